/*
 * gvo_b200.h — C ABI of the B200-native volume-enumeration core of the
 * arXiv 2107.01143 hardware-metric estimator ("gvo").
 *
 * The reference estimator is pure Python (pkg/src/gvo); it has no FFI.
 * SURVEY.md §8(b) places the thin native boundary under pkg/bindings.
 * Every entry point below replaces one Python seam of the reference and
 * cites it.  All structs are POD, all buffers are caller-owned; the
 * library never returns owned memory.  "d_" arguments are device
 * pointers (e.g. torch tensors' data_ptr()), "h_" arguments host pointers.
 *
 * Threading: one gvo_ctx per host thread; a context is used from one
 * caller thread at a time (reference SPEC.md:484-485).  Results never
 * depend on launch schedule.
 *
 * There is no CPU fallback and no backend dispatch: every entry point
 * runs sm_100a kernels or fails with a status code.
 */
#ifndef GVO_B200_H
#define GVO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GVO_ABI_VERSION 4

/* ---- status codes: map 1:1 onto the reference's exception classes ---- */
enum gvo_status {
  GVO_OK = 0,
  GVO_ERR_EXPR = 1,             /* gvo.expr.ExprError            expr.py:27   */
  GVO_ERR_ADDRESS_OVERFLOW = 2, /* gvo.expr.AddressOverflowError expr.py:37   */
  GVO_ERR_KERNEL = 3,           /* gvo.kernels.KernelError       kernels.py:34 */
  GVO_ERR_FOOTPRINT = 4,        /* gvo.footprint.FootprintError  footprint.py:30 */
  GVO_ERR_MACHINE = 5,          /* gvo.machine.MachineError      machine.py:22 */
  GVO_ERR_PERF = 6,             /* gvo.perf.PerfError            perf.py:24   */
  GVO_ERR_CAPACITY = 7,         /* engine scratch capacity exceeded (no reference analogue) */
  GVO_ERR_UNSUPPORTED = 8,      /* input outside the documented engine limits */
  GVO_ERR_INVALID = 15,         /* bad argument to the C ABI itself */
  GVO_ERR_CUDA = 16,
  GVO_ERR_NCCL = 17
};

/* ---- engine limits (documented in DESIGN.md §limits) ---- */
#define GVO_MAX_FIELDS 16
#define GVO_MAX_ACCESSES 1024      /* per template */
#define GVO_MAX_CODE 256           /* bytecode instructions per access */
#define GVO_MAX_BLOCK_SAMPLES 32   /* representative blocks per config */
#define GVO_MAX_UNIQUE_WAVES 16    /* => wave_samples <= 15 */

/* Machine descriptor; mirrors gvo.machine.MachineDescriptor
 * (reference machine.py:27-43) including the four Gompertz triples of
 * fit.py:22 in role order (l1, l2_load, l2_store, overmiss). */
typedef struct gvo_machine {
  int64_t sm_count;
  double clock_ghz;
  int64_t l1_capacity_bytes;
  int64_t l2_capacity_bytes;
  int64_t l1_line_bytes;
  int64_t sector_bytes;
  int64_t l1_banks;
  int64_t bank_width_bytes;
  double mem_bandwidth_gbps;
  double l2_bandwidth_gbps;
  int64_t max_threads_per_sm;
  int64_t max_blocks_per_sm;
  int64_t max_threads_per_block;
  double flop_per_byte_balance;
  double fit[4][3]; /* [role][a,b,c] */
} gvo_machine;

/* Postfix bytecode of one address-expression tree (reference expr.py:47-98).
 * Leaves push, binary ops pop two and push one. */
enum gvo_opcode {
  GVO_OP_CONST = 0,    /* arg: int64 constant            (IntConstant) */
  GVO_OP_COORD = 1,    /* arg: 0..5 tidx,tidy,tidz,bidx,bidy,bidz (CoordRef) */
  GVO_OP_BDIM = 2,     /* arg: 0..2 BX,BY,BZ             (BlockDimRef) */
  GVO_OP_BASE = 3,     /* arg: field index -> alignment  (BaseRef) */
  GVO_OP_ADD = 4,
  GVO_OP_SUB = 5,
  GVO_OP_MUL = 6,
  GVO_OP_FLOORDIV = 7, /* binary; right operand is a positive GVO_OP_CONST */
  GVO_OP_MOD = 8       /* binary floor modulo; right operand positive constant */
};

typedef struct gvo_insn {
  int32_t op;
  int32_t pad;
  int64_t arg;
} gvo_insn;

/* A kernel template: fields + accesses of a KernelDescriptor
 * (reference kernels.py:113-141) with BX/BY/BZ left symbolic, so one
 * template serves every block shape of a sweep (SPEC "DESIGN DECISIONS":
 * block dimensions bound at evaluation time).  Host pointers. */
typedef struct gvo_template {
  int32_t n_fields;
  int32_t n_accesses;
  const int64_t* field_base;     /* [n_fields] base substitution = alignment */
  const int32_t* access_field;   /* [n_accesses] field index */
  const int32_t* access_kind;    /* [n_accesses] 0 load, 1 store */
  const int64_t* access_mult;    /* [n_accesses] multiplicity >= 1 */
  const int32_t* access_code_off;/* [n_accesses] offset into code */
  const int32_t* access_code_len;/* [n_accesses] */
  const gvo_insn* code;          /* [n_code] */
  int32_t n_code;
  int32_t pad;
} gvo_template;

/* One candidate configuration (a KernelFamily.build(SweepConfig) result,
 * reference kernels.py:412-434, reduced to what the path consumes). */
typedef struct gvo_config {
  int32_t template_id;
  int32_t machine_id;
  int32_t block[3];          /* LaunchConfig.block_dim */
  int32_t fold_rank;         /* rank of the folding *string* for the sort key
                                of perf.py:131: "2y"=0 < "2z"=1 < "none"=2 */
  int64_t grid[3];           /* LaunchConfig.grid_dim, in blocks */
  int64_t work_per_thread;   /* LaunchConfig.work_per_thread */
  int64_t flops_per_lup;     /* KernelDescriptor.flops_per_lup */
} gvo_config;

/* Sampling knobs of evaluate_kernel (reference perf.py:70-89). */
typedef struct gvo_sampling {
  int32_t block_samples;            /* default 5 */
  int32_t wave_samples;             /* default 2 */
  int64_t blocks_per_wave_override; /* 0 = computed (footprint.py:66 'or') */
  int32_t phases;                   /* bitmask: 1 block stats (sample_block_stats),
                                       2 wave stats (sample_wave_stats),
                                       4 L1 cycles (l1_register_cycles);
                                       0 means all (evaluate_kernel) */
  int32_t pad;
} gvo_sampling;

/* ---- per-config integer numerators ("counts"), int64 layout ----
 * stride = gvo_counts_stride(F, S, W) with F fields (max over templates),
 * S = block_samples, W = wave_samples.  Offsets: */
#define GVO_C_STATUS 0        /* gvo_status */
#define GVO_C_ERR_PHASE 1     /* 0 block stats, 1 wave stats, 2 L1 cycles */
#define GVO_C_ERR_GROUP 2     /* group index inside the phase */
#define GVO_C_ERR_ACCESS 3    /* access index (kernel order) */
#define GVO_C_NSAMPLES 4      /* representative blocks actually picked */
#define GVO_C_NUWAVES 5       /* unique sampled waves (contiguous indices) */
#define GVO_C_NPAIRS 6        /* (prev, curr) pairs */
#define GVO_C_HASPRED 7       /* 1 if pairs have predecessors */
#define GVO_C_PERWAVE 8       /* blocks per wave */
#define GVO_C_NWAVES 9        /* waves in the grid */
#define GVO_C_L1BLOCK 10      /* linear index of the L1 block */
#define GVO_C_L1CYCLES 11     /* sum_a mult_a * warp cycles (integer) */
#define GVO_C_FIRSTWAVE 12    /* index of unique wave 0 */
#define GVO_C_FIRSTBLOCK 13   /* linear index of sample 0 (info) */
#define GVO_C_HDR 16
/* block part   [S][F][5]: load_unique_sectors, load_warp_requests,
 *                         load_unique_lines, store_unique_sectors,
 *                         store_warp_requests      (volumes.py:152-185)
 * wave part    [U][F][4]: |L_u|, |S_u|, |L_u u S_u|, |L_u n L_(u-1)|
 *                         (footprint.py:535-584, volumes.py:203-250)
 * wave lups    [U]      : blocks_in_wave * lups_per_block
 * with U = W + 1. */
static inline int64_t gvo_counts_stride(int32_t F, int32_t S, int32_t W) {
  return GVO_C_HDR + (int64_t)S * F * 5 + (int64_t)(W + 1) * F * 4 + (W + 1);
}

/* Effective counts stride of a call: S and W clamped to the engine limits
 * (S in [1, GVO_MAX_BLOCK_SAMPLES], W in [1, GVO_MAX_UNIQUE_WAVES-1]). */
int64_t gvo_counts_stride_eff(int32_t F, const gvo_sampling* sampling);

/* ---- per-config f64 record: the numeric columns of the 42-column
 * ranking record (reference report.py:162-255), in that order. ---- */
enum gvo_record_col {
  GVO_R_L1_CYCLES_PER_LUP = 0,
  GVO_R_L2L1_LOAD_COMP, GVO_R_L2L1_LOAD_RED, GVO_R_L2L1_LOAD_CAP, GVO_R_L2L1_LOAD_UP,
  GVO_R_L2L1_LOAD_DOWN, GVO_R_L2L1_LOAD_ALLOC, GVO_R_L2L1_LOAD_OVERSUB,
  GVO_R_L2L1_STORE_COMP, GVO_R_L2L1_STORE_RED, GVO_R_L2L1_STORE_CAP, GVO_R_L2L1_STORE_UP,
  GVO_R_L2L1_STORE_DOWN,
  GVO_R_DRAM_LOAD_COMP, GVO_R_DRAM_LOAD_RED, GVO_R_DRAM_LOAD_CAP, GVO_R_DRAM_LOAD_UP,
  GVO_R_DRAM_LOAD_DOWN, GVO_R_DRAM_LOAD_ALLOC, GVO_R_DRAM_LOAD_OVERSUB,
  GVO_R_DRAM_LOAD_UNIQUE, GVO_R_DRAM_LOAD_OVERLAP, GVO_R_DRAM_LOAD_OVERMISS,
  GVO_R_DRAM_LOAD_COVERAGE, /* NaN encodes None */
  GVO_R_DRAM_LOAD_REDL2,
  GVO_R_DRAM_STORE_COMP, GVO_R_DRAM_STORE_RED, GVO_R_DRAM_STORE_CAP, GVO_R_DRAM_STORE_UP,
  GVO_R_DRAM_STORE_DOWN, GVO_R_DRAM_STORE_UNIQUE,
  GVO_R_T_DRAM, GVO_R_T_L2, GVO_R_T_L1, GVO_R_T_FP,
  GVO_R_LIMITER, /* 0 dram, 1 l2, 2 l1, 3 fp (perf.py:21) */
  GVO_R_GLUPS,
  GVO_RECORD_LEN
};

typedef struct gvo_ctx gvo_ctx;

/* ---- context ---- */
int gvo_abi_version(void);
int gvo_open(int device, gvo_ctx** out);
void gvo_close(gvo_ctx* ctx);
const char* gvo_last_error(const gvo_ctx* ctx);

/* Upload kernel templates / machine descriptors; ids are positions.
 * Replaces the Python objects KernelDescriptor (kernels.py:113) and
 * MachineDescriptor (machine.py:27) on the device side. */
int gvo_set_templates(gvo_ctx* ctx, const gvo_template* h_tpls, int32_t n);
int gvo_set_machines(gvo_ctx* ctx, const gvo_machine* h_machines, int32_t n);

/* Batched configuration-space evaluation.  Replaces the per-config loop
 * of perf.rank_sweep (perf.py:115-130) → evaluate_kernel (perf.py:70) →
 * estimate_volumes (volumes.py:421) + l1_register_cycles (volumes.py:111)
 * + predict (perf.py:45).  F = max fields over the uploaded templates.
 * Fills counts [n][gvo_counts_stride(F,S,W)], stats [n][GVO_STATS_LEN(F)],
 * records [n][GVO_RECORD_LEN]; optionally field_down [n][4][F]
 * (per_field_down of l2l1 load/store, dram load/store) and
 * l1_access [n][l1_access_stride][3] (cycles, 2*sum metric, warps).
 * Returns GVO_OK when the launch sequence succeeded; per-config errors
 * are reported in counts[GVO_C_STATUS]. */
int gvo_eval_configs(gvo_ctx* ctx, const gvo_config* d_cfgs, int64_t n,
                     const gvo_sampling* sampling, int32_t F,
                     int64_t* d_counts, double* d_stats, double* d_records,
                     double* d_field_down, int64_t* d_l1_access,
                     int32_t l1_access_stride, void* stream);

/* Same with host buffers: copies in, evaluates, copies out, synchronises.
 * When every output buffer is page-locked (cudaHostAlloc / pinned) and the
 * call spans several batches, each batch's rows are copied to the host on a
 * second stream while the next batches compute (gvo_sweep_host* likewise). */
int gvo_eval_configs_host(gvo_ctx* ctx, const gvo_config* h_cfgs, int64_t n,
                          const gvo_sampling* sampling, int32_t F,
                          int64_t* h_counts, double* h_stats, double* h_records,
                          double* h_field_down, int64_t* h_l1_access,
                          int32_t l1_access_stride);

/* Ranking: order[i] = index of the i-th ranked config under the key
 * (-glups, block_dim, folding string, input index) of perf.py:131
 * (Python's sort is stable, hence the trailing input index). */
int gvo_rank(gvo_ctx* ctx, const double* d_records, const gvo_config* d_cfgs,
             int64_t n, int64_t* d_order, void* stream);

/* gvo_sweep_host plus the optional per-field down volumes and per-access
 * L1 outputs of gvo_eval_configs_host (either may be NULL): the one call
 * behind the drop-in rank_sweep (perf.py:98-132). */
int gvo_sweep_host_ex(gvo_ctx* ctx, const gvo_config* h_cfgs, int64_t n,
                      const gvo_sampling* sampling, int32_t F,
                      int64_t* h_counts, double* h_stats, double* h_records,
                      double* h_field_down, int64_t* h_l1_access, int32_t l1_access_stride,
                      int64_t* h_order);

/* Multi-GPU ranking of all-gathered shard records: d_rows
 * [n_rows][GVO_RECORD_LEN] as gathered rank-major, d_gidx[n_rows] the
 * global configuration index of each row (-1: all-gather padding, dropped),
 * d_cfgs [n_global] the whole space in global (input) order.  Rows are
 * scattered to global order (into d_records_global when non-NULL, else
 * library scratch) and ranked there, so ties break by the global input
 * index exactly as the reference's stable sort (perf.py:131) and padded
 * rows are never ranked.  Synchronises the stream (index validation). */
int gvo_rank_gathered(gvo_ctx* ctx, const double* d_rows, const int64_t* d_gidx, int64_t n_rows,
                      const gvo_config* d_cfgs, int64_t n_global, double* d_records_global,
                      int64_t* d_order, void* stream);

/* Build id of the loaded library: hash of the sources and compile flags
 * (profiles/ captures are tagged with it). */
const char* gvo_build_id(void);

/* Evaluate and rank host configurations in one call (one synchronisation):
 * the batch entry a sweep driver binds (perf.rank_sweep, perf.py:98-132).
 * h_order[i] = index of the i-th ranked config; other outputs as
 * gvo_eval_configs_host (h_stats may be NULL). */
int gvo_sweep_host(gvo_ctx* ctx, const gvo_config* h_cfgs, int64_t n,
                   const gvo_sampling* sampling, int32_t F,
                   int64_t* h_counts, double* h_stats, double* h_records,
                   int64_t* h_order);

/* ---- fine-grained parity entry points ---- */

/* One collaborative group given as runs of consecutive linear block
 * indices.  grid_iteration (footprint.py:441-471): per (field, kind)
 * unique granules and sum over access of mult * per-warp distinct.
 * out [F][2][2] = {unique, total} for kind load(0)/store(1). */
int gvo_group_footprint(gvo_ctx* ctx, int32_t template_id,
                        const int32_t block[3], const int64_t grid[3],
                        const int64_t* h_run_start, const int64_t* h_run_count,
                        int32_t n_runs, int64_t granularity, int64_t* h_out);

/* Ordered groups (waves), each one run.  For each group g and field f:
 * |L_g|, |S_g|, |L_g u S_g|, |L_g n L_(g-1)| at the given granularity
 * (wave_footprint / wave_overlap, footprint.py:535-584).  out [G][F][4]. */
int gvo_group_sets(gvo_ctx* ctx, int32_t template_id, const int32_t block[3],
                   const int64_t grid[3], const int64_t* h_run_start,
                   const int64_t* h_run_count, int32_t n_groups,
                   int64_t granularity, int64_t* h_out);

/* L1 bank-conflict cycles of one block (l1_register_cycles,
 * volumes.py:57-134).  out [A][3] = {warp cycles, 2*sum metric, warps}. */
int gvo_l1_cycles(gvo_ctx* ctx, int32_t template_id, const int32_t block[3],
                  const int64_t grid[3], int64_t block_linear,
                  int64_t bank_width_bytes, int64_t n_banks, int64_t* h_out);

/* Bulk evaluation of one access expression at explicit coordinates
 * (expr.evaluate_bulk, expr.py:281-304; int64 semantics after the
 * host-side value_bounds guard).  coords [n][6] → out [n]. */
int gvo_eval_addresses(gvo_ctx* ctx, int32_t template_id, int32_t access,
                       const int32_t block[3], const int64_t* h_coords,
                       int64_t n, int64_t* h_out);

/* ---- float statistics ("stats"), f64 layout per config, F fields ----
 * [0,5F)  BlockStats  load_comp, load_up, load_alloc, store_unique,
 *                     store_up            (volumes.py:141-149), [5][F]
 * [5F,8F) WaveStats   load_unique, load_overlap, store_unique [3][F]
 * 8F+0 prev_unique_total, 8F+1 alloc_total, 8F+2 wave_lups,
 * 8F+3 has_predecessor (0/1)               (volumes.py:188-199)
 * 8F+4 cycles_per_lup (L1CycleEstimate, volumes.py:47-54)
 * 8F+5 lups_per_block                      (kernels.py:108-110)
 * [8F+6, 10F+6) injected L2->L1 per_field_down (load, store) [2][F] and
 * 10F+6 flag: 1 = use them as the DRAM level's "up" instead of the values
 * assembled from the block stats (dram_to_l2_volume's l2l1 arguments,
 * volumes.py:354-363) */
#define GVO_STATS_LEN(F) (10 * (F) + 7)

/* Float assembly + prediction from (possibly injected) float statistics:
 * estimate_volumes with block_stats/wave_stats given (volumes.py:421-445),
 * then predict (perf.py:45-67).  machine_id/flops per config. */
int gvo_assemble_host(gvo_ctx* ctx, const double* h_stats, int32_t F,
                      const int32_t* h_machine_id, const int64_t* h_flops,
                      int64_t n, double* h_records, double* h_field_down);

/* Four-limiter prediction from given volumes (perf.predict, perf.py:45-67):
 * out [n][6] = t_dram, t_l2, t_l1, t_fp, limiter code, glups. */
int gvo_predict_host(gvo_ctx* ctx, const int32_t* h_machine_id, const double* h_dram_down,
                     const double* h_l2_down, const double* h_cycles_per_lup,
                     const int64_t* h_flops, int64_t n, double* h_out);

/* ---- ranking CSV (host) ----
 * Rows of render_ranking_csv (reference report.py:242-255, columns of
 * RANKING_CSV_COLUMNS report.py:162-205): for r in 0..n-1, config
 * i = order[r] (i = r when order is NULL): the caller's text prefix i
 * (prefixes[prefix_off[i] .. prefix_off[i+1]), i.e. "configKey,blockX,
 * blockY,blockZ,folding"), then the 37 record columns, each formatted as
 * Python format(v, ".10g") (NaN coverage = None -> empty cell), the
 * limiter by name, '\n' per row.  Pure host code, n_threads workers
 * (<= 0: all cores).  *len_out = bytes needed; GVO_ERR_CAPACITY when out is
 * NULL or cap is smaller (nothing written). */
int gvo_format_ranking_csv(const double* h_records, int64_t n, const int64_t* h_order,
                           const char* prefixes, const int64_t* prefix_off, int32_t n_threads,
                           char* out, int64_t cap, int64_t* len_out);

/* ---- instrumentation ---- */
/* Enable CUDA-event timing around every pipeline kernel (on the stream the
 * kernel is launched on). */
int gvo_set_timing(gvo_ctx* ctx, int enable);
/* Accumulated ms / launch counts per kernel: [0] setup, [1] warp stats,
 * [2] interval-union sets, [3] assembly, [4] rank; 8 slots. */
int gvo_kernel_times(gvo_ctx* ctx, double* ms_out, int64_t* count_out, int reset);
/* Profiling: enable per-unit statistics of the interval-union engine and
 * fetch those of the last batch: [item][runs, intervals, in-smem, cycles,
 * key bits, SM id]; items ordered (config, field, unit). */
int gvo_debug_units(gvo_ctx* ctx, int enable, int64_t* h_out, int64_t cap, int64_t* n_items);
/* Cross-configuration sharing of identical set problems (every
 * gvo_eval_configs* call; GVO_DEDUP=0 in the environment of gvo_open turns it
 * off).  enable_counting != 0 makes later calls count, and this returns the
 * last call's figures: units eligible for sharing and units that copied an
 * identical unit's counts instead of computing them.  Returns 1 when sharing
 * is on, 0 when off.  (No reference counterpart: the reference evaluates every
 * configuration from scratch, perf.py:115-130; results are identical.) */
int gvo_dedup_stats(gvo_ctx* ctx, int enable_counting, int64_t* shareable_units, int64_t* followers);
/* Turn the sharing on (1) or off (0) for later calls on this context: both
 * the set-problem sharing above and the plan sharing of k_setup (leader plans
 * of configurations equal up to field-base translation and machine
 * capacities; GVO_PLAN_SHARE=0 turns that one off alone). */
int gvo_set_dedup(gvo_ctx* ctx, int enable);
/* Configurations per device batch for later calls on this context (plan ->
 * sharing -> set kernel -> float assembly run batch by batch; default 65536,
 * or GVO_BATCH at gvo_open).  Results do not depend on it. */
int gvo_set_batch(gvo_ctx* ctx, int64_t configs_per_batch);
/* Measured INT32 issue rate of the device (ops/s), the integer roofline. */
int gvo_int_peak(gvo_ctx* ctx, double* ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* GVO_B200_H */
