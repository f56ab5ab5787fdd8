// gvo_kernels.h — host-side launchers of the device pipeline (internal).
#pragma once
#include <cuda_runtime.h>
#include "gvo_common.cuh"
#include "gvo_warp.cuh"

namespace gvo {

// The set kernel is built in two residencies (k_sets.cu, k_sets1.cu):
// sets2 = 2 CTAs x 512 threads per SM (64 registers, 110 KB shared memory
// each: latency hiding for small batches), sets1 = 1 CTA per SM (128
// registers, 222 KB: no spills, 2x wider bitmap ranges and sort buffers for
// throughput-bound batches).  kMaxSetsCtasPerSm sizes the per-CTA scratch.
#ifdef GVO_SETS2_CTAS
constexpr int kMaxSetsCtasPerSm = GVO_SETS2_CTAS;
#else
constexpr int kMaxSetsCtasPerSm = 2;
#endif

// plan sharing across configurations (k_setup.cu): a per-call key table
// and a cache of leader plans
struct PlanEntry {
  unsigned long long tag;  // 0 empty, else key hash | 1
  int ready;
  int slot;                // cache slot, -1 = cache full
  uint64_t key[6];
};
struct PlanShare {
  PlanEntry* table = nullptr;
  int64_t mask = 0;
  int64_t* cache = nullptr;      // cap slots of plan_slot_words(max_acc) int64
  int64_t cap = 0;
  unsigned long long* n_used = nullptr;
  int64_t* src = nullptr;        // per batch config: slot, -2 - slot (leader) or -1
  bool defer_rows = false;       // followers' coefficient rows / class tables by launch_plan_rows
  const uint8_t* need = nullptr; // per batch config: rows needed (a unit computes); null = all
};
void launch_plan_rows(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs, int64_t n,
                      const gvo_sampling& smp, int64_t* d_coefs, Geo* d_geos, int64_t* d_ctabs, const PlanShare& PS,
                      cudaStream_t st);
__host__ __device__ int64_t plan_slot_words(int64_t max_acc);
void launch_setup(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs,
                  int64_t n, const gvo_sampling& smp, int64_t* d_coefs, Geo* d_geos, int64_t* d_ctabs,
                  cudaStream_t st, const int32_t* d_mclass = nullptr, const PlanShare* share = nullptr);
void launch_classes(const TplView& T, const gvo_config* d_cfgs, int64_t n, const int64_t* d_coefs,
                    int64_t* d_ctabs, cudaStream_t st);

void launch_warp(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs, const Geo* d_geos, const int64_t* d_coefs,
                 int64_t n_items, int S_req, int64_t sector, int64_t bank_width, int64_t n_banks,
                 int mode, const int64_t* d_block_list, int64_t* d_counts, int64_t counts_stride,
                 int F_stride, int64_t* d_l1_access, int32_t l1_stride, unsigned long long* d_out,
                 int max_acc, int n_sm, cudaStream_t st);

struct SetsLaunch {
  TplView T;
  const gvo_machine* machines;
  const gvo_config* cfgs;
  const Geo* geos;
  const int64_t* coefs;
  const int64_t* ctabs;
  int64_t n_items;
  int S_req;
  int F_stride;
  int mode;
  int64_t granularity;
  const int64_t* run_start;
  const int64_t* run_count;
  int n_custom_runs;
  int64_t* counts;
  int64_t counts_stride;
  uint8_t* slab;
  int64_t slab_bytes;
  int64_t run_cap;
  int64_t elem_cap;
  int* status_out;
  int n_ctas;
  int64_t* unit_stats = nullptr;
  unsigned long long* work = nullptr;
  WarpArgs warp{};
  int64_t n_warp_items = 0;
  SplitState* split = nullptr;
  int64_t sm_cap = 0;
  int32_t seg_off = 0;
  int32_t pat_off = 0;
  int32_t wave_field_major = 1;
  int32_t epoch = 1;  // launch number, unique across both residencies (queue readiness tag)
  const int64_t* lead = nullptr;  // k_dedup: >= 0 = unit copied from another config's (skip)
  // work lists (k_dedup.cu k_worklist), mode 0; null = every item
  const int32_t* wl_wave = nullptr;
  const int32_t* wl_blk = nullptr;
  const int32_t* wl_warp = nullptr;
  const unsigned long long* wl_cnt = nullptr;
  // residency chosen on the device: the launch runs only if *run_if == run_if_val
  const int* run_if = nullptr;
  int run_if_val = 0;
  int handoff = 0;  // micro-tier handoffs of large block units to the CTA (large batches)
};
// *d_flag = 0 iff every config of the batch has a template with >= 3 fields (else 1)
void launch_batch_wide(const TplView& T, const gvo_config* d_cfgs, int64_t n, int* d_flag, cudaStream_t st);
namespace sets1 {
int64_t sets_ebuf_bytes();
void launch_sets(const SetsLaunch& L, cudaStream_t st);
}
namespace sets2 {
int64_t sets_ebuf_bytes();
void launch_sets(const SetsLaunch& L, cudaStream_t st);
}
int64_t sets_slab_bytes(int64_t run_cap, int64_t elem_cap);
int64_t split_slot_bytes(int64_t run_cap);

// cross-configuration sharing of identical set problems (k_dedup.cu)
struct DedupEntry {
  unsigned long long tag;  // 0 empty, else key hash | 1
  int64_t leader;          // global config index * 32 + field
  int ready;
  int pad;
  uint64_t key[9];
};
int64_t dedup_units(int64_t n, int F, int S);
void launch_dedup(const TplView& T, const gvo_machine* d_machines, const int32_t* d_mclass, const gvo_config* d_cfgs,
                  const Geo* d_geos, int64_t n, int F, int S, int64_t b0, DedupEntry* table, int64_t mask,
                  int64_t* d_lead, unsigned long long* d_stats, cudaStream_t st);
// work lists of the set kernel for one batch: wave units (in the kernel's
// wave order), block units and warp items that compute; d_list holds
// dedup_units(n, F, S) entries, d_cnt three counters
void launch_worklists(const TplView& T, const gvo_config* d_cfgs, const Geo* d_geos, int64_t n, int F, int S,
                      const int64_t* d_lead, int wave_field_major, int32_t* d_list, unsigned long long* d_cnt,
                      const int32_t** wl_wave, const int32_t** wl_blk, const int32_t** wl_warp, uint8_t* d_need,
                      cudaStream_t st);
void launch_dedup_copy(const gvo_config* d_cfgs, const Geo* d_geos, const TplView& T, int64_t* d_counts_all,
                       int64_t counts_stride, int64_t n, int F, int S, int64_t b0, const int64_t* d_lead,
                       int64_t* d_l1_access_all, int32_t l1_stride, cudaStream_t st);

// float assembly + prediction (k_assemble.cu)
void launch_finish(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs,
                   const Geo* d_geos, int64_t n, int S_req, int W_req, int F, int64_t* d_counts,
                   int64_t counts_stride, double* d_stats, double* d_records, double* d_field_down,
                   cudaStream_t st);
void launch_assemble_stats(const gvo_machine* d_machines, const int32_t* d_mid, const int64_t* d_flops,
                           int64_t n, int F, const double* d_stats, double* d_records,
                           double* d_field_down, cudaStream_t st);

void launch_predict(const gvo_machine* d_machines, const int32_t* d_mid, const double* dd, const double* ld,
                    const double* cyc, const int64_t* fl, int64_t n, double* out, cudaStream_t st);

int launch_int_peak(int n_sm, cudaStream_t st, double* ops_per_s);

// ranking (k_rank.cu)
int64_t rank_scratch_bytes(int64_t n);
void launch_rank(const double* d_records, const gvo_config* d_cfgs, int64_t n, int64_t* d_order,
                 void* d_scratch, cudaStream_t st);
void launch_scatter_gathered(const double* d_rows, const int64_t* d_gidx, int64_t n_rows, int64_t n_global,
                             double* d_out, unsigned int* d_bad, cudaStream_t st);

}  // namespace gvo
