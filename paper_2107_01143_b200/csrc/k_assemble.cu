// k_assemble.cu — float statistics, volume assembly and the four-limiter
// prediction, one thread per configuration.
//
// Bit-exactness: every expression follows the reference's operation order
// (Python evaluates left to right; sum() starts from int 0; int/int is a
// correctly rounded true division, identical to an IEEE double division
// while operands are < 2^53).  The file is compiled with --fmad=false so no
// multiply-add is contracted.
//   stats     : volumes.sample_block_stats / sample_wave_stats
//               (volumes.py:152-250), l1_register_cycles' per-LUP
//               normalisation (volumes.py:131-134)
//   assembly  : _assemble / _totals / l2_to_l1_volume / dram_to_l2_volume
//               (volumes.py:294-418), fit.evaluate (fit.py:51-57)
//   predict   : perf.predict / binding_limiter (perf.py:38-67)
#include "gvo_kernels.h"
#include "gvo_exp.cuh"

namespace gvo {

// Python's min(a, b) / max(a, b): the first argument wins ties.
__device__ __forceinline__ double pmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double pmax(double a, double b) { return b > a ? b : a; }

// fit.evaluate (fit.py:51-57)
__device__ inline double gompertz(const double* p, double x) {
  const double inner = (-p[2]) * x;
  if (inner > 700.0) return 0.0;
  const double value = p[0] * glibc_exp((-p[1]) * glibc_exp(inner));
  return pmin(1.0, pmax(0.0, value));
}

// perf.predict: the four limiter times, argmax with ties in the order
// (dram, l2, l1, fp), glups = 1e-9 / t_max (perf.py:38-67)
__device__ inline void predict_one(const gvo_machine& m, double dram_down, double l2_down,
                                   double cycles_per_lup, int64_t flops, double t[4], int* lim,
                                   double* glups) {
  const double mem_bps = m.mem_bandwidth_gbps * 1e9;
  const double l2_bps = m.l2_bandwidth_gbps * 1e9;
  const double clock_hz = m.clock_ghz * 1e9;
  t[0] = dram_down / mem_bps;
  t[1] = l2_down / l2_bps;
  t[2] = cycles_per_lup / ((double)m.sm_count * clock_hz);
  t[3] = (double)flops / (m.flop_per_byte_balance * mem_bps);
  int k = 0;
  for (int j = 1; j < 4; ++j)
    if (t[j] > t[k]) k = j;
  *lim = k;
  *glups = 1e-9 / t[k];
}

__global__ void k_predict(const gvo_machine* machines, const int32_t* mid, const double* dd,
                          const double* ld, const double* cyc, const int64_t* fl, int64_t n, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t[4], g;
  int lim;
  predict_one(machines[mid[i]], dd[i], ld[i], cyc[i], fl[i], t, &lim, &g);
  for (int k = 0; k < 4; ++k) out[i * 6 + k] = t[k];
  out[i * 6 + 4] = lim;
  out[i * 6 + 5] = g;
}

void launch_predict(const gvo_machine* d_machines, const int32_t* d_mid, const double* dd, const double* ld,
                    const double* cyc, const int64_t* fl, int64_t n, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_predict<<<(unsigned)((n + 63) / 64), 64, 0, st>>>(d_machines, d_mid, dd, ld, cyc, fl, n, out);
}

// Python's built-in sum() over floats (CPython >= 3.12, bltinmodule.c
// builtin_sum_impl): the int start 0 plus the first item is exact (0 + x),
// every further item is added with Neumaier's compensation, and the
// compensation is added at the end when it is nonzero and finite.  The
// reference sums per-field volumes with sum() (volumes.py:307-309, 332,
// 386, 401-404, 416); plain left-to-right addition differs in the last bit
// whenever the sum is inexact.
struct PySum {
  double s = 0.0, c = 0.0;
  bool any = false;
  __device__ __forceinline__ void add(double x) {
    if (!any) { s = 0.0 + x; any = true; return; }
    const double t = s + x;
    if (fabs(s) >= fabs(x)) c += (s - t) + x;
    else c += (x - t) + s;
    s = t;
  }
  __device__ __forceinline__ double value() const { return (c != 0.0 && isfinite(c)) ? s + c : s; }
};

// _assemble + _totals for F fields; writes (up, comp, red, cap, down)
__device__ inline void assemble_level(int F, const double* comp_f, const double* up_f,
                                      const double* basis_f, double ratio, double* down_f,
                                      double out[5]) {
  PySum Sc, Sr, Sk;
  for (int f = 0; f < F; ++f) {
    const double up = up_f[f];
    const double c = pmin(comp_f[f], up);
    const double r = pmax(0.0, up - c);
    const double k = pmin(pmax(ratio * basis_f[f], 0.0), r);
    down_f[f] = c + k;
    Sc.add(c);
    Sr.add(r);
    Sk.add(k);
  }
  const double sc = Sc.value(), sr = Sr.value();
  const double k = pmin(Sk.value(), sr);
  out[0] = sc + sr;
  out[1] = sc;
  out[2] = sr;
  out[3] = k;
  out[4] = sc + k;
}

// One configuration: stats (GVO_STATS_LEN(F) doubles) -> record, field_down.
__device__ void assemble_one(const gvo_machine& m, int F, const double* st, int64_t flops,
                             double* rec, double* fd /* [4][F] or null */) {
  const double* load_comp = st;
  const double* load_up = st + F;
  const double* load_alloc = st + 2 * F;
  const double* store_unique_b = st + 3 * F;
  const double* store_up_b = st + 4 * F;
  const double* w_load_unique = st + 5 * F;
  const double* w_load_overlap = st + 6 * F;
  const double* w_store_unique = st + 7 * F;
  const double prev_total = st[8 * F + 0];
  const double alloc_total = st[8 * F + 1];
  const double wave_lups = st[8 * F + 2];
  const bool has_pred = st[8 * F + 3] != 0.0;
  const double cycles_per_lup = st[8 * F + 4];
  const double lups_per_block = st[8 * F + 5];
  const bool inject_up = st[10 * F + 6] != 0.0;

  double basis[kMaxFields], d_l2l1_load[kMaxFields], d_l2l1_store[kMaxFields];
  double d_dram_load[kMaxFields], d_dram_store[kMaxFields];
  double tmp_a[kMaxFields], tmp_b[kMaxFields];
  double lv[5], sv[5], dl[5], ds[5];

  // ---- L2 -> L1 (volumes.py:313-351)
  PySum alloc_sum;
  for (int f = 0; f < F; ++f) alloc_sum.add(load_alloc[f]);
  const double alloc = alloc_sum.value() * lups_per_block;
  const double oversub1 = alloc / (double)m.l1_capacity_bytes;
  const double ratio1 = gompertz(m.fit[0], oversub1);
  for (int f = 0; f < F; ++f) basis[f] = pmax(0.0, load_up[f] - load_comp[f]);
  assemble_level(F, load_comp, load_up, basis, ratio1, d_l2l1_load, lv);
  for (int f = 0; f < F; ++f) basis[f] = pmax(0.0, store_up_b[f] - store_unique_b[f]);
  assemble_level(F, store_unique_b, store_up_b, basis, 1.0, d_l2l1_store, sv);
  if (inject_up)
    for (int f = 0; f < F; ++f) {
      d_l2l1_load[f] = st[8 * F + 6 + f];
      d_l2l1_store[f] = st[9 * F + 6 + f];
    }

  // ---- DRAM -> L2 (volumes.py:354-418)
  const double oversub2 = alloc_total / (double)m.l2_capacity_bytes;
  double* unique = tmp_a;
  double* overlap = tmp_b;
  for (int f = 0; f < F; ++f) {
    unique[f] = w_load_unique[f] / wave_lups;
    overlap[f] = w_load_overlap[f] / wave_lups;
  }
  bool has_cov = false;
  double coverage = 0.0, om_ratio = 0.0;
  if (has_pred && prev_total > 0.0) {
    PySum su, so;
    for (int f = 0; f < F; ++f) su.add(w_load_unique[f]);
    for (int f = 0; f < F; ++f) so.add(w_load_overlap[f]);
    const double net_new = su.value() - so.value();
    coverage = ((double)m.l2_capacity_bytes - net_new) / prev_total;
    has_cov = true;
    om_ratio = gompertz(m.fit[3], -coverage);
  } else {
    for (int f = 0; f < F; ++f) overlap[f] = 0.0;
  }
  double comp_raw[kMaxFields], red_basis[kMaxFields];
  PySum su, so, sb;
  for (int f = 0; f < F; ++f) {
    comp_raw[f] = (unique[f] - overlap[f]) + om_ratio * overlap[f];
    red_basis[f] = pmax(0.0, d_l2l1_load[f] - unique[f]);
  }
  const double ratio2 = gompertz(m.fit[1], oversub2);
  assemble_level(F, comp_raw, d_l2l1_load, red_basis, ratio2, d_dram_load, dl);
  for (int f = 0; f < F; ++f) su.add(unique[f]);
  for (int f = 0; f < F; ++f) so.add(overlap[f]);
  for (int f = 0; f < F; ++f) sb.add(red_basis[f]);
  const double wave_unique = su.value(), v_overlap = so.value(), overmiss = om_ratio * so.value(),
               v_red_l2 = sb.value();

  double* s_unique = tmp_a;  // unique/overlap no longer needed
  for (int f = 0; f < F; ++f) s_unique[f] = w_store_unique[f] / wave_lups;
  for (int f = 0; f < F; ++f) basis[f] = pmax(0.0, d_l2l1_store[f] - s_unique[f]);
  const double ratio3 = gompertz(m.fit[2], oversub2);
  assemble_level(F, s_unique, d_l2l1_store, basis, ratio3, d_dram_store, ds);
  PySum sw;
  for (int f = 0; f < F; ++f) sw.add(s_unique[f]);
  const double s_wave_unique = sw.value();

  // ---- predict (perf.py:45-67)
  double t[4];
  int lim;
  double glups;
  predict_one(m, dl[4] + ds[4], lv[4] + sv[4], cycles_per_lup, flops, t, &lim, &glups);

  double* r = rec;
  r[GVO_R_L1_CYCLES_PER_LUP] = cycles_per_lup;
  r[GVO_R_L2L1_LOAD_COMP] = lv[1];
  r[GVO_R_L2L1_LOAD_RED] = lv[2];
  r[GVO_R_L2L1_LOAD_CAP] = lv[3];
  r[GVO_R_L2L1_LOAD_UP] = lv[0];
  r[GVO_R_L2L1_LOAD_DOWN] = lv[4];
  r[GVO_R_L2L1_LOAD_ALLOC] = alloc;
  r[GVO_R_L2L1_LOAD_OVERSUB] = oversub1;
  r[GVO_R_L2L1_STORE_COMP] = sv[1];
  r[GVO_R_L2L1_STORE_RED] = sv[2];
  r[GVO_R_L2L1_STORE_CAP] = sv[3];
  r[GVO_R_L2L1_STORE_UP] = sv[0];
  r[GVO_R_L2L1_STORE_DOWN] = sv[4];
  r[GVO_R_DRAM_LOAD_COMP] = dl[1];
  r[GVO_R_DRAM_LOAD_RED] = dl[2];
  r[GVO_R_DRAM_LOAD_CAP] = dl[3];
  r[GVO_R_DRAM_LOAD_UP] = dl[0];
  r[GVO_R_DRAM_LOAD_DOWN] = dl[4];
  r[GVO_R_DRAM_LOAD_ALLOC] = alloc_total;
  r[GVO_R_DRAM_LOAD_OVERSUB] = oversub2;
  r[GVO_R_DRAM_LOAD_UNIQUE] = wave_unique;
  r[GVO_R_DRAM_LOAD_OVERLAP] = v_overlap;
  r[GVO_R_DRAM_LOAD_OVERMISS] = overmiss;
  r[GVO_R_DRAM_LOAD_COVERAGE] = has_cov ? coverage : __longlong_as_double(0x7ff8000000000000ll);
  r[GVO_R_DRAM_LOAD_REDL2] = v_red_l2;
  r[GVO_R_DRAM_STORE_COMP] = ds[1];
  r[GVO_R_DRAM_STORE_RED] = ds[2];
  r[GVO_R_DRAM_STORE_CAP] = ds[3];
  r[GVO_R_DRAM_STORE_UP] = ds[0];
  r[GVO_R_DRAM_STORE_DOWN] = ds[4];
  r[GVO_R_DRAM_STORE_UNIQUE] = s_wave_unique;
  r[GVO_R_T_DRAM] = t[0];
  r[GVO_R_T_L2] = t[1];
  r[GVO_R_T_L1] = t[2];
  r[GVO_R_T_FP] = t[3];
  r[GVO_R_LIMITER] = (double)lim;
  r[GVO_R_GLUPS] = glups;
  if (fd) {
    for (int f = 0; f < F; ++f) {
      fd[0 * F + f] = d_l2l1_load[f];
      fd[1 * F + f] = d_l2l1_store[f];
      fd[2 * F + f] = d_dram_load[f];
      fd[3 * F + f] = d_dram_store[f];
    }
  }
}

// counts -> header, stats, record
__device__ void finish_one(const TplView& T, const gvo_machine* machines, const gvo_config& cfg, const Geo& G,
                           int64_t c, int S_req, int W_req, int F, int64_t* row, double* stats, double* records,
                           double* field_down) {
  const gvo_machine m = machines[cfg.machine_id];
  const int64_t sets_status = row[GVO_C_STATUS];
  int status = G.status != GVO_OK ? G.status : (int)sets_status;
  row[GVO_C_STATUS] = status;
  row[GVO_C_ERR_PHASE] = G.err_phase;
  row[GVO_C_ERR_GROUP] = G.err_group;
  row[GVO_C_ERR_ACCESS] = G.err_access;
  row[GVO_C_NSAMPLES] = G.n_samples;
  row[GVO_C_NUWAVES] = G.n_uw;
  row[GVO_C_NPAIRS] = G.n_pairs;
  row[GVO_C_HASPRED] = G.has_pred;
  row[GVO_C_PERWAVE] = G.per_wave;
  row[GVO_C_NWAVES] = G.n_waves;
  row[GVO_C_FIRSTWAVE] = G.first_wave;
  row[GVO_C_FIRSTBLOCK] = G.n_samples ? G.sample_lin[0] : -1;
  int64_t* blk = row + GVO_C_HDR;
  int64_t* wv = blk + (int64_t)S_req * F * 5;
  int64_t* wl = wv + (int64_t)(W_req + 1) * F * 4;
  for (int u = 0; u < G.n_uw && u <= W_req; ++u) wl[u] = G.uw_count[u] * G.lups_per_block;
  double* rec = records + c * GVO_RECORD_LEN;
  const bool full = G.phases == 7 && status == GVO_OK;
  const bool ph0 = phase_ok(G, 0) && sets_status == GVO_OK;
  const bool ph1 = phase_ok(G, 1) && sets_status == GVO_OK;
  const bool ph2 = phase_ok(G, 2);
  const int Ft = T.n_fields[cfg.template_id];
  double st[10 * kMaxFields + 7];
  const double sector = (double)m.sector_bytes;
  const double lups = (double)G.lups_per_block;
  // ---- BlockStats (volumes.py:152-185)
  for (int k = 0; k < 10 * Ft + 7; ++k) st[k] = 0.0;
  // resolve deduplicated samples (unique counts copied from the
  // translate-equivalent sample; warp counts were computed per sample)
  for (int s = 0; ph0 && s < G.n_samples; ++s)
    for (int f = 0; f < Ft; ++f) {
      const int d = G.dup_of[f][s];
      if (d < 0) continue;
      int64_t* b = blk + ((int64_t)s * F + f) * 5;
      const int64_t* o = blk + ((int64_t)d * F + f) * 5;
      for (int k = 0; k < 5; ++k) b[k] = o[k];
    }
  for (int s = 0; ph0 && s < G.n_samples; ++s)
    for (int f = 0; f < Ft; ++f) {
      const int64_t* b = blk + ((int64_t)s * F + f) * 5;
      st[0 * Ft + f] = st[0 * Ft + f] + (double)(b[0] * m.sector_bytes) / lups;
      st[1 * Ft + f] = st[1 * Ft + f] + (double)(b[1] * m.sector_bytes) / lups;
      st[2 * Ft + f] = st[2 * Ft + f] + (double)(b[2] * m.l1_line_bytes) / lups;
      st[3 * Ft + f] = st[3 * Ft + f] + (double)(b[3] * m.sector_bytes) / lups;
      st[4 * Ft + f] = st[4 * Ft + f] + (double)(b[4] * m.sector_bytes) / lups;
    }
  const double ns = (double)G.n_samples;
  if (ph0)
    for (int k = 0; k < 5 * Ft; ++k) st[k] = st[k] / ns;
  // ---- WaveStats (volumes.py:203-250)
  double lu[kMaxFields], lo[kMaxFields], su[kMaxFields];
  for (int f = 0; f < Ft; ++f) lu[f] = lo[f] = su[f] = 0.0;
  double prev_total = 0.0, alloc_total = 0.0, wave_lups = 0.0;
  for (int p = 0; ph1 && p < G.n_pairs; ++p) {
    const int cu = G.has_pred ? p + 1 : 0;
    const int64_t* cw = wv + (int64_t)cu * F * 4;
    int64_t alloc = 0;
    for (int f = 0; f < Ft; ++f) {
      lu[f] = lu[f] + (double)cw[f * 4 + 0] * sector;
      su[f] = su[f] + (double)cw[f * 4 + 1] * sector;
      alloc += cw[f * 4 + 2];
    }
    alloc_total = alloc_total + (double)alloc * sector;
    wave_lups = wave_lups + (double)wl[cu];
    if (G.has_pred) {
      const int64_t* pw = wv + (int64_t)p * F * 4;
      int64_t ptot = 0;
      for (int f = 0; f < Ft; ++f) ptot += pw[f * 4 + 0];
      prev_total = prev_total + (double)ptot * sector;
      for (int f = 0; f < Ft; ++f) lo[f] = lo[f] + (double)cw[f * 4 + 3] * sector;
    }
  }
  if (ph1) {
    const double np = (double)G.n_pairs;
    for (int f = 0; f < Ft; ++f) {
      st[5 * Ft + f] = lu[f] / np;
      st[6 * Ft + f] = lo[f] / np;
      st[7 * Ft + f] = su[f] / np;
    }
    st[8 * Ft + 0] = prev_total / np;
    st[8 * Ft + 1] = alloc_total / np;
    st[8 * Ft + 2] = wave_lups / np;
    st[8 * Ft + 3] = G.has_pred ? 1.0 : 0.0;
  }
  if (ph2) st[8 * Ft + 4] = (double)row[GVO_C_L1CYCLES] / lups;
  st[8 * Ft + 5] = lups;
  if (stats) {
    // stored with the uniform stride F (fields beyond the template's are 0)
    double* o = stats + c * GVO_STATS_LEN(F);
    for (int k = 0; k < GVO_STATS_LEN(F); ++k) o[k] = 0.0;
    for (int blk5 = 0; blk5 < 8; ++blk5)
      for (int f = 0; f < Ft; ++f) o[blk5 * F + f] = st[blk5 * Ft + f];
    for (int k = 0; k < 6; ++k) o[8 * F + k] = st[8 * Ft + k];
  }
  if (!full) {
    for (int k = 0; k < GVO_RECORD_LEN; ++k) rec[k] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double fdl[4 * kMaxFields];
  assemble_one(m, Ft, st, cfg.flops_per_lup, rec, field_down ? fdl : nullptr);
  if (field_down) {
    double* o = field_down + c * 4 * F;
    for (int k = 0; k < 4 * F; ++k) o[k] = 0.0;
    for (int l = 0; l < 4; ++l)
      for (int f = 0; f < Ft; ++f) o[l * F + f] = fdl[l * Ft + f];
  }
}

// warp per config: stage the counts row and the plan in shared memory
// (coalesced), lane 0 runs the sequential float code from shared memory,
// the warp writes the resolved row back
constexpr int kFinishWarps = 4;
__global__ void __launch_bounds__(32 * kFinishWarps) k_finish(TplView T, const gvo_machine* machines,
                                                               const gvo_config* cfgs, const Geo* geos, int64_t n,
                                                               int S_req, int W_req, int F, int64_t* counts,
                                                               int64_t stride, double* stats, double* records,
                                                               double* field_down) {
  extern __shared__ int64_t fsh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kFinishWarps + warp;
  if (c >= n) return;
  const int64_t geo_words = (sizeof(Geo) + 7) / 8;
  int64_t* srow = fsh + warp * (stride + geo_words);
  Geo* sG = reinterpret_cast<Geo*>(srow + stride);
  int64_t* grow = counts + c * stride;
  for (int64_t i = lane; i < stride; i += 32) srow[i] = grow[i];
  const int64_t* gg = reinterpret_cast<const int64_t*>(geos + c);
  for (int64_t i = lane; i < (int64_t)(sizeof(Geo) / 8); i += 32) reinterpret_cast<int64_t*>(sG)[i] = gg[i];
  __syncwarp();
  if (lane == 0) {
    const gvo_config cfg = cfgs[c];
    finish_one(T, machines, cfg, *sG, c, S_req, W_req, F, srow, stats, records, field_down);
  }
  __syncwarp();
  for (int64_t i = lane; i < stride; i += 32) grow[i] = srow[i];
}

// thread per config (GVO_FINISH_THREAD, default): the float code is serial
// per configuration; the warp-per-config form keeps 31 of 32 lanes idle
// while lane 0 runs it — here every lane runs one configuration, reading its
// counts row and plan straight from global memory
__global__ void __launch_bounds__(128) k_finish_t(TplView T, const gvo_machine* machines, const gvo_config* cfgs,
                                                  const Geo* geos, int64_t n, int S_req, int W_req, int F,
                                                  int64_t* counts, int64_t stride, double* stats, double* records,
                                                  double* field_down) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const gvo_config cfg = cfgs[c];
  finish_one(T, machines, cfg, geos[c], c, S_req, W_req, F, counts + c * stride, stats, records, field_down);
}

// injected float stats (uniform stride F) -> record
__global__ void k_assemble_stats(const gvo_machine* machines, const int32_t* mid, const int64_t* flops,
                                 int64_t n, int F, const double* stats, double* records,
                                 double* field_down) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const gvo_machine m = machines[mid[c]];
  double fdl[4 * kMaxFields];
  assemble_one(m, F, stats + c * GVO_STATS_LEN(F), flops[c], records + c * GVO_RECORD_LEN,
               field_down ? fdl : nullptr);
  if (field_down)
    for (int k = 0; k < 4 * F; ++k) field_down[c * 4 * F + k] = fdl[k];
}

void launch_finish(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs,
                   const Geo* d_geos, int64_t n, int S_req, int W_req, int F, int64_t* d_counts,
                   int64_t counts_stride, double* d_stats, double* d_records, double* d_field_down,
                   cudaStream_t st) {
  if (n <= 0) return;
#ifndef GVO_FINISH_THREAD
#define GVO_FINISH_THREAD 1
#endif
  if (GVO_FINISH_THREAD) {
    k_finish_t<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(T, d_machines, d_cfgs, d_geos, n, S_req, W_req, F,
                                                             d_counts, counts_stride, d_stats, d_records,
                                                             d_field_down);
    return;
  }
  const size_t smem = kFinishWarps * (counts_stride + (sizeof(Geo) + 7) / 8) * sizeof(int64_t);
  k_finish<<<(unsigned)((n + kFinishWarps - 1) / kFinishWarps), 32 * kFinishWarps, smem, st>>>(
      T, d_machines, d_cfgs, d_geos, n, S_req, W_req, F, d_counts, counts_stride, d_stats, d_records,
      d_field_down);
}

void launch_assemble_stats(const gvo_machine* d_machines, const int32_t* d_mid, const int64_t* d_flops,
                           int64_t n, int F, const double* d_stats, double* d_records,
                           double* d_field_down, cudaStream_t st) {
  if (n <= 0) return;
  const int tb = 64;
  k_assemble_stats<<<(unsigned)((n + tb - 1) / tb), tb, 0, st>>>(d_machines, d_mid, d_flops, n, F, d_stats,
                                                                  d_records, d_field_down);
}

}  // namespace gvo
