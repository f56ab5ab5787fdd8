// k_setup.cu — per-config plan: affine coefficient tables, representative
// blocks, waves and wave pairs, and the int64 overflow guard.
//
// One warp per configuration.  Lanes stride over accesses.
//   coefficients      : reference expr.affine_parts (expr.py:171-212) with
//                       BX/BY/BZ and field bases bound per config
//   representative    : footprint.representative_blocks (footprint.py:591-613),
//                       closed form of the sorted interior-block meshgrid
//   waves / pairs     : footprint.blocks_per_wave / build_waves /
//                       representative_wave_pairs (footprint.py:48-78, 616-637)
//   overflow guard    : expr.value_bounds per (group, access) in the order the
//                       reference evaluates them: block samples
//                       (volumes.py:160-176), sampled waves current-first
//                       (volumes.py:227-239, footprint.py:541-545), the L1
//                       block (volumes.py:120-127).
#include "gvo_bytecode.cuh"
#include "gvo_kernels.h"

namespace gvo {

__device__ inline void interior(int64_t e, int64_t* off, int64_t* n) {
  if (e > 2) { *off = 1; *n = e - 2; }
  else { *off = 0; *n = e; }
}

// representative_blocks(kernel, samples) -> sorted linear indices; returns count
__device__ inline int representative(const int64_t g[3], int samples, int64_t* out, int cap) {
  int64_t ox, nx, oy, ny, oz, nz;
  interior(g[0], &ox, &nx);
  interior(g[1], &oy, &ny);
  interior(g[2], &oz, &nz);
  const int64_t n = nx * ny * nz;
  auto lin_of = [&](int64_t k) {
    const int64_t x = k % nx, y = (k / nx) % ny, z = k / (nx * ny);
    return (x + ox) + g[0] * ((y + oy) + g[1] * (z + oz));
  };
  int cnt = 0;
  if (n <= samples) {
    for (int64_t k = 0; k < n && cnt < cap; ++k) out[cnt++] = lin_of(k);
    return n <= cap ? (int)n : -1;
  }
  // np.unique(np.round(np.linspace(0, n-1, samples)))  (footprint.py:597-600)
  const double step = samples > 1 ? (double)(n - 1) / (double)(samples - 1) : 0.0;
  int64_t prev = -1;
  for (int i = 0; i < samples; ++i) {
    int64_t k;
    if (i == samples - 1 && samples > 1) k = n - 1;
    else k = (int64_t)rint(__dmul_rn((double)i, step));
    if (k == prev) continue;
    if (cnt >= cap) return -1;
    out[cnt++] = lin_of(k);
    prev = k;
  }
  return cnt;
}

// Coefficient classes of every (field, kind) slot (one warp).  Lanes find
// each access's representative (first earlier access of the slot with the
// same coefficients); lane 0 numbers the classes in slot order; lanes then
// gather each class's constants and sort them (insertion sort, unique).
__device__ void build_classes(const TplView& T, int tpl, const int64_t* crow, CTab ct, int16_t* rep_of) {
  const int lane = threadIdx.x & 31;
  const int32_t* fko = T.fk_off + tpl * (2 * kMaxFields + 1);
  for (int slot = 0; slot < 2 * kMaxFields; ++slot) {
    const int b = fko[slot], e = fko[slot + 1];
    for (int q = b + lane; q < e; q += 32) {
      const int a = T.fk_list[q];
      const int64_t* ca = crow + a * 8;
      int64_t r = -1;
      if (ca[7] == kAffine) {
        r = a;
        for (int q2 = b; q2 < q; ++q2) {
          const int a2 = T.fk_list[q2];
          const int64_t* cb = crow + a2 * 8;
          if (cb[7] != kAffine) continue;
          bool same = true;
          for (int k = 1; k < 7; ++k) same &= cb[k] == ca[k];
          if (same) { r = a2; break; }
        }
      }
      rep_of[a] = (int16_t)r;
    }
  }
  __syncwarp();
  if (lane == 0) {
    int64_t ncls = 0, off = 0;
    for (int slot = 0; slot < 2 * kMaxFields; ++slot) {
      ct.slot_first()[slot] = ncls;
      const int b = fko[slot], e = fko[slot + 1];
      for (int q = b; q < e; ++q) {
        const int a = T.fk_list[q];
        if (rep_of[a] != a) continue;
        int64_t members = 0;
        for (int q2 = q; q2 < e; ++q2) members += rep_of[T.fk_list[q2]] == a;
        ct.rep()[ncls] = a;
        ct.start()[ncls] = off;
        ct.cnt()[ncls] = members;
        off += members;
        ++ncls;
      }
    }
    ct.slot_first()[2 * kMaxFields] = ncls;
  }
  __syncwarp();
  const int64_t ncls = ct.slot_first()[2 * kMaxFields];
  for (int64_t c = lane; c < ncls; c += 32) {
    const int64_t r = ct.rep()[c];
    const int f = T.acc_field[T.acc_base[tpl] + r], k = T.acc_kind[T.acc_base[tpl] + r];
    const int b = fko[f * 2 + k], e = fko[f * 2 + k + 1];
    int64_t* P = ct.pts() + ct.start()[c];
    int64_t n = 0;
    for (int q = b; q < e; ++q) {
      const int a = T.fk_list[q];
      if (rep_of[a] != r) continue;
      const int64_t v = crow[a * 8];
      int64_t j = n;
      bool dup = false;
      while (j > 0 && P[j - 1] >= v) {
        if (P[j - 1] == v) { dup = true; break; }
        --j;
      }
      if (dup) continue;
      for (int64_t m = n; m > j; --m) P[m] = P[m - 1];
      P[j] = v;
      ++n;
    }
    ct.cnt()[c] = n;
  }
}

__global__ void k_setup(TplView T, const gvo_machine* machines, const gvo_config* cfgs,
                        int64_t n, gvo_sampling smp, int64_t* coefs, Geo* geos, int64_t* ctabs) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n) return;
  const gvo_config cfg = cfgs[c];
  const int tpl = cfg.template_id;
  const gvo_machine m = machines[cfg.machine_id];
  const int A = T.n_acc[tpl];
  const int F = T.n_fields[tpl];
  const int abase = T.acc_base[tpl];
  const int64_t* fbase = T.field_base + T.field_base_off[tpl];
  const int32_t bd[3] = {cfg.block[0], cfg.block[1], cfg.block[2]};
  const int64_t gd[3] = {cfg.grid[0], cfg.grid[1], cfg.grid[2]};
  int64_t* crow = coefs + c * (int64_t)T.max_acc * 8;

  // ---- coefficient tables (lane-parallel over accesses)
  for (int a = lane; a < A; a += 32) {
    const int ga = abase + a;
    AffineForm f;
    int flag = affine_extract(T.code + T.code_off[ga], T.code_len[ga], bd, fbase, &f);
    for (int k = 0; k < 7; ++k) crow[a * 8 + k] = flag == kAffine ? f.c[k] : 0;
    crow[a * 8 + 7] = flag;
  }
  __syncwarp();
  {
    extern __shared__ int16_t sh_rep[];
    build_classes(T, tpl, crow, CTab{ctabs + c * ctab_stride(T.max_acc), T.max_acc},
                  sh_rep + (threadIdx.x >> 5) * T.max_acc);
  }

  // ---- geometry (computed redundantly by every lane; cheap and uniform)
  Geo G;
  G.phases = smp.phases ? smp.phases : 7;
  G.status = GVO_OK;
  G.err_phase = G.err_group = G.err_access = -1;
  G.tpb = (int64_t)bd[0] * bd[1] * bd[2];
  G.lups_per_block = G.tpb * cfg.work_per_thread;
  G.total_blocks = gd[0] * gd[1] * gd[2];
  G.n_samples = 0;
  G.n_uw = 0;
  G.n_pairs = 0;
  G.has_pred = 0;
  G.per_wave = 0;
  G.n_waves = 0;
  G.first_wave = 0;
  G.l1_block = -1;

  auto fail = [&](int status, int phase, int group, int access) {
    G.status = status;
    G.err_phase = phase;
    G.err_group = group;
    G.err_access = access;
  };

  // coordinate-bounds guard for one group over all accesses in the given
  // order (by field then kernel order, optionally loads before stores);
  // returns the first failing access position or -1.
  auto guard = [&](int64_t rs, int64_t rc, int order) -> int {
    int64_t clo[6], chi[6];
    clo[0] = clo[1] = clo[2] = 0;
    chi[0] = bd[0] - 1; chi[1] = bd[1] - 1; chi[2] = bd[2] - 1;
    run_bid_bounds(rs, rc, gd, clo + 3, chi + 3);
    int best = INT32_MAX;  // order key
    int best_a = -1;
    for (int a = lane; a < A; a += 32) {
      const int ga = abase + a;
      int64_t lo, hi;
      if (bounds_check(T.code + T.code_off[ga], T.code_len[ga], clo, chi, bd, fbase, &lo, &hi) >= 0) {
        // order 0: field-major, kernel order inside (volumes.py:164-171)
        // order 1: field, loads before stores (footprint.py:541-545)
        // order 2: kernel order (volumes.py:126)
        const int f = order == 2 ? 0 : T.acc_field[ga];
        const int kind = order == 1 ? T.acc_kind[ga] : 0;
        const int key = (f * 2 + kind) * GVO_MAX_ACCESSES + a;
        if (key < best) { best = key; best_a = a; }
      }
    }
    for (int o = 16; o; o >>= 1) {
      int ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oa = __shfl_xor_sync(0xffffffffu, best_a, o);
      if (ob < best) { best = ob; best_a = oa; }
    }
    return best_a;
  };

  // ---- phase 0: block samples (volumes.py:152-185)
  if (!(G.phases & 1)) {
    // not requested
  } else if (smp.block_samples < 1) {
    fail(GVO_ERR_FOOTPRINT, 0, -1, 0);  // "sample count must be >= 1"
  } else {
    int ns = representative(gd, smp.block_samples, G.sample_lin, kMaxSamples);
    if (ns < 0) fail(GVO_ERR_UNSUPPORTED, 0, -1, 0);
    else G.n_samples = ns;
  }
  // ---- translation dedup of block samples (exact): all accesses of field f
  // affine with one common block-coordinate coefficient vector, and the
  // address shift between samples j and j' a multiple of the line size.
  for (int f = 0; f < kMaxFields; ++f)
    for (int j = 0; j < kMaxSamples; ++j) G.dup_of[f][j] = -1;
  if (G.status == GVO_OK && (G.phases & 1)) {
    const int32_t* fko = T.fk_off + tpl * (2 * kMaxFields + 1);
    for (int f = 0; f < F; ++f) {
      bool ok = true;
      const int64_t* c0 = nullptr;
      for (int q = fko[2 * f]; q < fko[2 * f + 2] && ok; ++q) {
        const int64_t* ca = crow + T.fk_list[q] * 8;
        if (ca[7] != kAffine) { ok = false; break; }
        if (!c0) c0 = ca;
        else ok = ca[4] == c0[4] && ca[5] == c0[5] && ca[6] == c0[6];
      }
      if (!ok || !c0) continue;
      const int64_t line = m.l1_line_bytes;
      for (int j = 1; j < G.n_samples; ++j) {
        const int64_t bj = G.sample_lin[j];
        const int64_t xj = bj % gd[0], yj = (bj / gd[0]) % gd[1], zj = bj / (gd[0] * gd[1]);
        for (int i = 0; i < j; ++i) {
          if (G.dup_of[f][i] >= 0) continue;
          const int64_t bi = G.sample_lin[i];
          const int64_t xi = bi % gd[0], yi = (bi / gd[0]) % gd[1], zi = bi / (gd[0] * gd[1]);
          const __int128 d = (__int128)c0[4] * (xj - xi) + (__int128)c0[5] * (yj - yi) + (__int128)c0[6] * (zj - zi);
          const __int128 r = d % line;
          if (r == 0) { G.dup_of[f][j] = (int8_t)i; break; }
        }
      }
    }
  }
  if (G.status == GVO_OK && (G.phases & 1)) {
    for (int s = 0; s < G.n_samples; ++s) {
      int a = guard(G.sample_lin[s], 1, 0);
      if (a >= 0) { fail(GVO_ERR_ADDRESS_OVERFLOW, 0, s, a); break; }
    }
  }

  // ---- phase 1: waves (volumes.py:203-250)
  if (G.status == GVO_OK && (G.phases & 2)) {
    int64_t per_wave = smp.blocks_per_wave_override;
    if (smp.wave_samples < 1) {
      fail(GVO_ERR_FOOTPRINT, 1, -1, 0);
    } else if (per_wave == 0) {
      // blocks_per_wave (footprint.py:48-57)
      if (G.tpb > m.max_threads_per_block) fail(GVO_ERR_FOOTPRINT, 1, -1, 1);
      else {
        int64_t per_sm = m.max_threads_per_sm / G.tpb;
        if (m.max_blocks_per_sm < per_sm) per_sm = m.max_blocks_per_sm;
        if (per_sm < 1) fail(GVO_ERR_FOOTPRINT, 1, -1, 2);
        else per_wave = m.sm_count * per_sm;
      }
    }
    if (G.status == GVO_OK && per_wave < 1) fail(GVO_ERR_FOOTPRINT, 1, -1, 3);
    if (G.status == GVO_OK) {
      G.per_wave = per_wave;
      G.n_waves = (G.total_blocks + per_wave - 1) / per_wave;
      int64_t start, count;
      if (G.n_waves == 1) {
        G.n_pairs = 1;
        G.has_pred = 0;
        G.n_uw = 1;
        G.first_wave = 0;
      } else {
        const int64_t hi = G.n_waves >= 3 ? G.n_waves - 2 : G.n_waves - 1;
        const int64_t lo = 1;
        count = smp.wave_samples < hi - lo + 1 ? smp.wave_samples : hi - lo + 1;
        const int64_t mid = (lo + hi) / 2;
        start = mid - (count - 1) / 2;
        if (start < lo) start = lo;
        if (start > hi - count + 1) start = hi - count + 1;
        if (count + 1 > kMaxUWaves) fail(GVO_ERR_UNSUPPORTED, 1, -1, 0);
        G.n_pairs = (int)count;
        G.has_pred = 1;
        G.n_uw = (int)count + 1;
        G.first_wave = start - 1;
      }
      if (G.status == GVO_OK) {
        for (int u = 0; u < G.n_uw; ++u) {
          const int64_t w = G.first_wave + u;
          G.uw_start[u] = w * per_wave;
          const int64_t rem = G.total_blocks - G.uw_start[u];
          G.uw_count[u] = rem < per_wave ? rem : per_wave;
        }
        // evaluation order: current of pair 0, its predecessor, then the
        // remaining currents (cached summaries are not re-evaluated)
        for (int k = 0; k < G.n_uw && G.status == GVO_OK; ++k) {
          int u = G.n_uw == 1 ? 0 : (k == 0 ? 1 : (k == 1 ? 0 : k));
          int a = guard(G.uw_start[u], G.uw_count[u], 1);
          if (a >= 0) fail(GVO_ERR_ADDRESS_OVERFLOW, 1, u, a);
        }
      }
    }
  }

  // ---- phase 2: L1 block = representative_blocks(k, 5)[len // 2]
  if (G.status == GVO_OK && (G.phases & 4)) {
    int64_t picks[5];
    int np = representative(gd, 5, picks, 5);
    G.l1_block = picks[np / 2];
    int a = guard(G.l1_block, 1, 2);
    if (a >= 0) fail(GVO_ERR_ADDRESS_OVERFLOW, 2, 0, a);
  }
  if (lane == 0) geos[c] = G;
}

void launch_setup(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs,
                  int64_t n, const gvo_sampling& smp, int64_t* d_coefs, Geo* d_geos, int64_t* d_ctabs,
                  cudaStream_t st) {
  const int wpb = 4;
  const int64_t blocks = (n + wpb - 1) / wpb;
  if (blocks > 0)
    k_setup<<<(unsigned)blocks, wpb * 32, wpb * T.max_acc * sizeof(int16_t), st>>>(T, d_machines, d_cfgs, n, smp,
                                                                                   d_coefs, d_geos, d_ctabs);
}

__global__ void k_classes_only(TplView T, const gvo_config* cfgs, int64_t n, const int64_t* coefs,
                               int64_t* ctabs) {
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n) return;
  extern __shared__ int16_t sh_rep2[];
  build_classes(T, cfgs[c].template_id, coefs + c * (int64_t)T.max_acc * 8,
                CTab{ctabs + c * ctab_stride(T.max_acc), T.max_acc}, sh_rep2 + (threadIdx.x >> 5) * T.max_acc);
}

void launch_classes(const TplView& T, const gvo_config* d_cfgs, int64_t n, const int64_t* d_coefs,
                    int64_t* d_ctabs, cudaStream_t st) {
  if (n > 0)
    k_classes_only<<<(unsigned)((n + 3) / 4), 128, 4 * T.max_acc * sizeof(int16_t), st>>>(T, d_cfgs, n, d_coefs,
                                                                                          d_ctabs);
}

}  // namespace gvo
