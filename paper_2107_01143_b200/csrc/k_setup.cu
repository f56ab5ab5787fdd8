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

#include <algorithm>

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

// Coefficient classes of every (field, kind) slot, all threads of the CTA.
// Representatives (first earlier access of the slot with identical
// coefficients) per access, member counts per representative, class
// numbering in slot order (thread 0, O(A)), then each class's constants
// gathered and sorted (insertion sort, unique) by one thread per class.
__device__ void build_classes_cta(const TplView& T, int tpl, const int64_t* crow, CTab ct, int16_t* rep_of,
                                  int16_t* members) {
  const int32_t* fko = T.fk_off + tpl * (2 * kMaxFields + 1);
  const int A = T.n_acc[tpl];
  const int abase = T.acc_base[tpl];
  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    const int slot = T.acc_field[abase + a] * 2 + T.acc_kind[abase + a];
    const int64_t* ca = crow + a * 8;
    int r = -1;
    if (ca[7] == kAffine) {
      r = a;
      for (int q2 = fko[slot]; q2 < fko[slot + 1]; ++q2) {
        const int a2 = T.fk_list[q2];
        if (a2 == a) break;
        const int64_t* cb = crow + a2 * 8;
        if (cb[7] != kAffine) continue;
        bool same = true;
        for (int k = 1; k < 7; ++k) same &= cb[k] == ca[k];
        if (same) { r = a2; break; }
      }
    }
    rep_of[a] = (int16_t)r;
  }
  __syncthreads();
  // class numbering in slot order: class = position q of fk_list holding a
  // representative; ranks by a warp-0 ballot scan over fk_list (which is
  // grouped by slot), then per-class distinct-constant counts
  __shared__ int s_ncls;
  int16_t* qrank = members;  // exclusive rank of representative positions, by fk_list position
  const int q0 = fko[0], q1 = fko[2 * kMaxFields];
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int base = 0;
    for (int qq = q0; qq < q1; qq += 32) {
      const int q = qq + lane;
      const bool isr = q < q1 && rep_of[T.fk_list[q]] == T.fk_list[q];
      const unsigned bal = __ballot_sync(0xffffffffu, isr);
      if (q < q1) qrank[q - q0] = (int16_t)(base + __popc(bal & ((1u << lane) - 1u)));
      base += __popc(bal);
    }
    if (lane == 0) s_ncls = base;
  }
  __syncthreads();
  const int ncls = s_ncls;
  for (int slot = threadIdx.x; slot <= 2 * kMaxFields; slot += blockDim.x) {
    const int q = fko[slot];
    ct.slot_first()[slot] = slot == 2 * kMaxFields ? ncls : (q < q1 ? qrank[q - q0] : ncls);
  }
  // class c = rank of its representative's fk_list position; member count
  int32_t* nu_start = reinterpret_cast<int32_t*>(members + ((T.max_acc + 1) & ~1));  // non-unique offsets (4-byte aligned)
  int32_t* n_uniq = nu_start + T.max_acc;
  for (int q = q0 + (int)threadIdx.x; q < q1; q += blockDim.x) {
    const int a = T.fk_list[q];
    if (rep_of[a] != a) continue;
    const int c = qrank[q - q0];
    const int slot = T.acc_field[abase + a] * 2 + T.acc_kind[abase + a];
    int m = 0;
    for (int q2 = fko[slot]; q2 < fko[slot + 1]; ++q2) m += rep_of[T.fk_list[q2]] == a;
    ct.rep()[c] = a;
    nu_start[c] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // ncls <= A
    int off = 0;
    for (int c = 0; c < ncls; ++c) { const int m = nu_start[c]; nu_start[c] = off; off += m; }
  }
  __syncthreads();
  // members placed at their rank (ties by position) in the scratch row:
  // each class's constants sorted, duplicates adjacent
  int64_t* tmp = ct.rep_of();
  for (int q = q0 + (int)threadIdx.x; q < q1; q += blockDim.x) {
    const int b = T.fk_list[q];
    const int r = rep_of[b];
    if (r < 0) continue;
    const int slot = T.acc_field[abase + b] * 2 + T.acc_kind[abase + b];
    const int64_t v = crow[b * 8];
    int rank = 0, qr = -1;
    for (int q2 = fko[slot]; q2 < fko[slot + 1]; ++q2) {
      const int b2 = T.fk_list[q2];
      if (b2 == r) qr = q2;
      if (rep_of[b2] != r) continue;
      const int64_t u = crow[b2 * 8];
      rank += (u < v) || (u == v && q2 < q);
    }
    tmp[nu_start[qrank[qr - q0]] + rank] = v;
  }
  __syncthreads();
  // distinct constants: a sorted element is kept unless it equals its predecessor
  for (int c = threadIdx.x; c < ncls; c += blockDim.x) {
    const int a = (int)ct.rep()[c];
    const int slot = T.acc_field[abase + a] * 2 + T.acc_kind[abase + a];
    int m = 0;
    for (int q2 = fko[slot]; q2 < fko[slot + 1]; ++q2) m += rep_of[T.fk_list[q2]] == a;
    const int e0 = nu_start[c];
    int u = 0;
    for (int i = 0; i < m; ++i) u += (i == 0 || tmp[e0 + i] != tmp[e0 + i - 1]);
    n_uniq[c] = u;
    ct.cnt()[c] = u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // class point offsets: exclusive scan of distinct counts
    int64_t off = 0;
    for (int c = 0; c < ncls; ++c) { ct.start()[c] = off; off += n_uniq[c]; }
  }
  __syncthreads();
  // compact: the thread of sorted element i writes it if it starts a new value
  for (int q = q0 + (int)threadIdx.x; q < q1; q += blockDim.x) {
    // element index within the scratch row = q - q0 covers every member once
    const int i = q - q0;
    // class of element i: last class whose non-unique start <= i (member
    // counts are positive, so starts are strictly increasing)
    int lo = 0, hi = ncls - 1;
    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (nu_start[mid] <= i) lo = mid; else hi = mid - 1; }
    if (ncls == 0) continue;
    const int c = lo;
    const int e0 = nu_start[c];
    const int e1 = c + 1 < ncls ? nu_start[c + 1] : -1;
    if (e1 >= 0 && i >= e1) continue;
    // elements beyond the last class (non-affine accesses) are not in any class
    const int a = (int)ct.rep()[c];
    if (e1 < 0) {
      const int slot = T.acc_field[abase + a] * 2 + T.acc_kind[abase + a];
      int m = 0;
      for (int q2 = fko[slot]; q2 < fko[slot + 1]; ++q2) m += rep_of[T.fk_list[q2]] == a;
      if (i >= e0 + m) continue;
    }
    if (i > e0 && tmp[i] == tmp[i - 1]) continue;
    int u = 0;
    for (int k = e0 + 1; k <= i; ++k) u += tmp[k] != tmp[k - 1];
    ct.pts()[ct.start()[c] + u] = tmp[i];
  }
  __syncthreads();
}

// dynamic shared memory of the setup kernels: rep_of and qrank (int16), the
// classes' non-unique offsets and distinct counts (int32)
static size_t setup_smem(int max_acc) {
  return (size_t)2 * (((max_acc + 1) & ~1) * sizeof(int16_t)) + 2 * (size_t)max_acc * sizeof(int32_t);
}

// evaluation-order key of a (phase, group, access) overflow failure
__device__ __forceinline__ unsigned long long fail_key(int phase, int gorder, int f, int kind, int a) {
  return ((unsigned long long)phase << 56) | ((unsigned long long)gorder << 40) |
         ((unsigned long long)(f * 2 + kind) << 16) | (unsigned long long)a;
}

// ------------------------------------------------------------------ plan sharing
// The plan of a configuration (coefficients, classes, geometry, overflow
// guard) depends only on its template's accesses, the launch and the
// machine's integer parameters — not on capacities, bandwidths or fits, and,
// for translation-safe templates (capi.cu translation_classes: every field
// base enters its accesses additively with coefficient 1), on the field
// bases only through a shift: moving base_f by D moves the constant of
// every affine access of field f, and every node interval of the guard,
// by o*D with |o| <= 8 (o = the node's base coefficient).  So one leader per
// key (translation class, block, grid, work per thread, machine class)
// computes the plan, and its followers take it with the constants shifted.
// Exactness: the leader's plan is shared only if its status is OK and every
// coefficient and every guard interval bound of every node is <= 2^62 in
// magnitude; a follower with |D| <= 2^58 then has every node within
// 2^62 + 8*2^58 < 2^63 - 1: the same affine flags and no overflow, which
// is what the reference computes for it.  Anything else computes itself.
// The reference recomputes every configuration (perf.py:115-130).
namespace {
constexpr int kPlanKey = 6;
constexpr int kPlanProbe = 64;
constexpr uint64_t kPlanMag = uint64_t(1) << 62;
constexpr int64_t kPlanShift = int64_t(1) << 58;

__device__ __forceinline__ uint64_t pmix(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 29);
}

// cache slot layout (int64 words): [0] share_ok, [1, 1+F) leader field
// bases, then Geo, the coefficient row and the class table row
__host__ __device__ inline int64_t plan_geo_off() { return (1 + kMaxFields + 1) & ~int64_t(1); }
__host__ __device__ inline int64_t plan_coef_off() { return plan_geo_off() + ((int64_t)sizeof(Geo) + 15) / 16 * 2; }
__host__ __device__ inline int64_t plan_ctab_off(int64_t A) { return plan_coef_off() + A * 8; }
}  // namespace

// slots start on 16-byte boundaries (TMA bulk copies of their Geo and coefficient rows)
__host__ __device__ int64_t plan_slot_words(int64_t max_acc) {
  return (plan_ctab_off(max_acc) + ctab_stride(max_acc) + 1) & ~int64_t(1);
}

// ---- TMA (cp.async.bulk) 1D copies through shared memory: the bulk-copy
// engine moves a follower's geometry and coefficient row (contiguous, 16-byte
// aligned, 1.1 KB and 64*A bytes) while the threads only patch constants
#ifndef GVO_PLAN_TMA
#define GVO_PLAN_TMA 1
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tma_bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// global -> shared, completion counted on bar (one thread)
__device__ __forceinline__ void tma_load_1d(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}
// shared -> global (one thread), after the shared-memory writes are fenced to the async proxy
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// One thread per configuration of the batch: src[c] = slot >= 0 (take the
// plan cached in slot), -2 - slot (leader: compute, then fill slot), -1
// (compute, not shared).
__global__ void k_plan_key(TplView T, const int32_t* mclass, const gvo_config* cfgs, int64_t n, PlanShare PS) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  PS.src[c] = -1;
  const gvo_config cfg = cfgs[c];
  if (cfg.work_per_thread < 0 || cfg.work_per_thread >= (int64_t(1) << 31)) return;
  const int tpl = cfg.template_id;
  const int tcls = T.tclass ? T.tclass[tpl] : -1;
  uint64_t key[kPlanKey];
  key[0] = tcls >= 0 ? (uint64_t)tcls : ((uint64_t)1 << 40) | (uint64_t)tpl;
  key[1] = (uint64_t)(uint32_t)cfg.block[0] | ((uint64_t)(uint32_t)cfg.block[1] << 21) |
           ((uint64_t)(uint32_t)cfg.block[2] << 42);
  key[2] = (uint64_t)cfg.grid[0];
  key[3] = (uint64_t)cfg.grid[1];
  key[4] = (uint64_t)cfg.grid[2];
  key[5] = (uint64_t)cfg.work_per_thread | ((uint64_t)(uint32_t)mclass[cfg.machine_id] << 32);
  uint64_t h = 0x13198a2e03707344ull;
#pragma unroll
  for (int k = 0; k < kPlanKey; ++k) h = pmix(h, key[k]);
  const uint64_t tag = h | 1ull;
  int64_t slot = (int64_t)(h >> 9) & PS.mask;
  for (int p = 0; p < kPlanProbe; ++p, slot = (slot + 1) & PS.mask) {
    PlanEntry& e = PS.table[slot];
    const unsigned long long old = atomicCAS(&e.tag, 0ull, (unsigned long long)tag);
    if (old == 0ull) {  // claimed: leader of its key
      const unsigned long long s = atomicAdd(PS.n_used, 1ull);
      const int cs = s < (unsigned long long)PS.cap ? (int)s : -1;
      for (int k = 0; k < kPlanKey; ++k) e.key[k] = key[k];
      e.slot = cs;
      __threadfence();
      atomicExch(&e.ready, 1);
      if (cs >= 0) PS.src[c] = -2 - cs;
      return;
    }
    if (old != tag) continue;
    while (atomicAdd(&e.ready, 0) == 0) __nanosleep(32);
    __threadfence();
    bool same = true;
#pragma unroll
    for (int k = 0; k < kPlanKey; ++k) same &= *reinterpret_cast<volatile uint64_t*>(&e.key[k]) == key[k];
    if (same) {
      const int cs = *reinterpret_cast<volatile int*>(&e.slot);
      PS.src[c] = cs >= 0 ? cs : -1;
      return;
    }
  }
}

// The plan of one configuration, all threads of the CTA (256).  A leader
// (src <= -2) also fills its cache slot.
__device__ void setup_one(const TplView& T, const gvo_machine* machines, const gvo_config* cfgs, int64_t c,
                          const gvo_sampling& smp, int64_t* coefs, Geo* geos, int64_t* ctabs, int64_t* cache_slot) {
  extern __shared__ int16_t sh16[];
  __shared__ Geo G;
  __shared__ unsigned long long first_fail;
  __shared__ unsigned long long s_mag;  // largest |coefficient| / |guard bound| of any node
  if (threadIdx.x == 0) s_mag = 0;
  __syncthreads();
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

  // ---- coefficient tables (thread per access)
  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    const int ga = abase + a;
    AffineForm f;
    uint64_t mag = 0;
    int flag = affine_extract(T.code + T.code_off[ga], T.code_len[ga], bd, fbase, &f, cache_slot ? &mag : nullptr);
    for (int k = 0; k < 7; ++k) crow[a * 8 + k] = flag == kAffine ? f.c[k] : 0;
    crow[a * 8 + 7] = flag;
    if (cache_slot && mag) atomicMax(&s_mag, (unsigned long long)mag);
  }
  __syncthreads();
  build_classes_cta(T, tpl, crow, CTab{ctabs + c * ctab_stride(T.max_acc), T.max_acc}, sh16, sh16 + ((T.max_acc + 1) & ~1));

  // ---- geometry (thread 0)
  if (threadIdx.x == 0) {
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
    for (int f = 0; f < kMaxFields; ++f)
      for (int j = 0; j < kMaxSamples; ++j) G.dup_of[f][j] = -1;
    first_fail = ~0ull;
    auto fail = [&](int status, int phase, int group, int access) {
      G.status = status;
      G.err_phase = phase;
      G.err_group = group;
      G.err_access = access;
    };
    // phase 0 geometry (volumes.py:152-185)
    if (G.phases & 1) {
      if (smp.block_samples < 1) fail(GVO_ERR_FOOTPRINT, 0, -1, 0);
      else {
        const int ns = representative(gd, smp.block_samples, G.sample_lin, kMaxSamples);
        if (ns < 0) fail(GVO_ERR_UNSUPPORTED, 0, -1, 0);
        else G.n_samples = ns;
      }
    }
    // phase 1 geometry (footprint.py:48-78, 616-637); its FootprintErrors are
    // raised only if phase 0 passes the overflow guard (resolved below)
    if (G.status == GVO_OK && (G.phases & 2)) {
      int64_t per_wave = smp.blocks_per_wave_override;
      int err = -1;
      if (smp.wave_samples < 1) err = 0;
      else if (per_wave == 0) {
        if (G.tpb > m.max_threads_per_block) err = 1;
        else {
          int64_t per_sm = m.max_threads_per_sm / G.tpb;
          if (m.max_blocks_per_sm < per_sm) per_sm = m.max_blocks_per_sm;
          if (per_sm < 1) err = 2;
          else per_wave = m.sm_count * per_sm;
        }
      }
      if (err < 0 && per_wave < 1) err = 3;
      if (err >= 0) {
        G.err_access = err;  // pending: becomes the status unless phase 0 fails first
        G.err_phase = 1;
        G.n_uw = 0;
      } else {
        G.per_wave = per_wave;
        G.n_waves = (G.total_blocks + per_wave - 1) / per_wave;
        if (G.n_waves == 1) {
          G.n_pairs = 1;
          G.has_pred = 0;
          G.n_uw = 1;
          G.first_wave = 0;
        } else {
          const int64_t hi = G.n_waves >= 3 ? G.n_waves - 2 : G.n_waves - 1;
          const int64_t count = smp.wave_samples < hi ? smp.wave_samples : hi;
          const int64_t mid = (1 + hi) / 2;
          int64_t start = mid - (count - 1) / 2;
          if (start < 1) start = 1;
          if (start > hi - count + 1) start = hi - count + 1;
          if (count + 1 > kMaxUWaves) { G.err_access = 100; G.err_phase = 1; }
          else {
            G.n_pairs = (int)count;
            G.has_pred = 1;
            G.n_uw = (int)count + 1;
            G.first_wave = start - 1;
          }
        }
        for (int u = 0; u < G.n_uw; ++u) {
          const int64_t w = G.first_wave + u;
          G.uw_start[u] = w * per_wave;
          const int64_t rem = G.total_blocks - G.uw_start[u];
          G.uw_count[u] = rem < per_wave ? rem : per_wave;
        }
      }
    }
    // phase 2 geometry: representative_blocks(k, 5)[len // 2]
    if (G.status == GVO_OK && (G.phases & 4)) {
      int64_t picks[5];
      const int np = representative(gd, 5, picks, 5);
      G.l1_block = picks[np / 2];
    }
  }
  __syncthreads();

  // ---- overflow guard: thread per (group, access), first failure in the
  // reference's evaluation order.  Groups: samples (order s), sampled waves
  // (current of pair 0, its predecessor, then the other currents), L1 block.
  if (G.status == GVO_OK) {
    const int ns = (G.phases & 1) ? G.n_samples : 0;
    const int nu = (G.phases & 2) ? G.n_uw : 0;
    const int nl = (G.phases & 4) ? 1 : 0;
    const int ng = ns + nu + nl;
    for (int t = threadIdx.x; t < ng * A; t += blockDim.x) {
      const int gi = t / A, a = t % A;
      int phase, gorder, rs_idx;
      int64_t rs, rc;
      if (gi < ns) { phase = 0; gorder = gi; rs = G.sample_lin[gi]; rc = 1; rs_idx = gi; }
      else if (gi < ns + nu) {
        const int k = gi - ns;
        const int u = G.n_uw == 1 ? 0 : (k == 0 ? 1 : (k == 1 ? 0 : k));
        phase = 1; gorder = k; rs = G.uw_start[u]; rc = G.uw_count[u]; rs_idx = u;
      } else { phase = 2; gorder = 0; rs = G.l1_block; rc = 1; rs_idx = 0; }
      int64_t clo[6], chi[6];
      clo[0] = clo[1] = clo[2] = 0;
      chi[0] = bd[0] - 1; chi[1] = bd[1] - 1; chi[2] = bd[2] - 1;
      run_bid_bounds(rs, rc, gd, clo + 3, chi + 3);
      const int ga = abase + a;
      int64_t lo, hi;
      uint64_t mag = 0;
      const int bad = bounds_check(T.code + T.code_off[ga], T.code_len[ga], clo, chi, bd, fbase, &lo, &hi,
                                   cache_slot ? &mag : nullptr);
      if (cache_slot && mag) atomicMax(&s_mag, (unsigned long long)mag);
      if (bad >= 0) {
        // order inside a group: phase 0 field-major (volumes.py:164-171);
        // phase 1 field, loads before stores (footprint.py:541-545);
        // phase 2 kernel order (volumes.py:126)
        const int f = phase == 2 ? 0 : T.acc_field[ga];
        const int kind = phase == 1 ? T.acc_kind[ga] : 0;
        unsigned long long key = fail_key(phase, gorder, f, kind, a);
        key |= (unsigned long long)rs_idx << 32;  // carries the group index (determined by gorder)
        atomicMin(&first_fail, key);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long k = first_fail;
    const int fphase = k == ~0ull ? 3 : (int)(k >> 56);
    // resolve in evaluation order: phase-0 overflow, phase-1 footprint
    // precondition, phase-1 overflow, phase-2 overflow
    if (G.status == GVO_OK) {
      const bool pending1 = G.err_phase == 1;
      if (fphase == 0) {
        G.status = GVO_ERR_ADDRESS_OVERFLOW; G.err_phase = 0;
        G.err_group = (int)((k >> 32) & 0xff); G.err_access = (int)(k & 0xffff);
      } else if (pending1) {
        G.status = G.err_access == 100 ? GVO_ERR_UNSUPPORTED : GVO_ERR_FOOTPRINT;
        if (G.err_access == 100) G.err_access = 0;
        G.err_group = -1;
      } else if (fphase <= 2) {
        G.status = GVO_ERR_ADDRESS_OVERFLOW; G.err_phase = fphase;
        G.err_group = (int)((k >> 32) & 0xff); G.err_access = (int)(k & 0xffff);
      }
    }
  }
  __syncthreads();

  // ---- translation dedup of block samples (thread per field)
  if (G.status == GVO_OK && (G.phases & 1)) {
    const int32_t* fko = T.fk_off + tpl * (2 * kMaxFields + 1);
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
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
          if (d % line == 0) { G.dup_of[f][j] = (int8_t)i; break; }
        }
      }
    }
  }
  __syncthreads();
  // copy the plan out
  {
    const int words = (int)(sizeof(Geo) / 4);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&G);
    uint32_t* dst = reinterpret_cast<uint32_t*>(geos + c);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  }
  if (cache_slot) {  // leader: the plan into the call's cache
    const int64_t A8 = (int64_t)T.max_acc * 8, CS = ctab_stride(T.max_acc);
    if (threadIdx.x == 0) cache_slot[0] = G.status == GVO_OK && s_mag <= kPlanMag;
    for (int f = threadIdx.x; f < kMaxFields; f += blockDim.x) cache_slot[1 + f] = f < F ? fbase[f] : 0;
    const int words = (int)(sizeof(Geo) / 4);
    uint32_t* gdst = reinterpret_cast<uint32_t*>(cache_slot + plan_geo_off());
    const uint32_t* gsrc = reinterpret_cast<const uint32_t*>(&G);
    for (int i = threadIdx.x; i < words; i += blockDim.x) gdst[i] = gsrc[i];
    for (int64_t i = threadIdx.x; i < (int64_t)A * 8; i += blockDim.x) cache_slot[plan_coef_off() + i] = crow[i];
    // the class table's defined words: slot heads, per-class start/cnt/rep, the points
    const CTab src{ctabs + c * CS, T.max_acc}, dst{cache_slot + plan_ctab_off(T.max_acc), T.max_acc};
    const int ncls = (int)src.slot_first()[2 * kMaxFields];
    for (int i = threadIdx.x; i <= 2 * kMaxFields; i += blockDim.x) dst.slot_first()[i] = src.slot_first()[i];
    for (int i = threadIdx.x; i < ncls; i += blockDim.x) {
      dst.start()[i] = src.start()[i];
      dst.cnt()[i] = src.cnt()[i];
      dst.rep()[i] = src.rep()[i];
    }
    const int64_t npts = ncls ? src.start()[ncls - 1] + src.cnt()[ncls - 1] : 0;
    for (int64_t i = threadIdx.x; i < npts; i += blockDim.x) dst.pts()[i] = src.pts()[i];
    (void)A8;
  }
}

// One CTA per configuration: leaders and unshared configurations.
__global__ void __launch_bounds__(256) k_setup(TplView T, const gvo_machine* machines, const gvo_config* cfgs,
                                               int64_t n, gvo_sampling smp, int64_t* coefs, Geo* geos,
                                               int64_t* ctabs, PlanShare PS) {
  const int64_t c = blockIdx.x;
  if (c >= n) return;
  const int64_t ps = PS.src ? PS.src[c] : -1;
  if (ps >= 0) return;  // a follower: k_plan_follow
  setup_one(T, machines, cfgs, c, smp, coefs, geos, ctabs,
            ps <= -2 ? PS.cache + (-2 - ps) * plan_slot_words(T.max_acc) : nullptr);
}

// One CTA per configuration: followers take their leader's plan with the
// field-base shifts, or compute it when the leader's plan is not shareable.
// Phase 0: the geometry (what sharing, work lists and the float assembly
// read) or the whole plan of a follower that computes itself; phase 1 (after
// the work lists): coefficient rows and class tables, only for followers
// with a unit that computes (need[c]; null = all) — most followers copy
// every count from another configuration and never read them.
__global__ void __launch_bounds__(256) k_plan_follow(TplView T, const gvo_machine* machines, const gvo_config* cfgs,
                                                     int64_t n, gvo_sampling smp, int64_t* coefs, Geo* geos,
                                                     int64_t* ctabs, PlanShare PS, int phase) {
  const int64_t c = blockIdx.x;
  if (c >= n) return;
  const int64_t ps = PS.src[c];
  if (ps < 0) return;
  if (phase == 1 && PS.need && !PS.need[c]) return;
  const int64_t* slot = PS.cache + ps * plan_slot_words(T.max_acc);
  const gvo_config cfg = cfgs[c];
  const int tpl = cfg.template_id;
  const int F = T.n_fields[tpl], A = T.n_acc[tpl], abase = T.acc_base[tpl];
  const int64_t* fbase = T.field_base + T.field_base_off[tpl];
  __shared__ int64_t dlt[kMaxFields];
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    bool ok = slot[0] != 0;
    for (int f = 0; f < F && ok; ++f) {
      const __int128 d = (__int128)fbase[f] - slot[1 + f];
      ok = d >= -kPlanShift && d <= kPlanShift;
      dlt[f] = ok ? (int64_t)d : 0;
    }
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) {
    if (phase == 0) setup_one(T, machines, cfgs, c, smp, coefs, geos, ctabs, nullptr);
    return;
  }
#if GVO_PLAN_TMA
  extern __shared__ __align__(16) int16_t sh16[];
  __shared__ __align__(8) uint64_t tbar;
  int64_t* sbuf = reinterpret_cast<int64_t*>(sh16);  // Geo (phase 0) / coefficient row (phase 1)
  const uint32_t bytes = phase == 0 ? (uint32_t)sizeof(Geo) : (uint32_t)A * 64u;
  if (bytes == 0) return;  // no accesses: nothing to move
  if (threadIdx.x == 0) {
    tma_bar_init(&tbar);
    tma_load_1d(sbuf, phase == 0 ? (const void*)(slot + plan_geo_off()) : (const void*)(slot + plan_coef_off()),
                bytes, &tbar);
  }
  __syncthreads();
  tma_wait(&tbar, 0);
  if (phase == 0) {
    if (threadIdx.x == 0) {
      tma_store_1d(geos + c, sbuf, bytes);
      tma_store_commit_wait();
    }
    return;
  }
  // coefficients: the constant of an affine access moves with its field's base
  for (int a = threadIdx.x; a < A; a += blockDim.x)
    if (sbuf[a * 8 + 7] == kAffine) sbuf[a * 8] += dlt[T.acc_field[abase + a]];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_1d(coefs + c * (int64_t)T.max_acc * 8, sbuf, bytes);
    tma_store_commit_wait();
  }
#else
  if (phase == 0) {
    const int words = (int)(sizeof(Geo) / 4);
    const uint32_t* gsrc = reinterpret_cast<const uint32_t*>(slot + plan_geo_off());
    uint32_t* gdst = reinterpret_cast<uint32_t*>(geos + c);
    for (int i = threadIdx.x; i < words; i += blockDim.x) gdst[i] = gsrc[i];
    return;
  }
  // coefficients: the constant of an affine access moves with its field's base
  const int64_t* csrc = slot + plan_coef_off();
  int64_t* crow = coefs + c * (int64_t)T.max_acc * 8;
  for (int i = threadIdx.x; i < A * 8; i += blockDim.x) {
    const int a = i >> 3, k = i & 7;
    int64_t v = csrc[i];
    if (k == 0 && csrc[a * 8 + 7] == kAffine) v += dlt[T.acc_field[abase + a]];
    crow[i] = v;
  }
#endif
  // class table: same classes, each class's sorted constants shifted by its field's delta
  const int64_t CS = ctab_stride(T.max_acc);
  const int64_t* tsrc = slot + plan_ctab_off(T.max_acc);
  int64_t* tdst = ctabs + c * CS;
  const CTab sct{const_cast<int64_t*>(tsrc), T.max_acc}, dct{tdst, T.max_acc};
  const int ncls = (int)sct.slot_first()[2 * kMaxFields];
  for (int i = threadIdx.x; i <= 2 * kMaxFields; i += blockDim.x) dct.slot_first()[i] = sct.slot_first()[i];
  for (int i = threadIdx.x; i < ncls; i += blockDim.x) {
    dct.start()[i] = sct.start()[i];
    dct.cnt()[i] = sct.cnt()[i];
    dct.rep()[i] = sct.rep()[i];
  }
  for (int cl = threadIdx.x; cl < ncls; cl += blockDim.x) {
    const int64_t d = dlt[T.acc_field[abase + (int)sct.rep()[cl]]];
    const int64_t s0 = sct.start()[cl], m = sct.cnt()[cl];
    for (int64_t q = 0; q < m; ++q) dct.pts()[s0 + q] = sct.pts()[s0 + q] + d;
  }
}

// dynamic shared memory of k_plan_follow: a follower that computes its own
// plan (setup_one) or the TMA staging buffer (Geo / coefficient row)
static size_t follow_smem(int max_acc) {
  const size_t tma = std::max(sizeof(Geo), (size_t)max_acc * 64) + 16;
  const size_t need = std::max(setup_smem(max_acc), tma);
  static size_t attr = 0;
  if (need > 48 * 1024 && need > attr) {
    cudaFuncSetAttribute(k_plan_follow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    attr = need;
  }
  return need;
}

void launch_setup(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs,
                  int64_t n, const gvo_sampling& smp, int64_t* d_coefs, Geo* d_geos, int64_t* d_ctabs,
                  cudaStream_t st, const int32_t* d_mclass, const PlanShare* share) {
  if (n <= 0) return;
  PlanShare PS{};
  if (share && share->table && d_mclass) {
    PS = *share;
    k_plan_key<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(T, d_mclass, d_cfgs, n, PS);
  }
  k_setup<<<(unsigned)n, 256, setup_smem(T.max_acc), st>>>(T, d_machines, d_cfgs, n, smp, d_coefs, d_geos, d_ctabs,
                                                           PS);
  if (PS.src) {
    k_plan_follow<<<(unsigned)n, 256, follow_smem(T.max_acc), st>>>(T, d_machines, d_cfgs, n, smp, d_coefs, d_geos,
                                                                    d_ctabs, PS, 0);
    if (!PS.defer_rows)
      k_plan_follow<<<(unsigned)n, 256, follow_smem(T.max_acc), st>>>(T, d_machines, d_cfgs, n, smp, d_coefs, d_geos,
                                                                      d_ctabs, PS, 1);
  }
}

void launch_plan_rows(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs, int64_t n,
                      const gvo_sampling& smp, int64_t* d_coefs, Geo* d_geos, int64_t* d_ctabs, const PlanShare& PS,
                      cudaStream_t st) {
  if (n > 0 && PS.src)
    k_plan_follow<<<(unsigned)n, 256, follow_smem(T.max_acc), st>>>(T, d_machines, d_cfgs, n, smp, d_coefs, d_geos,
                                                                    d_ctabs, PS, 1);
}

__global__ void k_classes_only(TplView T, const gvo_config* cfgs, int64_t n, const int64_t* coefs,
                               int64_t* ctabs) {
  const int64_t c = blockIdx.x;
  if (c >= n) return;
  extern __shared__ int16_t sh_rep2[];
  build_classes_cta(T, cfgs[c].template_id, coefs + c * (int64_t)T.max_acc * 8,
                    CTab{ctabs + c * ctab_stride(T.max_acc), T.max_acc}, sh_rep2, sh_rep2 + ((T.max_acc + 1) & ~1));
}

void launch_classes(const TplView& T, const gvo_config* d_cfgs, int64_t n, const int64_t* d_coefs,
                    int64_t* d_ctabs, cudaStream_t st) {
  if (n > 0)
    k_classes_only<<<(unsigned)n, 128, setup_smem(T.max_acc), st>>>(T, d_cfgs, n, d_coefs, d_ctabs);
}

}  // namespace gvo
