// k_sets.cu — exact unique-granule counting for blocks and waves.
//
// Replaces the reference's set machinery: GranuleSet/_SetBuilder bitmaps and
// sorted-unique arrays (footprint.py:141-227), grid_iteration's unique
// counts (footprint.py:441-471), wave_footprint / overlap_bytes
// (footprint.py:535-584) and the unique counts of sample_block_stats /
// sample_wave_stats (volumes.py:152-250).
//
// Instead of materialising every address, each (access, block box) is an
// affine image of a box of thread/block coordinates.  Its dimensions are
// collapsed like a strided tensor (contiguous strides merge), the innermost
// dimensions whose gaps never exceed one granule fold into a byte "span",
// and accesses that differ only by a translation along a remaining
// dimension (stencil rays) or by less than span+granule (clusters) merge
// into one lattice.  Each lattice point then contributes one granule
// INTERVAL.  All intervals of a unit (one field of one block, or one field
// over all sampled waves, loads and stores tagged separately) are radix
// sorted by their first granule in shared memory (or a per-CTA global slab
// when they do not fit) and every requested union / intersection count is
// a tagged prefix-max sweep.  Every step is an exact set identity; no
// address sampling, no hashing.
#include "gvo_bytecode.cuh"
#include "gvo_kernels.h"
#include "gvo_warp.cuh"
#if defined(GVO_DEBUG_SYNC) && GVO_DEBUG_SYNC
#include <cstdio>
#endif

// residency of this build of the set kernel (k_sets1.cu includes this file
// with 1); each residency lives in its own namespace
#ifndef GVO_SETS_CTAS_PER_SM
#define GVO_SETS_CTAS_PER_SM 2
#endif
#if GVO_SETS_CTAS_PER_SM == 1
#define GVO_SETS_NS sets1
#else
#define GVO_SETS_NS sets2
#endif

namespace gvo {
namespace GVO_SETS_NS {
// the small-batch residency's shape can be overridden for experiments
// (GVO_SETS2_CTAS / GVO_SETS2_NT, e.g. 4 x 256)
#if GVO_SETS_CTAS_PER_SM != 1 && defined(GVO_SETS2_CTAS)
constexpr int kSetsCtasPerSm = GVO_SETS2_CTAS;
#else
constexpr int kSetsCtasPerSm = GVO_SETS_CTAS_PER_SM;
#endif
#if GVO_SETS_CTAS_PER_SM != 1 && defined(GVO_SETS2_SMEM_KB)
constexpr int kSetsSmemBytes = GVO_SETS2_SMEM_KB * 1024;  // experiment: leave more of the SM's 256 KB to L1
#else
constexpr int kSetsSmemBytes = kSetsCtasPerSm == 1 ? 222 * 1024 : kSetsCtasPerSm == 2 ? 110 * 1024 : 54 * 1024;
#endif

// per-CTA phase accounting for tools/unit_profile.py (build with
// GVO_PHASE_STATS=1); compiled out of the product kernel
#if defined(GVO_PHASE_STATS) && GVO_PHASE_STATS
#define GVO_PH(...) __VA_ARGS__
#else
#define GVO_PH(...)
#endif
#if defined(GVO_PHASE_STATS) && GVO_PHASE_STATS && !(defined(GVO_BM_PROF) && GVO_BM_PROF)
#define GVO_PHN(...) __VA_ARGS__  // slots 12..15 (segment counters, run-building split) unless GVO_BM_PROF
#else
#define GVO_PHN(...)
#endif

// out-of-line set-engine stages (own register allocation, fewer spills in
// the monolithic kernel); GVO_HOT_NOINLINE=0 inlines them (A/B builds)
#ifndef GVO_HOT_NOINLINE
#define GVO_HOT_NOINLINE 1
#endif
#if GVO_HOT_NOINLINE
#define GVO_NOINL __noinline__
#else
#define GVO_NOINL
#endif
// Instruction footprint: the kernel is one ~1.5 MB SASS image and
// instruction-fetch stalls were 18 % of its warp samples (ncu, C5).  Device
// functions inlined at several call sites are kept as one out-of-line copy
// where that measured faster; GVO_OUTLINE is a bit mask (A/B builds):
//   1 wl_emit_lattice (3 call sites in cover_warp; C5 sample -11 %),
//   2 box_lattice, 4 wl_emit_normalized, 8 run_interval, 16 wl_normalize
//   (each within +-2 % or slower), 32 run_base's dimension loop not unrolled
//   (-2.6 %), 64 bytecode evaluator / interval guard out of line
//   (gvo_bytecode.cuh; +0.5 %), 128 wl_normalize's loops not unrolled (-2.4 %)
//   256 the other WLat emission loops not unrolled (-1.5 %), 512
//   cover_segments' loops (neutral)
#ifndef GVO_OUTLINE
#define GVO_OUTLINE 417
#endif
#if GVO_OUTLINE & 1
#define GVO_OL_EMIT __noinline__
#else
#define GVO_OL_EMIT __forceinline__
#endif
#if GVO_OUTLINE & 2
#define GVO_OL_BOX __noinline__
#else
#define GVO_OL_BOX inline
#endif
#if GVO_OUTLINE & 4
#define GVO_OL_EMITN __noinline__
#else
#define GVO_OL_EMITN __forceinline__
#endif
#if GVO_OUTLINE & 8
#define GVO_OL_RIV __noinline__
#else
#define GVO_OL_RIV __forceinline__
#endif
#if GVO_OUTLINE & 16
#define GVO_OL_NORM __noinline__
#else
#define GVO_OL_NORM __forceinline__
#endif

// threads per CTA.  2 CTAs/SM: 320 threads (96 registers; A/B on C2:
// 320 > 384 > 256 > 512, the 64-register build spills its stack to DRAM);
// 1 CTA/SM: 512 (128 registers).
#ifndef GVO_SETS2_NT
#define GVO_SETS2_NT 320
#endif
#ifndef GVO_SETS1_NT
#define GVO_SETS1_NT 512
#endif
#if GVO_SETS_CTAS_PER_SM != 1
constexpr int kNT = GVO_SETS2_NT;
#else
constexpr int kNT = GVO_SETS1_NT;
#endif
constexpr int kNW = kNT / 32;
constexpr int kMaxSrc = 64;        // sources per unit
constexpr int kMaxSub = 72;        // subsets per unit
constexpr int kSmemRuns = 1024;    // run offsets kept in shared memory
constexpr int kClassPts = 64;      // points per coefficient class chunk

struct UnitSh {
  int64_t cfg;
  int field;
  int kind;      // 0 block sample, 1 waves, 2 custom footprint
  int j;         // sample index (kind 0)
  int n_src;
  int64_t src_start[kMaxSrc], src_count[kMaxSrc];
  int src_kind[kMaxSrc], src_tag[kMaxSrc];
  int n_sub;
  uint32_t sub_mask[kMaxSub];
  int64_t sub_r[kMaxSub];
  int sub_sh[kMaxSub];      // log2(sub_r) when a power of two, else -1
  int64_t sub_val[kMaxSub];
  uint32_t sub_cm[kMaxSub];  // bitmap tier: subset masks over the compact tags
  int64_t g, R;
  int status;
  int n_runs;
  int64_t key_lo, key_hi;  // granule bounds over all runs
  int64_t N;
  int has_pattern;          // pattern runs present: bitmap tier only
};

// ------------------------------------------------------------------ lattice
// A lattice of addresses base + sum_d st_d * k_d (k_d < ex_d) with an inner
// granule-contiguous byte span.  Two register-resident forms, so that no
// lattice ever lives in local memory (a per-thread array indexed by a
// runtime dimension would, and under a 2x110 KB shared-memory carve-out the
// L1 cannot hold the stacks of 640 threads: the previous per-thread form
// moved ~190 MB of stack through DRAM per C2 launch):
//  * WLat — held by a whole warp, lane d < nd holding dimension d; every
//    step (normalise, split, emit) is warp-cooperative with shuffles.  Used
//    for the box lattices and the translate covers (a handful of lattices
//    per task, emitted one after another by the warp);
//  * Lat4 — per lane, at most kSegDims dimensions, every loop unrolled with
//    compile-time indices.  Used by the segment cover, whose lanes emit one
//    segment box each.
constexpr unsigned kFull = 0xffffffffu;
constexpr int kSegDims = 4;

struct WLat {
  int64_t base;   // warp-uniform
  uint64_t span;  // warp-uniform
  int nd;         // warp-uniform
  uint64_t st;    // lane d < nd: stride of dimension d (0 elsewhere)
  int64_t ex;     // lane d < nd: extent of dimension d (1 elsewhere)
};

struct Lat4 {
  int64_t base;
  uint64_t span;
  int nd;
  uint64_t st[kSegDims];
  int64_t ex[kSegDims];
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Merge dims whose union is again an arithmetic progression (sorted by
// stride, st_j % st_i == 0 && st_j / st_i <= ex_i), then fold the leading
// dims whose point gaps stay <= g into the granule-contiguous span.
// Warp-cooperative; dims with ex <= 1 or st == 0 are dropped.
__device__ GVO_OL_NORM void wl_normalize(WLat& L, int64_t g) {
  const int lane = threadIdx.x & 31;
  const bool keep = lane < L.nd && L.ex > 1 && L.st != 0;
  const unsigned kmask = __ballot_sync(kFull, keep);
  // rank among kept dims by (stride, dim)
  int r = 0;
#if GVO_OUTLINE & 128
#pragma unroll 1
#endif
  for (int j = 0; j < L.nd; ++j) {
    const uint64_t sj = __shfl_sync(kFull, L.st, j);
    r += ((kmask >> j) & 1u) && (sj < L.st || (sj == L.st && j < lane));
  }
  uint64_t s2 = 0;
  int64_t e2 = 1;
#if GVO_OUTLINE & 128
#pragma unroll 1
#endif
  for (int j = 0; j < L.nd; ++j) {
    const int rj = __shfl_sync(kFull, r, j);
    const uint64_t sj = __shfl_sync(kFull, L.st, j);
    const int64_t ej = __shfl_sync(kFull, L.ex, j);
    if (((kmask >> j) & 1u) && rj == lane) { s2 = sj; e2 = ej; }
  }
  const int m = __popc(kmask);
  uint64_t so = 0;
  int64_t eo = 1;
  int o = 0;
#if GVO_OUTLINE & 128
#pragma unroll 1
#endif
  for (int i = 0; i < m; ++i) {
    const uint64_t si = __shfl_sync(kFull, s2, i);
    const int64_t ei = __shfl_sync(kFull, e2, i);
    if (o > 0) {
      const uint64_t sc = __shfl_sync(kFull, so, o - 1);
      const int64_t sn = __shfl_sync(kFull, eo, o - 1);
      if (si % sc == 0 && si / sc <= (uint64_t)sn) {
        if (lane == o - 1) eo = sn + (int64_t)(si / sc) * (ei - 1);
        continue;
      }
    }
    if (lane == o) { so = si; eo = ei; }
    ++o;
  }
  uint64_t span = L.span;
  int k = 0;
  while (k < o) {
    const uint64_t sk = __shfl_sync(kFull, so, k);
    const int64_t ek = __shfl_sync(kFull, eo, k);
    if ((unsigned __int128)sk > (unsigned __int128)span + (uint64_t)g) break;
    span += sk * (uint64_t)(ek - 1);
    ++k;
  }
  const uint64_t s3 = __shfl_sync(kFull, so, (lane + k) & 31);
  const int64_t e3 = __shfl_sync(kFull, eo, (lane + k) & 31);
  L.nd = o - k;
  L.span = span;
  L.st = lane < L.nd ? s3 : 0;
  L.ex = lane < L.nd ? e3 : 1;
}

__device__ inline bool contains(const int64_t* P, int n, int64_t v) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    if (P[mid] == v) return true;
    if (P[mid] < v) lo = mid + 1; else hi = mid - 1;
  }
  return false;
}

struct RunSink {
  Run* runs;
  int cap;
  int* n_runs;
  int* status;
  int64_t* key_lo;
  int64_t* key_hi;
  int* has_pattern = nullptr;  // set when a pattern run is emitted (bitmap tier only)
};

// Emit normalised lattices that share their dims (held by the warp) and
// differ in their base: one run per active lane (`act`, this lane's base
// `b`).  Warp-cooperative: one slot reservation, the dims written by the
// lanes that hold them.
__device__ GVO_OL_EMITN void wl_emit_normalized(const RunSink& S, const WLat& L, int64_t b, bool act, int tag,
                                                const Granule& G) {
  const int lane = threadIdx.x & 31;
  int64_t count = 1;
  uint64_t ext_span = L.span;
  bool over = false;
  bool mono = true;
  unsigned __int128 reach = (unsigned __int128)L.span;
#if GVO_OUTLINE & 256
  #pragma unroll 1
#endif
  for (int d = 0; d < L.nd; ++d) {
    const uint64_t sd = __shfl_sync(kFull, L.st, d);
    const int64_t ed = __shfl_sync(kFull, L.ex, d);
    if (count > (int64_t(1) << 40) / ed) over = true;
    else count *= ed;
    ext_span += sd * (uint64_t)(ed - 1);
    if (d > 0 && (unsigned __int128)sd <= reach) mono = false;
    reach += (unsigned __int128)sd * (uint64_t)(ed - 1);
  }
  const unsigned am = __ballot_sync(kFull, act);
  if (!am) return;
  if (over) {
    if (lane == 0) atomicExch(S.status, GVO_ERR_CAPACITY);
    return;
  }
  const int64_t len = (int64_t)(L.span / (uint64_t)G.g) + 2;
  const int64_t pieces = (len + kPiece - 1) / kPiece;
  mono = mono && pieces == 1;
  int slot0 = 0;
  if (lane == 0) slot0 = atomicAdd(S.n_runs, __popc(am));
  slot0 = __shfl_sync(kFull, slot0, 0);
  if (slot0 + __popc(am) > S.cap) {
    if (lane == 0) atomicExch(S.status, GVO_ERR_CAPACITY);
    return;
  }
  if (act) {
    Run* r = S.runs + slot0 + __popc(am & lanemask_lt());
    r->base = b;
    r->span = L.span;
    r->nd = L.nd;
    r->tag = tag;
    r->kind = 0;
    r->access = -1;
    r->pieces = pieces;
    r->count = count * pieces;
    r->mono = mono ? 1 : 0;
    r->run_start = r->run_count = 0;
  }
  // dims: lanes d < kMaxDims write dimension d of every emitted run
  for (int q = 0; q < __popc(am); ++q) {
    Run* r = S.runs + slot0 + q;
    if (lane < kMaxDims) {
      r->stride[lane] = lane < L.nd ? (int64_t)L.st : 0;
      r->ext[lane] = lane < L.nd ? L.ex : 1;
    }
  }
  // key bounds: warp min/max, one atomic each
  long long lo = act ? (long long)G.of(b) : LLONG_MAX;
  long long hi = act ? (long long)G.of((int64_t)((uint64_t)b + ext_span)) : LLONG_MIN;
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFull, lo, o));
    hi = max(hi, __shfl_xor_sync(kFull, hi, o));
  }
  if (lane == 0) {
    atomicMin((long long*)S.key_lo, lo);
    atomicMax((long long*)S.key_hi, hi);
  }
}

// Normalise, then split off the dimensions that interleave with faster
// ones (a stride not beyond the reach of the kept faster dimensions, e.g. a
// translate pair 192 B apart on a 120 B-stride row): the sub-lattices over
// the remaining dimensions are monotone, so key ranges can bisect them
// instead of scanning.  Splitting is bounded (<= 64 sub-lattices, emitted
// by the lanes in parallel); beyond that the lattice is emitted as one
// non-monotone run.  Warp-cooperative.
__device__ GVO_OL_EMIT void wl_emit_lattice(const RunSink& S, WLat L, int tag, const Granule& G) {
  const int lane = threadIdx.x & 31;
  wl_normalize(L, G.g);
  unsigned smask = 0;
  int64_t combos = 1;
  {
    unsigned __int128 reach = (unsigned __int128)L.span;
#if GVO_OUTLINE & 256
    #pragma unroll 1
#endif
    for (int d = 0; d < L.nd; ++d) {
      const uint64_t sd = __shfl_sync(kFull, L.st, d);
      const int64_t ed = __shfl_sync(kFull, L.ex, d);
      if (d > 0 && (unsigned __int128)sd <= reach) {
        smask |= 1u << d;
        combos = combos > 64 || ed > 64 ? 65 : combos * ed;
      } else {
        reach += (unsigned __int128)sd * (uint64_t)(ed - 1);
      }
    }
  }
  if (smask == 0 || combos > 64) {
    wl_emit_normalized(S, L, L.base, lane == 0, tag, G);
    return;
  }
  // K: the kept dims, compacted
  const unsigned ndmask = L.nd >= 32 ? kFull : ((1u << L.nd) - 1u);
  const unsigned kept = ndmask & ~smask;
  WLat K;
  K.span = L.span;
  K.nd = __popc(kept);
  K.base = L.base;
  K.st = 0;
  K.ex = 1;
#if GVO_OUTLINE & 256
  #pragma unroll 1
#endif
  for (int d = 0; d < L.nd; ++d) {
    const uint64_t sd = __shfl_sync(kFull, L.st, d);
    const int64_t ed = __shfl_sync(kFull, L.ex, d);
    if (((kept >> d) & 1u) && __popc(kept & ((1u << d) - 1u)) == lane) { K.st = sd; K.ex = ed; }
  }
  // sub-lattice m: base + sum over split dims (ascending) of st_d * digit_d(m)
  for (int m0 = 0; m0 < combos; m0 += 32) {
    const int m = m0 + lane;
    int64_t r = m;
    uint64_t b = (uint64_t)L.base;
#if GVO_OUTLINE & 256
    #pragma unroll 1
#endif
    for (int d = 0; d < L.nd; ++d) {
      const uint64_t sd = __shfl_sync(kFull, L.st, d);
      const int64_t ed = __shfl_sync(kFull, L.ex, d);
      if ((smask >> d) & 1u) {
        b += sd * (uint64_t)(r % ed);
        r /= ed;
      }
    }
    wl_emit_normalized(S, K, (int64_t)b, m < combos, tag, G);
  }
}

// ---- per-lane lattices of at most kSegDims dims (segment boxes)
// every loop over dims has compile-time bounds and indices: registers only
__device__ __forceinline__ void l4_cswap(uint64_t& sa, int64_t& ea, uint64_t& sb, int64_t& eb) {
  if (sb < sa) {
    const uint64_t ts = sa; sa = sb; sb = ts;
    const int64_t te = ea; ea = eb; eb = te;
  }
}

__device__ __forceinline__ void l4_normalize(Lat4& L, int64_t g) {
  uint64_t s[kSegDims];
  int64_t e[kSegDims];
#pragma unroll
  for (int d = 0; d < kSegDims; ++d) {
    const bool ok = d < L.nd && L.ex[d] > 1 && L.st[d] != 0;
    s[d] = ok ? L.st[d] : ~0ull;  // dropped dims sort last
    e[d] = ok ? L.ex[d] : 1;
  }
  l4_cswap(s[0], e[0], s[1], e[1]);
  l4_cswap(s[2], e[2], s[3], e[3]);
  l4_cswap(s[0], e[0], s[2], e[2]);
  l4_cswap(s[1], e[1], s[3], e[3]);
  l4_cswap(s[1], e[1], s[2], e[2]);
  uint64_t os[kSegDims];
  int64_t oe[kSegDims];
#pragma unroll
  for (int d = 0; d < kSegDims; ++d) { os[d] = 0; oe[d] = 1; }
  int m = 0;
  uint64_t sc = 0;
  int64_t sn = 1;
  bool have = false;
#pragma unroll
  for (int i = 0; i < kSegDims; ++i) {
    if (s[i] == ~0ull) continue;
    if (have && s[i] % sc == 0 && s[i] / sc <= (uint64_t)sn) {
      sn = sn + (int64_t)(s[i] / sc) * (e[i] - 1);
      continue;
    }
    if (have) {
#pragma unroll
      for (int j = 0; j < kSegDims; ++j)
        if (j == m) { os[j] = sc; oe[j] = sn; }
      ++m;
    }
    sc = s[i];
    sn = e[i];
    have = true;
  }
  if (have) {
#pragma unroll
    for (int j = 0; j < kSegDims; ++j)
      if (j == m) { os[j] = sc; oe[j] = sn; }
    ++m;
  }
  uint64_t span = L.span;
  int k = 0;
  bool stop = false;
#pragma unroll
  for (int j = 0; j < kSegDims; ++j) {
    if (!stop && j < m && (unsigned __int128)os[j] <= (unsigned __int128)span + (uint64_t)g) {
      span += os[j] * (uint64_t)(oe[j] - 1);
      k = j + 1;
    } else {
      stop = true;
    }
  }
  L.span = span;
  L.nd = m - k;
#pragma unroll
  for (int j = 0; j < kSegDims; ++j) {
    uint64_t sv = 0;
    int64_t ev = 1;
#pragma unroll
    for (int q = 0; q < kSegDims; ++q)
      if (q == j + k) { sv = os[q]; ev = oe[q]; }
    L.st[j] = j < L.nd ? sv : 0;
    L.ex[j] = j < L.nd ? ev : 1;
  }
}

__device__ __forceinline__ void l4_emit_normalized(const RunSink& S, const Lat4& L, int tag, const Granule& G) {
  int64_t count = 1;
  uint64_t ext_span = L.span;
  bool mono = true;
  unsigned __int128 reach = (unsigned __int128)L.span;
#pragma unroll
  for (int d = 0; d < kSegDims; ++d) {
    if (d >= L.nd) continue;
    if (count > (int64_t(1) << 40) / L.ex[d]) { atomicExch(S.status, GVO_ERR_CAPACITY); return; }
    count *= L.ex[d];
    ext_span += L.st[d] * (uint64_t)(L.ex[d] - 1);
    if (d > 0 && (unsigned __int128)L.st[d] <= reach) mono = false;
    reach += (unsigned __int128)L.st[d] * (uint64_t)(L.ex[d] - 1);
  }
  const int64_t len = (int64_t)(L.span / (uint64_t)G.g) + 2;
  const int64_t pieces = (len + kPiece - 1) / kPiece;
  const int slot = atomicAdd(S.n_runs, 1);
  if (slot >= S.cap) { atomicExch(S.status, GVO_ERR_CAPACITY); return; }
  Run* r = S.runs + slot;  // written field by field (no local struct copy)
  r->base = L.base;
  r->span = L.span;
  r->nd = L.nd;
#pragma unroll
  for (int d = 0; d < kMaxDims; ++d) {
    r->stride[d] = d < kSegDims && d < L.nd ? (int64_t)L.st[d < kSegDims ? d : 0] : 0;
    r->ext[d] = d < kSegDims && d < L.nd ? L.ex[d < kSegDims ? d : 0] : 1;
  }
  r->tag = tag;
  r->kind = 0;
  r->access = -1;
  r->pieces = pieces;
  r->count = count * pieces;
  r->mono = mono && pieces == 1 ? 1 : 0;
  r->run_start = r->run_count = 0;
  atomicMin((long long*)S.key_lo, (long long)G.of(L.base));
  atomicMax((long long*)S.key_hi, (long long)G.of((int64_t)((uint64_t)L.base + ext_span)));
}

// per-lane twin of wl_emit_lattice
__device__ __forceinline__ void l4_emit_lattice(const RunSink& S, Lat4 L, int tag, const Granule& G) {
  l4_normalize(L, G.g);
  unsigned smask = 0;
  int64_t combos = 1;
  {
    unsigned __int128 reach = (unsigned __int128)L.span;
#pragma unroll
    for (int d = 0; d < kSegDims; ++d) {
      if (d >= L.nd) continue;
      if (d > 0 && (unsigned __int128)L.st[d] <= reach) {
        smask |= 1u << d;
        combos = combos > 64 || L.ex[d] > 64 ? 65 : combos * L.ex[d];
      } else {
        reach += (unsigned __int128)L.st[d] * (uint64_t)(L.ex[d] - 1);
      }
    }
  }
  if (smask == 0 || combos > 64) { l4_emit_normalized(S, L, tag, G); return; }
  Lat4 K;
  K.span = L.span;
  K.nd = 0;
#pragma unroll
  for (int j = 0; j < kSegDims; ++j) { K.st[j] = 0; K.ex[j] = 1; }
#pragma unroll
  for (int d = 0; d < kSegDims; ++d) {
    if (d >= L.nd || ((smask >> d) & 1u)) continue;
#pragma unroll
    for (int j = 0; j < kSegDims; ++j)
      if (j == K.nd) { K.st[j] = L.st[d]; K.ex[j] = L.ex[d]; }
    ++K.nd;
  }
  for (int64_t m = 0; m < combos; ++m) {
    int64_t r = m;
    uint64_t b = (uint64_t)L.base;
#pragma unroll
    for (int d = 0; d < kSegDims; ++d) {
      if (!((smask >> d) & 1u)) continue;
      b += L.st[d] * (uint64_t)(r % L.ex[d]);
      r /= L.ex[d];
    }
    K.base = (int64_t)b;
    l4_emit_normalized(S, K, tag, G);
  }
}

// Pattern run (Run::kind 2): rows of cells along a stride s0 in which every
// cell holds the same set of residue words {t*dg : bit t of pm}: one element
// per row, its interval spans the row, and the bitmap tier sets the row's
// sectors from the periodic per-period pattern (lcm(s0, g) / g sectors) word
// by word instead of one interval per cell and residue cluster.  Returns
// false (nothing emitted) when the rows would not be monotone.  Per lane.
constexpr int64_t kPatMinCells = 32;
__device__ inline int64_t gcd64(int64_t a, int64_t b);
__device__ __forceinline__ uint32_t pattern_bits(int64_t cell0, uint64_t pm, int64_t dg, int64_t s0, int64_t P,
                                                 int64_t nph, int64_t g, int shift, int part, int nparts);
__device__ inline bool emit_pattern(const RunSink& S, const Lat4& Lbox, uint64_t cell0, int tag, const Granule& G,
                                    uint64_t pm, int64_t dg, int64_t s0) {
  int64_t n0 = Lbox.ex[0];
  // outer dims (rows) with ex > 1, sorted by stride (rank sort, static indices)
  uint64_t s[kSegDims - 1];
  int64_t e[kSegDims - 1];
#pragma unroll
  for (int d = 1; d < kSegDims; ++d) {
    const bool ok = d < Lbox.nd && Lbox.ex[d] > 1;
    s[d - 1] = ok ? Lbox.st[d] : ~0ull;
    e[d - 1] = ok ? Lbox.ex[d] : 1;
  }
  l4_cswap(s[0], e[0], s[1], e[1]);
  l4_cswap(s[1], e[1], s[2], e[2]);
  l4_cswap(s[0], e[0], s[1], e[1]);
  int nd = 0;
#pragma unroll
  for (int d = 0; d < kSegDims - 1; ++d) nd += s[d] != ~0ull;
  // rows that continue the cell sequence merge into n0
  int k = 0;
#pragma unroll
  for (int d = 0; d < kSegDims - 1; ++d) {
    if (k == d && d < nd && s[d] == (uint64_t)(n0 * s0)) { n0 *= e[d]; ++k; }
  }
  uint64_t rs[kSegDims - 1];
  int64_t re[kSegDims - 1];
#pragma unroll
  for (int j = 0; j < kSegDims - 1; ++j) {
    rs[j] = 0; re[j] = 1;
#pragma unroll
    for (int q = 0; q < kSegDims - 1; ++q)
      if (q == j + k) { rs[j] = s[q]; re[j] = e[q]; }
  }
  nd -= k;
  if (n0 >= (int64_t(1) << 31)) return false;
  const int64_t rmin = (int64_t)__ffsll((long long)pm) - 1, rmax = 63 - __clzll((long long)pm);
  const uint64_t span = (uint64_t)((n0 - 1) * s0 + (rmax - rmin) * dg);
  unsigned __int128 reach = span;
  int64_t count = 1;
  uint64_t ext_span = span;
#pragma unroll
  for (int d = 0; d < kSegDims - 1; ++d) {
    if (d >= nd) continue;
    if ((unsigned __int128)rs[d] <= reach) return false;  // rows must be monotone
    reach += (unsigned __int128)rs[d] * (uint64_t)(re[d] - 1);
    if (count > (int64_t(1) << 40) / re[d]) return false;
    count *= re[d];
    ext_span += rs[d] * (uint64_t)(re[d] - 1);
  }
  const int slot = atomicAdd(S.n_runs, 1);
  if (slot >= S.cap) { atomicExch(S.status, GVO_ERR_CAPACITY); return true; }
  const uint64_t base = cell0 + (uint64_t)(rmin * dg);
  Run* r = S.runs + slot;
  r->base = (int64_t)base;
  r->span = span;
  r->nd = nd;
#pragma unroll
  for (int d = 0; d < kMaxDims; ++d) {
    r->stride[d] = d < kSegDims - 1 && d < nd ? (int64_t)rs[d < kSegDims - 1 ? d : 0] : 0;
    r->ext[d] = d < kSegDims - 1 && d < nd ? re[d < kSegDims - 1 ? d : 0] : 1;
  }
  r->tag = tag;
  r->kind = 2;
  r->access = (int32_t)n0;       // cells per row
  r->pad_ = (int32_t)dg;         // residue unit (bytes)
  r->run_start = (int64_t)pm;    // residues present, in units of dg
  r->run_count = s0;             // cell stride (bytes)
  r->mono = 1;
  {  // period pattern of rows with this run's phase (cell0 mod g), kept in `pieces`
    const int64_t gc = gcd64(s0, G.g);
    const int64_t ph = floormod((int64_t)cell0, G.g);
    const uint32_t pat = pattern_bits((int64_t)cell0, pm, dg, s0, s0 / gc, G.g / gc, G.g, G.shift, 0, 1);
    r->pieces = (int64_t)(((uint64_t)ph << 32) | pat);
  }
  r->count = count;
  atomicMin((long long*)S.key_lo, (long long)G.of((int64_t)base));
  atomicMax((long long*)S.key_hi, (long long)G.of((int64_t)(base + ext_span)));
  if (S.has_pattern) atomicExch(S.has_pattern, 1);
  return true;
}

__device__ inline int64_t gcd64(int64_t a, int64_t b) {  // a, b >= 0
  while (b) { const int64_t t = a % b; a = b; b = t; }
  return a;
}

// Maximal ray from translate i along stride s: members (bitmask over P) and
// length.  P sorted and unique.
__device__ __forceinline__ int ray_from(const int64_t* P, int n, int i, int64_t s, uint64_t* mem_out) {
  uint64_t mem = 1ull << i;
  int len = 1, pos = i;
  while (pos + 1 < n) {
    // the successor v + s, if present, is after pos
    const int64_t t = P[pos] + s;
    int lo = pos + 1, hi = n - 1, f = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if (P[mid] == t) { f = mid; break; }
      if (P[mid] < t) lo = mid + 1; else hi = mid - 1;
    }
    if (f < 0) break;
    mem |= 1ull << f;
    ++len;
    pos = f;
  }
  *mem_out = mem;
  return len;
}

// Translate cover of one coefficient class: the class's translates P[0..n)
// (n <= 64, sorted, unique) live in shared memory.  Rays of one dimension
// are disjoint (every point starts or continues exactly one maximal ray
// along that stride), so all rays of a dimension are judged in parallel
// (lane per translate) against the points not yet covered by larger-stride
// rays; the warp then emits them one after another.
__device__ GVO_NOINL void cover_warp(const RunSink& S, const WLat& L0, const int64_t* P, int n, int tag,
                                     const Granule& G) {
  const int lane = threadIdx.x & 31;
  uint64_t req = n >= 64 ? ~0ull : ((1ull << n) - 1);
  for (int d = L0.nd - 1; d >= 0 && req; --d) {
    const int64_t s = (int64_t)__shfl_sync(kFull, L0.st, d);
    uint64_t clear = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      bool ray = false;
      int len = 0;
      uint64_t mem = 0;
      if (i < n && !contains(P, n, P[i] - s)) {  // a ray start
        len = ray_from(P, n, i, s, &mem);
        ray = len >= 2 && __popcll(mem & req) >= 2;
      }
      if (ray) clear |= mem;
      for (unsigned rm = __ballot_sync(kFull, ray); rm; rm &= rm - 1) {
        const int src = __ffs(rm) - 1;
        WLat L = L0;
        L.base = __shfl_sync(kFull, i < n ? P[i < n ? i : 0] : 0, src);
        const int ln = __shfl_sync(kFull, len, src);
        if (lane == d) L.ex += ln - 1;
        wl_emit_lattice(S, L, tag, G);
      }
    }
    const unsigned lo32 = __reduce_or_sync(kFull, (unsigned)clear);
    const unsigned hi32 = __reduce_or_sync(kFull, (unsigned)(clear >> 32));
    req &= ~(((uint64_t)hi32 << 32) | lo32);
  }
  // rays along a stride that is not a lattice dimension (e.g. +-z offsets of
  // a one-layer block): the smallest gap between consecutive uncovered
  // translates, if wider than span + g, becomes an added dimension
  const unsigned __int128 tol0 = (unsigned __int128)L0.span + (uint64_t)G.g;
  for (int iter = 0; iter < 3 && __popcll(req) >= 2 && L0.nd < kMaxDims; ++iter) {
    int64_t gap = INT64_MAX;
    for (int i = lane; i < n; i += 32) {
      if (!((req >> i) & 1ull)) continue;
      int k = i + 1;
      while (k < n && !((req >> k) & 1ull)) ++k;
      if (k < n) gap = min(gap, P[k] - P[i]);
    }
    for (int o = 16; o; o >>= 1) gap = min(gap, __shfl_xor_sync(kFull, gap, o));
    if (gap == INT64_MAX || (unsigned __int128)(uint64_t)gap <= tol0) break;
    uint64_t clear = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      bool ray = false;
      int len = 0;
      uint64_t mem = 0;
      if (i < n && !contains(P, n, P[i] - gap)) {
        len = ray_from(P, n, i, gap, &mem);
        ray = len >= 2 && __popcll(mem & req) >= 2;
      }
      if (ray) clear |= mem;
      for (unsigned rm = __ballot_sync(kFull, ray); rm; rm &= rm - 1) {
        const int src = __ffs(rm) - 1;
        WLat L = L0;
        L.base = __shfl_sync(kFull, i < n ? P[i < n ? i : 0] : 0, src);
        const int ln = __shfl_sync(kFull, len, src);
        if (lane == L0.nd) { L.st = (uint64_t)gap; L.ex = ln; }
        L.nd = L0.nd + 1;
        wl_emit_lattice(S, L, tag, G);
      }
    }
    const unsigned lo32 = __reduce_or_sync(kFull, (unsigned)clear);
    const unsigned hi32 = __reduce_or_sync(kFull, (unsigned)(clear >> 32));
    const uint64_t cl = ((uint64_t)hi32 << 32) | lo32;
    if (!cl) break;
    req &= ~cl;
  }
  if (!req) return;
  // clusters: consecutive translates closer than span + g widen the span
  const unsigned __int128 tol = (unsigned __int128)L0.span + (uint64_t)G.g;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    bool start = false;
    int64_t width = 0;
    if (i < n && !(i > 0 && (unsigned __int128)(uint64_t)(P[i] - P[i - 1]) <= tol)) {
      int j = i;
      uint64_t mem = 1ull << i;
      while (j + 1 < n && (unsigned __int128)(uint64_t)(P[j + 1] - P[j]) <= tol) { ++j; mem |= 1ull << j; }
      start = (mem & req) != 0;
      width = P[j] - P[i];
    }
    for (unsigned rm = __ballot_sync(kFull, start); rm; rm &= rm - 1) {
      const int src = __ffs(rm) - 1;
      WLat L = L0;
      L.base = __shfl_sync(kFull, i < n ? P[i < n ? i : 0] : 0, src);
      L.span = L0.span + (uint64_t)__shfl_sync(kFull, width, src);
      wl_emit_lattice(S, L, tag, G);
    }
  }
}

// ------------------------------------------------------------------ segments
// Translates of a point lattice whose residues modulo the fastest stride
// tile whole cells (zyxf layouts: the Q components of a cell are adjacent
// words, and every pull load is the same lattice shifted by a neighbour
// cell).  cover_warp finds no rays or clusters there and each translate
// stays a lattice of points.  Instead: write every translate as
// residue + lattice-coordinate offset, so translate p covers the box
// B_p = prod_d [k_pd, k_pd + ex_d) with its residue.  The boundaries of all
// B_p cut coordinate space into segment boxes on which the set of present
// translates is fixed; their residues cluster into spans, and where every
// translate is present the cluster covers a whole cell, folds into the span
// and rows collapse into intervals.  Exact: the segment boxes partition the
// union of the B_p (any decomposition of the offsets is valid).
constexpr int kSegBpAll = 248;      // breakpoints over all dimensions (flat)
constexpr int kSegMaxBoxes = 4096;
constexpr int kSegScratch = 2688;   // bytes of per-warp scratch
#ifndef GVO_SEG_RUN_WEIGHT
#define GVO_SEG_RUN_WEIGHT 16
#endif
constexpr int64_t kSegRunWeight = GVO_SEG_RUN_WEIGHT;  // element-equivalents of one extra run (A/B on C3: 16 > 32 > 48 > 100)
struct SegScratch {
  uint64_t l0st[kSegDims];   // the class lattice's dims (read by any lane)
  int64_t l0ex[kSegDims];
  int32_t kv[kSegDims][64];  // offsets per dimension, by translate
  int32_t bpf[kSegBpAll];    // breakpoints, dimension d at boff[d]
  int32_t boff[kSegDims];
  int32_t rs[64];            // residues, sorted
  int32_t tmp[64];
  int32_t nb[kSegDims];
  uint8_t ord[64];           // sorted position -> translate
};
static_assert(sizeof(SegScratch) <= kSegScratch, "segment scratch");

__device__ __forceinline__ int64_t floordiv128(__int128 a, __int128 b, __int128* rem) {
  __int128 q = a / b;
  __int128 r = a - q * b;
  if (r != 0 && ((r < 0) != (b < 0))) { q -= 1; r += b; }
  *rem = r;
  return (int64_t)q;
}

// Returns false (nothing emitted) when the class is not of that shape or
// the segment plan is not cheaper than cover_warp's.
__device__ __noinline__ bool cover_segments(const RunSink& S, const WLat& L0, const int64_t* P, int n, int tag,
                               const Granule& G, SegScratch* sc, bool allow_pattern) {
  const int lane = threadIdx.x & 31;
  const int nd = L0.nd;
  if (nd < 1 || nd > kSegDims || n < 2 || n > 64) return false;
  const uint64_t s0 = __shfl_sync(kFull, L0.st, 0);
  if (s0 >= (uint64_t(1) << 30) || L0.span >= s0) return false;
  if (__any_sync(kFull, lane < nd && (L0.ex >= (int64_t(1) << 29) || L0.st >= (uint64_t(1) << 62)))) return false;
  __syncwarp();
  if (lane < kSegDims) {
    sc->l0st[lane] = lane < nd ? L0.st : 0;
    sc->l0ex[lane] = lane < nd ? L0.ex : 1;
  }
  __syncwarp();
  const int64_t tol = (int64_t)L0.span + G.g;
  if ((int64_t)n * tol < (int64_t)s0) return false;  // n residues cannot tile a cell
  {  // cheap screen: distinct residues mod s0 (one match per lane) must be able to tile it
    int distinct = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const bool v = i < n;
      const int64_t r = v ? floormod((int64_t)((uint64_t)P[i] - (uint64_t)L0.base), (int64_t)s0) : -1;
      const unsigned act = __ballot_sync(0xffffffffu, v);
      unsigned peers = 0;
      if (v) peers = __match_any_sync(act, (unsigned long long)r);
      distinct += __popc(__ballot_sync(0xffffffffu, v && (__ffs(peers) - 1) == lane));
    }
    if ((int64_t)distinct * tol < (int64_t)s0) return false;
  }
  // 1. offsets: round to nearest along the outer dims, floor along dim 0
  bool ok = true;
  for (int i = lane; i < n; i += 32) {
    const __int128 off0 = (__int128)P[i] - (__int128)L0.base;
    if (off0 > -(__int128(1) << 60) && off0 < (__int128(1) << 60)) {
      int64_t off = (int64_t)off0;  // strides < 2^62: no overflow below
      for (int d = nd - 1; d >= 1; --d) {
        const int64_t s = (int64_t)sc->l0st[d];
        const int64_t k = floordiv(off + s / 2, s);
        off -= k * s;
        if (k < -(int64_t(1) << 28) || k > (int64_t(1) << 28)) ok = false;
        sc->kv[d][i] = (int32_t)k;
      }
      const int64_t k0 = floordiv(off, (int64_t)s0);
      if (k0 < -(int64_t(1) << 28) || k0 > (int64_t(1) << 28)) ok = false;
      sc->kv[0][i] = (int32_t)k0;
      sc->tmp[i] = (int32_t)(off - k0 * (int64_t)s0);  // [0, s0)
    } else {
      __int128 off = off0, rem;
      for (int d = nd - 1; d >= 1; --d) {
        const __int128 s = (__int128)sc->l0st[d];
        const int64_t k = floordiv128(off + s / 2, s, &rem);
        off -= (__int128)k * s;
        if (k < -(int64_t(1) << 28) || k > (int64_t(1) << 28)) ok = false;
        sc->kv[d][i] = (int32_t)k;
      }
      const int64_t k0 = floordiv128(off, (__int128)s0, &rem);
      if (k0 < -(int64_t(1) << 28) || k0 > (int64_t(1) << 28)) ok = false;
      sc->kv[0][i] = (int32_t)k0;
      sc->tmp[i] = (int32_t)rem;  // [0, s0)
    }
  }
  if (!__all_sync(0xffffffffu, ok)) return false;
  __syncwarp();
  // 2. residues sorted (rank sort, ties by index); ord maps back
  {
    int32_t v[2];
    int rk[2];
    for (int t = 0; t < 2; ++t) {
      const int i = lane + 32 * t;
      rk[t] = -1;
      if (i < n) {
        v[t] = sc->tmp[i];
        int r = 0;
        for (int j = 0; j < n; ++j) {
          const int32_t u = sc->tmp[j];
          r += (u < v[t]) || (u == v[t] && j < i);
        }
        rk[t] = r;
      }
    }
    __syncwarp();
    for (int t = 0; t < 2; ++t)
      if (rk[t] >= 0) { sc->rs[rk[t]] = v[t]; sc->ord[rk[t]] = (uint8_t)(lane + 32 * t); }
    __syncwarp();
  }
  // residues must tile the cell: consecutive gaps (and the wrap) <= span + g
  bool cont = true;
  for (int r = lane; r < n; r += 32) {
    const int64_t nx = r + 1 < n ? (int64_t)sc->rs[r + 1] : (int64_t)sc->rs[0] + (int64_t)s0;
    if (nx - (int64_t)sc->rs[r] > tol) cont = false;
  }
  if (!__all_sync(0xffffffffu, cont)) return false;
  // 3. breakpoints per dimension: distinct offsets D, merged with D + ex
  int64_t nbox = 1;
#if GVO_OUTLINE & 512
  #pragma unroll 1
#endif
  for (int d = 0; d < nd; ++d) {
    const int32_t ex = (int32_t)sc->l0ex[d];
    int32_t v[2];
    int rk[2];
    for (int t = 0; t < 2; ++t) {
      const int i = lane + 32 * t;
      rk[t] = -1;
      if (i < n) {
        v[t] = sc->kv[d][i];
        int r = 0;
        bool first = true;
        for (int j = 0; j < n; ++j) {
          const int32_t u = sc->kv[d][j];
          if (u == v[t] && j < i) first = false;
          r += u < v[t];
        }
        // rank among distinct values = #distinct values below v
        if (first) rk[t] = r;
      }
    }
    // compact: distinct rank = number of distinct values below -> count of
    // first occurrences below (computed by ballot over sorted ranks)
    __syncwarp();
    // tmp[r] = value for first occurrences at their (non-distinct) rank
    for (int j = lane; j < n; j += 32) sc->tmp[j] = INT32_MIN;
    __syncwarp();
    for (int t = 0; t < 2; ++t) if (rk[t] >= 0) sc->tmp[rk[t]] = v[t];
    __syncwarp();
    // distinct sorted values: the non-sentinel entries of tmp in order
    int m = 0;
    {
      const int32_t a0 = lane < n ? sc->tmp[lane] : INT32_MIN;
      const int32_t a1 = lane + 32 < n ? sc->tmp[lane + 32] : INT32_MIN;
      const unsigned b0 = __ballot_sync(0xffffffffu, a0 != INT32_MIN);
      const unsigned b1 = __ballot_sync(0xffffffffu, a1 != INT32_MIN);
      const int p0 = __popc(b0 & ((1u << lane) - 1u));
      const int p1 = __popc(b0) + __popc(b1 & ((1u << lane) - 1u));
      m = __popc(b0) + __popc(b1);
      __syncwarp();
      if (a0 != INT32_MIN) sc->tmp[p0] = a0;  // p0 <= lane: safe after the reads above
      __syncwarp();
      if (a1 != INT32_MIN) sc->tmp[p1] = a1;
      __syncwarp();
    }
    // merge D (tmp[0..m), sorted distinct) with D + ex, common values once
    auto lbD = [&](int32_t x) {  // #D elements < x
      int lo = 0, hi = m;
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (sc->tmp[mid] < x) lo = mid + 1; else hi = mid; }
      return lo;
    };
    uint64_t both = 0;  // D elements y with y - ex in D (y in D and in D + ex)
    for (int t = 0; t < 2; ++t) {
      const int i = lane + 32 * t;
      bool f = false;
      if (i < m) { const int32_t y = sc->tmp[i] - ex; const int j = lbD(y); f = j < m && sc->tmp[j] == y; }
      const unsigned bb = __ballot_sync(0xffffffffu, f);
      both |= (uint64_t)bb << (32 * t);
    }
    const int nmerged = 2 * m - __popcll(both);
    const int b0 = d == 0 ? 0 : sc->boff[d - 1] + sc->nb[d - 1];
    if (b0 + nmerged > kSegBpAll) return false;
    if (lane == 0) sc->boff[d] = b0;
    __syncwarp();
    for (int t = 0; t < 2; ++t) {
      const int i = lane + 32 * t;
      if (i >= m) continue;
      const int32_t x = sc->tmp[i];
      const uint64_t below_i = i ? (~0ull >> (64 - i)) : 0ull;
      sc->bpf[sc->boff[d] + (i + lbD(x - ex) - __popcll(both & below_i))] = x;
      const int32_t y = x + ex;
      const int j = lbD(y);
      if (!(j < m && sc->tmp[j] == y)) {
        const uint64_t below_j = j ? (j >= 64 ? ~0ull : (~0ull >> (64 - j))) : 0ull;
        sc->bpf[sc->boff[d] + (j + i - __popcll(both & below_j))] = y;
      }
    }
    if (lane == 0) sc->nb[d] = nmerged;
    nbox *= nmerged - 1;
    if (nbox > kSegMaxBoxes) return false;
    __syncwarp();
  }
  // 4. per-dimension segment masks over sorted positions (lane holds
  // segments lane and lane + 32)
  bool fly = false;  // a dimension with > 64 segments: masks computed per box
#if GVO_OUTLINE & 512
  #pragma unroll 1
#endif
  for (int d = 0; d < nd; ++d) fly |= sc->nb[d] - 1 > 64;
  uint64_t segm[kSegDims][2];
#pragma unroll
  for (int d = 0; d < kSegDims; ++d) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      segm[d][h] = 0;
      const int sg = lane + 32 * h;
      if (!fly && d < nd && sg < sc->nb[d] - 1) {
        const int32_t lo = sc->bpf[sc->boff[d] + (sg)], hi = sc->bpf[sc->boff[d] + (sg + 1)];
        const int32_t ex = (int32_t)sc->l0ex[d];
        for (int r = 0; r < n; ++r) {
          const int32_t k = sc->kv[d][sc->ord[r]];
          if (k <= lo && hi <= k + ex) segm[d][h] |= 1ull << r;
        }
      }
    }
  }
  // 5. plan: elements and runs of the segment cover vs. cover_warp's clusters
  double vol0 = 1.0;
#if GVO_OUTLINE & 512
  #pragma unroll 1
#endif
  for (int d = 0; d < nd; ++d) vol0 *= (double)sc->l0ex[d];
  double seg_el = 0.0;
  int64_t seg_runs = 0;
  for (int64_t b0 = 0; b0 < nbox; b0 += 32) {
    const int64_t b = b0 + lane;
    int sd[kSegDims];
    {
      int64_t r = b < nbox ? b : 0;
#pragma unroll
      for (int d = 0; d < kSegDims; ++d) {
        if (d < nd) { const int ns = sc->nb[d] - 1; sd[d] = (int)(r % ns); r /= ns; } else sd[d] = 0;
      }
    }
    uint64_t M = ~0ull;
    if (!fly) {
#pragma unroll
      for (int d = 0; d < kSegDims; ++d) {
        const uint64_t v0 = __shfl_sync(0xffffffffu, segm[d][0], sd[d] & 31);
        const uint64_t v1 = __shfl_sync(0xffffffffu, segm[d][1], sd[d] & 31);
        if (d < nd) M &= sd[d] >= 32 ? v1 : v0;
      }
    } else if (b < nbox) {
      M = 0;
      for (int r2 = 0; r2 < n; ++r2) {
        bool in = true;
#if GVO_OUTLINE & 512
        #pragma unroll 1
#endif
        for (int d = 0; d < nd && in; ++d) {
          const int32_t k = sc->kv[d][sc->ord[r2]];
          in = k <= sc->bpf[sc->boff[d] + sd[d]] && sc->bpf[sc->boff[d] + sd[d] + 1] <= k + (int32_t)sc->l0ex[d];
        }
        if (in) M |= 1ull << r2;
      }
    }
    if (b >= nbox || !M) continue;
    double vol = 1.0;
#if GVO_OUTLINE & 512
    #pragma unroll 1
#endif
    for (int d = 0; d < nd; ++d) vol *= (double)(sc->bpf[sc->boff[d] + sd[d] + 1] - sc->bpf[sc->boff[d] + sd[d]]);
    const double len0 = (double)(sc->bpf[sc->boff[0] + sd[0] + 1] - sc->bpf[sc->boff[0] + sd[0]]);
    uint64_t mm = M;
    while (mm) {
      const int r0 = __ffsll((long long)mm) - 1;
      int r1 = r0;
      mm &= mm - 1;
      while (mm) {
        const int q = __ffsll((long long)mm) - 1;
        if ((int64_t)sc->rs[q] - (int64_t)sc->rs[r1] > tol) break;
        r1 = q;
        mm &= mm - 1;
      }
      const bool fold = (int64_t)s0 <= (int64_t)L0.span + (sc->rs[r1] - sc->rs[r0]) + G.g;
      seg_el += fold ? vol / len0 : vol;
      ++seg_runs;
    }
  }
  int64_t n_cl = 0;  // cover_warp's clusters of consecutive translates
  for (int i = lane; i < n; i += 32)
    if (i == 0 || (unsigned __int128)(uint64_t)(P[i] - P[i - 1]) > (unsigned __int128)(uint64_t)tol) ++n_cl;
  for (int o = 16; o; o >>= 1) {
    seg_el += __shfl_xor_sync(0xffffffffu, seg_el, o);
    seg_runs += __shfl_xor_sync(0xffffffffu, seg_runs, o);
    n_cl += __shfl_xor_sync(0xffffffffu, n_cl, o);
  }
  if (seg_el + (double)(kSegRunWeight * seg_runs) >= (double)n_cl * vol0 + (double)(kSegRunWeight * n_cl)) return false;
  // 6. emit
  for (int64_t b0 = 0; b0 < nbox; b0 += 32) {
    const int64_t b = b0 + lane;
    int sd[kSegDims];
    {
      int64_t r = b < nbox ? b : 0;
#pragma unroll
      for (int d = 0; d < kSegDims; ++d) {
        if (d < nd) { const int ns = sc->nb[d] - 1; sd[d] = (int)(r % ns); r /= ns; } else sd[d] = 0;
      }
    }
    uint64_t M = ~0ull;
    if (!fly) {
#pragma unroll
      for (int d = 0; d < kSegDims; ++d) {
        const uint64_t v0 = __shfl_sync(0xffffffffu, segm[d][0], sd[d] & 31);
        const uint64_t v1 = __shfl_sync(0xffffffffu, segm[d][1], sd[d] & 31);
        if (d < nd) M &= sd[d] >= 32 ? v1 : v0;
      }
    } else if (b < nbox) {
      M = 0;
      for (int r2 = 0; r2 < n; ++r2) {
        bool in = true;
#if GVO_OUTLINE & 512
        #pragma unroll 1
#endif
        for (int d = 0; d < nd && in; ++d) {
          const int32_t k = sc->kv[d][sc->ord[r2]];
          in = k <= sc->bpf[sc->boff[d] + sd[d]] && sc->bpf[sc->boff[d] + sd[d] + 1] <= k + (int32_t)sc->l0ex[d];
        }
        if (in) M |= 1ull << r2;
      }
    }
    if (b >= nbox || !M) continue;
    Lat4 L;
    L.nd = nd;
    L.span = L0.span;
    uint64_t base = (uint64_t)L0.base;
#pragma unroll
    for (int d = 0; d < kSegDims; ++d) {
      if (d < nd) {
        L.st[d] = sc->l0st[d];
        L.ex[d] = (int64_t)(sc->bpf[sc->boff[d] + sd[d] + 1] - sc->bpf[sc->boff[d] + sd[d]]);
        base += sc->l0st[d] * (uint64_t)(int64_t)sc->bpf[sc->boff[d] + sd[d]];
      } else {
        L.st[d] = 0;
        L.ex[d] = 1;
      }
    }
    L.base = (int64_t)base;
    // partial cells along a long row: one pattern run instead of one
    // lattice per residue cluster (unless the clusters fold into the span)
    if (allow_pattern && L0.span == 0 && L.ex[0] >= kPatMinCells) {
      const int rf = __ffsll((long long)M) - 1, rl = 63 - __clzll((long long)M);
      int64_t dg = (int64_t)s0;
      int ncl = 0;
      int64_t prev = -1;
      for (uint64_t m2 = M; m2; m2 &= m2 - 1) {
        const int q = __ffsll((long long)m2) - 1;
        dg = gcd64(dg, (int64_t)sc->rs[q]);
        if (prev < 0 || (int64_t)sc->rs[q] - prev > tol) ++ncl;
        prev = sc->rs[q];
      }
      const bool folds = ncl == 1 && (int64_t)s0 <= (int64_t)(sc->rs[rl] - sc->rs[rf]) + G.g;
      const int64_t per = (int64_t)s0 / gcd64((int64_t)s0, G.g);  // sectors per pattern period
      if (!folds && (int64_t)s0 / dg <= 64 && per <= 32) {
        uint64_t pm = 0;
        for (uint64_t m2 = M; m2; m2 &= m2 - 1) pm |= 1ull << (sc->rs[__ffsll((long long)m2) - 1] / dg);
        if (emit_pattern(S, L, base, tag, G, pm, dg, (int64_t)s0)) continue;
      }
    }
    uint64_t mm = M;
    while (mm) {
      const int r0 = __ffsll((long long)mm) - 1;
      int r1 = r0;
      mm &= mm - 1;
      while (mm) {
        const int q = __ffsll((long long)mm) - 1;
        if ((int64_t)sc->rs[q] - (int64_t)sc->rs[r1] > tol) break;
        r1 = q;
        mm &= mm - 1;
      }
      Lat4 C = L;
      C.base = (int64_t)(base + (uint64_t)(int64_t)sc->rs[r0]);
      C.span = L0.span + (uint64_t)(sc->rs[r1] - sc->rs[r0]);
      l4_emit_lattice(S, C, tag, G);
    }
  }
  return true;
}

// lattice of one coefficient vector over one block box, translation 0
// (warp-cooperative: lane k < 6 holds coordinate k = tid x/y/z, bid x/y/z)
__device__ GVO_OL_BOX WLat box_lattice(const int64_t* c, const int32_t bd[3], const Box& b, const Granule& G) {
  const int lane = threadIdx.x & 31;
  int64_t ext = 1, co = 0;
  uint64_t contrib = 0;
  if (lane < 6) {
    ext = lane == 0 ? bd[0] : lane == 1 ? bd[1] : lane == 2 ? bd[2] : lane == 3 ? b.n[0] : lane == 4 ? b.n[1] : b.n[2];
    co = c[1 + lane];
    if (lane >= 3) contrib = (uint64_t)co * (uint64_t)(lane == 3 ? b.lo[0] : lane == 4 ? b.lo[1] : b.lo[2]);
    if (ext > 1 && co < 0) contrib += (uint64_t)co * (uint64_t)(ext - 1);
  }
  for (int o = 4; o; o >>= 1) contrib += __shfl_xor_sync(kFull, contrib, o);
  WLat L;
  L.base = (int64_t)__shfl_sync(kFull, contrib, 0);
  L.span = 0;
  L.nd = 6;
  L.st = lane < 6 && ext > 1 && co != 0 ? (co < 0 ? (uint64_t)0 - (uint64_t)co : (uint64_t)co) : 0;
  L.ex = lane < 6 ? ext : 1;
  wl_normalize(L, G.g);
  return L;
}


// ------------------------------------------------------------------ decode
// tuple k of a lattice run -> base address (dim 0 fastest).  The 64-bit
// decode (k >= 2^31, rare) is kept out of line: its divisions would
// otherwise be inlined at every call site (~1.3 k instructions each, the
// largest share of the kernel's 1.5 MB of code and of its instruction-fetch
// stalls).
__device__ __noinline__ uint64_t run_base_wide(const Run& r, int64_t k) {
  uint64_t b = (uint64_t)r.base;
  for (int d = 0; d < r.nd; ++d) {
    const int64_t idx = k % r.ext[d];
    k /= r.ext[d];
    b += (uint64_t)r.stride[d] * (uint64_t)idx;
  }
  return b;
}

__device__ __forceinline__ uint64_t run_base(const Run& r, int64_t k) {
  if (k >= (int64_t(1) << 31)) return run_base_wide(r, k);
  uint64_t b = (uint64_t)r.base;
  uint32_t k32 = (uint32_t)k;
#if GVO_OUTLINE & 32
#pragma unroll 1
#endif
  for (int d = 0; d < r.nd; ++d) {
    const uint32_t ex = (uint32_t)r.ext[d];
    const uint32_t q = k32 / ex;
    b += (uint64_t)r.stride[d] * (uint64_t)(k32 - q * ex);
    k32 = q;
  }
  return b;
}

// element k of a points run (non-affine access: one bytecode evaluation per
// (block, thread)) -> its granule; out of line like run_base_wide (cold in
// affine workloads, the interpreter is large)
__device__ __noinline__ int64_t run_point_granule(const Run& r, int64_t k, const Granule& Gr, const TplView& T,
                                                  int abase, const int64_t* fbase, const int32_t* bd,
                                                  const int64_t* gd, int64_t tpb) {
  const int64_t blk = r.run_start + k / tpb;
  const int64_t th = k % tpb;
  int64_t crd[6];
  crd[0] = th % bd[0];
  crd[1] = (th / bd[0]) % bd[1];
  crd[2] = th / ((int64_t)bd[0] * bd[1]);
  crd[3] = blk % gd[0];
  crd[4] = (blk / gd[0]) % gd[1];
  crd[5] = blk / (gd[0] * gd[1]);
  const int ga = abase + r.access;
  return Gr.of(eval_point(T.code + T.code_off[ga], T.code_len[ga], crd, bd, fbase));
}

// element k of any run -> absolute granule interval [glo, ghi]
__device__ GVO_OL_RIV void run_interval(const Run& r, int64_t k, const Granule& Gr, const TplView& T, int abase,
                                             const int64_t* fbase, const int32_t bd[3], const int64_t gd[3],
                                             int64_t tpb, int64_t* glo, int64_t* ghi) {
  if (r.kind == 0) {
    int64_t piece = 0;
    if (r.pieces > 1) { piece = k % r.pieces; k /= r.pieces; }
    const uint64_t b = run_base(r, k);
    int64_t lo = Gr.of((int64_t)b), hi = Gr.of((int64_t)(b + r.span));
    if (r.pieces > 1) {
      int64_t plo = lo + piece * kPiece;
      if (plo > hi) plo = lo;
      hi = min(hi, plo + kPiece - 1);
      lo = plo;
    }
    *glo = lo;
    *ghi = hi;
  } else {
    *glo = *ghi = run_point_granule(r, k, Gr, T, abase, fbase, bd, gd, tpb);
  }
}

// first tuple k of a monotone run with (hi ? interval end : start) >= v
__device__ inline int64_t mono_first(const Run& r, const Granule& Gr, int64_t kbase, int64_t v, bool hi) {
  // f(k) = base + sum_d stride_d k_d increases with the tuple index (the
  // monotone condition), so floor((f + span?)/g) - kbase >= v <=> f >= T:
  // the digits of the first such tuple follow greedily from the slowest dim.
  // Loops over dims are unrolled with constant indices (registers only).
  const __int128 T = ((__int128)v + (__int128)kbase) * (__int128)Gr.g - (hi ? (__int128)r.span : (__int128)0);
  const __int128 R0 = T - (__int128)r.base;
  if (R0 <= 0) return 0;
  const int nd = r.nd;
  int64_t st[kMaxDims], ex[kMaxDims], M[kMaxDims];  // M[d]: reach of the dims faster than d
  uint64_t acc = 0;
#pragma unroll
  for (int d = 0; d < kMaxDims; ++d) {
    st[d] = d < nd ? r.stride[d] : 0;
    ex[d] = d < nd ? r.ext[d] : 1;
    M[d] = (int64_t)acc;
    acc += (uint64_t)st[d] * (uint64_t)(ex[d] - 1);
  }
  if (R0 > (__int128)acc) return r.count;
  int64_t R = (int64_t)R0;
  int64_t mul = 1;
#pragma unroll
  for (int d = 0; d < kMaxDims; ++d) mul *= ex[d];
  int64_t idx = 0;
#pragma unroll
  for (int d = kMaxDims - 1; d >= 0; --d) {
    mul /= ex[d];
    int64_t k = 0;
    if (d < nd && R > M[d]) {
      const uint64_t s1 = (uint64_t)st[d];
      k = (int64_t)(((uint64_t)(R - M[d]) + s1 - 1) / s1);
      if (k > ex[d] - 1) k = ex[d] - 1;
      R -= (int64_t)((uint64_t)k * s1);
    }
    idx += k * mul;
  }
  return idx;
}

// ------------------------------------------------------------------ sort
// CTA-wide stable LSD radix sort (8-bit digits) of packed 64-bit elements
// on bits [bit0, bit0 + nbits).  a/b may live in shared or global memory.
__device__ GVO_NOINL uint64_t* cta_sort(uint64_t* a, uint64_t* b, int64_t n, int bit0, int nbits,
                              uint32_t* hist /* kNW*256 */, uint32_t* tot /* 256 */) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = (((n + kNW - 1) / kNW) + 255) & ~int64_t(255);
  const int64_t beg = min(n, (int64_t)w * chunk), end = min(n, beg + chunk);
  for (int sh = bit0; sh < bit0 + nbits; sh += 8) {
    for (int i = threadIdx.x; i < kNW * 256; i += kNT) hist[i] = 0;
    __syncthreads();
    for (int64_t i0 = beg; i0 < end; i0 += 256) {
      uint32_t dg[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t i = i0 + k * 32 + lane;
        dg[k] = i < end ? (uint32_t)(a[i] >> sh) & 255u : 256u;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (dg[k] < 256u) atomicAdd(&hist[w * 256 + dg[k]], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 256) {
      const int d = threadIdx.x;
      uint32_t s = 0;
      for (int k = 0; k < kNW; ++k) s += hist[k * 256 + d];
      tot[d] = s;
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of 256 digit totals, 8 per lane
      uint32_t v[8], run = 0;
      for (int k = 0; k < 8; ++k) { v[k] = run; run += tot[lane * 8 + k]; }
      uint32_t incl = run;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t excl = incl - run;
      for (int k = 0; k < 8; ++k) tot[lane * 8 + k] = excl + v[k];
    }
    __syncthreads();
    if (threadIdx.x < 256) {
      const int d = threadIdx.x;
      uint32_t run = tot[d];
      for (int k = 0; k < kNW; ++k) {
        uint32_t h = hist[k * 256 + d];
        hist[k * 256 + d] = run;
        run += h;
      }
    }
    __syncthreads();
    for (int64_t i0 = beg; i0 < end; i0 += 256) {
      uint64_t ev[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t i = i0 + k * 32 + lane;
        ev[k] = i < end ? a[i] : 0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t i = i0 + k * 32 + lane;
        const bool v = i < end;
        const unsigned act = __ballot_sync(0xffffffffu, v);
        if (!act) break;
        const uint32_t d = (uint32_t)(ev[k] >> sh) & 255u;
        unsigned peers = 0;
        if (v) {
          peers = __match_any_sync(act, d);
          const uint32_t pos = hist[w * 256 + d] + __popc(peers & ((1u << lane) - 1u));
          b[pos] = ev[k];
        }
        __syncwarp();
        if (v && (31 - __clz(peers)) == lane) hist[w * 256 + d] += __popc(peers);
        __syncwarp();
      }
    }
    __syncthreads();
    uint64_t* t = a; a = b; b = t;
  }
  return a;
}

// ------------------------------------------------------------------ sweep
// Union counts of tagged subsets over the sorted elements in one pass pair.
// Each warp owns a contiguous chunk, each lane a contiguous sub-chunk (odd
// length: conflict-free 8-byte shared loads).  Pass 1: per-lane maxima of the
// rescaled interval ends for every subset; warp and CTA exclusive max-scans
// give each lane the running maximum R before its sub-chunk.  Pass 2: a
// sequential walk adds max(0, hi - max(lo - 1, R)) per selected interval.
#ifndef GVO_SWEEP_GROUP
#define GVO_SWEEP_GROUP 4
#endif
constexpr int kSubGroup = GVO_SWEEP_GROUP;  // subsets swept per pass (A/B: 4 = 6 > 12)
__device__ GVO_NOINL void sweep(const uint64_t* e, int64_t n, UnitSh& U, int64_t* wmax /* kMaxSub*kNW */) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = (n + kNW - 1) / kNW;
  const int64_t beg = min(n, (int64_t)w * chunk), end = min(n, beg + chunk);
  int64_t sub = (end - beg + 31) / 32;
  if (sub > 0 && !(sub & 1)) ++sub;
  const int64_t lb = min(end, beg + lane * sub), le = min(end, lb + sub);
  for (int s0 = 0; s0 < U.n_sub; s0 += kSubGroup) {
    const int sn = min(kSubGroup, U.n_sub - s0);
    uint32_t mask[kSubGroup];
    int sh[kSubGroup];
    int64_t r[kSubGroup], R[kSubGroup], cnt[kSubGroup];
#pragma unroll
    for (int q = 0; q < kSubGroup; ++q) {
      mask[q] = q < sn ? U.sub_mask[s0 + q] : 0u;
      sh[q] = q < sn ? U.sub_sh[s0 + q] : 0;
      r[q] = q < sn ? U.sub_r[s0 + q] : 1;
      R[q] = -1;
      cnt[q] = 0;
    }
    // pass 1: lane maxima
    for (int64_t i = lb; i < le; ++i) {
      const uint64_t x = e[i];
      const uint32_t tag = (uint32_t)(x & 31u);
      const int64_t hi0 = (int64_t)(x >> kKeyShift) + (int64_t)((x >> kTagBits) & kLenMask);
#pragma unroll
      for (int q = 0; q < kSubGroup; ++q)
        if ((mask[q] >> tag) & 1u) R[q] = max(R[q], sh[q] >= 0 ? (hi0 >> sh[q]) : hi0 / r[q]);
    }
    // warp exclusive max-scan per subset; warp totals to shared memory
#pragma unroll
    for (int q = 0; q < kSubGroup; ++q) {
      int64_t inc = R[q];
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = max(inc, t);
      }
      int64_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) ex = -1;
      R[q] = ex;
      if (lane == 31 && q < sn) wmax[q * kNW + w] = inc;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kSubGroup; ++q) {
      if (q >= sn) continue;
      int64_t c = -1;
      for (int k = 0; k < w; ++k) c = max(c, wmax[q * kNW + k]);
      R[q] = max(R[q], c);
    }
    __syncthreads();
    // pass 2: contributions
    for (int64_t i = lb; i < le; ++i) {
      const uint64_t x = e[i];
      const uint32_t tag = (uint32_t)(x & 31u);
      const int64_t lo0 = (int64_t)(x >> kKeyShift);
      const int64_t hi0 = lo0 + (int64_t)((x >> kTagBits) & kLenMask);
#pragma unroll
      for (int q = 0; q < kSubGroup; ++q) {
        if (!((mask[q] >> tag) & 1u)) continue;
        const int64_t lo = sh[q] >= 0 ? (lo0 >> sh[q]) : lo0 / r[q];
        const int64_t hi = sh[q] >= 0 ? (hi0 >> sh[q]) : hi0 / r[q];
        if (lo > R[q]) cnt[q] += hi - lo + 1;
        else if (hi > R[q]) cnt[q] += hi - R[q];
        R[q] = max(R[q], hi);
      }
    }
#pragma unroll
    for (int q = 0; q < kSubGroup; ++q) {
      int64_t v = cnt[q];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && q < sn) wmax[q * kNW + w] = v;
    }
    __syncthreads();
    if (threadIdx.x < sn) {
      int64_t v = 0;
      for (int k = 0; k < kNW; ++k) v += wmax[threadIdx.x * kNW + k];
      U.sub_val[s0 + threadIdx.x] = v;
    }
    __syncthreads();
  }
}

// exclusive prefix sum of a[0..n) in place, total in a[n] (all threads)
__device__ void cta_scan_excl(int64_t* a, int64_t n, int64_t* wtmp /* kNW */) {
  const int64_t per = (n + kNT - 1) / kNT;
  const int64_t b0 = min(n, (int64_t)threadIdx.x * per), b1 = min(n, b0 + per);
  int64_t s = 0;
  for (int64_t i = b0; i < b1; ++i) s += a[i];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t inc = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wtmp[w] = inc;
  __syncthreads();
  int64_t run = inc - s;
  for (int k = 0; k < w; ++k) run += wtmp[k];
  for (int64_t i = b0; i < b1; ++i) { const int64_t v = a[i]; a[i] = run; run += v; }
  if (threadIdx.x == kNT - 1) a[n] = run;
  __syncthreads();
}

// ------------------------------------------------------------------ bitmap tier
// Exact set measures of one key range [a, b) by bitmaps: bit (t, x) is set
// iff granule a + x lies in an interval of tag t.  Every in-range element of
// the unit's runs sets its clipped bits (single-word intervals by one
// shared-memory atomicOr, longer ones word by word), then each requested
// measure is the popcount of the OR of its tags' words, at granule or at
// line resolution (groups of r bits, r | 32, a aligned to r).
__device__ __forceinline__ void bm_set(uint32_t* bm, int64_t x, int64_t y) {
  const int64_t w0 = x >> 5, w1 = y >> 5;
  const uint32_t m0 = ~0u << (x & 31), m1 = ~0u >> (31 - (y & 31));
  if (w0 == w1) { atomicOr(bm + w0, m0 & m1); return; }
  atomicOr(bm + w0, m0);
  for (int64_t w = w0 + 1; w < w1; ++w) bm[w] = ~0u;  // idempotent: races with atomicOr are benign
  atomicOr(bm + w1, m1);
}

__device__ __forceinline__ uint32_t bm_lines(uint32_t v, int r) {
  // one bit per group of r bits that has any bit set (bit at the group's low end)
  uint32_t low = 0;
  for (int k = 0; k < 32; k += r) low |= 1u << k;
  uint32_t o = v;
  for (int k = 1; k < r; k <<= 1) o |= o >> k;  // OR-fold within groups (r a power of two)
  return o & low;
}

// Bits of elements [k, k + cnt) of one monotone lattice run in the bitmap of
// its tag (bit x = granule kb0 + x, x < w).  Dim 0 is stepped incrementally;
// single-granule intervals landing in the same word are OR-ed in a register
// and written with one atomicOr.  Kept out of line: few live values, no spills.
__device__ __noinline__ void bm_lattice(uint32_t* bmt, const Run* rrp, int64_t k, int64_t cnt, int64_t kb0,
                                        int64_t w, int64_t g, int shift) {
  const Run& rr = *rrp;
  const int nd = rr.nd;
  // two-level cursor: dims 0 and 1 stepped incrementally, a full decode only
  // when dim 1 wraps (segment boxes are often 1-2 cells wide along dim 0)
  const uint64_t st0 = nd > 0 ? (uint64_t)rr.stride[0] : 0;
  const int64_t ex0 = nd > 0 ? rr.ext[0] : 1;
  const uint64_t st1 = nd > 1 ? (uint64_t)rr.stride[1] : 0;
  const int64_t ex1 = nd > 1 ? rr.ext[1] : 1;
  const uint64_t back0 = st0 * (uint64_t)(ex0 - 1);
  const uint64_t span = rr.span;
  uint64_t bb = run_base(rr, k);
  int64_t i0 = k % ex0, i1 = (k / ex0) % ex1;
  uint32_t* cur_p = nullptr;
  uint32_t cur_m = 0;
  for (int64_t t = 0; t < cnt; ++t) {
    int64_t lo, hi;
    if (shift >= 0) { lo = ((int64_t)bb >> shift) - kb0; hi = ((int64_t)(bb + span) >> shift) - kb0; }
    else { lo = floordiv((int64_t)bb, g) - kb0; hi = floordiv((int64_t)(bb + span), g) - kb0; }
    lo = max(lo, (int64_t)0);
    hi = min(hi, w - 1);
    if (lo == hi) {
      uint32_t* p = bmt + (lo >> 5);
      const uint32_t bit = 1u << (lo & 31);
      if (p == cur_p) cur_m |= bit;
      else {
        if (cur_p) atomicOr(cur_p, cur_m);
        cur_p = p;
        cur_m = bit;
      }
    } else if (lo < hi) {
      bm_set(bmt, lo, hi);
    }
    if (++i0 < ex0) bb += st0;
    else {
      i0 = 0;
      if (++i1 < ex1) bb += st1 - back0;
      else { i1 = 0; if (t + 1 < cnt) bb = run_base(rr, k + t + 1); }
    }
  }
  if (cur_p) atomicOr(cur_p, cur_m);
}

// Bits of elements [k, k + cnt) of a pattern run (emit_pattern): per row the
// sectors of cells c < n0 and residues t*dg (bit t of pm) relative to the
// row's first cell.  The sector set of an unbounded row is periodic with
// P = s0 / gcd(s0, g) sectors (nph = g / gcd cells); clipped to the row's own
// first and last sector it is exact: a virtual cell beyond either end can only
// touch the end sector, which the end cell touches itself.  Each bitmap word
// is one 32-bit window of the period pattern repeated over 128 bits.
// Period pattern of a row whose first cell starts at byte cell0: bit j set
// iff some cell c < nph touches sector G(cell0) + j (mod P).  Depends only on
// cell0 mod g.
__device__ __forceinline__ uint32_t pattern_bits(int64_t cell0, uint64_t pm, int64_t dg, int64_t s0, int64_t P,
                                                 int64_t nph, int64_t g, int shift, int part, int nparts) {
  // relative to S0 = G(cell0): sector of byte cell0 + y is (ph + y) / g, ph = cell0 mod g
  const int64_t ph = floormod(cell0, g);
  const int nt = __popcll(pm);
  uint32_t pat = 0;
  for (int64_t p = part; p < nph * nt; p += nparts) {
    const int64_t c = p / nt;
    int ti = (int)(p - c * nt);
    uint64_t m = pm;
    for (; ti > 0; --ti) m &= m - 1;
    const int64_t y = ph + c * s0 + (int64_t)(__ffsll((long long)m) - 1) * dg;
    int64_t j = shift >= 0 ? (y >> shift) : y / g;  // y >= 0
    while (j >= P) j -= P;
    pat |= 1u << j;
  }
  return pat;
}

// Thread mode: this thread sets every word of elements [k, k + cnt); the
// period pattern is rebuilt only when a row's phase (cell0 mod g) changes.
__device__ __noinline__ void bm_pattern(uint32_t* bmt, const Run* rrp, int64_t k, int64_t cnt, int64_t kb0,
                                        int64_t w, int64_t g, int shift) {
  const Run& rr = *rrp;
  const int64_t dg = rr.pad_, s0 = rr.run_count;
  const uint64_t pm = (uint64_t)rr.run_start;
  const int64_t rmin = (int64_t)(__ffsll((long long)pm) - 1) * dg;
  const int64_t gc = gcd64(s0, g), P = s0 / gc, nph = g / gc;
  auto G = [&](int64_t x) { return shift >= 0 ? (x >> shift) : floordiv(x, g); };
  int64_t phase = (int64_t)((uint64_t)rr.pieces >> 32);  // the stored pattern's phase
  unsigned __int128 pp = (uint32_t)rr.pieces;
  for (int64_t sh = P; sh < 128; sh += P) pp |= (unsigned __int128)(uint32_t)rr.pieces << sh;
  for (int64_t e = 0; e < cnt; ++e) {
    const uint64_t bel = run_base(rr, k + e);
    const int64_t cell0 = (int64_t)bel - rmin;
    int64_t lo = G((int64_t)bel) - kb0, hi = G((int64_t)(bel + rr.span)) - kb0;
    lo = max(lo, (int64_t)0);
    hi = min(hi, w - 1);
    if (lo > hi) continue;
    const int64_t S0 = G(cell0);
    const int64_t ph = floormod(cell0, g);
    if (ph != phase) {
      phase = ph;
      const uint32_t pat = pattern_bits(cell0, pm, dg, s0, P, nph, g, shift, 0, 1);
      pp = pat;
      for (int64_t sh = P; sh < 128; sh += P) pp |= (unsigned __int128)pat << sh;
    }
    const int64_t w0 = lo >> 5, w1 = hi >> 5;
    int64_t off = floormod(kb0 + (w0 << 5) - S0, P);  // pattern phase of the first word's bit 0
    const int64_t step = 32 % P;
    for (int64_t ww = w0; ww <= w1; ++ww) {
      uint32_t v = (uint32_t)(pp >> off);
      if (ww == w0) v &= ~0u << (lo & 31);
      if (ww == w1) v &= ~0u >> (31 - (hi & 31));
      if (v) atomicOr(bmt + ww, v);
      off += step;
      if (off >= P) off -= P;
    }
  }
}

// One element (row) of a pattern run by one warp: lanes build the period
// pattern together and stride over the row's words.
__device__ __noinline__ void bm_pattern_warp(uint32_t* bmt, const Run* rrp, int64_t k, int64_t kb0, int64_t w,
                                             int64_t g, int shift) {
  const Run& rr = *rrp;
  const int lane = threadIdx.x & 31;
  const int64_t dg = rr.pad_, s0 = rr.run_count;
  const uint64_t pm = (uint64_t)rr.run_start;
  const int64_t rmin = (int64_t)(__ffsll((long long)pm) - 1) * dg;
  const int64_t gc = gcd64(s0, g), P = s0 / gc, nph = g / gc;
  auto G = [&](int64_t x) { return shift >= 0 ? (x >> shift) : floordiv(x, g); };
  const uint64_t bel = run_base(rr, k);
  const int64_t cell0 = (int64_t)bel - rmin;
  int64_t lo = G((int64_t)bel) - kb0, hi = G((int64_t)(bel + rr.span)) - kb0;
  lo = max(lo, (int64_t)0);
  hi = min(hi, w - 1);
  if (lo > hi) return;  // warp-uniform
  const int64_t S0 = G(cell0);
  const uint32_t pat = floormod(cell0, g) == (int64_t)((uint64_t)rr.pieces >> 32)
                           ? (uint32_t)rr.pieces
                           : __reduce_or_sync(0xffffffffu, pattern_bits(cell0, pm, dg, s0, P, nph, g, shift, lane, 32));
  unsigned __int128 pp = pat;
  for (int64_t sh = P; sh < 128; sh += P) pp |= (unsigned __int128)pat << sh;
  const int64_t w0 = lo >> 5, w1 = hi >> 5;
  int64_t off = floormod(kb0 + ((w0 + lane) << 5) - S0, P);
  const int64_t step = (32 * 32) % P;
  for (int64_t ww = w0 + lane; ww <= w1; ww += 32) {
    uint32_t v = (uint32_t)(pp >> off);
    if (ww == w0) v &= ~0u << (lo & 31);
    if (ww == w1) v &= ~0u >> (31 - (hi & 31));
    if (v) atomicOr(bmt + ww, v);
    off += step;
    if (off >= P) off -= P;
  }
}

// popcounts of the atoms of NT bitmap planes over words [0, wp): acc[p] =
// bits set in exactly the planes of p (p = 1 .. 2^NT - 1), this thread's words
#ifndef GVO_BM_ATOMS
#define GVO_BM_ATOMS 1  // 0: the per-measure OR-select pass only (A/B)
#endif
constexpr int kAtomTags = 4;
template <int NT>
__device__ __forceinline__ void atom_counts(const uint32_t* bm, int64_t wp, int32_t (&acc)[1 << kAtomTags]) {
#pragma unroll
  for (int p = 0; p < (1 << kAtomTags); ++p) acc[p] = 0;
  for (int64_t i = threadIdx.x; i < wp; i += kNT) {
    uint32_t tw[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) tw[t] = bm[(int64_t)t * wp + i];
#pragma unroll
    for (int p = 1; p < (1 << NT); ++p) {
      uint32_t v = ~0u;
#pragma unroll
      for (int t = 0; t < NT; ++t) v &= ((p >> t) & 1) ? tw[t] : ~tw[t];
      acc[p] += __popc(v);
    }
  }
}

// GVO_BM_PROF (with GVO_PHASE_STATS): bitmap-tier sub-phases into the
// phase slots 12..15 (zeroing, element pass, big runs, measures) instead of
// the segment counters (tools/phase_profile.py reads them under those names)
#if defined(GVO_BM_PROF) && GVO_BM_PROF
#define GVO_BMP(...) __VA_ARGS__
#else
#define GVO_BMP(...)
#endif
__device__ __noinline__ void bitmap_range(uint32_t* bm, const Run* druns, const int64_t* rcnt, const int64_t* rka, int nr,
                             int64_t N, int64_t a, int64_t b, int64_t kbase, int n_tags, const Granule& Gr,
                             const TplView& T, int abase, const int64_t* fbase, const int32_t bd[3],
                             const int64_t gd[3], int64_t tpb, UnitSh& U, int64_t* wmax, bool nonmono,
                             uint32_t tag_mask, int* big_list, int big_cap GVO_BMP(, long long* php)) {
  GVO_BMP(long long tb0 = clock64();)
  const int64_t wp = (b - a + 31) >> 5;
  // runs whose every interval covers >= kBigWords bitmap words (folded rows,
  // merged layers) are filled by the whole CTA after the element pass: one
  // thread per such interval would hold the CTA at the barrier
#ifndef GVO_BIG_WORDS
#define GVO_BIG_WORDS 256  // A/B on C4 / a C5 sample: 8, 16, 32 (r01), 64, 128, 256, 1024 -> 256 best (-3 %)
#endif
  constexpr int64_t kBigWords = GVO_BIG_WORDS;
  const uint64_t big_span = (uint64_t)(kBigWords * 32) * (uint64_t)Gr.g;
  __shared__ int n_big;
  if (threadIdx.x == 0) n_big = 0;
  for (int64_t i = threadIdx.x; i < (int64_t)n_tags * wp; i += kNT) bm[i] = 0u;
  __syncthreads();
  GVO_BMP(if (threadIdx.x == 0) { const long long t = clock64(); php[12] += t - tb0; tb0 = t; })
  // monotone runs: elements rka[r] .. rka[r] + count, contiguous per thread.
  // Dim 0 is stepped incrementally; single-granule intervals that land in
  // the same bitmap word are OR-ed in a register before one atomicOr.
  {
    const int64_t per = (N + kNT - 1) / kNT;
    const int64_t e0 = min(N, (int64_t)threadIdx.x * per), e1 = min(N, e0 + per);
    int ri = 0;
    if (e0 < e1) {
      int lo = 0, hi = nr - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rcnt[mid] <= e0) lo = mid; else hi = mid - 1;
      }
      ri = lo;
    }
    int64_t i = e0;
    while (i < e1) {
      while (rcnt[ri + 1] <= i) ++ri;
      const int64_t iend = min(e1, rcnt[ri + 1]);
      if (rka[ri] < 0) { i = iend; continue; }
      const Run& rr = druns[ri];
      if (rr.kind != 1 && rr.span >= big_span) {  // whole-CTA pass below
        if (rcnt[ri] >= e0) {  // listed once, by the thread owning its first element
          const int slot = atomicAdd(&n_big, 1);
          if (slot < big_cap / 2 - 1) big_list[slot] = ri;
        }
        i = iend;
        continue;
      }
      uint32_t* bmt = bm + (int64_t)__popc(tag_mask & ((1u << rr.tag) - 1u)) * wp;
      int64_t k = rka[ri] + (i - rcnt[ri]);
      const int64_t kend = k + (iend - i);
      if (rr.kind == 2) {
        bm_pattern(bmt, &rr, k, kend - k, kbase + a, b - a, Gr.g, Gr.shift);
        i = iend;
        continue;
      }
      if (rr.kind != 0) {
        for (; k < kend; ++k) {
          int64_t lo, hi;
          run_interval(rr, k, Gr, T, abase, fbase, bd, gd, tpb, &lo, &hi);
          lo = max(lo - kbase, a);
          hi = min(hi - kbase, b - 1);
          if (lo <= hi) bm_set(bmt, lo - a, hi - a);
        }
        i = iend;
        continue;
      }
      bm_lattice(bmt, &rr, k, kend - k, kbase + a, b - a, Gr.g, Gr.shift);
      i = iend;
    }
  }
  // non-monotone runs: every element, clipped
  for (int r = 0; r < (nonmono ? nr : 0); ++r) {
    if (rka[r] >= 0) continue;
    const Run& rr = druns[r];
    for (int64_t k = threadIdx.x; k < rr.count; k += kNT) {
      int64_t lo, hi;
      run_interval(rr, k, Gr, T, abase, fbase, bd, gd, tpb, &lo, &hi);
      lo = max(lo - kbase, a);
      hi = min(hi - kbase, b - 1);
      if (lo <= hi) bm_set(bm + (int64_t)__popc(tag_mask & ((1u << rr.tag) - 1u)) * wp, lo - a, hi - a);
    }
  }
  __syncthreads();
  GVO_BMP(if (threadIdx.x == 0) { const long long t = clock64(); php[13] += t - tb0; tb0 = t; })
  // big runs: their (run, element) pairs dealt to warps, lanes over words
  {
    const int nb = min(n_big, big_cap / 2 - 1);
    int* pref = big_list + big_cap / 2;  // exclusive prefix of the listed runs' element counts
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int carry = 0;
      for (int q0 = 0; q0 < nb; q0 += 32) {
        const int q = q0 + lane;
        const int v = q < nb ? (int)(rcnt[big_list[q] + 1] - rcnt[big_list[q]]) : 0;
        int inc = v;
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += t;
        }
        if (q < nb) pref[q] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) pref[nb] = carry;
    }
    __syncthreads();
    const int total = pref[nb];
    const int wq = threadIdx.x >> 5, lq = threadIdx.x & 31;
    for (int f = wq; f < total; f += kNW) {
      int lo = 0, hi = nb - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pref[mid] <= f) lo = mid; else hi = mid - 1;
      }
      const int r = big_list[lo];
      const Run& rr = druns[r];
      uint32_t* pl = bm + (int64_t)__popc(tag_mask & ((1u << rr.tag) - 1u)) * wp;
      const int64_t kk = rka[r] + (f - pref[lo]);
      if (rr.kind == 2) {
        bm_pattern_warp(pl, &rr, kk, kbase + a, b - a, Gr.g, Gr.shift);
        continue;
      }
      const uint64_t bb = run_base(rr, kk);
      int64_t glo = Gr.of((int64_t)bb) - kbase - a, ghi = Gr.of((int64_t)(bb + rr.span)) - kbase - a;
      glo = max(glo, (int64_t)0);
      ghi = min(ghi, b - a - 1);
      if (glo > ghi) continue;
      const int64_t w0 = glo >> 5, w1 = ghi >> 5;
      for (int64_t ww = w0 + lq; ww <= w1; ww += 32) {
        uint32_t m = ~0u;
        if (ww == w0) m &= ~0u << (glo & 31);
        if (ww == w1) m &= ~0u >> (31 - (ghi & 31));
        if (m == ~0u) pl[ww] = ~0u; else atomicOr(pl + ww, m);
      }
    }
    if (n_big > nb) {  // list overflow: the unlisted big runs, one warp per element
      for (int r = 0; r < nr; ++r) {
        const Run& rr = druns[r];
        if (rka[r] < 0 || rr.kind == 1 || rr.span < big_span) continue;
        bool listed = false;
        for (int q = 0; q < nb && !listed; ++q) listed = big_list[q] == r;
        if (listed) continue;
        uint32_t* pl = bm + (int64_t)__popc(tag_mask & ((1u << rr.tag) - 1u)) * wp;
        for (int64_t e = wq; e < rcnt[r + 1] - rcnt[r]; e += kNW) {
          if (rr.kind == 2) { bm_pattern_warp(pl, &rr, rka[r] + e, kbase + a, b - a, Gr.g, Gr.shift); continue; }
          const uint64_t bb = run_base(rr, rka[r] + e);
          int64_t glo = max(Gr.of((int64_t)bb) - kbase, a) - a, ghi = min(Gr.of((int64_t)(bb + rr.span)) - kbase, b - 1) - a;
          if (glo > ghi) continue;
          for (int64_t ww = (glo >> 5) + lq; ww <= (ghi >> 5); ww += 32) {
            uint32_t m = ~0u;
            if (ww == (glo >> 5)) m &= ~0u << (glo & 31);
            if (ww == (ghi >> 5)) m &= ~0u >> (31 - (ghi & 31));
            atomicOr(pl + ww, m);
          }
        }
      }
    }
  }
  __syncthreads();
  GVO_BMP(if (threadIdx.x == 0) { const long long t = clock64(); php[14] += t - tb0; tb0 = t; })
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // granule-resolution measures over <= 4 planes (wave-unit pieces): per word
  // the popcounts of the 2^T - 1 atoms (bits in exactly the planes of p), and
  // |union of the planes in S| = sum of the atoms p that meet S — T-1 ANDs per
  // atom instead of one OR-select per plane and measure
  bool all_r1 = GVO_BM_ATOMS != 0;
  for (int q = 0; q < U.n_sub; ++q) all_r1 &= U.sub_r[q] == 1;
  if (all_r1 && n_tags <= kAtomTags) {
    if (threadIdx.x < U.n_sub) {
      uint32_t cmq = 0;
      for (uint32_t m = U.sub_mask[threadIdx.x] & tag_mask; m; m &= m - 1)
        cmq |= 1u << __popc(tag_mask & ((1u << (__ffs(m) - 1)) - 1u));
      U.sub_cm[threadIdx.x] = cmq;
    }
    int32_t acc[1 << kAtomTags];
    switch (n_tags) {
      case 1: atom_counts<1>(bm, wp, acc); break;
      case 2: atom_counts<2>(bm, wp, acc); break;
      case 3: atom_counts<3>(bm, wp, acc); break;
      default: atom_counts<4>(bm, wp, acc); break;
    }
    const int np = 1 << n_tags;
#pragma unroll
    for (int p = 1; p < (1 << kAtomTags); ++p) {
      if (p < np) {
        int32_t v = acc[p];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) wmax[p * kNW + w] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x < U.n_sub) {
      const uint32_t cm = U.sub_cm[threadIdx.x];
      int64_t t = 0;
      for (int p = 1; p < np; ++p)
        if (p & cm)
          for (int k = 0; k < kNW; ++k) t += wmax[p * kNW + k];
      U.sub_val[threadIdx.x] = t;
    }
    __syncthreads();
    GVO_BMP(if (threadIdx.x == 0) php[15] += clock64() - tb0;)
    return;
  }
  constexpr int kPcSub = 16, kPcTags = 8;
  if (U.n_sub <= kPcSub && n_tags <= kPcTags) {
    // every requested measure in one pass over the words
    if (threadIdx.x < U.n_sub) {
      uint32_t cmq = 0;
      for (uint32_t m = U.sub_mask[threadIdx.x] & tag_mask; m; m &= m - 1)
        cmq |= 1u << __popc(tag_mask & ((1u << (__ffs(m) - 1)) - 1u));
      U.sub_cm[threadIdx.x] = cmq;
    }
    __syncthreads();
    int32_t c[kPcSub];
#pragma unroll
    for (int q = 0; q < kPcSub; ++q) c[q] = 0;
    for (int64_t i = threadIdx.x; i < wp; i += kNT) {
      uint32_t tw[kPcTags];
#pragma unroll
      for (int t = 0; t < kPcTags; ++t) tw[t] = t < n_tags ? bm[(int64_t)t * wp + i] : 0u;
#pragma unroll
      for (int q = 0; q < kPcSub; ++q) {
        if (q >= U.n_sub) break;
        const uint32_t mask = U.sub_cm[q];
        uint32_t v = 0;
#pragma unroll
        for (int t = 0; t < kPcTags; ++t) v |= ((mask >> t) & 1u) ? tw[t] : 0u;
        const int r = (int)U.sub_r[q];
        c[q] += __popc(r == 1 ? v : bm_lines(v, r));
      }
    }
#pragma unroll
    for (int q = 0; q < kPcSub; ++q) {
      if (q >= U.n_sub) break;
      int32_t v = c[q];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) wmax[q * kNW + w] = v;
    }
    __syncthreads();
    if (threadIdx.x < U.n_sub) {
      int64_t t = 0;
      for (int k = 0; k < kNW; ++k) t += wmax[threadIdx.x * kNW + k];
      U.sub_val[threadIdx.x] = t;
    }
    __syncthreads();
    return;
  }
  for (int q = 0; q < U.n_sub; ++q) {
    uint32_t mask = 0;
    for (uint32_t m = U.sub_mask[q] & tag_mask; m; m &= m - 1)
      mask |= 1u << __popc(tag_mask & ((1u << (__ffs(m) - 1)) - 1u));
    const int r = (int)U.sub_r[q];
    int64_t c = 0;
    for (int64_t i = threadIdx.x; i < wp; i += kNT) {
      uint32_t v = 0;
      for (int t = 0; t < n_tags; ++t)
        if ((mask >> t) & 1u) v |= bm[(int64_t)t * wp + i];
      c += __popc(r == 1 ? v : bm_lines(v, r));
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) wmax[w] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int k = 0; k < kNW; ++k) t += wmax[k];
      U.sub_val[q] = t;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ kernel
struct SetsArgs {
  TplView T;
  const gvo_machine* machines;
  const gvo_config* cfgs;
  const Geo* geos;
  const int64_t* coefs;
  const int64_t* ctabs;
  int64_t n_items;
  int S_req;
  int F_stride;
  int mode;                 // 0 standard, 1 custom wave sets, 2 custom footprint
  int64_t granularity;      // modes 1/2
  const int64_t* run_start; // mode 2 runs
  const int64_t* run_count;
  int n_custom_runs;
  int64_t* counts;          // mode 0: counts rows; modes 1/2: output
  int64_t counts_stride;
  uint8_t* slab;            // per-CTA scratch
  int64_t slab_bytes;
  int64_t run_cap;
  int64_t elem_cap;
  int* status_out;          // modes 1/2: unit status
  int64_t* unit_stats;      // optional [n_items][10]: runs, N, smem?, cycles, key bits, sm, t_runs, t_emit, t_sort, t_sweep
  unsigned long long* work; // dynamic work counter (zeroed before launch)
  WarpArgs warp;            // fused warp-statistics items (appended after the set units)
  int64_t n_warp_items;
  SplitState* split;        // key-range splitting of oversized units (may be null)
  int64_t sm_cap;           // test hook: cap on shared-memory elements (0 = none)
  int32_t seg_off;          // A/B hook: no segment cover
  int32_t pat_off;          // A/B hook: no pattern runs
  int32_t wave_field_major; // wave units ordered field-major (heavy fields first)
  int32_t epoch;            // launch number; queue slots are ready when ready == epoch
  const int64_t* lead;      // mode 0, k_dedup.cu: >= 0 = unit copied from an identical one (skip); may be null
  // mode 0 work lists (k_dedup.cu k_worklist): the wave units, block units
  // and warp items that compute, in item order; counts on the device.  The
  // work queue then hands out list entries only (copied and empty units are
  // never fetched, bundles of block units are dense).  May be null.
  const int32_t* wl_wave;
  const int32_t* wl_blk;
  const int32_t* wl_warp;
  const unsigned long long* wl_cnt;
  const int* run_if;        // residency picked on the device: run only if *run_if == run_if_val
  int run_if_val;
  int handoff;              // micro handoffs on (large batches)
};

// ------------------------------------------------------------------ micro tier
// Small units (one field of one sample block, typically 50-500 intervals)
// are processed by ONE warp: 16 units per CTA concurrently.  The warp builds
// the unit's lattices (warp-cooperative cover), emits the intervals into its
// own shared-memory slice, bitonic-sorts them in place (the sweep needs key
// order only, not stability) and sweeps.  Units that do not fit fall back to
// the CTA path.
#ifndef GVO_TASK_DYN
#define GVO_TASK_DYN 1
#endif
#ifndef GVO_BLOCK_POOL
#define GVO_BLOCK_POOL 0  // A/B: 1 = warp-scheduled block-unit pool (C5 stencil part 330 vs 312 ms: rejected)
#endif
constexpr int kMicroElems = 512;
constexpr int kMicroRuns = 64;          // run offsets kept per warp
constexpr int kMicroRunCap = 256;       // runs per warp in the global slab
struct Handoff {
  int64_t bidx, N, key_lo, key_hi;
  int w, nr;
};
struct MicroCnt {
  int n_runs, status;
  int64_t key_lo, key_hi;
  int64_t N;  // intervals of a handoff
};
constexpr int kMicroBytes = (int)(((sizeof(MicroCnt) + 15) & ~15) + (kMicroRuns + 1) * 8 + kMicroElems * 8);

static_assert(kMicroElems * 8 >= kSegScratch, "segment scratch in the micro element buffer");
static_assert(kNW * 256 * 4 + 256 * 4 + kMaxSub * kNW * 8 + (kSmemRuns + 1) * 8 + kSmemRuns * 8 >= kNW * kSegScratch,
              "segment scratch in the sort/sweep region");
static_assert(((sizeof(UnitSh) + 15) & ~size_t(15)) + kNW * kClassPts * 8 + (size_t)kNW * kMicroBytes <=
                  (size_t)kSetsSmemBytes,
              "micro tier does not fit the set kernel's shared memory");

__device__ __forceinline__ void warp_bitonic(uint64_t* a, int p) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= p; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < p; i += 32) {
        const int l = i ^ j;
        if (l > i) {
          const uint64_t x = a[i], y = a[l];
          const bool up = (i & k) == 0;
          if ((x > y) == up) { a[i] = y; a[l] = x; }
        }
      }
      __syncwarp();
    }
  }
}

// returns false when the unit must be processed by the whole CTA
// Micro units whose intervals or runs exceed the warp's slice take their
// element buffer / run offsets from the CTA's overflow pool (the shared
// memory beyond the micro slices, bump-allocated per bundle) instead of
// falling back to the CTA path, which would build the runs again with 2 of
// its 10 warps busy (C5: those fallbacks were ~23 % of a stencil batch).
#ifndef GVO_MICRO_POOL
#define GVO_MICRO_POOL 0  // A/B (rejected: a warp on a large unit holds its bundle; C2 0.42 -> 1.03 ms, C5 LBM 169 -> 199 ms)
#endif
struct MicroPool {
  uint8_t* base;
  uint32_t bytes;
  unsigned int* used;
};

__device__ __forceinline__ void* micro_alloc(const MicroPool& M, uint32_t bytes) {
  const int lane = threadIdx.x & 31;
  bytes = (bytes + 15u) & ~15u;
  unsigned int off = 0;
  if (lane == 0) off = M.used ? atomicAdd(M.used, bytes) : ~0u;
  off = __shfl_sync(0xffffffffu, off, 0);
  if (!M.used || off > M.bytes || bytes > M.bytes - off) return nullptr;
  return M.base + off;
}

// Returns 1 when the unit is done, 0 when the CTA path must process it from
// scratch, 2 when its runs are built (wruns, metadata in the warp's
// MicroCnt) but its intervals exceed the warp's slice: the CTA emits, sorts
// and sweeps them after the bundle (handoff, GVO_MICRO_HANDOFF) instead of
// building the runs again with the 2 of 10 warps a block unit's few lattice
// tasks keep busy.
#ifndef GVO_MICRO_HANDOFF
#define GVO_MICRO_HANDOFF 1
#endif
__device__ int micro_unit(const SetsArgs& P, int64_t bidx, uint8_t* reg, int64_t* wpts, Run* wruns,
                          const MicroPool& pool) {
  const int lane = threadIdx.x & 31;
  const int F = P.F_stride, S = P.S_req;
  const int64_t c = bidx / ((int64_t)F * S);
  const int f = (int)((bidx / S) % F);
  const int j = (int)(bidx % S);
  const Geo& G = P.geos[c];
  const gvo_config cfg = P.cfgs[c];
  const int tpl = cfg.template_id;
  if (f >= P.T.n_fields[tpl] || !phase_ok(G, 0) || j >= G.n_samples || G.dup_of[f][j] >= 0) return 1;
  if (P.lead && P.lead[(int64_t)F * (P.n_items / ((int64_t)F * (S + 1))) + bidx] >= 0) return 1;
  MicroCnt* cnt = reinterpret_cast<MicroCnt*>(reg);
  int64_t* roff = reinterpret_cast<int64_t*>(reg + ((sizeof(MicroCnt) + 15) & ~size_t(15)));
  uint64_t* el = reinterpret_cast<uint64_t*>(roff + kMicroRuns + 1);
  const gvo_machine& mach = P.machines[cfg.machine_id];
  const Granule Gr = Granule::make(mach.sector_bytes);
  const int64_t R = mach.l1_line_bytes / mach.sector_bytes;
  const int abase = P.T.acc_base[tpl];
  const int64_t* fbase = P.T.field_base + P.T.field_base_off[tpl];
  const int32_t bd[3] = {cfg.block[0], cfg.block[1], cfg.block[2]};
  const int64_t gd[3] = {cfg.grid[0], cfg.grid[1], cfg.grid[2]};
  const int64_t* crow = P.coefs + c * (int64_t)P.T.max_acc * 8;
  const int64_t blk = G.sample_lin[j];
  SegScratch* seg = reinterpret_cast<SegScratch*>(el);  // free until the intervals are emitted
  if (lane == 0) {
    cnt->n_runs = 0;
    cnt->status = GVO_OK;
    cnt->key_lo = INT64_MAX;
    cnt->key_hi = INT64_MIN;
  }
  __syncwarp();
  RunSink sink{wruns, kMicroRunCap, &cnt->n_runs, &cnt->status, &cnt->key_lo, &cnt->key_hi};
  const CTab ct{const_cast<int64_t*>(P.ctabs) + c * ctab_stride(P.T.max_acc), P.T.max_acc};
  const int32_t* fko = P.T.fk_off + tpl * (2 * kMaxFields + 1);
  Box box;
  box.lo[0] = blk % gd[0]; box.lo[1] = (blk / gd[0]) % gd[1]; box.lo[2] = blk / (gd[0] * gd[1]);
  box.n[0] = box.n[1] = box.n[2] = 1;
  for (int kind = 0; kind < 2; ++kind) {
    const int slot = f * 2 + kind;
    // non-affine accesses: points runs
    for (int q = fko[slot] + lane; q < fko[slot + 1]; q += 32) {
      const int a = P.T.fk_list[q];
      if (crow[a * 8 + 7] == kAffine) continue;
      int64_t clo[6], chi[6];
      clo[0] = clo[1] = clo[2] = 0;
      chi[0] = bd[0] - 1; chi[1] = bd[1] - 1; chi[2] = bd[2] - 1;
      run_bid_bounds(blk, 1, gd, clo + 3, chi + 3);
      int64_t lo, hi;
      bounds_check(P.T.code + P.T.code_off[abase + a], P.T.code_len[abase + a], clo, chi, bd, fbase, &lo, &hi);
      const int sr = atomicAdd(&cnt->n_runs, 1);
      if (sr >= kMicroRunCap) { atomicExch(&cnt->status, GVO_ERR_CAPACITY); continue; }
      Run r;
      r.kind = 1; r.access = a; r.tag = kind; r.run_start = blk; r.run_count = 1; r.count = G.tpb;
      r.mono = 0; r.pieces = 1; r.nd = 0; r.base = 0; r.span = 0;
      wruns[sr] = r;
      atomicMin((long long*)&cnt->key_lo, (long long)Gr.of(lo));
      atomicMax((long long*)&cnt->key_hi, (long long)Gr.of(hi));
    }
    // lattices per coefficient class
    const int64_t cl0 = ct.slot_first()[slot], cl1 = ct.slot_first()[slot + 1];
    for (int64_t cls = cl0; cls < cl1; ++cls) {
      const int64_t* ca = crow + ct.rep()[cls] * 8;
      const WLat L0 = box_lattice(ca, bd, box, Gr);
      const int64_t* cp = ct.pts() + ct.start()[cls];
      const int64_t np = ct.cnt()[cls];
      for (int64_t p0 = 0; p0 < np; p0 += kClassPts) {
        const int m = (int)((np - p0) < kClassPts ? (np - p0) : kClassPts);
        __syncwarp();
        for (int k = lane; k < m; k += 32) wpts[k] = (int64_t)((uint64_t)L0.base + (uint64_t)cp[p0 + k]);
        __syncwarp();
        if (P.seg_off || !cover_segments(sink, L0, wpts, m, kind, Gr, seg, false))
          cover_warp(sink, L0, wpts, m, kind, Gr);
      }
    }
  }
  __syncwarp();
  const int nr = cnt->n_runs;
  if (cnt->status != GVO_OK) return 0;
#if GVO_MICRO_HANDOFF
  {
    int64_t nl = 0;
    for (int r = lane; r < nr; r += 32) nl += wruns[r].count;
    for (int o = 16; o; o >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, o);
    if (nr > kMicroRuns || nl > kMicroElems) {
      const int64_t kb = nr ? floordiv(cnt->key_lo, R) * R : 0;
      if (nl > P.elem_cap || nr > kMicroRunCap ||
          (nr && (uint64_t)(cnt->key_hi - kb) >= (uint64_t(1) << kKeyBits)))
        return 0;
      if (lane == 0) cnt->N = nl;
      __syncwarp();
      return 2;
    }
  }
#endif
  if (nr > kMicroRuns) {  // run offsets from the overflow pool
    if (!GVO_MICRO_POOL || nr > kMicroRunCap) return 0;
    roff = reinterpret_cast<int64_t*>(micro_alloc(pool, (uint32_t)(nr + 1) * 8u));
    if (!roff) return 0;
  }
  // offsets
  if (lane == 0) {
    int64_t acc = 0;
    for (int r = 0; r < nr; ++r) { roff[r] = acc; acc += wruns[r].count; }
    roff[nr] = acc;
  }
  __syncwarp();
  const int64_t N = roff[nr];
  const int64_t kbase = nr ? floordiv(cnt->key_lo, R) * R : 0;
  if (nr && (uint64_t)(cnt->key_hi - kbase) >= (uint64_t(1) << kKeyBits)) return 0;
  int p = 32;
  while (p < N) p <<= 1;
  if (N > kMicroElems) {  // element buffer from the overflow pool
    if (!GVO_MICRO_POOL || N > (int64_t)(pool.bytes / 8)) return 0;
    el = reinterpret_cast<uint64_t*>(micro_alloc(pool, (uint32_t)p * 8u));
    if (!el) return 0;
  }
  const int64_t tpb = G.tpb;
  for (int64_t i = lane; i < p; i += 32) {
    if (i >= N) { el[i] = ~0ull; continue; }
    int lo = 0, hi = nr - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (roff[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const Run& rr = wruns[lo];
    int64_t glo, ghi;
    run_interval(rr, i - roff[lo], Gr, P.T, abase, fbase, bd, gd, tpb, &glo, &ghi);
    el[i] = ((uint64_t)(glo - kbase) << kKeyShift) | ((uint64_t)(ghi - glo) << kTagBits) | (uint64_t)rr.tag;
  }
  __syncwarp();
  warp_bitonic(el, p);
  // sweep: loads (sectors), loads (lines), stores (sectors)
  const uint32_t masks[3] = {1u, 1u, 2u};
  const int64_t rs[3] = {1, R, 1};
  int rsh = -1;
  if ((R & (R - 1)) == 0) { rsh = 0; while ((int64_t(1) << rsh) < R) ++rsh; }
  const int sub = p / 32;
  const int lb = lane * sub;
  int64_t res[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int64_t mx = -1;
    for (int i = lb; i < lb + sub && i < N; ++i) {
      const uint64_t x = el[i];
      if (!((masks[q] >> (x & 31u)) & 1u)) continue;
      int64_t hi0 = (int64_t)(x >> kKeyShift) + (int64_t)((x >> kTagBits) & kLenMask);
      if (rs[q] != 1) hi0 = rsh >= 0 ? hi0 >> rsh : hi0 / rs[q];
      mx = max(mx, hi0);
    }
    int64_t inc = mx;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc = max(inc, t);
    }
    int64_t Rm = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) Rm = -1;
    int64_t cntv = 0;
    for (int i = lb; i < lb + sub && i < N; ++i) {
      const uint64_t x = el[i];
      if (!((masks[q] >> (x & 31u)) & 1u)) continue;
      int64_t lo0 = (int64_t)(x >> kKeyShift);
      int64_t hi0 = lo0 + (int64_t)((x >> kTagBits) & kLenMask);
      if (rs[q] != 1) {
        lo0 = rsh >= 0 ? lo0 >> rsh : lo0 / rs[q];
        hi0 = rsh >= 0 ? hi0 >> rsh : hi0 / rs[q];
      }
      if (lo0 > Rm) cntv += hi0 - lo0 + 1;
      else if (hi0 > Rm) cntv += hi0 - Rm;
      Rm = max(Rm, hi0);
    }
    for (int o = 16; o; o >>= 1) cntv += __shfl_xor_sync(0xffffffffu, cntv, o);
    res[q] = cntv;
  }
  if (lane == 0) {
    int64_t* row = P.counts + c * P.counts_stride;
    int64_t* b = row + GVO_C_HDR + ((int64_t)j * P.F_stride + f) * 5;
    b[0] = res[0];
    b[2] = res[1];
    b[3] = res[2];
  }
  __syncwarp();
  return 1;
}

// Write a finished unit's measures (union counts per subset) to the outputs.
template <class V>
__device__ void write_unit_outputs(const SetsArgs& P, int64_t c, int field, int kind, int j, int n_uw,
                                   const V* v /* [n_sub] */) {
  const int f = field;
  if (P.mode == 0) {
    int64_t* row = P.counts + c * P.counts_stride;
    if (kind == 0) {
      int64_t* b = row + GVO_C_HDR + ((int64_t)j * P.F_stride + f) * 5;
      b[0] = (int64_t)v[0];
      b[2] = (int64_t)v[1];
      b[3] = (int64_t)v[2];
    } else {
      int64_t* wv = row + GVO_C_HDR + (int64_t)P.S_req * P.F_stride * 5;
      for (int u = 0; u < n_uw; ++u) {
        int64_t* o = wv + ((int64_t)u * P.F_stride + f) * 4;
        o[0] = (int64_t)v[4 * u + 0];
        o[1] = (int64_t)v[4 * u + 1];
        o[2] = (int64_t)v[4 * u + 2];
        o[3] = u ? (int64_t)(v[4 * u] + v[4 * (u - 1)] - v[4 * u + 3]) : 0;
      }
    }
  } else if (P.mode == 1) {
    for (int u = 0; u < n_uw; ++u) {
      int64_t* o = P.counts + ((int64_t)u * P.F_stride + f) * 4;
      o[0] = (int64_t)v[4 * u + 0];
      o[1] = (int64_t)v[4 * u + 1];
      o[2] = (int64_t)v[4 * u + 2];
      o[3] = u ? (int64_t)(v[4 * u] + v[4 * (u - 1)] - v[4 * u + 3]) : 0;
    }
  } else {
    P.counts[f * 2 + 0] = (int64_t)v[0];
    P.counts[f * 2 + 1] = (int64_t)v[1];
  }
}

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__global__ void __launch_bounds__(kNT, kSetsCtasPerSm) k_sets(SetsArgs P) {
  if (P.run_if && *P.run_if != P.run_if_val) return;  // the other residency runs this batch
  extern __shared__ __align__(16) uint8_t smem[];
  UnitSh& U = *reinterpret_cast<UnitSh*>(smem);
  size_t off = (sizeof(UnitSh) + 15) & ~size_t(15);
  int64_t* cpts = reinterpret_cast<int64_t*>(smem + off); off += kNW * kClassPts * 8;
  uint8_t* micro_region = smem + off;  // reused by the warp-per-unit tier
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + off); off += kNW * 256 * 4;
  uint32_t* tot = reinterpret_cast<uint32_t*>(smem + off); off += 256 * 4;
  int64_t* wmax = reinterpret_cast<int64_t*>(smem + off); off += kMaxSub * kNW * 8;
  int64_t* roff_sh = reinterpret_cast<int64_t*>(smem + off); off += (kSmemRuns + 1) * 8;
  int64_t* rka_sh = reinterpret_cast<int64_t*>(smem + off); off += kSmemRuns * 8;
  uint64_t* ebuf = reinterpret_cast<uint64_t*>(smem + off);
  const int64_t sm_elems = P.sm_cap > 0 ? min((int64_t)(kSetsSmemBytes - off) / 16, P.sm_cap)
                                         : (int64_t)(kSetsSmemBytes - off) / 16;

  uint8_t* slab = P.slab + (int64_t)blockIdx.x * P.slab_bytes;
  Run* runs = reinterpret_cast<Run*>(slab);
  int64_t* roff_gl = reinterpret_cast<int64_t*>(slab + P.run_cap * sizeof(Run));
  int64_t* rka_gl = roff_gl + (P.run_cap + 1);
  uint64_t* gbuf = reinterpret_cast<uint64_t*>(slab + P.run_cap * sizeof(Run) + 2 * (P.run_cap + 1) * 8);
  SplitState* SS = P.split;

  __shared__ int64_t next_item;
  __shared__ int next_kind;  // 0 main item, 1 range item, 2 exit
  __shared__ RangeItem cur_range;
  __shared__ int main_done;
  __shared__ int64_t fb_list[kNW];  // micro units that fell back to the CTA path
  __shared__ int fb_n, fb_i;
  __shared__ int64_t stat_idx;
  __shared__ long long t_runs_sh;
  // debug phase accounting (thread 0): 0 fetch wait, 1 warp items, 2 micro
  // bundles, 3 unit run building, 4 unit sort/sweep, 5 range counting,
  // 6 range bitmap, 7 range emit/sort/sweep, 8 ranges, 9 bitmap ranges,
  // 10 sum range N, 11 sum range runs
  GVO_PH(__shared__ long long ph[16];)
  GVO_PH(if (threadIdx.x < 16) ph[threadIdx.x] = 0;)
  if (threadIdx.x == 0) { main_done = 0; fb_n = 0; fb_i = 0; }
  // micro overflow pool: the shared memory beyond the micro slices (reset per bundle at fetch)
  __shared__ unsigned int pool_used;
  // micro handoffs of the current bundle (reset at fetch)
  __shared__ Handoff ho[kNW];
  __shared__ int ho_n;
  const size_t pool_off = ((size_t)(micro_region - smem) + (size_t)kNW * kMicroBytes + 15) & ~size_t(15);
  const MicroPool mpool{smem + pool_off, (uint32_t)(kSetsSmemBytes > (int)pool_off ? kSetsSmemBytes - pool_off : 0),
                        &pool_used};
  // item space (mode 0): wave units | bundles of kNW block units (micro) | warp items;
  // block units falling back to the CTA path re-enter as kBlkBase + index
  const bool micro_on = P.mode == 0 && P.S_req > 0;
  const int64_t n_cfg_u = P.mode == 0 ? P.n_items / ((int64_t)P.F_stride * (P.S_req + 1)) : 0;
  const int64_t n_wave_u = n_cfg_u * P.F_stride;
  const int64_t n_blk_u = n_cfg_u * P.F_stride * P.S_req;
  const int64_t n_bund = micro_on ? (n_blk_u + kNW - 1) / kNW : 0;
  const int64_t n_set_main = micro_on ? n_wave_u + n_bund : P.n_items;
  const int64_t n_main = n_set_main + P.n_warp_items;
  // work lists: the queue runs over list entries (virtual items), mapped back
  // to the item space at fetch
  const bool use_wl = micro_on && P.wl_cnt != nullptr;
  const int64_t n_wave_l = use_wl ? (int64_t)P.wl_cnt[0] : n_wave_u;
  const int64_t n_blk_l = use_wl ? (int64_t)P.wl_cnt[1] : n_blk_u;
  const int64_t n_bund_l = use_wl ? (n_blk_l + kNW - 1) / kNW : n_bund;
  const int64_t n_set_main_l = use_wl ? n_wave_l + n_bund_l : n_set_main;
  const int64_t n_main_l = use_wl ? n_set_main_l + (P.n_warp_items > 0 ? (int64_t)P.wl_cnt[2] : 0) : n_main;
  const int64_t kBlkBase = int64_t(1) << 40;

#if defined(GVO_DEBUG_SYNC) && GVO_DEBUG_SYNC
  // debug build: every warp counts its passes through the item loop; after
  // the fetch barrier thread 0 checks that all warps are on the same pass
  __shared__ int dbg_iter[kNW];
  if ((threadIdx.x & 31) == 0) dbg_iter[threadIdx.x >> 5] = 0;
  __syncthreads();
#endif
  for (;;) {
#if defined(GVO_DEBUG_SYNC) && GVO_DEBUG_SYNC
    if ((threadIdx.x & 31) == 0) dbg_iter[threadIdx.x >> 5] += 1;
#endif
    // ---------------- fetch: queued key ranges first, then main items
    const long long t_fetch = clock64();
    if (threadIdx.x == 0) {
      int kind = 2;
      int64_t it = -1;
      // a unit that may split needs one of this CTA's descriptor slots free
      auto slot_free = [&]() {
        if (!SS) return true;
        const volatile int32_t* sb = SS->slot_busy + (int64_t)blockIdx.x * kSplitSlotsPerCta;
        for (int q = 0; q < kSplitSlotsPerCta; ++q)
          if (sb[q] == 0) return true;
        return false;
      };
      for (;;) {
        if (fb_i < fb_n && slot_free()) {
          kind = 0;
          it = kBlkBase + fb_list[fb_i++];
          if (fb_i == fb_n) fb_i = fb_n = 0;
          if (SS) atomicAdd(&SS->pending, 1ull);
          break;
        }
        if (SS) {
          const unsigned long long t = min(vload(&SS->qtail), (unsigned long long)SS->q_cap);
          const unsigned long long h = vload(&SS->qhead);
          if (h < t) {
            if (atomicCAS(&SS->qhead, h, h + 1) == h) {
              volatile int32_t* rd = &SS->queue[h].ready;
              while (*rd != P.epoch) __nanosleep(64);
              __threadfence();
              cur_range = SS->queue[h];
              if (cur_range.desc < 0) {  // a micro unit handed back to the CTA path
                kind = 0;
                it = kBlkBase + (-1 - cur_range.desc);
              } else {
                kind = 1;
              }
              break;
            }
            continue;
          }
        }
        if (!main_done) {
          // wave units (mode 0) and custom units may split; bundles and warp
          // items never do (the counter only grows, so a peek past the wave
          // units stays past them)
          const int64_t peek = (int64_t)vload(P.work);
          const bool may_split = P.mode != 0 || peek < n_wave_l;
          if (!may_split || slot_free()) {
            const unsigned long long m = atomicAdd(P.work, 1ull);
            if ((int64_t)m < n_main_l) {
              kind = 0;
              it = (int64_t)m;
              if (use_wl) {  // list entry -> item (bundles stay virtual: their warps read the block list)
                if (it < n_wave_l) it = P.wl_wave[it];
                else if (it < n_set_main_l) it = n_wave_u + (it - n_wave_l);
                else it = n_set_main + P.wl_warp[it - n_set_main_l];
              }
              if (SS) atomicAdd(&SS->pending, 1ull);
              break;
            }
            main_done = 1;
          }
        }
        if (!SS || (main_done && fb_n == 0 && vload(&SS->pending) == 0 &&
                    vload(&SS->qhead) >= min(vload(&SS->qtail), (unsigned long long)SS->q_cap)))
          break;
        __nanosleep(256);
      }
      next_kind = kind;
      pool_used = 0;
      ho_n = 0;
      next_item = it;
    }
    __syncthreads();
    const int kind_fetched = next_kind;
    const int64_t item = next_item;
#if defined(GVO_DEBUG_SYNC) && GVO_DEBUG_SYNC
    if (threadIdx.x == 0) {
      for (int w = 1; w < kNW; ++w)
        if (dbg_iter[w] != dbg_iter[0]) {
          printf("GVO_DEBUG_SYNC block %d: warp %d on pass %d, warp 0 on pass %d (kind %d item %lld)\n", blockIdx.x, w,
                 dbg_iter[w], dbg_iter[0], kind_fetched, (long long)item);
          break;
        }
    }
#endif
    GVO_PH(if (threadIdx.x == 0) ph[0] += clock64() - t_fetch;)
    if (kind_fetched == 2) break;

    int64_t range_a = 0, range_b = 0;
    SplitHdr* hdr = nullptr;
    bool in_range = kind_fetched == 1;
    const long long t_start = clock64();
    // emission + sort + sweeps + outputs of an unsplit unit described by U,
    // runs urun[0, U.n_runs) with offsets roff: the CTA path's units and the
    // micro tier's handoffs (runs built by one warp, too many intervals for
    // its slice)
    auto finish_unsplit = [&](const Run* urun, int64_t* roff) {
      const int64_t c = U.cfg;
      const Geo& G = P.geos[c];
      const gvo_config cfg = P.cfgs[c];
      const int tpl = cfg.template_id;
      const int abase = P.T.acc_base[tpl];
      const int64_t* fbase = P.T.field_base + P.T.field_base_off[tpl];
      const int32_t bd[3] = {cfg.block[0], cfg.block[1], cfg.block[2]};
      const int64_t gd[3] = {cfg.grid[0], cfg.grid[1], cfg.grid[2]};
      const Granule Gr = Granule::make(U.g);
      const int64_t tpb = G.tpb;
      const int nr = min(U.n_runs, (int)P.run_cap);
      const long long t_runs = t_runs_sh;
    const int64_t N = U.N;
      uint64_t* A0;
      uint64_t* B0;
      if (N <= sm_elems) { A0 = ebuf; B0 = ebuf + sm_elems; }
      else { A0 = gbuf; B0 = gbuf + P.elem_cap; }
      const int64_t kbase = U.key_lo;

      // ---------------- emission: each thread owns a contiguous element range
      // (one binary search for its first run, then a cursor), outer-tuple
      // decode in 32-bit arithmetic when the run's extents allow it.
      {
        const int64_t per = (N + kNT - 1) / kNT;
        const int64_t e0 = min(N, (int64_t)threadIdx.x * per), e1 = min(N, e0 + per);
        int ri = 0;
        if (e0 < e1) {
          int lo = 0, hi = nr - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (roff[mid] <= e0) lo = mid; else hi = mid - 1;
          }
          ri = lo;
        }
        for (int64_t i = e0; i < e1; ++i) {
          while (roff[ri + 1] <= i) ++ri;
          const Run& r = urun[ri];
          int64_t k = i - roff[ri];
          int64_t glo, ghi;
          if (r.kind == 0) {
            int64_t piece = 0;
            if (r.pieces > 1) { piece = k % r.pieces; k /= r.pieces; }
            uint64_t b = (uint64_t)r.base;
            if (k < (int64_t(1) << 31)) {
              uint32_t k32 = (uint32_t)k;
              for (int d = r.nd - 1; d >= 0; --d) {
                const uint32_t ex = (uint32_t)r.ext[d];
                const uint32_t q = ex ? k32 / ex : 0;
                b += (uint64_t)r.stride[d] * (uint64_t)(k32 - q * ex);
                k32 = q;
              }
            } else {
              for (int d = r.nd - 1; d >= 0; --d) {
                const int64_t idx = k % r.ext[d];
                k /= r.ext[d];
                b += (uint64_t)r.stride[d] * (uint64_t)idx;
              }
            }
            glo = Gr.of((int64_t)b);
            ghi = Gr.of((int64_t)(b + r.span));
            if (r.pieces > 1) {
              int64_t plo = glo + piece * kPiece;
              if (plo > ghi) plo = glo;
              const int64_t phi = min(ghi, plo + kPiece - 1);
              glo = plo;
              ghi = phi;
            }
          } else {
            const int64_t blk = r.run_start + k / tpb;
            const int64_t th = k % tpb;
            int64_t crd[6];
            crd[0] = th % bd[0];
            crd[1] = (th / bd[0]) % bd[1];
            crd[2] = th / ((int64_t)bd[0] * bd[1]);
            crd[3] = blk % gd[0];
            crd[4] = (blk / gd[0]) % gd[1];
            crd[5] = blk / (gd[0] * gd[1]);
            const int ga = abase + r.access;
            glo = ghi = Gr.of(eval_point(P.T.code + P.T.code_off[ga], P.T.code_len[ga], crd, bd, fbase));
          }
          A0[i] = ((uint64_t)(glo - kbase) << kKeyShift) | ((uint64_t)(ghi - glo) << kTagBits) |
                  (uint64_t)r.tag;
        }
      }
      __syncthreads();

      const long long t_emit = clock64();
      // ---------------- sort + sweeps
      int kb = 0;
      {
        uint64_t span = (uint64_t)(U.key_hi - kbase);
        while (span) { ++kb; span >>= 1; }
      }
      const int nbits = ((kb + 7) / 8) * 8;
      const uint64_t* sorted = cta_sort(A0, B0, N, kKeyShift, nbits, hist, tot);
      const long long t_sort = clock64();
      sweep(sorted, N, U, wmax);
      const long long t_sweep = clock64();
      GVO_PH(if (threadIdx.x == 0) ph[4] += t_sweep - t_runs;)

      // ---------------- outputs
      if (threadIdx.x == 0 && P.unit_stats) {
        int64_t* us = P.unit_stats + stat_idx * 10;
        us[6] = t_runs - t_start;
        us[7] = t_emit - t_runs;
        us[8] = t_sort - t_emit;
        us[9] = t_sweep - t_sort;
        us[0] = nr;
        us[1] = N;
        us[2] = N <= sm_elems;
        us[3] = clock64() - t_start;
        us[4] = nbits;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        us[5] = smid;
      }
      if (threadIdx.x == 0) write_unit_outputs(P, c, U.field, U.kind, U.j, P.mode == 2 ? 0 : G.n_uw, U.sub_val);
    };

    if (!in_range && item >= n_set_main && item < kBlkBase) {
#if defined(GVO_DEBUG_SYNC) && GVO_DEBUG_SYNC
      if (threadIdx.x < 3) gvo_dbg_wexit[threadIdx.x] = 0;
#endif
      warp_item(P.warp, item - n_set_main, reinterpret_cast<unsigned long long*>(ebuf));
      __syncthreads();
#if defined(GVO_DEBUG_SYNC) && GVO_DEBUG_SYNC
      if (threadIdx.x == 0 && gvo_dbg_wexit[0] != kNW && gvo_dbg_wexit[1] != kNW && gvo_dbg_wexit[2] != kNW)
        printf("GVO_DEBUG_SYNC block %d: warp item %lld exits %d/%d/%d\n", blockIdx.x, (long long)(item - n_set_main),
               gvo_dbg_wexit[0], gvo_dbg_wexit[1], gvo_dbg_wexit[2]);
      __syncthreads();
#endif
      GVO_PH(if (threadIdx.x == 0) ph[1] += clock64() - t_start;)
      if (threadIdx.x == 0 && SS) atomicAdd(&SS->pending, ~0ull);
      continue;
    }
    if (!in_range && micro_on && item >= n_wave_u && item < n_set_main) {
      // block units, one per warp: the bundle's kNW units.  A/B
      // GVO_BLOCK_POOL=1: a bundle item lets the CTA join a block-unit pool
      // (every warp takes units from a global counter until it is drained,
      // no CTA barrier between units) — slower on C5 (330 vs 312 ms for the
      // stencil part): the CTAs in the pool stop taking queued key ranges
      // and CTA-path fallbacks, which then pile up in the tail.
      const int w = threadIdx.x >> 5;
#if GVO_BLOCK_POOL
      for (;;) {
        unsigned long long v = 0;
        if ((threadIdx.x & 31) == 0) v = atomicAdd(P.work + 1, 1ull);
        v = __shfl_sync(0xffffffffu, v, 0);
        if ((int64_t)v >= n_blk_l) break;
        const int64_t bidx = use_wl ? (int64_t)P.wl_blk[v] : (int64_t)v;
#else
      for (int once = 0; once < 1; ++once) {
        int64_t bidx = (item - n_wave_u) * kNW + w;
        if (use_wl) bidx = bidx < n_blk_l ? P.wl_blk[bidx] : n_blk_u;
        if (bidx >= n_blk_u) break;
#endif
        const int res0 = micro_unit(P, bidx, micro_region + w * kMicroBytes, cpts + w * kClassPts,
                                    runs + w * kMicroRunCap, mpool);
        // the pool has no per-bundle handoff list; small batches spread the
        // large units over idle CTAs through the queue instead (C2: 0.45 vs
        // 0.56 ms with handoffs)
        const int res = (GVO_BLOCK_POOL || !P.handoff) && res0 == 2 ? 0 : res0;
        if (res == 2 && (threadIdx.x & 31) == 0) {  // runs built: the CTA finishes it after the bundle
          const MicroCnt* mc = reinterpret_cast<const MicroCnt*>(micro_region + w * kMicroBytes);
          Handoff& H = ho[atomicAdd(&ho_n, 1)];
          H.bidx = bidx;
          H.N = mc->N;
          H.key_lo = mc->key_lo;
          H.key_hi = mc->key_hi;
          H.w = w;
          H.nr = mc->n_runs;
        }
        if (res == 0 && (threadIdx.x & 31) == 0) {
          bool queued = false;
          if (SS) {
            atomicAdd(&SS->pending, 1ull);
            const unsigned long long slot = atomicAdd(&SS->qtail, 1ull);
            if ((int64_t)slot < SS->q_cap) {
              RangeItem it;
              it.desc = -1 - bidx;
              it.a = it.b = 0;
              it.ready = 0;
              it.pad = 0;
              SS->queue[slot] = it;
              __threadfence();
              *reinterpret_cast<volatile int32_t*>(&SS->queue[slot].ready) = P.epoch;
              queued = true;
            } else {
              atomicAdd(&SS->pending, ~0ull);
            }
          }
          if (!queued) {
            const int q = atomicAdd(&fb_n, 1);
            if (q < kNW) {
              fb_list[q] = bidx;
            } else {  // local list full too: the configuration fails loudly
              atomicSub(&fb_n, 1);
              int64_t* row = P.counts + (bidx / ((int64_t)P.F_stride * P.S_req)) * P.counts_stride;
              atomicExch((unsigned long long*)&row[GVO_C_STATUS], (unsigned long long)GVO_ERR_CAPACITY);
            }
          }
        }
        __syncwarp();
      }
      __syncthreads();
      // handoffs: units whose runs a warp built but whose intervals exceed
      // its slice — emission, sort, sweep and outputs by the whole CTA
      const int nho = ho_n;
      for (int h = 0; h < nho; ++h) {
        const int hnr = ho[h].nr;
        const Run* urun = runs + ho[h].w * kMicroRunCap;
        if (threadIdx.x == 0) {
          const Handoff& H = ho[h];
          const int64_t c = H.bidx / ((int64_t)P.F_stride * P.S_req);
          const gvo_machine& mach = P.machines[P.cfgs[c].machine_id];
          const int64_t R = mach.l1_line_bytes / mach.sector_bytes;
          U.cfg = c;
          U.field = (int)((H.bidx / P.S_req) % P.F_stride);
          U.j = (int)(H.bidx % P.S_req);
          U.kind = 0;
          U.status = GVO_OK;
          U.n_runs = hnr;
          U.N = H.N;
          U.g = mach.sector_bytes;
          U.R = R;
          U.key_lo = hnr ? floordiv(H.key_lo, R) * R : 0;
          U.key_hi = H.key_hi;
          U.n_sub = 3;
          U.sub_mask[0] = 1; U.sub_r[0] = 1;  // load sectors
          U.sub_mask[1] = 1; U.sub_r[1] = R;  // load lines
          U.sub_mask[2] = 2; U.sub_r[2] = 1;  // store sectors
          for (int q = 0; q < 3; ++q) {
            const int64_t r = U.sub_r[q];
            int sh = -1;
            if (r > 0 && (r & (r - 1)) == 0) { sh = 0; while ((int64_t(1) << sh) < r) ++sh; }
            U.sub_sh[q] = sh;
          }
          stat_idx = n_wave_u + H.bidx;
          t_runs_sh = clock64();
        }
        // run offsets (<= kMicroRunCap runs): exclusive scan by warp 0
        if (threadIdx.x < 32) {
          int64_t carry = 0;
          for (int r0 = 0; r0 < hnr; r0 += 32) {
            const int r = r0 + (int)threadIdx.x;
            const int64_t v = r < hnr ? urun[r].count : 0;
            int64_t inc = v;
            for (int o = 1; o < 32; o <<= 1) {
              const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
              if ((int)threadIdx.x >= o) inc += t;
            }
            if (r < hnr) roff_sh[r] = carry + inc - v;
            carry += __shfl_sync(0xffffffffu, inc, 31);
          }
          if (threadIdx.x == 0) roff_sh[hnr] = carry;
        }
        __syncthreads();
        finish_unsplit(urun, roff_sh);
        __syncthreads();
      }
      __syncthreads();  // every thread has read ho_n before the next fetch resets it
      if (threadIdx.x == 0 && P.unit_stats && SS) {
        const unsigned long long slot =
            atomicAdd(reinterpret_cast<unsigned long long*>(P.unit_stats + P.n_items * 10), 1ull);
        if (slot < 4096) {
          int64_t* us = P.unit_stats + P.n_items * 10 + 10 + slot * 10;
          us[0] = -1; us[1] = item; us[2] = fb_n; us[3] = 0; us[4] = clock64() - t_start; us[5] = 0;
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          us[6] = smid; us[7] = 0; us[8] = 3;
        }
      }
      GVO_PH(if (threadIdx.x == 0) ph[2] += clock64() - t_start;)
      if (threadIdx.x == 0 && SS) atomicAdd(&SS->pending, ~0ull);
      continue;
    }

    if (!in_range) {
    // ---------------- unit description
      if (threadIdx.x == 0) {
        U.status = GVO_OK;
        U.n_runs = 0;
        U.has_pattern = 0;
        U.key_lo = INT64_MAX;
        U.key_hi = INT64_MIN;
        U.n_src = 0;
        U.n_sub = 0;
        int64_t c, f;
        int j = 0;
        bool skip = false;
        if (P.mode == 0) {
          if (item < n_wave_u) {
            // field-major: every config's first field (the stencil source /
            // pdf pull field: the heavy units) before the lighter ones
            if (P.wave_field_major) { f = item / n_cfg_u; c = item % n_cfg_u; }
            else { c = item / P.F_stride; f = item % P.F_stride; }
            j = P.S_req;
            stat_idx = item;
          } else {
            const int64_t r = item >= kBlkBase ? item - kBlkBase : item - n_wave_u;
            c = r / ((int64_t)P.F_stride * P.S_req);
            f = (r / P.S_req) % P.F_stride;
            j = (int)(r % P.S_req);
            stat_idx = n_wave_u + r;
          }
        } else {
          c = 0;
          f = item;
          stat_idx = item;
        }
        const Geo& G = P.geos[c];
        const gvo_config& cfg = P.cfgs[c];
        if (f >= P.T.n_fields[cfg.template_id]) skip = true;
        if (P.mode == 0 && !phase_ok(G, j < P.S_req ? 0 : 1)) skip = true;
        // identical unit of another configuration (k_dedup.cu): copied after the launch
        if (P.mode == 0 && P.lead && !skip &&
            P.lead[j < P.S_req ? n_wave_u + (c * P.F_stride + f) * P.S_req + j : c * P.F_stride + f] >= 0)
          skip = true;
        U.cfg = c;
        U.field = (int)f;
        U.j = j;
        if (!skip && P.mode == 0 && j < P.S_req) {
          if (j >= G.n_samples || G.dup_of[f][j] >= 0) skip = true;
          else {
            U.kind = 0;
            U.n_src = 2;
            for (int k = 0; k < 2; ++k) {
              U.src_start[k] = G.sample_lin[j];
              U.src_count[k] = 1;
              U.src_kind[k] = k;
              U.src_tag[k] = k;
            }
            U.n_sub = 3;
            U.sub_mask[0] = 1; U.sub_r[0] = 1;            // load sectors
            U.sub_mask[1] = 1; U.sub_r[1] = 1;            // load lines (r set below)
            U.sub_mask[2] = 2; U.sub_r[2] = 1;            // store sectors
          }
        } else if (!skip && P.mode != 2) {
          U.kind = 1;
          U.n_src = 2 * G.n_uw;
          for (int u = 0; u < G.n_uw; ++u)
            for (int k = 0; k < 2; ++k) {
              U.src_start[2 * u + k] = G.uw_start[u];
              U.src_count[2 * u + k] = G.uw_count[u];
              U.src_kind[2 * u + k] = k;
              U.src_tag[2 * u + k] = 2 * u + k;
            }
          int q = 0;
          for (int u = 0; u < G.n_uw; ++u) {
            U.sub_mask[q] = 1u << (2 * u); U.sub_r[q++] = 1;
            U.sub_mask[q] = 1u << (2 * u + 1); U.sub_r[q++] = 1;
            U.sub_mask[q] = 3u << (2 * u); U.sub_r[q++] = 1;
            U.sub_mask[q] = u ? (1u << (2 * u)) | (1u << (2 * u - 2)) : 0u; U.sub_r[q++] = 1;
          }
          U.n_sub = q;
        } else if (!skip) {
          U.kind = 2;
          U.n_src = 0;
          if (2 * P.n_custom_runs > kMaxSrc) { skip = true; atomicExch(P.status_out, GVO_ERR_UNSUPPORTED); }
          for (int r = 0; r < P.n_custom_runs && U.n_src + 2 <= kMaxSrc; ++r)
            for (int k = 0; k < 2; ++k) {
              U.src_start[U.n_src] = P.run_start[r];
              U.src_count[U.n_src] = P.run_count[r];
              U.src_kind[U.n_src] = k;
              U.src_tag[U.n_src] = k;
              ++U.n_src;
            }
          U.n_sub = 2;
          U.sub_mask[0] = 1; U.sub_r[0] = 1;
          U.sub_mask[1] = 2; U.sub_r[1] = 1;
        }
        if (skip) U.n_src = -1;
      }
      __syncthreads();
      __syncthreads();
      if (U.n_src < 0) {
        if (threadIdx.x == 0 && SS) atomicAdd(&SS->pending, ~0ull);
        __syncthreads();
        continue;
      }
    }

    // ---------------- main unit: run building, element count
    if (!in_range) {
    const int64_t c = U.cfg;
      const Geo& G = P.geos[c];
      const gvo_config cfg = P.cfgs[c];
      const int tpl = cfg.template_id;
      const int abase = P.T.acc_base[tpl];
      const int64_t* fbase = P.T.field_base + P.T.field_base_off[tpl];
      const int32_t bd[3] = {cfg.block[0], cfg.block[1], cfg.block[2]};
      const int64_t gd[3] = {cfg.grid[0], cfg.grid[1], cfg.grid[2]};
      const int64_t* crow = P.coefs + c * (int64_t)P.T.max_acc * 8;
      const gvo_machine& mach = P.machines[cfg.machine_id];
      const int64_t g = P.mode == 0 ? mach.sector_bytes : P.granularity;
      const Granule Gr = Granule::make(g);
      const int64_t R = P.mode == 0 ? mach.l1_line_bytes / mach.sector_bytes : 1;
      if (threadIdx.x == 0) {
        U.g = g;
        U.R = R;
        if (U.kind == 0) U.sub_r[1] = R;
        for (int q = 0; q < U.n_sub; ++q) {
          const int64_t r = U.sub_r[q];
          int sh = -1;
          if (r > 0 && (r & (r - 1)) == 0) { sh = 0; while ((int64_t(1) << sh) < r) ++sh; }
          U.sub_sh[q] = sh;
        }
      }
      const int64_t tpb = G.tpb;
      RunSink sink{runs, (int)P.run_cap, &U.n_runs, &U.status, &U.key_lo, &U.key_hi, &U.has_pattern};
      __syncthreads();

      // ---------------- run building
      // (a) points runs for non-affine accesses: one task per (source, access)
      const int32_t* fko = P.T.fk_off + tpl * (2 * kMaxFields + 1);
      for (int task = threadIdx.x; task < U.n_src * 64; task += kNT) {
        const int s = task >> 6;
        const int slot = U.field * 2 + U.src_kind[s];
        const int fk = fko[slot], na = fko[slot + 1] - fk;
        for (int q = task & 63; q < na; q += 64) {
          const int a = P.T.fk_list[fk + q];
          if (crow[a * 8 + 7] == kAffine) continue;
          int64_t clo[6], chi[6];
          clo[0] = clo[1] = clo[2] = 0;
          chi[0] = bd[0] - 1; chi[1] = bd[1] - 1; chi[2] = bd[2] - 1;
          run_bid_bounds(U.src_start[s], U.src_count[s], gd, clo + 3, chi + 3);
          int64_t lo, hi;
          const int ga = abase + a;
          bounds_check(P.T.code + P.T.code_off[ga], P.T.code_len[ga], clo, chi, bd, fbase, &lo, &hi);
          const int slot_r = atomicAdd(&U.n_runs, 1);
          if (slot_r >= P.run_cap) { atomicExch(&U.status, GVO_ERR_CAPACITY); continue; }
          Run r;
          r.kind = 1;
          r.access = a;
          r.tag = U.src_tag[s];
          r.run_start = U.src_start[s];
          r.run_count = U.src_count[s];
          r.count = U.src_count[s] * tpb;
          r.mono = 0;
          r.pieces = 1;
          r.nd = 0;
          r.base = 0;
          r.span = 0;
          runs[slot_r] = r;
          atomicMin((long long*)&U.key_lo, (long long)Gr.of(lo));
          atomicMax((long long*)&U.key_hi, (long long)Gr.of(hi));
        }
      }
      // (b) lattices: one WARP per (source, box, coefficient class)
      GVO_PHN(__syncthreads(); if (threadIdx.x == 0) ph[14] += clock64() - t_start;)
      GVO_PH(const long long t_lat = clock64();)
      {
        const CTab ct{const_cast<int64_t*>(P.ctabs) + c * ctab_stride(P.T.max_acc), P.T.max_acc};
        const int slot0 = U.field * 2;
        const int ncl0 = (int)(ct.slot_first()[slot0 + 1] - ct.slot_first()[slot0]);
        const int ncl1 = (int)(ct.slot_first()[slot0 + 2] - ct.slot_first()[slot0 + 1]);
        const int ncl = max(ncl0, ncl1);
        const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
        int64_t* wpts = cpts + wid * kClassPts;
        // hist .. rka are free while runs are built
        SegScratch* seg = reinterpret_cast<SegScratch*>(micro_region + wid * kSegScratch);
        // the real (source, box, class) tasks, compacted so that warps share
        // them evenly (empty store sources and absent boxes are skipped);
        // the element buffer is free while runs are built
        __shared__ int n_tasks_sh;
        __shared__ int task_next;  // GVO_TASK_DYN: next lattice task
        int* tlist = reinterpret_cast<int*>(ebuf);
        const int tcap = (int)min((int64_t)1 << 20, sm_elems * 4);
        if (threadIdx.x == 0) {
          int nt = 0;
          for (int s2 = 0; s2 < U.n_src && nt >= 0; ++s2) {
            const int slot = slot0 + U.src_kind[s2];
            const int nc = (int)(ct.slot_first()[slot + 1] - ct.slot_first()[slot]);
            if (nc <= 0) continue;
            const int nb = run_box_count(U.src_start[s2], U.src_count[s2], gd);
            for (int bi = 0; bi < nb && nt >= 0; ++bi)
              for (int ci = 0; ci < nc; ++ci) {
                if (nt >= tcap) { nt = -1; break; }
                tlist[nt++] = (s2 << 20) | (bi << 16) | ci;  // n_src <= 64, boxes < 8, classes < 65536
              }
          }
          n_tasks_sh = nt;
          task_next = kNW;
        }
        __syncthreads();
        const int n_tasks = n_tasks_sh;
        const bool listed = n_tasks >= 0 && ncl < 65536;
        const int n_iter = listed ? n_tasks : U.n_src * 5 * ncl;
#if GVO_TASK_DYN
        // tasks taken from a shared counter (their costs differ by an order of
        // magnitude: a 25-point load class vs a one-point store class)
        for (int task = wid;;) {
          if (task >= n_iter) break;
#else
        for (int task = wid; task < n_iter; task += kNW) {
#endif
         do {
          int s, bi, ci;
          if (listed) {
            const int t = tlist[task];
            s = t >> 20; bi = (t >> 16) & 15; ci = t & 0xffff;
          } else {
            s = task / (5 * ncl); const int rem = task % (5 * ncl); bi = rem / ncl; ci = rem % ncl;
          }
          const int slot = slot0 + U.src_kind[s];
          const int64_t cl0 = ct.slot_first()[slot];
          if (ci >= ct.slot_first()[slot + 1] - cl0) break;
          Box box;
          if (!run_box_at(U.src_start[s], U.src_count[s], gd, bi, &box)) break;
          const int64_t cls = cl0 + ci;
          const int64_t* ca = crow + ct.rep()[cls] * 8;
          const WLat L0 = box_lattice(ca, bd, box, Gr);
          const int64_t* cp = ct.pts() + ct.start()[cls];
          const int64_t np = ct.cnt()[cls];
          for (int64_t p0 = 0; p0 < np; p0 += kClassPts) {
            const int m = (int)((np - p0) < kClassPts ? (np - p0) : kClassPts);
            __syncwarp();
            for (int k = lane; k < m; k += 32) wpts[k] = (int64_t)((uint64_t)L0.base + (uint64_t)cp[p0 + k]);
            __syncwarp();
            const bool segd = !P.seg_off && cover_segments(sink, L0, wpts, m, U.src_tag[s], Gr, seg,
                                                            !P.pat_off && (U.kind != 0 || P.mode != 0));
            if (!segd) cover_warp(sink, L0, wpts, m, U.src_tag[s], Gr);
            GVO_PHN(if (lane == 0) atomicAdd((unsigned long long*)&ph[segd ? 12 : 13], 1ull);)
          }
         } while (0);
#if GVO_TASK_DYN
          int nxt = 0;
          if (lane == 0) nxt = atomicAdd(&task_next, 1);
          task = __shfl_sync(0xffffffffu, nxt, 0);
#endif
        }
      }
      __syncthreads();
      GVO_PHN(if (threadIdx.x == 0) ph[15] += clock64() - t_lat;)

    if (threadIdx.x == 0) { t_runs_sh = clock64(); GVO_PH(ph[3] += t_runs_sh - t_start;) }
    // ---------------- offsets of runs, element count
      const int nr = min(U.n_runs, (int)P.run_cap);
      int64_t* roff = nr <= kSmemRuns ? roff_sh : roff_gl;
      // run counts loaded in parallel, exclusive scan by warp 0
      for (int r = threadIdx.x; r < nr; r += kNT) roff[r] = runs[r].count;
      __syncthreads();
      if (threadIdx.x < 32) {
        int64_t carry = 0;
        for (int r0 = 0; r0 < nr; r0 += 32) {
          const int r = r0 + (int)threadIdx.x;
          const int64_t v = r < nr ? roff[r] : 0;
          int64_t inc = v;
          for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if ((int)threadIdx.x >= o) inc += t;
          }
          if (r < nr) roff[r] = carry + inc - v;
          carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (threadIdx.x == 0) roff[nr] = carry;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int64_t acc = roff[nr];
        U.N = acc;

        const int64_t base = floordiv(U.key_lo, U.R) * U.R;
        U.key_lo = base;
        if (U.status == GVO_OK) {
          if (nr > 0 && (uint64_t)(U.key_hi - base) >= (uint64_t(1) << kKeyBits)) U.status = GVO_ERR_UNSUPPORTED;
          // oversized units are split into key ranges below when the split
          // queue exists; only an unsplittable unit is capacity-bound
          if (acc > P.elem_cap && !SS) U.status = GVO_ERR_CAPACITY;
        }
      }
      __syncthreads();
      if (U.status != GVO_OK) {
        if (threadIdx.x == 0) {
          if (P.mode == 0) {
            int64_t* row = P.counts + c * P.counts_stride;
            atomicExch((unsigned long long*)&row[GVO_C_STATUS], (unsigned long long)U.status);
          } else {
            atomicExch(P.status_out, U.status);
          }
          if (SS) atomicAdd(&SS->pending, ~0ull);
        }
        __syncthreads();
        continue;
      }

      // too big for shared memory: turn the unit into a split descriptor
      // and continue as its first key range [0, span]
      if ((U.N > sm_elems || U.has_pattern) && SS) {
        __shared__ int64_t desc_off;
        if (threadIdx.x == 0) {
          desc_off = -1;
          int slot = -1;
          for (int q = 0; q < kSplitSlotsPerCta && slot < 0; ++q) {
            const int sq = (int)blockIdx.x * kSplitSlotsPerCta + q;
            if (*reinterpret_cast<volatile int32_t*>(SS->slot_busy + sq) == 0) slot = sq;
          }
          if (slot >= 0 && nr <= P.run_cap) {
            SS->slot_busy[slot] = 1;  // only this CTA claims its own slots
            desc_off = (int64_t)slot * SS->slot_bytes;
          }
          if (desc_off >= 0) {
            SplitHdr* h = reinterpret_cast<SplitHdr*>(SS->arena + desc_off);
            h->cfg = c; h->field = U.field; h->kind = U.kind; h->j = U.j; h->n_sub = U.n_sub; h->nr = nr;
            h->n_uw = P.mode == 2 ? 0 : G.n_uw;
            h->g = U.g; h->R = U.R; h->kbase = U.key_lo; h->span = U.key_hi - U.key_lo; h->tpb = G.tpb;
            for (int q = 0; q < U.n_sub; ++q) {
              h->sub_mask[q] = U.sub_mask[q]; h->sub_r[q] = U.sub_r[q]; h->sub_sh[q] = U.sub_sh[q]; h->acc[q] = 0ull;
            }
            h->outstanding = 1;
            h->status = GVO_OK;
            h->tag_mask = 0;
            h->slot = slot;
            h->has_pattern = U.has_pattern;
          }
        }
        __syncthreads();
        if (desc_off >= 0) {
          Run* dr = reinterpret_cast<Run*>(SS->arena + desc_off + ((sizeof(SplitHdr) + 15) & ~size_t(15)));
          int64_t* lim = reinterpret_cast<int64_t*>(dr + nr);  // [first, last] granule (relative) per run
          SplitHdr* h = reinterpret_cast<SplitHdr*>(SS->arena + desc_off);
          uint32_t tm = 0;
          for (int r = threadIdx.x; r < nr; r += kNT) {
            const Run& rr = runs[r];
            dr[r] = rr;
            tm |= 1u << rr.tag;
            int64_t lo = INT64_MIN, hi = INT64_MAX;  // points runs: unknown extent
            if (rr.kind != 1) {
              uint64_t ext = rr.span;
#if GVO_OUTLINE & 256
              #pragma unroll 1
#endif
              for (int d = 0; d < rr.nd; ++d) ext += (uint64_t)rr.stride[d] * (uint64_t)(rr.ext[d] - 1);
              lo = Gr.of(rr.base) - U.key_lo;
              hi = Gr.of((int64_t)((uint64_t)rr.base + ext)) - U.key_lo;
            }
            lim[2 * r] = lo;
            lim[2 * r + 1] = hi;
          }
          tm = __reduce_or_sync(0xffffffffu, tm);
          if ((threadIdx.x & 31) == 0 && tm) atomicOr(&h->tag_mask, tm);
          __threadfence();
          __syncthreads();
          hdr = reinterpret_cast<SplitHdr*>(SS->arena + desc_off);
          if (threadIdx.x == 0 && P.unit_stats) {  // debug: split unit record
            const unsigned long long slot =
                atomicAdd(reinterpret_cast<unsigned long long*>(P.unit_stats + P.n_items * 10), 1ull);
            if (slot < 4096) {
              int64_t* us = P.unit_stats + P.n_items * 10 + 10 + slot * 10;
              us[0] = U.field; us[1] = U.kind; us[2] = U.j; us[3] = U.N; us[4] = 0; us[5] = nr;
              us[6] = U.key_hi - U.key_lo; us[7] = c; us[8] = 4;
            }
          }
          in_range = true;
          range_a = 0;
          range_b = ((U.key_hi - U.key_lo) / U.R + 1) * U.R;
        }
      }
      if (!in_range && (U.N > P.elem_cap || U.has_pattern)) {  // no descriptor slot free (pattern runs need ranges)
        if (threadIdx.x == 0) {
          if (P.mode == 0) {
            int64_t* row = P.counts + c * P.counts_stride;
            atomicExch((unsigned long long*)&row[GVO_C_STATUS], (unsigned long long)GVO_ERR_CAPACITY);
          } else {
            atomicExch(P.status_out, GVO_ERR_CAPACITY);
          }
          if (SS) atomicAdd(&SS->pending, ~0ull);
        }
        __syncthreads();
        continue;
      }
    } else {
      if (threadIdx.x == 0) {
        hdr = reinterpret_cast<SplitHdr*>(SS->arena + cur_range.desc);
      }
      range_a = cur_range.a;
      range_b = cur_range.b;
      hdr = reinterpret_cast<SplitHdr*>(SS->arena + cur_range.desc);
      if (threadIdx.x == 0) {
        U.cfg = hdr->cfg; U.field = hdr->field; U.kind = hdr->kind; U.j = hdr->j; U.n_sub = hdr->n_sub;
        U.g = hdr->g; U.R = hdr->R; U.key_lo = hdr->kbase;
        for (int q = 0; q < hdr->n_sub; ++q) {
          U.sub_mask[q] = hdr->sub_mask[q]; U.sub_r[q] = hdr->sub_r[q]; U.sub_sh[q] = hdr->sub_sh[q];
        }
        U.status = GVO_OK;
      }
      __syncthreads();
    }

    if (in_range) {
      // ================= key-range processing of a split unit =================
      const int64_t c = hdr->cfg;
      const gvo_config cfg = P.cfgs[c];
      const int tpl = cfg.template_id;
      const int abase = P.T.acc_base[tpl];
      const int64_t* fbase = P.T.field_base + P.T.field_base_off[tpl];
      const int32_t bd[3] = {cfg.block[0], cfg.block[1], cfg.block[2]};
      const int64_t gd[3] = {cfg.grid[0], cfg.grid[1], cfg.grid[2]};
      const Granule Gr = Granule::make(hdr->g);
      const int64_t kbase = hdr->kbase, R = hdr->R, tpb = hdr->tpb;
      const int nr = hdr->nr;
      const Run* druns = reinterpret_cast<const Run*>(reinterpret_cast<const uint8_t*>(hdr) +
                                                      ((sizeof(SplitHdr) + 15) & ~size_t(15)));
      const int64_t* dlim = reinterpret_cast<const int64_t*>(druns + nr);
      const uint32_t tag_mask = *reinterpret_cast<volatile const uint32_t*>(&hdr->tag_mask);
      int64_t* rcnt = nr <= kSmemRuns ? roff_sh : roff_gl;
      int64_t* rka = nr <= kSmemRuns ? rka_sh : rka_gl;
      __shared__ int64_t s_N;
      __shared__ int s_split, s_bm, s_nonmono, s_m;
      __shared__ int64_t s_width;
      __shared__ unsigned long long s_pmask;
      __shared__ uint32_t s_rtags;
      int64_t a = range_a, b = range_b;
      const long long t_r0 = clock64();
      // tags present in the runs (the bitmap keeps one plane per present
      // tag) and whether every rescale divides a 32-bit word
      const int n_tags = __popc(tag_mask);
      bool bm_r_ok = true;
      for (int q = 0; q < U.n_sub; ++q)
        bm_r_ok = bm_r_ok && U.sub_r[q] >= 1 && U.sub_r[q] <= 32 && (32 % U.sub_r[q]) == 0;
      const int64_t bm_words = sm_elems * 4;  // ebuf holds 2*sm_elems 8-byte elements
      const bool has_pat = *reinterpret_cast<volatile const int32_t*>(&hdr->has_pattern) != 0;
      // reset here and by thread 0 when a pass continues (before the pass's
      // last barrier): the loop-exit read of s_split is a vector load that
      // also covers s_nonmono, so a reset at the top of the loop would race
      // with it
      if (threadIdx.x == 0) { s_nonmono = 0; s_rtags = 0u; }
      for (;;) {
        // count in-range elements per run (monotone runs: closed form)
        __syncthreads();
        uint32_t my_tags = 0;  // tags of the runs with elements in [a, b)
        for (int r = threadIdx.x; r < nr; r += kNT) {
          const int64_t first = dlim[2 * r], last = dlim[2 * r + 1];
          if (last < a || first >= b) {  // whole run outside [a, b)
            rka[r] = 0;
            rcnt[r] = 0;
            continue;
          }
          const Run& rr = druns[r];
          if (rr.kind != 1 && rr.mono) {
            const int64_t ka = first >= a ? 0 : mono_first(rr, Gr, kbase, a, true);
            const int64_t kb = last < b ? rr.count : mono_first(rr, Gr, kbase, b, false);
            rka[r] = ka;
            rcnt[r] = kb > ka ? kb - ka : 0;
            if (kb > ka) my_tags |= 1u << rr.tag;
          } else {
            rka[r] = -1;
            rcnt[r] = 0;
            s_nonmono = 1;
            my_tags |= 1u << rr.tag;  // conservatively present
          }
        }
        my_tags = __reduce_or_sync(0xffffffffu, my_tags);
        if ((threadIdx.x & 31) == 0 && my_tags) atomicOr(&s_rtags, my_tags);
        __syncthreads();
        // non-monotone runs: scan all their elements (rare)
        for (int r = 0; r < (s_nonmono ? nr : 0); ++r) {
          if (rka[r] >= 0) continue;
          const Run& rr = druns[r];
          int64_t local = 0;
          for (int64_t k = threadIdx.x; k < rr.count; k += kNT) {
            int64_t lo, hi;
            run_interval(rr, k, Gr, P.T, abase, fbase, bd, gd, tpb, &lo, &hi);
            lo -= kbase; hi -= kbase;
            local += (lo < b && hi >= a) ? 1 : 0;
          }
          for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
          if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = local;
          __syncthreads();
          if (threadIdx.x == 0) {
            int64_t t = 0;
            for (int w = 0; w < kNW; ++w) t += wmax[w];
            rcnt[r] = t;
          }
          __syncthreads();
        }
        cta_scan_excl(rcnt, nr, wmax);
        if (threadIdx.x == 0) {
          const int64_t acc = rcnt[nr];
          s_N = acc;
          s_split = 0;
          // bitmap tier: one bit per granule and tag over [a, b) in the
          // element buffer, when the range is narrow enough and dense enough
          // that setting bits beats emitting + radix sorting intervals
          const int64_t wp = (b - a + 31) >> 5;
          // bitmap planes only for the tags present in this range
          const int n_tags_r = max(1, __popc(s_rtags & tag_mask));
          const bool bm_fit = bm_r_ok && (int64_t)n_tags_r * wp <= bm_words;
          const bool bm_cheaper = acc * 96 > (int64_t)n_tags * wp * 2 + wp * 3 * (int64_t)U.n_sub;
          // pattern runs exist only as bitmaps: such units always take that tier
          s_bm = bm_fit && (acc > sm_elems || bm_cheaper || has_pat) ? 1 : 0;
          s_m = 1;
          if (!s_bm && acc > 0 && (acc > sm_elems || has_pat) && b - a > R) {
            // split into pieces sized for the tier the density favours (one
            // level instead of repeated halving); piece 0 is processed here
            const double dens = (double)acc / (double)(b - a);
            const bool bm_pref = bm_r_ok && n_tags > 0 &&
                                 (has_pat || dens * 96.0 * 32.0 > 2.0 * n_tags + 3.0 * U.n_sub);
            // pieces of a wave unit mostly hold one wave's tags
            int est_tags = max(1, U.kind == 1 && hdr->n_uw > 1 ? (n_tags_r + hdr->n_uw - 1) / hdr->n_uw : n_tags_r);
            if ((bm_words / est_tags) * 32 >= b - a) est_tags = n_tags_r;  // the estimate would not split
            int64_t width = bm_pref ? (bm_words / est_tags) * 32
                                    : (int64_t)((double)(b - a) * 0.8 * (double)sm_elems / (double)acc);
            width = max(R, (width / R) * R);
            if (width >= b - a) width = max(R, (((b - a) / 2) / R) * R);  // always make progress
            int64_t m = (b - a + width - 1) / width;
            if (m > 64) {
              m = 64;
              width = (((b - a) / 64) / R + 1) * R;
              m = (b - a + width - 1) / width;
            }
            s_m = (int)m;
            s_width = width;
            s_pmask = 0ull;
          }
        }
        __syncthreads();
        if (s_m > 1) {
          // pieces no run reaches are not queued (sparse units: rows far apart)
          const int64_t width = s_width;
          const int m = s_m;
          for (int r = threadIdx.x; r < nr; r += kNT) {
            const int64_t f0 = max(dlim[2 * r], a), f1 = min(dlim[2 * r + 1], b - 1);
            if (f0 > f1) continue;
            const int p0 = (int)((f0 - a) / width), p1 = (int)min((int64_t)m - 1, (f1 - a) / width);
            const uint64_t bits = (p1 - p0 >= 63 ? ~0ull : ((2ull << (p1 - p0)) - 1ull)) << p0;
            atomicOr(&s_pmask, (unsigned long long)bits);
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            const uint64_t pm = s_pmask & ~1ull;  // piece 0 stays here
            const int nq = __popcll(pm);
            if (nq > 0) {
              atomicAdd(&hdr->outstanding, nq);
              atomicAdd(&SS->pending, (unsigned long long)nq);
              const unsigned long long slot0 = atomicAdd(&SS->qtail, (unsigned long long)nq);
              const int64_t desc = (int64_t)(reinterpret_cast<uint8_t*>(hdr) - SS->arena);
              int qi = 0;
              for (uint64_t mm = pm; mm; mm &= mm - 1, ++qi) {
                const int t = __ffsll((long long)mm) - 1;
                const unsigned long long slot = slot0 + (unsigned long long)qi;
                if ((int64_t)slot < SS->q_cap) {
                  RangeItem it;
                  it.desc = desc;
                  it.a = a + (int64_t)t * width;
                  it.b = min(b, a + ((int64_t)t + 1) * width);
                  it.ready = 0;
                  it.pad = 0;
                  SS->queue[slot] = it;
                  __threadfence();
                  *reinterpret_cast<volatile int32_t*>(&SS->queue[slot].ready) = P.epoch;
                } else {  // queue full: the piece is lost, the unit fails loudly
                  atomicExch(&hdr->status, GVO_ERR_CAPACITY);
                  atomicSub(&hdr->outstanding, 1);
                  atomicAdd(&SS->pending, ~0ull);
                }
              }
            }
            s_split = 1;
            s_nonmono = 0;  // the next pass's
            s_rtags = 0u;
            cur_range.a = a;
            cur_range.b = a + width;
          }
        } else if (threadIdx.x == 0) {
          cur_range.a = a;
          cur_range.b = b;
        }
        __syncthreads();
        b = cur_range.b;
        if (!s_split) break;
      }
      const int64_t N = s_N;
      const long long t_r1 = clock64();
      GVO_PH(if (threadIdx.x == 0) { ph[5] += t_r1 - t_r0; ph[8] += 1; ph[9] += s_bm; ph[10] += N; ph[11] += nr; })
      if (N == 0) {
        // empty key range (sparse units: rows far apart): every measure adds 0
      } else if (s_bm) {
        bitmap_range(reinterpret_cast<uint32_t*>(ebuf), druns, rcnt, rka, nr, N, a, b, kbase,
                     max(1, __popc(s_rtags & tag_mask)), Gr, P.T, abase,
                     fbase, bd, gd, tpb, U, wmax, s_nonmono != 0, s_rtags & tag_mask, reinterpret_cast<int*>(hist),
                     kNW * 256 GVO_BMP(, ph));
        if (threadIdx.x < U.n_sub) atomicAdd(&hdr->acc[threadIdx.x], (unsigned long long)U.sub_val[threadIdx.x]);
        GVO_PH(if (threadIdx.x == 0) ph[6] += clock64() - t_r1;)
      } else if (N > P.elem_cap || has_pat) {
        if (threadIdx.x == 0) atomicExch(&hdr->status, has_pat ? GVO_ERR_UNSUPPORTED : GVO_ERR_CAPACITY);
      } else {
        uint64_t* A0 = N <= sm_elems ? ebuf : gbuf;
        uint64_t* B0 = N <= sm_elems ? ebuf + sm_elems : gbuf + P.elem_cap;
        // emission (clipped to [a, b), keys relative to a); dim 0 stepped
        {
          const int64_t per = (N + kNT - 1) / kNT;
          const int64_t e0 = min(N, (int64_t)threadIdx.x * per), e1 = min(N, e0 + per);
          int ri = 0;
          if (e0 < e1) {
            int lo = 0, hi = nr - 1;
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (rcnt[mid] <= e0) lo = mid; else hi = mid - 1;
            }
            ri = lo;
          }
          int64_t i = e0;
          while (i < e1) {
            while (rcnt[ri + 1] <= i) ++ri;
            const int64_t iend = min(e1, rcnt[ri + 1]);
            if (rka[ri] < 0) { i = iend; continue; }  // non-monotone runs: compacted below
            const Run& rr = druns[ri];
            const uint64_t tg = (uint64_t)rr.tag;
            int64_t k = rka[ri] + (i - rcnt[ri]);
            if (rr.kind != 0) {
              for (; i < iend; ++i, ++k) {
                int64_t lo, hi;
                run_interval(rr, k, Gr, P.T, abase, fbase, bd, gd, tpb, &lo, &hi);
                lo = max(lo - kbase, a);
                hi = min(hi - kbase, b - 1);
                A0[i] = ((uint64_t)(lo - a) << kKeyShift) | ((uint64_t)(hi - lo) << kTagBits) | tg;
              }
              continue;
            }
            const int nd = rr.nd;
            const uint64_t st0 = nd ? (uint64_t)rr.stride[0] : 0;
            const int64_t ex0 = nd ? rr.ext[0] : 1;
            const uint64_t span = rr.span;
            uint64_t bb = run_base(rr, k);
            int64_t i0 = nd ? k % ex0 : 0;
            for (; i < iend; ++i, ++k) {
              int64_t lo = Gr.of((int64_t)bb) - kbase, hi = Gr.of((int64_t)(bb + span)) - kbase;
              lo = max(lo, a);
              hi = min(hi, b - 1);
              A0[i] = ((uint64_t)(lo - a) << kKeyShift) | ((uint64_t)(hi - lo) << kTagBits) | tg;
              if (++i0 < ex0) bb += st0;
              else { i0 = 0; if (i + 1 < iend) bb = run_base(rr, k + 1); }
            }
          }
        }
        __shared__ unsigned long long fillc;
        for (int r = 0; r < (s_nonmono ? nr : 0); ++r) {
          if (rka[r] >= 0) continue;
          if (threadIdx.x == 0) fillc = 0;
          __syncthreads();
          const Run& rr = druns[r];
          for (int64_t k = threadIdx.x; k < rr.count; k += kNT) {
            int64_t lo, hi;
            run_interval(rr, k, Gr, P.T, abase, fbase, bd, gd, tpb, &lo, &hi);
            lo -= kbase; hi -= kbase;
            if (lo < b && hi >= a) {
              lo = max(lo, a);
              hi = min(hi, b - 1);
              const unsigned long long slot = atomicAdd(&fillc, 1ull);
              A0[rcnt[r] + (int64_t)slot] = ((uint64_t)(lo - a) << kKeyShift) | ((uint64_t)(hi - lo) << kTagBits) |
                                            (uint64_t)rr.tag;
            }
          }
          __syncthreads();
        }
        __syncthreads();
        int kb = 0;
        {
          uint64_t span = (uint64_t)(b - a - 1);
          while (span) { ++kb; span >>= 1; }
        }
        const uint64_t* sorted = cta_sort(A0, B0, N, kKeyShift, ((kb + 7) / 8) * 8, hist, tot);
        sweep(sorted, N, U, wmax);
        if (threadIdx.x < U.n_sub) atomicAdd(&hdr->acc[threadIdx.x], (unsigned long long)U.sub_val[threadIdx.x]);
        GVO_PH(if (threadIdx.x == 0) ph[7] += clock64() - t_r1;)
      }
      if (threadIdx.x == 0 && P.unit_stats) {
        // range statistics after the unit slots: [idx][10]
        const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(P.unit_stats + P.n_items * 10), 1ull);
        if (slot < 4096) {
          int64_t* us = P.unit_stats + P.n_items * 10 + 10 + slot * 10;
          us[0] = (int64_t)(reinterpret_cast<uint8_t*>(hdr) - SS->arena);
          us[1] = a; us[2] = b; us[3] = N; us[4] = clock64() - t_start; us[5] = nr;
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          us[6] = smid; us[7] = hdr->cfg; us[8] = kind_fetched;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        if (atomicSub(&hdr->outstanding, 1) == 1) {
          __threadfence();
          if (hdr->status != GVO_OK) {
            if (P.mode == 0) {
              int64_t* row = P.counts + c * P.counts_stride;
              atomicExch((unsigned long long*)&row[GVO_C_STATUS], (unsigned long long)hdr->status);
            } else {
              atomicExch(P.status_out, hdr->status);
            }
          } else {
            write_unit_outputs(P, c, hdr->field, hdr->kind, hdr->j, hdr->n_uw,
                               reinterpret_cast<const volatile unsigned long long*>(hdr->acc));
          }
          __threadfence();
          atomicExch(SS->slot_busy + hdr->slot, 0);  // the descriptor is dead: its slot is free
        }
        atomicAdd(&SS->pending, ~0ull);
      }
      __syncthreads();
      continue;
    }

    // ================= unsplit unit: one sort in shared (or slab) memory =================
    {
      const int nr_u = min(U.n_runs, (int)P.run_cap);
      finish_unsplit(runs, nr_u <= kSmemRuns ? roff_sh : roff_gl);
      if (threadIdx.x == 0 && SS) atomicAdd(&SS->pending, ~0ull);
      __syncthreads();
    }
  }
  GVO_PH(if (P.unit_stats && threadIdx.x < 16 && blockIdx.x < 1024))
    GVO_PH(P.unit_stats[P.n_items * 10 + 10 + 4096 * 10 + blockIdx.x * 16 + threadIdx.x] = ph[threadIdx.x];)
}

void launch_sets(const SetsLaunch& L, cudaStream_t st) {
  SetsArgs P;
  P.T = L.T;
  P.machines = L.machines;
  P.cfgs = L.cfgs;
  P.geos = L.geos;
  P.coefs = L.coefs;
  P.ctabs = L.ctabs;
  P.n_items = L.n_items;
  P.S_req = L.S_req;
  P.F_stride = L.F_stride;
  P.mode = L.mode;
  P.granularity = L.granularity;
  P.run_start = L.run_start;
  P.run_count = L.run_count;
  P.n_custom_runs = L.n_custom_runs;
  P.counts = L.counts;
  P.counts_stride = L.counts_stride;
  P.slab = L.slab;
  P.slab_bytes = L.slab_bytes;
  P.run_cap = L.run_cap;
  P.elem_cap = L.elem_cap;
  P.status_out = L.status_out;
  P.unit_stats = L.unit_stats;
  P.work = L.work;
  P.warp = L.warp;
  P.n_warp_items = L.n_warp_items;
  P.split = L.split;
  P.sm_cap = L.sm_cap;
  P.seg_off = L.seg_off;
  P.pat_off = L.pat_off;
  P.lead = L.lead;
  P.wl_wave = L.wl_wave;
  P.wl_blk = L.wl_blk;
  P.wl_warp = L.wl_warp;
  P.wl_cnt = L.wl_cnt;
  P.run_if = L.run_if;
  P.run_if_val = L.run_if_val;
  P.handoff = L.handoff;
  P.wave_field_major = L.wave_field_major;
  P.epoch = L.epoch;  // never 0 (the zeroed initial state), unique per launch
  if (P.n_items + P.n_warp_items <= 0) return;
  cudaMemsetAsync(P.work, 0, 2 * sizeof(unsigned long long), st);  // item counter, block-unit pool
  // head, tail, pending (descriptor slots are all free again when a launch ends)
  if (P.split) cudaMemsetAsync(P.split, 0, 4 * sizeof(unsigned long long), st);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sets, cudaFuncAttributeMaxDynamicSharedMemorySize, kSetsSmemBytes);
    attr = true;
  }
  const int64_t tot = P.n_items + P.n_warp_items;
  const int64_t grid = tot < L.n_ctas ? tot : L.n_ctas;
  k_sets<<<(unsigned)grid, kNT, kSetsSmemBytes, st>>>(P);
}

// bytes of the shared element buffer (what a fused warp item may use)
int64_t sets_ebuf_bytes() {
  size_t off = (sizeof(UnitSh) + 15) & ~size_t(15);
  off += kNW * 256 * 4 + 256 * 4 + kMaxSub * kNW * 8 + (kSmemRuns + 1) * 8 + kNW * kClassPts * 8 + kSmemRuns * 8;
  return (int64_t)kSetsSmemBytes - (int64_t)off;
}

}  // namespace GVO_SETS_NS

#if GVO_SETS_CTAS_PER_SM != 1
int64_t split_slot_bytes(int64_t run_cap) {
  const int64_t hb = (sizeof(SplitHdr) + 15) & ~int64_t(15);
  return (hb + run_cap * (int64_t)(sizeof(Run) + 16) + 255) & ~int64_t(255);
}

int64_t sets_slab_bytes(int64_t run_cap, int64_t elem_cap) {
  return ((run_cap * (int64_t)sizeof(Run) + 2 * (run_cap + 1) * 8 + 2 * elem_cap * 8) + 255) & ~int64_t(255);
}

#endif

}  // namespace gvo
