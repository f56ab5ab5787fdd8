// gvo_common.cuh — device-side types and helpers shared by every kernel of
// the B200 volume-enumeration core.  See DESIGN.md for the data layout.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/gvo_b200.h"

namespace gvo {

constexpr int kWarp = 32;
constexpr int kHalfWarp = 16;  // reference machine.py:19
constexpr int kMaxFields = GVO_MAX_FIELDS;
constexpr int kMaxSamples = GVO_MAX_BLOCK_SAMPLES;
constexpr int kMaxUWaves = GVO_MAX_UNIQUE_WAVES;
constexpr int kStack = 32;     // bytecode evaluation stack depth

// coefficient-table flags per (config, access)
enum CoefFlag : int64_t {
  kAffine = 0,     // address = C + sum_i c_i * coord_i exactly
  kNonAffine = 1,  // contains // or %, or a product of coordinate terms
};

// ---------------------------------------------------------------- integers
// Python floor semantics (reference footprint.py:234-237 uses an arithmetic
// shift for powers of two and np.floor_divide otherwise; both are floor).
__host__ __device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  int64_t r = a - q * b;
  return (r != 0 && ((r < 0) != (b < 0))) ? q - 1 : q;
}
__host__ __device__ __forceinline__ int64_t floormod(int64_t a, int64_t b) {
  int64_t r = a % b;
  return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}
// granule index with a precomputed shift when g is a power of two
struct Granule {
  int64_t g;
  int shift;  // >= 0 when g is a power of two, else -1
  __host__ __device__ static Granule make(int64_t g) {
    Granule r;
    r.g = g;
    r.shift = -1;
    if (g > 0 && (g & (g - 1)) == 0) {
      int s = 0;
      while ((int64_t(1) << s) < g) ++s;
      r.shift = s;
    }
    return r;
  }
  __host__ __device__ __forceinline__ int64_t of(int64_t a) const {
    return shift >= 0 ? (a >> shift) : floordiv(a, g);
  }
};

__device__ __forceinline__ bool fits_i64(__int128 v) {
  return v >= (__int128)INT64_MIN && v <= (__int128)INT64_MAX;
}

// ---------------------------------------------------------------- templates
// Device copy of all uploaded templates, flattened.  Accesses of template t
// live at [acc_base[t], acc_base[t] + n_acc[t]); fk_off gives, per template
// and (field, kind) slot f*2+kind, the range of fk_list holding the access
// indices (kernel order) of that field/kind.
struct TplView {
  int32_t n_tpl;
  const int32_t* n_fields;
  const int32_t* n_acc;
  const int32_t* acc_base;
  const int32_t* field_base_off;
  const int64_t* field_base;
  const int32_t* acc_field;
  const int32_t* acc_kind;
  const int64_t* acc_mult;
  const int32_t* code_off;
  const int32_t* code_len;
  const gvo_insn* code;
  const int32_t* fk_off;   // [n_tpl][2*kMaxFields+1]
  const int32_t* fk_list;  // global access index (within template) lists
  int32_t max_acc;         // max accesses over templates (coef row stride)
  // translation classes for cross-config sharing (k_dedup.cu; host-built in
  // capi.cu): fclass[field_base_off[t] + f] / tclass[t], -1 = never shared
  const int32_t* fclass;
  const int32_t* tclass;
};

// ---------------------------------------------------------------- classes
// Per config "class table" (int64 words), written by k_setup.  Affine
// accesses of one (field, kind) slot with identical thread/block
// coefficients form a class: translates of one lattice by their constants.
//   [0, 2F+1)          first class of each slot (F = kMaxFields)
//   start[A], cnt[A]   class -> range of its sorted unique constants in pts
//   rep[A]             class -> representative access
//   pts[A]             constants, sorted ascending, unique per class
//   rep_of[A]          access -> representative access (-1: non-affine)
__host__ __device__ constexpr int64_t ctab_stride(int64_t A) { return 2 * kMaxFields + 1 + 5 * A; }
struct CTab {
  int64_t* base;
  int64_t A;
  __host__ __device__ int64_t* slot_first() const { return base; }
  __host__ __device__ int64_t* start() const { return base + 2 * kMaxFields + 1; }
  __host__ __device__ int64_t* cnt() const { return start() + A; }
  __host__ __device__ int64_t* rep() const { return cnt() + A; }
  __host__ __device__ int64_t* pts() const { return rep() + A; }
  __host__ __device__ int64_t* rep_of() const { return pts() + A; }
};

// ---------------------------------------------------------------- geometry
// Per-config plan written by the setup kernel.
struct Geo {
  int32_t phases;      // requested phase mask (1 blocks, 2 waves, 4 L1)
  int32_t status;
  int32_t err_phase, err_group, err_access;
  int32_t n_samples;   // representative blocks picked
  int32_t n_uw;        // unique waves (consecutive wave indices)
  int32_t n_pairs;
  int32_t has_pred;
  int64_t tpb, lups_per_block, total_blocks;
  int64_t per_wave, n_waves, first_wave;
  int64_t l1_block;
  int64_t sample_lin[kMaxSamples];
  int64_t uw_start[kMaxUWaves];
  int64_t uw_count[kMaxUWaves];
  // block-sample dedup: dup_of[f][j] = earlier sample whose unique-granule
  // sets of field f are exact translates of sample j's by a multiple of the
  // line size (so every sector/line count is identical), or -1
  int8_t dup_of[kMaxFields][kMaxSamples];
};

// A unit of phase p runs when the phase was requested and no error was
// raised at or before it (the reference raises at the first failing group,
// so later phases never run, earlier ones completed).
__host__ __device__ inline bool phase_ok(const Geo& G, int phase) {
  if (!((G.phases >> phase) & 1)) return false;
  return G.status == GVO_OK || G.err_phase > phase;
}

// A collaborative group restricted to one run of consecutive linear block
// indices, split into <= 5 boxes in (bx, by, bz) (x-fastest linearisation,
// reference footprint.py:112-115).
struct Box {
  int64_t lo[3];
  int64_t n[3];
};

__host__ __device__ inline int run_boxes(int64_t s, int64_t cnt, const int64_t g[3], Box* out) {
  const int64_t L = g[0], P = g[0] * g[1];
  const int64_t e = s + cnt;
  int nb = 0;
  int64_t cur = s;
  while (cur < e) {
    Box b;
    if (cur % L != 0 || e - cur < L) {
      int64_t end = (cur / L + 1) * L;
      if (end > e) end = e;
      b.lo[0] = cur % L; b.n[0] = end - cur;
      b.lo[1] = (cur / L) % g[1]; b.n[1] = 1;
      b.lo[2] = cur / P; b.n[2] = 1;
      cur = end;
    } else if (cur % P != 0 || e - cur < P) {
      int64_t y0 = (cur / L) % g[1];
      int64_t rows = (e - cur) / L;
      if (rows > g[1] - y0) rows = g[1] - y0;
      b.lo[0] = 0; b.n[0] = L;
      b.lo[1] = y0; b.n[1] = rows;
      b.lo[2] = cur / P; b.n[2] = 1;
      cur += rows * L;
    } else {
      int64_t layers = (e - cur) / P;
      b.lo[0] = 0; b.n[0] = L;
      b.lo[1] = 0; b.n[1] = g[1];
      b.lo[2] = cur / P; b.n[2] = layers;
      cur += layers * P;
    }
    out[nb++] = b;
  }
  return nb;
}

// The bi-th box of run_boxes (false when the run has fewer boxes) and the
// box count, without a box array (no local-memory array in the callers).
__host__ __device__ __forceinline__ bool run_box_at(int64_t s, int64_t cnt, const int64_t g[3], int bi, Box* out) {
  const int64_t L = g[0], P = g[0] * g[1];
  const int64_t e = s + cnt;
  int64_t cur = s;
  for (int k = 0; cur < e; ++k) {
    Box b;
    if (cur % L != 0 || e - cur < L) {
      int64_t end = (cur / L + 1) * L;
      if (end > e) end = e;
      b.lo[0] = cur % L; b.n[0] = end - cur;
      b.lo[1] = (cur / L) % g[1]; b.n[1] = 1;
      b.lo[2] = cur / P; b.n[2] = 1;
      cur = end;
    } else if (cur % P != 0 || e - cur < P) {
      int64_t y0 = (cur / L) % g[1];
      int64_t rows = (e - cur) / L;
      if (rows > g[1] - y0) rows = g[1] - y0;
      b.lo[0] = 0; b.n[0] = L;
      b.lo[1] = y0; b.n[1] = rows;
      b.lo[2] = cur / P; b.n[2] = 1;
      cur += rows * L;
    } else {
      int64_t layers = (e - cur) / P;
      b.lo[0] = 0; b.n[0] = L;
      b.lo[1] = 0; b.n[1] = g[1];
      b.lo[2] = cur / P; b.n[2] = layers;
      cur += layers * P;
    }
    if (k == bi) { *out = b; return true; }
  }
  return false;
}

__host__ __device__ inline int run_box_count(int64_t s, int64_t cnt, const int64_t g[3]) {
  const int64_t L = g[0], P = g[0] * g[1];
  const int64_t e = s + cnt;
  int64_t cur = s;
  int nb = 0;
  while (cur < e) {
    if (cur % L != 0 || e - cur < L) {
      int64_t end = (cur / L + 1) * L;
      cur = end > e ? e : end;
    } else if (cur % P != 0 || e - cur < P) {
      int64_t rows = (e - cur) / L;
      const int64_t y0 = (cur / L) % g[1];
      if (rows > g[1] - y0) rows = g[1] - y0;
      cur += rows * L;
    } else {
      cur += ((e - cur) / P) * P;
    }
    ++nb;
  }
  return nb;
}

// Coordinate bounds of a run of blocks (min/max of each block coordinate),
// as the reference's _GroupEval computes them (footprint.py:262-269).
__host__ __device__ inline void run_bid_bounds(int64_t s, int64_t cnt, const int64_t g[3],
                                               int64_t lo[3], int64_t hi[3]) {
  const int64_t e = s + cnt - 1;
  const int64_t r0 = s / g[0], r1 = e / g[0];
  if (r0 == r1) { lo[0] = s % g[0]; hi[0] = e % g[0]; }
  else { lo[0] = 0; hi[0] = g[0] - 1; }
  if (r0 / g[1] == r1 / g[1]) { lo[1] = r0 % g[1]; hi[1] = r1 % g[1]; }
  else { lo[1] = 0; hi[1] = g[1] - 1; }
  lo[2] = s / (g[0] * g[1]);
  hi[2] = e / (g[0] * g[1]);
}

// ---------------------------------------------------------------- runs
// A collapsed lattice of addresses: base + sum_d stride[d]*k_d (k_d < ext[d])
// plus an inner byte span that is granule-contiguous, i.e. each outer tuple
// contributes the granule interval [floor(b/g), floor((b+span)/g)].
// Points runs (non-affine accesses) enumerate (block, thread) pairs and
// evaluate the bytecode per point.
constexpr int kMaxDims = 7;
struct Run {
  int64_t base;
  uint64_t span;
  int64_t stride[kMaxDims];
  int64_t ext[kMaxDims];
  int32_t nd;
  int32_t tag;
  int32_t kind;     // 0 lattice, 1 points
  int32_t access;   // template-local access index (points runs)
  int32_t mono;     // lattice whose interval starts/ends increase with the
                    // tuple index (dim 0 fastest): range counts by bisection
  int32_t pad_;
  int64_t count;    // intervals emitted by this run (incl. splitting)
  int64_t pieces;   // pieces per interval (long intervals are split)
  int64_t run_start, run_count;  // points runs: group blocks
};

// packed interval element: key (35 bits) | len (24 bits) | tag (5 bits)
constexpr int kTagBits = 5;
constexpr int kLenBits = 24;
constexpr int kKeyShift = kTagBits + kLenBits;  // 29
constexpr uint64_t kLenMask = (uint64_t(1) << kLenBits) - 1;
constexpr int64_t kPiece = int64_t(1) << kLenBits;  // max granules per piece
constexpr int kKeyBits = 64 - kKeyShift;            // 35

// ---------------------------------------------------------------- splitting
// Units whose intervals exceed the shared-memory sort capacity are split by
// granule-key range: every set measure is additive over disjoint key
// ranges once intervals are clipped at the boundaries.  The run table is
// copied into a descriptor in a global arena; ranges are queued for any CTA.
constexpr int kMaxSubC = 72;
struct SplitHdr {
  int64_t cfg;
  int32_t field, kind, j, n_sub, nr, n_uw;
  int64_t g, R, kbase, span;
  int64_t tpb;
  uint32_t sub_mask[kMaxSubC];
  int64_t sub_r[kMaxSubC];
  int32_t sub_sh[kMaxSubC];
  unsigned long long acc[kMaxSubC];
  int32_t outstanding;
  int32_t status;
  uint32_t tag_mask;  // tags present in the runs (bitmap tier: compact tags)
  int32_t slot;       // descriptor slot (freed when the last range completes)
  int32_t has_pattern;  // pattern runs present: every range takes the bitmap tier
  int32_t pad2_;
};
struct RangeItem {
  int64_t desc;  // byte offset of the SplitHdr in the arena
  int64_t a, b;  // relative key range [a, b)
  int32_t ready;
  int32_t pad;
};
// Descriptors live in fixed slots, kSplitSlotsPerCta per CTA, each sized for
// run_cap runs: a CTA only starts a unit that may split while one of its
// slots is free, and the CTA that completes a descriptor's last range frees
// its slot, so descriptor memory is bounded whatever the batch size.
constexpr int kSplitSlotsPerCta = 4;
struct SplitState {
  unsigned long long qhead, qtail, pending, arena_top;
  int64_t q_cap, arena_bytes;
  RangeItem* queue;
  uint8_t* arena;        // n_ctas * kSplitSlotsPerCta slots of slot_bytes
  int32_t* slot_busy;    // one flag per slot (0 free)
  int64_t slot_bytes;
};

}  // namespace gvo
