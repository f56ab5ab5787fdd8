// k_dedup.cu — exact sharing of identical set problems across configurations.
//
// A configuration space repeats the same integer problem many times: the
// reference evaluates every configuration from scratch (perf.py:115-130),
// while the unique-granule counts of a unit depend only on
//   * the field's access expressions up to the field base (the alignment),
//   * the launch (block, grid, work per thread),
//   * the machine's integer parameters (sector/line size, banks, SM count and
//     per-SM limits: the waves), and
//   * the sampling knobs (one per call),
// not on L2/L1 capacities, bandwidths, clocks or fit parameters (those only
// enter the float assembly, k_assemble.cu).  Moving a field's base by Δ
// translates every address of the field by Δ (the host checks that every
// access is `base_f + E(coords)` with E base-free: capi.cu field_classes), and
// translating a set by a multiple of the granule leaves every unique count
// unchanged:
//   wave units   (|L|, |S|, |L∪S|, |L∪L'| at sector granularity)  Δ ≡ 0 mod sector
//   block units  (sectors and 128 B lines)                         Δ ≡ 0 mod line
//   warp items   (distinct sectors per warp)                       Δ ≡ 0 mod sector
//   L1 items     (bank wavefronts: ids shift, banks rotate)        Δ ≡ 0 mod bank width × banks
// The residue of each base is part of the key, so two units with equal keys
// are exact translates: the first one to claim the key computes it, the
// others copy its counts after the set kernel.  Keys are compared word by
// word (no hashing without verification); the table persists over all
// batches of one call, so a later batch can reuse an earlier batch's counts.
#include "gvo_kernels.h"

#include <algorithm>

namespace gvo {

namespace {

constexpr int kKeyWords = 9;
constexpr int kMaxProbe = 64;

__device__ __forceinline__ uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 29);
}

// packed residues of every field base (8 bits each, 16 fields in two words);
// false when a residue does not fit 8 bits
__device__ __forceinline__ bool pack_residues(const int64_t* fb, int nf, int64_t m, uint64_t* w0, uint64_t* w1) {
  if (m <= 0 || m > 256) return false;
  uint64_t a = 0, b = 0;
  for (int f = 0; f < nf; ++f) {
    const uint64_t r = (uint64_t)floormod(fb[f], m);
    if (f < 8) a |= r << (8 * f); else b |= r << (8 * (f - 8));
  }
  *w0 = a;
  *w1 = b;
  return true;
}

}  // namespace

// One thread per unit of the batch.  Unit index space (local to the batch):
//   [0, n*F)                 wave unit (c, f)       at c*F + f
//   [n*F, n*F*(S+1))         block unit (c, f, j)   at n*F + (c*F + f)*S + j
//   [n*F*(S+1), +n*(S+1))    warp item (c, j)       j == S: the L1 item
// lead[u] = -1: the unit computes; >= 0: leader code (global config index *
// 32 + field) whose counts it copies.
// returns 0 not shareable, 1 leader, 2 follower
__device__ __forceinline__ int dedup_unit(const TplView& T, const gvo_machine* machines, const int32_t* mclass,
                                          const gvo_config* cfgs, const Geo* geos, int64_t n, int F, int S,
                                          int64_t b0, DedupEntry* table, int64_t mask, int64_t* lead, int64_t u) {
  const int64_t nw = n * F, nb = n * F * S;
  int kind, f = 0, j = 0;
  int64_t c;
  if (u < nw) { kind = 1; c = u / F; f = (int)(u % F); }
  else if (u < nw + nb) { const int64_t r = u - nw; kind = 2; c = r / ((int64_t)F * S); f = (int)((r / S) % F); j = (int)(r % S); }
  else { const int64_t r = u - nw - nb; c = r / (S + 1); j = (int)(r % (S + 1)); kind = j == S ? 4 : 3; }
  lead[u] = -1;
  const Geo& G = geos[c];
  if (G.status != GVO_OK) return 0;
  const gvo_config cfg = cfgs[c];
  const int tpl = cfg.template_id;
  const int nf = T.n_fields[tpl];
  const int64_t* fb = T.field_base + T.field_base_off[tpl];
  const gvo_machine& m = machines[cfg.machine_id];
  uint64_t key[kKeyWords];
  key[0] = (uint64_t)kind | ((uint64_t)j << 8) | ((uint64_t)(uint32_t)mclass[cfg.machine_id] << 32);
  key[2] = (uint64_t)(uint32_t)cfg.block[0] | ((uint64_t)(uint32_t)cfg.block[1] << 21) |
           ((uint64_t)(uint32_t)cfg.block[2] << 42);
  key[3] = (uint64_t)cfg.grid[0];
  key[4] = (uint64_t)cfg.grid[1];
  key[5] = (uint64_t)cfg.grid[2];
  key[6] = (uint64_t)cfg.work_per_thread;
  key[7] = key[8] = 0;
  if (kind <= 2) {
    if (f >= nf) return 0;
    if (kind == 1 && !phase_ok(G, 1)) return 0;
    if (kind == 2 && (!phase_ok(G, 0) || j >= G.n_samples || G.dup_of[f][j] >= 0)) return 0;
    const int cls = T.fclass[T.field_base_off[tpl] + f];
    if (cls < 0) return 0;
    key[1] = (uint64_t)cls;
    key[7] = (uint64_t)floormod(fb[f], kind == 1 ? m.sector_bytes : m.l1_line_bytes);
  } else {
    if (!phase_ok(G, kind == 4 ? 2 : 0)) return 0;
    if (kind == 3 && j >= G.n_samples) return 0;
    const int cls = T.tclass[tpl];
    if (cls < 0) return 0;
    key[1] = (uint64_t)cls;
    if (!pack_residues(fb, nf, kind == 3 ? m.sector_bytes : m.bank_width_bytes * m.l1_banks, &key[7], &key[8])) return 0;
  }
  uint64_t h = 0x243f6a8885a308d3ull;
#pragma unroll
  for (int k = 0; k < kKeyWords; ++k) h = mix(h, key[k]);
  const uint64_t tag = h | 1ull;
  const int64_t code = (b0 + c) * 32 + f;
  int64_t slot = (int64_t)(h >> 7) & mask;
  for (int p = 0; p < kMaxProbe; ++p, slot = (slot + 1) & mask) {
    DedupEntry& e = table[slot];
    const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(&e.tag), 0ull,
                                             (unsigned long long)tag);
    if (old == 0ull) {  // claimed: this unit is the leader of its key
      for (int k = 0; k < kKeyWords; ++k) e.key[k] = key[k];
      e.leader = code;
      __threadfence();
      atomicExch(&e.ready, 1);
      return 1;
    }
    if (old != tag) continue;
    while (atomicAdd(&e.ready, 0) == 0) __nanosleep(32);
    __threadfence();
    bool same = true;
#pragma unroll
    for (int k = 0; k < kKeyWords; ++k) same &= *reinterpret_cast<volatile uint64_t*>(&e.key[k]) == key[k];
    if (same) {
      lead[u] = *reinterpret_cast<volatile int64_t*>(&e.leader);
      return 2;
    }
  }
  return 1;  // table crowded: the unit computes itself (correct, just not shared)
}

__global__ void k_dedup(TplView T, const gvo_machine* machines, const int32_t* mclass, const gvo_config* cfgs,
                        const Geo* geos, int64_t n, int F, int S, int64_t b0, DedupEntry* table, int64_t mask,
                        int64_t* lead, unsigned long long* stats) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t units = n * F * (S + 1) + n * (S + 1);
  const int st = u < units ? dedup_unit(T, machines, mclass, cfgs, geos, n, F, S, b0, table, mask, lead, u) : 0;
  if (stats) {  // [0] shareable units, [1] followers (warp-aggregated)
    const unsigned sh = __ballot_sync(0xffffffffu, st != 0), fo = __ballot_sync(0xffffffffu, st == 2);
    if ((threadIdx.x & 31) == 0) {
      if (sh) atomicAdd(&stats[0], (unsigned long long)__popc(sh));
      if (fo) atomicAdd(&stats[1], (unsigned long long)__popc(fo));
    }
  }
}


// After the set kernel: followers copy their leader's counts (same unit
// kind, field and sample; the leader's row lives anywhere in the call's
// counts array, d_counts_all).
__global__ void k_dedup_copy(const gvo_config* cfgs, const Geo* geos, const TplView T, int64_t* counts_all,
                             int64_t counts_stride, int64_t n, int F, int S, int64_t b0, const int64_t* lead,
                             int64_t* l1_access_all, int32_t l1_stride) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nw = n * F, nb = n * F * S, nwi = n * (S + 1);
  if (u >= nw + nb + nwi) return;
  const int64_t ld = lead[u];
  if (ld < 0) return;
  const int64_t lc = ld >> 5;
  const int lf = (int)(ld & 31);
  // a set-kernel failure of the leader's configuration (capacity) is the
  // follower's too: same problem, same runs
  const int64_t lst = counts_all[lc * counts_stride + GVO_C_STATUS];
  int64_t c;
  int64_t* dst;
  const int64_t* src;
  if (u < nw) {
    c = u / F;
    const int f = (int)(u % F);
    const Geo& G = geos[c];
    dst = counts_all + (b0 + c) * counts_stride + GVO_C_HDR + (int64_t)S * F * 5;
    src = counts_all + lc * counts_stride + GVO_C_HDR + (int64_t)S * F * 5;
    for (int w = 0; w < G.n_uw; ++w)
      for (int k = 0; k < 4; ++k) dst[((int64_t)w * F + f) * 4 + k] = src[((int64_t)w * F + lf) * 4 + k];
  } else if (u < nw + nb) {
    const int64_t r = u - nw;
    c = r / ((int64_t)F * S);
    const int f = (int)((r / S) % F);
    const int j = (int)(r % S);
    dst = counts_all + (b0 + c) * counts_stride + GVO_C_HDR + ((int64_t)j * F + f) * 5;
    src = counts_all + lc * counts_stride + GVO_C_HDR + ((int64_t)j * F + lf) * 5;
    dst[0] = src[0];
    dst[2] = src[2];
    dst[3] = src[3];
  } else {
    const int64_t r = u - nw - nb;
    c = r / (S + 1);
    const int j = (int)(r % (S + 1));
    int64_t* row = counts_all + (b0 + c) * counts_stride;
    const int64_t* lrow = counts_all + lc * counts_stride;
    if (j < S) {
      const int nf = T.n_fields[cfgs[c].template_id];
      for (int f = 0; f < nf; ++f) {
        row[GVO_C_HDR + ((int64_t)j * F + f) * 5 + 1] = lrow[GVO_C_HDR + ((int64_t)j * F + f) * 5 + 1];
        row[GVO_C_HDR + ((int64_t)j * F + f) * 5 + 4] = lrow[GVO_C_HDR + ((int64_t)j * F + f) * 5 + 4];
      }
    } else {
      row[GVO_C_L1CYCLES] = lrow[GVO_C_L1CYCLES];
      row[GVO_C_L1BLOCK] = lrow[GVO_C_L1BLOCK];
      if (l1_access_all) {
        const int A = T.n_acc[cfgs[c].template_id];
        for (int a = 0; a < A && a < l1_stride; ++a)
          for (int k = 0; k < 3; ++k)
            l1_access_all[((b0 + c) * l1_stride + a) * 3 + k] = l1_access_all[(lc * l1_stride + a) * 3 + k];
      }
    }
  }
  if (lst != GVO_OK)
    atomicExch(reinterpret_cast<unsigned long long*>(counts_all + (b0 + c) * counts_stride + GVO_C_STATUS),
               (unsigned long long)lst);
}

int64_t dedup_units(int64_t n, int F, int S) { return n * F * (S + 1) + n * (S + 1); }

void launch_dedup(const TplView& T, const gvo_machine* d_machines, const int32_t* d_mclass, const gvo_config* d_cfgs,
                  const Geo* d_geos, int64_t n, int F, int S, int64_t b0, DedupEntry* table, int64_t mask,
                  int64_t* d_lead, unsigned long long* d_stats, cudaStream_t st) {
  const int64_t units = dedup_units(n, F, S);
  if (units == 0) return;
  k_dedup<<<(unsigned)((units + 255) / 256), 256, 0, st>>>(T, d_machines, d_mclass, d_cfgs, d_geos, n, F, S, b0,
                                                           table, mask, d_lead, d_stats);
}

void launch_dedup_copy(const gvo_config* d_cfgs, const Geo* d_geos, const TplView& T, int64_t* d_counts_all,
                       int64_t counts_stride, int64_t n, int F, int S, int64_t b0, const int64_t* d_lead,
                       int64_t* d_l1_access_all, int32_t l1_stride, cudaStream_t st) {
  const int64_t units = dedup_units(n, F, S);
  if (units == 0) return;
  k_dedup_copy<<<(unsigned)((units + 255) / 256), 256, 0, st>>>(d_cfgs, d_geos, T, d_counts_all, counts_stride, n, F,
                                                                S, b0, d_lead, d_l1_access_all, l1_stride);
}

// ------------------------------------------------------------------ work lists
// The set kernel's queue hands out every unit of the batch; after sharing
// most of them are copies (k_dedup) or empty (fields a template lacks,
// samples beyond the grid, translate-duplicate samples, failed phases).
// One thread per unit of a segment (0 wave units in the kernel's wave order,
// 1 block units, 2 warp items) keeps the units that compute; warp-aggregated
// appends keep the lists close to item order (heavy wave fields first).
// The set kernel re-checks every condition, so the lists only need to be a
// superset of the computing units.
__global__ void k_worklist(TplView T, const gvo_config* cfgs, const Geo* geos, int64_t n, int F, int S,
                           const int64_t* lead, int seg, int wave_fm, int32_t* out, unsigned long long* cnt,
                           uint8_t* need) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = seg == 0 ? n * F : seg == 1 ? n * F * S : n * (S + 1);
  bool keep = false;
  if (i < total) {
    int64_t c, u;
    int f = 0, j = 0;
    if (seg == 0) {
      if (wave_fm) { f = (int)(i / n); c = i % n; }
      else { c = i / F; f = (int)(i % F); }
      u = c * F + f;
    } else if (seg == 1) {
      c = i / ((int64_t)F * S); f = (int)((i / S) % F); j = (int)(i % S);
      u = n * F + i;
    } else {
      c = i / (S + 1); j = (int)(i % (S + 1));
      u = n * F * (S + 1) + i;
    }
    const Geo& G = geos[c];
    const int nf = T.n_fields[cfgs[c].template_id];
    keep = !lead || lead[u] < 0;
    if (seg == 0) keep = keep && f < nf && phase_ok(G, 1);
    else if (seg == 1) keep = keep && f < nf && phase_ok(G, 0) && j < G.n_samples && G.dup_of[f][j] < 0;
    else keep = keep && (j == S ? phase_ok(G, 2) : phase_ok(G, 0) && j < G.n_samples);
    if (keep && need) need[c] = 1;  // this configuration's plan rows are read
  }
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0 && bal) base = atomicAdd(&cnt[seg], (unsigned long long)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) out[base + __popc(bal & ((1u << lane) - 1u))] = (int32_t)i;
}

void launch_worklists(const TplView& T, const gvo_config* d_cfgs, const Geo* d_geos, int64_t n, int F, int S,
                      const int64_t* d_lead, int wave_field_major, int32_t* d_list, unsigned long long* d_cnt,
                      const int32_t** wl_wave, const int32_t** wl_blk, const int32_t** wl_warp, uint8_t* d_need,
                      cudaStream_t st) {
  const int64_t seg_n[3] = {n * F, n * F * S, n * (S + 1)};
  cudaMemsetAsync(d_cnt, 0, 3 * sizeof(unsigned long long), st);
  if (d_need) cudaMemsetAsync(d_need, 0, (size_t)n, st);
  int32_t* out = d_list;
  const int32_t** dst[3] = {wl_wave, wl_blk, wl_warp};
  for (int seg = 0; seg < 3; ++seg) {
    *dst[seg] = out;
    if (seg_n[seg] > 0)
      k_worklist<<<(unsigned)((seg_n[seg] + 255) / 256), 256, 0, st>>>(T, d_cfgs, d_geos, n, F, S, d_lead, seg,
                                                                        wave_field_major, out, d_cnt, d_need);
    out += seg_n[seg];
  }
}

// *flag = 1 when some config of the batch has a template with < 3 fields
__global__ void k_batch_wide(TplView T, const gvo_config* cfgs, int64_t n, int* flag) {
  bool narrow = false;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    narrow |= T.n_fields[cfgs[c].template_id] < 3;
  if (__syncthreads_or(narrow) && threadIdx.x == 0) atomicExch(flag, 1);
}

void launch_batch_wide(const TplView& T, const gvo_config* d_cfgs, int64_t n, int* d_flag, cudaStream_t st) {
  cudaMemsetAsync(d_flag, 0, sizeof(int), st);
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 1024);
  k_batch_wide<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(T, d_cfgs, n, d_flag);
}

}  // namespace gvo
