// gvo_warp.cuh — warp-granular statistics of one thread block (device
// function shared by the standalone k_warp kernel and the fused k_sets
// work queue).
//
// (1) coalesced requests: for every access instance and every warp of the
//     block, the number of distinct granules the warp touches (reference
//     footprint._warp_unique_count, footprint.py:371-388); summed with the
//     access multiplicity per (field, kind) (volumes.py:173, footprint.py:468).
// (2) L1 bank-conflict wavefronts of the L1 block (volumes.py:57-134): per
//     half-warp the maximum number of distinct 8-byte ids in one bank,
//     summed over half-warps, or the warp's distinct-id count when every
//     half-warp collapses into the same single bank.
//
// A hardware warp evaluates exactly one modelled warp: lane i computes the
// address of thread 32*w + i, so dedup is a register-level __match_any_sync
// on the 64-bit granule, no shared memory traffic.
//
// Translation dedup: two affine accesses with the same coefficient vector
// differ by a constant K (incl. the block terms).  The distinct granules of a
// warp depend only on K mod g, and its bank wavefronts only on
// K mod (bank width * banks): shifting every address by a multiple of the
// modulus shifts every id by a whole number of granules / bank rounds.  So
// per item the accesses are grouped by (field, kind, coefficients, residue)
// and only one access per group is evaluated per modelled warp, weighted by
// the group's summed multiplicity (stencil loads: 25 accesses -> 4 groups
// for sectors, 9 for banks).
#pragma once
#include "gvo_bytecode.cuh"

namespace gvo {

__device__ __forceinline__ int64_t access_address(const int64_t* coef, const gvo_insn* code, int len,
                                                  const int64_t crd[6], const int32_t bd[3],
                                                  const int64_t* fbase) {
  if (coef[7] == kAffine) {
    uint64_t v = (uint64_t)coef[0];
#pragma unroll
    for (int k = 0; k < 6; ++k) v += (uint64_t)coef[1 + k] * (uint64_t)crd[k];
    return (int64_t)v;
  }
  return eval_point(code, len, crd, bd, fbase);
}

__device__ __forceinline__ int max_half(int v) {
  // max within each 16-lane half (xor offsets < 16 stay inside the half)
  for (int o = 8; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct WarpArgs {
  TplView T;
  const gvo_machine* machines;
  const gvo_config* cfgs;
  const Geo* geos;
  const int64_t* coefs;
  int64_t n_items;
  int S_req;
  int64_t sector, bank_width, n_banks;
  int mode;  // 0 standard items (config, sample-or-L1); 1 block list totals; 2 one L1 block
  const int64_t* block_list;
  int64_t* counts;
  int64_t counts_stride;
  int F_stride;
  int64_t* l1_access;
  int32_t l1_stride;
  unsigned long long* out_totals;
  const int64_t* lead;  // mode 0: k_dedup marks, indexed by item (>= 0: copied, skip); may be null
};

constexpr int kWarpDedupAcc = 256;   // grouping is quadratic in the access count: off beyond

// shared memory bytes needed for max_acc accesses: accumulators, coefficient
// rows, group multiplicities (int64), group representative and key list
__host__ __device__ inline size_t warp_item_smem(int max_acc) {
  return (2 * kMaxFields + 14 * (size_t)max_acc) * sizeof(unsigned long long) + 3 * (size_t)max_acc * sizeof(int32_t);
}

// One item, all threads of the CTA (blockDim.x multiple of 32).
#if defined(GVO_DEBUG_SYNC) && GVO_DEBUG_SYNC
// debug build: which exit each warp took (0 not run, 1 all fields copied, 2 end)
__shared__ int gvo_dbg_wexit[3];
#define GVO_DBG_WEXIT(k) do { if ((threadIdx.x & 31) == 0) atomicAdd(&gvo_dbg_wexit[k], 1); } while (0)
#else
#define GVO_DBG_WEXIT(k) do { } while (0)
#endif

// inlined into its callers: as an out-of-line call (early returns before
// its barriers) compute-sanitizer synccheck reports a divergent barrier at
// the caller's next __syncthreads although every warp takes the same exit
// (checked at run time with -DGVO_DEBUG_SYNC); inlined, synccheck is clean.
// GVO_WARP_ITEM_INLINE=0 restores the call (A/B).
#ifndef GVO_WARP_ITEM_INLINE
#define GVO_WARP_ITEM_INLINE 1
#endif
#if GVO_WARP_ITEM_INLINE
#define GVO_WI_ATTR __forceinline__
#else
#define GVO_WI_ATTR __noinline__
#endif
static __device__ GVO_WI_ATTR void warp_item(const WarpArgs& W, int64_t item, unsigned long long* sh) {
  const TplView& T = W.T;
  const gvo_machine* machines = W.machines;
  const gvo_config* cfgs = W.cfgs;
  const Geo* geos = W.geos;
  const int64_t* coefs = W.coefs;
  const int S_req = W.S_req;
  const int64_t sector = W.sector, bank_width = W.bank_width, n_banks = W.n_banks;
  const int mode = W.mode;
  const int64_t* block_list = W.block_list;
  int64_t* counts = W.counts;
  const int64_t counts_stride = W.counts_stride;
  const int F_stride = W.F_stride;
  int64_t* l1_access = W.l1_access;
  const int32_t l1_stride = W.l1_stride;
  unsigned long long* out_totals = W.out_totals;
  unsigned long long* acc_fk = sh;
  unsigned long long* acc_l1 = sh + 2 * kMaxFields;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  {

    int64_t c, blk;
    bool is_l1;
    int j = 0;
    if (mode == 0) {
      c = item / (S_req + 1);
      j = (int)(item % (S_req + 1));
      const Geo& G = geos[c];
      is_l1 = j == S_req;
      // whether the item runs is decided once, by thread 0, and broadcast:
      // every thread takes the same path to the barriers below
      __shared__ int s_run;
      __shared__ int64_t s_blk;
      if (threadIdx.x == 0) {
        bool run = !(W.lead && W.lead[item] >= 0);  // else counts copied from an identical item (k_dedup.cu)
        run = run && phase_ok(G, is_l1 ? 2 : 0) && (is_l1 || j < G.n_samples);
        s_run = run;
        s_blk = run ? (is_l1 ? G.l1_block : G.sample_lin[j]) : 0;
      }
      __syncthreads();
      if (!s_run) { GVO_DBG_WEXIT(0); return; }
      blk = s_blk;
    } else {
      c = 0;
      blk = block_list[item];
      is_l1 = mode == 2;
    }
    const gvo_config cfg = cfgs[c];
    const int tpl = cfg.template_id;
    const int A = T.n_acc[tpl];
    const int abase = T.acc_base[tpl];
    const int64_t* fbase = T.field_base + T.field_base_off[tpl];
    const int32_t bd[3] = {cfg.block[0], cfg.block[1], cfg.block[2]};
    const int64_t tpb = (int64_t)bd[0] * bd[1] * bd[2];
    const int64_t nw = (tpb + 31) / 32;
    const int64_t* crow = coefs + c * (int64_t)T.max_acc * 8;
    const int64_t gx = cfg.grid[0], gy = cfg.grid[1];
    const int64_t bc[3] = {blk % gx, (blk / gx) % gy, blk / (gx * gy)};
    int64_t sec = sector, bw = bank_width, nbk = n_banks;
    if (mode == 0) {
      const gvo_machine& mm = machines[cfg.machine_id];
      sec = mm.sector_bytes;
      bw = mm.bank_width_bytes;
      nbk = mm.l1_banks;
    }
    const Granule G = Granule::make(is_l1 ? bw : sec);

    for (int i = threadIdx.x; i < 2 * kMaxFields + 3 * A; i += blockDim.x) sh[i] = 0;
    // stage this config's coefficient rows (8 x int64 per access) in shared memory
    int64_t* scoef = reinterpret_cast<int64_t*>(acc_l1 + 3 * A);
    for (int i = threadIdx.x; i < 8 * A; i += blockDim.x) scoef[i] = crow[i];
    int64_t* msum = scoef + 8 * A;                          // group multiplicity, by key index
    uint64_t* fp = reinterpret_cast<uint64_t*>(msum + A);    // group fingerprint, by access
    int64_t* kres = reinterpret_cast<int64_t*>(fp + A);      // constant residue, by access
    int32_t* rep = reinterpret_cast<int32_t*>(kres + A);     // group representative, by access
    int32_t* keys = rep + A;                                 // representatives in access order
    int32_t* kidx = keys + A;                                // key index of a representative
    const bool dedup = A <= kWarpDedupAcc;
    // fields whose sample is a translate of an earlier one (thread 0 reads
    // the plan, the CTA shares the mask)
    __shared__ uint32_t s_skip;
    if (threadIdx.x == 0) {
      uint32_t m = 0;
      if (mode == 0 && !is_l1)
        for (int f = 0; f < kMaxFields; ++f) m |= (geos[c].dup_of[f][j] >= 0 ? 1u : 0u) << f;
      s_skip = m;
    }
    __syncthreads();
    const uint32_t skip_field = s_skip;
    // every field of this sample is a translate of an earlier sample: k_finish
    // copies all its counts, nothing to evaluate (uniform across the CTA)
    {
      const int nf = T.n_fields[tpl];
      const uint32_t all = nf >= 32 ? ~0u : ((1u << nf) - 1u);
      if (mode == 0 && !is_l1 && nf > 0 && (skip_field & all) == all) { GVO_DBG_WEXIT(1); return; }
    }
    // group of each access: first access of the same field, kind and
    // coefficients whose constant (block terms included) has the same residue
    const int64_t modulus = is_l1 ? bw * nbk : sec;
    for (int a = threadIdx.x; a < A; a += blockDim.x) {
      const int64_t* ca = scoef + a * 8;
      const int ga = abase + a;
      uint64_t h = ~(uint64_t)a;  // unique: never grouped
      int64_t ra = 0;
      if (dedup && ca[7] == kAffine && modulus > 0) {
        const int64_t ka = (int64_t)((uint64_t)ca[0] + (uint64_t)ca[4] * (uint64_t)bc[0] +
                                     (uint64_t)ca[5] * (uint64_t)bc[1] + (uint64_t)ca[6] * (uint64_t)bc[2]);
        ra = floormod(ka, modulus);
        h = 0x9e3779b97f4a7c15ull * (uint64_t)(T.acc_field[ga] * 2 + T.acc_kind[ga] + 1);
        for (int k = 1; k <= 6; ++k) h = (h ^ (uint64_t)ca[k]) * 0xff51afd7ed558ccdull;
        h = ((h ^ (uint64_t)ra) * 0xc4ceb9fe1a85ec53ull) & ~(uint64_t(1) << 63);  // top bit clear
      }
      fp[a] = h;
      kres[a] = ra;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < A; a += blockDim.x) {
      int r = a;
      const uint64_t h = fp[a];
      if (!(h >> 63)) {
        const int64_t* ca = scoef + a * 8;
        const int ga = abase + a;
        for (int b = 0; b < a; ++b) {
          if (fp[b] != h) continue;
          const int64_t* cb = scoef + b * 8;
          const int gb = abase + b;
          if (cb[1] == ca[1] && cb[2] == ca[2] && cb[3] == ca[3] && cb[4] == ca[4] && cb[5] == ca[5] &&
              cb[6] == ca[6] && T.acc_field[gb] == T.acc_field[ga] && T.acc_kind[gb] == T.acc_kind[ga] &&
              kres[b] == kres[a]) {
            r = b;
            break;
          }
        }
      }
      rep[a] = r;
    }
    __syncthreads();
    __shared__ int n_keys;
    if (wid == 0) {  // representatives compacted in access order
      int base = 0;
      for (int a0 = 0; a0 < A; a0 += 32) {
        const int a = a0 + lane;
        const bool isk = a < A && rep[a] == a;
        const unsigned bal = __ballot_sync(0xffffffffu, isk);
        const int pos = base + __popc(bal & ((1u << lane) - 1u));
        if (isk) { keys[pos] = a; msum[pos] = 0; kidx[a] = pos; }
        base += __popc(bal);
      }
      if (lane == 0) n_keys = base;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < A; a += blockDim.x)
      atomicAdd(reinterpret_cast<unsigned long long*>(&msum[kidx[rep[a]]]), (unsigned long long)T.acc_mult[abase + a]);
    __syncthreads();
    const int NK = n_keys;

    // each hardware warp owns a contiguous range of (modelled warp, group)
    // tasks, so thread coordinates are recomputed only when the warp changes
    const int64_t ntask = nw * NK;
    const int64_t per = (ntask + nwarps - 1) / nwarps;
    const int64_t t0 = wid * per, t1 = min(ntask, t0 + per);
    int64_t w = NK ? t0 / NK : 0;
    int ki = (int)(t0 - w * NK);
    int64_t crd[6];
    bool act = false;
    unsigned am = 0;
    bool fresh = true;
    for (int64_t t = t0; t < t1; ++t, ++ki) {
      if (ki == NK) { ki = 0; ++w; fresh = true; }
      const int a = keys[ki];
      if (fresh) {
        fresh = false;
        const int64_t th = w * 32 + lane;
        act = th < tpb;
        am = __ballot_sync(0xffffffffu, act);
        crd[0] = th % bd[0];
        crd[1] = (th / bd[0]) % bd[1];
        crd[2] = th / ((int64_t)bd[0] * bd[1]);
        crd[3] = bc[0]; crd[4] = bc[1]; crd[5] = bc[2];
      }
      const int ga = abase + a;
      const int fa = T.acc_field[ga];
      if ((skip_field >> fa) & 1u) continue;
      int64_t gid = 0;
      if (act) {
        const int64_t* cf = scoef + a * 8;
        int64_t addr;
        if (cf[7] == kAffine) {
          uint64_t v = (uint64_t)cf[0];
#pragma unroll
          for (int k = 0; k < 6; ++k) v += (uint64_t)cf[1 + k] * (uint64_t)crd[k];
          addr = (int64_t)v;
        } else {
          addr = eval_point(T.code + T.code_off[ga], T.code_len[ga], crd, bd, fbase);
        }
        gid = G.of(addr);
      }
      // distinct granules of the warp
      unsigned peers = act ? __match_any_sync(am, (unsigned long long)gid) : 0u;
      const bool lead = act && (__ffs(peers) - 1) == lane;
      const int distinct = __popc(__ballot_sync(0xffffffffu, lead));
      if (!is_l1) {
        if (lane == 0) {
          const int slot = fa * 2 + T.acc_kind[ga];
          atomicAdd(&acc_fk[slot], (unsigned long long)(msum[ki] * distinct));
        }
        continue;
      }
      // ---- bank conflicts (volumes.py:57-108)
      const unsigned hmask = lane < 16 ? 0x0000ffffu : 0xffff0000u;
      const bool hlead = act && (__ffs(peers & hmask) - 1) == lane;  // first of its id in the half
      const unsigned hleads = __ballot_sync(0xffffffffu, hlead);
      const int64_t bank = floormod(gid, nbk);
      unsigned bpeers = act ? __match_any_sync(am, (unsigned long long)bank) : 0u;
      bpeers &= hleads & hmask;  // distinct ids of this bank in this half
      const int per_bank = hlead ? __popc(bpeers) : 0;
      const int hw_max = max_half(per_bank);
      const bool blead = hlead && (__ffs(bpeers) - 1) == lane;
      const unsigned bleads = __ballot_sync(0xffffffffu, blead);
      const int touched0 = __popc(bleads & 0x0000ffffu), touched1 = __popc(bleads & 0xffff0000u);
      const bool half0 = (am & 0x0000ffffu) != 0, half1 = (am & 0xffff0000u) != 0;
      const int hw0 = __shfl_sync(0xffffffffu, hw_max, 0);
      const int hw1 = __shfl_sync(0xffffffffu, hw_max, 16);
      const int64_t b0 = __shfl_sync(0xffffffffu, bank, bleads & 0x0000ffffu ? __ffs(bleads & 0x0000ffffu) - 1 : 0);
      const int64_t b1 = __shfl_sync(0xffffffffu, bank, bleads & 0xffff0000u ? __ffs(bleads & 0xffff0000u) - 1 : 16);
      bool full = (!half0 || touched0 == 1) && (!half1 || touched1 == 1);
      if (full && half0 && half1) full = b0 == b1;
      int64_t cyc, met2;
      if (full) {
        cyc = distinct;
        met2 = 2 * (int64_t)distinct;
      } else {
        cyc = (half0 ? hw0 : 0) + (half1 ? hw1 : 0);
        met2 = (half0 && half1) ? cyc : 2 * cyc;
      }
      if (lane == 0) {
        atomicAdd(&acc_l1[3 * a + 0], (unsigned long long)cyc);
        atomicAdd(&acc_l1[3 * a + 1], (unsigned long long)met2);
        atomicAdd(&acc_l1[3 * a + 2], 1ull);
      }
    }
    __syncthreads();
    // group members take their representative's per-access L1 numbers
    if (is_l1)
      for (int a = threadIdx.x; a < A; a += blockDim.x)
        if (rep[a] >= 0 && rep[a] != a) {
          const int r = rep[a];  // the representative's access index
          acc_l1[3 * a + 0] = acc_l1[3 * r + 0];
          acc_l1[3 * a + 1] = acc_l1[3 * r + 1];
          acc_l1[3 * a + 2] = acc_l1[3 * r + 2];
        }
    __syncthreads();
    if (mode == 0) {
      int64_t* row = counts + c * counts_stride;
      if (!is_l1) {
        for (int f = threadIdx.x; f < F_stride; f += blockDim.x) {
          int64_t* b = row + GVO_C_HDR + ((int64_t)j * F_stride + f) * 5;
          b[1] = (int64_t)acc_fk[f * 2 + 0];
          b[4] = (int64_t)acc_fk[f * 2 + 1];
        }
      } else {
        if (threadIdx.x == 0) {
          int64_t tot = 0;
          for (int a = 0; a < A; ++a) tot += T.acc_mult[abase + a] * (int64_t)acc_l1[3 * a];
          row[GVO_C_L1CYCLES] = tot;
          row[GVO_C_L1BLOCK] = blk;
        }
        if (l1_access) {
          for (int a = threadIdx.x; a < A && a < l1_stride; a += blockDim.x) {
            int64_t* o = l1_access + (c * l1_stride + a) * 3;
            o[0] = (int64_t)acc_l1[3 * a];
            o[1] = (int64_t)acc_l1[3 * a + 1];
            o[2] = (int64_t)acc_l1[3 * a + 2];
          }
        }
      }
    } else if (mode == 1) {
      for (int s = threadIdx.x; s < 2 * kMaxFields; s += blockDim.x)
        if (acc_fk[s]) atomicAdd(&out_totals[s], acc_fk[s]);
    } else {
      for (int a = threadIdx.x; a < A; a += blockDim.x)
        for (int k = 0; k < 3; ++k) out_totals[3 * a + k] = acc_l1[3 * a + k];
    }
    __syncthreads();
    GVO_DBG_WEXIT(2);
  
  }
}

}  // namespace gvo
