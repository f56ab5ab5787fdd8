// k_rank.cu — global ranking of evaluated configurations.
//
// Reference perf.rank_sweep sorts rows with
//   key = (-glups, block_dim, folding)            (perf.py:131)
// using Python's stable sort, so equal keys keep input order; folding is
// compared as a string ("2y" < "2z" < "none").  Here: LSD radix sort of
// (key, index) pairs, first on the secondary key (block_dim, folding rank),
// then on the primary key ~bits(glups) (glups > 0, so the IEEE bit pattern
// orders like the value; complementing it gives descending order).  Each
// digit pass is stable, so ties end in input order exactly as in Python.
#include "gvo_kernels.h"

namespace gvo {

constexpr int kRT = 256;              // threads per CTA
constexpr int kRPer = 8;              // elements per thread
constexpr int kTile = kRT * kRPer;    // 2048
constexpr int kRW = kRT / 32;

__global__ void k_rank_keys(const double* rec, const gvo_config* cfgs, int64_t n, uint64_t* k1,
                            uint64_t* k2, uint32_t* idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double g = rec[i * GVO_RECORD_LEN + GVO_R_GLUPS];
  uint64_t b = (uint64_t)__double_as_longlong(g);
  // total order for doubles, then complement for descending
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  k1[i] = ~b;
  const gvo_config c = cfgs[i];
  k2[i] = ((uint64_t)(c.block[0] & 0xfffff) << 42) | ((uint64_t)(c.block[1] & 0xfffff) << 22) |
          ((uint64_t)(c.block[2] & 0xfffff) << 2) | (uint64_t)(c.fold_rank & 3);
  idx[i] = (uint32_t)i;
}

__global__ void k_gather(const uint64_t* k1, const uint32_t* idx, int64_t n, uint64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = k1[idx[i]];
}

__global__ void k_tile_hist(const uint64_t* key, int64_t n, int sh, uint32_t* hist, int64_t n_tiles) {
  __shared__ uint32_t h[256];
  for (int d = threadIdx.x; d < 256; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kTile;
  for (int k = threadIdx.x; k < kTile; k += blockDim.x) {
    const int64_t i = t0 + k;
    if (i < n) atomicAdd(&h[(key[i] >> sh) & 255], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[(int64_t)d * n_tiles + blockIdx.x] = h[d];
}

// exclusive scan of m values in one CTA of 1024 threads
__global__ void k_scan(uint32_t* v, int64_t m) {
  __shared__ uint32_t part[1024];
  const int64_t per = (m + 1023) / 1024;
  const int64_t b = threadIdx.x * per, e = min(m, b + per);
  uint32_t s = 0;
  for (int64_t i = b; i < e; ++i) s += v[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    uint32_t t = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s;
  for (int64_t i = b; i < e; ++i) {
    const uint32_t x = v[i];
    v[i] = run;
    run += x;
  }
}

__global__ void k_tile_scatter(const uint64_t* key, const uint32_t* idx, int64_t n, int sh,
                               const uint32_t* offs, int64_t n_tiles, uint64_t* okey, uint32_t* oidx) {
  __shared__ uint32_t wh[kRW * 256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int d = threadIdx.x; d < kRW * 256; d += blockDim.x) wh[d] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kTile + (int64_t)w * (kTile / kRW);
  // per-warp digit histogram of its contiguous slice
  for (int k = lane; k < kTile / kRW; k += 32) {
    const int64_t i = t0 + k;
    if (i < n) atomicAdd(&wh[w * 256 + ((key[i] >> sh) & 255)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    uint32_t run = offs[(int64_t)d * n_tiles + blockIdx.x];
    for (int k = 0; k < kRW; ++k) {
      const uint32_t h = wh[k * 256 + d];
      wh[k * 256 + d] = run;
      run += h;
    }
  }
  __syncthreads();
  for (int k0 = 0; k0 < kTile / kRW; k0 += 32) {
    const int64_t i = t0 + k0 + lane;
    const bool v = i < n;
    const uint64_t kk = v ? key[i] : 0;
    const uint32_t d = (uint32_t)(kk >> sh) & 255u;
    const unsigned act = __ballot_sync(0xffffffffu, v);
    unsigned peers = 0;
    if (v) {
      peers = __match_any_sync(act, d);
      const uint32_t pos = wh[w * 256 + d] + __popc(peers & ((1u << lane) - 1u));
      okey[pos] = kk;
      oidx[pos] = idx[i];
    }
    __syncwarp();
    if (v && (31 - __clz(peers)) == lane) wh[w * 256 + d] += __popc(peers);
    __syncwarp();
  }
}

// Small batches: one CTA computes each element's rank by counting the
// elements ordered before it (lexicographic (k1, k2, index) => stable), one
// launch instead of 51.
constexpr int kSmallRank = 2048;
__global__ void __launch_bounds__(1024) k_rank_small(const double* rec, const gvo_config* cfgs, int64_t n,
                                                     int64_t* order) {
  __shared__ uint64_t s1[kSmallRank], s2[kSmallRank];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    uint64_t b = (uint64_t)__double_as_longlong(rec[i * GVO_RECORD_LEN + GVO_R_GLUPS]);
    b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    s1[i] = ~b;
    const gvo_config c = cfgs[i];
    s2[i] = ((uint64_t)(c.block[0] & 0xfffff) << 42) | ((uint64_t)(c.block[1] & 0xfffff) << 22) |
            ((uint64_t)(c.block[2] & 0xfffff) << 2) | (uint64_t)(c.fold_rank & 3);
  }
  __syncthreads();
  // one warp per element: lanes count a strided share of the others, then reduce
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t i = wid; i < n; i += nw) {
    const uint64_t a1 = s1[i], a2 = s2[i];
    int r = 0;
    for (int64_t j = lane; j < n; j += 32) {
      const uint64_t b1 = s1[j], b2 = s2[j];
      r += (b1 < a1) || (b1 == a1 && (b2 < a2 || (b2 == a2 && j < i)));
    }
    r = __reduce_add_sync(0xffffffffu, r);
    if (lane == 0) order[r] = i;
  }
}

__global__ void k_order_out(const uint32_t* idx, int64_t n, int64_t* order) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) order[i] = idx[i];
}

// Multi-GPU ranking: rows gathered rank-major from every shard
// carry their global configuration index (-1: all-gather padding).  Scatter
// them back to global order so the stable sort breaks ties by the input
// index exactly as perf.py:131 does, and padding never reaches the ranking.
__global__ void k_scatter_gathered(const double* rows, const int64_t* gidx, int64_t n_rows, int64_t n_global,
                                   double* out, unsigned int* bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = t / GVO_RECORD_LEN, c = t % GVO_RECORD_LEN;
  if (r >= n_rows) return;
  const int64_t g = gidx[r];
  if (g < 0) return;
  if (g >= n_global) { if (c == 0) atomicOr(bad, 1u); return; }
  out[g * GVO_RECORD_LEN + c] = rows[r * GVO_RECORD_LEN + c];
}

void launch_scatter_gathered(const double* d_rows, const int64_t* d_gidx, int64_t n_rows, int64_t n_global,
                             double* d_out, unsigned int* d_bad, cudaStream_t st) {
  if (n_rows <= 0) return;
  const int64_t tot = n_rows * GVO_RECORD_LEN;
  k_scatter_gathered<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d_rows, d_gidx, n_rows, n_global, d_out, d_bad);
}

int64_t rank_scratch_bytes(int64_t n) {
  const int64_t n_tiles = (n + kTile - 1) / kTile;
  return n * 8 * 3 + n * 4 * 2 + 256 * n_tiles * 4 + 1024;
}

void launch_rank(const double* d_records, const gvo_config* d_cfgs, int64_t n, int64_t* d_order,
                 void* d_scratch, cudaStream_t st) {
  if (n <= 0) return;
  if (n <= kSmallRank) {
    k_rank_small<<<1, 1024, 0, st>>>(d_records, d_cfgs, n, d_order);
    return;
  }
  const int64_t n_tiles = (n + kTile - 1) / kTile;
  uint8_t* p = (uint8_t*)d_scratch;
  uint64_t* k1 = (uint64_t*)p; p += n * 8;
  uint64_t* ka = (uint64_t*)p; p += n * 8;
  uint64_t* kb = (uint64_t*)p; p += n * 8;
  uint32_t* ia = (uint32_t*)p; p += n * 4;
  uint32_t* ib = (uint32_t*)p; p += n * 4;
  uint32_t* hist = (uint32_t*)p;
  const unsigned eb = (unsigned)((n + 255) / 256);
  k_rank_keys<<<eb, 256, 0, st>>>(d_records, d_cfgs, n, k1, ka, ia);
  for (int phase = 0; phase < 2; ++phase) {
    if (phase == 1) k_gather<<<eb, 256, 0, st>>>(k1, ia, n, ka);
    for (int sh = 0; sh < 64; sh += 8) {
      k_tile_hist<<<(unsigned)n_tiles, kRT, 0, st>>>(ka, n, sh, hist, n_tiles);
      k_scan<<<1, 1024, 0, st>>>(hist, 256 * n_tiles);
      k_tile_scatter<<<(unsigned)n_tiles, kRT, 0, st>>>(ka, ia, n, sh, hist, n_tiles, kb, ib);
      uint64_t* tk = ka; ka = kb; kb = tk;
      uint32_t* ti = ia; ia = ib; ib = ti;
    }
  }
  k_order_out<<<eb, 256, 0, st>>>(ia, n, d_order);
}

}  // namespace gvo
