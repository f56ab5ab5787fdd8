// k_warp.cu — standalone launcher of the warp-statistics items (custom
// groups of the fine-grained C ABI; the batched pipeline runs the same
// device function inside the fused k_sets work queue).
#include "gvo_warp.cuh"
#include "gvo_kernels.h"

namespace gvo {

__global__ void __launch_bounds__(256, 4) k_warp(WarpArgs W) {
  extern __shared__ unsigned long long sh[];
  for (int64_t item = blockIdx.x; item < W.n_items; item += gridDim.x) warp_item(W, item, sh);
}

void launch_warp(const TplView& T, const gvo_machine* d_machines, const gvo_config* d_cfgs, const Geo* d_geos, const int64_t* d_coefs,
                 int64_t n_items, int S_req, int64_t sector, int64_t bank_width, int64_t n_banks,
                 int mode, const int64_t* d_block_list, int64_t* d_counts, int64_t counts_stride,
                 int F_stride, int64_t* d_l1_access, int32_t l1_stride, unsigned long long* d_out,
                 int max_acc, int n_sm, cudaStream_t st) {
  if (n_items <= 0) return;
  const size_t smem = warp_item_smem(max_acc);
  int64_t grid = n_items < (int64_t)n_sm * 8 ? n_items : (int64_t)n_sm * 8;
  WarpArgs W{T, d_machines, d_cfgs, d_geos, d_coefs, n_items, S_req, sector, bank_width, n_banks, mode,
             d_block_list, d_counts, counts_stride, F_stride, d_l1_access, l1_stride, d_out};
  k_warp<<<(unsigned)grid, 256, smem, st>>>(W);
}

}  // namespace gvo
