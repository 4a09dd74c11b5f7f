// Subspace Hankel-SVT instantiations for 248 < d <= 496 (svt_subspace.cuh):
// the HUGE variant -- a 32-column block and 16-row chunks so that the d x 32
// block, one chunk of the lifted matrix and the Rayleigh-Ritz work area fit
// in 227 KB of shared memory; ranks beyond the block go down the deflation
// chain in steps of 24 Ritz pairs.
#include "svt_subspace.cuh"
#include "svt_subspace_launch.cuh"

namespace shlr_b200 {

namespace {
template <int DP, bool L2>
void launch_huge(const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    SHLR_CUDA(cudaFuncSetAttribute(svt_subspace_kernel<DP, kSubspaceKBHuge, 16, true, L2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = true;
  }
  svt_subspace_kernel<DP, kSubspaceKBHuge, 16, true, L2><<<total, kSubNT, smem, stream>>>(prm);
  SHLR_LAUNCH_CHECK();
}
template <bool L2>
bool dispatch_huge(int dp, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  switch (dp) {
    case 320: launch_huge<320, L2>(prm, total, smem, stream); return true;
    case 384: launch_huge<384, L2>(prm, total, smem, stream); return true;
    case 496: launch_huge<496, L2>(prm, total, smem, stream); return true;
    default: return false;
  }
}
}  // namespace

bool launch_sub_huge(int dp, bool l2, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  return l2 ? dispatch_huge<true>(dp, prm, total, smem, stream) : dispatch_huge<false>(dp, prm, total, smem, stream);
}

}  // namespace shlr_b200
