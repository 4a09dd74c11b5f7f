// Subspace Hankel-SVT instantiations for 128 < d <= 248 (svt_subspace.cuh):
// the large-d variant (spectra and adjoint not resident in shared memory).
#include "svt_subspace.cuh"
#include "svt_subspace_launch.cuh"

namespace shlr_b200 {

namespace {
template <bool L2>
bool dispatch_big(int dp, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  constexpr int KB = L2 ? kSubspaceKBBig : kSubspaceKB;
  switch (dp) {
    case 120:  // 112 < d <= 120 level 1, two CTAs per SM (hankel_svt.cu launch_level)
      if constexpr (!L2) {
        launch_sub<120, KB, true, L2, 2>(prm, total, smem, stream);
        return true;
      }
      return false;
    case 160: launch_sub<160, KB, true, L2>(prm, total, smem, stream); return true;
    case 192: launch_sub<192, KB, true, L2>(prm, total, smem, stream); return true;
    case 248: launch_sub<248, KB, true, L2>(prm, total, smem, stream); return true;
    default: return false;
  }
}
}  // namespace

bool launch_sub_big(int dp, bool l2, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  return l2 ? dispatch_big<true>(dp, prm, total, smem, stream) : dispatch_big<false>(dp, prm, total, smem, stream);
}

}  // namespace shlr_b200
