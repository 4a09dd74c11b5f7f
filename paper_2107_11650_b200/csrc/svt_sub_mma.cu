// Subspace Hankel-SVT instantiations whose chunk contractions run as 3xTF32
// on the tensor cores (svt_mma.cuh): 48-column level 1 at 72 <= d <= 128 in
// the resident layout, and the co-located large-d layout at d = 120.
#include "svt_subspace.cuh"
#include "svt_subspace_launch.cuh"

namespace shlr_b200 {

bool launch_sub_mma(int dp, bool coloc, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  if (coloc) {
    if (dp != 120) return false;
    launch_sub<120, kSubspaceKB, true, false, 2, true>(prm, total, smem, stream);
    return true;
  }
  switch (dp) {
    case 120: launch_sub<120, kSubspaceKB, false, false, 1, true>(prm, total, smem, stream); return true;
    default: return false;
  }
}

}  // namespace shlr_b200
