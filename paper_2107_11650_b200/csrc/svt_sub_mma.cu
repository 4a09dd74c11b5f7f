// Subspace Hankel-SVT instantiations whose chunk contractions run as 3xTF32
// on the tensor cores (svt_mma.cuh): the 48-column level 1 at d = 120 in the
// resident layout and in the co-located large-d layout (config 2), and the
// parameter path's PE lifts at d = 104 (32-column level 1, 48-column level 2).
#include "svt_subspace.cuh"
#include "svt_subspace_launch.cuh"

namespace shlr_b200 {

bool launch_sub_mma(int dp, int kb, bool l2, bool coloc, const SvtParams& prm, int total, size_t smem,
                    cudaStream_t stream) {
  if (coloc) {  // the large-d layout, two CTAs per SM
    if (l2) return false;
    if (dp == 120 && kb == kSubspaceKB) {
      launch_sub<120, kSubspaceKB, true, false, 2, true>(prm, total, smem, stream);
      return true;
    }
    if (dp == 104 && kb == kSubspaceKB1) {
      launch_sub<104, kSubspaceKB1, true, false, 2, true>(prm, total, smem, stream);
      return true;
    }
    if (dp == 72 && kb == kSubspaceKB) {
      launch_sub<72, kSubspaceKB, true, false, 2, true>(prm, total, smem, stream);
      return true;
    }
    return false;
  }
  if (dp == 120 && kb == kSubspaceKB && !l2) {
    launch_sub<120, kSubspaceKB, false, false, 1, true>(prm, total, smem, stream);
    return true;
  }
  if (dp == 72 && kb == kSubspaceKB && !l2) {
    launch_sub<72, kSubspaceKB, false, false, 1, true>(prm, total, smem, stream);
    return true;
  }
  if (dp == 104 && kb == kSubspaceKB1 && !l2) {
    launch_sub<104, kSubspaceKB1, false, false, 1, true>(prm, total, smem, stream);
    return true;
  }
  if (dp == 104 && kb == kSubspaceKB && l2) {
    launch_sub<104, kSubspaceKB, false, true, 1, true>(prm, total, smem, stream);
    return true;
  }
  return false;
}

}  // namespace shlr_b200
