// Launchers of the subspace Hankel-SVT kernel, one translation unit per
// dimension class (instantiations of svt_subspace_kernel, svt_subspace.cuh).
// Each returns false (nothing launched) for a dimension outside its class.
#pragma once
#include <cstddef>

#include "hankel_svt.cuh"

namespace shlr_b200 {

size_t svt_subspace_smem_bytes(int DP, int KB, int R, int maxB, int maxLen, int maxE, bool big, bool coloc = false);
// d <= 128 (svt_sub_small.cu): DP in {72, ..., 128}, KB in {32, 48}
bool launch_sub_small(int dp, int kb, bool l2, const SvtParams& prm, int total, size_t smem, cudaStream_t stream);
// 128 < d <= 248 (svt_sub_big.cu): DP in {160, 192, 248}; level 1 KB 48, level 2 / 3 KB 64
bool launch_sub_big(int dp, bool l2, const SvtParams& prm, int total, size_t smem, cudaStream_t stream);
// 3xTF32 tensor-core contractions (svt_sub_mma.cu): level 1 with 48 columns;
// coloc = the co-located large-d layout (d = 120, two CTAs per SM)
bool launch_sub_mma(int dp, int kb, bool l2, bool coloc, const SvtParams& prm, int total, size_t smem,
                    cudaStream_t stream);
// 248 < d <= 496 (svt_sub_huge.cu): DP in {320, 384, 496}; KB 32, 16-row chunks;
// l2 = the deflation-chain launches
bool launch_sub_huge(int dp, bool l2, const SvtParams& prm, int total, size_t smem, cudaStream_t stream);

}  // namespace shlr_b200
