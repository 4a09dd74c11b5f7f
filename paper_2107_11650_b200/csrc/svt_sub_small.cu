// Subspace Hankel-SVT instantiations for 40 <= d <= 128 (svt_subspace.cuh).
#include <cstdlib>

#include "svt_subspace.cuh"
#include "svt_subspace_launch.cuh"

namespace shlr_b200 {

namespace {
template <int KB, bool L2>
bool dispatch_small(int dp, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  switch (dp) {
    case 72: launch_sub<72, KB, false, L2>(prm, total, smem, stream); return true;
    case 80: launch_sub<80, KB, false, L2>(prm, total, smem, stream); return true;
    case 88: launch_sub<88, KB, false, L2>(prm, total, smem, stream); return true;
    case 96: launch_sub<96, KB, false, L2>(prm, total, smem, stream); return true;
    case 104: launch_sub<104, KB, false, L2>(prm, total, smem, stream); return true;
    case 112: launch_sub<112, KB, false, L2>(prm, total, smem, stream); return true;
    case 120: launch_sub<120, KB, false, L2>(prm, total, smem, stream); return true;
    case 128: launch_sub<128, KB, false, L2>(prm, total, smem, stream); return true;
    default: return false;
  }
}
// 40 <= d < 72: 16-column level 1, 32-column level 2
template <int KB, bool L2>
bool dispatch_smalld(int dp, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  // two CTAs per SM (64 registers per thread) when the shared memory allows it:
  // one matrix's barrier-bound QR / Rayleigh-Ritz phases overlap the other's
  // chunk products (SHLR_SMALLD_COLOC=0: one CTA per SM)
  static const bool coloc = !std::getenv("SHLR_SMALLD_COLOC") || std::atoi(std::getenv("SHLR_SMALLD_COLOC")) != 0;
  if (coloc && 2 * (smem + 1024) <= 227 * 1024) {
    switch (dp) {
      case 40: launch_sub<40, KB, false, L2, 2>(prm, total, smem, stream); return true;
      case 48: launch_sub<48, KB, false, L2, 2>(prm, total, smem, stream); return true;
      case 56: launch_sub<56, KB, false, L2, 2>(prm, total, smem, stream); return true;
      case 64: launch_sub<64, KB, false, L2, 2>(prm, total, smem, stream); return true;
      default: return false;
    }
  }
  switch (dp) {
    case 40: launch_sub<40, KB, false, L2>(prm, total, smem, stream); return true;
    case 48: launch_sub<48, KB, false, L2>(prm, total, smem, stream); return true;
    case 56: launch_sub<56, KB, false, L2>(prm, total, smem, stream); return true;
    case 64: launch_sub<64, KB, false, L2>(prm, total, smem, stream); return true;
    default: return false;
  }
}
}  // namespace

bool launch_sub_small(int dp, int kb, bool l2, const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  // d < 72: level 1 kSubspaceKBSmall, level 2 kSubspaceKB1 columns
  if (dp < 72) {
    if (l2) return kb == kSubspaceKB1 && dispatch_smalld<kSubspaceKB1, true>(dp, prm, total, smem, stream);
    return kb == kSubspaceKBSmall && dispatch_smalld<kSubspaceKBSmall, false>(dp, prm, total, smem, stream);
  }
  // level 2 of 72 <= d <= 128 always has kSubspaceKB columns; level 1 kSubspaceKB1 or kSubspaceKB
  if (l2) return kb == kSubspaceKB && dispatch_small<kSubspaceKB, true>(dp, prm, total, smem, stream);
  if (kb == kSubspaceKB1) return dispatch_small<kSubspaceKB1, false>(dp, prm, total, smem, stream);
  return kb == kSubspaceKB && dispatch_small<kSubspaceKB, false>(dp, prm, total, smem, stream);
}

}  // namespace shlr_b200
