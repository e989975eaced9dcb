// Generated: fast-path kernels for 4-QAM, N = 17..24.
#include "traverse_inst.cuh"

namespace mpnl {
cudaError_t launch_fast_l2_p2(int n, int kind, const DetectArgs& a, const TreeParams& tp,
                                    unsigned grid, int threads, size_t smem, int extra,
                                    cudaStream_t st) {
  return launch_fast_part<2, 17>(n, kind, a, tp, grid, threads, smem, extra, st);
}
}  // namespace mpnl
