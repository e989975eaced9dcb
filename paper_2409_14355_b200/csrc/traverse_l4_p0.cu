// Generated: fast-path and fp64 kernels for 16-QAM, N = 1..8.
#include "traverse_inst.cuh"

namespace mpnl {
cudaError_t launch_fast_l4_p0(int n, int kind, const DetectArgs& a, const TreeParams& tp,
                                    unsigned grid, int threads, size_t smem, int extra,
                                    cudaStream_t st) {
  return launch_fast_part<4, 1>(n, kind, a, tp, grid, threads, smem, extra, st);
}
cudaError_t launch_exact_l4_p0(int n, const ExactArgs& a, const TreeParams& tp, int grid,
                                     cudaStream_t st) {
  return launch_exact_part<4, 1>(n, a, tp, grid, st);
}
}  // namespace mpnl
