// Generated: fast-path kernels for 64-QAM, N = 1..8.
#include "traverse_inst.cuh"

namespace mpnl {
cudaError_t launch_fast_l8_p0(int n, int kind, const DetectArgs& a, const TreeParams& tp,
                                    unsigned grid, int threads, size_t smem, int extra,
                                    cudaStream_t st) {
  return launch_fast_part<8, 1>(n, kind, a, tp, grid, threads, smem, extra, st);
}
}  // namespace mpnl
