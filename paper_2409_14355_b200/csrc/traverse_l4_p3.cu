// Generated: fast-path kernels for 16-QAM, N = 25..32.
#include "traverse_inst.cuh"

namespace mpnl {
cudaError_t launch_fast_l4_p3(int n, int kind, const DetectArgs& a, const TreeParams& tp,
                                    unsigned grid, int threads, size_t smem, int extra,
                                    cudaStream_t st) {
  return launch_fast_part<4, 25>(n, kind, a, tp, grid, threads, smem, extra, st);
}
}  // namespace mpnl
