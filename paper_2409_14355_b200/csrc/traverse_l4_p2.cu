// Generated: traversal kernels for 16-QAM, N = 17..24.
#include "traverse_inst.cuh"

namespace mpnl {
cudaError_t launch_traverse_l4_p2(int n, const TraverseArgs& a, const TreeParams& tp,
                                        int threads, unsigned grid, size_t smem, cudaStream_t st) {
  return launch_traverse_part<4, 17>(n, a, tp, threads, grid, smem, st);
}
}  // namespace mpnl
