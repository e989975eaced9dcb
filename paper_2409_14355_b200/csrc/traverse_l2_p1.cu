// Generated: traversal kernels for 4-QAM, N = 9..16.
#include "traverse_inst.cuh"

namespace mpnl {
cudaError_t launch_traverse_l2_p1(int n, const TraverseArgs& a, const TreeParams& tp,
                                        int threads, unsigned grid, size_t smem, cudaStream_t st) {
  return launch_traverse_part<2, 9>(n, a, tp, threads, grid, smem, st);
}
}  // namespace mpnl
