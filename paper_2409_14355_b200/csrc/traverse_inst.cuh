// Explicit instantiation of the traversal kernel for one QAM order (L levels
// per axis) and a range of N, plus the launcher the C ABI dispatches to.
// Included by the generated traverse_l<L>_p<part>.cu units (one per
// constellation x N-range of 8, compiled in parallel).
#pragma once
#include "traverse.cuh"

namespace mpnl {

template <int NN, int L>
cudaError_t launch_traverse_one(const TraverseArgs& a, const TreeParams& tp, int threads,
                                unsigned grid, size_t smem, cudaStream_t st) {
  auto k = traverse_kernel<NN, L>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, threads, smem, st>>>(a, tp);
  return cudaGetLastError();
}

template <int L, int N0>
cudaError_t launch_traverse_part(int n, const TraverseArgs& a, const TreeParams& tp, int threads,
                                 unsigned grid, size_t smem, cudaStream_t st) {
  switch (n - N0) {
    case 0: return launch_traverse_one<N0 + 0, L>(a, tp, threads, grid, smem, st);
    case 1: return launch_traverse_one<N0 + 1, L>(a, tp, threads, grid, smem, st);
    case 2: return launch_traverse_one<N0 + 2, L>(a, tp, threads, grid, smem, st);
    case 3: return launch_traverse_one<N0 + 3, L>(a, tp, threads, grid, smem, st);
    case 4: return launch_traverse_one<N0 + 4, L>(a, tp, threads, grid, smem, st);
    case 5: return launch_traverse_one<N0 + 5, L>(a, tp, threads, grid, smem, st);
    case 6: return launch_traverse_one<N0 + 6, L>(a, tp, threads, grid, smem, st);
    case 7: return launch_traverse_one<N0 + 7, L>(a, tp, threads, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mpnl
