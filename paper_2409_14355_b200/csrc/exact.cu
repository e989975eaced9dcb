// Host dispatch of the fp64 exact kernel (exact.cuh), instantiated per
// (N, L) in the traverse_l<L>_p<part>.cu units.
#include "exact_args.cuh"

namespace mpnl {

#define MPNL_DECL(LL, PP)                                                                 \
  cudaError_t launch_exact_l##LL##_p##PP(int n, const ExactArgs& a, const TreeParams& tp, \
                                         int grid, cudaStream_t st);
MPNL_DECL(2, 0) MPNL_DECL(2, 1) MPNL_DECL(2, 2) MPNL_DECL(2, 3)
MPNL_DECL(4, 0) MPNL_DECL(4, 1) MPNL_DECL(4, 2) MPNL_DECL(4, 3)
MPNL_DECL(8, 0) MPNL_DECL(8, 1) MPNL_DECL(8, 2) MPNL_DECL(8, 3)
#undef MPNL_DECL

cudaError_t launch_exact(const ExactArgs& a, const TreeParams& tp, int grid, cudaStream_t st) {
  const int part = (a.n - 1) / 8;
#define MPNL_PART(LL)                                                   \
  switch (part) {                                                       \
    case 0: return launch_exact_l##LL##_p0(a.n, a, tp, grid, st);      \
    case 1: return launch_exact_l##LL##_p1(a.n, a, tp, grid, st);      \
    case 2: return launch_exact_l##LL##_p2(a.n, a, tp, grid, st);      \
    default: return launch_exact_l##LL##_p3(a.n, a, tp, grid, st);     \
  }
  if (a.L == 2) { MPNL_PART(2) }
  if (a.L == 4) { MPNL_PART(4) }
  MPNL_PART(8)
#undef MPNL_PART
}

}  // namespace mpnl
