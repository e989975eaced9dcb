// Batched linear ZF / MMSE detection with max-log LLRs.
//
// Follows linear_detect_batch (pkg/src/mpnlsim/detect.py:528-557) and the
// per-symbol max-log demapper it calls (core.py:191-206):
//   A = H^H H (+ nv I for MMSE), soft = A^-1 H^H y, d = diag(A^-1)
//   ZF:   est = soft,        nv_eff = nv d
//   MMSE: beta = max(1 - nv d, 1e-12), est = soft / beta,
//         nv_eff = max((1 - beta) / beta, 1e-15)
//   labels = nearest point (first minimum, np.argmin), llr = (d1 - d0) / nv_eff
//   clipped to +-clip (NaN kept, as np.clip).
// The reference inverts A with LAPACK; here A (Hermitian, positive definite
// unless the channel is rank deficient) is factorised by Cholesky in fp64:
// soft from two triangular solves, diag(A^-1) as the row sums of |L^-1|^2.
// Same quantities, different rounding: the parity tests compare soft values
// and LLRs within a stated tolerance and the hard labels exactly.  Singular A:
// the reference's np.linalg.inv (LAPACK getrf) raises LinAlgError only on an
// exactly zero LU pivot, so a Cholesky pivot at rounding level of its diagonal
// entry only makes the vector SUSPECT; suspects are re-factorised by an
// unblocked partially pivoted LU (zgetf2's pivot rule) and counted in
// *n_singular when that LU meets an exactly zero pivot.
//
// Layout: a lane GROUP of G = 8 / 16 / 32 lanes per vector (N <= G), several
// vectors per warp for small N.  Lane j owns column / stream j.  H and y are
// read straight from global memory (a group's H row is one coalesced 16 N-byte
// segment; the other columns are broadcast loads that hit L1); A = L L^H lives
// in the group's slice of shared memory (N x (N+1) complex, lower triangle =
// L, upper triangle = the transposed columns of L^-1 for diag(A^-1)):
//   Gram + matched filter: lane j accumulates column j, 4 rows of A at a time;
//   Cholesky (left-looking): per column a group reduction for the pivot, then
//     lane i > j forms L[i][j] from its own row;
//   forward / back solves column-oriented (one shuffle broadcast per step);
//   L^-1: lane j solves its own column of L^-1 (no cross-lane dependency).
// fp64 throughout; bound by the FP64 pipe for large N, by HBM (16 (MN + M)
// input bytes per vector) for small N.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kMaxN = 32;
constexpr int kThreads = 128;

__device__ __forceinline__ double2 cmul_conj_a(double2 a, double2 b) {   // conj(a) * b
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}


// column j of A = H^H H (+ nv I): the lower triangle (full = false) or all rows
// (full = true, for the LU check); x (optional) += (H^H y)_j
template <int G>
__device__ __forceinline__ void gram_column(double2* A, int ns, const double2* hv,
                                            const double2* yv, int m, int n, int j, int mmse,
                                            double nv, bool full, double2* x) {
  if (j >= n) return;
  for (int i0 = 0; i0 < n; i0 += 4) {
    double2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = make_double2(0.0, 0.0);
    for (int r = 0; r < m; ++r) {
      const double2 hj = hv[r * n + j];
      if (i0 == 0 && x) {
        const double2 t = cmul_conj_a(hj, yv[r]);
        x->x += t.x;
        x->y += t.y;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u < n) {
          const double2 t = cmul_conj_a(hv[r * n + i0 + u], hj);   // conj(H[r][i]) H[r][j]
          acc[u].x += t.x;
          acc[u].y += t.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u;
      if (i < n && (full || i >= j)) A[i * ns + j] = acc[u];
    }
  }
  if (mmse) A[j * ns + j].x += nv;
}

// left-looking Cholesky of the lower triangle in place (pivots as |d|, zero -> 1).
// suspect: a pivot at rounding level of its diagonal entry (or zero /
// non-finite).  The reciprocal of L[c][c] goes to the padding column A[c][n].
template <int G>
__device__ __forceinline__ bool cholesky(double2* A, int ns, int n, int j) {
  bool suspect = false;
  for (int c = 0; c < n; ++c) {
    double p = 0.0;
    if (j < c) {
      const double2 l = A[c * ns + j];
      p = fma(l.x, l.x, l.y * l.y);
    }
    const double acc = A[c * ns + c].x;
    double d = acc - group_sum<G>(p);
    if (!(d > 64.0 * 2.220446049250313e-16 * acc) || !isfinite(d)) suspect = true;
    if (!(d != 0.0) || !isfinite(d)) d = 1.0;
    const double lcc = sqrt(fabs(d)), rc = 1.0 / lcc;
    if (j > c && j < n) {
      double2 s = A[j * ns + c];
      for (int k = 0; k < c; ++k) {   // - L[j][k] conj(L[c][k])
        const double2 a = A[j * ns + k], b = A[c * ns + k];
        s.x -= fma(a.x, b.x, a.y * b.y);
        s.y -= fma(a.y, b.x, -a.x * b.y);
      }
      A[j * ns + c] = make_double2(s.x * rc, s.y * rc);
    }
    __syncwarp();
    if (j == c) {
      A[c * ns + c] = make_double2(lcc, 0.0);
      A[c * ns + n] = make_double2(rc, 0.0);
    }
    __syncwarp();
  }
  return suspect;
}

// Unblocked LU with partial pivoting on the full matrix A (zgetf2: pivot = first
// maximum of |Re| + |Im| in the column, multipliers by the pivot's reciprocal);
// returns true when a pivot is exactly zero (np.linalg.inv's LinAlgError).
// Lane j owns column j.  Destroys A.
template <int G>
__device__ __forceinline__ bool lu_zero_pivot(double2* A, int ns, int n, int j) {
  bool zero = false;
  for (int k = 0; k < n; ++k) {
    // pivot row: lanes i >= k propose row i's |Re| + |Im| in column k
    double bv = -1.0;
    int bi = 0x7fffffff;
    if (j >= k && j < n) {
      const double2 a = A[j * ns + k];
      bv = fabs(a.x) + fabs(a.y);
      bi = j;
    }
#pragma unroll
    for (int o = G / 2; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o, G);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o, G);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    // zgetf2: a zero pivot sets info and skips the elimination (control flow
    // stays warp-uniform: several groups may share the warp)
    const bool piv = bv != 0.0;
    if (!piv) zero = true;
    if (piv && bi != k && j < n) {              // swap rows k and bi (lane = column)
      const double2 t = A[k * ns + j];
      A[k * ns + j] = A[bi * ns + j];
      A[bi * ns + j] = t;
    }
    __syncwarp();
    const double2 pv = A[k * ns + k];
    const double den = pv.x * pv.x + pv.y * pv.y;
    const double2 rp = make_double2(pv.x / den, -pv.y / den);   // 1 / pivot
    if (piv && j > k && j < n) {
      // column j of the trailing block: A[i][j] -= (A[i][k] / p) A[k][j]
      const double2 akj = A[k * ns + j];
      for (int i = k + 1; i < n; ++i) {
        const double2 a = A[i * ns + k];
        const double2 l = make_double2(a.x * rp.x - a.y * rp.y, a.x * rp.y + a.y * rp.x);
        double2 v = A[i * ns + j];
        v.x -= l.x * akj.x - l.y * akj.y;
        v.y -= l.x * akj.y + l.y * akj.x;
        A[i * ns + j] = v;
      }
    }
    __syncwarp();
  }
  return zero;
}

template <int G, int HB>
__global__ void __launch_bounds__(kThreads)
linear_detect_kernel(const double2* __restrict__ h, const double2* __restrict__ y,
                     int64_t n_vectors, int m, int n, int half_bits, int mmse,
                     double nv_scalar, const double* __restrict__ nv_vec, double clip,
                     uint8_t* __restrict__ labels_out, double* __restrict__ llr_out,
                     double2* __restrict__ est_out, int32_t* __restrict__ n_singular) {
  extern __shared__ double2 lsm[];
  constexpr int GPC = kThreads / G;   // vectors (groups) per CTA
  const int g = threadIdx.x / G, j = threadIdx.x % G;
  const int ns = n + 1;               // row stride of A; column n holds 1 / L[r][r]
  double2* A = lsm + (int64_t)g * n * ns;
  const int64_t v = (int64_t)blockIdx.x * GPC + g;
  const bool live = v < n_vectors;    // dead groups still run the shuffles (full masks)
  const int64_t vv = live ? v : 0;
  const double nv = nv_vec ? nv_vec[vv] : nv_scalar;
  const double2* hv = h + vv * (int64_t)m * n;
  const double2* yv = y + vv * (int64_t)m;
  const bool own = j < n;

  // ---- Gram (column j, 4 rows at a time) and matched filter x_j = (H^H y)_j ----
  double2 x = make_double2(0.0, 0.0);
  gram_column<G>(A, ns, hv, yv, m, n, j, mmse, nv, /*full=*/false, &x);
  __syncwarp();

  // ---- Cholesky A = L L^H (left-looking, in place on the lower triangle) ----
  // A suspect pivot does not decide singularity: np.linalg.inv (LAPACK getrf)
  // raises only on an exactly zero LU pivot, so suspects are re-examined below.
  const bool suspect = cholesky<G>(A, ns, n, j);
  // rare path: decide singularity as LAPACK's zgetf2 would (exact zero pivot
  // of the partially pivoted LU), then rebuild the Cholesky factor
  if (__any_sync(0xffffffffu, suspect && live)) {
    // (suspect is group-uniform; every group of the warp runs the LU)
    gram_column<G>(A, ns, hv, yv, m, n, j, mmse, nv, /*full=*/true, nullptr);
    __syncwarp();
    const bool singular = lu_zero_pivot<G>(A, ns, n, j);
    if (suspect && singular && j == 0 && live && n_singular) atomicAdd(n_singular, 1);
    __syncwarp();
    gram_column<G>(A, ns, hv, yv, m, n, j, mmse, nv, /*full=*/false, nullptr);
    __syncwarp();
    cholesky<G>(A, ns, n, j);
  }

  // ---- forward L w = x, then back L^H soft = w (column-oriented) ----
  const double rjj = own ? A[j * ns + n].x : 1.0;   // 1 / L[j][j]
  for (int c = 0; c < n; ++c) {
    if (j == c) { x.x *= rjj; x.y *= rjj; }
    const double wr = __shfl_sync(0xffffffffu, x.x, c, G), wi = __shfl_sync(0xffffffffu, x.y, c, G);
    if (j > c && j < n) {   // x_j -= L[j][c] w_c
      const double2 l = A[j * ns + c];
      x.x -= fma(l.x, wr, -l.y * wi);
      x.y -= fma(l.x, wi, l.y * wr);
    }
  }
  for (int c = n - 1; c >= 0; --c) {
    if (j == c) { x.x *= rjj; x.y *= rjj; }
    const double sr = __shfl_sync(0xffffffffu, x.x, c, G), si = __shfl_sync(0xffffffffu, x.y, c, G);
    if (j < c) {            // w_j -= conj(L[c][j]) s_c
      const double2 l = A[c * ns + j];
      x.x -= fma(l.x, sr, l.y * si);
      x.y -= fma(l.x, si, -l.y * sr);
    }
  }

  // ---- diag(A^-1)_j = sum_r |(L^-1)[r][j]|^2: lane j solves column j of L^-1,
  // its entries r > j kept in the (free) upper triangle, row j ----
  double dg = 0.0;
  if (own) {
    const double ujj = rjj;
    dg = ujj * ujj;
    for (int r = j + 1; r < n; ++r) {
      // u_rj = - (L[r][j] u_jj + sum_{j<k<r} L[r][k] u_kj) / L[r][r]
      const double2 lrj = A[r * ns + j];
      double sr = lrj.x * ujj, si = lrj.y * ujj;
      for (int k = j + 1; k < r; ++k) {
        const double2 l = A[r * ns + k], u = A[j * ns + k];
        sr = fma(l.x, u.x, fma(-l.y, u.y, sr));
        si = fma(l.x, u.y, fma(l.y, u.x, si));
      }
      const double rr = A[r * ns + n].x;   // 1 / L[r][r]
      const double2 u = make_double2(-sr * rr, -si * rr);
      A[j * ns + r] = u;
      dg = fma(u.x, u.x, fma(u.y, u.y, dg));
    }
  }

  if (!own || !live) return;
  double er, ei, nv_eff;
  if (mmse) {
    const double beta = fmax(1.0 - nv * dg, 1e-12);
    er = x.x / beta;
    ei = x.y / beta;
    nv_eff = fmax((1.0 - beta) / beta, 1e-15);
  } else {
    er = x.x;
    ei = x.y;
    nv_eff = nv * dg;
  }
  if (est_out) est_out[v * n + j] = x;   // raw (biased) soft
  // per-axis Gray levels (core.py:56-63) divided by the unit-energy scale
  // (core.py:73) once; the points are the same doubles the reference divides
  constexpr int NL = 1 << HB, Q = NL * NL, BPS = 2 * HB;
  const double norm = sqrt(2.0 * (double)(Q - 1) / 3.0);
  double lvn[NL];
#pragma unroll
  for (int pos = 0; pos < NL; ++pos) lvn[pos ^ (pos >> 1)] = double(NL - 1 - 2 * pos) / norm;
  // nearest point (first minimum) and max-log bit metrics over all Q points
  double d0[BPS], d1[BPS];
#pragma unroll
  for (int b = 0; b < BPS; ++b) { d0[b] = INFINITY; d1[b] = INFINITY; }
  double best = INFINITY;
  int best_lab = 0;
#pragma unroll
  for (int lab = 0; lab < Q; ++lab) {
    const double dr = er - lvn[lab >> HB], di = ei - lvn[lab & (NL - 1)];
    const double d = dr * dr + di * di;
    if (d < best) { best = d; best_lab = lab; }
#pragma unroll
    for (int b = 0; b < BPS; ++b) {
      if ((lab >> (BPS - 1 - b)) & 1) d1[b] = fmin(d1[b], d);
      else d0[b] = fmin(d0[b], d);
    }
  }
  labels_out[v * n + j] = (uint8_t)best_lab;
  double* lo = llr_out + (v * n + j) * BPS;
  const double rnv = 1.0 / nv_eff;
#pragma unroll
  for (int b = 0; b < BPS; ++b) {   // np.clip keeps NaN (fmin/fmax would not)
    double l = (d1[b] - d0[b]) * rnv;
    if (l < -clip) l = -clip;
    if (l > clip) l = clip;
    lo[b] = l;
  }
}

}  // namespace

namespace mpnl {

cudaError_t launch_linear_detect(const void* h, const void* y, int64_t n_vectors, int m, int n,
                                 int half_bits, int mmse, double nv_scalar, const double* nv_vec,
                                 double clip, uint8_t* labels_out, double* llr_out,
                                 void* est_out, int32_t* n_singular, cudaStream_t stream) {
  if (n_vectors == 0) return cudaSuccess;
  auto launch = [&](auto kern, int G) {
    const int gpc = kThreads / G;
    const size_t smem = (size_t)gpc * n * (n + 1) * sizeof(double2);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned blocks = (unsigned)((n_vectors + gpc - 1) / gpc);
    kern<<<blocks, kThreads, smem, stream>>>((const double2*)h, (const double2*)y, n_vectors, m,
                                             n, half_bits, mmse, nv_scalar, nv_vec, clip,
                                             labels_out, llr_out, (double2*)est_out, n_singular);
  };
#define MPNL_LIN(G)                                                                   \
  (half_bits == 1 ? launch(linear_detect_kernel<G, 1>, G)                             \
                  : half_bits == 2 ? launch(linear_detect_kernel<G, 2>, G)            \
                                   : launch(linear_detect_kernel<G, 3>, G))
  if (n <= 8) MPNL_LIN(8);
  else if (n <= 16) MPNL_LIN(16);
  else MPNL_LIN(32);
#undef MPNL_LIN
  return cudaGetLastError();
}

int linear_max_n() { return kMaxN; }

}  // namespace mpnl
