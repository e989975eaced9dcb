// Batched linear ZF / MMSE detection with max-log LLRs.
//
// Follows linear_detect_batch (pkg/src/mpnlsim/detect.py:528-557) and the
// per-symbol max-log demapper it calls (core.py:191-206):
//   A = H^H H (+ nv I for MMSE), soft = A^-1 H^H y, d = diag(A^-1)
//   ZF:   est = soft,        nv_eff = nv d
//   MMSE: beta = max(1 - nv d, 1e-12), est = soft / beta,
//         nv_eff = max((1 - beta) / beta, 1e-15)
//   labels = nearest point (first minimum, np.argmin), llr = (d1 - d0) / nv_eff
//   clipped to +-clip.
// The reference inverts A with LAPACK; here A (Hermitian, positive definite
// unless the channel is rank deficient) is factorised by Cholesky in fp64
// per-thread local memory, soft comes from two triangular solves and diag(A^-1)
// from the column norms of L^-1.  Same quantities, different rounding: the
// parity tests compare soft values and LLRs within a stated tolerance and the
// hard labels exactly.  An exactly zero (or non-finite) pivot marks the vector
// singular, where the reference's np.linalg.inv (LAPACK getrf) raises
// LinAlgError; the count goes to *n_singular.
//
// One thread per vector: O(M N^2 + N^3) fp64 flops on 16 (M N + M) input bytes
// per vector; vectors are independent.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kMaxN = 16;

struct cd { double re, im; };
struct Tri {          // strided view: element e of this thread's triangle
  double2* p;
  int s;
  __device__ __forceinline__ double2& operator[](int e) const { return p[e * s]; }
};
struct Row {          // row i of the triangle
  Tri t;
  int o;
  __device__ __forceinline__ double2& operator[](int k) const { return t[o + k]; }
};
__device__ __forceinline__ cd cmul_conj_a(cd a, cd b) {  // conj(a) * b
  return {a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}

// NT > 0: stream count known at compile time (loops unroll, small arrays stay
// in registers); NT = 0: run-time n <= kMaxN.
template <int NT>
__global__ void __launch_bounds__(128)
linear_detect_kernel(const double2* __restrict__ h, const double2* __restrict__ y,
                     int64_t n_vectors, int m, int n_rt, int half_bits, int mmse,
                     double nv_scalar, const double* __restrict__ nv_vec, double clip,
                     uint8_t* __restrict__ labels_out, double* __restrict__ llr_out,
                     double2* __restrict__ est_out, int32_t* __restrict__ n_singular) {
  constexpr int kN = NT ? NT : kMaxN;
  const int n = NT ? NT : n_rt;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n_vectors) return;
  const double nv = nv_vec ? nv_vec[v] : nv_scalar;
  const double2* hv = h + v * (int64_t)m * n;
  const double2* yv = y + v * (int64_t)m;

  // packed lower triangle (row i at i(i+1)/2) in thread-local memory.  A
  // shared-memory triangle (element-major across the CTA) measured slower:
  // 12x12 3.30 -> 3.80 ms, 16x16 8.4 -> 22 ms (occupancy capped by 139 KB/CTA)
  double2 tri_local[kN * (kN + 1) / 2];
  Tri L{tri_local, 1};
  cd x[kN];
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j <= i; ++j) L[i * (i + 1) / 2 + j] = make_double2(0.0, 0.0);
    x[i] = {0.0, 0.0};
  }
  // Gram lower triangle and matched filter H^H y (detect.py:533-534)
  for (int r = 0; r < m; ++r) {
    const double2 yr = yv[r];
    for (int i = 0; i < n; ++i) {
      const double2 hi = hv[r * n + i];
      const cd a{hi.x, hi.y};
      const cd t = cmul_conj_a(a, {yr.x, yr.y});
      x[i].re += t.re; x[i].im += t.im;
      for (int j = 0; j <= i; ++j) {
        const double2 hj = hv[r * n + j];
        const cd g = cmul_conj_a(a, {hj.x, hj.y});
        double2& e = L[i * (i + 1) / 2 + j];
        e.x += g.re;
        e.y += g.im;
      }
    }
  }
  if (mmse)
    for (int i = 0; i < n; ++i) L[i * (i + 1) / 2 + i].x += nv;
  // Cholesky A = L L^H in place (row i of L: L[i][j], j <= i)
  bool singular = false;
  for (int j = 0; j < n; ++j) {
    const Row rj{L, j * (j + 1) / 2};
    double d = rj[j].x;
    for (int k = 0; k < j; ++k) d -= rj[k].x * rj[k].x + rj[k].y * rj[k].y;
    // LAPACK getrf (np.linalg.inv) raises only on an exactly zero pivot: flag
    // a zero / non-finite pivot; a rounding-level negative one goes on as |d|
    // (A is then numerically singular and, as in the reference, the outputs
    // are whatever the factorisation gives)
    if (!(d != 0.0) || !isfinite(d)) { singular = true; d = 1.0; }
    d = fabs(d);
    const double ljj = sqrt(d), inv = 1.0 / ljj;
    rj[j] = make_double2(ljj, 0.0);
    for (int i = j + 1; i < n; ++i) {
      const Row ri{L, i * (i + 1) / 2};
      double sr = ri[j].x, si = ri[j].y;
      for (int k = 0; k < j; ++k) {   // - L[i][k] conj(L[j][k])
        sr -= ri[k].x * rj[k].x + ri[k].y * rj[k].y;
        si -= ri[k].y * rj[k].x - ri[k].x * rj[k].y;
      }
      ri[j] = make_double2(sr * inv, si * inv);
    }
  }
  if (singular && n_singular) atomicAdd(n_singular, 1);
  // forward L w = H^H y, back L^H soft = w
  for (int i = 0; i < n; ++i) {
    const Row ri{L, i * (i + 1) / 2};
    double sr = x[i].re, si = x[i].im;
    for (int k = 0; k < i; ++k) {
      sr -= ri[k].x * x[k].re - ri[k].y * x[k].im;
      si -= ri[k].x * x[k].im + ri[k].y * x[k].re;
    }
    x[i] = {sr / ri[i].x, si / ri[i].x};
  }
  for (int i = n - 1; i >= 0; --i) {
    double sr = x[i].re, si = x[i].im;
    for (int k = i + 1; k < n; ++k) {   // - conj(L[k][i]) x[k]
      const double2 lk = L[k * (k + 1) / 2 + i];
      sr -= lk.x * x[k].re + lk.y * x[k].im;
      si -= lk.x * x[k].im - lk.y * x[k].re;
    }
    const double lii = L[i * (i + 1) / 2 + i].x;
    x[i] = {sr / lii, si / lii};
  }

  // per-axis Gray levels (core.py:56-63) and the unit-energy scale (core.py:73)
  const int nl = 1 << half_bits;
  double lv[8];
  for (int pos = 0; pos < nl; ++pos) lv[pos ^ (pos >> 1)] = double(nl - 1 - 2 * pos);
  const double norm = sqrt(2.0 * (double)((1 << (2 * half_bits)) - 1) / 3.0);
  const int q = 1 << (2 * half_bits), bps = 2 * half_bits;

  for (int i = 0; i < n; ++i) {
    // diag(A^-1)_i = || column i of L^-1 ||^2: solve L w = e_i from row i on
    cd w[kN];
    double dg = 0.0;
    for (int r = i; r < n; ++r) {
      const Row rr{L, r * (r + 1) / 2};
      double sr = (r == i) ? 1.0 : 0.0, si = 0.0;
      for (int k = i; k < r; ++k) {
        sr -= rr[k].x * w[k].re - rr[k].y * w[k].im;
        si -= rr[k].x * w[k].im + rr[k].y * w[k].re;
      }
      w[r] = {sr / rr[r].x, si / rr[r].x};
      dg += w[r].re * w[r].re + w[r].im * w[r].im;
    }
    double er, ei, nv_eff;
    if (mmse) {
      const double beta = fmax(1.0 - nv * dg, 1e-12);
      er = x[i].re / beta; ei = x[i].im / beta;
      nv_eff = fmax((1.0 - beta) / beta, 1e-15);
    } else {
      er = x[i].re; ei = x[i].im;
      nv_eff = nv * dg;
    }
    if (est_out) est_out[v * n + i] = make_double2(x[i].re, x[i].im);   // raw (biased) soft
    // nearest point (first minimum) and max-log bit metrics over all Q points
    double d0[6], d1[6];
    for (int b = 0; b < bps; ++b) { d0[b] = INFINITY; d1[b] = INFINITY; }
    double best = INFINITY;
    int best_lab = 0;
    for (int lab = 0; lab < q; ++lab) {
      const double pr = lv[lab >> half_bits] / norm, pi = lv[lab & (nl - 1)] / norm;
      const double dr = er - pr, di = ei - pi;
      const double d = dr * dr + di * di;
      if (d < best) { best = d; best_lab = lab; }
      for (int b = 0; b < bps; ++b) {
        if ((lab >> (bps - 1 - b)) & 1) d1[b] = fmin(d1[b], d);
        else d0[b] = fmin(d0[b], d);
      }
    }
    labels_out[v * n + i] = (uint8_t)best_lab;
    double* lo = llr_out + (v * n + i) * bps;
    for (int b = 0; b < bps; ++b) {   // np.clip keeps NaN (fmin/fmax would not)
      double l = (d1[b] - d0[b]) / nv_eff;
      if (l < -clip) l = -clip;
      if (l > clip) l = clip;
      lo[b] = l;
    }
  }
}

}  // namespace

namespace mpnl {

cudaError_t launch_linear_detect(const void* h, const void* y, int64_t n_vectors, int m, int n,
                                 int half_bits, int mmse, double nv_scalar, const double* nv_vec,
                                 double clip, uint8_t* labels_out, double* llr_out,
                                 void* est_out, int32_t* n_singular, cudaStream_t stream) {
  if (n_vectors == 0) return cudaSuccess;
  const int threads = 128;
  const unsigned blocks = (unsigned)((n_vectors + threads - 1) / threads);
#define MPNL_LIN(NT)                                                                     \
  linear_detect_kernel<NT><<<blocks, threads, 0, stream>>>(                              \
      (const double2*)h, (const double2*)y, n_vectors, m, n, half_bits, mmse, nv_scalar, \
      nv_vec, clip, labels_out, llr_out, (double2*)est_out, n_singular)
  // compile-time N measured faster only for small N (2x2 QPSK 0.040 -> 0.026 ms);
  // 12 and 16 unrolled spill more and ran slower (3.27 -> 4.15, 8.35 -> 8.96 ms)
  switch (n) {
    case 2: MPNL_LIN(2); break;
    case 4: MPNL_LIN(4); break;
    case 8: MPNL_LIN(8); break;
    default: MPNL_LIN(0); break;
  }
#undef MPNL_LIN
  return cudaGetLastError();
}

int linear_max_n() { return kMaxN; }

}  // namespace mpnl
