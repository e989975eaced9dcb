// K1 — per-channel planning: fp64 sorted (column-pivoted) complex QR and the
// fp32 traversal tables.
//
// Follows the reference planner `mpnl_plan_batch` / `_sorted_qr_batch`
// (`/root/reference/pkg/src/mpnlsim/detect.py:321-388`):
//   * right-looking modified Gram-Schmidt on A = H, or [H; sqrt(nv) I] when
//     N > M (detect.py:373-381);
//   * pivot = first argmax (in current column order) of the *downdated* norms
//     max(norm_j - |r_kj|^2, 0) (detect.py:335, 357);
//   * r_kk recomputed from the pivot column, floored at 1e-300 (348-350);
//   * Q^H = top M rows of Q, conjugate-transposed (383).
//
// B200 mapping: channels of up to 32 rows (every BASELINE config) take
// `plan_qr_reg_kernel`: a lane group of 8 / 16 / 32 lanes per channel, lane j
// holding column j of A in registers, no block barriers (see the kernel's
// comment).  Taller channels (m, or m + n when augmented, above 32) take
// `plan_qr_kernel`: one 4-warp CTA per channel, lane j owning *physical* column
// j of A in shared memory (A[m][j], padded rows), the column bookkeeping
// (norms, logical positions) replicated identically in every warp so that
// column swaps are pure bookkeeping, each warp owning a quarter of the rows for
// the projections and updates (partials summed in a fixed order), r_kk a block
// reduction over rows.  One kernel per shape, whatever the number of channels:
// plans never depend on the batch size.
// Everything is fp64; the fast path's fp32 tables are derived at the end.
#include "common.cuh"

namespace mpnl {

template <typename TIn>
__device__ inline double2 load_c(const TIn* p, int64_t i);
template <>
__device__ inline double2 load_c<float2>(const float2* p, int64_t i) {
  float2 v = p[i];
  return make_double2(v.x, v.y);
}
template <>
__device__ inline double2 load_c<double2>(const double2* p, int64_t i) {
  return p[i];
}

__device__ inline double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Outputs of a finished plan (shared by both plan kernels): perm, R and Q^H in
// logical order, and the fp32 traversal tables (TableLayout).  Threads t of T.
// perm, R (logical order) and the R-derived fp32 tables; threads t of T
__device__ inline void plan_epilogue_r(const double2* Rp, const int* phys_of, int64_t c, int m,
                                       int n, int L, int32_t* __restrict__ perm_out,
                                       double2* __restrict__ r_out, float* __restrict__ tables,
                                       int t, int T) {
  int32_t* pc = perm_out + c * n;
  double2* rc = r_out + c * (int64_t)n * n;
  for (int idx = t; idx < n; idx += T) pc[idx] = phys_of[idx];
  for (int idx = t; idx < n * n; idx += T) {
    const int i = idx / n, j = idx - i * n;
    rc[idx] = (j >= i) ? Rp[i * n + phys_of[j]] : make_double2(0.0, 0.0);
  }
  if (tables == nullptr) return;
  const TableLayout tl(m, n);
  float* tc = tables + c * (int64_t)tl.total;
  const double nrm = qam_norm_d(L);
  const double sc = 2.0 / nrm;
  const double lv = (double)(L - 1) / nrm;
  for (int idx = t; idx < n * 2 * tl.npp; idx += T) {
    const int pos = idx / (2 * tl.npp), k = idx % (2 * tl.npp);   // column pos, row k
    float2 v = make_float2(0.f, 0.f);
    if (k < pos) {
      const double2 r = Rp[k * n + phys_of[pos]];
      v = make_float2((float)(sc * r.x), (float)(sc * r.y));
    }
    float* blk = tc + tl.off_rcol + 4 * (pos * tl.npp + (k >> 1)) + 2 * (k & 1);
    blk[0] = v.x;   // {rr_2q, ri_2q, rr_2q+1, ri_2q+1}
    blk[1] = v.y;
  }
  for (int k = t; k < n; k += T) {
    double sr = 0.0, si = 0.0, sabs = 0.0;
    for (int j = k; j < n; ++j) {
      const double2 r = Rp[k * n + phys_of[j]];
      sr += r.x;
      si += r.y;
      if (j > k) sabs += (double)fabsf((float)(sc * r.x)) + (double)fabsf((float)(sc * r.y));
    }
    // shift = (L-1)(1+i)/norm * sum_{j>=k} r_kj
    const double shr = lv * (sr - si), shi = lv * (sr + si);
    reinterpret_cast<double2*>(tc + tl.off_shift)[k] = make_double2(shr, shi);
    const double rkk = Rp[k * n + phys_of[k]].x;
    const double c2r = sc * rkk;
    float* ly = tc + tl.off_lay + 4 * k;
    ly[0] = (float)(-1.0 / c2r);   // kx: acc -> level-index units
    ly[1] = (float)c2r;
    // guard input S_k = sum_{j>k} |Re r''| + |Im r''| (as stored)
    ly[2] = (float)(sabs * (1.0 + 1e-6));
    // kxs: acc -> saturated slicing domain [0, 1] (level index / (L - 1))
    ly[3] = (float)(-1.0 / (c2r * (double)(L - 1)));
  }
}

// The same plus Q^H (outputs and the table's transposed copy) from A in shared memory.
__device__ inline void plan_epilogue(const double2* A, int ns, const double2* Rp,
                                     const int* phys_of, int64_t c, int m, int n, int L,
                                     int32_t* __restrict__ perm_out, double2* __restrict__ r_out,
                                     double2* __restrict__ qh_out, float* __restrict__ tables,
                                     int t, int T) {
  double2* qc = qh_out + c * (int64_t)n * m;
  for (int idx = t; idx < n * m; idx += T) {
    const int k = idx / m, r = idx - k * m;
    const double2 q = A[r * ns + phys_of[k]];
    qc[idx] = make_double2(q.x, -q.y);
  }
  if (tables != nullptr) {
    const TableLayout tl(m, n);
    double2* qt = reinterpret_cast<double2*>(tables + c * (int64_t)tl.total + tl.off_qh);
    for (int idx = t; idx < n * m; idx += T) {
      const int r = idx / n, k = idx - r * n;   // transposed: qhT[r][k] = conj(q_k[r])
      const double2 q = A[r * ns + phys_of[k]];
      qt[idx] = make_double2(q.x, -q.y);
    }
  }
  plan_epilogue_r(Rp, phys_of, c, m, n, L, perm_out, r_out, tables, t, T);
}

#define PLAN_THREADS 128
#define PLAN_WARPS (PLAN_THREADS / 32)

template <typename TIn>
__global__ void __launch_bounds__(PLAN_THREADS)
plan_qr_kernel(const TIn* __restrict__ h, int64_t n_ch, int m, int n, int L,
               double noise_var, int augmented, int32_t* __restrict__ perm_out,
               double2* __restrict__ r_out, double2* __restrict__ qh_out,
               float* __restrict__ tables) {
  extern __shared__ double2 smem[];
  const int ma = augmented ? m + n : m;
  const int ns = n + 1;           // padded row stride: row-parallel column access spreads banks
  double2* A = smem;              // [ma][ns] physical columns
  double2* Rp = smem + ma * ns;   // [n][n] rows of R by physical column
  double2* red = Rp + n * n;      // [PLAN_WARPS][32] partial dot products
  double* rkp = reinterpret_cast<double*>(red + PLAN_WARPS * 32);   // [PLAN_WARPS] partial norms
  const int64_t c = blockIdx.x;
  if (c >= n_ch) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  // ---- load A (coalesced over the (m, n) row-major input) ----
  const TIn* hc = h + c * (int64_t)m * n;
  for (int idx = tid; idx < m * n; idx += PLAN_THREADS) {
    const int r = idx / n, j = idx - r * n;
    A[r * ns + j] = load_c<TIn>(hc, idx);
  }
  if (augmented) {
    const double s = sqrt(noise_var);
    for (int idx = tid; idx < n * n; idx += PLAN_THREADS) {
      int i = idx / n, j = idx % n;
      A[(m + i) * ns + j] = make_double2(i == j ? s : 0.0, 0.0);
    }
  }
  for (int idx = tid; idx < n * n; idx += PLAN_THREADS) Rp[idx] = make_double2(0.0, 0.0);
  __syncthreads();

  // Column bookkeeping in warp 0: lane j owns physical column j (downdated
  // norm, logical position); the pivot and the chosen set are published
  // through shared memory for the other warps.
  __shared__ int piv_s;
  __shared__ unsigned chosen_s;
  const bool own = lane < n;
  double norm = 0.0;
  if (w == 0 && own)
    for (int r = 0; r < ma; ++r) {
      double2 a = A[r * ns + lane];
      norm = fma(a.x, a.x, fma(a.y, a.y, norm));
    }
  int logpos = lane;     // logical position of my physical column (warp 0)
  bool chosen = !own;
  int my_final = -1;     // final logical position (== step at which chosen)
  // rows of this warp for the column updates
  const int rb = (ma + PLAN_WARPS - 1) / PLAN_WARPS;
  const int r0 = w * rb, r1 = min(ma, r0 + rb);

  for (int k = 0; k < n; ++k) {
    if (w == 0) {
      // pivot: max downdated norm, ties -> smallest logical position (first max)
      double bv = chosen ? -1.0 : norm;
      int bp = chosen ? 0x7fffffff : logpos;
      int bl = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int op = __shfl_xor_sync(0xffffffffu, bp, o);
        int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bl = ol; }
      }
      // exchange logical positions of column-at-k and the pivot column
      if (!chosen && logpos == k) logpos = bp;
      if (lane == bl) { logpos = k; chosen = true; my_final = k; }
      const unsigned cm = __ballot_sync(0xffffffffu, chosen);
      if (lane == 0) { piv_s = bl; chosen_s = cm; }
    }
    __syncthreads();
    const int cp = piv_s;                   // physical pivot column
    const bool ch = (chosen_s >> lane) & 1u;

    // r_kk from the pivot column (thread per row, fixed-order block reduction)
    double part = 0.0;
    if (tid < ma) {
      const double2 a = A[tid * ns + cp];
      part = fma(a.x, a.x, a.y * a.y);
    }
    part = warp_sum_d(part);
    if (lane == 0) rkp[w] = part;
    __syncthreads();
    double rkk = 0.0;
    if (lane == 0) {   // one sqrt per warp (the MUFU/slow path is costly), then broadcast
      double ss = 0.0;
#pragma unroll
      for (int i = 0; i < PLAN_WARPS; ++i) ss += rkp[i];
      rkk = fmax(sqrt(ss), 1e-300);
    }
    rkk = __shfl_sync(0xffffffffu, rkk, 0);
    if (tid < ma) {
      const double2 a = A[tid * ns + cp];
      A[tid * ns + cp] = make_double2(a.x / rkk, a.y / rkk);
    }
    if (tid == 0) Rp[k * n + cp] = make_double2(rkk, 0.0);
    __syncthreads();
    // proj_j = q^H a_j over this warp's rows -> partials -> fixed-order sum
    double pr = 0.0, pi = 0.0;
    if (!ch) {
      double pr2 = 0.0, pi2 = 0.0;
      int r = r0;
      for (; r + 2 <= r1; r += 2) {
        const double2 q = A[r * ns + cp], a = A[r * ns + lane];
        const double2 q2 = A[(r + 1) * ns + cp], a2 = A[(r + 1) * ns + lane];
        pr = fma(q.x, a.x, fma(q.y, a.y, pr));      // conj(q) * a
        pi = fma(q.x, a.y, fma(-q.y, a.x, pi));
        pr2 = fma(q2.x, a2.x, fma(q2.y, a2.y, pr2));
        pi2 = fma(q2.x, a2.y, fma(-q2.y, a2.x, pi2));
      }
      if (r < r1) {
        const double2 q = A[r * ns + cp], a = A[r * ns + lane];
        pr = fma(q.x, a.x, fma(q.y, a.y, pr));
        pi = fma(q.x, a.y, fma(-q.y, a.x, pi));
      }
      red[w * 32 + lane] = make_double2(pr + pr2, pi + pi2);
    }
    __syncthreads();
    if (!ch) {
      pr = 0.0;
      pi = 0.0;
#pragma unroll
      for (int i = 0; i < PLAN_WARPS; ++i) { pr += red[i * 32 + lane].x; pi += red[i * 32 + lane].y; }
      if (w == 0) Rp[k * n + lane] = make_double2(pr, pi);
      for (int rr = r0; rr < r1; ++rr) {
        const double2 q = A[rr * ns + cp];
        double2 a = A[rr * ns + lane];
        a.x -= q.x * pr - q.y * pi;
        a.y -= q.x * pi + q.y * pr;
        A[rr * ns + lane] = a;
      }
      norm = fmax(norm - (pr * pr + pi * pi), 0.0);
    }
    // (no barrier here: the next step's pivot needs only warp 0's own norms,
    // and its first barrier orders these updates before the next reads of A)
  }
  __syncthreads();

  // ---- outputs in logical order ----
  __shared__ int phys_of[MPNL_MAX_N];
  if (w == 0 && own) phys_of[my_final] = lane;
  __syncthreads();
  plan_epilogue(A, ns, Rp, phys_of, c, m, n, L, perm_out, r_out, qh_out, tables, tid,
                PLAN_THREADS);
}


// ---------------------------------------------------------------------------
// Register-resident plan kernel (ma <= 32): a lane GROUP of G >= n lanes per
// channel (32 / G channels per warp, no block barriers), lane j of the group
// owning physical column j of A *in registers* (MA rows, zero-padded).  Per
// step: group argmax of the downdated norms -> the pivot lane publishes its
// column to the group's shared-memory slot -> lane r normalises row r (r_kk by
// a group butterfly over the rows, one sqrt and two divisions per lane) and
// writes Q^H's row k straight to the outputs (the pivot column is final) ->
// every unchosen lane projects and updates its own column from registers,
// reading q as shared-memory broadcasts.  R is kept by physical column in
// shared memory and put in logical order at the end.  Against the CTA kernel
// (one block barrier chain per column, A in shared memory): C5's 2,048
// 24 x 24 channels 131 -> 90 us, 8,192 8 x 8 channels 66 -> 25 us.
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ double group_sum_d(double v) {
#pragma unroll
  for (int o = G / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct PlanRegSmem {   // per group, in double2 units
  int rp, q, phys, total;
  __host__ __device__ PlanRegSmem(int n) {
    rp = 0;              // [n][n] rows of R by physical column
    q = rp + n * n;      // [32] the step's pivot column (raw, then normalised; zero tail)
    phys = q + 32;       // [n] int: physical column of each logical position
    total = phys + (n + 3) / 4;
  }
};

#if defined(__CUDACC_VER_MAJOR__) && (__CUDACC_VER_MAJOR__ * 100 + __CUDACC_VER_MINOR__ >= 1204)
#define MPNL_MAXNREG(N) __maxnreg__(N)
#else
#define MPNL_MAXNREG(N)
#endif

// 16 resident warps per SM for MA <= 24 (128 registers): C5's 2,048 channels in one wave
template <int MA, int G, typename TIn>
__global__ void MPNL_MAXNREG(MA <= 24 ? 128 : 248)
plan_qr_reg_kernel(const TIn* __restrict__ h, int64_t n_ch, int m, int n, int L, double noise_var,
                   int augmented, int32_t* __restrict__ perm_out, double2* __restrict__ r_out,
                   double2* __restrict__ qh_out, float* __restrict__ tables) {
  extern __shared__ double2 smem[];
  constexpr int GPW = 32 / G;             // channels per warp
  constexpr int RPL0 = (MA + G - 1) / G;
  constexpr int RPL = RPL0 <= 1 ? 1 : (RPL0 <= 2 ? 2 : 4);   // rows per lane, row-parallel phases
  static_assert(RPL * G <= 32, "pivot column slot");
  const int ma = augmented ? m + n : m;
  const PlanRegSmem so(n);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gl = lane % G, gi = lane / G;
  const int64_t cg = ((int64_t)blockIdx.x * (blockDim.x >> 5) + w) * GPW + gi;
  const bool valid = cg < n_ch;
  const int64_t c = valid ? cg : n_ch - 1;   // idle groups shadow the last channel (stores masked)
  double2* base = smem + (int64_t)(w * GPW + gi) * so.total;
  double2* Rp = base + so.rp;
  double2* qb = base + so.q;
  int* phys_of = reinterpret_cast<int*>(base + so.phys);
  const TableLayout tl(m, n);
  const bool own = gl < n;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (gi * G));

  // ---- my column into registers (rows >= ma are zero, and stay zero) ----
  double2 col[MA];
  {
    const TIn* hc = h + c * (int64_t)m * n;
    const double s = augmented ? sqrt(noise_var) : 0.0;
#pragma unroll
    for (int r = 0; r < MA; ++r) {
      double2 v = make_double2(0.0, 0.0);
      if (own && r < m) v = load_c<TIn>(hc, r * n + gl);
      else if (own && r < ma && r - m == gl) v = make_double2(s, 0.0);
      col[r] = v;
    }
  }
  qb[gl] = make_double2(0.0, 0.0);
  if (G < 32) {
#pragma unroll
    for (int i = 1; i < 32 / G; ++i) qb[gl + i * G] = make_double2(0.0, 0.0);
  }
  double norm = 0.0;
#pragma unroll
  for (int r = 0; r < MA; ++r) norm = fma(col[r].x, col[r].x, fma(col[r].y, col[r].y, norm));
  int logpos = gl;
  bool chosen = !own;
  int my_final = -1;
  // Q^H row k is written by lane r = row (outputs [k][r], table copy [r][k])
  double2* qc = qh_out + c * (int64_t)n * m;
  double2* qt = reinterpret_cast<double2*>(tables + c * (int64_t)tl.total + tl.off_qh);
  const bool wq = valid, wt = valid && tables != nullptr;
  __syncwarp();

  for (int k = 0; k < n; ++k) {
    // pivot: max downdated norm, ties -> smallest logical position (first max).
    // norm >= 0, so its bit pattern orders as an unsigned integer: three group
    // reductions (high word, low word among the high-word maxima, logical position
    // among the maxima) replace a five-round shuffle butterfly on (double, int, int)
    const unsigned nh = (unsigned)__double2hiint(norm), nl = (unsigned)__double2loint(norm);
    const unsigned hk = chosen ? 0u : nh + 1u;
    const unsigned mh = __reduce_max_sync(gmask, hk);
    const unsigned ml = __reduce_max_sync(gmask, hk == mh ? nl : 0u);
    const bool cand = !chosen && hk == mh && nl == ml;
    const int bp = (int)__reduce_min_sync(gmask, cand ? (unsigned)logpos : 0x7fffffffu);
    const unsigned wb = __ballot_sync(0xffffffffu, cand && logpos == bp);
    const int cp = __ffs((int)((wb >> (gi * G)) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u)))) - 1;
    if (!chosen && logpos == k) logpos = bp;
    const bool piv = gl == cp;
    if (piv) {
      logpos = k;
      chosen = true;
      my_final = k;
#pragma unroll
      for (int r = 0; r < MA; ++r) qb[r] = col[r];
    }
    __syncwarp();
    // r_kk and the normalised column, row-parallel (lane gl: rows gl, gl + G, ...);
    // the sum follows a 32-lane butterfly over the rows (offsets 16, 8, ..): the
    // in-lane rows gl + i G are its highest offsets
    double2 a[RPL];
    double pr_[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      a[i] = qb[gl + i * G];
      pr_[i] = fma(a[i].x, a[i].x, a[i].y * a[i].y);
    }
#pragma unroll
    for (int o = RPL / 2; o; o >>= 1)
#pragma unroll
      for (int i = 0; i < o; ++i) pr_[i] += pr_[i + o];
    const double ss = group_sum_d<G>(pr_[0]);
    const double rkk = fmax(sqrt(ss), 1e-300);
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = gl + i * G;
      // (padding rows stay zero; dividing them would send the warp down the
      // division's slow path for tiny numerators)
      double2 q = make_double2(0.0, 0.0);
      if (r < ma) q = make_double2(a[i].x / rkk, a[i].y / rkk);
      qb[r] = q;
      if (r < m) {   // Q^H row k (logical): final at this step
        const double2 qcj = make_double2(q.x, -q.y);
        if (wq) qc[k * m + r] = qcj;
        if (wt) qt[r * n + k] = qcj;
      }
    }
    if (piv) Rp[k * n + gl] = make_double2(rkk, 0.0);
    __syncwarp();
    if (!chosen) {
      // proj = q^H a_j: four interleaved chains over the rows (zero rows are exact no-ops)
      double pr[4] = {0.0, 0.0, 0.0, 0.0}, pi[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int r = 0; r < MA; ++r) {
        const double2 q = qb[r];
        pr[r & 3] = fma(q.x, col[r].x, fma(q.y, col[r].y, pr[r & 3]));      // conj(q) * a
        pi[r & 3] = fma(q.x, col[r].y, fma(-q.y, col[r].x, pi[r & 3]));
      }
      const double sr = (pr[0] + pr[1]) + (pr[2] + pr[3]);
      const double si = (pi[0] + pi[1]) + (pi[2] + pi[3]);
      Rp[k * n + gl] = make_double2(sr, si);
#pragma unroll
      for (int r = 0; r < MA; ++r) {
        const double2 q = qb[r];
        col[r].x = fma(-q.x, sr, fma(q.y, si, col[r].x));   // a_j -= q r_kj
        col[r].y = fma(-q.x, si, fma(-q.y, sr, col[r].y));
      }
      norm = fmax(norm - (sr * sr + si * si), 0.0);
    }
    __syncwarp();
  }
  if (own) phys_of[my_final] = gl;
  __syncwarp();
  if (!valid) return;
  plan_epilogue_r(Rp, phys_of, c, m, n, L, perm_out, r_out, tables, gl, G);
}

template __global__ void plan_qr_kernel<float2>(const float2*, int64_t, int, int, int, double,
                                                int, int32_t*, double2*, double2*, float*);
template __global__ void plan_qr_kernel<double2>(const double2*, int64_t, int, int, int, double,
                                                 int, int32_t*, double2*, double2*, float*);

template <int MA, int G, typename TIn>
static cudaError_t launch_plan_reg(const TIn* h, int64_t n_ch, int m, int n, int L, double noise_var,
                                   int augmented, int32_t* perm, double2* r64, double2* qh64,
                                   float* tables, cudaStream_t st) {
  constexpr int WARPS = 2, GPC = WARPS * (32 / G);   // groups (channels) per CTA
  const size_t smem = (size_t)GPC * PlanRegSmem(n).total * sizeof(double2);
  auto k = plan_qr_reg_kernel<MA, G, TIn>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<(unsigned)((n_ch + GPC - 1) / GPC), 32 * WARPS, smem, st>>>(h, n_ch, m, n, L, noise_var,
                                                                 augmented, perm, r64, qh64, tables);
  return cudaGetLastError();
}

template <typename TIn>
static cudaError_t launch_plan_t(const TIn* h, int64_t n_ch, int m, int n, int L, double noise_var,
                                 int augmented, int32_t* perm, double2* r64, double2* qh64,
                                 float* tables, cudaStream_t st) {
  const int ma = augmented ? m + n : m;
  if (ma <= 32) {
    // lane group per channel, columns in registers (row count bucket x group width)
#define MPNL_PR(MA_, G_) \
    return launch_plan_reg<MA_, G_, TIn>(h, n_ch, m, n, L, noise_var, augmented, perm, r64, qh64, \
                                         tables, st)
    if (n <= 8) {
      if (ma <= 8) MPNL_PR(8, 8);
      if (ma <= 16) MPNL_PR(16, 8);
      if (ma <= 24) MPNL_PR(24, 8);
      MPNL_PR(32, 8);
    }
    if (n <= 16) {
      if (ma <= 16) MPNL_PR(16, 16);
      if (ma <= 24) MPNL_PR(24, 16);
      MPNL_PR(32, 16);
    }
    if (ma <= 24) MPNL_PR(24, 32);
    MPNL_PR(32, 32);
#undef MPNL_PR
  }
  // taller channels (m (+ n) > 32): one 4-warp CTA per channel, A in shared memory
  const size_t smem = (size_t)(ma * (n + 1) + n * n + PLAN_WARPS * 32) * sizeof(double2) +
                      PLAN_WARPS * sizeof(double);
  cudaFuncSetAttribute(plan_qr_kernel<TIn>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  plan_qr_kernel<TIn><<<(unsigned)n_ch, PLAN_THREADS, smem, st>>>(h, n_ch, m, n, L, noise_var,
                                                                  augmented, perm, r64, qh64, tables);
  return cudaGetLastError();
}

cudaError_t launch_plan(const void* h, int h_is_f64, int64_t n_ch, int m, int n, int L,
                        double noise_var, int augmented, int32_t* perm, double2* r64,
                        double2* qh64, float* tables, cudaStream_t st) {
  if (n_ch == 0) return cudaSuccess;
  if (h_is_f64)
    return launch_plan_t<double2>((const double2*)h, n_ch, m, n, L, noise_var, augmented, perm, r64,
                                  qh64, tables, st);
  return launch_plan_t<float2>((const float2*)h, n_ch, m, n, L, noise_var, augmented, perm, r64,
                               qh64, tables, st);
}

}  // namespace mpnl
