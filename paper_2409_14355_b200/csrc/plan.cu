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
// B200 mapping: one 4-warp CTA per channel.  Lane j owns *physical* column j
// of A in shared memory (A[m][j], padded rows); the column bookkeeping (norms,
// logical positions) is replicated identically in every warp, so column swaps
// are pure bookkeeping and no data moves.  Each warp owns a quarter of the
// rows for the projections and updates (partials summed in a fixed order);
// r_kk is a block reduction over rows.
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
__device__ inline void plan_epilogue(const double2* A, int ns, const double2* Rp,
                                     const int* phys_of, int64_t c, int m, int n, int L,
                                     int32_t* __restrict__ perm_out, double2* __restrict__ r_out,
                                     double2* __restrict__ qh_out, float* __restrict__ tables,
                                     int t, int T) {
  int32_t* pc = perm_out + c * n;
  double2* rc = r_out + c * (int64_t)n * n;
  double2* qc = qh_out + c * (int64_t)n * m;
  for (int idx = t; idx < n; idx += T) pc[idx] = phys_of[idx];
  for (int idx = t; idx < n * n; idx += T) {
    const int i = idx / n, j = idx - i * n;
    rc[idx] = (j >= i) ? Rp[i * n + phys_of[j]] : make_double2(0.0, 0.0);
  }
  for (int idx = t; idx < n * m; idx += T) {
    const int k = idx / m, r = idx - k * m;
    const double2 q = A[r * ns + phys_of[k]];
    qc[idx] = make_double2(q.x, -q.y);
  }
  if (tables == nullptr) return;
  const TableLayout tl(m, n);
  float* tc = tables + c * (int64_t)tl.total;
  const double nrm = qam_norm_d(L);
  const double sc = 2.0 / nrm;
  const double lv = (double)(L - 1) / nrm;
  double2* qt = reinterpret_cast<double2*>(tc + tl.off_qh);
  for (int idx = t; idx < n * m; idx += T) {
    const int r = idx / n, k = idx - r * n;   // transposed: qhT[r][k] = conj(q_k[r])
    const double2 q = A[r * ns + phys_of[k]];
    qt[idx] = make_double2(q.x, -q.y);
  }
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

#ifndef MPNL_PLAN_WARP_MAXN
#define MPNL_PLAN_WARP_MAXN 16   // channels with n <= this (and m (+n) <= 32) ...
#endif
#ifndef MPNL_PLAN_WARP_MINCH
#define MPNL_PLAN_WARP_MINCH 1024   // ... in batches of >= this many: warp kernel
#endif
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


// Small channels (ma <= 32, n <= 16): one WARP per channel, several channels per
// CTA and no block barriers.  A (physical columns, padded rows) and R (rows by
// physical column) live in the warp's slice of shared memory.  Lane j owns
// physical column j's bookkeeping (downdated norm, logical position) and, per
// step, that column's projection q^H a_j and update a_j -= q r_kj (sequential
// over the rows, four interleaved partial sums); the pivot is a warp argmax and
// r_kk a lane-per-row warp reduction — in the CTA kernel's arithmetic order,
// so the two give bit-identical plans.  Used for batches of many small
// channels (one H per vector: C1 pv 8,192 channels 123 -> 55 us); a few
// hundred channels (273 RBs) run faster as 4-warp CTAs, and 24 x 24 ones were
// measured slower in this layout (per-warp chains too long — DESIGN §8).
struct PlanWarpSmem {   // per warp, in double2 units
  int ns, r, total;
  __host__ __device__ PlanWarpSmem(int ma, int n) {
    ns = n + 1;
    r = ma * ns;
    total = r + n * n + 16;   // + 256 B for phys_of
  }
};

template <typename TIn>
__global__ void __launch_bounds__(128)
plan_qr_warp_kernel(const TIn* __restrict__ h, int64_t n_ch, int m, int n, int L,
                    double noise_var, int augmented, int32_t* __restrict__ perm_out,
                    double2* __restrict__ r_out, double2* __restrict__ qh_out,
                    float* __restrict__ tables) {
  extern __shared__ double2 smem[];
  const int ma = augmented ? m + n : m;
  const PlanWarpSmem so(ma, n);
  const int ns = so.ns;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (c >= n_ch) return;                       // warp-uniform: no block barriers below
  double2* A = smem + (int64_t)w * so.total;   // [ma][ns] physical columns
  double2* Rp = A + so.r;                      // [n][n] rows of R by physical column
  int* phys_of = reinterpret_cast<int*>(Rp + n * n);
  const TIn* hc = h + c * (int64_t)m * n;
  for (int idx = lane; idx < m * n; idx += 32) {
    const int r = idx / n, j = idx - r * n;
    A[r * ns + j] = load_c<TIn>(hc, idx);
  }
  if (augmented) {
    const double s = sqrt(noise_var);
    for (int idx = lane; idx < n * n; idx += 32) {
      const int i = idx / n, j = idx - i * n;
      A[(m + i) * ns + j] = make_double2(i == j ? s : 0.0, 0.0);
    }
  }
  for (int idx = lane; idx < n * n; idx += 32) Rp[idx] = make_double2(0.0, 0.0);
  __syncwarp();
  const bool own = lane < n;
  double norm = 0.0;
  if (own)
    for (int r = 0; r < ma; ++r) {
      const double2 a = A[r * ns + lane];
      norm = fma(a.x, a.x, fma(a.y, a.y, norm));
    }
  int logpos = lane;
  bool chosen = !own;
  int my_final = -1;
  for (int k = 0; k < n; ++k) {
    // pivot: max downdated norm, ties -> smallest logical position (first max)
    double bv = chosen ? -1.0 : norm;
    int bp = chosen ? 0x7fffffff : logpos;
    int bl = lane;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bl = ol; }
    }
    const int cp = bl;
    if (!chosen && logpos == k) logpos = bp;
    if (lane == cp) { logpos = k; chosen = true; my_final = k; }
    double part = 0.0;
    if (lane < ma) {
      const double2 a = A[lane * ns + cp];
      part = fma(a.x, a.x, a.y * a.y);
    }
    part = warp_sum_d(part);
    const double rkk = fmax(sqrt(part), 1e-300);
    if (lane < ma) {
      const double2 a = A[lane * ns + cp];
      A[lane * ns + cp] = make_double2(a.x / rkk, a.y / rkk);
    }
    if (lane == 0) Rp[k * n + cp] = make_double2(rkk, 0.0);
    __syncwarp();
    if (!chosen) {
      // q^H a_j in EXACTLY the CTA kernel's order (PLAN_WARPS row ranges, two
      // interleaved chains each, range partials summed in order), so both
      // kernels give bit-identical plans whichever one a batch size selects
      const int rb = (ma + PLAN_WARPS - 1) / PLAN_WARPS;
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int w4 = 0; w4 < PLAN_WARPS; ++w4) {
        const int r0 = w4 * rb, r1 = min(ma, r0 + rb);
        double pr = 0.0, pi = 0.0, pr2 = 0.0, pi2 = 0.0;
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
        sr += pr + pr2;
        si += pi + pi2;
      }
      Rp[k * n + lane] = make_double2(sr, si);
      for (int rr = 0; rr < ma; ++rr) {
        const double2 q = A[rr * ns + cp];
        double2 a = A[rr * ns + lane];
        a.x -= q.x * sr - q.y * si;
        a.y -= q.x * si + q.y * sr;
        A[rr * ns + lane] = a;
      }
      norm = fmax(norm - (sr * sr + si * si), 0.0);
    }
    __syncwarp();
  }
  if (own) phys_of[my_final] = lane;
  __syncwarp();
  plan_epilogue(A, ns, Rp, phys_of, c, m, n, L, perm_out, r_out, qh_out, tables, lane, 32);
}

template __global__ void plan_qr_kernel<float2>(const float2*, int64_t, int, int, int, double,
                                                int, int32_t*, double2*, double2*, float*);
template __global__ void plan_qr_kernel<double2>(const double2*, int64_t, int, int, int, double,
                                                 int, int32_t*, double2*, double2*, float*);

cudaError_t launch_plan(const void* h, int h_is_f64, int64_t n_ch, int m, int n, int L,
                        double noise_var, int augmented, int32_t* perm, double2* r64,
                        double2* qh64, float* tables, cudaStream_t st) {
  if (n_ch == 0) return cudaSuccess;
  const int ma = augmented ? m + n : m;
  if (ma <= 32 && n <= MPNL_PLAN_WARP_MAXN && n_ch >= MPNL_PLAN_WARP_MINCH) {
    // many small channels: warp per channel, 4 per CTA (bit-identical plans)
    const size_t smem = (size_t)4 * PlanWarpSmem(ma, n).total * sizeof(double2);
    const unsigned grid = (unsigned)((n_ch + 3) / 4);
    if (h_is_f64) {
      cudaFuncSetAttribute(plan_qr_warp_kernel<double2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      plan_qr_warp_kernel<double2><<<grid, 128, smem, st>>>(
          (const double2*)h, n_ch, m, n, L, noise_var, augmented, perm, r64, qh64, tables);
    } else {
      cudaFuncSetAttribute(plan_qr_warp_kernel<float2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      plan_qr_warp_kernel<float2><<<grid, 128, smem, st>>>(
          (const float2*)h, n_ch, m, n, L, noise_var, augmented, perm, r64, qh64, tables);
    }
    return cudaGetLastError();
  }
  size_t smem = (size_t)(ma * (n + 1) + n * n + PLAN_WARPS * 32) * sizeof(double2) +
                PLAN_WARPS * sizeof(double);
  if (h_is_f64) {
    cudaFuncSetAttribute(plan_qr_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    plan_qr_kernel<double2><<<(unsigned)n_ch, PLAN_THREADS, smem, st>>>(
        (const double2*)h, n_ch, m, n, L, noise_var, augmented, perm, r64, qh64, tables);
  } else {
    cudaFuncSetAttribute(plan_qr_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    plan_qr_kernel<float2><<<(unsigned)n_ch, PLAN_THREADS, smem, st>>>(
        (const float2*)h, n_ch, m, n, L, noise_var, augmented, perm, r64, qh64, tables);
  }
  return cudaGetLastError();
}

}  // namespace mpnl
