// fp32 list max-log LLRs fused with the path traversal (SURVEY §8f-1 sketch).
//
// Reference semantics: `mpnl_detect_batch` then `_candidate_llrs_batch`
// (pkg/src/mpnlsim/detect.py:473-488, 439-453; the link simulator's MPNL soft
// output, linksim.py:151-155): per stream n and bit j
//     llr = clip((min over paths with the bit set - min over paths with it clear) / nv)
// over the P candidate paths' metrics ||y - Hx||^2.  The common offset
// ||y||^2 - ||Q^H y||^2 cancels in the difference, so the fp32 PEDs of the
// traversal are all that is needed; no candidate list is materialised.
//
// Mapping: the prep kernel's outputs (z', guard thresholds, selection lists)
// are consumed as by the hard-output traversal.  A warp owns a vector and
// walks its paths in batches of 32 (lane = path, `traverse_paths` in its
// label-recording form).  After a batch every lane publishes its PED and its
// path's N log2(Q) label bits to the warp's shared memory, and the lanes
// switch roles: lane l then owns the (stream, bit) pairs l, l + 32, ... and
// folds the 32 paths into its two running minima per pair (broadcast reads,
// no cross-lane reductions).  The epilogue forms the fp64 LLRs in stream order.
//
// Exactness: the reference decides every layer in fp64.  A path with an fp32
// decision within the guard bound of a boundary (the traversal's `evm` mask)
// is settled right here: the warp re-decides its marked layers in fp64 from
// the path's own prefix (the check kernel's routines) and, where the
// reference takes the other branch, continues that branch in fp64 (exact SIC)
// and substitutes its labels and metric.  The candidate set is then the
// reference's, and metrics carry the fp32 PED error only: LLRs agree with
// the reference within 2 ped_tol / nv (about 1e-6 of the metrics / nv).
// Vectors whose partial-layer selection was a near-tie (EV_CUT events of the
// prep / select kernels) or whose event log overflowed are FLAGGED instead
// (flags[b] = 1): their LLRs must come from the fp64 list path
// (`mpnl_detect_full` + `mpnl_candidate_llrs`); the host shim does that.
#pragma once
#include "traverse.cuh"

namespace mpnl {

// warp_sic_f64 that also records the continued path's level indices (labw[q], q <= pos)
__device__ __forceinline__ double warp_sic_f64_lab(const DetectArgs& a, int64_t c, int n, int L,
                                                   int pos, int* labw, int ir0, int ii0,
                                                   double zr, double zi) {
  const int lane = threadIdx.x & 31;
  const double nrm = qam_norm_d(L);
  const double2* R = a.r64 + c * (int64_t)n * n;
  if (lane < n) {
    const int j0 = lane > pos ? lane : pos + 1;
#pragma unroll 4
    for (int j = j0; j < n; ++j) {
      const double sr = level_value_rt(labw[j] >> 3, L), si = level_value_rt(labw[j] & 7, L);
      const double2 r = R[lane * n + j];
      zr -= r.x * sr - r.y * si;
      zi -= r.x * si + r.y * sr;
    }
  } else {
    zr = 0.0;
    zi = 0.0;
  }
  double ped = (lane > pos && lane < n) ? zr * zr + zi * zi : 0.0;
  for (int q = pos; q >= 0; --q) {
    int ir = ir0, ii = ii0;
    if (q != pos) {
      const double rqq = R[q * n + q].x;
      const int lr = nearest_level_f64(zr / rqq, L, nrm), li = nearest_level_f64(zi / rqq, L, nrm);
      ir = __shfl_sync(0xffffffffu, lr, q);
      ii = __shfl_sync(0xffffffffu, li, q);
    }
    if (lane == 0) labw[q] = ir * 8 + ii;
    const double sr = level_value_rt(ir, L), si = level_value_rt(ii, L);
    if (lane <= q) {
      const double2 r = R[lane * n + q];
      zr -= r.x * sr - r.y * si;
      zi -= r.x * si + r.y * sr;
    }
    if (lane == q) ped += zr * zr + zi * zi;
  }
  __syncwarp();
  return warp_sum_d(ped);
}

struct SoftSmem {
  int tpo, tab, tab0, tabn, wbuf, wsz, total_bytes;   // floats / bytes
  int nwl;   // label-bit words per path
  __host__ __device__ SoftSmem(int m, int n, int bps, int warps) {
    TableLayout tl(m, n);
    int o = 0;
    tpo = o; o += TableLayout::up4((int)(sizeof(TreeParams) / 4));
    tab0 = tl.off_lay;
    tabn = tl.total - tl.off_lay;
    tab = o; o += tabn;
    nwl = (n * bps + 31) / 32;
    // per warp: 32 PEDs | 32 x nwl label-bit words | MPNL_MAX_N level indices (fp64 settling)
    wsz = TableLayout::up4(32 + 32 * nwl + MPNL_MAX_N);
    wbuf = o; o += warps * wsz;
    total_bytes = o * 4;
  }
};

template <int N, int L>
__global__ void __launch_bounds__(128)
soft_llr_kernel(const DetectArgs a, const TreeParams tparam) {
  const SoftArgs& sa = a.soft;
  constexpr int BPS = L == 2 ? 2 : (L == 4 ? 4 : 6);
  constexpr int H = BPS / 2;
  constexpr int NPP = (N + 1) / 2, N4 = (N + 3) & ~3;
  constexpr int NK = N * BPS;              // (layer, bit) pairs
  constexpr int NWL = (NK + 31) / 32;      // label-bit words per path = pairs per lane
  extern __shared__ __align__(16) float sm[];
  const SoftSmem so(a.m, N, BPS, (int)(blockDim.x >> 5));
  const TableLayout tl(a.m, N);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float INF = __int_as_float(0x7f800000);
  TreeParams& tp = *reinterpret_cast<TreeParams*>(sm + so.tpo);
  {
    const int* s = reinterpret_cast<const int*>(&tparam);
    int* d = reinterpret_cast<int*>(&tp);
    for (int i = tid; i < (int)(sizeof(TreeParams) / 4); i += blockDim.x) d[i] = s[i];
  }
  const int c = blockIdx.x / sa.chunks, chunk = blockIdx.x - c * sa.chunks;
  const float* tabg = a.tables + (int64_t)c * tl.total;   // the channel's blob (fp64 Q^H for settling)
  {
    const float4* src = reinterpret_cast<const float4*>(tabg + so.tab0);
    float4* dst = reinterpret_cast<float4*>(sm + so.tab);
    for (int i = tid; i < so.tabn / 4; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const TabPtrs T = tab_ptrs(sm + so.tab - so.tab0, a.m, N);
  float* pedw = sm + so.wbuf + warp * so.wsz;                     // [32]
  unsigned* bitw = reinterpret_cast<unsigned*>(pedw + 32);        // [32][NWL]
  int* labw = reinterpret_cast<int*>(bitw + 32 * NWL);            // [N]
  const int P = tp.n_paths, lbytes = tp.list_bytes;
  const int V = (int)a.V;
  const int v1 = min(V, (chunk + 1) * sa.vc);
  const int32_t* pc = a.perm + (int64_t)c * N;
  const double nrm = qam_norm_d(L);
  for (int v = chunk * sa.vc + warp; v < v1; v += (int)(blockDim.x >> 5)) {
    const int64_t gv = (int64_t)c * V + v;
    const float4* zs = a.zq + gv * NPP;
    const float* thr = a.thrg + gv * N4;
    const uint8_t* lch = a.lists + gv * lbytes;
    float mn1[NWL], mn0[NWL];   // running minima of pair 32 r + lane (bit set / clear)
#pragma unroll
    for (int r = 0; r < NWL; ++r) mn1[r] = mn0[r] = INF;
    bool zdone = false;
    double zr = 0.0, zi = 0.0;
    for (int p0 = 0; p0 < P; p0 += 32) {
      const int p = p0 + lane;
      const bool ok = p < P;
      const int vl[1] = {0}, pp[1] = {ok ? p : 0};
      const int64_t gvl[1] = {0};
      float ped[1], evp[1], pre[N];
      unsigned evm[1];
      int lab[N];
      traverse_paths<N, L, 1, true, true>(T, zs, thr, lch, tp, lbytes, vl, gvl, pp, ped, evm, evp,
                                          lab, pre, -1, nullptr);
      // ---- settle marked decisions in fp64 (rare): the reference's branch and metric ----
      unsigned mk = __ballot_sync(0xffffffffu, ok && evm[0] != 0u);
      while (mk) {
        const int l = __ffs(mk) - 1;
        mk &= mk - 1;
        __syncwarp();
        if (lane == l) {
#pragma unroll
          for (int pos = 0; pos < N; ++pos) labw[pos] = lab[pos];
        }
        __syncwarp();
        if (!zdone) { warp_z_f64(a, tabg, gv, N, zr, zi); zdone = true; }
        unsigned mask = __shfl_sync(0xffffffffu, evm[0], l);
        bool changed = false;
        double m64 = 0.0;
        while (mask) {
          const int pos = 31 - __clz(mask);
          mask &= ~(1u << pos);
          double cr, ci;
          warp_centre_f64(a, c, N, L, pos, labw, zr, zi, cr, ci);
          const int ir = nearest_level_f64(cr, L, nrm), ii = nearest_level_f64(ci, L, nrm);
          if (ir * 8 + ii != labw[pos]) {
            __syncwarp();
            m64 = warp_sic_f64_lab(a, c, N, L, pos, labw, ir, ii, zr, zi);
            changed = true;
            break;
          }
        }
        __syncwarp();
        if (changed && lane == l) {
#pragma unroll
          for (int pos = 0; pos < N; ++pos) lab[pos] = labw[pos];
          ped[0] = (float)m64;
        }
      }
      // ---- publish (PED, label bits): bit pos * BPS + j = bit j (MSB first) of the Gray label ----
      unsigned words[NWL];
#pragma unroll
      for (int r = 0; r < NWL; ++r) words[r] = 0u;
#pragma unroll
      for (int pos = 0; pos < N; ++pos) {
        const int ir = lab[pos] >> 3, ii = lab[pos] & 7;
        const unsigned lb = (unsigned)((gray_code(ir) << H) | gray_code(ii));
        const unsigned rv = __brev(lb) >> (32 - BPS);   // bit j of rv = label bit BPS - 1 - j
        const int bit = pos * BPS, w = bit >> 5, sh = bit & 31;
        words[w] |= rv << sh;
        if (sh + BPS > 32) words[w + 1] |= rv >> (32 - sh);
      }
      __syncwarp();
      pedw[lane] = ok ? ped[0] : INF;
#pragma unroll
      for (int r = 0; r < NWL; ++r) bitw[lane * NWL + r] = words[r];
      __syncwarp();
      // ---- lanes own (stream, bit) pairs: fold the batch's paths into the running minima ----
#pragma unroll 4
      for (int q = 0; q < 32; ++q) {
        const float m = pedw[q];
#pragma unroll
        for (int r = 0; r < NWL; ++r) {
          const bool bit = (bitw[q * NWL + r] >> lane) & 1u;
          mn1[r] = fminf(mn1[r], bit ? m : INF);
          mn0[r] = fminf(mn0[r], bit ? INF : m);
        }
      }
    }
    // ---- LLRs in stream order ----
    const double nv = sa.noise_var, clip = sa.clip;
#pragma unroll
    for (int r = 0; r < NWL; ++r) {
      const int kk = 32 * r + lane;
      if (kk < NK) {
        const int pos = kk / BPS, j = kk - pos * BPS;
        double x = __ddiv_rn(__dsub_rn((double)mn1[r], (double)mn0[r]), nv);
        if (x < -clip) x = -clip;   // np.clip (NaN stays NaN)
        if (x > clip) x = clip;
        sa.llr[(gv * N + pc[pos]) * BPS + j] = x;
      }
    }
    if (lane == 0) sa.flags[gv] = 0;   // (near-tie selections are flagged afterwards)
  }
}

}  // namespace mpnl
