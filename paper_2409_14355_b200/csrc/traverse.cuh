// K2+K3+K4 — fp32 parallel-path traversal with in-kernel argmin (hard output).
//
// Reference semantics (`/root/reference/pkg/src/mpnlsim/detect.py`):
//   z = Q^H y                                   detect.py:481
//   per layer pos = N-1..0: centre = (z_pos - acc_pos) / r_pp,
//   children = e_pos nearest points (stable)    detect.py:415-427
//   path index mixed radix, top layer most significant
//   metric = ||y - Hx||^2 (= PED for M = N)     detect.py:484-486
//   best = argmin (metric, labels[0], ...)      detect.py:465-470
//   hard = labels[best] in stream order         cli.py:239, detect.py:431-437
//
// B200 design (one CTA = one resource-block channel x a chunk of Vc vectors):
//   phase A  stage the channel's fp32 tables + the chunk's y in shared memory,
//            rotate z' = Q^H y - shift (fp32), per-chunk guard thresholds;
//   phase B  per (vector, parent) selection lists for *partial* expansion
//            layers (e < Q): e nearest of Q by a staircase rank over the
//            per-axis Schnorr-Euchner orders (only the SET matters for hard
//            output; the cut margin is guarded);
//   phase C  lane = path, PT paths per lane: every path is an independent
//            SIC chain.  Symbols are level indices held as exact small floats,
//            the interference of each decided symbol is pushed into the
//            per-row accumulators (4 FFMA per row, r'' broadcast from smem by
//            128-bit loads shared by PT paths), slicing is FMUL.SAT + a
//            magic-number round, the partial Euclidean distance accumulates
//            in registers.  Warp-shuffle argmin over paths on (metric, path);
//   phase D  one thread per vector re-traces its winning path with the very
//            same arithmetic (bit-identical), writes Gray labels in stream
//            order + the metric, and raises a flag when a guarded decision
//            on a competitive path or a near-tie could differ from fp64.
// Flagged vectors are recomputed by the fp64 kernel (exact.cu).
#pragma once
#include "common.cuh"

namespace mpnl {

struct TraverseArgs {
  const float* tables;      // per channel blob (TableLayout)
  const void* y;            // (n_ch, V, M) complex64 or complex128
  const int32_t* perm;      // (n_ch, N)
  uint8_t* hard;            // (n_ch, V, N) Gray labels, stream order
  float* metric;            // (n_ch, V)
  uint8_t* flags;           // (n_ch, V) or null
  int32_t* flag_count;      // device counter
  int64_t* flag_list;       // global vector indices needing fp64 recompute
  int64_t n_ch, V;
  int m;
  int y_f64;
  int vc;                   // vectors per CTA chunk
  int chunks;               // chunks per channel
  int vpi;                  // vectors per work item (VPI mode) or 1
  int bpv;                  // path batches per vector (batch mode) or 1
  int has_partial;          // any partial expansion layer (phase B needed)
  int metric_offset;        // 1 when M > N: add ||y||^2 - ||z||^2
  float tau;                // guard: relative fp32 error scale
};

#define MPNL_GROUP 8          // lanes per phase-B item
#define MPNL_GSCR 96          // floats of phase-B scratch per group
#define MPNL_MAGIC 8388608.0f // 2^23: fma(a, L-1, 2^23) rounds a to an integer

// shared-memory carve-up (offsets in floats; lists in bytes), host == device
struct TravSmem {
  int tab, y, z, thr, vb1, vb2, vfm, vbp, vcorr, misc, gscr, lists, total_bytes;
  __host__ __device__ TravSmem(int m, int n, int vc, int list_bytes, int ngroups) {
    TableLayout tl(m, n);
    int o = 0;
    tab = o; o += tl.total;
    y = o; o += TableLayout::up4(2 * vc * m);
    z = o; o += TableLayout::up4(2 * vc * n);
    thr = o; o += TableLayout::up4(n);
    vb1 = o; o += TableLayout::up4(vc);
    vb2 = o; o += TableLayout::up4(vc);
    vfm = o; o += TableLayout::up4(vc);
    vbp = o; o += TableLayout::up4(vc);
    vcorr = o; o += TableLayout::up4(vc);
    misc = o; o += 4;                        // [0] max ||y||, [1] E_acc max
    gscr = o; o += ngroups * MPNL_GSCR;
    lists = o * 4;
    total_bytes = lists + ((vc * list_bytes + 15) & ~15);
  }
};

struct Best {
  float b1, b2, fm;
  int bp;
};

__device__ __forceinline__ Best best_merge(Best a, Best b) {
  Best r;
  if (b.b1 < a.b1 || (b.b1 == a.b1 && b.bp < a.bp)) {
    r.b1 = b.b1; r.bp = b.bp; r.b2 = fminf(a.b1, b.b2);
  } else {
    r.b1 = a.b1; r.bp = a.bp; r.b2 = fminf(a.b2, b.b1);
  }
  r.fm = fminf(a.fm, b.fm);
  return r;
}

__device__ __forceinline__ Best best_shfl(Best a, int off) {
  Best o;
  o.b1 = __shfl_xor_sync(0xffffffffu, a.b1, off);
  o.b2 = __shfl_xor_sync(0xffffffffu, a.b2, off);
  o.fm = __shfl_xor_sync(0xffffffffu, a.fm, off);
  o.bp = __shfl_xor_sync(0xffffffffu, a.bp, off);
  return best_merge(a, o);
}

// Level indices of path p's symbol at an expanded layer pos.
template <int L>
__device__ __forceinline__ void expanded_symbol(const TreeParams& tp, int pos, int p,
                                                const uint8_t* vlist, int& ir, int& ii) {
  const int e = tp.e[pos];
  const int d = p / tp.stride[pos];
  if (e == L * L) {
    const int dd = d % e;          // full layer: any digit -> point bijection
    ir = dd / L;
    ii = dd - ir * L;
  } else {
    const uint8_t b = vlist[tp.list_off[pos] + d];
    ir = b >> 3;
    ii = b & 7;
  }
}

// One traversal of NS independent paths (tab = the channel's table blob in smem).
// GUARD: keep the PED prefix of any near-boundary decision in fped.
// LAB:   capture level indices (ir*8+ii) per position (NS must be 1).
template <int N, int L, int NS, bool GUARD, bool LAB>
__device__ __forceinline__ void traverse_paths(const float* __restrict__ tab,
                                               const float2* __restrict__ zs,
                                               const float* __restrict__ thr,
                                               const uint8_t* __restrict__ lists,
                                               const TreeParams& tp, int list_bytes,
                                               const int (&vl)[NS], const int (&p)[NS],
                                               float (&ped)[NS], float (&fped)[NS],
                                               int (&lab)[N], int m) {
  constexpr int NP = (N + 1) & ~1;
  const TableLayout tl(m, N);
  const float4* lay4 = reinterpret_cast<const float4*>(tab + tl.off_lay);
  const float* rcol = tab + tl.off_rcol;
  float ar[NS][N], ai[NS][N];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const float2 z = zs[vl[s] * N + k];
      ar[s][k] = z.x;
      ai[s][k] = z.y;
    }
    ped[s] = 0.f;
    fped[s] = __int_as_float(0x7f800000);
  }
  const int top_lo = N - tp.n_top;   // layers pos >= top_lo are expanded
#pragma unroll
  for (int pos = N - 1; pos >= 0; --pos) {
    const float4 ly = lay4[pos];
    const float kneg = ly.x, c2r = ly.y;
    float fr[NS], fi[NS];
    if (pos >= top_lo) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        int ir, ii;
        expanded_symbol<L>(tp, pos, p[s], lists + vl[s] * list_bytes, ir, ii);
        fr[s] = (float)ir;
        fi[s] = (float)ii;
        if (LAB) lab[pos] = ir * 8 + ii;
      }
    } else {
      float th = 0.f;
      if (GUARD) th = thr[pos];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const float sr = __saturatef(__fmul_rn(ar[s][pos], kneg));
        const float si = __saturatef(__fmul_rn(ai[s][pos], kneg));
        const float mr = __fmaf_rn(sr, (float)(L - 1), MPNL_MAGIC);
        const float mi = __fmaf_rn(si, (float)(L - 1), MPNL_MAGIC);
        fr[s] = __fsub_rn(mr, MPNL_MAGIC);
        fi[s] = __fsub_rn(mi, MPNL_MAGIC);
        if (GUARD) {
          const float tr = __fmaf_rn(sr, (float)(L - 1), -fr[s]);
          const float ti = __fmaf_rn(si, (float)(L - 1), -fi[s]);
          if (fabsf(tr) > th || fabsf(ti) > th) fped[s] = fminf(fped[s], ped[s]);
        }
        if (LAB) lab[pos] = (int)fr[s] * 8 + (int)fi[s];
      }
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float er = __fmaf_rn(c2r, fr[s], ar[s][pos]);
      const float ei = __fmaf_rn(c2r, fi[s], ai[s][pos]);
      ped[s] = __fmaf_rn(er, er, ped[s]);
      ped[s] = __fmaf_rn(ei, ei, ped[s]);
    }
    // push this layer's symbols into the rows below: acc_k += r''_k,pos * s
    const float4* rc = reinterpret_cast<const float4*>(rcol + 2 * NP * pos);
#pragma unroll
    for (int k = 0; k < pos; k += 2) {
      const float4 r2 = rc[k >> 1];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        ar[s][k] = __fmaf_rn(r2.x, fr[s], ar[s][k]);
        ar[s][k] = __fmaf_rn(-r2.y, fi[s], ar[s][k]);
        ai[s][k] = __fmaf_rn(r2.x, fi[s], ai[s][k]);
        ai[s][k] = __fmaf_rn(r2.y, fr[s], ai[s][k]);
        if (k + 1 < pos) {
          ar[s][k + 1] = __fmaf_rn(r2.z, fr[s], ar[s][k + 1]);
          ar[s][k + 1] = __fmaf_rn(-r2.w, fi[s], ar[s][k + 1]);
          ai[s][k + 1] = __fmaf_rn(r2.z, fi[s], ai[s][k + 1]);
          ai[s][k + 1] = __fmaf_rn(r2.w, fr[s], ai[s][k + 1]);
        }
      }
    }
  }
}

template <int N>
struct TravCfg {
  static constexpr int PT = N <= 8 ? 4 : 2;              // paths per lane
  static constexpr int MAXT = N <= 16 ? 256 : 128;       // threads per CTA
  static constexpr int MINB = 2;                         // CTAs per SM
};

template <int N, int L>
__global__ void __launch_bounds__(TravCfg<N>::MAXT, TravCfg<N>::MINB)
traverse_kernel(const TraverseArgs a, const TreeParams tp) {
  constexpr int PT = TravCfg<N>::PT;
  constexpr int S = 32 * PT;
  extern __shared__ __align__(16) float sm[];
  const int ngroups = blockDim.x / MPNL_GROUP;
  const TravSmem so(a.m, N, a.vc, tp.list_bytes, ngroups);
  const TableLayout tl(a.m, N);
  const int m = a.m;
  const int64_t c = blockIdx.x / a.chunks;
  const int v0 = (blockIdx.x % a.chunks) * a.vc;
  const int vce = (int)min((int64_t)a.vc, a.V - v0);
  const int tid = threadIdx.x, nth = blockDim.x;
  const int P = tp.n_paths;

  float* tab = sm + so.tab;
  float2* ys = reinterpret_cast<float2*>(sm + so.y);
  float2* zs = reinterpret_cast<float2*>(sm + so.z);
  float* thr = sm + so.thr;
  float* vb1 = sm + so.vb1;
  float* vb2 = sm + so.vb2;
  float* vfm = sm + so.vfm;
  int* vbp = reinterpret_cast<int*>(sm + so.vbp);
  float* vcorr = sm + so.vcorr;
  float* misc = sm + so.misc;
  uint8_t* lists = reinterpret_cast<uint8_t*>(sm) + so.lists;

  // ---------------- phase A: stage + rotate ----------------
  {
    const float4* src = reinterpret_cast<const float4*>(a.tables + c * (int64_t)tl.total);
    float4* dst = reinterpret_cast<float4*>(tab);
    for (int i = tid; i < tl.total / 4; i += nth) dst[i] = src[i];
    const int64_t ybase = (c * a.V + v0) * (int64_t)m;
    if (a.y_f64) {
      const double2* yd = reinterpret_cast<const double2*>(a.y) + ybase;
      for (int i = tid; i < vce * m; i += nth) {
        const double2 v = yd[i];
        ys[i] = make_float2((float)v.x, (float)v.y);
      }
    } else {
      const float2* yf = reinterpret_cast<const float2*>(a.y) + ybase;
      for (int i = tid; i < vce * m; i += nth) ys[i] = yf[i];
    }
    for (int i = tid; i < a.vc; i += nth) {
      vfm[i] = __int_as_float(0x7f800000);
      vcorr[i] = 0.f;
    }
    if (tid == 0) { misc[0] = 0.f; misc[1] = 0.f; }
  }
  __syncthreads();
  {
    const float2* qh = reinterpret_cast<const float2*>(tab + tl.off_qh);
    const float2* sh = reinterpret_cast<const float2*>(tab + tl.off_shift);
    for (int i = tid; i < vce * N; i += nth) {
      const int v = i / N, k = i - v * N;
      float zr = 0.f, zi = 0.f;
      for (int r = 0; r < m; ++r) {
        const float2 q = qh[k * m + r], yv = ys[v * m + r];
        zr = __fmaf_rn(q.x, yv.x, zr);
        zr = __fmaf_rn(-q.y, yv.y, zr);
        zi = __fmaf_rn(q.x, yv.y, zi);
        zi = __fmaf_rn(q.y, yv.x, zi);
      }
      zs[i] = make_float2(__fsub_rn(zr, sh[k].x), __fsub_rn(zi, sh[k].y));
    }
    for (int v = tid; v < vce; v += nth) {
      float yn = 0.f;
      for (int r = 0; r < m; ++r) {
        const float2 yv = ys[v * m + r];
        yn = __fmaf_rn(yv.x, yv.x, __fmaf_rn(yv.y, yv.y, yn));
      }
      if (a.metric_offset) vcorr[v] = yn;
      atomicMax(reinterpret_cast<int*>(misc), __float_as_int(sqrtf(yn)));
    }
  }
  __syncthreads();
  {
    const float4* lay4 = reinterpret_cast<const float4*>(tab + tl.off_lay);
    const float ymax = misc[0];
    float eacc = 0.f;
    for (int k = tid; k < N; k += nth) {
      const float4 ly = lay4[k];
      const float ek = a.tau * (ymax + ly.z);          // acc-domain error bound
      thr[k] = 0.5f - ek / ly.y;                        // index-domain threshold
      eacc = fmaxf(eacc, ek);
    }
    if (tid < N) atomicMax(reinterpret_cast<int*>(misc + 1), __float_as_int(eacc));
    if (a.metric_offset) {
      const float2* sh = reinterpret_cast<const float2*>(tab + tl.off_shift);
      for (int v = tid; v < vce; v += nth) {
        float zn = 0.f;
        for (int k = 0; k < N; ++k) {
          const float2 z = zs[v * N + k];
          const float zr = z.x + sh[k].x, zi = z.y + sh[k].y;
          zn = __fmaf_rn(zr, zr, __fmaf_rn(zi, zi, zn));
        }
        vcorr[v] = vcorr[v] - zn;
      }
    }
  }
  __syncthreads();

  // ---------------- phase B: partial-layer selection lists ----------------
  if (a.has_partial) {
    constexpr int NP = (N + 1) & ~1;
    const float* rcol = tab + tl.off_rcol;
    const float4* lay4 = reinterpret_cast<const float4*>(tab + tl.off_lay);
    const int gid = tid / MPNL_GROUP, gl = tid % MPNL_GROUP;
    float* gs = sm + so.gscr + gid * MPNL_GSCR;   // dx[8] dy[8] key[64] ox/oy(4) de de1
    float* gdx = gs;
    float* gdy = gs + 8;
    float* gkey = gs + 16;
    uint8_t* gox = reinterpret_cast<uint8_t*>(gs + 80);
    uint8_t* goy = gox + 8;
    const int top_lo = N - tp.n_top;
    for (int pos = N - 1; pos >= top_lo; --pos) {
      const int e = tp.e[pos];
      if (e == L * L) continue;
      const int npar = P / tp.stride[pos + 1];
      const int K = tp.stair_cnt[pos];
      const int items = vce * npar;
      const float4 lyp = lay4[pos];
      for (int it0 = 0; it0 < items; it0 += ngroups) {
        const int it = it0 + gid;
        const bool act = it < items;
        const int vl = act ? it / npar : 0;
        const int par = act ? it - vl * npar : 0;
        const int p0 = par * tp.stride[pos + 1];
        const uint8_t* vlist = lists + vl * tp.list_bytes;
        // prefix: acc at every prefix layer (phase-C order), PED prefix, acc at pos
        float pedp = 0.f, xr = 0.f, xi = 0.f;
        for (int j = N - 1; j >= pos; --j) {
          const float2 zj = zs[vl * N + j];
          float ar_ = zj.x, ai_ = zj.y;
          for (int l = N - 1; l > j; --l) {
            int ir, ii;
            expanded_symbol<L>(tp, l, p0, vlist, ir, ii);
            const float fr = (float)ir, fi = (float)ii;
            const float2 r2 = reinterpret_cast<const float2*>(rcol + 2 * NP * l)[j];
            ar_ = __fmaf_rn(r2.x, fr, ar_);
            ar_ = __fmaf_rn(-r2.y, fi, ar_);
            ai_ = __fmaf_rn(r2.x, fi, ai_);
            ai_ = __fmaf_rn(r2.y, fr, ai_);
          }
          if (j > pos) {
            int ir, ii;
            expanded_symbol<L>(tp, j, p0, vlist, ir, ii);
            const float c2r = lay4[j].y;
            const float er = __fmaf_rn(c2r, (float)ir, ar_);
            const float ei = __fmaf_rn(c2r, (float)ii, ai_);
            pedp = __fmaf_rn(er, er, pedp);
            pedp = __fmaf_rn(ei, ei, pedp);
          } else {
            xr = ar_; xi = ai_;
          }
        }
        // centre in level-index units (unclamped)
        const float cx = __fmul_rn(__fmul_rn(xr, lyp.x), (float)(L - 1));
        const float cy = __fmul_rn(__fmul_rn(xi, lyp.x), (float)(L - 1));
        if (gl == 0 && act) {
          // per-axis Schnorr-Euchner (closest-first) level orders
#pragma unroll
          for (int ax = 0; ax < 2; ++ax) {
            const float x = ax ? cy : cx;
            float* dd = ax ? gdy : gdx;
            uint8_t* oo = ax ? goy : gox;
            const int n0 = (int)rintf(fminf(fmaxf(x, 0.f), (float)(L - 1)));
            int lo = n0 - 1, hi = n0 + 1;
            oo[0] = (uint8_t)n0;
            dd[0] = (x - n0) * (x - n0);
#pragma unroll
            for (int r = 1; r < L; ++r) {
              const bool th = (hi < L) && (lo < 0 || (hi - x) < (x - lo));
              const int lev = th ? hi : lo;
              if (th) ++hi; else --lo;
              oo[r] = (uint8_t)lev;
              dd[r] = (x - lev) * (x - lev);
            }
          }
        }
        __syncwarp();
        // staircase(e+1) candidates (i, j) with (i+1)(j+1) <= e+1
        for (int cc = gl; cc < K; cc += MPNL_GROUP) {
          int i = 0, rem = cc;
          while (true) {
            const int w = min(L, (e + 1) / (i + 1));
            if (rem < w) break;
            rem -= w;
            ++i;
          }
          if (act) gkey[cc] = gdx[i] + gdy[rem];
        }
        __syncwarp();
        for (int cc = gl; cc < K; cc += MPNL_GROUP) {
          int i = 0, rem = cc;
          while (true) {
            const int w = min(L, (e + 1) / (i + 1));
            if (rem < w) break;
            rem -= w;
            ++i;
          }
          if (!act) continue;
          const float key = gkey[cc];
          int rank = 0;
          for (int c2 = 0; c2 < K; ++c2) {
            const float k2 = gkey[c2];
            rank += (k2 < key) || (k2 == key && c2 < cc);
          }
          if (rank < e) lists[vl * tp.list_bytes + tp.list_off[pos] + par * e + rank] =
                            (uint8_t)((gox[i] << 3) | goy[rem]);
          if (rank == e - 1) gs[84] = key;
          if (rank == e) gs[85] = key;
        }
        __syncwarp();
        if (gl == 0 && act) {
          const float E = fmaxf(0.5f - thr[pos], 0.f);
          const float de = gs[84], de1 = gs[85];
          const float bound = 2.8284272f * E * (sqrtf(de) + sqrtf(de1)) + 4.f * E * E +
                              4.8e-7f * de1;
          if (de1 - de <= bound)
            atomicMin(reinterpret_cast<int*>(vfm + vl), __float_as_int(pedp));
        }
        __syncwarp();
      }
      __syncthreads();
    }
  }

  // ---------------- phase C: path traversal + warp argmin ----------------
  {
    const int warp = tid >> 5, lane = tid & 31, nw = nth >> 5;
    const int items = (a.bpv > 1 || a.vpi == 1) ? (a.bpv > 1 ? vce : (vce + a.vpi - 1) / a.vpi)
                                                : (vce + a.vpi - 1) / a.vpi;
    int dummy_lab[N];
    for (int item = warp; item < items; item += nw) {
      Best run = {__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                  __int_as_float(0x7f800000), 0x7fffffff};
      for (int b = 0; b < a.bpv; ++b) {
        int vl[PT], pp[PT];
        bool ok[PT];
#pragma unroll
        for (int t = 0; t < PT; ++t) {
          const int s = t * 32 + lane;
          if (a.bpv > 1 || a.vpi == 1) {
            vl[t] = item;
            pp[t] = b * S + s;
            ok[t] = pp[t] < P;
          } else {
            vl[t] = item * a.vpi + s / P;
            pp[t] = s % P;
            ok[t] = vl[t] < vce;
          }
          if (!ok[t]) { vl[t] = 0; pp[t] = 0; }
        }
        float ped[PT], fped[PT];
        traverse_paths<N, L, PT, true, false>(tab, zs, thr, lists, tp, tp.list_bytes, vl, pp,
                                              ped, fped, dummy_lab, m);
        if (a.bpv > 1 || a.vpi == 1) {
#pragma unroll
          for (int t = 0; t < PT; ++t) {
            Best x = {ok[t] ? ped[t] : __int_as_float(0x7f800000), __int_as_float(0x7f800000),
                      ok[t] ? fped[t] : __int_as_float(0x7f800000), ok[t] ? pp[t] : 0x7fffffff};
            run = best_merge(run, x);
          }
        } else if (P >= 32) {
          const int g = P >> 5;   // t-slots per vector
#pragma unroll
          for (int t0 = 0; t0 < PT; ++t0) {
            if (t0 % g) continue;
            Best x = {__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                      __int_as_float(0x7f800000), 0x7fffffff};
#pragma unroll
            for (int t = 0; t < PT; ++t)
              if (t >= t0 && t < t0 + g) {
                Best y = {ok[t] ? ped[t] : __int_as_float(0x7f800000),
                          __int_as_float(0x7f800000),
                          ok[t] ? fped[t] : __int_as_float(0x7f800000), pp[t]};
                x = best_merge(x, y);
              }
#pragma unroll
            for (int o = 16; o; o >>= 1) x = best_shfl(x, o);
            const int v = item * a.vpi + t0 / g;
            if (lane == 0 && v < vce) {
              vb1[v] = x.b1; vb2[v] = x.b2; vbp[v] = x.bp; vfm[v] = fminf(vfm[v], x.fm);
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < PT; ++t) {
            Best x = {ok[t] ? ped[t] : __int_as_float(0x7f800000), __int_as_float(0x7f800000),
                      ok[t] ? fped[t] : __int_as_float(0x7f800000), pp[t]};
            for (int o = P >> 1; o; o >>= 1) x = best_shfl(x, o);
            const int v = item * a.vpi + (t * 32 + lane) / P;
            if ((lane % P) == 0 && v < vce) {
              vb1[v] = x.b1; vb2[v] = x.b2; vbp[v] = x.bp; vfm[v] = fminf(vfm[v], x.fm);
            }
          }
        }
      }
      if (a.bpv > 1 || a.vpi == 1) {
#pragma unroll
        for (int o = 16; o; o >>= 1) run = best_shfl(run, o);
        if (lane == 0) {
          vb1[item] = run.b1; vb2[item] = run.b2; vbp[item] = run.bp;
          vfm[item] = fminf(vfm[item], run.fm);
        }
      }
    }
  }
  __syncthreads();

  // ---------------- phase D: re-trace winners, labels, guard verdict ----------------
  {
    const int h = (L == 2) ? 1 : (L == 4 ? 2 : 3);
    const float eacc = misc[1];
    const int32_t* pc = a.perm + c * N;
    for (int v = tid; v < vce; v += nth) {
      int vl[1] = {v}, pp[1] = {vbp[v]};
      float ped[1], fped[1];
      int lab[N];
      traverse_paths<N, L, 1, false, true>(tab, zs, thr, lists, tp, tp.list_bytes, vl, pp, ped,
                                           fped, lab, m);
      const int64_t gv = c * a.V + v0 + v;
      uint8_t* out = a.hard + gv * N;
#pragma unroll
      for (int pos = 0; pos < N; ++pos) {
        const int ir = lab[pos] >> 3, ii = lab[pos] & 7;
        out[pc[pos]] = (uint8_t)((gray_code(ir) << h) | gray_code(ii));
      }
      const float b1 = vb1[v], b2 = vb2[v], fm = vfm[v];
      a.metric[gv] = b1 + vcorr[v];
      const float tolm = 4.f * sqrtf((float)N * b1) * eacc + 2.f * N * eacc * eacc + 2e-6f * b1;
      const bool flag = (b2 - b1 <= 2e-5f * b1 + tolm) || (fm <= b1 + tolm);
      if (a.flags) a.flags[gv] = flag ? 1 : 0;
      if (flag) {
        const int slot = atomicAdd(a.flag_count, 1);
        a.flag_list[slot] = gv;
      }
    }
  }
}

}  // namespace mpnl
