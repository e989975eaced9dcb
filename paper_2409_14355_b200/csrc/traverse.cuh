// K2 + K3 + K4 — the fp32 hard-output fast path, as three uniform kernels.
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
// select_kernel   (K2, only for partial layers 1 < e < Q) one thread per
//                 (vector, parent): the e nearest points by a k-smallest-sum
//                 merge of the two per-axis Schnorr-Euchner orders (only the SET
//                 matters for hard output); a cut closer than the fp32 error
//                 bound is logged as an event.
// traverse_kernel (K3, the hot kernel) CTA = a channel's chunk of vectors; the
//                 channel's tables are staged in shared memory once, then every
//                 warp loops over its vectors with no block barrier: rotate
//                 z' = Q^H y - shift (lane = row), per-vector per-layer fp32
//                 error bounds, then lane = path (PT paths per lane): each path
//                 is an independent SIC chain; symbols are level indices held as
//                 exact small floats, each decided symbol is pushed into the
//                 per-row accumulators (4 FFMA per row; one 128-bit LDS of r''
//                 serves 2 rows x PT paths), slicing = FMUL.SAT + magic-number
//                 round, the PED accumulates in registers.  A decision closer to
//                 a boundary than the bound sets a bit in a per-path mask
//                 (branch-free); paths with a competitive marked decision are
//                 logged.  Top-3 (metric, path) per vector with warp REDUX.
// verify_kernel   (K4) thread per vector: re-trace the winner with the very same
//                 arithmetic (bit-identical), write Gray labels in stream order;
//                 settle a 2-way near-tie in fp64.  Thread per logged event:
//                 re-decide the marked decisions of competitive paths in fp64
//                 from the path's own prefix.  Disagreements, 3-way ties and
//                 overflows go to the fp64 kernel (exact.cu).
#pragma once
#include "common.cuh"
#include "fp64dec.cuh"

namespace mpnl {

// Soft-output (fp32 list max-log LLR) kernel arguments (soft.cuh)
struct SoftArgs {
  double* llr;        // (B, N, bps) fp64, stream order
  uint8_t* flags;     // (B,) 1 = recompute in fp64
  double noise_var;
  double clip;
  int vc;             // vectors per CTA
  int chunks;         // CTAs per channel
};

struct DetectArgs {
  const float* tables;      // (n_ch, T) per channel blob (TableLayout)
  const void* y;            // (n_ch, V, M) complex64 or complex128
  const int32_t* perm;      // (n_ch, N)
  const double2* r64;       // (n_ch, N, N)
  const double2* qh64;      // (n_ch, N, M)
  uint8_t* hard;            // (B, N) Gray labels, stream order
  float* metric;            // (B,)
  // workspace
  int32_t* counters;        // [0] fix-up count, [1] event count
  int64_t* fix_list;        // (B,) vectors for the fp64 kernel
  uint32_t* vflag;          // (B,) 1 = sent to fp64
  float4* vres;             // (B,) b1, b2, b3, E_acc (L2)
  int2* vpath;              // (B,) p1, p2
  int4* events;             // (ev_cap,) {path, mask|pos, vector, type}
  uint8_t* lists;           // (B, list_bytes) partial-layer selections
  float4* zq;               // (B, NPP) z' row pairs (prep kernel)
  float* thrg;              // (B, N) per-layer index-domain guard thresholds (prep kernel)
  float2* vaux;             // (B,) E_acc (L2 over layers), metric offset ||y||^2-||z||^2
  int32_t* stats;           // diagnostics (may be null)
  int64_t n_ch, V;
  int m;
  int y_f64;
  int ev_cap;
  int vpi, bpv;             // vectors per warp item (VPI mode) / path batches per vector
  int metric_offset;        // 1 when M > N: add ||y||^2 - ||z||^2
  float guard_scale;        // scales the fp32 error bound (1 = rigorous)
  int wpc;                  // traversal: 1 = a warp per channel (few vectors per channel)
  SoftArgs soft;            // soft_llr_kernel only
};

#define MPNL_XMAX 3             // expanded (e > 1) layers handled by the fast path
#define MPNL_VPI_MAX 8          // vectors per warp item in VPI mode
#define MPNL_MAGIC 12582912.0f  // 1.5 * 2^23: fma(acc, kx, MAGIC) rounds x to an integer
#define MPNL_U 5.9604645e-08f   // 2^-24
#define EV_NODE 0   // (a NODE event's .w carries -evp: negative, see ev_node_w)
#define EV_CUT 1
#define TRAV_EV_CAP 512         // per-CTA event buffer of the traversal kernel
#define MPNL_XS_STRIDE 128      // = traversal threads per CTA (per-thread symbol slots)

// ---------------------------------------------------------------------------
// arithmetic shared by all kernels: keeping it in one place makes the
// re-traces bit-identical to the traversal.
// ---------------------------------------------------------------------------

template <int L>
__device__ __forceinline__ void expanded_symbol(const TreeParams& tp, int pos, int p,
                                                const uint8_t* vlist, int& ir, int& ii) {
  const unsigned e = (unsigned)tp.e[pos];
  const unsigned d = fast_div((unsigned)p, (unsigned)tp.stride[pos], tp.ms[pos]);
  if (e == (unsigned)(L * L)) {
    const unsigned dd = d - fast_div(d, e, tp.me[pos]) * e;   // full layer: digit -> point
    ir = (int)(dd / L);
    ii = (int)(dd % L);
  } else {
    const uint8_t b = vlist[tp.list_off[pos] + d];
    ir = b >> 3;
    ii = b & 7;
  }
}

// slice one axis (kxs = -1/(c2r (L-1)), the saturated scale): s = sat(acc kxs)
// in [0, 1], so n = round(s (L-1)) (1.5 * 2^23 magic number, exact) is the
// nearest level index already clamped to [0, L-1], t = s (L-1) - n.  Returns
// -n (the traversal carries negated level indices: a decision is then one
// FMUL.SAT per axis + FFMA2 + FADD2, with no min/max clamping).  The packed
// twin in traverse_paths performs the very same per-element operations, so
// both are bit-identical.
template <int L>
__device__ __forceinline__ float slice_axis(float acc, float kxs, float& t) {
  const float s = __saturatef(__fmul_rn(acc, kxs));
  const float mm = __fmaf_rn(s, (float)(L - 1), MPNL_MAGIC);
  const float nf = __fsub_rn(MPNL_MAGIC, mm);   // -n
  t = __fmaf_rn(s, (float)(L - 1), nf);
  return nf;
}

__device__ __forceinline__ float ped_step(float ped, float c2r, float fr, float fi, float ur,
                                          float ui) {
  const float er = __fmaf_rn(c2r, fr, ur);
  const float ei = __fmaf_rn(c2r, fi, ui);
  ped = __fmaf_rn(er, er, ped);
  return __fmaf_rn(ei, ei, ped);
}

// scalar twin of the packed row-pair update in traverse_paths (same fmas, same order)
__device__ __forceinline__ void acc_step(float& ar, float& ai, float rr, float ri, float fr,
                                         float fi) {
  ar = __fmaf_rn(rr, fr, ar);
  ar = __fmaf_rn(ri, -fi, ar);
  ai = __fmaf_rn(rr, fi, ai);
  ai = __fmaf_rn(ri, fr, ai);
}

// ---- packed f32x2 (Blackwell FFMA2: two IEEE fmas per lane per instruction) ----
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo32(u64 v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi32(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 fsub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ---- cp.async (LDGSTS): global -> shared without staging registers ----
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }
// r''(row k, column pos) from the row-pair table
__device__ __forceinline__ float2 rcol_at(const float* rcol, int npp, int k, int pos) {
  const float* b = rcol + 4 * (pos * npp + (k >> 1)) + 2 * (k & 1);
  return make_float2(b[0], b[1]);
}

__device__ __forceinline__ float2 load_y32(const DetectArgs& a, int64_t idx) {
  if (a.y_f64) {
    const double2 v = reinterpret_cast<const double2*>(a.y)[idx];
    return make_float2((float)v.x, (float)v.y);
  }
  return reinterpret_cast<const float2*>(a.y)[idx];
}

// z'_k = fl32((Q^H y)_k - shift_k): rotation in fp64, one rounding at the end
// (identical sequence everywhere).  yat(r) returns y_r as float2.
template <typename YF>
__device__ __forceinline__ float2 rotate_row(const float* tab, int m, int n, int k, YF yat) {
  const TableLayout tl(m, n);
  const double2* qt = reinterpret_cast<const double2*>(tab + tl.off_qh);
  double zr = 0.0, zi = 0.0;
  for (int r = 0; r < m; ++r) {
    const double2 q = qt[r * n + k];
    const float2 yv = yat(r);
    const double yr = yv.x, yi = yv.y;
    zr = fma(q.x, yr, zr);
    zr = fma(-q.y, yi, zr);
    zi = fma(q.x, yi, zi);
    zi = fma(q.y, yr, zi);
  }
  const double2 sh = reinterpret_cast<const double2*>(tab + tl.off_shift)[k];
  return make_float2((float)(zr - sh.x), (float)(zi - sh.y));
}

// acc-domain fp32 error bound of row k's decision variable:
//   u [ c_y sqrt2 |y| + (2(N-1-k)+2) (|z'_k| + (L-1) S_k) ] + 1e-12 |y|
// (c_y = 1 when y arrived in fp64 and was rounded to fp32; the fp64 rotation
//  itself contributes ~1e-16 |y|)
__device__ __forceinline__ float row_bound(float ynorm, float2 zk, float4 lyk, int k, int m, int n,
                                           int L, float gs, int y_f64) {
  (void)m;
  const float za = fmaxf(fabsf(zk.x), fabsf(zk.y));
  const float xk = za + (float)(L - 1) * lyk.z;
  return gs * (MPNL_U * 1.01f * ((y_f64 ? 1.4142136f * ynorm : 0.f) +
                                 (2.f * (n - 1 - k) + 2.f) * xk) +
               1e-12f * ynorm);
}

// fp32 PED error bound from the L2 norm of the per-layer acc bounds
// (sqrt.approx: <= 2 ulp below the true root; the 1 + 2^-19 factor makes it an
// upper bound, and every kernel evaluates the identical instruction sequence)
__device__ __forceinline__ float sqrt_up(float b) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
  return __fmul_ru(r, 1.0000020f);
}
__device__ __forceinline__ float ped_tol(float b, float eacc, int n) {
  return __fadd_ru(__fadd_ru(__fmul_ru(__fmul_ru(2.f, sqrt_up(b)), eacc), __fmul_ru(eacc, eacc)),
                   __fmul_ru(2.f * n * MPNL_U, b));
}

// a vector's final event bound: a marked decision whose PED prefix exceeds it cannot
// affect the result.  One explicit instruction sequence, because the traversal's
// flush and the check kernel must agree on it exactly.
__device__ __forceinline__ float node_lim(float4 res, int n) {
  return __fmaf_rn(2.f, ped_tol(res.x, res.w, n), res.x);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct TabPtrs {
  const float4* lay4;
  const float* rcol;   // 16-byte aligned columns of NPP float4 row pairs
};

__device__ __forceinline__ TabPtrs tab_ptrs(const float* tab, int m, int n) {
  const TableLayout tl(m, n);
  TabPtrs t;
  t.lay4 = reinterpret_cast<const float4*>(tab + tl.off_lay);
  t.rcol = reinterpret_cast<const float*>(__builtin_assume_aligned(tab + tl.off_rcol, 16));
  return t;
}

// guard bookkeeping as two predicated instructions (no branch, no selects):
// if (d > th) { evm |= bit; evp = min(evp, pre); }
__device__ __forceinline__ void guard_mark(float d, float th, unsigned bit, float pre,
                                           unsigned& evm, float& evp) {
  asm("{\n\t.reg .pred p;\n\tsetp.gt.f32 p, %2, %3;\n\t@p or.b32 %0, %0, %4;\n\t"
      "@p min.f32 %1, %1, %5;\n\t}"
      : "+r"(evm), "+f"(evp)
      : "f"(d), "f"(th), "r"(bit), "f"(pre));
}

// K3 inner loop: NS independent paths.  Per path: PED, mask of layers whose
// decision was within the bound, and a lower bound of the PED prefix at the
// first such layer (Ped<>::bound: the prefix itself, or its real half in the packed
// mode; taken with a predicated min).
// Accumulators are per row (re, im) f32x2 registers; decided symbols are held
// as NEGATED level indices g = -n (what the magic-number rounding yields for
// free), so every product with g uses a negated table operand -- exact, hence
// bit-identical to the positive-form scalar twins (acc_step, warp_retrace).
// The update of row k is
//   acc_k = FFMA2(-rr_k (bcast), g, acc_k);  acc_k = FFMA2((-gi, gr), -ri_k (bcast), acc_k)
// i.e. per element exactly acc_step's fma sequence, with no register moves
// (swap, partial and broadcast negations are free FFMA2 operand modifiers).
// One 128-bit LDS of r'' ({rr_2q, ri_2q, rr_2q+1, ri_2q+1}) feeds 4 FFMA2 per path.
// zs: per vector NPP float4 {re_2q, im_2q, re_2q+1, im_2q+1}.
// LAB (NS == 1): record level indices lab[pos] and PED prefix pre[pos] and
// stop after layer `stop` (phase re-traces).
// SH (NS == 2): the lane's two paths are siblings under the top layer (same
// top symbol): the top layer's PED term and row updates are computed once.
#ifndef MPNL_QDESC
#define MPNL_QDESC 1
#endif
// PED accumulation.  Scalar: one chain ped += er^2; ped += ei^2 -- the guard then sees the
// FULL prefix of a marked decision, so far fewer non-competitive paths are logged as
// events (C5/P1024: 1.8 -> 0.76 per vector, verify + checks 1,493 -> 996 us for +120 us
// of traversal).  Packed: the (sum er^2, sum ei^2) pair of one FFMA2 per layer, whose real
// half is the guard's prefix bound -- kept where events are rare anyway and the extra issue
// slot per layer only costs (16-QAM / QPSK with N <= 16: C2 traversal 300 vs 305 us).
// The choice is a function of (N, L) only, so every re-trace twin makes the same one.
#ifndef MPNL_PED_SCALAR
#define MPNL_PED_SCALAR 1
#endif
template <int N, int L>
__host__ __device__ constexpr bool ped_scalar() {
  return MPNL_PED_SCALAR && !(L <= 4 && N <= 16);
}
template <bool SCALAR>
struct Ped;
template <>
struct Ped<true> {
  typedef float T;
  static __device__ __forceinline__ T zero() { return 0.f; }
  static __device__ __forceinline__ T add(u64 e2, T p) {
    const float er = lo32(e2), ei = hi32(e2);
    return __fmaf_rn(ei, ei, __fmaf_rn(er, er, p));
  }
  static __device__ __forceinline__ float bound(T p) { return p; }   // <= the PED prefix
  static __device__ __forceinline__ float value(T p) { return p; }
};
template <>
struct Ped<false> {
  typedef u64 T;
  static __device__ __forceinline__ T zero() { return 0ull; }
  static __device__ __forceinline__ T add(u64 e2, T p) { return ffma2(e2, e2, p); }
  static __device__ __forceinline__ float bound(T p) { return lo32(p); }
  static __device__ __forceinline__ float value(T p) { return lo32(p) + hi32(p); }
};
template <int N, int L, int NS, bool GUARD, bool LAB, bool SAMEV = false, bool SH = false>
__device__ __forceinline__ void traverse_paths(const TabPtrs& T, const float4* __restrict__ zs,
                                               const float* __restrict__ thr,
                                               const uint8_t* __restrict__ lists,
                                               const TreeParams& tp, int list_bytes,
                                               const int (&vl)[NS], const int64_t (&gvl)[NS],
                                               const int (&p)[NS], float (&ped)[NS],
                                               unsigned (&evm)[NS], float (&evp)[NS],
                                               int* lab = nullptr, float* pre = nullptr,
                                               int stop = -1, const u64* xs = nullptr) {
  constexpr int NPP = (N + 1) / 2;
  constexpr int N4 = (N + 3) & ~3;
  constexpr int XM = N < MPNL_XMAX ? N : MPNL_XMAX;
  const float INF = __int_as_float(0x7f800000);
  u64 acc[NS][2 * NPP];
  using PA = Ped<ped_scalar<N, L>()>;
  typename PA::T ped2[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
#pragma unroll
    for (int q = 0; q < NPP; ++q) {
      const float4 z = zs[(SAMEV ? 0 : vl[s]) * NPP + q];
      acc[s][2 * q] = pk2(z.x, z.y);
      acc[s][2 * q + 1] = pk2(z.z, z.w);
    }
    ped2[s] = PA::zero();
    evm[s] = 0u;
    evp[s] = INF;
  }
  const int top_lo = N - tp.n_top;   // layers pos >= top_lo are expanded (n_top <= XM)
  const float4* rc4 = reinterpret_cast<const float4*>(T.rcol);
  const u64 MAGIC2 = pk2(MPNL_MAGIC, MPNL_MAGIC);
  const u64 LM2 = pk2((float)(L - 1), (float)(L - 1));
#pragma unroll
  for (int pos = N - 1; pos >= 0; --pos) {
    const float4 ly = T.lay4[pos];
    const float kxs = ly.w, c2r = ly.y;
    u64 g2[NS];   // negated level indices (-ir, -ii)
    if (pos >= N - XM && pos >= top_lo) {
      if (xs != nullptr) {
        // per-lane precomputed symbols (paths fixed per lane): a negated float
        // pair for a full layer, the list index for a partial one
        const bool full = tp.e[pos] == L * L;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const u64 x = xs[((N - 1 - pos) * NS + s) * MPNL_XS_STRIDE];
          if (full) {
            g2[s] = x;
          } else {
            const unsigned b = lists[(SAMEV ? 0 : (int)gvl[s]) * list_bytes + (int)(unsigned)x];
            // -(float)k for k < 8 without I2F: MAGIC - (MAGIC + k), one FADD2
            g2[s] = fsub2(pk2(MPNL_MAGIC, MPNL_MAGIC),
                          pk2(__uint_as_float(0x4B400000u | (b >> 3)),
                              __uint_as_float(0x4B400000u | (b & 7u))));
          }
        }
      } else {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          int ir, ii;
          expanded_symbol<L>(tp, pos, p[s], lists + gvl[s] * list_bytes, ir, ii);
          g2[s] = pk2(-(float)ir, -(float)ii);
        }
      }
    } else {
      // packed slicing of (re, im): the per-element twin of slice_axis
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const u64 s2 = pk2(__saturatef(__fmul_rn(lo32(acc[s][pos]), kxs)),
                           __saturatef(__fmul_rn(hi32(acc[s][pos]), kxs)));
        const u64 mm = ffma2(s2, LM2, MAGIC2);
        g2[s] = fsub2(MAGIC2, mm);
        if (GUARD) {
          const u64 t2 = ffma2(s2, LM2, g2[s]);
          const float th = thr[(SAMEV ? 0 : vl[s]) * N4 + pos];
          guard_mark(fmaxf(fabsf(lo32(t2)), fabsf(hi32(t2))), th, 1u << pos, PA::bound(ped2[s]),
                     evm[s], evp[s]);
        }
      }
    }
    if (LAB) {
      lab[pos] = (int)(-lo32(g2[0])) * 8 + (int)(-hi32(g2[0]));
      pre[pos] = PA::value(ped2[0]);
      if (pos == stop) return;
    }
    constexpr bool SH2 = SH && NS == 2;
    const bool shared = SH2 && pos == N - 1;   // compile-time in the unrolled loop
    const int ns = shared ? 1 : NS;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s >= ns) break;
      const u64 e2 = ffma2(pk2(-c2r, -c2r), g2[s], acc[s][pos]);   // c2r n + u
      ped2[s] = PA::add(e2, ped2[s]);
    }
    // push this layer's symbols into the rows below: acc_k += r''_k,pos * s.
    // Row pairs are walked top-down so the row the next layer slices (pos - 1)
    // is updated first and the other rows' updates fill its latency.
    const float4* rc = rc4 + pos * NPP;
#pragma unroll
    for (int qq = 0; qq < (pos + 1) / 2; ++qq) {
#if MPNL_QDESC
      const int q = (pos + 1) / 2 - 1 - qq;
#else
      const int q = qq;
#endif
      const float4 r = rc[q];              // {rr_2q, ri_2q, rr_2q+1, ri_2q+1}
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (s >= ns) break;
        const u64 gs = pk2(-hi32(g2[s]), lo32(g2[s]));   // (fi, -fr): operand modifiers
        acc[s][2 * q] = ffma2(pk2(-r.x, -r.x), g2[s], acc[s][2 * q]);
        acc[s][2 * q] = ffma2(gs, pk2(-r.y, -r.y), acc[s][2 * q]);
        if (2 * q + 1 < pos) {
          acc[s][2 * q + 1] = ffma2(pk2(-r.z, -r.z), g2[s], acc[s][2 * q + 1]);
          acc[s][2 * q + 1] = ffma2(gs, pk2(-r.w, -r.w), acc[s][2 * q + 1]);
        }
      }
    }
    if (shared) {   // the sibling continues from the shared state (register renaming)
#pragma unroll
      for (int k = 0; k < 2 * NPP; ++k) acc[NS - 1][k] = acc[0][k];
      ped2[NS - 1] = ped2[0];
    }
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) ped[s] = PA::value(ped2[s]);
}

// Single-path re-trace with the identical arithmetic: level indices lab[pos]
// (ir*8+ii) and the PED prefix pre[pos] before layer pos, for pos >= stop.
// zs: this vector's NPP float4 row pairs.  vlist: this vector's lists.
template <int N, int L>
__device__ __forceinline__ void retrace_inline(const float* tab, int m, const float4* zs,
                                               const uint8_t* vlist, const TreeParams& tp, int p,
                                               int stop, int* lab, float* pre) {
  const TabPtrs T = tab_ptrs(tab, m, N);
  const int vl[1] = {0}, pp[1] = {p};
  const int64_t gvl[1] = {0};
  float ped[1], evp[1];
  unsigned evm[1];
  traverse_paths<N, L, 1, false, true>(T, zs, nullptr, vlist, tp, 0, vl, gvl, pp, ped, evm, evp,
                                       lab, pre, stop);
}

// Paths per lane: more paths amortise the r'' loads and add ILP, but the
// fully unrolled traversal grows as PT * N^2 instructions; beyond N = 16 the
// two-path loop no longer fits the instruction cache (ncu: no_instruction
// stalls dominate), so large N runs one path per lane at twice the warps.
#ifndef MPNL_PT_SMALL
#define MPNL_PT_SMALL 4
#endif
#ifndef MPNL_PT_MID
#define MPNL_PT_MID 2
#endif
#ifndef MPNL_PT_LARGE
#define MPNL_PT_LARGE 1
#endif
#ifndef MPNL_MINB_SMALL
#define MPNL_MINB_SMALL 0
#endif
#ifndef MPNL_MINB_MID
#define MPNL_MINB_MID 0
#endif
#ifndef MPNL_MINB_LARGE
#define MPNL_MINB_LARGE 0
#endif
template <int N>
struct TravCfg {
  static constexpr int PT = N <= 8 ? MPNL_PT_SMALL : (N <= 16 ? MPNL_PT_MID : MPNL_PT_LARGE);
  static constexpr int MAXT = 128;                       // threads per CTA
  static constexpr int MB = N <= 8 ? MPNL_MINB_SMALL : (N <= 16 ? MPNL_MINB_MID : MPNL_MINB_LARGE);
  static constexpr int MINB = MB ? MB : (PT * N <= 24 ? 4 : 3);   // CTAs per SM (no spills)
};

// A NODE event's type word is the NEGATED lower bound evp of the path's PED
// prefix at its first marked layer (sign bit set, so never equal to EV_CUT /
// EV_TIE): the check kernel drops the event before any re-trace when evp
// already exceeds the vector's final bound.
__device__ __forceinline__ int ev_node_w(float evp) {
  return (int)(__float_as_uint(evp) | 0x80000000u);
}
__device__ __forceinline__ bool ev_is_node(int w) { return w < 0; }
__device__ __forceinline__ float ev_node_evp(int w) {
  return __uint_as_float((unsigned)w & 0x7fffffffu);
}

// mark vector gv for the fp64 kernel (the first marker appends it to the list)
// reasons (stats[4 + reason]): 0 three-way tie, 1 fp64-level tie, 2 fp64
// disagreement at a guarded decision, 3 event-log overflow
__device__ __forceinline__ void send_to_fp64(const DetectArgs& a, int64_t gv, int reason) {
  if (atomicExch(a.vflag + gv, 1u) == 0u) {
    const int slot = atomicAdd(a.counters, 1);
    a.fix_list[slot] = gv;
    if (a.stats) {
      atomicAdd(a.stats + 3, 1);
      atomicAdd(a.stats + 4 + reason, 1);
    }
  }
}

__device__ __forceinline__ void log_event(const DetectArgs& a, int4 e) {
  const int idx = atomicAdd(a.counters + 1, 1);
  if (a.stats) atomicAdd(a.stats, 1);
  if (idx < a.ev_cap) a.events[idx] = e;
  else send_to_fp64(a, (int64_t)(unsigned)e.z, 3);
}

// ---------------------------------------------------------------------------
// top-3 (metric, path) bookkeeping
// ---------------------------------------------------------------------------
struct Top3 {
  float m1, m2, m3;
  unsigned p1, p2;
};

__device__ __forceinline__ bool tless(float a, unsigned pa, float b, unsigned pb) {
  return a < b || (a == b && pa < pb);
}

__device__ __forceinline__ void top3_insert(Top3& t, float m, unsigned p) {
  // branch-free: (m1,p1) <= (m2,p2) <= (m3) in the (metric, path) order
  const bool lt1 = tless(m, p, t.m1, t.p1), lt2 = tless(m, p, t.m2, t.p2);
  t.m3 = lt2 ? t.m2 : fminf(t.m3, m);
  const float m2 = lt1 ? t.m1 : (lt2 ? m : t.m2);
  const unsigned p2 = lt1 ? t.p1 : (lt2 ? p : t.p2);
  t.m2 = m2;
  t.p2 = p2;
  t.m1 = lt1 ? m : t.m1;
  t.p1 = lt1 ? p : t.p1;
}

__device__ __forceinline__ void top3_pop(Top3& t) {
  t.m1 = t.m2; t.p1 = t.p2; t.m2 = t.m3; t.p2 = 0xffffffffu;
  t.m3 = __int_as_float(0x7f800000);
}

// warp-wide three smallest (metric, path) (metrics >= 0 order like uints: REDUX.MIN)
__device__ __forceinline__ void warp_top3(Top3 t, float& b1, unsigned& q1, float& b2,
                                          unsigned& q2, float& b3) {
  unsigned k = __reduce_min_sync(0xffffffffu, __float_as_uint(t.m1));
  unsigned q = __reduce_min_sync(0xffffffffu, __float_as_uint(t.m1) == k ? t.p1 : 0xffffffffu);
  b1 = __uint_as_float(k);
  q1 = q;
  if (__float_as_uint(t.m1) == k && t.p1 == q) top3_pop(t);
  k = __reduce_min_sync(0xffffffffu, __float_as_uint(t.m1));
  q = __reduce_min_sync(0xffffffffu, __float_as_uint(t.m1) == k ? t.p1 : 0xffffffffu);
  b2 = __uint_as_float(k);
  q2 = q;
  if (__float_as_uint(t.m1) == k && t.p1 == q) top3_pop(t);
  b3 = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(t.m1)));
}

// shuffle-based variant for groups of `width` < 32 lanes (VPI mode)
__device__ __forceinline__ void group_top3(Top3 t, int width, float& b1, unsigned& q1, float& b2,
                                           unsigned& q2, float& b3) {
  for (int o = width >> 1; o; o >>= 1) {
    Top3 u;
    u.m1 = __shfl_xor_sync(0xffffffffu, t.m1, o);
    u.m2 = __shfl_xor_sync(0xffffffffu, t.m2, o);
    u.m3 = __shfl_xor_sync(0xffffffffu, t.m3, o);
    u.p1 = __shfl_xor_sync(0xffffffffu, t.p1, o);
    u.p2 = __shfl_xor_sync(0xffffffffu, t.p2, o);
    Top3 r = t;
    top3_insert(r, u.m1, u.p1);
    top3_insert(r, u.m2, u.p2);
    r.m3 = fminf(r.m3, u.m3);
    t = r;
  }
  b1 = t.m1; q1 = t.p1; b2 = t.m2; q2 = t.p2; b3 = t.m3;
}

// ===========================================================================
// K2: partial-layer selection lists
// ===========================================================================
// K2 (templated on the expansion count E of the partial layer): one thread per
// (vector, parent), block = (parents, vectors).  The E nearest points of the
// centre are the E smallest sums dx_i + dy_j of the two per-axis
// Schnorr-Euchner distance orders (only the SET matters for hard output): a
// register-resident k-smallest-sums merge, E + 1 picks (the (E+1)-th sum is
// the guard's cut partner).
template <int K, typename T>
__device__ __forceinline__ T dyn_at(const T (&v)[K], int i) {
  T r = v[0];
#pragma unroll
  for (int k = 1; k < K; ++k) r = (i == k) ? v[k] : r;
  return r;
}

// per-axis levels sorted by distance to x (level-index units): lev[r], d[r]
template <int L>
__device__ __forceinline__ void se_order(float x, int (&lev)[L], float (&d)[L]) {
  const int n0 = (int)rintf(fminf(fmaxf(x, 0.f), (float)(L - 1)));
  int lo = n0 - 1, hi = n0 + 1;
  lev[0] = n0;
  d[0] = (x - n0) * (x - n0);
#pragma unroll
  for (int r = 1; r < L; ++r) {
    const bool up = (hi < L) && (lo < 0 || (hi - x) < (x - lo));
    const int l = up ? hi : lo;
    hi += up ? 1 : 0;
    lo -= up ? 0 : 1;
    lev[r] = l;
    d[r] = (x - l) * (x - l);
  }
}

// The E nearest points (E <= EMAX) of the centre (xl, yl) in level-index units
// (unclamped): packed label bytes (ir << 3 | ii) in `words`, the E-th and
// (E+1)-th smallest squared distances (index units) in kprev / knext.  th =
// the thread's slot in the per-thread shared-memory arrays (L = 8, EMAX > 4).
template <int L, int EMAX>
__device__ __forceinline__ void select_nearest(float xl, float yl, int E, int th,
                                               unsigned (&words)[(EMAX + 3) / 4], float& kprev,
                                               float& knext) {
  const float INF = __int_as_float(0x7f800000);
  int ox[L], oy[L];
  float dx[L], dy[L];
  se_order<L>(xl, ox, dx);
  se_order<L>(yl, oy, dy);
  constexpr int NW = (EMAX + 3) / 4;
#pragma unroll
  for (int i = 0; i < NW; ++i) words[i] = 0u;
  kprev = 0.f;
  knext = 0.f;
  if constexpr (EMAX <= 4) {
    // E <= 4: the E + 1 smallest sums lie in row 0, column 0 or at (1,1)
    // ((i+1)(j+1) <= 5): a two-pointer merge of row 0 and column 0 plus the corner
    constexpr int K = (L - 1) < 4 ? (L - 1) : 4;
    float ra[K], cb[K];
    unsigned la[K], lb[K];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      ra[t] = dx[0] + dy[t + 1];
      cb[t] = dx[t + 1] + dy[0];
      la[t] = ((unsigned)ox[0] << 3) | (unsigned)oy[t + 1];
      lb[t] = ((unsigned)ox[t + 1] << 3) | (unsigned)oy[0];
    }
    const float cc = dx[1] + dy[1];
    const unsigned lc = ((unsigned)ox[1] << 3) | (unsigned)oy[1];
    words[0] = ((unsigned)ox[0] << 3) | (unsigned)oy[0];
    kprev = dx[0] + dy[0];
    int i = 0, j = 0;
    bool ct = false;
#pragma unroll
    for (int k = 1; k <= 4; ++k) {
      if (k > E) break;
      const float va = i < K ? dyn_at(ra, i) : INF;
      const float vb = j < K ? dyn_at(cb, j) : INF;
      const float vc = (i >= 1 && j >= 1 && !ct) ? cc : INF;
      const bool ta = va <= vb && va <= vc, tb = !ta && vb <= vc;
      const float v = ta ? va : (tb ? vb : vc);
      if (k < E) {
        const unsigned b = ta ? dyn_at(la, i) : (tb ? dyn_at(lb, j) : lc);
        words[k >> 2] |= b << (8 * (k & 3));
        kprev = v;
      } else {
        knext = v;
      }
      i += ta ? 1 : 0;
      j += tb ? 1 : 0;
      ct = ct || (!ta && !tb);
    }
  } else if constexpr (L == 8) {
    // 64-QAM, E > 4.  Row i of the merge (the x-axis order's i-th level) offers the sum
    // dx_i + dy_{w_i}; its KEY is that sum with the three low mantissa bits replaced by
    // i, so the frontier's minimum and its row come out of one min tree (FMNMX3) and a
    // mask instead of a compare/select chain.  Keys and per-axis distances live in
    // per-thread (transposed) shared memory, so every data-dependent access is one
    // conflict-free LDS / STS.  Keys are non-decreasing along a row, hence the picks are exactly
    // the E smallest cells in KEY order; that order differs from the exact one only
    // between sums closer than 8 ulp, and the returned kprev / knext are keys (within
    // 8 ulp below the sums): select_cut_slack() widens the cut guard accordingly, so a
    // cut that the truncation could have changed is always logged and re-selected in
    // fp64 by the check kernel.
    __shared__ float sdx[L][128], sdy[L][128], snk[L][128];
    const float BIG = 1e30f;
    auto mkkey = [](float v, unsigned row) {
      return __uint_as_float((__float_as_uint(v) & ~7u) | row);
    };
    // level orders and the rows' column counters as 4-bit fields of three registers
    // (byte arrays in shared memory cost 2-4-way bank conflicts per lookup)
    unsigned oxp = 0u, oyp = 0u, swp = 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      sdx[i][th] = dx[i];
      sdy[i][th] = dy[i];
      snk[i][th] = mkkey(dx[i] + dy[0], (unsigned)i);
      oxp |= (unsigned)ox[i] << (4 * i);
      oyp |= (unsigned)oy[i] << (4 * i);
    }
#pragma unroll
    for (int pick = 0; pick <= EMAX; ++pick) {
      if (pick > E) break;
      const float best =
          fminf(fminf(fminf(fminf(snk[0][th], snk[1][th]), snk[2][th]),
                      fminf(fminf(snk[3][th], snk[4][th]), snk[5][th])),
                fminf(snk[6][th], snk[7][th]));
      if (pick < E) {
        const unsigned sel = __float_as_uint(best) & 7u;
        const unsigned col = (swp >> (4u * sel)) & 15u;
        const unsigned b = (((oxp >> (4u * sel)) & 7u) << 3) | ((oyp >> (4u * col)) & 7u);
        const unsigned cn = col + 1u < (unsigned)L ? col + 1u : (unsigned)(L - 1);
        const float nxt = (col + 1u < (unsigned)L) ? sdx[sel][th] + sdy[cn][th] : BIG;
        snk[sel][th] = mkkey(nxt, sel);
        swp += 1u << (4u * sel);
        words[pick >> 2] |= b << (8 * (pick & 3));
        kprev = best;
      } else {
        knext = best;
      }
    }
  } else {
    // L <= 4: a register-resident merge (the orders are short select chains)
    int w[L];
    float nk[L];
#pragma unroll
    for (int i = 0; i < L; ++i) { w[i] = 0; nk[i] = dx[i] + dy[0]; }
#pragma unroll
    for (int pick = 0; pick <= EMAX; ++pick) {
      if (pick > E) break;
      int sel = 0;
      float best = nk[0];
#pragma unroll
      for (int i = 1; i < L; ++i) {
        const bool lt = nk[i] < best;
        best = lt ? nk[i] : best;
        sel = lt ? i : sel;
      }
      if (pick < E) {
        const int col = dyn_at(w, sel);
        const unsigned b = (unsigned)((dyn_at(ox, sel) << 3) | dyn_at(oy, col));
        const float nxt = (col + 1 < L) ? dyn_at(dx, sel) + dyn_at(dy, col + 1) : INF;
        words[pick >> 2] |= b << (8 * (pick & 3));
        kprev = best;
#pragma unroll
        for (int i = 0; i < L; ++i)
          if (i == sel) { w[i] = col + 1; nk[i] = nxt; }
      } else {
        knext = best;
      }
    }
  }
}

// first K entries of the per-axis Schnorr-Euchner order (levels by distance
// to x, ties to the lower level), K <= L
template <int L, int K>
__device__ __forceinline__ void se_order_k(float x, int (&lev)[K], float (&d)[K]) {
  if constexpr (L == 4) {
    // 16-QAM axis: the order is fixed by the interval of x among the midpoints
    // {0.5, 1, 1.5, 2, 2.5} (ties to the lower level): idx = ceil(2x - 1)
    // clamped to [0, 5], then 2-bit levels from a 6-byte table.  Same distances
    // as the generic walk; the order can differ only between equidistant
    // levels, which the selection's cut guard covers (equal keys at the cut).
    const int idx = min(max(__float2int_ru(fmaf(x, 2.f, -1.f)), 0), 5);
    const unsigned code = (unsigned)(0x1B1E36C9E1E4ull >> (8 * idx));
#pragma unroll
    for (int r = 0; r < K; ++r) {
      lev[r] = (int)((code >> (2 * r)) & 3u);
      d[r] = (x - lev[r]) * (x - lev[r]);
    }
    return;
  }
  const int n0 = (int)rintf(fminf(fmaxf(x, 0.f), (float)(L - 1)));
  int lo = n0 - 1, hi = n0 + 1;
  lev[0] = n0;
  d[0] = (x - n0) * (x - n0);
#pragma unroll
  for (int r = 1; r < K; ++r) {
    const bool up = (hi < L) && (lo < 0 || (hi - x) < (x - lo));
    const int l = up ? hi : lo;
    hi += up ? 1 : 0;
    lo -= up ? 0 : 1;
    lev[r] = l;
    d[r] = (x - l) * (x - l);
  }
}

// select_nearest for a compile-time E <= 4: the same two-pointer merge of
// row 0 / column 0 / corner (1,1), fully unrolled (no E-dependent branches)
// over only the min(L, E + 1) leading entries of each axis order.
template <int L, int E>
__device__ __forceinline__ void select_nearest_e(float xl, float yl, unsigned& word, float& kprev,
                                                 float& knext) {
  static_assert(E >= 2 && E <= 4, "E in 2..4");
  constexpr int KK = (E + 1) < L ? (E + 1) : L;   // entries per axis
  constexpr int K = KK - 1;                        // row-0 / column-0 candidates
  const float INF = __int_as_float(0x7f800000);
  int ox[KK], oy[KK];
  float dx[KK], dy[KK];
  se_order_k<L, KK>(xl, ox, dx);
  se_order_k<L, KK>(yl, oy, dy);
  if constexpr ((E == 2 || E == 4) && KK >= 3) {
    // The merge below, resolved in closed form (same picks, same tie rules,
    // same kprev / knext values).  R_t = dx0 + dy_t (row 0), C_t = dx_t + dy0
    // (column 0), D = dx1 + dy1; both runs ascend and D >= R1, C1.
    auto R = [&](int t) { return t < KK ? dx[0] + dy[t] : INF; };
    auto C = [&](int t) { return t < KK ? dx[t] + dy[0] : INF; };
    auto lr = [&](int t) { return ((unsigned)ox[0] << 3) | (unsigned)oy[t < KK ? t : 0]; };
    auto lcl = [&](int t) { return ((unsigned)ox[t < KK ? t : 0] << 3) | (unsigned)oy[0]; };
    const float R1 = R(1), C1 = C(1), R2 = R(2), C2 = C(2);
    word = ((unsigned)ox[0] << 3) | (unsigned)oy[0];
    if constexpr (E == 2) {
      const bool ta = R1 <= C1;
      word |= (ta ? lr(1) : lcl(1)) << 8;
      kprev = ta ? R1 : C1;
      knext = ta ? fminf(R2, C1) : fminf(R1, C2);
    } else {
      const float R3 = R(3), C3 = C(3), D = dx[1] + dy[1];
      const unsigned ld = ((unsigned)ox[1] << 3) | (unsigned)oy[1];
      const bool rr = R2 <= C1;               // picks R1, R2, then R3 | C1
      const bool cc = !rr && C2 < R1;         // picks C1, C2, then C3 | R1
      const bool t3r = R3 <= C1, t3c = R1 <= C3;
      const bool a3 = R2 <= C2 && R2 <= D, b3 = !a3 && C2 <= D;   // mid: R1, C1, then
      unsigned b1, b2, b3l;
      float k3, k4;
      if (rr) {
        b1 = lr(1); b2 = lr(2);
        b3l = t3r ? lr(3) : lcl(1);
        k3 = t3r ? R3 : C1;
        k4 = t3r ? fminf(R(4), C1) : fminf(fminf(R3, C2), D);
      } else if (cc) {
        b1 = lcl(1); b2 = lcl(2);
        b3l = t3c ? lr(1) : lcl(3);
        k3 = t3c ? R1 : C3;
        k4 = t3c ? fminf(fminf(R2, C3), D) : fminf(R1, C(4));
      } else {
        b1 = lr(1); b2 = lcl(1);
        b3l = a3 ? lr(2) : (b3 ? lcl(2) : ld);
        k3 = a3 ? R2 : (b3 ? C2 : D);
        k4 = a3 ? fminf(fminf(R3, C2), D) : (b3 ? fminf(fminf(R2, C3), D) : fminf(R2, C2));
      }
      word |= (b1 << 8) | (b2 << 16) | (b3l << 24);
      kprev = k3;
      knext = k4;
    }
    return;
  }
  float ra[K], cb[K];
  unsigned la[K], lb[K];
#pragma unroll
  for (int t = 0; t < K; ++t) {
    ra[t] = dx[0] + dy[t + 1];
    cb[t] = dx[t + 1] + dy[0];
    la[t] = ((unsigned)ox[0] << 3) | (unsigned)oy[t + 1];
    lb[t] = ((unsigned)ox[t + 1] << 3) | (unsigned)oy[0];
  }
  const float cc = dx[1] + dy[1];
  const unsigned lc = ((unsigned)ox[1] << 3) | (unsigned)oy[1];
  word = ((unsigned)ox[0] << 3) | (unsigned)oy[0];
  kprev = dx[0] + dy[0];
  knext = INF;
  int i = 0, j = 0;
  bool ct = false;
#pragma unroll
  for (int k = 1; k <= E; ++k) {
    const float va = i < K ? dyn_at(ra, i) : INF;
    const float vb = j < K ? dyn_at(cb, j) : INF;
    const float vc = (i >= 1 && j >= 1 && !ct) ? cc : INF;
    const bool ta = va <= vb && va <= vc, tb = !ta && vb <= vc;
    const float v = ta ? va : (tb ? vb : vc);
    if (k < E) {
      const unsigned b = ta ? dyn_at(la, i) : (tb ? dyn_at(lb, j) : lc);
      word |= b << (8 * k);
      kprev = v;
    } else {
      knext = v;
    }
    i += ta ? 1 : 0;
    j += tb ? 1 : 0;
    ct = ct || (!ta && !tb);
  }
}

// write E label bytes of one parent's selection
template <int EMAX>
__device__ __forceinline__ void store_selection(uint8_t* out, int E,
                                                const unsigned (&words)[(EMAX + 3) / 4]) {
  constexpr int NW = (EMAX + 3) / 4;
  if ((E & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0) {
#pragma unroll
    for (int i = 0; i < NW; ++i)
      if (4 * i < E) reinterpret_cast<unsigned*>(out)[i] = words[i];
  } else {
#pragma unroll
    for (int k = 0; k < EMAX; ++k)
      if (k < E) out[k] = (uint8_t)(words[k >> 2] >> (8 * (k & 3)));
  }
}

// cut guard: distance keys are within 2 sqrt2 E (sqrt k) + 2E^2 (+ rounding).
// slack_u: extra relative slack in units of u = 2^-24 (select_cut_slack: the key-ordered
// 64-QAM merge returns sums truncated by up to 8 ulp = 16 u each and may order sums
// closer than that either way).
__device__ __forceinline__ bool cut_near(float kprev, float knext, float Eb, float slack_u = 0.f) {
  const float bound = 2.8284272f * Eb * (sqrt_up(kprev) + sqrt_up(knext)) + 4.f * Eb * Eb +
                      (8.f + slack_u) * MPNL_U * (fmaxf(knext, kprev) + 1.f);
  return knext - kprev <= bound;
}
template <int L, int EMAX>
__device__ __forceinline__ constexpr float select_cut_slack() {
  return (L == 8 && EMAX > 4) ? 64.f : 0.f;
}

#ifndef MPNL_SELECT_MINB
#define MPNL_SELECT_MINB 1   // minimum CTAs per SM asked of the compiler (register cap)
#endif
template <int N, int L, int EMAX>
__global__ void __launch_bounds__(128, MPNL_SELECT_MINB)
select_kernel(const DetectArgs a, const TreeParams tp, int pos, int npar, int vblocks) {
  const int E = tp.e[pos];   // <= EMAX
  constexpr int XM = N < MPNL_XMAX ? N : MPNL_XMAX;
  constexpr int NPP = (N + 1) / 2, N4 = (N + 3) & ~3;
  // grid.x = channel x vector block, grid.y = parent block: no per-thread division
  const int c = blockIdx.x / vblocks;
  const int vi = (blockIdx.x - c * vblocks) * blockDim.y + threadIdx.y;
  const int par = blockIdx.y * blockDim.x + threadIdx.x;
  if (par >= npar || vi >= a.V) return;
  const int64_t gv = (int64_t)c * a.V + vi;
  const float* tab = a.tables + (int64_t)c * TableLayout(a.m, N).total;
  const TabPtrs T = tab_ptrs(tab, a.m, N);
  const int p0 = par * tp.stride[pos + 1];
  uint8_t* vlist = a.lists + gv * tp.list_bytes;
  const float thr_pos = __ldg(a.thrg + gv * N4 + pos);   // issued early (used by the guard)
  // acc of row pos after the expanded layers above it (the traversal's fma order)
  const float2 z = reinterpret_cast<const float2*>(a.zq + gv * NPP)[pos];
  float xr = z.x, xi = z.y;
#pragma unroll
  for (int q = 0; q < XM; ++q) {
    const int j = N - 1 - q;
    if (j > pos) {
      int ir, ii;
      expanded_symbol<L>(tp, j, p0, vlist, ir, ii);
      const float2 r2 = rcol_at(T.rcol, NPP, pos, j);
      acc_step(xr, xi, r2.x, r2.y, (float)ir, (float)ii);
    }
  }
  const float kx = T.lay4[pos].x;
  unsigned words[(EMAX + 3) / 4];
  float kprev, knext;
  select_nearest<L, EMAX>(__fmul_rn(xr, kx), __fmul_rn(xi, kx), E,
                          threadIdx.y * blockDim.x + threadIdx.x, words, kprev, knext);
  store_selection<EMAX>(vlist + tp.list_off[pos] + par * E, E, words);
  if (cut_near(kprev, knext, 0.5f - thr_pos, select_cut_slack<L, EMAX>()))
    log_event(a, make_int4(p0, pos, (int)gv, EV_CUT));
}

// ===========================================================================
// K1b': per-vector preparation fused with the partial-layer selection.
// Thread = vector (CTA = 128 vectors of one channel).  The channel's fp64 Q^H
// (transposed) and shifts are staged in shared memory and read as broadcasts;
// each thread rotates its own y in fp64 in blocks of RB rows (y re-read from
// L1), writes its z' row pairs, guard thresholds and (E_acc, corr) as
// contiguous 16-byte stores, and then -- when the tree's only partial layer
// sits at the top or right below a full top layer (every BASELINE config) --
// selects that layer's E nearest points for each of its parents from the
// fp32 z' it just produced, with the traversal's arithmetic (select_nearest).
// ===========================================================================
template <int N>
struct Prep2Smem {
  // qt | shift | lay | y rows of the CTA's vectors (odd stride: conflict-free per-thread reads)
  __host__ __device__ static constexpr int ystride(int m) { return m | 1; }
  __host__ __device__ static constexpr int bytes(int m, int vpc, int yb) {
    return 16 * m * N + 16 * N + 16 * N + vpc * ystride(m) * yb;
  }
};

template <int N, int L, int E, int TPV>
__global__ void __launch_bounds__(128)
prep2_kernel(const DetectArgs a, const TreeParams tp, int chunks, int pos_sel) {
  constexpr int NPP = (N + 1) / 2, N4 = (N + 3) & ~3;
  // rows per block (even, a multiple of 4); thread j of a vector's TPV group
  // rotates blocks j, j + TPV, ... and selects for parents j, j + TPV, ...
  constexpr int RB = TPV == 1 ? (N < 8 ? N4 : 8) : 4;
  constexpr int NB = (N + RB - 1) / RB;
  constexpr int VPC = 128 / TPV;                     // vectors per CTA
  extern __shared__ __align__(16) uint8_t psm2[];
  const int m = a.m;
  double2* qt = reinterpret_cast<double2*>(psm2);
  double2* sh = qt + m * N;
  float4* ly = reinterpret_cast<float4*>(sh + N);
  const TableLayout tl(m, N);
  const int64_t c = blockIdx.x / chunks;
  const int j = threadIdx.x % TPV;
  const int v = (blockIdx.x - (int)c * chunks) * VPC + threadIdx.x / TPV;
  const float* tab = a.tables + c * (int64_t)tl.total;
  const int sy = Prep2Smem<N>::ystride(m);
  const int v0 = (blockIdx.x - (int)c * chunks) * VPC;
  const int nvc = (int)min((int64_t)VPC, a.V - v0);
  float2* ys32 = reinterpret_cast<float2*>(ly + N);
  double2* ys64 = reinterpret_cast<double2*>(ly + N);
  {
    const double2* q = reinterpret_cast<const double2*>(tab + tl.off_qh);
    for (int i = threadIdx.x; i < m * N; i += 128) qt[i] = q[i];
    const double2* s2 = reinterpret_cast<const double2*>(tab + tl.off_shift);
    const float4* l4 = reinterpret_cast<const float4*>(tab + tl.off_lay);
    for (int i = threadIdx.x; i < N; i += 128) { sh[i] = s2[i]; ly[i] = l4[i]; }
    // the CTA's y rows: one coalesced flat copy into the padded layout
    // ((v, r) by a float reciprocal: exact for i < 2^13 >= VPC * m)
    const int64_t g0 = (c * a.V + v0) * m;
    const float rm = 1.f / (float)m;
    for (int i = threadIdx.x; i < nvc * m; i += 128) {
      const int vv = (int)(((float)i + 0.5f) * rm), r = i - vv * m;
      if (a.y_f64) ys64[vv * sy + r] = reinterpret_cast<const double2*>(a.y)[g0 + i];
      else ys32[vv * sy + r] = reinterpret_cast<const float2*>(a.y)[g0 + i];
    }
  }
  __syncthreads();
  const bool live = v < a.V;   // (whole TPV groups share liveness: shuffles stay in-group)
  const int64_t gv = c * a.V + (live ? v : 0);
  const int vl = live ? v - v0 : 0;
  auto yat = [&](int r) -> double2 {
    if (a.y_f64) return ys64[vl * sy + r];
    const float2 f = ys32[vl * sy + r];
    return make_double2(f.x, f.y);
  };
  // ||y|| (every thread of the group: the per-row bounds need it)
  double yn = 0.0;
  for (int r = 0; r < m; ++r) {
    const double2 y = yat(r);
    yn = fma(y.x, y.x, fma(y.y, y.y, yn));
  }
  const float ynf = (float)sqrt(yn) * 1.0001f;
  float4* zo = a.zq + gv * NPP;
  float4* to = reinterpret_cast<float4*>(a.thrg + gv * N4);
  double e2 = 0.0, zn = 0.0;
  float zsr = 0.f, zsi = 0.f, thsel = 0.f;
#pragma unroll
  for (int b0 = 0; b0 < NB; b0 += TPV) {
    const int k0 = (b0 + j) * RB;
    if (k0 < N) {
      double zr[RB], zi[RB];
#pragma unroll
      for (int t = 0; t < RB; ++t) { zr[t] = 0.0; zi[t] = 0.0; }
      for (int r = 0; r < m; ++r) {
        const double2 y = yat(r);
#pragma unroll
        for (int t = 0; t < RB; ++t) {
          if (k0 + t < N) {
            const double2 q = qt[r * N + k0 + t];
            zr[t] = fma(q.x, y.x, zr[t]);
            zr[t] = fma(-q.y, y.y, zr[t]);
            zi[t] = fma(q.x, y.y, zi[t]);
            zi[t] = fma(q.y, y.x, zi[t]);
          }
        }
      }
      float zf[2 * RB], th[RB];
#pragma unroll
      for (int t = 0; t < RB; ++t) {
        const int k = k0 + t;
        zf[2 * t] = 0.f; zf[2 * t + 1] = 0.f; th[t] = 0.5f;
        if (k < N) {
          const double2 shk = sh[k];
          const float2 z = make_float2((float)(zr[t] - shk.x), (float)(zi[t] - shk.y));
          zf[2 * t] = z.x; zf[2 * t + 1] = z.y;
          const float4 lk = ly[k];
          const float e = row_bound(ynf, z, lk, k, m, N, L, a.guard_scale, 0);
          th[t] = 0.5f - e / lk.y - MPNL_U * 3.f * L;
          e2 += (double)e * e;
          zn += zr[t] * zr[t] + zi[t] * zi[t];
          if (k == pos_sel) { zsr = z.x; zsi = z.y; thsel = th[t]; }
        }
      }
      if (live) {
#pragma unroll
        for (int q = 0; q < RB / 2; ++q)
          if (k0 / 2 + q < NPP)
            zo[k0 / 2 + q] = make_float4(zf[4 * q], zf[4 * q + 1], zf[4 * q + 2], zf[4 * q + 3]);
#pragma unroll
        for (int q = 0; q < RB / 4; ++q)
          if (k0 + 4 * q < N4)
            to[k0 / 4 + q] = make_float4(th[4 * q], th[4 * q + 1], th[4 * q + 2], th[4 * q + 3]);
      }
    }
  }
  if (TPV > 1) {
    // group sums (fixed xor order) and the selected row from its owner thread
#pragma unroll
    for (int o = 1; o < TPV; o <<= 1) {
      e2 += __shfl_xor_sync(0xffffffffu, e2, o);
      zn += __shfl_xor_sync(0xffffffffu, zn, o);
    }
    if (E > 0 && pos_sel >= 0) {
      const int src = (threadIdx.x & 31 & ~(TPV - 1)) + (pos_sel / RB) % TPV;
      zsr = __shfl_sync(0xffffffffu, zsr, src);
      zsi = __shfl_sync(0xffffffffu, zsi, src);
      thsel = __shfl_sync(0xffffffffu, thsel, src);
    }
  }
  if (!live) return;
  if (j == 0) a.vaux[gv] = make_float2((float)sqrt(e2) * 1.001f, (float)(yn - zn));
  if constexpr (E > 0) {
    // partial layer pos_sel (tp.e[pos_sel] == E): parents = the full top
    // layer's L^2 points (or one parent when pos_sel is the top layer); centre
    // of parent (ir, ii) = z'_pos + r''_{pos,N-1} (ir, ii) with the traversal's
    // fma sequence
    const int npar = pos_sel == N - 1 ? 1 : L * L;
    const float kx = ly[pos_sel].x;
    const float Eb = 0.5f - thsel;
    const float2 r2 = pos_sel == N - 1 ? make_float2(0.f, 0.f)
                                       : rcol_at(tab + tl.off_rcol, NPP, pos_sel, N - 1);
    uint8_t* out = a.lists + gv * tp.list_bytes + tp.list_off[pos_sel];
    const int st = tp.stride[pos_sel + 1];
#pragma unroll 2
    for (int par = j; par < npar; par += TPV) {
      float xr = zsr, xi = zsi;
      if (npar > 1) acc_step(xr, xi, r2.x, r2.y, (float)(par / L), (float)(par % L));
      unsigned word;
      float kprev, knext;
      select_nearest_e<L, E>(__fmul_rn(xr, kx), __fmul_rn(xi, kx), word, kprev, knext);
      if (E == 4) {
        *reinterpret_cast<unsigned*>(out + par * 4) = word;
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k) out[par * E + k] = (uint8_t)(word >> (8 * k));
      }
      if (cut_near(kprev, knext, Eb)) log_event(a, make_int4(par * st, pos_sel, (int)gv, EV_CUT));
    }
  }
}

// ===========================================================================
// K3: traversal (hot kernel)
//
// Persistent CTAs: the grid is sized to the resident capacity and CTA b owns
// the contiguous item range [b I / G, (b+1) I / G) (MPNL is fixed-complexity,
// so static ranges are balanced).  An item is one vector (or, when P < 32 PT,
// `vpi` vectors of the same channel).  The range is walked channel segment by
// channel segment: the channel's tables are staged in shared memory once per
// segment; each warp owns a balanced sub-range of the segment and walks it in
// chunks of consecutive vectors.  A chunk's z' rows, guard thresholds,
// selection lists and (E_acc, corr) are contiguous in the workspace, so one
// lane fetches the next chunk with four TMA bulk copies (cp.async.bulk,
// completion on a per-buffer mbarrier) into the warp's second buffer while the
// warp traverses the current one.
// ===========================================================================
#ifndef MPNL_CHUNK_V
#define MPNL_CHUNK_V 8          // vectors per warp chunk (one bulk-copy group)
#endif
struct TravSmem {
  int tpo, tab, wbuf, bufsz, zs, thr, lst, eac, mbar, xs, ev, evn, total_bytes;   // floats / bytes
  int ck, cv;   // items and vectors per chunk
  int tab0, tabn;   // staged slice of the channel's table blob (per-layer float4 + r'' columns)
  // wpc: warp-per-channel mode, every warp stages its own channel's table slice
  __host__ __device__ TravSmem(int m, int n, int warps, int nvi, int list_bytes, bool wpc = false) {
    TableLayout tl(m, n);
    const int npp = (n + 1) / 2, n4 = (n + 3) & ~3;
    // chunk: up to MPNL_CHUNK_V vectors, at most ~2 KB per buffer (large
    // selection lists -> fewer vectors per chunk; occupancy is kept)
    const int bv = 16 * npp + 4 * n4 + list_bytes + 8;
    ck = MPNL_CHUNK_V / nvi;
    if (ck * nvi * bv > 2048) ck = 2048 / (nvi * bv);
    if (ck < 1) ck = 1;
    cv = ck * nvi;
    // per-warp chunk buffer (floats): z' row pairs | thresholds | lists |
    // (E_acc, corr) pairs from the even vector at or below the chunk start
    zs = 0;
    thr = zs + 4 * cv * npp;
    lst = thr + cv * n4;
    eac = lst + cv * list_bytes / 4;
    bufsz = eac + TableLayout::up4(2 * (cv + 2));
    int o = 0;
    tpo = o; o += TableLayout::up4((int)(sizeof(TreeParams) / 4));
    // Q^H and the shift are not read here: wide channels (whose fp64 Q^H is the
    // bulk of the blob) stage only the per-layer and r'' blocks; small ones keep
    // the whole blob (measured: C2 traversal 300 vs 306 us with the slice)
    tab0 = n > 16 ? tl.off_lay : 0;
    tabn = tl.total - tab0;
    tab = o; o += (wpc ? warps : 1) * tabn;
    wbuf = o; o += warps * 2 * bufsz;
    mbar = o; o += warps * 2 * 2;                  // u64 mbarrier per warp buffer
    xs = o; o += 2 * MPNL_XMAX * MPNL_PT_SMALL * MPNL_XS_STRIDE;   // u64 per-thread symbols
    ev = o; o += 4 * TRAV_EV_CAP;                  // int4 event buffer
    evn = o; o += 4;
    total_bytes = o * 4;
  }
};

// ---- TMA bulk copies (cp.async.bulk, completion on an mbarrier) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(void* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(void* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, void* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// issue the bulk copies of vectors gv0 .. gv0+nv-1 into the warp buffer `buf`
// (lane 0 only; the buffer's previous contents must be consumed).  Every
// source block is contiguous and 16-byte aligned; the (E_acc, corr) pairs are
// fetched from the even vector at or below gv0 (workspace padded for it).
template <int N>
__device__ __forceinline__ void trav_issue(const DetectArgs& a, const TravSmem& so, float* buf,
                                           void* bar, int gv0, int nv, int list_bytes) {
  constexpr int NPP = (N + 1) / 2, N4 = (N + 3) & ~3;
  const unsigned bz = nv * NPP * 16, bt = nv * N4 * 4, bl = nv * list_bytes;
  const int e0 = gv0 & ~1;
  const unsigned be = ((gv0 - e0 + nv) * 8 + 15) & ~15u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before async writes
  mbar_expect_tx(bar, bz + bt + bl + be);
  bulk_g2s(buf + so.zs, a.zq + (int64_t)gv0 * NPP, bz, bar);
  bulk_g2s(buf + so.thr, a.thrg + (int64_t)gv0 * N4, bt, bar);
  if (bl) bulk_g2s(buf + so.lst, a.lists + (int64_t)gv0 * list_bytes, bl, bar);
  bulk_g2s(buf + so.eac, a.vaux + e0, be, bar);
}

// VPI = false: one vector per item, its P paths in bpv batches of 32 PT paths
//              (every path of a lane is on the same vector);
// VPI = true : vpi = 32 PT / P vectors per item, one batch.
// SH: (non-VPI, PT = 2) lane l holds the sibling paths 2l, 2l + 1 of a batch
// (same top symbol: requires an even top-layer stride), sharing the top layer.
// ONEB: (SH, P == 32 PT) every vector is exactly one full batch: the path
// bookkeeping is compile-time (loop-invariant) and the lane's two paths are
// ordered with one compare instead of running top-3 inserts.
template <int N, int L, bool VPI, bool SH = false, bool ONEB = false, bool WPC = false>
__global__ void __launch_bounds__(TravCfg<N>::MAXT, TravCfg<N>::MINB)
traverse_kernel(const DetectArgs a, const TreeParams tparam) {
  constexpr int PT = TravCfg<N>::PT;
  constexpr int S = 32 * PT;
  extern __shared__ __align__(16) float sm[];
  const int nth = blockDim.x, nw = nth >> 5;
  const int nvi = VPI ? a.vpi : 1;                          // vectors per item
  // Warp-per-channel mode (a.wpc; channels with only a few vectors, e.g. one H
  // per vector as in the reference's own bench, cli.py:227-239): every warp
  // walks whole channels with its own table slot and no block barrier, instead
  // of the CTA staging one channel and splitting its vectors over the warps.
  // (a template parameter: the CTA-mode instances keep their instruction schedule)
  constexpr bool wpc = WPC;
  static_assert(!WPC || (!SH && !ONEB), "warp-per-channel mode: plain or VPI instances");
  const TravSmem so(a.m, N, nw, nvi, tparam.list_bytes, wpc);
  const TableLayout tl(a.m, N);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float INF = __int_as_float(0x7f800000);
  TreeParams& tp = *reinterpret_cast<TreeParams*>(sm + so.tpo);
  float* tabs = sm + so.tab + (wpc ? warp * so.tabn : 0);   // staged slice [tab0, total)
  float* tab = tabs - so.tab0;                               // virtual blob base
  float* wb0 = sm + so.wbuf + warp * 2 * so.bufsz;
  uint64_t* wbar = reinterpret_cast<uint64_t*>(sm + so.mbar) + 2 * warp;
  if (lane == 0) {
    mbar_init(wbar, 1);
    mbar_init(wbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned phase = 0u;   // parity bit per buffer
  int4* evb = reinterpret_cast<int4*>(sm + so.ev);
  int* evn = reinterpret_cast<int*>(sm + so.evn);
  {
    const int* s = reinterpret_cast<const int*>(&tparam);
    int* d = reinterpret_cast<int*>(&tp);
    for (int i = tid; i < (int)(sizeof(TreeParams) / 4); i += nth) d[i] = s[i];
    if (tid == 0) { evn[0] = 0; evn[1] = 0; evn[2] = 0; evn[3] = 0; }
  }
  const int P = tparam.n_paths;
  const int lbytes = tparam.list_bytes;
  static_assert(!ONEB || (SH && !VPI && TravCfg<N>::PT == 2), "ONEB needs sibling pairs");
  const int bpv = (VPI || ONEB) ? 1 : a.bpv;
  // paths are fixed per lane when one batch covers them: precompute the
  // expanded layers' symbols (float pair) / list indices once
  u64* xs = reinterpret_cast<u64*>(sm + so.xs) + tid;
  const bool use_xs = bpv == 1;
  if (use_xs) {
    constexpr int XM = N < MPNL_XMAX ? N : MPNL_XMAX;
#pragma unroll
    for (int t = 0; t < PT; ++t) {
      const int s = SH ? 2 * lane + t : t * 32 + lane;
      const int p = VPI ? s % P : s;
#pragma unroll
      for (int j = 0; j < XM; ++j) {
        const int pos = N - 1 - j;
        u64 x = 0ull;
        if (j < tparam.n_top && p < P) {
          const int e = tparam.e[pos];
          const int d = p / tparam.stride[pos];
          if (e == L * L) {
            const int dd = d % e;
            x = pk2(-(float)(dd / L), -(float)(dd % L));   // negated level indices
          } else {
            x = (u64)(unsigned)(tparam.list_off[pos] + d);
          }
        }
        xs[(j * PT + t) * MPNL_XS_STRIDE] = x;
      }
    }
  }
  const int V = (int)a.V;
  const int ipc = (V + nvi - 1) / nvi;                      // items per channel
  const int64_t I = a.n_ch * (int64_t)ipc;
  const int it_begin = (int)((int64_t)blockIdx.x * I / gridDim.x);
  const int it_end = (int)((int64_t)(blockIdx.x + 1) * I / gridDim.x);
  const TabPtrs T = tab_ptrs(tab, a.m, N);

#ifdef MPNL_SKEW_NS
  // co-resident CTAs (b, b + G/k, ...) start out of phase: their warps share
  // the SM sub-partitions and would otherwise hit the update-heavy top layers
  // and the latency-bound bottom layers in lockstep
  {
    int nsm = 148;
    const int slot = (int)(blockIdx.x / (unsigned)nsm);
    if (slot) __nanosleep((unsigned)(slot * MPNL_SKEW_NS));
  }
#endif
  if (wpc) __syncthreads();   // xs / tp ready (the CTA mode's first segment barrier does it)
  const int64_t wstep = (int64_t)gridDim.x * nw * ipc;   // wpc: this warp's channel stride, in items
  const int64_t wseg0 = ((int64_t)blockIdx.x * nw + warp) * ipc;
  const int seg_stop = wpc ? (int)I : it_end;
  for (int seg = wpc ? (int)min(wseg0, I) : it_begin; seg < seg_stop;) {
    const int c = seg / ipc;
    const int ibase = c * ipc, vbase = c * V;
    const int seg_end = wpc ? ibase + ipc : min(it_end, ibase + ipc);
    // warp w owns the balanced item range [wb, we) of the segment (the whole
    // channel in wpc mode), walked in chunks of so.ck items (contiguous vectors,
    // one bulk-copy group each); the first chunk's copies are issued before the
    // table staging (they overlap)
    const int wb = wpc ? seg : seg + (int)((int64_t)warp * (seg_end - seg) / nw);
    const int we = wpc ? seg_end : seg + (int)((int64_t)(warp + 1) * (seg_end - seg) / nw);
    const int nchunk = (we - wb + so.ck - 1) / so.ck;
    int k = 0;
    int ch = 0;
    if (ch < nchunk && lane == 0) {
      const int i0 = wb;
      const int i1 = min(we, i0 + so.ck);
      trav_issue<N>(a, so, wb0, wbar, vbase + (i0 - ibase) * nvi,
                    min((i1 - ibase) * nvi, V) - (i0 - ibase) * nvi, lbytes);
    }
    // previous segment's tables no longer in use (and xs / tp ready)
    if (wpc) __syncwarp(); else __syncthreads();
    {
      const float4* src = reinterpret_cast<const float4*>(a.tables + (int64_t)c * tl.total + so.tab0);
      float4* dst = reinterpret_cast<float4*>(tabs);
      for (int i = wpc ? lane : tid; i < so.tabn / 4; i += wpc ? 32 : nth) dst[i] = src[i];
    }
    if (wpc) __syncwarp(); else __syncthreads();
    for (; ch < nchunk; ++ch, k ^= 1) {
      if (ch + 1 < nchunk && lane == 0) {
        const int i0 = wb + (ch + 1) * so.ck;
        const int i1 = min(we, i0 + so.ck);
        trav_issue<N>(a, so, wb0 + (k ^ 1) * so.bufsz, wbar + (k ^ 1),
                      vbase + (i0 - ibase) * nvi, min((i1 - ibase) * nvi, V) - (i0 - ibase) * nvi,
                      lbytes);
      }
      mbar_wait(wbar + k, (phase >> k) & 1u);
      phase ^= 1u << k;
      const float* cbuf = wb0 + k * so.bufsz;
      const int ci0 = wb + ch * so.ck;
      const int ci1 = min(we, ci0 + so.ck);
      const int eo = (vbase + (ci0 - ibase) * nvi) & 1;   // (E_acc, corr) window offset
    for (int it = ci0; it < ci1; ++it) {
      const int jl = (it - ci0) * nvi;                      // vector offset in the chunk
      const float4* zs = reinterpret_cast<const float4*>(cbuf + so.zs) + jl * ((N + 1) / 2);
      const float* thr = cbuf + so.thr + jl * ((N + 3) & ~3);
      const float* weacc = cbuf + so.eac + 2 * (eo + jl);   // (E_acc, corr) pairs
      const uint8_t* lch = reinterpret_cast<const uint8_t*>(cbuf + so.lst) + jl * lbytes;
      const int jv = (it - ibase) * nvi;
      const int gbase = vbase + jv;
      const int vce = min(nvi, V - jv);

      Top3 run = {INF, INF, INF, 0xffffffffu, 0xffffffffu};
      float wbest = INF;   // warp-wide best so far of this vector
      // multi-batch: start with the batch holding the top layer's nearest point
      // (the SIC family), so the event filter has a good bound from the start;
      // the result does not depend on the batch order (total order on paths)
      int b0 = 0;
      if (!VPI && bpv > 1 && tp.e[N - 1] == L * L) {
        const float4 zt = zs[(N - 1) >> 1];
        const float ur = ((N - 1) & 1) ? zt.z : zt.x, ui = ((N - 1) & 1) ? zt.w : zt.y;
        float t0;
        const float kxt = T.lay4[N - 1].w;
        const int d0 = (int)(-slice_axis<L>(ur, kxt, t0)) * L + (int)(-slice_axis<L>(ui, kxt, t0));
        b0 = (d0 * tp.stride[N - 1]) / S;
      }
      for (int bi = 0; bi < bpv; ++bi) {
        const int b = (VPI || bpv == 1) ? 0 : (b0 + bi < bpv ? b0 + bi : b0 + bi - bpv);
        int vl[PT], pp[PT];
        int64_t gvl[PT];
        bool ok[PT];
#pragma unroll
        for (int t = 0; t < PT; ++t) {
          const int s = SH ? 2 * lane + t : t * 32 + lane;
          if (ONEB) {
            vl[t] = 0;
            pp[t] = s;
            ok[t] = true;
          } else if (!VPI) {
            vl[t] = 0;
            pp[t] = b * S + s;
            ok[t] = pp[t] < P;
          } else {
            vl[t] = s / P;
            pp[t] = s % P;
            ok[t] = vl[t] < vce;
          }
          if (!ok[t]) { vl[t] = 0; pp[t] = 0; }
          gvl[t] = vl[t];   // lists of the item's vectors in the warp buffer
        }
        float ped[PT], evp[PT];
        unsigned evm[PT];
        traverse_paths<N, L, PT, true, false, !VPI, SH>(T, zs, thr, lch, tp, lbytes, vl, gvl, pp, ped,
                                                    evm, evp, nullptr, nullptr, -1,
                                                    use_xs ? xs : nullptr);
        if (ONEB) {   // the lane's two paths, ordered (path 2l < 2l + 1)
          const bool sw = ped[1] < ped[0];
          run.m1 = sw ? ped[1] : ped[0];
          run.p1 = (unsigned)(sw ? pp[1] : pp[0]);
          run.m2 = sw ? ped[0] : ped[1];
          run.p2 = (unsigned)(sw ? pp[0] : pp[1]);
          wbest = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(run.m1)));
        } else if (!VPI) {   // running top-3; the event bound includes this batch's own best
#pragma unroll
          for (int t = 0; t < PT; ++t)
            if (ok[t]) top3_insert(run, ped[t], (unsigned)pp[t]);
          wbest = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(run.m1)));
        }
        // log paths with a marked decision whose prefix may still be competitive
#pragma unroll
        for (int t = 0; t < PT; ++t) {
          if (ok[t] && evm[t] != 0u) {
            const float bnd = (wbest == INF) ? INF : wbest + 2.f * ped_tol(wbest, weacc[0], N);
            if (evp[t] <= bnd) {
              const int4 e4 = make_int4(pp[t], (int)evm[t], gbase + vl[t], ev_node_w(evp[t]));
              const int idx = atomicAdd(evn, 1);
              if (idx < TRAV_EV_CAP) evb[idx] = e4;
              else log_event(a, e4);
            }
          }
        }
        if (!VPI) {
        } else if (P >= 32) {
          const int g = P >> 5;   // t-slots per vector
#pragma unroll
          for (int t0 = 0; t0 < PT; ++t0) {
            if (t0 % g) continue;
            Top3 x = {INF, INF, INF, 0xffffffffu, 0xffffffffu};
#pragma unroll
            for (int t = 0; t < PT; ++t)
              if (t >= t0 && t < t0 + g && ok[t]) top3_insert(x, ped[t], (unsigned)pp[t]);
            float b1, b2, b3;
            unsigned q1, q2;
            warp_top3(x, b1, q1, b2, q2, b3);
            const int j = t0 / g;
            if (lane == 0 && j < vce) {
              a.vres[gbase + j] = make_float4(b1, b2, b3, weacc[2 * j]);
              a.vpath[gbase + j] = make_int2((int)q1, (int)q2);
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < PT; ++t) {
            Top3 x = {INF, INF, INF, 0xffffffffu, 0xffffffffu};
            if (ok[t]) top3_insert(x, ped[t], (unsigned)pp[t]);
            float b1, b2, b3;
            unsigned q1, q2;
            group_top3(x, P, b1, q1, b2, q2, b3);
            const int j = (t * 32 + lane) / P;
            if ((lane % P) == 0 && j < vce) {
              a.vres[gbase + j] = make_float4(b1, b2, b3, weacc[2 * j]);
              a.vpath[gbase + j] = make_int2((int)q1, (int)q2);
            }
          }
        }
      }
      if (!VPI) {
        // b1 = wbest; the 2nd path and the 3rd metric only matter for a near-tie
        const unsigned k1 = __float_as_uint(wbest);
        unsigned q1;
        if (ONEB) {
          // lane l holds paths 2l, 2l + 1: the lowest lane holding the best
          // metric holds the lowest such path (no second reduction on the chain)
          const int wl = __ffs(__ballot_sync(0xffffffffu, __float_as_uint(run.m1) == k1)) - 1;
          q1 = __shfl_sync(0xffffffffu, run.p1, wl);
          if (lane == wl) top3_pop(run);
        } else {
          q1 = __reduce_min_sync(0xffffffffu,
                                 __float_as_uint(run.m1) == k1 ? run.p1 : 0xffffffffu);
          if (__float_as_uint(run.m1) == k1 && run.p1 == q1) top3_pop(run);
        }
        const float b2 = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(run.m1)));
        unsigned q2 = 0xffffffffu;
        float b3 = b2;
        if (b2 - wbest <= ped_tol(wbest, weacc[0], N) + ped_tol(b2, weacc[0], N)) {
          q2 = __reduce_min_sync(0xffffffffu,
                                 __float_as_uint(run.m1) == __float_as_uint(b2) ? run.p1 : 0xffffffffu);
          if (__float_as_uint(run.m1) == __float_as_uint(b2) && run.p1 == q2) top3_pop(run);
          b3 = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(run.m1)));
        }
        if (lane == 0) {
          a.vres[gbase] = make_float4(wbest, b2, b3, weacc[0]);
          a.vpath[gbase] = make_int2((int)q1, (int)q2);
        }
      }
    }
      __syncwarp();   // the chunk buffer is refilled by the next issue into it
    }
    if (wpc) {
      const int64_t nx = (int64_t)seg + wstep;
      seg = nx < (int64_t)seg_stop ? (int)nx : seg_stop;
    } else {
      seg = seg_end;
    }
  }
  // ---- flush the CTA's event buffer to the global log ----
  // A NODE event was logged against the vector's RUNNING best; every vector of
  // this CTA is finished now, so the event is first tested against the FINAL
  // bound -- the very test check_kernel applies before doing any work
  // (node_lim) -- and only the survivors reach the global log (C5/P1024: 2.0 ->
  // 0.8 events per vector).
  __syncthreads();
  const int n_ev = min(evn[0], TRAV_EV_CAP);
  for (int i0 = 0; i0 < n_ev; i0 += nth) {
    const int i = i0 + tid;
    bool keep = i < n_ev;
    if (keep) {
      const int4 e = evb[i];
      if (ev_is_node(e.w)) {
        keep = ev_node_evp(e.w) <= node_lim(__ldcg(a.vres + (unsigned)e.z), N);
        if (!keep) evb[i].y = 0;   // a logged NODE event always has a non-zero mask
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0 && bal) atomicAdd(evn + 2, __popc(bal));
  }
  __syncthreads();
  const int n_keep = evn[2];
  if (tid == 0) {
    evn[1] = n_keep ? atomicAdd(a.counters + 1, n_keep) : 0;
    if (a.stats && n_keep) atomicAdd(a.stats, n_keep);
  }
  __syncthreads();
  const int base = evn[1];
  for (int i0 = 0; i0 < n_ev; i0 += nth) {
    const int i = i0 + tid;
    int4 e = make_int4(0, 0, 0, 0);
    bool keep = i < n_ev;
    if (keep) {
      e = evb[i];
      keep = !(ev_is_node(e.w) && e.y == 0);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    int slot = 0;
    if (lane == 0 && bal) slot = atomicAdd(evn + 3, __popc(bal));
    slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(bal & ((1u << lane) - 1u));
    if (keep) {
      if (base + slot < a.ev_cap) a.events[base + slot] = e;
      else send_to_fp64(a, (int64_t)(unsigned)e.z, 3);
    }
  }
}

// ===========================================================================
// K4a: winners — one thread per vector re-traces its best path
// ===========================================================================
#define EV_TIE 2

template <int N, int L>
__global__ void __launch_bounds__(128)
verify_kernel(const DetectArgs a, const TreeParams tparam, int unused) {
  (void)unused;
  constexpr int NPP = (N + 1) / 2;
  constexpr int TW = N + N * NPP;   // float4 of (lay, rcol) per channel
  __shared__ TreeParams tp;
  __shared__ float4 tabs[2][TW];    // the CTA's (at most two) channels' traversal tables
  const int m = a.m;
  const TableLayout tl(m, N);
  const int64_t B = a.n_ch * a.V;
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t c0 = g0 / a.V, c1 = min(g0 + (int64_t)blockDim.x, B) - 1;
  const int nst = (c1 / a.V - c0) < 2 ? (int)(c1 / a.V - c0) + 1 : 0;   // staged channels
  {
    const int* s = reinterpret_cast<const int*>(&tparam);
    int* d = reinterpret_cast<int*>(&tp);
    for (int i = threadIdx.x; i < (int)(sizeof(TreeParams) / 4); i += blockDim.x) d[i] = s[i];
    for (int i = threadIdx.x; i < nst * TW; i += blockDim.x) {
      const int j = i / TW, o = i - j * TW;
      tabs[j][o] = reinterpret_cast<const float4*>(a.tables + (c0 + j) * (int64_t)tl.total +
                                                   tl.off_lay)[o];
    }
  }
  // the CTA's z' rows (contiguous) and its output labels go through shared
  // memory: coalesced 16-byte loads in, 4-byte stores out
  // (N <= 16; larger N reads its rows directly: static shared memory limit)
  constexpr bool STZ = N <= 16;
  __shared__ float4 zsh[STZ ? 128 * NPP : 1];
  __shared__ __align__(16) uint8_t osh[128 * N];
  const int nvb = (int)min((int64_t)blockDim.x, B - g0);
  if (STZ)
    for (int i = threadIdx.x; i < nvb * NPP; i += blockDim.x) zsh[i] = a.zq[g0 * NPP + i];
  __syncthreads();
  const int h = (L == 2) ? 1 : (L == 4 ? 2 : 3);
  const int64_t gv = g0 + threadIdx.x;
  const bool live = gv < B;
  if (live) {
  const int64_t c = gv / a.V;
  TabPtrs T;
  if (c - c0 < nst) {
    T.lay4 = tabs[c - c0];
    T.rcol = reinterpret_cast<const float*>(tabs[c - c0] + N);
  } else {
    T = tab_ptrs(a.tables + c * (int64_t)tl.total, m, N);
  }
  float4 zreg[STZ ? 1 : NPP];
  if (!STZ) {
#pragma unroll
    for (int q = 0; q < (STZ ? 1 : NPP); ++q) zreg[q] = a.zq[gv * NPP + q];
  }
  const float4* zl = STZ ? zsh + threadIdx.x * NPP : zreg;
  const uint8_t* vlist = a.lists + gv * tp.list_bytes;
  const float4 res = a.vres[gv];
  const int2 pth = a.vpath[gv];
  int lab[N];
  float pre[N];
  {
    const int vl[1] = {0}, pp[1] = {pth.x};
    const int64_t gvl[1] = {0};
    float pd[1], ep[1];
    unsigned em[1];
    traverse_paths<N, L, 1, false, true>(T, zl, nullptr, vlist, tp, 0, vl, gvl, pp, pd, em, ep,
                                         lab, pre, 0);
  }
  if (res.y - res.x <= ped_tol(res.x, res.w, N) + ped_tol(res.y, res.w, N)) {
    // near-tie of the two best paths: a three-way tie goes to the fp64 kernel,
    // a two-way tie is settled in fp64 by the check kernel (which may rewrite
    // this vector's outputs with the second path)
    // (pth.y < 0: the traversal judged it no near-tie, a rounding-level
    // disagreement of the two evaluations of the test -> fp64, conservatively)
    if (pth.y < 0 || res.z - res.x <= ped_tol(res.x, res.w, N) + ped_tol(res.z, res.w, N))
      send_to_fp64(a, gv, 0);
    else
      log_event(a, make_int4(pth.x, pth.y, (int)gv, EV_TIE));
  }
  const float corr = a.metric_offset ? a.vaux[gv].y : 0.f;
  const int32_t* pc = a.perm + c * N;
  uint8_t* out = osh + threadIdx.x * N;
#pragma unroll
  for (int pos = 0; pos < N; ++pos) {
    const int ir = lab[pos] >> 3, ii = lab[pos] & 7;
    out[pc[pos]] = (uint8_t)((gray_code(ir) << h) | gray_code(ii));
  }
  a.metric[gv] = res.x + corr;
  }
  __syncthreads();
  uint8_t* dst = a.hard + g0 * N;
  const int nb = nvb * N;
  if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
    for (int i = threadIdx.x; i < nb / 4; i += blockDim.x)
      reinterpret_cast<unsigned*>(dst)[i] = reinterpret_cast<const unsigned*>(osh)[i];
    for (int i = (nb & ~3) + threadIdx.x; i < nb; i += blockDim.x) dst[i] = osh[i];
  } else {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) dst[i] = osh[i];
  }
}

// ===========================================================================
// K4b: event checks — one warp per logged event
//   NODE: re-decide each marked, competitive decision in fp64
//   CUT : re-select a near-tied partial-layer cut in fp64
//   TIE : settle a two-way near-tie of the best metrics in fp64
// The fp32 re-trace is warp-cooperative (lane = tree row) with exactly the
// traversal's per-row fma sequence, so it reproduces the traversal bit for bit.
// ===========================================================================
// fp32 re-trace of path p with lanes = rows; labw[pos] / prew[pos] (smem) for pos >= stop.
// T / zrow may point to global or (staged) shared memory.
// (An early exit at the first layer whose prefix exceeds the event bound was measured
// slower: the exit test in every unrolled layer costs more than the layers it skips.)
template <int N, int L>
__device__ __forceinline__ void warp_retrace(const TabPtrs& T, const float4* zrow,
                                             const uint8_t* vlist, const TreeParams& tp, int p,
                                             int stop, int* labw, float* prew) {
  constexpr int NPP = (N + 1) / 2;
  constexpr int XM = N < MPNL_XMAX ? N : MPNL_XMAX;
  const int lane = threadIdx.x & 31;
  float ar = 0.f, ai = 0.f;
  if (lane < N) {
    const float2 zf = reinterpret_cast<const float2*>(zrow)[lane];
    ar = zf.x;
    ai = zf.y;
  }
  using PA = Ped<ped_scalar<N, L>()>;
  typename PA::T ped2 = PA::zero();
  const int top_lo = N - tp.n_top;
#pragma unroll
  for (int pos = N - 1; pos >= 0; --pos) {
    if (pos < stop) break;
    const float4 ly = T.lay4[pos];
    const float2 rr = (lane < pos) ? rcol_at(T.rcol, NPP, lane, pos) : make_float2(0.f, 0.f);
    float fr, fi;
    if (pos >= N - XM && pos >= top_lo) {
      int ir, ii;
      expanded_symbol<L>(tp, pos, p, vlist, ir, ii);
      fr = (float)ir;
      fi = (float)ii;
    } else {
      float tr, ti;
      const float sr = -slice_axis<L>(ar, ly.w, tr);   // level indices (positive form)
      const float si = -slice_axis<L>(ai, ly.w, ti);
      fr = __shfl_sync(0xffffffffu, sr, pos);
      fi = __shfl_sync(0xffffffffu, si, pos);
    }
    const float ur = __shfl_sync(0xffffffffu, ar, pos), ui = __shfl_sync(0xffffffffu, ai, pos);
    if (lane == 0) {
      labw[pos] = (int)fr * 8 + (int)fi;
      prew[pos] = PA::value(ped2);
    }
    if (pos == stop) break;
    const float er = __fmaf_rn(ly.y, fr, ur);
    const float ei = __fmaf_rn(ly.y, fi, ui);
    const u64 e2 = pk2(er, ei);
    ped2 = PA::add(e2, ped2);
    if (lane < pos) {
      ar = __fmaf_rn(rr.x, fr, ar);
      ar = __fmaf_rn(rr.y, -fi, ar);
      ai = __fmaf_rn(rr.x, fi, ai);
      ai = __fmaf_rn(rr.y, fr, ai);
    }
  }
  __syncwarp();
}

// fp64 rotation z_k = (Q^H y)_k for lane k < n (sequential over the receive
// rows; the channel's transposed Q^H from its table blob, coalesced over k;
// y_r broadcast by shuffles from the lane that loaded it).
__device__ __forceinline__ void warp_z_f64(const DetectArgs& a, const float* tab, int64_t gv,
                                           int n, double& zr, double& zi) {
  const int lane = threadIdx.x & 31;
  const int m = a.m;
  const double2* qt = reinterpret_cast<const double2*>(tab + TableLayout(m, n).off_qh);
  double y0r = 0.0, y0i = 0.0, y1r = 0.0, y1i = 0.0;   // y_lane, y_{lane+32}
  if (a.y_f64) {
    const double2* yp = reinterpret_cast<const double2*>(a.y) + gv * m;
    if (lane < m) { const double2 v = yp[lane]; y0r = v.x; y0i = v.y; }
    if (lane + 32 < m) { const double2 v = yp[lane + 32]; y1r = v.x; y1i = v.y; }
  } else {
    const float2* yp = reinterpret_cast<const float2*>(a.y) + gv * m;
    if (lane < m) { const float2 v = yp[lane]; y0r = v.x; y0i = v.y; }
    if (lane + 32 < m) { const float2 v = yp[lane + 32]; y1r = v.x; y1i = v.y; }
  }
  const int k = lane < n ? lane : n - 1;
  zr = 0.0;
  zi = 0.0;
#pragma unroll 8
  for (int r = 0; r < m; ++r) {
    const double2 q = qt[r * n + k];
    const double yr = __shfl_sync(0xffffffffu, r < 32 ? y0r : y1r, r & 31);
    const double yi = __shfl_sync(0xffffffffu, r < 32 ? y0i : y1i, r & 31);
    zr = fma(q.x, yr, fma(-q.y, yi, zr));
    zi = fma(q.x, yi, fma(q.y, yr, zi));
  }
}

// One row of the fp64 rotation, z_k = (Q^H y)_k, with the M products spread over the
// lanes (lane = receive row) and a butterfly sum: every lane gets the same value.  An
// event check needs only the marked layer's row: one load round trip and ~45
// instructions instead of the M sequential steps of warp_z_f64.
__device__ __forceinline__ void warp_zrow_f64(const DetectArgs& a, const float* tab, int64_t gv,
                                              int n, int k, double& zr, double& zi) {
  const int lane = threadIdx.x & 31;
  const int m = a.m;
  const double2* qt = reinterpret_cast<const double2*>(tab + TableLayout(m, n).off_qh);
  double sr = 0.0, si = 0.0;
  for (int r = lane; r < m; r += 32) {
    double yr, yi;
    if (a.y_f64) {
      const double2 v = reinterpret_cast<const double2*>(a.y)[gv * m + r];
      yr = v.x; yi = v.y;
    } else {
      const float2 v = reinterpret_cast<const float2*>(a.y)[gv * m + r];
      yr = v.x; yi = v.y;
    }
    const double2 q = qt[r * n + k];
    sr = fma(q.x, yr, fma(-q.y, yi, sr));
    si = fma(q.x, yi, fma(q.y, yr, si));
  }
  zr = warp_sum_d(sr);
  zi = warp_sum_d(si);
}

// fp64 centre of layer pos for the path whose level indices above pos are labw (smem),
// from that layer's rotated value (zp_r, zp_i) alone
__device__ __forceinline__ void warp_centre_f64_row(const DetectArgs& a, int64_t c, int n, int L,
                                                    int pos, const int* labw, double zp_r,
                                                    double zp_i, double& cr, double& ci) {
  const int lane = threadIdx.x & 31;
  const double* R = reinterpret_cast<const double*>(a.r64 + (c * n + pos) * (int64_t)n);
  double sr_ = 0.0, si_ = 0.0;
  const int j = pos + 1 + lane;
  if (j < n) {
    const double sr = level_value_rt(labw[j] >> 3, L), si = level_value_rt(labw[j] & 7, L);
    const double rr = R[2 * j], ri = R[2 * j + 1];
    sr_ = rr * sr - ri * si;
    si_ = rr * si + ri * sr;
  }
  sr_ = warp_sum_d(sr_);
  si_ = warp_sum_d(si_);
  const double rpp = R[2 * pos];
  cr = (zp_r - sr_) / rpp;
  ci = (zp_i - si_) / rpp;
}

// fp64 centre of layer pos for the path whose level indices above pos are labw
// (smem); zr/zi = this lane's fp64 rotation (warp_z_f64)
__device__ __forceinline__ void warp_centre_f64(const DetectArgs& a, int64_t c, int n, int L,
                                                int pos, const int* labw, double zr, double zi,
                                                double& cr, double& ci) {
  const int lane = threadIdx.x & 31;
  const double nrm = qam_norm_d(L);
  const double* R = reinterpret_cast<const double*>(a.r64 + (c * n + pos) * (int64_t)n);
  double sr_ = 0.0, si_ = 0.0;
  const int j = pos + 1 + lane;
  if (j < n) {
    const double sr = level_value_rt(labw[j] >> 3, L), si = level_value_rt(labw[j] & 7, L);
    const double rr = R[2 * j], ri = R[2 * j + 1];
    sr_ = rr * sr - ri * si;
    si_ = rr * si + ri * sr;
  }
  sr_ = warp_sum_d(sr_);
  si_ = warp_sum_d(si_);
  const double zp_r = __shfl_sync(0xffffffffu, zr, pos), zp_i = __shfl_sync(0xffffffffu, zi, pos);
  const double rpp = R[2 * pos];
  cr = (zp_r - sr_) / rpp;
  ci = (zp_i - si_) / rpp;
}

// fp64 PED ||z - R x||^2 of the path with level indices labw (smem), lanes = rows
__device__ __forceinline__ double warp_ped_f64(const DetectArgs& a, int64_t c, int n, int L,
                                               const int* labw, double zr, double zi) {
  const int lane = threadIdx.x & 31;
  const double nrm = qam_norm_d(L);
  double acc = 0.0;
  if (lane < n) {
    const double2* R = a.r64 + (c * n + lane) * (int64_t)n;
#pragma unroll 4
    for (int j = lane; j < n; ++j) {
      const double sr = level_value_rt(labw[j] >> 3, L), si = level_value_rt(labw[j] & 7, L);
      const double2 r = R[j];
      zr -= r.x * sr - r.y * si;
      zi -= r.x * si + r.y * sr;
    }
    acc = zr * zr + zi * zi;
  }
  return warp_sum_d(acc);
}

// The reference's path from layer pos down, in fp64: prefix symbols labw[j > pos],
// the fp64 decision (ir0, ii0) at pos, exact SIC below.  Returns its fp64 PED.
// Lanes = rows; zr/zi = this lane's fp64 rotation.
__device__ __forceinline__ double warp_sic_f64(const DetectArgs& a, int64_t c, int n, int L,
                                               int pos, const int* labw, int ir0, int ii0,
                                               double zr, double zi) {
  const int lane = threadIdx.x & 31;
  const double nrm = qam_norm_d(L);
  const double2* R = a.r64 + c * (int64_t)n * n;
  if (lane < n) {
    // interference of the prefix symbols (j > pos); rows above pos also add
    // their own symbol and become prefix residuals
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
    const double sr = level_value_rt(ir, L), si = level_value_rt(ii, L);
    if (lane <= q) {
      const double2 r = R[lane * n + q];
      zr -= r.x * sr - r.y * si;
      zi -= r.x * si + r.y * sr;
    }
    if (lane == q) ped += zr * zr + zi * zi;
  }
  return warp_sum_d(ped);
}

// K4b event checks: one warp per event, events strided over all warps.  Each
// warp double-buffers its events' traversal tables (lay + r'' columns, one
// contiguous block of the channel's blob) and z' rows in shared memory with
// cp.async, so the next event's fetch overlaps this event's re-trace.
#define CHECK_WARPS 4
template <int N>
struct CheckSmem {
  static constexpr int NPP = (N + 1) / 2;
  static constexpr int TW = N + N * NPP;   // float4: lay | rcol
  float4 tab[CHECK_WARPS][2][TW];
  float4 z[CHECK_WARPS][2][NPP];
  int labs[CHECK_WARPS][2][MPNL_MAX_N];
  float pres[CHECK_WARPS][MPNL_MAX_N];
  TreeParams tp;
};

template <int N>
__device__ __forceinline__ void check_fetch(const DetectArgs& a, const TableLayout& tl, int4 e4,
                                            float4* tb, float4* zb, int lane) {
  constexpr int NPP = (N + 1) / 2, TW = N + N * NPP;
  const int64_t gv = (int64_t)(unsigned)e4.z;
  const int64_t c = gv / a.V;
  const float4* src = reinterpret_cast<const float4*>(a.tables + c * (int64_t)tl.total + tl.off_lay);
  for (int i = lane; i < TW; i += 32) cp_async16(tb + i, src + i);
  if (lane < NPP) cp_async16(zb + lane, a.zq + gv * NPP + lane);
  cp_async_commit();
}

template <int N, int L>
__global__ void __launch_bounds__(32 * CHECK_WARPS)
check_kernel(const DetectArgs a, const TreeParams tparam, int unused) {
  (void)unused;
  extern __shared__ __align__(16) uint8_t csm_raw[];
  CheckSmem<N>& S = *reinterpret_cast<CheckSmem<N>*>(csm_raw);
  TreeParams& tp = S.tp;
  {
    const int* s = reinterpret_cast<const int*>(&tparam);
    int* d = reinterpret_cast<int*>(&tp);
    for (int i = threadIdx.x; i < (int)(sizeof(TreeParams) / 4); i += blockDim.x) d[i] = s[i];
  }
  __syncthreads();
  const int m = a.m;
  const TableLayout tl(m, N);
  const int h = (L == 2) ? 1 : (L == 4 ? 2 : 3);
  const double nrm = qam_norm_d(L);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* lab = S.labs[warp][0];
  int* lab2 = S.labs[warp][1];
  float* pre = S.pres[warp];
  const int nev = min(a.counters[1], a.ev_cap);
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  int i = blockIdx.x * (blockDim.x >> 5) + warp;
  int k = 0;
  int4 e4 = make_int4(0, 0, 0, 0);
  if (i < nev) {
    e4 = a.events[i];
    check_fetch<N>(a, tl, e4, S.tab[warp][0], S.z[warp][0], lane);
  }
  for (; i < nev; i += nwarps, k ^= 1) {
    int4 en = make_int4(0, 0, 0, 0);
    if (i + nwarps < nev) {
      en = a.events[i + nwarps];
      check_fetch<N>(a, tl, en, S.tab[warp][k ^ 1], S.z[warp][k ^ 1], lane);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int64_t gv = (int64_t)(unsigned)e4.z;
    if (!a.vflag[gv]) {
      const int64_t c = gv / a.V;
      const float* tab = a.tables + c * (int64_t)tl.total;
      TabPtrs T;
      T.lay4 = S.tab[warp][k];
      T.rcol = reinterpret_cast<const float*>(S.tab[warp][k] + N);
      const float4* zrow = S.z[warp][k];
      const uint8_t* vlist = a.lists + gv * tp.list_bytes;
      const float4 res = a.vres[gv];
      const float lim = node_lim(res, N);
      if (ev_is_node(e4.w)) {
        // every marked layer's prefix is >= evp: nothing can compete, no re-trace
        if (ev_node_evp(e4.w) <= lim) {
          const unsigned mask = (unsigned)e4.y;
          const int lowest = __ffs(mask) - 1;
          warp_retrace<N, L>(T, zrow, vlist, tp, e4.x, lowest, lab, pre);
          // marked layers from the top down; prefixes only grow on the way down
          for (unsigned mm = mask; mm;) {
            const int pos = 31 - __clz(mm);
            mm &= ~(1u << pos);
            if (pre[pos] > lim) break;
            if (a.stats && lane == 0) atomicAdd(a.stats + 1, 1);
            double cr, ci, zpr, zpi;
            warp_zrow_f64(a, tab, gv, N, pos, zpr, zpi);   // only this layer's row of Q^H y
            warp_centre_f64_row(a, c, N, L, pos, lab, zpr, zpi, cr, ci);
            const int ir = nearest_level_f64(cr, L, nrm), ii = nearest_level_f64(ci, L, nrm);
            if (ir * 8 + ii != lab[pos]) {
              // the reference takes the other branch here.  Our fp32 path is then
              // a candidate the reference lacks: harmless unless it is one of our
              // two best.  The reference's path instead: harmless unless its exact
              // metric could beat our winner.
              const int2 pth = a.vpath[gv];
              bool bad = e4.x == pth.x || e4.x == pth.y;
              if (!bad) {
                double zr, zi;
                warp_z_f64(a, tab, gv, N, zr, zi);   // the continuation needs every row
                const double malt = warp_sic_f64(a, c, N, L, pos, lab, ir, ii, zr, zi);
                bad = malt <= (double)lim;
              }
              if (bad && lane == 0) send_to_fp64(a, gv, 2);
              break;
            }
          }
        }
      } else if (e4.w == EV_CUT) {
        const int pos = e4.y;
        if (pos < N - 1) warp_retrace<N, L>(T, zrow, vlist, tp, e4.x, pos + 1, lab, pre);
        const float prefix = (pos < N - 1) ? pre[pos + 1] : 0.f;   // <= PED prefix at pos
        if (prefix <= lim) {
          if (a.stats && lane == 0) atomicAdd(a.stats + 1, 1);
          double zpr, zpi, cr, ci;
          warp_zrow_f64(a, tab, gv, N, pos, zpr, zpi);
          warp_centre_f64_row(a, c, N, L, pos, lab, zpr, zpi, cr, ci);
          if (lane == 0) {
            const int e = tp.e[pos];
            const unsigned long long m64 = nearest_set_f64(cr, ci, L, nrm, e);
            const int par = e4.x / tp.stride[pos + 1];
            const uint8_t* lst = vlist + tp.list_off[pos] + par * e;
            unsigned long long m32 = 0ull;
            for (int r = 0; r < e; ++r) m32 |= 1ull << ((lst[r] >> 3) * L + (lst[r] & 7));
            if (m32 != m64) send_to_fp64(a, gv, 2);
          }
        }
      } else {   // EV_TIE: fp64 metrics of the two best paths
        if (a.stats && lane == 0) atomicAdd(a.stats + 2, 1);
        warp_retrace<N, L>(T, zrow, vlist, tp, e4.x, 0, lab, pre);
        warp_retrace<N, L>(T, zrow, vlist, tp, e4.y, 0, lab2, pre);
        double zr, zi;
        warp_z_f64(a, tab, gv, N, zr, zi);
        const double m1 = warp_ped_f64(a, c, N, L, lab, zr, zi);
        const double m2 = warp_ped_f64(a, c, N, L, lab2, zr, zi);
        if (fabs(m1 - m2) <= 1e-12 * fmax(m1, m2)) {
          if (lane == 0) send_to_fp64(a, gv, 1);   // tie at fp64 level: exact total order
        } else if (m2 < m1) {
          // the second path wins: rewrite labels and metric (fp32 value of that path)
          const int32_t* pc = a.perm + c * N;
          if (lane < N) {
            const int ir = lab2[lane] >> 3, ii = lab2[lane] & 7;
            a.hard[gv * N + pc[lane]] = (uint8_t)((gray_code(ir) << h) | gray_code(ii));
          }
          if (lane == 0) a.metric[gv] = a.metric[gv] - res.x + res.y;
        }
      }
    }
    __syncwarp();   // this buffer is refilled by the fetch two events ahead
    e4 = en;
  }
}

}  // namespace mpnl
