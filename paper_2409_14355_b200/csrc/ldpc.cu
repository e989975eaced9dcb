// LDPC stage after detection: the reference's
// normalized min-sum decoder, systematic encoder, syndrome and the
// shortening / puncturing rate match (pkg/src/mpnlsim/fec.py:136-220, 262-326).
//
// Decoder (fec.py:156-220), flooding schedule, fp64, bit-identical to the
// reference: per word, with total = llr and m_cv = 0 to start,
//   loop: hard = total < 0; converged if every check's parity is 0; stop
//         after max_iter updates.  Update: for each check, over its edges e
//         (variable v(e)), m_vc = total[v] - m_cv[e]; par = xor(m_vc < 0);
//         first argmin / min1 / min2 of |m_vc|;
//         m_cv[e] = +-(alpha * (e == argmin ? min2 : min1)), sign par ^ (m_vc < 0);
//         then total[v] = llr[v] + sum of m_cv over v's padded edge row in
//         numpy's add.reduce order (sequential under 8 terms, 8-way pairwise
//         blocks from 8 on), with explicit _rn intrinsics (no FMA contraction).
// m_vc is not stored: it is re-formed from total and the previous m_cv, which
// is the reference's own `total[check_vars] - m_cv` (fec.py:214).
//
// Layout: one CTA per codeword (grid-stride over the batch), the graph
// (uint16 check->variable and variable->edge tables), m_cv, total and the
// channel LLRs of the word in shared memory; thread per check, then thread
// per variable.  The rate match is fused into the LLR load: mother position
// [0,k_tb) <- llr_tx[0,k_tb), [k_tb,k) <- shortened_llr (known zeros),
// [k,k+p) <- llr_tx[k_tb,n_tx), [k+p,n) <- 0 (punctured), p = n_tx - k_tb.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/mpnl_b200.h"

namespace {

constexpr uint16_t kPad = 0xFFFF;
constexpr int kDecThreads = 256;

struct DecLayout {   // dynamic shared memory (bytes)
  int mcv, tot, llr, cv, ve, total;
  DecLayout(int m, int n, int dc, int dv) {
    int o = 0;
    mcv = o; o += 8 * m * dc;
    tot = o; o += 8 * n;
    llr = o; o += 8 * n;
    cv = o; o += 2 * m * dc;
    ve = o; o += 2 * n * dv;
    total = (o + 15) & ~15;
  }
};

__device__ __forceinline__ double edge_val(const double* mcv, const uint16_t* ve, int i) {
  const uint16_t e = ve[i];
  return e == kPad ? 0.0 : mcv[e];
}

// numpy add.reduce over one contiguous float64 row of dv terms (padded with 0)
__device__ __forceinline__ double np_row_sum(const double* mcv, const uint16_t* ve, int dv) {
  if (dv < 8) {
    double s = 0.0;
    for (int j = 0; j < dv; ++j) s = __dadd_rn(s, edge_val(mcv, ve, j));
    return s;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = edge_val(mcv, ve, j);
  int i = 8;
  for (; i + 8 <= dv; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], edge_val(mcv, ve, i + j));
  }
  double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < dv; ++i) s = __dadd_rn(s, edge_val(mcv, ve, i));
  return __dadd_rn(0.0, s);
}

__global__ void __launch_bounds__(kDecThreads)
ldpc_decode_kernel(const uint16_t* __restrict__ g_cv, const uint16_t* __restrict__ g_ve, int m,
                   int n, int dc, int dv, const double* __restrict__ llr_tx, int64_t n_words,
                   int n_tx, int k_tb, int max_iter, double alpha, double shortened,
                   uint8_t* __restrict__ info_out, uint8_t* __restrict__ conv_out,
                   int32_t* __restrict__ iters_out, int32_t* __restrict__ n_nonfinite,
                   DecLayout lo) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* mcv = reinterpret_cast<double*>(sm + lo.mcv);
  double* tot = reinterpret_cast<double*>(sm + lo.tot);
  double* llr = reinterpret_cast<double*>(sm + lo.llr);
  uint16_t* cv = reinterpret_cast<uint16_t*>(sm + lo.cv);
  uint16_t* ve = reinterpret_cast<uint16_t*>(sm + lo.ve);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int k = n - m, p = n_tx - k_tb;
  for (int i = tid; i < m * dc; i += nt) cv[i] = g_cv[i];
  for (int i = tid; i < n * dv; i += nt) ve[i] = g_ve[i];
  for (int64_t w = blockIdx.x; w < n_words; w += gridDim.x) {
    const double* lt = llr_tx + w * (int64_t)n_tx;
    int bad = 0;
    for (int v = tid; v < n; v += nt) {
      double x;
      if (v < k_tb) x = lt[v];
      else if (v < k) x = shortened;
      else if (v < k + p) x = lt[k_tb + (v - k)];
      else x = 0.0;
      bad |= !isfinite(x);
      llr[v] = x;
      tot[v] = x;
    }
    for (int i = tid; i < m * dc; i += nt) mcv[i] = 0.0;
    if (__syncthreads_or(bad) && tid == 0 && n_nonfinite) atomicAdd(n_nonfinite, 1);
    int it = 0, converged = 0;
    for (;;) {
      // ---- syndrome of the current hard decision + check-node update ----
      int synd = 0;
      for (int r = tid; r < m; r += nt) {
        const uint16_t* row = cv + r * dc;
        double* mr = mcv + r * dc;
        double min1 = INFINITY, min2 = INFINITY;
        int amin = 0, par = 0, sp = 0;
        unsigned negm = 0u;
        for (int s = 0; s < dc; ++s) {
          const uint16_t v = row[s];
          if (v == kPad) continue;   // padded slot: |m_vc| = inf, not negative
          const double t = tot[v];
          sp ^= (t < 0.0);
          const double x = __dsub_rn(t, mr[s]);
          const int ng = x < 0.0;
          negm |= (unsigned)ng << s;
          par ^= ng;
          const double a = fabs(x);
          if (a < min1) { min2 = min1; min1 = a; amin = s; }
          else if (a < min2) { min2 = a; }
        }
        synd |= sp;
        const double a1 = __dmul_rn(alpha, min1), a2 = __dmul_rn(alpha, min2);
        for (int s = 0; s < dc; ++s) {
          if (row[s] == kPad) continue;
          const double e = s == amin ? a2 : a1;
          mr[s] = (par ^ (int)((negm >> s) & 1u)) ? -e : e;
        }
      }
      if (!__syncthreads_or(synd)) { converged = 1; break; }
      if (it == max_iter) break;
      // ---- variable-node update ----
      for (int v = tid; v < n; v += nt)
        tot[v] = __dadd_rn(llr[v], np_row_sum(mcv, ve + v * dv, dv));
      __syncthreads();
      ++it;
    }
    uint8_t* out = info_out + w * (int64_t)k_tb;
    for (int v = tid; v < k_tb; v += nt) out[v] = tot[v] < 0.0 ? 1 : 0;
    if (tid == 0) {
      conv_out[w] = (uint8_t)converged;
      if (iters_out) iters_out[w] = it;
    }
    __syncthreads();   // smem reused by the next word
  }
}

// ---------------------------------------------------------------------------
// Fast path for small-degree codes (the default code: check degree <= 6,
// variable degree <= 3): one thread owns one check and up to two variables for
// the whole batch, so the graph lives in registers as shared-memory byte
// offsets.  The owning thread keeps its check's previous messages COMPRESSED
// in registers — (alpha*min1, alpha*min2) and a meta word (argmin slot, sign
// parity, sign mask), from which each m_cv[e] re-forms exactly (a select and
// a sign flip of the same doubles) for m_vc = total - m_cv_old — and stores
// the full messages in shared memory for the variable phase.  Same
// arithmetic, same order as the generic kernel: bit-identical.
// ---------------------------------------------------------------------------
constexpr int kFastDC = 6, kFastDV = 3, kFastThreads = 672;

__device__ __forceinline__ double msg_of(double a1, double a2, unsigned meta, int s) {
  // meta: bits 0-2 argmin slot, bit 3 sign parity, bits 4.. per-slot sign
  const double e = (int)(meta & 7u) == s ? a2 : a1;
  return (((meta >> 3) ^ (meta >> (4 + s))) & 1u) ? -e : e;
}

__device__ __forceinline__ double lds_f64(const unsigned char* base, int off) {
  return *reinterpret_cast<const double*>(base + off);
}

__global__ void __launch_bounds__(kFastThreads, 2)
ldpc_decode_fast_kernel(const uint16_t* __restrict__ g_cv, const uint16_t* __restrict__ g_ve,
                        int m, int n, int dc, int dv, const double* __restrict__ llr_tx,
                        int64_t n_words, int n_tx, int k_tb, int max_iter, double alpha,
                        double shortened, uint8_t* __restrict__ info_out,
                        uint8_t* __restrict__ conv_out, int32_t* __restrict__ iters_out,
                        int32_t* __restrict__ n_nonfinite) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned char* mcv_b = sm;                                   // m * dc doubles
  double* tot = reinterpret_cast<double*>(sm + 8 * m * dc);    // n
  double* llr = tot + n;                                       // n
  const unsigned char* tot_b = reinterpret_cast<const unsigned char*>(tot);
  const int tid = threadIdx.x;
  const int k = n - m, p = n_tx - k_tb;
  // graph of this thread's check (r = tid) and variables (tid, tid + blockDim)
  // as byte offsets into tot / mcv (-1 = padded slot)
  const bool own_c = tid < m;
  int toff[kFastDC];
#pragma unroll
  for (int s = 0; s < kFastDC; ++s) {
    const uint16_t v = (own_c && s < dc) ? g_cv[tid * dc + s] : kPad;
    toff[s] = v == kPad ? -1 : 8 * (int)v;
  }
  int eoff[2][kFastDV];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int v = tid + j * kFastThreads;
#pragma unroll
    for (int d = 0; d < kFastDV; ++d) {
      const uint16_t e = (v < n && d < dv) ? g_ve[v * dv + d] : kPad;
      eoff[j][d] = e == kPad ? -1 : 8 * (int)e;
    }
  }
  double* mrow = reinterpret_cast<double*>(mcv_b) + tid * dc;
  for (int64_t w = blockIdx.x; w < n_words; w += gridDim.x) {
    const double* lt = llr_tx + w * (int64_t)n_tx;
    int bad = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int v = tid + j * kFastThreads;
      if (v < n) {
        double x;
        if (v < k_tb) x = lt[v];
        else if (v < k) x = shortened;
        else if (v < k + p) x = lt[k_tb + (v - k)];
        else x = 0.0;
        bad |= !isfinite(x);
        llr[v] = x;
        tot[v] = x;
      }
    }
    if (__syncthreads_or(bad) && tid == 0 && n_nonfinite) atomicAdd(n_nonfinite, 1);
    double o1 = 0.0, o2 = 0.0;   // this check's previous messages (all +0.0 at first)
    unsigned om = 0u;
    int it = 0, converged = 0;
    for (;;) {
      int sp = 0;
      if (own_c) {
        double min1 = INFINITY, min2 = INFINITY;
        int amin = 0, par = 0;
        unsigned negm = 0u;
#pragma unroll
        for (int s = 0; s < kFastDC; ++s) {
          if (toff[s] < 0) continue;
          const double t = lds_f64(tot_b, toff[s]);
          sp ^= (t < 0.0);
          const double x = __dsub_rn(t, msg_of(o1, o2, om, s));
          const int ng = x < 0.0;
          negm |= (unsigned)ng << s;
          par ^= ng;
          const double a = fabs(x);
          if (a < min1) { min2 = min1; min1 = a; amin = s; }
          else if (a < min2) { min2 = a; }
        }
        o1 = __dmul_rn(alpha, min1);
        o2 = __dmul_rn(alpha, min2);
        om = (unsigned)amin | ((unsigned)par << 3) | (negm << 4);
#pragma unroll
        for (int s = 0; s < kFastDC; ++s)
          if (toff[s] >= 0) mrow[s] = msg_of(o1, o2, om, s);
      }
      if (!__syncthreads_or(sp)) { converged = 1; break; }
      if (it == max_iter) break;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int v = tid + j * kFastThreads;
        if (v < n) {
          double acc = 0.0;   // numpy order (dv < 8): 0 + e0 + e1 + ..., padded terms add +0
#pragma unroll
          for (int d = 0; d < kFastDV; ++d)
            if (eoff[j][d] >= 0) acc = __dadd_rn(acc, lds_f64(mcv_b, eoff[j][d]));
          tot[v] = __dadd_rn(llr[v], acc);
        }
      }
      __syncthreads();
      ++it;
    }
    uint8_t* out = info_out + w * (int64_t)k_tb;
    for (int v = tid; v < k_tb; v += kFastThreads) out[v] = tot[v] < 0.0 ? 1 : 0;
    if (tid == 0) {
      conv_out[w] = (uint8_t)converged;
      if (iters_out) iters_out[w] = it;
    }
    __syncthreads();
  }
}

// parity[r] = popc(E[r] & info) & 1 over the zero-padded k info bits;
// tx = [info (k_tb), parity[0, n_tx - k_tb)]  (fec.py:136-148, 262-278)
__global__ void ldpc_encode_kernel(const uint32_t* __restrict__ enc, int m, int k,
                                   const uint8_t* __restrict__ info, int64_t n_words, int k_tb,
                                   int n_tx, uint8_t* __restrict__ tx) {
  extern __shared__ uint32_t bits[];
  const int kw = (k + 31) / 32, p = n_tx - k_tb;
  for (int64_t w = blockIdx.x; w < n_words; w += gridDim.x) {
    const uint8_t* in = info + w * (int64_t)k_tb;
    for (int i = threadIdx.x; i < kw; i += blockDim.x) {
      uint32_t word = 0u;
      for (int j = 0; j < 32; ++j) {
        const int b = 32 * i + j;
        if (b < k_tb && (in[b] & 1)) word |= 1u << j;
      }
      bits[i] = word;
    }
    __syncthreads();
    uint8_t* out = tx + w * (int64_t)n_tx;
    for (int i = threadIdx.x; i < k_tb; i += blockDim.x) out[i] = in[i] & 1;
    for (int r = threadIdx.x; r < p; r += blockDim.x) {
      const uint32_t* er = enc + (int64_t)r * kw;
      int par = 0;
      for (int i = 0; i < kw; ++i) par ^= __popc(er[i] & bits[i]);
      out[k_tb + r] = (uint8_t)(par & 1);
    }
    __syncthreads();
  }
}

// syndrome (B, m): parity of the bits on each check (fec.py:151-153)
__global__ void ldpc_syndrome_kernel(const uint16_t* __restrict__ cv, int m, int dc,
                                     const uint8_t* __restrict__ bits, int64_t n_words, int n,
                                     uint8_t* __restrict__ synd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_words * m) return;
  const int64_t w = i / m;
  const int r = (int)(i % m);
  int par = 0;
  for (int s = 0; s < dc; ++s) {
    const uint16_t v = cv[r * dc + s];
    if (v != kPad) par ^= bits[w * n + v] & 1;
  }
  synd[i] = (uint8_t)par;
}

}  // namespace

namespace mpnl {
int set_error(int code, const char* msg);   // abi.cu: the thread's mpnl_last_error
}

extern "C" {

int mpnl_ldpc_graph_dims(const uint8_t* H, int m, int n, int* max_dc, int* max_dv) {
  if (!H || m < 1 || n <= m) return mpnl::set_error(MPNL_EINVAL, "parity-check matrix must be m x n with m < n");
  std::vector<int> dcs(m, 0), dvs(n, 0);
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < n; ++c)
      if (H[(int64_t)r * n + c]) { ++dcs[r]; ++dvs[c]; }
  int a = 0, b = 0;
  for (int x : dcs) a = x > a ? x : a;
  for (int x : dvs) b = x > b ? x : b;
  *max_dc = a;
  *max_dv = b;
  if (a > 32 || b > 32 || (int64_t)m * a >= kPad || n >= kPad)
    return mpnl::set_error(MPNL_EUNSUPPORTED, "LDPC graph too large (degree > 32 or >= 65535 edges)");
  return MPNL_OK;
}

int mpnl_ldpc_build(const uint8_t* H, int m, int n, int max_dc, int max_dv, uint16_t* check_vars,
                    uint16_t* var_edges, uint32_t* encoder) {
  int dc = 0, dv = 0;
  if (int rc = mpnl_ldpc_graph_dims(H, m, n, &dc, &dv)) return rc;
  if (dc != max_dc || dv != max_dv) return mpnl::set_error(MPNL_EINVAL, "graph dimensions mismatch");
  // edges enumerated row-major (np.nonzero order), fec.py:107-133
  std::vector<int> sc(m, 0), sv(n, 0);
  for (int64_t i = 0; i < (int64_t)m * dc; ++i) check_vars[i] = kPad;
  for (int64_t i = 0; i < (int64_t)n * dv; ++i) var_edges[i] = kPad;
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < n; ++c)
      if (H[(int64_t)r * n + c]) {
        check_vars[r * dc + sc[r]] = (uint16_t)c;
        var_edges[c * dv + sv[c]] = (uint16_t)(r * dc + sc[r]);
        ++sc[r];
        ++sv[c];
      }
  // systematic encoder: GF(2) elimination on the parity columns (fec.py:60-81)
  const int k = n - m, kw = (k + 31) / 32;
  std::vector<uint8_t> w(H, H + (int64_t)m * n);
  for (int r = 0; r < m; ++r) {
    const int c = k + r;
    int p = -1;
    for (int i = r; i < m; ++i)
      if (w[(int64_t)i * n + c]) { p = i; break; }
    if (p < 0) return mpnl::set_error(MPNL_EINVAL, "parity submatrix is singular");
    if (p != r)
      for (int j = 0; j < n; ++j) std::swap(w[(int64_t)r * n + j], w[(int64_t)p * n + j]);
    for (int i = 0; i < m; ++i)
      if (i != r && w[(int64_t)i * n + c])
        for (int j = 0; j < n; ++j) w[(int64_t)i * n + j] ^= w[(int64_t)r * n + j];
  }
  for (int r = 0; r < m; ++r)
    for (int i = 0; i < kw; ++i) {
      uint32_t word = 0u;
      for (int j = 0; j < 32 && 32 * i + j < k; ++j)
        if (w[(int64_t)r * n + 32 * i + j]) word |= 1u << j;
      encoder[(int64_t)r * kw + i] = word;
    }
  return MPNL_OK;
}

int mpnl_ldpc_decode(const uint16_t* check_vars, const uint16_t* var_edges, int m, int n,
                     int max_dc, int max_dv, const double* llr_tx, int64_t n_words, int n_tx,
                     int k_tb, int max_iter, double alpha, double shortened_llr,
                     uint8_t* info_out, uint8_t* converged, int32_t* iterations,
                     int32_t* n_nonfinite, void* stream) {
  const int k = n - m;
  if (m < 1 || n <= m || max_dc < 1 || max_dc > 32 || max_dv < 1 || max_dv > 32)
    return mpnl::set_error(MPNL_EINVAL, "invalid LDPC graph dimensions");
  if (k_tb < 1 || k_tb > k || n_tx - k_tb < 0 || n_tx - k_tb > m)
    return mpnl::set_error(MPNL_EINVAL, "invalid rate match (k_tb, n_tx)");
  if (max_iter < 0 || n_words < 0) return mpnl::set_error(MPNL_EINVAL, "negative max_iter or batch");
  if (n_words == 0) return MPNL_OK;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st = (cudaStream_t)stream;
  if (max_dc <= kFastDC && max_dv <= kFastDV && m <= kFastThreads && n <= 2 * kFastThreads) {
    const int smem = 8 * m * max_dc + 16 * n;
    cudaFuncSetAttribute(ldpc_decode_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ldpc_decode_fast_kernel, kFastThreads, smem);
    const int64_t grid = std::min<int64_t>(n_words, (int64_t)sms * std::max(per_sm, 1));
    ldpc_decode_fast_kernel<<<(unsigned)grid, kFastThreads, smem, st>>>(
        check_vars, var_edges, m, n, max_dc, max_dv, llr_tx, n_words, n_tx, k_tb, max_iter, alpha,
        shortened_llr, info_out, converged, iterations, n_nonfinite);
  } else {
    const DecLayout lo(m, n, max_dc, max_dv);
    if (lo.total > 200 * 1024) return mpnl::set_error(MPNL_EUNSUPPORTED, "LDPC code too large for one CTA");
    cudaFuncSetAttribute(ldpc_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lo.total);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ldpc_decode_kernel, kDecThreads, lo.total);
    const int64_t grid = std::min<int64_t>(n_words, (int64_t)sms * std::max(per_sm, 1));
    ldpc_decode_kernel<<<(unsigned)grid, kDecThreads, lo.total, st>>>(
        check_vars, var_edges, m, n, max_dc, max_dv, llr_tx, n_words, n_tx, k_tb, max_iter, alpha,
        shortened_llr, info_out, converged, iterations, n_nonfinite, lo);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return mpnl::set_error(MPNL_ECUDA, cudaGetErrorString(e));
  return MPNL_OK;
}

int mpnl_ldpc_encode(const uint32_t* encoder, int m, int n, const uint8_t* info, int64_t n_words,
                     int k_tb, int n_tx, uint8_t* tx_out, void* stream) {
  const int k = n - m;
  if (m < 1 || n <= m) return mpnl::set_error(MPNL_EINVAL, "invalid LDPC code dimensions");
  if (k_tb < 1 || k_tb > k || n_tx - k_tb < 0 || n_tx - k_tb > m)
    return mpnl::set_error(MPNL_EINVAL, "invalid rate match (k_tb, n_tx)");
  if (n_words <= 0) return n_words < 0 ? mpnl::set_error(MPNL_EINVAL, "negative batch") : MPNL_OK;
  const int grid = (int)std::min<int64_t>(n_words, 148 * 8);
  const size_t smem = 4 * (size_t)((k + 31) / 32);
  ldpc_encode_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(encoder, m, k, info, n_words,
                                                                  k_tb, n_tx, tx_out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return mpnl::set_error(MPNL_ECUDA, cudaGetErrorString(e));
  return MPNL_OK;
}

int mpnl_ldpc_syndrome(const uint16_t* check_vars, int m, int max_dc, const uint8_t* bits,
                       int64_t n_words, int n, uint8_t* syndrome_out, void* stream) {
  if (m < 1 || n <= m || max_dc < 1) return mpnl::set_error(MPNL_EINVAL, "invalid LDPC graph dimensions");
  if (n_words <= 0) return n_words < 0 ? mpnl::set_error(MPNL_EINVAL, "negative batch") : MPNL_OK;
  const int64_t tot = n_words * m;
  ldpc_syndrome_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      check_vars, m, max_dc, bits, n_words, n, syndrome_out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return mpnl::set_error(MPNL_ECUDA, cudaGetErrorString(e));
  return MPNL_OK;
}

}  // extern "C"
