// List max-log LLRs over a candidate list.
//
// Reference: `_candidate_llrs_batch` (pkg/src/mpnlsim/detect.py:439-453) with the
// bit expansion of `bits_from_labels` (core.py:209-213, MSB first) and LLR_CLIP
// (core.py:21).  Per vector b, stream n and bit j:
//     min1 = min over paths with bit j of labels[b,p,n] set   of metrics[b,p]
//     min0 = min over paths with the bit clear                of metrics[b,p]
//     llr[b,n,j] = clip((min1 - min0) / nv_b, -clip, clip)
// A bit no path sets (or clears) has min = +inf and saturates, exactly as
// numpy does.  All arithmetic is one IEEE fp64 subtraction and one correctly
// rounded fp64 division, so the result is bit-identical to the reference.
//
// Layout: labels (B, P, N) uint8, metrics (B, P) fp64, llr (B, N, bps) fp64 — the
// mpnl_detect_full outputs as they sit in HBM.  The kernel is HBM-bound byte
// work: one warp per vector, lane = stream, so every path is one coalesced
// N-byte row read plus a broadcast metric; the 2·bps running minima live in
// registers.  A warp takes G = 32 / N vectors at once (lane = (vector, stream)),
// so short vectors do not idle most of the warp.  Grid: persistent warps
// strided over vector groups.
#include <cstdint>
#include <cuda_runtime.h>

#include <cstddef>

namespace mpnl {

template <int BPS>
__global__ void __launch_bounds__(256) candidate_llr_kernel(
    const uint8_t* __restrict__ labels, const double* __restrict__ metrics, int64_t B,
    int64_t P, int n, double nv, const double* __restrict__ nv_vec, double clip,
    double* __restrict__ llr) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int G = 32 / n;                        // vectors per warp pass
  const int gi = lane / n, ln = lane - gi * n;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  for (int64_t b0 = warp * G; b0 < B; b0 += n_warps * G) {
    const int64_t b = b0 + gi;
    const bool active = gi < G && b < B;
    const int64_t bb = active ? b : b0;        // inactive lanes read a valid row
    double mn1[BPS], mn0[BPS];
#pragma unroll
    for (int j = 0; j < BPS; ++j) mn1[j] = mn0[j] = inf;
    const uint8_t* lab = labels + bb * P * n + ln;
    const double* met = metrics + bb * P;
    int64_t p = 0;
    for (; p + 4 <= P; p += 4) {
      unsigned l4[4];
      double m4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        l4[u] = active ? __ldg(lab + (p + u) * n) : 0u;
        m4[u] = __ldg(met + p + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int j = 0; j < BPS; ++j) {
          const bool bit = (l4[u] >> (BPS - 1 - j)) & 1u;
          if (bit) mn1[j] = m4[u] < mn1[j] ? m4[u] : mn1[j];
          else mn0[j] = m4[u] < mn0[j] ? m4[u] : mn0[j];
        }
      }
    }
    for (; p < P; ++p) {
      const unsigned l = active ? __ldg(lab + p * n) : 0u;
      const double m = __ldg(met + p);
#pragma unroll
      for (int j = 0; j < BPS; ++j) {
        const bool bit = (l >> (BPS - 1 - j)) & 1u;
        if (bit) mn1[j] = m < mn1[j] ? m : mn1[j];
        else mn0[j] = m < mn0[j] ? m : mn0[j];
      }
    }
    if (active) {
      const double v = nv_vec ? nv_vec[b] : nv;
      double* out = llr + (b * n + ln) * BPS;
#pragma unroll
      for (int j = 0; j < BPS; ++j) {
        double x = __ddiv_rn(__dsub_rn(mn1[j], mn0[j]), v);
        // np.clip: NaN stays NaN, otherwise min(max(x, -clip), clip)
        if (x < -clip) x = -clip;
        if (x > clip) x = clip;
        out[j] = x;
      }
    }
  }
}

// Staged variant (16-byte aligned lists): the G vectors' label rows and metrics
// of a chunk of CP paths are copied into the warp's shared memory with 16-byte
// loads (one instruction per 512 bytes per warp instead of one byte load per
// lane and path), then every lane runs the same per-path minima from shared
// memory.  Same comparisons in the same path order: bit-identical outputs.
constexpr int kCP = 64;   // paths per chunk

template <int BPS>
__global__ void __launch_bounds__(256) candidate_llr_staged_kernel(
    const uint8_t* __restrict__ labels, const double* __restrict__ metrics, int64_t B,
    int64_t P, int n, double nv, const double* __restrict__ nv_vec, double clip,
    double* __restrict__ llr) {
  extern __shared__ __align__(16) unsigned char lsm_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int G = 32 / n;
  // per warp: G x kCP x n label bytes (rounded to 16) | G x kCP metrics
  const int lab_b = (G * kCP * n + 15) & ~15;
  unsigned char* wl = lsm_raw + (size_t)wid * (lab_b + G * kCP * 8);
  double* wm = reinterpret_cast<double*>(wl + lab_b);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int gi = lane / n, ln = lane - gi * n;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  for (int64_t b0 = warp * G; b0 < B; b0 += n_warps * G) {
    const int gv = (int)min((int64_t)G, B - b0);   // vectors in this pass
    const int64_t b = b0 + gi;
    const bool active = gi < gv;
    double mn1[BPS], mn0[BPS];
#pragma unroll
    for (int j = 0; j < BPS; ++j) mn1[j] = mn0[j] = inf;
    for (int64_t p0 = 0; p0 < P; p0 += kCP) {
      const int cp = (int)min((int64_t)kCP, P - p0);
      const int rowb = cp * n;                        // label bytes per vector in the chunk
      __syncwarp();
      for (int g = 0; g < gv; ++g) {
        const uint4* src = reinterpret_cast<const uint4*>(labels + ((b0 + g) * P + p0) * n);
        uint4* dst = reinterpret_cast<uint4*>(wl + g * kCP * n);
        for (int i = lane; i < rowb / 16; i += 32) dst[i] = __ldg(src + i);
        const double2* ms = reinterpret_cast<const double2*>(metrics + (b0 + g) * P + p0);
        double2* md = reinterpret_cast<double2*>(wm + g * kCP);
        for (int i = lane; i < cp / 2; i += 32) md[i] = __ldg(ms + i);
      }
      __syncwarp();
      if (active) {
        const unsigned char* lab = wl + gi * kCP * n + ln;
        const double* met = wm + gi * kCP;
#pragma unroll 4
        for (int p = 0; p < cp; ++p) {
          const unsigned l = lab[p * n];
          const double m = met[p];
#pragma unroll
          for (int j = 0; j < BPS; ++j) {
            const bool bit = (l >> (BPS - 1 - j)) & 1u;
            if (bit) mn1[j] = m < mn1[j] ? m : mn1[j];
            else mn0[j] = m < mn0[j] ? m : mn0[j];
          }
        }
      }
    }
    if (active) {
      const double v = nv_vec ? nv_vec[b] : nv;
      double* out = llr + (b * n + ln) * BPS;
#pragma unroll
      for (int j = 0; j < BPS; ++j) {
        double x = __ddiv_rn(__dsub_rn(mn1[j], mn0[j]), v);
        if (x < -clip) x = -clip;
        if (x > clip) x = clip;
        out[j] = x;
      }
    }
  }
}

cudaError_t launch_candidate_llrs(const uint8_t* labels, const double* metrics, int64_t B,
                                  int64_t P, int n, int bps, double nv, const double* nv_vec,
                                  double clip, double* llr, cudaStream_t st) {
  const int threads = 256;
  const int64_t warps_needed = (B + 32 / n - 1) / (32 / n);
  int64_t blocks = (warps_needed + (threads / 32) - 1) / (threads / 32);
  const int64_t cap = 148 * 8;  // 8 resident 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // 16-byte staging when every chunk row starts aligned: P N and kCP N multiples
  // of 16 bytes, P even (metric pairs) and 16-byte aligned bases
  const bool staged = (P * n) % 16 == 0 && (kCP * n) % 16 == 0 && P % 2 == 0 &&
                      (reinterpret_cast<uintptr_t>(labels) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(metrics) & 15) == 0;
  if (staged) {
    const int G = 32 / n;
    const size_t per_warp = (size_t)((G * kCP * n + 15) & ~15) + (size_t)G * kCP * 8;
    const size_t smem = per_warp * (threads / 32);
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<(unsigned)blocks, threads, smem, st>>>(labels, metrics, B, P, n, nv, nv_vec, clip,
                                                    llr);
    };
    switch (bps) {
      case 2: go(candidate_llr_staged_kernel<2>); break;
      case 4: go(candidate_llr_staged_kernel<4>); break;
      case 6: go(candidate_llr_staged_kernel<6>); break;
      default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
  switch (bps) {
    case 2:
      candidate_llr_kernel<2><<<(unsigned)blocks, threads, 0, st>>>(labels, metrics, B, P, n,
                                                                    nv, nv_vec, clip, llr);
      break;
    case 4:
      candidate_llr_kernel<4><<<(unsigned)blocks, threads, 0, st>>>(labels, metrics, B, P, n,
                                                                    nv, nv_vec, clip, llr);
      break;
    case 6:
      candidate_llr_kernel<6><<<(unsigned)blocks, threads, 0, st>>>(labels, metrics, B, P, n,
                                                                    nv, nv_vec, clip, llr);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace mpnl
