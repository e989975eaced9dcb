// Slot I/O around the detector: the per-RE receive grid and
// the DMRS least-squares channel estimate of the reference link simulator
// (pkg/src/mpnlsim/linksim.py:117-137, 200-226).
//
//   slot_receive:  y[b, t, f, :] = H[t, f] x[b, t, f] + noise[b, t, f]
//                  (linksim.py:207, einsum "tfmn,btfn->btfm" + noise);
//                  thread per (b, t, f, m), fp64 complex MACs over the N streams
//                  in numpy's einsum order: bit-identical.
//   dmrs_ls:       per stream v (DMRS symbol t_v, pilot subcarriers sc_v[p]):
//                  h_pilot = obs[t_v, sc_v[p], :] / pilot_v[p] (numpy's complex
//                  division, Smith's algorithm, bit for bit), nearest pilot
//                  subcarrier (first minimum of |sc - sc_v[p]|), the same value
//                  for every symbol of the slot (linksim.py:117-137);
//                  thread per (subcarrier, antenna, stream), S stores each.
//   select_symbols: the data-symbol rows of a grid (h[data_syms] /
//                  y[:, data_syms], linksim.py:211-216) as one gather.
// All three are HBM-bound streaming kernels.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mpnl_b200.h"

namespace mpnl {
int set_error(int code, const char* msg);
}

namespace {

// numpy's complex128 division (npy_cdouble, Smith's method; no FMA contraction)
__device__ __forceinline__ double2 np_cdiv(double2 a, double2 b) {
  const double ar = fabs(b.x), ai = fabs(b.y);
  if (ar >= ai) {
    if (ar == 0.0 && ai == 0.0) return make_double2(a.x / ar, a.y / ar);
    const double rat = __ddiv_rn(b.y, b.x);
    const double scl = __ddiv_rn(1.0, __dadd_rn(b.x, __dmul_rn(b.y, rat)));
    return make_double2(__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, rat)), scl),
                        __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, rat)), scl));
  }
  const double rat = __ddiv_rn(b.x, b.y);
  const double scl = __ddiv_rn(1.0, __dadd_rn(b.y, __dmul_rn(b.x, rat)));
  return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(a.x, rat), a.y), scl),
                      __dmul_rn(__dsub_rn(__dmul_rn(a.y, rat), a.x), scl));
}

__global__ void slot_receive_kernel(const double2* __restrict__ h, const double2* __restrict__ x,
                                    const double2* __restrict__ noise, int64_t frames, int s,
                                    int sc, int m, int n, double2* __restrict__ y) {
  const int64_t total = frames * s * sc * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int mm = (int)(i % m);
    const int64_t tf = (i / m) % ((int64_t)s * sc);   // (t, f)
    const int64_t b = i / ((int64_t)m * s * sc);
    const double2* hr = h + (tf * m + mm) * n;
    const double2* xr = x + (b * s * sc + tf) * n;
    // numpy's einsum order: sequential over the streams from 0, each complex
    // product's two real products rounded separately, then + noise (no FMA)
    double re = 0.0, im = 0.0;
    for (int k = 0; k < n; ++k) {
      const double2 a = hr[k], v = xr[k];
      re = __dadd_rn(re, __dsub_rn(__dmul_rn(a.x, v.x), __dmul_rn(a.y, v.y)));
      im = __dadd_rn(im, __dadd_rn(__dmul_rn(a.x, v.y), __dmul_rn(a.y, v.x)));
    }
    if (noise) {
      const double2 w = noise[i];
      re = __dadd_rn(re, w.x);
      im = __dadd_rn(im, w.y);
    }
    y[i] = make_double2(re, im);
  }
}

__global__ void dmrs_ls_kernel(const double2* __restrict__ obs, const double2* __restrict__ pilots,
                               const int32_t* __restrict__ port_sym,
                               const int32_t* __restrict__ port_sc, int s, int sc, int m, int n,
                               int np_, double2* __restrict__ h_est) {
  const int64_t total = (int64_t)sc * m * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % n);
    const int mm = (int)((i / n) % m);
    const int f = (int)(i / ((int64_t)n * m));
    const int32_t* scs = port_sc + (int64_t)v * np_;
    int best = 0, bd = abs(f - scs[0]);
    for (int p = 1; p < np_; ++p) {   // first minimum (np.argmin)
      const int d = abs(f - scs[p]);
      if (d < bd) { bd = d; best = p; }
    }
    const double2 o = obs[((int64_t)port_sym[v] * sc + scs[best]) * m + mm];
    const double2 hv = np_cdiv(o, pilots[(int64_t)v * np_ + best]);
    for (int t = 0; t < s; ++t) h_est[(((int64_t)t * sc + f) * m + mm) * n + v] = hv;
  }
}

__global__ void select_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ rows,
                                   int n_sel, int s, int64_t row_u4, int64_t batch,
                                   uint4* __restrict__ dst) {
  const int64_t total = batch * n_sel * row_u4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i % row_u4;
    const int64_t r = (i / row_u4) % n_sel;
    const int64_t b = i / (row_u4 * n_sel);
    dst[i] = src[(b * s + rows[r]) * row_u4 + w];
  }
}

unsigned grid_for(int64_t total) {
  const int64_t b = (total + 255) / 256;
  return (unsigned)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

int cuda_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MPNL_OK : mpnl::set_error(MPNL_ECUDA, cudaGetErrorString(e));
}

}  // namespace

extern "C" {

int mpnl_slot_receive(const void* h, const void* x, const void* noise, int64_t frames,
                      int symbols, int subcarriers, int m, int n, void* y, void* stream) {
  if (frames < 0 || symbols < 1 || subcarriers < 1 || m < 1 || n < 1)
    return mpnl::set_error(MPNL_EINVAL, "invalid slot grid dimensions");
  const int64_t total = frames * symbols * subcarriers * m;
  if (total == 0) return MPNL_OK;
  slot_receive_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      (const double2*)h, (const double2*)x, (const double2*)noise, frames, symbols, subcarriers,
      m, n, (double2*)y);
  return cuda_check("slot receive");
}

int mpnl_dmrs_ls_estimate(const void* grid_obs, const void* pilots, const int32_t* port_symbol,
                          const int32_t* port_subcarriers, int symbols, int subcarriers, int m,
                          int n, int n_pilot, void* h_est, void* stream) {
  if (symbols < 1 || subcarriers < 1 || m < 1 || n < 1 || n_pilot < 1)
    return mpnl::set_error(MPNL_EINVAL, "invalid DMRS estimate dimensions");
  const int64_t total = (int64_t)subcarriers * m * n;
  dmrs_ls_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      (const double2*)grid_obs, (const double2*)pilots, port_symbol, port_subcarriers, symbols,
      subcarriers, m, n, n_pilot, (double2*)h_est);
  return cuda_check("dmrs ls");
}

int mpnl_select_symbols(const void* src, int64_t batch, int symbols, int64_t row_bytes,
                        const int32_t* rows, int n_rows, void* dst, void* stream) {
  if (batch < 0 || symbols < 1 || n_rows < 0 || row_bytes < 0 || row_bytes % 16)
    return mpnl::set_error(MPNL_EINVAL, "invalid symbol selection (row bytes must be 16k)");
  const int64_t total = batch * n_rows * (row_bytes / 16);
  if (total == 0) return MPNL_OK;
  select_rows_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      (const uint4*)src, rows, n_rows, symbols, row_bytes / 16, batch, (uint4*)dst);
  return cuda_check("select symbols");
}

}  // extern "C"
