// Shared definitions for the MPNL B200 kernels (sm_100a).
//
// Numbering convention used everywhere: *tree position* pos = 0..N-1, with
// pos = N-1 the top (first-detected, weakest) layer, exactly as the reference
// (`detect.py:221-231`, `detect.py:403-428`).  Per-axis QAM symbols are held as
// *level indices* i = 0..L-1 (value (L-1-2i)/norm, Gray label i ^ (i>>1)),
// see `core.cuh`-free maps in `paper_2409_14355_b200/core.py`.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define MPNL_MAX_N 32
#define MPNL_MAX_M 64

namespace mpnl {

// --------------------------------------------------------------------------
// Per-channel fp32 table blob written by the plan kernel and read by the
// traversal kernel.  All offsets are in floats; every block starts 16-byte
// aligned so it can be fetched with 128-bit loads.
// --------------------------------------------------------------------------
struct TableLayout {
  int m, n;
  int off_qh;     // M x N double2 : Q^H transposed (fp64): qhT[r][k], for z = Q^H y
  int off_shift;  // N double2     : constant symbol offset folded into z (fp64)
  int off_lay;    // N float4      : per layer (kx = -1/c2r, c2r, S_k, kxs = kx/(L-1))
  int off_rcol;   // N columns x NPP float4: column pos, row pair q holds
                  // {rr_2q, ri_2q, rr_2q+1, ri_2q+1} of r''[k][pos] (0 for k >= pos)
  int npp;        // row pairs, (N+1)/2
  int total;      // floats per channel

  __host__ __device__ static int up4(int x) { return (x + 3) & ~3; }
  __host__ __device__ TableLayout(int m_, int n_) : m(m_), n(n_) {
    off_qh = 0;
    off_shift = up4(off_qh + 4 * n * m);
    off_lay = up4(off_shift + 4 * n);
    off_rcol = up4(off_lay + 4 * n);
    npp = (n + 1) / 2;
    total = up4(off_rcol + 4 * n * npp);
  }
};

// Expansion structure of a plan, passed by value (constant bank).
struct TreeParams {
  int n_paths;                 // realized P = prod(e)
  int n_top;                   // number of expanded layers (e > 1); they are
                               // positions N-1 .. N-n_top
  int e[MPNL_MAX_N];           // expansions by tree position
  int stride[MPNL_MAX_N + 1];  // prod_{j<pos} e_j (stride[N] = P)
  int list_off[MPNL_MAX_N];    // byte offset of the partial-layer list (per vector)
  int list_bytes;              // list bytes per vector (stride, multiple of 16)
  unsigned ms[MPNL_MAX_N];     // magic for p / stride[pos]   (fast_div)
  unsigned me[MPNL_MAX_N];     // magic for d / e[pos]
};

// floor(p / d) for p < 2^24 with m = floor((2^32 - 1) / d): the umulhi estimate
// is exact or one short; one upward correction makes it exact.
__host__ __device__ inline unsigned div_magic(unsigned d) { return 0xffffffffu / d; }
__device__ __forceinline__ unsigned fast_div(unsigned p, unsigned d, unsigned m) {
  unsigned q = __umulhi(p, m);
  return q + ((q + 1) * d <= p ? 1u : 0u);
}

__host__ __device__ inline float qam_norm(int L) {
  // sqrt(2 (L^2 - 1) / 3): 4-QAM sqrt(2), 16-QAM sqrt(10), 64-QAM sqrt(42)
  return L == 2 ? 1.4142135623730951f : (L == 4 ? 3.1622776601683795f : 6.48074069840786f);
}
__host__ __device__ inline double qam_norm_d(int L) {
  return L == 2 ? 1.4142135623730951 : (L == 4 ? 3.1622776601683795 : 6.48074069840786);
}
__host__ __device__ inline int gray_code(int i) { return i ^ (i >> 1); }

}  // namespace mpnl
