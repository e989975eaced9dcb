// Explicit instantiation of the fast-path kernels (select / traverse / verify)
// for one QAM order (L levels per axis) and a range of 8 N values, plus the
// launcher the C ABI dispatches to.  Included by the traverse_l<L>_p<part>.cu
// units (one per constellation x N-range, compiled in parallel).
#pragma once
#include <algorithm>

#include "exact.cuh"
#include <cstdlib>

#include "traverse.cuh"
#include "soft.cuh"

#ifndef MPNL_TRAV_WAVES
#define MPNL_TRAV_WAVES 4
#endif

namespace mpnl {

// kind 0 = select_kernel (extra = layer), 1 = traverse_kernel, 2 = verify_kernel,
// 3 = check_kernel, 5 = prep2_kernel (fused prep + top selection), 6 = soft_llr_kernel
template <int NN, int L>
cudaError_t launch_fast_one(int kind, const DetectArgs& a, const TreeParams& tp, unsigned grid,
                            int threads, size_t smem, int extra, cudaStream_t st) {
  if (kind == 0) {
    // block = (parents, vectors); the smallest unrolled pick count >= e
    const int pos = extra, e = tp.e[pos];
    const int npar = tp.n_paths / tp.stride[pos + 1];
    const int px = std::min(npar, 128), vy = std::max(1, 128 / px);
    const int vblocks = (int)((a.V + vy - 1) / vy);
    const dim3 blk(px, vy), grd((unsigned)(a.n_ch * vblocks), (unsigned)((npar + px - 1) / px));
    if constexpr (L == 2) {
      select_kernel<NN, L, 4><<<grd, blk, 0, st>>>(a, tp, pos, npar, vblocks);
    } else if constexpr (L == 4) {
      if (e <= 4) select_kernel<NN, L, 4><<<grd, blk, 0, st>>>(a, tp, pos, npar, vblocks);
      else select_kernel<NN, L, 16><<<grd, blk, 0, st>>>(a, tp, pos, npar, vblocks);
    } else {
      if (e <= 4) select_kernel<NN, L, 4><<<grd, blk, 0, st>>>(a, tp, pos, npar, vblocks);
      else if (e <= 16) select_kernel<NN, L, 16><<<grd, blk, 0, st>>>(a, tp, pos, npar, vblocks);
      else select_kernel<NN, L, 64><<<grd, blk, 0, st>>>(a, tp, pos, npar, vblocks);
    }
  } else if (kind == 1) {
    // persistent: grid = resident capacity (capped by the item count `extra`)
    // top-layer sharing of sibling path pairs (PT = 2, one vector per batch, even top stride)
    constexpr bool CAN_SH = TravCfg<NN>::PT == 2;
    const bool sh = CAN_SH && a.vpi <= 1 && tp.n_top >= 1 && tp.stride[NN - 1] % 2 == 0 &&
                    tp.n_paths % 2 == 0;
    const bool oneb = sh && a.bpv == 1 && tp.n_paths == 32 * TravCfg<NN>::PT;
    auto k = a.vpi > 1 ? traverse_kernel<NN, L, true>
                       : (oneb ? traverse_kernel<NN, L, false, CAN_SH, CAN_SH>
                               : (sh ? traverse_kernel<NN, L, false, CAN_SH>
                                     : traverse_kernel<NN, L, false>));
    if (a.wpc)   // a warp per channel (few vectors per channel): plain or VPI instance
      k = a.vpi > 1 ? traverse_kernel<NN, L, true, false, false, true>
                    : traverse_kernel<NN, L, false, false, false, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (grid == 0) {
      int nb = 0, dev = 0, sms = 148;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, threads, smem);
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      // waves of CTAs over the resident capacity: the block scheduler refills
      // the slot of a CTA that finished early (the SM's warp schedulers favour
      // the oldest warps, so co-resident CTAs finish at different times)
      // (measured: C2 338 -> 326 us, C4 1161 -> 1119 us at 4 waves).  Small
      // batches (< 64 path batches per resident warp) keep one wave: their
      // per-CTA table staging would not be amortised.
      static const int env_waves = [] {
        const char* e = getenv("MPNL_TRAV_WAVES");
        return e ? atoi(e) : 0;
      }();
      const long long cap = (long long)std::max(nb, 1) * sms;
      const long long work = (long long)extra * std::max(a.bpv, 1);
      // (very long grids -- C5 at P >= 256: over 1,000 path batches per resident warp --
      // gain another 0.5% from six waves; C2 / C3 / C4 are best at four or fewer)
      int waves = work >= 64LL * cap * (threads / 32) ? MPNL_TRAV_WAVES : 1;
      if (work >= 1024LL * cap * (threads / 32)) waves = MPNL_TRAV_WAVES + MPNL_TRAV_WAVES / 2;
      if (env_waves > 0) waves = env_waves;
      grid = (unsigned)std::min<long long>(cap * waves, (long long)extra);
      if (a.wpc)   // a warp per channel: one wave of CTAs, never more warps than channels
        grid = (unsigned)std::min<long long>(cap, (a.n_ch + threads / 32 - 1) / (threads / 32));
    }
    k<<<grid, threads, smem, st>>>(a, tp);
  } else if (kind == 5) {
    // fused prep + top partial-layer selection (E = 2 or 4); extra = pos_sel (-1:
    // none), threads = threads per vector (1, or 4 for small batches)
    const int pos = extra;
    const int tpv = threads == 4 ? 4 : 1;
    const int sm = Prep2Smem<NN>::bytes(a.m, 128 / tpv, a.y_f64 ? 16 : 8);
    const int chunks = (int)((a.V + 128 / tpv - 1) / (128 / tpv));
    auto launch = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      kern<<<(unsigned)(a.n_ch * chunks), 128, sm, st>>>(a, tp, chunks, pos);
    };
    const int e = pos >= 0 ? tp.e[pos] : 0;   // 0, 2 or 4 (abi.cu)
    if (tpv == 1) {
      if (e == 0) launch(prep2_kernel<NN, L, 0, 1>);
      else if (e == 2) launch(prep2_kernel<NN, L, 2, 1>);
      else launch(prep2_kernel<NN, L, 4, 1>);
    } else {
      if (e == 0) launch(prep2_kernel<NN, L, 0, 4>);
      else if (e == 2) launch(prep2_kernel<NN, L, 2, 4>);
      else launch(prep2_kernel<NN, L, 4, 4>);
    }
  } else if (kind == 6) {
    // fp32 list LLRs: CTA = (channel, chunk of vectors), tables staged per CTA
    auto k = soft_llr_kernel<NN, L>;
    const int sm = SoftSmem(a.m, NN, L == 2 ? 2 : (L == 4 ? 4 : 6), 4).total_bytes;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    k<<<(unsigned)(a.n_ch * a.soft.chunks), 128, sm, st>>>(a, tp);
  } else if (kind == 2) {
    verify_kernel<NN, L><<<grid, threads, 0, st>>>(a, tp, extra);
  } else {
    // events strided over all warps; at most the resident capacity
    auto k = check_kernel<NN, L>;
    const int sm = (int)sizeof(CheckSmem<NN>);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    int nb = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 32 * CHECK_WARPS, sm);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = (unsigned)std::min<long long>((long long)std::max(nb, 1) * sms, (long long)grid);
    k<<<grid, 32 * CHECK_WARPS, sm, st>>>(a, tp, extra);
  }
  return cudaGetLastError();
}

template <int L, int N0>
cudaError_t launch_fast_part(int n, int kind, const DetectArgs& a, const TreeParams& tp,
                             unsigned grid, int threads, size_t smem, int extra, cudaStream_t st) {
  switch (n - N0) {
#define MPNL_C(I) \
    case I: return launch_fast_one<N0 + I, L>(kind, a, tp, grid, threads, smem, extra, st);
    MPNL_C(0) MPNL_C(1) MPNL_C(2) MPNL_C(3) MPNL_C(4) MPNL_C(5) MPNL_C(6) MPNL_C(7)
#undef MPNL_C
    default: return cudaErrorInvalidValue;
  }
}

template <int L, int N0>
cudaError_t launch_exact_part(int n, const ExactArgs& a, const TreeParams& tp, int grid,
                              cudaStream_t st) {
  switch (n - N0) {
#define MPNL_C(I) \
    case I: return launch_exact_t<N0 + I, L>(a, tp, grid, st);
    MPNL_C(0) MPNL_C(1) MPNL_C(2) MPNL_C(3) MPNL_C(4) MPNL_C(5) MPNL_C(6) MPNL_C(7)
#undef MPNL_C
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mpnl
