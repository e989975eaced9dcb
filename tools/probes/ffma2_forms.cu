// FFMA2 operand-form throughput probe (sm_100a): what bounds the traversal's inner loop?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_forms tools/probes/ffma2_forms.cu
// Variants (all: 128-thread CTAs, `ctas` per SM resident, NACC independent f32x2 accumulators):
//   0  acc = fma2(acc, x, b)                        same pair operands everywhere (bench.py's probe)
//   1  acc_k = fma2(bcast(-r_j), g, acc_k)          scalar-broadcast operand, distinct r registers
//   2  1 + the swapped/partially negated pair       the traversal's two-FFMA2 row update
//   3  2 with r from broadcast LDS.128              adds the shared-memory wavefronts (0.5 / FFMA2)
//   4  2 with r from LDS.128, two paths per load    0.25 wavefront / FFMA2
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float lo32(u64 v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi32(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

template <int V, int NACC>
__global__ void __launch_bounds__(128, 4) probe(float* out, const float* tab, int iters) {
  __shared__ __align__(16) float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 128) sm[i] = tab[i];
  __syncthreads();
  const float t = threadIdx.x * 1e-3f;
  u64 acc[NACC], acc2[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { acc[k] = pk2(t + k, t - k); acc2[k] = pk2(t - k, t + k); }
  u64 g = pk2(-1.f - t * 1e-6f, -3.f), h = pk2(-5.f, -7.f - t * 1e-6f);
  const u64 x = pk2(0.999999f, 0.999998f), b = pk2(1e-7f, 1e-7f);
  float r[2 * NACC];
#pragma unroll
  for (int k = 0; k < 2 * NACC; ++k) r[k] = sm[k] * 1e-3f;
  const float4* s4 = reinterpret_cast<const float4*>(sm);
  for (int i = 0; i < iters; ++i) {
    if (V == 0) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) { acc[k] = ffma2(acc[k], x, b); acc[k] = ffma2(acc[k], x, b); }
    } else if (V == 1) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) {
        acc[k] = ffma2(pk2(-r[2 * k], -r[2 * k]), g, acc[k]);
        acc[k] = ffma2(pk2(-r[2 * k + 1], -r[2 * k + 1]), h, acc[k]);
      }
    } else if (V == 2) {
      const u64 gs = pk2(-hi32(g), lo32(g));
#pragma unroll
      for (int k = 0; k < NACC; ++k) {
        acc[k] = ffma2(pk2(-r[2 * k], -r[2 * k]), g, acc[k]);
        acc[k] = ffma2(gs, pk2(-r[2 * k + 1], -r[2 * k + 1]), acc[k]);
      }
    } else {
      const u64 gs = pk2(-hi32(g), lo32(g)), hs = pk2(-hi32(h), lo32(h));
      const float4* p = s4 + (i & 7) * (NACC / 2);
#pragma unroll
      for (int q = 0; q < NACC / 2; ++q) {
        const float4 rr = p[q];
        acc[2 * q] = ffma2(pk2(-rr.x, -rr.x), g, acc[2 * q]);
        acc[2 * q] = ffma2(gs, pk2(-rr.y, -rr.y), acc[2 * q]);
        acc[2 * q + 1] = ffma2(pk2(-rr.z, -rr.z), g, acc[2 * q + 1]);
        acc[2 * q + 1] = ffma2(gs, pk2(-rr.w, -rr.w), acc[2 * q + 1]);
        if (V == 4) {
          acc2[2 * q] = ffma2(pk2(-rr.x, -rr.x), h, acc2[2 * q]);
          acc2[2 * q] = ffma2(hs, pk2(-rr.y, -rr.y), acc2[2 * q]);
          acc2[2 * q + 1] = ffma2(pk2(-rr.z, -rr.z), h, acc2[2 * q + 1]);
          acc2[2 * q + 1] = ffma2(hs, pk2(-rr.w, -rr.w), acc2[2 * q + 1]);
        }
      }
    }
    // a data dependence that keeps g / h live and varying (one FFMA2 per iteration)
    g = ffma2(g, x, b);
    h = ffma2(h, x, b);
  }
  u64 s = 0;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s ^= acc[k] ^ acc2[k];
  out[blockIdx.x * 128 + threadIdx.x] = lo32(s) + hi32(s);
}

template <int V, int NACC>
void run(const char* name, int ctas_per_sm, float* out, float* tab) {
  const int iters = 20000, grid = 148 * ctas_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<V, NACC><<<grid, 128>>>(out, tab, 200);
  cudaEventRecord(e0);
  probe<V, NACC><<<grid, 128>>>(out, tab, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double per_iter = (V == 4 ? 4.0 : 2.0) * NACC + 2;   // FFMA2 per thread per iteration
  const double tf = (double)grid * 128 * iters * per_iter * 4 / (ms * 1e-3) / 1e12;
  printf("%-44s NACC=%2d ctas/SM=%d  %7.2f TFLOP/s  (%.3f of 74.45)  %s\n", name, NACC, ctas_per_sm, tf,
         tf / 74.45, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float *out, *tab;
  cudaMalloc(&out, 148 * 8 * 128 * 4);
  cudaMalloc(&tab, 4096);
  float h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 0.001f * (i % 37) - 0.01f;
  cudaMemcpy(tab, h, 4096, cudaMemcpyHostToDevice);
  for (int c = 2; c <= 4; c += 2) {
    run<0, 12>("0 pair operands, shared x/b", c, out, tab);
    run<1, 12>("1 scalar-broadcast operand", c, out, tab);
    run<2, 12>("2 scalar + swapped/negated pair", c, out, tab);
    run<3, 12>("3 form 2, r'' by broadcast LDS.128 (1 path)", c, out, tab);
    run<4, 12>("4 form 2, r'' by LDS.128 shared by 2 paths", c, out, tab);
    run<2, 24>("2 scalar + swapped/negated pair", c, out, tab);
    run<3, 24>("3 form 2, r'' by broadcast LDS.128 (1 path)", c, out, tab);
  }
  return 0;
}
