// Argument block and shared-memory layout of the fp64 exact kernel (exact.cu),
// shared with the C ABI host code (abi.cu).
#pragma once
#include "common.cuh"

namespace mpnl {

struct ExactArgs {
  const double2* r64;    // (n_ch, N, N)
  const double2* qh64;   // (n_ch, N, M)
  const int32_t* perm;   // (n_ch, N)
  const void* y;         // (n_ch, V, M)
  int y_f64;
  int64_t n_ch, V;
  int m, n, L;
  double noise_var;
  int augmented;
  const int64_t* list;     // flagged vector ids, or null -> vectors [0, n_tasks)
  const int32_t* count;    // device count of `list`
  int64_t n_tasks;
  uint8_t* hard;           // (B, N) Gray labels (hard mode) or null
  float* metric;           // (B,) hard mode metric (fp32) or null
  double* metric64;        // (B,) hard mode metric (fp64) or null
  uint8_t* full_labels;    // (B, P, N) or null
  double* full_metrics;    // (B, P) or null
  int64_t* full_best;      // (B,) or null
  int exact_order;         // 1: full layers in stable distance order too
  int split;               // > 1: a thread-block cluster of `split` CTAs shares one vector
                           // (its paths and their parents' lists are divided; fix-up mode)
};

}  // namespace mpnl
