// C ABI of the MPNL B200 library (declared in include/mpnl_b200.h).
//
// Host side: argument validation with the reference's error behaviour, the
// integer expansion allocator (C++ port of detect.py:221-280), the tree /
// chunking parameters, and the kernel launches.  No host synchronisation,
// no hidden allocations: scratch comes from the caller's workspace.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mpnl_b200.h"
#include "common.cuh"
#include "traverse.cuh"

namespace mpnl {
cudaError_t launch_plan(const void* h, int h_is_f64, int64_t n_ch, int m, int n, int L,
                        double noise_var, int augmented, int32_t* perm, double2* r64,
                        double2* qh64, float* tables, cudaStream_t st);
#define MPNL_DECL_PART(LL, PP)                                                                 \
  cudaError_t launch_fast_l##LL##_p##PP(int n, int kind, const DetectArgs& a, const TreeParams& tp, \
                                        unsigned grid, int threads, size_t smem, int extra,       \
                                        cudaStream_t st);
MPNL_DECL_PART(2, 0) MPNL_DECL_PART(2, 1) MPNL_DECL_PART(2, 2) MPNL_DECL_PART(2, 3)
MPNL_DECL_PART(4, 0) MPNL_DECL_PART(4, 1) MPNL_DECL_PART(4, 2) MPNL_DECL_PART(4, 3)
MPNL_DECL_PART(8, 0) MPNL_DECL_PART(8, 1) MPNL_DECL_PART(8, 2) MPNL_DECL_PART(8, 3)
#undef MPNL_DECL_PART
}  // namespace mpnl

#include "exact_args.cuh"

namespace mpnl {
cudaError_t launch_exact(const ExactArgs& a, const TreeParams& tp, int grid, cudaStream_t st);
cudaError_t launch_linear_detect(const void* h, const void* y, int64_t n_vectors, int m, int n,
                                 int half_bits, int mmse, double nv_scalar, const double* nv_vec,
                                 double clip, uint8_t* labels_out, double* llr_out,
                                 void* est_out, int32_t* n_singular, cudaStream_t stream);
int linear_max_n();
cudaError_t launch_candidate_llrs(const uint8_t* labels, const double* metrics, int64_t B,
                                  int64_t P, int n, int bps, double nv, const double* nv_vec,
                                  double clip, double* llr, cudaStream_t st);
}

__global__ void flags_kernel(uint8_t* flags, const uint32_t* vflag, int64_t B, int all) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) flags[i] = (all || vflag[i]) ? 1 : 0;
}

static cudaError_t launch_flags(uint8_t* flags, const uint32_t* vflag, int64_t B, int all,
                                cudaStream_t st) {
  flags_kernel<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(flags, vflag, B, all);
  return cudaGetLastError();
}

using namespace mpnl;

namespace {

thread_local std::string g_err;   // mpnl_last_error(): per calling thread

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(MPNL_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int levels_for(int q) { return q == 4 ? 2 : (q == 16 ? 4 : (q == 64 ? 8 : 0)); }

// detect.py:240-251 — greedy non-increasing factorisation of `budget`
bool split_budget(int64_t budget, int slots, int64_t cap, std::vector<int64_t>& out) {
  if (budget == 1) return true;
  if (slots == 0) return false;
  for (int64_t d = std::min(cap, budget); d >= 2; --d) {
    if (budget % d) continue;
    out.push_back(d);
    if (split_budget(budget / d, slots - 1, d, out)) return true;
    out.pop_back();
  }
  return false;
}

int64_t ipow_sat(int64_t b, int e, int64_t cap) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) {
    if (r > cap / b) return cap + 1;
    r *= b;
  }
  return r;
}

struct TreeBuild {
  TreeParams tp;
  bool ok;
  std::string err;
};

TreeBuild build_tree(int n, int L, const int64_t* ex) {
  TreeBuild b;
  std::memset(&b.tp, 0, sizeof(b.tp));
  b.ok = false;
  const int q = L * L;
  int64_t stride = 1;
  b.tp.stride[0] = 1;
  for (int pos = 0; pos < n; ++pos) {
    if (ex[pos] < 1 || ex[pos] > q) { b.err = "expansions out of range [1, q]"; return b; }
    b.tp.e[pos] = (int)ex[pos];
    stride *= ex[pos];
    if (stride > (1 << 24)) { b.err = "path budget too large (> 2^24)"; return b; }
    b.tp.stride[pos + 1] = (int)stride;
  }
  b.tp.n_paths = (int)stride;
  int ntop = 0;
  for (int pos = n - 1; pos >= 0 && b.tp.e[pos] > 1; --pos) ++ntop;
  for (int pos = n - 1 - ntop; pos >= 0; --pos)
    if (b.tp.e[pos] != 1) { b.err = "expansions must be non-increasing from the top layer"; return b; }
  b.tp.n_top = ntop;
  int off = 0;
  for (int pos = n - 1; pos >= n - ntop; --pos) {
    const int e = b.tp.e[pos];
    if (e < q) {
      b.tp.list_off[pos] = off;
      off += b.tp.n_paths / b.tp.stride[pos];
    }
  }
  for (int pos = 0; pos < n; ++pos) {
    b.tp.ms[pos] = div_magic((unsigned)b.tp.stride[pos]);
    b.tp.me[pos] = div_magic((unsigned)b.tp.e[pos]);
  }
  b.tp.list_bytes = (off + 15) & ~15;   // 16-byte rows (cp.async staging)
  b.ok = true;
  return b;
}

int check_dims(int m, int n, int q) {
  if (n < 1 || m < 1) return fail(MPNL_EINVAL, "inconsistent channel/observation dimensions");
  if (n > MPNL_MAX_N) return fail(MPNL_EUNSUPPORTED, "N > 32 streams is not supported");
  if (m > MPNL_MAX_M || (n > m && m + n > MPNL_MAX_M))
    return fail(MPNL_EUNSUPPORTED, "M (or M+N when augmented) > 64 is not supported");
  if (!levels_for(q)) return fail(MPNL_EUNSUPPORTED, "unsupported constellation order " + std::to_string(q));
  return MPNL_OK;
}

int trav_pt(int n) {
  switch ((n + 7) / 8) {
    case 1: return TravCfg<8>::PT;
    case 2: return TravCfg<16>::PT;
    case 3: return TravCfg<24>::PT;
    default: return TravCfg<32>::PT;
  }
}

cudaError_t launch_fast(int n, int L, int kind, const DetectArgs& a, const TreeParams& tp,
                        unsigned grid, int threads, size_t smem, int extra, cudaStream_t st) {
  const int part = (n - 1) / 8;
#define MPNL_PART(LL)                                                                       \
  switch (part) {                                                                           \
    case 0: return launch_fast_l##LL##_p0(n, kind, a, tp, grid, threads, smem, extra, st); \
    case 1: return launch_fast_l##LL##_p1(n, kind, a, tp, grid, threads, smem, extra, st); \
    case 2: return launch_fast_l##LL##_p2(n, kind, a, tp, grid, threads, smem, extra, st); \
    default: return launch_fast_l##LL##_p3(n, kind, a, tp, grid, threads, smem, extra, st); \
  }
  if (L == 2) { MPNL_PART(2) }
  if (L == 4) { MPNL_PART(4) }
  MPNL_PART(8)
#undef MPNL_PART
}

// Workspace carve-up (byte offsets), identical in mpnl_workspace_bytes and the launches.
struct Workspace {
  int64_t counters, fix_list, vflag, vres, vpath, events, lists, zq, thrg, vaux, total;
  int64_t ev_cap;
  Workspace(int64_t B, int list_bytes, int n) {
    auto up = [](int64_t x) { return (x + 255) & ~int64_t(255); };
    B = std::max<int64_t>(B, 1);
    ev_cap = std::min<int64_t>(8 * B + 4096, int64_t(1) << 30);
    int64_t o = 0;
    counters = o; o = up(o + 64);   // 4 work counters + 8 diagnostic event counters
    fix_list = o; o = up(o + 8 * B);
    vflag = o; o = up(o + 4 * B);
    vres = o; o = up(o + 16 * B);
    vpath = o; o = up(o + 8 * B);
    events = o; o = up(o + 16 * ev_cap);
    lists = o; o = up(o + B * (int64_t)list_bytes);
    zq = o; o = up(o + B * 16 * (int64_t)((n + 1) / 2));
    thrg = o; o = up(o + B * 4 * (int64_t)((n + 3) & ~3));
    vaux = o; o = up(o + B * 8 + 16);   // +16: the traversal's aligned bulk-copy window
    total = o;
  }
};

}  // namespace

namespace mpnl {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace mpnl

// ------------------------------------------------------------------------------------------
extern "C" {

const char* mpnl_last_error(void) { return g_err.c_str(); }

int mpnl_version(void) { return 0x000100; }

int mpnl_alloc_expansions(int n_layers, int q, int64_t n_paths, int n_forced,
                          int64_t* expansions_out, int64_t* realized_out, int* warned) {
  if (n_paths < 1) return fail(MPNL_EINVAL, "n_paths must be >= 1");
  if (n_layers < 1 || q < 2) return fail(MPNL_EINVAL, "n_layers must be >= 1 and q >= 2");
  const int64_t cap = int64_t(1) << 40;
  const int64_t full = ipow_sat(q, n_layers, cap);
  if (full <= cap) n_paths = std::min(n_paths, full);
  if (warned) *warned = 0;
  if (n_forced > 0) {
    const int64_t qf = ipow_sat(q, n_forced, cap);
    if (n_paths < qf && warned) *warned = 1;
  }
  const int forced = std::min(n_forced, n_layers);
  for (int64_t target = n_paths; target >= 1; --target) {
    std::vector<int64_t> fac;
    int64_t budget = target;
    bool ok = true;
    for (int i = 0; i < forced; ++i) {
      if (budget >= q && budget % q == 0) { fac.push_back(q); budget /= q; }
      else if (budget >= q) { ok = false; break; }
      else { fac.push_back(budget); budget = 1; }
    }
    if (!ok) continue;
    std::vector<int64_t> rest;
    const int64_t cap0 = std::min<int64_t>(q, fac.empty() ? q : fac.back());
    if (!split_budget(budget, n_layers - forced, cap0, rest)) continue;
    fac.insert(fac.end(), rest.begin(), rest.end());
    while ((int)fac.size() < n_layers) fac.push_back(1);
    std::sort(fac.begin(), fac.end(), [](int64_t x, int64_t y) { return x > y; });
    for (int i = 0; i < n_layers; ++i) expansions_out[n_layers - 1 - i] = fac[i];
    *realized_out = target;
    return MPNL_OK;
  }
  return fail(MPNL_EINVAL, "unreachable: no representable path budget");
}

int64_t mpnl_tables_floats(int m, int n) { return TableLayout(m, n).total; }

int64_t mpnl_workspace_stats_offset(void) { return 16; }

int64_t mpnl_workspace_bytes(int64_t n_vectors, int n, int q, const int64_t* expansions) {
  const int L = levels_for(q);
  if (!L || n < 1 || n > MPNL_MAX_N) return -1;
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return -1;
  return Workspace(n_vectors, tb.tp.list_bytes, n).total;
}

int mpnl_plan(const void* h, int h_is_f64, int64_t n_ch, int m, int n, int q, double noise_var,
              int32_t* perm, void* r64, void* qh64, float* tables, void* stream) {
  if (int rc = check_dims(m, n, q)) return rc;
  if (n_ch < 0) return fail(MPNL_EINVAL, "negative batch");
  if (n > m && !(noise_var > 0)) return fail(MPNL_EINVAL, "noise_var must be positive");
  cudaError_t e = launch_plan(h, h_is_f64, n_ch, m, n, levels_for(q), noise_var, n > m ? 1 : 0,
                              perm, (double2*)r64, (double2*)qh64, tables, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "plan kernel");
  return MPNL_OK;
}

int mpnl_detect_hard_stage(int stage, const int32_t* perm, const void* r64, const void* qh64,
                           const float* tables, const void* y, int y_is_f64, int64_t n_ch,
                           int64_t v_per_ch, int m, int n, int q, const int64_t* expansions,
                           double noise_var, uint8_t* hard, float* metric, uint8_t* flags,
                           void* workspace, int64_t workspace_bytes, void* stream) {
  if (int rc = check_dims(m, n, q)) return rc;
  const int L = levels_for(q);
  const int64_t B = n_ch * v_per_ch;
  if (n_ch < 0 || v_per_ch < 0) return fail(MPNL_EINVAL, "negative batch");
  if (B == 0) return MPNL_OK;
  if (B > 0x7fffffffLL) return fail(MPNL_EUNSUPPORTED, "more than 2^31 vectors per call");
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return fail(MPNL_EINVAL, tb.err);
  const TreeParams& tp = tb.tp;
  const Workspace W(B, tp.list_bytes, n);
  if (workspace_bytes < W.total) return fail(MPNL_EINVAL, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = reinterpret_cast<char*>(workspace);
  DetectArgs a;
  std::memset(&a, 0, sizeof(a));
  a.tables = tables;
  a.y = y;
  a.y_f64 = y_is_f64;
  a.perm = perm;
  a.r64 = (const double2*)r64;
  a.qh64 = (const double2*)qh64;
  a.hard = hard;
  a.metric = metric;
  a.counters = reinterpret_cast<int32_t*>(ws + W.counters);
  a.fix_list = reinterpret_cast<int64_t*>(ws + W.fix_list);
  a.vflag = reinterpret_cast<uint32_t*>(ws + W.vflag);
  a.vres = reinterpret_cast<float4*>(ws + W.vres);
  a.vpath = reinterpret_cast<int2*>(ws + W.vpath);
  a.events = reinterpret_cast<int4*>(ws + W.events);
  a.lists = reinterpret_cast<uint8_t*>(ws + W.lists);
  a.zq = reinterpret_cast<float4*>(ws + W.zq);
  a.thrg = reinterpret_cast<float*>(ws + W.thrg);
  a.vaux = reinterpret_cast<float2*>(ws + W.vaux);
  a.stats = a.counters + 4;   // diagnostic counters (mpnl_workspace_stats)
  a.n_ch = n_ch;
  a.V = v_per_ch;
  a.m = m;
  a.ev_cap = (int)W.ev_cap;
  a.metric_offset = m > n;
  a.guard_scale = 1.0f;   // rigorous fp32 error bound
  // overloaded channels and trees with more than MPNL_XMAX expanded layers
  // (e.g. full enumeration) are detected entirely by the fp64 kernel
  const bool augmented = n > m;
  const bool slow = augmented || tp.n_top > MPNL_XMAX ||
                    TravSmem(m, n, 4, MPNL_VPI_MAX, tp.list_bytes).total_bytes > 160 * 1024;
  cudaError_t e = cudaSuccess;
  if (stage == 1) {   // reset + partial-layer selection
    e = cudaMemsetAsync(a.counters, 0, 64, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.vflag, 0, 4 * B, st);
    if (e != cudaSuccess) return cuda_fail(e, "memset");
    if (slow) return MPNL_OK;
    // partial (1 < e < Q) layers among the expanded ones; the top one is
    // selected inside the fused prep kernel when it is the top layer or sits
    // right below a full top layer, any other by the generic select kernel
    int fused = -1;
    for (int pos = n - 1; pos >= n - tp.n_top; --pos) {
      if (tp.e[pos] == L * L) continue;
      if ((tp.e[pos] == 2 || tp.e[pos] == 4) &&
          (pos == n - 1 || (pos == n - 2 && tp.e[n - 1] == L * L)))
        fused = pos;
      break;
    }
    // one thread per vector for large batches; 4 (rows and parents split) when
    // a thread per vector would leave the SMs short of warps
    // (with no fused selection to divide, one thread per vector already pays at two CTAs per
    // SM: C4's 45,864 vectors 72 -> 51 us, C5 at 256-512 RBs -5% of the step; with 64 fused
    // parent selections per vector -- C3 -- four threads stay better until the SMs are full)
    const int tpv = B >= 148 * 128 * (fused < 0 ? 2 : 8) ? 1 : 4;
    const int64_t pch = (v_per_ch + 128 / tpv - 1) / (128 / tpv);
    if (n_ch * pch > 0x7fffffffLL) return fail(MPNL_EUNSUPPORTED, "grid too large");
    if (16 * (m + 2) * n + 128 * 16 * (m | 1) > 200 * 1024)
      return fail(MPNL_EUNSUPPORTED, "channel too large");
    e = launch_fast(n, L, 5, a, tp, 0, tpv, 0, fused, st);
    if (e != cudaSuccess) return cuda_fail(e, "prep kernel");
    for (int pos = n - 1; pos >= n - tp.n_top; --pos) {
      if (tp.e[pos] == L * L || pos == fused) continue;
      const int npar = tp.n_paths / tp.stride[pos + 1];
      const int px = std::min(npar, 128), vy = std::max(1, 128 / px);
      if (n_ch * ((v_per_ch + vy - 1) / vy) > 0x7fffffffLL || (npar + px - 1) / px > 65535)
        return fail(MPNL_EUNSUPPORTED, "selection grid too large");
      e = launch_fast(n, L, 0, a, tp, 0, 128, 0, pos, st);
      if (e != cudaSuccess) return cuda_fail(e, "select kernel");
    }
    return MPNL_OK;
  }
  if (stage == 2 || stage == 3) {
    if (slow) return MPNL_OK;
    const int pt = trav_pt(n), S = 32 * pt, P = tp.n_paths;
    int vpi = 1, bpv = 1;
    if (P < S && S % P == 0) vpi = std::min(S / P, MPNL_VPI_MAX);
    else bpv = (P + S - 1) / S;
    a.vpi = vpi;
    a.bpv = bpv;
    const int threads = 128, warps = threads / 32;
    const int nvi = (bpv > 1 || vpi == 1) ? 1 : vpi;
    const int64_t items = n_ch * ((v_per_ch + nvi - 1) / nvi);
    if (items > 0x7fffffffLL) return fail(MPNL_EUNSUPPORTED, "too many work items");
    // channels with fewer than two path batches per warp: a warp per channel
    a.wpc = ((v_per_ch + nvi - 1) / nvi) * (int64_t)bpv < 2 * warps && n_ch >= 2 * warps ? 1 : 0;
    if (stage == 2) {
      const TravSmem so(m, n, warps, nvi, tp.list_bytes, a.wpc != 0);
      e = launch_fast(n, L, 1, a, tp, 0, threads, so.total_bytes, (int)items, st);
      if (e != cudaSuccess) return cuda_fail(e, "traverse kernel");
    } else {
      // winners: one thread per vector; then events/ties: one warp per event
      const int64_t vb = (B + 127) / 128;
      e = launch_fast(n, L, 2, a, tp, (unsigned)vb, 128, 0, 0, st);
      if (e != cudaSuccess) return cuda_fail(e, "verify kernel");
      const int64_t cb = 148 * 16;   // capped at the resident capacity by the launcher
      e = launch_fast(n, L, 3, a, tp, (unsigned)cb, 128, 0, 0, st);
      if (e != cudaSuccess) return cuda_fail(e, "check kernel");
    }
    return MPNL_OK;
  }
  // stage 4: fp64 fix-up of the listed vectors (or of every vector on the slow path)
  ExactArgs ea;
  std::memset(&ea, 0, sizeof(ea));
  ea.r64 = (const double2*)r64;
  ea.qh64 = (const double2*)qh64;
  ea.perm = perm;
  ea.y = y;
  ea.y_f64 = y_is_f64;
  ea.n_ch = n_ch;
  ea.V = v_per_ch;
  ea.m = m;
  ea.n = n;
  ea.L = L;
  ea.noise_var = noise_var;
  ea.augmented = augmented;
  ea.hard = hard;
  ea.metric = metric;
  int grid;
  // one CTA per vector (grid-stride over the task list)
  if (slow) {
    ea.list = nullptr;
    ea.n_tasks = B;
    grid = (int)std::min<int64_t>(B, 148 * 8);
  } else {
    ea.list = a.fix_list;
    ea.count = a.counters;
    // a cluster of 4 CTAs per flagged vector when there are paths to divide (the latency
    // tail of the step: C5/P1024 fix-up 158 -> 86 us, C4 57 -> 41; below 256 paths the
    // cluster launch and its two barriers cost what the division saves)
    ea.split = tp.n_paths >= 256 ? 4 : 1;
    grid = 148 * 2;   // a handful of flagged vectors: few, long-lived CTAs
  }
  e = launch_exact(ea, tp, grid, st);
  if (e != cudaSuccess) return cuda_fail(e, "exact kernel");
  if (flags) {
    e = launch_flags(flags, a.vflag, B, slow ? 1 : 0, st);
    if (e != cudaSuccess) return cuda_fail(e, "flags kernel");
  }
  return MPNL_OK;
}

int mpnl_detect_hard(const int32_t* perm, const void* r64, const void* qh64, const float* tables,
                     const void* y, int y_is_f64, int64_t n_ch, int64_t v_per_ch, int m, int n,
                     int q, const int64_t* expansions, double noise_var, uint8_t* hard,
                     float* metric, uint8_t* flags, void* workspace, int64_t workspace_bytes,
                     void* stream) {
  for (int stage = 1; stage <= 4; ++stage) {
    const int rc = mpnl_detect_hard_stage(stage, perm, r64, qh64, tables, y, y_is_f64, n_ch,
                                          v_per_ch, m, n, q, expansions, noise_var, hard, metric,
                                          flags, workspace, workspace_bytes, stream);
    if (rc) return rc;
  }
  return MPNL_OK;
}

}  // extern "C"

// soft path: vectors whose partial-layer selection was a near-tie (EV_CUT events of
// the prep / select kernels) or that the event log dropped go to the fp64 list path
__global__ void soft_flag_kernel(const int4* __restrict__ events, const int32_t* __restrict__ counters,
                                 int ev_cap, const uint32_t* __restrict__ vflag, int64_t B,
                                 uint8_t* __restrict__ flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int nev = min(counters[1], ev_cap);
  for (int64_t k = i; k < nev; k += stride) {
    const int4 e = events[k];
    if (e.w == EV_CUT) flags[(unsigned)e.z] = 1;
  }
  for (int64_t k = i; k < B; k += stride)
    if (vflag[k]) flags[k] = 1;
}

extern "C" {

int mpnl_detect_llrs_fast(const int32_t* perm, const void* r64, const void* qh64,
                          const float* tables, const void* y, int y_is_f64, int64_t n_ch,
                          int64_t v_per_ch, int m, int n, int q, const int64_t* expansions,
                          double noise_var, double llr_noise_var, double clip, double* llr,
                          uint8_t* flags, void* workspace, int64_t workspace_bytes,
                          void* stream) {
  if (int rc = check_dims(m, n, q)) return rc;
  const int L = levels_for(q);
  const int64_t B = n_ch * v_per_ch;
  if (n_ch < 0 || v_per_ch < 0) return fail(MPNL_EINVAL, "negative batch");
  if (!(llr_noise_var > 0)) return fail(MPNL_EINVAL, "noise_var must be positive");
  if (B == 0) return MPNL_OK;
  if (B > 0x7fffffffLL) return fail(MPNL_EUNSUPPORTED, "more than 2^31 vectors per call");
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return fail(MPNL_EINVAL, tb.err);
  const TreeParams& tp = tb.tp;
  if (n > m || tp.n_top > MPNL_XMAX ||
      TravSmem(m, n, 4, MPNL_VPI_MAX, tp.list_bytes).total_bytes > 160 * 1024)
    return fail(MPNL_EUNSUPPORTED,
                "no fp32 path for this plan (overloaded channel or > 3 expanded layers): "
                "use mpnl_detect_full + mpnl_candidate_llrs");
  // reset + rotation + guard thresholds + partial-layer selection, as for the hard output
  if (int rc = mpnl_detect_hard_stage(1, perm, r64, qh64, tables, y, y_is_f64, n_ch, v_per_ch, m,
                                      n, q, expansions, noise_var, nullptr, nullptr, nullptr,
                                      workspace, workspace_bytes, stream))
    return rc;
  const Workspace W(B, tp.list_bytes, n);
  char* ws = reinterpret_cast<char*>(workspace);
  DetectArgs a;
  std::memset(&a, 0, sizeof(a));
  a.tables = tables;
  a.y = y;
  a.y_f64 = y_is_f64;
  a.perm = perm;
  a.r64 = (const double2*)r64;
  a.qh64 = (const double2*)qh64;
  a.counters = reinterpret_cast<int32_t*>(ws + W.counters);
  a.vflag = reinterpret_cast<uint32_t*>(ws + W.vflag);
  a.events = reinterpret_cast<int4*>(ws + W.events);
  a.ev_cap = (int)W.ev_cap;
  a.lists = reinterpret_cast<uint8_t*>(ws + W.lists);
  a.zq = reinterpret_cast<float4*>(ws + W.zq);
  a.thrg = reinterpret_cast<float*>(ws + W.thrg);
  a.vaux = reinterpret_cast<float2*>(ws + W.vaux);
  a.n_ch = n_ch;
  a.V = v_per_ch;
  a.m = m;
  a.soft.llr = llr;
  a.soft.flags = flags;
  a.soft.noise_var = llr_noise_var;
  a.soft.clip = clip;
  a.soft.vc = 8;   // vectors per CTA (two per warp): the 5 KB table slice is staged per CTA
  a.soft.chunks = (int)((v_per_ch + a.soft.vc - 1) / a.soft.vc);
  if (n_ch * (int64_t)a.soft.chunks > 0x7fffffffLL) return fail(MPNL_EUNSUPPORTED, "grid too large");
  cudaError_t e = launch_fast(n, L, 6, a, tp, 0, 128, 0, 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "soft llr kernel");
  soft_flag_kernel<<<148 * 4, 256, 0, (cudaStream_t)stream>>>(a.events, a.counters, a.ev_cap, a.vflag,
                                                            B, flags);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "soft flag kernel");
  return MPNL_OK;
}

int mpnl_detect_full(const int32_t* perm, const void* r64, const void* qh64, const void* y,
                     int y_is_f64, int64_t n_ch, int64_t v_per_ch, int m, int n, int q,
                     const int64_t* expansions, double noise_var, uint8_t* labels,
                     double* metrics, int64_t* best, void* stream) {
  if (int rc = check_dims(m, n, q)) return rc;
  const int L = levels_for(q);
  const int64_t B = n_ch * v_per_ch;
  if (B == 0) return MPNL_OK;
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return fail(MPNL_EINVAL, tb.err);
  ExactArgs ea;
  std::memset(&ea, 0, sizeof(ea));
  ea.r64 = (const double2*)r64;
  ea.qh64 = (const double2*)qh64;
  ea.perm = perm;
  ea.y = y;
  ea.y_f64 = y_is_f64;
  ea.n_ch = n_ch;
  ea.V = v_per_ch;
  ea.m = m;
  ea.n = n;
  ea.L = L;
  ea.noise_var = noise_var;
  ea.augmented = n > m;
  ea.n_tasks = B;
  ea.full_labels = labels;
  ea.full_metrics = metrics;
  ea.full_best = best;
  ea.exact_order = 1;
  const int grid = (int)std::min<int64_t>(B, 148 * 8);
  cudaError_t e = launch_exact(ea, tb.tp, grid, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "exact kernel");
  return MPNL_OK;
}

int mpnl_candidate_llrs(const uint8_t* labels, const double* metrics, int64_t n_vectors,
                        int64_t n_paths, int n, int q, double noise_var,
                        const double* noise_var_per_vector, double clip, double* llr_out,
                        void* stream) {
  if (n_paths < 1) return fail(MPNL_EINVAL, "empty candidate list");
  if (n < 1 || n_vectors < 0) return fail(MPNL_EINVAL, "inconsistent candidate list dimensions");
  if (n > MPNL_MAX_N) return fail(MPNL_EUNSUPPORTED, "N > 32 streams is not supported");
  const int L = levels_for(q);
  if (!L) return fail(MPNL_EUNSUPPORTED, "unsupported constellation order " + std::to_string(q));
  if (n_vectors == 0) return MPNL_OK;
  const int bps = q == 4 ? 2 : (q == 16 ? 4 : 6);
  cudaError_t e = launch_candidate_llrs(labels, metrics, n_vectors, n_paths, n, bps, noise_var,
                                        noise_var_per_vector, clip, llr_out,
                                        (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "candidate llr kernel");
  return MPNL_OK;
}

int mpnl_linear_detect(const void* h, const void* y, int64_t n_vectors, int m, int n, int q,
                       int mode, double noise_var, const double* noise_var_per_vector,
                       double clip, uint8_t* labels_out, double* llr_out, void* est_out,
                       int32_t* n_singular, void* stream) {
  if (mode != 0 && mode != 1)
    return fail(MPNL_EINVAL, "unknown linear mode " + std::to_string(mode));
  if (n < 1 || m < 1 || n_vectors < 0) return fail(MPNL_EINVAL, "inconsistent h/y dimensions");
  if (n > linear_max_n()) return fail(MPNL_EUNSUPPORTED, "N > 32 streams is not supported");
  const int L = levels_for(q);
  if (!L) return fail(MPNL_EUNSUPPORTED, "unsupported constellation order " + std::to_string(q));
  const int half = q == 4 ? 1 : (q == 16 ? 2 : 3);
  cudaError_t e = launch_linear_detect(h, y, n_vectors, m, n, half, mode, noise_var,
                                       noise_var_per_vector, clip, labels_out, llr_out, est_out,
                                       n_singular, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "linear detect kernel");
  return MPNL_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------
// Host-buffer drop-in: h, y and the outputs in (pinned) host memory.  Channels are
// processed in chunks through two device slots; three streams overlap the upload
// of chunk k+1, the plan + detection of chunk k (caller's stream) and the download
// of chunk k-1.  Results are identical to mpnl_plan + mpnl_detect_hard on the
// whole batch (channels and vectors are independent).
// ------------------------------------------------------------------------------------------
namespace {

struct HostSlot {   // one of the two per-chunk device slots
  int64_t y, hard, metric, ws, total;
  int64_t ws_bytes;
  HostSlot(int64_t C, int64_t V, int m, int n, int yb, int list_bytes) {
    auto up = [](int64_t x) { return (x + 255) & ~int64_t(255); };
    int64_t o = 0;
    y = o; o = up(o + C * V * m * yb);
    hard = o; o = up(o + C * V * n);
    metric = o; o = up(o + C * V * 4);
    ws_bytes = Workspace(C * V, list_bytes, n).total;
    ws = o; o = up(o + ws_bytes);
    total = o;
  }
};

struct HostPlan {   // the whole batch's channels and plans (planned once, up front)
  int64_t h, perm, r64, qh64, tables, total;
  HostPlan(int64_t n_ch, int m, int n, int hb) {
    auto up = [](int64_t x) { return (x + 255) & ~int64_t(255); };
    int64_t o = 0;
    h = o; o = up(o + n_ch * m * n * hb);
    perm = o; o = up(o + n_ch * n * 4);
    r64 = o; o = up(o + n_ch * n * n * 16);
    qh64 = o; o = up(o + n_ch * n * m * 16);
    tables = o; o = up(o + n_ch * TableLayout(m, n).total * 4);
    total = o;
  }
};

#define HOST_SLOTS 3
struct HostPipe {
  bool init = false;
  cudaStream_t up = nullptr, down = nullptr, cs[HOST_SLOTS];
  cudaEvent_t in_ready[HOST_SLOTS], done[HOST_SLOTS], out_done[HOST_SLOTS], fin, planned;
};
// streams/events are device objects: one pipe per (calling thread, device)
#define PIPE_MAX_DEV 16
thread_local HostPipe g_pipes[PIPE_MAX_DEV];
thread_local HostPipe* g_pipe_cur = nullptr;
#define g_pipe (*g_pipe_cur)

int pipe_init() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= PIPE_MAX_DEV)
    return fail(MPNL_ECUDA, "host pipeline: no current CUDA device");
  g_pipe_cur = &g_pipes[dev];
  if (g_pipe.init) return MPNL_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&g_pipe.up, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g_pipe.down, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_pipe.planned, cudaEventDisableTiming);
  for (int i = 0; i < HOST_SLOTS && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithFlags(&g_pipe.cs[i], cudaStreamNonBlocking);
    if (e != cudaSuccess) break;
    e = cudaEventCreateWithFlags(&g_pipe.in_ready[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_pipe.done[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_pipe.out_done[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_pipe.fin, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(e, "pipeline streams");
  g_pipe.init = true;
  return MPNL_OK;
}

}  // namespace

extern "C" int64_t mpnl_host_workspace_bytes(int64_t n_ch, int64_t chunk_channels,
                                             int64_t v_per_ch, int m, int n, int q,
                                             int h_is_f64, int y_is_f64,
                                             const int64_t* expansions) {
  const int L = levels_for(q);
  if (!L || n < 1 || n > MPNL_MAX_N || chunk_channels < 1 || n_ch < 0) return -1;
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return -1;
  const HostSlot hs(std::min(chunk_channels, std::max<int64_t>(n_ch, 1)), v_per_ch, m, n,
                    y_is_f64 ? 16 : 8, tb.tp.list_bytes);
  return HostPlan(n_ch, m, n, h_is_f64 ? 16 : 8).total + HOST_SLOTS * hs.total;
}

extern "C" int mpnl_detect_hard_host(const void* h, int h_is_f64, const void* y, int y_is_f64,
                                     int64_t n_ch, int64_t v_per_ch, int m, int n, int q,
                                     const int64_t* expansions, double noise_var, uint8_t* hard,
                                     float* metric, int64_t chunk_channels, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  if (int rc = check_dims(m, n, q)) return rc;
  if (n_ch < 0 || v_per_ch < 0) return fail(MPNL_EINVAL, "negative batch");
  if (n_ch == 0 || v_per_ch == 0) return MPNL_OK;
  if (chunk_channels < 1) return fail(MPNL_EINVAL, "chunk_channels must be >= 1");
  const int L = levels_for(q);
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return fail(MPNL_EINVAL, tb.err);
  const int64_t C = std::min(chunk_channels, n_ch);
  const int hb = h_is_f64 ? 16 : 8, yb = y_is_f64 ? 16 : 8;
  const HostPlan hp(n_ch, m, n, hb);
  const HostSlot hs(C, v_per_ch, m, n, yb, tb.tp.list_bytes);
  if (workspace_bytes < hp.total + HOST_SLOTS * hs.total)
    return fail(MPNL_EINVAL, "workspace too small");
  if (int rc = pipe_init()) return rc;
  cudaStream_t comp = (cudaStream_t)stream, up = g_pipe.up, down = g_pipe.down;
  char* pb = reinterpret_cast<char*>(workspace);
  char* base = pb + hp.total;
  const int64_t tf = TableLayout(m, n).total;
  cudaError_t e = cudaSuccess;
  // the uploads must not start before work already queued on the caller's stream
  e = cudaEventRecord(g_pipe.fin, comp);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(up, g_pipe.fin, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(down, g_pipe.fin, 0);
  // all channels first (small), planned in one launch while the observations stream in
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(pb + hp.h, h, n_ch * m * n * hb, cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess) e = cudaEventRecord(g_pipe.fin, up);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, g_pipe.fin, 0);
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline");
  if (int rc = mpnl_plan(pb + hp.h, h_is_f64, n_ch, m, n, q, noise_var,
                         reinterpret_cast<int32_t*>(pb + hp.perm), pb + hp.r64, pb + hp.qh64,
                         reinterpret_cast<float*>(pb + hp.tables), comp))
    return rc;
  e = cudaEventRecord(g_pipe.planned, comp);
  for (int i = 0; i < HOST_SLOTS && e == cudaSuccess; ++i)
    e = cudaStreamWaitEvent(g_pipe.cs[i], g_pipe.planned, 0);
  // chunk schedule: tapered ends (a quarter chunk first and last) when the batch
  // spans more than two chunks, so the kernels start after a short first upload
  // and the un-overlapped tail (last chunk's kernels + download) stays short
  std::vector<int64_t> starts;
  {
    const int64_t taper = std::max<int64_t>(1, C / 4);
    const bool tap = n_ch > 2 * C;
    int64_t pos = 0;
    if (tap) { starts.push_back(0); pos = taper; }
    while (pos < n_ch) {
      starts.push_back(pos);
      const int64_t rem = n_ch - pos;
      pos += (tap && rem > taper && rem <= C + taper) ? rem - taper : std::min(C, rem);
    }
  }
  const int64_t K = (int64_t)starts.size();
  for (int64_t k = 0; k < K && e == cudaSuccess; ++k) {
    const int sl = (int)(k % HOST_SLOTS);
    cudaStream_t cst = g_pipe.cs[sl];   // one compute stream per slot: chunk tails overlap
    char* sb = base + sl * hs.total;
    const int64_t c0 = starts[k], cn = (k + 1 < K ? starts[k + 1] : n_ch) - c0;
    // upload (slot free once the compute of its previous chunk is done)
    if (k >= HOST_SLOTS) e = cudaStreamWaitEvent(up, g_pipe.done[sl], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(sb + hs.y, (const char*)y + c0 * v_per_ch * m * yb,
                          cn * v_per_ch * m * yb, cudaMemcpyHostToDevice, up);
    if (e == cudaSuccess) e = cudaEventRecord(g_pipe.in_ready[sl], up);
    // detect (outputs free once the slot's previous chunk is downloaded)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cst, g_pipe.in_ready[sl], 0);
    if (e == cudaSuccess && k >= HOST_SLOTS) e = cudaStreamWaitEvent(cst, g_pipe.out_done[sl], 0);
    if (e != cudaSuccess) break;
    const int rc = mpnl_detect_hard(
        reinterpret_cast<int32_t*>(pb + hp.perm) + c0 * n,
        reinterpret_cast<double2*>(pb + hp.r64) + c0 * n * n,
        reinterpret_cast<double2*>(pb + hp.qh64) + c0 * n * m,
        reinterpret_cast<float*>(pb + hp.tables) + c0 * tf, sb + hs.y, y_is_f64, cn, v_per_ch,
        m, n, q, expansions, noise_var, reinterpret_cast<uint8_t*>(sb + hs.hard),
        reinterpret_cast<float*>(sb + hs.metric), nullptr, sb + hs.ws, hs.ws_bytes, cst);
    if (rc) return rc;
    e = cudaEventRecord(g_pipe.done[sl], cst);
    // download
    if (e == cudaSuccess) e = cudaStreamWaitEvent(down, g_pipe.done[sl], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hard + c0 * v_per_ch * n, sb + hs.hard, cn * v_per_ch * n,
                          cudaMemcpyDeviceToHost, down);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(metric + c0 * v_per_ch, sb + hs.metric, cn * v_per_ch * 4,
                          cudaMemcpyDeviceToHost, down);
    if (e == cudaSuccess) e = cudaEventRecord(g_pipe.out_done[sl], down);
  }
  // the caller's stream completes after the last download
  if (e == cudaSuccess) e = cudaEventRecord(g_pipe.fin, down);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, g_pipe.fin, 0);
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline");
  return MPNL_OK;
}

// ------------------------------------------------------------------------------------------
// Device-buffer plan + hard detection of a whole batch in channel groups on forked
// streams.  Channels are independent, so group g's latency-bound stages (plan, the
// verify/check of its events, the fp64 fix-up of its few flagged vectors) overlap
// the other groups' traversal instead of idling the GPU between dependent launches.
// Results are identical to mpnl_plan + mpnl_detect_hard on the whole batch.
// ------------------------------------------------------------------------------------------
namespace {
#define GROUP_MAX 4
struct GroupPipe {
  bool init = false;
  cudaStream_t gs[GROUP_MAX];
  cudaEvent_t fork, done[GROUP_MAX];
};
thread_local GroupPipe g_grps[PIPE_MAX_DEV];   // per (calling thread, device)
thread_local GroupPipe* g_grp_cur = nullptr;
#define g_grp (*g_grp_cur)

int group_init() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= PIPE_MAX_DEV)
    return fail(MPNL_ECUDA, "group streams: no current CUDA device");
  g_grp_cur = &g_grps[dev];
  if (g_grp.init) return MPNL_OK;
  int lo = 0, hi = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);   // hi = greatest priority
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_grp.fork, cudaEventDisableTiming);
  for (int i = 0; i < GROUP_MAX && e == cudaSuccess; ++i) {
    // earlier groups first: their short tail kernels take free SM slots ahead
    // of the next group's traversal CTAs
    const int pr = std::min(lo, hi + i);
    e = cudaStreamCreateWithPriority(&g_grp.gs[i], cudaStreamNonBlocking, pr);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_grp.done[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(e, "group streams");
  g_grp.init = true;
  return MPNL_OK;
}

struct GroupLayout {
  HostPlan plan;
  int64_t ws0, ws_bytes, total;
  GroupLayout(int64_t n_ch, int64_t v, int m, int n, int groups, int list_bytes)
      : plan(n_ch, m, n, 0) {
    const int64_t cg = (n_ch + groups - 1) / groups;
    ws_bytes = (Workspace(cg * v, list_bytes, n).total + 255) & ~int64_t(255);
    ws0 = plan.total;
    total = ws0 + groups * ws_bytes;
  }
};
}  // namespace

extern "C" int64_t mpnl_group_workspace_bytes(int64_t n_ch, int64_t v_per_ch, int m, int n,
                                              int q, const int64_t* expansions, int groups) {
  const int L = levels_for(q);
  if (!L || n < 1 || n > MPNL_MAX_N || n_ch < 0 || groups < 1 || groups > GROUP_MAX) return -1;
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return -1;
  return GroupLayout(n_ch, v_per_ch, m, n, groups, tb.tp.list_bytes).total;
}

extern "C" int mpnl_plan_detect_hard(const void* h, int h_is_f64, const void* y, int y_is_f64,
                                     int64_t n_ch, int64_t v_per_ch, int m, int n, int q,
                                     const int64_t* expansions, double noise_var, uint8_t* hard,
                                     float* metric, int groups, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  if (int rc = check_dims(m, n, q)) return rc;
  if (n_ch < 0 || v_per_ch < 0) return fail(MPNL_EINVAL, "negative batch");
  if (groups < 1 || groups > GROUP_MAX) return fail(MPNL_EINVAL, "groups must be in 1..4");
  if (n_ch == 0 || v_per_ch == 0) return MPNL_OK;
  const int L = levels_for(q);
  TreeBuild tb = build_tree(n, L, expansions);
  if (!tb.ok) return fail(MPNL_EINVAL, tb.err);
  const int G = (int)std::min<int64_t>(groups, n_ch);
  const GroupLayout gl(n_ch, v_per_ch, m, n, G, tb.tp.list_bytes);
  if (workspace_bytes < gl.total) return fail(MPNL_EINVAL, "workspace too small");
  if (int rc = group_init()) return rc;
  cudaStream_t main = (cudaStream_t)stream;
  char* pb = reinterpret_cast<char*>(workspace);
  const int64_t tf = TableLayout(m, n).total;
  const int hb = h_is_f64 ? 16 : 8, yb = y_is_f64 ? 16 : 8;
  const int64_t cg = (n_ch + G - 1) / G;
  cudaError_t e = cudaEventRecord(g_grp.fork, main);
  for (int g = 0; g < G && e == cudaSuccess; ++g) {
    const int64_t c0 = g * cg, cn = std::min(cg, n_ch - c0);
    if (cn <= 0) break;
    cudaStream_t st = g_grp.gs[g];
    e = cudaStreamWaitEvent(st, g_grp.fork, 0);
    if (e != cudaSuccess) break;
    int32_t* perm = reinterpret_cast<int32_t*>(pb + gl.plan.perm) + c0 * n;
    double2* r64 = reinterpret_cast<double2*>(pb + gl.plan.r64) + c0 * n * n;
    double2* qh64 = reinterpret_cast<double2*>(pb + gl.plan.qh64) + c0 * n * m;
    float* tab = reinterpret_cast<float*>(pb + gl.plan.tables) + c0 * tf;
    if (int rc = mpnl_plan((const char*)h + c0 * m * n * hb, h_is_f64, cn, m, n, q, noise_var,
                           perm, r64, qh64, tab, st))
      return rc;
    if (int rc = mpnl_detect_hard(perm, r64, qh64, tab, (const char*)y + c0 * v_per_ch * m * yb,
                                  y_is_f64, cn, v_per_ch, m, n, q, expansions, noise_var,
                                  hard + c0 * v_per_ch * n, metric + c0 * v_per_ch, nullptr,
                                  pb + gl.ws0 + g * gl.ws_bytes, gl.ws_bytes, st))
      return rc;
    e = cudaEventRecord(g_grp.done[g], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(main, g_grp.done[g], 0);
  }
  if (e != cudaSuccess) return cuda_fail(e, "group streams");
  return MPNL_OK;
}

// ---- FFMA throughput probe (roofline denominator) ----
__global__ void ffma_probe_kernel(float* out, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
  float x4 = x0 + 4.f, x5 = x0 + 5.f, x6 = x0 + 6.f, x7 = x0 + 7.f;
  const float a = 0.999999f, b = 1e-7f;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// packed FFMA2 throughput (the instruction the traversal is built on):
// 8 independent f32x2 accumulators, a register pair and a broadcast operand
__global__ void ffma2_probe_kernel(float* out, int iters) {
  typedef unsigned long long u64;
  auto pk = [](float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
  };
  auto fma2 = [](u64 a, u64 b, u64 c) {
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
  };
  const float t = threadIdx.x * 1e-3f;
  const u64 x = pk(0.999999f + t * 1e-9f, 0.999998f), b = pk(1e-7f, 1e-7f);
  u64 a0 = pk(t, t + 1.f), a1 = pk(t + 2.f, t + 3.f), a2 = pk(t + 4.f, t + 5.f),
      a3 = pk(t + 6.f, t + 7.f), a4 = pk(t + 8.f, t + 9.f), a5 = pk(t + 10.f, t + 11.f),
      a6 = pk(t + 12.f, t + 13.f), a7 = pk(t + 14.f, t + 15.f);
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    a0 = fma2(a0, x, b); a1 = fma2(a1, x, b); a2 = fma2(a2, x, b); a3 = fma2(a3, x, b);
    a4 = fma2(a4, x, b); a5 = fma2(a5, x, b); a6 = fma2(a6, x, b); a7 = fma2(a7, x, b);
  }
  const u64 s = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float((unsigned)s);
}

extern "C" int64_t mpnl_ffma2_probe(float* out, int blocks, int threads, int iters, void* stream) {
  ffma2_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, iters);
  if (cudaGetLastError() != cudaSuccess) return -1;
  return (int64_t)blocks * threads * iters * 8 * 2 * 2;
}

extern "C" int64_t mpnl_ffma_probe(float* out, int blocks, int threads, int iters, void* stream) {
  ffma_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, iters);
  if (cudaGetLastError() != cudaSuccess) return -1;
  return (int64_t)blocks * threads * iters * 8 * 2;
}
