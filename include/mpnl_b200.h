/*
 * mpnl_b200 — C ABI of the B200-native MPNL parallel-path MIMO detector.
 *
 * Plain pointers and sizes only.  Device pointers are CUDA device memory
 * (e.g. torch.Tensor.data_ptr()), `stream` is a cudaStream_t (0 = legacy).
 * Every call returns 0 on success, a negative MPNL_E* code otherwise;
 * mpnl_last_error() gives the message of the calling thread's last failure.
 *
 * Reference interfaces replaced (the Python package `mpnlsim`, detect.py):
 *   mpnl_alloc_expansions  <- allocate_expansions   detect.py:221-280
 *   mpnl_plan              <- mpnl_plan_batch / _sorted_qr_batch
 *                                                    detect.py:321-388
 *   mpnl_detect_hard       <- mpnl_detect_batch + take_along_axis(labels, best)
 *                             (the hard-output composition of cli.py:236-239
 *                              and test_acceptance.py:114-117)
 *   mpnl_detect_full       <- mpnl_detect_batch      detect.py:473-488
 *   mpnl_candidate_llrs    <- _candidate_llrs_batch  detect.py:439-453
 *   mpnl_detect_llrs_fast  <- mpnl_detect_batch + _candidate_llrs_batch, the link
 *                             simulator's MPNL soft output (linksim.py:151-155),
 *                             in fp32 without the candidate list
 *   mpnl_linear_detect     <- linear_detect_batch    detect.py:528-557
 * INTEGRATION.md shows the ctypes binding a maintainer adds to detect.py.
 */
#ifndef MPNL_B200_H
#define MPNL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPNL_OK 0
#define MPNL_EINVAL (-1)      /* invalid argument (reference: ValueError)      */
#define MPNL_EUNSUPPORTED (-2) /* N > 32, M > 64, Q not in {4,16,64}          */
#define MPNL_ECUDA (-3)       /* CUDA runtime error                            */

/* Last error message of the calling thread ("" if none). */
const char* mpnl_last_error(void);

/* Library / ABI version, e.g. 0x000100 for 0.1.0. */
int mpnl_version(void);

/* Per-layer expansion counts (indexed by tree position, n_layers-1 = top) and
 * the realized path count.  *warned = 1 when n_paths < q^n_forced (the
 * reference's UserWarning).  Errors: n_paths < 1 -> MPNL_EINVAL
 * ("n_paths must be >= 1").  Host function. */
int mpnl_alloc_expansions(int n_layers, int q, int64_t n_paths, int n_forced,
                          int64_t* expansions_out, int64_t* realized_out,
                          int* warned);

/* floats per channel of the fp32 traversal table blob. */
int64_t mpnl_tables_floats(int m, int n);

/* Plan n_ch channels h (n_ch, m, n) row-major complex64 (h_is_f64 = 0) or
 * complex128 (1).  Augmented planning ([H; sqrt(nv) I]) when n > m.
 * Outputs (device): perm (n_ch, n) int32, r64 (n_ch, n, n) complex128,
 * qh64 (n_ch, n, m) complex128, tables (n_ch, mpnl_tables_floats) float32. */
int mpnl_plan(const void* h, int h_is_f64, int64_t n_ch, int m, int n, int q,
              double noise_var, int32_t* perm, void* r64, void* qh64,
              float* tables, void* stream);

/* Scratch bytes mpnl_detect_hard needs for n_vectors received vectors of a
 * plan with these expansions (-1 on invalid arguments). */
int64_t mpnl_workspace_bytes(int64_t n_vectors, int n, int q,
                             const int64_t* expansions);

/* Hard-output detection of y (n_ch, v_per_ch, m) (complex64 or complex128)
 * against the plan: writes hard (n_ch*v_per_ch, n) uint8 point labels in
 * stream order and metric (n_ch*v_per_ch) float32 = ||y - H x_hat||^2.
 * expansions: host array of n int64 (from mpnl_alloc_expansions).
 * flags (optional, may be NULL): 1 where the fp32 pass was re-done in fp64.
 * Launches stages 1-4 of mpnl_detect_hard_stage in order (no host sync). */
int mpnl_detect_hard(const int32_t* perm, const void* r64, const void* qh64,
                     const float* tables, const void* y, int y_is_f64,
                     int64_t n_ch, int64_t v_per_ch, int m, int n, int q,
                     const int64_t* expansions, double noise_var,
                     uint8_t* hard, float* metric, uint8_t* flags,
                     void* workspace, int64_t workspace_bytes, void* stream);

/* The stages of mpnl_detect_hard, for timing (all four, in order, equal
 * mpnl_detect_hard): 1 = reset + fp64 rotation/guard-bound kernel +
 * partial-layer selection kernel, 2 = fp32 traversal kernel (the hot kernel),
 * 3 = verification kernel (winner labels, near-ties) + fp64 re-decision of
 * guarded decisions, 4 = fp64 fix-up kernel (+ flags). */
int mpnl_detect_hard_stage(int stage, const int32_t* perm, const void* r64,
                           const void* qh64, const float* tables, const void* y,
                           int y_is_f64, int64_t n_ch, int64_t v_per_ch, int m,
                           int n, int q, const int64_t* expansions,
                           double noise_var, uint8_t* hard, float* metric,
                           uint8_t* flags, void* workspace,
                           int64_t workspace_bytes, void* stream);

/* Host-buffer drop-in for the reference's numpy call sites (cli.py:236-239):
 * h (n_ch, m, n), y (n_ch, v_per_ch, m) and the outputs hard (n_ch*v_per_ch, n)
 * uint8 / metric float32 live in HOST memory (pinned for asynchronous
 * copies).  Uploads all channels and plans them in one launch, then detects
 * chunk_channels channels at a time through two device slots, overlapping the
 * upload of the next chunk's observations, the computation of the current one
 * (on `stream`) and the download of the previous one.  Same
 * results as mpnl_plan + mpnl_detect_hard on the whole batch.  The outputs
 * are complete when `stream` reaches this point. */
int64_t mpnl_host_workspace_bytes(int64_t n_ch, int64_t chunk_channels, int64_t v_per_ch,
                                  int m, int n, int q, int h_is_f64, int y_is_f64,
                                  const int64_t* expansions);
int mpnl_detect_hard_host(const void* h, int h_is_f64, const void* y, int y_is_f64,
                          int64_t n_ch, int64_t v_per_ch, int m, int n, int q,
                          const int64_t* expansions, double noise_var, uint8_t* hard,
                          float* metric, int64_t chunk_channels, void* workspace,
                          int64_t workspace_bytes, void* stream);

/* Device-buffer plan + hard detection of a whole batch (the cli._bench_chunk
 * call, cli.py:236-239, on device-resident h and y): the channels are split
 * into `groups` (1..4) contiguous ranges, each planned and detected on its own
 * internal stream forked from / joined back into `stream`, so one group's
 * latency-bound stages overlap another's traversal.  Same results as
 * mpnl_plan + mpnl_detect_hard on the whole batch.  Workspace: device bytes
 * from mpnl_group_workspace_bytes (plans of all channels + one detection
 * workspace per group). */
int64_t mpnl_group_workspace_bytes(int64_t n_ch, int64_t v_per_ch, int m, int n, int q,
                                   const int64_t* expansions, int groups);
int mpnl_plan_detect_hard(const void* h, int h_is_f64, const void* y, int y_is_f64,
                          int64_t n_ch, int64_t v_per_ch, int m, int n, int q,
                          const int64_t* expansions, double noise_var, uint8_t* hard,
                          float* metric, int groups, void* workspace,
                          int64_t workspace_bytes, void* stream);

/* Full candidate list (reference-compatible mpnl_detect_batch), fp64:
 * labels (B, P, n) uint8 in path order and stream order, metrics (B, P)
 * float64, best (B,) int64, B = n_ch * v_per_ch, P = prod(expansions). */
int mpnl_detect_full(const int32_t* perm, const void* r64, const void* qh64,
                     const void* y, int y_is_f64, int64_t n_ch,
                     int64_t v_per_ch, int m, int n, int q,
                     const int64_t* expansions, double noise_var,
                     uint8_t* labels, double* metrics, int64_t* best,
                     void* stream);

/* fp32 list max-log LLRs fused with the path traversal: the MPNL soft output
 * of the link simulator (linksim.py:151-155 = mpnl_detect_batch, detect.py:473-488,
 * then _candidate_llrs_batch, detect.py:439-453) without materialising the
 * candidate list.  Plan and observation arguments as mpnl_detect_hard;
 * llr_noise_var and clip are _candidate_llrs_batch's noise_var and clip.
 * llr_out (B, n, log2 q) float64 and flags_out (B,) uint8 are device buffers.
 * Path metrics are the traversal's fp32 PEDs: an LLR differs from the
 * reference's by at most 2 ped_tol / noise_var (about 1e-6 relative to the
 * metrics).  flags_out[b] = 1 marks a vector in which an fp32 decision within
 * the guard bound of a decision boundary sits on a path that can reach an
 * unclipped LLR: recompute those vectors with mpnl_detect_full +
 * mpnl_candidate_llrs (the Python shim does) and every LLR is then the
 * reference's within that tolerance.
 * Errors: overloaded channels (n > m) and plans with more than 3 expanded layers
 * have no fp32 path -> MPNL_EUNSUPPORTED. */
int mpnl_detect_llrs_fast(const int32_t* perm, const void* r64, const void* qh64,
                          const float* tables, const void* y, int y_is_f64, int64_t n_ch,
                          int64_t v_per_ch, int m, int n, int q, const int64_t* expansions,
                          double noise_var, double llr_noise_var, double clip, double* llr_out,
                          uint8_t* flags_out, void* workspace, int64_t workspace_bytes,
                          void* stream);

/* List max-log LLRs over a candidate list (replaces _candidate_llrs_batch,
 * detect.py:439-453; bits as bits_from_labels, core.py:209-213, MSB first).
 * labels (B, P, n) uint8 and metrics (B, P) float64 as mpnl_detect_full
 * writes them (device); llr_out (B, n, log2 q) float64 (device).  noise_var
 * is used when noise_var_per_vector is NULL, else that device float64 (B,)
 * array is (the reference's array-valued noise_var).  Bit-identical to the
 * reference: bits no path sets/clears saturate at +-clip.
 * Errors: P < 1 -> MPNL_EINVAL ("empty candidate list"). */
int mpnl_candidate_llrs(const uint8_t* labels, const double* metrics, int64_t n_vectors,
                        int64_t n_paths, int n, int q, double noise_var,
                        const double* noise_var_per_vector, double clip, double* llr_out,
                        void* stream);

/* Batched linear ZF (mode 0) / MMSE (mode 1) detection with max-log LLRs
 * (replaces linear_detect_batch, detect.py:528-557).  Device pointers:
 * h (B,M,N) and y (B,M) complex128 (interleaved re/im), noise_var scalar or
 * per vector (noise_var_per_vector, B doubles, or NULL).  Outputs: labels
 * uint8 (B,N) nearest points, llr float64 (B,N,log2 Q) clipped to +-clip,
 * optional est complex128 (B,N) raw equalised symbols A^-1 H^H y (the biased
 * MMSE output, detect.py:129-136; NULL skips), optional
 * device int32 *n_singular += vectors whose A had an exactly zero (or
 * non-finite) Cholesky pivot, where the reference's np.linalg.inv (LAPACK
 * getrf) raises LinAlgError.
 * Errors: unknown mode -> MPNL_EINVAL; N > 32 or Q not in {4,16,64} -> MPNL_EUNSUPPORTED. */
int mpnl_linear_detect(const void* h, const void* y, int64_t n_vectors, int m, int n, int q,
                       int mode, double noise_var, const double* noise_var_per_vector,
                       double clip, uint8_t* labels_out, double* llr_out, void* est_out,
                       int32_t* n_singular, void* stream);

/* Byte offset, inside the mpnl_detect_hard workspace, of eight int32
 * diagnostic counters the last call on that workspace left (valid once the
 * stream reaches the end of the call; reset by the next call): [0] events
 * logged, [1] guarded decisions re-decided in fp64, [2] two-way near-ties
 * settled in fp64, [3] vectors sent to the fp64 kernel, of which [4] three-way
 * ties, [5] fp64-level ties, [6] fp64 disagreements, [7] event-log overflows.
 * (There is no process-global state: all scratch lives in the caller's
 * workspace.) */
int64_t mpnl_workspace_stats_offset(void);

/* ---- LDPC stage after detection (mpnlsim fec.py) ---- */

/* Maximum check / variable degree of a dense m x n parity-check matrix H
 * (host, row-major uint8).  MPNL_EINVAL unless 1 <= m < n ("parity-check
 * matrix must be m x n with m < n"); MPNL_EUNSUPPORTED for degrees > 32 or
 * >= 65535 edges.  Replaces LdpcCode.__post_init__ / _graph (fec.py:91-133). */
int mpnl_ldpc_graph_dims(const uint8_t* H, int m, int n, int* max_dc, int* max_dv);

/* Host: the decoder graph and the systematic encoder of H.
 * check_vars (m*max_dc) uint16 variable of each check's slot, var_edges
 * (n*max_dv) uint16 flat edge index (check*max_dc + slot) of each variable's
 * slot — edges in np.nonzero order, 0xFFFF padding, as LdpcCode._graph
 * (fec.py:107-133); encoder (m * ceil(k/32)) uint32 rows of E (bit j of word
 * i = E[r, 32 i + j]), parity = E info mod 2 (fec.py:60-81, _encoder).
 * MPNL_EINVAL "parity submatrix is singular" as the reference's ValueError. */
int mpnl_ldpc_build(const uint8_t* H, int m, int n, int max_dc, int max_dv,
                    uint16_t* check_vars, uint16_t* var_edges, uint32_t* encoder);

/* Normalized min-sum decoding of n_words rate-matched words (replaces
 * ldpc_decode, fec.py:156-220, and decode_rate_matched, fec.py:296-326), fp64,
 * bit-identical to the reference.  Device: graph from mpnl_ldpc_build,
 * llr_tx (n_words, n_tx) float64 (positive = bit 0); mother positions
 * [0,k_tb) <- llr_tx[:, :k_tb], [k_tb,k) <- shortened_llr, [k,k+p) <-
 * llr_tx[:, k_tb:], rest 0 (punctured), p = n_tx - k_tb (plain ldpc_decode:
 * k_tb = k, n_tx = n).  Outputs: info_out (n_words, k_tb) uint8 bits of the
 * hard decision at convergence (else after max_iter iterations), converged
 * (n_words) uint8, iterations (optional, int32), *n_nonfinite (optional
 * device int32) += words with a non-finite LLR (the reference raises
 * ValueError("LLRs must be finite")). */
int mpnl_ldpc_decode(const uint16_t* check_vars, const uint16_t* var_edges, int m, int n,
                     int max_dc, int max_dv, const double* llr_tx, int64_t n_words, int n_tx,
                     int k_tb, int max_iter, double alpha, double shortened_llr,
                     uint8_t* info_out, uint8_t* converged, int32_t* iterations,
                     int32_t* n_nonfinite, void* stream);

/* Systematic (rate-matched) encoding (replaces ldpc_encode, fec.py:136-148,
 * and encode_rate_matched, fec.py:278-293): info (n_words, k_tb) uint8 bits,
 * zero-padded to k, tx_out (n_words, n_tx) = [info, parity[0, n_tx - k_tb)]. */
int mpnl_ldpc_encode(const uint32_t* encoder, int m, int n, const uint8_t* info,
                     int64_t n_words, int k_tb, int n_tx, uint8_t* tx_out, void* stream);

/* Syndrome (n_words, m) uint8 of bits (n_words, n) (replaces ldpc_syndrome,
 * fec.py:151-153). */
int mpnl_ldpc_syndrome(const uint16_t* check_vars, int m, int max_dc, const uint8_t* bits,
                       int64_t n_words, int n, uint8_t* syndrome_out, void* stream);

/* ---- slot I/O around the detector (mpnlsim linksim.py) ---- */

/* Receive grid y (frames, S, SC, m) = H x + noise per resource element
 * (replaces linksim.py:207, einsum "tfmn,btfn->btfm" + noise): device
 * complex128 h (S, SC, m, n), x (frames, S, SC, n), noise (frames, S, SC, m)
 * or NULL. */
int mpnl_slot_receive(const void* h, const void* x, const void* noise, int64_t frames,
                      int symbols, int subcarriers, int m, int n, void* y, void* stream);

/* DMRS least-squares channel estimate (replaces estimate_channel_ls,
 * linksim.py:117-137): grid_obs (S, SC, m) complex128, pilots (n, n_pilot)
 * complex128, port_symbol (n) int32 DMRS symbol of each stream, port_subcarriers
 * (n, n_pilot) int32 its pilot subcarriers (device).  h_est (S, SC, m, n):
 * obs / pilot (numpy's complex division, bit-identical) at the nearest pilot
 * subcarrier (first minimum), the same for every symbol. */
int mpnl_dmrs_ls_estimate(const void* grid_obs, const void* pilots, const int32_t* port_symbol,
                          const int32_t* port_subcarriers, int symbols, int subcarriers, int m,
                          int n, int n_pilot, void* h_est, void* stream);

/* Gather the rows `rows` (device int32, n_rows) of a (batch, symbols, row)
 * grid into (batch, n_rows, row): the per-RE flattening of the data symbols
 * (h[data_syms], y[:, data_syms], linksim.py:211-216).  row_bytes % 16 == 0. */
int mpnl_select_symbols(const void* src, int64_t batch, int symbols, int64_t row_bytes,
                        const int32_t* rows, int n_rows, void* dst, void* stream);

/* FFMA throughput probe (for the roofline denominator): runs `iters` dependent
 * FFMA chains on every SM; returns FLOPs executed.  out: device float[blocks*threads]. */
int64_t mpnl_ffma_probe(float* out, int blocks, int threads, int iters, void* stream);

/* Same for the packed fma.rn.f32x2 (FFMA2) instruction the traversal uses. */
int64_t mpnl_ffma2_probe(float* out, int blocks, int threads, int iters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPNL_B200_H */
