/*
 * tnsample.h -- C ABI of the B200 boundary-MPS sampler (libtnsample.so).
 *
 * Implements the data-parallel hot path of arXiv 2507.11424 (Rudolph & Tindall,
 * "Simulating and Sampling from Quantum Circuits with 2D Tensor Networks"):
 * generalised boundary-MPS sampling of bitstrings from a planar tensor-network state.
 * Citations: P:n = /root/reference/PAPER.md line n; readings R1..R24 = SURVEY.md 8(c),
 * restated in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Return value: 0 = TN_OK, < 0 = error code below. tn_last_error() returns a
 *    thread-local, NUL-terminated message for the last failing call on this thread.
 *  - Host pointers are borrowed for the duration of the call only (copied to the device).
 *    "_dev" variants take device pointers and a cudaStream_t (passed as void*), do not
 *    synchronise the stream, and leave the caller responsible for the buffers' lifetime
 *    until the stream has passed the call.
 *  - A tn_state is owned by the caller from tn_load_state until tn_free_state. Calls on one
 *    state must be serialised by the caller; distinct states may be used concurrently.
 *    The state is immutable after load except for internal caches keyed by
 *    (row order, chi_env): the device layout of the tensors and the norm environments.
 *  - All work runs on the CUDA device current at tn_load_state. There is no CPU fallback:
 *    without a usable device, calls fail with TN_E_CUDA.
 */
#ifndef TNSAMPLE_H
#define TNSAMPLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TN_OK 0
#define TN_E_ARG (-1)     /* NULL pointer, n <= 0, chi_env < 1, uniform not finite or not in [0,1) */
#define TN_E_GRAPH (-2)   /* vertex id out of range, self-loop, duplicate edge, bond dim not in [1,chi],
                             tensor shape inconsistent with the graph */
#define TN_E_ROWS (-3)    /* row order not a grid-layered line partition (R1) */
#define TN_E_NOMEM (-4)   /* device or host allocation failed */
#define TN_E_CUDA (-5)    /* CUDA runtime error or no device */
#define TN_E_NCCL (-6)    /* NCCL error (tn_comm_unique_id, tn_set_comm, sharded tn_prepare) */
#define TN_E_NUMERIC (-7) /* non-finite value in the norm-environment precompute */

/* Per-sample incident flags (not errors). */
#define TN_FLAG_CLAMPED 1u   /* a one-site weight Re w_s < 0 was clamped to 0 */
#define TN_FLAG_ZERO_MASS 2u /* w_0 + w_1 == 0: P0 := 1/2 was used */
#define TN_FLAG_NONFINITE 4u /* a non-finite weight appeared; logp is NaN */

typedef struct tn_state tn_state; /* opaque */

/* Graph of the tensor network state |psi> (one tensor per qubit, one virtual
 * index per edge). edges: [n_edges][2] vertex ids, 0 <= u,v < n_vertices, u != v, no
 * duplicates. bond_dims: [n_edges], 1 <= dim <= chi. */
typedef struct {
  int32_t n_vertices;
  int32_t n_edges;
  const int32_t* edges;
  const int32_t* bond_dims;
} tn_graph;

/* Load a TNS (D1). tensors[v] points to interleaved complex128 (re, im) data in
 * C order with shape (2, d_e1, d_e2, ...), where e1 < e2 < ... are the ids of the edges
 * incident to v (physical index first). chi >= max bond dim. The data are converted to
 * complex64 on the device (R24). On success *out owns a new state. */
int tn_load_state(const tn_graph* g, const double* const* tensors, int32_t chi, tn_state** out);

/* Norm-environment precompute (a1, "contract the norm network once (independent of the
 * number of samples)"): M_{N_b -> N_b-1} ... M_{2->1} at bond <= chi_env for the row
 * order given as CSR: row_ptr[n_rows+1], row_vertices[n_vertices] (the partition b = 1..N_b
 * in sampling order, vertices of a row in their within-row order, R1/R2). Cached in the
 * state; tn_sample calls it implicitly when the cache misses. Sets the state's current
 * row order (used by tn_amplitude). */
int tn_prepare(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows,
               int32_t chi_env);

/* Sharded norm-environment precompute. The double-layer
 * fits of tn_prepare loop over chunks of their output-bond rows (the mid contraction
 * L.M.A.conj(A) of one chunk at a time); after tn_set_comm, chunk ci is computed only by rank
 * ci % world and broadcast from it over NCCL (NVLink), and every rank assembles the chunks in
 * the same order as one GPU: the environments are bitwise identical on every rank and to a
 * one-GPU tn_prepare. All ranks must call tn_prepare with the same arguments. Everything else
 * (sampling) stays rank-local; the sample shards are the caller's (paper_2507_11424_b200.dist).
 * tn_comm_unique_id: rank 0 creates the id (TN_COMM_ID_BYTES opaque bytes), the caller
 * distributes it; tn_set_comm: every rank joins (blocking until all have joined) on the
 * state's device. Errors: TN_E_ARG, TN_E_NCCL, TN_E_CUDA. */
#define TN_COMM_ID_BYTES 128
int tn_comm_unique_id(uint8_t* out_id);
int tn_set_comm(tn_state* st, const uint8_t* id, int32_t rank, int32_t world);

/* Draw n_samples bitstrings from q(x). uniforms[k][v] in [0,1) is
 * the random number of sample k at vertex id v: x_v = 0 iff u < P0 (R10). Outputs are
 * caller-allocated host arrays: out_bits[k][v] in {0,1} by vertex id, out_logp[k] =
 * ln q(x_k), the natural log of the product of the sampled conditionals (R11). */
int tn_sample(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows,
              int32_t chi_env, int64_t n_samples, const double* uniforms, uint8_t* out_bits,
              double* out_logp);

/* Extended form. sample_offset: global index of the first sample (bookkeeping only; the
 * uniforms given are used as-is, so results do not depend on batching or GPU count,
 * SURVEY 8(b) "Determinism"). out_cond[k][v] (optional, may be NULL): P(x_v | earlier
 * vertices) of the drawn bit. out_flags[k] (optional): OR of TN_FLAG_*. */
int tn_sample_ex(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows,
                 int32_t chi_env, int64_t n_samples, int64_t sample_offset, const double* uniforms,
                 uint8_t* out_bits, double* out_logp, double* out_cond, uint32_t* out_flags);

/* Device-pointer form of tn_sample_ex (for the torch driver / benchmarks): uniforms_dev
 * [n][N] float64, out_bits_dev [n][N] uint8, out_logp_dev [n] float64, out_cond_dev and
 * out_flags_dev optional (NULL). stream: cudaStream_t or NULL for the legacy stream.
 * Requires a prior tn_prepare for this row order and chi_env (TN_E_ROWS otherwise). */
int tn_sample_dev(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows,
                  int32_t chi_env, int64_t n_samples, const double* uniforms_dev, uint8_t* out_bits_dev,
                  double* out_logp_dev, double* out_cond_dev, uint32_t* out_flags_dev, void* stream);

/* tn_sample plus the amplitude carried along each sample's own sampling path (PAPER.md:293:
 * "if the MPS dimension R_x used is large enough such that only minimal truncations are made
 * in the fitting procedures ... [p(x)] is the square of the MPS-MPS contraction
 * m_{N_b-1 -> N_b} . X_{N_b}"): out_logabs[k] = ln|a_k|, out_phase[k] = arg a_k, where a_k is
 * the product of the row fits' norms, the merge normalisations and the final scalar of the
 * projected rows; p(x_k) ~ |a_k|^2 (exact when no fit truncates, else an approximation --
 * tn_certify gives the independent contraction). Host arrays [n_samples]; compress-then-sample
 * order only (TN_E_ARG under option order = 1). Other arguments and errors as tn_sample. */
int tn_sample_path(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows,
                   int32_t chi_env, int64_t n_samples, const double* uniforms, uint8_t* out_bits,
                   double* out_logq, double* out_logabs, double* out_phase);

/* Amplitudes <x|psi> (D3) of n bitstrings bits[k][v] (by vertex id), contracted by
 * boundary MPS of bond <= chi_env over the state's current row order (the last one given to
 * tn_prepare / tn_sample; TN_E_ROWS if none) ("separate contraction of
 * the network <x|psi>"). out_logabs[k] = ln|<x|psi>| (-inf for an exactly zero amplitude),
 * out_phase[k] = arg <x|psi> in radians. Unnormalised: sum_x |<x|psi>|^2 = <psi|psi>. */
int tn_amplitude(tn_state* st, const uint8_t* bits, int64_t n, int32_t chi_env, double* out_logabs,
                 double* out_phase);

/* ln <psi|psi> ~ ln <M_{2->1}, T_1> for the current row order and chi_env (R12). */
int tn_log_norm(tn_state* st, int32_t chi_env, double* out_lognorm);

/* Sample certification. For n samples bits[k][v]
 * with their sampled log-probabilities logq[k] = ln q(x_k) (from tn_sample), computes
 * out_logp[k] = ln p(x_k) = 2 ln|<x_k|psi>| by a separate boundary-MPS contraction at bond
 * chi_env_verify (the paper's verification rank, 2 chi by default, P:130 / R15) over the
 * state's current row order, and the statistics of the importance weights w_k = p_k / q_k:
 *   log_norm_estimate  ln( (1/n) sum_k w_k ): the unbiased estimator E_q[p/q] = <psi|psi>
 *                      (P:116-121), evaluated with a log-sum-exp;
 *   norm_rel_stderr    standard error of (1/n) sum_k w_k divided by that mean (0 if n == 1);
 *   kld                (1/n) sum_k (ln q_k - ln p_k + ln Z), the sample KLD of Eq. (kld)
 *                       with p normalised by Z (R12): ln Z = log_z if finite,
 *                      else ln Z = log_norm_estimate;
 *   ess                (sum w)^2 / sum w^2, the effective sample size of the weights.
 * Samples with logq or logp = -inf/NaN are excluded from the statistics and counted in
 * n_excluded. Host arrays; out_logp may be NULL. Errors: TN_E_ARG (NULL, n <= 0, bits not
 * 0/1), TN_E_ROWS (no row order prepared), TN_E_CUDA. */
typedef struct {
  double log_norm_estimate;
  double norm_rel_stderr;
  double kld;
  double ess;
  int64_t n_used;
  int64_t n_excluded;
} tn_cert_stats;
int tn_certify(tn_state* st, const uint8_t* bits, const double* logq, int64_t n, int32_t chi_env_verify,
               double log_z, double* out_logp, tn_cert_stats* out);

/* Sample observables ("importance sampling" formula;
 * PAPER.md:174 magnetisation pass rate). For n samples bits[k][v] (host, [n][n_vertices]) with
 * ln q (sampled, from tn_sample) and ln p (from tn_certify or tn_sample_path), on the current
 * device:
 *   out_z_weighted[v] = sum_k w_k z_v(x_k) / sum_k w_k, w_k = p_k / q_k, z_v = 1 - 2 x_v: the
 *                       importance-sampled <psi|Z_v|psi> / <psi|psi> (self-normalised, N = the
 *                       mean ratio as in P:299-300); samples with a non-finite ratio weigh 0;
 *   out_z_plain[v]    = (1/n) sum_k z_v(x_k) (the uncorrected sample mean under q);
 *   out_pass_rate     = fraction of samples whose number of ones in each group g
 *                       (group_of[v] in [0, n_groups), -1 = no group) equals target_ones[g]
 *                       (the magnetisation / particle-number sector; n_groups = 0 -> 1);
 *   out_pass_rate_weighted (optional) = the same fraction with the importance weights.
 * Sums are in FP64 with a fixed reduction order (deterministic). n_groups <= 8.
 * Errors: TN_E_ARG (NULL, n <= 0, n_groups out of range), TN_E_CUDA. */
int tn_observables(const uint8_t* bits, const double* logq, const double* logp, int64_t n, int32_t n_vertices,
                   const int32_t* group_of, int32_t n_groups, const int32_t* target_ones,
                   double* out_z_weighted, double* out_z_plain, double* out_pass_rate,
                   double* out_pass_rate_weighted);

/* TNS construction on the GPU, complex FP64: the
 * state a circuit of two-qubit gates leaves, by belief propagation and the BP-gauged simple
 * update -- the oracle generator's algorithm (O7) on the device.
 *   tn_su_create: product state |bits> (bits[v] in {0,1}) on the graph edges [n_edges][2]
 *                 (every bond of dimension 1).
 *   tn_su_bp:     BP on the norm network (identity-initialised normalised messages,
 *                 synchronous sweeps, stop when the largest message change < tol or after
 *                 max_sweeps; R20); *out_residual, *out_sweeps (optional).
 *   tn_su_apply2: gate on edge e (gate: 4 x 4 complex, interleaved (re, im), row-major, index
 *                 2 x_u + x_v with u < v the edge's vertices) with the current BP messages as
 *                 the gauge: sqrt-message gauging (eigen-based, relative cutoff 1e-12),
 *                 orthonormal reduction of both sites, SVD, keep min(chi, #{sigma^2 / sum >
 *                 cutoff}) >= 1 values, *out_eps = discarded weight (Eq. 1), sqrt(sigma)
 *                 split, ungauging, normalised tensors, both messages on e := diag(sigma_kept)
 *                 normalised. Run tn_su_bp before each layer of non-overlapping gates.
 *   tn_su_bond_dims: [n_edges] current bond dimensions.
 *   tn_su_export: tensors[v] (caller-allocated host complex128, C order (2, d_e1, d_e2, ...),
 *                 e1 < e2 < ... incident edge ids): the tn_load_state layout.
 *   tn_su_last_error: message of the last failing tn_su_* call on this thread.
 * Errors: TN_E_ARG, TN_E_GRAPH, TN_E_CUDA. */
typedef struct tn_su tn_su;
int tn_su_create(int32_t n_vertices, int32_t n_edges, const int32_t* edges, const uint8_t* bits, tn_su** out);
int tn_su_bp(tn_su* s, double tol, int32_t max_sweeps, double* out_residual, int32_t* out_sweeps);
int tn_su_apply2(tn_su* s, int32_t edge, const double* gate, int32_t chi, double cutoff, double* out_eps);
int tn_su_bond_dims(tn_su* s, int32_t* out);
int tn_su_export(tn_su* s, double* const* tensors);
int tn_su_free(tn_su* s);
const char* tn_su_last_error(void);

/* Options (SURVEY 5 "Config / flags"): "fit_half_sweeps" (nh, default 2, R5), "init_seed"
 * (default 0x2507114240, R4), "gemm" (0 = auto, 1 = force SIMT FP32, 2 = force tcgen05
 * FP16x3), "max_batch" (0 = auto from free device memory), "order" (within-row sampling
 * order: 0 = compress-then-sample, R3, default; 1 = the paper's literal order, PAPER.md:
 * 289-290 -- sample row b against the uncompressed m_{b-1}.psi_b five-layer ladder, then fit
 * the projected row; its environments hold chi_env^3 chi^2 entries, meant for chi_env <=
 * chi), "chunk_elems" (element budget of one chunk of the double-layer mid contraction in
 * tn_prepare, 0 = default 2^30; smaller = more chunks, e.g. to spread a sharded precompute).
 * Changing fit_half_sweeps / init_seed / gemm / chunk_elems invalidates cached environments.
 * Unknown name or value -> TN_E_ARG. */
int tn_set_option(tn_state* st, const char* name, int64_t value);

/* Kernel launches and wall-clock of the last call on this state (instrumentation). */
int tn_get_stats(tn_state* st, int64_t* out_launches, double* out_precompute_s);

int tn_free_state(tn_state* st);

const char* tn_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* TNSAMPLE_H */
