/*
 * pe.h -- C ABI of the B200-native Polar Express hot path.
 *
 * Polar Express (arXiv 2505.16932; /root/reference/PAPER.md, cited P:<line>)
 * approximates polar(M) = U V^T (eq. (matrixsign)) of a rectangular
 * matrix M by a composition of odd polynomials (eq. (composition)/(iteration),
 * P:121-128).  The library has the paper's two stages (Alg. 1):
 *
 *   offline (host, fp64): pe_coeffs / pe_coeffs_ex -- greedy minimax
 *       polynomials (Theorem 1; Alg. 2 / Listing 1),
 *       cushioning, recentring and the 1.01 safety factor.
 *   online (device): pe_polar -- Listing 2: normalise by
 *       ||X||_F * 1.01 + 1e-7, transpose when rows > cols, then T steps of
 *       A = X X^T; B = b A + c A^2; X = a X + B X, transpose back.
 *       Variants: pe_polar_ex (fp32 in / bf16 arithmetic / fp32 out),
 *       pe_polar_host (host buffers), pe_muon_step (one fused Muon step,
 *       P:41-49), pe_set_spectrum_init (App. G first step).
 *   multi-GPU: pe_nccl_unique_id / pe_attach_comm / pe_polar_sharded (each
 *       rank its pe_shard_plan share, results broadcast to every rank) and
 *       pe_polar_split (one matrix split by columns, all-reduced Gram).
 *
 * Conventions common to every call:
 *   - plain C: no C++ types, no exceptions cross this boundary; every call
 *     returns pe_status and never aborts the process.
 *   - matrices are row-major and contiguous (leading dimension = cols),
 *     16-byte aligned; "shapes" is an int64 array of 2*count entries
 *     (rows_0, cols_0, rows_1, cols_1, ...).
 *   - device pointers are CUDA device addresses on the context's device;
 *     host pointers are ordinary (preferably pinned) host memory.
 *   - the caller owns every buffer it passes; the context owns its workspace.
 *   - argument errors are reported synchronously, before any launch;
 *     asynchronous CUDA faults surface as PE_ERR_CUDA on a later call.
 *   - no CPU fallback exists: without a usable sm_100 device the online calls
 *     return PE_ERR_CUDA / PE_ERR_UNSUPPORTED.
 */
#ifndef PE_H_
#define PE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PE_OK = 0,
  PE_ERR_INVALID_ARG = 1,     /* bad shape / pointer / parameter              */
  PE_ERR_UNSUPPORTED = 2,     /* e.g. degree not in {3,5}, no sm_100 device   */
  PE_ERR_NO_CONVERGENCE = 3,  /* Remez exceeded 50 iterations (reading R6)    */
  PE_ERR_CUDA = 4,            /* CUDA runtime/driver error (sticky errors too) */
  PE_ERR_NCCL = 5,            /* NCCL missing or failed (multi-GPU calls)     */
  PE_ERR_WORKSPACE = 6,       /* device allocation failed                     */
  PE_ERR_NONFINITE = 7        /* PE_DEBUG_CHECK_FINITE found NaN / Inf        */
} pe_status;

typedef enum { PE_BF16 = 0, PE_FP32 = 1 } pe_dtype;

/* Flags of pe_coeffs_ex (reading R5 and App. F). */
#define PE_SAFETY_ALL 1       /* scale every tuple, Pade tail too (Alg.1 l.5) */
#define PE_SAFETY_NOT_FINAL 2 /* leave the final tuple unscaled              */
#define PE_NO_RECENTER 4      /* skip Listing 1's recentring             */

/* Human-readable name of a status code (static storage). */
const char* pe_status_string(pe_status s);

/* Library version string, e.g. "pe-b200 0.1 sm_100a". */
const char* pe_version(void);

/* Detail of the last error raised on the calling thread (static storage,
 * empty string if none). */
const char* pe_last_error_message(void);

/*
 * Offline stage (Alg. 1 offline box; Listing 1, P:537-554;
 * Listing 2's safety comprehension).  Host-only, fp64, pure and
 * thread-safe; microseconds.
 *
 *   ell    lower bound on the normalised singular values, 0 < ell <= 1
 *          (P:261 recommends 1e-3).
 *   degree 3 (closed form, eq. (deg3_solution)) or 5 (Alg. 2,
 *          P:862-886); anything else -> PE_ERR_UNSUPPORTED (general Remez is
 *          only cited by the paper).
 *   T      number of polynomials, T >= 1.
 *   safety safety factor >= 1 (P:486 uses 1.01): p_t(x) -> p_t(x / safety).
 *   coeffs caller-owned output of T * (degree+1)/2 doubles, tuple t at
 *          coeffs[t*(degree+1)/2 ...] = (a_t, b_t[, c_t]) with
 *          p_t(x) = a_t x + b_t x^3 [+ c_t x^5].
 * Cushion = 0.02407327424182761 (Listing 1) for degree 5 and the
 * analogous 0.039327193224439 for degree 3 (reading R3).  Tuples produced by
 * the Pade branch (l/u >= 1 - 5e-6) are emitted as the exact limit
 * (15/8, -10/8, 3/8) and left unscaled (readings R4, R5), reproducing the
 * printed table P:475-487.
 * Errors: PE_ERR_INVALID_ARG (ell, T, safety, NULL), PE_ERR_UNSUPPORTED
 * (degree), PE_ERR_NO_CONVERGENCE (Remez > 50 iterations).
 */
pe_status pe_coeffs(double ell, int degree, int T, double safety, double* coeffs);

/*
 * As pe_coeffs with the knobs exposed:
 *   cushion    < 0 selects the default above; otherwise the cushion ratio c
 *              of max(l_t, c*u_t) (Alg.1 line 4 uses 0.1).
 *   flags      PE_SAFETY_ALL | PE_SAFETY_NOT_FINAL | PE_NO_RECENTER.
 *   ell_trace  optional (NULL ok) output of T+1 doubles: l_1..l_{T+1} of the
 *              pre-safety recurrence l_{t+1} = p_t(l_t) (eq. (newbounds),
 *              P:196); the certified error is 1 - l_{T+1}.
 */
pe_status pe_coeffs_ex(double ell, int degree, int T, double safety, double cushion,
                       int flags, double* coeffs, double* ell_trace);

/* ------------------------------------------------------------------------ */
/* Online stage (device).  One context per device; a context is not          */
/* thread-safe (serialise calls on it) and its calls must be ordered on one  */
/* stream (it caches up to 8 plans over one workspace and keeps a ring of 4  */
/* pinned per-call upload buffers, so up to 4 calls may be in flight).       */
/* ------------------------------------------------------------------------ */
typedef struct pe_ctx_s* pe_ctx;

/* Create a context on CUDA device `device`.  Its default table is
 * pe_coeffs(1e-3, 5, 8, 1.01) (Listing 2's coeffs_list).
 * Errors: PE_ERR_INVALID_ARG (NULL), PE_ERR_UNSUPPORTED (device is not
 * compute capability 10.0), PE_ERR_CUDA. */
pe_status pe_create(pe_ctx* ctx, int device);

/* Destroy a context and free its workspace (synchronises its device). */
pe_status pe_destroy(pe_ctx ctx);

/* Replace the coefficient table: `ntuples` tuples of (degree+1)/2 doubles,
 * degree 3 or 5 (e.g. Newton-Schulz P:78, Jordan P:82, a degree-3 table).
 * The kernels receive them rounded to fp32.  Copied; caller keeps ownership.
 * Errors: PE_ERR_INVALID_ARG (NULL, ntuples < 1, non-finite entries),
 * PE_ERR_UNSUPPORTED (degree). */
pe_status pe_set_coeffs(pe_ctx ctx, const double* coeffs, int ntuples, int degree);

/* Pre-size the workspace and build the plan for a batch (shape list and
 * dtype) so that a later pe_polar / pe_muon_step on it performs no allocation
 * or synchronisation.  Workspace per matrix (m = min side, n = max side): two
 * bf16 m x n iterate buffers, two m x m buffers (A, B), a norm slot; PE_FP32
 * holds each buffer as three bf16 planes (3x the bytes).
 * CUDA graphs: a pe_polar / pe_muon_step issued on a stream that is being
 * captured requires a prior pe_reserve of the same shape list and dtype; it
 * then allocates nothing, does not synchronise, and consumes one of the
 * upload slots pe_reserve keeps in reserve (4 per call of pe_reserve,
 * iters <= 64) for the lifetime of the context, since the graph's copy node
 * re-reads it at every replay. Graph replays see the current contents of the
 * captured buffers.  A captured graph stays valid until pe_destroy: the plan
 * and the workspace it points into are retired, never freed, when the
 * workspace later grows or the plan leaves the context's 8-plan cache.  A
 * one-step (iters = 1) call whose outputs overlap its inputs uses a separate
 * plan (see pe_polar) that pe_reserve does not build: issue it once
 * uncaptured before capturing it.  Errors: PE_ERR_INVALID_ARG,
 * PE_ERR_WORKSPACE (also: a captured call without a reservation). */
pe_status pe_reserve(pe_ctx ctx, const int64_t* shapes, int count, pe_dtype dtype);

/*
 * Polar Express on a batch of `count` matrices (Listing 2).
 *   in[i], out[i]  device pointers to rows_i x cols_i row-major matrices of
 *                  element type `dtype` (PE_BF16: bf16 tensor-core path with
 *                  fp32 accumulation; PE_FP32: fp32 values, every product
 *                  on the same tensor cores as six bf16 plane products
 *                  P_i Q_j^T, i + j <= 2, of the three-plane split
 *                  v = p0 + p1 + p2; relF <= 1e-5).  in[i] == out[i]
 *                  (in place) is allowed; distinct matrices must not overlap.
 *                  (With iters = 1 the single update reads the inputs while
 *                  it stores results, so a call whose outputs overlap its
 *                  inputs stores through the workspace plus one copy pass.)
 *   iters          T >= 1; tuples past the table repeat its last tuple
 *                  (P:495-496).
 *   stream         a cudaStream_t (NULL = legacy default stream); all work is
 *                  enqueued on it, the call does not synchronise.
 * Per matrix: s = ||M||_F * 1.01 + 1e-7 (reading R1; fp64 sum of
 * squares), X_0 = M / s, oriented so that the Gram is on the smaller side
 * (strict rows > cols, R10; bf16 X_0 is never rounded: 1/s is applied
 * in the first Gram / update epilogues, on the caller's M or on an exact
 * oriented copy M 2^e, R2); then T x (Gram, b A + c A^2, a X + B X)
 * on sm_100a tcgen05 tensor cores; the result is written to out[i] in the
 * caller's orientation.  A zero matrix gives zeros (R9).
 * Errors: PE_ERR_INVALID_ARG (count < 0, NULL pointer, rows/cols < 1 or
 * > 2^20, a pointer not 16-byte aligned, iters < 1), PE_ERR_WORKSPACE
 * (device allocation), PE_ERR_CUDA (launch / earlier asynchronous fault).
 */
pe_status pe_polar(pe_ctx ctx, const void* const* in, void* const* out, const int64_t* shapes,
                   int count, int iters, pe_dtype dtype, void* stream);

/*
 * pe_polar with separate element types for the caller's input, the caller's
 * output and the arithmetic: Listing 2 casts the (usually
 * fp32) Muon momentum to bf16 and iterates in bf16, and returns bf16.
 *   compute = PE_BF16: in_dtype and out_dtype each PE_BF16 or PE_FP32.  An
 *     fp32 input is normalised in fp32 (s from the fp64 sum of its squares,
 *     P:494) and rounded once to bf16 as X_0 = bf16(fp32(x) * inv) (reading
 *     R16: the fp32 values, not a bf16 copy of them, are normalised); an fp32
 *     output receives the bf16 result exactly (no further rounding).  These
 *     matrices go through the copy passes instead of being folded into the
 *     first / last GEMM, so in == out requires in_dtype == out_dtype.
 *   compute = PE_FP32: in_dtype = out_dtype = PE_FP32 only (= pe_polar).
 * Same pointers, shapes, streams and errors as pe_polar, plus
 * PE_ERR_UNSUPPORTED for other type combinations.  Under CUDA-graph capture a
 * mixed-type call needs its plan built by an earlier uncaptured call with the
 * same shapes and types (pe_reserve covers in = out = compute only).
 */
pe_status pe_polar_ex(pe_ctx ctx, const void* const* in, void* const* out, const int64_t* shapes,
                      int count, int iters, pe_dtype in_dtype, pe_dtype out_dtype, pe_dtype compute,
                      void* stream);

/*
 * End-to-end variant on HOST buffers: copies in[i] (host) to device staging
 * owned by the context, runs pe_polar, copies the results back to out[i]
 * (host) and synchronises `stream` before returning.  The batch is cut into
 * up to 8 groups of about equal bytes that are software-pipelined over the
 * caller's stream and two context-owned copy streams (H2D of group g+1 and
 * D2H of group g-1 overlap the compute of group g).  Same semantics and
 * errors as pe_polar; host buffers should be pinned for full PCIe bandwidth.
 */
pe_status pe_polar_host(pe_ctx ctx, const void* const* in, void* const* out, const int64_t* shapes,
                        int count, int iters, pe_dtype dtype, void* stream);

/*
 * One Muon optimizer step on a batch of `count` bf16 layer
 * matrices, with the polar factor computed exactly as pe_polar computes it:
 *   M <- bf16(fp32(beta) * M + fp32(1 - beta) * G)      (fp32 arithmetic,
 *                                                         no FMA contraction)
 *   X  = pe_polar(M) (bf16, T = iters, the context's table)
 *   W <- bf16(fp32(W) - fp32(lr) * X)
 * W[i], M[i], G[i]: device pointers to rows_i x cols_i row-major bf16
 * matrices, 16-byte aligned; W and M are updated in place, G is read; the
 * three sets must not overlap. beta, lr: finite (the paper's default beta =
 * 0.9). The momentum update is fused into the norm pass and the weight
 * update into the last update GEMM's epilogue (matrices with cols % 8 == 0;
 * the others update W in the final copy pass), so neither M_t nor X makes an
 * extra HBM round trip. Asynchronous on `stream` like pe_polar.
 * Errors: PE_ERR_INVALID_ARG (NULL or overlapping pointers, misalignment,
 * bad shapes, iters < 1, non-finite beta/lr), PE_ERR_WORKSPACE, PE_ERR_CUDA.
 */
pe_status pe_muon_step(pe_ctx ctx, void* const* W, void* const* M, const void* const* G,
                       const int64_t* shapes, int count, double beta, double lr, int iters, void* stream);

/*
 * Intra-matrix sharding: one wide matrix
 * M = [M_0 | M_1 | ... ] (m x n, column blocks on different ranks) is
 * orthogonalised jointly; this rank passes its column block M_r (rows = m,
 * cols = n_r, row-major bf16, cols % 8 == 0, 16-byte aligned) and receives
 * the same columns of pe_polar(M) in `out` (m x n_r).  Per iteration
 * A = sum_r M_r M_r^T is formed by an all-reduce of the fp32 partial Grams
 * (rounded once to bf16 afterwards, reading R8), B = b A + c A^2 is
 * computed redundantly on every rank and X_r <- a X_r + B X_r stays local
 * (P:500); ||M||_F^2 is all-reduced first.  rows may exceed cols
 * here (the Gram side is always `rows`).
 * allreduce(buf, count, dtype, user, stream): the caller's in-place SUM
 * all-reduce over all ranks of `count` elements (dtype 0 = fp32, 1 = fp64)
 * of device buffer `buf`, enqueued on `stream` (e.g. ncclAllReduce); called
 * 1 + iters times per call, from the calling thread, between kernel
 * launches; return PE_OK or an error, which aborts the call.  allreduce =
 * NULL uses the context's own communicator (pe_attach_comm): an in-place
 * ncclAllReduce (SUM) on `stream`; `user` is then ignored.
 * Errors: PE_ERR_INVALID_ARG (also: NULL allreduce without a communicator),
 * PE_ERR_UNSUPPORTED (cols % 8 != 0, capture),
 * PE_ERR_WORKSPACE, PE_ERR_CUDA, or the callback's status.
 */
typedef pe_status (*pe_allreduce_fn)(void* buf, int64_t count, int dtype, void* user, void* stream);
pe_status pe_polar_split(pe_ctx ctx, const void* in, void* out, int64_t rows, int64_t cols, int iters,
                           pe_allreduce_fn allreduce, void* user, void* stream);

/*
 * pe_polar_split with the cross-rank sums done by the library's own kernels
 * over peer-visible memory instead of an all-reduce call.
 * slots[r] (r = 0..world-1, 256-byte aligned, pe_split_slot_bytes(rows, cols)
 * bytes each) is rank r's slot, readable by every rank: on several GPUs a
 * P2P-mapped (cudaIpc / symmetric-memory) allocation over NVLink, on one GPU
 * plain device memory.  Rank r's kernels write its partial results straight
 * into slots[rank] -- ||M_r||^2 from the norm pass, the partial Gram from the
 * Gram epilogue (double-buffered by iteration parity) -- and after the
 * barrier the next kernel sums all slots in rank order (bit-identical on every
 * rank) and rounds A once to bf16 (R8).  barrier(user, stream) is called on
 * the host: it must return once the work enqueued on `stream` so far is
 * complete on this rank and every rank has reached the same barrier (one per
 * iteration plus one for the norm).  Errors: PE_ERR_INVALID_ARG (NULL,
 * misaligned slot, rank outside [0, world)), the barrier's status, and
 * pe_polar_split's.
 */
typedef pe_status (*pe_barrier_fn)(void* user, void* stream);
pe_status pe_split_slot_bytes(int64_t rows, int64_t cols, int64_t* bytes);
pe_status pe_polar_split_peers(pe_ctx ctx, const void* in, void* out, int64_t rows, int64_t cols, int iters,
                               void* const* slots, int rank, int world, pe_barrier_fn barrier, void* user,
                               void* stream);

/*
 * Spectrum-aware first step (App. G, k = 1; reading R17), for
 * inputs with one large outlying singular value.  power_iters > 0 turns it
 * on for the context's later bf16 pe_polar / pe_polar_ex / pe_polar_host
 * calls (0 = off, the default): after Listing 2's normalisation X_0 = M / s,
 * power_iters steps of the power method on A_0 = X_0 X_0^T in fp32
 * (deterministic start vector v0_i = frac((i+1)/phi) + 0.5) give the
 * Rayleigh quotient lambda <= sigma_1(X_0)^2 and z = sqrt(lambda) / ||X_0||_F;
 * when
 * 1/sqrt(2) <= z <= 1 - 1e-6 the odd cubic p(x) = a x + b x^3 of
 * eq. (init_poly) (p(sqrt(1-z^2)) = p(z) = 1 on the unit-norm
 * scale) is applied before the T iterations, else the step is the identity.
 * Costs one extra Gram (which also stores its fp32 accumulator for the
 * power method) + one update (+ power_iters passes over A_0; fp32 inputs also
 * one pass over A_0's diagonal: ||X_0||_F^2 of the rounded X_0 as its trace);
 * matrices run
 * on the large path (the small-matrix path is bypassed).  fp32 calls and
 * pe_muon_step ignore it.  Errors: PE_ERR_INVALID_ARG (NULL, power_iters < 0
 * or > 1000).
 */
pe_status pe_set_spectrum_init(pe_ctx ctx, int power_iters);

/*
 * Same, with the bf16 stabilisation margin of reading R17 made explicit: the
 * cubic of eq. (init_poly) is divided by 1 + |b| * margin.  margin = 0 applies
 * eq. (init_poly) exactly as P:1256-1263 states it (what the oracle computes)
 * and is what pe_set_spectrum_init uses.  z comes from the power method on
 * the fp32 Gram of the first iteration (a second Gram launch that stores the
 * raw accumulator): on the bf16 Gram the Rayleigh quotient can exceed
 * sigma_1^2 by ~2^-9 relative, which breaks z <= sigma_1, lets
 * the tail bound sqrt(1 - z^2) fall below sigma_2 and lifted sigma_2 past 1
 * (NaN two iterations later); a margin > 0 is then a user choice.  Errors:
 * PE_ERR_INVALID_ARG (NULL, power_iters outside 0..1000, margin outside
 * [0, 1] or NaN).
 */
pe_status pe_set_spectrum_init_ex(pe_ctx ctx, int power_iters, double margin);

/*
 * Fast polynomial iteration for rectangular matrices (App. H, Alg. 4,
 * P:1303-1316), opt-in for the context's later bf16 pe_polar / pe_polar_ex /
 * pe_polar_host calls with a degree-5 table.  A matrix with min side
 * m > 128 and max side n > min_aspect * m (min_aspect <= 0: the paper's rule
 * n / m > 1.5 T / (T - 1)) is computed as
 *     Y = X X^T (+ shift I in the first application), Q_0 = I,
 *     R_t = Q_{t-1} Y Q_{t-1},  Q_t = Q_{t-1} h_t(R_t),  X' = Q X
 * (wide orientation; p_t(x) = x h_t(x^2), h_t(y) = a_t + b_t y + c_t y^2),
 * restarted every `restart` iterations (1 = Listing 2 exactly,
 * >= T = one application).  Rectangular products: 2 per application instead
 * of 2 per iteration; per further iteration four m x m products.  Other
 * matrices of the call run Listing 2 (a mixed call becomes two grouped
 * calls).  Rounding points (R19): Y, T = Y Q, R, H = b R + c R^2,
 * Q and X' each rounded once to bf16 from fp32 accumulators (R² is the
 * true product R R).  fp32 calls, degree-3 tables, pe_muon_step,
 * pe_polar_split and calls with the App. G step (pe_set_spectrum_init) run
 * Listing 2 as if it were off; a call under graph capture with a qualifying
 * matrix returns PE_ERR_UNSUPPORTED.  restart = 0 turns it off (the
 * default).  Errors: PE_ERR_INVALID_ARG (NULL, restart < 0, shift outside
 * [0, 1), NaN min_aspect).
 */
pe_status pe_set_rect_iteration(pe_ctx ctx, int restart, double min_aspect, double shift);

/*
 * Precision of the bf16 small-matrix path (one CTA per matrix, min side
 * <= 128; R8p).  planes = 2 (opt-in; applies when every matrix of
 * the call has max side <= 640): the Gram A and the polynomial B are kept as
 * two bf16 planes (16 significand bits) -- their bf16 rounding dominates the
 * R8 design's error at small m, and with two planes the small path meets
 * north_star's 2e-2 from m = 32 (tests/test_r8_spread.py); X and X' stay
 * bf16; the call takes ~1.4x longer (two MMA chains on the update).
 * planes = 1 (the default): Listing 2's R8 rounding points, bit-identical to
 * the large path, so a matrix's result does not depend on the batch it is
 * computed in (two-plane results do: the variant only exists on the small
 * path).  Errors: PE_ERR_INVALID_ARG (NULL, planes not 1 or 2).
 */
pe_status pe_set_small_planes(pe_ctx ctx, int planes);

/*
 * Debug aids (never on the hot path).
 * pe_count_nonfinite: *nonfinite = number of NaN / Inf elements over the
 *   `count` device buffers (rows x cols of `dtype` each); synchronises
 *   `stream`; PE_ERR_UNSUPPORTED under graph capture.  Uses a counter owned
 *   by the context: like every call on a context, not from two host threads
 *   at once.
 * pe_set_debug(ctx, PE_DEBUG_CHECK_FINITE): later pe_polar / pe_polar_ex
 *   calls scan their inputs before launching anything (non-finite inputs:
 *   PE_ERR_NONFINITE, nothing computed) and their outputs after the call
 *   (non-finite outputs of finite inputs: PE_ERR_NONFINITE); both scans
 *   synchronise the stream.  0 turns it off (the default: non-finite inputs
 *   then propagate, reading R9's contract).
 * Errors: PE_ERR_INVALID_ARG (NULL, unknown flag bits), PE_ERR_CUDA.
 */
#define PE_DEBUG_CHECK_FINITE 1
pe_status pe_count_nonfinite(pe_ctx ctx, const void* const* bufs, const int64_t* shapes, int count, pe_dtype dtype,
                             int64_t* nonfinite, void* stream);
pe_status pe_set_debug(pe_ctx ctx, int flags);

/* Number of kernel launches the last pe_polar / pe_polar_host enqueued (for
 * the benchmark's gpu_launches accounting). */
pe_status pe_last_launch_count(pe_ctx ctx, int* launches);

/*
 * Per-kernel timing for the benchmark's roofline report.  When enabled, every
 * launch of pe_polar is bracketed by CUDA events on the call's stream (no
 * extra synchronisation).  pe_profile_read synchronises those events, adds
 * their durations into ms[kind] and launch counts into counts[kind] for the
 * first `nkinds` kinds, and clears the pending list.  Kinds:
 *   0 norm (pe_norm_kernel)     1 scale/orient (pe_copy_kernel)
 *   2 Gram  3 poly  4 update (pe_gemm_sm100, one launch per phase; fp32 calls:
 *   the three-plane instantiation)   5 transpose-back (pe_copy_kernel)
 *   6 fused (pe_gemm_sm100 running every phase of the call in one launch;
 *     bf16 with PE_FUSED=1 set in the environment, otherwise one launch per phase)
 *   7 small (pe_small_sm100: the whole call in one launch, one CTA per
 *     matrix, when every matrix has min side <= 128 and max side <= 768
 *     (bf16) / 128 (fp32); PE_SMALL=0 disables it)
 */
#define PE_PROFILE_KINDS 8
pe_status pe_profile_enable(pe_ctx ctx, int on);
pe_status pe_profile_read(pe_ctx ctx, double* ms, int* counts, int nkinds);

/*
 * Deterministic matrix-to-rank partition for data-parallel Muon:
 * longest-processing-time greedy on the per-matrix cost 3 m^2 n + m^3
 * (m = min side), run bucket by bucket over pe_polar_sharded's buckets
 * (pe_shard_nbuckets / pe_shard_buckets): largest first, to the rank with
 * the least work in the bucket, ties to the least total work, then the
 * lowest rank.  Every bucket is balanced, hence the whole set; every rank
 * computes the same plan with no communication.  owner[i] in [0, world).
 * Errors: PE_ERR_INVALID_ARG (world < 1, count < 0, NULL, a side < 1).
 */
pe_status pe_shard_plan(const int64_t* shapes, int count, int world, int* owner);

/*
 * Bucket boundaries pe_polar_sharded uses: consecutive index ranges of about
 * equal total cost 3 m^2 n + m^3, identical on every rank.  begin[0..nbuckets]
 * (caller-owned, nbuckets + 1 ints) receives the first index of each bucket
 * and `count` at the end (trailing empty buckets repeat `count`).
 * Errors: PE_ERR_INVALID_ARG.
 */
pe_status pe_shard_buckets(const int64_t* shapes, int count, int nbuckets, int* begin);

/*
 * Data-parallel Muon across GPUs.  Every rank holds
 * every momentum matrix and needs every polar factor for its weight update
 * W <- W - lr * polar(M); the matrices are independent (the
 * iteration runs per parameter).  NCCL is loaded at run time (the copy
 * already in the process, else $PE_NCCL_LIB, else libnccl.so.2); without it
 * these calls return PE_ERR_NCCL and everything else still works.
 *
 * pe_nccl_unique_id: a fresh ncclUniqueId (128 bytes, caller-owned `id`),
 *   made on one rank and handed to the others out of band.
 * pe_attach_comm: collective over the `world` ranks (ncclCommInitRank inside);
 *   binds a communicator to the context's device and creates a side stream
 *   for the exchange.  Calling it again replaces the communicator.
 * pe_comm_info: the attached rank / world (world = 0 when none is attached).
 * pe_polar_sharded: same arguments and semantics as pe_polar, called by every
 *   rank with the same shape list.  Rank r computes the matrices
 *   pe_shard_plan(shapes, count, world) assigns to it, in buckets of
 *   consecutive matrices (pe_shard_buckets; their number pe_shard_nbuckets
 *   gives, or $PE_SHARD_BUCKETS); as soon as bucket b is computed it is
 *   exchanged on the side stream while bucket b+1 is computed:
 *     - if out[] is the pe_shard_layout of one flat buffer (out[i] =
 *       base + offsets[i] on every rank), the owned matrices' last update
 *       epilogues store straight into this rank's chunk and ONE in-place
 *       all-gather per bucket (ncclAllGather, or the exchange function's
 *       PE_EXCHANGE_ALLGATHER) fills the other chunks -- no packing copy;
 *     - otherwise every matrix is broadcast from its owner into every rank's
 *       out[i] (ncclBroadcast, one NCCL group per bucket, or
 *       PE_EXCHANGE_BROADCAST per matrix).
 *   When the work enqueued on `stream` completes, out[i] holds polar(M_i) on
 *   every rank.  in[i] is read only on the owner of matrix i (it may be NULL
 *   elsewhere); out[i] must be valid on every rank; in[i] == out[i] is
 *   allowed.  On an error after part of the exchange was enqueued, `stream`
 *   still waits for what was enqueued before the error returns.
 *   Errors: PE_ERR_INVALID_ARG (no communicator, bad arguments),
 *   PE_ERR_NCCL (NCCL missing or failed; an earlier asynchronous NCCL error),
 *   the exchange function's status, and pe_polar's.
 */
pe_status pe_nccl_unique_id(char id[128]);
pe_status pe_attach_comm(pe_ctx ctx, const char id[128], int rank, int world);
pe_status pe_comm_info(pe_ctx ctx, int* rank, int* world);
pe_status pe_polar_sharded(pe_ctx ctx, const void* const* in, void* const* out, const int64_t* shapes,
                           int count, int iters, pe_dtype dtype, void* stream);

/*
 * The exchange step of pe_polar_sharded alone: every rank's out[i] for the
 * matrices it owns (pe_shard_plan) already hold their results; the same
 * buckets, collectives (all-gather over the pe_shard_layout buffer, else
 * per-matrix broadcasts) and stream ordering bring every out[i] to every
 * rank.  No compute.  Errors as pe_polar_sharded.
 */
pe_status pe_sharded_exchange(pe_ctx ctx, void* const* out, const int64_t* shapes, int count, pe_dtype dtype,
                              void* stream);

/*
 * Caller-supplied exchange instead of NCCL (virtual ranks, other transports).
 * pe_polar_sharded calls fn on the enqueueing host thread, after the bucket's
 * compute is ordered before `stream` (the side stream, a cudaStream_t), with
 *   op = PE_EXCHANGE_ALLGATHER: buf holds world chunks of `bytes` bytes; this
 *        rank's chunk (index `root` = this rank) is complete once `stream`
 *        reaches this point; fn must make every chunk complete on `stream`;
 *   op = PE_EXCHANGE_BROADCAST: `bytes` bytes at buf, complete on rank `root`,
 *        to be made complete on every rank on `stream`.
 * fn returns PE_OK or an error, which pe_polar_sharded returns.
 * pe_attach_exchange replaces any attached communicator.
 * Errors: PE_ERR_INVALID_ARG (NULL ctx or fn, rank outside [0, world)).
 */
#define PE_EXCHANGE_ALLGATHER 0
#define PE_EXCHANGE_BROADCAST 1
typedef pe_status (*pe_exchange_fn)(int op, void* buf, int64_t bytes, int root, void* user, void* stream);
pe_status pe_attach_exchange(pe_ctx ctx, int rank, int world, pe_exchange_fn fn, void* user);

/*
 * Bucket count pe_polar_sharded uses for this shape list and world: one
 * bucket per ~2.4 TFLOP of per-rank work (about 2 ms of compute, long next to
 * a bucket's fixed fill/drain cost; the exposed tail is the last bucket's
 * exchange), at most 8; 1 when world = 1; $PE_SHARD_BUCKETS overrides.
 */
pe_status pe_shard_nbuckets(const int64_t* shapes, int count, int world, int* nbuckets);

/*
 * Flat output layout for pe_polar_sharded's zero-copy all-gather: bucket after
 * bucket (pe_shard_nbuckets buckets, pe_shard_buckets boundaries), each bucket
 * `world` equal chunks of the largest rank's share, rank r's matrices of the
 * bucket packed in index order inside chunk r, each at a 256-byte granule.
 * offsets[i] (caller-owned, count int64) receives matrix i's byte offset,
 * chunk_bytes[b] (caller-owned, pe_shard_nbuckets int64, or NULL) bucket b's
 * per-rank chunk size (bucket b spans world * chunk_bytes[b] bytes, buckets
 * back to back from offset 0), *total_bytes the buffer size; the same on
 * every rank.  Matrix i of dtype's
 * element size then lives at base + offsets[i] (row-major, lda = cols).
 * Errors: PE_ERR_INVALID_ARG.
 */
pe_status pe_shard_layout(const int64_t* shapes, int count, int world, pe_dtype dtype, int64_t* offsets,
                          int64_t* chunk_bytes, int64_t* total_bytes);

/* Algorithmic flops of one pe_polar call (symmetric Gram and A^2 counted
 * once): sum_i T [ m(m+1) n + m^2 (m+1) + 2 m^2 n ]; degree-3
 * tables drop the A^2 term.  Written to *flops. */
pe_status pe_flops(const int64_t* shapes, int count, int iters, int degree, double* flops);

#ifdef __cplusplus
}
#endif

#endif /* PE_H_ */
