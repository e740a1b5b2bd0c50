/*
 * prohd.h — C ABI of the B200-native ProHD hot path (arxiv 2511.18207).
 *
 * The library (libprohd.so, sm_100a only) exposes the paper's problem
 * statement: given two point clouds A (nA x D) and B (nB x D), compute
 *   - the exact directed Hausdorff distance h(A,B) = max_{a in A} min_{b in B} ||a-b||_2
 *     (Eq. (1))                              -> directed_hd
 *   - the undirected H(A,B) = max{h(A,B), h(B,A)}      -> hausdorff
 *   - the ProHD estimate H^ of Alg. 3 "ProjHausdorff":
 *     centroid axis (Alg. 1) + top-k principal directions of A u B
 *     (Alg. 2), top/bottom-m extremes per direction (P:205-214,
 *     P:242-251), union, exact HD on the subsets
 *                                                                      -> prohd_estimate
 * Notation (BASELINE.json): k = number of principal directions (the paper's
 * m = floor(sqrt D)), m = points kept per (set, direction, tail) (the paper's
 * k_X = max{1, floor(alpha n_X)}).
 *
 * Conventions shared by every call
 *   - Point clouds are fp32, row-major, contiguous, leading dimension D
 *     (row i starts at X + i*D). They may be DEVICE pointers (CUDA memory on the
 *     context's device) or HOST pointers; host inputs are copied into the
 *     workspace inside the call (cudaMemcpyAsync on the context stream), so the
 *     workspace must have been sized with PROHD_WS_HOST_INPUTS.
 *   - Alignment: when D % 4 == 0, DEVICE point-cloud pointers must be 16-byte
 *     aligned (the kernels read rows with 16-byte vector loads, bulk copies and
 *     TMA); a misaligned device pointer returns PROHD_E_INVALID before any launch.
 *     torch / cudaMalloc buffers and whole-row offsets of them always qualify;
 *     host inputs are staged into the (aligned) workspace and may be unaligned.
 *   - Ownership: the caller owns every input/output buffer and the workspace;
 *     the library never frees caller memory and allocates no device memory of
 *     its own beyond its context (TMA descriptors live in kernel parameters).
 *   - All calls enqueue on the context's CUDA stream and are BLOCKING: they
 *     synchronize that stream before filling the host result struct.
 *   - Distances are Euclidean, returned in fp64: `dist` is the fp64 direct
 *     re-evaluation sum_k (a_k - b_k)^2 of the witness pair, square-rooted.
 *   - Ties: nearest neighbour = lowest
 *     column index among equal fp64 distances; directed maximum = lowest row
 *     among equal row minima; undirected witness = the A->B side on equality.
 *   - Errors: every call returns a prohd_status; no exception crosses the ABI.
 *     prohd_last_error(ctx) returns a NUL-terminated message for the last
 *     failing call on that context (valid until the next call).
 *   - Thread-safety: a context may be used by one host thread at a time.
 */
#ifndef PROHD_H_
#define PROHD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PROHD_OK = 0,
  PROHD_E_INVALID = 2,   /* null pointer, n < 1, D < 1, k < 0 or k > D, m < 1, bad shard */
  PROHD_E_DATA = 3,      /* non-finite input (detected from the row norms / moments)     */
  PROHD_E_INTERNAL = 4,  /* an internal invariant failed                                 */
  PROHD_E_CUDA = 5,      /* a CUDA runtime/driver call failed (message has the name)     */
  PROHD_E_WORKSPACE = 6, /* workspace missing or smaller than prohd_workspace_bytes()    */
  PROHD_E_NOTIMPL = 7,   /* feature not built (e.g. not an sm_100 device)                */
  PROHD_E_DEVICE = 8     /* the context's device is not a compute-capability 10.0 GPU    */
} prohd_status;

/* flags for prohd_workspace_bytes */
#define PROHD_WS_HOST_INPUTS 1u /* inputs may be host pointers: reserve staging space */
#define PROHD_WS_CERTIFIED 2u   /* include prohd_estimate_certified (full-set operands)  */

typedef struct prohd_ctx prohd_ctx; /* opaque: device, stream, workspace, last error */

/* Create a context on `device` that enqueues on `cuda_stream` (a cudaStream_t;
 * NULL = the legacy default stream). Returns PROHD_E_DEVICE if the device is
 * not sm_100. *out is set to NULL on failure. */
int prohd_create(int device, void* cuda_stream, prohd_ctx** out);
int prohd_destroy(prohd_ctx* ctx);
int prohd_set_stream(prohd_ctx* ctx, void* cuda_stream);
const char* prohd_last_error(const prohd_ctx* ctx);
/* Library version string, e.g. "prohd-b200 0.1 sm_100a". Never NULL. */
const char* prohd_version(void);
/* Kernels this process has launched through the library so far (all contexts; tracing and
 * the benchmark's gpu_launches). *out (HOST) receives the count; PROHD_E_INVALID if NULL. */
int prohd_launch_count(int64_t* out);
/* Variant options (process-wide, all contexts). Each forces another DEVICE variant of the same
 * computation for A/B measurement and tests; none is a CPU path, and the defaults (value -1,
 * "unset") are the measured-best variants. They are only ever set through this call (the
 * library reads no environment variables). Names and values:
 *   "k6_variant"    1 single 128-row A block per CTA, 2 two-SM pair (directed), 3 two A blocks
 *   "k6_split3"     1: literal 3xTF32 distance products (three TF32 MMAs on fp32 hi/lo)
 *   "k6_bidir_2a"   fused bidirectional sweep on: 0 the single-block kernel, 1 the two-A kernel,
 *                   2 the CTA-pair kernel (default for D >= 128: 2 up to nA nB D = 1e14, 0 above)
 *   "k6_splits_2x"  1: the earlier fill-twice column-split rule
 *   "k1_path"       0 fp64 DMMA Gram, 1 int8 tcgen05 Gram (the default for D <= 256, D % 4 == 0),
 *                   2 legacy tile moments kernel
 *   "k1_ctas", "k1_cs_sms", "k1_beta_milli"   Gram scheduling knobs
 *   "shift"         0 never / 1 always shift the Gram by the sample mean
 *   "k3_simt"       1: SIMT projection kernel instead of tcgen05
 *   "eig_stop"      1|2|3: stop the eigen-solver after that stage (timing prefixes only)
 *   "eig_cl"        8: tridiagonalisation on the portable 8-CTA cluster (default 16 CTAs)
 *   "k1_ablate"     1|2: int8 Gram timing ablations (skip slicing / MMAs; WRONG results, dev only)
 *   "k4_sampled"    0: radix K4 over all projections; 1: sampled-threshold K4 wherever it applies
 *                   (default: sampled for n >= 262144, same selected indices either way);
 *                   2|3: timing ablations of the fused K3 epilogue (no tests / no appends; the
 *                   lists then fail certification and the radix K4 reruns)
 *   "k1_i8_ctas"    n > 0: at most n CTAs in the int8 Gram (tests force mid-sweep drains with it)
 * value < 0 restores the default. PROHD_E_INVALID for an unknown name or NULL pointer. */
int prohd_set_option(const char* name, int64_t value);
int prohd_get_option(const char* name, int64_t* value);

/* Bytes of device workspace any call below needs for these sizes (max over
 * directed_hd, hausdorff and prohd_estimate). Pure host arithmetic. */
size_t prohd_workspace_bytes(int64_t nA, int64_t nB, int32_t D, int32_t k, int64_t m,
                             uint32_t flags);
/* Attach a caller-owned device buffer (>= 256-byte aligned) as workspace. */
int prohd_set_workspace(prohd_ctx* ctx, void* dptr, size_t bytes);

/* ---------------------------------------------------------------- results */
typedef struct {
  double dist;   /* h = sqrt(dist2)                                          */
  double dist2;  /* fp64 direct-form squared distance of the witness pair    */
  int64_t a;     /* witness row in the FIRST argument (the argmax row)       */
  int64_t b;     /* witness row in the SECOND argument (a's nearest point)   */
  double dist2_tc; /* the kernel's 3xTF32 row minimum of row a (diagnostic)  */
} prohd_directed;

typedef struct {
  double value;      /* max(ab.dist, ba.dist)                                */
  prohd_directed ab; /* h(A,B): a in A, b in B                               */
  prohd_directed ba; /* h(B,A): a in B, b in A                               */
} prohd_hd;

typedef struct {
  double value;      /* H^ = max(h(A_sel,B_sel), h(B_sel,A_sel)), Alg. 3 l.6-7 */
  prohd_directed ab; /* witnesses are ORIGINAL indices into A and B          */
  prohd_directed ba;
  int64_t size_a;    /* |I^A| (Alg. 3 return value)                   */
  int64_t size_b;    /* |I^B|                                                */
  int32_t n_dirs;    /* directions used: 1 + number of PCs kept (<= k+1)     */
  int32_t _pad;
} prohd_est;

/* ---------------------------------------------------------------- exact HD */
/* h(A,B) (Eq. 1). Cost nA*nB*D; the fused distance kernel never writes the
 * nA x nB distance matrix. Errors: PROHD_E_INVALID for null/empty/D<1,
 * PROHD_E_DATA for non-finite input, PROHD_E_WORKSPACE, PROHD_E_CUDA. */
int directed_hd(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB,
                int32_t D, prohd_directed* out);

/* H(A,B) = max(h(A,B), h(B,A)). */
int hausdorff(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB,
              int32_t D, prohd_hd* out);

/* Test hook: per-row minima of A against B, d2_i = min_j ||a_i - b_j||^2 as the
 * kernel computes them (split-precision tensor-core products, fp32 accumulation), written
 * to rowmin_dev (DEVICE, nA floats). */
int directed_hd_rowmin(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB,
                       int32_t D, float* rowmin_dev);

/* Test hook (SURVEY.md §8(c4) L6 for the undirected H): exactly the hausdorff()
 * launch sequence (one fused bidirectional K6 sweep for D >= 128, two directed sweeps below, both
 * about centre(A, B)), additionally exporting the per-row minima of both directions:
 * rowmin_dev[i] = min_j ||a_i - b_j||^2 (nA floats) and colmin_dev[j] = min_i ||a_i - b_j||^2
 * (nB floats), both DEVICE, as the kernel computes them; *out as hausdorff(). Errors as hausdorff()
 * plus PROHD_E_INVALID for null / host minima pointers. */
int hausdorff_minima(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                     float* rowmin_dev, float* colmin_dev, prohd_hd* out);

/* Test hook: step 1a of prohd_estimate alone -- the mean mu of A u B and
 * the covariance C = (1/N) sum (p - mu)(p - mu)^T (Alg. 2 lines 1-2) as the
 * library computes them for the directions, through the same Gram path (int8 tensor cores for
 * D <= 256 with D % 4 == 0 unless option k1_path = 0, else fp64 DMMA; the int8 pass falls
 * back to DMMA when a value leaves its sampled fixed-point range). mu_out (HOST, D), C_out (HOST,
 * D x D row-major), *path_out (HOST) = 1 if the int8 Gram produced C, 0 if the DMMA Gram did.
 * Workspace: prohd_workspace_bytes(nA, nB, D, 0, 1, flags). Errors as prohd_estimate. */
int prohd_covariance(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                     double* mu_out, double* C_out, int32_t* path_out);

/* Test hook (K3, Alg. 1 line 4 / Alg. 2 line 5; pi = x^T u,
 * P:139): the fp32 projections the selection starts from. X (DEVICE, n x D fp32 row-major),
 * dirs (DEVICE, L x D fp64, row l = direction u_l, 1 <= L <= 32; rounded to fp32 first);
 * proj_out (DEVICE, L x n fp32, direction-major: proj_out[l * n + i] ~= x_i . u_l);
 * *eps_out (HOST) = the bound the selection's fp64 re-rank band assumes:
 * |proj_out[l * n + i] - x_i . u_l (exact)| <= eps_out for every i, l. Workspace >= L*D*4 + 256
 * bytes. Errors: PROHD_E_INVALID (null, host pointers, bad sizes), PROHD_E_WORKSPACE,
 * PROHD_E_CUDA. */
int prohd_project(prohd_ctx* ctx, const float* X, int64_t n, int32_t D, const double* dirs, int32_t L,
                  float* proj_out, double* eps_out);

/* ---------------------------------------------------------------- ProHD   */
/* Alg. 3 with k principal directions plus the centroid axis and m points per
 * (set, direction, tail). 0 <= k <= D, m >= 1; if 2m >= n_X all of X is kept.
 * The device eigen-solver holds C in one thread-block cluster's shared memory (8 or 16 CTAs):
 * k > 0 needs D <= 512 (else PROHD_E_NOTIMPL); k = 0 (centroid axis only) takes any D.
 * Optional outputs (NULL to skip), HOST pointers:
 *   dirs_out  D x (k+1) fp64, column-major by direction (dirs_out[l*D + d]);
 *             column 0 is the centroid axis; columns >= n_dirs are zero.
 *   idxA_out  capacity min(nA, 2m(k+1)): sorted unique I^A (size_a entries)
 *   idxB_out  capacity min(nB, 2m(k+1)): sorted unique I^B (size_b entries) */
int prohd_estimate(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB,
                   int32_t D, int32_t k, int64_t m, prohd_est* out,
                   double* dirs_out, int64_t* idxA_out, int64_t* idxB_out);

/* Certified subset-full estimate: same selection as
 * prohd_estimate, then
 *   H^_sf = max( max_{a in A_sel} min_{b in B} ||a-b||, max_{b in B_sel} min_{a in A} ||b-a|| )
 * which never exceeds H(A,B) (each term is an exact directed distance of a subset of
 * the rows), restoring the paper's "never overestimates" claim that
 * Alg. 3's subset-subset estimate does not satisfy. Witness b indices refer to the full
 * sets. Cost |A_sel| nB + |B_sel| nA pairs. Workspace: PROHD_WS_CERTIFIED. */
int prohd_estimate_certified(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB,
                             int32_t D, int32_t k, int64_t m, prohd_est* out,
                             double* dirs_out, int64_t* idxA_out, int64_t* idxB_out);

/* Paper-literal parameterisation: Alg. 3 line 1
 * k = m_pc = max(1, floor(sqrt D)) principal directions, alpha' = alpha / m_pc; per-tail counts
 * max{1, floor(alpha n_X)} on the centroid axis (Alg. 1) and max{1, floor(alpha' n_X)}
 * on each PC (Alg. 2), per set. 0 < alpha < 1. Outputs as prohd_estimate (idx
 * capacities min(n_X, 2 (c0 + m_pc c1))). Workspace: prohd_workspace_bytes(nA, nB, D, m_pc,
 * max per-tail count, flags). */
int prohd_estimate_alpha(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB,
                         int32_t D, double alpha, prohd_est* out, double* dirs_out,
                         int64_t* idxA_out, int64_t* idxB_out);

/* H(A[idxA], B[idxB]) with witnesses as indices into A and B: the exact HD of two index
 * subsets (HOST or DEVICE int64 lists, 0 <= idx < n, duplicates allowed), one fused
 * bidirectional sweep. The paper's sampling baselines (Random Sampling, Systematic
 * Random Sampling) are this call on seeded index draws (datagen). Workspace:
 * prohd_workspace_bytes(max(nA,nB), max(nA,nB), D, 0, 1, flags) suffices. */
int hausdorff_subsets(prohd_ctx* ctx, const float* A, int64_t nA, const int64_t* idxA, int64_t kA,
                      const float* B, int64_t nB, const int64_t* idxB, int64_t kB, int32_t D,
                      prohd_hd* out);

/* Bound report for directions `dirs` (HOST, n_dirs x D fp64, row l =
 * u_l, 1 <= n_dirs <= 32), e.g. dirs_out of prohd_estimate:
 *   per_dir_out (HOST, n_dirs x 4): delta(u_l) through the origin (Eq. 2),
 *     delta(u_l) centred at the mean of A u B, h_u(A,B), h_u(B,A)
 *     (1-D Hausdorff distances of the projections);
 *   summary_out (HOST, 3): H_U = max_l H_u, min delta over both frames and all
 *     directions, and H_U + 2 min delta (the upper end of Eq. 4).
 * delta is evaluated from fp32 dot products and inflated by a bound of their rounding error, so
 * it never falls below the exact value (the interval stays valid); H_u uses the fp32
 * projections (|error| <= 2 (D+8) 2^-24 max ||p||). One extra pass over A and B plus a radix
 * sort of the n x n_dirs projections of each set. */
int prohd_bounds(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                 const double* dirs, int32_t n_dirs, double* per_dir_out, double* summary_out);

/* Test hook: steps 2-4 with caller-supplied directions
 * `dirs` (HOST, fp64, D x n_dirs, same layout as dirs_out; n_dirs >= 1). */
int prohd_estimate_with_dirs(prohd_ctx* ctx, const float* A, int64_t nA, const float* B,
                             int64_t nB, int32_t D, int32_t n_dirs, int64_t m,
                             const double* dirs, prohd_est* out, int64_t* idxA_out,
                             int64_t* idxB_out);

/* ---------------------------------------------------------------- sharding */
/* Row-sharded exact HD: this rank holds rows
 * [row_offset, row_offset + nA_local) of the full A and all of B. Writes the
 * rank's packed key  (float_bits(d2_tc) << 32) | (0xFFFFFFFF - global_row)
 * (max over ranks = global argmax, lowest row on ties) to *key_out (HOST).
 * The caller all-reduces the key (MAX), then calls directed_hd_witness on the
 * rank that owns the winning row. `centre` (HOST or DEVICE, D fp64, or NULL): the
 * common translation applied before the tensor-core distances (K0); NULL = the
 * default of directed_hd, prohd_centre(NULL, 0, B, nB), so any shard count reproduces
 * directed_hd's key bit for bit. The sharded subset HD passes prohd_centre(A_sel, B_sel),
 * the centre prohd_estimate uses. */
int directed_hd_local(prohd_ctx* ctx, const float* A_local, int64_t nA_local, int64_t row_offset,
                      const float* B, int64_t nB, int32_t D, const double* centre, uint64_t* key_out);
/* Common centre of a pair (HOST out, D fp64): the fp64 mean of the first min(nX, 4096)
 * rows of X and the first min(nY, 4096) rows of Y (DEVICE inputs; either count may be 0),
 * per-set sums added last so centre(X, Y) == centre(Y, X) bit for bit. The distance
 * operands are prepared about this point (directed_hd: centre(-, B); hausdorff and the
 * subset HD of prohd_estimate: centre(A, B) of the pair they compare). Workspace: 2D
 * doubles. */
int prohd_centre(prohd_ctx* ctx, const float* X, int64_t nX, const float* Y, int64_t nY, int32_t D,
                 double* centre_out);
/* fp64 nearest neighbour of one point a (HOST or DEVICE, D floats) in B:
 * fills out->b, out->dist2, out->dist (out->a is left to the caller). */
int directed_hd_witness(prohd_ctx* ctx, const float* a, const float* B, int64_t nB, int32_t D,
                        prohd_directed* out);

/* ------------------------------------------------- sharded ProHD (phase calls)
 * Alg. 3 with the rows of A and of B split across ranks. The caller
 * (paper_2511_18207_b200/dist.py) runs the collectives between the calls:
 *   s = prohd_shift(rank 0's first rows)            -> broadcast s
 *   prohd_local_colmax(own rows, s)                 -> all_reduce(MAX)      (C0, int8 Gram)
 *   prohd_local_moments[_i8](own rows, s[, colmax]) -> all_reduce(SUM)      (C1)
 *   prohd_directions(reduced moments)               (replicated, deterministic)
 *   prohd_local_candidates(own rows, global offset) -> all_gather           (C2)
 *   prohd_merge_union(all lists)                    (replicated)
 *   prohd_gather_owned(own rows of the union)       -> all_gather           (C3)
 *   directed_hd_local on a row shard of each subset -> all_reduce(MAX)      (C4)
 * The merged lists equal the single-GPU lists (same fp64 values, same order).
 * Workspace: prohd_shard_workspace_bytes(max local rows, max total rows, D, k, m, flags). */
size_t prohd_shard_workspace_bytes(int64_t n_local_max, int64_t n_total_max, int32_t D, int32_t k,
                                   int64_t m, uint32_t flags);
/* Shift s (HOST out, D fp64): the fp64 mean m of the first min(n, 4096) rows of A and of
 * B if that offset is large against the rows' spread (sum m_f^2 > 1024 sum var_f), else all
 * zeros (the moments are then taken about the origin: fp32 products are exact in fp64,
 * and the bounded offset bounds the cancellation in C = G/N - mu mu^T). Any s is valid
 * for prohd_local_moments / prohd_directions as long as every rank uses the same one. */
int prohd_shift(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                double* shift_out);
/* This rank's moments about s (HOST, D fp64): moments_out (DEVICE, 2D + D*D fp64) =
 * [S_A | S_B | G], S_X = sum (x - s), G = sum over own A and B rows of (p - s)(p - s)^T
 * (full, row-major). n_local may be 0. */
int prohd_local_moments(prohd_ctx* ctx, const float* A_local, int64_t nA_local, const float* B_local,
                        int64_t nB_local, int32_t D, const double* shift, double* moments_out);
/* The same moments on the int8 tensor cores (the Gram prohd_estimate uses, k_gram_i8.cu), in two
 * calls around one MAX all-reduce so that every rank quantises on the same fixed-point grid
 * (Alg. 2 lines 1-2; SURVEY.md §8(e) "shard the Gram and centroid sums"):
 *   prohd_local_colmax: colmax_out (DEVICE, D fp32) = max over own A and B rows of |x_f - s_f|
 *     (+inf for non-finite input; 0 without rows)                 -> all_reduce(MAX)
 *   prohd_local_moments_i8: moments_out (DEVICE, 2D + D*D fp64) exactly as prohd_local_moments,
 *     from the int8 Gram on the grid of colmax (DEVICE, D fp32, the all-reduced maxima), re-expressed
 *     about s. A non-finite colmax entry selects the fp64 DMMA Gram (whose sums then carry the
 *     non-finite value to prohd_directions: PROHD_E_DATA there).
 * Both need D <= 256 and D % 4 == 0 (else PROHD_E_NOTIMPL: use prohd_local_moments); shift is
 * HOST (D fp64, the broadcast prohd_shift). n_local may be 0. Blocking. */
int prohd_local_colmax(prohd_ctx* ctx, const float* A_local, int64_t nA_local, const float* B_local,
                       int64_t nB_local, int32_t D, const double* shift, float* colmax_out);
int prohd_local_moments_i8(prohd_ctx* ctx, const float* A_local, int64_t nA_local, const float* B_local,
                           int64_t nB_local, int32_t D, const double* shift, const float* colmax,
                           double* moments_out);
/* Directions from the all-reduced moments (DEVICE) of nA + nB points: dirs_out (DEVICE,
 * (k+1) x D fp64, row l = direction l, row 0 = centroid axis), *n_dirs_out (HOST). */
int prohd_directions(prohd_ctx* ctx, const double* moments, int64_t nA, int64_t nB, int32_t D, int32_t k,
                     const double* shift, double* dirs_out, int32_t* n_dirs_out);
/* Local top/bottom-m per direction of rows X_local (global rows row_offset + i): lists
 * (DEVICE, [n_dirs][2 (top, bottom)][m]) of fp64 projection values and GLOBAL indices, in
 * list order; empty slots have index -1. */
int prohd_local_candidates(prohd_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset,
                           int32_t D, const double* dirs, int32_t n_dirs, int64_t m,
                           double* cand_val_out, int64_t* cand_idx_out);
/* Merge G ranks' lists (DEVICE, [G][n_dirs][2][m]) into the sorted unique union of global
 * indices (DEVICE out, capacity min(n_total, 2 m n_dirs)); *count_out (HOST). */
int prohd_merge_union(prohd_ctx* ctx, const double* cand_val, const int64_t* cand_idx, int32_t G,
                      int32_t n_dirs, int64_t m, int64_t n_total, int64_t* union_out,
                      int64_t* count_out);
/* Rows of X_local (DEVICE) whose global index is in the sorted union (DEVICE), in union
 * order -> rows_out (DEVICE); *first_out = their position in the union, *count_out. */
int prohd_gather_owned(prohd_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset,
                       int32_t D, const int64_t* union_idx, int64_t union_count, float* rows_out,
                       int64_t* first_out, int64_t* count_out);

/* ---------------------------------------------------------------- tracing */
/* Per-phase device times of the LAST call on this context, measured with CUDA
 * events recorded on the context stream around each phase (enable first;
 * disabled by default; costs two event records per phase). A phase that did
 * not run reads 0. */
typedef struct {
  double total_ms;          /* first to last enqueued operation of the call          */
  double h2d_ms;            /* staging copies of host inputs                        */
  double prep_ms;           /* K0 TF32 hi/lo split + norms (full sets)              */
  double dist_ms;           /* K6 fused distance kernel, summed over its launches   */
  double reduce_ms;         /* K7 row-max key + fp64 witness search                 */
  double moments_ms;        /* K1 centroid sums + covariance                        */
  double eigen_ms;          /* K2 top-k eigenvectors                                */
  double select_ms;         /* K3 projection + K4 selection + K5 union (both sets)  */
  double subset_ms;         /* step 4: gather + K0 + K6 + K7 on the subsets         */
  int32_t dist_launches;    /* number of K6 launches in dist_ms                     */
  int32_t kernel_launches;  /* all kernels this call launched                       */
} prohd_timings;
int prohd_enable_timing(prohd_ctx* ctx, int on);
int prohd_last_timings(const prohd_ctx* ctx, prohd_timings* out);

#ifdef __cplusplus
}
#endif
#endif /* PROHD_H_ */
