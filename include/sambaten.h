/*
 * sambaten.h -- C-ABI of the B200-native SamBaTen per-batch incremental CP update.
 *
 * Paper: Gujral, Pasricha, Papalexakis, "SamBaTen: Sampling-based Batch Incremental Tensor
 * Decomposition", arXiv 1709.00668.  "P:n" below is line n of the paper's text;
 * "Rn" is reading n in DESIGN.md section 2 (where the paper is silent or garbled).
 *
 * General conventions
 *  - All functions return a sambaten_status; SAMBATEN_OK == 0.  The message of the last
 *    failure on the calling thread is available from sambaten_last_error().
 *  - A dense tensor X of dims (I, J, K) is a float32 array with X(i,j,k) at
 *    vals[i + I*(j + J*k)]: i fastest, frontal slices X(:,:,k) contiguous.
 *  - A sparse tensor is COO: int32 idx[0..2][n] (0-based i, j, k) and float32 vals[n].
 *    Inputs to sambaten_init / sambaten_update must be canonical: sorted by (k, j, i),
 *    without duplicates or explicit zeros (R28); violations return SAMBATEN_E_INVALID.
 *  - Factor matrices are float32 row-major [rows][R] (R innermost); lambda is float32[R].
 *  - Pointers passed to stateless primitives (sambaten_marginals ... sambaten_fit) are
 *    DEVICE pointers unless stated otherwise; work is enqueued on `stream` (a cudaStream_t,
 *    NULL = legacy default stream) and the call returns without synchronising.
 *  - Handle-based calls accept host or device buffers for tensors and factors (the copy
 *    direction is taken from the pointer; sambaten_tensor.on_device is advisory) and
 *    synchronise their stream once before returning, so that they can report a status.
 *  - Only sm_100a (B200) devices are supported.  There is no CPU fallback: without a
 *    usable CUDA device every compute call returns SAMBATEN_E_CUDA.
 *  - A handle is not thread-safe; distinct handles may be used from distinct threads.
 */
#ifndef SAMBATEN_H_
#define SAMBATEN_H_

#include <stdint.h>

#if defined(__GNUC__)
#define SAMBATEN_API __attribute__((visibility("default")))
#else
#define SAMBATEN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sambaten_s* sambaten_t; /* opaque; owns the tensor store, model, workspaces */

typedef enum {
  SAMBATEN_OK = 0,
  SAMBATEN_E_INVALID = -1,          /* bad argument (NULL, negative size, R > 32, ...)      */
  SAMBATEN_E_SHAPE = -2,            /* I or J of a batch differs from the state's    */
  SAMBATEN_E_DEGENERATE = -3,       /* all-zero initial tensor                      */
  SAMBATEN_E_EMPTY_BATCH = -4,      /* batch with zero slices                       */
  SAMBATEN_E_INDEX_RANGE = -5,      /* index outside its mode                        */
  SAMBATEN_E_NUMERICAL = -6,        /* non-finite value in ALS                      */
  SAMBATEN_E_BATCH_REJECTED = -7,   /* every repetition failed the acceptance test (R26)    */
  SAMBATEN_E_FIXEDPOINT_RANGE = -8, /* batch value outside the fixed-point range (R7)       */
  SAMBATEN_E_OOM = -9,              /* device allocation failed / capacity exceeded         */
  SAMBATEN_E_CUDA = -10             /* CUDA runtime error (message has the CUDA string)     */
} sambaten_status;

enum { SAMBATEN_DENSE = 0, SAMBATEN_COO = 1 };
enum { SAMBATEN_MOI_ABS = 0,  /* phi(x) = |x|  (BASELINE north_star, R1)   */
       SAMBATEN_MOI_SQ = 1 }; /* phi(x) = x^2  (Eq. 1)         */

typedef struct {
  int fmt;                /* SAMBATEN_DENSE or SAMBATEN_COO                                 */
  int64_t dims[3];        /* I, J, K (K = number of frontal slices in this tensor / batch)  */
  const float* vals;      /* dense: I*J*K values (layout above); COO: nnz values            */
  const int32_t* idx[3];  /* COO only: i, j, k coordinates (k relative to this tensor)      */
  int64_t nnz;            /* COO only                                                       */
  int on_device;          /* 1 if vals/idx are device pointers (advisory)                   */
} sambaten_tensor;

typedef struct {
  int als_max_iters;      /* ALS iterations per summary (R11); default 30                     */
  double als_tol;         /* stop when it >= 2 and |fit - fit_prev| < tol; 0 = fixed count   */
  int moi;                /* SAMBATEN_MOI_ABS (default) or SAMBATEN_MOI_SQ (R1)              */
  int s_mode[3];          /* per-mode sampling factor; 0 = use the `s` argument      */
  int merge_policy;       /* 0 = update zero entries only (default); 1 = overwrite    */
                          /*     the sampled rows (R17)                              */
  double accept_tau;      /* rep acceptance threshold on min_f S(f, pi f) (R26); default 0.9 */
  int full_fit;           /* 1: sambaten_update also computes the full relative error of the   */
                          /*    model it commits (a7): on dense handles kept up to date from the */
                          /*    previous model's per-component inner products (the batch's      */
                          /*    slices plus the rows the merge changed; exact algebra, O(batch)  */
                          /*    bytes), else one pass over the tensor;                           */
                          /* 2: lag-1 fused fit: the relative error of the */
                          /*    model the PREVIOUS update (or init) committed is computed inside  */
                          /*    this update's marginal pass over the old slices, which reads the  */
                          /*    same bytes (dense handles, full marginals, fit-stream shapes),    */
                          /*    reported as info.fit_full_prev (info.fit_full = -1); where it     */
                          /*    does not apply (incremental marginals, COO, unsupported shape)    */
                          /*    it behaves as 1.  sambaten_relative_error gives the last model's. */
  int64_t capacity;       /* dense: total K slices to preallocate; COO: total nnz; 0 = 2x X0 */
  int64_t capacity_k;     /* COO: mode-3 rows of C to preallocate; 0 = 2 K0 + 1024          */
  int init_max_iters;     /* sambaten_init: ALS iterations on X0 (default 1000)       */
  double init_tol;        /* sambaten_init: tolerance (default 1e-6)                         */
  void* stream;           /* cudaStream_t for all work of this handle; NULL = default       */
  int borrow_store;       /* dense init only: X0->vals is a DEVICE buffer with room for       */
                          /* `capacity` slices (I % 4 == 0); the handle uses it as its tensor */
                          /* store in place (no copy of X0).  sambaten_init_factors_dist: the */
                          /* rank's slab buffer holds Kcap_local = K0_local + ceil((capacity -*/
                          /* K0_global) / world) + 1 slices.  The caller keeps it alive and   */
                          /* unmodified until sambaten_destroy.  Default 0 (copy).            */
  int incremental_marginals; /* 1: a1 adds the batch's contribution to the marginals kept from */
                          /* the previous update instead of re-reading the whole tensor --    */
                          /* bit-identical (integer sums); the first     */
                          /* update after init / restore makes the full pass.  Default 0.     */
  int getrank;            /* 1: before each summary decomposition run GetRank (Alg. 2,        */
                          /* P:279-294) on the summary and decompose at the rank it returns;  */
                          /* only those components are matched and merged (P:264-266,        */
                          /* readings R29-R33).  Dense and COO handles (COO: the sparse       */
                          /* CorConDia), single-GPU and sharded (each rank rates its owned    */
                          /* repetitions, the ranks are allgathered).  Default 0.             */
  int getrank_trials;     /* CP runs per candidate rank (Alg. 2 `it`); default 1              */
  double getrank_threshold; /* CorConDia cut-off of R31; default 90                           */
  int warm_start;         /* 1: each summary ALS starts from the model's rows (A(I_s), B(J_s),  */
                          /* C(K_s) diag(lambda), zero rows for the new slices   */
                          /* NEXT #4, reading R34) instead of the Philox point.  Dense and    */
                          /* COO handles, single-GPU and sharded; not with getrank (else      */
                          /* SAMBATEN_E_INVALID).                                             */
  int pipelined;          /* 1: update t+1 samples from the marginals update t committed (the  */
                          /* tensor BEFORE its batch, reading R36),*/
                          /* so sampling and gather do not wait for this update's marginal    */
                          /* pass, which runs on a side stream overlapped with a2..a7 and is  */
                          /* committed for the next update.  Dense single-GPU handles (else   */
                          /* SAMBATEN_E_INVALID).  Default 0.                                 */
} sambaten_opts;

typedef struct {
  double fit_summary;          /* mean over repetitions of the summary ALS fit (R21)         */
  double fit_full;             /* 1 - ||X - model||/||X|| over the whole tensor if full_fit,  */
                               /* else -1                                         */
  int als_iters_max;           /* largest ALS iteration count over repetitions               */
  int64_t k_total;             /* slices (mode-3 extent) after the update                    */
  uint32_t reps_rejected_mask; /* bit rho set if repetition rho was rejected (R26; r <= 32)  */
  int scale_exp;               /* fixed-point exponent S of the marginals (R7)                */
  int kernel_launches;         /* CUDA kernels this update launched (all are this library's) */
  uint32_t reps_pinv_mask;     /* bit rho set if repetition rho's ALS used the pseudo-inverse  */
                               /* fallback (R12) at least once                                */
  double step_ms[8];           /* device time of steps a0..a7 (CUDA events)                   */
  int als_iters_sum;           /* ALS iterations summed over the repetitions (work accounting) */
  int rep_rank[32];            /* rank each repetition decomposed its summary at (R unless    */
                               /* opts.getrank reduced it, R33); entries >= r are 0           */
  int als_plan[4];             /* the a4 launch plan this update ran:                          */
                               /* [0] kind: 0 multi-kernel ALS, 1 cluster ALS (one thread-    */
                               /* block cluster per repetition), 2 grid ALS (CTA groups of one */
                               /* cooperative grid, global-memory exchange), COO handles: 3   */
                               /* persistent cooperative ALS (k_coo_als.cu), 4 per-mode kernel */
                               /* pipeline (R > 16 / SAMBATEN_COO_ALS_MULTI); -1 none (GetRank)*/
                               /* [1] CTAs per repetition, [2] RB (padded rank width),        */
                               /* [3] 1 if D lives in shared memory, 0 if in global memory     */
  int64_t summary_entries;     /* entries (dense) or nonzeros (COO) of the summaries this      */
                               /* rank decomposed, summed over its repetitions (work units of  */
                               /* a3 / a4 for the rooflines)                                   */
  double fit_full_prev;        /* full_fit = 2: 1 - ||X_prev - model_prev||/||X_prev|| of the    */
                               /* model the previous update committed, over the tensor it was   */
                               /* committed on (computed in this update's a1 pass); else -1     */
  int fit_path;                /* how the full fit was obtained: 0 none, 1 separate pass over  */
                               /* the tensor, 2 lag-1 inside a1, 3 incremental (the batch plus */
                               /* the rows the merge changed), 4 incremental plan fell back to */
                               /* one full per-component pass                                   */
} sambaten_info;

/* Fill *opts with the defaults listed above. */
SAMBATEN_API void sambaten_default_opts(sambaten_opts* opts);

/* ---------------------------------------------------------------------------------------
 * Handle API: the incremental update of Problem 1 and Alg. 1.
 * ------------------------------------------------------------------------------------- */

/* Create a handle from the existing tensor X0 (I x J x K0) and decompose it with full
 * CP-ALS at rank R (the "existing data"; Philox init R10, update_id 0).
 * s: sampling factor for every mode unless opts->s_mode overrides it;
 * r: repetitions per batch, 1 <= r <= 32; seed: Philox key (R6); 1 <= R <= 32.
 * Errors: E_INVALID, E_DEGENERATE (all-zero X0), E_INDEX_RANGE, E_OOM, E_CUDA. On error
 * *h is set to NULL. */
SAMBATEN_API sambaten_status sambaten_init(sambaten_t* h, const sambaten_tensor* X0, int R, int s, int r,
                              uint64_t seed, const sambaten_opts* opts);

/* As sambaten_init, but the model [lambda; A, B, C] (float32, host or device; C has K0
 * rows) is given instead of computed.  Used for parity tests and the throughput bench. */
SAMBATEN_API sambaten_status sambaten_init_factors(sambaten_t* h, const sambaten_tensor* X0, int R, int s,
                                      int r, uint64_t seed, const float* A, const float* B,
                                      const float* C, const float* lambda,
                                      const sambaten_opts* opts);

/* One SamBaTen update with the batch X_new (I x J x K_new, K_new >= 1): steps a0..a7 of
 * DESIGN.md (ingest, marginals, sampling, gather, batched CP-ALS, matching, merge, fit).
 * On success the model has K_old + K_new rows of C.  If A, B, C, lambda are
 * non-NULL the updated factors are copied there (host or device; C gets K_old+K_new rows).
 * info may be NULL.  Strong guarantee: on any error the state is unchanged.
 * Errors: E_INVALID, E_SHAPE, E_EMPTY_BATCH, E_INDEX_RANGE, E_FIXEDPOINT_RANGE,
 * E_BATCH_REJECTED, E_NUMERICAL, E_OOM (capacity exceeded), E_CUDA. */
SAMBATEN_API sambaten_status sambaten_update(sambaten_t h, const sambaten_tensor* batch, float* A, float* B,
                                float* C, float* lambda, sambaten_info* info);

/* Device pointers to the current model (valid until the next mutating call) and dims. */
SAMBATEN_API sambaten_status sambaten_get_factors(sambaten_t h, const float** A, const float** B,
                                     const float** C, const float** lambda, int64_t dims[3],
                                     int* R);

/* Copy the current model into caller buffers (host or device by pointer; any may be NULL):
 * A [I][R], B [J][R], C [K][R] (K = current mode-3 extent), lambda [R], float32 row-major.
 * Synchronises the handle's stream. */
SAMBATEN_API sambaten_status sambaten_copy_factors(sambaten_t h, float* A, float* B, float* C,
                                      float* lambda);

/* Sample sets of the last update, copied to caller (host or device) buffers of
 * r * n_mode int32 each (rep-major): I_s, J_s, K_s (sorted, R9).  Any pointer may be NULL.
 * n_out[3] receives n_I, n_J, n_Ks. */
SAMBATEN_API sambaten_status sambaten_last_samples(sambaten_t h, int32_t* Is, int32_t* Js, int32_t* Ks,
                                      int64_t n_out[3]);

/* Full relative error ||X - [[lambda; A, B, C]]||_F / ||X||_F of the current model over the
 * whole retained tensor. */
SAMBATEN_API sambaten_status sambaten_relative_error(sambaten_t h, double* relerr);

/* In-memory checkpoint of (model, K extent, update counter) and its restore; the tensor
 * store is append-only, so restore discards slices appended after the checkpoint.
 * Deterministic resume: Philox counters depend only on (seed, update_id, rep, mode, index). */
SAMBATEN_API sambaten_status sambaten_checkpoint(sambaten_t h);
SAMBATEN_API sambaten_status sambaten_restore(sambaten_t h);

SAMBATEN_API void sambaten_destroy(sambaten_t h);

/* ---------------------------------------------------------------------------------------
 * Sharded update over G ranks (one process per GPU, NCCL, DESIGN.md
 * "Multi-GPU").  Every rank holds the frontal slices it ingested (its slab of X0 and its
 * share of every batch); marginals are combined by one int64 allreduce, repetition rho is
 * decomposed on rank rho mod G from summary slices exchanged by one all-to-all-v, and the
 * per-repetition results are allgathered before the (replicated) merge.  Dense and COO
 * stores (the COO handle keeps the canonical entries of its slices; R32).
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int rank, world;              /* this process and the number of ranks                     */
  unsigned char nccl_id[128];   /* from sambaten_dist_unique_id on one rank, broadcast by the */
                                /* caller's own process-group plumbing                        */
  int64_t k0;                   /* first global frontal slice of this rank's slab of X0       */
  int64_t K0_global;            /* mode-3 extent of the whole initial tensor                   */
} sambaten_dist;

/* A fresh NCCL unique id (128 bytes) for sambaten_dist.nccl_id. */
SAMBATEN_API sambaten_status sambaten_dist_unique_id(unsigned char id[128]);

/* Collective: every rank passes its slab X0_local (dims[2] slices starting at global slice
 * dist->k0; the slabs must tile [0, K0_global) exactly) and the same replicated model
 * (C has K0_global rows).  r must be a multiple of world.  opts->capacity is the GLOBAL
 * mode-3 capacity.  Errors as sambaten_init_factors, plus E_INVALID for a bad tiling. */
SAMBATEN_API sambaten_status sambaten_init_factors_dist(sambaten_t* h, const sambaten_tensor* X0_local,
                                           const sambaten_dist* dist, int R, int s, int r,
                                           uint64_t seed, const float* A, const float* B,
                                           const float* C, const float* lambda,
                                           const sambaten_opts* opts);

/* Host-only (no GPU): the summary-exchange plan of one rank.  Kp: the r K' lists (global
 * slice indices, rep-major, nKp each); owner_old[k]: rank storing slice k < K_old; the new
 * slices [K_old, K_old + K_new) are split by sambaten_batch_partition.  Repetition rho is
 * owned by rank rho % world.  send_slices[g] / recv_slices[g] (world entries each): summary
 * slices this rank sends to / receives from rank g (0 for g == rank).  Used by the sharded
 * update; exposed for testing the plan across processes. */
SAMBATEN_API sambaten_status sambaten_dist_plan(const int32_t* Kp, int r, int64_t nKp,
                                   const int32_t* owner_old, int64_t K_old, int64_t K_new,
                                   int world, int rank, int64_t* send_slices, int64_t* recv_slices);

/* The slices [K_old + *k_begin, K_old + *k_begin + *k_count) of a batch of K_new slices that
 * this rank passes to sambaten_update (contiguous, balanced; single-GPU handles: all). */
SAMBATEN_API sambaten_status sambaten_batch_partition(sambaten_t h, int64_t K_new, int64_t* k_begin,
                                         int64_t* k_count);

/* ---------------------------------------------------------------------------------------
 * Stateless primitives (device pointers, enqueue on `stream`, no synchronisation).
 * ------------------------------------------------------------------------------------- */

/* Fixed-point exponent S = 62 - ceil(log2 cap_entries) - ceil(log2 max_phi) - 8, clamped
 * to [-60, 120] (R7).  Host-only arithmetic; max_phi must be > 0. */
SAMBATEN_API int sambaten_fixed_point_scale(int64_t cap_entries, double max_phi);

/* Measure of importance (Eq. 1; R1, R7): with q(x) = RNE(phi(x) * 2^S) in int64,
 * x1[i] = sum_{j,k} q(X(i,j,k)), x2[j] = sum_{i,k} q, x3[k] = sum_{i,j} q, over the dense or
 * COO tensor X (device).  x1, x2, x3: device int64 arrays of I, J, K entries, OVERWRITTEN.
 * Exact and independent of launch configuration (integer sums). */
SAMBATEN_API sambaten_status sambaten_marginals(const sambaten_tensor* X, int moi, int scale_exp,
                                   int64_t* x1, int64_t* x2, int64_t* x3, void* stream);

/* Importance sample without replacement (Alg. 1 line 3 P:211; R4-R6): the n_s
 * smallest (key_i, i), key_i = -ln(u_i)/w[i] (+inf if w[i] == 0), u_i from Philox4x32-10
 * with key = seed and counter (i, 0, update_id, 1<<24 | rep<<8 | mode), written sorted
 * ascending to out_idx[0..n_s).  w: device int64[n]; 0 <= n_s <= n. */
SAMBATEN_API sambaten_status sambaten_sample(const int64_t* w, int64_t n, int64_t n_s, uint64_t seed,
                                uint32_t update_id, uint32_t rep, uint32_t mode,
                                int32_t* out_idx, void* stream);

/* Summary gather (Alg. 1 line 4 P:212): Y(p,q,u) = X(Is[p], Js[q], Ks[u]).
 * Dense X: out_dense is float32 [nK][nJ][nI] (p fastest).  COO X: the entries whose three
 * coordinates are sampled, relabelled to (p, q, u), in canonical (u, q, p) order, written
 * to out_idx[0..2] / out_vals (capacity out_cap entries); *out_nnz (device int64) gets the
 * count.  Index lists: device int32, sorted ascending, distinct. */
SAMBATEN_API sambaten_status sambaten_gather(const sambaten_tensor* X, const int32_t* Is, int64_t nI,
                                const int32_t* Js, int64_t nJ, const int32_t* Ks, int64_t nK,
                                float* out_dense, int32_t* out_idx_i, int32_t* out_idx_j,
                                int32_t* out_idx_k, float* out_vals, int64_t out_cap,
                                int64_t* out_nnz, void* stream);

/* MTTKRP: M = X_(mode) (Khatri-Rao product of the other two factors), i.e.
 * M(i,f) = sum_{j,k} X(i,j,k) U1(j,f) U2(k,f) for mode 0 and likewise for modes 1, 2.
 * U0, U1, U2: device float32 row-major [dims[m]][R] (the one of `mode` is ignored);
 * M: device float32 [dims[mode]][R].  1 <= R <= 32.  fp32 products, fp64 partial sums. */
SAMBATEN_API sambaten_status sambaten_mttkrp(const sambaten_tensor* X, const float* U0, const float* U1,
                                const float* U2, int R, int mode, float* M, void* stream);

/* CP-ALS on one tensor, starting from U0, U1, U2 (device float32, overwritten by
 * the column-normalised result); lambda_out: device float64[R].  Iterations as in R11:
 * modes 0,1,2 each: M = mttkrp, V = Hadamard of the other Grams, U = M V^-1 (Cholesky,
 * pseudo-inverse fallback R12), lambda = column 2-norms, normalise.  fit_out: device
 * float64[1], iters_out: device int32[1]. */
SAMBATEN_API sambaten_status sambaten_cp_als(const sambaten_tensor* X, int R, float* U0, float* U1,
                                float* U2, double* lambda_out, int max_iters, double tol,
                                double* fit_out, int32_t* iters_out, void* stream);

/* ---------------------------------------------------------------------------------------
 * Full-tensor CP-ALS: the evaluation's CP_ALS baseline and relative
 * fitness, and the distributed initial decomposition.
 * ------------------------------------------------------------------------------------- */

/* The CP_ALS baseline of the paper's evaluation ("re-compute CP using CP_ALS every time
 * a new batch update arrives"; P:232 ALS): full CP-ALS at the handle's rank of its CURRENT
 * tensor (all stored slices), from the Philox U(0,1) point with counter update_id = the
 * handle's update count and repetition 255 (reading R35), at most max_iters iterations, stop
 * when |fit - fit_prev| < tol (R11).  Sharded dense handles: collective, the slabs' MTTKRP
 * partials all-reduced (NCCL), every rank gets the same factors.  The handle's model is not
 * touched.  A [I][R], B [J][R], C [K][R], lambda [R] (host or device, NULL = not copied);
 * relerr: 1 - the final ALS fit = relative error of that model; iters: the count.
 * Errors: E_INVALID (NULL handle, max_iters < 1, sharded COO), E_OOM, E_CUDA. */
SAMBATEN_API sambaten_status sambaten_recompute(sambaten_t h, int max_iters, double tol, float* A, float* B,
                                                float* C, float* lambda, double* relerr, int* iters);

/* Relative fitness = ||X - X_SamBaTen|| / ||X - X_CPALS|| of the handle's committed
 * model against sambaten_recompute's; also returns both relative errors (NULL = not
 * returned).  Lower is better; 1 = as good as recomputing.  Collective on sharded handles. */
SAMBATEN_API sambaten_status sambaten_relative_fitness(sambaten_t h, int max_iters, double tol, double* rf,
                                                       double* relerr_sambaten, double* relerr_baseline);

/* The sharded handle initialised by the DISTRIBUTED full CP-ALS of X0 ("10% as
 * existing"; R10 Philox init, update_id 0, rep 0; opts->init_max_iters / init_tol): every rank
 * passes its slab [dist->k0, dist->k0 + dims[2]) of X0; the slabs' MTTKRP partials are
 * all-reduced and the mode-2 rows all-gathered (NCCL) so every rank holds the same model.
 * Dense tensors only.  Errors as sambaten_init_factors_dist. */
SAMBATEN_API sambaten_status sambaten_init_dist(sambaten_t* h, const sambaten_tensor* X0_local,
                                                const sambaten_dist* dist, int R, int s, int r, uint64_t seed,
                                                const sambaten_opts* opts);

/* The a4 plan (sambaten_info.als_plan layout) the library would pick for r dense summaries of
 * shape nI x nJ x nK at rank R on the current device (no handle; host call that queries the
 * device's cluster occupancy).  Lets a test assert that a small problem runs the same kernel
 * instantiation as a large one.  Errors: E_INVALID (bad sizes), E_CUDA. */
SAMBATEN_API sambaten_status sambaten_als_plan(int nI, int nJ, int nK, int R, int r, int plan[4]);

/* ---- GetRank quality control (Alg. 2) ------------------------
 * Core consistency (CorConDia, P:266 [bro2003new]; reading R29) of the rank-F model
 * [[lambda; A, B, C]] of the tensor X: with lambda absorbed into A, the least-squares core
 * G = X x1 pinv(A) x2 pinv(B) x3 pinv(C) and cc = 100 (1 - sum (G - T)^2 / F), T the
 * superdiagonal unit core.  Dense X, or a canonical COO X in DEVICE memory (sorted by (k,j,i)):
 * the core is then formed from the nonzeros fibre by fibre ("exploits sparsity").
 * A, B, C: device float32 [dims][F] row-major; lambda: device float64[F]; cc: host or device
 * float64[1].  fp64 throughout; E_INVALID on bad arguments. */
SAMBATEN_API sambaten_status sambaten_corcondia(const sambaten_tensor* X, int F, const float* A, const float* B,
                                   const float* C, const double* lambda, double* cc, void* stream);

/* Alg. 2 on the (summary) tensor X, dense or canonical COO in device memory (the COO ALS and
 * the sparse CorConDia): for every candidate rank F = 1..R_max and trial
 * j < trials, CP-ALS (max_iters, tol as sambaten_cp_als) from the Philox initialisation with
 * update_id = 0x47520000 + F and repetition j (R30), rated by CorConDia; R_new = the largest F
 * whose best trial reaches `threshold` (R31; 90 is customary), else 1.  cc: host float64
 * [R_max][trials] (may be NULL); the call synchronises the stream. */
SAMBATEN_API sambaten_status sambaten_getrank(const sambaten_tensor* X, int R_max, int trials, uint64_t seed,
                                 int max_iters, double tol, double threshold, int* R_new, double* cc,
                                 void* stream);

/* Relative error ||X - [[lambda; A, B, C]]||_F / ||X||_F of a dense or COO
 * tensor X against a model (device float32); relerr: device float64[1]. */
SAMBATEN_API sambaten_status sambaten_fit(const sambaten_tensor* X, const float* lambda, const float* A,
                             const float* B, const float* C, int R, double* relerr,
                             void* stream);

/* Philox4x32-10 (R6) on device for the cross-check tests: out[4*t..4*t+3] = Philox(counter
 * (c0 + t, c1, c2, c3), key) for t < n.  out: device uint32[4n]. */
SAMBATEN_API sambaten_status sambaten_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                uint64_t key, int64_t n, uint32_t* out, void* stream);

/* detlog (R7) on device: out[t] = detlog(u[t]) for u in (0,1). Device float64 arrays. */
SAMBATEN_API sambaten_status sambaten_detlog(const double* u, int64_t n, double* out, void* stream);

/* Message of the last failure on this thread ("" if none). */
SAMBATEN_API const char* sambaten_last_error(void);

/* Library version string. */
SAMBATEN_API const char* sambaten_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SAMBATEN_H_ */
