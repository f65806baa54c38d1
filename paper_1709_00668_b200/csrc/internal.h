// internal.h -- launchers shared between the kernel translation units and the engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

namespace sbt {

// ---- errors ---------------------------------------------------------------------------
void set_error(const std::string& msg);
#define SBT_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      ::sbt::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));            \
      return SAMBATEN_E_CUDA;                                                          \
    }                                                                                  \
  } while (0)

// ---- dense tensor view: X(i,j,k) at base[(k*J + j)*pitch + i] ---------------------------
struct DenseView {
  const float* base;
  int64_t I, J, K;
  int64_t pitch;
};

// a1: marginals over slices [k0, k0+nk) of a dense view; x1/x2/x3 (x3 indexed by absolute
// k) are accumulated with integer atomics (callers zero them first).
cudaError_t launch_marginals_dense(const DenseView& X, int64_t k0, int64_t nk, int moi, int S,
                                   int64_t* x1, int64_t* x2, int64_t* x3, cudaStream_t st);
// x1/x2/x3 are added to.  rep_ws (nrep * (I + J) int64, nrep = marg_coo_replicas(...) >= 2):
// the replicated kernel for large Zipf-hot stores; NULL: one global atomic per entry and mode.
constexpr int kMargCooMaxRep = 16;
int marg_coo_replicas(int64_t nnz, int64_t I, int64_t J);
cudaError_t launch_marginals_coo(const int32_t* i, const int32_t* j, const int32_t* k,
                                 const float* v, int64_t nnz, int moi, int S, int64_t* x1,
                                 int64_t* x2, int64_t* x3, cudaStream_t st, int64_t I = 0, int64_t J = 0,
                                 int64_t* rep_ws = nullptr, int nrep = 0);
// max phi over a dense view (slices [k0,k0+nk)) or COO values; result as double bits in
// *out (callers zero it; phi >= 0 so the bit pattern is monotone).
// a0 fused copy + max |x| of a contiguous device batch (n floats, n % 4 == 0, 16 B aligned)
cudaError_t launch_ingest_dense(const float* src, float* dst, int64_t n, int moi, unsigned long long* out,
                                cudaStream_t st);
cudaError_t launch_max_phi_dense(const DenseView& X, int64_t k0, int64_t nk, int moi,
                                 unsigned long long* out, cudaStream_t st);
cudaError_t launch_max_phi_vals(const float* v, int64_t n, int moi, unsigned long long* out,
                                cudaStream_t st);

// a2: one block per (rep, mode) segment.
struct SampleSeg {
  const int64_t* w;   // weights (device)
  int64_t n;          // population size
  int64_t ns;         // sample size
  int32_t* out;       // sorted sample (device, ns entries)
  int32_t* loc;       // optional local-index map [n]: position in out or -1 (may be null)
  uint64_t* keys;     // workspace [n]
  uint32_t rep, mode;
  int32_t* kp_tail;   // optional: write kp_tail[t] = tail0 + t after out (t < ntail)
  int64_t tail0, ntail;
};
cudaError_t launch_sample(const SampleSeg* segs_dev, int nseg, uint64_t seed, uint32_t update_id,
                          cudaStream_t st);

// a3 dense: Y[rep][u][q][p] = X(Is[rep][p], Js[rep][q], Kp[rep][u]) ; Y pitch = nI.
// ysq_part (optional) [rep][gridDim.x] gets per-block sums of squares (fp64).
// Y rows have pitch pI (>= nI); Yt (optional, may be null) is the per-slice transpose
// Yt[rep][u][p][q] with row pitch pJ (>= nJ) and the same y_stride.
cudaError_t launch_gather_dense(const DenseView& X, const int32_t* Is, const int32_t* Js,
                                const int32_t* Kp, int nI, int nJ, int nK, int r,
                                int64_t idx_stride_I, int64_t idx_stride_J, int64_t idx_stride_K,
                                float* Y, int64_t y_stride, cudaStream_t st, float* Yt = nullptr,
                                int pI = 0, int pJ = 0, int32_t* order_ws = nullptr, int64_t nslices = 0);
// (order_ws: r * nK int32 scratch for the slice-ordered walk; nslices: slices of the store K'
// indexes, <= 8192 for the ordering, else the plain (rep, slice) order)

// ---- dense batched CP-ALS -------------------------------------------------------------
struct DenseAls {
  const float* Y;  int64_t y_stride;   // [r][nK][nJ][pitch]
  const float* Yt;                     // optional per-slice transpose [r][nK][nI][nJ] (cluster path)
  int64_t pitch;
  int nI, nJ, nK, R, r;
  float* U[3]; int64_t u_stride[3];    // [r][n_m][R]
  double* G;       // [r][3][R][R]
  double* lam;     // [r][R]
  double* ysq;     // [r]
  double* fit;     // [r]
  double* fit_prev;// [r]
  int* iters;      // [r]
  int* done;       // [r]
  int* flags;      // [r]: bit0 pinv used, bit1 non-finite
  double* part0;   int nb0;  int64_t rows_per_block0;   // [r][nb0][nI][R]
  float* D;                            // [r][nK][nJ][R]
  double* M;       int64_t m_stride;   // [r][max n][R]
  double* Uscr;                        // [r][max n][R]
  int maxit; double tol;
};
// ws sizes for a given problem (bytes); fills nb0/rows_per_block0 in *a.
size_t dense_als_workspace(DenseAls* a);
cudaError_t dense_als_bind_workspace(DenseAls* a, void* ws);
cudaError_t launch_als_init(const DenseAls& a, uint64_t seed, uint32_t update_id,
                            uint32_t rep0, bool init_factors, cudaStream_t st);
// factor init only (Philox U(0,1) -> fp32, R10) and per-rep state reset
cudaError_t launch_als_init_factors(const DenseAls& a, uint64_t seed, uint32_t update_id,
                                    uint32_t rep0, cudaStream_t st, uint32_t rep_stride = 1);
// cluster-per-repetition ALS (k_als_cluster.cu): all iterations in one launch
struct ClusterPlan {
  int CS = 0; size_t smem = 0; int act = 0; int RB = 0; int stage_fl = 0; int dsh = 0;
  int grid = 0;   // 1: CS plain CTAs per repetition in one cooperative grid (global-memory comm)
};
// row pitch (floats) of the summary layouts Y[u][q][p] / Yt[u][p][q] the cluster path reads
int cluster_pitch(int n);
bool plan_als_cluster(const DenseAls& a, ClusterPlan* pl);
size_t als_cluster_dscratch_bytes(const DenseAls& a, const ClusterPlan& pl);
void als_phase_dump();   // SBT_ALS_PHASES builds only (debug)
cudaError_t run_als_cluster(const DenseAls& a, const ClusterPlan& pl, float* Dglob, cudaStream_t st);
cudaError_t launch_sumsq_dense(const float* Y, int64_t y_stride, int64_t rows, int64_t pitch,
                               int64_t ncols, int r, double* out, cudaStream_t st);
cudaError_t run_dense_als(const DenseAls& a, cudaStream_t st);
// Collectives the sharded full-tensor ALS needs (capi_dist.inc binds them to NCCL; a world-1
// handle to plain copies): in-place sum all-reduce and an all-gather of n doubles per rank.
struct AlsComm {
  void* ctx;
  cudaError_t (*sum_d)(void* ctx, double* buf, size_t n, cudaStream_t st);
  cudaError_t (*gather_d)(void* ctx, const double* send, double* recv, size_t n, cudaStream_t st);
  int world;
};
// Full-tensor CP-ALS over a time-sharded store.  loc: this rank's slab
// (r = 1, nK = local slices, workspace of dense_als_workspace; U[0] = glob.U[0], U[1] =
// glob.U[1], U[2] = a local buffer of the slab's C rows), glob: the replicated factors (nK =
// global slices; dense_als_small_bind; factors initialised, Grams and ysq (all-reduced) set);
// kmap: local -> global slice (device, loc.nK); gidx: [world][kpad] global slice of every
// rank's padded row (or -1); stage: kpad * R doubles; gathered: world * kpad * R doubles.
cudaError_t run_dense_als_sharded(const DenseAls& loc, const DenseAls& glob, const int32_t* kmap,
                                  const int32_t* gidx, int kpad, double* stage, double* gathered,
                                  const AlsComm& c, cudaStream_t st);
size_t dense_als_small_workspace(const DenseAls& a);
void dense_als_small_bind(DenseAls* a, void* ws);
// single-mode MTTKRP for the stateless API (r = 1): M (fp32 [n_mode][R])
cudaError_t dense_mttkrp_single(const DenseAls& a, int mode, float* M, cudaStream_t st);

// GetRank (k_getrank.cu): CorConDia of nm models of dense tensors X + model * x_stride (fp64)
size_t corcondia_ws_doubles(int I, int J, int K, int F, int nm);
cudaError_t launch_corcondia(const float* X, int64_t x_stride, int64_t pitch, int I, int J, int K, int F,
                             int nm, const float* const U[3], const int64_t u_stride[3], const double* lam,
                             double* ws, double* cc, cudaStream_t st);
// the same for a canonical COO tensor (sorted by (k, j, i)): T1 / T2 from the nonzeros (sparse
// CorConDia); ws: corcondia_coo_ws_doubles
size_t corcondia_coo_ws_doubles(int I, int J, int K, int F, int nm);
cudaError_t launch_corcondia_coo(const int32_t* ci, const int32_t* cj, const int32_t* ck, const float* cv,
                                 int64_t nnz, int I, int J, int K, int F, int nm, const float* const U[3],
                                 const int64_t u_stride[3], const double* lam, double* ws, double* cc,
                                 cudaStream_t st);
// Warm start (R34): U0 = A(I_s), U1 = B(J_s), U2 = [fp32(C(K_s) lambda); 0] per repetition
// (Is [r][nI], Js [r][nJ], Kp [r][nK] with the first nKs entries the old slices K_s)
cudaError_t launch_warm_init(const DenseAls& a, const float* A, const float* B, const float* C, const float* lam,
                             const int32_t* Is, const int32_t* Js, const int32_t* Kp, int nKs, cudaStream_t st,
                             int rep0 = 0, int rep_stride = 1);
// GetRank inside the update (R33): copy the r = 1 rank-src.R decomposition `src` into
// repetition rho of the rank-dst.R candidate buffers of `dst` (columns >= src.R and their
// lambda zero; fit / iters / flags copied)
cudaError_t launch_rank_pad(const DenseAls& src, const DenseAls& dst, int rho, cudaStream_t st);

// a5 / a6
struct MatchArgs {
  const float *A, *B, *C;            // model snapshot (fp32)
  int R, r;
  const int32_t* Is; const int32_t* Js; const int32_t* Ks;   // [r][nI] ...
  int nI, nJ, nKs, nK;
  int64_t ks_stride;                  // stride between reps' K_s lists (K' rows: nK)
  int64_t is_stride, js_stride;       // strides between reps' I_s / J_s lists (0 = nI / nJ)
  const float* U[3]; int64_t u_stride[3];
  const double* lamp;                 // [r][R]
  double tau;
  int* pi;           // [r][R]
  double* scale;     // [r][3][R]
  double* lam_hat;   // [r][R]
  double* score_min; // [r]
  int* accepted;     // [r]
  const int* rnew;   // [r] or null: rank of rep's candidate (GetRank, R33); only old components
                     // matched to a real column (pi f < rnew) count for acceptance and merge
  double* part;      // [r][3][match_chunks][R*R + 2R] partial anchor sums (workspace)
};
int match_chunks(const MatchArgs& m);
size_t match_part_doubles(const MatchArgs& m);
cudaError_t launch_match(const MatchArgs& m, cudaStream_t st);

struct MergeArgs {
  const float *A, *B, *C, *lam;      // old model
  float *An, *Bn, *Cn, *lamn;        // new model (pre-filled copy of the old one)
  int64_t I, J, Ko, Kn; int R, r;
  const int32_t* loc[3];             // [r][n_m] local index maps (-1 = not sampled)
  int nKs;
  const float* U[3]; int64_t u_stride[3];
  const int* pi; const double* scale; const double* lam_hat; const int* accepted;
  const int* rnew;                   // [r] or null (see MatchArgs::rnew)
  int policy;
};
cudaError_t launch_merge(const MergeArgs& m, cudaStream_t st);

// a7: relative error of [[lam; A, B, C]] over a dense view (slices [0,K)); writes relerr.
cudaError_t launch_fit_dense(const DenseView& X, const float* lam, const float* A,
                             const float* B, const float* C, int R, double* ws /* >= 4 + nb */,
                             double* relerr, cudaStream_t st);
size_t fit_dense_ws_doubles(const DenseView& X);

// ---- COO (k_coo.cu) -----------------------------------------------------------------
struct CooView {                       // canonical COO tensor, device arrays
  const int32_t *i, *j, *k;
  const float* v;
  int64_t nnz, I, J, K;
};
struct CooModePlan {                   // per-mode MTTKRP layout (k_coo.cu)
  int64_t nrow, n;                     // r * rows, entries
  const int64_t* ptr;                  // [nrow + 1] row pointers into the mode's order
  int64_t* pstart;                     // [nrow + 1] first piece of each row (scan)
  int64_t* pb;                         // [pieces] first entry of each piece
  int32_t* prow;                       // [pieces] row (rep * rows + row) of each piece
  const int32_t *sa, *sb;              // other two indices in the mode's order
  const float* sv;                     // values in the mode's order
  double* partial;                     // [pieces][R] partial sums of multi-piece rows
  int32_t* plist;                      // optional [pieces]: warp pieces at [0, nlist[0]), short
  unsigned* nlist;                     //   pieces at plist[P - 1 - j], j < nlist[1] (any order)
};
struct CooAls {                        // the r COO summaries (concatenated) + ALS buffers
  int nI, nJ, nK, R, RB, r;
  CooModePlan plan[3];
  float* U[3]; int64_t u_stride[3];
  const float* Up[3]; int64_t up_stride[3];   // optional copies of U with rows padded to RB floats
  double* M[3]; int64_t m_stride[3];
  const int* done;
};
size_t coo_plan_elems(int64_t nrow, int64_t n);
cudaError_t coo_build_plan(CooModePlan& pl, const int32_t* perm, const int32_t* ia, const int32_t* ib,
                           const float* v, int64_t n, int64_t* cnt, int64_t* sws, cudaStream_t st);
cudaError_t launch_coo_validate(const int32_t* i, const int32_t* j, const int32_t* k, const float* v,
                                int64_t n, int64_t I, int64_t J, int64_t K, unsigned* flags,
                                cudaStream_t st);
cudaError_t launch_coo_append(const int32_t* bi, const int32_t* bj, const int32_t* bk, const float* bv,
                              int64_t n, int32_t k_shift, int32_t* si, int32_t* sj, int32_t* sk,
                              float* sv, cudaStream_t st);
cudaError_t launch_build_mask(const int32_t* loc, int64_t n, int r, uint32_t* mask, int64_t total,
                              cudaStream_t st);
int64_t coo_gather_blocks(int64_t nnz);
cudaError_t launch_coo_gather_count(const CooView& X, const uint32_t* mI, const uint32_t* mJ,
                                    const uint32_t* mK, int r, int64_t* counts, cudaStream_t st);
cudaError_t launch_coo_gather_write(const CooView& X, const uint32_t* mI, const uint32_t* mJ,
                                    const uint32_t* mK, const int32_t* locI, const int32_t* locJ,
                                    const int32_t* locK, int64_t Ko, int nKs, int r,
                                    const int64_t* offsets, int32_t* op, int32_t* oq, int32_t* ou,
                                    float* ov, cudaStream_t st);
size_t scan_ws_elems(int64_t n);
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* ws, cudaStream_t st);
size_t radix_ws_elems(int64_t n);
cudaError_t launch_coo_permute4(const int32_t* perm, const int32_t* a, const int32_t* b, const int32_t* c,
                                const float* v, int64_t n, int32_t* oa, int32_t* ob, int32_t* oc, float* ov,
                                cudaStream_t st);
cudaError_t coo_sort_by_index(const int32_t* idx, const int64_t* off, int r, int kb, int64_t n,
                              uint32_t* keys, int32_t* perm, uint32_t* ws_keys, int32_t* ws_vals,
                              int64_t* hist, int64_t* offs, int64_t* sws, cudaStream_t st);
cudaError_t coo_make_keys(const int32_t* idx, const int64_t* off, int r, int kb, int64_t n,
                          uint32_t* keys, cudaStream_t st);
cudaError_t coo_row_pointers(const uint32_t* sorted_keys, int64_t n, int kb, int r, int64_t rows,
                             int64_t* cnt, int64_t* ptr, int64_t* sws, cudaStream_t st);
cudaError_t launch_coo_mttkrp(const CooAls& a, int mode, cudaStream_t st);
cudaError_t launch_coo_sumsq(const float* v, const int64_t* off, int r, double* ysq, cudaStream_t st);
size_t coo_fit_ws_doubles(int64_t I, int64_t J, int64_t K);
cudaError_t launch_coo_fit_partial(const CooView& X, const float* lam, const float* A, const float* B,
                                   const float* C, int R, const int32_t* kmap, double* ws, double* out2,
                                   cudaStream_t st);
cudaError_t launch_coo_fit(const CooView& X, const float* lam, const float* A, const float* B,
                           const float* C, int R, double* ws, double* relerr, cudaStream_t st);
cudaError_t launch_coo_max_phi(const float* v, int64_t n, int moi, unsigned long long* out, cudaStream_t st);
// row-parallel ALS solve steps (k_als_rows.cu), R <= 16
struct RowsAls {
  int nI, nJ, nK, R, r, maxit;
  double tol;
  float* U[3]; int64_t u_stride[3];
  float* Up[3]; int64_t up_stride[3]; int RBp;   // optional padded copies (16 B rows), kept in sync
  const double* M[3]; int64_t m_stride[3];
  double* X; int64_t x_stride;         // [r][maxn][R] solved rows
  double* Vi;                          // [r][R][R]
  double* part;                        // [r][tiles][R*R + 1]
  double* G;                           // [r][3][R][R]
  double* lam;                         // [r][R]
  double* ysq; double* fit; double* fit_prev;
  int* iters; int* done; int* flags; int* stop;
};
cudaError_t launch_als_rows_mode(const RowsAls& a, int mode, cudaStream_t st);
// Up[m] = U[m] with rows padded to RBp floats (zeros), every mode and repetition
cudaError_t launch_pad_factors(const RowsAls& a, cudaStream_t st);
struct GramArgs {                      // G[rep][m] = U_m^T U_m for m < 3, rep < r (fp64)
  const float* U[3]; int64_t u_stride[3]; int n[3];
  int R, r, tmax;                      // tmax = gram_tiles_for(max n)
  double* part;                        // gram_part_doubles(max n, R, r)
  double* G; int64_t g_stride;         // per-rep stride of G (>= 3 R^2)
};
size_t gram_part_doubles(int maxn, int R, int r);
int gram_tiles_for(int n);
cudaError_t launch_gram_tiles(const GramArgs& g, cudaStream_t st);
cudaError_t launch_als_rows_commit(const RowsAls& a, cudaStream_t st);
size_t als_rows_part_doubles(int maxn, int R, int r);
// the whole batched COO ALS (every iteration and mode) in one cooperative launch (k_coo_als.cu);
// R <= 16 with padded factors; bar: one zeroed-by-the-launch counter
bool coo_als_persist_supported(int R);
size_t coo_als_persist_ctr_words(int maxit);   // size of `bar` (barrier + work counters)
cudaError_t launch_coo_als_persist(const CooAls& ca, const RowsAls& ra, unsigned* bar, cudaStream_t st);
// ALS pieces shared with the COO path (k_als.cu)
cudaError_t launch_als_solve(const DenseAls& a, int mode, cudaStream_t st);
cudaError_t launch_als_gram(const DenseAls& a, cudaStream_t st);
// Grams of three factors, fp64 [3][R][R] (k_stream.cu), ws: gram3_ws_doubles
size_t gram3_ws_doubles(int64_t I, int64_t J, int64_t K, int R);
cudaError_t launch_gram3(const float* A, const float* B, const float* C, int64_t I, int64_t J,
                         int64_t K, int R, double* G, double* ws, cudaStream_t st);

// ---- distributed data movement (k_dist.cu) ----------------------------------------------
struct SliceJob { int rep; int32_t k_local; float* dY; float* dYt; };
struct CopyJob { const float* src; float* dY; float* dYt; };
struct CopyBytes { const void* src; void* dst; int64_t bytes; };
cudaError_t launch_multi_copy(const CopyBytes* jobs, int njobs, int64_t max_bytes, cudaStream_t st);
cudaError_t launch_slice_gather(const DenseView& X, const SliceJob* jobs, int njobs, const int32_t* Is_all,
                                const int32_t* Js_all, int nI, int nJ, int pI, int pJ, cudaStream_t st);
cudaError_t launch_slice_copy(const CopyJob* jobs, int njobs, int64_t nY, int64_t nYt, cudaStream_t st);
cudaError_t launch_add_i64(int64_t* dst, const int64_t* src, int64_t n, cudaStream_t st);
cudaError_t launch_local_kmaps(const int32_t* kmap, int64_t Kl, const uint32_t* mK, const int32_t* locK, int64_t Ko,
                               int nKs, int r, uint32_t* mKl, int32_t* locKl, cudaStream_t st);
cudaError_t launch_x3_scatter(const int64_t* x3l, const int32_t* kmap, int64_t n, int64_t* x3g,
                              cudaStream_t st);
// fit partials of a slab: inner/sq summed into out2[0..1] (kmap: local slice -> global row of C)
cudaError_t launch_fit_stream_partial(const DenseView& X, const float* lam, const float* A, const float* B,
                                      const float* C, int R, const int32_t* kmap, double* ws,
                                      double* out2, cudaStream_t st);
// relerr from the (globally summed) inner/sq and the model's Grams
cudaError_t launch_fit_finish(const double* in2, const float* lam, const float* A, const float* B,
                              const float* C, int64_t I, int64_t J, int64_t K, int R, double* ws,
                              double* relerr, cudaStream_t st);

// k_stream.cu: TMA-ring streaming passes over the dense store (pitch % 4 == 0, 16 B aligned)
bool stream_supported(const DenseView& X);
bool fit_stream_supported(const DenseView& X, int R);
// qb: every q = RNE(phi 2^S) of the pass is <= 2^qb (64: unknown); qb <= 27 -> 32-bit arithmetic
// phimax / d_phimax (device fp64 bits, may be NULL): upper bounds on phi of the pass's data (the
// larger counts); a bound q < 2^22 selects the FMA rounding of the 32-bit kernel (MOI 0)
cudaError_t launch_marginals_stream(const DenseView& X, int64_t k0, int64_t nk, int moi, int S,
                                    int64_t* x1, int64_t* x2, int64_t* x3, cudaStream_t st, int qb = 64,
                                    double phimax = 1e300, const unsigned long long* d_phimax = nullptr);
size_t fit_stream_ws_doubles(const DenseView& X);
// a1 over slices [0, nk) fused with the fit partials of the model (lam; A, B, C) over the same
// slices (SURVEY 8(f) NEXT #1 lag-1 fit): x1/x2/x3 accumulate (zero them first); out2 =
// {<X, M>, ||X||^2} of those slices (finish with launch_fit_finish); kmap: local slice -> model
// row (sharded stores) or NULL; ws: fit_stream_ws_doubles; needs fit_stream_supported(X, R)
// ---- incremental exact fit (k_fitinc.cu) ---------------------------------
// per-component sums P[f] += sum over a row set of the store of sum_i X(i,j,k) As(i,f) w(j,k,f),
// w = (U - Usub)(j,f) (V - Vsub)(kmap(k), f); column R of the outputs: sum of X^2 over the rows
struct FitRows {
  const float* X; int64_t pitch; int I, J, R;
  int kind;                  // 0: slices [k0, k1), every j; 1: j in list, k in [k0, k1); 2: k in list, every j
  int64_t k0, k1;
  const int32_t* list; const int* nlist;   // kinds 1, 2 (device count)
  const float* As;                         // I x R
  const float *U, *Usub, *V, *Vsub;        // J x R and (model rows) x R; Usub / Vsub may be NULL
  const int32_t* kmap;                     // store slice -> model row (sharded) or NULL
  const int* gate; int gate_val;           // run only if *gate == gate_val (NULL: always)
};
struct FitPlanArgs {
  const float *A0, *A1, *B0, *B1, *C0, *C1;   // old / new model
  int64_t I, J, Kold; int R;
  const double* st_old;                        // [P[R], ||X||^2, valid]
  double budget_rows; int allow_c;             // allow_c = 0: a changed old C row forces the full pass
  int32_t *jlist, *klist; int* counts;          // counts[0] = changed B rows, [1] = changed old C rows
  int* mode;                                    // 1 incremental, 2 full pass
};
struct FitFinishArgs {
  const double* terms[4]; int nparts[4];       // 0 new slices, 1 dB, 2 dC (incremental), 3 full pass
  const double* reduced;                       // sharded: all-reduced [R + 1] sums, else NULL
  const int* mode; int R, RB;
  const double* st_old; double* st_new;
  const float* lam; const double* G;           // new lambda, Grams [3][R][R]
  double* relerr;
};
// COO stores (k_fitinc.cu): per-component sums P[f] = sum_e v_e A(i_e,f) B(j_e,f) C(k_e,f) and
// sum_e v_e^2 over the store entries [n0, n1), in fitrows' partial layout (the term of new slices,
// entries appended after n0, or the full pass); gate as in FitRows
struct CooFitRows {
  const int32_t *i, *j, *k; const float* v; int64_t n0, n1;
  const float *A, *B, *C; int R;
  const int* gate; int gate_val;
  // difference term (old entries): sum over entries with a changed row of v (A'B'C' - ABC)_f;
  // A0 / B0 / C0 the previous model, changed-row bitmaps, *any == 0: nothing to do
  const float *A0, *B0, *C0; const uint32_t *bA, *bB, *bC; const int* any;
};
// changed-row bitmaps of A, B and the old rows of C (zeroed by the caller, with *any) and the
// plan mode (1: incremental when the old state is valid, else 2: the full pass)
struct CooFitFlags {
  const float *A0, *A1, *B0, *B1, *C0, *C1; int64_t I, J, Kold; int R;
  uint32_t *bA, *bB, *bC; int* any; const double* st_old; int* mode;
};
cudaError_t launch_coo_fit_flags(const CooFitFlags& f, cudaStream_t st);
cudaError_t launch_coo_fitrows(const CooFitRows& a, double* part, cudaStream_t st);   // part: fitrows_blocks() x (RB + 1)
int fitrows_rb_of(int R);
bool fitrows_supported(int64_t pitch, int R);   // pitch % 4 == 0 and the transposed As fits in shared memory
int fitrows_blocks();
cudaError_t launch_fitrows(FitRows a, double* part, cudaStream_t st);   // part: fitrows_blocks() x (RB + 1)
cudaError_t launch_fitinc_plan(const FitPlanArgs& p, cudaStream_t st);
cudaError_t launch_fitinc_finish(const FitFinishArgs& a, cudaStream_t st);
cudaError_t launch_fitinc_sum(const FitFinishArgs& a, double* out, cudaStream_t st);

bool margfit_supported(const DenseView& X, int R);
// qb: every quantised value q = RNE(phi 2^S) of the pass is <= 2^qb (32-bit arithmetic when small)
cudaError_t launch_marg_fit_stream(const DenseView& X, int64_t nk, int moi, int S, int qb, const float* lam,
                                   const float* A, const float* B, const float* C, int R, const int32_t* kmap,
                                   int64_t* x1, int64_t* x2, int64_t* x3, double* ws, double* out2,
                                   cudaStream_t st);
cudaError_t launch_fit_stream(const DenseView& X, const float* lam, const float* A, const float* B,
                              const float* C, int R, double* ws, double* relerr, cudaStream_t st);

cudaError_t launch_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t key,
                          int64_t n, uint32_t* out, cudaStream_t st);
cudaError_t launch_detlog(const double* u, int64_t n, double* out, cudaStream_t st);

}  // namespace sbt
