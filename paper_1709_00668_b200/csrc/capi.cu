// capi.cu -- the C-ABI (include/sambaten.h) and the per-handle engine that sequences the
// hot path a0..a7 on one CUDA stream.  Host code here only validates, sizes buffers and
// launches; every step of the method runs in the kernels of k_*.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <tuple>
#include <string>
#include <functional>
#include <vector>

#include "../../include/sambaten.h"
#include "common.cuh"
#include "internal.h"

namespace sbt {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace sbt

using namespace sbt;

#define FAIL(code, msg)        \
  do {                         \
    sbt::set_error(msg);       \
    return (code);             \
  } while (0)

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      sbt::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));     \
      return e_ == cudaErrorMemoryAllocation ? SAMBATEN_E_OOM : SAMBATEN_E_CUDA; \
    }                                                                         \
  } while (0)

// a1 / a7 dispatch: the TMA-ring streaming kernels when the view allows them (pitch % 4 == 0,
// 16 B aligned; R <= 16 for the fit), else the tiled kernels.
static cudaError_t marginals_any(const DenseView& V, int64_t k0, int64_t nk, int moi, int S,
                                 int64_t* x1, int64_t* x2, int64_t* x3, cudaStream_t st, int qb = 64,
                                 double phimax = 1e300, const unsigned long long* d_phimax = nullptr) {
  if (stream_supported(V)) return launch_marginals_stream(V, k0, nk, moi, S, x1, x2, x3, st, qb, phimax, d_phimax);
  return launch_marginals_dense(V, k0, nk, moi, S, x1, x2, x3, st);
}
static size_t fit_ws_doubles_any(const DenseView& V) {
  return std::max(fit_dense_ws_doubles(V), fit_stream_ws_doubles(V));
}
static cudaError_t fit_any(const DenseView& V, const float* lam, const float* A, const float* B,
                           const float* C, int R, double* ws, double* relerr, cudaStream_t st) {
  if (fit_stream_supported(V, R)) return launch_fit_stream(V, lam, A, B, C, R, ws, relerr, st);
  return launch_fit_dense(V, lam, A, B, C, R, ws, relerr, st);
}

static int ceil_log2_d(double v) {
  int e;
  const double m = frexp(v, &e);
  return m == 0.5 ? e - 1 : e;
}

// ---------------------------------------------------------------------------------------
// device buffer helper
// ---------------------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t b) {
    if (b <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    // growth by small steps (K grows with every batch) reallocates once per ~12%, not per call
    size_t want = grown ? ((b + b / 8 + 255) & ~(size_t)255) : b;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess && want > b) {
      cudaGetLastError();
      want = b;
      e = cudaMalloc(&p, want);
    }
    if (e == cudaSuccess) bytes = want;
    grown = true;
    return e;
  }
  bool grown = false;
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct HostStatus {        // pinned; filled by one D2H copy at the end of an update
  unsigned long long maxphi_bits;
  unsigned vflags;
  int accepted[kMaxReps];
  int iters[kMaxReps];
  int flags[kMaxReps];
  double fit[kMaxReps];
  double relerr, relerr_prev;
  int fit_mode;
};

struct DistState;   // capi_dist.inc

struct sambaten_s {
  int fmt = SAMBATEN_DENSE;
  DistState* dist = nullptr;   // set for handles of the sharded update (sambaten_init_factors_dist)
  int64_t I = 0, J = 0, K = 0, Kcap = 0, pitch = 0;
  bool X_borrowed = false;   // opts.borrow_store: X is the caller's buffer
  int als_plan[4] = {-1, 0, 0, 0};   // the a4 plan of the last update (sambaten_info.als_plan)
  int64_t summ_entries = 0;          // summary entries / nnz of the update in flight (sambaten_info)
  bool lag_now = false;              // this update computes the previous model's fit in a1 (full_fit = 2)
  bool pipe_now = false;             // this update's a1 runs on the side stream (opts.pipelined, R36)
  int fit_path = 0;                  // sambaten_info.fit_path of the update in flight
  const int* d_fit_mode = nullptr;   // device plan of the incremental fit (1 incremental, 2 full)
  cudaStream_t st2 = nullptr;     // side stream: host batch copy overlapped with a1 (old slices)
  cudaEvent_t ev_side[2] = {nullptr, nullptr};
  cudaEvent_t ev_pl[2] = {nullptr, nullptr};   // pipelined a1 on the side stream (timing)
  DevBuf xm, xm_ck;          // committed marginals of the current tensor (incremental a1)
  bool xm_valid = false, xm_ck_valid = false;
  int R = 0, r = 0, s[3] = {1, 1, 1};
  uint64_t seed = 0;
  uint32_t update_id = 0;
  sambaten_opts opts;
  cudaStream_t st = nullptr;
  int S = 0, maxphi_log2 = 0;
  double phimax_run = 1e300;   // upper bound on phi over the store (X0 and committed batches; restore keeps it)
  // store and model
  DevBuf X;
  DevBuf model[2];          // A | B | C | lam | fit state, double-buffered (merge writes the shadow)
  DevBuf fiws;              // incremental-fit workspace (k_fitinc.cu)
  DevBuf mrep;              // replicated COO marginals (k_marginals.cu)
  DevBuf gord;              // the gather's (rep, slice) pairs in source-slice order
  int cur = 0;
  DevBuf ck;                // checkpoint of the model
  int64_t K_ck = -1;
  uint32_t uid_ck = 0;
  // workspaces
  DevBuf marg, samp, summ, fac, als, match, misc, segs, fitws;
  // COO store (fmt == SAMBATEN_COO): i | j | k (int32) and v (fp32), capacity nnz_cap
  int64_t nnz = 0, nnz_cap = 0, nnz_ck = 0;
  DevBuf coo_ws;            // gather / sort / ALS workspace of the COO path
  DevBuf grws, grk;         // GetRank in the update (R33): trial workspace, per-rep ranks [r]
  DevBuf grc[4];            // COO GetRank in the update: ALS workspace, factors, CorConDia, offsets
  int rep_rank[kMaxReps] = {};   // rank each rep of the last update decomposed at
  int32_t* ci() const { return X.as<int32_t>(); }
  int32_t* cj() const { return ci() + nnz_cap; }
  int32_t* ck_() const { return cj() + nnz_cap; }
  float* cv() const { return reinterpret_cast<float*>(ck_() + nnz_cap); }
  CooView coo_view(int64_t n) const { return CooView{ci(), cj(), ck_(), cv(), n, I, J, K}; }
  SampleSeg* segs_host = nullptr;   // pinned
  HostStatus* hs = nullptr;         // pinned
  cudaEvent_t ev[9] = {};
  // last sample sizes
  int64_t last_n[3] = {0, 0, 0};
  int64_t last_nKp = 0;
  // cluster-ALS plans by summary shape (host-side planning kept out of the timed path)
  struct PlanEntry { int nI, nJ, nK, R, r; bool ok; ClusterPlan pl; };
  std::vector<PlanEntry> plans;

  float* A(int b) const { return model[b].as<float>(); }
  float* B(int b) const { return A(b) + I * R; }
  float* C(int b) const { return B(b) + J * R; }
  float* lam(int b) const { return C(b) + Kcap * R; }
  // the incremental fit's state rides in the model buffer (so merge copies, checkpoint and
  // restore carry it): [P[0..R), ||X||^2, valid] fp64 after lambda (k_fitinc.cu)
  size_t fit_off() const { return ((size_t)(I + J + Kcap + 1) * R + 1) & ~(size_t)1; }
  double* fitst(int b) const { return reinterpret_cast<double*>(model[b].as<float>() + fit_off()); }
  size_t model_floats() const { return fit_off() + 2 * (size_t)(R + 2); }
  DenseView view() const { return DenseView{X.as<float>(), I, J, K, pitch}; }
  DenseView view_local() const;   // the local slab of a sharded handle (capi_dist.inc)
};

static bool cluster_plan(sambaten_s* h, const DenseAls& a, ClusterPlan* pl) {
  if (a.r < 2 || getenv("SAMBATEN_NO_CLUSTER_ALS")) return false;
  for (auto& e : h->plans)
    if (e.nI == a.nI && e.nJ == a.nJ && e.nK == a.nK && e.R == a.R && e.r == a.r) {
      *pl = e.pl;
      return e.ok;
    }
  sambaten_s::PlanEntry e{a.nI, a.nJ, a.nK, a.R, a.r, false, ClusterPlan{}};
  e.ok = plan_als_cluster(a, &e.pl);
  if (getenv("SAMBATEN_DEBUG"))
    fprintf(stderr, "[sambaten] cluster ALS plan nI=%d nJ=%d nK=%d R=%d r=%d -> ok=%d CS=%d smem=%zu act=%d RB=%d stage_fl=%d dsh=%d\n",
            a.nI, a.nJ, a.nK, a.R, a.r, (int)e.ok, e.pl.CS, e.pl.smem, e.pl.act, e.pl.RB,
            e.pl.stage_fl, e.pl.dsh);
  h->plans.push_back(e);
  *pl = e.pl;
  return e.ok;
}

// bound on the quantised values of the stored tensor: phi <= 2^(maxphi_log2 + 8) (R7: a batch
// beyond it is rejected), so q = RNE(phi 2^S) <= 2^(maxphi_log2 + 8 + S) (x^2 measure: the
// log of the squared bound)
static int qbits(const sambaten_s* h) { return h->maxphi_log2 + 8 + h->S; }

// a1 over the COO store entries [n0, n1), added to x1 / x2 / x3 (replicated kernel when large)
static cudaError_t coo_marginals(sambaten_s* h, int64_t n0, int64_t n1, int64_t* x1, int64_t* x2, int64_t* x3,
                                 cudaStream_t st) {
  const int nrep = marg_coo_replicas(n1 - n0, h->I, h->J);
  if (nrep >= 2) {
    cudaError_t e = h->mrep.ensure(sizeof(int64_t) * (size_t)nrep * (h->I + h->J));
    if (e != cudaSuccess) return e;
  }
  return launch_marginals_coo(h->ci() + n0, h->cj() + n0, h->ck_() + n0, h->cv() + n0, n1 - n0, h->opts.moi,
                              h->S, x1, x2, x3, st, h->I, h->J, nrep >= 2 ? h->mrep.as<int64_t>() : nullptr, nrep);
}

// ---- incremental exact fit (k_fitinc.cu) --------------------------------------------------------
static size_t align256(size_t b);
// Workspace: 4 term partials, the changed-row lists, counts, mode, Grams and their tiles.
struct FitIncWs {
  double* parts[4]; int32_t *jlist, *klist; int *counts, *mode; double *G, *gws, *red;
  uint32_t* bits; int64_t wA, wB, wC;   // COO: changed-row bitmaps of A, B, C (words) + the any flag
};
static cudaError_t fitinc_ws(sambaten_s* h, FitIncWs* w) {
  const int R = h->R, RB = fitrows_rb_of(R), nb = fitrows_blocks();
  const size_t pb = align256(sizeof(double) * (size_t)nb * (RB + 1));
  const size_t lb = align256(sizeof(int32_t) * (size_t)std::max<int64_t>(std::max(h->J, h->Kcap), 1));
  const size_t gw = align256(sizeof(double) * gram3_ws_doubles(h->I, h->J, h->Kcap, R));
  w->wA = (h->I + 31) / 32; w->wB = (h->J + 31) / 32; w->wC = (h->Kcap + 31) / 32;
  const size_t bb = align256(sizeof(uint32_t) * (size_t)(w->wA + w->wB + w->wC + 1));
  const size_t need = 4 * pb + 2 * lb + 256 + align256(sizeof(double) * 3 * R * R) + gw + 256 + bb;
  cudaError_t e = h->fiws.ensure(need);
  if (e != cudaSuccess) return e;
  char* p = h->fiws.as<char>();
  for (int t = 0; t < 4; ++t) { w->parts[t] = reinterpret_cast<double*>(p); p += pb; }
  w->jlist = reinterpret_cast<int32_t*>(p); p += lb;
  w->klist = reinterpret_cast<int32_t*>(p); p += lb;
  w->counts = reinterpret_cast<int*>(p); w->mode = w->counts + 2; w->red = reinterpret_cast<double*>(p + 64); p += 256;
  w->G = reinterpret_cast<double*>(p); p += align256(sizeof(double) * 3 * R * R);
  w->gws = reinterpret_cast<double*>(p); p += gw;
  w->bits = reinterpret_cast<uint32_t*>(p);
  return cudaSuccess;
}

// Fit of model nb over the slices [0, K) of view V: incremental from model b's state over the
// first Ko slices when the plan allows, else one full pass (decided on the device).
// full_only: skip the plan (initial state).  kmap: store slice -> model row (sharded) or NULL;
// allow_c: the dC term may run (its slice list holds store slices = model rows; single GPU).
// reduce: sharded all-reduce of the [R + 1] sums (NULL on one GPU).
static cudaError_t fitinc_run(sambaten_s* h, const DenseView& V, int64_t Ko_store, int64_t Ko_model, int64_t K_model,
                              int b, int nb, bool full_only, const int32_t* kmap, bool allow_c,
                              double* relerr, cudaStream_t st,
                              const std::function<cudaError_t(double*, size_t)>& reduce = nullptr) {
  const int R = h->R;
  FitIncWs w;
  cudaError_t e = fitinc_ws(h, &w);
  if (e != cudaSuccess) return e;
  if (full_only) {
    const int two = 2;
    e = cudaMemcpyAsync(w.mode, &two, sizeof(int), cudaMemcpyHostToDevice, st);
  } else {
    FitPlanArgs p{};
    p.A0 = h->A(b); p.A1 = h->A(nb); p.B0 = h->B(b); p.B1 = h->B(nb); p.C0 = h->C(b); p.C1 = h->C(nb);
    p.I = h->I; p.J = h->J; p.Kold = Ko_model; p.R = R;
    p.st_old = h->fitst(b);
    // incremental while its rows stay under half of a full pass; the dC term only where allowed
    p.budget_rows = 0.5 * (double)h->J * (double)Ko_model;
    p.allow_c = allow_c ? 1 : 0;
    p.jlist = w.jlist; p.klist = w.klist; p.counts = w.counts; p.mode = w.mode;
    e = launch_fitinc_plan(p, st);
  }
  if (e != cudaSuccess) return e;
  FitRows base{};
  base.X = V.base; base.pitch = V.pitch; base.I = (int)h->I; base.J = (int)h->J; base.R = R;
  base.kmap = kmap;
  // term 0: the new slices with the new model
  FitRows t0 = base;
  t0.kind = 0; t0.k0 = Ko_store; t0.k1 = V.K; t0.As = h->A(nb); t0.U = h->B(nb); t0.V = h->C(nb);
  t0.gate = w.mode; t0.gate_val = 1;
  // term 1: changed B rows over the old slices: A (B' - B) C'
  FitRows t1 = base;
  t1.kind = 1; t1.k0 = 0; t1.k1 = Ko_store; t1.list = w.jlist; t1.nlist = w.counts;
  t1.As = h->A(b); t1.U = h->B(nb); t1.Usub = h->B(b); t1.V = h->C(nb); t1.gate = w.mode; t1.gate_val = 1;
  // term 2: changed old C rows: A B (C' - C)   (store slice = model row: single GPU only)
  FitRows t2 = base;
  t2.kind = 2; t2.list = w.klist; t2.nlist = w.counts + 1;
  t2.As = h->A(b); t2.U = h->B(b); t2.V = h->C(nb); t2.Vsub = h->C(b); t2.gate = w.mode; t2.gate_val = 1;
  // term 3: the full pass with the new model
  FitRows t3 = base;
  t3.kind = 0; t3.k0 = 0; t3.k1 = V.K; t3.As = h->A(nb); t3.U = h->B(nb); t3.V = h->C(nb);
  t3.gate = w.mode; t3.gate_val = 2;
  if (!full_only) {
    if (Ko_store < V.K && (e = launch_fitrows(t0, w.parts[0], st)) != cudaSuccess) return e;
    if (Ko_store > 0 && (e = launch_fitrows(t1, w.parts[1], st)) != cudaSuccess) return e;
    if (allow_c && (e = launch_fitrows(t2, w.parts[2], st)) != cudaSuccess) return e;
  }
  if (V.K > 0 && (e = launch_fitrows(t3, w.parts[3], st)) != cudaSuccess) return e;
  e = launch_gram3(h->A(nb), h->B(nb), h->C(nb), h->I, h->J, K_model, R, w.G, w.gws, st);
  if (e != cudaSuccess) return e;
  FitFinishArgs f{};
  const int nbk = fitrows_blocks();
  f.terms[0] = (!full_only && Ko_store < V.K) ? w.parts[0] : nullptr;
  f.terms[1] = (!full_only && Ko_store > 0) ? w.parts[1] : nullptr;
  f.terms[2] = (!full_only && allow_c) ? w.parts[2] : nullptr;
  f.terms[3] = V.K > 0 ? w.parts[3] : nullptr;
  for (int t = 0; t < 4; ++t) f.nparts[t] = nbk;
  f.mode = w.mode; f.R = R; f.RB = fitrows_rb_of(R);
  f.st_old = h->fitst(b); f.st_new = h->fitst(nb); f.lam = h->lam(nb); f.G = w.G; f.relerr = relerr;
  if (reduce) {
    if ((e = launch_fitinc_sum(f, w.red, st)) != cudaSuccess) return e;
    if ((e = reduce(w.red, (size_t)R + 1)) != cudaSuccess) return e;
    f.reduced = w.red;
  }
  return launch_fitinc_finish(f, st);
}

// The same for a COO store.  Term 0: the entries appended after n_old (the batch's new slices)
// with the new model.  Term 1: the old entries with a changed A, B or old C row (bitmaps), each
// adding v (A'B'C' - ABC)_f -- the telescoped difference in one product, since the store has no
// per-row index; it reads the old entries' indices only when some row changed.  The full pass
// over [0, n_tot) only when the old state is not valid.
static cudaError_t fitinc_run_coo(sambaten_s* h, int64_t n_old, int64_t n_tot, int64_t Ko_model, int64_t K_model,
                                  int b, int nb, bool full_only, double* relerr, cudaStream_t st) {
  const int R = h->R;
  FitIncWs w;
  cudaError_t e = fitinc_ws(h, &w);
  if (e != cudaSuccess) return e;
  uint32_t *bA = w.bits, *bB = bA + w.wA, *bC = bB + w.wB;
  int* any = reinterpret_cast<int*>(bC + w.wC);
  if (full_only) {
    const int two = 2;
    e = cudaMemcpyAsync(w.mode, &two, sizeof(int), cudaMemcpyHostToDevice, st);
  } else {
    e = cudaMemsetAsync(w.bits, 0, sizeof(uint32_t) * (size_t)(w.wA + w.wB + w.wC + 1), st);
    CooFitFlags p{};
    p.A0 = h->A(b); p.A1 = h->A(nb); p.B0 = h->B(b); p.B1 = h->B(nb); p.C0 = h->C(b); p.C1 = h->C(nb);
    p.I = h->I; p.J = h->J; p.Kold = Ko_model; p.R = R;
    p.bA = bA; p.bB = bB; p.bC = bC; p.any = any; p.st_old = h->fitst(b); p.mode = w.mode;
    if (e == cudaSuccess) e = launch_coo_fit_flags(p, st);
  }
  if (e != cudaSuccess) return e;
  CooFitRows base{};
  base.i = h->ci(); base.j = h->cj(); base.k = h->ck_(); base.v = h->cv(); base.R = R;
  base.A = h->A(nb); base.B = h->B(nb); base.C = h->C(nb); base.gate = w.mode;
  CooFitRows t0 = base, t1 = base, t3 = base;
  t0.n0 = n_old; t0.n1 = n_tot; t0.gate_val = 1;
  t1.n0 = 0; t1.n1 = n_old; t1.gate_val = 1;
  t1.A0 = h->A(b); t1.B0 = h->B(b); t1.C0 = h->C(b); t1.bA = bA; t1.bB = bB; t1.bC = bC; t1.any = any;
  t3.n0 = 0; t3.n1 = n_tot; t3.gate_val = 2;
  const bool term0 = !full_only && n_old < n_tot, term1 = !full_only && n_old > 0;
  if (term0 && (e = launch_coo_fitrows(t0, w.parts[0], st)) != cudaSuccess) return e;
  if (term1 && (e = launch_coo_fitrows(t1, w.parts[1], st)) != cudaSuccess) return e;
  if ((e = launch_coo_fitrows(t3, w.parts[3], st)) != cudaSuccess) return e;
  e = launch_gram3(h->A(nb), h->B(nb), h->C(nb), h->I, h->J, K_model, R, w.G, w.gws, st);
  if (e != cudaSuccess) return e;
  FitFinishArgs f{};
  f.terms[0] = term0 ? w.parts[0] : nullptr;
  f.terms[1] = term1 ? w.parts[1] : nullptr;
  f.terms[3] = w.parts[3];
  for (int t = 0; t < 4; ++t) f.nparts[t] = fitrows_blocks();
  f.mode = w.mode; f.R = R; f.RB = fitrows_rb_of(R);
  f.st_old = h->fitst(b); f.st_new = h->fitst(nb); f.lam = h->lam(nb); f.G = w.G; f.relerr = relerr;
  return launch_fitinc_finish(f, st);
}

static void set_plan_report(sambaten_s* h, bool cluster, const ClusterPlan& pl, int R) {
  h->als_plan[0] = cluster ? (pl.grid ? 2 : 1) : 0;
  h->als_plan[1] = cluster ? pl.CS : 1;
  h->als_plan[2] = cluster ? pl.RB : R;
  h->als_plan[3] = cluster ? pl.dsh : 0;
}

extern "C" {

void sambaten_default_opts(sambaten_opts* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->als_max_iters = 30;
  o->als_tol = 1e-6;
  o->moi = SAMBATEN_MOI_ABS;
  o->merge_policy = 0;
  o->accept_tau = 0.9;
  o->full_fit = 0;
  o->capacity = 0;
  o->init_max_iters = 1000;
  o->init_tol = 1e-6;
  o->stream = nullptr;
  o->getrank = 0;
  o->getrank_trials = 1;
  o->getrank_threshold = 90.0;
}

const char* sambaten_last_error(void) { return sbt::g_err.c_str(); }
const char* sambaten_version(void) { return "sambaten-b200 0.1 (sm_100a)"; }

int sambaten_fixed_point_scale(int64_t cap_entries, double max_phi) {
  if (!(max_phi > 0.0)) return 0;
  int S = 62 - ceil_log2_d((double)std::max<int64_t>(cap_entries, 1)) - ceil_log2_d(max_phi) - 8;
  return std::min(std::max(S, -60), 120);
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// validation helpers
// ---------------------------------------------------------------------------------------
static sambaten_status check_dense(const sambaten_tensor* X, const char* what) {
  if (!X) FAIL(SAMBATEN_E_INVALID, std::string(what) + ": NULL tensor");
  if (X->fmt != SAMBATEN_DENSE && X->fmt != SAMBATEN_COO)
    FAIL(SAMBATEN_E_INVALID, std::string(what) + ": unknown format");
  for (int m = 0; m < 3; ++m)
    if (X->dims[m] < 0) FAIL(SAMBATEN_E_INVALID, std::string(what) + ": negative dimension");
  if (X->fmt == SAMBATEN_DENSE && X->dims[0] * X->dims[1] * X->dims[2] > 0 && !X->vals)
    FAIL(SAMBATEN_E_INVALID, std::string(what) + ": NULL values");
  return SAMBATEN_OK;
}

static cudaStream_t stream_of(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------------------
// handle creation
// ---------------------------------------------------------------------------------------
static sambaten_status create_common(sambaten_t* out, const sambaten_tensor* X0, int R, int s,
                                     int r, uint64_t seed, const sambaten_opts* opts) {
  if (!out) FAIL(SAMBATEN_E_INVALID, "init: NULL handle pointer");
  *out = nullptr;
  if (sambaten_status st = check_dense(X0, "init")) return st;
  if (X0->fmt == SAMBATEN_COO && X0->nnz > 0 && (!X0->idx[0] || !X0->idx[1] || !X0->idx[2] || !X0->vals))
    FAIL(SAMBATEN_E_INVALID, "init: NULL COO array");
  if (X0->fmt == SAMBATEN_COO && X0->nnz < 1) FAIL(SAMBATEN_E_DEGENERATE, "init: empty COO tensor");
  if (R < 1 || R > kMaxR) FAIL(SAMBATEN_E_INVALID, "init: R must be in [1, 32]");
  if (r < 1 || r > kMaxReps) FAIL(SAMBATEN_E_INVALID, "init: r must be in [1, 32]");
  if (s < 1) FAIL(SAMBATEN_E_INVALID, "init: s must be >= 1");
  if (X0->dims[0] < 1 || X0->dims[1] < 1 || X0->dims[2] < 1)
    FAIL(SAMBATEN_E_INVALID, "init: empty initial tensor");
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) FAIL(SAMBATEN_E_CUDA, "init: needs an sm_100 (B200) device");

  auto* h = new sambaten_s();
  if (opts) h->opts = *opts; else sambaten_default_opts(&h->opts);
  h->fmt = X0->fmt;
  h->I = X0->dims[0]; h->J = X0->dims[1]; h->K = X0->dims[2];
  h->R = R; h->r = r; h->seed = seed; h->update_id = 0;
  for (int m = 0; m < 3; ++m) h->s[m] = h->opts.s_mode[m] > 0 ? h->opts.s_mode[m] : s;
  if (h->fmt == SAMBATEN_DENSE) {
    h->Kcap = h->opts.capacity > 0 ? h->opts.capacity : 2 * h->K;
    if (h->Kcap < h->K) { delete h; FAIL(SAMBATEN_E_INVALID, "init: capacity < K0"); }
  } else {
    h->nnz = X0->nnz;
    h->nnz_cap = h->opts.capacity > 0 ? h->opts.capacity : 2 * X0->nnz;
    if (h->nnz_cap < h->nnz) { delete h; FAIL(SAMBATEN_E_INVALID, "init: capacity < nnz0"); }
    h->Kcap = h->opts.capacity_k > 0 ? h->opts.capacity_k : 2 * h->K + 1024;
    if (h->Kcap < h->K) { delete h; FAIL(SAMBATEN_E_INVALID, "init: capacity_k < K0"); }
  }
  if (h->opts.warm_start && h->opts.getrank) {
    delete h;
    FAIL(SAMBATEN_E_INVALID, "init: warm_start and getrank are exclusive (R34)");
  }
  if (h->opts.pipelined && h->fmt != SAMBATEN_DENSE) {
    delete h;
    FAIL(SAMBATEN_E_INVALID, "init: pipelined needs a dense tensor (R36)");
  }
  if (h->opts.getrank) {
    // dense or COO (the sparse summaries are rated by the COO CorConDia); single-GPU
    // (the sharded init refuses it)
    if (h->opts.getrank_trials < 1 || h->opts.getrank_trials > kMaxReps) {
      delete h; FAIL(SAMBATEN_E_INVALID, "init: getrank_trials must be in [1, 32]");
    }
  }
  h->st = stream_of(h->opts.stream);
  h->pitch = (h->I + 3) & ~int64_t(3);
  *out = h;
  return SAMBATEN_OK;
}

// Rows of `width` bytes between pitched buffers: one linear copy when both sides are
// contiguous (a 2D copy of many short rows runs far below the link rate from host memory),
// else a 2D copy.
static cudaError_t copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                             size_t rows, cudaStream_t st) {
  if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * rows, cudaMemcpyDefault, st);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDefault, st);
}

static sambaten_status alloc_store_and_model(sambaten_s* h, const sambaten_tensor* X0) {
  if (h->fmt == SAMBATEN_DENSE) {
    const size_t store = (size_t)h->Kcap * h->J * h->pitch * sizeof(float);
    if (h->opts.borrow_store) {
      // the caller's device buffer becomes the store (X0 in place, room for Kcap slices)
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, X0->vals) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        FAIL(SAMBATEN_E_INVALID, "init: borrow_store needs X0 in device memory");
      }
      if (h->pitch != h->I) FAIL(SAMBATEN_E_INVALID, "init: borrow_store needs I % 4 == 0");
      if (h->opts.capacity <= 0) FAIL(SAMBATEN_E_INVALID, "init: borrow_store needs opts.capacity (slices in the buffer)");
      h->X.p = const_cast<float*>(X0->vals);
      h->X.bytes = store;
      h->X_borrowed = true;
    } else {
      CK(h->X.ensure(store));
      CK(cudaMemsetAsync(h->X.p, 0, store, h->st));
      CK(copy_rows(h->X.p, h->pitch * sizeof(float), X0->vals, h->I * sizeof(float),
                        h->I * sizeof(float), h->J * h->K, h->st));
    }
  } else {
    CK(h->X.ensure((size_t)h->nnz_cap * (3 * sizeof(int32_t) + sizeof(float))));
    const size_t n = (size_t)h->nnz;
    CK(cudaMemcpyAsync(h->ci(), X0->idx[0], n * sizeof(int32_t), cudaMemcpyDefault, h->st));
    CK(cudaMemcpyAsync(h->cj(), X0->idx[1], n * sizeof(int32_t), cudaMemcpyDefault, h->st));
    CK(cudaMemcpyAsync(h->ck_(), X0->idx[2], n * sizeof(int32_t), cudaMemcpyDefault, h->st));
    CK(cudaMemcpyAsync(h->cv(), X0->vals, n * sizeof(float), cudaMemcpyDefault, h->st));
  }
  for (int b = 0; b < 2; ++b) {
    CK(h->model[b].ensure(h->model_floats() * sizeof(float)));
    CK(cudaMemsetAsync(h->model[b].p, 0, h->model_floats() * sizeof(float), h->st));
  }
  CK(cudaMallocHost(&h->segs_host, sizeof(SampleSeg) * 3 * kMaxReps));
  CK(cudaMallocHost(&h->hs, sizeof(HostStatus)));
  for (int e = 0; e < 9; ++e) CK(cudaEventCreate(&h->ev[e]));
  // fixed-point scale from X0 (R7)
  CK(h->misc.ensure(4096));
  CK(cudaMemsetAsync(h->misc.p, 0, 16, h->st));
  if (h->fmt == SAMBATEN_DENSE) {
    CK(launch_max_phi_dense(h->view(), 0, h->K, h->opts.moi, h->misc.as<unsigned long long>(), h->st));
  } else {
    CK(launch_coo_max_phi(h->cv(), h->nnz, h->opts.moi, h->misc.as<unsigned long long>(), h->st));
    // the initial tensor must be canonical (R28)
    CK(launch_coo_validate(h->ci(), h->cj(), h->ck_(), h->cv(), h->nnz, h->I, h->J, h->K,
                           reinterpret_cast<unsigned*>(h->misc.as<char>() + 8), h->st));
  }
  unsigned long long bits = 0;
  unsigned vflags = 0;
  CK(cudaMemcpyAsync(&vflags, h->misc.as<char>() + 8, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaMemcpyAsync(&bits, h->misc.p, 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  double maxphi;
  memcpy(&maxphi, &bits, 8);
  if (vflags & 1u) FAIL(SAMBATEN_E_INDEX_RANGE, "init: COO index out of range (S:77)");
  if (vflags & 6u) FAIL(SAMBATEN_E_INVALID, "init: COO tensor not canonical (sorted by (k,j,i), unique, nonzero; R28)");
  if (!(maxphi > 0.0)) FAIL(SAMBATEN_E_DEGENERATE, "init: all-zero initial tensor");
  const int64_t cap_entries = h->fmt == SAMBATEN_DENSE ? h->I * h->J * h->Kcap : h->nnz_cap;
  h->S = sambaten_fixed_point_scale(cap_entries, maxphi);
  h->maxphi_log2 = ceil_log2_d(maxphi);
  h->phimax_run = maxphi;
  return SAMBATEN_OK;
}

static void dist_destroy(DistState* d);

extern "C" void sambaten_destroy(sambaten_t h) {
  if (!h) return;
  cudaStreamSynchronize(h->st);
  dist_destroy(h->dist);
  h->dist = nullptr;
  if (h->st2) {
    cudaStreamSynchronize(h->st2);
    cudaStreamDestroy(h->st2);
    cudaEventDestroy(h->ev_side[0]);
    cudaEventDestroy(h->ev_side[1]);
    if (h->ev_pl[0]) { cudaEventDestroy(h->ev_pl[0]); cudaEventDestroy(h->ev_pl[1]); }
  }
  if (h->X_borrowed) h->X.p = nullptr;   // the caller's buffer: not ours to free
  h->X.release();
  h->model[0].release(); h->model[1].release(); h->ck.release();
  h->marg.release(); h->xm.release(); h->xm_ck.release(); h->samp.release(); h->summ.release(); h->fac.release();
  h->als.release(); h->match.release(); h->misc.release(); h->segs.release(); h->fitws.release();
  h->coo_ws.release(); h->grws.release(); h->grk.release(); h->fiws.release(); h->gord.release();
  if (h->segs_host) cudaFreeHost(h->segs_host);
  if (h->hs) cudaFreeHost(h->hs);
  for (int e = 0; e < 9; ++e)
    if (h->ev[e]) cudaEventDestroy(h->ev[e]);
  delete h;
}

__global__ static void lam_to_f32_kernel(const double* l, int R, float* out) {
  if (threadIdx.x < R) out[threadIdx.x] = (float)l[threadIdx.x];
}

static sambaten_status init_als_coo(sambaten_s* h);
static cudaError_t compute_committed_marginals(sambaten_s* h);

// The incremental fit's state of the initial model (one per-component pass over X0; untimed
// init work) when the updates will report the full fit of a dense handle (full_fit = 1).
static cudaError_t init_fit_state(sambaten_s* h) {
  if (h->opts.full_fit != 1 || h->dist || getenv("SAMBATEN_FULL_FIT_PASS") ||
      (h->fmt == SAMBATEN_DENSE && !fitrows_supported(h->pitch, h->R)))
    return cudaSuccess;
  cudaError_t e = h->misc.ensure(4096);
  if (e != cudaSuccess) return e;
  double* scratch = reinterpret_cast<double*>(h->misc.as<char>() + 512);
  if (h->fmt == SAMBATEN_COO)
    return fitinc_run_coo(h, 0, h->nnz, 0, h->K, h->cur, h->cur, true, scratch, h->st);
  return fitinc_run(h, h->view(), 0, 0, h->K, h->cur, h->cur, true, nullptr, false, scratch, h->st);
}

extern "C" sambaten_status sambaten_init(sambaten_t* out, const sambaten_tensor* X0, int R, int s,
                                         int r, uint64_t seed, const sambaten_opts* opts) {
  if (sambaten_status e = create_common(out, X0, R, s, r, seed, opts)) return e;
  sambaten_s* h = *out;
  if (sambaten_status e = alloc_store_and_model(h, X0)) { sambaten_destroy(h); *out = nullptr; return e; }
  if (h->fmt == SAMBATEN_COO) {
    if (sambaten_status e = init_als_coo(h)) { sambaten_destroy(h); *out = nullptr; return e; }
    const cudaError_t ce = init_fit_state(h);
    if (ce != cudaSuccess || cudaStreamSynchronize(h->st) != cudaSuccess) {
      set_error(std::string("init fit state: ") + cudaGetErrorString(ce));
      sambaten_destroy(h); *out = nullptr;
      return SAMBATEN_E_CUDA;
    }
    return SAMBATEN_OK;
  }
  // full CP-ALS on X0, r = 1, Philox init with update_id 0 (R10)
  DenseAls a{};
  a.Y = h->X.as<float>(); a.y_stride = 0; a.pitch = h->pitch;
  a.nI = (int)h->I; a.nJ = (int)h->J; a.nK = (int)h->K; a.R = R; a.r = 1;
  a.U[0] = h->A(h->cur); a.U[1] = h->B(h->cur); a.U[2] = h->C(h->cur);
  a.u_stride[0] = a.u_stride[1] = a.u_stride[2] = 0;
  a.maxit = h->opts.init_max_iters; a.tol = h->opts.init_tol;
  DevBuf ws;
  cudaError_t ce = ws.ensure(dense_als_workspace(&a));
  if (ce == cudaSuccess) ce = dense_als_bind_workspace(&a, ws.p);
  if (ce == cudaSuccess) ce = launch_als_init(a, seed, 0, 0, true, h->st);
  if (ce == cudaSuccess) ce = run_dense_als(a, h->st);
  if (ce == cudaSuccess) {
    lam_to_f32_kernel<<<1, 32, 0, h->st>>>(a.lam, R, h->lam(h->cur));
    ce = init_fit_state(h);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->st);
  }
  ws.release();
  if (ce != cudaSuccess) {
    set_error(std::string("init ALS: ") + cudaGetErrorString(ce));
    sambaten_destroy(h); *out = nullptr;
    return ce == cudaErrorMemoryAllocation ? SAMBATEN_E_OOM : SAMBATEN_E_CUDA;
  }
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_init_factors(sambaten_t* out, const sambaten_tensor* X0, int R,
                                                 int s, int r, uint64_t seed, const float* A,
                                                 const float* B, const float* C,
                                                 const float* lambda, const sambaten_opts* opts) {
  if (!A || !B || !C || !lambda) FAIL(SAMBATEN_E_INVALID, "init_factors: NULL factor");
  if (sambaten_status e = create_common(out, X0, R, s, r, seed, opts)) return e;
  sambaten_s* h = *out;
  if (sambaten_status e = alloc_store_and_model(h, X0)) { sambaten_destroy(h); *out = nullptr; return e; }
  const int b = h->cur;
  cudaError_t ce = cudaMemcpyAsync(h->A(b), A, sizeof(float) * h->I * R, cudaMemcpyDefault, h->st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(h->B(b), B, sizeof(float) * h->J * R, cudaMemcpyDefault, h->st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(h->C(b), C, sizeof(float) * h->K * R, cudaMemcpyDefault, h->st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(h->lam(b), lambda, sizeof(float) * R, cudaMemcpyDefault, h->st);
  if (ce == cudaSuccess) ce = init_fit_state(h);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->st);
  if (ce != cudaSuccess) {
    set_error(std::string("init_factors: ") + cudaGetErrorString(ce));
    sambaten_destroy(h); *out = nullptr;
    return SAMBATEN_E_CUDA;
  }
  return SAMBATEN_OK;
}

// ---------------------------------------------------------------------------------------
// the update (Alg. 1)
// ---------------------------------------------------------------------------------------
static inline int64_t sample_n(int64_t n, int s) { return std::min<int64_t>(n, (n + s - 1) / s); }

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// ---------------------------------------------------------------------------------------
// update steps shared by the dense and COO paths
// ---------------------------------------------------------------------------------------
// a2: sampling (R4-R6); K_s from the old slices only, then K' = K_s ++ new.  Outputs point
// into h->samp: Is [r][nI], Js [r][nJ], Kp [r][nKp], loc maps [r][I], [r][J], [r][Ko].
static cudaError_t run_sampling(sambaten_s* h, const int64_t* x1, const int64_t* x2, const int64_t* x3,
                                int64_t Ko, int64_t Kn, int64_t nI, int64_t nJ, int64_t nKs,
                                int64_t nKp, uint32_t uid, int32_t** Is_, int32_t** Js_, int32_t** Kp_,
                                int32_t** locI_, int32_t** locJ_, int32_t** locK_) {
  const int r = h->r;
  const size_t is_b = align256(sizeof(int32_t) * r * nI), js_b = align256(sizeof(int32_t) * r * nJ);
  const size_t kp_b = align256(sizeof(int32_t) * r * nKp);
  const size_t li_b = align256(sizeof(int32_t) * r * h->I), lj_b = align256(sizeof(int32_t) * r * h->J);
  const size_t lk_b = align256(sizeof(int32_t) * r * std::max<int64_t>(Ko, 1));
  const size_t key_b = align256(sizeof(uint64_t) * 3 * r * std::max(h->I, std::max(h->J, Ko)));
  cudaError_t e = h->samp.ensure(is_b + js_b + kp_b + li_b + lj_b + lk_b + key_b);
  if (e != cudaSuccess) return e;
  char* sp = h->samp.as<char>();
  int32_t* Is = (int32_t*)sp; sp += is_b;
  int32_t* Js = (int32_t*)sp; sp += js_b;
  int32_t* Kp = (int32_t*)sp; sp += kp_b;
  int32_t* locI = (int32_t*)sp; sp += li_b;
  int32_t* locJ = (int32_t*)sp; sp += lj_b;
  int32_t* locK = (int32_t*)sp; sp += lk_b;
  uint64_t* keys = (uint64_t*)sp;
  const int64_t kstride = std::max(h->I, std::max(h->J, Ko));
  for (int rho = 0; rho < r; ++rho) {
    for (int m = 0; m < 3; ++m) {
      SampleSeg& g = h->segs_host[rho * 3 + m];
      g.rep = rho; g.mode = m;
      g.keys = keys + (int64_t)(rho * 3 + m) * kstride;
      g.kp_tail = nullptr; g.tail0 = 0; g.ntail = 0;
      if (m == 0) { g.w = x1; g.n = h->I; g.ns = nI; g.out = Is + rho * nI; g.loc = locI + rho * h->I; }
      if (m == 1) { g.w = x2; g.n = h->J; g.ns = nJ; g.out = Js + rho * nJ; g.loc = locJ + rho * h->J; }
      if (m == 2) {
        g.w = x3; g.n = Ko; g.ns = nKs; g.out = Kp + rho * nKp; g.loc = locK + rho * Ko;
        g.kp_tail = Kp + rho * nKp + nKs; g.tail0 = Ko; g.ntail = Kn;
      }
    }
  }
  e = h->segs.ensure(sizeof(SampleSeg) * 3 * kMaxReps);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(h->segs.p, h->segs_host, sizeof(SampleSeg) * 3 * r, cudaMemcpyHostToDevice, h->st);
  if (e != cudaSuccess) return e;
  e = launch_sample(h->segs.as<SampleSeg>(), 3 * r, h->seed, uid, h->st);
  *Is_ = Is; *Js_ = Js; *Kp_ = Kp; *locI_ = locI; *locJ_ = locJ; *locK_ = locK;
  return e;
}

// a5 (match against the batch-start model, R13-R16, R26) and a6 (merge into the shadow model,
// P:216-227).  Records ev[6] between the two.
// GetRank (Alg. 2; readings R29-R31) on nsum dense summaries Y + s * y_stride
// ([K][J][pitch] each): for every candidate rank F = 1..R_max, `trials` CP-ALS runs (Philox
// update_id 0x47520000 + F, rep = s * trials + j, R30) rated by CorConDia; R_new[s] = the largest
// F whose best trial reaches `threshold` (R31), else 1.  cc (host, optional) gets [s][F-1][j].
// Synchronises st: the rank fixes the launch shapes of what follows.
static cudaError_t getrank_batch(const float* Y, int64_t y_stride, int64_t pitch, int I, int J, int K,
                                 int nsum, int R_max, int trials, uint64_t seed, int max_iters, double tol,
                                 double threshold, DevBuf& ws, cudaStream_t st, int* R_new, double* cc,
                                 int* launches, uint32_t rep_base = 0) {
  constexpr uint32_t kGetRankId = 0x47520000u;   // R30
  // trials == 1: the nsum summaries are one batch of models (rep = s); else one batch of
  // `trials` models per summary (rep = s * trials + j)
  const bool by_summary = trials == 1;
  const int groups = by_summary ? 1 : nsum, nm = by_summary ? nsum : trials;
  DenseAls a{};
  a.y_stride = by_summary ? y_stride : 0; a.pitch = pitch;
  a.nI = I; a.nJ = J; a.nK = K; a.R = R_max; a.r = nm;
  a.maxit = max_iters; a.tol = tol;
  const size_t ub = align256(sizeof(float) * (size_t)nm * (I + J + K) * R_max);
  const size_t als_b = align256(dense_als_workspace(&a));
  const size_t ccn = corcondia_ws_doubles(I, J, K, R_max, nm);
  const size_t cc_b = align256(sizeof(double) * (ccn + (size_t)groups * R_max * nm));
  cudaError_t e = ws.ensure(ub + als_b + cc_b);
  if (e != cudaSuccess) return e;
  char* base = ws.as<char>();
  double* ccws = reinterpret_cast<double*>(base + ub + als_b);
  double* ccd = ccws + ccn;   // [group][F-1][nm]
  int nl = 0;
  for (int g = 0; g < groups; ++g) {
    a.Y = Y + (by_summary ? 0 : g * y_stride);
    for (int F = 1; F <= R_max; ++F) {
      a.R = F;
      a.U[0] = reinterpret_cast<float*>(base);
      a.U[1] = a.U[0] + (size_t)nm * I * F;
      a.U[2] = a.U[1] + (size_t)nm * J * F;
      a.u_stride[0] = (int64_t)I * F; a.u_stride[1] = (int64_t)J * F; a.u_stride[2] = (int64_t)K * F;
      dense_als_workspace(&a);
      if ((e = dense_als_bind_workspace(&a, base + ub)) != cudaSuccess) return e;
      if ((e = launch_als_init(a, seed, kGetRankId + (uint32_t)F, rep_base + (uint32_t)(g * trials), true, st)) !=
          cudaSuccess)
        return e;
      if ((e = run_dense_als(a, st)) != cudaSuccess) return e;
      const float* U[3] = {a.U[0], a.U[1], a.U[2]};
      e = launch_corcondia(a.Y, a.y_stride, pitch, I, J, K, F, nm, U, a.u_stride, a.lam, ccws,
                           ccd + ((size_t)g * R_max + F - 1) * nm, st);
      if (e != cudaSuccess) return e;
      nl += 4 + 7 * max_iters + 4;
    }
  }
  std::vector<double> hc((size_t)groups * R_max * nm);
  if ((e = cudaMemcpyAsync(hc.data(), ccd, sizeof(double) * hc.size(), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  for (int s = 0; s < nsum; ++s) {
    int best = 1;
    for (int F = 1; F <= R_max; ++F) {
      double m = -1e300;
      for (int j = 0; j < trials; ++j) {
        const double v = by_summary ? hc[(size_t)(F - 1) * nm + s] : hc[((size_t)s * R_max + F - 1) * nm + j];
        if (cc) cc[((size_t)s * R_max + F - 1) * trials + j] = v;
        m = std::max(m, v);
      }
      if (m >= threshold) best = F;
    }
    R_new[s] = best;
  }
  if (launches) *launches += nl;
  return cudaSuccess;
}

// a4 with GetRank's ranks (R33): every repetition decomposes its summary at its own rank
// R_new[rho] (Philox rep rho, as the plain path) and is padded with zero columns into the
// R-column candidate buffers of `a` (whose workspace is bound).
static cudaError_t rank_als(sambaten_s* h, const DenseAls& a, const int* R_new, uint32_t uid,
                            cudaStream_t st, int* launches, uint32_t rep0 = 0, uint32_t rep_stride = 1) {
  DenseAls b{};
  b.y_stride = 0; b.pitch = a.pitch; b.nI = a.nI; b.nJ = a.nJ; b.nK = a.nK; b.r = 1;
  b.maxit = a.maxit; b.tol = a.tol;
  b.R = a.R;
  const size_t ub = align256(sizeof(float) * (size_t)(a.nI + a.nJ + a.nK) * a.R);
  cudaError_t e = h->grws.ensure(ub + align256(dense_als_workspace(&b)));
  if (e != cudaSuccess) return e;
  for (int rho = 0; rho < a.r; ++rho) {
    b.Y = a.Y + rho * a.y_stride;
    b.R = R_new[rho];
    b.U[0] = h->grws.as<float>();
    b.U[1] = b.U[0] + (size_t)a.nI * b.R;
    b.U[2] = b.U[1] + (size_t)a.nJ * b.R;
    b.u_stride[0] = (int64_t)a.nI * b.R; b.u_stride[1] = (int64_t)a.nJ * b.R; b.u_stride[2] = (int64_t)a.nK * b.R;
    dense_als_workspace(&b);
    if ((e = dense_als_bind_workspace(&b, h->grws.as<char>() + ub)) != cudaSuccess) return e;
    if ((e = launch_als_init(b, h->seed, uid, rep0 + (uint32_t)rho * rep_stride, true, st)) != cudaSuccess) return e;
    if ((e = run_dense_als(b, st)) != cudaSuccess) return e;
    if ((e = launch_rank_pad(b, a, rho, st)) != cudaSuccess) return e;
    *launches += 4 + 7 * a.maxit + 1;
  }
  return cudaSuccess;
}

static cudaError_t run_match_merge(sambaten_s* h, const DenseAls& a, const int32_t* Is, const int32_t* Js,
                                   const int32_t* Kp, const int32_t* locI, const int32_t* locJ,
                                   const int32_t* locK, int64_t Ko, int64_t Kn, int64_t nI, int64_t nJ,
                                   int64_t nKs, int64_t nKp, int** accepted, const int* rnew = nullptr) {
  const int R = h->R, r = h->r;
  cudaStream_t st = h->st;
  const int b = h->cur, nb = 1 - h->cur;
  MatchArgs ma{};
  ma.A = h->A(b); ma.B = h->B(b); ma.C = h->C(b); ma.R = R; ma.r = r;
  ma.Is = Is; ma.Js = Js; ma.Ks = Kp;
  ma.nI = (int)nI; ma.nJ = (int)nJ; ma.nKs = (int)nKs; ma.nK = (int)nKp; ma.ks_stride = nKp;
  const size_t part_b = align256(sizeof(double) * match_part_doubles(ma));
  cudaError_t e = h->match.ensure(align256(sizeof(int) * r * R) + align256(sizeof(double) * r * 3 * R) +
                                  align256(sizeof(double) * r * R) + align256(sizeof(double) * r) +
                                  align256(sizeof(int) * r) + part_b);
  if (e != cudaSuccess) return e;
  char* mp = h->match.as<char>();
  ma.part = reinterpret_cast<double*>(mp + h->match.bytes - part_b);
  for (int m = 0; m < 3; ++m) { ma.U[m] = a.U[m]; ma.u_stride[m] = a.u_stride[m]; }
  ma.lamp = a.lam; ma.tau = h->opts.accept_tau;
  ma.pi = (int*)mp; mp += align256(sizeof(int) * r * R);
  ma.scale = (double*)mp; mp += align256(sizeof(double) * r * 3 * R);
  ma.lam_hat = (double*)mp; mp += align256(sizeof(double) * r * R);
  ma.score_min = (double*)mp; mp += align256(sizeof(double) * r);
  ma.accepted = (int*)mp;
  ma.rnew = rnew;
  e = launch_match(ma, st);
  if (e != cudaSuccess) return e;
  e = cudaEventRecord(h->ev[6], st);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(h->model[nb].p, h->model[b].p, h->model_floats() * sizeof(float),
                      cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  MergeArgs g{};
  g.A = h->A(b); g.B = h->B(b); g.C = h->C(b); g.lam = h->lam(b);
  g.An = h->A(nb); g.Bn = h->B(nb); g.Cn = h->C(nb); g.lamn = h->lam(nb);
  g.I = h->I; g.J = h->J; g.Ko = Ko; g.Kn = Kn; g.R = R; g.r = r;
  g.loc[0] = locI; g.loc[1] = locJ; g.loc[2] = locK; g.nKs = (int)nKs;
  for (int m = 0; m < 3; ++m) { g.U[m] = a.U[m]; g.u_stride[m] = a.u_stride[m]; }
  g.pi = ma.pi; g.scale = ma.scale; g.lam_hat = ma.lam_hat; g.accepted = ma.accepted;
  g.rnew = rnew;
  g.policy = h->opts.merge_policy;
  *accepted = ma.accepted;
  return launch_merge(g, st);
}

// Status readback, validation outcome, commit (strong guarantee: nothing above is visible
// before this point), info and copy-out.
static sambaten_status finish_update(sambaten_s* h, const DenseAls& a, const int* accepted,
                                     const unsigned long long* d_maxphi, const unsigned* d_vflags,
                                     const double* d_relerr, int64_t Ko, int64_t Kn, int64_t nI,
                                     int64_t nJ, int64_t nKs, int64_t nKp, int b, int nb, int launches,
                                     int64_t batch_nnz, float* Aout, float* Bout, float* Cout,
                                     float* lamout, sambaten_info* info) {
  const int R = h->R, r = h->r;
  cudaStream_t st = h->st;
  (void)b;
  HostStatus* hs = h->hs;
  unsigned vflags = 0;
  CK(cudaMemcpyAsync(&hs->maxphi_bits, d_maxphi, 8, cudaMemcpyDeviceToHost, st));
  if (d_vflags) CK(cudaMemcpyAsync(&hs->vflags, d_vflags, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hs->accepted, accepted, sizeof(int) * r, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hs->iters, a.iters, sizeof(int) * r, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hs->flags, a.flags, sizeof(int) * r, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hs->fit, a.fit, sizeof(double) * r, cudaMemcpyDeviceToHost, st));
  const bool fit_now = h->opts.full_fit == 1 || (h->opts.full_fit == 2 && !h->lag_now);
  if (fit_now) CK(cudaMemcpyAsync(&hs->relerr, d_relerr, 8, cudaMemcpyDeviceToHost, st));
  if (h->lag_now) CK(cudaMemcpyAsync(&hs->relerr_prev, d_relerr + 4, 8, cudaMemcpyDeviceToHost, st));
  if (h->d_fit_mode) CK(cudaMemcpyAsync(&hs->fit_mode, h->d_fit_mode, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (d_vflags) vflags = hs->vflags;
  if (vflags & 1u) FAIL(SAMBATEN_E_INDEX_RANGE, "update: COO index out of range (S:77)");
  if (vflags & 6u) FAIL(SAMBATEN_E_INVALID, "update: COO batch not canonical (sorted by (k,j,i), unique, nonzero; R28)");
  double maxphi;
  memcpy(&maxphi, &hs->maxphi_bits, 8);
  if (maxphi > ldexp(1.0, h->maxphi_log2 + 8))
    FAIL(SAMBATEN_E_FIXEDPOINT_RANGE, "update: batch value outside the fixed-point range (R7)");
  if (maxphi > h->phimax_run) h->phimax_run = maxphi;   // (a later failure only leaves it an upper bound)
  uint32_t rejected = 0, pm = 0;
  int nacc = 0, itmax = 0, itsum = 0;
  double fsum = 0.0;
  for (int rho = 0; rho < r; ++rho) {
    if (hs->accepted[rho]) ++nacc; else rejected |= 1u << rho;
    if (hs->flags[rho] & 1) pm |= 1u << rho;
    itmax = std::max(itmax, hs->iters[rho]);
    itsum += hs->iters[rho];
    fsum += hs->fit[rho];
  }
  if (nacc == 0) FAIL(SAMBATEN_E_BATCH_REJECTED, "update: every repetition was rejected (R26)");
  // commit
  if (h->opts.incremental_marginals || h->opts.pipelined) {   // this update's marginals are the new committed ones
    std::swap(h->marg, h->xm);
    h->xm_valid = true;
  }
  h->cur = nb;
  h->K = Ko + Kn;
  if (h->fmt == SAMBATEN_COO) h->nnz += batch_nnz;
  h->update_id += 1;
  h->last_n[0] = nI; h->last_n[1] = nJ; h->last_n[2] = nKs; h->last_nKp = nKp;
  if (info) {
    info->fit_summary = fsum / r;
    info->fit_full = fit_now ? 1.0 - hs->relerr : -1.0;
    info->fit_full_prev = h->lag_now ? 1.0 - hs->relerr_prev : -1.0;
    info->fit_path = h->d_fit_mode ? (hs->fit_mode == 1 ? 3 : 4) : (h->lag_now ? 2 : (fit_now ? 1 : 0));
    info->als_iters_max = itmax;
    info->als_iters_sum = itsum;
    info->k_total = h->K;
    info->reps_rejected_mask = rejected;
    info->scale_exp = h->S;
    info->reps_pinv_mask = pm;
    info->kernel_launches = launches;
    for (int rho = 0; rho < 32; ++rho) info->rep_rank[rho] = rho < r ? (h->opts.getrank ? h->rep_rank[rho] : R) : 0;
    for (int e = 0; e < 4; ++e) info->als_plan[e] = h->als_plan[e];
    info->summary_entries = h->summ_entries;
    for (int e = 0; e < 8; ++e) {
      float ms = 0.f;
      if (e == 1 && h->pipe_now) cudaEventElapsedTime(&ms, h->ev_pl[0], h->ev_pl[1]);   // a1 on the side stream
      else cudaEventElapsedTime(&ms, h->ev[e], h->ev[e + 1]);
      info->step_ms[e] = ms;
    }
  }
  if (Aout) CK(cudaMemcpyAsync(Aout, h->A(nb), sizeof(float) * h->I * R, cudaMemcpyDefault, st));
  if (Bout) CK(cudaMemcpyAsync(Bout, h->B(nb), sizeof(float) * h->J * R, cudaMemcpyDefault, st));
  if (Cout) CK(cudaMemcpyAsync(Cout, h->C(nb), sizeof(float) * h->K * R, cudaMemcpyDefault, st));
  if (lamout) CK(cudaMemcpyAsync(lamout, h->lam(nb), sizeof(float) * R, cudaMemcpyDefault, st));
  if (Aout || Bout || Cout || lamout) CK(cudaStreamSynchronize(st));
  return SAMBATEN_OK;
}

// ---------------------------------------------------------------------------------------
// COO: batched CP-ALS on r concatenated COO summaries (entries [off[rho], off[rho+1]) of rep
// rho, canonical (u, q, p)).  Mode-0/1 row structure by stable radix sort, mode 2 by the
// natural order; per iteration and mode: MTTKRP (warp per row) -> R x R solve / normalise /
// Gram / fit (k_als.cu solve kernel).  Returns the ALS state in `d`.
// ---------------------------------------------------------------------------------------
struct Bump {
  char* base = nullptr;
  size_t off = 0;
  template <class T> T* take(size_t n) {
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += (sizeof(T) * n + 255) & ~(size_t)255;
    return p;
  }
};

// pinned host words for the COO ALS's done flags (kMaxReps; one per host thread)
static int* pinned_done_flags() {
  thread_local int* p = nullptr;
  if (!p && cudaHostAlloc(reinterpret_cast<void**>(&p), sizeof(int) * kMaxReps, cudaHostAllocDefault) != cudaSuccess)
    p = nullptr;
  return p;
}

static int bits_for(int64_t n) { int b = 1; while (((int64_t)1 << b) < n) ++b; return b; }

// which batched COO ALS the last coo_als call ran (sambaten_info.als_plan[0]: 3 persistent, 4 per mode)
static thread_local int g_coo_als_kind = -1;

// the model rows a warm-started summary ALS begins from (R34): A(I_s), B(J_s), C(K_s) diag(lambda)
struct WarmRows {
  const float *A, *B, *C, *lam;
  const int32_t *Is, *Js, *Kp;
  int nKs;
};

static sambaten_status coo_als(DevBuf& wsbuf, cudaStream_t st, int R, const int32_t* p, const int32_t* q,
                               const int32_t* u, const float* v, const int64_t* d_off, int64_t ntot,
                               int nI, int nJ, int nK, int r, float* U0, float* U1, float* U2,
                               uint64_t seed, uint32_t uid, int maxit, double tol, bool init_factors,
                               DenseAls* d, int* launches, uint32_t rep0 = 0, uint32_t rep_stride = 1,
                               const WarmRows* warm = nullptr) {
  const int64_t maxn = std::max<int64_t>(nI, std::max<int64_t>(nJ, nK));
  const int kb0 = bits_for(nI), kb1 = bits_for(nJ), kb2 = bits_for(nK);
  const int64_t n = std::max<int64_t>(ntot, 1);
  const int64_t pmax = (int64_t)r * maxn + 1;
  const size_t sws_n = std::max(scan_ws_elems(radix_ws_elems(n)), scan_ws_elems(pmax));
  auto layout = [&](Bump& b, bool assign) {
    uint32_t* keys = b.take<uint32_t>(n);
    int32_t* perm0 = b.take<int32_t>(n);
    int32_t* perm1 = b.take<int32_t>(n);
    uint32_t* wk = b.take<uint32_t>(n);
    int32_t* wv = b.take<int32_t>(n);
    int64_t* hist = b.take<int64_t>(radix_ws_elems(n));
    int64_t* offs = b.take<int64_t>(radix_ws_elems(n));
    int64_t* sws = b.take<int64_t>(sws_n);
    int64_t* cnt = b.take<int64_t>(pmax);
    int64_t* ptr0 = b.take<int64_t>((int64_t)r * nI + 1);
    int64_t* ptr1 = b.take<int64_t>((int64_t)r * nJ + 1);
    int64_t* ptr2 = b.take<int64_t>((int64_t)r * nK + 1);
    double* G = b.take<double>((size_t)r * 3 * R * R);
    double* lam = b.take<double>((size_t)r * R);
    double* ysq = b.take<double>((size_t)r * 257);
    double* gpart = b.take<double>(gram_part_doubles((int)maxn, R, r));
    double* fit = b.take<double>(r);
    double* fitp = b.take<double>(r);
    int* iters = b.take<int>(r);
    int* done = b.take<int>(r);
    int* flags = b.take<int>(r);
    double* M0 = b.take<double>((size_t)r * nI * R);
    double* Mb = b.take<double>((size_t)r * maxn * R);
    double* Us = b.take<double>((size_t)r * maxn * R);
    double* Vi = b.take<double>((size_t)r * R * R);
    double* rpart = b.take<double>(als_rows_part_doubles((int)maxn, R, r));
    int* stop = b.take<int>(r);
    unsigned* gbar = b.take<unsigned>(coo_als_persist_ctr_words(maxit));
    const int RBp = R <= 4 ? 4 : R <= 8 ? 8 : R <= 12 ? 12 : R <= 16 ? 16 : R <= 24 ? 24 : 32;
    const bool padded = R <= 16;   // the row-parallel solve keeps the padded copies in sync
    float* Upad = padded ? b.take<float>((size_t)r * ((int64_t)nI + nJ + nK) * RBp) : nullptr;
    // per-mode MTTKRP plans: row pieces, sorted copies (modes 0, 1), piece partials
    const int rows_m[3] = {nI, nJ, nK};
    CooModePlan plan[3];
    for (int m = 0; m < 3; ++m) {
      const int64_t nrow = (int64_t)r * rows_m[m];
      const size_t pe = coo_plan_elems(nrow, n);
      plan[m].nrow = nrow; plan[m].n = ntot;
      plan[m].pstart = b.take<int64_t>(nrow + 1);
      plan[m].pb = b.take<int64_t>(pe);
      plan[m].prow = b.take<int32_t>(pe);
      plan[m].partial = b.take<double>(pe * R);
      plan[m].plist = b.take<int32_t>(pe);
      plan[m].nlist = b.take<unsigned>(2);
      if (m < 2) {
        plan[m].sa = b.take<int32_t>(n); plan[m].sb = b.take<int32_t>(n); plan[m].sv = b.take<float>(n);
      }
    }
    if (!assign) return;
    plan[0].ptr = ptr0; plan[1].ptr = ptr1; plan[2].ptr = ptr2;
    plan[2].sa = p; plan[2].sb = q; plan[2].sv = v;
    *d = DenseAls{};
    d->nI = nI; d->nJ = nJ; d->nK = nK; d->R = R; d->r = r;
    d->U[0] = U0; d->U[1] = U1; d->U[2] = U2;
    d->u_stride[0] = (int64_t)nI * R; d->u_stride[1] = (int64_t)nJ * R; d->u_stride[2] = (int64_t)nK * R;
    d->G = G; d->lam = lam; d->ysq = ysq; d->fit = fit; d->fit_prev = fitp; d->iters = iters;
    d->done = done; d->flags = flags; d->part0 = M0; d->nb0 = 1; d->rows_per_block0 = 0;
    d->M = Mb; d->m_stride = maxn * R; d->Uscr = Us; d->maxit = maxit; d->tol = tol;
    // sort / row pointers
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = coo_sort_by_index(p, d_off, r, kb0, ntot, keys, perm0, wk, wv, hist, offs, sws, st);
    if (e == cudaSuccess) e = coo_row_pointers(keys, ntot, kb0, r, nI, cnt, ptr0, sws, st);
    if (e == cudaSuccess) e = coo_sort_by_index(q, d_off, r, kb1, ntot, keys, perm1, wk, wv, hist, offs, sws, st);
    if (e == cudaSuccess) e = coo_row_pointers(keys, ntot, kb1, r, nJ, cnt, ptr1, sws, st);
    if (e == cudaSuccess) e = coo_make_keys(u, d_off, r, kb2, ntot, keys, st);
    if (e == cudaSuccess) e = coo_row_pointers(keys, ntot, kb2, r, nK, cnt, ptr2, sws, st);
    if (e == cudaSuccess) e = coo_build_plan(plan[0], perm0, q, u, v, ntot, cnt, sws, st);
    if (e == cudaSuccess) e = coo_build_plan(plan[1], perm1, p, u, v, ntot, cnt, sws, st);
    if (e == cudaSuccess) e = coo_build_plan(plan[2], nullptr, p, q, v, ntot, cnt, sws, st);
    CooAls a{};
    a.nI = nI; a.nJ = nJ; a.nK = nK; a.R = R; a.r = r;
    a.RB = R <= 4 ? 4 : R <= 8 ? 8 : R <= 12 ? 12 : R <= 16 ? 16 : R <= 24 ? 24 : 32;
    for (int m = 0; m < 3; ++m) a.plan[m] = plan[m];
    for (int m = 0; m < 3; ++m) { a.U[m] = d->U[m]; a.u_stride[m] = d->u_stride[m]; }
    a.M[0] = M0; a.m_stride[0] = (int64_t)nI * R;
    a.M[1] = a.M[2] = Mb; a.m_stride[1] = a.m_stride[2] = maxn * R;
    a.done = done;
    float* Up3[3] = {nullptr, nullptr, nullptr};
    if (padded) {
      Up3[0] = Upad;
      Up3[1] = Up3[0] + (size_t)r * nI * RBp;
      Up3[2] = Up3[1] + (size_t)r * nJ * RBp;
    }
    const int64_t ups[3] = {(int64_t)nI * RBp, (int64_t)nJ * RBp, (int64_t)nK * RBp};
    for (int m = 0; m < 3; ++m) { a.Up[m] = Up3[m]; a.up_stride[m] = ups[m]; }
    if (e == cudaSuccess && init_factors) e = launch_als_init_factors(*d, seed, uid, rep0, st, rep_stride);
    if (e == cudaSuccess && warm)   // R34: the model's rows replace the Philox point (before the Grams)
      e = launch_warm_init(*d, warm->A, warm->B, warm->C, warm->lam, warm->Is, warm->Js, warm->Kp, warm->nKs, st,
                           (int)rep0, (int)rep_stride);
    if (e == cudaSuccess && !init_factors) e = cudaMemsetAsync(done, 0, sizeof(int) * r, st);
    if (e == cudaSuccess && !init_factors) e = cudaMemsetAsync(iters, 0, sizeof(int) * r, st);
    if (e == cudaSuccess && !init_factors) e = cudaMemsetAsync(flags, 0, sizeof(int) * r, st);
    if (e == cudaSuccess && !init_factors) e = cudaMemsetAsync(fit, 0, sizeof(double) * r, st);
    if (e == cudaSuccess) {
      GramArgs ga{};
      for (int m = 0; m < 3; ++m) { ga.U[m] = d->U[m]; ga.u_stride[m] = d->u_stride[m]; }
      ga.n[0] = nI; ga.n[1] = nJ; ga.n[2] = nK; ga.R = R; ga.r = r;
      ga.tmax = gram_tiles_for((int)maxn); ga.part = gpart; ga.G = G; ga.g_stride = 3 * R * R;
      e = launch_gram_tiles(ga, st);
    }
    if (e == cudaSuccess) e = launch_coo_sumsq(v, d_off, r, ysq, st);
    // row-parallel solve steps (k_als_rows.cu) for R <= 16, the one-block solve otherwise
    RowsAls ra{};
    ra.nI = nI; ra.nJ = nJ; ra.nK = nK; ra.R = R; ra.r = r; ra.maxit = maxit; ra.tol = tol;
    for (int m = 0; m < 3; ++m) { ra.U[m] = d->U[m]; ra.u_stride[m] = d->u_stride[m]; }
    ra.M[0] = M0; ra.m_stride[0] = (int64_t)nI * R;
    ra.M[1] = ra.M[2] = Mb; ra.m_stride[1] = ra.m_stride[2] = maxn * R;
    ra.X = Us; ra.x_stride = maxn * R; ra.Vi = Vi; ra.part = rpart; ra.G = G; ra.lam = lam;
    ra.ysq = ysq; ra.fit = fit; ra.fit_prev = fitp; ra.iters = iters; ra.done = done;
    ra.flags = flags; ra.stop = stop;
    for (int m = 0; m < 3; ++m) { ra.Up[m] = Up3[m]; ra.up_stride[m] = ups[m]; }
    ra.RBp = RBp;
    if (e == cudaSuccess) e = launch_pad_factors(ra, st);
    const bool rows = R <= 16;
    if (e == cudaSuccess) e = cudaMemsetAsync(stop, 0, sizeof(int) * r, st);
    if (e == cudaSuccess && rows && coo_als_persist_supported(R)) {
      // every iteration in one persistent cooperative kernel (k_coo_als.cu)
      e = launch_coo_als_persist(a, ra, gbar, st);
      *launches = 2 * 3 + 9 + 3 + 3 + 3 + 1;
      g_coo_als_kind = 3;
    } else {
      // the per-mode pipeline: the stop test runs on the device; the host looks at the done
      // flags after iterations 3, 6, 10, 15, ... (one small read each) and stops launching once
      // every repetition is done
      int nit = 0, next_check = 3, gap = 3;
      for (int it = 0; it < maxit && e == cudaSuccess; ++it, ++nit) {
        if (rows && it > 0) e = launch_als_rows_commit(ra, st);
        for (int m = 0; m < 3 && e == cudaSuccess; ++m) {
          e = launch_coo_mttkrp(a, m, st);
          if (e == cudaSuccess) e = rows ? launch_als_rows_mode(ra, m, st) : launch_als_solve(*d, m, st);
        }
        int* hd = pinned_done_flags();
        if (hd && rows && e == cudaSuccess && it + 1 == next_check && it + 1 < maxit) {
          next_check += ++gap;
          e = launch_als_rows_commit(ra, st);
          if (e == cudaSuccess) e = cudaMemcpyAsync(hd, done, sizeof(int) * r, cudaMemcpyDeviceToHost, st);
          if (e == cudaSuccess) e = cudaStreamSynchronize(st);
          int nd = 0;
          for (int t = 0; t < r; ++t) nd += hd[t] != 0;
          if (nd == r) { ++nit; break; }
        }
      }
      *launches = 2 * 3 + 9 + 3 + 3 + 3 + (rows ? 16 : 6) * nit;
      g_coo_als_kind = 4;
    }
    if (e != cudaSuccess) {
      set_error(std::string("COO ALS: ") + cudaGetErrorString(e));
      d->nI = -1;
    }
  };
  Bump sz;
  layout(sz, false);
  CK(wsbuf.ensure(sz.off));
  Bump b{wsbuf.as<char>(), 0};
  layout(b, true);
  if (d->nI < 0) return SAMBATEN_E_CUDA;
  return SAMBATEN_OK;
}

__global__ static void two_offsets_kernel(int64_t* off, int64_t n) {
  if (threadIdx.x == 0) { off[0] = 0; off[1] = n; }
}

// Full CP-ALS of the initial COO tensor: the store itself is the single "summary"
// (identity maps p = i, q = j, u = k), Philox init with update_id 0 (R10).
static sambaten_status init_als_coo(sambaten_s* h) {
  DevBuf offb;
  CK(offb.ensure(2 * sizeof(int64_t)));
  two_offsets_kernel<<<1, 32, 0, h->st>>>(offb.as<int64_t>(), h->nnz);
  DenseAls d{};
  int nl = 0;
  if (sambaten_status e = coo_als(h->coo_ws, h->st, h->R, h->ci(), h->cj(), h->ck_(), h->cv(),
                                  offb.as<int64_t>(), h->nnz, (int)h->I, (int)h->J, (int)h->K, 1,
                                  h->A(h->cur), h->B(h->cur), h->C(h->cur), h->seed, 0,
                                  h->opts.init_max_iters, h->opts.init_tol, true, &d, &nl))
    return e;
  lam_to_f32_kernel<<<1, 32, 0, h->st>>>(d.lam, h->R, h->lam(h->cur));
  CK(cudaStreamSynchronize(h->st));
  return SAMBATEN_OK;
}

__global__ static void rep_offsets_kernel(const int64_t* scan, int64_t nb, int r, int64_t* off) {
  const int t = threadIdx.x;
  if (t <= r) off[t] = scan[(int64_t)t * nb];
}

static sambaten_status getrank_coo_one(DevBuf* ws, const int32_t* ti, const int32_t* tj, const int32_t* tk,
                                       const float* tv, int64_t nnz, int I, int J, int K, int R_max, int trials,
                                       uint32_t rep_base, uint64_t seed, int max_iters, double tol,
                                       double threshold, int* R_new, double* cc, cudaStream_t st, int* launches);

// The COO update (Alg. 1 with the sparse store): see the dense update for the step structure.
static sambaten_status update_coo(sambaten_t h, const sambaten_tensor* batch, float* Aout,
                                  float* Bout, float* Cout, float* lamout, sambaten_info* info) {
  const int64_t Kn = batch->dims[2];
  const int64_t bn = batch->nnz;
  if (bn < 0) FAIL(SAMBATEN_E_INVALID, "update: negative nnz");
  if (bn > 0 && (!batch->idx[0] || !batch->idx[1] || !batch->idx[2] || !batch->vals))
    FAIL(SAMBATEN_E_INVALID, "update: NULL COO array");
  const int64_t Ko = h->K;
  if (Ko + Kn > h->Kcap) FAIL(SAMBATEN_E_OOM, "update: mode-3 capacity exceeded (opts.capacity_k)");
  if (h->nnz + bn > h->nnz_cap) FAIL(SAMBATEN_E_OOM, "update: nnz capacity exceeded (opts.capacity)");
  cudaStream_t st = h->st;
  const int R = h->R, r = h->r;
  const uint32_t uid = h->update_id + 1;
  const int64_t nI = sample_n(h->I, h->s[0]), nJ = sample_n(h->J, h->s[1]);
  const int64_t nKs = sample_n(Ko, h->s[2]), nKp = nKs + Kn;
  const int64_t ntot = h->nnz + bn;
  int launches = 0;

  CK(cudaEventRecord(h->ev[0], st));
  // ---- a0: validate + append the batch (not visible until commit), max phi ---------------
  CK(h->misc.ensure(4096));
  unsigned long long* d_maxphi = h->misc.as<unsigned long long>();
  unsigned* d_vflags = reinterpret_cast<unsigned*>(h->misc.as<char>() + 8);
  double* d_relerr = reinterpret_cast<double*>(h->misc.as<char>() + 64);
  CK(cudaMemsetAsync(h->misc.p, 0, 16, st));
  // copy (host or device arrays) into the store capacity, validate there, then shift k
  int32_t* ti = h->ci() + h->nnz;
  int32_t* tj = h->cj() + h->nnz;
  int32_t* tk = h->ck_() + h->nnz;
  float* tv = h->cv() + h->nnz;
  if (bn > 0) {
    CK(cudaMemcpyAsync(ti, batch->idx[0], sizeof(int32_t) * bn, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(tj, batch->idx[1], sizeof(int32_t) * bn, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(tk, batch->idx[2], sizeof(int32_t) * bn, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(tv, batch->vals, sizeof(float) * bn, cudaMemcpyDefault, st));
  }
  CK(launch_coo_validate(ti, tj, tk, tv, bn, h->I, h->J, Kn, d_vflags, st));
  CK(launch_coo_append(ti, tj, tk, tv, bn, (int32_t)Ko, ti, tj, tk, tv, st));
  CK(launch_coo_max_phi(h->cv() + h->nnz, bn, h->opts.moi, d_maxphi, st));
  launches += 3;
  CK(cudaEventRecord(h->ev[1], st));
  // ---- a1: marginals over X_old U X_new (R2, R3) ----------------------------------------
  const size_t marg_bytes = sizeof(int64_t) * (h->I + h->J + h->Kcap);
  CK(h->marg.ensure(marg_bytes));
  int64_t* x1 = h->marg.as<int64_t>();
  int64_t* x2 = x1 + h->I;
  int64_t* x3 = x2 + h->J;
  if (h->opts.incremental_marginals && h->xm_valid) {
    CK(cudaMemcpyAsync(x1, h->xm.p, sizeof(int64_t) * (h->I + h->J + Ko), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(x3 + Ko, 0, sizeof(int64_t) * (h->Kcap - Ko), st));
    CK(coo_marginals(h, h->nnz, ntot, x1, x2, x3, st));
  } else {
    CK(cudaMemsetAsync(x1, 0, marg_bytes, st));
    CK(coo_marginals(h, 0, ntot, x1, x2, x3, st));
  }
  launches += 1;
  CK(cudaEventRecord(h->ev[2], st));
  // ---- a2: sampling ---------------------------------------------------------------------
  int32_t *Is, *Js, *Kp, *locI, *locJ, *locK;
  CK(run_sampling(h, x1, x2, x3, Ko, Kn, nI, nJ, nKs, nKp, uid, &Is, &Js, &Kp, &locI, &locJ, &locK));
  launches += 1;
  CK(cudaEventRecord(h->ev[3], st));
  // ---- a3: gather (membership bitmaps, count, scan, write) ------------------------------
  const int64_t nbk = coo_gather_blocks(ntot);
  Bump gsz;
  auto glayout = [&](Bump& b) {
    b.take<uint32_t>(h->I); b.take<uint32_t>(h->J); b.take<uint32_t>(Ko + Kn);
    b.take<int64_t>((int64_t)r * nbk + 1); b.take<int64_t>((int64_t)r * nbk + 1);
    b.take<int64_t>(scan_ws_elems((int64_t)r * nbk + 1)); b.take<int64_t>(r + 1);
  };
  glayout(gsz);
  CK(h->summ.ensure(gsz.off));
  Bump gb{h->summ.as<char>(), 0};
  uint32_t* mI = gb.take<uint32_t>(h->I);
  uint32_t* mJ = gb.take<uint32_t>(h->J);
  uint32_t* mK = gb.take<uint32_t>(Ko + Kn);
  int64_t* counts = gb.take<int64_t>((int64_t)r * nbk + 1);
  int64_t* goffs = gb.take<int64_t>((int64_t)r * nbk + 1);
  int64_t* gsws = gb.take<int64_t>(scan_ws_elems((int64_t)r * nbk + 1));
  int64_t* d_off = gb.take<int64_t>(r + 1);
  CK(launch_build_mask(locI, h->I, r, mI, h->I, st));
  CK(launch_build_mask(locJ, h->J, r, mJ, h->J, st));
  CK(launch_build_mask(locK, Ko, r, mK, Ko + Kn, st));
  CK(cudaMemsetAsync(counts + (int64_t)r * nbk, 0, sizeof(int64_t), st));
  const CooView Xall = h->coo_view(ntot);
  CK(launch_coo_gather_count(Xall, mI, mJ, mK, r, counts, st));
  CK(exclusive_scan_i64(counts, (int64_t)r * nbk + 1, goffs, gsws, st));
  rep_offsets_kernel<<<1, 64, 0, st>>>(goffs, nbk, r, d_off);
  CK(cudaGetLastError());
  int64_t h_off[kMaxReps + 1];
  CK(cudaMemcpyAsync(h_off, d_off, sizeof(int64_t) * (r + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));   // summary sizes decide the allocation below
  const int64_t nsum = h_off[r];
  h->summ_entries = nsum;
  const size_t sbytes = align256(sizeof(int32_t) * std::max<int64_t>(nsum, 1));
  CK(h->fac.ensure(4 * sbytes + align256(sizeof(float) * r * (nI + nJ + nKp) * R)));
  int32_t* sp = h->fac.as<int32_t>();
  int32_t* sq = reinterpret_cast<int32_t*>(h->fac.as<char>() + sbytes);
  int32_t* su = reinterpret_cast<int32_t*>(h->fac.as<char>() + 2 * sbytes);
  float* sv = reinterpret_cast<float*>(h->fac.as<char>() + 3 * sbytes);
  float* U0 = reinterpret_cast<float*>(h->fac.as<char>() + 4 * sbytes);
  float* U1 = U0 + (size_t)r * nI * R;
  float* U2 = U1 + (size_t)r * nJ * R;
  CK(launch_coo_gather_write(Xall, mI, mJ, mK, locI, locJ, locK, Ko, (int)nKs, r, goffs, sp, sq, su, sv, st));
  launches += 3 + 1 + 3 + 1 + 1;
  CK(cudaEventRecord(h->ev[4], st));
  // ---- a4: batched CP-ALS on the COO summaries ----------------------------------------------
  DenseAls a{};
  int als_launches = 0;
  // GetRank on every sparse summary (Alg. 2; R33), rep numbering as the dense path
  // (trial j of summary s is Philox rep s * trials + j)
  const int* d_rnew = nullptr;
  if (h->opts.getrank) {
    bool deficient = false;
    for (int s = 0; s < r; ++s) {
      if (sambaten_status e = getrank_coo_one(h->grc, sp + h_off[s], sq + h_off[s], su + h_off[s], sv + h_off[s],
                                              h_off[s + 1] - h_off[s], (int)nI, (int)nJ, (int)nKp, R,
                                              h->opts.getrank_trials, (uint32_t)(s * h->opts.getrank_trials),
                                              h->seed, h->opts.als_max_iters, h->opts.als_tol,
                                              h->opts.getrank_threshold, &h->rep_rank[s], nullptr, st,
                                              &als_launches))
        return e;
      deficient |= h->rep_rank[s] < R;
    }
    if (deficient) {
      CK(h->grk.ensure(sizeof(int) * r));
      CK(cudaMemcpyAsync(h->grk.p, h->rep_rank, sizeof(int) * r, cudaMemcpyHostToDevice, st));
      d_rnew = h->grk.as<int>();
    }
  }
  const WarmRows wr{h->A(h->cur), h->B(h->cur), h->C(h->cur), h->lam(h->cur), Is, Js, Kp, (int)nKs};
  if (sambaten_status e = coo_als(h->coo_ws, st, R, sp, sq, su, sv, d_off, nsum, (int)nI, (int)nJ,
                                  (int)nKp, r, U0, U1, U2, h->seed, uid, h->opts.als_max_iters,
                                  h->opts.als_tol, true, &a, &als_launches, 0, 1,
                                  h->opts.warm_start ? &wr : nullptr))
    return e;
  h->als_plan[0] = g_coo_als_kind; h->als_plan[1] = 0; h->als_plan[2] = R; h->als_plan[3] = 0;
  if (d_rnew) {
    // the repetitions GetRank reduced: decomposed alone at R_new (Philox rep s, as in the batch)
    // and written, zero-padded to R columns, over their batch result (R33)
    CK(h->grws.ensure(sizeof(float) * (size_t)(nI + nJ + nKp) * R + 256));
    for (int s = 0; s < r; ++s) {
      if (h->rep_rank[s] >= R) continue;
      const int F = h->rep_rank[s];
      CK(h->grc[3].ensure(2 * sizeof(int64_t)));
      two_offsets_kernel<<<1, 32, 0, st>>>(h->grc[3].as<int64_t>(), h_off[s + 1] - h_off[s]);
      float* V0 = h->grws.as<float>();
      float* V1 = V0 + (size_t)nI * F;
      float* V2 = V1 + (size_t)nJ * F;
      DenseAls b{};
      if (sambaten_status e = coo_als(h->grc[0], st, F, sp + h_off[s], sq + h_off[s], su + h_off[s], sv + h_off[s],
                                      h->grc[3].as<int64_t>(), h_off[s + 1] - h_off[s], (int)nI, (int)nJ, (int)nKp,
                                      1, V0, V1, V2, h->seed, uid, h->opts.als_max_iters, h->opts.als_tol, true,
                                      &b, &als_launches, (uint32_t)s, 1))
        return e;
      CK(launch_rank_pad(b, a, s, st));
      ++als_launches;
    }
  }
  launches += als_launches;
  CK(cudaEventRecord(h->ev[5], st));
  // ---- a5 / a6: match and merge (format independent) -----------------------------------------
  const int b = h->cur, nbuf = 1 - h->cur;
  int* accepted = nullptr;
  CK(run_match_merge(h, a, Is, Js, Kp, locI, locJ, locK, Ko, Kn, nI, nJ, nKs, nKp, &accepted, d_rnew));
  launches += 1 + 4;
  CK(cudaEventRecord(h->ev[7], st));
  // ---- a7: full fit of the new model (optional) ----------------------------------------------
  if (h->opts.full_fit && !getenv("SAMBATEN_FULL_FIT_PASS")) {
    // the new model's exact fit from the previous one's per-component state: the batch's entries,
    // or one full pass when an old row changed (decided on the device)
    CK(fitinc_run_coo(h, h->nnz, ntot, Ko, Ko + Kn, b, nbuf, false, d_relerr, st));
    FitIncWs w;
    CK(fitinc_ws(h, &w));
    h->d_fit_mode = w.mode;
    launches += 6;
  } else if (h->opts.full_fit) {
    CK(h->fitws.ensure(sizeof(double) * coo_fit_ws_doubles(h->I, h->J, h->Kcap)));
    CooView Xn = Xall;
    Xn.K = Ko + Kn;
    CK(launch_coo_fit(Xn, h->lam(nbuf), h->A(nbuf), h->B(nbuf), h->C(nbuf), R, h->fitws.as<double>(),
                      d_relerr, st));
    CK(cudaMemsetAsync(h->fitst(nbuf) + R + 1, 0, sizeof(double), st));   // per-component state not kept
    launches += 3;
  } else {
    CK(cudaMemsetAsync(h->fitst(nbuf) + R + 1, 0, sizeof(double), st));
  }
  CK(cudaEventRecord(h->ev[8], st));
  return finish_update(h, a, accepted, d_maxphi, d_vflags, d_relerr, Ko, Kn, nI, nJ, nKs, nKp, b, nbuf,
                       launches, bn, Aout, Bout, Cout, lamout, info);
}

static sambaten_status update_coo_dist(sambaten_t h, const sambaten_tensor* batch, float* Aout, float* Bout,
                                       float* Cout, float* lamout, sambaten_info* info);
static sambaten_status update_dense_dist(sambaten_t h, const sambaten_tensor* batch, float* Aout,
                                         float* Bout, float* Cout, float* lamout, sambaten_info* info);

extern "C" sambaten_status sambaten_update(sambaten_t h, const sambaten_tensor* batch, float* Aout,
                                           float* Bout, float* Cout, float* lamout,
                                           sambaten_info* info) {
  if (!h) FAIL(SAMBATEN_E_INVALID, "update: NULL handle");
  if (sambaten_status e = check_dense(batch, "update")) return e;
  if (batch->fmt != h->fmt) FAIL(SAMBATEN_E_INVALID, "update: batch format differs from the state's");
  if (batch->dims[0] != h->I || batch->dims[1] != h->J)
    FAIL(SAMBATEN_E_SHAPE, "update: batch I x J differs from the state's (S:68)");
  h->als_plan[0] = -1; h->als_plan[1] = h->als_plan[2] = h->als_plan[3] = 0;   // set by the dense paths
  h->summ_entries = 0;
  h->lag_now = false;
  h->pipe_now = false;
  h->fit_path = 0;
  h->d_fit_mode = nullptr;
  if (h->dist)
    return h->fmt == SAMBATEN_COO ? update_coo_dist(h, batch, Aout, Bout, Cout, lamout, info)
                                  : update_dense_dist(h, batch, Aout, Bout, Cout, lamout, info);
  const int64_t Kn = batch->dims[2];
  if (Kn < 1) FAIL(SAMBATEN_E_EMPTY_BATCH, "update: empty batch (S:275)");
  if (h->fmt == SAMBATEN_COO) return update_coo(h, batch, Aout, Bout, Cout, lamout, info);
  const int64_t Ko = h->K;
  if (Ko + Kn > h->Kcap) FAIL(SAMBATEN_E_OOM, "update: capacity exceeded (opts.capacity)");
  cudaStream_t st = h->st;
  const int R = h->R, r = h->r;
  const uint32_t uid = h->update_id + 1;
  const int64_t nI = sample_n(h->I, h->s[0]), nJ = sample_n(h->J, h->s[1]);
  const int64_t nKs = sample_n(Ko, h->s[2]), nKp = nKs + Kn;
  // R36 pipelined: sample from the committed marginals of X_old (the first update after init
  // computes them once); this update's a1 runs on the side stream, off the critical path
  const bool pipe = h->opts.pipelined;
  if (pipe) {
    CK(compute_committed_marginals(h));
    if (!h->st2) {
      CK(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h->ev_side[0], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_side[1], cudaEventDisableTiming));
    }
    if (!h->ev_pl[0]) {
      CK(cudaEventCreate(&h->ev_pl[0]));
      CK(cudaEventCreate(&h->ev_pl[1]));
    }
  }
  h->pipe_now = pipe;
  const cudaStream_t sa1 = pipe ? h->st2 : st;   // the stream a1 runs on

  CK(cudaEventRecord(h->ev[0], st));
  // ---- a0: ingest into the preallocated capacity (not visible until commit) --------------
  float* dst = h->X.as<float>() + Ko * h->J * h->pitch;
  CK(h->misc.ensure(4096));
  unsigned long long* d_maxphi = h->misc.as<unsigned long long>();
  double* d_relerr = reinterpret_cast<double*>(h->misc.as<char>() + 64);
  CK(cudaMemsetAsync(d_maxphi, 0, 8, st));
  DenseView V = h->view();
  V.K = Ko + Kn;
  const int64_t nb_fl = h->I * h->J * Kn;
  const size_t marg_bytes = sizeof(int64_t) * (h->I + h->J + h->Kcap);
  CK(h->marg.ensure(marg_bytes));
  int64_t* x1 = h->marg.as<int64_t>();
  int64_t* x2 = x1 + h->I;
  int64_t* x3 = x2 + h->J;
  const bool inc = h->opts.incremental_marginals && h->xm_valid;
  const bool dev_batch = is_device_ptr(batch->vals);
  // full_fit = 2: the previous model's fit rides on the marginal pass over the old slices
  DenseView Vold = V;
  Vold.K = Ko;
  const bool lag = h->opts.full_fit == 2 && !inc && Ko > 0 && margfit_supported(Vold, R);
  h->lag_now = lag;
  double* d_fit2 = reinterpret_cast<double*>(h->misc.as<char>() + 112);
  double* d_relerr_prev = d_relerr + 4;
  if (lag) CK(h->fitws.ensure(sizeof(double) * fit_ws_doubles_any(V)));
  auto old_pass = [&]() -> cudaError_t {   // a1 over [0, Ko), with the lag-1 fit when asked
    if (!lag) return marginals_any(V, 0, Ko, h->opts.moi, h->S, x1, x2, x3, sa1, qbits(h), h->phimax_run);
    cudaError_t e = launch_marg_fit_stream(Vold, Ko, h->opts.moi, h->S, qbits(h), h->lam(h->cur), h->A(h->cur),
                                           h->B(h->cur), h->C(h->cur), R, nullptr, x1, x2, x3,
                                           h->fitws.as<double>(), d_fit2, sa1);
    if (e != cudaSuccess) return e;
    return launch_fit_finish(d_fit2, h->lam(h->cur), h->A(h->cur), h->B(h->cur), h->C(h->cur), h->I, h->J, Ko,
                             R, h->fitws.as<double>(), d_relerr_prev, sa1);
  };
  // A host batch crosses PCIe on a side stream while a1 reads the old slices (they do not
  // depend on it); the batch's own marginals follow once it has landed.  (Pipelined updates
  // run the whole a1 on the side stream instead.)
  const bool overlap = !dev_batch && !inc && Ko > 0 && !pipe;
  if (overlap) {
    if (!h->st2) {
      CK(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h->ev_side[0], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_side[1], cudaEventDisableTiming));
    }
    CK(cudaEventRecord(h->ev_side[0], st));
    CK(cudaStreamWaitEvent(h->st2, h->ev_side[0], 0));
    CK(copy_rows(dst, h->pitch * sizeof(float), batch->vals, h->I * sizeof(float),
                        h->I * sizeof(float), h->J * Kn, h->st2));
    CK(cudaEventRecord(h->ev_side[1], h->st2));
    CK(cudaMemsetAsync(x1, 0, marg_bytes, st));
    CK(old_pass());   // a1, old slices (+ the previous model's fit)
    CK(cudaStreamWaitEvent(st, h->ev_side[1], 0));
    CK(launch_max_phi_dense(V, Ko, Kn, h->opts.moi, d_maxphi, st));
  } else if (h->pitch == h->I && nb_fl % 4 == 0 && dev_batch &&
             (((uintptr_t)batch->vals | (uintptr_t)dst) & 15) == 0) {
    // device batch, contiguous store: one pass copies and tracks max |x|
    CK(launch_ingest_dense(batch->vals, dst, nb_fl, h->opts.moi, d_maxphi, st));
  } else {
    CK(copy_rows(dst, h->pitch * sizeof(float), batch->vals, h->I * sizeof(float),
                        h->I * sizeof(float), h->J * Kn, st));
    CK(launch_max_phi_dense(V, Ko, Kn, h->opts.moi, d_maxphi, st));
  }
  CK(cudaEventRecord(h->ev[1], st));
  // ---- a1: marginals over X_old U X_new (R2, R3) ----------------------------------------
  if (pipe) {   // the side stream, after the ingest
    CK(cudaEventRecord(h->ev_side[0], st));
    CK(cudaStreamWaitEvent(sa1, h->ev_side[0], 0));
    CK(cudaEventRecord(h->ev_pl[0], sa1));
  }
  if (overlap) {
    CK(marginals_any(V, Ko, Kn, h->opts.moi, h->S, x1, x2, x3, sa1, qbits(h), 0.0, d_maxphi));   // the batch's slices
  } else if (inc) {
    // committed marginals of X_old plus the batch's contribution (integer sums: bit-identical
    // to the full pass)
    CK(cudaMemcpyAsync(x1, h->xm.p, sizeof(int64_t) * (h->I + h->J + Ko), cudaMemcpyDeviceToDevice, sa1));
    CK(cudaMemsetAsync(x3 + Ko, 0, sizeof(int64_t) * (h->Kcap - Ko), sa1));
    CK(marginals_any(V, Ko, Kn, h->opts.moi, h->S, x1, x2, x3, sa1, qbits(h), 0.0, d_maxphi));
  } else if (lag) {
    CK(cudaMemsetAsync(x1, 0, marg_bytes, sa1));
    CK(old_pass());
    CK(marginals_any(V, Ko, Kn, h->opts.moi, h->S, x1, x2, x3, sa1, qbits(h), 0.0, d_maxphi));   // the batch's slices
  } else {
    CK(cudaMemsetAsync(x1, 0, marg_bytes, sa1));
    CK(marginals_any(V, 0, Ko + Kn, h->opts.moi, h->S, x1, x2, x3, sa1, qbits(h), h->phimax_run, d_maxphi));
  }
  if (pipe) {
    CK(cudaEventRecord(h->ev_pl[1], sa1));
    CK(cudaEventRecord(h->ev_side[1], sa1));   // joined before the commit
  }
  CK(cudaEventRecord(h->ev[2], st));
  // ---- a2: sampling (pipelined: from the committed marginals of X_old, R36) ---------------
  int32_t *Is, *Js, *Kp, *locI, *locJ, *locK;
  {
    const int64_t* sx1 = pipe ? h->xm.as<int64_t>() : x1;
    CK(run_sampling(h, sx1, sx1 + h->I, sx1 + h->I + h->J, Ko, Kn, nI, nJ, nKs, nKp, uid, &Is, &Js, &Kp, &locI,
                    &locJ, &locK));
  }
  CK(cudaEventRecord(h->ev[3], st));
  // ---- a3: gather the r summaries ------------------------------------------------------
  int64_t y_stride = (nKp * nJ * nI + 3) & ~int64_t(3);
  const size_t u0 = align256(sizeof(float) * r * nI * R), u1 = align256(sizeof(float) * r * nJ * R);
  const size_t u2 = align256(sizeof(float) * r * nKp * R);
  CK(h->fac.ensure(u0 + u1 + u2));
  DenseAls a{};
  a.y_stride = y_stride; a.pitch = nI;
  a.nI = (int)nI; a.nJ = (int)nJ; a.nK = (int)nKp; a.R = R; a.r = r;
  a.U[0] = h->fac.as<float>();
  a.U[1] = reinterpret_cast<float*>(h->fac.as<char>() + u0);
  a.U[2] = reinterpret_cast<float*>(h->fac.as<char>() + u0 + u1);
  a.u_stride[0] = nI * R; a.u_stride[1] = nJ * R; a.u_stride[2] = nKp * R;
  a.maxit = h->opts.als_max_iters; a.tol = h->opts.als_tol;
  a.Yt = reinterpret_cast<const float*>(1);   // planning only needs "transpose available"
  ClusterPlan cpl;
  const bool use_cluster = cluster_plan(h, a, &cpl);
  set_plan_report(h, use_cluster, cpl, R);
  h->summ_entries = (int64_t)r * nI * nJ * nKp;
  const int pI = use_cluster ? cluster_pitch((int)nI) : (int)nI;
  const int pJ = use_cluster ? cluster_pitch((int)nJ) : (int)nJ;
  if (use_cluster) y_stride = (nKp * std::max<int64_t>(nJ * pI, nI * pJ) + 3) & ~int64_t(3);
  a.y_stride = y_stride;
  a.pitch = pI;
  CK(h->summ.ensure(sizeof(float) * r * y_stride * (use_cluster ? 2 : 1)));
  float* Y = h->summ.as<float>();
  float* Yt = use_cluster ? Y + r * y_stride : nullptr;
  a.Y = Y;
  a.Yt = Yt;
  CK(h->gord.ensure(sizeof(int32_t) * r * nKp));
  CK(launch_gather_dense(V, Is, Js, Kp, (int)nI, (int)nJ, (int)nKp, r, nI, nJ, nKp, Y, y_stride, st,
                         Yt, pI, pJ, h->gord.as<int32_t>(), Ko + Kn));
  CK(cudaEventRecord(h->ev[4], st));
  // ---- a4: batched CP-ALS ---------------------------------------------------------------
  const size_t ws_als = align256(dense_als_workspace(&a));
  const size_t ws_d = use_cluster ? als_cluster_dscratch_bytes(a, cpl) : 0;
  CK(h->als.ensure(ws_als + ws_d));
  CK(dense_als_bind_workspace(&a, h->als.p));
  int als_launches = 0;
  // GetRank on every summary (Alg. 2; R33): a rep whose summary shows fewer than R
  // consistent components is decomposed at that rank and matches / merges only those
  const int* d_rnew = nullptr;
  if (h->opts.getrank) {
    CK(getrank_batch(Y, y_stride, pI, (int)nI, (int)nJ, (int)nKp, r, R, h->opts.getrank_trials, h->seed,
                     h->opts.als_max_iters, h->opts.als_tol, h->opts.getrank_threshold, h->grws, st,
                     h->rep_rank, nullptr, &als_launches));
    bool deficient = false;
    for (int rho = 0; rho < r; ++rho) deficient |= h->rep_rank[rho] < R;
    if (deficient) {
      CK(h->grk.ensure(sizeof(int) * r));
      CK(cudaMemcpyAsync(h->grk.p, h->rep_rank, sizeof(int) * r, cudaMemcpyHostToDevice, st));
      d_rnew = h->grk.as<int>();
    }
  }
  if (d_rnew) {
    h->als_plan[0] = -1;   // per-rep ranks: the multi-kernel ALS at each rep's R_new
    CK(rank_als(h, a, h->rep_rank, uid, st, &als_launches));
  } else if (use_cluster) {
    CK(launch_als_init_factors(a, h->seed, uid, 0, st));
    if (h->opts.warm_start) {   // R34: the model's rows replace the Philox point
      CK(launch_warm_init(a, h->A(h->cur), h->B(h->cur), h->C(h->cur), h->lam(h->cur), Is, Js, Kp, (int)nKs, st));
      ++als_launches;
    }
    CK(run_als_cluster(a, cpl, reinterpret_cast<float*>(h->als.as<char>() + ws_als), st));
    if (getenv("SAMBATEN_DEBUG")) als_phase_dump();
    als_launches += 2;
  } else {
    if (h->opts.warm_start) {
      // R34: the model's rows replace the Philox point BEFORE the Grams are formed (the first
      // sweep's normal equations must see the warm factors)
      CK(launch_als_init_factors(a, h->seed, uid, 0, st));
      CK(launch_warm_init(a, h->A(h->cur), h->B(h->cur), h->C(h->cur), h->lam(h->cur), Is, Js, Kp, (int)nKs, st));
      CK(launch_als_gram(a, st));
      CK(launch_sumsq_dense(a.Y, a.y_stride, (int64_t)a.nK * a.nJ, a.pitch, a.nI, a.r, a.ysq, st));
      ++als_launches;
    } else {
      CK(launch_als_init(a, h->seed, uid, 0, true, st));
    }
    CK(run_dense_als(a, st));
    als_launches += 4 + 7 * a.maxit;
  }
  CK(cudaEventRecord(h->ev[5], st));
  // ---- a5 / a6: match and merge -----------------------------------------------------------
  const int b = h->cur, nb = 1 - h->cur;
  int* accepted = nullptr;
  CK(run_match_merge(h, a, Is, Js, Kp, locI, locJ, locK, Ko, Kn, nI, nJ, nKs, nKp, &accepted, d_rnew));
  CK(cudaEventRecord(h->ev[7], st));
  // ---- a7: full fit of the new model (optional; with full_fit = 2 it rides on the next a1) --
  const bool fit_now = h->opts.full_fit == 1 || (h->opts.full_fit == 2 && !lag);
  if (fit_now && h->opts.full_fit == 1 && !getenv("SAMBATEN_FULL_FIT_PASS") && fitrows_supported(h->pitch, R)) {
    // the new model's exact fit kept up to date from the previous one (k_fitinc.cu): the batch's
    // slices plus the rows the merge changed, or one full pass when the plan says so
    CK(fitinc_run(h, V, Ko, Ko, Ko + Kn, b, nb, false, nullptr, true, d_relerr, st));
    FitIncWs w;
    CK(fitinc_ws(h, &w));
    h->d_fit_mode = w.mode;
  } else if (fit_now) {
    // separate workspace: reallocating misc here would lose the max-phi word written in a0
    const size_t need = sizeof(double) * fit_ws_doubles_any(V);
    CK(h->fitws.ensure(need));
    CK(fit_any(V, h->lam(nb), h->A(nb), h->B(nb), h->C(nb), R, h->fitws.as<double>(), d_relerr, st));
    CK(cudaMemsetAsync(h->fitst(nb) + R + 1, 0, sizeof(double), st));   // per-component state not kept
  } else {
    CK(cudaMemsetAsync(h->fitst(nb) + R + 1, 0, sizeof(double), st));
  }
  CK(cudaEventRecord(h->ev[8], st));
  // a0 ingest or max_phi (+ the old-slice marginal pass when a host batch overlaps its copy),
  // a1 marginals (lag: fused pass + pair sum + 2 Gram kernels + finish, then the batch's
  // marginals), a2 sample, a3 gather, a4 ALS, a5 match partial + match, a6 merge, a7 fit + two
  // Gram kernels + combine
  const int launches = 1 + (overlap ? 1 : 0) + 1 + (lag ? 5 : 0) + 1 + 1 + als_launches + 2 + 1 + (fit_now ? 4 : 0);
  if (pipe) CK(cudaStreamWaitEvent(st, h->ev_side[1], 0));   // this update's marginals, committed for the next
  return finish_update(h, a, accepted, d_maxphi, nullptr, d_relerr, Ko, Kn, nI, nJ, nKs, nKp, b, nb,
                       launches, 0, Aout, Bout, Cout, lamout, info);
}

#include "capi_dist.inc"

DenseView sambaten_s::view_local() const {
  return DenseView{X.as<float>(), I, J, dist ? dist->K_local : K, pitch};
}

extern "C" sambaten_status sambaten_get_factors(sambaten_t h, const float** A, const float** B,
                                                const float** C, const float** lambda,
                                                int64_t dims[3], int* R) {
  if (!h) FAIL(SAMBATEN_E_INVALID, "get_factors: NULL handle");
  if (A) *A = h->A(h->cur);
  if (B) *B = h->B(h->cur);
  if (C) *C = h->C(h->cur);
  if (lambda) *lambda = h->lam(h->cur);
  if (dims) { dims[0] = h->I; dims[1] = h->J; dims[2] = h->K; }
  if (R) *R = h->R;
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_copy_factors(sambaten_t h, float* A, float* B, float* C,
                                                 float* lambda) {
  if (!h) FAIL(SAMBATEN_E_INVALID, "copy_factors: NULL handle");
  const int b = h->cur, R = h->R;
  if (A) CK(cudaMemcpyAsync(A, h->A(b), sizeof(float) * h->I * R, cudaMemcpyDefault, h->st));
  if (B) CK(cudaMemcpyAsync(B, h->B(b), sizeof(float) * h->J * R, cudaMemcpyDefault, h->st));
  if (C) CK(cudaMemcpyAsync(C, h->C(b), sizeof(float) * h->K * R, cudaMemcpyDefault, h->st));
  if (lambda) CK(cudaMemcpyAsync(lambda, h->lam(b), sizeof(float) * R, cudaMemcpyDefault, h->st));
  CK(cudaStreamSynchronize(h->st));
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_last_samples(sambaten_t h, int32_t* Is, int32_t* Js,
                                                 int32_t* Ks, int64_t n_out[3]) {
  if (!h) FAIL(SAMBATEN_E_INVALID, "last_samples: NULL handle");
  if (h->update_id == 0) FAIL(SAMBATEN_E_INVALID, "last_samples: no update yet");
  const int64_t nI = h->last_n[0], nJ = h->last_n[1], nKs = h->last_n[2], nKp = h->last_nKp;
  const int r = h->r;
  const size_t is_b = align256(sizeof(int32_t) * r * nI), js_b = align256(sizeof(int32_t) * r * nJ);
  const char* sp = h->samp.as<char>();
  if (Is) CK(cudaMemcpyAsync(Is, sp, sizeof(int32_t) * r * nI, cudaMemcpyDefault, h->st));
  if (Js) CK(cudaMemcpyAsync(Js, sp + is_b, sizeof(int32_t) * r * nJ, cudaMemcpyDefault, h->st));
  if (Ks)
    CK(cudaMemcpy2DAsync(Ks, sizeof(int32_t) * nKs, sp + is_b + js_b, sizeof(int32_t) * nKp,
                         sizeof(int32_t) * nKs, r, cudaMemcpyDefault, h->st));
  if (n_out) { n_out[0] = nI; n_out[1] = nJ; n_out[2] = nKs; }
  CK(cudaStreamSynchronize(h->st));
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_relative_error(sambaten_t h, double* relerr) {
  if (!h || !relerr) FAIL(SAMBATEN_E_INVALID, "relative_error: NULL argument");
  if (h->fmt == SAMBATEN_COO) {
    DevBuf ws;
    CK(ws.ensure(sizeof(double) * (coo_fit_ws_doubles(h->I, h->J, h->Kcap) + 8)));
    double* d = ws.as<double>();
    CK(launch_coo_fit(h->coo_view(h->nnz), h->lam(h->cur), h->A(h->cur), h->B(h->cur), h->C(h->cur),
                      h->R, d + 8, d, h->st));
    CK(cudaMemcpyAsync(relerr, d, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return SAMBATEN_OK;
  }
  DenseView V = h->view();
  DevBuf ws;
  CK(ws.ensure(sizeof(double) * (fit_ws_doubles_any(V) + 8)));
  double* d = ws.as<double>();
  CK(fit_any(V, h->lam(h->cur), h->A(h->cur), h->B(h->cur), h->C(h->cur), h->R, d + 8, d, h->st));
  CK(cudaMemcpyAsync(relerr, d, 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  ws.release();
  return SAMBATEN_OK;
}

// Committed marginals of the current tensor for the incremental a1 (one full pass; single-GPU
// handles -- a sharded handle computes them in its first update).
static cudaError_t compute_committed_marginals(sambaten_s* h) {
  if (h->dist || h->xm_valid || !(h->opts.incremental_marginals || h->opts.pipelined)) return cudaSuccess;
  const size_t xb = sizeof(int64_t) * (h->I + h->J + h->Kcap);
  cudaError_t e = h->xm.ensure(xb);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->xm.p, 0, xb, h->st);
  int64_t* x1 = h->xm.as<int64_t>();
  if (e == cudaSuccess) {
    if (h->fmt == SAMBATEN_DENSE)
      e = marginals_any(h->view(), 0, h->K, h->opts.moi, h->S, x1, x1 + h->I, x1 + h->I + h->J, h->st, qbits(h),
                        h->phimax_run);
    else
      e = coo_marginals(h, 0, h->nnz, x1, x1 + h->I, x1 + h->I + h->J, h->st);
  }
  if (e == cudaSuccess) h->xm_valid = true;
  return e;
}

extern "C" sambaten_status sambaten_checkpoint(sambaten_t h) {
  if (!h) FAIL(SAMBATEN_E_INVALID, "checkpoint: NULL handle");
  CK(compute_committed_marginals(h));
  CK(h->ck.ensure(h->model_floats() * sizeof(float)));
  CK(cudaMemcpyAsync(h->ck.p, h->model[h->cur].p, h->model_floats() * sizeof(float),
                     cudaMemcpyDeviceToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  h->K_ck = h->K;
  h->nnz_ck = h->nnz;
  h->xm_ck_valid = h->xm_valid;
  if (h->xm_valid) {
    const size_t xb = sizeof(int64_t) * (h->I + h->J + h->K);
    CK(h->xm_ck.ensure(xb));
    CK(cudaMemcpyAsync(h->xm_ck.p, h->xm.p, xb, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaStreamSynchronize(h->st));
  }
  if (h->dist) h->dist->K_local_ck = h->dist->K_local;
  h->uid_ck = h->update_id;
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_restore(sambaten_t h) {
  if (!h) FAIL(SAMBATEN_E_INVALID, "restore: NULL handle");
  if (h->K_ck < 0) FAIL(SAMBATEN_E_INVALID, "restore: no checkpoint");
  CK(cudaMemcpyAsync(h->model[h->cur].p, h->ck.p, h->model_floats() * sizeof(float),
                     cudaMemcpyDeviceToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  h->K = h->K_ck;
  h->nnz = h->nnz_ck;
  h->xm_valid = h->xm_ck_valid;
  if (h->xm_valid) {
    CK(cudaMemcpyAsync(h->xm.p, h->xm_ck.p, sizeof(int64_t) * (h->I + h->J + h->K), cudaMemcpyDeviceToDevice,
                       h->st));
    CK(cudaStreamSynchronize(h->st));
  }
  if (h->dist) {
    h->dist->K_local = h->dist->K_local_ck;
    h->dist->kmap_h.resize(h->dist->K_local);
    for (int64_t k = h->K; k < (int64_t)h->dist->owner.size(); ++k) { h->dist->owner[k] = -1; h->dist->kloc[k] = -1; }
  }
  h->update_id = h->uid_ck;
  return SAMBATEN_OK;
}

// ---------------------------------------------------------------------------------------
// stateless primitives
// ---------------------------------------------------------------------------------------
static DenseView user_view(const sambaten_tensor* X) {
  return DenseView{X->vals, X->dims[0], X->dims[1], X->dims[2], X->dims[0]};
}

extern "C" sambaten_status sambaten_marginals(const sambaten_tensor* X, int moi, int scale_exp,
                                              int64_t* x1, int64_t* x2, int64_t* x3, void* stream) {
  if (sambaten_status e = check_dense(X, "marginals")) return e;
  if (!x1 || !x2 || !x3) FAIL(SAMBATEN_E_INVALID, "marginals: NULL output");
  if (moi != 0 && moi != 1) FAIL(SAMBATEN_E_INVALID, "marginals: moi must be 0 or 1");
  cudaStream_t st = stream_of(stream);
  CK(cudaMemsetAsync(x1, 0, sizeof(int64_t) * X->dims[0], st));
  CK(cudaMemsetAsync(x2, 0, sizeof(int64_t) * X->dims[1], st));
  CK(cudaMemsetAsync(x3, 0, sizeof(int64_t) * X->dims[2], st));
  if (X->fmt == SAMBATEN_DENSE) {
    if (X->dims[0] > 4096) FAIL(SAMBATEN_E_INVALID, "marginals: dense I > 4096 not supported");
    // SAMBATEN_MARG_QB (test hook): the caller asserts every q <= 2^qb (qb <= 27: 32-bit kernel)
    // SAMBATEN_MARG_PHIMAX (test hook): ... and every phi <= this bound (q < 2^22: FMA rounding)
    const char* qe = getenv("SAMBATEN_MARG_QB");
    const char* pe = getenv("SAMBATEN_MARG_PHIMAX");
    CK(marginals_any(user_view(X), 0, X->dims[2], moi, scale_exp, x1, x2, x3, st, qe ? atoi(qe) : 64,
                     pe ? atof(pe) : 1e300));
  } else {
    const int nrep = marg_coo_replicas(X->nnz, X->dims[0], X->dims[1]);
    int64_t* rws = nullptr;
    if (nrep >= 2) CK(cudaMallocAsync(reinterpret_cast<void**>(&rws), sizeof(int64_t) * (size_t)nrep *
                                      (X->dims[0] + X->dims[1]), st));
    const cudaError_t e = launch_marginals_coo(X->idx[0], X->idx[1], X->idx[2], X->vals, X->nnz, moi, scale_exp,
                                               x1, x2, x3, st, X->dims[0], X->dims[1], rws, nrep);
    if (rws) CK(cudaFreeAsync(rws, st));
    CK(e);
  }
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_sample(const int64_t* w, int64_t n, int64_t n_s, uint64_t seed,
                                           uint32_t update_id, uint32_t rep, uint32_t mode,
                                           int32_t* out_idx, void* stream) {
  if (n < 0 || n_s < 0 || n_s > n) FAIL(SAMBATEN_E_INVALID, "sample: need 0 <= n_s <= n");
  if (n > 0 && (!w || (n_s > 0 && !out_idx))) FAIL(SAMBATEN_E_INVALID, "sample: NULL pointer");
  if (n >= (int64_t)1 << 31) FAIL(SAMBATEN_E_INVALID, "sample: n >= 2^31");
  if (n == 0) return SAMBATEN_OK;
  cudaStream_t st = stream_of(stream);
  const size_t bytes = align256(sizeof(SampleSeg)) + sizeof(uint64_t) * n;
  void* p = nullptr;
  CK(cudaMallocAsync(&p, bytes, st));
  SampleSeg g{};
  g.w = w; g.n = n; g.ns = n_s; g.out = out_idx; g.loc = nullptr;
  g.keys = reinterpret_cast<uint64_t*>(static_cast<char*>(p) + align256(sizeof(SampleSeg)));
  g.rep = rep; g.mode = mode; g.kp_tail = nullptr; g.tail0 = 0; g.ntail = 0;
  CK(cudaMemcpyAsync(p, &g, sizeof(g), cudaMemcpyHostToDevice, st));
  CK(launch_sample(static_cast<SampleSeg*>(p), 1, seed, update_id, st));
  CK(cudaStreamSynchronize(st));   // g lives on this stack frame
  CK(cudaFreeAsync(p, st));
  return SAMBATEN_OK;
}

__global__ static void loc_from_list_kernel(const int32_t* list, int64_t n, int64_t nall, int32_t* loc,
                                            unsigned* bad) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = list[t];
    if (x < 0 || x >= nall) { atomicOr(bad, 1u); continue; }
    loc[x] = (int32_t)t;
  }
}

__global__ static void store_i64_kernel(const int64_t* src, int64_t* dst) {
  if (threadIdx.x == 0) *dst = *src;
}

extern "C" sambaten_status sambaten_gather(const sambaten_tensor* X, const int32_t* Is, int64_t nI,
                                           const int32_t* Js, int64_t nJ, const int32_t* Ks,
                                           int64_t nK, float* out_dense, int32_t* oi, int32_t* oj,
                                           int32_t* ok, float* ov, int64_t out_cap,
                                           int64_t* out_nnz, void* stream) {
  if (sambaten_status e = check_dense(X, "gather")) return e;
  if (nI < 0 || nJ < 0 || nK < 0) FAIL(SAMBATEN_E_INVALID, "gather: negative size");
  cudaStream_t st = stream_of(stream);
  if (X->fmt == SAMBATEN_DENSE) {
    if (!out_dense) FAIL(SAMBATEN_E_INVALID, "gather: NULL output");
    CK(launch_gather_dense(user_view(X), Is, Js, Ks, (int)nI, (int)nJ, (int)nK, 1, nI, nJ, nK,
                           out_dense, nK * nJ * nI, st));
    return SAMBATEN_OK;
  }
  // COO: membership bitmaps of the three index lists (r = 1), count, scan, write
  if (!oi || !oj || !ok || !ov || !out_nnz) FAIL(SAMBATEN_E_INVALID, "gather: NULL COO output");
  const int64_t I = X->dims[0], J = X->dims[1], K = X->dims[2], n = X->nnz;
  const CooView V{X->idx[0], X->idx[1], X->idx[2], X->vals, n, I, J, K};
  const int64_t nb = coo_gather_blocks(n);
  DevBuf ws;
  Bump sz;
  auto lay = [&](Bump& b) {
    int32_t* lI = b.take<int32_t>(I); int32_t* lJ = b.take<int32_t>(J); int32_t* lK = b.take<int32_t>(K);
    uint32_t* mI = b.take<uint32_t>(I); uint32_t* mJ = b.take<uint32_t>(J); uint32_t* mK = b.take<uint32_t>(K);
    int64_t* cnt = b.take<int64_t>(nb + 1); int64_t* off = b.take<int64_t>(nb + 1);
    int64_t* sws = b.take<int64_t>(scan_ws_elems(nb + 1));
    unsigned* bad = b.take<unsigned>(1);
    return std::make_tuple(lI, lJ, lK, mI, mJ, mK, cnt, off, sws, bad);
  };
  lay(sz);
  CK(ws.ensure(sz.off));
  Bump b{ws.as<char>(), 0};
  auto [lI, lJ, lK, mI, mJ, mK, cnt, off, sws, bad] = lay(b);
  CK(cudaMemsetAsync(lI, 0xff, sizeof(int32_t) * I, st));
  CK(cudaMemsetAsync(lJ, 0xff, sizeof(int32_t) * J, st));
  CK(cudaMemsetAsync(lK, 0xff, sizeof(int32_t) * K, st));
  CK(cudaMemsetAsync(bad, 0, sizeof(unsigned), st));
  CK(cudaMemsetAsync(cnt + nb, 0, sizeof(int64_t), st));
  if (nI) loc_from_list_kernel<<<64, 256, 0, st>>>(Is, nI, I, lI, bad);
  if (nJ) loc_from_list_kernel<<<64, 256, 0, st>>>(Js, nJ, J, lJ, bad);
  if (nK) loc_from_list_kernel<<<64, 256, 0, st>>>(Ks, nK, K, lK, bad);
  CK(launch_build_mask(lI, I, 1, mI, I, st));
  CK(launch_build_mask(lJ, J, 1, mJ, J, st));
  CK(launch_build_mask(lK, K, 1, mK, K, st));
  CK(launch_coo_gather_count(V, mI, mJ, mK, 1, cnt, st));
  CK(exclusive_scan_i64(cnt, nb + 1, off, sws, st));
  int64_t tot = 0;
  unsigned hbad = 0;
  CK(cudaMemcpyAsync(&tot, off + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hbad, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  store_i64_kernel<<<1, 32, 0, st>>>(off + nb, out_nnz);
  if (hbad) FAIL(SAMBATEN_E_INDEX_RANGE, "gather: sampled index outside its mode");
  if (tot > out_cap) {
    CK(cudaStreamSynchronize(st));
    FAIL(SAMBATEN_E_INVALID, "gather: out_cap smaller than the summary's nnz (*out_nnz has the size)");
  }
  CK(launch_coo_gather_write(V, mI, mJ, mK, lI, lJ, lK, K, (int)nK, 1, off, oi, oj, ok, ov, st));
  CK(cudaStreamSynchronize(st));   // ws is released on return
  return SAMBATEN_OK;
}

__global__ static void f64_to_f32_kernel(const double* in, int64_t n, float* out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (float)in[t];
}

// MTTKRP of one COO tensor (r = 1): stable sort by the mode's index (modes 0, 1), row pointers,
// warp-per-row sums; fp64 result rounded to fp32.
static sambaten_status coo_mttkrp_single(const sambaten_tensor* X, const float* U0, const float* U1,
                                         const float* U2, int R, int mode, float* M, cudaStream_t st) {
  const int64_t I = X->dims[0], J = X->dims[1], K = X->dims[2], n = X->nnz;
  const int64_t rows = mode == 0 ? I : mode == 1 ? J : K;
  const int kb = bits_for(rows);
  const int64_t nn = std::max<int64_t>(n, 1);
  DevBuf ws;
  Bump sz;
  const size_t pe = coo_plan_elems(rows, nn);
  auto lay = [&](Bump& b) {
    uint32_t* keys = b.take<uint32_t>(nn); int32_t* perm = b.take<int32_t>(nn);
    uint32_t* wk = b.take<uint32_t>(nn); int32_t* wv = b.take<int32_t>(nn);
    int64_t* hist = b.take<int64_t>(radix_ws_elems(nn)); int64_t* offs = b.take<int64_t>(radix_ws_elems(nn));
    int64_t* sws = b.take<int64_t>(std::max(scan_ws_elems(radix_ws_elems(nn)), scan_ws_elems(rows + 1)));
    int64_t* cnt = b.take<int64_t>(rows + 1); int64_t* ptr = b.take<int64_t>(rows + 1);
    int64_t* off = b.take<int64_t>(2); double* Md = b.take<double>(rows * R); int* done = b.take<int>(1);
    CooModePlan pl{};
    pl.nrow = rows; pl.n = n;
    pl.pstart = b.take<int64_t>(rows + 1); pl.pb = b.take<int64_t>(pe); pl.prow = b.take<int32_t>(pe);
    pl.partial = b.take<double>(pe * R);
    pl.sa = b.take<int32_t>(nn); pl.sb = b.take<int32_t>(nn); pl.sv = b.take<float>(nn);
    pl.ptr = ptr;
    return std::make_tuple(keys, perm, wk, wv, hist, offs, sws, cnt, ptr, off, Md, done, pl);
  };
  lay(sz);
  CK(ws.ensure(sz.off));
  Bump b{ws.as<char>(), 0};
  auto [keys, perm, wk, wv, hist, offs, sws, cnt, ptr, off, Md, done, pl] = lay(b);
  two_offsets_kernel<<<1, 32, 0, st>>>(off, n);
  CK(cudaMemsetAsync(done, 0, sizeof(int), st));
  const int32_t* idx = X->idx[mode];
  if (mode < 2) CK(coo_sort_by_index(idx, off, 1, kb, n, keys, perm, wk, wv, hist, offs, sws, st));
  else CK(coo_make_keys(idx, off, 1, kb, n, keys, st));
  CK(coo_row_pointers(keys, n, kb, 1, rows, cnt, ptr, sws, st));
  const int oa = mode == 0 ? 1 : 0, ob = mode == 2 ? 1 : 2;
  if (mode == 2) { pl.sa = X->idx[0]; pl.sb = X->idx[1]; pl.sv = X->vals; }
  CK(coo_build_plan(pl, mode < 2 ? perm : nullptr, X->idx[oa], X->idx[ob], X->vals, n, cnt, sws, st));
  CooAls a{};
  a.nI = (int)I; a.nJ = (int)J; a.nK = (int)K; a.R = R; a.r = 1;
  a.RB = R <= 4 ? 4 : R <= 8 ? 8 : R <= 12 ? 12 : R <= 16 ? 16 : R <= 24 ? 24 : 32;
  a.plan[mode] = pl;
  a.U[0] = const_cast<float*>(U0); a.U[1] = const_cast<float*>(U1); a.U[2] = const_cast<float*>(U2);
  a.u_stride[0] = a.u_stride[1] = a.u_stride[2] = 0;
  a.M[mode] = Md; a.m_stride[mode] = rows * R;
  a.done = done;
  CK(launch_coo_mttkrp(a, mode, st));
  f64_to_f32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * R, 256), 4096), 256, 0, st>>>(Md, rows * R, M);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));   // ws is released on return
  return SAMBATEN_OK;
}

static sambaten_status single_als_setup(const sambaten_tensor* X, int R, float* U0, float* U1,
                                        float* U2, DenseAls* a) {
  if (sambaten_status e = check_dense(X, "mttkrp/cp_als")) return e;
  if (R < 1 || R > kMaxR) FAIL(SAMBATEN_E_INVALID, "R must be in [1, 32]");
  if (X->fmt != SAMBATEN_DENSE) FAIL(SAMBATEN_E_INVALID, "COO MTTKRP not available in this build");
  *a = DenseAls{};
  a->Y = X->vals; a->y_stride = 0; a->pitch = X->dims[0];
  a->nI = (int)X->dims[0]; a->nJ = (int)X->dims[1]; a->nK = (int)X->dims[2]; a->R = R; a->r = 1;
  a->U[0] = U0; a->U[1] = U1; a->U[2] = U2;
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_mttkrp(const sambaten_tensor* X, const float* U0, const float* U1,
                                           const float* U2, int R, int mode, float* M, void* stream) {
  if (mode < 0 || mode > 2) FAIL(SAMBATEN_E_INVALID, "mttkrp: mode must be 0, 1 or 2");
  if (!M) FAIL(SAMBATEN_E_INVALID, "mttkrp: NULL output");
  if (X && X->fmt == SAMBATEN_COO) {
    if (R < 1 || R > kMaxR) FAIL(SAMBATEN_E_INVALID, "R must be in [1, 32]");
    return coo_mttkrp_single(X, U0, U1, U2, R, mode, M, stream_of(stream));
  }
  DenseAls a;
  if (sambaten_status e = single_als_setup(X, R, (float*)U0, (float*)U1, (float*)U2, &a)) return e;
  cudaStream_t st = stream_of(stream);
  void* ws = nullptr;
  CK(cudaMallocAsync(&ws, dense_als_workspace(&a), st));
  CK(dense_als_bind_workspace(&a, ws));
  CK(dense_mttkrp_single(a, mode, M, st));
  CK(cudaFreeAsync(ws, st));
  return SAMBATEN_OK;
}

__global__ static void copy_als_out_kernel(const double* lam, const double* fit, const int* iters,
                                           int R, double* lam_out, double* fit_out, int* iters_out) {
  if (threadIdx.x < R && lam_out) lam_out[threadIdx.x] = lam[threadIdx.x];
  if (threadIdx.x == 0) {
    if (fit_out) *fit_out = *fit;
    if (iters_out) *iters_out = *iters;
  }
}

extern "C" sambaten_status sambaten_cp_als(const sambaten_tensor* X, int R, float* U0, float* U1,
                                           float* U2, double* lambda_out, int max_iters, double tol,
                                           double* fit_out, int32_t* iters_out, void* stream) {
  if (max_iters < 1) FAIL(SAMBATEN_E_INVALID, "cp_als: max_iters >= 1");
  if (X && X->fmt == SAMBATEN_COO) {
    if (R < 1 || R > kMaxR) FAIL(SAMBATEN_E_INVALID, "R must be in [1, 32]");
    cudaStream_t st = stream_of(stream);
    DevBuf ws, offb;
    CK(offb.ensure(2 * sizeof(int64_t)));
    two_offsets_kernel<<<1, 32, 0, st>>>(offb.as<int64_t>(), X->nnz);
    DenseAls d{};
    int nl = 0;
    if (sambaten_status e = coo_als(ws, st, R, X->idx[0], X->idx[1], X->idx[2], X->vals, offb.as<int64_t>(),
                                    X->nnz, (int)X->dims[0], (int)X->dims[1], (int)X->dims[2], 1, U0, U1,
                                    U2, 0, 0, max_iters, tol, false, &d, &nl))
      return e;
    copy_als_out_kernel<<<1, 32, 0, st>>>(d.lam, d.fit, d.iters, R, lambda_out, fit_out, iters_out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return SAMBATEN_OK;
  }
  DenseAls a;
  if (sambaten_status e = single_als_setup(X, R, U0, U1, U2, &a)) return e;
  a.maxit = max_iters; a.tol = tol;
  cudaStream_t st = stream_of(stream);
  void* ws = nullptr;
  CK(cudaMallocAsync(&ws, dense_als_workspace(&a), st));
  CK(dense_als_bind_workspace(&a, ws));
  CK(launch_als_init(a, 0, 0, 0, false, st));
  CK(run_dense_als(a, st));
  copy_als_out_kernel<<<1, 32, 0, st>>>(a.lam, a.fit, a.iters, R, lambda_out, fit_out, iters_out);
  CK(cudaGetLastError());
  CK(cudaFreeAsync(ws, st));
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_als_plan(int nI, int nJ, int nK, int R, int r, int plan[4]) {
  if (nI < 1 || nJ < 1 || nK < 1 || R < 1 || R > kMaxR || r < 1 || r > kMaxReps || !plan)
    FAIL(SAMBATEN_E_INVALID, "als_plan: bad argument");
  DenseAls a{};
  a.nI = nI; a.nJ = nJ; a.nK = nK; a.R = R; a.r = r;
  a.Yt = reinterpret_cast<float*>(16);   // the plan only needs to know a transposed layout exists
  ClusterPlan pl{};
  const bool ok = r >= 2 && !getenv("SAMBATEN_NO_CLUSTER_ALS") && plan_als_cluster(a, &pl);
  cudaGetLastError();
  plan[0] = ok ? (pl.grid ? 2 : 1) : 0;
  plan[1] = ok ? pl.CS : 1;
  plan[2] = ok ? pl.RB : R;
  plan[3] = ok ? pl.dsh : 0;
  return SAMBATEN_OK;
}

// GetRank (Alg. 2; R29-R31) on one canonical COO tensor (device arrays; dims I x J x
// K): each candidate rank F and trial j runs the COO ALS (r = 1, Philox update_id 0x47520000 + F,
// rep rep_base + j: R30, the dense path's numbering) and the sparse CorConDia rates it;
// R_new = the largest F whose best trial reaches `threshold` (R31), else 1.  Synchronises st.
// ws: [0] ALS workspace, [1] factors, [2] CorConDia workspace + ratings, [3] offsets.
static sambaten_status getrank_coo_one(DevBuf* ws, const int32_t* ti, const int32_t* tj, const int32_t* tk,
                                       const float* tv, int64_t nnz, int I, int J, int K, int R_max, int trials,
                                       uint32_t rep_base, uint64_t seed, int max_iters, double tol,
                                       double threshold, int* R_new, double* cc, cudaStream_t st, int* launches) {
  constexpr uint32_t kGetRankId = 0x47520000u;   // R30
  CK(ws[3].ensure(2 * sizeof(int64_t)));
  two_offsets_kernel<<<1, 32, 0, st>>>(ws[3].as<int64_t>(), nnz);
  CK(ws[1].ensure(sizeof(float) * ((size_t)I + J + K) * R_max + 256));
  const size_t ccn = corcondia_coo_ws_doubles(I, J, K, R_max, 1);
  CK(ws[2].ensure(sizeof(double) * (ccn + (size_t)R_max * trials + 8)));
  double* ccws = ws[2].as<double>();
  double* ccd = ccws + ccn;
  for (int F = 1; F <= R_max; ++F) {
    float* U0 = ws[1].as<float>();
    float* U1 = U0 + (size_t)I * F;
    float* U2 = U1 + (size_t)J * F;
    for (int j = 0; j < trials; ++j) {
      DenseAls d{};
      int nl = 0;
      if (sambaten_status e = coo_als(ws[0], st, F, ti, tj, tk, tv, ws[3].as<int64_t>(), nnz, I, J, K, 1, U0, U1,
                                      U2, seed, kGetRankId + (uint32_t)F, max_iters, tol, true, &d, &nl,
                                      rep_base + (uint32_t)j, 1))
        return e;
      const float* U[3] = {U0, U1, U2};
      const int64_t us[3] = {0, 0, 0};
      CK(launch_corcondia_coo(ti, tj, tk, tv, nnz, I, J, K, F, 1, U, us, d.lam, ccws,
                              ccd + (size_t)(F - 1) * trials + j, st));
      if (launches) *launches += nl + 4;
    }
  }
  std::vector<double> hc((size_t)R_max * trials);
  CK(cudaMemcpyAsync(hc.data(), ccd, sizeof(double) * hc.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int best = 1;
  for (int F = 1; F <= R_max; ++F) {
    double m = -1e300;
    for (int j = 0; j < trials; ++j) {
      m = std::max(m, hc[(size_t)(F - 1) * trials + j]);
      if (cc) cc[(size_t)(F - 1) * trials + j] = hc[(size_t)(F - 1) * trials + j];
    }
    if (m >= threshold) best = F;
  }
  *R_new = best;
  return SAMBATEN_OK;
}

static sambaten_status getrank_coo(const sambaten_tensor* X, int R_max, int trials, uint64_t seed, int max_iters,
                                   double tol, double threshold, int* R_new, double* cc, cudaStream_t st) {
  DevBuf ws[4];
  return getrank_coo_one(ws, X->idx[0], X->idx[1], X->idx[2], X->vals, X->nnz, (int)X->dims[0], (int)X->dims[1],
                         (int)X->dims[2], R_max, trials, 0, seed, max_iters, tol, threshold, R_new, cc, st, nullptr);
}

extern "C" sambaten_status sambaten_corcondia(const sambaten_tensor* X, int F, const float* A, const float* B,
                                              const float* C, const double* lambda, double* cc, void* stream) {
  if (sambaten_status e = check_dense(X, "corcondia")) return e;
  if (F < 1 || F > kMaxR || !A || !B || !C || !lambda || !cc) FAIL(SAMBATEN_E_INVALID, "corcondia: bad argument");
  cudaStream_t st = stream_of(stream);
  const int I = (int)X->dims[0], J = (int)X->dims[1], K = (int)X->dims[2];
  if (X->fmt == SAMBATEN_COO) {   // sparse CorConDia: device arrays, canonical order
    DevBuf ws;
    CK(ws.ensure(sizeof(double) * (corcondia_coo_ws_doubles(I, J, K, F, 1) + 1)));
    double* out = ws.as<double>() + corcondia_coo_ws_doubles(I, J, K, F, 1);
    const float* U[3] = {A, B, C};
    const int64_t us[3] = {0, 0, 0};
    CK(launch_corcondia_coo(X->idx[0], X->idx[1], X->idx[2], X->vals, X->nnz, I, J, K, F, 1, U, us, lambda,
                            ws.as<double>(), out, st));
    CK(cudaMemcpyAsync(cc, out, sizeof(double), cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    return SAMBATEN_OK;
  }
  void* ws = nullptr;
  CK(cudaMallocAsync(&ws, sizeof(double) * (corcondia_ws_doubles(I, J, K, F, 1) + 1), st));
  double* out = static_cast<double*>(ws) + corcondia_ws_doubles(I, J, K, F, 1);
  const float* U[3] = {A, B, C};
  const int64_t us[3] = {0, 0, 0};
  CK(launch_corcondia(X->vals, 0, X->dims[0], I, J, K, F, 1, U, us, lambda, static_cast<double*>(ws), out, st));
  CK(cudaMemcpyAsync(cc, out, sizeof(double), cudaMemcpyDefault, st));
  CK(cudaFreeAsync(ws, st));
  CK(cudaStreamSynchronize(st));
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_getrank(const sambaten_tensor* X, int R_max, int trials, uint64_t seed,
                                            int max_iters, double tol, double threshold, int* R_new, double* cc,
                                            void* stream) {
  if (sambaten_status e = check_dense(X, "getrank")) return e;
  if (R_max < 1 || R_max > kMaxR || trials < 1 || trials > kMaxReps || max_iters < 1 || !R_new)
    FAIL(SAMBATEN_E_INVALID, "getrank: bad argument");
  if (X->fmt == SAMBATEN_COO)
    return getrank_coo(X, R_max, trials, seed, max_iters, tol, threshold, R_new, cc, stream_of(stream));
  DevBuf ws;
  const cudaError_t e = getrank_batch(X->vals, 0, X->dims[0], (int)X->dims[0], (int)X->dims[1], (int)X->dims[2],
                                      1, R_max, trials, seed, max_iters, tol, threshold, ws, stream_of(stream),
                                      R_new, cc, nullptr);
  ws.release();
  CK(e);
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_fit(const sambaten_tensor* X, const float* lambda, const float* A,
                                        const float* B, const float* C, int R, double* relerr,
                                        void* stream) {
  if (sambaten_status e = check_dense(X, "fit")) return e;
  if (R < 1 || R > kMaxR || !relerr) FAIL(SAMBATEN_E_INVALID, "fit: bad argument");
  cudaStream_t st = stream_of(stream);
  if (X->fmt == SAMBATEN_COO) {
    const CooView V{X->idx[0], X->idx[1], X->idx[2], X->vals, X->nnz, X->dims[0], X->dims[1], X->dims[2]};
    void* ws = nullptr;
    CK(cudaMallocAsync(&ws, sizeof(double) * coo_fit_ws_doubles(V.I, V.J, V.K), st));
    CK(launch_coo_fit(V, lambda, A, B, C, R, static_cast<double*>(ws), relerr, st));
    CK(cudaFreeAsync(ws, st));
    return SAMBATEN_OK;
  }
  const DenseView V = user_view(X);
  void* ws = nullptr;
  CK(cudaMallocAsync(&ws, sizeof(double) * fit_ws_doubles_any(V), st));
  CK(fit_any(V, lambda, A, B, C, R, static_cast<double*>(ws), relerr, st));
  CK(cudaFreeAsync(ws, st));
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                           uint64_t key, int64_t n, uint32_t* out, void* stream) {
  if (n < 0 || (n > 0 && !out)) FAIL(SAMBATEN_E_INVALID, "philox: bad argument");
  CK(launch_philox(c0, c1, c2, c3, key, n, out, stream_of(stream)));
  return SAMBATEN_OK;
}

extern "C" sambaten_status sambaten_detlog(const double* u, int64_t n, double* out, void* stream) {
  if (n < 0 || (n > 0 && (!u || !out))) FAIL(SAMBATEN_E_INVALID, "detlog: bad argument");
  CK(launch_detlog(u, n, out, stream_of(stream)));
  return SAMBATEN_OK;
}
