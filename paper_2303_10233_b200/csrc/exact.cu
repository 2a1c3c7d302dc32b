// exact.cu — SURVEY §8(f) NEXT-2: a P1-quality (exact) M_Q solve at scale, and the
// preconditioners built on it.
//
// The exact pressure block of P1 solves the augmented system [[M_Q, k], [k^T, 0]] (P:409-427,
// P:515-516), which the n <= 32 path does with a dense inverse.  Here the Q0 block of
// M_Q = [[Q_k, R^T], [R, Q_0]] (Prop 2.1; R = h^2/4 per cell vertex, Q_0 = h^2 I) is
// eliminated, leaving the Q1-vertex Schur complement S_k = Q_k - R^T Q_0^{-1} R (9-point,
// symmetric positive semidefinite, null space = constants).  With a = 1 + R^T 1 / h^2 the
// augmented solve becomes (reading R21, pinned by
// tests/test_oracle_mg_mass.py::test_schur_reduction_equals_augmented_solve):
//   lambda = k^T r / 1^T a,   g = r_k - R^T r_0 / h^2 - lambda a        (1^T g = 0)
//   zhat   = S_k^+ g                          (PCG, preconditioned by one Q1-GMG V-cycle on S_k)
//   beta   = ((1^T r_0 + lambda n_0) / h^2 - a^T zhat) / 1^T a
//   z_k    = zhat + beta 1,   z_0 = (r_0 - R z_k + lambda 1) / h^2
// so that M_Q z + lambda k = r and k^T z = 0 hold to the PCG tolerance.
//
// The PCG loops run as CUDA-graph WHILE conditional nodes: the convergence test is taken on the
// device (last block of the residual reduction) and ends the loop without a host round trip, so
// the whole preconditioner — and the MINRES iteration around it — stays one captured graph.
// Outside a capture the same code is captured into a temporary graph and launched once.
//
// Preconditioners (include/etq.h):
//   ETQ_PC_P3      = diag(one Q2-GMG V-cycle, exact M_Q)            (P2's velocity block, P1's M_Q)
//   ETQ_PC_P1_ITER = diag(A^{-1} by V-cycle-PCG, exact M_Q)         (P1 at any n)
#include "etq_internal.cuh"
#include <cmath>
#include <cstdio>
#include <vector>
#include "device_common.cuh"

using namespace etqd;

namespace {

// reduction slots of PcgWs::red
constexpr int SL_R0 = 0, SL_RZ = 1, SL_PQ = 2, SL_RR = 3, SL_SUMS = 4 /* 4,5 */, SL_ADOT = 6;
// PcExactMass::sc
constexpr int MX_SK = 0, MX_S0 = 1, MX_LAM = 2, MX_ADOT = 3, MX_BETA = 4;

__device__ __forceinline__ bool pcg_done(const double* sc) { return sc[PG_DONE] != 0.0; }

__device__ __forceinline__ void pcg_stop(double* sc, cudaGraphConditionalHandle h, int use_h) {
  sc[PG_DONE] = 1.0;
  if (use_h) cudaGraphSetConditional(h, 0u);
}

__global__ void k_pcg_start(double* sc, const double* outer_done, cudaGraphConditionalHandle h, int use_h) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const bool d = outer_done && *outer_done != 0.0;
  sc[PG_DONE] = d ? 1.0 : 0.0;
  sc[PG_IT] = 0.0;
  if (!d) sc[PG_CALLS] += 1.0;
  if (use_h) cudaGraphSetConditional(h, d ? 0u : 1u);
}

// x = 0, r = b, r0 = b^T b
__global__ void __launch_bounds__(BS) k_pcg_init(const double* b, double* x, double* r, int64_t n, RedSite site,
                                                 double* sc, cudaGraphConditionalHandle h, int use_h) {
  if (pcg_done(sc)) return;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = b[i];
    x[i] = 0.0; r[i] = v; s += v * v;
  }
  double a[1] = {s};
  if (reduce_finish<1>(a, site, SL_R0, sc + PG_R0)) {
    if (!(sc[PG_R0] > 0.0)) pcg_stop(sc, h, use_h);
  }
}

__global__ void __launch_bounds__(BS) k_pcg_p0(double* p, const double* z, int64_t n, const double* sc) {
  if (pcg_done(sc)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i];
}

// q = A p, pq = p^T q (NC = 2: the scalar velocity operator on both components, node-permuted
// SELL; NC = 1: a Q1 operator in natural row order).  Also moves rz_new into rz_old.
template <int NC>
__global__ void __launch_bounds__(BS) k_pcg_spmv(Sell A, int nq, const double* p, double* q, RedSite site,
                                                 double* sc) {
  if (pcg_done(sc)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[PG_RZ0] = sc[PG_RZ1];
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double s = 0.0;
  for (int64_t sl = gw; sl < A.nslices; sl += nw) {
    const int64_t t = sl * SELL_C + lane;
    if (NC == 2) {
      const int row = A.perm[t];
      double a0 = 0.0, a1 = 0.0;
      sell_row2(A, sl, lane, row, p, p + nq, a0, a1);
      if (row >= 0) {
        q[row] = a0; q[nq + row] = a1;
        s += a0 * p[row] + a1 * p[nq + row];
      }
    } else {
      const int row = A.perm ? A.perm[t] : (t < A.nrows ? (int)t : -1);
      const double v = sell_row1(A, sl, lane, p);
      if (row >= 0) { q[row] = v; s += v * p[row]; }
    }
  }
  double a[1] = {s};
  reduce_finish<1>(a, site, SL_PQ, sc + PG_PQ);
}

// q = S_k p (matrix-free, level 0 of the S_k hierarchy: w = h^2 / 144), pq = p^T q
__global__ void __launch_bounds__(BS) k_pcg_spmv_sk(int n, double w, const double* p, double* q, RedSite site,
                                                    double* sc) {
  if (pcg_done(sc)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[PG_RZ0] = sc[PG_RZ1];
  const int n1 = n + 1;
  const int64_t nk = (int64_t)n1 * n1;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / n1), a = (int)(i - (int64_t)c * n1);
    double d7;
    const double v = w * sk_stencil(i, a, c, n, p, &d7);
    q[i] = v;
    s += v * p[i];
  }
  double a[1] = {s};
  reduce_finish<1>(a, site, SL_PQ, sc + PG_PQ);
}

// alpha = rz / pq; x += alpha p; r -= alpha q; stop test ||r||^2 <= tol^2 ||b||^2 or it >= maxit
__global__ void __launch_bounds__(BS) k_pcg_xr(double* x, double* r, const double* p, const double* q, int64_t n,
                                               RedSite site, double* sc, cudaGraphConditionalHandle h, int use_h) {
  if (pcg_done(sc)) return;
  const double pq = sc[PG_PQ];
  const double alpha = pq > 0.0 ? sc[PG_RZ0] / pq : 0.0;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double v = r[i] - alpha * q[i];
    r[i] = v; s += v * v;
  }
  double a[1] = {s};
  if (reduce_finish<1>(a, site, SL_RR, sc + PG_RR)) {
    const double it = sc[PG_IT] + 1.0;
    sc[PG_IT] = it;
    sc[PG_ITTOT] += 1.0;
    if (!(pq > 0.0) || sc[PG_RR] <= sc[PG_TOL2] * sc[PG_R0] || it >= sc[PG_MAXIT]) pcg_stop(sc, h, use_h);
  }
}

__global__ void __launch_bounds__(BS) k_pcg_p(double* p, const double* z, int64_t n, const double* sc) {
  if (pcg_done(sc)) return;
  const double beta = sc[PG_RZ1] / sc[PG_RZ0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// ---------------------------------------------------------------- exact M_Q pieces
__device__ __forceinline__ int cells_at(int a, int n) { return (a > 0) + (a < n); }

// sums of r_k and r_0 -> lambda = (1^T r_k - 1^T r_0) / (n_k + n_0)   (1^T a = n_k + n_0)
__global__ void __launch_bounds__(BS) k_mq_sums(const double* r_p, int nk, int n0, RedSite site, double* msc,
                                                const double* done) {
  if (is_done(done)) return;
  double s[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk + n0; i += (int64_t)gridDim.x * blockDim.x)
    s[i < nk ? 0 : 1] += r_p[i];
  if (reduce_finish<2>(s, site, SL_SUMS, msc + MX_SK)) msc[MX_LAM] = (msc[MX_SK] - msc[MX_S0]) / (double)(nk + n0);
}

// g_p = r_k[p] - (1/4) sum_{T ni p} r_0[T] - lambda (1 + #{T ni p} / 4)
__global__ void __launch_bounds__(BS) k_mq_g(const double* r_p, double* g, int n, const double* msc, const double* done) {
  if (is_done(done)) return;
  const int n1 = n + 1, nk = n1 * n1;
  const double* r0 = r_p + nk;
  const double lam = msc[MX_LAM];
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nk; p += gridDim.x * blockDim.x) {
    const int a = p % n1, c = p / n1;
    double s = 0.0;
    for (int f = max(0, c - 1); f <= min(n - 1, c); ++f)
      for (int e = max(0, a - 1); e <= min(n - 1, a); ++e) s += r0[e + n * f];
    const double cnt = (double)(cells_at(a, n) * cells_at(c, n));
    g[p] = r_p[p] - 0.25 * s - lam * (1.0 + 0.25 * cnt);
  }
}

// a^T zhat -> beta = ((1^T r_0 + lambda n_0) / h^2 - a^T zhat) / (n_k + n_0)
__global__ void __launch_bounds__(BS) k_mq_adot(const double* zh, int n, double h2, RedSite site, double* msc,
                                                const double* done) {
  if (is_done(done)) return;
  const int n1 = n + 1, nk = n1 * n1, n0 = n * n;
  double s = 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nk; p += gridDim.x * blockDim.x) {
    const int a = p % n1, c = p / n1;
    s += (1.0 + 0.25 * (double)(cells_at(a, n) * cells_at(c, n))) * zh[p];
  }
  double v[1] = {s};
  if (reduce_finish<1>(v, site, SL_ADOT, msc + MX_ADOT))
    msc[MX_BETA] = ((msc[MX_S0] + msc[MX_LAM] * n0) / h2 - msc[MX_ADOT]) / (double)(nk + n0);
}

// z_k = zhat + beta; z_0[T] = (r_0[T] - (h^2/4) sum_{p in T} z_k[p] + lambda) / h^2; optional z^T w
__global__ void __launch_bounds__(BS) k_mq_final(const double* zh, const double* r_p, double* z_p, int n, double h2,
                                                 const double* msc, const double* dw, RedSite site, int slot,
                                                 double* out, const double* done) {
  if (is_done(done)) return;
  const int n1 = n + 1, nk = n1 * n1, n0 = n * n;
  const double beta = msc[MX_BETA], lam = msc[MX_LAM];
  double dot = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nk + n0; i += gridDim.x * blockDim.x) {
    double v;
    if (i < nk) {
      v = zh[i] + beta;
    } else {
      const int t = i - nk, e = t % n, f = t / n;
      const int p = e + n1 * f;
      const double s = (zh[p] + zh[p + 1] + zh[p + n1] + zh[p + n1 + 1]) + 4.0 * beta;
      v = (r_p[i] - 0.25 * h2 * s + lam) / h2;
    }
    z_p[i] = v;
    if (dw) dot += v * dw[i];
  }
  if (out) { double a[1] = {dot}; reduce_finish<1>(a, site, slot, out); }
}

// ---------------------------------------------------------------- two-field Lp^+ (NEXT-4)
// sums of the Q1 and P0 parts of x -> out[0], out[1]
__global__ void __launch_bounds__(BS) k_field_sums(const double* x, int nk, int n0, RedSite site, int slot,
                                                   double* out, const double* done) {
  if (is_done(done)) return;
  double s[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk + n0; i += (int64_t)gridDim.x * blockDim.x)
    s[i < nk ? 0 : 1] += x[i];
  reduce_finish<2>(s, site, slot, out);
}
// y = x - (mean of each field) (projection onto range(Lp) = the zero-mean fields)
__global__ void __launch_bounds__(BS) k_field_sub(const double* x, double* y, int nk, int n0, const double* sums,
                                                  const double* done) {
  if (is_done(done)) return;
  const double m1 = sums[0] / nk, m0 = sums[1] / n0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk + n0; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] - (i < nk ? m1 : m0);
}

// ---------------------------------------------------------------- PCG driver
// A and M issue their launches on the given stream; M must write z = M r and the dot r^T z into
// sc[PG_RZ1] through (site, SL_RZ) and honour done = sc + PG_DONE.
struct PcgOps {
  int nc;                         // 2: velocity (Sell with node perm), 1: Q1
  const Sell* A; int nq;
  const Problem* P; const Hierarchy* H;
};

static void pcg_apply_A(const PcgWs& W, const PcgOps& o, cudaStream_t st) {
  const int gs = grid_for(o.A->nslices * 32, BS, 4096);
  if (o.nc == 1 && o.H->op == 1)
    k_pcg_spmv_sk<<<grid_for(W.n, BS, RED_BLOCKS * 2), BS, 0, st>>>(o.H->lv[0].g.n, o.H->sk_w, W.p, W.q, W.red, W.sc);
  else if (o.nc == 2) k_pcg_spmv<2><<<gs, BS, 0, st>>>(*o.A, o.nq, W.p, W.q, W.red, W.sc);
  else k_pcg_spmv<1><<<gs, BS, 0, st>>>(*o.A, o.nq, W.p, W.q, W.red, W.sc);
  etq_count_launch();
}

static etq_status pcg_apply_M(const PcgWs& W, const PcgOps& o, cudaStream_t st) {
  return vcycle_apply_ex(*o.P, *o.H, W.r, W.z, &W.red, SL_RZ, W.sc + PG_RZ1, W.r, W.sc + PG_DONE, st, true);
}

static etq_status pcg_body(const PcgWs& W, const PcgOps& o, double* x, cudaGraphConditionalHandle h, int use_h,
                           cudaStream_t st) {
  pcg_apply_A(W, o, st);
  k_pcg_xr<<<grid_for(W.n, BS, RED_BLOCKS), BS, 0, st>>>(x, W.r, W.p, W.q, W.n, W.red, W.sc, h, use_h);
  etq_count_launch();
  ETQ_TRY(pcg_apply_M(W, o, st));
  k_pcg_p<<<grid_for(W.n, BS, 4096), BS, 0, st>>>(W.p, W.z, W.n, W.sc); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

// x = A^+ b to the relative tolerance W.rtol (at most W.maxit iterations).  `st` must be capturing.
static etq_status pcg_captured(PcgWs& W, const PcgOps& o, const double* b, double* x, const double* outer_done,
                               cudaStream_t st) {
  cudaStreamCaptureStatus cst;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  ETQ_CHECK(cudaStreamGetCaptureInfo(st, &cst, nullptr, &g, &deps, &nd));
  if (cst != cudaStreamCaptureStatusActive) return ETQ_ECUDA;
  cudaGraphConditionalHandle h;
  ETQ_CHECK(cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault));
  const int64_t l0 = etq_launch_total();
  k_pcg_start<<<1, 32, 0, st>>>(W.sc, outer_done, h, 1); etq_count_launch();
  k_pcg_init<<<grid_for(W.n, BS, RED_BLOCKS), BS, 0, st>>>(b, x, W.r, W.n, W.red, W.sc, h, 1); etq_count_launch();
  ETQ_TRY(pcg_apply_M(W, o, st));
  k_pcg_p0<<<grid_for(W.n, BS, 4096), BS, 0, st>>>(W.p, W.z, W.n, W.sc); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  W.fixed_nodes = etq_launch_total() - l0;
  // while (cond) { body }
  ETQ_CHECK(cudaStreamGetCaptureInfo(st, &cst, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  ETQ_CHECK(cudaGraphAddNode(&node, g, deps, nd, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  ETQ_CHECK(cudaStreamBeginCaptureToGraph(W.cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  const int64_t l1 = etq_launch_total();
  etq_status s = pcg_body(W, o, x, h, 1, W.cs);
  W.body_nodes = etq_launch_total() - l1;
  cudaGraph_t tmp;
  cudaError_t e = cudaStreamEndCapture(W.cs, &tmp);
  if (s < 0) return s;
  ETQ_CHECK(e);
  ETQ_CHECK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  return ETQ_OK;
}

// Run `issue(st)` (which may contain PCG loops) inside the caller's capture, or — outside any
// capture — as a temporary graph launched once and synchronised.  Launch accounting: a captured
// loop body is counted once at capture; the extra iterations are added from the device counters.
template <class F>
static etq_status run_graphed(const Problem& P, cudaStream_t st, F issue) {
  cudaStreamCaptureStatus cst;
  ETQ_CHECK(cudaStreamIsCapturing(st, &cst));
  if (cst == cudaStreamCaptureStatusActive) return issue(st);
  double i0m = 0, c0m = 0, i0v = 0, c0v = 0;
  ETQ_TRY(pcg_stats(P, 0, &i0m, &c0m));
  ETQ_TRY(pcg_stats(P, 1, &i0v, &c0v));
  cudaGraph_t g;
  ETQ_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  etq_status s = issue(st);
  cudaError_t e = cudaStreamEndCapture(st, &g);
  if (s < 0) { if (e == cudaSuccess) cudaGraphDestroy(g); return s; }
  ETQ_CHECK(e);
  cudaGraphExec_t ex;
  cudaError_t ei = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  ETQ_CHECK(ei);
  ETQ_CHECK(cudaGraphLaunch(ex, st));
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaGraphExecDestroy(ex);
  etq_count_launch(pcg_launches_since(P, i0m, c0m, i0v, c0v));
  return ETQ_OK;
}

static etq_status pcg_alloc(PcgWs& W, int64_t n, double rtol, int maxit) {
  if (W.n != n) {
    cudaFree(W.r); cudaFree(W.z); cudaFree(W.p); cudaFree(W.q);
    W.r = W.z = W.p = W.q = nullptr;
    ETQ_TRY(dalloc(&W.r, n)); ETQ_TRY(dalloc(&W.z, n)); ETQ_TRY(dalloc(&W.p, n)); ETQ_TRY(dalloc(&W.q, n));
    W.n = n;
  }
  if (!W.sc) {
    ETQ_TRY(dalloc(&W.sc, PG_COUNT));
    W.red.nslot = RED_SLOTS;
    ETQ_TRY(dalloc(&W.red.partials, (size_t)RED_SLOTS * RED_MAXB));
    ETQ_TRY(dalloc(&W.red.counter, RED_SLOTS));
    ETQ_CHECK(cudaMemset(W.red.counter, 0, sizeof(unsigned) * RED_SLOTS));
    ETQ_CHECK(cudaStreamCreateWithFlags(&W.cs, cudaStreamNonBlocking));
  }
  W.rtol = rtol; W.maxit = maxit;
  std::vector<double> h(PG_COUNT, 0.0);
  h[PG_TOL2] = rtol * rtol; h[PG_MAXIT] = maxit;
  ETQ_CHECK(cudaMemcpy(W.sc, h.data(), sizeof(double) * PG_COUNT, cudaMemcpyHostToDevice));
  return ETQ_OK;
}

static void pcg_free(PcgWs& W) {
  cudaFree(W.r); cudaFree(W.z); cudaFree(W.p); cudaFree(W.q); cudaFree(W.sc);
  cudaFree(W.red.partials); cudaFree(W.red.counter);
  if (W.cs) cudaStreamDestroy(W.cs);
  W = PcgWs{};
}

static etq_status exact_mass_issue(PcExactMass& X, const Problem& P, const double* r_p, double* z_p,
                                   const RedSite* site, int slot, double* dot_out, const double* dot_with,
                                   const double* done, cudaStream_t st) {
  const Geo& g = P.g;
  const double h2 = g.h * g.h;
  k_mq_sums<<<grid_for((int64_t)g.nk + g.n0, BS, RED_BLOCKS), BS, 0, st>>>(r_p, g.nk, g.n0, X.cg.red, X.sc, done);
  etq_count_launch();
  k_mq_g<<<grid_for(g.nk, BS, 4096), BS, 0, st>>>(r_p, X.g, g.n, X.sc, done); etq_count_launch();
  PcgOps o{1, &X.sH.lv[0].A, g.nk, &P, &X.sH};
  ETQ_TRY(pcg_captured(X.cg, o, X.g, X.zh, done, st));
  k_mq_adot<<<grid_for(g.nk, BS, RED_BLOCKS), BS, 0, st>>>(X.zh, g.n, h2, X.cg.red, X.sc, done); etq_count_launch();
  RedSite dummy{};
  k_mq_final<<<grid_for((int64_t)g.nk + g.n0, BS, RED_BLOCKS), BS, 0, st>>>(
      X.zh, r_p, z_p, g.n, h2, X.sc, dot_with, site ? *site : dummy, slot, dot_out, done);
  etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

static etq_status vel_iter_issue(PcVelIter& V, const Problem& P, const double* r_u, double* z_u,
                                 const RedSite* site, int slot, double* dot_out, const double* dot_with,
                                 const double* done, cudaStream_t st) {
  PcgOps o{2, &P.Lv, P.g.nq, &P, &P.mg};
  ETQ_TRY(pcg_captured(V.cg, o, r_u, z_u, done, st));
  if (dot_out && site) launch_dot(z_u, dot_with, P.n_u, const_cast<RedSite*>(site), slot, dot_out, done, st);
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

static etq_status lp_pinv_issue(PcLp& X, const Problem& P, const double* r, double* z, const double* done,
                                cudaStream_t st) {
  const int nk = P.g.nk, n0 = P.g.n0;
  const int64_t np = (int64_t)nk + n0;
  const int gs = grid_for(np, BS, RED_BLOCKS);
  k_field_sums<<<gs, BS, 0, st>>>(r, nk, n0, X.cg.red, SL_SUMS, X.sc, done); etq_count_launch();
  k_field_sub<<<grid_for(np, BS, 4096), BS, 0, st>>>(r, X.rp, nk, n0, X.sc, done); etq_count_launch();
  PcgOps o{1, &X.H.lv[0].A, (int)np, &P, &X.H};
  ETQ_TRY(pcg_captured(X.cg, o, X.rp, z, done, st));
  k_field_sums<<<gs, BS, 0, st>>>(z, nk, n0, X.cg.red, SL_SUMS, X.sc + 2, done); etq_count_launch();
  k_field_sub<<<grid_for(np, BS, 4096), BS, 0, st>>>(z, z, nk, n0, X.sc + 2, done); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

}  // namespace

etq_status exact_mass_setup(Problem& P) {
  PcExactMass& X = P.mx;
  const etq_pc_params& prm = P.params;
  if (X.sH.built) free_hierarchy(X.sH);
  const int nc = std::min(P.g.n, prm.inner_coarse_n);
  ETQ_TRY(build_ap_hierarchy(P, X.sH, nc, 0.18, 1.8, 3, 1));   // lambda_max(D^-1 S_k) = 12/7 (pinned)
  if (!X.g) {
    ETQ_TRY(dalloc(&X.g, P.g.nk));
    ETQ_TRY(dalloc(&X.zh, P.g.nk));
    ETQ_TRY(dalloc(&X.sc, 8));
  }
  ETQ_TRY(pcg_alloc(X.cg, P.g.nk, prm.inner_rtol, prm.inner_maxit));
  X.ready = true;
  return ETQ_OK;
}

etq_status vel_iter_setup(Problem& P) {
  if (!P.mg.built) return ETQ_ENOTSETUP;
  ETQ_TRY(pcg_alloc(P.vi.cg, P.n_u, P.params.inner_rtol, P.params.inner_maxit));
  P.vi.ready = true;
  return ETQ_OK;
}

void exact_free(Problem& P) {
  if (P.mx.sH.built) free_hierarchy(P.mx.sH);
  cudaFree(P.mx.g); cudaFree(P.mx.zh); cudaFree(P.mx.sc);
  pcg_free(P.mx.cg);
  P.mx = PcExactMass{};
  pcg_free(P.vi.cg);
  P.vi = PcVelIter{};
}

etq_status exact_mass_apply(const Problem& P, const double* r_p, double* z_p, const RedSite* site, int slot,
                            double* dot_out, const double* dot_with, const double* done, cudaStream_t st) {
  NvtxRange nvtx_("exact M_Q solve");
  if (!P.mx.ready) return ETQ_ENOTSETUP;
  PcExactMass& X = const_cast<PcExactMass&>(P.mx);
  return run_graphed(P, st, [&](cudaStream_t s) {
    return exact_mass_issue(X, P, r_p, z_p, site, slot, dot_out, dot_with, done, s);
  });
}

etq_status vel_iter_apply(const Problem& P, const double* r_u, double* z_u, const RedSite* site, int slot,
                          double* dot_out, const double* dot_with, const double* done, cudaStream_t st) {
  if (!P.vi.ready) return ETQ_ENOTSETUP;
  PcVelIter& V = const_cast<PcVelIter&>(P.vi);
  return run_graphed(P, st, [&](cudaStream_t s) {
    return vel_iter_issue(V, P, r_u, z_u, site, slot, dot_out, dot_with, done, s);
  });
}

// which 0: exact M_Q PCG, 1: velocity PCG.  Device counters (accumulated over all calls).
etq_status pcg_stats(const Problem& P, int which, double* it_total, double* calls) {
  const PcgWs& W = which == 0 ? P.mx.cg : P.vi.cg;
  *it_total = 0.0; *calls = 0.0;
  if (!W.sc) return ETQ_OK;
  double h[PG_COUNT];
  ETQ_CHECK(cudaMemcpy(h, W.sc, sizeof(h), cudaMemcpyDeviceToHost));
  *it_total = h[PG_ITTOT]; *calls = h[PG_CALLS];
  return ETQ_OK;
}

// kernel launches executed beyond the once-counted captured loop bodies since the given counters
int64_t pcg_launches_since(const Problem& P, double it0_m, double calls0_m, double it0_v, double calls0_v) {
  double im, cm, iv, cv;
  if (pcg_stats(P, 0, &im, &cm) < 0 || pcg_stats(P, 1, &iv, &cv) < 0) return 0;
  const double em = (im - it0_m) - (cm - calls0_m), ev = (iv - it0_v) - (cv - calls0_v);
  return (int64_t)(std::max(0.0, em) * (double)P.mx.cg.body_nodes + std::max(0.0, ev) * (double)P.vi.cg.body_nodes);
}

// ---------------------------------------------------------------- Lp^+ (NEXT-4)
// Two-field pressure Laplacian Lp = B Mdiag^-1 B^T: Q1 + P0 multigrid (rediscretised Lp, bilinear and
// piecewise-constant transfers, Chebyshev-3 on [0.21, 2.1] in D^-1 Lp: lambda_max = 1.93 on fine
// levels, reading R25), coarse pseudo-inverse at n_c = 2; CG to inner_rtol on the zero-mean fields.
etq_status lp_setup(Problem& P) {
  PcLp& X = P.lp;
  if (X.ready) return ETQ_OK;
  ETQ_TRY(build_ap_hierarchy(P, X.H, 2, 0.21, 2.1, 3, 2));
  if (!X.rp) { ETQ_TRY(dalloc(&X.rp, P.n_p)); ETQ_TRY(dalloc(&X.sc, 8)); }
  ETQ_TRY(pcg_alloc(X.cg, P.n_p, P.params.inner_rtol, P.params.inner_maxit));
  X.ready = true;
  return ETQ_OK;
}

etq_status lp_pinv_apply(const Problem& P, const double* r, double* z, const double* done, cudaStream_t st) {
  if (!P.lp.ready) return ETQ_ENOTSETUP;
  PcLp& X = const_cast<PcLp&>(P.lp);
  return run_graphed(P, st, [&](cudaStream_t s) { return lp_pinv_issue(X, P, r, z, done, s); });
}

void lp_free(Problem& P) {
  if (P.lp.H.built) free_hierarchy(P.lp.H);
  cudaFree(P.lp.rp); cudaFree(P.lp.sc);
  pcg_free(P.lp.cg);
  P.lp = PcLp{};
}
