// solvers.cu — block preconditioner composition and preconditioned MINRES (Algorithm 1).
//
// MINRES keeps every scalar of Algorithm 1 in device memory: one single-thread
// kernel evaluates lines 10-18 (gamma_{j+1}, alpha_0..3, c, s, eta) from the two fused dot
// products, so an iteration is a fixed kernel sequence with no host round trip inside it.
// One iteration is captured in a CUDA graph (two graphs: the v/z/w buffers alternate with
// period 2); the host only reads a done flag after each graph launch.
#include "etq_internal.cuh"
#include <cmath>
#include <cstring>
#include <vector>

namespace {
constexpr int BS = 256;
inline int grid_for(int64_t n, int cap = 4096) {
  int64_t g = (n + BS - 1) / BS;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

__global__ void k_scale_copy(double* y, const double* x, double a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i];
}
__global__ void k_lincomb3(double* w, const double* a, double ca, const double* b, double cb, const double* c,
                           double cc, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = ca * a[i] + cb * b[i] + cc * c[i];
}
__global__ void k_sub(double* y, const double* a, const double* b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a[i] - b[i];
}

// MINRES line 8: v_new = q - (delta/gamma) v - (gamma/gamma_prev) v_prev   (in place on v_prev)
__global__ void k_minres_v(const double* q, const double* v, double* vp, const double* sc, int64_t n) {
  if (sc[S_DONE] != 0.0) return;
  const double g = sc[S_GAMMA], gp = sc[S_GAMMA_PREV], d = sc[S_DELTA];
  const double a = d / g;
  const double b = (gp != 0.0) ? g / gp : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    vp[i] = (b != 0.0) ? (q[i] - a * v[i] - b * vp[i]) : (q[i] - a * v[i]);
}

// MINRES lines 10-19 on one thread
__global__ void k_minres_scalars(double* sc, double* hist, int hist_cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  sc[S_TMP0] = sc[S_DONE];            // done flag seen by this iteration's w/x update
  if (sc[S_DONE] != 0.0) return;
  const double zv = sc[S_DOT0] + sc[S_DOT1];
  if (!(zv >= 0.0)) {
    sc[S_STATUS] = (zv != zv) ? (double)ETQ_ENAN : (double)ETQ_EINDEFINITE;
    sc[S_DONE] = 1.0; sc[S_TMP0] = 1.0;
    return;
  }
  const double gamma = sc[S_GAMMA], delta = sc[S_DELTA];
  const double c = sc[S_C], cp = sc[S_C_PREV], s = sc[S_S], sp = sc[S_S_PREV];
  const double eta = sc[S_ETA];
  const double gn = sqrt(zv);                                    // line 10
  const double a0 = c * delta - cp * s * gamma;                  // line 11
  const double a1 = sqrt(a0 * a0 + gn * gn);                     // line 12
  const double a2 = s * delta + cp * c * gamma;                  // line 13
  const double a3 = sp * gamma;                                  // line 14
  if (a1 == 0.0 || a1 != a1) {
    sc[S_STATUS] = (a1 != a1) ? (double)ETQ_ENAN : (double)ETQ_EBREAKDOWN;
    sc[S_DONE] = 1.0; sc[S_TMP0] = 1.0;
    return;
  }
  const double cn = a0 / a1, sn = gn / a1;                       // line 15
  sc[S_A1] = a1; sc[S_A2] = a2; sc[S_A3] = a3;
  sc[S_CE_PREV] = sc[S_CNEW_ETA];                                // the previous iteration's (deferred x update)
  sc[S_CNEW_ETA] = cn * eta;                                     // line 17 coefficient
  sc[S_TMP1] = 1.0 / gamma;                                      // z^{(j)} / gamma_j in line 16
  const double etan = -sn * eta;                                 // line 18
  sc[S_ETA] = etan;
  sc[S_C_PREV] = c; sc[S_C] = cn; sc[S_S_PREV] = s; sc[S_S] = sn;
  sc[S_GAMMA_PREV] = gamma; sc[S_GAMMA] = gn;
  sc[S_INV_GAMMA] = gn > 0.0 ? 1.0 / gn : 0.0;
  const int it = (int)sc[S_IT];
  if (it < hist_cap) {
    hist[it] = fabs(etan);
    hist[hist_cap + it] = delta;
    hist[2 * hist_cap + it] = gn;
  }
  sc[S_IT] = it + 1;
  if (fabs(etan) / sc[S_GAMMA1] < sc[S_RTOL]) sc[S_DONE] = 1.0;   // line 19
  else if (it + 1 >= (int)sc[S_MAXIT]) sc[S_DONE] = 1.0;
}

// line 16-17: w_new = (z/gamma - a3 w_prev - a2 w)/a1 (in place on w_prev); x += c eta w_new.
// The x update of an odd iteration is deferred to the next (even) iteration's call, which holds
// both directions (w = w_{j-1} is an operand of line 16 anyway): x is read and written every
// other iteration (8 N fewer bytes per iteration), by the same two multiply-adds in the same order.
//   xmode 0: odd iteration, x untouched; 1: even iteration, x += ce_{j-1} w_{j-1} + ce_j w_j;
//   2: the last iteration of a solve when it is odd (tail): x += ce_j w_j
// Tail calls (w0 != nullptr) also flush the pending odd update when the iteration they belong to
// never ran (the loop stopped inside the two-iteration graph body, or on an error status).
__global__ void k_minres_wx(const double* z, const double* w, double* wp, double* x, const double* sc, int64_t n,
                            int xmode, const double* w0) {
  if (sc[S_TMP0] != 0.0) {
    if (w0 && (((int)sc[S_IT]) & 1)) {
      const double ce = sc[S_CNEW_ETA];
      for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = fma(ce, w0[i], x[i]);
    }
    return;
  }
  const double ig = sc[S_TMP1], a1 = sc[S_A1], a2 = sc[S_A2], a3 = sc[S_A3], ce = sc[S_CNEW_ETA];
  const double cep = sc[S_CE_PREV];
  const double inv_a1 = 1.0 / a1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double wo = w[i];
    const double wn = (z[i] * ig - a3 * wp[i] - a2 * wo) * inv_a1;
    wp[i] = wn;
    if (xmode == 1) x[i] = fma(ce, wn, fma(cep, wo, x[i]));
    else if (xmode == 2) x[i] = fma(ce, wn, x[i]);
  }
}

// P1 pressure refinement (below): s = r - s ; z += t
__global__ void k_sub_from(const double* r, double* s, int64_t n, const double* done) {
  if (done && *done != 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s[i] = r[i] - s[i];
}
__global__ void k_add_to(double* z, const double* t, int64_t n, const double* done) {
  if (done && *done != 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] += t[i];
}

__global__ void k_minres_init(double* sc) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double zv = sc[S_DOT0] + sc[S_DOT1];
  if (!(zv >= 0.0)) {
    sc[S_STATUS] = (zv != zv) ? (double)ETQ_ENAN : (double)ETQ_EINDEFINITE;
    sc[S_DONE] = 1.0;
    return;
  }
  const double g = sqrt(zv);                                     // line 3
  sc[S_GAMMA] = g; sc[S_GAMMA1] = g; sc[S_ETA] = g;              // line 4
  sc[S_GAMMA_PREV] = 0.0;
  sc[S_C] = 1.0; sc[S_C_PREV] = 1.0; sc[S_S] = 0.0; sc[S_S_PREV] = 0.0;
  sc[S_INV_GAMMA] = g > 0.0 ? 1.0 / g : 0.0;
  sc[S_IT] = 0.0;
  sc[S_DONE] = (g == 0.0) ? 1.0 : 0.0;
  sc[S_STATUS] = 0.0;
}
}  // namespace

void vec_scale_copy(double* y, const double* x, double a, int64_t n, cudaStream_t st) {
  k_scale_copy<<<grid_for(n), BS, 0, st>>>(y, x, a, n); etq_count_launch();
}
void vec_lincomb3(double* w, const double* a, double ca, const double* b, double cb, const double* c, double cc,
                  int64_t n, cudaStream_t st) {
  k_lincomb3<<<grid_for(n), BS, 0, st>>>(w, a, ca, b, cb, c, cc, n); etq_count_launch();
}

// z = P^{-1} r for the block-diagonal Stokes preconditioners; optional dot partials
// <z_u, w_u> -> out_u and <z_p, w_p> -> out_p.
etq_status precond_apply_ex(const Problem& P, etq_pc_kind kind, const double* r, double* z, const double* w,
                            double* out_u, double* out_p, const double* done, cudaStream_t st) {
  NvtxRange nvtx_("preconditioner apply");
  const RedSite* site = &P.red[0];
  const int64_t nu = P.n_u, np = P.n_p;
  if (kind == ETQ_PC_OSEEN_M1 || kind == ETQ_PC_OSEEN_PCD1 || kind == ETQ_PC_OSEEN_M2 || kind == ETQ_PC_OSEEN_LSC)
    return oseen_precond_apply(P, kind, r, z, st);
  if (kind == ETQ_PC_P1_EXACT) {
    if (!P.p1.ready) return ETQ_ENOTSETUP;
    dense_gemv(P.p1.Ainv, P.g.nq, 2, r, P.g.nq, z, P.g.nq, done, st);
    dense_gemv(P.p1.MQinv, (int)np, 1, r + nu, np, z + nu, np, done, st);
    // one step of iterative refinement of the augmented M_Q solve: the dense inverse
    // W = (M_Q + k k^T)^{-1} - k k^T/(k^T k)^2 carries an error ~ cond(M_Q + k k^T) eps; with
    // s = r_p - M_Q z_p, z_p += W s restores M_Q z_p = r_p - lambda k to rounding (k^T W s = 0)
    double* s = P.p1.tmp;
    double* t = P.p1.tmp + np;
    mass_apply(P.g, z + nu, s, st);
    k_sub_from<<<grid_for(np, 1024), BS, 0, st>>>(r + nu, s, np, done); etq_count_launch();
    dense_gemv(P.p1.MQinv, (int)np, 1, s, np, t, np, done, st);
    k_add_to<<<grid_for(np, 1024), BS, 0, st>>>(z + nu, t, np, done); etq_count_launch();
    if (out_u) launch_dot(z, w, nu, const_cast<RedSite*>(site), 1, out_u, done, st);
    if (out_p) launch_dot(z + nu, w + nu, np, const_cast<RedSite*>(site), 2, out_p, done, st);
    return ETQ_OK;
  }
  if (kind == ETQ_PC_P3 || kind == ETQ_PC_P1_ITER) {
    if (!P.mx.ready || (kind == ETQ_PC_P1_ITER && !P.vi.ready)) return ETQ_ENOTSETUP;
    // exact M_Q solve on the aux stream, velocity block (one V-cycle or V-cycle-PCG) on the main stream
    ETQ_CHECK(cudaEventRecord(P.ev_fork, st));
    ETQ_CHECK(cudaStreamWaitEvent(P.aux, P.ev_fork, 0));
    ETQ_TRY(exact_mass_apply(P, r + nu, z + nu, site, 2, out_p, w ? w + nu : nullptr, done, P.aux));
    if (kind == ETQ_PC_P3) ETQ_TRY(vcycle_apply_ex(P, P.mg, r, z, site, 1, out_u, w, done, st, true));
    else ETQ_TRY(vel_iter_apply(P, r, z, site, 1, out_u, w, done, st));
    ETQ_CHECK(cudaEventRecord(P.ev_join, P.aux));
    ETQ_CHECK(cudaStreamWaitEvent(st, P.ev_join, 0));
    return ETQ_OK;
  }
  if (kind == ETQ_PC_P2_GMG) {
    if (!P.p2_ready) return ETQ_ENOTSETUP;
    // pressure branch on the aux stream, velocity V-cycle on the main stream
    ETQ_CHECK(cudaEventRecord(P.ev_fork, st));
    ETQ_CHECK(cudaStreamWaitEvent(P.aux, P.ev_fork, 0));
    if (P.plain) {   // plain Q2-Q1: z_p1 = Chebyshev-Jacobi(Q_k) r_p1, z_p0 = 0 (etq.h, etq_grid.enriched)
      const int64_t nk = P.g.nk;
      qk_cheb_ws(P, r + nu, z + nu, P.params.mass_cheb_steps, P.plain_w, done, P.aux);
      ETQ_CHECK(cudaMemsetAsync(z + nu + nk, 0, sizeof(double) * (np - nk), P.aux));
      if (out_p) launch_dot(z + nu, w + nu, np, const_cast<RedSite*>(site), 2, out_p, done, P.aux);
    } else {
      ETQ_TRY(mass_pc_apply_ex(P, r + nu, z + nu, site, 2, out_p, w ? w + nu : nullptr, done, P.aux));
    }
    ETQ_TRY(vcycle_apply_ex(P, P.mg, r, z, site, 1, out_u, w, done, st, g_p2_vc_pdl));
    ETQ_CHECK(cudaEventRecord(P.ev_join, P.aux));
    ETQ_CHECK(cudaStreamWaitEvent(st, P.ev_join, 0));
    return ETQ_OK;
  }
  return ETQ_ENOTSETUP;
}

// device-side MINRES loop: the WHILE node's condition is "not done" (set before the loop and at the
// end of every two-iteration body)
__global__ void k_minres_cond(const double* sc, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0 && blockIdx.x == 0) cudaGraphSetConditional(h, sc[S_DONE] != 0.0 ? 0u : 1u);
}

void drop_minres_graphs(Problem& P) {
  for (int g = 0; g < 2; ++g)
    if (P.minres_graph[g]) { cudaGraphExecDestroy(P.minres_graph[g]); P.minres_graph[g] = nullptr; }
  P.minres_graph_kind = -1;
  P.minres_graph_x = nullptr;
  if (P.minres_wgraph) { cudaGraphExecDestroy(P.minres_wgraph); P.minres_wgraph = nullptr; }
  P.minres_wgraph_kind = -1;
  P.minres_wgraph_x = nullptr;
}

static etq_status minres_alloc(Problem& P) {
  if (!P.wside) {
    int lo = 0, hi = 0;
    ETQ_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ETQ_CHECK(cudaStreamCreateWithPriority(&P.wside, cudaStreamNonBlocking, hi));
    ETQ_CHECK(cudaEventCreateWithFlags(&P.ev_wfork, cudaEventDisableTiming));
    ETQ_CHECK(cudaEventCreateWithFlags(&P.ev_wjoin, cudaEventDisableTiming));
  }
  if (P.nkv >= 7) return ETQ_OK;
  for (int i = P.nkv; i < 7; ++i) ETQ_TRY(dalloc(&P.kv[i], P.N));
  P.nkv = 7;
  return ETQ_OK;
}

static etq_status minres_iteration(Problem& P, etq_pc_kind kind, int cur, double* x, cudaStream_t st) {
  double* V[2] = {P.kv[0], P.kv[1]};
  double* Z[2] = {P.kv[2], P.kv[3]};
  double* W[2] = {P.kv[4], P.kv[5]};
  double* Q = P.kv[6];
  double* sc = P.dscal;
  const int64_t N = P.N;
  const double* done = sc + S_DONE;
  // lines 16-17 of the PREVIOUS iteration (w, x update; skipped via S_TMP0 when there is none or the
  // solve had already stopped) on a side stream, beside this iteration's saddle apply: they share
  // no vector and no scalar (the update reads z_{j-1}, w and x; the apply reads z_j and writes q and
  // delta), and this iteration's preconditioner, which overwrites z_{j-1}, starts after the join
  ETQ_CHECK(cudaEventRecord(P.ev_wfork, st));
  ETQ_CHECK(cudaStreamWaitEvent(P.wside, P.ev_wfork, 0));
  k_minres_wx<<<grid_for(N), BS, 0, P.wside>>>(Z[1 - cur], W[1 - cur], W[cur], x, sc, N, cur == 1 ? 1 : 0, nullptr);
  etq_count_launch();
  ETQ_CHECK(cudaEventRecord(P.ev_wjoin, P.wside));
  // line 6-7: q = K (z / gamma), delta = <q, z / gamma>
  launch_saddle_ex(P, P.plain, Z[cur], Q, sc + S_INV_GAMMA, &P.red[0], 0, sc + S_DELTA, done, st);
  ETQ_CHECK(cudaStreamWaitEvent(st, P.ev_wjoin, 0));
  // line 8
  k_minres_v<<<grid_for(N), BS, 0, st>>>(Q, V[cur], V[1 - cur], sc, N); etq_count_launch();
  // line 9-10 (dot products fused into the preconditioner's last kernels)
  ETQ_TRY(precond_apply_ex(P, kind, V[1 - cur], Z[1 - cur], V[1 - cur], sc + S_DOT0, sc + S_DOT1, done, st));
  // lines 10-19 (lines 16-17 of this iteration run at the start of the next one, or in minres_wx_tail)
  k_minres_scalars<<<1, 32, 0, st>>>(sc, P.dhist, P.hist_cap); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

// lines 16-17 of the last iteration run (parity cur), after the loop
static etq_status minres_wx_tail(Problem& P, int cur, double* x, cudaStream_t st) {
  double* Z[2] = {P.kv[2], P.kv[3]};
  double* W[2] = {P.kv[4], P.kv[5]};
  // parity-0 last iteration = an even one (both pending directions); parity 1 = an odd one (its own only)
  k_minres_wx<<<grid_for(P.N), BS, 0, st>>>(Z[cur], W[cur], W[1 - cur], x, P.dscal, P.N, cur == 0 ? 1 : 2, W[0]);
  etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status minres_run(Problem& P, etq_pc_kind kind, const double* b, double* x, double rtol, int maxit,
                      etq_report* rep) {
  NvtxRange nvtx_("minres (Algorithm 1)");
  if (maxit < 1) return ETQ_EINVAL;
  ETQ_TRY(minres_alloc(P));
  cudaStream_t st = P.stream;
  const int64_t N = P.N;
  double* V[2] = {P.kv[0], P.kv[1]};
  double* Z[2] = {P.kv[2], P.kv[3]};
  double* W[2] = {P.kv[4], P.kv[5]};
  double* Q = P.kv[6];
  double* sc = P.dscal;
  if (P.hist_cap < maxit + 1) {
    // the cached graphs capture (dhist, hist_cap) as kernel arguments: rebuild them
    drop_minres_graphs(P);
    if (P.dhist) cudaFree(P.dhist);
    P.hist_cap = maxit + 1;
    ETQ_TRY(dalloc(&P.dhist, 3 * (size_t)P.hist_cap));
  }
  ETQ_CHECK(cudaEventRecord(P.ev_t0, st));
  // scalars
  std::vector<double> h(S_COUNT, 0.0);
  h[S_RTOL] = rtol; h[S_MAXIT] = maxit;
  h[S_TMP0] = 1.0;   // no previous iteration: the first deferred w/x update is skipped
  ETQ_CHECK(cudaMemcpyAsync(sc, h.data(), sizeof(double) * S_COUNT, cudaMemcpyHostToDevice, st));
  // line 1-2: v^(0) = 0, w^(0) = w^(1) = 0, v^(1) = b - K x0
  ETQ_CHECK(cudaMemsetAsync(V[0], 0, N * sizeof(double), st));
  ETQ_CHECK(cudaMemsetAsync(W[0], 0, N * sizeof(double), st));
  ETQ_CHECK(cudaMemsetAsync(W[1], 0, N * sizeof(double), st));
  launch_saddle_ex(P, P.plain, x, Q, nullptr, nullptr, 0, nullptr, nullptr, st);
  k_sub<<<grid_for(N), BS, 0, st>>>(V[1], b, Q, N); etq_count_launch();
  // line 3
  ETQ_TRY(precond_apply_ex(P, kind, V[1], Z[1], V[1], sc + S_DOT0, sc + S_DOT1, nullptr, st));
  k_minres_init<<<1, 32, 0, st>>>(sc); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());

  const bool graphs = P.params.use_graphs != 0;
  const bool devloop = graphs && g_minres_devloop;
  if (devloop && (P.minres_wgraph_kind != (int)kind || P.minres_wgraph_x != x || !P.minres_wgraph)) {
    // one graph: while (!done) { iteration(cur = 1); iteration(cur = 0); cond = !done }
    if (P.minres_wgraph) { cudaGraphExecDestroy(P.minres_wgraph); P.minres_wgraph = nullptr; }
    if (!P.wcs) ETQ_CHECK(cudaStreamCreateWithFlags(&P.wcs, cudaStreamNonBlocking));
    cudaGraph_t graph;
    const int64_t before = etq_launch_total();
    ETQ_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    cudaStreamCaptureStatus cst;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    etq_status s = ETQ_OK;
    cudaGraphConditionalHandle hc;
    cudaError_t e = cudaStreamGetCaptureInfo(st, &cst, nullptr, &cg, &deps, &nd);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hc, cg, 1u, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) { k_minres_cond<<<1, 32, 0, st>>>(sc, hc); etq_count_launch(); e = cudaGetLastError(); }
    if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(st, &cst, nullptr, &cg, &deps, &nd);
    cudaGraphNode_t node;
    cudaGraphNodeParams np = {};
    if (e == cudaSuccess) {
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = hc;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      e = cudaGraphAddNode(&node, cg, deps, nd, &np);
    }
    const int64_t b0 = etq_launch_total();
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(P.wcs, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                            cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      s = minres_iteration(P, kind, 1, x, P.wcs);
      if (s >= 0) s = minres_iteration(P, kind, 0, x, P.wcs);
      if (s >= 0) { k_minres_cond<<<1, 32, 0, P.wcs>>>(sc, hc); etq_count_launch(); }
      cudaGraph_t tmp;
      cudaError_t e2 = cudaStreamEndCapture(P.wcs, &tmp);
      if (e == cudaSuccess) e = e2;
    }
    P.minres_wbody_nodes = etq_launch_total() - b0;
    if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies);
    cudaError_t e3 = cudaStreamEndCapture(st, &graph);
    P.minres_wfixed_nodes = (etq_launch_total() - before) - P.minres_wbody_nodes;
    etq_count_launch(-(etq_launch_total() - before));   // captured, not launched
    if (s < 0) return s;
    ETQ_CHECK(e);
    ETQ_CHECK(e3);
    ETQ_CHECK(cudaGraphInstantiate(&P.minres_wgraph, graph, 0));
    cudaGraphDestroy(graph);
    P.minres_wgraph_kind = (int)kind;
    P.minres_wgraph_x = x;
  }
  if (graphs && !devloop && (P.minres_graph_kind != (int)kind || P.minres_graph_x != x || !P.minres_graph[0])) {
    for (int g = 0; g < 2; ++g) {
      if (P.minres_graph[g]) { cudaGraphExecDestroy(P.minres_graph[g]); P.minres_graph[g] = nullptr; }
    }
    for (int g = 0; g < 2; ++g) {
      cudaGraph_t graph;
      const int64_t before = etq_launch_total();
      ETQ_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      etq_status s = minres_iteration(P, kind, g, x, st);
      cudaError_t e = cudaStreamEndCapture(st, &graph);
      P.minres_graph_nodes[g] = etq_launch_total() - before;
      etq_count_launch(-P.minres_graph_nodes[g]);   // captured, not launched
      if (s < 0) return s;
      ETQ_CHECK(e);
      ETQ_CHECK(cudaGraphInstantiate(&P.minres_graph[g], graph, 0));
      cudaGraphDestroy(graph);
    }
    P.minres_graph_kind = (int)kind;
    P.minres_graph_x = x;
  }
  double pi0m = 0, pc0m = 0, pi0v = 0, pc0v = 0;   // inner CG counters (loop bodies run a variable count)
  const bool inner = kind == ETQ_PC_P3 || kind == ETQ_PC_P1_ITER;
  if (inner) {
    ETQ_CHECK(cudaStreamSynchronize(st));
    ETQ_TRY(pcg_stats(P, 0, &pi0m, &pc0m));
    ETQ_TRY(pcg_stats(P, 1, &pi0v, &pc0v));
  }
  int cur = 1;
  int it = 0;
  if (devloop) {
    ETQ_CHECK(cudaGraphLaunch(P.minres_wgraph, st));
    ETQ_TRY(minres_wx_tail(P, 0, x, st));   // the body ends with the parity-0 iteration
    ETQ_CHECK(cudaStreamSynchronize(st));
    ETQ_CHECK(cudaMemcpy(P.hscal, sc, sizeof(double) * 20, cudaMemcpyDeviceToHost));
    const int its = (int)P.hscal[S_IT];
    etq_count_launch(P.minres_wfixed_nodes + (int64_t)((its + 1) / 2) * P.minres_wbody_nodes);
  }
  for (; !devloop;) {
    ETQ_CHECK(cudaMemcpyAsync(P.hscal, sc, sizeof(double) * 20, cudaMemcpyDeviceToHost, st));
    ETQ_CHECK(cudaStreamSynchronize(st));
    if (P.hscal[S_DONE] != 0.0) break;
    if (graphs) {
      ETQ_CHECK(cudaGraphLaunch(P.minres_graph[cur], st));
      etq_count_launch(P.minres_graph_nodes[cur]);
    }
    else ETQ_TRY(minres_iteration(P, kind, cur, x, st));
    cur = 1 - cur;
    if (++it > maxit + 2) break;   // safety net; the device flag ends the loop
  }
  if (!devloop) ETQ_TRY(minres_wx_tail(P, 1 - cur, x, st));   // last iteration run: parity 1 - cur
  ETQ_CHECK(cudaEventRecord(P.ev_t1, st));
  ETQ_CHECK(cudaMemcpyAsync(P.hscal, sc, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost, st));
  ETQ_CHECK(cudaStreamSynchronize(st));
  if (inner && graphs) etq_count_launch(pcg_launches_since(P, pi0m, pc0m, pi0v, pc0v));
  const int iters = (int)P.hscal[S_IT];
  const int status = (int)P.hscal[S_STATUS];
  const double g1 = P.hscal[S_GAMMA1];
  const double eta = std::fabs(P.hscal[S_ETA]);
  const bool conv = status == 0 && (g1 == 0.0 || eta / g1 < rtol);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1);
  if (rep) {
    rep->iterations = iters; rep->converged = conv ? 1 : 0; rep->restarts = 0; rep->status = status;
    rep->abs_res = eta; rep->rel_res = g1 > 0 ? eta / g1 : 0.0; rep->ms_total = ms;
    const int nh = std::min(iters, P.hist_cap);
    if (rep->history && rep->history_cap > 0) {
      const int k = std::min(nh, rep->history_cap);
      ETQ_CHECK(cudaMemcpy(rep->history, P.dhist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
    if (rep->lanczos_delta && rep->lanczos_cap > 0) {
      const int k = std::min(nh, rep->lanczos_cap);
      ETQ_CHECK(cudaMemcpy(rep->lanczos_delta, P.dhist + P.hist_cap, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
    if (rep->lanczos_gamma && rep->lanczos_cap > 0) {
      const int k = std::min(nh, rep->lanczos_cap);
      ETQ_CHECK(cudaMemcpy(rep->lanczos_gamma, P.dhist + 2 * P.hist_cap, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
  }
  if (status < 0) return status;
  return conv ? ETQ_OK : ETQ_NOT_CONVERGED;
}
