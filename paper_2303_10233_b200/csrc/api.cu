// api.cu — the extern "C" boundary of libetq (declared and documented in include/etq.h).
#include "etq_internal.cuh"
#include "../../include/etq_debug.h"
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

struct etq_problem { Problem P; };

#include <atomic>
static std::atomic<int64_t> g_launches{0};
bool g_cheb_tile_enabled = true;   // etq_set_option(0): temporally blocked smoothing on/off
int g_cheb_tile_min_n = 64;         // etq_set_option(1): coarsest level n that uses it
bool g_saddle_mf = true;            // etq_set_option(2): matrix-free Stokes saddle apply
bool g_minres_devloop = true;       // etq_set_option(3): MINRES loop as a CUDA-graph while node
bool g_sgs_high_prio = false;       // etq_set_option(4): Chebyshev-SGS kernels at the highest priority
bool g_tail_sm = true;              // etq_set_option(5): shared-memory matrix-free coarse-level tail
bool g_saddle_tile = true;          // etq_set_option(6): shared-memory tiled matrix-free saddle apply
bool g_sgs_pdl = true;              // etq_set_option(7): programmatic dependent launches in the SGS chain
bool g_cheb_tile3 = true;
bool g_p2_vc_pdl = true;
bool g_oseen_mf = true;
bool g_sgs_yp_ldg = true; 
int g_sgs_window = 0;               // etq_debug_set_option(16): Chebyshev-SGS window 0 auto, 1 64x64, 2 64x32, 3 64x32 / 512 threads          // etq_debug_set_option(15): Chebyshev-SGS y_prev loaded in the Q pass             // etq_debug_set_option(14): matrix-free interior rows of the cavity-wind F levels           // etq_debug_set_option(13): programmatic dependent launches inside P2's V-cycle           // etq_debug_set_option(12): smoother with the residual in registers (k_cheb_tile3)
bool g_cheb_tile2 = true;           // etq_set_option(11): leaner temporally blocked smoother (k_cheb_tile2)
bool g_sgs_planar = false;          // etq_set_option(10): Chebyshev-SGS on parity planes with TMA windows
bool g_vc_pdl = true;               // etq_set_option(8): programmatic dependent launches in the V-cycle
bool g_prolong_tile = true;         // etq_set_option(9): tiled nested-Q2 prolongation
bool g_ct_prefetch = true;          // etq_debug_set_option(18): L2 prefetch of a later tile's window in the tiled smoother
bool g_oseen_vc_pdl = true;         // etq_debug_set_option(17): programmatic dependent launches in the F V-cycle of the Oseen preconditioners
void etq_count_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
int64_t etq_launch_total() { return g_launches.load(std::memory_order_relaxed); }

void etq_last_cuda_error(cudaError_t e, const char* file, int line) {
  std::fprintf(stderr, "[etq] CUDA error %s (%d) at %s:%d\n", cudaGetErrorString(e), (int)e, file, line);
}

etq_status dev_alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes > 0 ? bytes : 8);
  if (e != cudaSuccess) {
    etq_last_cuda_error(e, __FILE__, __LINE__);
    *p = nullptr;
    return e == cudaErrorMemoryAllocation ? ETQ_ENOMEM : ETQ_ECUDA;
  }
  return ETQ_OK;
}

void sell_free(Sell& s) {
  if (s.own_perm && s.perm) cudaFree(s.perm);
  if (s.sptr) cudaFree(s.sptr);
  if (s.slen) cudaFree(s.slen);
  if (s.col) cudaFree(s.col);
  if (s.val) cudaFree(s.val);
  if (s.fval) cudaFree(s.fval);
  if (s.skind) cudaFree(s.skind);
  if (s.stoff) cudaFree(s.stoff);
  if (s.stval) cudaFree(s.stval);
  s = Sell{};
}

namespace {
// Order the library's work stream after the caller's stream and vice versa.
struct StreamScope {
  const Problem& P;
  explicit StreamScope(const Problem& p) : P(p) {
    cudaEventRecord(P.ev_in, P.ustream);
    cudaStreamWaitEvent(P.stream, P.ev_in, 0);
  }
  ~StreamScope() {
    cudaEventRecord(P.ev_out, P.stream);
    cudaStreamWaitEvent(P.ustream, P.ev_out, 0);
  }
};

etq_pc_params default_params(const Problem& P) {
  etq_pc_params d;
  std::memset(&d, 0, sizeof(d));
  d.cheb_sgs_steps = 20;
  d.cheb_sgs_lo = 0.0;
  d.lanczos_steps = 60;
  d.smooth_degree = 3;
  d.smooth_hi = 1.6;
  d.smooth_lo = 0.16;
  d.coarse_n = P.oseen ? 32 : 2;
  d.mass_cheb_steps = 10;
  d.use_graphs = 1;
  d.inner_rtol = 1e-10;
  d.inner_maxit = 100;
  d.inner_coarse_n = 16;
  return d;
}

etq_pc_params merge_params(const Problem& P, const etq_pc_params* in) {
  etq_pc_params d = default_params(P);
  if (!in) return d;
  if (in->cheb_sgs_steps > 0) d.cheb_sgs_steps = in->cheb_sgs_steps;
  if (in->cheb_sgs_lo > 0) d.cheb_sgs_lo = in->cheb_sgs_lo;
  if (in->lanczos_steps > 0) d.lanczos_steps = in->lanczos_steps;
  if (in->smooth_degree > 0) d.smooth_degree = in->smooth_degree;
  if (in->smooth_hi > 0) { d.smooth_hi = in->smooth_hi; d.smooth_lo = in->smooth_hi / 10.0; }
  if (in->smooth_lo > 0) d.smooth_lo = in->smooth_lo;
  if (in->coarse_n > 0) d.coarse_n = in->coarse_n;
  if (in->mass_cheb_steps > 0) d.mass_cheb_steps = in->mass_cheb_steps;
  d.use_graphs = in->use_graphs;
  if (in->inner_rtol > 0) d.inner_rtol = in->inner_rtol;
  if (in->inner_maxit > 0) d.inner_maxit = in->inner_maxit;
  if (in->inner_coarse_n > 0) d.inner_coarse_n = in->inner_coarse_n;
  return d;
}

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// deterministic start vector of the automatic Lanczos estimate (splitmix64 -> [-1, 1))
void auto_start_vector(std::vector<double>& v) {
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (auto& x : v) {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x = 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
  }
}
}  // namespace

extern "C" {

const char* etq_status_string(etq_status s) {
  switch (s) {
    case ETQ_OK: return "ok";
    case ETQ_NOT_CONVERGED: return "not converged (maxit reached)";
    case ETQ_EINVAL: return "invalid argument";
    case ETQ_ENOMEM: return "out of device memory";
    case ETQ_ECUDA: return "CUDA error";
    case ETQ_EINDEFINITE: return "indefinite preconditioner (<z,v> < 0)";
    case ETQ_EBREAKDOWN: return "breakdown";
    case ETQ_ENOTSETUP: return "preconditioner not set up";
    case ETQ_ENAN: return "NaN/Inf in scalar recurrence";
    default: return "unknown status";
  }
}

etq_status etq_assemble(const etq_grid* grid, double viscosity, const etq_wind* wind, void* cuda_stream,
                        etq_problem** out) {
  NvtxRange nvtx_("etq_assemble");
  if (!grid || !out) return ETQ_EINVAL;
  if (grid->n < 2 || grid->n > 4096 || (grid->bc != 0 && grid->bc != 1)) return ETQ_EINVAL;
  if (grid->storage < 0 || grid->storage > 2) return ETQ_EINVAL;
  if (grid->enriched != 0 && grid->enriched != 1) return ETQ_EINVAL;
  const bool oseen = wind && wind->kind != 0;
  if (!grid->enriched && oseen) return ETQ_EINVAL;      // plain Q2-Q1: Stokes only
  if (oseen && !(viscosity > 0.0)) return ETQ_EINVAL;
  if (wind && (wind->kind < 0 || wind->kind > 2)) return ETQ_EINVAL;
  etq_problem* h = new (std::nothrow) etq_problem();
  if (!h) return ETQ_ENOMEM;
  Problem& P = h->P;
  P.g = make_geo(grid->n);
  P.bc = grid->bc;
  P.storage = (oseen && wind->kind == 2) ? 2 : grid->storage;   // nodal winds refill explicit values
  P.oseen = oseen;
  P.plain = grid->enriched == 0;
  P.wind = oseen ? wind->kind : 0;
  P.nu = oseen ? viscosity : 1.0;
  P.n_u = 2LL * P.g.nq;
  P.n_p = (int64_t)P.g.nk + P.g.n0;
  P.N = P.n_u + P.n_p;
  P.ustream = reinterpret_cast<cudaStream_t>(cuda_stream);
  P.params = default_params(P);
  auto fail = [&](etq_status s) { etq_destroy(h); return s; };
#define A_CHECK(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) { etq_last_cuda_error(_e, __FILE__, __LINE__); return fail(ETQ_ECUDA); } } while (0)
#define A_TRY(expr) do { etq_status _s = (expr); if (_s < 0) return fail(_s); } while (0)
  {
    // the bandwidth-bound velocity V-cycle (main stream) has the higher priority; the latency-bound
    // pressure chain (aux stream) fills the SMs around it (measured: P2 apply 2.99 -> 2.69 ms, n=1024)
    int lo_prio = 0, hi_prio = 0;
    A_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    A_CHECK(cudaStreamCreateWithPriority(&P.stream, cudaStreamNonBlocking, hi_prio));
    A_CHECK(cudaStreamCreateWithPriority(&P.aux, cudaStreamNonBlocking, lo_prio));
  }
  cudaEvent_t* evs[4] = {&P.ev_in, &P.ev_out, &P.ev_fork, &P.ev_join};
  for (auto e : evs) A_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  A_CHECK(cudaEventCreate(&P.ev_t0));
  A_CHECK(cudaEventCreate(&P.ev_t1));
  A_CHECK(cudaEventRecord(P.ev_in, P.ustream));
  A_CHECK(cudaStreamWaitEvent(P.stream, P.ev_in, 0));
  int64_t nsl = 0;
  A_TRY(build_node_perm(P.g, &P.node_perm, &nsl, P.stream));
  A_TRY(assemble_velocity_op(P.g, P.oseen, P.nu, P.wind, P.node_perm, nsl, &P.Lv, P.stream));
  if (P.storage < 2) A_TRY(mark_implicit(P.g, P.oseen, P.nu, P.wind, P.Lv, P.stream, P.storage == 0));
  if (!P.oseen && P.storage == 0 && P.g.n >= 16 && P.Lv.stval) {   // matrix-free Stokes saddle apply
    A_TRY(class_weights(P.g, P.Lv, &P.so0));
    A_TRY(saddle_weights(P.g, &P.sst, P.stream));
    P.mf_on = true;
    P.bt_mf = true;
  } else if (P.oseen && P.storage == 0 && P.g.n >= 16) {
    // B / B^T do not depend on the wind: their class weights serve the matrix-free B^T of M1; the
    // cavity wind's F is applied matrix-free from nu L class stencils and 1D tables (k_saddle_mf<1>)
    A_TRY(saddle_weights(P.g, &P.sst, P.stream));
    P.bt_mf = true;
    if (P.wind == 1) A_TRY(oseen_tables(P.g, P.nu, &P.so_os, &P.os_tab0, P.stream));
  }
  A_TRY(assemble_bt(P.g, 0, 0, P.node_perm, nsl, &P.BxT1, P.stream));
  A_TRY(assemble_bt(P.g, 1, 0, P.node_perm, nsl, &P.ByT1, P.stream));
  A_TRY(assemble_bt(P.g, 0, 1, P.node_perm, nsl, &P.BxT0, P.stream));
  A_TRY(assemble_bt(P.g, 1, 1, P.node_perm, nsl, &P.ByT0, P.stream));
  A_TRY(assemble_b(P.g, &P.B, P.stream));
  RedSite& rs = P.red[0];
  rs.nslot = RED_SLOTS;
  A_TRY(dalloc(&rs.partials, (size_t)RED_SLOTS * RED_MAXB));
  A_TRY(dalloc(&rs.counter, RED_SLOTS));
  A_CHECK(cudaMemsetAsync(rs.counter, 0, sizeof(unsigned) * RED_SLOTS, P.stream));
  A_TRY(dalloc(&P.dscal, S_COUNT));
  A_CHECK(cudaMemsetAsync(P.dscal, 0, sizeof(double) * S_COUNT, P.stream));
  A_CHECK(cudaMallocHost(&P.hscal, sizeof(double) * S_COUNT));
  A_CHECK(cudaStreamSynchronize(P.stream));
#undef A_CHECK
#undef A_TRY
  *out = h;
  return ETQ_OK;
}

etq_status etq_sizes(const etq_problem* h, int64_t* n_u, int64_t* n_k, int64_t* n_0) {
  if (!h) return ETQ_EINVAL;
  if (n_u) *n_u = h->P.n_u;
  if (n_k) *n_k = h->P.g.nk;
  if (n_0) *n_0 = h->P.g.n0;
  return ETQ_OK;
}

etq_status etq_build_rhs(const etq_problem* h, const double* f_nodal, double* b) {
  if (!h || !b) return ETQ_EINVAL;
  StreamScope sc(h->P);
  ETQ_TRY(build_rhs_dev(h->P, f_nodal, b));
  const Problem& P = h->P;
  if (P.plain)   // plain Q2-Q1: no P0 rows (the reduced right-hand side [f; g1])
    ETQ_CHECK(cudaMemsetAsync(b + P.n_u + P.g.nk, 0, sizeof(double) * P.g.n0, P.stream));
  return ETQ_OK;
}

etq_status etq_apply_saddle(const etq_problem* h, int32_t reduced, const double* x, double* y) {
  if (!h || !x || !y || x == y) return ETQ_EINVAL;
  const Problem& P = h->P;
  StreamScope sc(P);
  launch_saddle_ex(P, reduced != 0 || P.plain, x, y, nullptr, nullptr, 0, nullptr, nullptr, P.stream);
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status etq_precond_setup(etq_problem* h, etq_pc_kind kind, const etq_pc_params* params) {
  NvtxRange nvtx_("etq_precond_setup");
  if (!h) return ETQ_EINVAL;
  Problem& P = h->P;
  StreamScope sc(P);
  const etq_pc_params prm = merge_params(P, params);
  P.params = prm;
  // cached MINRES graphs bake in hierarchy buffers that a new setup may replace
  drop_minres_graphs(P);
  if (P.plain && kind != ETQ_PC_P2_GMG) return ETQ_EINVAL;   // plain Q2-Q1: only the Taylor-Hood P2
  if (kind == ETQ_PC_P3 || kind == ETQ_PC_P1_ITER) {
    if (P.oseen) return ETQ_EINVAL;
    if (!is_pow2(P.g.n) || !is_pow2(prm.coarse_n) || prm.coarse_n > P.g.n || !is_pow2(prm.inner_coarse_n))
      return ETQ_EINVAL;
    if (P.mg.built) free_hierarchy(P.mg);
    ETQ_TRY(build_hierarchy(P, P.mg, prm.coarse_n, prm.smooth_lo, prm.smooth_hi, prm.smooth_degree));
    ETQ_TRY(exact_mass_setup(P));
    if (kind == ETQ_PC_P1_ITER) ETQ_TRY(vel_iter_setup(P));
    ETQ_CHECK(cudaStreamSynchronize(P.stream));
    return ETQ_OK;
  }
  if (kind == ETQ_PC_P1_EXACT) {
    if (P.oseen || P.g.nq > 4225) return ETQ_EINVAL;   // dense exact solves: n <= 32
    if (!P.p1.Ainv) {
      ETQ_TRY(dalloc(&P.p1.Ainv, (size_t)P.g.nq * P.g.nq));
      ETQ_TRY(dalloc(&P.p1.MQinv, (size_t)P.n_p * P.n_p));
      ETQ_TRY(dalloc(&P.p1.tmp, 2 * (size_t)P.n_p));
    }
    ETQ_TRY(dense_from_sell(P.Lv, P.g.nq, P.p1.Ainv, P.stream));
    ETQ_TRY(dense_inverse_spd(P.p1.Ainv, P.g.nq, P.stream));
    ETQ_TRY(p1_build_mass_inverse(P.g, P.p1.MQinv, P.stream));
    ETQ_CHECK(cudaStreamSynchronize(P.stream));
    P.p1.ready = true;
    return ETQ_OK;
  }
  if (kind == ETQ_PC_P2_GMG) {
    if (P.oseen) return ETQ_EINVAL;
    if (!is_pow2(P.g.n) || !is_pow2(prm.coarse_n) || prm.coarse_n > P.g.n) return ETQ_EINVAL;
    // a failed re-setup must not leave the previous setup marked ready on a rebuilt hierarchy
    P.p2_ready = false;
    P.pm.ready = false;
    if (P.mg.built) free_hierarchy(P.mg);
    ETQ_TRY(build_hierarchy(P, P.mg, prm.coarse_n, prm.smooth_lo, prm.smooth_hi, prm.smooth_degree));
    if (P.plain) {   // plain Q2-Q1: the pressure block is Chebyshev-Jacobi on Q_k (no M_Q, no k)
      if (prm.mass_cheb_steps < 1) return ETQ_EINVAL;
      if (!P.plain_w) ETQ_TRY(dalloc(&P.plain_w, 3 * (size_t)P.g.nk));
      P.p2_ready = true;
      drop_minres_graphs(P);
      ETQ_CHECK(cudaStreamSynchronize(P.stream));
      return ETQ_OK;
    }
    ETQ_TRY(mass_pc_alloc(P));
    P.pm.m = prm.cheb_sgs_steps;
    double a = prm.cheb_sgs_lo;
    if (!(a > 0.0)) {
      std::vector<double> v0(P.n_p);
      auto_start_vector(v0);
      double* dv;
      ETQ_TRY(dalloc(&dv, P.n_p));
      ETQ_CHECK(cudaMemcpy(dv, v0.data(), sizeof(double) * P.n_p, cudaMemcpyHostToDevice));
      double lam = 0.0;
      const etq_status ls = lanczos_sgs_lo(P, dv, std::min<int64_t>(prm.lanczos_steps, P.n_p / 2), &lam);
      cudaFree(dv);
      if (ls < 0) return ls;
      const double floor_ = 2.0 / ((double)P.pm.m * P.pm.m);   // reading R7: a = max(lam, 2/m^2)
      a = lam > floor_ ? lam : floor_;
    }
    if (!(a > 0.0 && a < 1.0)) return ETQ_EINVAL;
    P.pm.a = a;
    P.pm.ready = true;
    P.p2_ready = true;
    drop_minres_graphs(P);
    ETQ_CHECK(cudaStreamSynchronize(P.stream));
    return ETQ_OK;
  }
  if (kind == ETQ_PC_OSEEN_M1 || kind == ETQ_PC_OSEEN_PCD1 || kind == ETQ_PC_OSEEN_M2 || kind == ETQ_PC_OSEEN_LSC) {
    if (!P.oseen) return ETQ_EINVAL;
    if (!is_pow2(P.g.n)) return ETQ_EINVAL;
    if (kind == ETQ_PC_OSEEN_M1) {   // Chebyshev-SGS for the -(1/nu) M_Q~ block
      ETQ_TRY(mass_pc_alloc(P));
      P.pm.m = prm.cheb_sgs_steps;
      double a = prm.cheb_sgs_lo;
      if (!(a > 0.0)) a = 2.0 / ((double)P.pm.m * P.pm.m);
      P.pm.a = a;
      P.pm.ready = true;
    }
    ETQ_TRY(oseen_setup(P, kind));
    if (P.wind == 2) ETQ_TRY(picard_refresh(P));   // new levels / F1 get the current nodal wind
    if (P.gmres_graph) { cudaGraphExecDestroy(P.gmres_graph); P.gmres_graph = nullptr; }
    ETQ_CHECK(cudaStreamSynchronize(P.stream));
    return ETQ_OK;
  }
  return ETQ_EINVAL;
}

etq_status etq_apply_precond(const etq_problem* h, etq_pc_kind kind, const double* r, double* z) {
  if (!h || !r || !z || r == z) return ETQ_EINVAL;
  const Problem& P = h->P;
  StreamScope sc(P);
  return precond_apply_ex(P, kind, r, z, nullptr, nullptr, nullptr, nullptr, P.stream);
}

etq_status etq_apply_vcycle(const etq_problem* h, etq_pc_kind kind, const double* r_u, double* z_u) {
  if (!h || !r_u || !z_u) return ETQ_EINVAL;
  const Problem& P = h->P;
  if (kind == ETQ_PC_P1_EXACT || !P.mg.built) return ETQ_ENOTSETUP;
  StreamScope sc(P);
  return vcycle_apply_ex(P, P.mg, r_u, z_u, nullptr, 0, nullptr, nullptr, nullptr, P.stream);
}

etq_status etq_apply_mass_pc(const etq_problem* h, const double* r_p, double* z_p) {
  if (!h || !r_p || !z_p) return ETQ_EINVAL;
  const Problem& P = h->P;
  if (!P.pm.ready) return ETQ_ENOTSETUP;
  StreamScope sc(P);
  return mass_pc_apply_ex(P, r_p, z_p, &P.red[0], 2, nullptr, nullptr, nullptr, P.stream);
}

etq_status etq_apply_mass_exact(const etq_problem* h, const double* r_p, double* z_p, int32_t* cg_iterations) {
  if (!h || !r_p || !z_p || r_p == z_p) return ETQ_EINVAL;
  const Problem& P = h->P;
  if (!P.mx.ready) return ETQ_ENOTSETUP;
  StreamScope sc(P);
  double i0, c0, i1, c1;
  ETQ_TRY(pcg_stats(P, 0, &i0, &c0));
  ETQ_TRY(exact_mass_apply(P, r_p, z_p, nullptr, 0, nullptr, nullptr, nullptr, P.stream));
  ETQ_CHECK(cudaStreamSynchronize(P.stream));
  ETQ_TRY(pcg_stats(P, 0, &i1, &c1));
  if (cg_iterations) *cg_iterations = (int32_t)(i1 - i0);
  return ETQ_OK;
}

etq_status etq_inner_stats(const etq_problem* h, int32_t which, double* iterations, double* solves) {
  if (!h || !iterations || !solves || which < 0 || which > 1) return ETQ_EINVAL;
  cudaStreamSynchronize(h->P.stream);
  return pcg_stats(h->P, which, iterations, solves);
}

etq_status etq_apply_mass(const etq_problem* h, const double* x_p, double* y_p) {
  if (!h || !x_p || !y_p || x_p == y_p) return ETQ_EINVAL;
  const Problem& P = h->P;
  StreamScope sc(P);
  mass_apply(P.g, x_p, y_p, P.stream);
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status etq_sgs_sweep(const etq_problem* h, const double* r_p, const double* y_p, double* z_p) {
  if (!h || !r_p || !z_p) return ETQ_EINVAL;
  Problem& P = const_cast<Problem&>(h->P);
  ETQ_TRY(mass_pc_alloc(P));
  StreamScope sc(P);
  sgs_sweep_dev(P.g, r_p, y_p, z_p, P.pm.t, P.stream);
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status etq_estimate_sgs_lo(etq_problem* h, const double* v0, int32_t steps, double* lam) {
  if (!h || !v0 || !lam || steps < 1) return ETQ_EINVAL;
  StreamScope sc(h->P);
  return lanczos_sgs_lo(h->P, v0, steps, lam);
}

etq_status etq_get_cheb_sgs_lo(const etq_problem* h, double* a) {
  if (!h || !a) return ETQ_EINVAL;
  if (!h->P.pm.ready) return ETQ_ENOTSETUP;
  *a = h->P.pm.a;
  return ETQ_OK;
}

etq_status etq_minres_solve(etq_problem* h, etq_pc_kind kind, const double* b, double* x, double rtol,
                            int32_t maxit, etq_report* report) {
  if (!h || !b || !x || !(rtol > 0.0) || maxit < 1) return ETQ_EINVAL;
  if (kind != ETQ_PC_P1_EXACT && kind != ETQ_PC_P2_GMG && kind != ETQ_PC_P3 && kind != ETQ_PC_P1_ITER)
    return ETQ_EINVAL;
  Problem& P = h->P;
  StreamScope sc(P);
  return minres_run(P, kind, b, x, rtol, maxit, report);
}

etq_status etq_minres_solve_host(etq_problem* h, etq_pc_kind kind, const double* b_host, double* x_host,
                                 double rtol, int32_t maxit, etq_report* report) {
  if (!h || !b_host || !x_host || !(rtol > 0.0) || maxit < 1) return ETQ_EINVAL;
  if (kind != ETQ_PC_P1_EXACT && kind != ETQ_PC_P2_GMG && kind != ETQ_PC_P3 && kind != ETQ_PC_P1_ITER)
    return ETQ_EINVAL;
  Problem& P = h->P;
  // persistent device staging buffers (the cached MINRES graphs stay valid across calls)
  if (!P.kv[7]) ETQ_TRY(dalloc(&P.kv[7], P.N));
  if (!P.kv[8]) ETQ_TRY(dalloc(&P.kv[8], P.N));
  double* db = P.kv[7];
  double* dx = P.kv[8];
  StreamScope sc(P);
  ETQ_CHECK(cudaMemcpyAsync(db, b_host, sizeof(double) * P.N, cudaMemcpyHostToDevice, P.stream));
  ETQ_CHECK(cudaMemcpyAsync(dx, x_host, sizeof(double) * P.N, cudaMemcpyHostToDevice, P.stream));
  const etq_status s = minres_run(P, kind, db, dx, rtol, maxit, report);
  if (s >= 0) {
    ETQ_CHECK(cudaMemcpyAsync(x_host, dx, sizeof(double) * P.N, cudaMemcpyDeviceToHost, P.stream));
    ETQ_CHECK(cudaStreamSynchronize(P.stream));
  }
  return s;
}

etq_status etq_apply_saddle_f32(etq_problem* h, int32_t reduced, const float* x, float* y) {
  if (!h || !x || !y || (const void*)x == (const void*)y) return ETQ_EINVAL;
  Problem& P = h->P;
  ETQ_TRY(ensure_f32(P));
  StreamScope sc(P);
  launch_saddle_f32(P, reduced != 0, x, y, P.stream);
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status etq_apply_vcycle_f32(etq_problem* h, const float* r_u, float* z_u) {
  if (!h || !r_u || !z_u) return ETQ_EINVAL;
  Problem& P = h->P;
  if (!P.mg.built || P.mg.kind != 0 || P.oseen) return ETQ_ENOTSETUP;
  ETQ_TRY(ensure_f32(P));
  StreamScope sc(P);
  return vcycle_f32(P, r_u, z_u, P.stream);
}

etq_status etq_apply_pcd_schur(const etq_problem* h, const double* r_p1, double* z_p1) {
  if (!h || !r_p1 || !z_p1) return ETQ_EINVAL;
  const Problem& P = h->P;
  StreamScope sc(P);
  return pcd_schur_apply(P, r_p1, z_p1, P.stream);
}

etq_status etq_gmres_solve(etq_problem* h, int32_t reduced, etq_pc_kind kind, const double* b, double* x,
                           double rtol, int32_t restart, int32_t maxit, etq_report* report) {
  if (!h || !b || !x || !(rtol > 0.0) || restart < 1 || restart > ETQ_MAX_RESTART || maxit < 1) return ETQ_EINVAL;
  if (kind != ETQ_PC_OSEEN_M1 && kind != ETQ_PC_OSEEN_PCD1 && kind != ETQ_PC_OSEEN_M2 && kind != ETQ_PC_OSEEN_LSC)
    return ETQ_EINVAL;
  if ((kind == ETQ_PC_OSEEN_M2 || kind == ETQ_PC_OSEEN_LSC) && reduced) return ETQ_EINVAL;   // full system only
  if (kind == ETQ_PC_OSEEN_PCD1 && !reduced) return ETQ_EINVAL;   // PCD1 preconditions the reduced system
  Problem& P = h->P;
  StreamScope sc(P);
  const double* bb = b;
  if (reduced) {
    double* bred;
    ETQ_TRY(make_reduced_rhs(P, b, &bred));
    bb = bred;
  }
  // tolerance relative to ||b|| (reading R14): computed on the device inside gmres_run
  const double nb = host_norm(P, bb, P.N);
  return gmres_run(P, reduced != 0, kind, bb, x, rtol * nb, restart, maxit, report, nullptr);
}

etq_status etq_two_stage_solve(etq_problem* h, const double* b, double* x, double eta, double c, int32_t restart,
                               int32_t maxit, etq_report* st1, etq_report* st2, double bound_out[2]) {
  if (!h || !b || !x || !(eta > 0.0) || !(c > 0.0) || restart < 1 || restart > ETQ_MAX_RESTART || maxit < 1)
    return ETQ_EINVAL;
  Problem& P = h->P;
  StreamScope sc(P);
  return two_stage_run(P, b, x, eta, c, restart, maxit, st1, st2, bound_out);
}

etq_status etq_set_wind(etq_problem* h, const double* w) {
  if (!h || !w) return ETQ_EINVAL;
  Problem& P = h->P;
  StreamScope sc(P);
  return picard_set_wind(P, w);
}

etq_status etq_picard_solve(etq_problem* h, int32_t steps, double eta, double c, int32_t restart, int32_t maxit,
                            double* x, int32_t* its, double* res, double* ms_total) {
  if (!h || !x || steps < 0 || !(eta > 0.0) || !(c > 0.0) || restart < 1 || restart > ETQ_MAX_RESTART || maxit < 1)
    return ETQ_EINVAL;
  Problem& P = h->P;
  StreamScope sc(P);
  return picard_run(P, steps, eta, c, restart, maxit, x, its, res, ms_total);
}

etq_status etq_export_operator(const etq_problem* h, int32_t which, int32_t level, int64_t* nrows, int64_t* nnz,
                               int64_t* rowptr, int32_t* col, double* val) {
  if (!h || !nrows || !nnz) return ETQ_EINVAL;
  const Problem& P = h->P;
  std::vector<std::pair<const Sell*, std::pair<int64_t, int64_t>>> parts;   // (matrix, (row offset, col offset))
  int64_t R = 0;
  if (which == 0) {
    if (level < 0) return ETQ_EINVAL;
    if (level == 0) parts.push_back({&P.Lv, {0, 0}});
    else {
      if (!P.mg.built || level >= (int)P.mg.lv.size()) return ETQ_EINVAL;
      parts.push_back({&P.mg.lv[level].A, {0, 0}});
    }
    R = parts[0].first->nrows;
  } else if (which == 1) {
    parts.push_back({&P.B, {0, 0}});
    R = P.n_p;
  } else if (which == 3) {
    if (!P.apH.built || level < 0 || level >= (int)P.apH.lv.size()) return ETQ_EINVAL;
    parts.push_back({&P.apH.lv[level].A, {0, 0}});
    R = P.apH.lv[level].A.nrows;
  } else if (which == 6) {
    if (!P.lp.H.built || level < 0 || level >= (int)P.lp.H.lv.size()) return ETQ_EINVAL;
    parts.push_back({&P.lp.H.lv[level].A, {0, 0}});
    R = P.lp.H.lv[level].A.nrows;
  } else if (which == 5) {
    if (!P.mx.sH.built || level < 0 || level >= (int)P.mx.sH.lv.size()) return ETQ_EINVAL;
    parts.push_back({&P.mx.sH.lv[level].A, {0, 0}});
    R = P.mx.sH.lv[level].A.nrows;
  } else if (which == 4) {
    if (!P.pcd_ready) return ETQ_EINVAL;
    parts.push_back({&P.F1, {0, 0}});
    R = P.F1.nrows;
  } else if (which == 2) {
    parts.push_back({&P.BxT1, {0, 0}});
    parts.push_back({&P.BxT0, {0, P.g.nk}});
    parts.push_back({&P.ByT1, {P.g.nq, 0}});
    parts.push_back({&P.ByT0, {P.g.nq, P.g.nk}});
    R = P.n_u;
  } else {
    return ETQ_EINVAL;
  }
  cudaStreamSynchronize(P.stream);
  std::vector<std::vector<std::pair<int32_t, double>>> rows(R);
  for (auto& pr : parts) {
    const Sell& S = *pr.first;
    std::vector<int64_t> sptr(S.nslices + 1);
    std::vector<int> slen(S.nslices), perm(S.nslices * SELL_C), c(S.nnz_stored);
    std::vector<double> v(S.nnz_stored);
    ETQ_CHECK(cudaMemcpy(sptr.data(), S.sptr, sizeof(int64_t) * (S.nslices + 1), cudaMemcpyDeviceToHost));
    ETQ_CHECK(cudaMemcpy(slen.data(), S.slen, sizeof(int) * S.nslices, cudaMemcpyDeviceToHost));
    if (S.perm) ETQ_CHECK(cudaMemcpy(perm.data(), S.perm, sizeof(int) * S.nslices * SELL_C, cudaMemcpyDeviceToHost));
    ETQ_CHECK(cudaMemcpy(c.data(), S.col, sizeof(int) * S.nnz_stored, cudaMemcpyDeviceToHost));
    ETQ_CHECK(cudaMemcpy(v.data(), S.val, sizeof(double) * S.nnz_stored, cudaMemcpyDeviceToHost));
    for (int64_t s = 0; s < S.nslices; ++s)
      for (int l = 0; l < SELL_C; ++l) {
        const int64_t t = s * SELL_C + l;
        const int64_t row = S.perm ? perm[t] : (t < S.nrows ? t : -1);
        if (row < 0) continue;
        for (int k = 0; k < slen[s]; ++k) {
          const int64_t e = sptr[s] + l + (int64_t)k * SELL_C;
          if (v[e] != 0.0) rows[row + pr.second.first].push_back({(int32_t)(c[e] + pr.second.second), v[e]});
        }
      }
  }
  int64_t total = 0;
  for (auto& r : rows) total += (int64_t)r.size();
  *nrows = R; *nnz = total;
  if (!rowptr) return ETQ_OK;
  int64_t k = 0;
  for (int64_t i = 0; i < R; ++i) {
    rowptr[i] = k;
    for (auto& e : rows[i]) { if (col) col[k] = e.first; if (val) val[k] = e.second; ++k; }
  }
  rowptr[R] = k;
  return ETQ_OK;
}

etq_status etq_est_minres(const double* delta, const double* gamma, int32_t k, double* gamma2) {
  if (!delta || !gamma2 || k < 0 || (k > 1 && !gamma)) return ETQ_EINVAL;
  *gamma2 = std::nan("");
  if (k == 0) return ETQ_OK;
  auto off = [&](int i) { return gamma[i]; };   // between rows i and i+1
  auto count_below = [&](double x) {             // Sturm count of eigenvalues < x
    int c = 0; double d = 1.0;
    for (int i = 0; i < k; ++i) {
      d = delta[i] - x - (i > 0 ? off(i - 1) * off(i - 1) / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0) ++c;
    }
    return c;
  };
  const int nneg = count_below(0.0);
  if (nneg == 0) return ETQ_OK;
  double lo = 0.0;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::fabs(off(i - 1)) : 0.0) + (i < k - 1 ? std::fabs(off(i)) : 0.0);
    lo = std::fmin(lo, delta[i] - r);
  }
  double hi = 0.0;
  for (int it = 0; it < 200; ++it) {   // the nneg-th smallest eigenvalue = largest negative one
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) >= nneg) hi = mid; else lo = mid;
  }
  const double mu = 0.5 * (lo + hi);
  *gamma2 = mu * (mu - 1.0);
  return ETQ_OK;
}

etq_status etq_launch_count(int64_t* count) {
  if (count) *count = etq_launch_total();
  return ETQ_OK;
}

etq_status etq_time_kernel(etq_problem* h, int32_t which, int32_t reps, double* ms, double* bytes) {
  if (!h || reps < 1 || !ms || !bytes) return ETQ_EINVAL;
  Problem& P = h->P;
  if (which < 0 || which > 12) return ETQ_EINVAL;
  if ((which >= 2 && which <= 6 && which != 5) && !P.p2_ready) return ETQ_ENOTSETUP;
  if (which >= 10 && !P.p2_ready) return ETQ_ENOTSETUP;
  if (which >= 7 && which <= 9 && !P.mx.ready) return ETQ_ENOTSETUP;
  if (which >= 5) {
    ETQ_TRY(ensure_f32(P));
    if (!P.tkf) {
      ETQ_TRY(dalloc(&P.tkf, 2 * (size_t)P.N));
      ETQ_CHECK(cudaMemset(P.tkf, 0, sizeof(float) * 2 * (size_t)P.N));
    }
  }
  if (!P.tk) {
    ETQ_TRY(dalloc(&P.tk, 3 * (size_t)P.N));
    std::vector<double> v(P.N);
    auto_start_vector(v);
    for (int i = 0; i < 3; ++i)
      ETQ_CHECK(cudaMemcpy(P.tk + (size_t)i * P.N, v.data(), sizeof(double) * P.N, cudaMemcpyHostToDevice));
  }
  if (which == 1 && !P.mg.built) return ETQ_ENOTSETUP;
  StreamScope sc(P);
  cudaStream_t st = P.stream;
  double* a = P.tk; double* b = P.tk + P.N; double* c = P.tk + 2 * P.N;
  auto one = [&](int k) -> etq_status {
    switch (which) {
      case 0: launch_saddle_ex(P, false, a, b, nullptr, nullptr, 0, nullptr, nullptr, st); break;
      case 1: cheb_step_level0(P, (k & 1) ? b : a, (k & 1) ? a : b, st); break;
      case 2: ETQ_TRY(vcycle_apply_ex(P, P.mg, a, b, nullptr, 0, nullptr, nullptr, nullptr, st)); break;
      case 3: ETQ_TRY(mass_pc_apply_ex(P, a + P.n_u, b + P.n_u, &P.red[0], 2, nullptr, nullptr, nullptr, st)); break;
      case 4: ETQ_TRY(precond_apply_ex(P, ETQ_PC_P2_GMG, a, c, nullptr, nullptr, nullptr, nullptr, st)); break;
      case 5: launch_saddle_f32(P, false, P.tkf, P.tkf + P.N, st); break;
      case 6: ETQ_TRY(vcycle_f32(P, P.tkf, P.tkf + P.N, st)); break;
      case 7: ETQ_TRY(exact_mass_apply(P, a + P.n_u, b + P.n_u, nullptr, 0, nullptr, nullptr, nullptr, st)); break;
      case 8: ETQ_TRY(vcycle_apply_ex(P, P.mx.sH, a + P.n_u, b + P.n_u, nullptr, 0, nullptr, nullptr, nullptr, st)); break;
      case 9: ETQ_TRY(precond_apply_ex(P, ETQ_PC_P3, a, c, nullptr, nullptr, nullptr, nullptr, st)); break;
      case 10: sgs_step_bench(P, a + P.n_u, b + P.n_u, c + P.n_u, (k & 1) ? b + P.n_u : c + P.n_u, st); break;
      case 11: ETQ_TRY(cheb_tile_bench(P, false, a, nullptr, b, c, st)); break;
      case 12: ETQ_TRY(cheb_tile_bench(P, true, a, b, nullptr, nullptr, st)); break;
    }
    return ETQ_OK;
  };
  cudaGraphExec_t gx = nullptr;
  if (which == 7 || which == 9) {   // the inner CG loops are graph while-nodes: time replays of one graph
    cudaGraph_t g;
    ETQ_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    etq_status s1 = one(0);
    cudaError_t e = cudaStreamEndCapture(st, &g);
    if (s1 < 0) return s1;
    ETQ_CHECK(e);
    cudaError_t ei = cudaGraphInstantiate(&gx, g, 0);
    cudaGraphDestroy(g);
    ETQ_CHECK(ei);
    ETQ_CHECK(cudaGraphLaunch(gx, st));   // warm-up
  } else {
    ETQ_TRY(one(0));   // warm-up
  }
  ETQ_CHECK(cudaEventRecord(P.ev_t0, st));
  for (int k = 0; k < reps; ++k) {
    if (gx) ETQ_CHECK(cudaGraphLaunch(gx, st));
    else ETQ_TRY(one(k));
  }
  ETQ_CHECK(cudaEventRecord(P.ev_t1, st));
  ETQ_CHECK(cudaEventSynchronize(P.ev_t1));
  float t = 0.f;
  ETQ_CHECK(cudaEventElapsedTime(&t, P.ev_t0, P.ev_t1));
  *ms = (double)t / reps;
  if (gx) cudaGraphExecDestroy(gx);
  const double nnz_all = (double)(P.Lv.nnz + P.BxT1.nnz + P.ByT1.nnz + P.BxT0.nnz + P.ByT0.nnz + P.B.nnz);
  switch (which) {
    case 0:   // matrix-free apply: x in, y out; stored rows: every stored value / index once + x + y
      *bytes = (P.mf_on && g_saddle_mf) ? 16.0 * P.N
               : 12.0 * nnz_all - 4.0 * P.Lv.nnz_implicit - 8.0 * P.Lv.nnz_implicit_vals + 4.0 * P.Lv.nslices * SELL_C + 16.0 * P.N;
      break;
    case 1: *bytes = cheb_step_bytes(P.mg.lv[0]); break;
    case 2: *bytes = vcycle_bytes(P.mg); break;
    case 3: *bytes = mass_pc_bytes(P); break;
    case 4: *bytes = vcycle_bytes(P.mg) + mass_pc_bytes(P); break;   // both branches
    case 5: *bytes = 8.0 * nnz_all + 4.0 * P.Lv.nslices * SELL_C + 8.0 * P.N; break;
    case 6: *bytes = vcycle_bytes_f32(P.mg); break;
    case 10: *bytes = 32.0 * (double)P.n_p; break;            // r, y, yp in; out
    case 11: *bytes = 48.0 * (double)P.g.nq; break;           // b in; x, r out (2 components)
    case 12: *bytes = 64.0 * (double)P.g.nq; break;           // x, b in; x, d out (2 components)
    default: *bytes = 0.0;
  }
  return ETQ_OK;
}

etq_status etq_debug_set_option(int32_t option, int32_t value) {
  if (option == 0) { g_cheb_tile_enabled = value != 0; return ETQ_OK; }
  if (option == 1) { if (value < 2) return ETQ_EINVAL; g_cheb_tile_min_n = value; return ETQ_OK; }
  if (option == 2) { g_saddle_mf = value != 0; return ETQ_OK; }
  if (option == 3) { g_minres_devloop = value != 0; return ETQ_OK; }
  if (option == 4) { g_sgs_high_prio = value != 0; return ETQ_OK; }
  if (option == 5) { g_tail_sm = value != 0; return ETQ_OK; }
  if (option == 6) { g_saddle_tile = value != 0; return ETQ_OK; }
  if (option == 7) { g_sgs_pdl = value != 0; return ETQ_OK; }
  if (option == 8) { g_vc_pdl = value != 0; return ETQ_OK; }
  if (option == 9) { g_prolong_tile = value != 0; return ETQ_OK; }
  if (option == 10) { g_sgs_planar = value != 0; return ETQ_OK; }
  if (option == 11) { g_cheb_tile2 = value != 0; return ETQ_OK; }
  if (option == 12) { g_cheb_tile3 = value != 0; return ETQ_OK; }
  if (option == 13) { g_p2_vc_pdl = value != 0; return ETQ_OK; }
  if (option == 14) { g_oseen_mf = value != 0; return ETQ_OK; }
  if (option == 15) { g_sgs_yp_ldg = value != 0; return ETQ_OK; }
  if (option == 18) { g_ct_prefetch = value != 0; return ETQ_OK; }
  if (option == 17) { g_oseen_vc_pdl = value != 0; return ETQ_OK; }
  if (option == 16) { if (value < 0 || value > 3) return ETQ_EINVAL; g_sgs_window = value; return ETQ_OK; }
  return ETQ_EINVAL;
}

void etq_destroy(etq_problem* h) {
  if (!h) return;
  Problem& P = h->P;
  if (P.stream) cudaStreamSynchronize(P.stream);
  for (int g = 0; g < 2; ++g) if (P.minres_graph[g]) cudaGraphExecDestroy(P.minres_graph[g]);
  if (P.minres_wgraph) cudaGraphExecDestroy(P.minres_wgraph);
  if (P.wcs) cudaStreamDestroy(P.wcs);
  if (P.wside) cudaStreamDestroy(P.wside);
  if (P.ev_wfork) cudaEventDestroy(P.ev_wfork);
  if (P.ev_wjoin) cudaEventDestroy(P.ev_wjoin);
  free_hierarchy(P.mg);
  exact_free(P);
  oseen_free(P);
  cudaFree(P.wnod); cudaFree(P.lv_lap); cudaFree(P.f1_lap); cudaFree(P.os_tab0);
  P.Lv.perm = nullptr; P.BxT1.perm = nullptr; P.ByT1.perm = nullptr; P.BxT0.perm = nullptr; P.ByT0.perm = nullptr;
  sell_free(P.Lv); sell_free(P.BxT1); sell_free(P.ByT1); sell_free(P.BxT0); sell_free(P.ByT0); sell_free(P.B);
  if (P.node_perm) cudaFree(P.node_perm);
  cudaFree(P.p1.Ainv); cudaFree(P.p1.MQinv); cudaFree(P.p1.tmp);
  cudaFree(P.pm.t); cudaFree(P.pm.y0); cudaFree(P.pm.y1); cudaFree(P.pm.rr);
  cudaFree(P.pm.rp); cudaFree(P.pm.yp[0]); cudaFree(P.pm.yp[1]);
  cudaFree(P.plain_w);
  cudaFree(P.red[0].partials); cudaFree(P.red[0].counter);
  cudaFree(P.dscal); cudaFree(P.dhist); cudaFree(P.tk); cudaFree(P.tkf);
  if (P.hscal) cudaFreeHost(P.hscal);
  for (int i = 0; i < 10; ++i) cudaFree(P.kv[i]);
  cudaEvent_t evs[6] = {P.ev_in, P.ev_out, P.ev_fork, P.ev_join, P.ev_t0, P.ev_t1};
  for (auto e : evs) if (e) cudaEventDestroy(e);
  if (P.aux) cudaStreamDestroy(P.aux);
  if (P.stream) cudaStreamDestroy(P.stream);
  delete h;
}

}  // extern "C"
