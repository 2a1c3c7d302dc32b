// etq_internal.cuh — internal data structures and device helpers of libetq (sm_100a).
//
// Layout in HBM:
//   * SELL-32 sliced ELLPACK: rows are processed by one thread each, 32 rows (one warp) per
//     slice; entry k of lane l of slice s lives at sptr[s] + 32 k + l, so a warp reads 256 B of
//     values and 128 B of column indices per k, fully coalesced.  Row order inside the slices is
//     a permutation `perm` grouping Q2 nodes by class (i mod 2, j mod 2), so all rows of a slice
//     have the same stencil width (25 / 15 / 15 / 9 for the Laplacian) and padding is confined
//     to slices that touch the boundary.
//   * The scalar velocity operator (L or F_s) is stored ONCE and applied to both components.
//   * B^T is stored as four SELL blocks over the velocity-node permutation (x/y component times
//     Q1/P0 pressure part) so the reduced Taylor-Hood operator can skip the P0 part.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <vector>
#include <string>
#include "../../include/etq.h"
#include <nvtx3/nvToolsExt.h>

// NVTX range for a solver phase / kernel family (header-only NVTX v3: no link dependency; a
// profiler such as Nsight Systems picks the ranges up through its injection library).  The
// ranges cover host time: eager launches, graph captures and graph launches.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

#define ETQ_CHECK(call)                                                        \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      etq_last_cuda_error(_e, __FILE__, __LINE__);                             \
      return (_e == cudaErrorMemoryAllocation) ? ETQ_ENOMEM : ETQ_ECUDA;       \
    }                                                                          \
  } while (0)

#define ETQ_TRY(expr)                                                          \
  do {                                                                         \
    etq_status _s = (expr);                                                    \
    if (_s < 0) return _s;                                                     \
  } while (0)

void etq_last_cuda_error(cudaError_t e, const char* file, int line);
void etq_count_launch(int64_t k = 1);
extern bool g_cheb_tile_enabled;          // api.cu; etq_set_option(0)
extern int g_cheb_tile_min_n;             // api.cu; etq_set_option(1)
extern bool g_minres_devloop;             // api.cu; etq_set_option(3)
extern bool g_saddle_mf;                  // api.cu; etq_set_option(2)
extern bool g_sgs_high_prio;              // api.cu; etq_set_option(4)
extern bool g_tail_sm;                    // api.cu; etq_set_option(5)
extern bool g_saddle_tile;                // api.cu; etq_set_option(6)
extern bool g_sgs_pdl;                    // api.cu; etq_set_option(7)
extern bool g_sgs_planar;                 // api.cu; etq_set_option(10)
extern int g_sgs_window;                  // api.cu; etq_debug_set_option(16)
extern bool g_sgs_yp_ldg;                 // api.cu; etq_debug_set_option(15)
extern bool g_oseen_mf;                   // api.cu; etq_debug_set_option(14)
extern bool g_p2_vc_pdl;                  // api.cu; etq_debug_set_option(13)
extern bool g_cheb_tile3;                 // api.cu; etq_debug_set_option(12)
extern bool g_cheb_tile2;                 // api.cu; etq_set_option(11)
extern bool g_vc_pdl;                     // api.cu; etq_set_option(8)
extern bool g_ct_prefetch;                // api.cu; etq_debug_set_option(18)
extern bool g_oseen_vc_pdl;               // api.cu; etq_debug_set_option(17)
extern bool g_prolong_tile;               // api.cu; etq_set_option(9)

constexpr int SELL_C = 32;           // slice height = warp size
constexpr int RED_BLOCKS = 592;      // 4 x 148 SMs: grid of plain reduction kernels
constexpr int RED_MAXB = 8192;       // max blocks of any reducing kernel
constexpr int RED_SLOTS = 16;        // reduction slots per site (see solvers.cu for the map)

// ---------------------------------------------------------------- SELL-32
struct Sell {
  int64_t nrows = 0;       // logical rows
  int64_t nslices = 0;
  int64_t nnz_stored = 0;  // padded entries
  int64_t nnz = 0;         // true entries
  int* perm = nullptr;     // [nslices*32] row id or -1 (may be shared, not owned)
  bool own_perm = false;
  int64_t* sptr = nullptr; // [nslices+1]
  int* slen = nullptr;     // [nslices]
  int* col = nullptr;      // [nnz_stored]
  double* val = nullptr;   // [nnz_stored]
  float* fval = nullptr;   // optional fp32 copy of val (c5 sweep)
  // implicit column indices (velocity operators): slice s with skind[s] = c + 1 holds rows of node
  // class c with the full interior stencil, so col = row + stoff[c * 32 + k] and col[] is not read
  //   skind[s] = c + 5: additionally every value equals stval[c * 32 + k] bitwise (translation-
  //   invariant interior rows), so val[] is not read either
  int8_t* skind = nullptr; // [nslices] or nullptr
  int* stoff = nullptr;    // [4 * 32] stencil offsets per class
  double* stval = nullptr; // [4 * 32] stencil values per class (Stokes), or nullptr
  int64_t nnz_implicit = 0;        // entries without stored indices
  int64_t nnz_implicit_vals = 0;   // entries without stored values
};

// ---------------------------------------------------------------- grid geometry
struct Geo {
  int n;        // elements per side
  int m;        // 2n+1 Q2 nodes per side
  int nq;       // m*m
  int nk;       // (n+1)^2
  int n0;       // n^2
  double h;     // 2/n
};

inline Geo make_geo(int n) {
  Geo g; g.n = n; g.m = 2 * n + 1; g.nq = g.m * g.m; g.nk = (n + 1) * (n + 1); g.n0 = n * n;
  g.h = 2.0 / n; return g;
}

// ---------------------------------------------------------------- deterministic reductions
// A reduction "site" owns RED_BLOCKS partial sums per slot and a completion counter; the last
// block to finish sums the partials in fixed order (no fp64 atomics on result paths).
struct RedSite {
  double* partials = nullptr;   // [nslot * RED_BLOCKS]
  unsigned* counter = nullptr;  // [1]
  int nslot = 0;
};

// ---------------------------------------------------------------- interior stencil
// Interior rectangle [lo, hi]^2 of a translation-invariant (Stokes) level, processed in natural
// node order with per-class tap weights (dj outer, di inner; 0 where a class has no tap), i.e.
// the same summation order as the SELL rows, so the results are bitwise identical.
struct StencilOp {
  int m = 0, lo = 0, hi = -1, nseg_x = 0;
  int64_t nseg = 0;
  double w[4][25];
  double dcls[4] = {0.0, 0.0, 0.0, 0.0};   // D^-1 of the non-Dirichlet rows per class
};

// translation-invariant B / B^T weights of the Stokes saddle operator (matrix-free k_saddle_mf)
struct SaddleSt {
  double bt1[4][2][9];        // B^T Q1 part per velocity class: vertices (i/2 + da, j/2 + dc), dc outer
  double bt0[4][2][4];        // B^T P0 part per velocity class: cells (i/2 + de, j/2 + df), de, df in {-1, 0}
  double b1[2][25];           // B Q1 rows: velocity nodes (2a + di, 2c + dj), dj outer, per component
  double b0[2][9];            // B P0 rows: velocity nodes (2e + di, 2f + dj), di, dj in {0, 1, 2}
};

// ---------------------------------------------------------------- MG level
struct Level {
  Geo g;
  Sell A;                     // scalar operator (Q2: identity Dirichlet rows; Q1: Ap)
  double* dinv = nullptr;     // [nrows]
  int nrows = 0;              // nq (Q2 velocity) or nk (Q1 pressure)
  double bim = 0.0;           // imaginary semi-axis of the smoother ellipse (0: real interval)
  bool st_on = false;         // interior stencil + frame SELL (Afr) instead of A for the smoother
  bool ct2 = false;           // its stencils equal the constant-bank table of k_cheb_tile2
  StencilOp so;
  Sell Afr;                   // rows outside the interior rectangle (own permutation)
  double* os_tab = nullptr;   // Oseen cavity-wind levels: 1D convection tables A1, T2 [2][m][5] (matrix-free interior)
  // two-component work vectors, each [2*nq]
  double *b = nullptr, *x = nullptr, *r = nullptr, *d0 = nullptr, *d1 = nullptr;
  double* coarse_inv = nullptr;   // dense inverse (coarsest level only), nq x nq row-major
  double* wind = nullptr;         // nodal Q2 wind on this level (Picard, levels >= 1; injection)
  double* lapval = nullptr;       // nu L values of A as assembled (Picard refills F = nu L + N)
  // fp32 copies for the c5 sweep (sweep32.cu)
  float *f_dinv = nullptr, *f_b = nullptr, *f_x = nullptr, *f_r = nullptr, *f_d0 = nullptr, *f_d1 = nullptr;
  float* f_coarse = nullptr;
};

// device-side description of one level of the fused coarse-level tail (ops.cu)
struct TailLevel {
  Sell A; const double* dinv; double *b, *x, *r, *d0, *d1;
  int nq, m; double c1[4], c2[4]; const double* coarse_inv;
};

// the same tail with its vectors in shared memory and the class stencils (Stokes levels only)
constexpr int TAIL_SM_MAXLEV = 8;
struct TailSmArgs {
  StencilOp so;               // class stencils and D^-1 (identical on every Stokes level)
  int nlev = 0, degree = 3;
  int m[TAIL_SM_MAXLEV];
  double c1[TAIL_SM_MAXLEV][4], c2[TAIL_SM_MAXLEV][4];
  double itheta = 0.0;
  const double* b0 = nullptr; const double* d00 = nullptr; double* x0 = nullptr;   // first tail level (global)
  const double* coarse_inv = nullptr;
  const double* done = nullptr;
  int smem_bytes = 0;
};

struct Hierarchy {
  std::vector<Level> lv;
  double lo = 0.16, hi = 1.6;
  int degree = 3;
  int kind = 0;               // 0: Q2 velocity (2 components, Dirichlet rows); 1: Q1 pressure (Ap / S_k)
  int op = 0;                 // kind 1: 0 = Ap (SELL), 1 = S_k / 4^l (matrix-free stencil kernels)
  double sk_w = 0.0;          // op 1: h_0^2 / 144, the stencil scale shared by all levels
  int ncomp = 2;
  bool built = false;
  bool f32 = false;           // fp32 copies present
  int tail_start = -1;        // first level run by the fused coarse-level tail kernel (-1: none)
  TailLevel* tail = nullptr;  // device array, levels tail_start .. L-1
  bool tail_sm = false;       // shared-memory matrix-free tail available (Stokes, storage 0)
  TailSmArgs tsm;             // its launch arguments (done filled per launch)
};

// ---------------------------------------------------------------- device scalars (MINRES / GMRES)
enum ScalarIdx {
  S_GAMMA = 0, S_GAMMA_PREV, S_DELTA, S_ETA, S_C, S_C_PREV, S_S, S_S_PREV, S_GAMMA1,
  S_A2, S_A3, S_A1, S_CNEW_ETA, S_DONE, S_STATUS, S_IT, S_RTOL, S_MAXIT,
  S_DOT0, S_DOT1, S_DOT2, S_DOT3, S_DOT4, S_DOT5, S_KR, S_KY, S_INV_GAMMA, S_TMP0, S_TMP1,
  S_APSUM, S_CE_PREV,
  // GMRES (solvers in oseen.cu)
  G_J = 32, G_JW, G_HN, G_RES, G_TOL, G_DONE, G_BREAK, G_TOT, G_BETA, G_MAXIT, G_NRM_P0, G_CAP,
  S_COUNT = 64
};

struct PcP1 {
  bool ready = false;
  double* Ainv = nullptr;     // nq x nq inverse of the scalar velocity block (Dirichlet rows)
  double* MQinv = nullptr;    // n_p x n_p inverse of (M_Q + k k^T)
  double* tmp = nullptr;      // [2 n_p] residual and correction of the refinement step
};

struct PcMass {               // Chebyshev-SGS on M_Q (P2 / M1 pressure block)
  bool ready = false;
  double a = 0.0;             // lower end of the SGS-preconditioned spectrum
  int m = 20;
  double *t = nullptr, *y0 = nullptr, *y1 = nullptr, *rr = nullptr;   // n_p work vectors
  // parity-plane ("planar") copies of r and of the Chebyshev iterates (ops.cu, k_sgs_plane): 8 planes
  // (4 vertex, 4 cell parities) of ph x pw entries, zero outside the domain; TMA descriptors of y
  int pw = 0, ph = 0;
  double *rp = nullptr, *yp[2] = {nullptr, nullptr};
  alignas(64) unsigned char tmap[2][128];   // CUtensorMap of yp[0], yp[1] (opaque, 64-byte aligned)
  bool planar = false;
};

// ---------------------------------------------------------------- PCG inner solves (exact.cu)
enum PcgScalar {
  PG_R0 = 0, PG_RZ0, PG_RZ1, PG_PQ, PG_RR, PG_DONE, PG_IT, PG_TOL2, PG_MAXIT, PG_ITTOT, PG_CALLS,
  PG_COUNT = 16
};
struct PcgWs {                // one preconditioned CG instance: device scalars, vectors, own slots
  int64_t n = 0;
  double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
  double* sc = nullptr;       // [PG_COUNT]
  RedSite red{};              // RED_SLOTS slots: 0 r0, 1 rz, 2 pq, 3 rr, 4.. callers
  cudaStream_t cs = nullptr;  // stream used to capture the conditional loop body
  double rtol = 1e-10;
  int maxit = 50;
  int64_t body_nodes = 0;     // kernel launches per loop iteration (captured body)
  int64_t fixed_nodes = 0;    // kernel launches outside the loop per call
};
struct PcExactMass {          // exact augmented M_Q solve through S_k (NEXT-2, reading R21)
  bool ready = false;
  Hierarchy sH;               // Q1 hierarchy of S_k (level l scaled by 4^-l)
  PcgWs cg;
  double* g = nullptr;        // [n_k] reduced right-hand side
  double* zh = nullptr;       // [n_k] S_k^+ g
  double* sc = nullptr;       // [8] sums, lambda, a^T zhat, beta
};
struct PcLp {                 // Lp^+ for the two-field PCD / LSC Schur approximations (NEXT-4)
  bool ready = false;
  Hierarchy H;                // Q1 + P0 hierarchy of Lp = B Mdiag^-1 B^T
  PcgWs cg;
  double* rp = nullptr;       // [n_p] projected right-hand side
  double* sc = nullptr;       // [8] field sums
};
struct PcVelIter {            // A^{-1} by V-cycle-preconditioned CG (P1 at scale)
  bool ready = false;
  PcgWs cg;
};

struct Problem {
  Geo g;
  int bc = 0;
  int storage = 0;                            // etq_grid.storage
  int wind = 0;
  bool plain = false;                         // etq_grid.enriched == 0: plain Q2-Q1 (p_0 block inert)
  double* plain_w = nullptr;                  // [3 n_k] scratch of the plain P2 pressure block
  double nu = 1.0;
  bool oseen = false;
  int64_t n_u = 0, n_p = 0, N = 0;
  cudaStream_t stream = nullptr;              // library work stream (capturable)
  cudaStream_t ustream = nullptr;             // caller's stream (may be the legacy stream)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaStream_t aux = nullptr;                 // pressure branch of the block preconditioner
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;

  Sell Lv;                                    // scalar velocity operator, level-0 rows, node perm
  Sell BxT1, ByT1, BxT0, ByT0;                // B^T split by component and pressure part
  Sell B;                                     // pressure rows (Q1 then P0) over [u_x; u_y]
  bool mf_on = false;                         // Stokes storage 0: matrix-free saddle apply (k_saddle_mf)
  bool bt_mf = false;                         // storage 0: sst holds the B / B^T class weights (any wind)
  double* os_tab0 = nullptr;                  // Oseen cavity wind, storage 0: 1D convection tables of level 0
  StencilOp so_os;                            // ... and the nu L class stencils (matrix-free Oseen saddle apply)
  StencilOp so0;                              // class stencil of L (level 0)
  SaddleSt sst;                               // B / B^T weights
  int* node_perm = nullptr;                   // shared by Lv and the B^T blocks

  Hierarchy mg;                               // velocity-block V-cycle
  PcP1 p1;
  PcMass pm;
  etq_pc_params params{};
  bool p2_ready = false;

  // reductions and device scalars
  RedSite red[1];                             // RED_SLOTS slots (map in solvers.cu)
  double* dscal = nullptr;                    // [S_COUNT]
  double* hscal = nullptr;                    // pinned host mirror
  double* dhist = nullptr;                    // [4 * hist_cap]: |eta|, delta, gamma
  int hist_cap = 0;

  // Oseen preconditioners (oseen.cu)
  Hierarchy apH;                              // Q1 hierarchy for Ap (PCD)
  Sell F1;                                    // PCD convection-diffusion on Q1
  bool pcd_ready = false, m1_ready = false;
  double* pw[3] = {nullptr, nullptr, nullptr};   // n_k work vectors of the PCD chain
  double* tu = nullptr;                       // [n_u] r_u - B^T z_p
  // GMRES workspace
  double* gV = nullptr; int gm = 0;           // (m+1) x N Arnoldi basis (stride gld)
  int64_t gld = 0;                            // basis stride: N rounded up to 32 elements
  double* gH = nullptr;                       // (m+1) x m Hessenberg (column-major)
  double* gsm = nullptr;                      // cs[m], sn[m], g[m+1], y[m], hh[m+1]
  double* gW = nullptr; double* gZ = nullptr; double* gT = nullptr; double* gU = nullptr;
  double* ghist = nullptr; int ghist_cap = 0;
  RedSite gred{};                             // 64 slots for the CGS2 multi-dots
  cudaGraphExec_t gmres_graph = nullptr; int gmres_graph_key = -1;
  int64_t gmres_graph_nodes = 0;

  // NEXT-3: nodal (Picard) wind, wind kind 2 (picard.cu)
  double* wnod = nullptr;                     // [n_u] Q2 nodal wind [w_x | w_y]
  double* lv_lap = nullptr;                   // nu L values of Lv as assembled
  double* f1_lap = nullptr;                   // diffusion values of F1 as assembled

  // NEXT-2: exact M_Q solve (P3, P1_ITER) and iterative A^{-1} (P1_ITER)
  PcExactMass mx;
  PcVelIter vi;
  PcLp lp;                                    // NEXT-4: Lp^+ (oseen2 Schur approximations)
  double* minv = nullptr;                     // [nq] 1 / Mdiag (scalar velocity mass diagonal)
  double* s2w[4] = {nullptr, nullptr, nullptr, nullptr};   // [n_u] work vectors of M2 / LSC

  // Krylov workspace (length N each)
  double* kv[10] = {nullptr};
  int nkv = 0;
  cudaGraphExec_t minres_graph[2] = {nullptr, nullptr};
  int minres_graph_kind = -1;
  const double* minres_graph_x = nullptr;     // graphs bake in the caller's x pointer
  int64_t minres_graph_nodes[2] = {0, 0};     // kernel launches per graph launch
  cudaGraphExec_t minres_wgraph = nullptr;    // device-side loop: while (!done) { 2 iterations }
  int minres_wgraph_kind = -1;
  const double* minres_wgraph_x = nullptr;
  int64_t minres_wbody_nodes = 0, minres_wfixed_nodes = 0;
  cudaStream_t wcs = nullptr;                 // capture stream of the loop body
  cudaStream_t wside = nullptr;               // MINRES w/x update beside the next saddle apply
  cudaEvent_t ev_wfork = nullptr, ev_wjoin = nullptr;
  double* tk = nullptr;                       // scratch for etq_time_kernel (3 x N)
  float* tkf = nullptr;                       // fp32 scratch (2 x N)
};

// ---------------------------------------------------------------- helpers (host)
etq_status dev_alloc(void** p, size_t bytes);
template <class T> inline etq_status dalloc(T** p, size_t count) {
  return dev_alloc(reinterpret_cast<void**>(p), count * sizeof(T));
}
void sell_free(Sell& s);

// assemble.cu
etq_status build_node_perm(const Geo& g, int** perm, int64_t* nslices, cudaStream_t st);
etq_status assemble_velocity_op(const Geo& g, bool oseen, double nu, int wind, int* perm,
                                int64_t nslices, Sell* out, cudaStream_t st);
etq_status assemble_bt(const Geo& g, int comp, int part, int* perm, int64_t nslices, Sell* out,
                       cudaStream_t st);
etq_status assemble_b(const Geo& g, Sell* out, cudaStream_t st);
etq_status velocity_dinv_dev(const Geo& g, bool oseen, double nu, int wind, double* dinv, cudaStream_t st);
etq_status oseen_gershgorin(const Geo& g, double nu, int wind, double* bim, cudaStream_t st);
etq_status assemble_ap(const Geo& g, Sell* out, cudaStream_t st);
etq_status assemble_f1(const Geo& g, double nu, int wind, Sell* out, cudaStream_t st);
etq_status assemble_sk(const Geo& g, double scale, Sell* out, cudaStream_t st);
etq_status assemble_lp(const Geo& g, Sell* out, cudaStream_t st);
etq_status velocity_mdiag_inv(const Geo& g, double* out, cudaStream_t st);
etq_status sell_diag_inv(const Sell& A, double* dinv, cudaStream_t st);
etq_status build_rhs_dev(const Problem& P, const double* f_nodal, double* b);
etq_status mark_implicit(const Geo& g, bool oseen, double nu, int wind, Sell& S, cudaStream_t st, bool values);
etq_status build_stencil_level(const Geo& g, const Sell& A, StencilOp* so, Sell* frame, cudaStream_t st);
etq_status build_oseen_stencil_level(const Geo& g, double nu, StencilOp* so, Sell* frame, double** tab,
                                     cudaStream_t st);
etq_status oseen_tables(const Geo& g, double nu, StencilOp* so, double** tab, cudaStream_t st);
etq_status saddle_weights(const Geo& g, SaddleSt* out, cudaStream_t st);
etq_status class_weights(const Geo& g, const Sell& A, StencilOp* so);

// ops.cu
void launch_saddle_ex(const Problem& P, bool reduced, const double* x, double* y, const double* inv_scale,
                      const RedSite* site, int slot, double* dot_out, const double* done, cudaStream_t st);
void launch_vel_spmv(const Sell& A, const double* x, double* y, int nq, cudaStream_t st);
void launch_dot(const double* a, const double* b, int64_t n, RedSite* site, int slot, double* out,
                const double* done, cudaStream_t st);
etq_status build_hierarchy(Problem& P, Hierarchy& H, int coarse_n, double lo, double hi, int degree);
etq_status build_ap_hierarchy(Problem& P, Hierarchy& H, int coarse_n, double lo, double hi, int degree, int op = 0);
void free_hierarchy(Hierarchy& H);
etq_status dense_inverse_pivot(double* A, int m, cudaStream_t st);
etq_status vcycle_apply_ex(const Problem& P, const Hierarchy& H, const double* r_u, double* z_u,
                           const RedSite* site, int slot, double* dot_out, const double* dot_with,
                           const double* done, cudaStream_t st, bool pdl = false);
void mass_apply(const Geo& g, const double* x, double* y, cudaStream_t st);
void sgs_sweep_dev(const Geo& g, const double* r, const double* y, double* z, double* t, cudaStream_t st);
etq_status mass_pc_alloc(Problem& P);
etq_status mass_pc_apply_ex(const Problem& P, const double* r_p, double* z_p, const RedSite* site, int slot,
                            double* dot_out, const double* dot_with, const double* done, cudaStream_t st,
                            double scale = 1.0);
etq_status dense_inverse_spd(double* A, int m, cudaStream_t st);
etq_status dense_from_sell(const Sell& A, int m, double* D, cudaStream_t st);
etq_status p1_build_mass_inverse(const Geo& g, double* W, cudaStream_t st);
void dense_gemv(const double* A, int m, int ncomp, const double* x, int64_t xstride, double* y,
                int64_t ystride, const double* done, cudaStream_t st, bool pdl = false);
etq_status lanczos_sgs_lo(Problem& P, const double* v0, int steps, double* lam);
int64_t etq_launch_total();
void cheb_step_level0(const Problem& P, const double* d_in, double* d_out, cudaStream_t st);
double vcycle_bytes(const Hierarchy& H);
double mass_pc_bytes(const Problem& P);
double cheb_step_bytes(const Level& L);
void sgs_step_bench(const Problem& P, const double* r, const double* y, const double* yp, double* out,
                    cudaStream_t st);
etq_status cheb_tile_bench(const Problem& P, bool post, const double* in_b, const double* in_x, double* o1,
                           double* o2, cudaStream_t st);

// oseen.cu
etq_status oseen_setup(Problem& P, etq_pc_kind kind);
etq_status oseen_precond_apply(const Problem& P, etq_pc_kind kind, const double* r, double* z, cudaStream_t st);
etq_status gmres_run(Problem& P, bool reduced, etq_pc_kind kind, const double* b, double* x, double tol_abs,
                     int restart, int maxit, etq_report* rep, double* p0_res_norm);
void oseen_free(Problem& P);
etq_status pcd_schur_apply(const Problem& P, const double* r, double* z, cudaStream_t st);
// out = m_p-step Chebyshev-Jacobi approximation of Q_k^{-1} r on [1/4, 9/4] (reading R13); ws: 3 n_k scratch
void qk_cheb_ws(const Problem& P, const double* r, double* out, int steps, double* ws, const double* done,
                cudaStream_t st);
etq_status make_reduced_rhs(Problem& P, const double* b, double** bred);
double host_norm(Problem& P, const double* v, int64_t n);
etq_status two_stage_run(Problem& P, const double* b, double* x, double eta, double c, int restart, int maxit,
                         etq_report* r1, etq_report* r2, double* bound);
etq_status ap_solve(const Problem& P, const Hierarchy& H, const double* r, double* z, double* sum_slot,
                    const double* done, cudaStream_t st);

// sweep32.cu
etq_status ensure_f32(Problem& P);
void launch_saddle_f32(const Problem& P, bool reduced, const float* x, float* y, cudaStream_t st);
etq_status vcycle_f32(const Problem& P, const float* r_u, float* z_u, cudaStream_t st);
double vcycle_bytes_f32(const Hierarchy& H);

// solvers.cu
void vec_scale_copy(double* y, const double* x, double a, int64_t n, cudaStream_t st);
void vec_lincomb3(double* w, const double* a, double ca, const double* b, double cb, const double* c,
                  double cc, int64_t n, cudaStream_t st);
etq_status precond_apply_ex(const Problem& P, etq_pc_kind kind, const double* r, double* z, const double* w,
                            double* out_u, double* out_p, const double* done, cudaStream_t st);
etq_status minres_run(Problem& P, etq_pc_kind kind, const double* b, double* x, double rtol,
                      int maxit, etq_report* rep);
// destroy every cached MINRES graph (they bake in hierarchy buffers, x and the history buffer)
void drop_minres_graphs(Problem& P);

// exact.cu (NEXT-2: exact M_Q solve through S_k, iterative A^{-1}, preconditioners P3 / P1_ITER)
etq_status exact_mass_setup(Problem& P);
etq_status vel_iter_setup(Problem& P);
void exact_free(Problem& P);
etq_status exact_mass_apply(const Problem& P, const double* r_p, double* z_p, const RedSite* site, int slot,
                            double* dot_out, const double* dot_with, const double* done, cudaStream_t st);
etq_status vel_iter_apply(const Problem& P, const double* r_u, double* z_u, const RedSite* site, int slot,
                          double* dot_out, const double* dot_with, const double* done, cudaStream_t st);
etq_status pcg_stats(const Problem& P, int which, double* it_total, double* calls);
int64_t pcg_launches_since(const Problem& P, double it0_m, double calls0_m, double it0_v, double calls0_v);

// picard.cu (NEXT-3: nodal Q2 wind, Picard loop)
etq_status picard_refresh(Problem& P);
etq_status picard_set_wind(Problem& P, const double* w);
etq_status picard_rhs_convection(const Problem& P, double* b);
etq_status picard_run(Problem& P, int steps, double eta, double c, int restart, int maxit, double* x,
                      int* its, double* res, double* ms_total);
etq_status refresh_tail(Hierarchy& H);   // ops.cu: rewrite the fused tail's level table (c1, c2)
etq_status lp_setup(Problem& P);
etq_status lp_pinv_apply(const Problem& P, const double* r, double* z, const double* done, cudaStream_t st);
void lp_free(Problem& P);
etq_status schur2_apply(const Problem& P, etq_pc_kind kind, const double* r_p, double* z_p, const double* done,
                        cudaStream_t st);
