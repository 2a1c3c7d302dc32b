// ops.cu — hot-path kernels of libetq (sm_100a, fp64):
//   * fused block SpMV  y = [A B^T; B 0] x  (Oseen P:756-773) with the optional
//     MINRES dot delta = <K z, z> fused into the same pass (Algorithm 1 line 7);
//   * Q2 geometric-multigrid V-cycle: Chebyshev-3 smoothing fused with the SpMV, matrix-free
//     nested-Q2 restriction/prolongation, dense coarse solve (reading R9);
//   * matrix-free 5-colour symmetric Gauss-Seidel on the singular M_Q = [[Qk, R^T],[R, Q0]]
//     and its Chebyshev semi-iteration with the symmetric k-projection Pi C Pi
//     (readings R6/R7);
//   * deterministic reductions (block partials + last-block fixed-order sum), dense
//     Gauss-Jordan inverse and GEMV for the exact (P1) and coarse solves.
#include "etq_internal.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <vector>
#include <utility>
#include <complex>

#include "device_common.cuh"
// SpMV-type kernels: 8 resident 256-thread blocks per SM (<= 32 registers) gave the highest
// bandwidth among the measured variants (unroll 2/4/8 x min-blocks 1/6/8, n = 1024).
#ifndef SPMV_MINB
#define SPMV_MINB 8
#endif
using namespace etqd;

namespace {
// ================================================================ fused saddle SpMV
struct SaddleArgs {
  Sell L, BxT1, ByT1, BxT0, ByT0, B;
  int nq, nk;
  int64_t n_u, n_p;
  int reduced;
  const double* x;
  double* y;
  const double* inv_scale;   // optional device scalar s: y = K (s x)
  RedSite site; int slot; double* dot_out;   // optional: dot_out = <y, s x>
  const double* done;
};

__global__ void __launch_bounds__(BS) k_saddle(SaddleArgs a) {
  if (is_done(a.done)) return;
  const double sc = a.inv_scale ? *a.inv_scale : 1.0;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsv = a.L.nslices, nsp = a.B.nslices;
  const double* xu = a.x;
  const double* xv = a.x + a.nq;
  const double* p1 = a.x + a.n_u;
  const double* p0 = p1 + a.nk;
  double dot = 0.0;
  for (int64_t s = gw; s < nsv + nsp; s += nw) {
    if (s < nsv) {
      const int row = a.L.perm[s * SELL_C + lane];
      double ax = 0.0, ay = 0.0;
      sell_row2(a.L, s, lane, row, xu, xv, ax, ay);
      ax += sell_row1(a.BxT1, s, lane, p1);
      ay += sell_row1(a.ByT1, s, lane, p1);
      if (!a.reduced) {
        ax += sell_row1(a.BxT0, s, lane, p0);
        ay += sell_row1(a.ByT0, s, lane, p0);
      }
      if (row >= 0) {
        ax *= sc; ay *= sc;
        a.y[row] = ax; a.y[a.nq + row] = ay;
        if (a.dot_out) dot += ax * (sc * xu[row]) + ay * (sc * xv[row]);
      }
    } else {
      const int64_t sp = s - nsv;
      const int64_t row = sp * SELL_C + lane;
      double acc = sell_row1(a.B, sp, lane, xu);
      if (row < a.n_p) {
        acc *= sc;
        if (a.reduced && row >= a.nk) acc = 0.0;
        a.y[a.n_u + row] = acc;
        if (a.dot_out) dot += acc * (sc * p1[row]);
      }
    }
  }
  if (a.dot_out) {
    double v[1] = {dot};
    reduce_finish<1>(v, a.site, a.slot, a.dot_out);
  }
}

// Matrix-free saddle apply for the Stokes operator (storage 0): every non-Dirichlet row of L, B^T and
// B is a translation-invariant class stencil (Dirichlet columns removed, reading R2), so only the
// vectors are streamed: 16 B per unknown (x in, y out) plus cached neighbour gathers, instead of the
// ~0.9 GB of B / B^T entries per apply at n = 1024.  Per-row arithmetic and summation order are those
// of k_saddle over the stored rows (bitwise-identical results).
struct SaddleMfArgs {
  StencilOp so; SaddleSt w;
  int nq, nk; int64_t n_u, n_p; int reduced;
  const double* x; double* y; const double* inv_scale;
  RedSite site; int slot; double* dot_out; const double* done;
  const double* tab;          // OS: 1D convection tables A1, T2 [2][m][5] of the cavity wind
};
// OS = 1: the Oseen operator [F B^T; B 0] of the cavity wind, F = nu L + N with the interior weights
// nu L_class(di, dj) + A1_i(di) T2_j(dj) - T2_i(di) A1_j(dj) (reading R9'; not the stored-row order)
template <int OS>
__global__ void __launch_bounds__(BS) k_saddle_mf(SaddleMfArgs a) {
  if (is_done(a.done)) return;
  const double sc = a.inv_scale ? *a.inv_scale : 1.0;
  const int m = a.so.m, n = (m - 1) / 2, n1 = n + 1;
  const double* xu = a.x;
  const double* xv = a.x + a.nq;
  const double* p1 = a.x + a.n_u;
  const double* p0 = p1 + a.nk;
  double dot = 0.0;
  const int64_t tot = (int64_t)a.nq + a.n_p;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < a.nq) {
      const int node = (int)t, i = node % m, j = node / m;
      double ax, ay;
      if (i == 0 || j == 0 || i == m - 1 || j == m - 1) {   // identity row; B^T rows are empty
        ax = fma(1.0, xu[node], 0.0) + 0.0;
        ay = fma(1.0, xv[node], 0.0) + 0.0;
        if (!a.reduced) { ax += 0.0; ay += 0.0; }
      } else {
        const int cl = (j & 1) * 2 + (i & 1);
        const double* w = a.so.w[cl];
        const bool near = i < 3 || j < 3 || i > m - 4 || j > m - 4;
        double a0 = 0.0, a1 = 0.0;
        double ai[5], ti[5];
        if (OS) {
#pragma unroll
          for (int d = 0; d < 5; ++d) { ai[d] = __ldg(a.tab + 5 * i + d); ti[d] = __ldg(a.tab + 5 * (m + i) + d); }
        }
        for (int dj = -2; dj <= 2; ++dj) {
          if ((j & 1) && (dj == 2 || dj == -2)) continue;
          const int jt = j + dj;
          if (near && (jt <= 0 || jt >= m - 1)) continue;
          const int rb = node + dj * m;
          double aj = 0.0, tj = 0.0;
          if (OS) { aj = __ldg(a.tab + 5 * j + dj + 2); tj = __ldg(a.tab + 5 * (m + j) + dj + 2); }
#pragma unroll
          for (int di = -2; di <= 2; ++di) {
            if (near && (i + di <= 0 || i + di >= m - 1)) continue;
            double wv = w[(dj + 2) * 5 + (di + 2)];
            if (OS) wv = fma(ai[di + 2], tj, fma(-ti[di + 2], aj, wv));
            a0 = fma(wv, __ldg(xu + rb + di), a0);
            a1 = fma(wv, __ldg(xv + rb + di), a1);
          }
        }
        // B^T Q1 part: vertices (i/2 + da, j/2 + dc) in [0, n]^2, dc outer
        double bx = 0.0, by = 0.0;
        const int ia = i / 2, jc = j / 2;
#pragma unroll
        for (int dc = -1; dc <= 1; ++dc) {
          const int c = jc + dc;
          if (c < 0 || c > n) continue;
#pragma unroll
          for (int da = -1; da <= 1; ++da) {
            const int aa = ia + da;
            if (aa < 0 || aa > n) continue;
            const double pv = __ldg(p1 + aa + (int64_t)n1 * c);
            bx = fma(a.w.bt1[cl][0][(dc + 1) * 3 + da + 1], pv, bx);
            by = fma(a.w.bt1[cl][1][(dc + 1) * 3 + da + 1], pv, by);
          }
        }
        ax = a0 + bx; ay = a1 + by;
        if (!a.reduced) {
          double cx = 0.0, cy = 0.0;
#pragma unroll
          for (int df = -1; df <= 0; ++df) {
            const int f = jc + df;
            if (f < 0 || f >= n) continue;
#pragma unroll
            for (int de = -1; de <= 0; ++de) {
              const int e = ia + de;
              if (e < 0 || e >= n) continue;
              const double pv = __ldg(p0 + e + (int64_t)n * f);
              cx = fma(a.w.bt0[cl][0][(df + 1) * 2 + de + 1], pv, cx);
              cy = fma(a.w.bt0[cl][1][(df + 1) * 2 + de + 1], pv, cy);
            }
          }
          ax += cx; ay += cy;
        }
      }
      ax *= sc; ay *= sc;
      a.y[node] = ax; a.y[a.nq + node] = ay;
      if (a.dot_out) dot += ax * (sc * xu[node]) + ay * (sc * xv[node]);
    } else {
      const int64_t row = t - a.nq;
      double acc = 0.0;
      if (row < a.nk) {
        const int aa = (int)(row % n1), c = (int)(row / n1);
        for (int dj = -2; dj <= 2; ++dj) {
          const int jj = 2 * c + dj;
          if (jj < 1 || jj > m - 2) continue;
#pragma unroll
          for (int di = -2; di <= 2; ++di) {
            const int ii = 2 * aa + di;
            if (ii < 1 || ii > m - 2) continue;
            const int64_t v = ii + (int64_t)m * jj;
            acc = fma(a.w.b1[0][(dj + 2) * 5 + di + 2], __ldg(xu + v), acc);
            acc = fma(a.w.b1[1][(dj + 2) * 5 + di + 2], __ldg(xv + v), acc);
          }
        }
      } else {
        const int tt = (int)(row - a.nk), e = tt % n, f = tt / n;
        for (int dj = 0; dj <= 2; ++dj) {
          const int jj = 2 * f + dj;
          if (jj < 1 || jj > m - 2) continue;
#pragma unroll
          for (int di = 0; di <= 2; ++di) {
            const int ii = 2 * e + di;
            if (ii < 1 || ii > m - 2) continue;
            const int64_t v = ii + (int64_t)m * jj;
            acc = fma(a.w.b0[0][dj * 3 + di], __ldg(xu + v), acc);
            acc = fma(a.w.b0[1][dj * 3 + di], __ldg(xv + v), acc);
          }
        }
      }
      acc *= sc;
      if (a.reduced && row >= a.nk) acc = 0.0;
      a.y[a.n_u + row] = acc;
      if (a.dot_out) dot += acc * (sc * p1[row]);
    }
  }
  if (a.dot_out) {
    double v[1] = {dot};
    reduce_finish<1>(v, a.site, a.slot, a.dot_out);
  }
}

// scalar operator on two components: y_c = A x_c
__global__ void __launch_bounds__(BS) k_vel_spmv2(Sell A, int nq, const double* x, double* y) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < A.nslices; s += nw) {
    const int row = A.perm[s * SELL_C + lane];
    double a0 = 0.0, a1 = 0.0;
    sell_row2(A, s, lane, row, x, x + nq, a0, a1);
    if (row >= 0) { y[row] = a0; y[nq + row] = a1; }
  }
}

// ================================================================ V-cycle kernels
__device__ __forceinline__ int sell_row_id(const Sell& A, int64_t s, int lane) {
  const int64_t t = s * SELL_C + lane;
  return A.perm ? A.perm[t] : (t < A.nrows ? (int)t : -1);
}

// One Chebyshev step fused with the level SpMV (Saad Alg. 12.1; readings R9/R9'), NC components
// (2: both velocity components share the scalar operator; 1: the Q1 pressure operator Ap):
//   x_out = x_in + d_in ; r_out = r_in - A d_in ; d_out = c1 d_in + c2 D^{-1} r_out
struct ChebArgs {
  Sell A; const double* dinv; int nq;
  const double* d_in; const double* r_in; const double* x_in;
  double* x_out; double* r_out; double* d_out;
  double c1, c2;
  const double* done;
};
template <int NC>
__global__ void __launch_bounds__(BS, SPMV_MINB) k_cheb_step(ChebArgs a) {
  if (is_done(a.done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < a.A.nslices; s += nw) {
    const int row = sell_row_id(a.A, s, lane);
    double q[2] = {0.0, 0.0};
    if (NC == 2) sell_row2(a.A, s, lane, row, a.d_in, a.d_in + a.nq, q[0], q[1]);
    else q[0] = sell_row1(a.A, s, lane, a.d_in);
    if (row < 0) continue;
    const double di = a.dinv[row];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int64_t idx = (int64_t)c * a.nq + row;
      const double dd = a.d_in[idx];
      const double ro = a.r_in[idx] - q[c];
      a.x_out[idx] = (a.x_in ? a.x_in[idx] : 0.0) + dd;
      if (a.r_out) a.r_out[idx] = ro;
      if (a.d_out) a.d_out[idx] = a.c1 * dd + a.c2 * (di * ro);
    }
  }
}

// ---- interior stencil path (Stokes levels): natural node order, contiguous gathers
// acc_c = sum_{dj, di} w[class][dj][di] x_c[(i+di) + m (j+dj)] in the SELL row order
__device__ __forceinline__ void stencil_row2(const StencilOp& so, int i, int j, const double* __restrict__ x0,
                                             const double* __restrict__ x1, double& a0, double& a1) {
  const int ce = (j & 1) * 2, cl = ce + (i & 1);
  const int node = i + so.m * j;
  a0 = 0.0; a1 = 0.0;
#pragma unroll
  for (int dj = -2; dj <= 2; ++dj) {
    if ((j & 1) && (dj == 2 || dj == -2)) continue;   // classes 2, 3 have no |dj| = 2 taps (warp-uniform)
    const int rb = node + dj * so.m;
#pragma unroll
    for (int di = -2; di <= 2; ++di) {
      const double w = so.w[cl][(dj + 2) * 5 + (di + 2)];
      const double v0 = __ldg(x0 + rb + di), v1 = __ldg(x1 + rb + di);
      a0 = fma(w, v0, a0);
      a1 = fma(w, v1, a1);
    }
  }
}

struct ChebStArgs {
  StencilOp so; Sell F; const double* dinv; int nq;
  const double* d_in; const double* r_in; const double* x_in;
  double* x_out; double* r_out; double* d_out;
  double c1, c2; int post; double itheta;   // post: r = b - A x, d = D^{-1} r / theta (x_in = x, r_in = b; itheta = 1 / theta)
  const double* done;
};
__device__ __forceinline__ void cheb_update2(const ChebStArgs& a, int row, double q0, double q1) {
  const double di = a.dinv[row];
  if (a.post) {
    const double r0 = a.r_in[row] - q0, r1 = a.r_in[a.nq + row] - q1;
    a.r_out[row] = r0; a.r_out[a.nq + row] = r1;
    a.d_out[row] = di * r0 * a.itheta; a.d_out[a.nq + row] = di * r1 * a.itheta;
    return;
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int64_t idx = (int64_t)c * a.nq + row;
    const double dd = a.d_in[idx];
    const double ro = a.r_in[idx] - (c == 0 ? q0 : q1);
    a.x_out[idx] = (a.x_in ? a.x_in[idx] : 0.0) + dd;
    if (a.r_out) a.r_out[idx] = ro;
    if (a.d_out) a.d_out[idx] = a.c1 * dd + a.c2 * (di * ro);
  }
}
// one launch: interior segments (32 consecutive nodes of one grid row per warp) + frame SELL slices
#ifndef STENCIL_MINB
#define STENCIL_MINB 6
#endif
__global__ void __launch_bounds__(BS, STENCIL_MINB) k_cheb_step_st(ChebStArgs a) {
  pdl_wait();
  if (is_done(a.done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* g = a.post ? a.x_in : a.d_in;   // gathered vector
  for (int64_t s = gw; s < a.so.nseg + a.F.nslices; s += nw) {
    if (s < a.so.nseg) {
      const int j = a.so.lo + (int)(s / a.so.nseg_x);
      const int i = a.so.lo + (int)(s % a.so.nseg_x) * 32 + lane;
      if (i > a.so.hi) continue;
      double q0, q1;
      stencil_row2(a.so, i, j, g, g + a.nq, q0, q1);
      cheb_update2(a, i + a.so.m * j, q0, q1);
    } else {
      const int64_t sf = s - a.so.nseg;
      const int row = a.F.perm[sf * SELL_C + lane];
      double q0 = 0.0, q1 = 0.0;
      sell_row2(a.F, sf, lane, row, g, g + a.nq, q0, q1);
      if (row >= 0) cheb_update2(a, row, q0, q1);
    }
  }
}

// Oseen levels with the cavity wind (reading R9'): interior row (i, j) of F_s = nu L + N, both
// components from one set of weights w = nu L_class(di, dj) + A1_i(di) T2_j(dj) - T2_i(di) A1_j(dj)
// (tab: A1 then T2, [m][5] each; the tables hold 0 outside the 1D supports, so the full 5 x 5
// (odd j: 5 x 3) loop needs no per-lane branches).  Not the stored-row summation order.
__device__ __forceinline__ void oseen_row2(const StencilOp& so, const double* __restrict__ tab, int i, int j,
                                           const double* __restrict__ x0, const double* __restrict__ x1, double& a0,
                                           double& a1) {
  const int cl = (j & 1) * 2 + (i & 1);
  const int node = i + so.m * j;
  const double* __restrict__ tA = tab;
  const double* __restrict__ tT = tab + 5 * so.m;
  double ai[5], ti[5];
#pragma unroll
  for (int d = 0; d < 5; ++d) { ai[d] = __ldg(tA + 5 * i + d); ti[d] = __ldg(tT + 5 * i + d); }
  a0 = 0.0; a1 = 0.0;
#pragma unroll
  for (int dj = -2; dj <= 2; ++dj) {
    if ((j & 1) && (dj == 2 || dj == -2)) continue;   // warp-uniform
    const double aj = __ldg(tA + 5 * j + dj + 2), tj = __ldg(tT + 5 * j + dj + 2);
    const int rb = node + dj * so.m;
#pragma unroll
    for (int di = -2; di <= 2; ++di) {
      const double w = fma(ai[di + 2], tj, fma(-ti[di + 2], aj, so.w[cl][(dj + 2) * 5 + (di + 2)]));
      a0 = fma(w, __ldg(x0 + rb + di), a0);
      a1 = fma(w, __ldg(x1 + rb + di), a1);
    }
  }
}

#ifndef OS_MINB
#define OS_MINB 4
#endif
__global__ void __launch_bounds__(BS, OS_MINB) k_cheb_step_os(ChebStArgs a, const double* __restrict__ tab) {
  pdl_wait();
  if (is_done(a.done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* g = a.post ? a.x_in : a.d_in;
  for (int64_t s = gw; s < a.so.nseg + a.F.nslices; s += nw) {
    if (s < a.so.nseg) {
      const int j = a.so.lo + (int)(s / a.so.nseg_x);
      const int i = a.so.lo + (int)(s % a.so.nseg_x) * 32 + lane;
      if (i > a.so.hi) continue;
      double q0, q1;
      oseen_row2(a.so, tab, i, j, g, g + a.nq, q0, q1);
      cheb_update2(a, i + a.so.m * j, q0, q1);
    } else {
      const int64_t sf = s - a.so.nseg;
      const int row = a.F.perm[sf * SELL_C + lane];
      double q0 = 0.0, q1 = 0.0;
      sell_row2(a.F, sf, lane, row, g, g + a.nq, q0, q1);
      if (row >= 0) cheb_update2(a, row, q0, q1);
    }
  }
}

// ---- temporally blocked Chebyshev smoothing (Stokes levels, storage 0): all three steps of a
// pre- or post-smoothing pass in one kernel.  A CTA owns a CT_T x CT_T tile of one velocity
// component and stages a CT_R x CT_R window (halo CT_H = 3 steps x stencil radius 2) of each
// vector in shared memory; each step shrinks the valid region by 2.  Within a step a lane owns
// a column pair (even i, odd i + 1) and a warp walks a strip of rows with a 5-row x 6-column
// register window (one 128-bit shared load per two values, each value reused by up to 25 taps).
// Row parity is compile-time in the unrolled walk, so the four stencil classes' weights are
// compile-time constant-bank operands.  Every non-Dirichlet row of a translation-invariant
// Stokes level equals its class stencil with the Dirichlet-node taps removed (identity rows and
// eliminated columns, reading R2): the level is matrix-free.  Per-row arithmetic and summation
// order are those of k_cheb_step_st / k_post_residual (interior rows bitwise identical).
// Bytes per node and component: pre 24 (b in; x, r out), post 32 (x, b in; x, d out) instead of
// 3 x ~52 + 16 for the unfused steps.
constexpr int CT_T = 56, CT_H = 6, CT_R = CT_T + 2 * CT_H, CT_THREADS = 256, CT_STRIP = 8;
constexpr int CT_ARR = CT_R * CT_R;            // one staged array, row-major (stride CT_R, even)
constexpr int CT_SMEM = 3 * CT_ARR * (int)sizeof(double);
static_assert(CT_R % 2 == 0 && CT_H % 2 == 0 && CT_T % 2 == 0, "column pairs need even offsets");
static_assert((CT_R - 4) / 2 <= 32, "a warp covers the widest step region with column pairs");
static_assert((CT_R - 4) <= CT_STRIP * (CT_THREADS / 32), "the warps' strips cover the widest step region");
struct ChebTileArgs {
  StencilOp so; int nq; int tiles_x;
  const double* b; const double* x_in;
  double* x_out; double* r_out; double* d_out;
  double itheta, c1[3], c2[3];
  const double* done;
  // finest post pass only: z = x + d2 written here (instead of d_out) and <z, dot_with>
  double* z_out; const double* dot_with; RedSite site; int slot; double* dot_out;
  int prefetch;   // L2 prefetch of a later CTA's window (k_cheb_tile3)
};

// class stencil of one output from the register window: win[slot][col], rows jj-2..jj+2 in
// slots (R0 + dj) % 5 (R0: slot of the output row, compile-time), cols ii-2..ii+3 with the
// output at column offset OC
// class stencils in the constant bank for k_cheb_tile2 (the Stokes Q2 Laplacian stencils are
// h-independent: every Stokes level's StencilOp equals this table bitwise, checked at launch)
__constant__ double c_ct_w[4][25];
__constant__ double c_ct_dcls[4];
// symmetric groups of the class stencils (reflections in x and y; classes 0 and 3 also the
// transpose): class 0 weights of |offset| (0,0) (1,0) (1,1) (2,0) (2,1) (2,2); class 1 (i odd,
// j even) (0,0) (1,0) (0,1) (1,1) (1,2); class 2 = class 1 transposed; class 3 (0,0) (1,0) (1,1)
__constant__ double c_ct_g0[6], c_ct_g1[5], c_ct_g3[3];

// grouped evaluation: sums of the mirrored taps first (independent adds), then one multiply-add
// per distinct weight.  Not the stored-row summation order (rounding-level differences).
template <int C, int OC, int R0>
__device__ __forceinline__ double ct_group_sum(const double (&win)[5][6]) {
#define W_(di, dj) win[(R0 + (dj) + 5) % 5][OC + (di) + 2]
  if (C == 0) {
    const double g10 = (W_(-1, 0) + W_(1, 0)) + (W_(0, -1) + W_(0, 1));
    const double g11 = (W_(-1, -1) + W_(1, -1)) + (W_(-1, 1) + W_(1, 1));
    const double g20 = (W_(-2, 0) + W_(2, 0)) + (W_(0, -2) + W_(0, 2));
    const double g21 = ((W_(-2, -1) + W_(2, -1)) + (W_(-2, 1) + W_(2, 1))) +
                       ((W_(-1, -2) + W_(1, -2)) + (W_(-1, 2) + W_(1, 2)));
    const double g22 = (W_(-2, -2) + W_(2, -2)) + (W_(-2, 2) + W_(2, 2));
    double a = c_ct_g0[0] * W_(0, 0);
    a = fma(c_ct_g0[1], g10, a);
    a = fma(c_ct_g0[2], g11, a);
    a = fma(c_ct_g0[3], g20, a);
    a = fma(c_ct_g0[4], g21, a);
    return fma(c_ct_g0[5], g22, a);
  } else if (C == 1 || C == 2) {
    // class 1 groups (|di|, |dj|); class 2 is its transpose (swap di and dj)
    constexpr bool T = C == 2;
#define V_(u, v) (T ? W_(v, u) : W_(u, v))
    const double g10 = V_(-1, 0) + V_(1, 0);
    const double g01 = V_(0, -1) + V_(0, 1);
    const double g11 = (V_(-1, -1) + V_(1, -1)) + (V_(-1, 1) + V_(1, 1));
    const double g12 = (V_(-1, -2) + V_(1, -2)) + (V_(-1, 2) + V_(1, 2));
#undef V_
    double a = c_ct_g1[0] * W_(0, 0);
    a = fma(c_ct_g1[1], g10, a);
    a = fma(c_ct_g1[2], g01, a);
    a = fma(c_ct_g1[3], g11, a);
    return fma(c_ct_g1[4], g12, a);
  } else {
    const double g10 = (W_(-1, 0) + W_(1, 0)) + (W_(0, -1) + W_(0, 1));
    const double g11 = (W_(-1, -1) + W_(1, -1)) + (W_(-1, 1) + W_(1, 1));
    double a = c_ct_g3[0] * W_(0, 0);
    a = fma(c_ct_g3[1], g10, a);
    return fma(c_ct_g3[2], g11, a);
  }
#undef W_
}

template <int C, int OC, int R0, bool CW = false>
__device__ __forceinline__ double ct_tap_sum(const StencilOp& so, const double (&win)[5][6]) {
  if (CW) return ct_group_sum<C, OC, R0>(win);
  constexpr int PI = C & 1, PJ = C >> 1, RX = PI ? 1 : 2, RY = PJ ? 1 : 2;
  double a = 0.0;
#pragma unroll
  for (int dj = -RY; dj <= RY; ++dj) {
#pragma unroll
    for (int di = -RX; di <= RX; ++di) {
      if (CW) {
        // taps the Stokes enumeration drops (exact Kronecker cancellations: weight 0, and
        // fma(0, v, a) == a for the finite window values) are skipped at compile time
        if ((di == 2 || di == -2) && dj == 0 && PJ) continue;
        if ((dj == 2 || dj == -2) && di == 0 && PI) continue;
        a = fma(c_ct_w[C][(dj + 2) * 5 + di + 2], win[(R0 + dj + 5) % 5][OC + di + 2], a);
      } else {
        a = fma(so.w[C][(dj + 2) * 5 + di + 2], win[(R0 + dj + 5) % 5][OC + di + 2], a);
      }
    }
  }
  return a;
}

// window row load: columns ii-2 .. ii+3 of window row jj (three 128-bit loads); EDGE: Dirichlet
// nodes read as 0 (their columns are eliminated from every non-Dirichlet row)
template <bool EDGE>
__device__ __forceinline__ void ct_load_row(const double* __restrict__ v, int ii, int jj, int i, int j, int m,
                                            double (&dst)[6]) {
  const double2* p = reinterpret_cast<const double2*>(v + (ii - 2) + CT_R * jj);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double2 t = p[k];
    dst[2 * k] = t.x; dst[2 * k + 1] = t.y;
  }
  if (EDGE) {
    const bool rowd = j <= 0 || j >= m - 1;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int it = i - 2 + k;
      if (rowd || it <= 0 || it >= m - 1) dst[k] = 0.0;
    }
  }
}

// row t of a warp's strip (compile-time t: window slots and stencil classes are constants)
template <int S, int MODE, bool EDGE, int t, bool CW = false>
__device__ __forceinline__ void ct_row_t(const ChebTileArgs& a, int i0, int j0, double* RS, const double* v,
                                         const double* din, double* dout, double c1, double c2, int jb, int ii,
                                         int i, bool lok, double (&win)[5][6]) {
  const int m = a.so.m;
  const int jj = jb + t;
  if (jj >= CT_R - S) return;                          // W even, strips even: whole pairs
  if (jj + 2 < CT_R) ct_load_row<EDGE>(v, ii, jj + 2, i, j0 + jj + 2, m, win[(t + 4) % 5]);
  constexpr int RSLOT = (t + 2) % 5;
  double qq[2];
  if ((t & 1) == 0) {                                  // jj even (jb even): classes 0 (i even), 1 (i odd)
    qq[0] = ct_tap_sum<0, 0, RSLOT, CW>(a.so, win);
    qq[1] = ct_tap_sum<1, 1, RSLOT, CW>(a.so, win);
  } else {
    qq[0] = ct_tap_sum<2, 0, RSLOT, CW>(a.so, win);
    qq[1] = ct_tap_sum<3, 1, RSLOT, CW>(a.so, win);
  }
  const int j = j0 + jj;
  if (!lok || (EDGE && (j < 0 || j >= m))) return;   // interior tiles lie inside the domain
  constexpr int C0 = (t & 1) * 2;
  const int base = ii + CT_R * jj;
  const double2 rr = *reinterpret_cast<const double2*>(RS + base);
  double ro[2] = {rr.x, rr.y};
  double outd[2];
  double dd[2] = {0.0, 0.0};
  if (MODE == 0 && dout) {
    const double2 t2 = *reinterpret_cast<const double2*>(din + base);
    dd[0] = t2.x; dd[1] = t2.y;
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int ik = i + k;
    const bool dir = EDGE && (ik == 0 || j == 0 || ik == m - 1 || j == m - 1);   // interior tiles: never
    if (EDGE && dir) qq[k] = fma(1.0, v[base + k], 0.0);   // identity row (unmasked centre)
    const double di = dir ? 1.0 : (CW ? c_ct_dcls[C0 + k] : a.so.dcls[C0 + k]);
    ro[k] = ro[k] - qq[k];
    if (MODE == 1) outd[k] = di * ro[k] * a.itheta;
    else outd[k] = c1 * dd[k] + c2 * (di * ro[k]);
  }
  // the odd column of the last pair may lie outside the domain (never read by valid rows)
  *reinterpret_cast<double2*>(RS + base) = make_double2(ro[0], ro[1]);
  if (MODE == 1 || dout) *reinterpret_cast<double2*>(dout + base) = make_double2(outd[0], outd[1]);
}

template <int S, int MODE, bool EDGE, bool CW, int... Ts>
__device__ __forceinline__ void ct_rows(const ChebTileArgs& a, int i0, int j0, double* RS, const double* v,
                                        const double* din, double* dout, double c1, double c2, int jb, int ii,
                                        int i, bool lok, double (&win)[5][6], std::integer_sequence<int, Ts...>) {
  (ct_row_t<S, MODE, EDGE, Ts, CW>(a, i0, j0, RS, v, din, dout, c1, c2, jb, ii, i, lok, win), ...);
}

// One Chebyshev update over the square [S, CT_R - S)^2 of the window.  MODE 0: r <- r - A v,
// dout <- c1 din + c2 D^-1 r (dout null: r only); MODE 1 (post-smoothing start, v = x):
// r <- b - A x (r holds b), dout <- D^-1 r / theta.
template <int S, int MODE, bool EDGE, bool CW = false>
__device__ __forceinline__ void ct_step(const ChebTileArgs& a, int i0, int j0, double* RS, const double* v,
                                        const double* din, double* dout, double c1, double c2) {
  constexpr int W = CT_R - 2 * S;
  const int m = a.so.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jb = S + CT_STRIP * warp;                 // first row of this warp's strip (even)
  if (jb >= CT_R - S) return;
  const bool lok = lane < W / 2;
  const int ii = S + 2 * (lok ? lane : 0);            // even column of the pair
  const int i = i0 + ii;
  double win[5][6];
  // rows jb-2 .. jb+1 into slots 0..3 (slot of row jj = (jj - jb + 2) % 5)
#pragma unroll
  for (int r = 0; r < 4; ++r) ct_load_row<EDGE>(v, ii, jb - 2 + r, i, j0 + jb - 2 + r, m, win[r]);
  ct_rows<S, MODE, EDGE, CW>(a, i0, j0, RS, v, din, dout, c1, c2, jb, ii, i, lok, win,
                             std::make_integer_sequence<int, CT_STRIP>{});
}

template <int POST>
__global__ void __launch_bounds__(CT_THREADS, 2) k_cheb_tile(ChebTileArgs a) {
  pdl_wait();
  if (is_done(a.done)) return;
  extern __shared__ __align__(16) double ct_sm[];
  double* D0 = ct_sm;
  double* D1 = ct_sm + CT_ARR;     // POST: holds x until the second step overwrites it
  double* RS = ct_sm + 2 * CT_ARR;
  const int m = a.so.m;
  const int comp = blockIdx.y;
  const int tx = blockIdx.x % a.tiles_x, ty = blockIdx.x / a.tiles_x;
  const int i0 = tx * CT_T - CT_H, j0 = ty * CT_T - CT_H;
  const int64_t off = (int64_t)comp * a.nq;
  const double* b = a.b + off;
  const int tid = threadIdx.x;
  const bool edge = i0 < 3 || j0 < 3 || i0 + CT_R > m - 3 || j0 + CT_R > m - 3;   // block-uniform
  // ---- stage the window (coalesced along i); outside the domain everything is 0.  All of a
  // thread's global loads are issued before any is used (one memory latency per CTA, not 19).
  constexpr int NST = (CT_ARR + CT_THREADS - 1) / CT_THREADS;
  double lb[NST], lx[NST];
#pragma unroll
  for (int k = 0; k < NST; ++k) {
    const int idx = tid + k * CT_THREADS;
    const int ii = idx % CT_R, jj = idx / CT_R;
    const int i = i0 + ii, j = j0 + jj;
    const bool in = idx < CT_ARR && i >= 0 && j >= 0 && i < m && j < m;
    const int node = in ? i + m * j : 0;
    lb[k] = in ? __ldg(b + node) : 0.0;
    if (POST) lx[k] = in ? __ldg(a.x_in + off + node) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < NST; ++k) {
    const int idx = tid + k * CT_THREADS;
    if (idx >= CT_ARR) break;
    const int ii = idx % CT_R, jj = idx / CT_R;
    const int i = i0 + ii, j = j0 + jj;
    const double bv = lb[k];
    RS[idx] = bv;
    if (POST) {
      D1[idx] = lx[k];
      D0[idx] = 0.0;
    } else {
      const bool in = i >= 0 && j >= 0 && i < m && j < m;
      double di = 1.0;
      if (!(i == 0 || j == 0 || i == m - 1 || j == m - 1)) di = a.so.dcls[(i & 1) + 2 * (j & 1)];
      D0[idx] = in ? di * bv * a.itheta : 0.0;   // k_cheb_init
      D1[idx] = 0.0;
    }
  }
  __syncthreads();
  // x lives in the output array between steps (T region only; L2-resident re-reads)
  constexpr int NTP = (CT_T * CT_T + CT_THREADS - 1) / CT_THREADS;
  auto tile_pos = [&](int k, int& w, int64_t& g) {
    const int o = tid + k * CT_THREADS;
    const int ii = CT_H + o % CT_T, jj = CT_H + o / CT_T;
    const int i = i0 + ii, j = j0 + jj;
    w = ii + CT_R * jj;
    g = off + i + (int64_t)m * j;
    return o < CT_T * CT_T && i < m && j < m;
  };
  auto tile_pass = [&](auto&& f) {
#pragma unroll
    for (int k = 0; k < NTP; ++k) {
      int w; int64_t g;
      if (tile_pos(k, w, g)) f(w, g);
    }
  };
  // x_out[T] += D[T] with all loads first
  auto tile_accum = [&](const double* D) {
    double xv[NTP];
#pragma unroll
    for (int k = 0; k < NTP; ++k) {
      int w; int64_t g;
      xv[k] = tile_pos(k, w, g) ? a.x_out[g] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NTP; ++k) {
      int w; int64_t g;
      if (tile_pos(k, w, g)) a.x_out[g] = xv[k] + D[w];
    }
  };
#define CT_STEP(S_, MODE_, RS_, V_, DIN_, DOUT_, C1_, C2_)                              \
  do {                                                                                  \
    if (edge) ct_step<S_, MODE_, true>(a, i0, j0, RS_, V_, DIN_, DOUT_, C1_, C2_);      \
    else ct_step<S_, MODE_, false>(a, i0, j0, RS_, V_, DIN_, DOUT_, C1_, C2_);          \
  } while (0)
  if (!POST) {
    CT_STEP(2, 0, RS, D0, D0, D1, a.c1[0], a.c2[0]);
    __syncthreads();
    tile_pass([&](int w, int64_t g) { a.x_out[g] = (0.0 + D0[w]) + D1[w]; });   // x2 = (0 + d0) + d1
    __syncthreads();
    CT_STEP(4, 0, RS, D1, D1, D0, a.c1[1], a.c2[1]);
    __syncthreads();
    tile_accum(D0);                                                              // x3 = x2 + d2
    CT_STEP(6, 0, RS, D0, D0, (double*)nullptr, 0.0, 0.0);
    __syncthreads();
    pdl_trigger();
    tile_pass([&](int w, int64_t g) { a.r_out[g] = RS[w]; });
  } else {
    CT_STEP(2, 1, RS, D1, (const double*)nullptr, D0, 0.0, 0.0);   // r0 = b - A x, d0 = D^-1 r0 / theta
    __syncthreads();
    tile_pass([&](int w, int64_t g) { a.x_out[g] = D1[w] + D0[w]; });   // x += d0
    __syncthreads();                                                     // x (in D1) no longer read
    CT_STEP(4, 0, RS, D0, D0, D1, a.c1[0], a.c2[0]);
    __syncthreads();
    tile_accum(D1);                                                      // x += d1
    CT_STEP(6, 0, RS, D1, D1, D0, a.c1[1], a.c2[1]);                   // d2 (deferred)
    __syncthreads();
    pdl_trigger();
    if (a.z_out) {   // finest level: the V-cycle's result z = x + d2 (k_final_add fused), <z, w>
      double xv[NTP], wv[NTP];
#pragma unroll
      for (int k = 0; k < NTP; ++k) {
        int w; int64_t g;
        const bool ok = tile_pos(k, w, g);
        xv[k] = ok ? a.x_out[g] : 0.0;
        wv[k] = (ok && a.dot_with) ? __ldg(a.dot_with + g) : 0.0;
      }
      double dot = 0.0;
#pragma unroll
      for (int k = 0; k < NTP; ++k) {
        int w; int64_t g;
        if (!tile_pos(k, w, g)) continue;
        const double v = xv[k] + D0[w];
        a.z_out[g] = v;
        dot += a.dot_with ? v * wv[k] : v;
      }
      if (a.dot_out) { double v1[1] = {dot}; reduce_finish<1>(v1, a.site, a.slot, a.dot_out, true); }
    } else {
      tile_pass([&](int w, int64_t g) { a.d_out[g] = D0[w]; });
    }
  }
#undef CT_STEP
}

// k_cheb_tile with fewer instructions per output (the smoother was issue-bound: 29 k warp
// instructions per CTA, a quarter of them in the staging loop's index arithmetic and a fifth in the
// tile passes): the class weights and D^-1 are constant-bank operands with the structurally zero
// taps skipped (no uniform-register reloads), the window is staged by row strips of column pairs
// (one 128-bit shared store per pair, no division), and the tile passes use the same pair layout.
// Same per-row arithmetic and summation order as k_cheb_tile: bitwise-identical outputs.
constexpr int CT2_TP = CT_T / 2;                       // tile column pairs (28) = active lanes in tile passes
constexpr int CT2_TR = CT_T / (CT_THREADS / 32);       // tile rows per warp (7)
static_assert(CT2_TP <= 32 && CT_T % (CT_THREADS / 32) == 0, "tile pass layout");

template <int POST, bool EDGE>
__device__ __forceinline__ void ct2_body(const ChebTileArgs& a, double* D0, double* D1, double* RS, int i0, int j0,
                                         int64_t off) {
  const int m = a.so.m;
  const double* __restrict__ b = a.b + off;
  const double* __restrict__ xin = POST ? a.x_in + off : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- staging: column pairs in window order, pair p = tid + 256 k (row p / 34); all loads of a
  //      group are issued before its stores; interior tiles need no bounds tests
  constexpr int PR = CT_R / 2, NP = PR * CT_R, NK = (NP + CT_THREADS - 1) / CT_THREADS, G = NK;   // one group: every load of the window in flight together
#pragma unroll
  for (int k0 = 0; k0 < NK; k0 += G) {
    double lb[G][2], lx[G][2];
#pragma unroll
    for (int kk = 0; kk < G; ++kk) {
      const int p = tid + CT_THREADS * (k0 + kk);
      const int jj = p / PR, pp = p - PR * jj;
      const int j = j0 + jj, i = i0 + 2 * pp;
      const int64_t g = (int64_t)m * j + i;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool in = (k0 + kk < NK) && p < NP && (!EDGE || (j >= 0 && j < m && i + e >= 0 && i + e < m));
        lb[kk][e] = in ? __ldg(b + g + e) : 0.0;
        if (POST) lx[kk][e] = in ? __ldg(xin + g + e) : 0.0;
      }
    }
#pragma unroll
    for (int kk = 0; kk < G; ++kk) {
      const int p = tid + CT_THREADS * (k0 + kk);
      if (k0 + kk >= NK || p >= NP) continue;
      const int jj = p / PR, pp = p - PR * jj;
      const int idx = 2 * pp + CT_R * jj;
      *reinterpret_cast<double2*>(RS + idx) = make_double2(lb[kk][0], lb[kk][1]);
      if (POST) {
        *reinterpret_cast<double2*>(D1 + idx) = make_double2(lx[kk][0], lx[kk][1]);
        *reinterpret_cast<double2*>(D0 + idx) = make_double2(0.0, 0.0);
      } else {
        const int odd = jj & 1;                            // j0 even: the row parity of j
        double dv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double di = c_ct_dcls[e + 2 * odd];
          if (EDGE) {
            const int j = j0 + jj, ie = i0 + 2 * pp + e;
            if (ie == 0 || j == 0 || ie == m - 1 || j == m - 1) di = 1.0;
            const bool in = ie >= 0 && j >= 0 && ie < m && j < m;
            dv[e] = in ? di * lb[kk][e] * a.itheta : 0.0;
          } else {
            dv[e] = di * lb[kk][e] * a.itheta;             // k_cheb_init
          }
        }
        *reinterpret_cast<double2*>(D0 + idx) = make_double2(dv[0], dv[1]);
        *reinterpret_cast<double2*>(D1 + idx) = make_double2(0.0, 0.0);
      }
    }
  }
  __syncthreads();
  // ---- tile passes: lane L < 28 owns the column pair (CT_H + 2L, +1) of the warp's 7 tile rows
  const bool tl = lane < CT2_TP;
  const int tii = CT_H + 2 * (tl ? lane : 0);
  const int ti = i0 + tii;
  auto tile_pass = [&](auto&& f) {
    if (!tl) return;
#pragma unroll
    for (int r = 0; r < CT2_TR; ++r) {
      const int tjj = CT_H + warp * CT2_TR + r;
      const int j = j0 + tjj;
      if (EDGE && j >= m) continue;
      const int w = tii + CT_R * tjj;
      const int64_t g = off + ti + (int64_t)m * j;
      f(w, g, !EDGE || ti + 1 < m, !EDGE || ti < m, r);
    }
  };
  // the tile's x accumulates in registers (pair r of the warp's rows): no global round trips
  double xs[CT2_TR][2];
  auto tile_acc = [&](const double* D, bool init, const double* D2) {
    if (!tl) return;
#pragma unroll
    for (int r = 0; r < CT2_TR; ++r) {
      const int w = tii + CT_R * (CT_H + warp * CT2_TR + r);
      const double2 p = *reinterpret_cast<const double2*>(D + w);
      if (init) {   // x = v0 + d (v0 from D2: POST x, pre 0 + d0)
        const double2 q = *reinterpret_cast<const double2*>(D2 + w);
        xs[r][0] = POST ? q.x + p.x : (0.0 + q.x) + p.x;
        xs[r][1] = POST ? q.y + p.y : (0.0 + q.y) + p.y;
      } else {
        xs[r][0] = xs[r][0] + p.x;
        xs[r][1] = xs[r][1] + p.y;
      }
    }
  };
  if (!POST) {
    ct_step<2, 0, EDGE, true>(a, i0, j0, RS, D0, D0, D1, a.c1[0], a.c2[0]);
    __syncthreads();
    tile_acc(D1, true, D0);                                  // x2 = (0 + d0) + d1
    __syncthreads();
    ct_step<4, 0, EDGE, true>(a, i0, j0, RS, D1, D1, D0, a.c1[1], a.c2[1]);
    __syncthreads();
    tile_acc(D0, false, nullptr);                            // x3 = x2 + d2
    ct_step<6, 0, EDGE, true>(a, i0, j0, RS, D0, D0, (double*)nullptr, 0.0, 0.0);
    __syncthreads();
    pdl_trigger();
    tile_pass([&](int w, int64_t g, bool ok1, bool ok0, int r) {
      const double2 p = *reinterpret_cast<const double2*>(RS + w);
      if (ok0) { a.r_out[g] = p.x; a.x_out[g] = xs[r][0]; }
      if (ok1) { a.r_out[g + 1] = p.y; a.x_out[g + 1] = xs[r][1]; }
    });
  } else {
    ct_step<2, 1, EDGE, true>(a, i0, j0, RS, D1, (const double*)nullptr, D0, 0.0, 0.0);   // r0 = b - A x, d0
    __syncthreads();
    tile_acc(D0, true, D1);                                  // x += d0
    __syncthreads();                                         // x (in D1) no longer read
    ct_step<4, 0, EDGE, true>(a, i0, j0, RS, D0, D0, D1, a.c1[0], a.c2[0]);
    __syncthreads();
    tile_acc(D1, false, nullptr);                            // x += d1
    ct_step<6, 0, EDGE, true>(a, i0, j0, RS, D1, D1, D0, a.c1[1], a.c2[1]);   // d2 (deferred)
    __syncthreads();
    pdl_trigger();
    if (a.z_out) {   // finest level: z = x + d2, <z, w>
      double dot = 0.0;
      tile_pass([&](int w, int64_t g, bool ok1, bool ok0, int r) {
        const double2 p = *reinterpret_cast<const double2*>(D0 + w);
        if (ok0) {
          const double v = xs[r][0] + p.x;
          a.z_out[g] = v;
          dot += a.dot_with ? v * __ldg(a.dot_with + g) : v;
        }
        if (ok1) {
          const double v = xs[r][1] + p.y;
          a.z_out[g + 1] = v;
          dot += a.dot_with ? v * __ldg(a.dot_with + g + 1) : v;
        }
      });
      if (a.dot_out) { double v1[1] = {dot}; reduce_finish<1>(v1, a.site, a.slot, a.dot_out, true); }
    } else {
      tile_pass([&](int w, int64_t g, bool ok1, bool ok0, int r) {
        const double2 p = *reinterpret_cast<const double2*>(D0 + w);
        if (ok0) { a.d_out[g] = p.x; a.x_out[g] = xs[r][0]; }
        if (ok1) { a.d_out[g + 1] = p.y; a.x_out[g + 1] = xs[r][1]; }
      });
    }
  }
}

template <int POST>
__global__ void __launch_bounds__(CT_THREADS, 2) k_cheb_tile2(ChebTileArgs a) {
  pdl_wait();
  if (is_done(a.done)) return;
  extern __shared__ __align__(16) double ct_sm[];
  const int m = a.so.m;
  const int tx = blockIdx.x % a.tiles_x, ty = blockIdx.x / a.tiles_x;
  const int i0 = tx * CT_T - CT_H, j0 = ty * CT_T - CT_H;
  const int64_t off = (int64_t)blockIdx.y * a.nq;
  const bool edge = i0 < 3 || j0 < 3 || i0 + CT_R > m - 3 || j0 + CT_R > m - 3;   // block-uniform
  if (edge) ct2_body<POST, true>(a, ct_sm, ct_sm + CT_ARR, ct_sm + 2 * CT_ARR, i0, j0, off);
  else ct2_body<POST, false>(a, ct_sm, ct_sm + CT_ARR, ct_sm + 2 * CT_ARR, i0, j0, off);
}

// k_cheb_tile2 with the residual in registers (k_cheb_tile3).  ncu on k_cheb_tile2: the shared-memory
// pipe is the bound (20.9 M wavefronts per finest pass ~ 72 us at one wavefront per clock per SM;
// short-scoreboard and MIO-throttle stalls lead), not the fp64 pipe (~30 us).  Here every thread
// keeps ONE output map for all three steps - lane L owns window columns 2 + 2L, 3 + 2L, warp w the
// rows 2 + 8w .. 9 + 8w (the widest step region [2, 66)^2) - so:
//   * r lives in registers (no shared r array, no r load / store per row),
//   * the step's own d_k is the centre of the register window (no din load),
//   * the tile's outputs are written straight from the last step's row loop (no trailing tile
//     passes and their barriers); x = d0 + d1 + d2 (resp. x + d0 + d1) is summed there from the
//     two earlier d arrays in the same order as k_cheb_tile2 (bitwise-identical outputs).
// Per row and lane: 3 window loads + 1 d store (step 3: + 2 loads on tile rows) instead of 7.
// Lanes / rows outside a step's region compute finite garbage from unused window entries that no
// valid output reads (each region lies inside the previous one shrunk by the stencil radius 2).
template <int S, int MODE, bool EDGE, int FIN, int t>
__device__ __forceinline__ void ct3_row(const ChebTileArgs& a, int i0, int j0, const double* __restrict__ v,
                                        double* __restrict__ dout, const double* __restrict__ e0,
                                        const double* __restrict__ e1, double c1, double c2, int jb, int ii,
                                        int lane, double (&win)[5][6], double (&rr)[CT_STRIP][2], double& dot) {
  const int m = a.so.m;
  const int jj = jb + t;
  if (jj + 2 < CT_R) ct_load_row<EDGE>(v, ii, jj + 2, i0 + ii, j0 + jj + 2, m, win[(t + 4) % 5]);
  if (jj < S || jj >= CT_R - S) return;               // warp-uniform
  const int j = j0 + jj;
  if (EDGE && (j < 0 || j >= m)) return;
  constexpr int RSLOT = (t + 2) % 5;
  double qq[2];
  if ((t & 1) == 0) {                                  // jj even (jb even): classes 0 (i even), 1 (i odd)
    qq[0] = ct_tap_sum<0, 0, RSLOT, true>(a.so, win);
    qq[1] = ct_tap_sum<1, 1, RSLOT, true>(a.so, win);
  } else {
    qq[0] = ct_tap_sum<2, 0, RSLOT, true>(a.so, win);
    qq[1] = ct_tap_sum<3, 1, RSLOT, true>(a.so, win);
  }
  constexpr int C0 = (t & 1) * 2;
  const int i = i0 + ii;
  const int base = ii + CT_R * jj;
  double outd[2], dd[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int ik = i + k;
    const bool dir = EDGE && (ik == 0 || j == 0 || ik == m - 1 || j == m - 1);
    dd[k] = win[RSLOT][2 + k];                         // d_k at the output (interior: unmasked)
    if (EDGE && dir) {
      dd[k] = v[base + k];                             // Dirichlet centre: the unmasked value
      qq[k] = fma(1.0, dd[k], 0.0);                    // identity row
    }
    const double di = dir ? 1.0 : c_ct_dcls[C0 + k];
    rr[t][k] = rr[t][k] - qq[k];
    if (MODE == 1) outd[k] = di * rr[t][k] * a.itheta;
    else outd[k] = c1 * dd[k] + c2 * (di * rr[t][k]);
  }
  if (FIN == 0) {
    *reinterpret_cast<double2*>(dout + base) = make_double2(outd[0], outd[1]);
    return;
  }
  // last step: the tile's outputs (tile rows / columns [CT_H, CT_H + CT_T) only)
  if (jj < CT_H || jj >= CT_H + CT_T || ii < CT_H || ii >= CT_H + CT_T) return;
  const double2 p0 = *reinterpret_cast<const double2*>(e0 + base);
  const double2 p1 = *reinterpret_cast<const double2*>(e1 + base);
  const double q0[2] = {p0.x, p0.y}, q1[2] = {p1.x, p1.y};
  const int64_t g = (int64_t)blockIdx.y * a.nq + i + (int64_t)m * j;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (EDGE && i + k >= m) continue;
    if (FIN == 1) {                                    // pre: r out, x3 = ((0 + d0) + d1) + d2
      a.r_out[g + k] = rr[t][k];
      a.x_out[g + k] = ((0.0 + q0[k]) + q1[k]) + dd[k];
    } else {                                           // post: x = (x + d0) + d1, d2 = MODE-0 output
      const double x = (q0[k] + q1[k]) + dd[k];
      if (FIN == 3) {                                  // finest: z = x + d2, <z, w>
        const double z = x + outd[k];
        a.z_out[g + k] = z;
        dot += a.dot_with ? z * __ldg(a.dot_with + g + k) : z;
      } else {
        a.d_out[g + k] = outd[k];
        a.x_out[g + k] = x;
      }
    }
  }
}

template <int S, int MODE, bool EDGE, int FIN, int... Ts>
__device__ __forceinline__ void ct3_rows(const ChebTileArgs& a, int i0, int j0, const double* v, double* dout,
                                         const double* e0, const double* e1, double c1, double c2, int jb, int ii,
                                         int lane, double (&win)[5][6], double (&rr)[CT_STRIP][2], double& dot,
                                         std::integer_sequence<int, Ts...>) {
  (ct3_row<S, MODE, EDGE, FIN, Ts>(a, i0, j0, v, dout, e0, e1, c1, c2, jb, ii, lane, win, rr, dot), ...);
}

// FIN: 0 = intermediate step (d out to shared memory), 1 = last pre step, 2 = last post step
// (x, d out), 3 = last post step of the finest level (z out + dot)
template <int S, int MODE, bool EDGE, int FIN>
__device__ __forceinline__ void ct3_step(const ChebTileArgs& a, int i0, int j0, const double* v, double* dout,
                                         const double* e0, const double* e1, double c1, double c2,
                                         double (&rr)[CT_STRIP][2], double& dot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jb = 2 + CT_STRIP * warp;
  const int ii = 2 + 2 * lane;
  double win[5][6];
#pragma unroll
  for (int r = 0; r < 4; ++r) ct_load_row<EDGE>(v, ii, jb - 2 + r, i0 + ii, j0 + jb - 2 + r, a.so.m, win[r]);
  ct3_rows<S, MODE, EDGE, FIN>(a, i0, j0, v, dout, e0, e1, c1, c2, jb, ii, lane, win, rr, dot,
                               std::make_integer_sequence<int, CT_STRIP>{});
}

static_assert(2 + 2 * 31 + 3 < CT_R && 2 + CT_STRIP * (CT_THREADS / 32) == CT_R - 2, "tile3 output map");

template <int POST, bool EDGE>
__device__ __forceinline__ void ct3_body(const ChebTileArgs& a, double* A0, double* A1, double* A2, int i0, int j0,
                                         int64_t off) {
  const int m = a.so.m;
  const double* __restrict__ b = a.b + off;
  const double* __restrict__ xin = POST ? a.x_in + off : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- r = b at the thread's own outputs (registers; 16-byte coalesced rows), issued first
  double rr[CT_STRIP][2];
  {
    const int i = i0 + 2 + 2 * lane;
#pragma unroll
    for (int t = 0; t < CT_STRIP; ++t) {
      const int j = j0 + 2 + CT_STRIP * warp + t;
      const int64_t g = (int64_t)m * j + i;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool in = !EDGE || (j >= 0 && j < m && i + e >= 0 && i + e < m);
        rr[t][e] = in ? __ldg(b + g + e) : 0.0;
      }
    }
  }
  // ---- staging of the first step's window: pre d0 = D^-1 b / theta (k_cheb_init) into A0; post x
  //      into A0.  Column pairs in window order, all loads of a group before its stores
  constexpr int PR = CT_R / 2, NP = PR * CT_R, NK = (NP + CT_THREADS - 1) / CT_THREADS, G = NK;   // one group: every load of the window in flight together
#pragma unroll
  for (int k0 = 0; k0 < NK; k0 += G) {
    double lv[G][2];
#pragma unroll
    for (int kk = 0; kk < G; ++kk) {
      const int p = tid + CT_THREADS * (k0 + kk);
      const int jj = p / PR, pp = p - PR * jj;
      const int j = j0 + jj, i = i0 + 2 * pp;
      const int64_t g = (int64_t)m * j + i;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool in = (k0 + kk < NK) && p < NP && (!EDGE || (j >= 0 && j < m && i + e >= 0 && i + e < m));
        lv[kk][e] = in ? __ldg((POST ? xin : b) + g + e) : 0.0;
      }
    }
#pragma unroll
    for (int kk = 0; kk < G; ++kk) {
      const int p = tid + CT_THREADS * (k0 + kk);
      if (k0 + kk >= NK || p >= NP) continue;
      const int jj = p / PR, pp = p - PR * jj;
      const int idx = 2 * pp + CT_R * jj;
      if (POST) {
        *reinterpret_cast<double2*>(A0 + idx) = make_double2(lv[kk][0], lv[kk][1]);
      } else {
        const int odd = jj & 1;
        double dv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double di = c_ct_dcls[e + 2 * odd];
          if (EDGE) {
            const int j = j0 + jj, ie = i0 + 2 * pp + e;
            if (ie == 0 || j == 0 || ie == m - 1 || j == m - 1) di = 1.0;
            const bool in = ie >= 0 && j >= 0 && ie < m && j < m;
            dv[e] = in ? di * lv[kk][e] * a.itheta : 0.0;
          } else {
            dv[e] = di * lv[kk][e] * a.itheta;
          }
        }
        *reinterpret_cast<double2*>(A0 + idx) = make_double2(dv[0], dv[1]);
      }
    }
  }
  __syncthreads();
  double dot = 0.0;
  if (!POST) {
    ct3_step<2, 0, EDGE, 0>(a, i0, j0, A0, A1, nullptr, nullptr, a.c1[0], a.c2[0], rr, dot);   // d1
    __syncthreads();
    ct3_step<4, 0, EDGE, 0>(a, i0, j0, A1, A2, nullptr, nullptr, a.c1[1], a.c2[1], rr, dot);   // d2
    __syncthreads();
    pdl_trigger();
    ct3_step<6, 0, EDGE, 1>(a, i0, j0, A2, nullptr, A0, A1, 0.0, 0.0, rr, dot);               // r, x3
  } else {
    ct3_step<2, 1, EDGE, 0>(a, i0, j0, A0, A1, nullptr, nullptr, 0.0, 0.0, rr, dot);          // r0, d0
    __syncthreads();
    ct3_step<4, 0, EDGE, 0>(a, i0, j0, A1, A2, nullptr, nullptr, a.c1[0], a.c2[0], rr, dot);   // d1
    __syncthreads();
    pdl_trigger();
    if (a.z_out) {
      ct3_step<6, 0, EDGE, 3>(a, i0, j0, A2, nullptr, A0, A1, a.c1[1], a.c2[1], rr, dot);      // z = x + d2
      if (a.dot_out) { double v1[1] = {dot}; reduce_finish<1>(v1, a.site, a.slot, a.dot_out, true); }
    } else {
      ct3_step<6, 0, EDGE, 2>(a, i0, j0, A2, nullptr, A0, A1, a.c1[1], a.c2[1], rr, dot);      // x, d2
    }
  }
}

// L2 prefetch of the window a later CTA will stage: the CTA that takes this one's place on the SM
// is about CT_PF_DIST blocks ahead in launch order (2 resident CTAs on each of 148 SMs), and the
// staging of a tile is one exposed DRAM latency at 16 warps per SM; with its lines already in L2
// that wait is an L2 hit.  One 128-byte line per prefetch, rows clamped to the grid.
constexpr int CT_PF_DIST = 2 * 148 + 32;
__device__ __forceinline__ void ct_prefetch_window(const double* __restrict__ v, int m, int i0, int j0, int tid) {
  if (tid >= CT_R) return;
  const int j = j0 + tid;
  if (j < 0 || j >= m) return;
  const int ia = max(i0, 0), ib = min(i0 + CT_R, m);        // [ia, ib)
  const char* p = reinterpret_cast<const char*>(v + (int64_t)m * j + ia);
  const char* e = reinterpret_cast<const char*>(v + (int64_t)m * j + ib);
  p = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)127);
  for (; p < e; p += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int POST>
__global__ void __launch_bounds__(CT_THREADS, 2) k_cheb_tile3(ChebTileArgs a) {
  pdl_wait();
  if (is_done(a.done)) return;
  extern __shared__ __align__(16) double ct_sm[];
  const int m = a.so.m;
  if (a.prefetch) {
    const int lin = blockIdx.x + gridDim.x * blockIdx.y + CT_PF_DIST;
    if (lin < (int)(gridDim.x * gridDim.y)) {
      const int bx = lin % gridDim.x, by = lin / gridDim.x;
      const int pi0 = (bx % a.tiles_x) * CT_T - CT_H, pj0 = (bx / a.tiles_x) * CT_T - CT_H;
      const int64_t poff = (int64_t)by * a.nq;
      ct_prefetch_window(a.b + poff, m, pi0, pj0, threadIdx.x);
      if (POST) ct_prefetch_window(a.x_in + poff, m, pi0, pj0, (int)threadIdx.x - 128);
    }
  }
  const int tx = blockIdx.x % a.tiles_x, ty = blockIdx.x / a.tiles_x;
  const int i0 = tx * CT_T - CT_H, j0 = ty * CT_T - CT_H;
  const int64_t off = (int64_t)blockIdx.y * a.nq;
  const bool edge = i0 < 3 || j0 < 3 || i0 + CT_R > m - 3 || j0 + CT_R > m - 3;   // block-uniform
  if (edge) ct3_body<POST, true>(a, ct_sm, ct_sm + CT_ARR, ct_sm + 2 * CT_ARR, i0, j0, off);
  else ct3_body<POST, false>(a, ct_sm, ct_sm + CT_ARR, ct_sm + 2 * CT_ARR, i0, j0, off);
}

// r = b - A x ; d = D^{-1} r / theta  (start of post-smoothing), NC components
template <int NC>
__global__ void __launch_bounds__(BS, SPMV_MINB) k_post_residual(Sell A, const double* dinv, int nq, const double* b,
                                                      const double* x, double* r, double* d, double itheta,
                                                      const double* done) {
  if (is_done(done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < A.nslices; s += nw) {
    const int row = sell_row_id(A, s, lane);
    double q[2] = {0.0, 0.0};
    if (NC == 2) sell_row2(A, s, lane, row, x, x + nq, q[0], q[1]);
    else q[0] = sell_row1(A, s, lane, x);
    if (row < 0) continue;
    const double di = dinv[row];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int64_t idx = (int64_t)c * nq + row;
      const double rr = b[idx] - q[c];
      r[idx] = rr;
      d[idx] = di * rr * itheta;
    }
  }
}

// Matrix-free S_k Chebyshev step / post-smoothing residual on a Q1 level (reading R21):
// same contract as k_cheb_step<1> (post = 0) and k_post_residual<1> (post = 1, v = x, r_in = b).
struct SkChebArgs {
  int n; double w;
  const double* v;                         // vector the operator is applied to (d_in, or x if post)
  const double* d_in; const double* r_in; const double* x_in;
  double* x_out; double* r_out; double* d_out;
  double c1, c2, itheta; int post;
  const double* done;
};
__global__ void __launch_bounds__(BS) k_cheb_sk(SkChebArgs a) {
  pdl_wait();
  if (is_done(a.done)) return;
  const int n1 = a.n + 1;
  const int64_t nk = (int64_t)n1 * n1;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nk; p += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(p / n1), ai = (int)(p - (int64_t)c * n1);
    double d7;
    const double q = a.w * sk_stencil(p, ai, c, a.n, a.v, &d7);
    const double di = 1.0 / (a.w * d7);
    const double ro = a.r_in[p] - q;
    if (a.post) {
      a.r_out[p] = ro;
      a.d_out[p] = di * ro * a.itheta;
    } else {
      const double dd = a.d_in[p];
      a.x_out[p] = (a.x_in ? a.x_in[p] : 0.0) + dd;
      if (a.r_out) a.r_out[p] = ro;
      if (a.d_out) a.d_out[p] = a.c1 * dd + a.c2 * (di * ro);
    }
  }
}

// d = D^{-1} b / theta (start of pre-smoothing from x = 0), NC components
__global__ void k_cheb_init(const double* dinv, int nq, int nc, const double* b, double* d, double itheta,
                            const double* done) {
  if (is_done(done)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)nc * nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i % nq);
    d[i] = dinv[row] * b[i] * itheta;
  }
}

// Q1 (pressure) transfers: nested bilinear interpolation, no boundary rows (no pressure BC)
// b_c = P^T r_f and d0_c = D_c^{-1} b_c / theta
__global__ void k_restrict_q1(int mf, int mc, const double* rf, double* bc, double* d0c, const double* dinvc,
                              double itheta, const double* done) {
  pdl_wait();
  if (is_done(done)) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)mc * mc;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int I = (int)(t % mc), J = (int)(t / mc);
    double s = 0.0;
    for (int dl = -1; dl <= 1; ++dl) {
      const int l = 2 * J + dl;
      if (l < 0 || l >= mf) continue;
      const double wy = dl == 0 ? 1.0 : 0.5;
      double tt = 0.0;
      for (int dk = -1; dk <= 1; ++dk) {
        const int k = 2 * I + dk;
        if (k < 0 || k >= mf) continue;
        tt = fma(dk == 0 ? 1.0 : 0.5, rf[(int64_t)l * mf + k], tt);
      }
      s = fma(wy, tt, s);
    }
    bc[t] = s;
    d0c[t] = dinvc[t] * s * itheta;
  }
}
// x_f += P (x_c + d_c)
__global__ void k_prolong_q1(int mf, int mc, const double* xc, const double* dc, double* xf, const double* done) {
  pdl_wait();
  if (is_done(done)) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)mf * mf;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(t % mf), l = (int)(t / mf);
    const int nx = (k & 1) ? 2 : 1, ny = (l & 1) ? 2 : 1;
    double s = 0.0;
    for (int q = 0; q < ny; ++q) {
      const int J = (l >> 1) + q;
      double tt = 0.0;
      for (int p = 0; p < nx; ++p) {
        const int I = (k >> 1) + p;
        const int64_t c = (int64_t)J * mc + I;
        tt = fma(nx == 2 ? 0.5 : 1.0, dc ? xc[c] + dc[c] : xc[c], tt);
      }
      s = fma(ny == 2 ? 0.5 : 1.0, tt, s);
    }
    xf[t] += s;
  }
}
// P0 (cell) transfers of the two-field hierarchy (NEXT-4): piecewise-constant prolongation
// (a coarse cell's value on its 4 children) and its transpose (sum of the 4 children)
__global__ void k_restrict_p0(int nf, int nc, const double* rf, double* bc, double* d0c, const double* dinvc,
                              double itheta, const double* done) {
  if (is_done(done)) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)nc * nc;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int E = (int)(t % nc), F = (int)(t / nc);
    const int64_t f0 = (int64_t)(2 * F) * nf + 2 * E;
    const double s = (rf[f0] + rf[f0 + 1]) + (rf[f0 + nf] + rf[f0 + nf + 1]);
    bc[t] = s;
    d0c[t] = dinvc[t] * s * itheta;
  }
}
__global__ void k_prolong_p0(int nf, int nc, const double* xc, const double* dc, double* xf, const double* done) {
  if (is_done(done)) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)nf * nf;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t % nf), f = (int)(t / nf);
    const int64_t c = (int64_t)(f >> 1) * nc + (e >> 1);
    xf[t] += dc ? xc[c] + dc[c] : xc[c];
  }
}
// A[i][j] += v for i, j in [r0, r1) (coarse pseudo-inverse of the two-field Laplacian)
__global__ void k_add_block(double* A, int m, int r0, int r1, double v) {
  const int w = r1 - r0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)w * w; t += (int64_t)gridDim.x * blockDim.x)
    A[(int64_t)(r0 + t / w) * m + r0 + t % w] += v;
}

// z -= (sum / n) 1 (mean-zero projection after the Ap V-cycle, reading R13)
__global__ void k_sub_mean(double* z, int64_t n, const double* sum, const double* done) {
  if (is_done(done)) return;
  const double m = *sum / (double)n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] -= m;
}

// 1D nested-Q2 transfer weights: coarse node I gathers fine nodes 2I + off
__device__ __forceinline__ int restrict_taps(int I, int* off, double* w) {
  if ((I & 1) == 0) {
    off[0] = -3; w[0] = -0.125; off[1] = -1; w[1] = 0.375; off[2] = 0; w[2] = 1.0;
    off[3] = 1; w[3] = 0.375; off[4] = 3; w[4] = -0.125;
    return 5;
  }
  off[0] = -1; w[0] = 0.75; off[1] = 0; w[1] = 1.0; off[2] = 1; w[2] = 0.75;
  return 3;
}

// b_c = Z_c P^T r_f (both components) and d0_c = D_c^{-1} b_c / theta
__global__ void k_restrict(int mf, int mc, int nqf, int nqc, const double* rf, double* bc, double* d0c,
                           const double* dinvc, double itheta, const double* done) {
  pdl_wait();
  if (is_done(done)) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)nqc;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int I = (int)(t % mc), J = (int)(t / mc);
    if (I == 0 || J == 0 || I == mc - 1 || J == mc - 1) {
      bc[t] = 0.0; bc[nqc + t] = 0.0; d0c[t] = 0.0; d0c[nqc + t] = 0.0;
      continue;
    }
    // fixed 5 x 5 tap frame (offsets -3, -1, 0, 1, 3): odd (element-midpoint) coarse indices take the
    // two outer taps with weight 0 and skip their loads, so the loops unroll and every load of a
    // row is in flight together; the sums start from 0, so the zero taps leave them bitwise unchanged
    const bool ei = (I & 1) == 0, ej = (J & 1) == 0;
    const double wo_i = ei ? -0.125 : 0.0, wn_i = ei ? 0.375 : 0.75;
    const double wo_j = ej ? -0.125 : 0.0, wn_j = ej ? 0.375 : 0.75;
    const double wx[5] = {wo_i, wn_i, 1.0, wn_i, wo_i}, wy[5] = {wo_j, wn_j, 1.0, wn_j, wo_j};
    constexpr int off[5] = {-3, -1, 0, 1, 3};
    const double di = dinvc[t];            // requested with the gathers, not after them
    const double* __restrict__ r0 = rf + (int64_t)(2 * J) * mf + 2 * I;
    const double* __restrict__ r1 = r0 + nqf;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      if ((q == 0 || q == 4) && !ej) continue;
      const int64_t ro = (int64_t)off[q] * mf;
      double v0[5], v1[5];
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        const bool on = ei || (p != 0 && p != 4);
        v0[p] = on ? r0[ro + off[p]] : 0.0;
        v1[p] = on ? r1[ro + off[p]] : 0.0;
      }
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        if ((p == 0 || p == 4) && !ei) continue;
        t0 = fma(wx[p], v0[p], t0);
        t1 = fma(wx[p], v1[p], t1);
      }
      s0 = fma(wy[q], t0, s0);
      s1 = fma(wy[q], t1, s1);
    }
    bc[t] = s0; bc[nqc + t] = s1;
    d0c[t] = di * s0 * itheta; d0c[nqc + t] = di * s1 * itheta;
  }
}

// fine node k interpolates coarse nodes: k even -> k/2 (weight 1); k = 4e+1 -> (3/8, 3/4, -1/8)
// on 2e..2e+2; k = 4e+3 -> (-1/8, 3/4, 3/8)
__device__ __forceinline__ int prolong_taps(int k, int* idx, double* w) {
  if ((k & 1) == 0) { idx[0] = k >> 1; w[0] = 1.0; return 1; }
  const int e = k >> 2;
  idx[0] = 2 * e; idx[1] = 2 * e + 1; idx[2] = 2 * e + 2;
  if ((k & 3) == 1) { w[0] = 0.375; w[1] = 0.75; w[2] = -0.125; }
  else { w[0] = -0.125; w[1] = 0.75; w[2] = 0.375; }
  return 3;
}

// x_f += Z_f P (x_c + d_c)
__global__ void k_prolong(int mf, int mc, int nqf, int nqc, const double* xc, const double* dc, double* xf,
                          const double* done) {
  pdl_wait();
  if (is_done(done)) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)nqf;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(t % mf), l = (int)(t / mf);
    if (k == 0 || l == 0 || k == mf - 1 || l == mf - 1) continue;
    int ix[3], iy[3]; double wx[3], wy[3];
    const int nx = prolong_taps(k, ix, wx), ny = prolong_taps(l, iy, wy);
    double s0 = 0.0, s1 = 0.0;
    for (int q = 0; q < ny; ++q) {
      double t0 = 0.0, t1 = 0.0;
      for (int p = 0; p < nx; ++p) {
        const int64_t c = (int64_t)iy[q] * mc + ix[p];
        const double v0 = dc ? xc[c] + dc[c] : xc[c];
        const double v1 = dc ? xc[nqc + c] + dc[nqc + c] : xc[nqc + c];
        t0 = fma(wx[p], v0, t0);
        t1 = fma(wx[p], v1, t1);
      }
      s0 = fma(wy[q], t0, s0);
      s1 = fma(wy[q], t1, s1);
    }
    xf[t] += s0; xf[nqf + t] += s1;
  }
}

// Tiled nested-Q2 prolongation xf += P (xc + dc) (same operations and order as k_prolong, so
// bitwise the same): a CTA owns a PT_X x PT_Y block of fine nodes; the coarse correction of its
// coarse window is staged in shared memory, each needed coarse row is interpolated along x once
// (the per-row partial sums t0 of k_prolong), then every fine node combines up to three of them
// along y.  Replaces up to 36 gathered coarse loads per fine node.
constexpr int PT_X = 64, PT_Y = 32, PT_THREADS = 256;
constexpr int PT_CX = PT_X / 2 + 3, PT_CY = PT_Y / 2 + 3;   // coarse window (origin K0/2 - 1, L0/2 - 1)
__global__ void __launch_bounds__(PT_THREADS) k_prolong_tile(int mf, int mc, int nqf, int nqc, const double* xc,
                                                            const double* dc, double* xf, const double* done) {
  pdl_wait();
  if (is_done(done)) return;
  __shared__ double ec[2][PT_CY][PT_CX];
  __shared__ double tx[2][PT_CY][PT_X];
  const int tilesx = (mf + PT_X - 1) / PT_X;
  const int K0 = (blockIdx.x % tilesx) * PT_X, L0 = (blockIdx.x / tilesx) * PT_Y;
  const int I0 = K0 / 2 - 1, J0 = L0 / 2 - 1;
  // the fine values this thread will update, requested first: their DRAM latency passes behind the
  // staging and the x pass instead of in front of the final read-modify-write
  constexpr int PT_NF = PT_Y * PT_X / PT_THREADS;
  double xf0[PT_NF], xf1[PT_NF];
#pragma unroll
  for (int q = 0; q < PT_NF; ++q) {
    const int idx = threadIdx.x + q * PT_THREADS;
    const int k = K0 + idx % PT_X, l = L0 + idx / PT_X;
    const bool on = k < mf && l < mf && k > 0 && l > 0 && k < mf - 1 && l < mf - 1;
    const int64_t t = on ? k + (int64_t)mf * l : 0;
    xf0[q] = on ? xf[t] : 0.0;
    xf1[q] = on ? xf[nqf + t] : 0.0;
  }
  for (int idx = threadIdx.x; idx < PT_CY * PT_CX; idx += PT_THREADS) {
    const int ci = I0 + idx % PT_CX, cj = J0 + idx / PT_CX;
    const bool in = ci >= 0 && cj >= 0 && ci < mc && cj < mc;
    const int64_t c = in ? ci + (int64_t)mc * cj : 0;
#pragma unroll
    for (int comp = 0; comp < 2; ++comp) {
      const int64_t cc = c + (int64_t)comp * nqc;
      ec[comp][idx / PT_CX][idx % PT_CX] = in ? (dc ? xc[cc] + dc[cc] : xc[cc]) : 0.0;
    }
  }
  __syncthreads();
  // x pass: t0(J, k) for the window's coarse rows and the tile's fine columns
  for (int idx = threadIdx.x; idx < PT_CY * PT_X; idx += PT_THREADS) {
    const int jr = idx / PT_X, kk = idx % PT_X, k = K0 + kk;
    if (k >= mf) continue;
    int ix[3]; double wx[3];
    const int nx = prolong_taps(k, ix, wx);
#pragma unroll
    for (int comp = 0; comp < 2; ++comp) {
      double t0 = 0.0;
      for (int p = 0; p < nx; ++p) t0 = fma(wx[p], ec[comp][jr][ix[p] - I0], t0);
      tx[comp][jr][kk] = t0;
    }
  }
  __syncthreads();
  // y pass
#pragma unroll
  for (int qq = 0; qq < PT_NF; ++qq) {
    const int idx = threadIdx.x + qq * PT_THREADS;
    const int kk = idx % PT_X, k = K0 + kk, l = L0 + idx / PT_X;
    if (k >= mf || l >= mf || k == 0 || l == 0 || k == mf - 1 || l == mf - 1) continue;
    int iy[3]; double wy[3];
    const int ny = prolong_taps(l, iy, wy);
    double s0 = 0.0, s1 = 0.0;
    for (int q = 0; q < ny; ++q) {
      s0 = fma(wy[q], tx[0][iy[q] - J0][kk], s0);
      s1 = fma(wy[q], tx[1][iy[q] - J0][kk], s1);
    }
    const int64_t t = k + (int64_t)mf * l;
    xf[t] = xf0[qq] + s0; xf[nqf + t] = xf1[qq] + s1;
  }
}

// z = x + d (d nullable), optional dot partial <z, w>
__global__ void __launch_bounds__(BS) k_final_add(const double* x, const double* d, double* z, int64_t n,
                                                  const double* dw, RedSite site, int slot, double* out,
                                                  const double* done) {
  pdl_wait();
  if (is_done(done)) return;
  double dot = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = d ? x[i] + d[i] : x[i];
    z[i] = v;
    dot += dw ? v * dw[i] : v;     // dw == nullptr: plain sum (mean projection)
  }
  if (out) { double a[1] = {dot}; reduce_finish<1>(a, site, slot, out); }
}

// ================================================================ dense helpers
// in-place Gauss-Jordan inverse without pivoting (SPD input), step p, part 1: save column, scale row
__global__ void k_gj_row(double* A, int m, int p, double* colp) {
  const double piv = A[(int64_t)p * m + p];
  const double pinv = 1.0 / piv;
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < m; i += blockDim.x * gridDim.x)
    colp[i] = A[(int64_t)i * m + p];
  __syncthreads();   // single block launch: column saved before the row changes
  for (int j = threadIdx.x; j < m; j += blockDim.x)
    A[(int64_t)p * m + j] = (j == p ? 1.0 : A[(int64_t)p * m + j]) * pinv;
}
__global__ void k_gj_update(double* A, int m, int p, const double* colp) {
  const int64_t total = (int64_t)m * m;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / m), j = (int)(t % m);
    if (i == p) continue;
    const double f = colp[i];
    A[t] = (j == p ? 0.0 : A[t]) - f * A[(int64_t)p * m + j];
  }
}

// y_c = A x_c for ncomp components (A dense m x m row-major), warp per row
__global__ void k_gemv(const double* A, int m, int ncomp, const double* x, int64_t xs, double* y, int64_t ys,
                       const double* done) {
  pdl_wait();
  if (is_done(done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // both components from one pass over the row (the matrix is read once; per component the
  // summation order is the lane-strided sum + warp_sum as before)
  for (int64_t r = gw; r < m; r += nw) {
    for (int c0 = 0; c0 < ncomp; c0 += 2) {
      const bool two = c0 + 1 < ncomp;
      const double* x0 = x + c0 * xs;
      const double* x1 = x + (c0 + 1) * xs;
      // four independent partial sums per component, the loads of four row chunks issued together
      // (the kernel was latency-bound at one load per iteration: 43 us for the 143 MB F coarse inverse)
      double p0[4] = {0.0, 0.0, 0.0, 0.0}, p1[4] = {0.0, 0.0, 0.0, 0.0};
      const double* __restrict__ Ar = A + r * m;
      int j = lane;
      for (; j + 96 < m; j += 128) {
        double a[4], u[4], v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a[k] = __ldg(Ar + j + 32 * k);
          u[k] = __ldg(x0 + j + 32 * k);
          v[k] = two ? __ldg(x1 + j + 32 * k) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) { p0[k] = fma(a[k], u[k], p0[k]); p1[k] = fma(a[k], v[k], p1[k]); }
      }
      for (; j < m; j += 32) {
        const double a = __ldg(Ar + j);
        p0[0] = fma(a, __ldg(x0 + j), p0[0]);
        if (two) p1[0] = fma(a, __ldg(x1 + j), p1[0]);
      }
      double s0 = warp_sum((p0[0] + p0[1]) + (p0[2] + p0[3]));
      double s1 = two ? warp_sum((p1[0] + p1[1]) + (p1[2] + p1[3])) : 0.0;
      if (lane == 0) { y[c0 * ys + r] = s0; if (two) y[(c0 + 1) * ys + r] = s1; }
    }
  }
}

// ================================================================ pressure mass (matrix-free)
// 1D Q1 mass entries (h/6)[[2,1],[1,2]] assembled: diag 4h/6 inside, 2h/6 at the ends, off h/6.
__device__ __forceinline__ double ml1(int n, double h, int a, int ap) {
  const int d = a - ap;
  if (d == 0) return (a == 0 || a == n) ? (2.0 * h / 6.0) : (4.0 * h / 6.0);
  return (d == 1 || d == -1) ? (h / 6.0) : 0.0;
}

struct MassGeo { int n; int nk; int n0; double h; };

// y = M_Q x  (Prop 2.1 matrix; R_{T,p} = h^2/4, Q0 = h^2)
__global__ void k_mass_apply(MassGeo g, const double* x, double* y) {
  const int n = g.n, n1 = n + 1; const double h = g.h, r = 0.25 * h * h, q0 = h * h;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)g.nk + g.n0;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < g.nk) {
      const int a = (int)(t % n1), c = (int)(t / n1);
      double s = 0.0;
      for (int cc = max(0, c - 1); cc <= min(n, c + 1); ++cc) {
        const double mc = ml1(n, h, c, cc);
        for (int aa = max(0, a - 1); aa <= min(n, a + 1); ++aa) s += mc * ml1(n, h, a, aa) * x[aa + n1 * cc];
      }
      double s0 = 0.0;
      for (int f = max(0, c - 1); f <= min(n - 1, c); ++f)
        for (int e = max(0, a - 1); e <= min(n - 1, a); ++e) s0 += x[g.nk + e + n * f];
      y[t] = s + r * s0;
    } else {
      const int te = (int)(t - g.nk), e = te % n, f = te / n;
      const double s1 = x[e + n1 * f] + x[e + 1 + n1 * f] + x[e + n1 * (f + 1)] + x[e + 1 + n1 * (f + 1)];
      y[t] = r * s1 + q0 * x[t];
    }
  }
}

// ---------------------------------------------------------------- temporally blocked SGS
// One launch = one symmetric Gauss-Seidel sweep S(y) on M_Q z = r' (r' = r - alpha k, reading R6)
// in the colour order 0,1,2,3,P0 | P0,3,2,1,0 (reading R7; the repeated P0 update is idempotent
// and done once), fused with the Chebyshev semi-iteration update of P:455 (mode 1):
//     out = omega (gam (S(y) - y) + y - yp) + yp = co_s S(y) + (co_y y + co_p yp)   (mode 0: S(y)).
// Each CTA owns a T x T tile of Q1 vertices (and the P0 cells whose lower-left vertex is in the
// tile), stages a W x W window (the tile plus the halo the 9 colour steps need, below) in
// shared memory, runs all colour steps there and writes only its tile: the 16.8 MB pressure
// vectors are read once per Chebyshev step instead of once per colour step.
//
// Layout: vertices AND cells are stored as four parity planes each (local (la, lc) -> plane
// (la & 1) + 2 (lc & 1), entry (lc >> 1, la >> 1)), and thread (tx, ty) owns plane entries
// (tx, ty + 16 m), m = 0, 1, of every plane in every phase (staging, sweeps, cells, output).  So a
// vertex update reads its 8 vertex and 4 cell neighbours at compile-time offsets from one base
// address, each warp access is 32 consecutive words (no bank conflicts), and the interior path
// (tiles away from the domain boundary) has no branches: the window-edge entries compute
// finite garbage that the halo absorbs.  On
// boundary tiles the 1D mass diagonal (2h/6 on the boundary) and the out-of-domain zeros are
// selects.  Every row uses the same operation sequence on both paths.
// Halo: garbage entering at the window edge moves one entry per colour step only when the
// updated colour has the parity of the entry next to the front, so along x (colour parities
// 0,1,0,1 | 1,0,1,0) it travels 7 entries from the left edge and 6 from the right, along y
// (0,0,1,1 | 1,1,0,0) only 3 from below and 2 from above (tests/test_sgs_halo.py simulates the
// dependency cone).  Halos 8 / 6 (x) and 4 / 2 (y) keep tile origins even (the colour of a local
// entry is its global colour): 50 x 58 tiles from a 64 x 64 window (1.5x the 44 x 44 tiles of
// a symmetric halo of 10).
constexpr int SGS_W = 64;              // staged window (both directions)
constexpr int SGS_HX = 8, SGS_HY = 4;  // left / bottom halo (right / top: 6 / 2)
constexpr int SGS_TTX = 50, SGS_TTY = 58;   // tile
constexpr int SGS_P = SGS_W / 2;       // plane side (32)
constexpr int SGS_PL = SGS_P * SGS_P;  // one plane
constexpr int SGS_TQ = SGS_TTX * SGS_TTY;  // tile entries (Q: vertices, then cells, row-major)
constexpr int SGS_PAD = 64;            // zeroed words before the vertex planes (edge reads at -33)
constexpr int SGS_TX = 32, SGS_TY = 16;
constexpr int SGS_SMEM = (SGS_PAD + 8 * SGS_PL + 2 * SGS_TQ) * (int)sizeof(double);
static_assert(SGS_W - SGS_HX - SGS_TTX >= 6 && SGS_W - SGS_HY - SGS_TTY >= 2, "right / top halo");
static_assert(SGS_HX % 2 == 0 && SGS_HY % 2 == 0 && SGS_TTX % 2 == 0 && SGS_TTY % 2 == 0, "even origins");
static_assert(SGS_TX == SGS_P && 2 * SGS_TY == SGS_P, "one thread per plane column, two rows");
// window geometry by height WY (64 or 32 rows; 64 columns) and plane rows per thread MR (2: 512 / 256
// threads, 1: 1024 / 512 threads); the halos are unchanged
#define SGS_GEO(WY_, MR_)                                                                         \
  constexpr int TY_ = (WY_) / 2 / (MR_), PL_ = SGS_P * ((WY_) / 2), TTY_ = (WY_) - 6, TQ_ = SGS_TTX * TTY_; \
  static_assert((MR_) * TY_ == (WY_) / 2 && TTY_ % 2 == 0, "MR plane rows per thread");          \
  (void)TQ_
template <int WY>
constexpr int sgs_smem() { return (SGS_PAD + 8 * SGS_P * (WY / 2) + 2 * SGS_TTX * (WY - 6)) * (int)sizeof(double); }

struct SgsK {                 // M_Q coefficients (Qk = Mlin x Mlin, R = h^2/4, Q0 = h^2)
  double w_in, w_bd, w_off, rq, c_dd, c_ed, inv_in2, inv_inbd, inv_bd2, inv_q0;
};

struct SgsTileArgs {
  MassGeo g;
  SgsK k;                   // filled by launch_sgs_tile (kernel parameters: constant-bank operands)
  const double* r;          // right-hand side (n_p)
  const double* kproj;      // optional device scalar k^T r: r' = r - (kproj / k^T k) k
  double inv_kk;
  const double* y;          // current iterate (nullable = 0)
  const double* yp;         // previous iterate (nullable = 0)
  double* out;
  int mode;                 // 0: out = S(y); 1: Chebyshev combination
  double omega, gam;
  int tiles_x;
  RedSite site; int slot; double* kout;   // optional k^T out
  const double* done;
  int pdl;                  // launched as a programmatic dependent of the previous SGS step
  int yp_ldg;               // y_prev read from global in the Q pass (1) or staged by cp.async (0)
};


__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

// update of colour (PX, PY): plane entries (i, j), j = ty + 16 m; vertex (2i + PX, 2j + PY)
template <int WY, int MR, int PX, int PY, bool IN>
__device__ __forceinline__ void sgs_colour(double* __restrict__ V, const double* __restrict__ Cc,
                                           const double (&rr)[MR], int A0, int C0, int n, const SgsK& k) {
  SGS_GEO(WY, MR);
  constexpr int c = PX + 2 * PY, cx = (1 - PX) + 2 * PY, cy = PX + 2 * (1 - PY), cxy = (1 - PX) + 2 * (1 - PY);
  constexpr int OW = PX - 1, OE = PX, OS = (PY - 1) * SGS_P, ON = PY * SGS_P;   // neighbour offsets
  const int i = threadIdx.x;
#pragma unroll
  for (int m = 0; m < MR; ++m) {
    const int j = threadIdx.y + TY_ * m;
    const int B = j * SGS_P + i;
    const double* vd = V + cxy * PL_ + B;
    const double* vx = V + cx * PL_ + B;
    const double* vy = V + cy * PL_ + B;
    const double sd = (vd[OS + OW] + vd[OS + OE]) + (vd[ON + OW] + vd[ON + OE]);
    const double sx = vx[OW] + vx[OE];
    const double sy = vy[OS] + vy[ON];
    // cells (la-1, lc-1), (la, lc-1), (la-1, lc), (la, lc)
    const double sc = (Cc[cxy * PL_ + B + OS + OW] + Cc[cy * PL_ + B + OS]) +
                      (Cc[cx * PL_ + B + OW] + Cc[c * PL_ + B]);
    double wx = k.c_ed, wy = k.c_ed, inv = k.inv_in2;
    bool in = true;
    if (!IN) {
      const int ga = A0 + 2 * i + PX, gc = C0 + 2 * j + PY;
      in = ga >= 0 && ga <= n && gc >= 0 && gc <= n;
      const bool bx = ga == 0 || ga == n, by = gc == 0 || gc == n;
      wx = by ? k.w_off * k.w_bd : k.c_ed;   // x-neighbours: M(a, a +- 1) M(c, c)
      wy = bx ? k.w_bd * k.w_off : k.c_ed;   // y-neighbours: M(a, a) M(c, c +- 1)
      inv = bx ? (by ? k.inv_bd2 : k.inv_inbd) : (by ? k.inv_inbd : k.inv_in2);
    }
    const double s = rr[m] - k.c_dd * sd - wx * sx - wy * sy - k.rq * sc;
    V[c * PL_ + B] = in ? s * inv : 0.0;
  }
}

// P0 cells of parity plane (PE, PF): cell (2i + PE, 2j + PF) from its four vertices
template <int WY, int MR, int PE, int PF, bool IN, bool ADJ = false>
__device__ __forceinline__ void sgs_cells(const double* __restrict__ V, double* __restrict__ Cc,
                                          const double (&rc)[MR], int A0, int C0, int n, const SgsK& k) {
  SGS_GEO(WY, MR);
  constexpr int p00 = PE + 2 * PF, p10 = (1 - PE) + 2 * PF, p01 = PE + 2 * (1 - PF), p11 = (1 - PE) + 2 * (1 - PF);
  const int i = threadIdx.x;
#pragma unroll
  for (int m = 0; m < MR; ++m) {
    const int j = ADJ ? 2 * (int)threadIdx.y + m : threadIdx.y + TY_ * m;
    const int B = j * SGS_P + i;
    const double sv = (V[p00 * PL_ + B] + V[p10 * PL_ + B + PE]) +
                      (V[p01 * PL_ + B + PF * SGS_P] + V[p11 * PL_ + B + PF * SGS_P + PE]);
    const double z = (rc[m] - k.rq * sv) * k.inv_q0;
    bool in = true;
    if (!IN) {
      const int e = A0 + 2 * i + PE, f = C0 + 2 * j + PF;
      in = e >= 0 && e < n && f >= 0 && f < n;
    }
    Cc[p00 * PL_ + B] = in ? z : 0.0;
  }
}

// Two ADJACENT plane rows per thread (j0 = 2 ty, j1 = j0 + 1; MR = 2 in k_sgs_tile): the rows
// j0 + PY - 1 .. j0 + PY + 1 of the diagonal and y-neighbour planes serve both updates (9 loads
// instead of 12), and the four cells of each vertex enter through sums formed once per sweep
// direction (the cells only change in the P0 phase between the two directions): 13 shared loads per
// colour and thread instead of 24.  Same expressions in the same order as sgs_colour (bitwise).
template <int WY>
__device__ __forceinline__ void sgs_cellsums(const double* __restrict__ Cc, double (&S)[4][2]) {
  SGS_GEO(WY, 2);
  const int i = threadIdx.x, j0 = 2 * threadIdx.y;
  const double* c00 = Cc;
  const double* c10 = Cc + PL_;
  const double* c01 = Cc + 2 * PL_;
  const double* c11 = Cc + 3 * PL_;
  double a11m[3], a11[3], a01[3], a10m[2], a10[2], a00[2];
#pragma unroll
  for (int r = 0; r < 3; ++r) {          // rows j0 - 1, j0, j1
    const int B = (j0 - 1 + r) * SGS_P + i;
    a11m[r] = c11[B - 1]; a11[r] = c11[B]; a01[r] = c01[B];
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {          // rows j0, j1
    const int B = (j0 + m) * SGS_P + i;
    a10m[m] = c10[B - 1]; a10[m] = c10[B]; a00[m] = c00[B];
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    S[0][m] = (a11m[m] + a01[m]) + (a10m[m] + a00[m]);            // colour (0, 0)
    S[1][m] = (a01[m] + a11[m]) + (a00[m] + a10[m]);              // colour (1, 0)
    S[2][m] = (a10m[m] + a00[m]) + (a11m[m + 1] + a01[m + 1]);    // colour (0, 1)
    S[3][m] = (a00[m] + a10[m]) + (a01[m + 1] + a11[m + 1]);      // colour (1, 1)
  }
}

template <int WY, int PX, int PY, bool IN>
__device__ __forceinline__ void sgs_colour_adj(double* __restrict__ V, const double (&sc)[2], const double (&rr)[2],
                                               int A0, int C0, int n, const SgsK& k) {
  SGS_GEO(WY, 2);
  constexpr int c = PX + 2 * PY, cx = (1 - PX) + 2 * PY, cy = PX + 2 * (1 - PY), cxy = (1 - PX) + 2 * (1 - PY);
  constexpr int OW = PX - 1, OE = PX;
  const int i = threadIdx.x, j0 = 2 * threadIdx.y;
  double D[3][2], Y[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {          // rows j0 + PY - 1 + r
    const int B = (j0 + PY - 1 + r) * SGS_P + i;
    D[r][0] = V[cxy * PL_ + B + OW]; D[r][1] = V[cxy * PL_ + B + OE];
    Y[r] = V[cy * PL_ + B];
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int j = j0 + m;
    const int B = j * SGS_P + i;
    const double sd = (D[m][0] + D[m][1]) + (D[m + 1][0] + D[m + 1][1]);
    const double sx = V[cx * PL_ + B + OW] + V[cx * PL_ + B + OE];
    const double sy = Y[m] + Y[m + 1];
    double wx = k.c_ed, wy = k.c_ed, inv = k.inv_in2;
    bool in = true;
    if (!IN) {
      const int ga = A0 + 2 * i + PX, gc = C0 + 2 * j + PY;
      in = ga >= 0 && ga <= n && gc >= 0 && gc <= n;
      const bool bx = ga == 0 || ga == n, by = gc == 0 || gc == n;
      wx = by ? k.w_off * k.w_bd : k.c_ed;
      wy = bx ? k.w_bd * k.w_off : k.c_ed;
      inv = bx ? (by ? k.inv_bd2 : k.inv_inbd) : (by ? k.inv_inbd : k.inv_in2);
    }
    const double s = rr[m] - k.c_dd * sd - wx * sx - wy * sy - k.rq * sc[m];
    V[c * PL_ + B] = in ? s * inv : 0.0;
  }
}

// The thread's own vertex values own[plane][m] (plane entries (i, j0 + m) of the four vertex planes)
// are kept in registers through the whole sweep: the thread is their only writer, so every read of
// column i on rows j0 / j1 comes from registers (7 shared loads per colour instead of 13, the P0
// phase's own-column vertices likewise).  Same values, same expressions, same order (bitwise).
template <int WY, int PX, int PY, bool IN>
__device__ __forceinline__ void sgs_colour_own(double* __restrict__ V, double (&own)[4][2], const double (&sc)[2],
                                               const double (&rr)[2], int A0, int C0, int n, const SgsK& k) {
  SGS_GEO(WY, 2);
  constexpr int c = PX + 2 * PY, cx = (1 - PX) + 2 * PY, cy = PX + 2 * (1 - PY), cxy = (1 - PX) + 2 * (1 - PY);
  constexpr int OW = PX - 1, OE = PX;
  constexpr int RL = PY == 0 ? 0 : 2;     // the one row of j0 + PY - 1 .. j0 + PY + 1 that is not own
  const int i = threadIdx.x, j0 = 2 * threadIdx.y;
  double D[3][2], Y[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {          // rows j0 + PY - 1 + r; own rows: r - PY + 1 in {0, 1}
    const int B = (j0 + PY - 1 + r) * SGS_P + i;
    if (r == RL) {
      D[r][0] = V[cxy * PL_ + B + OW]; D[r][1] = V[cxy * PL_ + B + OE];
      Y[r] = V[cy * PL_ + B];
    } else {
      const int m = r + PY - 1;
      if (PX == 0) { D[r][0] = V[cxy * PL_ + B + OW]; D[r][1] = own[cxy][m]; }   // OE = 0: own column
      else { D[r][0] = own[cxy][m]; D[r][1] = V[cxy * PL_ + B + OE]; }           // OW = 0: own column
      Y[r] = own[cy][m];
    }
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int j = j0 + m;
    const int B = j * SGS_P + i;
    const double sd = (D[m][0] + D[m][1]) + (D[m + 1][0] + D[m + 1][1]);
    const double sx = PX == 0 ? V[cx * PL_ + B + OW] + own[cx][m] : own[cx][m] + V[cx * PL_ + B + OE];
    const double sy = Y[m] + Y[m + 1];
    double wx = k.c_ed, wy = k.c_ed, inv = k.inv_in2;
    bool in = true;
    if (!IN) {
      const int ga = A0 + 2 * i + PX, gc = C0 + 2 * j + PY;
      in = ga >= 0 && ga <= n && gc >= 0 && gc <= n;
      const bool bx = ga == 0 || ga == n, by = gc == 0 || gc == n;
      wx = by ? k.w_off * k.w_bd : k.c_ed;
      wy = bx ? k.w_bd * k.w_off : k.c_ed;
      inv = bx ? (by ? k.inv_bd2 : k.inv_inbd) : (by ? k.inv_inbd : k.inv_in2);
    }
    const double s = rr[m] - k.c_dd * sd - wx * sx - wy * sy - k.rq * sc[m];
    const double v = in ? s * inv : 0.0;
    V[c * PL_ + B] = v;
    own[c][m] = v;
  }
}

// P0 cells of parity plane (PE, PF) on the rows j0, j1, own-column vertices from registers
template <int WY, int PE, int PF, bool IN>
__device__ __forceinline__ void sgs_cells_own(const double* __restrict__ V, const double (&own)[4][2],
                                              double* __restrict__ Cc, const double (&rc)[2], int A0, int C0, int n,
                                              const SgsK& k) {
  SGS_GEO(WY, 2);
  constexpr int p00 = PE + 2 * PF, p10 = (1 - PE) + 2 * PF, p01 = PE + 2 * (1 - PF), p11 = (1 - PE) + 2 * (1 - PF);
  const int i = threadIdx.x, j0 = 2 * threadIdx.y;
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int j = j0 + m;
    const int B = j * SGS_P + i;
    const bool up_own = PF == 0 || m == 0;          // row j + PF is own
    const double v00 = own[p00][m];
    const double v10 = PE == 0 ? own[p10][m] : V[p10 * PL_ + B + PE];
    const double v01 = up_own ? own[p01][m + PF] : V[p01 * PL_ + B + PF * SGS_P];
    const double v11 = (PE == 0 && up_own) ? own[p11][m + PF] : V[p11 * PL_ + B + PF * SGS_P + PE];
    const double sv = (v00 + v10) + (v01 + v11);
    const double z = (rc[m] - k.rq * sv) * k.inv_q0;
    bool in = true;
    if (!IN) {
      const int e = A0 + 2 * i + PE, f = C0 + 2 * j + PF;
      in = e >= 0 && e < n && f >= 0 && f < n;
    }
    Cc[p00 * PL_ + B] = in ? z : 0.0;
  }
}

// The same register forwarding with ONE plane row per thread (MR = 1, 512-thread 64 x 32 windows):
// own[plane] = the thread's entry (i, j); 5 shared loads per colour instead of 12 (cells by sums)
template <int WY>
__device__ __forceinline__ void sgs_cellsums1(const double* __restrict__ Cc, double (&S)[4]) {
  SGS_GEO(WY, 1);
  const int i = threadIdx.x, j = threadIdx.y;
  const double* c00 = Cc;
  const double* c10 = Cc + PL_;
  const double* c01 = Cc + 2 * PL_;
  const double* c11 = Cc + 3 * PL_;
  double a11m[2], a11[2], a01[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {          // rows j - 1, j
    const int B = (j - 1 + r) * SGS_P + i;
    a11m[r] = c11[B - 1]; a11[r] = c11[B]; a01[r] = c01[B];
  }
  const int B = j * SGS_P + i;
  const double a10m = c10[B - 1], a10 = c10[B], a00 = c00[B];
  S[0] = (a11m[0] + a01[0]) + (a10m + a00);
  S[1] = (a01[0] + a11[0]) + (a00 + a10);
  S[2] = (a10m + a00) + (a11m[1] + a01[1]);
  S[3] = (a00 + a10) + (a01[1] + a11[1]);
}

template <int WY, int PX, int PY, bool IN>
__device__ __forceinline__ void sgs_colour_own1(double* __restrict__ V, double (&own)[4], double sc, double rr,
                                                int A0, int C0, int n, const SgsK& k) {
  SGS_GEO(WY, 1);
  constexpr int c = PX + 2 * PY, cx = (1 - PX) + 2 * PY, cy = PX + 2 * (1 - PY), cxy = (1 - PX) + 2 * (1 - PY);
  constexpr int OW = PX - 1, OE = PX;
  const int i = threadIdx.x, j = threadIdx.y;
  const int B = j * SGS_P + i;
  constexpr int OS = (PY - 1) * SGS_P, ON = PY * SGS_P;
  // diagonal rows j + PY - 1 (S) and j + PY (N): the own row is N for PY = 0, S for PY = 1
  double dSW, dSE, dNW, dNE, ys, yn, sx;
  if (PY == 0) {
    dSW = V[cxy * PL_ + B + OS + OW]; dSE = V[cxy * PL_ + B + OS + OE];
    dNW = PX == 0 ? V[cxy * PL_ + B + OW] : own[cxy];
    dNE = PX == 0 ? own[cxy] : V[cxy * PL_ + B + OE];
    ys = V[cy * PL_ + B + OS]; yn = own[cy];
  } else {
    dSW = PX == 0 ? V[cxy * PL_ + B + OW] : own[cxy];
    dSE = PX == 0 ? own[cxy] : V[cxy * PL_ + B + OE];
    dNW = V[cxy * PL_ + B + ON + OW]; dNE = V[cxy * PL_ + B + ON + OE];
    ys = own[cy]; yn = V[cy * PL_ + B + ON];
  }
  sx = PX == 0 ? V[cx * PL_ + B + OW] + own[cx] : own[cx] + V[cx * PL_ + B + OE];
  const double sd = (dSW + dSE) + (dNW + dNE);
  const double sy = ys + yn;
  double wx = k.c_ed, wy = k.c_ed, inv = k.inv_in2;
  bool in = true;
  if (!IN) {
    const int ga = A0 + 2 * i + PX, gc = C0 + 2 * j + PY;
    in = ga >= 0 && ga <= n && gc >= 0 && gc <= n;
    const bool bx = ga == 0 || ga == n, by = gc == 0 || gc == n;
    wx = by ? k.w_off * k.w_bd : k.c_ed;
    wy = bx ? k.w_bd * k.w_off : k.c_ed;
    inv = bx ? (by ? k.inv_bd2 : k.inv_inbd) : (by ? k.inv_inbd : k.inv_in2);
  }
  const double s = rr - k.c_dd * sd - wx * sx - wy * sy - k.rq * sc;
  const double v = in ? s * inv : 0.0;
  V[c * PL_ + B] = v;
  own[c] = v;
}

template <int WY, int PE, int PF, bool IN>
__device__ __forceinline__ void sgs_cells_own1(const double* __restrict__ V, const double (&own)[4],
                                               double* __restrict__ Cc, double rc, int A0, int C0, int n,
                                               const SgsK& k) {
  SGS_GEO(WY, 1);
  constexpr int p00 = PE + 2 * PF, p10 = (1 - PE) + 2 * PF, p01 = PE + 2 * (1 - PF), p11 = (1 - PE) + 2 * (1 - PF);
  const int i = threadIdx.x, j = threadIdx.y;
  const int B = j * SGS_P + i;
  const double v00 = own[p00];
  const double v10 = PE == 0 ? own[p10] : V[p10 * PL_ + B + PE];
  const double v01 = PF == 0 ? own[p01] : V[p01 * PL_ + B + PF * SGS_P];
  const double v11 = (PE == 0 && PF == 0) ? own[p11] : V[p11 * PL_ + B + PF * SGS_P + PE];
  const double sv = (v00 + v10) + (v01 + v11);
  const double z = (rc - k.rq * sv) * k.inv_q0;
  bool in = true;
  if (!IN) {
    const int e = A0 + 2 * i + PE, f = C0 + 2 * j + PF;
    in = e >= 0 && e < n && f >= 0 && f < n;
  }
  Cc[p00 * PL_ + B] = in ? z : 0.0;
}

template <int WY, int MR, bool IN>
__device__ __forceinline__ void sgs_tile_body(const SgsTileArgs& a, double* V, double* Cc, double* Q, int A0, int C0) {
  SGS_GEO(WY, MR);
  const int i = threadIdx.x, ty = threadIdx.y;
  const int n = a.g.n, n1 = n + 1, nk = a.g.nk;
  const double alpha = a.kproj ? (*a.kproj * a.inv_kk) : 0.0;
  const double* __restrict__ r1 = a.r;
  const double* __restrict__ r0 = a.r + nk;
  const double co_y = a.mode ? a.omega * (1.0 - a.gam) : 0.0;
  const double co_p = a.mode ? 1.0 - a.omega : 0.0;
  const bool use_yp = a.mode && a.yp && co_p != 0.0;
  const double* ys = a.y ? a.y : a.r;      // valid source address for the zero-filling copies
  const double* yps = use_yp ? a.yp : a.r;
  // ---- one staging phase: y (window) and y_prev (tile) by cp.async in row-major order (each
  //      warp reads 32 consecutive words of a global row; the shared destinations are the parity
  //      planes / the tile-ordered Q), r into registers in plane order (the thread's own entries).
  //      Window: thread t stages column t mod 64 of rows t / 64 + 8q (plane and parity fixed per
  //      thread, addresses incremented)
  const int tid = i + SGS_TX * ty;
  {
    constexpr int RSTEP = SGS_TX * TY_ / SGS_W;              // window rows per pass (64 columns)
    static_assert(SGS_TX * TY_ % SGS_W == 0 && RSTEP % 2 == 0 && WY % RSTEP == 0, "fixed parity per thread");
    const int la = tid & (SGS_W - 1), lc0 = tid / SGS_W;
    const int ga = A0 + la;
    double* vdst = V + ((la & 1) + 2 * (lc0 & 1)) * PL_ + (lc0 >> 1) * SGS_P + (la >> 1);
    double* cdst = Cc + (vdst - V);
    const double* vsrc = ys + ga + (int64_t)n1 * (C0 + lc0);
    const double* csrc = ys + nk + ga + (int64_t)n * (C0 + lc0);
    const int64_t dv = (int64_t)RSTEP * n1, dc = (int64_t)RSTEP * n;
    const bool xin_v = IN || (ga >= 0 && ga <= n), xin_c = IN || (ga >= 0 && ga < n);
#pragma unroll 4
    for (int q = 0; q < WY / RSTEP; ++q) {
      const int gc = C0 + lc0 + RSTEP * q;
      const bool inv = IN || (xin_v && gc >= 0 && gc <= n);
      const bool inc = IN || (xin_c && gc >= 0 && gc < n);
      cp_async8(vdst, inv ? vsrc : ys, inv && a.y);
      cp_async8(cdst, inc ? csrc : ys, inc && a.y);
      vdst += (RSTEP / 2) * SGS_P; cdst += (RSTEP / 2) * SGS_P; vsrc += dv; csrc += dc;
    }
  }
  if (use_yp && !a.yp_ldg) {
    for (int idx = tid; idx < SGS_TTX * TTY_; idx += SGS_TX * TY_) {
      const int ga = A0 + SGS_HX + idx % SGS_TTX, gc = C0 + SGS_HY + idx / SGS_TTX;
      const bool okv = IN || (ga <= n && gc <= n), okc = IN || (ga < n && gc < n);
      cp_async8(Q + idx, yps + (okv ? ga + (int64_t)n1 * gc : 0), okv);
      cp_async8(Q + TQ_ + idx, yps + nk + (okc ? ga + (int64_t)n * gc : 0), okc);
    }
  }
  double rv[4][MR], rc[4][MR];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int j = MR == 2 ? 2 * ty + m : ty + TY_ * m;   // MR = 2: adjacent rows (sgs_colour_adj)
      const int ga = A0 + 2 * i + (c & 1), gc = C0 + 2 * j + (c >> 1);
      const bool inv = IN || (ga >= 0 && ga <= n && gc >= 0 && gc <= n);
      const bool inc = IN || (ga >= 0 && ga < n && gc >= 0 && gc < n);
      (void)inc; (void)inv; (void)rv; (void)rc;
    }
  // the vertices' right-hand side read per colour (L1 / L2) instead of held in registers; colour 0's
  // is requested here, behind the staging
  auto rv_of = [&](int c, double (&rr)[2]) {
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int j = 2 * ty + m;
      const int ga = A0 + 2 * i + (c & 1), gc = C0 + 2 * j + (c >> 1);
      const bool inv = IN || (ga >= 0 && ga <= n && gc >= 0 && gc <= n);
      rr[m] = inv ? __ldg(r1 + ga + (int64_t)n1 * gc) - alpha : 0.0;
    }
  };
  auto rv1 = [&](int c) {
    const int ga = A0 + 2 * i + (c & 1), gc = C0 + 2 * ty + (c >> 1);
    const bool inv = IN || (ga >= 0 && ga <= n && gc >= 0 && gc <= n);
    return inv ? __ldg(r1 + ga + (int64_t)n1 * gc) - alpha : 0.0;
  };
  double ra_[2] = {0.0, 0.0}, rb_[2];
  double r1a = 0.0;
  if constexpr (MR == 2) rv_of(0, ra_);
  else r1a = rv1(0);
  cp_async_wait_all();
  __syncthreads();
  // ---- the y / y_prev part of this thread's outputs (tile row-major), before the sweep
  //      overwrites y in place; the write phase below uses the same thread -> entry map
  if (use_yp && a.yp_ldg) {
    // y_prev read from global (L2) here instead of staged by cp.async (the default): fewer MIO
    // operations; all loads of the thread issued before their use (same values, same arithmetic)
    constexpr int NQ = (SGS_TTX * TTY_ + SGS_TX * TY_ - 1) / (SGS_TX * TY_);
    double pv[NQ], pc[NQ];
    // tile entries walked without divisions (see the write phase)
    constexpr int NT = SGS_TX * TY_, DC = NT % SGS_TTX, DR = NT / SGS_TTX;
    {
      int tc = tid % SGS_TTX, tr = tid / SGS_TTX;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int ga = A0 + SGS_HX + tc, gc = C0 + SGS_HY + tr;
        const bool ok = tr < TTY_;
        const bool okv = ok && (IN || (ga <= n && gc <= n)), okc = ok && (IN || (ga < n && gc < n));
        pv[q] = okv ? __ldg(yps + ga + (int64_t)n1 * gc) : 0.0;
        pc[q] = okc ? __ldg(yps + nk + ga + (int64_t)n * gc) : 0.0;
        tc += DC; tr += DR;
        if (tc >= SGS_TTX) { tc -= SGS_TTX; ++tr; }
      }
    }
    int tc = tid % SGS_TTX, tr = tid / SGS_TTX;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (tr >= TTY_) break;
      const int idx = tid + q * NT;
      const int la = SGS_HX + tc, lc = SGS_HY + tr;
      const int pl = ((la & 1) + 2 * (lc & 1)) * PL_ + (lc >> 1) * SGS_P + (la >> 1);
      Q[idx] = fma(co_y, V[pl], co_p * pv[q]);
      Q[TQ_ + idx] = fma(co_y, Cc[pl], co_p * pc[q]);
      tc += DC; tr += DR;
      if (tc >= SGS_TTX) { tc -= SGS_TTX; ++tr; }
    }
  } else {
    for (int idx = tid; idx < SGS_TTX * TTY_; idx += SGS_TX * TY_) {
      const int la = SGS_HX + idx % SGS_TTX, lc = SGS_HY + idx / SGS_TTX;
      const int pl = ((la & 1) + 2 * (lc & 1)) * PL_ + (lc >> 1) * SGS_P + (la >> 1);
      Q[idx] = fma(co_y, V[pl], use_yp ? co_p * Q[idx] : 0.0);
      Q[TQ_ + idx] = fma(co_y, Cc[pl], use_yp ? co_p * Q[TQ_ + idx] : 0.0);
    }
  }
  __syncthreads();
  const SgsK& k = a.k;
  if constexpr (MR == 2) {
    double S[4][2];
    double own[4][2];
    {
      const int j0 = 2 * ty;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int m = 0; m < 2; ++m) own[c][m] = V[c * PL_ + (j0 + m) * SGS_P + i];
    }
    sgs_cellsums<WY>(Cc, S);                                       // cells of the forward sweep
    // the right-hand side of colour c + 1 is requested before colour c is computed: its L2 latency
    // passes behind that colour's arithmetic and barrier instead of in front of the next one's
#define SGS_V(PX, PY, NX, NY, RA, RB) do { rv_of(NX + 2 * NY, RB); \
      sgs_colour_own<WY, PX, PY, IN>(V, own, S[PX + 2 * PY], RA, A0, C0, n, k); __syncthreads(); } while (0)
    SGS_V(0, 0, 1, 0, ra_, rb_); SGS_V(1, 0, 0, 1, rb_, ra_); SGS_V(0, 1, 1, 1, ra_, rb_);   // forward: 0, 1, 2
    // the cells' right-hand side read only now (L1 / L2): not held in registers through the
    // forward sweep, where the cell sums S are live
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        const int j = 2 * ty + m;
        const int ga = A0 + 2 * i + (c & 1), gc = C0 + 2 * j + (c >> 1);
        const bool inc = IN || (ga >= 0 && ga < n && gc >= 0 && gc < n);
        rc[c][m] = inc ? __ldg(r0 + ga + (int64_t)n * gc) + alpha : 0.0;
      }
    sgs_colour_own<WY, 1, 1, IN>(V, own, S[3], rb_, A0, C0, n, k); __syncthreads();          // colour 3
    sgs_cells_own<WY, 0, 0, IN>(V, own, Cc, rc[0], A0, C0, n, k);   // P0 (once: the backward sweep's
    sgs_cells_own<WY, 1, 0, IN>(V, own, Cc, rc[1], A0, C0, n, k);   // P0 update would repeat it exactly)
    sgs_cells_own<WY, 0, 1, IN>(V, own, Cc, rc[2], A0, C0, n, k);
    sgs_cells_own<WY, 1, 1, IN>(V, own, Cc, rc[3], A0, C0, n, k);
    __syncthreads();
    sgs_cellsums<WY>(Cc, S);                                       // cells after the P0 update
    // backward: colours 3, 2, 1, 0 (colour 3's right-hand side is still in rb_)
    SGS_V(1, 1, 0, 1, rb_, ra_); SGS_V(0, 1, 1, 0, ra_, rb_); SGS_V(1, 0, 0, 0, rb_, ra_);
    sgs_colour_own<WY, 0, 0, IN>(V, own, S[0], ra_, A0, C0, n, k); __syncthreads();
#undef SGS_V
  } else {
    static_assert(MR == 1, "one or two rows per thread");
    double S[4];
    double own[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) own[c] = V[c * PL_ + ty * SGS_P + i];
    sgs_cellsums1<WY>(Cc, S);
    // one row per thread: the same request-ahead of the next colour's right-hand side (rv1 below the
    // staging wait would add its L2 latency to every colour of a one-wave, latency-bound step)
#define SGS_V(PX, PY, NX, NY, RA, RB) do { RB = rv1(NX + 2 * NY); \
      sgs_colour_own1<WY, PX, PY, IN>(V, own, S[PX + 2 * PY], RA, A0, C0, n, k); __syncthreads(); } while (0)
    double qa = r1a, qb;
    SGS_V(0, 0, 1, 0, qa, qb); SGS_V(1, 0, 0, 1, qb, qa); SGS_V(0, 1, 1, 1, qa, qb);   // forward: 0, 1, 2
    double rc1[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int ga = A0 + 2 * i + (c & 1), gc = C0 + 2 * ty + (c >> 1);
      const bool inc = IN || (ga >= 0 && ga < n && gc >= 0 && gc < n);
      rc1[c] = inc ? __ldg(r0 + ga + (int64_t)n * gc) + alpha : 0.0;
    }
    sgs_colour_own1<WY, 1, 1, IN>(V, own, S[3], qb, A0, C0, n, k); __syncthreads();      // colour 3
    sgs_cells_own1<WY, 0, 0, IN>(V, own, Cc, rc1[0], A0, C0, n, k);
    sgs_cells_own1<WY, 1, 0, IN>(V, own, Cc, rc1[1], A0, C0, n, k);
    sgs_cells_own1<WY, 0, 1, IN>(V, own, Cc, rc1[2], A0, C0, n, k);
    sgs_cells_own1<WY, 1, 1, IN>(V, own, Cc, rc1[3], A0, C0, n, k);
    __syncthreads();
    sgs_cellsums1<WY>(Cc, S);
    SGS_V(1, 1, 0, 1, qb, qa); SGS_V(0, 1, 1, 0, qa, qb); SGS_V(1, 0, 0, 0, qb, qa);   // backward: 3, 2, 1
    sgs_colour_own1<WY, 0, 0, IN>(V, own, S[0], qa, A0, C0, n, k); __syncthreads();      // and 0
#undef SGS_V
  }
  // the next step's CTAs may launch once every CTA of this grid is writing its tile (they wait in
  // griddepcontrol.wait; triggering at the start would park them on SMs the V-cycle needs)
  asm volatile("griddepcontrol.launch_dependents;");
  // ---- write the tile: out = co_s S(y) + Q, row-major (coalesced global rows)
  const double co_s = a.mode ? a.omega * a.gam : 1.0;
  double kd = 0.0;
  // tile entries idx = tid + q NT walked without divisions: (column, row) and the two output
  // pointers advance by NT = 5 x 50 + 6 (256 threads) resp. 10 x 50 + 12 (512), with a wrap
  constexpr int NT = SGS_TX * TY_, DC = NT % SGS_TTX, DR = NT / SGS_TTX;
  int tc = tid % SGS_TTX, tr = tid / SGS_TTX;
  double* ov = a.out + (A0 + SGS_HX + tc) + (int64_t)n1 * (C0 + SGS_HY + tr);
  double* oc = a.out + nk + (A0 + SGS_HX + tc) + (int64_t)n * (C0 + SGS_HY + tr);
  const int64_t sv = DC + (int64_t)DR * n1, sc = DC + (int64_t)DR * n;
  for (int idx = tid; idx < SGS_TTX * TTY_; idx += NT) {
    const int la = SGS_HX + tc, lc = SGS_HY + tr, ga = A0 + la, gc = C0 + lc;
    const int pl = ((la & 1) + 2 * (lc & 1)) * PL_ + (lc >> 1) * SGS_P + (la >> 1);
    if (IN || (ga <= n && gc <= n)) {
      const double o = fma(co_s, V[pl], Q[idx]);
      *ov = o;
      kd += o;
    }
    if (IN || (ga < n && gc < n)) {
      const double o = fma(co_s, Cc[pl], Q[TQ_ + idx]);
      *oc = o;
      kd -= o;
    }
    tc += DC; tr += DR; ov += sv; oc += sc;
    if (tc >= SGS_TTX) { tc -= SGS_TTX; ++tr; ov += n1 - SGS_TTX; oc += n - SGS_TTX; }
  }
  if (a.kout) { double v[1] = {kd}; reduce_finish<1>(v, a.site, a.slot, a.kout); }
}

#ifndef SGS_MINB
#define SGS_MINB 2
#endif
template <int WY, int MR>
__global__ void __launch_bounds__(SGS_TX * (WY / 2 / MR), SGS_TX * (WY / 2 / MR) <= 256 ? 4 : (SGS_TX * (WY / 2 / MR) <= 512 ? SGS_MINB : 1))
    k_sgs_tile(SgsTileArgs a) {
  SGS_GEO(WY, MR);
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");   // previous step complete and visible
  if (is_done(a.done)) return;
  extern __shared__ double sm[];
  double* V = sm + SGS_PAD;
  double* Cc = V + 4 * PL_;
  double* Q = Cc + 4 * PL_;
  if (threadIdx.x + SGS_TX * threadIdx.y < SGS_PAD) sm[threadIdx.x + SGS_TX * threadIdx.y] = 0.0;
  const int n = a.g.n;
  const int A0 = (blockIdx.x % a.tiles_x) * SGS_TTX - SGS_HX, C0 = (blockIdx.x / a.tiles_x) * TTY_ - SGS_HY;
  const bool interior = A0 >= 1 && A0 + SGS_W - 1 <= n - 1 && C0 >= 1 && C0 + WY - 1 <= n - 1;
  if (interior) sgs_tile_body<WY, MR, true>(a, V, Cc, Q, A0, C0);
  else sgs_tile_body<WY, MR, false>(a, V, Cc, Q, A0, C0);
}

// ---------------------------------------------------------------- SGS on parity planes (TMA)
// The same Chebyshev-SGS step as k_sgs_tile (same colour updates sgs_colour / sgs_cells, same
// arithmetic, same outputs) on an internal "planar" copy of the pressure vectors: 8 planes (vertex
// parities q = px + 2 py, then cell parities) of ph x pw entries, plane q entry (i, j) = vertex
// (2i + px, 2j + py) (cell (2i + px, 2j + py)), zero outside the domain.  A window's 8 parity
// planes are then one dense 3D box {32, 32, 8} of the planar tensor: ONE TMA load
// (cp.async.bulk.tensor, hardware zero fill outside the tensor) replaces the 32 per-thread
// stride-2 cp.async gathers and their index arithmetic, and every global row access of the step
// (r, y, y_prev, out) is a contiguous plane row.  y (window) arrives by TMA; r is read into
// registers (coalesced) while the TMA is in flight; y and y_prev at the thread's own tile entries
// are read at write time (L2: y was just fetched, y_prev is prefetched to L2 by a TMA prefetch at
// the start), so the Q pass and its 46 KB of shared memory are gone (64 KB per CTA).
// The last step of a chain writes the ABI (lexicographic) layout directly.
struct SgsPlaneArgs {
  MassGeo g;
  SgsK k;
  int pw, ph; int64_t pl;        // planar geometry: plane row length, rows, plane size
  const double* rp;              // planar r (Pi applied on the fly: r - (kproj / k^T k) k)
  const double* kproj;
  double inv_kk;
  const double* yg;              // planar y (nullable = 0: first step); the TMA map describes it
  const double* ypg;             // planar y_prev (nullable)
  double* outp;                  // planar output (or null when out_abi is set)
  double* out_abi;               // ABI-layout output of the chain's last step
  double omega, gam;
  int tiles_x;
  RedSite site; int slot; double* kout;
  const double* done;
  int pdl;
};
constexpr int SGSP_PAD = 128;                                      // zero words before V (edge reads at -33)
// TMA box origins must be 16-byte aligned in the innermost dimension: the window's first plane
// column A0 / 2 must be even, so the tile is 48 wide (halo 8 / 8, the right one >= 6 as required)
// instead of k_sgs_tile's 50; vertically (dimension 1, no alignment rule) it is 26 (64 x 32
// windows, 256 threads, two adjacent plane rows per thread: the geometry and the register-forwarding
// sweep of k_sgs_tile<32, 2>).
constexpr int SGSP_TTX = 48;
constexpr int SGSP_WY = 32, SGSP_TY = SGSP_WY / 4, SGSP_TTY = SGSP_WY - 6;
constexpr int SGSP_PLW = SGS_P * (SGSP_WY / 2);                    // one plane of the window (32 x 16)
static_assert(SGS_W - SGS_HX - SGSP_TTX >= 6 && (SGSP_TTX / 2) % 2 == 0 && (SGS_HX / 2) % 2 == 0, "TMA-aligned tile");
constexpr int SGSP_BYTES = 8 * SGSP_PLW * (int)sizeof(double);     // one TMA box (8 planes x 16 x 32)
constexpr int SGSP_TAIL = 64;                                      // zero words after Cc (edge reads at +32)
constexpr int SGSP_SMEM = (SGSP_PAD + 8 * SGSP_PLW + SGSP_TAIL) * (int)sizeof(double) + 1024 + 64;   // + alignment slack, mbarrier

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <bool IN>
__device__ __forceinline__ void sgsp_body(const SgsPlaneArgs& a, double* V, double* Cc, unsigned bar, bool tma,
                                          int A0, int C0) {
  constexpr int WY = SGSP_WY;
  const int i = threadIdx.x, ty = threadIdx.y;
  const int n = a.g.n;
  const int pw = a.pw;
  const int64_t pl = a.pl;
  const int X0 = A0 >> 1, Y0 = C0 >> 1;                      // window origin in plane coordinates
  const double alpha = a.kproj ? (*a.kproj * a.inv_kk) : 0.0;
  const int64_t o0 = (int64_t)(Y0 + 2 * ty) * pw + (X0 + i);   // the thread's entry (i, 2 ty) of a plane
  if (tma) {
    // wait for the window (phase 0 of the single-use barrier)
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar)
        : "memory");
  }
  __syncthreads();
  const SgsK& k = a.k;
  double S[4][2];
  double own[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int m = 0; m < 2; ++m) own[c][m] = V[c * SGSP_PLW + (2 * ty + m) * SGS_P + i];
  sgs_cellsums<WY>(Cc, S);                                       // cells of the forward sweep
  // right-hand side of the thread's entries, one contiguous plane row per warp, read per colour
  auto rv_of = [&](int c, double (&rr)[2]) {
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int ga = A0 + 2 * i + (c & 1), gc = C0 + 2 * (2 * ty + m) + (c >> 1);
      const bool inv = IN || (ga >= 0 && ga <= n && gc >= 0 && gc <= n);
      rr[m] = inv ? __ldg(a.rp + c * pl + o0 + m * pw) - alpha : 0.0;
    }
  };
#define SGS_V(PX, PY) do { double rr_[2]; rv_of(PX + 2 * PY, rr_); \
    sgs_colour_own<WY, PX, PY, IN>(V, own, S[PX + 2 * PY], rr_, A0, C0, n, k); __syncthreads(); } while (0)
  SGS_V(0, 0); SGS_V(1, 0); SGS_V(0, 1); SGS_V(1, 1);          // forward: colours 0, 1, 2, 3
  {
    double rc[4][2];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int ga = A0 + 2 * i + (c & 1), gc = C0 + 2 * (2 * ty + m) + (c >> 1);
        const bool inc = IN || (ga >= 0 && ga < n && gc >= 0 && gc < n);
        rc[c][m] = inc ? __ldg(a.rp + (4 + c) * pl + o0 + m * pw) + alpha : 0.0;
      }
    sgs_cells_own<WY, 0, 0, IN>(V, own, Cc, rc[0], A0, C0, n, k);   // P0 (once; see k_sgs_tile)
    sgs_cells_own<WY, 1, 0, IN>(V, own, Cc, rc[1], A0, C0, n, k);
    sgs_cells_own<WY, 0, 1, IN>(V, own, Cc, rc[2], A0, C0, n, k);
    sgs_cells_own<WY, 1, 1, IN>(V, own, Cc, rc[3], A0, C0, n, k);
  }
  __syncthreads();
  sgs_cellsums<WY>(Cc, S);                                       // cells after the P0 update
  SGS_V(1, 1); SGS_V(0, 1); SGS_V(1, 0);
  {                                                              // backward colour 0: the write phase reads the
    double rr_[2]; rv_of(0, rr_);                                // thread's own entries only (registers / own cells)
    sgs_colour_own<WY, 0, 0, IN>(V, own, S[0], rr_, A0, C0, n, k);
  }
#undef SGS_V
  asm volatile("griddepcontrol.launch_dependents;");
  // ---- write the own tile entries: out = co_s S(y) + (co_y y + co_p y_prev), as k_sgs_tile; y and
  //      y_prev at the thread's entries come from L2 (y was just fetched by the TMA, y_prev by the
  //      prefetch), contiguous plane rows
  const bool tile_x = i >= SGS_HX / 2 && i < SGS_HX / 2 + SGSP_TTX / 2;
  const double co_s = a.omega * a.gam;
  const double co_y = a.omega * (1.0 - a.gam);
  const double co_p = 1.0 - a.omega;
  const bool use_yp = a.ypg && co_p != 0.0;
  const int n1 = n + 1, nk = a.g.nk;
  double kd = 0.0;
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int j = 2 * ty + m;
    if (!tile_x || j < SGS_HY / 2 || j >= SGS_HY / 2 + SGSP_TTY / 2) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {                      // vertex planes, then cell planes
    double yv[4], ypv[4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int64_t po = (4 * h + qq) * pl + o0 + m * pw;
      yv[qq] = a.yg ? __ldg(a.yg + po) : 0.0;
      ypv[qq] = use_yp ? __ldg(a.ypg + po) : 0.0;
    }
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int q = 4 * h + qq;
      const int px = q & 1, py = (q >> 1) & 1;
      const int ga = A0 + 2 * i + px, gc = C0 + 2 * j + py;
      const bool vert = q < 4;
      if (!IN && !(vert ? (ga <= n && gc <= n) : (ga < n && gc < n))) continue;
      const double sv = vert ? own[q & 3][m] : Cc[(q & 3) * SGSP_PLW + j * SGS_P + i];
      const double Q = fma(co_y, yv[qq], use_yp ? co_p * ypv[qq] : 0.0);
      const double o = fma(co_s, sv, Q);
      if (a.out_abi) {
        if (vert) a.out_abi[ga + (int64_t)n1 * gc] = o;
        else a.out_abi[nk + ga + (int64_t)n * gc] = o;
      } else {
        a.outp[q * pl + o0 + m * pw] = o;
      }
      kd += vert ? o : -o;
    }
    }
  }
  if (a.kout) { double v[1] = {kd}; reduce_finish<1>(v, a.site, a.slot, a.kout); }
}

__global__ void __launch_bounds__(SGS_TX * SGSP_TY, 4) k_sgs_plane(const __grid_constant__ SgsPlaneArgs a,
                                                                  const __grid_constant__ CUtensorMap tm_y,
                                                                  const __grid_constant__ CUtensorMap tm_yp) {
  extern __shared__ unsigned char sgsp_raw[];
  // 1024-byte aligned window: [pad | V (4 planes) | Cc (4 planes) | tail], mbarrier after it
  const unsigned base = smem_u32(sgsp_raw);
  const unsigned off = ((base + SGSP_PAD * 8 + 1023u) & ~1023u) - base;
  double* V = reinterpret_cast<double*>(sgsp_raw + off);
  double* Cc = V + 4 * SGSP_PLW;
  double* pad = V - SGSP_PAD;
  double* tail = Cc + 4 * SGSP_PLW;
  unsigned long long* barp = reinterpret_cast<unsigned long long*>(tail + SGSP_TAIL);
  const unsigned bar = smem_u32(barp);
  const int tid = threadIdx.x + SGS_TX * threadIdx.y;
  const int n = a.g.n;
  const int A0 = (blockIdx.x % a.tiles_x) * SGSP_TTX - SGS_HX, C0 = (blockIdx.x / a.tiles_x) * SGSP_TTY - SGS_HY;
  const bool tma = a.yg != nullptr;
  if (tid == 0) {
    if (a.ypg) {   // y_prev is only read at write time: start pulling its window into L2 now
      asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(&tm_yp), "r"(A0 >> 1),
                   "r"(C0 >> 1), "r"(0) : "memory");
    }
    if (tma) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();                                                  // barrier initialised before any wait
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");   // previous step complete and visible
  if (is_done(a.done)) return;
  if (tid < SGSP_PAD) pad[tid] = 0.0;
  if (tid < SGSP_TAIL) tail[tid] = 0.0;
  if (tma) {
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(SGSP_BYTES) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(smem_u32(V)), "l"(&tm_y), "r"(A0 >> 1), "r"(C0 >> 1), "r"(0), "r"(bar)
          : "memory");
    }
  } else {   // first step: y = 0
    for (int t = tid; t < 8 * SGSP_PLW; t += SGS_TX * SGSP_TY) V[t] = 0.0;
  }
  const bool interior = A0 >= 1 && A0 + SGS_W - 1 <= n - 1 && C0 >= 1 && C0 + SGSP_WY - 1 <= n - 1;
  if (interior) sgsp_body<true>(a, V, Cc, bar, tma, A0, C0);
  else sgsp_body<false>(a, V, Cc, bar, tma, A0, C0);
}

// planar copy of r (rp) fused with k^T r (the Pi projection coefficient of Pi C Pi, reading R6)
__global__ void __launch_bounds__(BS) k_kdot_planar(int n, int64_t np, int pw, int64_t pl, const double* x,
                                                    double* xp, RedSite site, int slot, double* out,
                                                    const double* done) {
  if (is_done(done)) return;
  const int n1 = n + 1;
  const int64_t nk = (int64_t)n1 * n1;
  double s = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < np; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[t];
    int a, c, q;
    if (t < nk) { a = (int)(t % n1); c = (int)(t / n1); q = (a & 1) + 2 * (c & 1); s += v; }
    else { const int64_t e = t - nk; a = (int)(e % n); c = (int)(e / n); q = 4 + (a & 1) + 2 * (c & 1); s -= v; }
    xp[q * pl + (int64_t)(c >> 1) * pw + (a >> 1)] = v;
  }
  double v[1] = {s};
  reduce_finish<1>(v, site, slot, out);
}

// k^T x
__global__ void __launch_bounds__(BS) k_kdot(int nk, int64_t np, const double* x, RedSite site, int slot,
                                             double* out, const double* done) {
  if (is_done(done)) return;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x)
    s += (i < nk) ? x[i] : -x[i];
  double v[1] = {s};
  reduce_finish<1>(v, site, slot, out);
}

// z = y - (ky / kk) k, optional partial <z, w>
__global__ void __launch_bounds__(BS) k_kproject_out(int nk, int64_t np, const double* y, const double* ky,
                                                     double inv_kk, double scale, double* z, const double* w,
                                                     RedSite site, int slot, double* out, const double* done) {
  if (is_done(done)) return;
  const double beta = *ky * inv_kk;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    double v = y[i] - beta * ((i < nk) ? 1.0 : -1.0);
    if (scale != 1.0) v *= scale;
    z[i] = v;
    if (w) s += v * w[i];
  }
  if (out) { double v[1] = {s}; reduce_finish<1>(v, site, slot, out); }
}

// generic dot product
__global__ void __launch_bounds__(BS) k_dot(const double* a, const double* b, int64_t n, RedSite site, int slot,
                                            double* out, const double* done) {
  if (is_done(done)) return;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  double v[1] = {s};
  reduce_finish<1>(v, site, slot, out);
}

// dense (M_Q + k k^T) for the P1 exact solve (small n only)
__global__ void k_dense_mq_kk(MassGeo g, double* D) {
  const int64_t np = (int64_t)g.nk + g.n0;
  const int n = g.n, n1 = n + 1; const double h = g.h;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < np * np; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / np, j = t % np;
    double v = 0.0;
    if (i < g.nk && j < g.nk) {
      const int a = (int)(i % n1), c = (int)(i / n1), aa = (int)(j % n1), cc = (int)(j / n1);
      v = ml1(n, h, a, aa) * ml1(n, h, c, cc);
    } else if (i >= g.nk && j >= g.nk) {
      v = (i == j) ? h * h : 0.0;
    } else {
      const int64_t p = i < g.nk ? i : j, T = (i < g.nk ? j : i) - g.nk;
      const int a = (int)(p % n1), c = (int)(p / n1), e = (int)(T % n), f = (int)(T / n);
      if ((a == e || a == e + 1) && (c == f || c == f + 1)) v = 0.25 * h * h;
    }
    const double ki = (i < g.nk) ? 1.0 : -1.0, kj = (j < g.nk) ? 1.0 : -1.0;
    D[t] = v + ki * kj;
  }
}
// W = Minv - k k^T / (k^T k)^2
__global__ void k_dense_fix_k(double* W, int nk, int64_t np) {
  const double kk = (double)np;
  const double f = 1.0 / (kk * kk);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < np * np; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / np, j = t % np;
    const double ki = (i < nk) ? 1.0 : -1.0, kj = (j < nk) ? 1.0 : -1.0;
    W[t] -= f * ki * kj;
  }
}
// dense copy of a scalar SELL operator (coarse level)
__global__ void k_sell_to_dense(Sell A, int m, double* D) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = t / SELL_C;
  if (s >= A.nslices) return;
  const int lane = (int)(t % SELL_C);
  const int row = A.perm ? A.perm[t] : (t < A.nrows ? (int)t : -1);
  if (row < 0) return;
  for (int k = 0; k < A.slen[s]; ++k) {
    const int64_t e = A.sptr[s] + lane + (int64_t)k * SELL_C;
    D[(int64_t)row * m + A.col[e]] += A.val[e];
  }
}

}  // namespace

// ================================================================ host side

static MassGeo mass_geo(const Geo& g) { MassGeo m{g.n, g.nk, g.n0, g.h}; return m; }

// ---------------------------------------------------------------- tiled matrix-free saddle apply
// y = [A B^T; B 0] x on the Stokes system (reduced: P0 columns / rows dropped) with x staged in
// shared memory: a CTA owns a 64 x 64 tile of Q2 nodes (both components), the 32 x 32 Q1 vertices
// and P0 cells at its even origin, and stages the node window with a halo of 2 (the stencil
// radius), split by column parity (E: even, O: odd columns) so that every warp access, for the
// node pairs of the velocity rows and for the stride-2 node gathers of the pressure rows, is 32
// consecutive words; plus the Q1 (34 x 34) and P0 (33 x 33) windows the B^T parts read.  All
// staging is cp.async (zero-filled outside the domain).  Velocity rows: lanes own a column pair
// (even i, odd i + 1), a warp walks 8 rows with a 5-row x 6-column register window, one
// component at a time.  Every row's arithmetic is that of k_saddle_mf in the same order
// (Dirichlet / outside nodes read as 0 where k_saddle_mf skips them; zero-weight taps skipped),
// so y is bitwise the same.
constexpr int ST_T = 64;               // tile side in Q2 nodes (even origin)
constexpr int ST_W = ST_T + 4;         // staged window (halo 2)
constexpr int ST_H = ST_W / 2;         // entries per parity row (34)
constexpr int ST_PW = ST_T / 2 + 2;    // Q1 window (vertices I0/2 - 1 ... I0/2 + 32)
constexpr int ST_CW = ST_T / 2 + 1;    // P0 window (cells I0/2 - 1 ... I0/2 + 31)
constexpr int ST_THREADS = 256;
constexpr int ST_ROWS = ST_T / (ST_THREADS / 32);   // 8 tile rows per warp
constexpr int ST_SCR = 2 * (ST_T / 2) * (ST_T / 2);   // component-0 partial sums of the tile's pressure rows
constexpr int ST_SMEM = (4 * ST_W * ST_H + ST_PW * ST_PW + ST_CW * ST_CW + ST_SCR) * (int)sizeof(double);
static_assert(ST_T == 2 * 32 && ST_ROWS % 2 == 0, "lane = column pair, even strips");

// Structural zeros of the B / B^T class weights (the kernel skips them at compile time; the launch
// checks that every weight outside these patterns is exactly 0, else the gather kernel runs).  The
// weights are products of 1D tables; per direction, for a Q2 node of type V (on a Q1 vertex) or
// M (element midpoint): the Q1 derivative table vanishes on the node's own vertex (V: vertices
// -1, +1; M: 0, +1), the Q1 mass table on the neighbouring vertices of a V node (V: 0; M: 0, +1);
// the P0 derivative table vanishes for M nodes (V: cells -1, 0), the P0 mass table is V: -1, 0,
// M: 0.  Component C takes the derivative table in direction C and the mass table in the other.
__host__ __device__ constexpr bool st_pat1(int p, bool deriv, int d) {     // d in {-1, 0, 1}
  return p == 0 ? (deriv ? d != 0 : d == 0) : (d == 0 || d == 1);
}
__host__ __device__ constexpr bool st_pat0(int p, bool deriv, int d) {     // d in {-1, 0}
  return p == 0 ? true : (deriv ? false : d == 0);
}
__host__ __device__ constexpr bool st_m_bt1(int cl, int C, int dc, int da) {
  return st_pat1(cl & 1, C == 0, da) && st_pat1(cl >> 1, C == 1, dc);
}
__host__ __device__ constexpr bool st_m_bt0(int cl, int C, int df, int de) {
  return st_pat0(cl & 1, C == 0, de) && st_pat0(cl >> 1, C == 1, df);
}
__host__ __device__ constexpr bool st_m_b1(int C, int dj, int di) {        // di, dj in -2 .. 2
  return (C == 0 ? di != 0 : (di >= -1 && di <= 1)) && (C == 1 ? dj != 0 : (dj >= -1 && dj <= 1));
}
__host__ __device__ constexpr bool st_m_b0(int C, int dj, int di) {        // di, dj in 0 .. 2
  return C == 0 ? di != 1 : dj != 1;
}
static bool saddle_masks_ok(const SaddleSt& w) {
  for (int cl = 0; cl < 4; ++cl)
    for (int C = 0; C < 2; ++C) {
      for (int dc = -1; dc <= 1; ++dc)
        for (int da = -1; da <= 1; ++da)
          if (!st_m_bt1(cl, C, dc, da) && w.bt1[cl][C][(dc + 1) * 3 + da + 1] != 0.0) return false;
      for (int df = -1; df <= 0; ++df)
        for (int de = -1; de <= 0; ++de)
          if (!st_m_bt0(cl, C, df, de) && w.bt0[cl][C][(df + 1) * 2 + de + 1] != 0.0) return false;
    }
  for (int C = 0; C < 2; ++C) {
    for (int dj = -2; dj <= 2; ++dj)
      for (int di = -2; di <= 2; ++di)
        if (!st_m_b1(C, dj, di) && w.b1[C][(dj + 2) * 5 + di + 2] != 0.0) return false;
    for (int dj = 0; dj <= 2; ++dj)
      for (int di = 0; di <= 2; ++di)
        if (!st_m_b0(C, dj, di) && w.b0[C][dj * 3 + di] != 0.0) return false;
  }
  return true;
}

struct SaddleTileArgs {
  StencilOp so; SaddleSt w;
  int m, n, nq, nk, tiles_x; int64_t n_u; int reduced;
  const double* x; double* y; const double* inv_scale;
  RedSite site; int slot; double* dot_out; const double* done;
};

// shared-memory layout (one dynamic array; every offset a compile-time constant): E0, O0, E1, O1
// (ST_W rows x ST_H), then the Q1 window (ST_PW x ST_PW), then the P0 window (ST_CW x ST_CW)
extern __shared__ __align__(16) double st_sm[];
constexpr int ST_OFF_P1 = 4 * ST_W * ST_H, ST_OFF_P0 = ST_OFF_P1 + ST_PW * ST_PW, ST_OFF_SCR = ST_OFF_P0 + ST_CW * ST_CW;
struct StSmem {
  __device__ __forceinline__ const double* E(int c) const { return st_sm + 2 * c * ST_W * ST_H; }
  __device__ __forceinline__ const double* O(int c) const { return st_sm + (2 * c + 1) * ST_W * ST_H; }
  __device__ __forceinline__ const double* P1() const { return st_sm + ST_OFF_P1; }
  __device__ __forceinline__ const double* P0() const { return st_sm + ST_OFF_P0; }
  // node at window (wi, wj) of component c
  __device__ __forceinline__ double node(int c, int wi, int wj) const {
    return (wi & 1) ? O(c)[wj * ST_H + (wi >> 1)] : E(c)[wj * ST_H + (wi >> 1)];
  }
};

// window row wr of component c for lane L: columns 2L .. 2L + 4 (the pair's taps: the even node
// at 2L + 2 reads 2L .. 2L + 4, the odd node at 2L + 3 reads 2L + 2 .. 2L + 4), Dirichlet /
// outside nodes as 0 on edge tiles
template <bool EDGE>
__device__ __forceinline__ void st_load_row(const StSmem& S, int c, int wr, int L, int I0, int J0, int m,
                                            double (&v)[5]) {
  const double* e = S.E(c) + wr * ST_H + L;
  const double* o = S.O(c) + wr * ST_H + L;
  v[0] = e[0]; v[1] = o[0]; v[2] = e[1]; v[3] = o[1]; v[4] = e[2];
  if (EDGE) {
    const int gj = J0 - 2 + wr;
    const bool rowd = gj <= 0 || gj >= m - 1;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int gi = I0 - 2 + 2 * L + k;
      if (rowd || gi <= 0 || gi >= m - 1) v[k] = 0.0;
    }
  }
}

// A-part of one velocity row of class CL from the register window (output at window column
// offset OC within the 6 loaded columns; RSLOT: ring slot of the output row)
template <int CL, int OC, int RSLOT>
__device__ __forceinline__ double st_lap(const StencilOp& so, const double (&win)[5][5]) {
  constexpr int PI = CL & 1, PJ = CL >> 1, RX = PI ? 1 : 2, RY = PJ ? 1 : 2;
  double a = 0.0;
#pragma unroll
  for (int dj = -RY; dj <= RY; ++dj)
#pragma unroll
    for (int di = -RX; di <= RX; ++di)
      a = fma(so.w[CL][(dj + 2) * 5 + di + 2], win[(RSLOT + dj + 5) % 5][OC + di], a);
  return a;
}

// one output row t of the warp's strip for component C (compile-time t: ring slots, classes)
template <int C, bool EDGE, int t>
__device__ __forceinline__ void st_vel_row(const SaddleTileArgs& a, const StSmem& S, int L, int tj0, int I0, int J0,
                                           double sc, double (&win)[5][5], double& dot) {
  const int m = a.m, n = a.n;
  if (t + 4 < ST_ROWS + 4) st_load_row<EDGE>(S, C, tj0 + t + 4, L, I0, J0, m, win[(t + 4) % 5]);
  constexpr int RS = (t + 2) % 5;
  constexpr int PJ = (t & 1);                 // tile rows start even: row parity = t parity
  const int tj = tj0 + t, j = J0 + tj;
  const int jc = j >> 1;
  const int pr = jc - (J0 >> 1) + 1;          // Q1 / P0 window row of jc
  double q[2];
  q[0] = st_lap<2 * PJ, 2, RS>(a.so, win);
  q[1] = st_lap<2 * PJ + 1, 3, RS>(a.so, win);
  double out[2] = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = I0 + 2 * L + k;
    if (EDGE && (i >= m || j >= m)) continue;
    const int cl = 2 * PJ + k;
    const double raw = S.node(C, 2 * L + 2 + k, tj + 2);
    double ax;
    if (EDGE && (i == 0 || j == 0 || i == m - 1 || j == m - 1)) {   // identity row; B^T rows are empty
      ax = fma(1.0, raw, 0.0) + 0.0;
      if (!a.reduced) ax += 0.0;
    } else {
      double bx = 0.0;
#pragma unroll
      for (int dc = -1; dc <= 1; ++dc)
#pragma unroll
        for (int da = -1; da <= 1; ++da) {
          if (!st_m_bt1(2 * PJ + k, C, dc, da)) continue;         // structural zero (compile time)
          bx = fma(a.w.bt1[cl][C][(dc + 1) * 3 + da + 1], S.P1()[(pr + dc) * ST_PW + L + 1 + da], bx);
        }
      ax = q[k] + bx;
      if (!a.reduced) {
        double cx = 0.0;
#pragma unroll
        for (int df = -1; df <= 0; ++df)
#pragma unroll
          for (int de = -1; de <= 0; ++de) {
            if (!st_m_bt0(2 * PJ + k, C, df, de)) continue;
            cx = fma(a.w.bt0[cl][C][(df + 1) * 2 + de + 1], S.P0()[(pr + df) * ST_CW + L + 1 + de], cx);
          }
        ax += cx;
      }
    }
    ax *= sc;
    if (EDGE) a.y[(int64_t)C * a.nq + i + (int64_t)m * j] = ax;
    out[k] = ax;
    if (a.dot_out) dot += ax * (sc * raw);
  }
  if (!EDGE) {
    // 16-byte stores of aligned pairs (a warp row = 512 contiguous bytes, no half-written
    // sectors); rows whose pair addresses are only 8-byte aligned (warp-uniform: lanes are 16 B
    // apart) pair lane L's odd column with lane L + 1's even one
    double* yr = a.y + (int64_t)C * a.nq + I0 + (int64_t)m * j + 2 * L;
    if ((reinterpret_cast<uintptr_t>(yr) & 15) == 0) {
      *reinterpret_cast<double2*>(yr) = make_double2(out[0], out[1]);
    } else {
      const double nx = __shfl_down_sync(0xffffffffu, out[0], 1);
      if (L == 0) yr[0] = out[0];
      if (L < 31) *reinterpret_cast<double2*>(yr + 1) = make_double2(out[1], nx);
      else yr[1] = out[1];
    }
  }
  // ---- pressure rows of the tile's vertex / cell (L, tj / 2) on even rows: the 5 x 5 (Q1) and
  //      3 x 3 (P0) node neighbourhoods of node (2 va, 2 vc) are exactly this lane's register
  //      window (columns 2L .. 2L + 4, rows tj - 2 .. tj + 2), so B u needs no further loads.
  //      Component 0's sum waits in the thread's own scratch entry for component 1's.
  if constexpr ((t & 1) == 0) {
    const int cr = tj >> 1;
    double q1 = 0.0, q0 = 0.0;
#pragma unroll
    for (int dj = -2; dj <= 2; ++dj)
#pragma unroll
      for (int di = -2; di <= 2; ++di)
        if (st_m_b1(C, dj, di)) q1 = fma(a.w.b1[C][(dj + 2) * 5 + di + 2], win[(RS + dj + 5) % 5][2 + di], q1);
#pragma unroll
    for (int dj = 0; dj <= 2; ++dj)
#pragma unroll
      for (int di = 0; di <= 2; ++di)
        if (st_m_b0(C, dj, di)) q0 = fma(a.w.b0[C][dj * 3 + di], win[(RS + dj) % 5][2 + di], q0);
    double* scr = st_sm + ST_OFF_SCR + cr * (ST_T / 2) + L;
    if (C == 0) {
      scr[0] = q1; scr[ST_SCR / 2] = q0;
    } else {
      const int va = (I0 >> 1) + L, vc = (J0 >> 1) + cr;
      if (!EDGE || (va <= n && vc <= n)) {
        const double acc = (scr[0] + q1) * sc;
        a.y[a.n_u + va + (int64_t)(n + 1) * vc] = acc;
        if (a.dot_out) dot += acc * (sc * S.P1()[(cr + 1) * ST_PW + L + 1]);
      }
      if (!EDGE || (va < n && vc < n)) {
        double acc = (scr[ST_SCR / 2] + q0) * sc;
        if (a.reduced) acc = 0.0;
        a.y[a.n_u + a.nk + va + (int64_t)n * vc] = acc;
        if (a.dot_out) dot += acc * (sc * S.P0()[(cr + 1) * ST_CW + L + 1]);
      }
    }
  }
}

template <int C, bool EDGE, int... Ts>
__device__ __forceinline__ void st_vel_rows(const SaddleTileArgs& a, const StSmem& S, int L, int tj0, int I0, int J0,
                                            double sc, double (&win)[5][5], double& dot, std::integer_sequence<int, Ts...>) {
  (st_vel_row<C, EDGE, Ts>(a, S, L, tj0, I0, J0, sc, win, dot), ...);
}

template <int C, bool EDGE>
__device__ __forceinline__ void st_vel(const SaddleTileArgs& a, const StSmem& S, int I0, int J0, double sc, double& dot) {
  const int L = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tj0 = ST_ROWS * w;                // first tile row of the strip; window row = tile row + 2
  double win[5][5];
#pragma unroll
  for (int r = 0; r < 4; ++r) st_load_row<EDGE>(S, C, tj0 + r, L, I0, J0, a.m, win[r]);   // rows tj0-2 .. tj0+1
  st_vel_rows<C, EDGE>(a, S, L, tj0, I0, J0, sc, win, dot, std::make_integer_sequence<int, ST_ROWS>{});
}

// node value for the pressure rows (Dirichlet / outside -> 0 on edge tiles)
template <bool EDGE>
__device__ __forceinline__ double st_pnode(const StSmem& S, int c, int wi, int wj, int I0, int J0, int m) {
  const double v = S.node(c, wi, wj);
  if (!EDGE) return v;
  const int gi = I0 - 2 + wi, gj = J0 - 2 + wj;
  return (gi <= 0 || gj <= 0 || gi >= m - 1 || gj >= m - 1) ? 0.0 : v;
}

template <bool EDGE>
__device__ __forceinline__ void st_body(const SaddleTileArgs& a, const StSmem& S, int I0, int J0, double sc) {
  double dot = 0.0;
  st_vel<0, EDGE>(a, S, I0, J0, sc, dot);
  st_vel<1, EDGE>(a, S, I0, J0, sc, dot);
  if (a.dot_out) { double v[1] = {dot}; reduce_finish<1>(v, a.site, a.slot, a.dot_out); }
}

#ifndef ST_MINB
#define ST_MINB 2
#endif
__global__ void __launch_bounds__(ST_THREADS, ST_MINB) k_saddle_tile(SaddleTileArgs a) {
  if (is_done(a.done)) return;
  const StSmem S;
  const int m = a.m, n = a.n, n1 = n + 1;
  const int I0 = (blockIdx.x % a.tiles_x) * ST_T, J0 = (blockIdx.x / a.tiles_x) * ST_T;
  const double sc = a.inv_scale ? *a.inv_scale : 1.0;
  const double* xu = a.x;
  const double* p1 = a.x + a.n_u;
  const double* p0 = p1 + a.nk;
  // ---- stage (cp.async).  Interior tiles: every window entry is inside the domain, and element
  //      idx = tid + 256 k of a window of width W is walked incrementally (row += 256 / W, column +=
  //      256 % W with a wrap) from one running source pointer; the shared destinations are linear in
  //      idx (node planes: idx / 2 within the thread's fixed parity plane).  Edge tiles: zero fill
  //      outside the domain.
  const bool edge = I0 - 2 < 1 || J0 - 2 < 1 || I0 + ST_T + 1 > m - 2 || J0 + ST_T + 1 > m - 2;
  if (!edge) {
    const int tid = threadIdx.x;
    {
      constexpr int TOT = ST_W * ST_W, NF = TOT / ST_THREADS, DJ = ST_THREADS / ST_W, DI = ST_THREADS % ST_W;
      static_assert(ST_W == 2 * ST_H && DI % 2 == 0 && ST_THREADS % 2 == 0, "fixed parity plane, linear destination");
      int wj = tid / ST_W, wi = tid - ST_W * wj;
      const double* src = xu + ((int64_t)m * (J0 - 2 + wj) + (I0 - 2 + wi));
      double* dst = st_sm + ((wi & 1) ? ST_W * ST_H : 0) + (tid >> 1);
      const int64_t step = (int64_t)DJ * m + DI, wrap = (int64_t)m - ST_W;
      // component 0 now, component 1 after the pressure windows, in a second cp.async group:
      // its latency passes behind component 0's velocity walk
#pragma unroll 6
      for (int k = 0; k < NF; ++k) {
        cp_async8(dst, src, true);
        dst += ST_THREADS / 2; src += step; wi += DI;
        if (wi >= ST_W) { wi -= ST_W; src += wrap; }
      }
      if (tid < TOT - NF * ST_THREADS) {
        const int idx = NF * ST_THREADS + tid, wj2 = idx / ST_W, wi2 = idx - ST_W * wj2;
        const double* s2 = xu + ((int64_t)m * (J0 - 2 + wj2) + (I0 - 2 + wi2));
        double* d2 = st_sm + ((wi2 & 1) ? ST_W * ST_H : 0) + (idx >> 1);
        cp_async8(d2, s2, true);
      }
      (void)wj;
    }
    {
      constexpr int TOT = ST_PW * ST_PW, DJ = ST_THREADS / ST_PW, DI = ST_THREADS % ST_PW;
      int pj = tid / ST_PW, pi = tid - ST_PW * pj;
      const double* src = p1 + ((int64_t)n1 * ((J0 >> 1) - 1 + pj) + ((I0 >> 1) - 1 + pi));
      const int64_t step = (int64_t)DJ * n1 + DI, wrap = (int64_t)n1 - ST_PW;
      for (int idx = tid; idx < TOT; idx += ST_THREADS) {
        cp_async8(st_sm + ST_OFF_P1 + idx, src, true);
        src += step; pi += DI;
        if (pi >= ST_PW) { pi -= ST_PW; src += wrap; }
      }
    }
    {
      constexpr int TOT = ST_CW * ST_CW, DJ = ST_THREADS / ST_CW, DI = ST_THREADS % ST_CW;
      int cj = tid / ST_CW, ci = tid - ST_CW * cj;
      const double* src = p0 + ((int64_t)n * ((J0 >> 1) - 1 + cj) + ((I0 >> 1) - 1 + ci));
      const int64_t step = (int64_t)DJ * n + DI, wrap = (int64_t)n - ST_CW;
      const bool on = !a.reduced;
      for (int idx = tid; idx < TOT; idx += ST_THREADS) {
        cp_async8(st_sm + ST_OFF_P0 + idx, on ? src : p0, on);
        src += step; ci += DI;
        if (ci >= ST_CW) { ci -= ST_CW; src += wrap; }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    {
      constexpr int TOT = ST_W * ST_W, NF = TOT / ST_THREADS, DJ = ST_THREADS / ST_W, DI = ST_THREADS % ST_W;
      int wj = tid / ST_W, wi = tid - ST_W * wj;
      const double* src = xu + a.nq + ((int64_t)m * (J0 - 2 + wj) + (I0 - 2 + wi));
      double* dst = st_sm + 2 * ST_W * ST_H + ((wi & 1) ? ST_W * ST_H : 0) + (tid >> 1);
      const int64_t step = (int64_t)DJ * m + DI, wrap = (int64_t)m - ST_W;
#pragma unroll 6
      for (int k = 0; k < NF; ++k) {
        cp_async8(dst, src, true);
        dst += ST_THREADS / 2; src += step; wi += DI;
        if (wi >= ST_W) { wi -= ST_W; src += wrap; }
      }
      if (tid < TOT - NF * ST_THREADS) {
        const int idx = NF * ST_THREADS + tid, wj2 = idx / ST_W, wi2 = idx - ST_W * wj2;
        const double* s2 = xu + a.nq + ((int64_t)m * (J0 - 2 + wj2) + (I0 - 2 + wi2));
        cp_async8(st_sm + 2 * ST_W * ST_H + ((wi2 & 1) ? ST_W * ST_H : 0) + (idx >> 1), s2, true);
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    {
      const double sc0 = sc;
      double dot = 0.0;
      st_vel<0, false>(a, S, I0, J0, sc0, dot);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      st_vel<1, false>(a, S, I0, J0, sc0, dot);
      if (a.dot_out) { double v[1] = {dot}; reduce_finish<1>(v, a.site, a.slot, a.dot_out); }
    }
    return;
  } else {
    for (int idx = threadIdx.x; idx < ST_W * ST_W; idx += ST_THREADS) {
      const int wi = idx % ST_W, wj = idx / ST_W;
      const int gi = I0 - 2 + wi, gj = J0 - 2 + wj;
      const bool in = gi >= 0 && gj >= 0 && gi < m && gj < m;
      const int64_t g = in ? gi + (int64_t)m * gj : 0;
      const int s = wj * ST_H + (wi >> 1);
      cp_async8(st_sm + ((wi & 1) ? ST_W * ST_H : 0) + s, xu + g, in);
      cp_async8(st_sm + ((wi & 1) ? 3 : 2) * ST_W * ST_H + s, xu + a.nq + g, in);
    }
    for (int idx = threadIdx.x; idx < ST_PW * ST_PW; idx += ST_THREADS) {
      const int pa = (I0 >> 1) - 1 + idx % ST_PW, pc = (J0 >> 1) - 1 + idx / ST_PW;
      const bool in = pa >= 0 && pc >= 0 && pa <= n && pc <= n;
      cp_async8(st_sm + ST_OFF_P1 + idx, p1 + (in ? pa + (int64_t)n1 * pc : 0), in);
    }
    for (int idx = threadIdx.x; idx < ST_CW * ST_CW; idx += ST_THREADS) {
      const int ce = (I0 >> 1) - 1 + idx % ST_CW, cf = (J0 >> 1) - 1 + idx / ST_CW;
      const bool in = !a.reduced && ce >= 0 && cf >= 0 && ce < n && cf < n;
      cp_async8(st_sm + ST_OFF_P0 + idx, p0 + (in ? ce + (int64_t)n * cf : 0), in);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (edge) st_body<true>(a, S, I0, J0, sc);
  else st_body<false>(a, S, I0, J0, sc);
}

void launch_saddle_ex(const Problem& P, bool reduced, const double* x, double* y, const double* inv_scale,
                      const RedSite* site, int slot, double* dot_out, const double* done, cudaStream_t st) {
  NvtxRange nvtx_("saddle apply");
  SaddleArgs a;
  a.L = P.Lv; a.BxT1 = P.BxT1; a.ByT1 = P.ByT1; a.BxT0 = P.BxT0; a.ByT0 = P.ByT0; a.B = P.B;
  a.nq = P.g.nq; a.nk = P.g.nk; a.n_u = P.n_u; a.n_p = P.n_p; a.reduced = reduced ? 1 : 0;
  a.x = x; a.y = y; a.inv_scale = inv_scale;
  a.site = site ? *site : RedSite{}; a.slot = slot; a.dot_out = dot_out; a.done = done;
  if (P.os_tab0 && g_oseen_mf) {   // Oseen cavity wind, storage 0: matrix-free F, B^T, B
    SaddleMfArgs b;
    b.so = P.so_os; b.w = P.sst;
    b.nq = P.g.nq; b.nk = P.g.nk; b.n_u = P.n_u; b.n_p = P.n_p; b.reduced = a.reduced;
    b.x = x; b.y = y; b.inv_scale = inv_scale; b.site = a.site; b.slot = slot; b.dot_out = dot_out; b.done = done;
    b.tab = P.os_tab0;
    k_saddle_mf<1><<<grid_for(P.N, BS, 8 * 148 * 2), BS, 0, st>>>(b); etq_count_launch();
    return;
  }
  if (P.mf_on && g_saddle_mf) {
    SaddleMfArgs b;
    b.so = P.so0; b.w = P.sst;
    b.nq = P.g.nq; b.nk = P.g.nk; b.n_u = P.n_u; b.n_p = P.n_p; b.reduced = a.reduced;
    b.x = x; b.y = y; b.inv_scale = inv_scale; b.site = a.site; b.slot = slot; b.dot_out = dot_out; b.done = done;
    const int tiles_x = (P.g.m + ST_T - 1) / ST_T;
    // a fused <K z, z> reduction keeps one partial per CTA: at most RED_MAXB of them per slot
    if (g_saddle_tile && (!dot_out || tiles_x * tiles_x <= RED_MAXB) && saddle_masks_ok(P.sst)) {
      static bool smem_set = false;
      if (!smem_set) {
        cudaFuncSetAttribute(k_saddle_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM);
        smem_set = true;
      }
      SaddleTileArgs t;
      t.so = P.so0; t.w = P.sst;
      t.m = P.g.m; t.n = P.g.n; t.nq = P.g.nq; t.nk = P.g.nk; t.n_u = P.n_u; t.reduced = a.reduced;
      t.tiles_x = tiles_x;
      t.x = x; t.y = y; t.inv_scale = inv_scale; t.site = a.site; t.slot = slot; t.dot_out = dot_out; t.done = done;
      k_saddle_tile<<<t.tiles_x * t.tiles_x, ST_THREADS, ST_SMEM, st>>>(t); etq_count_launch();
      return;
    }
    b.tab = nullptr;
    k_saddle_mf<0><<<grid_for(P.N, BS, 8 * 148 * 2), BS, 0, st>>>(b); etq_count_launch();
    return;
  }
  const int64_t warps = P.Lv.nslices + P.B.nslices;
  const int grid = grid_for(warps * 32, BS);
  k_saddle<<<grid, BS, 0, st>>>(a); etq_count_launch();
}

void launch_vel_spmv(const Sell& A, const double* x, double* y, int nq, cudaStream_t st) {
  k_vel_spmv2<<<grid_for(A.nslices * 32, BS), BS, 0, st>>>(A, nq, x, y); etq_count_launch();
}

void launch_dot(const double* a, const double* b, int64_t n, RedSite* site, int slot, double* out,
                const double* done, cudaStream_t st) {
  k_dot<<<grid_for(n, BS, RED_BLOCKS), BS, 0, st>>>(a, b, n, *site, slot, out, done); etq_count_launch();
}

// ---------------------------------------------------------------- dense inverse (setup)
etq_status dense_inverse_spd(double* A, int m, cudaStream_t st) {
  double* colp;
  ETQ_TRY(dalloc(&colp, m));
  const int64_t tot = (int64_t)m * m;
  const int g2 = grid_for(tot, BS, 4096);
  for (int p = 0; p < m; ++p) {
    k_gj_row<<<1, 1024, 0, st>>>(A, m, p, colp); etq_count_launch();
    k_gj_update<<<g2, BS, 0, st>>>(A, m, p, colp); etq_count_launch();
  }
  ETQ_CHECK(cudaGetLastError());
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(colp);
  return ETQ_OK;
}

// Gauss-Jordan with partial pivoting on the augmented [A | I] (m x 2m), for the nonsymmetric
// coarse F of the Oseen V-cycle.  Deterministic (ties -> smallest row index).
__global__ void k_piv_find(const double* Aug, int m, int p, int* piv) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = -1.0; int bidx = p;
  for (int i = p + threadIdx.x; i < m; i += blockDim.x) {
    const double v = fabs(Aug[(int64_t)i * 2 * m + p]);
    if (v > best) { best = v; bidx = i; }
  }
  bv[threadIdx.x] = best; bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = bv[threadIdx.x + s]; const int oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) { bv[threadIdx.x] = o; bi[threadIdx.x] = oi; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *piv = bi[0];
}
__global__ void k_piv_swap_scale(double* Aug, int m, int p, const int* piv, double* colp) {
  const int q = *piv;
  const int64_t w = 2LL * m;
  if (q != p)
    for (int j = threadIdx.x; j < 2 * m; j += blockDim.x) {
      const double t = Aug[(int64_t)p * w + j];
      Aug[(int64_t)p * w + j] = Aug[(int64_t)q * w + j];
      Aug[(int64_t)q * w + j] = t;
    }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) colp[i] = Aug[(int64_t)i * w + p];
  __syncthreads();
  const double pinv = 1.0 / colp[p];
  for (int j = threadIdx.x; j < 2 * m; j += blockDim.x) Aug[(int64_t)p * w + j] *= pinv;
}
__global__ void k_piv_update(double* Aug, int m, int p, const double* colp) {
  const int64_t w = 2LL * m;
  const int64_t ncol = w - p;
  const int64_t total = (int64_t)m * ncol;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / ncol);
    if (i == p) continue;
    const int64_t j = p + t % ncol;
    Aug[i * w + j] -= colp[i] * Aug[(int64_t)p * w + j];
  }
}
__global__ void k_aug_init(const double* A, double* Aug, int m) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2LL * m * m; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / (2 * m), j = t % (2 * m);
    Aug[t] = j < m ? A[i * m + j] : (j - m == i ? 1.0 : 0.0);
  }
}
__global__ void k_aug_extract(const double* Aug, double* A, int m) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)m * m; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / m, j = t % m;
    A[t] = Aug[i * 2 * m + m + j];
  }
}

void dense_gemv(const double* A, int m, int ncomp, const double* x, int64_t xstride, double* y, int64_t ystride,
                const double* done, cudaStream_t st, bool pdl) {
  launch_pdl(k_gemv, dim3(grid_for((int64_t)m * 32, BS, 4096)), dim3(BS), 0, st, pdl, A, m, ncomp, x, xstride, y, ystride,
             done);
  etq_count_launch();
}

etq_status dense_inverse_pivot(double* A, int m, cudaStream_t st) {
  double *Aug, *colp; int* piv;
  ETQ_TRY(dalloc(&Aug, 2 * (size_t)m * m));
  ETQ_TRY(dalloc(&colp, m));
  ETQ_TRY(dalloc(&piv, 1));
  k_aug_init<<<grid_for(2LL * m * m, BS, 8192), BS, 0, st>>>(A, Aug, m); etq_count_launch();
  for (int p = 0; p < m; ++p) {
    k_piv_find<<<1, 1024, 0, st>>>(Aug, m, p, piv);
    k_piv_swap_scale<<<1, 1024, 0, st>>>(Aug, m, p, piv, colp);
    k_piv_update<<<grid_for((int64_t)m * (2 * m - p), BS, 8192), BS, 0, st>>>(Aug, m, p, colp);
    etq_count_launch(3);
  }
  k_aug_extract<<<grid_for((int64_t)m * m, BS, 8192), BS, 0, st>>>(Aug, A, m); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(Aug); cudaFree(colp); cudaFree(piv);
  return ETQ_OK;
}

etq_status dense_from_sell(const Sell& A, int m, double* D, cudaStream_t st) {
  ETQ_CHECK(cudaMemsetAsync(D, 0, sizeof(double) * (size_t)m * m, st));
  k_sell_to_dense<<<(unsigned)((A.nslices * 32 + 255) / 256), 256, 0, st>>>(A, m, D); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status p1_build_mass_inverse(const Geo& g, double* W, cudaStream_t st) {
  const int64_t np = (int64_t)g.nk + g.n0;
  MassGeo mg = mass_geo(g);
  k_dense_mq_kk<<<grid_for(np * np, BS, 4096), BS, 0, st>>>(mg, W); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  ETQ_TRY(dense_inverse_spd(W, (int)np, st));
  k_dense_fix_k<<<grid_for(np * np, BS, 4096), BS, 0, st>>>(W, g.nk, np); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

// ---------------------------------------------------------------- coarse-level tail
// Levels with n <= TAIL_N are latency-bound (~55 us per level for ~10 tiny launches); one
// 1024-thread CTA runs them all with __syncthreads() between the same per-row operations as the
// level kernels (same formulas and order, so the results are identical).
namespace {
constexpr int TAIL_N = 16;
constexpr int TAIL_THREADS = 1024;

__device__ void tail_cheb_step(const TailLevel& L, const double* d_in, const double* r_in, const double* x_in,
                               double* x_out, double* r_out, double* d_out, double c1, double c2) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = TAIL_THREADS / 32;
  for (int64_t s = w; s < L.A.nslices; s += nw) {
    const int row = L.A.perm[s * SELL_C + lane];
    double q0 = 0.0, q1 = 0.0;
    sell_row2(L.A, s, lane, row, d_in, d_in + L.nq, q0, q1);
    if (row < 0) continue;
    const double di = L.dinv[row];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t idx = (int64_t)c * L.nq + row;
      const double dd = d_in[idx];
      const double ro = r_in[idx] - (c == 0 ? q0 : q1);
      x_out[idx] = (x_in ? x_in[idx] : 0.0) + dd;
      if (r_out) r_out[idx] = ro;
      if (d_out) d_out[idx] = c1 * dd + c2 * (di * ro);
    }
  }
}

__global__ void __launch_bounds__(TAIL_THREADS) k_vcycle_tail(const TailLevel* lvs, int nlev, int degree, double itheta,
                                                              const double* done) {
  if (is_done(done)) return;
  const int tid = threadIdx.x;
  // ---- down (level 0 of the tail: b and d0 were written by the restriction kernel above it)
  for (int l = 0; l < nlev - 1; ++l) {
    const TailLevel& L = lvs[l];
    double* din = L.d0; double* dout = L.d1;
    for (int k = 0; k < degree; ++k) {
      tail_cheb_step(L, din, k == 0 ? L.b : L.r, k == 0 ? nullptr : L.x, L.x, L.r, k == degree - 1 ? nullptr : dout,
                     L.c1[k], L.c2[k]);
      __syncthreads();
      double* t = din; din = dout; dout = t;
    }
    const TailLevel& Cv = lvs[l + 1];
    for (int t = tid; t < Cv.nq; t += TAIL_THREADS) {
      const int I = t % Cv.m, J = t / Cv.m;
      if (I == 0 || J == 0 || I == Cv.m - 1 || J == Cv.m - 1) {
        Cv.b[t] = 0.0; Cv.b[Cv.nq + t] = 0.0; Cv.d0[t] = 0.0; Cv.d0[Cv.nq + t] = 0.0;
        continue;
      }
      int ox[5], oy[5]; double wx[5], wy[5];
      const int nx = restrict_taps(I, ox, wx), ny = restrict_taps(J, oy, wy);
      double s0 = 0.0, s1 = 0.0;
      for (int q = 0; q < ny; ++q) {
        const int64_t rowf = (int64_t)(2 * J + oy[q]) * L.m;
        double t0 = 0.0, t1 = 0.0;
        for (int p = 0; p < nx; ++p) {
          const int64_t f = rowf + 2 * I + ox[p];
          t0 = fma(wx[p], L.r[f], t0);
          t1 = fma(wx[p], L.r[L.nq + f], t1);
        }
        s0 = fma(wy[q], t0, s0);
        s1 = fma(wy[q], t1, s1);
      }
      Cv.b[t] = s0; Cv.b[Cv.nq + t] = s1;
      const double di = Cv.dinv[t];
      Cv.d0[t] = di * s0 * itheta; Cv.d0[Cv.nq + t] = di * s1 * itheta;
    }
    __syncthreads();
  }
  // ---- coarse solve x = C^{-1} b (warp per row, both components)
  {
    const TailLevel& C = lvs[nlev - 1];
    const int lane = tid & 31, w = tid >> 5;
    for (int r = w; r < C.nq; r += TAIL_THREADS / 32)
      for (int c = 0; c < 2; ++c) {
        double s = 0.0;
        for (int j = lane; j < C.nq; j += 32) s = fma(C.coarse_inv[(int64_t)r * C.nq + j], C.b[(int64_t)c * C.nq + j], s);
        s = warp_sum(s);
        if (lane == 0) C.x[(int64_t)c * C.nq + r] = s;
      }
    __syncthreads();
  }
  // ---- up
  const double* pend_c = nullptr;
  for (int l = nlev - 2; l >= 0; --l) {
    const TailLevel& L = lvs[l];
    const TailLevel& Cv = lvs[l + 1];
    for (int64_t t = tid; t < L.nq; t += TAIL_THREADS) {
      const int k = (int)(t % L.m), ll = (int)(t / L.m);
      if (k == 0 || ll == 0 || k == L.m - 1 || ll == L.m - 1) continue;
      int ix[3], iy[3]; double wx[3], wy[3];
      const int nx = prolong_taps(k, ix, wx), ny = prolong_taps(ll, iy, wy);
      double s0 = 0.0, s1 = 0.0;
      for (int q = 0; q < ny; ++q) {
        double t0 = 0.0, t1 = 0.0;
        for (int p = 0; p < nx; ++p) {
          const int64_t c = (int64_t)iy[q] * Cv.m + ix[p];
          const double v0 = pend_c ? Cv.x[c] + pend_c[c] : Cv.x[c];
          const double v1 = pend_c ? Cv.x[Cv.nq + c] + pend_c[Cv.nq + c] : Cv.x[Cv.nq + c];
          t0 = fma(wx[p], v0, t0);
          t1 = fma(wx[p], v1, t1);
        }
        s0 = fma(wy[q], t0, s0);
        s1 = fma(wy[q], t1, s1);
      }
      L.x[t] += s0; L.x[L.nq + t] += s1;
    }
    __syncthreads();
    {   // r = b - A x ; d = D^{-1} r / theta
      const int lane = tid & 31, w = tid >> 5;
      for (int64_t s = w; s < L.A.nslices; s += TAIL_THREADS / 32) {
        const int row = L.A.perm[s * SELL_C + lane];
        double q0 = 0.0, q1 = 0.0;
        sell_row2(L.A, s, lane, row, L.x, L.x + L.nq, q0, q1);
        if (row < 0) continue;
        const double di = L.dinv[row];
        const double r0 = L.b[row] - q0, r1 = L.b[L.nq + row] - q1;
        L.r[row] = r0; L.r[L.nq + row] = r1;
        L.d0[row] = di * r0 * itheta; L.d0[L.nq + row] = di * r1 * itheta;
      }
    }
    __syncthreads();
    double* din = L.d0; double* dout = L.d1;
    for (int k = 0; k < degree - 1; ++k) {
      tail_cheb_step(L, din, L.r, L.x, L.x, k == degree - 2 ? nullptr : L.r, dout, L.c1[k], L.c2[k]);
      __syncthreads();
      double* t = din; din = dout; dout = t;
    }
    pend_c = din;
  }
  // ---- complete level 0 of the tail: x += pending correction (the caller prolongs from x)
  const TailLevel& L0 = lvs[0];
  for (int64_t i = tid; i < 2LL * L0.nq; i += TAIL_THREADS) L0.x[i] += pend_c[i];
}

// ---- the tail in shared memory (Stokes): every level's b, x, r, d0, d1 (two components) stay in
// shared memory, and each row product is the level's class stencil (the Q2 Laplacian is
// h-independent, so one StencilOp serves every level) with Dirichlet nodes read as 0 and
// identity rows on the boundary, summed in the tap order of stencil_row2 (= the stored row
// order).  Global traffic: the first level's b and d0 in, its x out, the coarse inverse.  The
// previous tail ran each of its ~40 dependent phases through L2 with index chains (~120 us).
__device__ __forceinline__ double tsm_at(const double* v, int m, int i, int j) {
  return (i <= 0 || j <= 0 || i >= m - 1 || j >= m - 1) ? 0.0 : v[i + m * j];
}
__device__ __forceinline__ void tsm_row2(const StencilOp& so, int m, int i, int j, const double* v0,
                                         const double* v1, double& a0, double& a1) {
  if (i == 0 || j == 0 || i == m - 1 || j == m - 1) {   // identity row
    const int t = i + m * j;
    a0 = fma(1.0, v0[t], 0.0); a1 = fma(1.0, v1[t], 0.0);
    return;
  }
  const int cl = (i & 1) + 2 * (j & 1);
  a0 = 0.0; a1 = 0.0;
#pragma unroll
  for (int dj = -2; dj <= 2; ++dj) {
    if ((j & 1) && (dj == 2 || dj == -2)) continue;
#pragma unroll
    for (int di = -2; di <= 2; ++di) {
      const double w = so.w[cl][(dj + 2) * 5 + (di + 2)];
      a0 = fma(w, tsm_at(v0, m, i + di, j + dj), a0);
      a1 = fma(w, tsm_at(v1, m, i + di, j + dj), a1);
    }
  }
}
__device__ __forceinline__ double tsm_dinv(const StencilOp& so, int m, int i, int j) {
  return (i == 0 || j == 0 || i == m - 1 || j == m - 1) ? 1.0 : so.dcls[(i & 1) + 2 * (j & 1)];
}
// one Chebyshev update on a level (same formulas as tail_cheb_step)
__device__ __forceinline__ void tsm_cheb_step(const StencilOp& so, int m, const double* d_in, const double* r_in,
                                              const double* x_in, double* x_out, double* r_out, double* d_out,
                                              double c1, double c2) {
  const int nq = m * m;
  for (int t = threadIdx.x; t < nq; t += TAIL_THREADS) {
    const int i = t % m, j = t / m;
    double q[2];
    tsm_row2(so, m, i, j, d_in, d_in + nq, q[0], q[1]);
    const double di = tsm_dinv(so, m, i, j);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int idx = c * nq + t;
      const double dd = d_in[idx];
      const double ro = r_in[idx] - q[c];
      x_out[idx] = (x_in ? x_in[idx] : 0.0) + dd;
      if (r_out) r_out[idx] = ro;
      if (d_out) d_out[idx] = c1 * dd + c2 * (di * ro);
    }
  }
}

__global__ void __launch_bounds__(TAIL_THREADS) k_vcycle_tail_sm(TailSmArgs a) {
  pdl_wait();
  if (is_done(a.done)) return;
  extern __shared__ double tsm[];
  const int tid = threadIdx.x;
  const int nlev = a.nlev, degree = a.degree;
  const double itheta = a.itheta;
  auto base = [&](int l) {
    int o = 0;
    for (int k = 0; k < l; ++k) o += 10 * a.m[k] * a.m[k];
    return tsm + o;
  };
  // vectors of level l: b, x, r, d0, d1 at offsets 0, 2nq, 4nq, 6nq, 8nq
  {
    const int nq = a.m[0] * a.m[0];
    double* B = base(0);
    for (int i = tid; i < 2 * nq; i += TAIL_THREADS) { B[i] = a.b0[i]; B[6 * nq + i] = a.d00[i]; }
  }
  __syncthreads();
  // ---- down
  for (int l = 0; l < nlev - 1; ++l) {
    const int m = a.m[l], nq = m * m;
    double* B = base(l);
    double *b = B, *x = B + 2 * nq, *r = B + 4 * nq;
    double* din = B + 6 * nq; double* dout = B + 8 * nq;
    for (int k = 0; k < degree; ++k) {
      tsm_cheb_step(a.so, m, din, k == 0 ? b : r, k == 0 ? nullptr : x, x, r, k == degree - 1 ? nullptr : dout,
                    a.c1[l][k], a.c2[l][k]);
      __syncthreads();
      double* t = din; din = dout; dout = t;
    }
    const int mc = a.m[l + 1], nqc = mc * mc;
    double* Bc = base(l + 1);
    for (int t = tid; t < nqc; t += TAIL_THREADS) {
      const int I = t % mc, J = t / mc;
      if (I == 0 || J == 0 || I == mc - 1 || J == mc - 1) {
        Bc[t] = 0.0; Bc[nqc + t] = 0.0; Bc[6 * nqc + t] = 0.0; Bc[6 * nqc + nqc + t] = 0.0;
        continue;
      }
      int ox[5], oy[5]; double wx[5], wy[5];
      const int nx = restrict_taps(I, ox, wx), ny = restrict_taps(J, oy, wy);
      double s0 = 0.0, s1 = 0.0;
      for (int q = 0; q < ny; ++q) {
        const int rowf = (2 * J + oy[q]) * m;
        double t0 = 0.0, t1 = 0.0;
        for (int p = 0; p < nx; ++p) {
          const int f = rowf + 2 * I + ox[p];
          t0 = fma(wx[p], r[f], t0);
          t1 = fma(wx[p], r[nq + f], t1);
        }
        s0 = fma(wy[q], t0, s0);
        s1 = fma(wy[q], t1, s1);
      }
      Bc[t] = s0; Bc[nqc + t] = s1;
      const double di = tsm_dinv(a.so, mc, I, J);
      Bc[6 * nqc + t] = di * s0 * itheta; Bc[6 * nqc + nqc + t] = di * s1 * itheta;
    }
    __syncthreads();
  }
  // ---- coarse solve x = C^{-1} b (warp per row, both components)
  {
    const int mc = a.m[nlev - 1], nqc = mc * mc;
    double* B = base(nlev - 1);
    const int lane = tid & 31, w = tid >> 5;
    for (int rr = w; rr < nqc; rr += TAIL_THREADS / 32)
      for (int c = 0; c < 2; ++c) {
        double s = 0.0;
        for (int j = lane; j < nqc; j += 32) s = fma(__ldg(a.coarse_inv + (int64_t)rr * nqc + j), B[c * nqc + j], s);
        s = warp_sum(s);
        if (lane == 0) B[2 * nqc + c * nqc + rr] = s;
      }
    __syncthreads();
  }
  // ---- up
  const double* pend_c = nullptr;
  for (int l = nlev - 2; l >= 0; --l) {
    const int m = a.m[l], nq = m * m, mc = a.m[l + 1], nqc = mc * mc;
    double* B = base(l);
    double *b = B, *x = B + 2 * nq, *r = B + 4 * nq;
    const double* xc = base(l + 1) + 2 * nqc;
    for (int t = tid; t < nq; t += TAIL_THREADS) {
      const int k = t % m, ll = t / m;
      if (k == 0 || ll == 0 || k == m - 1 || ll == m - 1) continue;
      int ix[3], iy[3]; double wx[3], wy[3];
      const int nx = prolong_taps(k, ix, wx), ny = prolong_taps(ll, iy, wy);
      double s0 = 0.0, s1 = 0.0;
      for (int q = 0; q < ny; ++q) {
        double t0 = 0.0, t1 = 0.0;
        for (int p = 0; p < nx; ++p) {
          const int c = iy[q] * mc + ix[p];
          const double v0 = pend_c ? xc[c] + pend_c[c] : xc[c];
          const double v1 = pend_c ? xc[nqc + c] + pend_c[nqc + c] : xc[nqc + c];
          t0 = fma(wx[p], v0, t0);
          t1 = fma(wx[p], v1, t1);
        }
        s0 = fma(wy[q], t0, s0);
        s1 = fma(wy[q], t1, s1);
      }
      x[t] += s0; x[nq + t] += s1;
    }
    __syncthreads();
    for (int t = tid; t < nq; t += TAIL_THREADS) {   // r = b - A x ; d = D^{-1} r / theta
      const int i = t % m, j = t / m;
      double q0, q1;
      tsm_row2(a.so, m, i, j, x, x + nq, q0, q1);
      const double di = tsm_dinv(a.so, m, i, j);
      const double r0 = b[t] - q0, r1 = b[nq + t] - q1;
      r[t] = r0; r[nq + t] = r1;
      B[6 * nq + t] = di * r0 * itheta; B[6 * nq + nq + t] = di * r1 * itheta;
    }
    __syncthreads();
    double* din = B + 6 * nq; double* dout = B + 8 * nq;
    for (int k = 0; k < degree - 1; ++k) {
      tsm_cheb_step(a.so, m, din, r, x, x, k == degree - 2 ? nullptr : r, dout, a.c1[l][k], a.c2[l][k]);
      __syncthreads();
      double* t = din; din = dout; dout = t;
    }
    pend_c = din;
  }
  // ---- complete level 0 of the tail: x += pending correction, to global (the caller prolongs it)
  pdl_trigger();
  {
    const int nq = a.m[0] * a.m[0];
    const double* x = base(0) + 2 * nq;
    for (int i = tid; i < 2 * nq; i += TAIL_THREADS) a.x0[i] = x[i] + pend_c[i];
  }
}
}  // namespace

// ---------------------------------------------------------------- hierarchy
static void cheb_coeffs(double lo, double hi, double bim, int degree, std::vector<double>& c1, std::vector<double>& c2);

static etq_status alloc_level_vectors(Level& L, int nc, bool need_b) {
  const size_t nv = (size_t)nc * L.nrows;
  if (need_b) ETQ_TRY(dalloc(&L.b, nv));
  ETQ_TRY(dalloc(&L.x, nv));
  ETQ_TRY(dalloc(&L.r, nv));
  ETQ_TRY(dalloc(&L.d0, nv));
  ETQ_TRY(dalloc(&L.d1, nv));
  return ETQ_OK;
}

static etq_status level_sizes(int n, int coarse_n, std::vector<int>& ns) {
  if (coarse_n < 1) return ETQ_EINVAL;
  int m = n;
  while (true) {
    ns.push_back(m);
    if (m <= coarse_n) break;
    if (m % 2) return ETQ_EINVAL;
    m /= 2;
  }
  return ETQ_OK;
}

// Velocity-block hierarchy (reading R9/R9'): rediscretised scalar operator L or F_s per level,
// Dirichlet identity rows, smoother ellipse per level (Oseen: imaginary semi-axis = Gershgorin
// radius of D^{-1}N), dense coarse inverse (Gauss-Jordan; pivoted for the nonsymmetric F).
// Constant-bank stencil table of k_cheb_tile2: uploaded once (setup time, never during capture);
// a level may use k_cheb_tile2 only if its class stencils and D^-1 equal the table bitwise.
// the grouped weights of ct_group_sum and the symmetry they rely on: every tap equals its group's
// representative (the + offsets) to within a few ulp (the assembled mirrored taps may differ in the
// last bit: different element-contribution order); the taps the Stokes enumeration drops are zero
static bool ct2_groups(const StencilOp& so, double g0[6], double g1[5], double g3[3]) {
  auto w = [&](int c, int di, int dj) { return so.w[c][(dj + 2) * 5 + di + 2]; };
  g0[0] = w(0, 0, 0); g0[1] = w(0, 1, 0); g0[2] = w(0, 1, 1); g0[3] = w(0, 2, 0); g0[4] = w(0, 2, 1); g0[5] = w(0, 2, 2);
  g1[0] = w(1, 0, 0); g1[1] = w(1, 1, 0); g1[2] = w(1, 0, 1); g1[3] = w(1, 1, 1); g1[4] = w(1, 1, 2);
  g3[0] = w(3, 0, 0); g3[1] = w(3, 1, 0); g3[2] = w(3, 1, 1);
  for (int dj = -2; dj <= 2; ++dj)
    for (int di = -2; di <= 2; ++di) {
      const int u = std::abs(di), v = std::abs(dj);
      const int lo = std::min(u, v), hi = std::max(u, v);
      const double e0 = (hi == 0) ? g0[0] : (hi == 1) ? (lo == 0 ? g0[1] : g0[2]) : (lo == 0 ? g0[3] : lo == 1 ? g0[4] : g0[5]);
      auto near = [](double x, double y) { return std::fabs(x - y) <= 8e-16 * std::fabs(y); };
      if (!near(w(0, di, dj), e0)) return false;
      if (u <= 1) {   // class 1 (i odd: |di| <= 1), class 2 = its transpose
        const double e1 = (u == 0 && v == 0) ? g1[0] : (u == 1 && v == 0) ? g1[1] : (u == 0 && v == 1) ? g1[2]
                        : (u == 1 && v == 1) ? g1[3] : (u == 1 && v == 2) ? g1[4] : 0.0;
        if (!near(w(1, di, dj), e1) || !near(w(2, dj, di), e1)) return false;
      }
      if (u <= 1 && v <= 1) {
        const double e3 = (u + v == 0) ? g3[0] : (u + v == 1) ? g3[1] : g3[2];
        if (!near(w(3, di, dj), e3)) return false;
      }
    }
  return true;
}

static bool ct2_register(const StencilOp& so) {
  static bool have = false;
  static double w[4][25], d[4];
  if (!have) {
    double g0[6], g1[5], g3[3];
    if (!ct2_groups(so, g0, g1, g3)) return false;
    if (cudaMemcpyToSymbol(c_ct_w, so.w, sizeof(w)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_ct_dcls, so.dcls, sizeof(d)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_ct_g0, g0, sizeof(g0)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_ct_g1, g1, sizeof(g1)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_ct_g3, g3, sizeof(g3)) != cudaSuccess)
      return false;
    std::memcpy(w, so.w, sizeof(w));
    std::memcpy(d, so.dcls, sizeof(d));
    have = true;
    return true;
  }
  return std::memcmp(w, so.w, sizeof(w)) == 0 && std::memcmp(d, so.dcls, sizeof(d)) == 0;
}

etq_status build_hierarchy(Problem& P, Hierarchy& H, int coarse_n, double lo, double hi, int degree) {
  std::vector<int> ns;
  ETQ_TRY(level_sizes(P.g.n, coarse_n, ns));
  H.kind = 0; H.ncomp = 2;
  H.lv.resize(ns.size());
  for (size_t l = 0; l < ns.size(); ++l) {
    Level& L = H.lv[l];
    L.g = make_geo(ns[l]);
    L.nrows = L.g.nq;
    if (l == 0) {
      L.A = P.Lv;   // shallow: owned by the problem
    } else {
      int* perm; int64_t nsl;
      ETQ_TRY(build_node_perm(L.g, &perm, &nsl, P.stream));
      ETQ_TRY(assemble_velocity_op(L.g, P.oseen, P.nu, P.wind, perm, nsl, &L.A, P.stream));
      if (P.storage < 2) ETQ_TRY(mark_implicit(L.g, P.oseen, P.nu, P.wind, L.A, P.stream, P.storage == 0));
      L.A.own_perm = true;
    }
    ETQ_TRY(dalloc(&L.dinv, L.g.nq));
    ETQ_TRY(velocity_dinv_dev(L.g, P.oseen, P.nu, P.wind, L.dinv, P.stream));
    L.bim = 0.0;
    if (P.oseen && l + 1 < ns.size()) ETQ_TRY(oseen_gershgorin(L.g, P.nu, P.wind, &L.bim, P.stream));
    ETQ_TRY(alloc_level_vectors(L, 2, l > 0));
  }
  Level& C = H.lv.back();
  ETQ_TRY(dalloc(&C.coarse_inv, (size_t)C.g.nq * C.g.nq));
  ETQ_TRY(dense_from_sell(C.A, C.g.nq, C.coarse_inv, P.stream));
  if (P.oseen) ETQ_TRY(dense_inverse_pivot(C.coarse_inv, C.g.nq, P.stream));
  else ETQ_TRY(dense_inverse_spd(C.coarse_inv, C.g.nq, P.stream));
  H.lo = lo; H.hi = hi; H.degree = degree; H.built = true;
  // interior stencil path for translation-invariant levels with n > TAIL_N
  for (size_t l = 0; l < H.lv.size(); ++l) {
    Level& lv = H.lv[l];
    if (!P.oseen && P.storage == 0 && lv.g.n > TAIL_N && lv.A.stval && l + 1 < H.lv.size()) {
      ETQ_TRY(build_stencil_level(lv.g, lv.A, &lv.so, &lv.Afr, P.stream));
      // D^-1 per stencil class, read at interior reference nodes (the tiled smoother's diagonal)
      for (int c = 0; c < 4; ++c) {
        const int64_t node = (int64_t)(lv.so.lo + (c & 1)) + (int64_t)lv.g.m * (lv.so.lo + (c >> 1));
        ETQ_CHECK(cudaMemcpyAsync(&lv.so.dcls[c], lv.dinv + node, sizeof(double), cudaMemcpyDeviceToHost, P.stream));
      }
      ETQ_CHECK(cudaStreamSynchronize(P.stream));
      lv.st_on = true;
      lv.ct2 = ct2_register(lv.so);
      if (std::getenv("ETQ_DEBUG")) std::fprintf(stderr, "[etq] level n=%d k_cheb_tile2 %s\n", lv.g.n, lv.ct2 ? "on" : "off");
    } else if (P.oseen && P.wind == 1 && P.storage == 0 && g_oseen_mf && lv.g.n >= 16 && l + 1 < H.lv.size()) {
      // cavity-wind F levels: matrix-free interior rows (k_cheb_step_os), stored frame rows
      ETQ_TRY(build_oseen_stencil_level(lv.g, P.nu, &lv.so, &lv.Afr, &lv.os_tab, P.stream));
      lv.st_on = true;
    }
  }
  // coarse-level tail: first level l >= 1 with n <= TAIL_N (degree <= 4)
  H.tail_start = -1;
  if (degree <= 4)
    for (size_t l = 1; l < H.lv.size(); ++l)
      if (H.lv[l].g.n <= TAIL_N && H.lv.size() - l >= 2) { H.tail_start = (int)l; break; }
  if (H.tail_start > 0) ETQ_TRY(refresh_tail(H));
  // shared-memory matrix-free tail: Stokes levels (translation invariant, the finest level's class
  // stencils and D^-1 hold on every level), degree <= 4, vectors within the shared-memory budget
  H.tail_sm = false;
  if (H.tail_start > 0 && !P.oseen && P.storage == 0 && H.lv[0].st_on &&
      (int)H.lv.size() - H.tail_start <= TAIL_SM_MAXLEV) {
    TailSmArgs& t = H.tsm;
    t = TailSmArgs{};
    t.so = H.lv[0].so; t.nlev = (int)H.lv.size() - H.tail_start; t.degree = degree;
    const double theta = 0.5 * (hi + lo);
    t.itheta = 1.0 / theta;
    std::vector<double> c1, c2;
    int words = 0;
    for (int k = 0; k < t.nlev; ++k) {
      const Level& lv = H.lv[H.tail_start + k];
      t.m[k] = lv.g.m;
      words += 10 * lv.g.m * lv.g.m;
      cheb_coeffs(lo, hi, lv.bim, degree, c1, c2);
      for (int q = 0; q < degree; ++q) { t.c1[k][q] = c1[q]; t.c2[k][q] = c2[q]; }
    }
    const Level& l0 = H.lv[H.tail_start];
    t.b0 = l0.b; t.d00 = l0.d0; t.x0 = l0.x; t.coarse_inv = H.lv.back().coarse_inv;
    t.smem_bytes = words * (int)sizeof(double);
    if (t.smem_bytes <= 200 * 1024) {
      ETQ_CHECK(cudaFuncSetAttribute(k_vcycle_tail_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem_bytes));
      H.tail_sm = true;
    }
  }
  ETQ_CHECK(cudaStreamSynchronize(P.stream));
  return ETQ_OK;
}

// (Re)write the fused tail's level table: operators, vectors and Chebyshev coefficients (the
// latter change when a Picard wind changes the smoother ellipses, picard.cu)
etq_status refresh_tail(Hierarchy& H) {
  if (H.tail_start <= 0) return ETQ_OK;
  std::vector<TailLevel> tl;
  std::vector<double> c1, c2;
  for (size_t l = H.tail_start; l < H.lv.size(); ++l) {
    const Level& lv = H.lv[l];
    TailLevel t{};
    t.A = lv.A; t.dinv = lv.dinv; t.b = lv.b; t.x = lv.x; t.r = lv.r; t.d0 = lv.d0; t.d1 = lv.d1;
    t.nq = lv.nrows; t.m = lv.g.m; t.coarse_inv = lv.coarse_inv;
    cheb_coeffs(H.lo, H.hi, lv.bim, H.degree, c1, c2);
    for (int k = 0; k < H.degree; ++k) { t.c1[k] = c1[k]; t.c2[k] = c2[k]; }
    tl.push_back(t);
  }
  if (!H.tail) ETQ_TRY(dalloc(&H.tail, tl.size()));
  ETQ_CHECK(cudaMemcpy(H.tail, tl.data(), sizeof(TailLevel) * tl.size(), cudaMemcpyHostToDevice));
  return ETQ_OK;
}

// W = (A + 1 1^T)^{-1} - 1 1^T / m^2 = A^+ for a symmetric A with null space span{1}
__global__ void k_add_ones(double* A, int m, double v) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)m * m; t += (int64_t)gridDim.x * blockDim.x)
    A[t] += v;
}

// Pressure hierarchy for Ap = B1 Mdiag^{-1} B1^T (reading R13; op 0) or the mass Schur complement
// S_k (reading R21; op 1, level l scaled by 4^-l so that it approximates the Galerkin product):
// Q1 levels n ... coarse_n, nested bilinear transfers, real Chebyshev smoother, coarse pseudo-inverse.
etq_status build_ap_hierarchy(Problem& P, Hierarchy& H, int coarse_n, double lo, double hi, int degree, int op) {
  std::vector<int> ns;
  ETQ_TRY(level_sizes(P.g.n, coarse_n, ns));
  H.kind = 1; H.ncomp = 1;
  H.lv.resize(ns.size());
  for (size_t l = 0; l < ns.size(); ++l) {
    Level& L = H.lv[l];
    L.g = make_geo(ns[l]);
    L.nrows = op == 2 ? L.g.nk + L.g.n0 : L.g.nk;
    if (op == 0) ETQ_TRY(assemble_ap(L.g, &L.A, P.stream));
    else if (op == 1) ETQ_TRY(assemble_sk(L.g, std::ldexp(1.0, -2 * (int)l), &L.A, P.stream));   // S_k / 4^l (R21)
    else ETQ_TRY(assemble_lp(L.g, &L.A, P.stream));                                                // two-field Lp
    if (op == 2) { ETQ_TRY(dalloc(&L.dinv, L.nrows)); ETQ_TRY(sell_diag_inv(L.A, L.dinv, P.stream));
                   L.bim = 0.0; ETQ_TRY(alloc_level_vectors(L, 1, true)); continue; }
    ETQ_TRY(dalloc(&L.dinv, L.g.nk));
    ETQ_TRY(sell_diag_inv(L.A, L.dinv, P.stream));
    L.bim = 0.0;
    ETQ_TRY(alloc_level_vectors(L, 1, true));
  }
  Level& C = H.lv.back();
  const int m = C.nrows;
  ETQ_TRY(dalloc(&C.coarse_inv, (size_t)m * m));
  ETQ_TRY(dense_from_sell(C.A, m, C.coarse_inv, P.stream));
  if (op == 2) {   // null space: the Q1 and the P0 constants; (A + sum c_i e_i e_i^T)^-1 - sum e_i e_i^T / (c_i |e_i|^4)
    const int nk = C.g.nk, n0 = C.g.n0;
    k_add_block<<<grid_for((int64_t)nk * nk, BS, 4096), BS, 0, P.stream>>>(C.coarse_inv, m, 0, nk, 1.0 / nk); etq_count_launch();
    k_add_block<<<grid_for((int64_t)n0 * n0, BS, 4096), BS, 0, P.stream>>>(C.coarse_inv, m, nk, m, 1.0 / n0); etq_count_launch();
    ETQ_TRY(dense_inverse_spd(C.coarse_inv, m, P.stream));
    k_add_block<<<grid_for((int64_t)nk * nk, BS, 4096), BS, 0, P.stream>>>(C.coarse_inv, m, 0, nk, -1.0 / nk); etq_count_launch();
    k_add_block<<<grid_for((int64_t)n0 * n0, BS, 4096), BS, 0, P.stream>>>(C.coarse_inv, m, nk, m, -1.0 / n0); etq_count_launch();
    H.lo = lo; H.hi = hi; H.degree = degree; H.built = true; H.op = op;
    ETQ_CHECK(cudaStreamSynchronize(P.stream));
    return ETQ_OK;
  }
  // c 1 1^T with c m ~ the operator's diagonal keeps A + c 1 1^T as well conditioned as A on 1^perp
  // (Ap: diagonal O(1); S_k / 4^l: diagonal (28/144) h_0^2 on every level)
  const double cs = op == 0 ? 1.0 : (28.0 / 144.0) * P.g.h * P.g.h / m;
  k_add_ones<<<grid_for((int64_t)m * m, BS, 4096), BS, 0, P.stream>>>(C.coarse_inv, m, cs); etq_count_launch();
  ETQ_TRY(dense_inverse_spd(C.coarse_inv, m, P.stream));
  k_add_ones<<<grid_for((int64_t)m * m, BS, 4096), BS, 0, P.stream>>>(C.coarse_inv, m, -1.0 / (cs * m * m)); etq_count_launch();
  H.lo = lo; H.hi = hi; H.degree = degree; H.built = true;
  H.op = op; H.sk_w = P.g.h * P.g.h / 144.0;
  ETQ_CHECK(cudaStreamSynchronize(P.stream));
  return ETQ_OK;
}

void free_hierarchy(Hierarchy& H) {
  for (size_t l = 0; l < H.lv.size(); ++l) {
    Level& L = H.lv[l];
    if (l == 0 && H.kind == 0) L.A.fval = nullptr;   // owned by the problem's Lv
    cudaFree(L.f_dinv); cudaFree(L.f_b); cudaFree(L.f_x); cudaFree(L.f_r); cudaFree(L.f_d0); cudaFree(L.f_d1);
    cudaFree(L.f_coarse);
    if (H.kind == 1 || l > 0) sell_free(L.A);
    sell_free(L.Afr);
    cudaFree(L.os_tab);
    cudaFree(L.dinv); cudaFree(L.b); cudaFree(L.x); cudaFree(L.r); cudaFree(L.d0); cudaFree(L.d1);
    cudaFree(L.coarse_inv);
    cudaFree(L.wind); cudaFree(L.lapval);
  }
  cudaFree(H.tail);
  H = Hierarchy{};
}

// Chebyshev coefficients c1_k = rho_{k+1} rho_k, c2_k = 2 rho_{k+1} / delta on the ellipse with
// centre theta, real semi-axis a and imaginary semi-axis bim (real interval when bim = 0).
static void cheb_coeffs(double lo, double hi, double bim, int degree, std::vector<double>& c1, std::vector<double>& c2) {
  c1.resize(degree); c2.resize(degree);
  const double theta = 0.5 * (hi + lo), a = 0.5 * (hi - lo);
  if (bim == 0.0) {
    const double delta = a, sigma = theta / delta;
    double rho = 1.0 / sigma;
    for (int k = 0; k < degree; ++k) {
      const double rn = 1.0 / (2.0 * sigma - rho);
      c1[k] = rn * rho; c2[k] = 2.0 * rn / delta;
      rho = rn;
    }
    return;
  }
  const std::complex<double> delta = std::sqrt(std::complex<double>(a * a - bim * bim, 0.0));
  const std::complex<double> sigma = theta / delta;
  std::complex<double> rho = 1.0 / sigma;
  for (int k = 0; k < degree; ++k) {
    const std::complex<double> rn = 1.0 / (2.0 * sigma - rho);
    c1[k] = (rn * rho).real(); c2[k] = (2.0 * rn / delta).real();
    rho = rn;
  }
}

static void launch_cheb_st(const Level& lv, const ChebArgs& c, bool post, double theta, cudaStream_t st,
                           bool pdl = false) {
  ChebStArgs a;
  a.so = lv.so; a.F = lv.Afr; a.dinv = c.dinv; a.nq = c.nq;
  a.d_in = c.d_in; a.r_in = c.r_in; a.x_in = c.x_in; a.x_out = c.x_out; a.r_out = c.r_out; a.d_out = c.d_out;
  a.c1 = c.c1; a.c2 = c.c2; a.post = post ? 1 : 0; a.itheta = 1.0 / theta; a.done = c.done;
  const int64_t warps = lv.so.nseg + lv.Afr.nslices;
  if (lv.os_tab) launch_pdl(k_cheb_step_os, dim3(grid_for(warps * 32, BS, 4096)), dim3(BS), 0, st, pdl, a,
                            (const double*)lv.os_tab);
  else launch_pdl(k_cheb_step_st, dim3(grid_for(warps * 32, BS, 4096)), dim3(BS), 0, st, pdl, a);
}

// Temporally blocked smoothing pass on an interior-stencil level (degree 3, real interval).
static void launch_cheb_tile(const Level& lv, bool post, const double* b, const double* x_in, double* x_out,
                             double* r_out, double* d_out, const std::vector<double>& c1,
                             const std::vector<double>& c2, double theta, const double* done, cudaStream_t st,
                             double* z_out = nullptr, const double* dot_with = nullptr,
                             const RedSite* site = nullptr, int slot = 0, double* dot_out = nullptr,
                             bool pdl = false) {
  static bool smem_set = false;
  if (!smem_set) {
    cudaFuncSetAttribute(k_cheb_tile<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, CT_SMEM);
    cudaFuncSetAttribute(k_cheb_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, CT_SMEM);
    cudaFuncSetAttribute(k_cheb_tile<0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_cheb_tile<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    smem_set = true;
  }
  ChebTileArgs a;
  a.so = lv.so; a.nq = lv.g.nq;
  a.tiles_x = (lv.g.m + CT_T - 1) / CT_T;
  a.b = b; a.x_in = x_in; a.x_out = x_out; a.r_out = r_out; a.d_out = d_out;
  a.itheta = 1.0 / theta;
  for (int k = 0; k < 3; ++k) { a.c1[k] = c1[k]; a.c2[k] = c2[k]; }
  a.done = done;
  a.z_out = z_out; a.dot_with = dot_with; a.site = site ? *site : RedSite{}; a.slot = slot; a.dot_out = dot_out;
  a.prefetch = g_ct_prefetch ? 1 : 0;
  dim3 grid(a.tiles_x * a.tiles_x, 2);
  if (lv.ct2 && g_cheb_tile3) {
    static bool smem3 = false;
    if (!smem3) {
      cudaFuncSetAttribute(k_cheb_tile3<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, CT_SMEM);
      cudaFuncSetAttribute(k_cheb_tile3<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, CT_SMEM);
      smem3 = true;
    }
    if (post) launch_pdl(k_cheb_tile3<1>, grid, dim3(CT_THREADS), CT_SMEM, st, pdl, a);
    else launch_pdl(k_cheb_tile3<0>, grid, dim3(CT_THREADS), CT_SMEM, st, pdl, a);
    return;
  }
  if (lv.ct2 && g_cheb_tile2) {
    static bool smem2 = false;
    if (!smem2) {
      cudaFuncSetAttribute(k_cheb_tile2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, CT_SMEM);
      cudaFuncSetAttribute(k_cheb_tile2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, CT_SMEM);
      smem2 = true;
    }
    if (post) launch_pdl(k_cheb_tile2<1>, grid, dim3(CT_THREADS), CT_SMEM, st, pdl, a);
    else launch_pdl(k_cheb_tile2<0>, grid, dim3(CT_THREADS), CT_SMEM, st, pdl, a);
    return;
  }
  if (post) launch_pdl(k_cheb_tile<1>, grid, dim3(CT_THREADS), CT_SMEM, st, pdl, a);
  else launch_pdl(k_cheb_tile<0>, grid, dim3(CT_THREADS), CT_SMEM, st, pdl, a);
}

static bool tile_ok(const Hierarchy& H, const Level& lv) {
  return lv.st_on && H.degree == 3 && lv.bim == 0.0 && H.ncomp == 2 && g_cheb_tile_enabled &&
         lv.g.n >= g_cheb_tile_min_n;
}

// One V-cycle (readings R9/R9'/R13) on H.ncomp components: z = V(r); optional partial
// <z, dot_with> into (site, slot) -> dot_out.
static void launch_cheb_sk(const Hierarchy& H, const Level& lv, const ChebArgs& c, int post, double theta,
                           cudaStream_t st, bool pdl = false) {
  SkChebArgs a;
  a.n = lv.g.n; a.w = H.sk_w;
  a.v = post ? c.x_in : c.d_in;
  a.d_in = c.d_in; a.r_in = c.r_in; a.x_in = c.x_in;
  a.x_out = c.x_out; a.r_out = c.r_out; a.d_out = c.d_out;
  a.c1 = c.c1; a.c2 = c.c2; a.itheta = 1.0 / theta; a.post = post; a.done = c.done;
  launch_pdl(k_cheb_sk, dim3(grid_for((int64_t)lv.g.nk, BS, 8 * 148)), dim3(BS), 0, st, pdl, a);
}

etq_status vcycle_apply_ex(const Problem& P, const Hierarchy& H, const double* r_u, double* z_u,
                           const RedSite* site, int slot, double* dot_out, const double* dot_with,
                           const double* done, cudaStream_t st, bool pdl) {
  NvtxRange nvtx_("V-cycle");
  const int L = (int)H.lv.size();
  const int nc = H.ncomp;
  const double theta = 0.5 * (H.hi + H.lo);
  RedSite dummy{};
  if (L == 1) {   // coarse solve only
    const Level& C = H.lv[0];
    dense_gemv(C.coarse_inv, C.nrows, nc, r_u, C.nrows, z_u, C.nrows, done, st);
    if (dot_out && site) {
      k_final_add<<<grid_for((int64_t)nc * C.nrows, BS, RED_BLOCKS), BS, 0, st>>>(
          z_u, nullptr, z_u, (int64_t)nc * C.nrows, dot_with, *site, slot, dot_out, done); etq_count_launch();
    }
    return ETQ_OK;
  }
  std::vector<const double*> bvec(L);
  std::vector<const double*> pend(L, nullptr);
  // programmatic dependent launches between the cycle's kernels: shorter cycle latency, but the
  // early-launched CTAs compete with a concurrent branch for SM slots; the caller decides (P3: on,
  // P2: off - measured: P3 solve 94 -> 88 ms, P2 solve 557 -> 564 ms)
  const bool vpdl = pdl && g_vc_pdl;
  std::vector<double> c1, c2;
  const bool use_tail = H.kind == 0 && nc == 2 && H.tail_start > 0 && H.tail != nullptr;
  const int Ld = use_tail ? H.tail_start + 1 : L;   // levels handled by the per-level kernels (+1)
  // ---- down
  for (int l = 0; l < Ld - 1; ++l) {
    const Level& lv = H.lv[l];
    const int nq = lv.nrows;
    cheb_coeffs(H.lo, H.hi, lv.bim, H.degree, c1, c2);
    const double* b = (l == 0) ? r_u : lv.b;
    bvec[l] = b;
    const bool tiled = tile_ok(H, lv);
    if (tiled) {
      launch_cheb_tile(lv, false, b, nullptr, lv.x, lv.r, nullptr, c1, c2, theta, done, st, nullptr, nullptr, nullptr,
                       0, nullptr, vpdl && l > 0);
      etq_count_launch();
    }
    if (l == 0 && !tiled) {
      k_cheb_init<<<grid_for((int64_t)nc * nq, BS, 4096), BS, 0, st>>>(lv.dinv, nq, nc, b, lv.d0, 1.0 / theta, done); etq_count_launch();
    }
    const int gs = grid_for(lv.A.nslices * 32, BS, 4096);
    double* din = lv.d0; double* dout = lv.d1;
    for (int k = 0; k < (tiled ? 0 : H.degree); ++k) {
      ChebArgs a;
      a.A = lv.A; a.dinv = lv.dinv; a.nq = nq;
      a.d_in = din; a.r_in = (k == 0) ? b : lv.r; a.x_in = (k == 0) ? nullptr : lv.x;
      a.x_out = lv.x; a.r_out = lv.r; a.d_out = (k == H.degree - 1) ? nullptr : dout;
      a.c1 = c1[k]; a.c2 = c2[k]; a.done = done;
      if (lv.st_on) launch_cheb_st(lv, a, false, theta, st, vpdl);
      else if (H.op == 1) launch_cheb_sk(H, lv, a, 0, theta, st, vpdl);
      else if (nc == 2) k_cheb_step<2><<<gs, BS, 0, st>>>(a);
      else k_cheb_step<1><<<gs, BS, 0, st>>>(a);
      etq_count_launch();
      std::swap(din, dout);
    }
    const Level& cv = H.lv[l + 1];
    if (H.kind == 0) {
      launch_pdl(k_restrict, dim3(grid_for(cv.g.nq, BS, 4096)), dim3(BS), 0, st, vpdl, lv.g.m, cv.g.m, nq, cv.g.nq,
                 (const double*)lv.r, cv.b, cv.d0, (const double*)cv.dinv, 1.0 / theta, done);
    } else {
      launch_pdl(k_restrict_q1, dim3(grid_for(cv.g.nk, BS, 4096)), dim3(BS), 0, st, vpdl && H.op == 1, lv.g.n + 1,
                 cv.g.n + 1, (const double*)lv.r, cv.b, cv.d0, (const double*)cv.dinv, 1.0 / theta, done);
      if (H.op == 2) {
        etq_count_launch();
        const int nkf = lv.g.nk, nkc = cv.g.nk;
        k_restrict_p0<<<grid_for(cv.g.n0, BS, 4096), BS, 0, st>>>(lv.g.n, cv.g.n, lv.r + nkf, cv.b + nkc, cv.d0 + nkc,
                                                                  cv.dinv + nkc, 1.0 / theta, done);
      }
    }
    etq_count_launch();
  }
  // ---- coarse (or the fused coarse-level tail, which leaves a complete x on its first level)
  if (use_tail) {
    if (H.tail_sm && g_tail_sm) {
      TailSmArgs ta = H.tsm;
      ta.done = done;
      launch_pdl(k_vcycle_tail_sm, dim3(1), dim3(TAIL_THREADS), ta.smem_bytes, st, vpdl, ta);
    } else {
      k_vcycle_tail<<<1, TAIL_THREADS, 0, st>>>(H.tail, L - H.tail_start, H.degree, 1.0 / theta, done);
    }
    etq_count_launch();
    pend[Ld - 1] = nullptr;
  } else {
    const Level& C = H.lv[L - 1];
    dense_gemv(C.coarse_inv, C.nrows, nc, C.b, C.nrows, C.x, C.nrows, done, st, vpdl);
    pend[L - 1] = nullptr;
  }
  // ---- up
  std::vector<const double*> xres(L, nullptr);   // where each level's smoothed x ends up
  for (int l = 0; l < L; ++l) xres[l] = H.lv[l].x;
  for (int l = Ld - 2; l >= 0; --l) {
    const Level& lv = H.lv[l];
    const Level& cv = H.lv[l + 1];
    const int nq = lv.nrows;
    cheb_coeffs(H.lo, H.hi, lv.bim, H.degree, c1, c2);
    if (H.kind == 0) {
      if (g_prolong_tile) {
        const int tx = (lv.g.m + PT_X - 1) / PT_X, ty = (lv.g.m + PT_Y - 1) / PT_Y;
        launch_pdl(k_prolong_tile, dim3(tx * ty), dim3(PT_THREADS), 0, st, vpdl, lv.g.m, cv.g.m, nq, cv.g.nq,
                   xres[l + 1], pend[l + 1], lv.x, done);
      } else {
        launch_pdl(k_prolong, dim3(grid_for(nq, BS, 4096)), dim3(BS), 0, st, vpdl, lv.g.m, cv.g.m, nq, cv.g.nq,
                   xres[l + 1], pend[l + 1], lv.x, done);
      }
    } else {
      launch_pdl(k_prolong_q1, dim3(grid_for(lv.g.nk, BS, 4096)), dim3(BS), 0, st, vpdl && H.op == 1, lv.g.n + 1,
                 cv.g.n + 1, xres[l + 1], pend[l + 1], lv.x, done);
      if (H.op == 2) {
        etq_count_launch();
        const int nkf = lv.g.nk, nkc = cv.g.nk;
        k_prolong_p0<<<grid_for(lv.g.n0, BS, 4096), BS, 0, st>>>(lv.g.n, cv.g.n, xres[l + 1] + nkc,
                                                                 pend[l + 1] ? pend[l + 1] + nkc : nullptr, lv.x + nkf, done);
      }
    }
    etq_count_launch();
    const int gs = grid_for(lv.A.nslices * 32, BS, 4096);
    if (tile_ok(H, lv)) {
      // residual + two steps in one pass; x goes to d1 (tiles read x halos), deferred d2 to d0.
      // Finest level: the pass writes z = x + d2 (and its dot partials) itself, unless z aliases
      // an input the other tiles still read or the reduction grid exceeds the partials buffer
      const int tx = (lv.g.m + CT_T - 1) / CT_T;
      const bool fuse = l == 0 && z_u != r_u && z_u != lv.x && z_u != lv.d1 && z_u != lv.d0 &&
                        2 * tx * tx <= RED_MAXB && (!dot_out || site);
      if (fuse) {
        launch_cheb_tile(lv, true, bvec[l], lv.x, lv.d1, nullptr, lv.d0, c1, c2, theta, done, st, z_u, dot_with,
                         site, slot, dot_out, vpdl);
        etq_count_launch();
        return ETQ_OK;
      }
      launch_cheb_tile(lv, true, bvec[l], lv.x, lv.d1, nullptr, lv.d0, c1, c2, theta, done, st, nullptr, nullptr,
                       nullptr, 0, nullptr, vpdl);
      etq_count_launch();
      xres[l] = lv.d1;
      pend[l] = lv.d0;
      continue;
    }
    if (lv.st_on) {
      ChebArgs a{};
      a.A = lv.A; a.dinv = lv.dinv; a.nq = nq; a.x_in = lv.x; a.r_in = bvec[l]; a.r_out = lv.r; a.d_out = lv.d0;
      a.done = done;
      launch_cheb_st(lv, a, true, theta, st, vpdl);
    } else if (H.op == 1) {
      ChebArgs a{};
      a.x_in = lv.x; a.r_in = bvec[l]; a.r_out = lv.r; a.d_out = lv.d0; a.done = done;
      launch_cheb_sk(H, lv, a, 1, theta, st, vpdl);
    } else if (nc == 2) {
      k_post_residual<2><<<gs, BS, 0, st>>>(lv.A, lv.dinv, nq, bvec[l], lv.x, lv.r, lv.d0, 1.0 / theta, done);
    } else {
      k_post_residual<1><<<gs, BS, 0, st>>>(lv.A, lv.dinv, nq, bvec[l], lv.x, lv.r, lv.d0, 1.0 / theta, done);
    }
    etq_count_launch();
    double* din = lv.d0; double* dout = lv.d1;
    for (int k = 0; k < H.degree - 1; ++k) {
      ChebArgs a;
      a.A = lv.A; a.dinv = lv.dinv; a.nq = nq;
      a.d_in = din; a.r_in = lv.r; a.x_in = lv.x;
      a.x_out = lv.x; a.r_out = (k == H.degree - 2) ? nullptr : lv.r; a.d_out = dout;
      a.c1 = c1[k]; a.c2 = c2[k]; a.done = done;
      if (lv.st_on) launch_cheb_st(lv, a, false, theta, st, vpdl);
      else if (H.op == 1) launch_cheb_sk(H, lv, a, 0, theta, st, vpdl);
      else if (nc == 2) k_cheb_step<2><<<gs, BS, 0, st>>>(a);
      else k_cheb_step<1><<<gs, BS, 0, st>>>(a);
      etq_count_launch();
      std::swap(din, dout);
    }
    pend[l] = din;   // last correction deferred to the consumer
  }
  const Level& F = H.lv[0];
  const int64_t nv = (int64_t)nc * F.nrows;
launch_pdl(k_final_add, dim3(grid_for(nv, BS, RED_BLOCKS)), dim3(BS), 0, st, vpdl, (const double*)xres[0], pend[0], z_u,
             nv, dot_with, site ? *site : dummy, slot, dot_out, done); etq_count_launch();
  return ETQ_OK;
}

// Ap^{-1} r ~ one Q1 V-cycle, then the mean-zero projection (reading R13)
etq_status ap_solve(const Problem& P, const Hierarchy& H, const double* r, double* z, double* sum_slot,
                    const double* done, cudaStream_t st) {
  ETQ_TRY(vcycle_apply_ex(P, H, r, z, nullptr, 0, nullptr, nullptr, done, st));
  const int64_t nk = H.lv[0].nrows;
  k_final_add<<<grid_for(nk, BS, RED_BLOCKS), BS, 0, st>>>(z, nullptr, z, nk, nullptr, P.red[0], 6, sum_slot, done);
  etq_count_launch();
  k_sub_mean<<<grid_for(nk, BS, 4096), BS, 0, st>>>(z, nk, sum_slot, done); etq_count_launch();
  return ETQ_OK;
}

// ---------------------------------------------------------------- mass / SGS
void mass_apply(const Geo& g, const double* x, double* y, cudaStream_t st) {
  k_mass_apply<<<grid_for((int64_t)g.nk + g.n0, BS, 4096), BS, 0, st>>>(mass_geo(g), x, y); etq_count_launch();
}

static void launch_sgs_tile(SgsTileArgs a, cudaStream_t st, bool pdl = false) {
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k_sgs_tile<64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sgs_smem<64>());
    cudaFuncSetAttribute(k_sgs_tile<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sgs_smem<32>());
    cudaFuncSetAttribute(k_sgs_tile<32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sgs_smem<32>());
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  a.tiles_x = (a.g.n + 1 + SGS_TTX - 1) / SGS_TTX;
  // 64 x 32 windows (256 threads, four CTAs per SM) by default: 12 % more redundant sweep work than
  // 64 x 64 windows (two per SM), but smaller CTAs fill the SMs left by the concurrent V-cycle
  // better (measured, n = 1024, interleaved: Pi C Pi 600 -> 574 us, c3 814 -> 825 it/s).  When the
  // tiles fit in one wave of 512-thread CTAs (n <= 512), one plane row per thread (512 threads):
  // the step is then the latency of one CTA, which this halves in the sweep
  const int tiles32 = a.tiles_x * ((a.g.n + 1 + (32 - 6) - 1) / (32 - 6));
  const int geo = g_sgs_window ? g_sgs_window : (tiles32 <= 2 * sms ? 3 : 2);
  const int wy = geo == 1 ? 64 : 32, mr = geo == 3 ? 1 : 2;
  const int tiles = a.tiles_x * ((a.g.n + 1 + (wy - 6) - 1) / (wy - 6));
  {
    SgsK& k = a.k;
    const double h = a.g.h;
    k.w_in = 4.0 * h / 6.0; k.w_bd = 2.0 * h / 6.0; k.w_off = h / 6.0; k.rq = 0.25 * h * h;
    k.c_dd = k.w_off * k.w_off; k.c_ed = k.w_off * k.w_in;
    k.inv_in2 = 1.0 / (k.w_in * k.w_in); k.inv_inbd = 1.0 / (k.w_in * k.w_bd); k.inv_bd2 = 1.0 / (k.w_bd * k.w_bd);
    k.inv_q0 = 1.0 / (h * h);
  }
  // the latency-bound pressure chain runs at the lowest priority so that the concurrent,
  // bandwidth-bound V-cycle blocks are scheduled first (the attribute is kept by graph capture)
  static int lo_prio = 1, hi_prio = 0;
  if (lo_prio == 1) cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles); cfg.blockDim = dim3(SGS_TX, wy / 2 / mr);
  cfg.dynamicSmemBytes = wy == 64 ? sgs_smem<64>() : sgs_smem<32>(); cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = g_sgs_high_prio ? hi_prio : lo_prio;
  // programmatic dependent launch on the previous SGS step: this grid's CTAs are launched while
  // the previous step drains and wait in griddepcontrol.wait (kernel-boundary bubble hidden)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  a.pdl = pdl && g_sgs_pdl ? 1 : 0;
  a.yp_ldg = g_sgs_yp_ldg ? 1 : 0;
  cfg.attrs = attr; cfg.numAttrs = a.pdl ? 2 : 1;
  if (geo == 1) cudaLaunchKernelEx(&cfg, k_sgs_tile<64, 2>, a);
  else if (geo == 3) cudaLaunchKernelEx(&cfg, k_sgs_tile<32, 1>, a);
  else cudaLaunchKernelEx(&cfg, k_sgs_tile<32, 2>, a);
  etq_count_launch();
}

// z = S(y) (one symmetric sweep from y; y nullable = 0); t is scratch for the in-place case
void sgs_sweep_dev(const Geo& g, const double* r, const double* y, double* z, double* t, cudaStream_t st) {
  SgsTileArgs a{};
  a.g = mass_geo(g); a.r = r; a.kproj = nullptr; a.inv_kk = 0.0;
  a.y = y; a.yp = nullptr; a.mode = 0; a.omega = 1.0; a.gam = 1.0;
  a.site = RedSite{}; a.slot = 0; a.kout = nullptr; a.done = nullptr;
  const int64_t np = (int64_t)g.nk + g.n0;
  if (y == z) {
    a.out = t;
    launch_sgs_tile(a, st);
    cudaMemcpyAsync(z, t, sizeof(double) * np, cudaMemcpyDeviceToDevice, st);
  } else {
    a.out = z;
    launch_sgs_tile(a, st);
  }
}

// z_p = Pi C Pi r_p (reading R6) with C = m-step Chebyshev semi-iteration on SGS (reading R7)
// Pi C Pi on the planar copies: k^T r fused with the planar copy of r, m steps of k_sgs_plane (TMA
// windows), the last one writing the lexicographic layout, then the k-projection of the output.
// Same operations and arithmetic as the lexicographic chain below (k^T out summed in another order).
static etq_status mass_pc_apply_planar(const Problem& P, const double* r_p, double* z_p, RedSite rs, int slot,
                                       double* dot_out, const double* dot_with, const double* done, cudaStream_t st,
                                       double scale) {
  const PcMass& M = P.pm;
  const Geo& g = P.g;
  const int64_t np = (int64_t)g.nk + g.n0;
  const int64_t pl = (int64_t)M.pw * M.ph;
  const double inv_kk = 1.0 / (double)np;
  const int gf = grid_for(np, BS, RED_BLOCKS);
  k_kdot_planar<<<gf, BS, 0, st>>>(g.n, np, M.pw, pl, r_p, M.rp, rs, 3, P.dscal + S_KR, done); etq_count_launch();
  static bool smem_set = false;
  if (!smem_set) {
    cudaFuncSetAttribute(k_sgs_plane, cudaFuncAttributeMaxDynamicSharedMemorySize, SGSP_SMEM);
    smem_set = true;
  }
  static int lo_prio = 1, hi_prio = 0;
  if (lo_prio == 1) cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  const double rho = 1.0 - M.a;
  const double gam = 2.0 / (2.0 - rho), rh = rho / (2.0 - rho);
  double omega = 1.0;
  int cur = -1, prev = -1;                  // planar buffer indices of y and y_prev
  SgsPlaneArgs a{};
  a.g = mass_geo(g);
  {
    SgsK& k = a.k;
    const double h = g.h;
    k.w_in = 4.0 * h / 6.0; k.w_bd = 2.0 * h / 6.0; k.w_off = h / 6.0; k.rq = 0.25 * h * h;
    k.c_dd = k.w_off * k.w_off; k.c_ed = k.w_off * k.w_in;
    k.inv_in2 = 1.0 / (k.w_in * k.w_in); k.inv_inbd = 1.0 / (k.w_in * k.w_bd); k.inv_bd2 = 1.0 / (k.w_bd * k.w_bd);
    k.inv_q0 = 1.0 / (h * h);
  }
  a.pw = M.pw; a.ph = M.ph; a.pl = pl;
  a.rp = M.rp; a.kproj = P.dscal + S_KR; a.inv_kk = inv_kk;
  a.gam = gam;
  a.tiles_x = (g.n + 1 + SGSP_TTX - 1) / SGSP_TTX;
  const int tiles = a.tiles_x * ((g.n + 1 + SGSP_TTY - 1) / SGSP_TTY);
  a.site = rs; a.slot = 4; a.done = done;
  for (int k = 0; k < M.m; ++k) {
    if (k == 1) omega = 1.0 / (1.0 - 0.5 * rh * rh);
    else if (k > 1) omega = 1.0 / (1.0 - 0.25 * rh * rh * omega);
    const bool last = k == M.m - 1;
    const int outb = (cur == 0) ? 1 : 0;    // never the buffer read as y (y_prev is overwritten in place)
    a.yg = cur >= 0 ? M.yp[cur] : nullptr;
    a.ypg = prev >= 0 ? M.yp[prev] : nullptr;
    a.outp = last ? nullptr : M.yp[outb];
    a.out_abi = last ? M.y0 : nullptr;
    a.omega = (k == 0) ? 1.0 : omega;
    a.kout = last ? P.dscal + S_KY : nullptr;
    a.pdl = (k > 0 && g_sgs_pdl) ? 1 : 0;
    const void* tm_y = M.tmap[cur >= 0 ? cur : 0];
    const void* tm_yp = M.tmap[prev >= 0 ? prev : 0];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles); cfg.blockDim = dim3(SGS_TX, SGSP_TY); cfg.dynamicSmemBytes = SGSP_SMEM; cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = g_sgs_high_prio ? hi_prio : lo_prio;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr; cfg.numAttrs = a.pdl ? 2 : 1;
    cudaLaunchKernelEx(&cfg, k_sgs_plane, a, *reinterpret_cast<const CUtensorMap*>(tm_y),
                       *reinterpret_cast<const CUtensorMap*>(tm_yp));
    etq_count_launch();
    prev = cur; cur = outb;
  }
  k_kproject_out<<<gf, BS, 0, st>>>(g.nk, np, M.y0, P.dscal + S_KY, inv_kk, scale, z_p, dot_with, rs, slot, dot_out,
                                    done); etq_count_launch();
  return ETQ_OK;
}

etq_status mass_pc_apply_ex(const Problem& P, const double* r_p, double* z_p, const RedSite* site, int slot,
                            double* dot_out, const double* dot_with, const double* done, cudaStream_t st,
                            double scale) {
  NvtxRange nvtx_("Pi C Pi (Chebyshev-SGS)");
  const PcMass& M = P.pm;
  if (!M.ready) return ETQ_ENOTSETUP;
  const Geo& g = P.g;
  const int64_t np = (int64_t)g.nk + g.n0;
  const double inv_kk = 1.0 / (double)np;
  const int gf = grid_for(np, BS, RED_BLOCKS);
  RedSite rs = *site;
  if (M.planar && g_sgs_planar && M.m >= 1) return mass_pc_apply_planar(P, r_p, z_p, rs, slot, dot_out, dot_with, done,
                                                                        st, scale);
  // k^T r (Pi applied on the fly inside the sweeps)
  k_kdot<<<gf, BS, 0, st>>>(g.nk, np, r_p, rs, 3, P.dscal + S_KR, done); etq_count_launch();
  const double rho = 1.0 - M.a;
  const double gam = 2.0 / (2.0 - rho), rh = rho / (2.0 - rho);
  double omega = 1.0;
  const double* cur = nullptr; const double* prev = nullptr;
  double* bufs[2] = {M.y0, M.y1};
  int nb = 0;
  for (int k = 0; k < M.m; ++k) {
    if (k == 1) omega = 1.0 / (1.0 - 0.5 * rh * rh);
    else if (k > 1) omega = 1.0 / (1.0 - 0.25 * rh * rh * omega);
    double* out = bufs[nb]; nb ^= 1;
    SgsTileArgs a{};
    a.g = mass_geo(g); a.r = r_p; a.kproj = P.dscal + S_KR; a.inv_kk = inv_kk;
    a.y = cur; a.yp = prev; a.out = out; a.mode = 1;
    a.omega = (k == 0) ? 1.0 : omega; a.gam = gam;
    a.site = rs; a.slot = 4; a.kout = (k == M.m - 1) ? P.dscal + S_KY : nullptr; a.done = done;
    launch_sgs_tile(a, st, k > 0);
    prev = cur; cur = out;
  }
  k_kproject_out<<<gf, BS, 0, st>>>(g.nk, np, cur, P.dscal + S_KY, inv_kk, scale, z_p, dot_with, rs, slot, dot_out,
                                    done); etq_count_launch();
  return ETQ_OK;
}

// ---- bench helpers (etq_time_kernel 10-12)
// one Chebyshev-SGS step (mode 1: the semi-iteration combination) on the pressure vectors
void sgs_step_bench(const Problem& P, const double* r, const double* y, const double* yp, double* out,
                    cudaStream_t st) {
  SgsTileArgs a{};
  a.g = mass_geo(P.g); a.r = r; a.kproj = nullptr; a.inv_kk = 0.0;
  a.y = y; a.yp = yp; a.out = out; a.mode = 1; a.omega = 1.2; a.gam = 1.1;
  a.site = RedSite{}; a.slot = 0; a.kout = nullptr; a.done = nullptr;
  launch_sgs_tile(a, st);
}

// the finest level's temporally blocked pre- (post = false) or post-smoothing pass
etq_status cheb_tile_bench(const Problem& P, bool post, const double* in_b, const double* in_x, double* o1,
                           double* o2, cudaStream_t st) {
  const Hierarchy& H = P.mg;
  if (!H.built || !tile_ok(H, H.lv[0])) return ETQ_ENOTSETUP;
  std::vector<double> c1, c2;
  cheb_coeffs(H.lo, H.hi, H.lv[0].bim, H.degree, c1, c2);
  const double theta = 0.5 * (H.hi + H.lo);
  // post: outputs into the level's own scratch (x -> d1, deferred d -> d0) exactly as in the V-cycle
  if (post) launch_cheb_tile(H.lv[0], true, in_b, in_x, H.lv[0].d1, nullptr, H.lv[0].d0, c1, c2, theta, nullptr, st);
  else launch_cheb_tile(H.lv[0], false, in_b, nullptr, o1, o2, nullptr, c1, c2, theta, nullptr, st);
  etq_count_launch();
  return ETQ_OK;
}

// TMA descriptor of a planar pressure vector: 3D tensor {pw, ph, 8 planes}, box {32, 16, 8} (one SGS
// window), zero fill outside (the domain edges of every window)
static etq_status encode_planar_map(void* tmap, double* base, int pw, int ph) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return ETQ_ECUDA;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)pw, (cuuint64_t)ph, 8};
  const cuuint64_t strides[2] = {(cuuint64_t)pw * sizeof(double), (cuuint64_t)pw * ph * sizeof(double)};
  const cuuint32_t box[3] = {SGS_P, SGSP_WY / 2, 8};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(reinterpret_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides,
                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? ETQ_OK : ETQ_ECUDA;
}

etq_status mass_pc_alloc(Problem& P) {
  const int64_t np = P.n_p;
  PcMass& M = P.pm;
  if (!M.t) {
    ETQ_TRY(dalloc(&M.t, np)); ETQ_TRY(dalloc(&M.y0, np)); ETQ_TRY(dalloc(&M.y1, np)); ETQ_TRY(dalloc(&M.rr, np));
  }
  if (!M.rp && P.g.n >= 2 && P.g.n % 2 == 0) {
    // planar copies (k_sgs_plane): pw even so that plane rows are 16-byte multiples (TMA strides)
    M.pw = ((P.g.n / 2 + 1) + 1) & ~1;
    M.ph = P.g.n / 2 + 1;
    const size_t sz = (size_t)8 * M.pw * M.ph;
    ETQ_TRY(dalloc(&M.rp, sz)); ETQ_TRY(dalloc(&M.yp[0], sz)); ETQ_TRY(dalloc(&M.yp[1], sz));
    // entries outside the domain stay zero forever (only in-domain entries are ever written)
    for (double* b : {M.rp, M.yp[0], M.yp[1]}) ETQ_CHECK(cudaMemset(b, 0, sz * sizeof(double)));
    for (int k = 0; k < 2; ++k) ETQ_TRY(encode_planar_map(M.tmap[k], M.yp[k], M.pw, M.ph));
    M.planar = true;
  }
  return ETQ_OK;
}

// Lanczos for the pencil (M_Q, C_sgs), start p_1 = M_Q v0 (reading R7); smallest Ritz value.
etq_status lanczos_sgs_lo(Problem& P, const double* v0, int steps, double* lam) {
  ETQ_TRY(mass_pc_alloc(P));
  const Geo& g = P.g;
  const int64_t np = P.n_p;
  cudaStream_t st = P.stream;
  double *p, *pp, *q, *w, *z;
  ETQ_TRY(dalloc(&p, np)); ETQ_TRY(dalloc(&pp, np)); ETQ_TRY(dalloc(&q, np)); ETQ_TRY(dalloc(&w, np));
  ETQ_TRY(dalloc(&z, np));
  RedSite rs = P.red[0];
  double* d0 = P.dscal + S_TMP0 + 8;
  auto dot = [&](const double* a, const double* b) -> double {
    launch_dot(a, b, np, &rs, 5, d0, nullptr, st);
    double h = 0;
    cudaMemcpyAsync(&h, d0, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return h;
  };
  mass_apply(g, v0, p, st);
  sgs_sweep_dev(g, p, nullptr, q, P.pm.t, st);
  const double b0 = std::sqrt(dot(q, p));
  std::vector<double> al, be;
  // scale p, q by 1/b0 ; pp = 0
  vec_scale_copy(p, p, 1.0 / b0, np, st);
  vec_scale_copy(q, q, 1.0 / b0, np, st);
  ETQ_CHECK(cudaMemsetAsync(pp, 0, np * 8, st));
  double beta_prev = 0.0;
  for (int j = 0; j < steps; ++j) {
    mass_apply(g, q, w, st);
    const double alpha = dot(q, w);
    vec_lincomb3(w, w, 1.0, p, -alpha, pp, -beta_prev, np, st);
    al.push_back(alpha);
    if (j == steps - 1) break;
    sgs_sweep_dev(g, w, nullptr, z, P.pm.t, st);
    const double zw = dot(z, w);
    if (!(zw > 0.0)) break;
    const double beta = std::sqrt(zw);
    be.push_back(beta);
    std::swap(pp, p);
    vec_scale_copy(p, w, 1.0 / beta, np, st);
    vec_scale_copy(q, z, 1.0 / beta, np, st);
    beta_prev = beta;
  }
  cudaStreamSynchronize(st);
  cudaFree(p); cudaFree(pp); cudaFree(q); cudaFree(w); cudaFree(z);
  // smallest eigenvalue of the tridiagonal by Sturm bisection
  const int k = (int)al.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::fabs(be[i - 1]) : 0.0) + (i < k - 1 ? std::fabs(be[i]) : 0.0);
    lo = std::fmin(lo, al[i] - r); hi = std::fmax(hi, al[i] + r);
  }
  auto count_below = [&](double x) {
    int c = 0; double d = 1.0;
    for (int i = 0; i < k; ++i) {
      d = al[i] - x - (i > 0 ? be[i - 1] * be[i - 1] / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0) ++c;
    }
    return c;
  };
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) >= 1) hi = mid; else lo = mid;
  }
  *lam = 0.5 * (lo + hi);
  return ETQ_OK;
}

// ---------------------------------------------------------------- bench helpers
// middle Chebyshev step of the finest level (x, r in place; d_in -> d_out)
void cheb_step_level0(const Problem& P, const double* d_in, double* d_out, cudaStream_t st) {
  const Level& lv = P.mg.lv[0];
  ChebArgs a;
  a.A = lv.A; a.dinv = lv.dinv; a.nq = lv.g.nq;
  a.d_in = d_in; a.r_in = lv.r; a.x_in = lv.x; a.x_out = lv.x; a.r_out = lv.r; a.d_out = d_out;
  a.c1 = 0.5; a.c2 = 0.1; a.done = nullptr;
  if (lv.st_on) launch_cheb_st(lv, a, false, 0.0, st);
  else k_cheb_step<2><<<grid_for(lv.A.nslices * 32, BS, 4096), BS, 0, st>>>(a);
  etq_count_launch();
}

// Algorithmic bytes: every stored value/index once (12 B per true nnz), the
// row permutation (4 B per slot), every vector element the kernel must read or write once.
double cheb_step_bytes(const Level& L) {
  const double nq = L.nrows;
  return 12.0 * L.A.nnz - 4.0 * L.A.nnz_implicit - 8.0 * L.A.nnz_implicit_vals + 4.0 * L.A.nslices * SELL_C + 8.0 * nq /*dinv*/ + 8.0 * 2 * nq * 6 /*d,r,x in; x,r,d out*/;
}

double vcycle_bytes(const Hierarchy& H) {
  double b = 0.0;
  const int L = (int)H.lv.size();
  const int deg = H.degree;
  for (int l = 0; l < L - 1; ++l) {
    const Level& lv = H.lv[l];
    const double nq = lv.g.nq, mat = 12.0 * lv.A.nnz - 4.0 * lv.A.nnz_implicit - 8.0 * lv.A.nnz_implicit_vals + 4.0 * lv.A.nslices * SELL_C + 8.0 * nq;
    const double v = 8.0 * 2 * nq;   // one two-component vector
    const bool tiled = tile_ok(H, lv);
    if (tiled) b += 3 * v;                                   // fused pre pass: b -> x, r (matrix-free)
    else {
      if (l == 0) b += 8.0 * nq + 2 * v;                     // init: dinv, b -> d
      for (int k = 0; k < deg; ++k)                          // pre-smoothing steps
        b += mat + v * ((k == 0 ? 2 : 3) + (k == deg - 1 ? 2 : 3));
    }
    const double nqc = H.lv[l + 1].g.nq, vc = 8.0 * 2 * nqc;
    b += v + 2 * vc + 8.0 * nqc;                             // restriction: r -> b_c, d0_c
    b += 2 * vc + 2 * v;                                     // prolongation: x_c + d_c -> x += P e
    if (tiled) b += 4 * v;                                   // fused post pass: x, b -> x, d
    else {
      b += mat + 2 * v + 2 * v;                              // post residual: b, x -> r, d
      for (int k = 0; k < deg - 1; ++k)                      // post steps
        b += mat + v * (3 + (k == deg - 2 ? 2 : 3));
    }
    if (l == 0) b -= tiled ? v : 0.0;                        // tiled finest post pass: z out, no x / d
    if (l == 0 && !tiled) b += 2 * v + v;                    // final: x + d -> z
  }
  const Level& C = H.lv[L - 1];
  b += 8.0 * (double)C.g.nq * C.g.nq + 4.0 * 8.0 * C.g.nq;  // dense coarse solve
  return b;
}

// Pi C Pi (mass_pc_apply_ex): k^T r (r in), step 0 (r in, out), step 1 (r, y in, out), steps
// 2..m-1 (r, y, y_prev in, out), projection (y in, z out); 640 n_p bytes at m = 20
double mass_pc_bytes(const Problem& P) {
  const double np = (double)P.g.nk + P.g.n0;
  const int m = P.pm.m;
  if (m < 1) return 0.0;
  double b = 8.0 * np + 16.0 * np;
  if (m >= 2) b += 24.0 * np + 32.0 * np * (m - 2);
  return b + 16.0 * np;
}

// fp32 V-cycle algorithmic bytes: 8 B per stored entry + 4 B index... i.e. values 4 B + index 4 B,
// fp32 vectors (half of the fp64 vector traffic)
double vcycle_bytes_f32(const Hierarchy& H) {
  double b = 0.0;
  const int L = (int)H.lv.size();
  const int deg = H.degree;
  for (int l = 0; l < L - 1; ++l) {
    const Level& lv = H.lv[l];
    const double nq = lv.nrows, mat = 8.0 * lv.A.nnz + 4.0 * lv.A.nslices * SELL_C + 4.0 * nq;
    const double v = 4.0 * 2 * nq;
    if (l == 0) b += 4.0 * nq + 2 * v;
    for (int k = 0; k < deg; ++k) b += mat + v * ((k == 0 ? 2 : 3) + (k == deg - 1 ? 2 : 3));
    const double nqc = H.lv[l + 1].nrows, vc = 4.0 * 2 * nqc;
    b += v + 2 * vc + 4.0 * nqc;
    b += 2 * vc + 2 * v;
    b += mat + 2 * v + 2 * v;
    for (int k = 0; k < deg - 1; ++k) b += mat + v * (3 + (k == deg - 2 ? 2 : 3));
    if (l == 0) b += 2 * v + v;
  }
  const Level& C = H.lv[L - 1];
  b += 4.0 * (double)C.nrows * C.nrows + 4.0 * 4.0 * C.nrows;
  return b;
}
