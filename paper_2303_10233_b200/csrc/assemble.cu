// assemble.cu — row-gather assembly of the Q2–Q1* blocks straight into SELL-32 slices.
//
// On the uniform grid every block is a sum of tensor products of 1D "global" matrices, so a
// thread computes its row from closed-form 1D element tables (no element loop, no atomics):
//   L   = M1 (x) K1 + K1 (x) M1                 a(u,v) = int grad u : grad v
//   B1x = -H1 (x) G1, B1y = -G1 (x) H1          b(u,p) = -int p div u
//   B0x = -W1 (x) E1, B0y = -E1 (x) W1          P0 rows, -int_T d_x phi
//   M_v = M1 (x) M1                              Galerkin load (reading R10)
//   N   = A1 (x) T2 - T2 (x) A1                  int (w . grad phi_j) phi_i for the separable
//                                                cavity wind w = (2y(1-x^2), -2x(1-y^2))
// (first factor acts on y / the slow index, second on x.)  The 1D tables are the exact
// integrals of the quadratic (Q2) and linear (Q1) Lagrange bases on one interval; A1 and T2
// use 3-point Gauss per interval, exact for their degree-5 integrands.
// Dirichlet handling (reading R2): boundary velocity rows are identity rows, boundary columns
// are dropped from L, F and B, and their contribution is lifted into the right-hand side.
#include "etq_internal.cuh"
#include <cstdio>
#include <cstring>
#include <vector>

namespace {

// ---------------------------------------------------------------- 1D element tables
__device__ __constant__ double cK2[3][3] = {{7.0 / 3, -8.0 / 3, 1.0 / 3},
                                           {-8.0 / 3, 16.0 / 3, -8.0 / 3},
                                           {1.0 / 3, -8.0 / 3, 7.0 / 3}};          // x 1/h
__device__ __constant__ double cM2[3][3] = {{4.0 / 30, 2.0 / 30, -1.0 / 30},
                                           {2.0 / 30, 16.0 / 30, 2.0 / 30},
                                           {-1.0 / 30, 2.0 / 30, 4.0 / 30}};       // x h
__device__ __constant__ double cG[2][3] = {{-5.0 / 6, 4.0 / 6, 1.0 / 6},
                                          {-1.0 / 6, -4.0 / 6, 5.0 / 6}};          // int N_a L_b'
__device__ __constant__ double cH[2][3] = {{1.0 / 6, 2.0 / 6, 0.0},
                                          {0.0, 2.0 / 6, 1.0 / 6}};                // x h
__device__ __constant__ double cE[3] = {-1.0, 0.0, 1.0};                          // int L_b'
__device__ __constant__ double cW[3] = {1.0 / 6, 4.0 / 6, 1.0 / 6};               // x h

__device__ __forceinline__ double lag2(int a, double x) {
  return a == 0 ? 2.0 * (x - 0.5) * (x - 1.0) : (a == 1 ? 4.0 * x * (1.0 - x) : 2.0 * x * (x - 0.5));
}
__device__ __forceinline__ double dlag2(int a, double x) {
  return a == 0 ? 4.0 * x - 3.0 : (a == 1 ? 4.0 - 8.0 * x : 4.0 * x - 1.0);
}

// Oseen 1D tables on element e: A1loc[a][b] = int (1-x^2) L_b' L_a dx, T2loc[a][b] = int 2x L_b L_a dx
__device__ double oseen_tab(int which, int n, double h, int e, int a, int b) {
  const double gx[3] = {0.5 - 0.5 * 0.7745966692414834, 0.5, 0.5 + 0.5 * 0.7745966692414834};
  const double gw[3] = {5.0 / 18, 8.0 / 18, 5.0 / 18};
  double s = 0.0;
  for (int q = 0; q < 3; ++q) {
    double x = -1.0 + (e + gx[q]) * h;
    if (which == 0) s += gw[q] * (1.0 - x * x) * dlag2(b, gx[q]) * lag2(a, gx[q]);
    else s += gw[q] * h * 2.0 * x * lag2(b, gx[q]) * lag2(a, gx[q]);
  }
  return s;
}

// 1D global Q2-Q2 entries: sum over the (<= 2) intervals containing both nodes
__device__ double k1(int n, double h, int i, int ip) {
  int lo = min(i, ip), hi = max(i, ip);
  if (hi - lo > 2) return 0.0;
  double s = 0.0;
  for (int e = lo / 2 - 1; e <= lo / 2; ++e)
    if (e >= 0 && e < n && 2 * e <= lo && hi <= 2 * e + 2) s += cK2[i - 2 * e][ip - 2 * e];
  return s / h;
}
__device__ double m1(int n, double h, int i, int ip) {
  int lo = min(i, ip), hi = max(i, ip);
  if (hi - lo > 2) return 0.0;
  double s = 0.0;
  for (int e = lo / 2 - 1; e <= lo / 2; ++e)
    if (e >= 0 && e < n && 2 * e <= lo && hi <= 2 * e + 2) s += cM2[i - 2 * e][ip - 2 * e];
  return s * h;
}
__device__ double osn1(int which, int n, double h, int i, int ip) {
  int lo = min(i, ip), hi = max(i, ip);
  if (hi - lo > 2) return 0.0;
  double s = 0.0;
  for (int e = lo / 2 - 1; e <= lo / 2; ++e)
    if (e >= 0 && e < n && 2 * e <= lo && hi <= 2 * e + 2)
      s += oseen_tab(which, n, h, e, i - 2 * e, ip - 2 * e);
  return s;
}
// Q1 (row a) x Q2 (column i)
__device__ double g1(int n, int a, int i) {
  double s = 0.0;
  for (int e = a - 1; e <= a; ++e)
    if (e >= 0 && e < n && i >= 2 * e && i <= 2 * e + 2) s += cG[a - e][i - 2 * e];
  return s;
}
__device__ double h1(int n, double h, int a, int i) {
  double s = 0.0;
  for (int e = a - 1; e <= a; ++e)
    if (e >= 0 && e < n && i >= 2 * e && i <= 2 * e + 2) s += cH[a - e][i - 2 * e];
  return s * h;
}
// P0 (element e) x Q2 (column i)
__device__ double e1(int e, int i) { return (i >= 2 * e && i <= 2 * e + 2) ? cE[i - 2 * e] : 0.0; }
__device__ double w1(double h, int e, int i) {
  return (i >= 2 * e && i <= 2 * e + 2) ? cW[i - 2 * e] * h : 0.0;
}

struct VelParams { Geo g; int oseen; double nu; };   // oseen: 0 Stokes, 1 cavity wind, 2 nodal wind (nu L part)

// entry of the scalar velocity operator between nodes (i,j) and (ii,jj), no Dirichlet masking
__device__ double vel_entry(const VelParams& P, int i, int j, int ii, int jj) {
  const int n = P.g.n; const double h = P.g.h;
  double v = m1(n, h, j, jj) * k1(n, h, i, ii) + k1(n, h, j, jj) * m1(n, h, i, ii);
  if (P.oseen == 1) {
    v = P.nu * v + osn1(0, n, h, i, ii) * osn1(1, n, h, j, jj) - osn1(1, n, h, i, ii) * osn1(0, n, h, j, jj);
  } else if (P.oseen == 2) {   // nodal (Picard) wind: nu L here, the convection is added by picard.cu
    v = P.nu * v;
  }
  return v;
}

__device__ __forceinline__ bool on_boundary(int i, int j, int m) {
  return i == 0 || j == 0 || i == m - 1 || j == m - 1;
}

// Enumerate row `node` of the Dirichlet-modified scalar operator.  Stokes drops the entries
// that cancel exactly in M1(x)K1 + K1(x)M1 (vertex-vertex distance 2 along a midpoint line).
template <class Emit>
__device__ int vel_row(const VelParams& P, int node, Emit& emit) {
  const int m = P.g.m;
  const int i = node % m, j = node / m;
  if (on_boundary(i, j, m)) { emit(node, 1.0); return 1; }
  const int rx = (i & 1) ? 1 : 2, ry = (j & 1) ? 1 : 2;
  int cnt = 0;
  for (int dj = -ry; dj <= ry; ++dj) {
    const int jj = j + dj;
    if (jj <= 0 || jj >= m - 1) continue;
    for (int di = -rx; di <= rx; ++di) {
      const int ii = i + di;
      if (ii <= 0 || ii >= m - 1) continue;
      if (!P.oseen) {
        if ((di == 2 || di == -2) && dj == 0 && (j & 1)) continue;
        if ((dj == 2 || dj == -2) && di == 0 && (i & 1)) continue;
      }
      emit(ii + m * jj, vel_entry(P, i, j, ii, jj));
      ++cnt;
    }
  }
  return cnt;
}

// B^T row (velocity node -> pressure columns): comp 0 = x, 1 = y; part 0 = Q1, 1 = P0
struct BtParams { Geo g; int comp; int part; };
template <class Emit>
__device__ int bt_row(const BtParams& P, int node, Emit& emit) {
  const int m = P.g.m, n = P.g.n; const double h = P.g.h;
  const int i = node % m, j = node / m;
  if (on_boundary(i, j, m)) return 0;
  int cnt = 0;
  if (P.part == 0) {
    for (int c = max(0, j / 2 - 1); c <= min(n, j / 2 + 1); ++c)
      for (int a = max(0, i / 2 - 1); a <= min(n, i / 2 + 1); ++a) {
        double v = P.comp == 0 ? -g1(n, a, i) * h1(n, h, c, j) : -h1(n, h, a, i) * g1(n, c, j);
        if (v != 0.0) { emit(a + (n + 1) * c, v); ++cnt; }
      }
  } else {
    for (int f = max(0, j / 2 - 1); f <= min(n - 1, j / 2); ++f)
      for (int e = max(0, i / 2 - 1); e <= min(n - 1, i / 2); ++e) {
        double v = P.comp == 0 ? -e1(e, i) * w1(h, f, j) : -w1(h, e, i) * e1(f, j);
        if (v != 0.0) { emit(e + n * f, v); ++cnt; }
      }
  }
  return cnt;
}

// B row: pressure dof (Q1 vertex rows first, then P0 rows) -> columns in [u_x; u_y]
struct BParams { Geo g; };
template <class Emit>
__device__ int b_row(const BParams& P, int row, Emit& emit) {
  const int m = P.g.m, n = P.g.n, nq = P.g.nq; const double h = P.g.h;
  int cnt = 0;
  if (row < P.g.nk) {
    const int a = row % (n + 1), c = row / (n + 1);
    for (int j = max(1, 2 * c - 2); j <= min(m - 2, 2 * c + 2); ++j) {
      const double hc = h1(n, h, c, j), gc = g1(n, c, j);
      for (int i = max(1, 2 * a - 2); i <= min(m - 2, 2 * a + 2); ++i) {
        const double vx = -g1(n, a, i) * hc, vy = -h1(n, h, a, i) * gc;
        if (vx != 0.0) { emit(i + m * j, vx); ++cnt; }
        if (vy != 0.0) { emit(nq + i + m * j, vy); ++cnt; }
      }
    }
  } else {
    const int t = row - P.g.nk;
    const int e = t % n, f = t / n;
    for (int j = max(1, 2 * f); j <= min(m - 2, 2 * f + 2); ++j)
      for (int i = max(1, 2 * e); i <= min(m - 2, 2 * e + 2); ++i) {
        const double vx = -e1(e, i) * w1(h, f, j), vy = -w1(h, e, i) * e1(f, j);
        if (vx != 0.0) { emit(i + m * j, vx); ++cnt; }
        if (vy != 0.0) { emit(nq + i + m * j, vy); ++cnt; }
      }
  }
  return cnt;
}

// Ap = B1 Mdiag^{-1} B1^T on Q1 vertices (reading R12/R13): row p gathers over the
// interior velocity nodes of its B1 support and accumulates into a 5 x 5 vertex window.
struct ApParams { Geo g; };
template <class Emit>
__device__ int ap_row(const ApParams& P, int row, Emit& emit) {
  const int m = P.g.m, n = P.g.n; const double h = P.g.h;
  const int a = row % (n + 1), c = row / (n + 1);
  double acc[25];
#pragma unroll
  for (int k = 0; k < 25; ++k) acc[k] = 0.0;
  for (int jj = max(1, 2 * c - 2); jj <= min(m - 2, 2 * c + 2); ++jj) {
    for (int ii = max(1, 2 * a - 2); ii <= min(m - 2, 2 * a + 2); ++ii) {
      const double bx = -g1(n, a, ii) * h1(n, h, c, jj), by = -h1(n, h, a, ii) * g1(n, c, jj);
      if (bx == 0.0 && by == 0.0) continue;
      const double md = m1(n, h, ii, ii) * m1(n, h, jj, jj);   // diagonal of the Q2 mass
      const double wx = bx / md, wy = by / md;
      for (int cc = max(0, jj / 2 - 1); cc <= min(n, jj / 2 + 1); ++cc) {
        if (cc - c > 2 || c - cc > 2) continue;
        for (int aa = max(0, ii / 2 - 1); aa <= min(n, ii / 2 + 1); ++aa) {
          if (aa - a > 2 || a - aa > 2) continue;
          const double qx = -g1(n, aa, ii) * h1(n, h, cc, jj), qy = -h1(n, h, aa, ii) * g1(n, cc, jj);
          acc[(cc - c + 2) * 5 + (aa - a + 2)] += wx * qx + wy * qy;
        }
      }
    }
  }
  int cnt = 0;
  for (int dc = -2; dc <= 2; ++dc)
    for (int da = -2; da <= 2; ++da) {
      const double v = acc[(dc + 2) * 5 + (da + 2)];
      if (v != 0.0) { emit((a + da) + (n + 1) * (c + dc), v); ++cnt; }
    }
  return cnt;
}

// Two-field pressure Laplacian Lp = B Mdiag^{-1} B^T on [Q1; P0] (NEXT-4: the B M^{-1} B^T of the
// two-field PCD and LSC approximations).  A Q1 row gathers over the
// interior velocity nodes of its B1 support into a 5 x 5 vertex window and a 4 x 4 cell window; a P0
// row over the interior nodes of its square into 4 x 4 vertices and 3 x 3 cells.  Q1 columns first.
struct LpParams { Geo g; };
template <class Emit>
__device__ int lp_row(const LpParams& P, int row, Emit& emit) {
  const int m = P.g.m, n = P.g.n; const double h = P.g.h;
  const int nk = P.g.nk;
  double acck[25], acc0[16];
#pragma unroll
  for (int k = 0; k < 25; ++k) acck[k] = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) acc0[k] = 0.0;
  const bool q1 = row < nk;
  int a, c, i0, i1, j0, j1, kw, ko, cw, co;   // vertex window (width kw, origin ko), cell window (cw, co)
  if (q1) {
    a = row % (n + 1); c = row / (n + 1);
    i0 = max(1, 2 * a - 2); i1 = min(m - 2, 2 * a + 2); j0 = max(1, 2 * c - 2); j1 = min(m - 2, 2 * c + 2);
    kw = 5; ko = 2; cw = 4; co = 2;
  } else {
    const int t = row - nk;
    a = t % n; c = t / n;
    i0 = max(1, 2 * a); i1 = min(m - 2, 2 * a + 2); j0 = max(1, 2 * c); j1 = min(m - 2, 2 * c + 2);
    kw = 4; ko = 1; cw = 3; co = 1;
  }
  for (int jj = j0; jj <= j1; ++jj) {
    for (int ii = i0; ii <= i1; ++ii) {
      double bx, by;
      if (q1) { bx = -g1(n, a, ii) * h1(n, h, c, jj); by = -h1(n, h, a, ii) * g1(n, c, jj); }
      else { bx = -e1(a, ii) * w1(h, c, jj); by = -w1(h, a, ii) * e1(c, jj); }
      if (bx == 0.0 && by == 0.0) continue;
      const double md = m1(n, h, ii, ii) * m1(n, h, jj, jj);   // diagonal of the Q2 mass
      const double wx = bx / md, wy = by / md;
      for (int cc = max(0, jj / 2 - 1); cc <= min(n, jj / 2 + 1); ++cc) {
        if (cc - c + ko < 0 || cc - c + ko >= kw) continue;
        for (int aa = max(0, ii / 2 - 1); aa <= min(n, ii / 2 + 1); ++aa) {
          if (aa - a + ko < 0 || aa - a + ko >= kw) continue;
          const double qx = -g1(n, aa, ii) * h1(n, h, cc, jj), qy = -h1(n, h, aa, ii) * g1(n, cc, jj);
          acck[(cc - c + ko) * kw + (aa - a + ko)] += wx * qx + wy * qy;
        }
      }
      for (int ff = max(0, (jj - 1) / 2); ff <= min(n - 1, jj / 2); ++ff) {
        if (2 * ff > jj || 2 * ff + 2 < jj || ff - c + co < 0 || ff - c + co >= cw) continue;
        for (int ee = max(0, (ii - 1) / 2); ee <= min(n - 1, ii / 2); ++ee) {
          if (2 * ee > ii || 2 * ee + 2 < ii || ee - a + co < 0 || ee - a + co >= cw) continue;
          const double px = -e1(ee, ii) * w1(h, ff, jj), py = -w1(h, ee, ii) * e1(ff, jj);
          acc0[(ff - c + co) * cw + (ee - a + co)] += wx * px + wy * py;
        }
      }
    }
  }
  int cnt = 0;
  for (int dc = 0; dc < kw; ++dc)
    for (int da = 0; da < kw; ++da) {
      const double v = acck[dc * kw + da];
      if (v != 0.0) { emit((a + da - ko) + (n + 1) * (c + dc - ko), v); ++cnt; }
    }
  for (int df = 0; df < cw; ++df)
    for (int de = 0; de < cw; ++de) {
      const double v = acc0[df * cw + de];
      if (v != 0.0) { emit(nk + (a + de - co) + n * (c + df - co), v); ++cnt; }
    }
  return cnt;
}

// 1 / diagonal of the scalar Q2 velocity mass (M = Mdiag of P:922-923), Dirichlet nodes 0
__global__ void k_vel_mdiag_inv(Geo g, double* out) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= g.nq) return;
  const int m = g.m, i = node % m, j = node / m;
  out[node] = (i == 0 || j == 0 || i == m - 1 || j == m - 1) ? 0.0 : 1.0 / (m1(g.n, g.h, i, i) * m1(g.n, g.h, j, j));
}

// S_k = Q_k - R^T Q_0^{-1} R on the Q1 vertices (the Schur complement of the Q0 block of M_Q,
// P:287-294 with R = h^2/4, Q0 = h^2): per cell T, (h^2/36) m_x m_y - h^2/16 for each vertex pair
// of T (m = 2 on the same 1D index, else 1); interior stencil (h^2/144) [-5 -2 -5; -2 28 -2; -5 -2 -5].
// `scale` multiplies the operator (4^-l on hierarchy level l, reading R21).
struct SkParams { Geo g; double scale; };
template <class Emit>
__device__ int sk_row(const SkParams& P, int row, Emit& emit) {
  const int n = P.g.n; const double h2 = P.g.h * P.g.h;
  const int a = row % (n + 1), c = row / (n + 1);
  double acc[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) acc[k] = 0.0;
  for (int f = max(0, c - 1); f <= min(n - 1, c); ++f)
    for (int e = max(0, a - 1); e <= min(n - 1, a); ++e)
      for (int cc = f; cc <= f + 1; ++cc)
        for (int aa = e; aa <= e + 1; ++aa) {
          const double mx = aa == a ? 2.0 : 1.0, my = cc == c ? 2.0 : 1.0;
          acc[(cc - c + 1) * 3 + (aa - a + 1)] += h2 * (mx * my / 36.0 - 1.0 / 16.0);
        }
  int cnt = 0;
  for (int dc = -1; dc <= 1; ++dc)
    for (int da = -1; da <= 1; ++da) {
      const int aa = a + da, cc = c + dc;
      if (aa < 0 || aa > n || cc < 0 || cc > n) continue;
      emit(aa + (n + 1) * cc, P.scale * acc[(dc + 1) * 3 + (da + 1)]); ++cnt;
    }
  return cnt;
}

// F1 = nu int grad psi_j . grad psi_i + int (w . grad psi_j) psi_i on Q1, natural
// boundary (reading R13); for the separable cavity wind the convection part is
// Aq (x) Tq - Tq (x) Aq with Aq = int (1-x^2) N_b' N_a, Tq = int 2x N_b N_a (3-point Gauss, exact).
__device__ double q1tab(int which, double h, int e, int a, int b) {
  const double gx[3] = {0.5 - 0.5 * 0.7745966692414834, 0.5, 0.5 + 0.5 * 0.7745966692414834};
  const double gw[3] = {5.0 / 18, 8.0 / 18, 5.0 / 18};
  double s = 0.0;
  for (int q = 0; q < 3; ++q) {
    const double xi = gx[q], x = -1.0 + (e + xi) * h;
    const double Na = a == 0 ? 1.0 - xi : xi, Nb = b == 0 ? 1.0 - xi : xi, dNb = b == 0 ? -1.0 : 1.0;
    if (which == 0) s += gw[q] * (1.0 - x * x) * dNb * Na;
    else s += gw[q] * h * 2.0 * x * Nb * Na;
  }
  return s;
}
__device__ double q1glob(int which, int n, double h, int a, int ap) {   // 0: Aq, 1: Tq, 2: K, 3: M
  double s = 0.0;
  for (int e = max(a, ap) - 1; e <= min(a, ap); ++e) {
    if (e < 0 || e >= n) continue;
    const int la = a - e, lb = ap - e;
    if (which <= 1) s += q1tab(which, h, e, la, lb);
    else if (which == 2) s += (la == lb ? 1.0 : -1.0) / h;
    else s += (la == lb ? 2.0 : 1.0) * h / 6.0;
  }
  return s;
}
struct F1Params { Geo g; double nu; int wind; };
template <class Emit>
__device__ int f1_row(const F1Params& P, int row, Emit& emit) {
  const int n = P.g.n; const double h = P.g.h;
  const int a = row % (n + 1), c = row / (n + 1);
  int cnt = 0;
  for (int cc = max(0, c - 1); cc <= min(n, c + 1); ++cc)
    for (int aa = max(0, a - 1); aa <= min(n, a + 1); ++aa) {
      double v = P.nu * (q1glob(2, n, h, a, aa) * q1glob(3, n, h, c, cc) + q1glob(3, n, h, a, aa) * q1glob(2, n, h, c, cc));
      if (P.wind == 1)
        v += q1glob(0, n, h, a, aa) * q1glob(1, n, h, c, cc) - q1glob(1, n, h, a, aa) * q1glob(0, n, h, c, cc);
      emit(aa + (n + 1) * cc, v); ++cnt;
    }
  return cnt;
}

struct CountEmit { __device__ void operator()(int, double) {} };
struct FillEmit {
  int* col; double* val; int64_t base; int k;
  __device__ void operator()(int c, double v) {
    col[base + (int64_t)k * SELL_C] = c; val[base + (int64_t)k * SELL_C] = v; ++k;
  }
};

struct VelFn { VelParams p; template <class E> __device__ int operator()(int r, E& e) const { return vel_row(p, r, e); } };
struct BtFn { BtParams p; template <class E> __device__ int operator()(int r, E& e) const { return bt_row(p, r, e); } };
struct BFn { BParams p; template <class E> __device__ int operator()(int r, E& e) const { return b_row(p, r, e); } };
struct ApFn { ApParams p; template <class E> __device__ int operator()(int r, E& e) const { return ap_row(p, r, e); } };
struct LpFn { LpParams p; template <class E> __device__ int operator()(int r, E& e) const { return lp_row(p, r, e); } };
struct SkFn { SkParams p; template <class E> __device__ int operator()(int r, E& e) const { return sk_row(p, r, e); } };
struct F1Fn { F1Params p; template <class E> __device__ int operator()(int r, E& e) const { return f1_row(p, r, e); } };

template <class Fn>
__global__ void k_sell_count(Fn fn, const int* perm, int64_t nrows, int64_t nslices, int* slen,
                             unsigned long long* nnz) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = t / SELL_C;
  if (s >= nslices) return;
  const int row = perm ? perm[t] : (t < nrows ? (int)t : -1);
  CountEmit ce;
  int len = row >= 0 ? fn(row, ce) : 0;
  int mx = len;
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int tot = len;
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if ((threadIdx.x & 31) == 0) { slen[s] = mx; atomicAdd(nnz, (unsigned long long)tot); }
}

template <class Fn>
__global__ void k_sell_fill(Fn fn, const int* perm, int64_t nrows, int64_t nslices, const int64_t* sptr,
                            const int* slen, int* col, double* val) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = t / SELL_C;
  if (s >= nslices) return;
  const int lane = (int)(t % SELL_C);
  const int row = perm ? perm[t] : (t < nrows ? (int)t : -1);
  FillEmit fe{col, val, sptr[s] + lane, 0};
  if (row >= 0) fn(row, fe);
  for (int k = fe.k; k < slen[s]; ++k) {
    col[sptr[s] + lane + (int64_t)k * SELL_C] = 0;
    val[sptr[s] + lane + (int64_t)k * SELL_C] = 0.0;
  }
}

// exclusive scan of 32 * slen into sptr (single block; setup only)
__global__ void k_scan_slices(const int* slen, int64_t nslices, int64_t* sptr) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t chunk = (nslices + 1023) / 1024;
  const int64_t b = tid * chunk, e = min(nslices, b + chunk);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += (int64_t)slen[i] * SELL_C;
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t acc = 0;
    for (int k = 0; k < 1024; ++k) { int64_t v = part[k]; part[k] = acc; acc += v; }
    sptr[nslices] = acc;
  }
  __syncthreads();
  int64_t acc = part[tid];
  for (int64_t i = b; i < e; ++i) { sptr[i] = acc; acc += (int64_t)slen[i] * SELL_C; }
}

// Row order of the velocity node slices: the grid is swept ONCE in bands of two node rows
// (j = 2b, 2b+1); inside a band the four node classes (i mod 2, j mod 2) form separate row
// segments, each padded to a multiple of 32, so every slice holds nodes of one class and one row
// (uniform stencil width) and the gathered x rows stay L2-resident while the band advances.
// Row order of the velocity node slices.  Class-major: the four node classes (i mod 2, j mod 2)
// one after the other, lexicographic inside a class, so every slice holds rows of one stencil
// width (25 / 15 / 15 / 9).  Band: the grid is swept once in bands of two node rows with the
// four class segments of the band padded to multiples of 32, so the gathered rows stay in L2
// while the band advances.  Measured (variants A/B, n = 1024 / 2048): class-major is faster
// while a two-component vector fits in the L2, band order beyond (etq_band_order).
__host__ __device__ inline int64_t pad32(int64_t v) { return (v + 31) / 32 * 32; }
__global__ void k_node_perm_class(int n, int64_t total, int* perm) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int m = 2 * n + 1;
  const int64_t nq = (int64_t)m * m;
  if (t >= nq) { perm[t] = -1; return; }
  const int64_t cnt[4] = {(int64_t)(n + 1) * (n + 1), (int64_t)n * (n + 1), (int64_t)(n + 1) * n, (int64_t)n * n};
  int c = 0; int64_t idx = t;
  while (idx >= cnt[c]) { idx -= cnt[c]; ++c; }
  const int px = c & 1, py = c >> 1;
  const int cx = px ? n : n + 1;
  const int ix = (int)(idx % cx), iy = (int)(idx / cx);
  perm[t] = (2 * ix + px) + m * (2 * iy + py);
}
__global__ void k_node_perm_band(int n, int64_t total, int* perm) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int m = 2 * n + 1;
  const int64_t pe = pad32(n + 1), po = pad32(n);        // even-i / odd-i segment sizes
  const int64_t band = 2 * (pe + po);
  const int64_t b = t / band;
  int64_t r = t % band;
  int j, i;
  if (r < pe) { j = 2 * (int)b; i = 2 * (int)r; if (r > n) { perm[t] = -1; return; } }
  else if ((r -= pe) < po) { j = 2 * (int)b; i = 2 * (int)r + 1; if (r >= n) { perm[t] = -1; return; } }
  else if ((r -= po) < pe) { j = 2 * (int)b + 1; i = 2 * (int)r; if (r > n) { perm[t] = -1; return; } }
  else { r -= pe; j = 2 * (int)b + 1; i = 2 * (int)r + 1; if (r >= n) { perm[t] = -1; return; } }
  if (j >= m) { perm[t] = -1; return; }
  perm[t] = i + m * j;
}

template <class Fn>
etq_status build_sell(Fn fn, int* perm, int64_t nrows, int64_t nslices, Sell* out, cudaStream_t st) {
  Sell& S = *out;
  S.nrows = nrows; S.nslices = nslices; S.perm = perm;
  ETQ_TRY(dalloc(&S.slen, nslices));
  ETQ_TRY(dalloc(&S.sptr, nslices + 1));
  unsigned long long* dnnz;
  ETQ_TRY(dalloc(&dnnz, 1));
  ETQ_CHECK(cudaMemsetAsync(dnnz, 0, sizeof(unsigned long long), st));
  const int64_t threads = nslices * SELL_C;
  const int bs = 256;
  const int64_t grid = (threads + bs - 1) / bs;
  k_sell_count<<<(unsigned)grid, bs, 0, st>>>(fn, perm, nrows, nslices, S.slen, dnnz); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  k_scan_slices<<<1, 1024, 0, st>>>(S.slen, nslices, S.sptr); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  int64_t total = 0; unsigned long long nnz = 0;
  ETQ_CHECK(cudaMemcpyAsync(&total, S.sptr + nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  ETQ_CHECK(cudaMemcpyAsync(&nnz, dnnz, sizeof(nnz), cudaMemcpyDeviceToHost, st));
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(dnnz);
  S.nnz_stored = total; S.nnz = (int64_t)nnz;
  ETQ_TRY(dalloc(&S.col, total > 0 ? total : 1));
  ETQ_TRY(dalloc(&S.val, total > 0 ? total : 1));
  k_sell_fill<<<(unsigned)grid, bs, 0, st>>>(fn, perm, nrows, nslices, S.sptr, S.slen, S.col, S.val); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

// ---------------------------------------------------------------- diagonal and RHS
__global__ void k_vel_dinv(VelParams P, double* dinv) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= P.g.nq) return;
  const int m = P.g.m, i = node % m, j = node / m;
  dinv[node] = on_boundary(i, j, m) ? 1.0 : 1.0 / vel_entry(P, i, j, i, j);
}

__device__ __forceinline__ double lid_ux(const Geo& g, int bc, int i, int j) {
  if (bc != 0 || j != g.m - 1) return 0.0;
  const double x = -1.0 + i * (g.h * 0.5);
  return 1.0 - x * x * x * x;   // reading R1: tangential lid velocity u_x = 1 - x^4
}

// f rows: boundary -> Dirichlet value; interior -> Galerkin load minus lifting (reading R2, R10)
__global__ void k_rhs_velocity(VelParams P, int bc, const double* f_nodal, double* b) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  const Geo& g = P.g;
  if (node >= g.nq) return;
  const int m = g.m, n = g.n; const double h = g.h;
  const int i = node % m, j = node / m;
  if (on_boundary(i, j, m)) {
    b[node] = lid_ux(g, bc, i, j);
    b[g.nq + node] = 0.0;
    return;
  }
  const int rx = (i & 1) ? 1 : 2, ry = (j & 1) ? 1 : 2;
  double fx = 0.0, fy = 0.0, lift = 0.0;
  for (int dj = -ry; dj <= ry; ++dj) {
    const int jj = j + dj;
    for (int di = -rx; di <= rx; ++di) {
      const int ii = i + di;
      const int col = ii + m * jj;
      if (f_nodal) {
        const double mv = m1(n, h, j, jj) * m1(n, h, i, ii);
        fx += mv * f_nodal[col];
        fy += mv * f_nodal[g.nq + col];
      }
      if (on_boundary(ii, jj, m)) {
        const double u = lid_ux(g, bc, ii, jj);
        if (u != 0.0) lift += vel_entry(P, i, j, ii, jj) * u;
      }
    }
  }
  b[node] = fx - lift;
  b[g.nq + node] = fy;
}

// g rows: -B[:, boundary] u_boundary (only the lid's u_x is non-zero)
__global__ void k_rhs_pressure(Geo g, int bc, double* bp) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= g.nk + g.n0) return;
  const int m = g.m, n = g.n; const double h = g.h;
  double s = 0.0;
  if (bc == 0) {
    const int j = m - 1;
    if (row < g.nk) {
      const int a = row % (n + 1), c = row / (n + 1);
      const double hc = h1(n, h, c, j);
      if (hc != 0.0)
        for (int i = max(0, 2 * a - 2); i <= min(m - 1, 2 * a + 2); ++i) {
          const double u = lid_ux(g, bc, i, j);
          s += -g1(n, a, i) * hc * u;
        }
    } else {
      const int t = row - g.nk, e = t % n, f = t / n;
      const double wf = w1(h, f, j);
      if (wf != 0.0)
        for (int i = 2 * e; i <= 2 * e + 2; ++i) s += -e1(e, i) * wf * lid_ux(g, bc, i, j);
    }
  }
  bp[row] = -s;
}


// max over interior rows of sum_{j != i} |N_ij| / |F_ii| (reading R9': imaginary semi-axis)
__global__ void k_gershgorin_n(VelParams P, unsigned long long* out) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= P.g.nq) return;
  const int m = P.g.m, n = P.g.n; const double h = P.g.h;
  const int i = node % m, j = node / m;
  if (on_boundary(i, j, m)) return;
  const int rx = (i & 1) ? 1 : 2, ry = (j & 1) ? 1 : 2;
  double s = 0.0;
  for (int dj = -ry; dj <= ry; ++dj) {
    const int jj = j + dj;
    if (jj <= 0 || jj >= m - 1) continue;
    for (int di = -rx; di <= rx; ++di) {
      const int ii = i + di;
      if (ii <= 0 || ii >= m - 1 || (di == 0 && dj == 0)) continue;
      s += fabs(osn1(0, n, h, i, ii) * osn1(1, n, h, j, jj) - osn1(1, n, h, i, ii) * osn1(0, n, h, j, jj));
    }
  }
  const double v = s / fabs(vel_entry(P, i, j, i, j));
  atomicMax(out, (unsigned long long)__double_as_longlong(v));
}

__global__ void k_sell_diag_inv(Sell A, double* dinv) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = t / SELL_C;
  if (s >= A.nslices) return;
  const int lane = (int)(t % SELL_C);
  const int row = A.perm ? A.perm[t] : (t < A.nrows ? (int)t : -1);
  if (row < 0) return;
  double d = 0.0;
  for (int k = 0; k < A.slen[s]; ++k) {
    const int64_t e = A.sptr[s] + lane + (int64_t)k * SELL_C;
    if (A.col[e] == row && A.val[e] != 0.0) d = A.val[e];
  }
  dinv[row] = 1.0 / d;
}
// A slice is implicit when every lane holds a row of the same node class whose stored columns are
// exactly row + off[class][k] (the full interior stencil in enumeration order).
// reference values of the interior rows of each node class (node (4 + px, 4 + py))
struct RefEmit {
  double* out; int k;
  __device__ void operator()(int, double v) { out[k++] = v; }
};
__global__ void k_ref_values(VelParams P, double* stval) {
  const int c = threadIdx.x;
  if (c >= 4) return;
  const int px = c & 1, py = c >> 1;
  RefEmit e{stval + c * 32, 0};
  vel_row(P, (4 + px) + P.g.m * (4 + py), e);
}

__global__ void k_mark_implicit(Sell S, const int* off, const int* len, const double* stval, int8_t* skind,
                                unsigned long long* nimp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = t / SELL_C;
  if (s >= S.nslices) return;
  const int lane = (int)(t % SELL_C);
  const int row = S.perm[t];
  int cls = -1;
  bool ok = row >= 0, vok = ok && stval != nullptr;
  const int m = len[4];                       // nodes per grid row
  if (ok) {
    const int i = row % m, j = row / m;
    cls = (i & 1) + 2 * (j & 1);
    ok = S.slen[s] == len[cls];
    for (int k = 0; ok && k < len[cls]; ++k) {
      const int64_t e = S.sptr[s] + lane + (int64_t)k * SELL_C;
      if (S.col[e] != row + off[cls * 32 + k] || S.val[e] == 0.0) ok = false;
      if (vok && S.val[e] != stval[cls * 32 + k]) vok = false;
    }
  }
  const int c0 = __shfl_sync(0xffffffffu, cls, 0);
  const bool all = __all_sync(0xffffffffu, ok && cls == c0);
  const bool allv = __all_sync(0xffffffffu, ok && vok && cls == c0);
  if (lane == 0) {
    skind[s] = allv ? (int8_t)(c0 + 5) : (all ? (int8_t)(c0 + 1) : (int8_t)0);
    if (all) atomicAdd(nimp, (unsigned long long)SELL_C * len[c0]);
    if (allv) atomicAdd(nimp + 1, (unsigned long long)SELL_C * len[c0]);
  }
}

}  // namespace

// ---------------------------------------------------------------- host entry points
bool etq_band_order(const Geo& g) {
  return 2.0 * 8.0 * (double)g.nq > 126.0e6;   // two-component vector larger than the 126 MB L2
}

etq_status build_node_perm(const Geo& g, int** perm, int64_t* nslices, cudaStream_t st) {
  const bool band = etq_band_order(g);
  const int64_t ns = band ? (2 * (pad32(g.n + 1) + pad32(g.n)) * (g.n + 1)) / SELL_C   // last odd row: padding
                          : ((int64_t)g.nq + SELL_C - 1) / SELL_C;
  ETQ_TRY(dalloc(perm, ns * SELL_C));
  const int64_t tot = ns * SELL_C;
  if (band) k_node_perm_band<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g.n, tot, *perm);
  else k_node_perm_class<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g.n, tot, *perm);
  etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  *nslices = ns;
  return ETQ_OK;
}

etq_status assemble_velocity_op(const Geo& g, bool oseen, double nu, int wind, int* perm,
                                int64_t nslices, Sell* out, cudaStream_t st) {
  VelFn fn{VelParams{g, oseen ? (wind == 1 ? 1 : 2) : 0, oseen ? nu : 1.0}};
  return build_sell(fn, perm, g.nq, nslices, out, st);
}

etq_status assemble_bt(const Geo& g, int comp, int part, int* perm, int64_t nslices, Sell* out,
                       cudaStream_t st) {
  BtFn fn{BtParams{g, comp, part}};
  return build_sell(fn, perm, g.nq, nslices, out, st);
}

etq_status assemble_b(const Geo& g, Sell* out, cudaStream_t st) {
  BFn fn{BParams{g}};
  const int64_t nrows = (int64_t)g.nk + g.n0;
  return build_sell(fn, nullptr, nrows, (nrows + SELL_C - 1) / SELL_C, out, st);
}

etq_status velocity_dinv_dev(const Geo& g, bool oseen, double nu, int wind, double* dinv, cudaStream_t st) {
  VelParams P{g, oseen ? (wind == 1 ? 1 : 2) : 0, oseen ? nu : 1.0};
  k_vel_dinv<<<(g.nq + 255) / 256, 256, 0, st>>>(P, dinv); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status build_rhs_dev(const Problem& P, const double* f_nodal, double* b) {
  VelParams vp{P.g, P.oseen ? (P.wind == 1 ? 1 : 2) : 0, P.oseen ? P.nu : 1.0};
  k_rhs_velocity<<<(P.g.nq + 255) / 256, 256, 0, P.stream>>>(vp, P.bc, f_nodal, b); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  k_rhs_pressure<<<(unsigned)((P.n_p + 255) / 256), 256, 0, P.stream>>>(P.g, P.bc, b + P.n_u); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  if (P.oseen && P.wind == 2) ETQ_TRY(picard_rhs_convection(P, b));   // - N(w)[:, boundary] u_boundary
  return ETQ_OK;
}

etq_status oseen_gershgorin(const Geo& g, double nu, int wind, double* bim, cudaStream_t st) {
  if (wind == 2) { *bim = 0.0; return ETQ_OK; }   // nodal wind: picard.cu recomputes it from the values
  VelParams P{g, wind == 1 ? 1 : 0, nu};
  unsigned long long* d;
  ETQ_TRY(dalloc(&d, 1));
  ETQ_CHECK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
  k_gershgorin_n<<<(g.nq + 255) / 256, 256, 0, st>>>(P, d); etq_count_launch();
  unsigned long long hv = 0;
  ETQ_CHECK(cudaMemcpyAsync(&hv, d, sizeof(hv), cudaMemcpyDeviceToHost, st));
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(d);
  double v;
  std::memcpy(&v, &hv, sizeof(v));
  *bim = v;
  return ETQ_OK;
}

etq_status assemble_ap(const Geo& g, Sell* out, cudaStream_t st) {
  ApFn fn{ApParams{g}};
  return build_sell(fn, nullptr, g.nk, ((int64_t)g.nk + SELL_C - 1) / SELL_C, out, st);
}

etq_status assemble_lp(const Geo& g, Sell* out, cudaStream_t st) {
  LpFn fn{LpParams{g}};
  const int64_t nr = (int64_t)g.nk + g.n0;
  return build_sell(fn, nullptr, nr, (nr + SELL_C - 1) / SELL_C, out, st);
}

etq_status velocity_mdiag_inv(const Geo& g, double* out, cudaStream_t st) {
  k_vel_mdiag_inv<<<(g.nq + 255) / 256, 256, 0, st>>>(g, out); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status assemble_sk(const Geo& g, double scale, Sell* out, cudaStream_t st) {
  SkFn fn{SkParams{g, scale}};
  return build_sell(fn, nullptr, g.nk, ((int64_t)g.nk + SELL_C - 1) / SELL_C, out, st);
}

etq_status assemble_f1(const Geo& g, double nu, int wind, Sell* out, cudaStream_t st) {
  F1Fn fn{F1Params{g, nu, wind}};
  return build_sell(fn, nullptr, g.nk, ((int64_t)g.nk + SELL_C - 1) / SELL_C, out, st);
}

etq_status sell_diag_inv(const Sell& A, double* dinv, cudaStream_t st) {
  k_sell_diag_inv<<<(unsigned)((A.nslices * SELL_C + 255) / 256), 256, 0, st>>>(A, dinv); etq_count_launch();
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

// Per-class interior stencil offsets in vel_row's enumeration order (dj outer, di inner), then
// mark the slices whose stored columns follow them (implicit column indices in the kernels).
etq_status mark_implicit(const Geo& g, bool oseen, double nu, int wind, Sell& S, cudaStream_t st, bool values) {
  if (!S.perm) return ETQ_OK;
  std::vector<int> off(4 * 32, 0), len(5, 0);
  for (int c = 0; c < 4; ++c) {
    const int px = c & 1, py = c >> 1, rx = px ? 1 : 2, ry = py ? 1 : 2;
    int k = 0;
    for (int dj = -ry; dj <= ry; ++dj)
      for (int di = -rx; di <= rx; ++di) {
        if (!oseen) {
          if ((di == 2 || di == -2) && dj == 0 && py) continue;
          if ((dj == 2 || dj == -2) && di == 0 && px) continue;
        }
        off[c * 32 + k++] = di + g.m * dj;
      }
    len[c] = k;
  }
  len[4] = g.m;
  int* dlen;
  unsigned long long* dn;
  ETQ_TRY(dalloc(&S.stoff, 4 * 32));
  ETQ_TRY(dalloc(&dlen, 5));
  ETQ_TRY(dalloc(&S.skind, S.nslices));
  ETQ_TRY(dalloc(&dn, 2));
  ETQ_CHECK(cudaMemcpyAsync(S.stoff, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice, st));
  ETQ_CHECK(cudaMemcpyAsync(dlen, len.data(), sizeof(int) * len.size(), cudaMemcpyHostToDevice, st));
  ETQ_CHECK(cudaMemsetAsync(dn, 0, 2 * sizeof(unsigned long long), st));
  // value dictionary only for the translation-invariant Stokes operator (n >= 4)
  if (values && !oseen && g.n >= 4) {
    ETQ_TRY(dalloc(&S.stval, 4 * 32));
    ETQ_CHECK(cudaMemsetAsync(S.stval, 0, sizeof(double) * 4 * 32, st));
    VelParams P{g, 0, 1.0};
    k_ref_values<<<1, 32, 0, st>>>(P, S.stval); etq_count_launch();
  }
  (void)nu; (void)wind;
  k_mark_implicit<<<(unsigned)((S.nslices * SELL_C + 255) / 256), 256, 0, st>>>(S, S.stoff, dlen, S.stval, S.skind, dn);
  etq_count_launch();
  unsigned long long h[2] = {0, 0};
  ETQ_CHECK(cudaMemcpyAsync(h, dn, sizeof(h), cudaMemcpyDeviceToHost, st));
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(dlen); cudaFree(dn);
  S.nnz_implicit = (int64_t)h[0];
  S.nnz_implicit_vals = (int64_t)h[1];
  return ETQ_OK;
}

// Interior stencil of a Stokes level: rectangle [4, m-5]^2, per-class weights
// from the verified value dictionary, and a SELL over the remaining (frame) rows.
// B / B^T weights at deep-interior reference positions (the same 1-D table products as bt_row / b_row;
// every non-Dirichlet row equals them, so the saddle operator can be applied matrix-free)
__global__ void k_saddle_weights(Geo g, SaddleSt* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = g.n; const double h = g.h;
  const int r = n / 2;
  for (int c = 0; c < 4; ++c) {
    const int i = 2 * r + (c & 1), j = 2 * r + (c >> 1);
    for (int dc = -1; dc <= 1; ++dc)
      for (int da = -1; da <= 1; ++da) {
        const int a = i / 2 + da, cc = j / 2 + dc;
        out->bt1[c][0][(dc + 1) * 3 + da + 1] = -g1(n, a, i) * h1(n, h, cc, j);
        out->bt1[c][1][(dc + 1) * 3 + da + 1] = -h1(n, h, a, i) * g1(n, cc, j);
      }
    for (int df = -1; df <= 0; ++df)
      for (int de = -1; de <= 0; ++de) {
        const int e = i / 2 + de, f = j / 2 + df;
        out->bt0[c][0][(df + 1) * 2 + de + 1] = -e1(e, i) * w1(h, f, j);
        out->bt0[c][1][(df + 1) * 2 + de + 1] = -w1(h, e, i) * e1(f, j);
      }
  }
  for (int dj = -2; dj <= 2; ++dj) {
    const int jj = 2 * r + dj;
    const double hc = h1(n, h, r, jj), gc = g1(n, r, jj);
    for (int di = -2; di <= 2; ++di) {
      const int ii = 2 * r + di;
      out->b1[0][(dj + 2) * 5 + di + 2] = -g1(n, r, ii) * hc;
      out->b1[1][(dj + 2) * 5 + di + 2] = -h1(n, h, r, ii) * gc;
    }
  }
  for (int dj = 0; dj <= 2; ++dj)
    for (int di = 0; di <= 2; ++di) {
      const int ii = 2 * r + di, jj = 2 * r + dj;
      out->b0[0][dj * 3 + di] = -e1(r, ii) * w1(h, r, jj);
      out->b0[1][dj * 3 + di] = -w1(h, r, ii) * e1(r, jj);
    }
}

etq_status saddle_weights(const Geo& g, SaddleSt* out, cudaStream_t st) {
  SaddleSt* d;
  ETQ_TRY(dalloc(&d, 1));
  k_saddle_weights<<<1, 32, 0, st>>>(g, d); etq_count_launch();
  ETQ_CHECK(cudaMemcpyAsync(out, d, sizeof(SaddleSt), cudaMemcpyDeviceToHost, st));
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(d);
  return ETQ_OK;
}

// class stencil w[4][25] of a Stokes velocity operator from its per-class dictionary (stval)
etq_status class_weights(const Geo& g, const Sell& A, StencilOp* so) {
  if (!A.stval || !A.stoff) return ETQ_EINVAL;
  std::vector<double> sv(4 * 32);
  ETQ_CHECK(cudaMemcpy(sv.data(), A.stval, sizeof(double) * sv.size(), cudaMemcpyDeviceToHost));
  StencilOp o;
  o.m = g.m; o.lo = 4; o.hi = g.m - 5;
  for (int c = 0; c < 4; ++c) {
    for (int t = 0; t < 25; ++t) o.w[c][t] = 0.0;
    const int px = c & 1, py = c >> 1, rx = px ? 1 : 2, ry = py ? 1 : 2;
    int k = 0;
    for (int dj = -ry; dj <= ry; ++dj)
      for (int di = -rx; di <= rx; ++di) {   // Stokes enumeration of vel_row (cancelled taps dropped)
        if ((di == 2 || di == -2) && dj == 0 && py) continue;
        if ((dj == 2 || dj == -2) && di == 0 && px) continue;
        o.w[c][(dj + 2) * 5 + (di + 2)] = sv[c * 32 + k++];
      }
  }
  *so = o;
  return ETQ_OK;
}

// Oseen levels with the separable cavity wind (oseen == 1, reading R9'): F_s = nu L + N with
// N((i,j),(i',j')) = A1(i,i') T2(j,j') - T2(i,i') A1(j,j') (the 1D tables of the file header).  The
// interior rows are applied matrix-free: nu times the (h-independent) Stokes class stencil plus the
// convection weights formed from two 1D tables per node index, tab[0][5 i + d] = A1(i, i + d - 2)
// and tab[1][5 i + d] = T2(i, i + d - 2); frame rows keep stored SELL rows.
namespace {
__global__ void k_oseen_tabs(Geo g, double nu, double* w, double* tab) {
  const int n = g.n, m = g.m;
  const double h = g.h;
  const int tot = 100 + 5 * m;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
    if (t < 100) {   // nu L class stencil at an interior reference node of class c
      const int c = t / 25, k = t % 25, dj = k / 5 - 2, di = k % 5 - 2;
      const int i = 4 + (c & 1), j = 4 + (c >> 1);
      w[t] = nu * (m1(n, h, j, j + dj) * k1(n, h, i, i + di) + k1(n, h, j, j + dj) * m1(n, h, i, i + di));
    } else {
      const int q = t - 100, i = q / 5, ii = i + q % 5 - 2;
      const bool ok = ii >= 0 && ii < m;
      tab[q] = ok ? osn1(0, n, h, i, ii) : 0.0;
      tab[5 * m + q] = ok ? osn1(1, n, h, i, ii) : 0.0;
    }
  }
}
}  // namespace

// nu L class stencils (so->w) and the 1D convection tables of the cavity wind on grid g
etq_status oseen_tables(const Geo& g, double nu, StencilOp* so, double** tab, cudaStream_t st) {
  StencilOp o;
  o.m = g.m; o.lo = 4; o.hi = g.m - 5;
  o.nseg_x = (o.hi - o.lo + 1 + 31) / 32;
  o.nseg = (int64_t)o.nseg_x * (o.hi - o.lo + 1);
  double* dw;
  ETQ_TRY(dalloc(&dw, 100));
  ETQ_TRY(dalloc(tab, (size_t)10 * g.m));
  k_oseen_tabs<<<(100 + 5 * g.m + 255) / 256, 256, 0, st>>>(g, nu, dw, *tab); etq_count_launch();
  ETQ_CHECK(cudaMemcpyAsync(&o.w[0][0], dw, sizeof(double) * 100, cudaMemcpyDeviceToHost, st));
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(dw);
  *so = o;
  return ETQ_OK;
}

etq_status build_oseen_stencil_level(const Geo& g, double nu, StencilOp* so, Sell* frame, double** tab,
                                     cudaStream_t st) {
  if (g.n < 16) return ETQ_EINVAL;
  StencilOp o;
  ETQ_TRY(oseen_tables(g, nu, &o, tab, st));
  std::vector<int> rows;
  for (int c = 0; c < 4; ++c)
    for (int j = (c >> 1); j < g.m; j += 2)
      for (int i = (c & 1); i < g.m; i += 2)
        if (i < o.lo || i > o.hi || j < o.lo || j > o.hi) rows.push_back(i + g.m * j);
  const int64_t ns = ((int64_t)rows.size() + SELL_C - 1) / SELL_C;
  rows.resize(ns * SELL_C, -1);
  int* perm;
  ETQ_TRY(dalloc(&perm, rows.size()));
  ETQ_CHECK(cudaMemcpy(perm, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
  VelFn fn{VelParams{g, 1, nu}};
  ETQ_TRY(build_sell(fn, perm, g.nq, ns, frame, st));
  frame->own_perm = true;
  *so = o;
  return ETQ_OK;
}

etq_status build_stencil_level(const Geo& g, const Sell& A, StencilOp* so, Sell* frame, cudaStream_t st) {
  if (!A.stval || !A.stoff || g.n < 16) return ETQ_EINVAL;
  std::vector<double> sv(4 * 32);
  ETQ_CHECK(cudaMemcpy(sv.data(), A.stval, sizeof(double) * sv.size(), cudaMemcpyDeviceToHost));
  StencilOp o;
  o.m = g.m; o.lo = 4; o.hi = g.m - 5;
  o.nseg_x = (o.hi - o.lo + 1 + 31) / 32;
  o.nseg = (int64_t)o.nseg_x * (o.hi - o.lo + 1);
  for (int c = 0; c < 4; ++c) {
    for (int t = 0; t < 25; ++t) o.w[c][t] = 0.0;
    const int px = c & 1, py = c >> 1, rx = px ? 1 : 2, ry = py ? 1 : 2;
    int k = 0;
    for (int dj = -ry; dj <= ry; ++dj)
      for (int di = -rx; di <= rx; ++di) {   // Stokes enumeration of vel_row (cancelled taps dropped)
        if ((di == 2 || di == -2) && dj == 0 && py) continue;
        if ((dj == 2 || dj == -2) && di == 0 && px) continue;
        o.w[c][(dj + 2) * 5 + (di + 2)] = sv[c * 32 + k++];
      }
  }
  // frame rows, class-major
  std::vector<int> rows;
  for (int c = 0; c < 4; ++c)
    for (int j = (c >> 1); j < g.m; j += 2)
      for (int i = (c & 1); i < g.m; i += 2)
        if (i < o.lo || i > o.hi || j < o.lo || j > o.hi) rows.push_back(i + g.m * j);
  const int64_t ns = ((int64_t)rows.size() + SELL_C - 1) / SELL_C;
  rows.resize(ns * SELL_C, -1);
  int* perm;
  ETQ_TRY(dalloc(&perm, rows.size()));
  ETQ_CHECK(cudaMemcpy(perm, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
  VelFn fn{VelParams{g, 0, 1.0}};
  ETQ_TRY(build_sell(fn, perm, g.nq, ns, frame, st));
  frame->own_perm = true;
  *so = o;
  return ETQ_OK;
}
