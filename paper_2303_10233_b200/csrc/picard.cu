// picard.cu — SURVEY §8(f) NEXT-3: Oseen systems with a nodal Q2 wind (the previous Picard
// iterate) and the Picard outer loop of the steady Navier–Stokes cavity ("5
// fixed-point iterations of the discretised Navier-Stokes system starting from the
// corresponding Stokes flow solution").
//
// A problem assembled with wind kind 2 stores F_s = nu L (explicit SELL, full 25/15/15/9 pattern)
// until etq_set_wind gives it a wind w_h in Q2; the convection N(w_h)_ij = int (w_h . grad phi_j)
// phi_i is then added on every MG level (coarse winds by injection at the nested Q2 nodes):
//   1. k_conv_local: per square, the 9 x 9 local matrix with 4 x 4 Gauss points (the integrand is
//      a degree-6 polynomial per direction for a Q2 wind; exact, pinned in the oracle);
//   2. k_fill_nodal: every stored entry F_pq = nu L_pq + sum over the squares containing p and q
//      (ascending square index) of the local entries; Dirichlet rows stay identity rows;
//   3. D^-1, the smoother ellipse's Gershgorin semi-axis b = max_i sum_{j!=i} |N_ij| / |F_ii|
//      (reading R9'), the coarse pivoted inverse and the tail coefficients are recomputed;
//   4. with PCD set up, F1 (Q1, natural boundary, reading R13) is refilled the same way.
// The lifting of the boundary data gains - N(w_h)[:, boundary] u_boundary (picard_rhs_convection).
#include "etq_internal.cuh"
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>
#include "device_common.cuh"

using namespace etqd;

namespace {

// 4-point Gauss–Legendre on [0, 1]
__device__ __forceinline__ void gauss4(double* x, double* w) {
  const double a = sqrt(3.0 / 7.0 - 2.0 / 7.0 * sqrt(6.0 / 5.0)), b = sqrt(3.0 / 7.0 + 2.0 / 7.0 * sqrt(6.0 / 5.0));
  const double wa = (18.0 + sqrt(30.0)) / 72.0, wb = (18.0 - sqrt(30.0)) / 72.0;
  x[0] = 0.5 - 0.5 * b; x[1] = 0.5 - 0.5 * a; x[2] = 0.5 + 0.5 * a; x[3] = 0.5 + 0.5 * b;
  w[0] = wb; w[1] = wa; w[2] = wa; w[3] = wb;
}
// quadratic Lagrange basis on {0, 1/2, 1} and derivative; linear on {0, 1}
__device__ __forceinline__ double q2v(int a, double t) {
  return a == 0 ? 2.0 * (t - 0.5) * (t - 1.0) : (a == 1 ? 4.0 * t * (1.0 - t) : 2.0 * t * (t - 0.5));
}
__device__ __forceinline__ double q2d(int a, double t) { return a == 0 ? 4.0 * t - 3.0 : (a == 1 ? 4.0 - 8.0 * t : 4.0 * t - 1.0); }
__device__ __forceinline__ double q1v(int a, double t) { return a == 0 ? 1.0 - t : t; }
__device__ __forceinline__ double q1d(int a) { return a == 0 ? -1.0 : 1.0; }

// Local convection matrices (Q2 test/trial, Q2 wind) of every square: nloc[e][i][j], 81 per square.
// One thread per (square, test function i).
__global__ void k_conv_local(Geo g, const double* __restrict__ wind, double* __restrict__ nloc) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = g.n, m = g.m, nq = g.nq;
  if (t >= (int64_t)n * n * 9) return;
  const int i = (int)(t % 9);
  const int64_t el = t / 9;
  const int e = (int)(el % n), f = (int)(el / n);
  const double h = g.h;
  double gx[4], gw[4];
  gauss4(gx, gw);
  // wind at the local nodes
  double wx[9], wy[9];
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int node = (2 * e + a) + m * (2 * f + b);
      wx[a + 3 * b] = wind[node]; wy[a + 3 * b] = wind[nq + node];
    }
  const int ia = i % 3, ib = i / 3;
  double acc[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) acc[j] = 0.0;
  for (int qy = 0; qy < 4; ++qy)
    for (int qx = 0; qx < 4; ++qx) {
      const double xi = gx[qx], eta = gx[qy], W = gw[qx] * gw[qy] * h * h;
      double vx[3], vy[3], dx[3], dy[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) { vx[a] = q2v(a, xi); vy[a] = q2v(a, eta); dx[a] = q2d(a, xi) / h; dy[a] = q2d(a, eta) / h; }
      double wqx = 0.0, wqy = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double p = vx[a] * vy[b];
          wqx += wx[a + 3 * b] * p; wqy += wy[a + 3 * b] * p;
        }
      const double phi_i = vx[ia] * vy[ib];
#pragma unroll
      for (int jb = 0; jb < 3; ++jb)
#pragma unroll
        for (int ja = 0; ja < 3; ++ja)
          acc[ja + 3 * jb] += W * (wqx * dx[ja] * vy[jb] + wqy * vx[ja] * dy[jb]) * phi_i;
    }
  double* out = nloc + el * 81 + i * 9;
#pragma unroll
  for (int j = 0; j < 9; ++j) out[j] = acc[j];
}

// Sum of the local entries (p, q) over the squares containing both Q2 nodes, ascending square index.
__device__ __forceinline__ double conv_entry(const Geo& g, const double* __restrict__ nloc, int i, int j, int ii, int jj) {
  const int n = g.n;
  double s = 0.0;
  for (int f = max(0, (max(j, jj) - 2 + 1) / 2); f <= min(n - 1, min(j, jj) / 2); ++f) {
    if (2 * f > min(j, jj) || 2 * f + 2 < max(j, jj)) continue;
    for (int e = max(0, (max(i, ii) - 2 + 1) / 2); e <= min(n - 1, min(i, ii) / 2); ++e) {
      if (2 * e > min(i, ii) || 2 * e + 2 < max(i, ii)) continue;
      const int lp = (i - 2 * e) + 3 * (j - 2 * f), lq = (ii - 2 * e) + 3 * (jj - 2 * f);
      s += nloc[((int64_t)e + (int64_t)n * f) * 81 + lp * 9 + lq];
    }
  }
  return s;
}

// F values of an explicit SELL (node-permuted rows): F = nu L + N(w) with nu L the values the
// level was assembled with (kept in lap); Dirichlet rows stay identity rows.  The row's entries are
// re-enumerated in assemble.cu's vel_row order (full Oseen pattern, Dirichlet columns dropped), so
// entry k of the row is slot k (padding slots untouched).
__global__ void k_fill_nodal(Sell A, const double* __restrict__ lap, Geo g, const double* __restrict__ nloc,
                             unsigned long long* gersh) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = t / SELL_C;
  if (s >= A.nslices) return;
  const int lane = (int)(t % SELL_C);
  const int row = A.perm[s * SELL_C + lane];
  if (row < 0) return;
  const int m = g.m;
  const int i = row % m, j = row / m;
  if (i == 0 || j == 0 || i == m - 1 || j == m - 1) return;   // identity row
  const int rx = (i & 1) ? 1 : 2, ry = (j & 1) ? 1 : 2;
  int k = 0;
  double off = 0.0, diag = 0.0;
  for (int dj = -ry; dj <= ry; ++dj) {
    const int jj = j + dj;
    if (jj <= 0 || jj >= m - 1) continue;
    for (int di = -rx; di <= rx; ++di) {
      const int ii = i + di;
      if (ii <= 0 || ii >= m - 1) continue;
      const int64_t idx = A.sptr[s] + (int64_t)k * SELL_C + lane;
      const double c = conv_entry(g, nloc, i, j, ii, jj);
      const double v = lap[idx] + c;
      A.val[idx] = v;
      if (di == 0 && dj == 0) diag = v; else off += fabs(c);
      ++k;
    }
  }
  // Gershgorin semi-axis of D^-1 N (reading R9'): max over rows of sum_{j != i} |N_ij| / |F_ii|
  if (gersh) atomicMax(gersh, (unsigned long long)__double_as_longlong(off / fabs(diag)));
}

__global__ void k_wind_inject(const double* wf, int mf, int nqf, double* wc, int mc, int nqc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nqc) return;
  const int I = t % mc, J = t / mc;
  const int64_t f = (int64_t)(2 * I) + (int64_t)mf * (2 * J);
  wc[t] = wf[f]; wc[nqc + t] = wf[nqf + f];
}

// b[p] -= sum over boundary nodes b of N(w)_pb u_b (the lid's u_x; the other data are 0)
__global__ void k_rhs_conv(Geo g, int bc, const double* __restrict__ nloc, double* b) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= g.nq || bc != 0) return;
  const int m = g.m;
  const int i = node % m, j = node / m;
  if (i == 0 || j == 0 || i == m - 1 || j == m - 1) return;
  if (j < m - 3) return;                                       // only rows coupled to the lid y = 1
  const double hh = g.h * 0.5;
  double lift = 0.0;
  const int jj = m - 1;
  for (int ii = max(0, i - 2); ii <= min(m - 1, i + 2); ++ii) {
    const double x = -1.0 + ii * hh;
    const double u = 1.0 - x * x * x * x;                      // reading R1
    if (u != 0.0) lift += conv_entry(g, nloc, i, j, ii, jj) * u;
  }
  b[node] -= lift;
}

// ---- Q1 (PCD F1) with a Q2 wind: local 4 x 4 convection per square, 4 x 4 Gauss points
__global__ void k_conv_local_q1(Geo g, const double* __restrict__ wind, double* __restrict__ nloc1) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = g.n, m = g.m, nq = g.nq;
  if (t >= (int64_t)n * n * 4) return;
  const int i = (int)(t % 4);
  const int64_t el = t / 4;
  const int e = (int)(el % n), f = (int)(el / n);
  const double h = g.h;
  double gx[4], gw[4];
  gauss4(gx, gw);
  double wx[9], wy[9];
  for (int b = 0; b < 3; ++b)
    for (int a = 0; a < 3; ++a) {
      const int node = (2 * e + a) + m * (2 * f + b);
      wx[a + 3 * b] = wind[node]; wy[a + 3 * b] = wind[nq + node];
    }
  const int ia = i % 2, ib = i / 2;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int qy = 0; qy < 4; ++qy)
    for (int qx = 0; qx < 4; ++qx) {
      const double xi = gx[qx], eta = gx[qy], W = gw[qx] * gw[qy] * h * h;
      double wqx = 0.0, wqy = 0.0;
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
          const double p = q2v(a, xi) * q2v(b, eta);
          wqx += wx[a + 3 * b] * p; wqy += wy[a + 3 * b] * p;
        }
      const double psi_i = q1v(ia, xi) * q1v(ib, eta);
      for (int jb = 0; jb < 2; ++jb)
        for (int ja = 0; ja < 2; ++ja)
          acc[ja + 2 * jb] += W * (wqx * q1d(ja) / h * q1v(jb, eta) + wqy * q1v(ja, xi) * q1d(jb) / h) * psi_i;
    }
  double* out = nloc1 + el * 16 + i * 4;
  for (int j = 0; j < 4; ++j) out[j] = acc[j];
}

// F1 values (natural row order, 9-point rows in assemble.cu's f1_row order): the diffusion values
// F1 was assembled with (lap) plus the local convection entries of the squares containing both
__global__ void k_fill_f1_nodal(Sell A, const double* __restrict__ lap, Geo g, const double* __restrict__ nloc1) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = t / SELL_C;
  if (s >= A.nslices) return;
  const int lane = (int)(t % SELL_C);
  const int64_t r = s * SELL_C + lane;
  if (r >= A.nrows) return;
  const int n = g.n, n1 = n + 1;
  const int a = (int)(r % n1), c = (int)(r / n1);
  int k = 0;
  for (int cc = max(0, c - 1); cc <= min(n, c + 1); ++cc)
    for (int aa = max(0, a - 1); aa <= min(n, a + 1); ++aa) {
      const int64_t idx = A.sptr[s] + (int64_t)k * SELL_C + lane;
      double v = lap[idx];
      for (int f = max(0, max(c, cc) - 1); f <= min(n - 1, min(c, cc)); ++f)
        for (int e = max(0, max(a, aa) - 1); e <= min(n - 1, min(a, aa)); ++e) {
          const int lp = (a - e) + 2 * (c - f), lq = (aa - e) + 2 * (cc - f);
          v += nloc1[((int64_t)e + (int64_t)n * f) * 16 + lp * 4 + lq];
        }
      A.val[idx] = v;
      ++k;
    }
}

}  // namespace

// keep the values a wind-kind-2 operator was assembled with (nu L, or F1's diffusion)
static etq_status keep_lap(const Sell& A, double** lap, cudaStream_t st) {
  if (*lap) return ETQ_OK;
  ETQ_TRY(dalloc(lap, (size_t)A.nnz_stored));
  ETQ_CHECK(cudaMemcpyAsync(*lap, A.val, sizeof(double) * A.nnz_stored, cudaMemcpyDeviceToDevice, st));
  return ETQ_OK;
}

static etq_status fill_level(const Geo& g, Sell& A, double** lap, double* dinv, const double* wind, double* nloc,
                             double* bim, bool need_bim, cudaStream_t st) {
  ETQ_TRY(keep_lap(A, lap, st));
  const int64_t nt = (int64_t)g.n * g.n * 9;
  k_conv_local<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(g, wind, nloc); etq_count_launch();
  const int64_t slots = A.nslices * SELL_C;
  unsigned long long* d = nullptr;
  if (need_bim) {
    ETQ_TRY(dalloc(&d, 1));
    ETQ_CHECK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
  }
  k_fill_nodal<<<(unsigned)((slots + 255) / 256), 256, 0, st>>>(A, *lap, g, nloc, d); etq_count_launch();
  if (dinv) ETQ_TRY(sell_diag_inv(A, dinv, st));
  if (need_bim) {
    unsigned long long hv = 0;
    ETQ_CHECK(cudaMemcpyAsync(&hv, d, sizeof(hv), cudaMemcpyDeviceToHost, st));
    ETQ_CHECK(cudaStreamSynchronize(st));
    cudaFree(d);
    std::memcpy(bim, &hv, sizeof(double));
  }
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

// Refill every operator that depends on the nodal wind (P.wnod): level-0 F (P.Lv), the MG levels,
// their D^-1, Gershgorin semi-axes, coarse inverse and tail coefficients, and F1 if PCD is set up.
etq_status picard_refresh(Problem& P) {
  if (!(P.oseen && P.wind == 2) || !P.wnod) return ETQ_OK;
  cudaStream_t st = P.stream;
  double* nloc;
  ETQ_TRY(dalloc(&nloc, (size_t)81 * P.g.n * P.g.n));
  double dummy = 0.0;
  if (!P.mg.built) {
    etq_status s = fill_level(P.g, P.Lv, &P.lv_lap, nullptr, P.wnod, nloc, &dummy, false, st);
    if (s < 0) { cudaFree(nloc); return s; }
  } else {
    Hierarchy& H = P.mg;
    const int L = (int)H.lv.size();
    for (int l = 0; l < L; ++l) {
      Level& lv = H.lv[l];
      const double* w = P.wnod;
      if (l > 0) {
        if (!lv.wind) ETQ_TRY(dalloc(&lv.wind, 2 * (size_t)lv.g.nq));
        const Level& fv = H.lv[l - 1];
        const double* wf = l == 1 ? P.wnod : fv.wind;
        k_wind_inject<<<(lv.g.nq + 255) / 256, 256, 0, st>>>(wf, fv.g.m, fv.g.nq, lv.wind, lv.g.m, lv.g.nq);
        etq_count_launch();
        w = lv.wind;
      }
      ETQ_TRY(fill_level(lv.g, lv.A, l == 0 ? &P.lv_lap : &lv.lapval, lv.dinv, w, nloc, &lv.bim, l + 1 < L, st));
    }
    Level& C = H.lv.back();
    ETQ_TRY(dense_from_sell(C.A, C.g.nq, C.coarse_inv, st));
    ETQ_TRY(dense_inverse_pivot(C.coarse_inv, C.g.nq, st));
    ETQ_TRY(refresh_tail(H));
  }
  if (P.F1.val) {
    double* nl1;
    ETQ_TRY(dalloc(&nl1, (size_t)16 * P.g.n * P.g.n));
    const int64_t nt = (int64_t)P.g.n * P.g.n * 4;
    k_conv_local_q1<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(P.g, P.wnod, nl1); etq_count_launch();
    const int64_t slots = P.F1.nslices * SELL_C;
    ETQ_TRY(keep_lap(P.F1, &P.f1_lap, st));
    k_fill_f1_nodal<<<(unsigned)((slots + 255) / 256), 256, 0, st>>>(P.F1, P.f1_lap, P.g, nl1); etq_count_launch();
    ETQ_CHECK(cudaStreamSynchronize(st));
    cudaFree(nl1);
  }
  ETQ_CHECK(cudaStreamSynchronize(st));
  cudaFree(nloc);
  // captured solver graphs bake in the Chebyshev coefficients (semi-axes changed)
  if (P.gmres_graph) { cudaGraphExecDestroy(P.gmres_graph); P.gmres_graph = nullptr; }
  P.gmres_graph_key = -1;
  return ETQ_OK;
}

etq_status picard_set_wind(Problem& P, const double* w) {
  if (!(P.oseen && P.wind == 2)) return ETQ_EINVAL;
  if (!P.wnod) ETQ_TRY(dalloc(&P.wnod, (size_t)P.n_u));
  ETQ_CHECK(cudaMemcpyAsync(P.wnod, w, sizeof(double) * P.n_u, cudaMemcpyDeviceToDevice, P.stream));
  return picard_refresh(P);
}

etq_status picard_rhs_convection(const Problem& P, double* b) {
  if (!P.wnod) return ETQ_OK;   // zero wind: nu L only
  double* nloc;
  ETQ_TRY(dalloc(&nloc, (size_t)81 * P.g.n * P.g.n));
  const int64_t nt = (int64_t)P.g.n * P.g.n * 9;
  k_conv_local<<<(unsigned)((nt + 255) / 256), 256, 0, P.stream>>>(P.g, P.wnod, nloc); etq_count_launch();
  k_rhs_conv<<<(P.g.nq + 255) / 256, 256, 0, P.stream>>>(P.g, P.bc, nloc, b); etq_count_launch();
  ETQ_CHECK(cudaStreamSynchronize(P.stream));
  cudaFree(nloc);
  return ETQ_OK;
}

// Picard loop: x^0 = the Stokes velocity (the wind-0 system nu L, whose velocity is
// the Stokes velocity), then `steps` Oseen solves with the wind of the previous iterate.  Every
// solve is the two-stage PCD strategy to ||r|| <= eta ||b||.  x (device) receives
// the last iterate; its[2k], its[2k+1] the Step I / Step II GMRES iterations of solve k and
// res[k] its true residual ||b_k - K_k x^k|| / ||b_k|| (host arrays, may be NULL).
etq_status picard_run(Problem& P, int steps, double eta, double c, int restart, int maxit, double* x,
                      int* its, double* res, double* ms_total) {
  NvtxRange nvtx_("Picard loop");
  if (!(P.oseen && P.wind == 2)) return ETQ_EINVAL;
  if (!P.pcd_ready || !P.m1_ready) return ETQ_ENOTSETUP;
  cudaStream_t st = P.stream;
  if (!P.wnod) ETQ_TRY(dalloc(&P.wnod, (size_t)P.n_u));
  double* b = nullptr;
  double* y = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // every exit below goes through this cleanup (no early return leaks b, y or the events)
  auto cleanup = [&](etq_status s) {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(b); cudaFree(y);
    return s;
  };
  if (dalloc(&b, P.N) != ETQ_OK || dalloc(&y, P.N) != ETQ_OK) return cleanup(ETQ_ENOMEM);
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return cleanup(ETQ_ECUDA);
  cudaEventRecord(e0, st);
  etq_status status = ETQ_OK;
  for (int k = 0; k <= steps; ++k) {
    cudaError_t ce = (k == 0) ? cudaMemsetAsync(P.wnod, 0, sizeof(double) * P.n_u, st)
                              : cudaMemcpyAsync(P.wnod, x, sizeof(double) * P.n_u, cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess) { status = ETQ_ECUDA; break; }
    etq_status s = picard_refresh(P);
    if (s < 0) { status = s; break; }
    s = build_rhs_dev(P, nullptr, b);
    if (s < 0) { status = s; break; }
    etq_report r1{}, r2{};
    s = two_stage_run(P, b, x, eta, c, restart, maxit, &r1, &r2, nullptr);
    if (s < 0) { status = s; break; }
    if (s == ETQ_NOT_CONVERGED) status = ETQ_NOT_CONVERGED;
    if (its) { its[2 * k] = r1.iterations; its[2 * k + 1] = r2.iterations; }
    if (res) {
      launch_saddle_ex(P, false, x, y, nullptr, nullptr, 0, nullptr, nullptr, st);
      vec_lincomb3(y, b, 1.0, y, -1.0, b, 0.0, P.N, st);
      res[k] = host_norm(P, y, P.N) / host_norm(P, b, P.N);
    }
  }
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (ms_total) *ms_total = ms;
  return cleanup(status);
}
