// sweep32.cu — fp32-value variants of the fused saddle SpMV and of the Q2 V-cycle for the kernel
// sweep of BASELINE.json configs[4] ("fp64 and fp32 values"): fp32 matrix values (SELL.fval),
// fp32 vectors and fp32 accumulation; compared with the fp64 oracle at 1e-5 relative.  The
// solvers always run in fp64; these entry points exist for the bandwidth sweep only.
#include "device_common.cuh"
#include <vector>

using namespace etqd;

namespace {

__device__ __forceinline__ float sell_row1f(const Sell& A, int64_t s, int lane, const float* __restrict__ x) {
  const int64_t base = A.sptr[s] + lane;
  const int len = A.slen[s];
  const int* __restrict__ cp = A.col + base;
  const float* __restrict__ vp = A.fval + base;
  float acc = 0.f;
  int k = 0;
  for (; k + 4 <= len; k += 4) {
    int c[4]; float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { c[u] = __ldg(cp + (k + u) * SELL_C); v[u] = __ldg(vp + (k + u) * SELL_C); }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = fmaf(v[u], __ldg(x + c[u]), acc);
  }
  for (; k < len; ++k) acc = fmaf(__ldg(vp + k * SELL_C), __ldg(x + __ldg(cp + k * SELL_C)), acc);
  return acc;
}
__device__ __forceinline__ void sell_row2f(const Sell& A, int64_t s, int lane, const float* __restrict__ x0,
                                           const float* __restrict__ x1, float& a0, float& a1) {
  const int64_t base = A.sptr[s] + lane;
  const int len = A.slen[s];
  const int* __restrict__ cp = A.col + base;
  const float* __restrict__ vp = A.fval + base;
  int k = 0;
  for (; k + 4 <= len; k += 4) {
    int c[4]; float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { c[u] = __ldg(cp + (k + u) * SELL_C); v[u] = __ldg(vp + (k + u) * SELL_C); }
#pragma unroll
    for (int u = 0; u < 4; ++u) { a0 = fmaf(v[u], __ldg(x0 + c[u]), a0); a1 = fmaf(v[u], __ldg(x1 + c[u]), a1); }
  }
  for (; k < len; ++k) {
    const int c = __ldg(cp + k * SELL_C); const float v = __ldg(vp + k * SELL_C);
    a0 = fmaf(v, __ldg(x0 + c), a0); a1 = fmaf(v, __ldg(x1 + c), a1);
  }
}
__device__ __forceinline__ int row_id(const Sell& A, int64_t s, int lane) {
  const int64_t t = s * SELL_C + lane;
  return A.perm ? A.perm[t] : (t < A.nrows ? (int)t : -1);
}

struct SaddleF {
  Sell L, BxT1, ByT1, BxT0, ByT0, B; int nq, nk; int64_t n_u, n_p; int reduced; const float* x; float* y;
};
__global__ void __launch_bounds__(BS) k_saddle_f32(SaddleF a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsv = a.L.nslices, nsp = a.B.nslices;
  const float* xu = a.x; const float* xv = a.x + a.nq;
  const float* p1 = a.x + a.n_u; const float* p0 = p1 + a.nk;
  for (int64_t s = gw; s < nsv + nsp; s += nw) {
    if (s < nsv) {
      const int row = row_id(a.L, s, lane);
      float ax = 0.f, ay = 0.f;
      sell_row2f(a.L, s, lane, xu, xv, ax, ay);
      ax += sell_row1f(a.BxT1, s, lane, p1);
      ay += sell_row1f(a.ByT1, s, lane, p1);
      if (!a.reduced) { ax += sell_row1f(a.BxT0, s, lane, p0); ay += sell_row1f(a.ByT0, s, lane, p0); }
      if (row >= 0) { a.y[row] = ax; a.y[a.nq + row] = ay; }
    } else {
      const int64_t sp = s - nsv, row = sp * SELL_C + lane;
      const float acc = sell_row1f(a.B, sp, lane, xu);
      if (row < a.n_p) a.y[a.n_u + row] = (a.reduced && row >= a.nk) ? 0.f : acc;
    }
  }
}

struct ChebF {
  Sell A; const float* dinv; int nq; const float* d_in; const float* r_in; const float* x_in;
  float* x_out; float* r_out; float* d_out; float c1, c2;
};
__global__ void __launch_bounds__(BS) k_cheb_step_f32(ChebF a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < a.A.nslices; s += nw) {
    const int row = row_id(a.A, s, lane);
    float q[2] = {0.f, 0.f};
    sell_row2f(a.A, s, lane, a.d_in, a.d_in + a.nq, q[0], q[1]);
    if (row < 0) continue;
    const float di = a.dinv[row];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t idx = (int64_t)c * a.nq + row;
      const float dd = a.d_in[idx], ro = a.r_in[idx] - q[c];
      a.x_out[idx] = (a.x_in ? a.x_in[idx] : 0.f) + dd;
      if (a.r_out) a.r_out[idx] = ro;
      if (a.d_out) a.d_out[idx] = a.c1 * dd + a.c2 * (di * ro);
    }
  }
}
__global__ void __launch_bounds__(BS) k_post_residual_f32(Sell A, const float* dinv, int nq, const float* b,
                                                          const float* x, float* r, float* d, float theta) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < A.nslices; s += nw) {
    const int row = row_id(A, s, lane);
    float q[2] = {0.f, 0.f};
    sell_row2f(A, s, lane, x, x + nq, q[0], q[1]);
    if (row < 0) continue;
    const float di = dinv[row];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t idx = (int64_t)c * nq + row;
      const float rr = b[idx] - q[c];
      r[idx] = rr; d[idx] = di * rr / theta;
    }
  }
}
__global__ void k_cheb_init_f32(const float* dinv, int nq, const float* b, float* d, float theta) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2LL * nq; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = dinv[i % nq] * b[i] / theta;
}
__device__ __forceinline__ int rtaps(int I, int* off, float* w) {
  if ((I & 1) == 0) {
    off[0] = -3; w[0] = -0.125f; off[1] = -1; w[1] = 0.375f; off[2] = 0; w[2] = 1.f; off[3] = 1; w[3] = 0.375f;
    off[4] = 3; w[4] = -0.125f;
    return 5;
  }
  off[0] = -1; w[0] = 0.75f; off[1] = 0; w[1] = 1.f; off[2] = 1; w[2] = 0.75f;
  return 3;
}
__global__ void k_restrict_f32(int mf, int mc, int nqf, int nqc, const float* rf, float* bc, float* d0c,
                               const float* dinvc, float theta) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nqc; t += (int64_t)gridDim.x * blockDim.x) {
    const int I = (int)(t % mc), J = (int)(t / mc);
    if (I == 0 || J == 0 || I == mc - 1 || J == mc - 1) { bc[t] = bc[nqc + t] = d0c[t] = d0c[nqc + t] = 0.f; continue; }
    int ox[5], oy[5]; float wx[5], wy[5];
    const int nx = rtaps(I, ox, wx), ny = rtaps(J, oy, wy);
    float s0 = 0.f, s1 = 0.f;
    for (int q = 0; q < ny; ++q) {
      const int64_t rowf = (int64_t)(2 * J + oy[q]) * mf;
      float t0 = 0.f, t1 = 0.f;
      for (int p = 0; p < nx; ++p) {
        const int64_t f = rowf + 2 * I + ox[p];
        t0 = fmaf(wx[p], rf[f], t0); t1 = fmaf(wx[p], rf[nqf + f], t1);
      }
      s0 = fmaf(wy[q], t0, s0); s1 = fmaf(wy[q], t1, s1);
    }
    bc[t] = s0; bc[nqc + t] = s1;
    d0c[t] = dinvc[t] * s0 / theta; d0c[nqc + t] = dinvc[t] * s1 / theta;
  }
}
__device__ __forceinline__ int ptaps(int k, int* idx, float* w) {
  if ((k & 1) == 0) { idx[0] = k >> 1; w[0] = 1.f; return 1; }
  const int e = k >> 2;
  idx[0] = 2 * e; idx[1] = 2 * e + 1; idx[2] = 2 * e + 2;
  if ((k & 3) == 1) { w[0] = 0.375f; w[1] = 0.75f; w[2] = -0.125f; } else { w[0] = -0.125f; w[1] = 0.75f; w[2] = 0.375f; }
  return 3;
}
__global__ void k_prolong_f32(int mf, int mc, int nqf, int nqc, const float* xc, const float* dc, float* xf) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nqf; t += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(t % mf), l = (int)(t / mf);
    if (k == 0 || l == 0 || k == mf - 1 || l == mf - 1) continue;
    int ix[3], iy[3]; float wx[3], wy[3];
    const int nx = ptaps(k, ix, wx), ny = ptaps(l, iy, wy);
    float s0 = 0.f, s1 = 0.f;
    for (int q = 0; q < ny; ++q) {
      float t0 = 0.f, t1 = 0.f;
      for (int p = 0; p < nx; ++p) {
        const int64_t c = (int64_t)iy[q] * mc + ix[p];
        t0 = fmaf(wx[p], dc ? xc[c] + dc[c] : xc[c], t0);
        t1 = fmaf(wx[p], dc ? xc[nqc + c] + dc[nqc + c] : xc[nqc + c], t1);
      }
      s0 = fmaf(wy[q], t0, s0); s1 = fmaf(wy[q], t1, s1);
    }
    xf[t] += s0; xf[nqf + t] += s1;
  }
}
__global__ void k_add_f32(const float* x, const float* d, float* z, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = d ? x[i] + d[i] : x[i];
}
__global__ void k_gemv_f32(const float* A, int m, const float* x, int64_t xs, float* y, int64_t ys) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < m; r += nw)
    for (int c = 0; c < 2; ++c) {
      float s = 0.f;
      for (int j = lane; j < m; j += 32) s = fmaf(A[r * m + j], x[c * xs + j], s);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) y[c * ys + r] = s;
    }
}
__global__ void k_to_float(const double* a, float* b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

etq_status sell_make_f32(Sell& S, cudaStream_t st) {
  if (S.fval || S.nnz_stored == 0) return ETQ_OK;
  ETQ_TRY(dalloc(&S.fval, S.nnz_stored));
  k_to_float<<<grid_for(S.nnz_stored, BS, 4096), BS, 0, st>>>(S.val, S.fval, S.nnz_stored); etq_count_launch();
  return ETQ_OK;
}
etq_status to_f32(const double* a, float** b, int64_t n, cudaStream_t st) {
  ETQ_TRY(dalloc(b, n));
  k_to_float<<<grid_for(n, BS, 4096), BS, 0, st>>>(a, *b, n); etq_count_launch();
  return ETQ_OK;
}
}  // namespace

// fp32 copies of the saddle blocks and of the Stokes V-cycle hierarchy (created on first use)
etq_status ensure_f32(Problem& P) {
  cudaStream_t st = P.stream;
  Sell* ms[6] = {&P.Lv, &P.BxT1, &P.ByT1, &P.BxT0, &P.ByT0, &P.B};
  for (Sell* m : ms) ETQ_TRY(sell_make_f32(*m, st));
  if (P.mg.built && !P.mg.f32) {
    if (P.mg.kind != 0) return ETQ_EINVAL;
    for (size_t l = 0; l < P.mg.lv.size(); ++l) {
      Level& L = P.mg.lv[l];
      if (l > 0) ETQ_TRY(sell_make_f32(L.A, st));
      ETQ_TRY(to_f32(L.dinv, &L.f_dinv, L.nrows, st));
      const size_t nv = 2 * (size_t)L.nrows;
      ETQ_TRY(dalloc(&L.f_b, nv)); ETQ_TRY(dalloc(&L.f_x, nv)); ETQ_TRY(dalloc(&L.f_r, nv));
      ETQ_TRY(dalloc(&L.f_d0, nv)); ETQ_TRY(dalloc(&L.f_d1, nv));
      if (L.coarse_inv) ETQ_TRY(to_f32(L.coarse_inv, &L.f_coarse, (int64_t)L.nrows * L.nrows, st));
    }
    P.mg.lv[0].A.fval = P.Lv.fval;
    P.mg.f32 = true;
  }
  ETQ_CHECK(cudaStreamSynchronize(st));
  return ETQ_OK;
}

void launch_saddle_f32(const Problem& P, bool reduced, const float* x, float* y, cudaStream_t st) {
  SaddleF a;
  a.L = P.Lv; a.BxT1 = P.BxT1; a.ByT1 = P.ByT1; a.BxT0 = P.BxT0; a.ByT0 = P.ByT0; a.B = P.B;
  a.nq = P.g.nq; a.nk = P.g.nk; a.n_u = P.n_u; a.n_p = P.n_p; a.reduced = reduced ? 1 : 0; a.x = x; a.y = y;
  k_saddle_f32<<<grid_for((P.Lv.nslices + P.B.nslices) * 32, BS), BS, 0, st>>>(a); etq_count_launch();
}

// same schedule as vcycle_apply_ex (real Chebyshev interval; Stokes hierarchy) in fp32
etq_status vcycle_f32(const Problem& P, const float* r_u, float* z_u, cudaStream_t st) {
  const Hierarchy& H = P.mg;
  if (!H.f32 || H.kind != 0) return ETQ_ENOTSETUP;
  const int L = (int)H.lv.size();
  const double theta = 0.5 * (H.hi + H.lo), delta = 0.5 * (H.hi - H.lo), sigma = theta / delta;
  std::vector<float> c1(H.degree), c2(H.degree);
  {
    double rho = 1.0 / sigma;
    for (int k = 0; k < H.degree; ++k) {
      const double rn = 1.0 / (2.0 * sigma - rho);
      c1[k] = (float)(rn * rho); c2[k] = (float)(2.0 * rn / delta);
      rho = rn;
    }
  }
  if (L == 1) {
    const Level& C = H.lv[0];
    k_gemv_f32<<<grid_for((int64_t)C.nrows * 32, BS, 4096), BS, 0, st>>>(C.f_coarse, C.nrows, r_u, C.nrows, z_u, C.nrows);
    etq_count_launch();
    return ETQ_OK;
  }
  std::vector<const float*> bvec(L), pend(L, nullptr);
  for (int l = 0; l < L - 1; ++l) {
    const Level& lv = H.lv[l];
    const int nq = lv.nrows;
    const float* b = (l == 0) ? r_u : lv.f_b;
    bvec[l] = b;
    if (l == 0) { k_cheb_init_f32<<<grid_for(2LL * nq, BS, 4096), BS, 0, st>>>(lv.f_dinv, nq, b, lv.f_d0, (float)theta); etq_count_launch(); }
    const int gs = grid_for(lv.A.nslices * 32, BS, 4096);
    float* din = lv.f_d0; float* dout = lv.f_d1;
    for (int k = 0; k < H.degree; ++k) {
      ChebF a;
      a.A = lv.A; a.dinv = lv.f_dinv; a.nq = nq; a.d_in = din; a.r_in = (k == 0) ? b : lv.f_r;
      a.x_in = (k == 0) ? nullptr : lv.f_x; a.x_out = lv.f_x; a.r_out = lv.f_r;
      a.d_out = (k == H.degree - 1) ? nullptr : dout; a.c1 = c1[k]; a.c2 = c2[k];
      k_cheb_step_f32<<<gs, BS, 0, st>>>(a); etq_count_launch();
      std::swap(din, dout);
    }
    const Level& cv = H.lv[l + 1];
    k_restrict_f32<<<grid_for(cv.nrows, BS, 4096), BS, 0, st>>>(lv.g.m, cv.g.m, nq, cv.nrows, lv.f_r, cv.f_b, cv.f_d0,
                                                               cv.f_dinv, (float)theta); etq_count_launch();
  }
  {
    const Level& C = H.lv[L - 1];
    k_gemv_f32<<<grid_for((int64_t)C.nrows * 32, BS, 4096), BS, 0, st>>>(C.f_coarse, C.nrows, C.f_b, C.nrows, C.f_x, C.nrows);
    etq_count_launch();
  }
  for (int l = L - 2; l >= 0; --l) {
    const Level& lv = H.lv[l];
    const Level& cv = H.lv[l + 1];
    const int nq = lv.nrows;
    k_prolong_f32<<<grid_for(nq, BS, 4096), BS, 0, st>>>(lv.g.m, cv.g.m, nq, cv.nrows, cv.f_x, pend[l + 1], lv.f_x);
    etq_count_launch();
    const int gs = grid_for(lv.A.nslices * 32, BS, 4096);
    k_post_residual_f32<<<gs, BS, 0, st>>>(lv.A, lv.f_dinv, nq, bvec[l], lv.f_x, lv.f_r, lv.f_d0, (float)theta);
    etq_count_launch();
    float* din = lv.f_d0; float* dout = lv.f_d1;
    for (int k = 0; k < H.degree - 1; ++k) {
      ChebF a;
      a.A = lv.A; a.dinv = lv.f_dinv; a.nq = nq; a.d_in = din; a.r_in = lv.f_r; a.x_in = lv.f_x; a.x_out = lv.f_x;
      a.r_out = (k == H.degree - 2) ? nullptr : lv.f_r; a.d_out = dout; a.c1 = c1[k]; a.c2 = c2[k];
      k_cheb_step_f32<<<gs, BS, 0, st>>>(a); etq_count_launch();
      std::swap(din, dout);
    }
    pend[l] = din;
  }
  const Level& F = H.lv[0];
  k_add_f32<<<grid_for(2LL * F.nrows, BS, 4096), BS, 0, st>>>(F.f_x, pend[0], z_u, 2LL * F.nrows); etq_count_launch();
  return ETQ_OK;
}
