// oseen.cu — Oseen hot path: block upper-triangular preconditioners, the Step-I
// pressure convection-diffusion Schur complement, right-preconditioned GMRES(m)
// with classical Gram-Schmidt applied twice (reading R18), and the two-stage driver
// (P:1058-1092).
//
// GMRES keeps the Hessenberg matrix, the Givens rotations and the residual estimate on the
// device; one Arnoldi step (copy of v_j, preconditioner, operator, 2 x (multi-dot + multi-axpy),
// norm, Givens, normalisation) is one CUDA graph whose kernels read the step index j from device
// memory, so the same graph serves every j.  The host reads a few scalars after each step.
#include "device_common.cuh"
#include <cmath>
#include <cstring>
#include <vector>

using namespace etqd;

extern void launch_saddle_ex(const Problem& P, bool reduced, const double* x, double* y, const double* inv_scale,
                             const RedSite* site, int slot, double* dot_out, const double* done, cudaStream_t st);

namespace {

// ---------------------------------------------------------------- PCD pieces
__device__ __forceinline__ double ml1q(int n, double h, int a, int ap) {
  const int d = a - ap;
  if (d == 0) return (a == 0 || a == n) ? (2.0 * h / 6.0) : (4.0 * h / 6.0);
  return (d == 1 || d == -1) ? (h / 6.0) : 0.0;
}
__device__ __forceinline__ double qk_apply_at(int n, double h, int a, int c, const double* x) {
  const int n1 = n + 1;
  double s = 0.0;
  for (int cc = max(0, c - 1); cc <= min(n, c + 1); ++cc) {
    const double mc = ml1q(n, h, c, cc);
    for (int aa = max(0, a - 1); aa <= min(n, a + 1); ++aa) s += mc * ml1q(n, h, a, aa) * x[aa + n1 * cc];
  }
  return s;
}

// Chebyshev-Jacobi on the Q1 mass Qk (Mp^{-1}, reading R13), matrix-free, one step:
//   x += d ; r -= Qk d ; d' = c1 d + c2 D^{-1} r     (x nullable on the first step)
__global__ void k_qk_cheb_step(int n, double h, const double* d_in, double* r, const double* x_in, double* x_out,
                               double* d_out, double c1, double c2, const double* done) {
  if (is_done(done)) return;
  const int n1 = n + 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n1 * n1;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(t % n1), c = (int)(t / n1);
    const double q = qk_apply_at(n, h, a, c, d_in);
    const double dd = d_in[t];
    const double ro = r[t] - q;
    x_out[t] = (x_in ? x_in[t] : 0.0) + dd;
    r[t] = ro;
    if (d_out) d_out[t] = c1 * dd + c2 * (ro / (ml1q(n, h, a, a) * ml1q(n, h, c, c)));
  }
}
// r = b (copy), d = D^{-1} b / theta
__global__ void k_qk_cheb_init(int n, double h, const double* b, double* r, double* d, double theta,
                               const double* done) {
  if (is_done(done)) return;
  const int n1 = n + 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n1 * n1;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(t % n1), c = (int)(t / n1);
    r[t] = b[t];
    d[t] = (b[t] / (ml1q(n, h, a, a) * ml1q(n, h, c, c))) / theta;
  }
}

// y = scale * A x (single component, SELL)
__global__ void __launch_bounds__(BS) k_spmv1(Sell A, const double* x, double* y, double scale, const double* done) {
  if (is_done(done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < A.nslices; s += nw) {
    const int64_t t = s * SELL_C + lane;
    const int row = A.perm ? A.perm[t] : (t < A.nrows ? (int)t : -1);
    const double v = sell_row1(A, s, lane, x);
    if (row >= 0) y[row] = scale * v;
  }
}

// t_u = r_u - B^T z_p over the velocity node slices (full: B1 and B0 parts; reduced: B1 only)
struct BtSubArgs {
  Sell BxT1, ByT1, BxT0, ByT0; int nq; int nk; int reduced;
  const double* r_u; const double* z_p; double* t_u; const double* done;
};
__global__ void __launch_bounds__(BS) k_bt_sub(BtSubArgs a) {
  if (is_done(a.done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* p1 = a.z_p;
  const double* p0 = a.z_p + a.nk;
  for (int64_t s = gw; s < a.BxT1.nslices; s += nw) {
    const int row = a.BxT1.perm[s * SELL_C + lane];
    double ax = sell_row1(a.BxT1, s, lane, p1), ay = sell_row1(a.ByT1, s, lane, p1);
    if (!a.reduced) { ax += sell_row1(a.BxT0, s, lane, p0); ay += sell_row1(a.ByT0, s, lane, p0); }
    if (row >= 0) {
      a.t_u[row] = a.r_u[row] - ax;
      a.t_u[a.nq + row] = a.r_u[a.nq + row] - ay;
    }
  }
}

// t_u = r_u - B^T z_p matrix-free (storage 0): every non-Dirichlet velocity row of B^T is its class
// stencil over the 3 x 3 Q1 vertices and 2 x 2 P0 cells around it (SaddleSt, wind-independent);
// Dirichlet rows of B^T are empty.  One thread per node, both components.
struct BtMfArgs {
  SaddleSt w; int m, n, nq, nk, reduced;
  const double* r_u; const double* z_p; double* t_u; const double* done;
};
__global__ void __launch_bounds__(BS) k_bt_sub_mf(BtMfArgs a) {
  if (is_done(a.done)) return;
  const int m = a.m, n = a.n, n1 = n + 1;
  const double* __restrict__ p1 = a.z_p;
  const double* __restrict__ p0 = a.z_p + a.nk;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < a.nq; t += (int64_t)gridDim.x * blockDim.x) {
    const int node = (int)t, i = node % m, j = node / m;
    double bx = 0.0, by = 0.0;
    if (!(i == 0 || j == 0 || i == m - 1 || j == m - 1)) {
      const int cl = (j & 1) * 2 + (i & 1);
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
        bx += cx; by += cy;
      }
    }
    a.t_u[node] = __ldg(a.r_u + node) - bx;
    a.t_u[a.nq + node] = __ldg(a.r_u + a.nq + node) - by;
  }
}

// t_u = minv o (B^T z_p) (both parts; minv = 1 / Mdiag, zero on Dirichlet nodes)
__global__ void __launch_bounds__(BS) k_bt_minv(BtSubArgs a, const double* minv) {
  if (is_done(a.done)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* p1 = a.z_p;
  const double* p0 = a.z_p + a.nk;
  for (int64_t s = gw; s < a.BxT1.nslices; s += nw) {
    const int row = a.BxT1.perm[s * SELL_C + lane];
    const double ax = sell_row1(a.BxT1, s, lane, p1) + sell_row1(a.BxT0, s, lane, p0);
    const double ay = sell_row1(a.ByT1, s, lane, p1) + sell_row1(a.ByT0, s, lane, p0);
    if (row >= 0) { a.t_u[row] = minv[row] * ax; a.t_u[a.nq + row] = minv[row] * ay; }
  }
}

// y = minv o x on both velocity components
__global__ void k_scale_minv(const double* x, const double* minv, double* y, int nq, const double* done) {
  if (is_done(done)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2LL * nq; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = minv[i % nq] * x[i];
}

// P0 convection-diffusion F0 (reading R25): y_T = sum over the interior edges e of T of
// (nu - (w_e . n_e) h / 2) (x_T - x_T'), w_e the wind at the edge midpoint (a Q2 node)
__global__ void k_f0_apply(Geo g, double nu, int wind, const double* wnod, const double* x, double* y,
                           double scale, const double* done) {
  if (is_done(done)) return;
  const int n = g.n, m = g.m; const double h = g.h;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t % n), f = (int)(t / n);
    const double xt = x[t] * scale;
    double acc = 0.0;
    for (int k = 0; k < 4; ++k) {
      const int de = k == 0 ? 1 : (k == 1 ? -1 : 0), df = k == 2 ? 1 : (k == 3 ? -1 : 0);
      const int e2 = e + de, f2 = f + df;
      if (e2 < 0 || e2 >= n || f2 < 0 || f2 >= n) continue;
      const int i = 2 * e + 1 + de, j = 2 * f + 1 + df;          // edge-midpoint Q2 node
      double wx = 0.0, wy = 0.0;
      if (wind == 1) {
        const double xx = -1.0 + i * (0.5 * h), yy = -1.0 + j * (0.5 * h);
        wx = 2.0 * yy * (1.0 - xx * xx); wy = -2.0 * xx * (1.0 - yy * yy);
      } else if (wind == 2 && wnod) {
        wx = wnod[i + m * j]; wy = wnod[g.nq + i + m * j];
      }
      const double flux = (wx * de + wy * df) * h / 2.0;
      acc += (nu - flux) * (xt - x[e2 + (int64_t)n * f2] * scale);
    }
    y[t] = acc;
  }
}

__global__ void k_fill(double* x, int64_t n, double v, const double* done) {
  if (is_done(done)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}

// ---------------------------------------------------------------- GMRES kernels
__global__ void k_copy_vj(const double* V, int64_t N, int64_t ld, const double* sc, double* T) {
  const int64_t j = (int64_t)sc[G_J];
  const double* vj = V + j * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    T[i] = vj[i];
}

// CGS2 (reading R18) in three passes over the basis instead of four:
//   A  h = V^T w                                   (k_multidot)
//   B  w <- w - V h, then h' = V^T w               (k_cgs_mid: the segment of every V_i is read
//                                                   twice by the same warp, the second time from L2)
//   C  w <- w - V h', ||w||^2                      (k_cgs_last)
// The basis vectors are stored with a stride ld (N rounded up to 32 elements) so that every V_i is
// 256-byte aligned and is streamed with 128-bit loads.  Dot products: each warp owns segments of
// CG_SEG consecutive elements (grid-stride over segments), lane l the pairs 2l + 64k; per segment
// and vector the lane sums its CG_K pairs, the warp sums its lanes (shuffles) and lane (i mod 32)
// keeps the warp's running total of vector i; warps are combined in warp order in shared memory,
// blocks in block order by the last block: deterministic for a fixed grid.
constexpr int CG_K = 4, CG_SEG = 64 * CG_K, MD_MAXV = 64;

__device__ __forceinline__ void cg_ld(const double* __restrict__ p, int64_t e, int64_t N, double& a, double& b) {
  if (e + 1 < N) { const double2 t = __ldg(reinterpret_cast<const double2*>(p + e)); a = t.x; b = t.y; }
  else { a = e < N ? __ldg(p + e) : 0.0; b = 0.0; }
}
__device__ __forceinline__ void cg_ldw(const double* p, int64_t e, int64_t N, double& a, double& b) {
  if (e + 1 < N) { const double2 t = *reinterpret_cast<const double2*>(p + e); a = t.x; b = t.y; }
  else { a = e < N ? p[e] : 0.0; b = 0.0; }
}
__device__ __forceinline__ void cg_st(double* p, int64_t e, int64_t N, double a, double b) {
  if (e + 1 < N) *reinterpret_cast<double2*>(p + e) = make_double2(a, b);
  else if (e < N) p[e] = a;
}

// running totals of a warp (lane i mod 32 holds vector i's) -> h[0..nv) through the grid reduction
__device__ __forceinline__ void md_finish(double t0, double t1, int nv, double* h, RedSite site) {
  __shared__ double part[BS / 32][MD_MAXV];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < nv) part[warp][lane] = t0;
  if (lane + 32 < nv) part[warp][lane + 32] = t1;
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += BS) {
    double b = 0.0;
    for (int wi = 0; wi < BS / 32; ++wi) b += part[wi][i];
    site.partials[(int64_t)i * MAXB + blockIdx.x] = b;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(site.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (last) {
    __threadfence();
    for (int i = warp; i < nv; i += BS / 32) {
      double sv = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) sv += __ldcg(site.partials + (int64_t)i * MAXB + b);
      sv = warp_sum(sv);
      if (lane == 0) h[i] = sv;
    }
    if (threadIdx.x == 0) site.counter[0] = 0u;
  }
}

// pass A: h_i = <V_i, W>, i = 0..j (j from device)
__global__ void __launch_bounds__(BS) k_multidot(const double* V, int64_t N, int64_t ld, const double* W,
                                                 const double* sc, double* h, RedSite site) {
  const int nv = min((int)sc[G_J] + 1, MD_MAXV);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nseg = (N + CG_SEG - 1) / CG_SEG;
  const int64_t nw = (int64_t)gridDim.x * (BS / 32);
  double t0 = 0.0, t1 = 0.0;
  for (int64_t sg = (int64_t)blockIdx.x * (BS / 32) + warp; sg < nseg; sg += nw) {
    const int64_t e0 = sg * CG_SEG + 2 * lane;
    double w[2 * CG_K];
#pragma unroll
    for (int k = 0; k < CG_K; ++k) cg_ldw(W, e0 + 64 * k, N, w[2 * k], w[2 * k + 1]);
#pragma unroll 2
    for (int i = 0; i < nv; ++i) {
      const double* vi = V + (int64_t)i * ld;
      double v[2 * CG_K];
#pragma unroll
      for (int k = 0; k < CG_K; ++k) cg_ld(vi, e0 + 64 * k, N, v[2 * k], v[2 * k + 1]);
      double sv = 0.0;
#pragma unroll
      for (int k = 0; k < 2 * CG_K; ++k) sv = fma(v[k], w[k], sv);
      sv = warp_sum(sv);
      if (lane == (i & 31)) { if (i < 32) t0 += sv; else t1 += sv; }
    }
  }
  md_finish(t0, t1, nv, h, site);
}

// pass B: W <- W - sum_i h_i V_i (in i order), then h'_i = <V_i, W> on the updated segment.  The
// second sweep re-reads the segment of every V_i: with one 16-byte pair per lane (512-byte
// segments) and 2 CTAs per SM the grid's working set between the two reads is about
// 2 x 148 x 8 warps x 512 B x (j + 1) (~50 MB at j = 40), so the re-read is served by L2.
constexpr int CGM_U = 8;   // loads in flight per lane
__global__ void __launch_bounds__(BS) k_cgs_mid(const double* V, int64_t N, int64_t ld, double* W, const double* h,
                                                const double* sc, double* h2, RedSite site) {
  const int nv = min((int)sc[G_J] + 1, MD_MAXV);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nseg = (N + 63) / 64;
  const int64_t nw = (int64_t)gridDim.x * (BS / 32);
  double t0 = 0.0, t1 = 0.0;
  for (int64_t sg = (int64_t)blockIdx.x * (BS / 32) + warp; sg < nseg; sg += nw) {
    const int64_t e = sg * 64 + 2 * lane;
    double w0, w1;
    cg_ldw(W, e, N, w0, w1);
    int i = 0;
    for (; i + CGM_U <= nv; i += CGM_U) {
      double v[CGM_U][2];
#pragma unroll
      for (int u = 0; u < CGM_U; ++u) cg_ld(V + (int64_t)(i + u) * ld, e, N, v[u][0], v[u][1]);
#pragma unroll
      for (int u = 0; u < CGM_U; ++u) { const double hi = __ldg(h + i + u); w0 -= hi * v[u][0]; w1 -= hi * v[u][1]; }
    }
    for (; i < nv; ++i) {
      double v0, v1;
      cg_ld(V + (int64_t)i * ld, e, N, v0, v1);
      const double hi = __ldg(h + i);
      w0 -= hi * v0; w1 -= hi * v1;
    }
    cg_st(W, e, N, w0, w1);
    // h'_i partials of this segment for 32 vectors at a time, reduced across the warp by recursive
    // halving (31 shuffles per 32 sums instead of 5 per sum): lane l ends with vector (32 c + l)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int base = 32 * c;
      if (base >= nv) break;
      double pp[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        double v0 = 0.0, v1 = 0.0;
        if (base + k < nv) cg_ld(V + (int64_t)(base + k) * ld, e, N, v0, v1);
        pp[k] = fma(v1, w1, v0 * w0);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < o; ++k) {
          const double keep = up ? pp[k + o] : pp[k];
          const double send = up ? pp[k] : pp[k + o];
          pp[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (c == 0) t0 += pp[0]; else t1 += pp[0];
    }
  }
  md_finish(t0, t1, nv, h2, site);
}

// pass C: W <- W - sum_i h'_i V_i, out = ||W||^2 (deterministic grid reduction)
__global__ void __launch_bounds__(BS) k_cgs_last(const double* V, int64_t N, int64_t ld, double* W, const double* h,
                                                 const double* sc, RedSite site, int slot, double* out) {
  const int nv = (int)sc[G_J] + 1;
  double s = 0.0;
  for (int64_t e = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); e < N; e += 2 * (int64_t)gridDim.x * blockDim.x) {
    double w0, w1;
    cg_ldw(W, e, N, w0, w1);
    int i = 0;
    for (; i + 4 <= nv; i += 4) {
      double v[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) cg_ld(V + (int64_t)(i + u) * ld, e, N, v[u][0], v[u][1]);
#pragma unroll
      for (int u = 0; u < 4; ++u) { const double c = __ldg(h + i + u); w0 -= c * v[u][0]; w1 -= c * v[u][1]; }
    }
    for (; i < nv; ++i) {
      double v0, v1;
      cg_ld(V + (int64_t)i * ld, e, N, v0, v1);
      const double c = __ldg(h + i);
      w0 -= c * v0; w1 -= c * v1;
    }
    cg_st(W, e, N, w0, w1);
    s = fma(w0, w0, s);
    if (e + 1 < N) s = fma(w1, w1, s);
  }
  double v1[1] = {s};
  reduce_finish<1>(v1, site, slot, out);
}

// W -= sum_{i <= j} coef_i V_i  (coef device array, count j + 1 from device); the vector loads of
// eight terms are issued before their updates (same update order)
__global__ void k_multiaxpy(double* W, const double* V, int64_t N, int64_t ld, const double* coef, const double* sc,
                            int cnt_slot, int cnt_add, double sign) {
  const int nv = (int)sc[cnt_slot] + cnt_add;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    double w = W[e];
    int i = 0;
    for (; i + 8 <= nv; i += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = V[(int64_t)(i + u) * ld + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) w -= sign * coef[i + u] * v[u];
    }
    for (; i < nv; ++i) w -= sign * coef[i] * V[(int64_t)i * ld + e];
    W[e] = w;
  }
}

// Arnoldi bookkeeping on one thread: H(:, j) = h + hh, H(j+1, j) = ||w||, previous rotations,
// new rotation, g, residual estimate |g_{j+1}|, stop flags.
// small GMRES arrays, padded segments of (m + 16): cs, sn, g, y, hh (2nd CGS pass), h (1st pass)
__host__ __device__ __forceinline__ int gseg(int m, int k) { return k * (m + 16); }

__global__ void k_gmres_scalar(double* sc, double* H, double* sm, int m, double* hist, int hist_cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double* cs = sm + gseg(m, 0); double* sn = sm + gseg(m, 1); double* g = sm + gseg(m, 2); double* hh = sm + gseg(m, 4);
  const int j = (int)sc[G_J];
  const int ld = m + 1;
  double* Hj = H + (int64_t)j * ld;
  for (int i = 0; i <= j; ++i) Hj[i] += hh[i];
  const double hn = sqrt(sc[G_HN]);
  sc[G_HN] = hn;
  Hj[j + 1] = hn;
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * Hj[i] + sn[i] * Hj[i + 1];
    Hj[i + 1] = -sn[i] * Hj[i] + cs[i] * Hj[i + 1];
    Hj[i] = t;
  }
  const double den = hypot(Hj[j], Hj[j + 1]);
  cs[j] = Hj[j] / den; sn[j] = Hj[j + 1] / den;
  Hj[j] = den; Hj[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  const double res = fabs(g[j + 1]);
  sc[G_RES] = res;
  const int tot = (int)sc[G_TOT];
  if (tot < hist_cap) hist[tot + 1] = res;
  sc[G_TOT] = tot + 1;
  sc[G_JW] = j;
  sc[G_J] = j + 1;
  if (res <= sc[G_TOL]) sc[G_DONE] = 1.0;
  if (hn == 0.0) sc[G_BREAK] = 1.0;
  if (den != den) { sc[G_BREAK] = 1.0; sc[G_DONE] = -1.0; }
}

__global__ void k_store_hcol(double* H, const double* h, const double* sc, int m) {
  const int j = (int)sc[G_J];
  for (int i = threadIdx.x; i <= j; i += blockDim.x) H[(int64_t)j * (m + 1) + i] = h[i];
}

// V_{j+1} = W / ||W||
__global__ void k_set_vnext(double* V, int64_t N, int64_t ld, const double* W, const double* sc) {
  const double hn = sc[G_HN];
  if (hn == 0.0) return;
  const int64_t jw = (int64_t)sc[G_JW];
  double* vn = V + (jw + 1) * ld;
  const double inv = 1.0 / hn;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    vn[i] = W[i] * inv;
}

// start of a restart cycle: V_0 = r / beta, g = beta e_1, j = 0
__global__ void k_cycle_init(double* V, int64_t N, const double* r, double* sc, double* sm, int m) {
  const double beta = sqrt(sc[G_BETA]);
  const double inv = 1.0 / beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    V[i] = r[i] * inv;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double* g = sm + gseg(m, 2);
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    sc[G_J] = 0.0; sc[G_DONE] = 0.0; sc[G_BREAK] = 0.0; sc[G_RES] = beta;
  }
}

// y = H(0:k, 0:k)^{-1} g(0:k), k = current j
__global__ void k_trisolve(const double* H, double* sm, const double* sc, int m) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int k = (int)sc[G_J];
  const double* g = sm + gseg(m, 2);
  double* y = sm + gseg(m, 3);
  const int ld = m + 1;
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int c = i + 1; c < k; ++c) s -= H[(int64_t)c * ld + i] * y[c];
    y[i] = s / H[(int64_t)i * ld + i];
  }
}

__global__ void k_axpy(double* x, const double* z, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += z[i];
}
__global__ void k_bsub(double* w, const double* b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = b[i] - w[i];
}
__global__ void k_zero_tail(double* x, int64_t from, int64_t n) {
  for (int64_t i = from + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = 0.0;
}
__global__ void __launch_bounds__(BS) k_dot2(const double* a, const double* b, int64_t n, RedSite site, int slot,
                                             double* out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  double v[1] = {s};
  reduce_finish<1>(v, site, slot, out);
}

}  // namespace

// ================================================================ host side
static double theta_of(double lo, double hi) { return 0.5 * (hi + lo); }

// Mp^{-1} r: m_p-step Chebyshev-Jacobi on Qk over [1/4, 9/4] from zero (reading R13); x -> out
static void qk_cheb_impl(const Problem& P, const double* r, double* out, int steps, double* rr, double* d0, double* d1,
                         const double* done, cudaStream_t st) {
  const int n = P.g.n; const double h = P.g.h;
  const int64_t nk = P.g.nk;
  const double lo = 0.25, hi = 2.25, theta = theta_of(lo, hi), delta = 0.5 * (hi - lo), sigma = theta / delta;
  const int gsz = grid_for(nk, BS, 4096);
  k_qk_cheb_init<<<gsz, BS, 0, st>>>(n, h, r, rr, d0, theta, done); etq_count_launch();
  double rho = 1.0 / sigma;
  double* din = d0; double* dout = d1;
  for (int k = 0; k < steps; ++k) {
    const double rn = 1.0 / (2.0 * sigma - rho);
    const double c1 = rn * rho, c2 = 2.0 * rn / delta;
    k_qk_cheb_step<<<gsz, BS, 0, st>>>(n, h, din, rr, k == 0 ? nullptr : out, out, k == steps - 1 ? nullptr : dout,
                                       c1, c2, done); etq_count_launch();
    rho = rn;
    std::swap(din, dout);
  }
}

static void qk_cheb(const Problem& P, const double* r, double* out, int steps, const double* done, cudaStream_t st) {
  qk_cheb_impl(P, r, out, steps, P.pw[1], P.pw[2], P.tu, done, st);   // scratch (tu is free at this point)
}

void qk_cheb_ws(const Problem& P, const double* r, double* out, int steps, double* ws, const double* done,
                cudaStream_t st) {
  qk_cheb_impl(P, r, out, steps, ws, ws + P.g.nk, ws + 2 * P.g.nk, done, st);
}

// z_p = -M_S^+ r_p for the two-field PCD (M2) or LSC (M3) approximation (NEXT-4, oracle.schur2)
etq_status schur2_apply(const Problem& P, etq_pc_kind kind, const double* r_p, double* z_p, const double* done,
                        cudaStream_t st) {
  if (!P.lp.ready || !P.minv) return ETQ_ENOTSETUP;
  const int nk = P.g.nk, n0 = P.g.n0, nq = P.g.nq;
  const int64_t np = (int64_t)nk + n0;
  double* u = P.s2w[0]; double* v = P.s2w[1]; double* w = P.s2w[2]; double* y = P.s2w[3];
  if (kind == ETQ_PC_OSEEN_M2) {
    if (!P.F1.val) return ETQ_ENOTSETUP;
    // [F1 Q1^{-1} r_1 ; F0 Q0^{-1} r_0], Q1^{-1} as in the Step-I PCD (R13), Q0 = h^2 I
    qk_cheb(P, r_p, v, P.params.mass_cheb_steps, done, st);
    k_spmv1<<<grid_for(P.F1.nslices * 32, BS, 4096), BS, 0, st>>>(P.F1, v, u, 1.0, done); etq_count_launch();
    k_f0_apply<<<grid_for(n0, BS, 4096), BS, 0, st>>>(P.g, P.nu, P.wind, P.wnod, r_p + nk, u + nk,
                                                      1.0 / (P.g.h * P.g.h), done); etq_count_launch();
    ETQ_TRY(lp_pinv_apply(P, u, z_p, done, st));
  } else if (kind == ETQ_PC_OSEEN_LSC) {
    // Lp^+ (B M^{-1} F M^{-1} B^T) Lp^+ r   (H = M, reading R26)
    ETQ_TRY(lp_pinv_apply(P, r_p, u, done, st));
    BtSubArgs a;
    a.BxT1 = P.BxT1; a.ByT1 = P.ByT1; a.BxT0 = P.BxT0; a.ByT0 = P.ByT0; a.nq = nq; a.nk = nk; a.reduced = 0;
    a.r_u = nullptr; a.z_p = u; a.t_u = v; a.done = done;
    k_bt_minv<<<grid_for(P.BxT1.nslices * 32, BS, 4096), BS, 0, st>>>(a, P.minv); etq_count_launch();
    launch_vel_spmv(P.Lv, v, w, nq, st);
    k_scale_minv<<<grid_for(2LL * nq, BS, 4096), BS, 0, st>>>(w, P.minv, v, nq, done); etq_count_launch();
    k_spmv1<<<grid_for(P.B.nslices * 32, BS, 4096), BS, 0, st>>>(P.B, v, y, 1.0, done); etq_count_launch();
    ETQ_TRY(lp_pinv_apply(P, y, z_p, done, st));
  } else {
    return ETQ_EINVAL;
  }
  vec_scale_copy(z_p, z_p, -1.0, np, st);
  ETQ_CHECK(cudaGetLastError());
  return ETQ_OK;
}

etq_status oseen_precond_apply(const Problem& P, etq_pc_kind kind, const double* r, double* z, cudaStream_t st) {
  NvtxRange nvtx_("Oseen block-triangular apply");
  const int64_t nu = P.n_u;
  const double* done = nullptr;
  if (kind == ETQ_PC_OSEEN_PCD1) {
    if (!P.pcd_ready) return ETQ_ENOTSETUP;
    // z_p1 = -Ap^{-1} F1 Mp^{-1} r_p1 (paper order, reading R11); z_p0 = 0 (reduced system)
    double* t1 = P.pw[0];
    qk_cheb(P, r + nu, t1, P.params.mass_cheb_steps, done, st);
    double* t2 = P.pw[1];
    k_spmv1<<<grid_for(P.F1.nslices * 32, BS, 4096), BS, 0, st>>>(P.F1, t1, t2, 1.0, done); etq_count_launch();
    ETQ_TRY(ap_solve(P, P.apH, t2, z + nu, P.dscal + S_APSUM, done, st));
    // negate z_p1 and zero z_p0
    vec_scale_copy(z + nu, z + nu, -1.0, P.g.nk, st);
    k_fill<<<grid_for(P.g.n0, BS, 4096), BS, 0, st>>>(z + nu + P.g.nk, P.g.n0, 0.0, done); etq_count_launch();
  } else if (kind == ETQ_PC_OSEEN_M2 || kind == ETQ_PC_OSEEN_LSC) {
    ETQ_TRY(schur2_apply(P, kind, r + nu, z + nu, done, st));
  } else if (kind == ETQ_PC_OSEEN_M1) {
    if (!P.m1_ready) return ETQ_ENOTSETUP;
    // z_p = -nu Pi C Pi r_p  ( -(1/nu) M_Q~ z_p = r_p, P:1006 )
    ETQ_TRY(mass_pc_apply_ex(P, r + nu, z + nu, &P.red[0], 2, nullptr, nullptr, done, st, -P.nu));
  } else {
    return ETQ_EINVAL;
  }
  if (P.bt_mf && g_oseen_mf) {
    BtMfArgs b;
    b.w = P.sst; b.m = P.g.m; b.n = P.g.n; b.nq = P.g.nq; b.nk = P.g.nk;
    b.reduced = kind == ETQ_PC_OSEEN_PCD1 ? 1 : 0;
    b.r_u = r; b.z_p = z + nu; b.t_u = P.tu; b.done = done;
    k_bt_sub_mf<<<grid_for(P.g.nq, BS, 8 * 148), BS, 0, st>>>(b); etq_count_launch();
  } else {
  BtSubArgs a;
  a.BxT1 = P.BxT1; a.ByT1 = P.ByT1; a.BxT0 = P.BxT0; a.ByT0 = P.ByT0; a.nq = P.g.nq; a.nk = P.g.nk;
  a.reduced = kind == ETQ_PC_OSEEN_PCD1 ? 1 : 0;
  a.r_u = r; a.z_p = z + nu; a.t_u = P.tu; a.done = done;
  k_bt_sub<<<grid_for(P.BxT1.nslices * 32, BS, 4096), BS, 0, st>>>(a); etq_count_launch();
  }
  // nothing runs beside the F V-cycle of a block-triangular preconditioner: programmatic dependent
  // launches between its kernels (as for P3) shorten the latency-bound cycle
  return vcycle_apply_ex(P, P.mg, P.tu, z, nullptr, 0, nullptr, nullptr, done, st, g_oseen_vc_pdl);
}

etq_status oseen_setup(Problem& P, etq_pc_kind kind) {
  if (!P.oseen) return ETQ_EINVAL;
  const etq_pc_params& prm = P.params;
  if (!P.mg.built) {
    const int cn = std::min(prm.coarse_n, P.g.n);
    ETQ_TRY(build_hierarchy(P, P.mg, cn, prm.smooth_lo, prm.smooth_hi, prm.smooth_degree));
  }
  if (!P.tu) ETQ_TRY(dalloc(&P.tu, P.n_u));
  if (kind == ETQ_PC_OSEEN_PCD1) {
    if (!P.pcd_ready) {
      ETQ_TRY(build_ap_hierarchy(P, P.apH, 2, prm.smooth_lo, prm.smooth_hi, prm.smooth_degree));
      ETQ_TRY(assemble_f1(P.g, P.nu, P.wind, &P.F1, P.stream));
      for (int i = 0; i < 3; ++i) ETQ_TRY(dalloc(&P.pw[i], P.g.nk));
      ETQ_CHECK(cudaStreamSynchronize(P.stream));
    }
    P.pcd_ready = true;
    return ETQ_OK;
  }
  if (kind == ETQ_PC_OSEEN_M1) {
    P.m1_ready = true;
    return ETQ_OK;
  }
  if (kind == ETQ_PC_OSEEN_M2 || kind == ETQ_PC_OSEEN_LSC) {
    ETQ_TRY(lp_setup(P));
    if (!P.minv) {
      ETQ_TRY(dalloc(&P.minv, P.g.nq));
      ETQ_TRY(velocity_mdiag_inv(P.g, P.minv, P.stream));
    }
    for (int i = 0; i < 4; ++i) if (!P.s2w[i]) ETQ_TRY(dalloc(&P.s2w[i], P.n_u));
    if (kind == ETQ_PC_OSEEN_M2) {
      if (!P.F1.val) ETQ_TRY(assemble_f1(P.g, P.nu, P.wind, &P.F1, P.stream));
      for (int i = 0; i < 3; ++i) if (!P.pw[i]) ETQ_TRY(dalloc(&P.pw[i], P.g.nk));
    }
    ETQ_CHECK(cudaStreamSynchronize(P.stream));
    return ETQ_OK;
  }
  return ETQ_EINVAL;
}

void oseen_free(Problem& P) {
  lp_free(P);
  cudaFree(P.minv); P.minv = nullptr;
  for (int i = 0; i < 4; ++i) { cudaFree(P.s2w[i]); P.s2w[i] = nullptr; }
  free_hierarchy(P.apH);
  sell_free(P.F1);
  for (int i = 0; i < 3; ++i) { cudaFree(P.pw[i]); P.pw[i] = nullptr; }
  cudaFree(P.tu); P.tu = nullptr;
  cudaFree(P.gV); cudaFree(P.gH); cudaFree(P.gsm); cudaFree(P.gW); cudaFree(P.gZ); cudaFree(P.gT); cudaFree(P.gU);
  cudaFree(P.ghist); cudaFree(P.gred.partials); cudaFree(P.gred.counter);
  if (P.gmres_graph) cudaGraphExecDestroy(P.gmres_graph);
  P.gmres_graph = nullptr;
}

static etq_status gmres_alloc(Problem& P, int m, int hist_cap) {
  if (P.gm != m) {
    cudaFree(P.gV); cudaFree(P.gH); cudaFree(P.gsm);
    P.gld = (P.N + 31) / 32 * 32;   // 256-byte aligned basis vectors (128-bit loads in CGS2)
    ETQ_TRY(dalloc(&P.gV, (size_t)(m + 1) * P.gld));
    ETQ_TRY(dalloc(&P.gH, (size_t)(m + 1) * m));
    ETQ_TRY(dalloc(&P.gsm, (size_t)gseg(m, 6)));
    P.gm = m;
    if (P.gmres_graph) { cudaGraphExecDestroy(P.gmres_graph); P.gmres_graph = nullptr; }
  }
  if (!P.gW) {
    ETQ_TRY(dalloc(&P.gW, P.N)); ETQ_TRY(dalloc(&P.gZ, P.N)); ETQ_TRY(dalloc(&P.gT, P.N)); ETQ_TRY(dalloc(&P.gU, P.N));
    P.gred.nslot = 64;
    ETQ_TRY(dalloc(&P.gred.partials, (size_t)64 * RED_MAXB));
    ETQ_TRY(dalloc(&P.gred.counter, 64));
    ETQ_CHECK(cudaMemset(P.gred.counter, 0, 64 * sizeof(unsigned)));
  }
  if (P.ghist_cap < hist_cap) {
    // the cached Arnoldi graph captures (ghist, ghist_cap) as kernel arguments: rebuild it
    if (P.gmres_graph) { cudaGraphExecDestroy(P.gmres_graph); P.gmres_graph = nullptr; }
    P.gmres_graph_key = -1;
    cudaFree(P.ghist);
    ETQ_TRY(dalloc(&P.ghist, hist_cap + 1));
    P.ghist_cap = hist_cap;
  }
  return ETQ_OK;
}

// one Arnoldi step (capturable): z = M^{-1} v_j, w = K z, CGS2, ||w||, Givens, v_{j+1}
static etq_status arnoldi_step(Problem& P, bool reduced, etq_pc_kind kind, cudaStream_t st) {
  const int m = P.gm;
  const int64_t N = P.N;
  double* sc = P.dscal;
  double* hh = P.gsm + gseg(m, 4);
  double* Hcol = P.gsm + gseg(m, 5);
  const int gN = grid_for(N, BS, RED_BLOCKS);
  const int64_t ld = P.gld;
  k_copy_vj<<<grid_for(N, BS, 4096), BS, 0, st>>>(P.gV, N, ld, sc, P.gT); etq_count_launch();
  ETQ_TRY(oseen_precond_apply(P, kind, P.gT, P.gZ, st));
  launch_saddle_ex(P, reduced, P.gZ, P.gW, nullptr, nullptr, 0, nullptr, nullptr, st);
  // CGS2: h = V^T w ; w -= V h ; h' = V^T w ; w -= V h' ; h += h' (k_gmres_scalar), in three passes
  const int gs = grid_for((N + CG_SEG - 1) / CG_SEG, BS / 32, RED_BLOCKS);
  k_multidot<<<gs, BS, 0, st>>>(P.gV, N, ld, P.gW, sc, Hcol, P.gred); etq_count_launch();
  k_cgs_mid<<<2 * 148, BS, 0, st>>>(P.gV, N, ld, P.gW, Hcol, sc, hh, P.gred); etq_count_launch();
  k_cgs_last<<<grid_for((N + 1) / 2, BS, RED_BLOCKS), BS, 0, st>>>(P.gV, N, ld, P.gW, hh, sc, P.red[0], 7, sc + G_HN);
  etq_count_launch();
  (void)gN;
  return ETQ_OK;
}


etq_status gmres_run(Problem& P, bool reduced, etq_pc_kind kind, const double* b, double* x, double tol_abs,
                     int restart, int maxit, etq_report* rep, double* p0_res_norm) {
  NvtxRange nvtx_("gmres (CGS2)");
  if (restart < 1 || maxit < 1) return ETQ_EINVAL;
  ETQ_TRY(gmres_alloc(P, restart, maxit + 1));
  cudaStream_t st = P.stream;
  const int m = restart;
  const int64_t N = P.N;
  double* sc = P.dscal;
  const int gN = grid_for(N, BS, RED_BLOCKS);
  ETQ_CHECK(cudaEventRecord(P.ev_t0, st));
  ETQ_CHECK(cudaMemsetAsync(P.gH, 0, sizeof(double) * (m + 1) * m, st));
  ETQ_CHECK(cudaMemsetAsync(P.gsm, 0, sizeof(double) * gseg(m, 6), st));
  {
    std::vector<double> h(S_COUNT - G_J, 0.0);
    h[G_TOL - G_J] = tol_abs; h[G_MAXIT - G_J] = maxit;
    ETQ_CHECK(cudaMemcpyAsync(sc + G_J, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st));
  }
  auto residual = [&]() -> etq_status {   // W = b - K x ; G_BETA = ||W||^2 ; G_NRM_P0 = ||W_p0||^2
    launch_saddle_ex(P, reduced, x, P.gW, nullptr, nullptr, 0, nullptr, nullptr, st);
    k_bsub<<<grid_for(N, BS, 4096), BS, 0, st>>>(P.gW, b, N); etq_count_launch();
    if (reduced) { k_zero_tail<<<grid_for(P.g.n0, BS, 4096), BS, 0, st>>>(P.gW, P.n_u + P.g.nk, N); etq_count_launch(); }
    k_dot2<<<gN, BS, 0, st>>>(P.gW, P.gW, N, P.red[0], 7, sc + G_BETA); etq_count_launch();
    const int64_t o0 = P.n_u + P.g.nk;
    k_dot2<<<grid_for(P.g.n0, BS, RED_BLOCKS), BS, 0, st>>>(P.gW + o0, P.gW + o0, P.g.n0, P.red[0], 8, sc + G_NRM_P0);
    etq_count_launch();
    return ETQ_OK;
  };
  auto read_sc = [&]() -> etq_status {
    ETQ_CHECK(cudaMemcpyAsync(P.hscal + G_J, sc + G_J, sizeof(double) * (S_COUNT - G_J), cudaMemcpyDeviceToHost, st));
    ETQ_CHECK(cudaStreamSynchronize(st));
    return ETQ_OK;
  };
  k_dot2<<<gN, BS, 0, st>>>(b, b, N, P.red[0], 9, sc + G_CAP); etq_count_launch();
  ETQ_TRY(residual());
  ETQ_TRY(read_sc());
  const double bnorm = std::sqrt(P.hscal[G_CAP]);
  const double beta0 = std::sqrt(P.hscal[G_BETA]);
  ETQ_CHECK(cudaMemcpyAsync(P.ghist, &beta0, sizeof(double), cudaMemcpyHostToDevice, st));
  // graph of one Arnoldi step
  const int key = (int)kind * 2 + (reduced ? 1 : 0);
  if (P.params.use_graphs && (P.gmres_graph == nullptr || P.gmres_graph_key != key)) {
    if (P.gmres_graph) { cudaGraphExecDestroy(P.gmres_graph); P.gmres_graph = nullptr; }
    cudaGraph_t graph;
    const int64_t before = etq_launch_total();
    ETQ_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    etq_status s = arnoldi_step(P, reduced, kind, st);
    k_store_hcol<<<1, 64, 0, st>>>(P.gH, P.gsm + gseg(m, 5), sc, m); etq_count_launch();
    k_gmres_scalar<<<1, 32, 0, st>>>(sc, P.gH, P.gsm, m, P.ghist, P.ghist_cap); etq_count_launch();
    k_set_vnext<<<grid_for(N, BS, 4096), BS, 0, st>>>(P.gV, N, P.gld, P.gW, sc); etq_count_launch();
    cudaError_t e = cudaStreamEndCapture(st, &graph);
    P.gmres_graph_nodes = etq_launch_total() - before;
    etq_count_launch(-P.gmres_graph_nodes);
    if (s < 0) return s;
    ETQ_CHECK(e);
    ETQ_CHECK(cudaGraphInstantiate(&P.gmres_graph, graph, 0));
    cudaGraphDestroy(graph);
    P.gmres_graph_key = key;
  }
  int restarts = 0;
  bool converged = std::sqrt(P.hscal[G_BETA]) <= tol_abs;
  int status = 0;
  while (!converged) {
    if (std::sqrt(P.hscal[G_BETA]) <= tol_abs) { converged = true; break; }
    if ((int)P.hscal[G_TOT] >= maxit) break;
    k_cycle_init<<<grid_for(N, BS, 4096), BS, 0, st>>>(P.gV, N, P.gW, sc, P.gsm, m); etq_count_launch();
    for (int j = 0; j < m; ++j) {
      if (P.params.use_graphs) {
        ETQ_CHECK(cudaGraphLaunch(P.gmres_graph, st));
        etq_count_launch(P.gmres_graph_nodes);
      } else {
        ETQ_TRY(arnoldi_step(P, reduced, kind, st));
        k_store_hcol<<<1, 64, 0, st>>>(P.gH, P.gsm + gseg(m, 5), sc, m); etq_count_launch();
        k_gmres_scalar<<<1, 32, 0, st>>>(sc, P.gH, P.gsm, m, P.ghist, P.ghist_cap); etq_count_launch();
        k_set_vnext<<<grid_for(N, BS, 4096), BS, 0, st>>>(P.gV, N, P.gld, P.gW, sc); etq_count_launch();
      }
      ETQ_TRY(read_sc());
      if (P.hscal[G_DONE] != 0.0 || P.hscal[G_BREAK] != 0.0 || (int)P.hscal[G_TOT] >= maxit) break;
    }
    if (P.hscal[G_DONE] < 0.0) { status = ETQ_ENAN; break; }
    // x += M^{-1} (V_k y)
    k_trisolve<<<1, 32, 0, st>>>(P.gH, P.gsm, sc, m); etq_count_launch();
    ETQ_CHECK(cudaMemsetAsync(P.gU, 0, sizeof(double) * N, st));
    k_multiaxpy<<<grid_for(N, BS, 4096), BS, 0, st>>>(P.gU, P.gV, N, P.gld, P.gsm + gseg(m, 3), sc, G_J, 0, -1.0);
    etq_count_launch();
    ETQ_TRY(oseen_precond_apply(P, kind, P.gU, P.gZ, st));
    k_axpy<<<grid_for(N, BS, 4096), BS, 0, st>>>(x, P.gZ, N); etq_count_launch();
    ++restarts;
    const bool est_conv = P.hscal[G_DONE] > 0.0;
    const bool brk = P.hscal[G_BREAK] != 0.0;
    ETQ_TRY(residual());
    ETQ_TRY(read_sc());
    if (est_conv) { converged = true; break; }
    if (brk && std::sqrt(P.hscal[G_BETA]) <= tol_abs) { converged = true; break; }
  }
  ETQ_CHECK(cudaEventRecord(P.ev_t1, st));
  ETQ_CHECK(cudaEventSynchronize(P.ev_t1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1);
  const int iters = (int)P.hscal[G_TOT];
  const double true_res = std::sqrt(P.hscal[G_BETA]);
  if (p0_res_norm) *p0_res_norm = std::sqrt(P.hscal[G_NRM_P0]);
  if (rep) {
    rep->iterations = iters; rep->converged = converged ? 1 : 0; rep->restarts = restarts; rep->status = status;
    rep->abs_res = true_res; rep->rel_res = bnorm > 0 ? true_res / bnorm : 0.0; rep->ms_total = ms;
    if (rep->history && rep->history_cap > 0) {
      const int k = std::min(iters + 1, rep->history_cap);
      ETQ_CHECK(cudaMemcpy(rep->history, P.ghist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
  }
  if (status < 0) return status;
  return converged ? ETQ_OK : ETQ_NOT_CONVERGED;
}

// z = M_S1^{-1} r = Ap^{-1} F1 Mp^{-1} r on the Q1 block (test hook; no sign change)
etq_status pcd_schur_apply(const Problem& P, const double* r, double* z, cudaStream_t st) {
  NvtxRange nvtx_("PCD Schur apply");
  if (!P.pcd_ready) return ETQ_ENOTSETUP;
  qk_cheb(P, r, P.pw[0], P.params.mass_cheb_steps, nullptr, st);
  k_spmv1<<<grid_for(P.F1.nslices * 32, BS, 4096), BS, 0, st>>>(P.F1, P.pw[0], P.pw[1], 1.0, nullptr); etq_count_launch();
  return ap_solve(P, P.apH, P.pw[1], z, P.dscal + S_APSUM, nullptr, st);
}

// ---------------------------------------------------------------- two-stage driver
namespace {
__global__ void k_copy_zero_p0(const double* b, double* out, int64_t p0_from, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < p0_from ? b[i] : 0.0;
}
}  // namespace

// b_red = [f; g1; 0] into P.gU (used by reduced GMRES as its right-hand side buffer)
etq_status make_reduced_rhs(Problem& P, const double* b, double** bred) {
  if (!P.kv[9]) ETQ_TRY(dalloc(&P.kv[9], P.N));
  k_copy_zero_p0<<<grid_for(P.N, BS, 4096), BS, 0, P.stream>>>(b, P.kv[9], P.n_u + P.g.nk, P.N); etq_count_launch();
  *bred = P.kv[9];
  return ETQ_OK;
}

double host_norm(Problem& P, const double* v, int64_t n) {
  k_dot2<<<grid_for(n, BS, RED_BLOCKS), BS, 0, P.stream>>>(v, v, n, P.red[0], 10, P.dscal + 30);
  etq_count_launch();
  double h = 0.0;
  cudaMemcpyAsync(&h, P.dscal + 30, sizeof(double), cudaMemcpyDeviceToHost, P.stream);
  cudaStreamSynchronize(P.stream);
  return std::sqrt(h);
}

// Two-stage PCD: Step I GMRES on the reduced system with PCD to c*eta*||b_red||,
// Step II GMRES on the full system with M1 from [u1*; q1*; 0] to eta*||b||.  bound[0] = ||z*||,
// bound[1] = sqrt(c^2 eta^2 ||b_red||^2 + ||g0 - B0 u1*||^2) (Prop 3.3, reading R16).
etq_status two_stage_run(Problem& P, const double* b, double* x, double eta, double c, int restart, int maxit,
                         etq_report* r1, etq_report* r2, double* bound) {
  NvtxRange nvtx_("two-stage PCD");
  if (!P.pcd_ready || !P.m1_ready) return ETQ_ENOTSETUP;
  cudaStream_t st = P.stream;
  double* bred;
  ETQ_TRY(make_reduced_rhs(P, b, &bred));
  const double nb_red = host_norm(P, bred, P.N), nb = host_norm(P, b, P.N);
  ETQ_CHECK(cudaMemsetAsync(x, 0, sizeof(double) * P.N, st));
  etq_status s1 = gmres_run(P, true, ETQ_PC_OSEEN_PCD1, bred, x, c * eta * nb_red, restart, maxit, r1, nullptr);
  if (s1 < 0) return s1;
  // transition residual z* of [u1*; q1*; 0] in the full system
  launch_saddle_ex(P, false, x, P.gW, nullptr, nullptr, 0, nullptr, nullptr, st);
  k_bsub<<<grid_for(P.N, BS, 4096), BS, 0, st>>>(P.gW, b, P.N); etq_count_launch();
  const double zstar = host_norm(P, P.gW, P.N);
  const double rp0 = host_norm(P, P.gW + P.n_u + P.g.nk, P.g.n0);
  if (bound) {
    bound[0] = zstar;
    bound[1] = std::sqrt((c * eta * nb_red) * (c * eta * nb_red) + rp0 * rp0);
  }
  etq_status s2 = gmres_run(P, false, ETQ_PC_OSEEN_M1, b, x, eta * nb, restart, maxit, r2, nullptr);
  if (s2 < 0) return s2;
  return (s1 == ETQ_OK && s2 == ETQ_OK) ? ETQ_OK : ETQ_NOT_CONVERGED;
}
