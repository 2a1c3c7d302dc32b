// device_common.cuh — device helpers shared by the kernel files of libetq: launch sizing,
// deterministic block/grid reductions, SELL-32 row products.
#pragma once
#include <utility>
#include "etq_internal.cuh"

// ================================================================ launch helpers
namespace etqd {
constexpr int BS = 256;
constexpr int MAXB = RED_MAXB;

inline int grid_for(int64_t work_items, int per_block, int cap = MAXB) {
  int64_t g = (work_items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

__device__ __forceinline__ bool is_done(const double* done) { return done && *done != 0.0; }

// programmatic dependent launch: wait until the preceding grid has completed and its writes are
// visible (a no-op when the grid was not launched as a programmatic dependent); allow the next
// grid, if launched as a programmatic dependent, to start launching
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// launch with the programmatic-stream-serialization attribute when pdl (the kernel must call
// pdl_wait() before touching anything the preceding kernel wrote)
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Linear thread index / block size (kernels may use 2D blocks).
__device__ __forceinline__ int lin_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
__device__ __forceinline__ int lin_bs() { return blockDim.x * blockDim.y * blockDim.z; }

// Block sum; the result is valid in thread 0.  Safe to call repeatedly in one kernel.
static __device__ double block_sum(double v) {
  __shared__ double sh[32];
  const int t = lin_tid();
  const int lane = t & 31, wid = t >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = (lin_bs() + 31) >> 5;
  v = (t < nw) ? sh[t] : 0.0;
  if (wid == 0) v = warp_sum(v);
  return v;
}

// Store this block's partial of NV sums into `site` and, in the last block to finish, sum the
// gridDim.x partials in a fixed order into out[0..NV).  Deterministic for a fixed grid.
// Returns true in exactly one thread (thread 0 of the last block) after out[] is written, so
// the caller can derive scalars from the finished sums.
template <int NV>
__device__ bool reduce_finish(const double (&v)[NV], RedSite site, int slot, double* out, bool grid2d = false) {
  __shared__ bool last;
  const int t = lin_tid(), bs = lin_bs();
  // linear block index / count (2D grids: blockIdx.y-major)
  const int bid = grid2d ? (int)(blockIdx.x + gridDim.x * blockIdx.y) : (int)blockIdx.x;
  const int nb = grid2d ? (int)(gridDim.x * gridDim.y) : (int)gridDim.x;
  double tot[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) tot[k] = block_sum(v[k]);
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) site.partials[(int64_t)(slot + k) * MAXB + bid] = tot[k];
    __threadfence();
    unsigned c = atomicAdd(site.counter + slot, 1u);
    last = (c == (unsigned)nb - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int i = t; i < nb; i += bs)
        s += __ldcg(site.partials + (int64_t)(slot + k) * MAXB + i);
      s = block_sum(s);
      if (t == 0) out[k] = s;
    }
    if (t == 0) site.counter[slot] = 0u;
  }
  return last && t == 0;
}

// ---------------------------------------------------------------- SELL row products
// One thread per row; entry k of the row at base + 32 k.  SELL_U entries are loaded before their
// gathers so SELL_U x 12 B of matrix data plus SELL_U gathers are in flight per thread (U = 4
// measured best among 2/4/6/8 and predicated variants, n = 1024).  Slices may carry implicit
// column indices (col = row + per-class offset) and implicit values (per-class dictionary).
#ifndef SELL_U
#define SELL_U 4
#endif
// matrix loads: read-only path (measured faster than the evict-first hint, variants A/E)
template <class T>
__device__ __forceinline__ T ld_mat(const T* p) { return __ldg(p); }
__device__ __forceinline__ double sell_row1(const Sell& A, int64_t s, int lane, const double* __restrict__ x) {
  const int64_t base = A.sptr[s] + lane;
  const int len = A.slen[s];
  const int* __restrict__ cp = A.col + base;
  const double* __restrict__ vp = A.val + base;
  double acc = 0.0;
  int k = 0;
  for (; k + SELL_U <= len; k += SELL_U) {
    int c[SELL_U]; double v[SELL_U];
#pragma unroll
    for (int u = 0; u < SELL_U; ++u) { c[u] = ld_mat(cp + (k + u) * SELL_C); v[u] = ld_mat(vp + (k + u) * SELL_C); }
#pragma unroll
    for (int u = 0; u < SELL_U; ++u) acc = fma(v[u], __ldg(x + c[u]), acc);
  }
  for (; k < len; ++k) acc = fma(ld_mat(vp + k * SELL_C), __ldg(x + ld_mat(cp + k * SELL_C)), acc);
  return acc;
}

__device__ __forceinline__ void sell_row2(const Sell& A, int64_t s, int lane, int row, const double* __restrict__ x0,
                                          const double* __restrict__ x1, double& a0, double& a1) {
  const int64_t base = A.sptr[s] + lane;
  const int len = A.slen[s];
  const double* __restrict__ vp = A.val + base;
  const int kind = A.skind ? (int)A.skind[s] : 0;
  if (kind >= 5) {   // implicit columns and values (warp-uniform branch): nothing streamed
    const int* __restrict__ off = A.stoff + (kind - 5) * 32;
    const double* __restrict__ sv = A.stval + (kind - 5) * 32;
    int k = 0;
    for (; k + SELL_U <= len; k += SELL_U) {
      int c[SELL_U]; double v[SELL_U];
#pragma unroll
      for (int u = 0; u < SELL_U; ++u) { c[u] = row + __ldg(off + k + u); v[u] = __ldg(sv + k + u); }
#pragma unroll
      for (int u = 0; u < SELL_U; ++u) { a0 = fma(v[u], __ldg(x0 + c[u]), a0); a1 = fma(v[u], __ldg(x1 + c[u]), a1); }
    }
    for (; k < len; ++k) {
      const int c = row + __ldg(off + k); const double v = __ldg(sv + k);
      a0 = fma(v, __ldg(x0 + c), a0); a1 = fma(v, __ldg(x1 + c), a1);
    }
    return;
  }
  if (kind) {   // implicit columns: col = row + offset (warp-uniform branch)
    const int* __restrict__ off = A.stoff + (kind - 1) * 32;
    int k = 0;
    for (; k + SELL_U <= len; k += SELL_U) {
      int c[SELL_U]; double v[SELL_U];
#pragma unroll
      for (int u = 0; u < SELL_U; ++u) { c[u] = row + __ldg(off + k + u); v[u] = ld_mat(vp + (k + u) * SELL_C); }
#pragma unroll
      for (int u = 0; u < SELL_U; ++u) { a0 = fma(v[u], __ldg(x0 + c[u]), a0); a1 = fma(v[u], __ldg(x1 + c[u]), a1); }
    }
    for (; k < len; ++k) {
      const int c = row + __ldg(off + k); const double v = ld_mat(vp + k * SELL_C);
      a0 = fma(v, __ldg(x0 + c), a0); a1 = fma(v, __ldg(x1 + c), a1);
    }
    return;
  }
  const int* __restrict__ cp = A.col + base;
  int k = 0;
  for (; k + SELL_U <= len; k += SELL_U) {
    int c[SELL_U]; double v[SELL_U];
#pragma unroll
    for (int u = 0; u < SELL_U; ++u) { c[u] = ld_mat(cp + (k + u) * SELL_C); v[u] = ld_mat(vp + (k + u) * SELL_C); }
#pragma unroll
    for (int u = 0; u < SELL_U; ++u) { a0 = fma(v[u], __ldg(x0 + c[u]), a0); a1 = fma(v[u], __ldg(x1 + c[u]), a1); }
  }
  for (; k < len; ++k) {
    const int c = ld_mat(cp + k * SELL_C); const double v = ld_mat(vp + k * SELL_C);
    a0 = fma(v, __ldg(x0 + c), a0); a1 = fma(v, __ldg(x1 + c), a1);
  }
}

// ---------------------------------------------------------------- matrix-free S_k (reading R21)
// (S_k v)_p / w with w = h_0^2 / 144 on every level of the scaled hierarchy (S_l / 4^l): per cell
// T of the Q1 vertex p = (a, c), (36^-1 m_x m_y - 16^-1) h^2 for each vertex pair of T, i.e.
//   7 ca cc v_p - cc (v_{p-1} + v_{p+1}) - ca (v_{p-n1} + v_{p+n1}) - 5 (corner neighbours)
// with ca, cc the numbers of cells adjacent to p along x and y (missing neighbours dropped).
// Returns the sum; *diag7 = 7 ca cc (the diagonal / w).
__device__ __forceinline__ double sk_stencil(int64_t p, int a, int c, int n, const double* __restrict__ v,
                                             double* diag7) {
  const int n1 = n + 1;
  const int ca = (a > 0) + (a < n), cc = (c > 0) + (c < n);
  const double d7 = 7.0 * (double)(ca * cc);
  double acc = d7 * __ldg(v + p);
  double ex = 0.0, ey = 0.0, co = 0.0;
  if (a > 0) ex += __ldg(v + p - 1);
  if (a < n) ex += __ldg(v + p + 1);
  if (c > 0) {
    ey += __ldg(v + p - n1);
    if (a > 0) co += __ldg(v + p - n1 - 1);
    if (a < n) co += __ldg(v + p - n1 + 1);
  }
  if (c < n) {
    ey += __ldg(v + p + n1);
    if (a > 0) co += __ldg(v + p + n1 - 1);
    if (a < n) co += __ldg(v + p + n1 + 1);
  }
  acc -= (double)cc * ex + (double)ca * ey + 5.0 * co;
  *diag7 = d7;
  return acc;
}
}  // namespace etqd
