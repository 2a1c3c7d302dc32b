// Standalone probe: one 3D TMA box {32,32,8} of fp64 from a {pw, ph, 8} tensor at given coordinates,
// checked against the expected values (zero outside).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int x, int y, double* out, int pre) {
  extern __shared__ unsigned char raw[];
  const unsigned base = (unsigned)__cvta_generic_to_shared(raw);
  const unsigned off = ((base + 1023u) & ~1023u) - base;
  double* V = reinterpret_cast<double*>(raw + off);
  unsigned long long* barp = reinterpret_cast<unsigned long long*>(V + 8192);
  const unsigned bar = (unsigned)__cvta_generic_to_shared(barp);
  if (threadIdx.x == 0) {
    if (pre) asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(&tm), "r"(x), "r"(y), "r"(0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(65536) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"((unsigned)__cvta_generic_to_shared(V)), "l"(&tm), "r"(x), "r"(y), "r"(0), "r"(bar) : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(bar) : "memory");
  for (int t = threadIdx.x; t < 8192; t += blockDim.x) out[blockIdx.x * 8192 + t] = V[t];
}

int main(int argc, char** argv) {
  const int pw = atoi(argv[1]), ph = atoi(argv[2]), x = atoi(argv[3]), y = atoi(argv[4]);
  const int ncta = argc > 5 ? atoi(argv[5]) : 1, pre = argc > 6 ? atoi(argv[6]) : 0;
  const size_t sz = (size_t)8 * pw * ph;
  std::vector<double> h(sz);
  for (size_t i = 0; i < sz; ++i) h[i] = (double)i + 1.0;
  double *d, *o;
  cudaMalloc(&d, sz * 8); cudaMalloc(&o, (size_t)ncta * 8192 * 8);
  cudaMemcpy(d, h.data(), sz * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  alignas(64) CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)pw, (cuuint64_t)ph, 8};
  const cuuint64_t str[2] = {(cuuint64_t)pw * 8, (cuuint64_t)pw * ph * 8};
  const cuuint32_t box[3] = {32, 32, 8}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 65536 + 1024 + 64;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_probe<<<ncta, 256, smem>>>(tm, x, y, o, pre);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> ho((size_t)ncta * 8192);
  cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int c = 0; c < ncta; ++c)
    for (int t = 0; t < 8192; ++t) {
      const int z = t >> 10, jj = (t >> 5) & 31, ii = t & 31, xx = x + ii, yy = y + jj;
      const double ex = (xx >= 0 && yy >= 0 && xx < pw && yy < ph) ? h[(size_t)z * pw * ph + (size_t)yy * pw + xx] : 0.0;
      if (ho[(size_t)c * 8192 + t] != ex) ++bad;
    }
  printf("pw=%d ph=%d x=%d y=%d ncta=%d pre=%d encode=%d err=%s bad=%ld\n", pw, ph, x, y, ncta, pre, (int)r,
         cudaGetErrorString(e), bad);
  return 0;
}
