// TMA geometry probe: dims d0 d1 d2, box b0 b1, coords c0 c1 c2, dst offset (doubles)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Maps { CUtensorMap a; };
__global__ void probe(const __grid_constant__ Maps m, double* out, int c0, int c1, int c2, unsigned bytes, int dst) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ alignas(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(smem_u32(sm + dst)), "l"(reinterpret_cast<unsigned long long>(&m.a)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n"
               ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < (int)(bytes / 8); i += blockDim.x) out[i] = sm[dst + i];
}
int main(int argc, char** argv) {
  if (argc < 10) { printf("usage\n"); return 2; }
  int d0 = atoi(argv[1]), d1 = atoi(argv[2]), d2 = atoi(argv[3]), b0 = atoi(argv[4]), b1 = atoi(argv[5]);
  int c0 = atoi(argv[6]), c1 = atoi(argv[7]), c2 = atoi(argv[8]), dst = atoi(argv[9]);
  size_t n = (size_t)d0 * d1 * d2;
  std::vector<double> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (double)i + 1;
  double *d, *o;
  cudaMalloc(&d, n * 8);
  cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  Maps m;
  memset(&m, 0, sizeof(m));
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t str[2] = {(cuuint64_t)d0 * 8, (cuuint64_t)d0 * d1 * 8};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned bytes = b0 * b1 * 8;
  probe<<<1, 128, 40000>>>(m, o, c0, c1, c2, bytes, dst);
  printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> rr(b0 * b1);
  cudaMemcpy(rr.data(), o, rr.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < b1; ++y)
    for (int x = 0; x < b0; ++x) {
      int gx = c0 + x, gy = c1 + y;
      double ex = (gx >= 0 && gx < d0 && gy >= 0 && gy < d1 && c2 >= 0 && c2 < d2) ? h[(size_t)c2 * d0 * d1 + gy * d0 + gx] : 0.0;
      if (rr[y * b0 + x] != ex) ++bad;
    }
  printf("dims %d %d %d box %d %d at %d %d %d dst %d: enc=%d %s bad=%d\n", d0, d1, d2, b0, b1, c0, c1, c2, dst, (int)r,
         cudaGetErrorString(e), bad);
  return 0;
}
