// Minimal TMA probe: one 3D box load through an mbarrier, variants by flags:
//  argv[1] dtype: 0 f64, 1 u64, 2 f32(x2 width)   argv[2] coords: 0 (-1,-1,1), 1 (0,0,1)
//  argv[3] desc: 0 grid_constant param, 1 global memory copy   argv[4] smem: 0 dynamic, 1 manual 1024 align
//  argv[5] box cols (default 34)   argv[6] l2promo 0 none / 1 256B
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

struct Maps { CUtensorMap a[1]; };

__global__ void probe(const __grid_constant__ Maps m, const CUtensorMap* gdesc, int use_g, int align1024, double* out,
                      int c0, int c1, int c2, unsigned bytes, int nout) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ alignas(8) unsigned long long bar;
  unsigned char* base = smraw;
  if (align1024) base = (unsigned char*)(((unsigned long long)smraw + 1023) & ~1023ull);
  double* sm = (double*)base;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    const CUtensorMap* mp = use_g ? gdesc : &m.a[0];
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(smem_u32(sm)), "l"(reinterpret_cast<unsigned long long>(mp)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < nout; i += blockDim.x) out[i] = sm[i];
  if (threadIdx.x == 0) out[nout] = (double)(smem_u32(sm) & 1023);
}

int main(int argc, char** argv) {
  int dt = argc > 1 ? atoi(argv[1]) : 0, cz = argc > 2 ? atoi(argv[2]) : 0, useg = argc > 3 ? atoi(argv[3]) : 0;
  int a1024 = argc > 4 ? atoi(argv[4]) : 0, bw = argc > 5 ? atoi(argv[5]) : 34, l2 = argc > 6 ? atoi(argv[6]) : 1;
  const int n3 = 40, n2 = 5, np = 3;
  std::vector<double> h(n3 * n2 * np);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 4096 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  Maps m;
  memset(&m, 0, sizeof(m));
  int mult = dt == 2 ? 2 : 1;
  CUtensorMapDataType ty = dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t dims[3] = {(cuuint64_t)n3 * mult, n2, np};
  cuuint64_t str[2] = {n3 * 8, (cuuint64_t)n3 * n2 * 8};
  cuuint32_t box[3] = {(cuuint32_t)(bw * mult), 9, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m.a[0], ty, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* gd;
  cudaMalloc(&gd, sizeof(CUtensorMap));
  cudaMemcpy(gd, &m.a[0], sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  int c0 = cz ? 0 : -1 * mult, c1 = cz ? 0 : -1, c2 = 1;
  unsigned bytes = bw * 9 * 8;
  int nout = bw * 9;
  size_t smem = bytes + 2048;
  probe<<<1, 128, smem>>>(m, gd, useg, a1024, o, c0, c1, c2, bytes, nout);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> rr(nout + 1);
  cudaMemcpy(rr.data(), o, rr.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int jj = 0; jj < 9; ++jj)
    for (int kk = 0; kk < bw; ++kk) {
      int j = jj + c1, k = kk + c0 / mult;
      double ex = (j >= 0 && j < n2 && k >= 0 && k < n3) ? h[(size_t)1 * n3 * n2 + j * n3 + k] : 0.0;
      if (rr[jj * bw + kk] != ex) ++bad;
    }
  printf("dt=%d coords0=%d gdesc=%d a1024=%d bw=%d l2=%d encode=%d -> %s, mismatches %d, smem%%1024=%g\n", dt, cz, useg,
         a1024, bw, l2, (int)r, cudaGetErrorString(e), bad, rr[nout]);
  return e != cudaSuccess;
}
