// Pointwise kernels of the path: lagged Spitzer face diffusivity (A3) and the
// PCG vector updates / deterministic dot-product reductions (A7).
#include "sts_common.cuh"

namespace sts {

// ----------------------------------------------------------------------------
// A3: kappa_f = kappa0 f_c(r_f) beta_Tcut(Tf) Tf^(5/2), Tf = (T_L + T_R)/2
// (PAPER.md:33 lagged diffusivity, :173 boxed term, :183 f_c, :187 beta_Tcut)
// ----------------------------------------------------------------------------
__device__ __forceinline__ double spitzer(double Tf, double kappa0, double T_cut) {
  double k = kappa0 * Tf * Tf * sqrt(Tf);           // kappa0 T^(5/2)
  if (T_cut > 0.0 && Tf < T_cut) {
    const double x = Tf / T_cut;
    k *= x * x * sqrt(x);                            // beta = (T/T_cut)^(5/2)
  }
  return k;
}

__device__ __forceinline__ double fc_profile(double r, double r0, double w) {
  return w > 0.0 ? 0.5 * (1.0 - tanh((r - r0) / w)) : 1.0;
}

__global__ void face_kappa_kernel(Geo G, FieldV T, double* __restrict__ k1, double* __restrict__ k2,
                                  double* __restrict__ k3, double kappa0, double T_cut, double fc_r0,
                                  double fc_w, const double* __restrict__ x1f, const double* __restrict__ x1c) {
  const long long n = (long long)G.nl * G.plane;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int il = (int)(e / G.plane);
    const long long rem = e - (long long)il * G.plane;
    const int j = (int)(rem / G.n3);
    const int k = (int)(rem - (long long)j * G.n3);
    const int ig = G.i0 + il;
    const double Tc = T.p[e];
    // r-face (i+1/2): needs T at il+1 (hi halo on the last local plane)
    double v1 = 0.0;
    if (ig + 1 < G.n1g) {
      const double Tn = (il + 1 < G.nl) ? T.p[e + G.plane] : T.hi[rem];
      v1 = spitzer(0.5 * (Tc + Tn), kappa0, T_cut) * fc_profile(x1f[ig + 1], fc_r0, fc_w);
    }
    double v2 = 0.0;
    if (j + 1 < G.n2) v2 = spitzer(0.5 * (Tc + T.p[e + G.n3]), kappa0, T_cut) * fc_profile(x1c[ig], fc_r0, fc_w);
    double v3 = 0.0;
    if (G.periodic3 || k + 1 < G.n3) {
      const long long en = (k + 1 < G.n3) ? e + 1 : e - k;  // wrap to k = 0
      v3 = spitzer(0.5 * (Tc + T.p[en]), kappa0, T_cut) * fc_profile(x1c[ig], fc_r0, fc_w);
    }
    k1[e] = v1;
    k2[e] = v2;
    k3[e] = v3;
  }
}

void launch_face_kappa(const Geo& G, FieldV T, double* k1, double* k2, double* k3, double kappa0,
                       double T_cut, double fc_r0, double fc_w, const double* x1f_d, const double* x1c_d,
                       cudaStream_t st) {
  const long long n = (long long)G.nl * G.plane;
  if (n == 0) return;
  long long nb = (n + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  face_kappa_kernel<<<(int)nb, 256, 0, st>>>(G, T, k1, k2, k3, kappa0, T_cut, fc_r0, fc_w, x1f_d, x1c_d);
  STS_CUDA(cudaGetLastError());
}

// ----------------------------------------------------------------------------
// A7: PCG pointwise updates (Fig. 1) and reductions
// ----------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// x += alpha p ; r -= alpha y ; z = r d ; partial r.z   (z is not stored: p-update recomputes it)
template <int NC>
__global__ void __launch_bounds__(256) pcg_update_kernel(long long n, long long cs, double* __restrict__ x,
                                                         double* __restrict__ r, const double* __restrict__ p,
                                                         const double* __restrict__ y, const double* __restrict__ d,
                                                         const PcgScal* __restrict__ sc, double* __restrict__ partials,
                                                         long long pstride) {
  double alpha[NC];
  bool act[NC];
  bool any = false;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    act[q] = !sc[q].done;
    alpha[q] = sc[q].alpha;
    any = any || act[q];
  }
  if (!any) return;
  double acc[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) acc[q] = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const double de = d[e];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      if (!act[q]) continue;
      const long long o = e + q * cs;
      x[o] += alpha[q] * p[o];
      const double rn = r[o] - alpha[q] * y[o];
      r[o] = rn;
      acc[q] += rn * (rn * de);
    }
  }
  __shared__ double red[NC][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const double s = warp_sum_d(acc[q]);
    if (lane == 0) red[q][wid] = s;
  }
  __syncthreads();
  if (threadIdx.x < NC) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[threadIdx.x][w];
    partials[threadIdx.x * pstride + blockIdx.x] = s;
  }
}

template <int NC>
__global__ void __launch_bounds__(256) pcg_pupdate_kernel(long long n, long long cs, double* __restrict__ p,
                                                          const double* __restrict__ r, const double* __restrict__ d,
                                                          const PcgScal* __restrict__ sc) {
  double beta[NC];
  bool act[NC];
  bool any = false;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    act[q] = !sc[q].done;
    beta[q] = sc[q].beta;
    any = any || act[q];
  }
  if (!any) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const double de = d[e];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      if (!act[q]) continue;
      const long long o = e + q * cs;
      p[o] = r[o] * de + beta[q] * p[o];
    }
  }
}

void launch_pcg_update(int ncomp, long long n, long long cs, double* x, double* r, const double* p,
                       const double* y, const double* d, const PcgScal* sc, double* partials,
                       long long pstride, cudaStream_t st) {
  switch (ncomp) {
    case 1: pcg_update_kernel<1><<<PW_BLOCKS, 256, 0, st>>>(n, cs, x, r, p, y, d, sc, partials, pstride); break;
    case 2: pcg_update_kernel<2><<<PW_BLOCKS, 256, 0, st>>>(n, cs, x, r, p, y, d, sc, partials, pstride); break;
    case 3: pcg_update_kernel<3><<<PW_BLOCKS, 256, 0, st>>>(n, cs, x, r, p, y, d, sc, partials, pstride); break;
    default: throw Error{STS_ERR_ARG, "ncomp"};
  }
  STS_CUDA(cudaGetLastError());
}

void launch_pcg_pupdate(int ncomp, long long n, long long cs, double* p, const double* r, const double* d,
                        const PcgScal* sc, cudaStream_t st) {
  switch (ncomp) {
    case 1: pcg_pupdate_kernel<1><<<PW_BLOCKS, 256, 0, st>>>(n, cs, p, r, d, sc); break;
    case 2: pcg_pupdate_kernel<2><<<PW_BLOCKS, 256, 0, st>>>(n, cs, p, r, d, sc); break;
    case 3: pcg_pupdate_kernel<3><<<PW_BLOCKS, 256, 0, st>>>(n, cs, p, r, d, sc); break;
    default: throw Error{STS_ERR_ARG, "ncomp"};
  }
  STS_CUDA(cudaGetLastError());
}

// scalar recurrences of Fig. 1 (one thread per component)
__device__ void pcg_phase(const double* sums, int c, int nq, int phase, PcgScal* sc, double rtol2) {
  PcgScal& s = sc[c];
  if (phase == PH_R0) {
    s.rz = sums[c * nq + 0];
    s.thresh = rtol2 * sums[c * nq + 1];
    s.iters = 0;
    s.done = (s.rz <= s.thresh) ? 1 : 0;   // DESIGN R8: already converged -> 0 iterations
    s.beta = 0.0;
  } else if (phase == PH_AP) {
    if (s.done) return;
    s.pAp = sums[c * nq];
    s.alpha = s.rz / s.pAp;                // alpha_k = r_r / (p_k . y_k)
  } else if (phase == PH_RZ) {
    if (s.done) return;
    s.rz_old = s.rz;
    s.rz = sums[c * nq];                   // r_r = r_{k+1} . z_{k+1}
    s.iters += 1;
    if (s.rz <= s.thresh) s.done = 1;      // check r_r for convergence
    else s.beta = s.rz / s.rz_old;         // beta_k = r_r / r_old
  }
}

// one CTA: fixed-order sums of the per-CTA partials (deterministic), then the phase
__global__ void __launch_bounds__(1024) pcg_reduce_kernel(const double* __restrict__ partials, long long pstride,
                                                          int nblocks, int ncomp, int nq, double* __restrict__ sums,
                                                          int phase, PcgScal* sc, double rtol2) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int row = 0; row < ncomp * nq; ++row) {
    const double* src = partials + row * pstride;
    double a = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) a += src[b];
    a = warp_sum_d(a);
    if (lane == 0) red[wid] = a;
    __syncthreads();
    if (wid == 0) {
      double v = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
      v = warp_sum_d(v);
      if (lane == 0) sums[row] = v;
    }
    __syncthreads();
  }
  if (phase != PH_NONE && threadIdx.x < ncomp) pcg_phase(sums, threadIdx.x, nq, phase, sc, rtol2);
}

__global__ void pcg_scalar_kernel(const double* sums, int ncomp, int nq, int phase, PcgScal* sc, double rtol2) {
  if (threadIdx.x < ncomp) pcg_phase(sums, threadIdx.x, nq, phase, sc, rtol2);
}

void launch_pcg_reduce(const double* partials, long long pstride, int nblocks, int ncomp, int nq, double* sums,
                       int phase, PcgScal* sc, double rtol2, cudaStream_t st) {
  pcg_reduce_kernel<<<1, 1024, 0, st>>>(partials, pstride, nblocks, ncomp, nq, sums, phase, sc, rtol2);
  STS_CUDA(cudaGetLastError());
}

void launch_pcg_scalar(const double* sums, int ncomp, int nq, int phase, PcgScal* sc, double rtol2,
                       cudaStream_t st) {
  pcg_scalar_kernel<<<1, 32, 0, st>>>(sums, ncomp, nq, phase, sc, rtol2);
  STS_CUDA(cudaGetLastError());
}

}  // namespace sts
