// Pointwise kernels of the path: lagged Spitzer face diffusivity (A3) and the
// PCG vector updates / deterministic dot-product reductions (A7).
#include "sts_common.cuh"
#include "pcg.cuh"

#include <algorithm>

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

// one thread per (theta, phi) column marching along r over planes [ib, ie): T of the
// next plane is loaded once (it is this plane's r-face neighbour and the next plane's
// own value), the phi neighbour comes from the next lane (lane 31 loads it), the theta
// neighbour is a coalesced row load; streaming stores (the face fields are re-read by a
// later pass, after far more than L2 has streamed through)
constexpr int FK_T = 256;
__global__ void __launch_bounds__(FK_T) face_kappa_kernel(Geo G, FieldV T, double* __restrict__ k1,
                                                          double* __restrict__ k2, double* __restrict__ k3,
                                                          double kappa0, double T_cut, double fc_r0, double fc_w,
                                                          const double* __restrict__ x1f,
                                                          const double* __restrict__ x1c, int ic) {
  const int k = blockIdx.x * FK_T + threadIdx.x, j = blockIdx.y;
  const int ib = blockIdx.z * ic, ie = min(ib + ic, G.nl);
  const bool in = k < G.n3;
  const bool jp = j + 1 < G.n2, kp = G.periodic3 || k + 1 < G.n3;
  const int kn = (k + 1 < G.n3) ? k + 1 : 0;    // (wrap to k = 0)
  const long long col = (long long)j * G.n3;
  const int lane = threadIdx.x & 31;
  // the phi neighbour is the next lane's own value unless it lies in another warp / wraps
  const bool shfl_ok = lane < 31 && k + 1 < G.n3;
  double Tc = (in && ib < ie) ? __ldg(T.p + (long long)ib * G.plane + col + k) : 0.0;
  for (int il = ib; il < ie; ++il) {
    const long long e = (long long)il * G.plane + col + k;
    const int ig = G.i0 + il;
    double Tn = 0.0;
    if (in && ig + 1 < G.n1g) Tn = (il + 1 < G.nl) ? __ldg(T.p + e + G.plane) : T.hi[col + k];
    const double Tk_s = __shfl_down_sync(0xffffffffu, Tc, 1);
    if (in) {
      const double Tk = shfl_ok ? Tk_s : __ldg(T.p + (long long)il * G.plane + col + kn);
      const double fcc = fc_profile(x1c[ig], fc_r0, fc_w);
      const double v1 = (ig + 1 < G.n1g) ? spitzer(0.5 * (Tc + Tn), kappa0, T_cut) * fc_profile(x1f[ig + 1], fc_r0, fc_w)
                                         : 0.0;
      const double v2 = jp ? spitzer(0.5 * (Tc + __ldg(T.p + e + G.n3)), kappa0, T_cut) * fcc : 0.0;
      const double v3 = kp ? spitzer(0.5 * (Tc + Tk), kappa0, T_cut) * fcc : 0.0;
      __stcs(k1 + e, v1);
      __stcs(k2 + e, v2);
      __stcs(k3 + e, v3);
    }
    Tc = Tn;
  }
}

// The same pass with two phi columns per thread (n3 even, 16 B-aligned arrays): double2
// loads / streaming stores, the next-but-one plane prefetched (two loads in flight per
// column pair besides the theta row), f_c evaluated once per plane (warp-uniform); the
// phi neighbour of the pair's second column is the next lane's first (lane 31 loads it).
constexpr int FK2_T = 128;
__global__ void __launch_bounds__(FK2_T) face_kappa2_kernel(Geo G, FieldV T, double* __restrict__ k1,
                                                            double* __restrict__ k2, double* __restrict__ k3,
                                                            double kappa0, double T_cut, double fc_r0, double fc_w,
                                                            const double* __restrict__ x1f,
                                                            const double* __restrict__ x1c, int ic) {
  const int k = 2 * (blockIdx.x * FK2_T + threadIdx.x), j = blockIdx.y;
  const int ib = blockIdx.z * ic, ie = min(ib + ic, G.nl);
  const bool in = k < G.n3;
  const bool jp = j + 1 < G.n2, kp = G.periodic3 || k + 2 < G.n3;
  const int kn = (k + 2 < G.n3) ? k + 2 : 0;    // (wrap to k = 0)
  const long long col = (long long)j * G.n3 + k;
  const int lane = threadIdx.x & 31;
  const bool shfl_ok = lane < 31 && k + 2 < G.n3;
  auto ld2 = [&](long long e) { return __ldg(reinterpret_cast<const double2*>(T.p + e)); };
  // T of local plane il (il = nl: the halo plane above, or nothing at r_max)
  auto plane = [&](int il) -> double2 {
    if (!in || il >= ie + 1 || G.i0 + il >= G.n1g) return make_double2(0.0, 0.0);
    if (il < G.nl) return ld2((long long)il * G.plane + col);
    return T.hi ? *reinterpret_cast<const double2*>(T.hi + col) : make_double2(0.0, 0.0);
  };
  double2 Tc = plane(ib), Tn = plane(ib + 1);
  for (int il = ib; il < ie; ++il) {
    const double2 Tnn = plane(il + 2);
    const long long e = (long long)il * G.plane + col;
    const int ig = G.i0 + il;
    const double Tk_s = __shfl_down_sync(0xffffffffu, Tc.x, 1);
    if (in) {
      const double Tk = shfl_ok ? Tk_s : __ldg(T.p + (long long)il * G.plane + (long long)j * G.n3 + kn);
      const double fcc = fc_profile(x1c[ig], fc_r0, fc_w);
      const bool rp = ig + 1 < G.n1g;
      const double fcf = rp ? fc_profile(x1f[ig + 1], fc_r0, fc_w) : 0.0;
      double2 v1, v2, v3;
      v1.x = rp ? spitzer(0.5 * (Tc.x + Tn.x), kappa0, T_cut) * fcf : 0.0;
      v1.y = rp ? spitzer(0.5 * (Tc.y + Tn.y), kappa0, T_cut) * fcf : 0.0;
      if (jp) {
        const double2 Tt = ld2(e + G.n3);
        v2.x = spitzer(0.5 * (Tc.x + Tt.x), kappa0, T_cut) * fcc;
        v2.y = spitzer(0.5 * (Tc.y + Tt.y), kappa0, T_cut) * fcc;
      } else {
        v2 = make_double2(0.0, 0.0);
      }
      v3.x = spitzer(0.5 * (Tc.x + Tc.y), kappa0, T_cut) * fcc;
      v3.y = kp ? spitzer(0.5 * (Tc.y + Tk), kappa0, T_cut) * fcc : 0.0;
      __stcs(reinterpret_cast<double2*>(k1 + e), v1);
      __stcs(reinterpret_cast<double2*>(k2 + e), v2);
      __stcs(reinterpret_cast<double2*>(k3 + e), v3);
    }
    Tc = Tn;
    Tn = Tnn;
  }
}

// Face coefficients of the isotropic operator with the metrics folded in, for the
// merged PCG pass (once per solve): K1 = k1 F1r F1t F1p (r face i+1/2), K2 = k2 F2r
// F2t F2p (theta face j+1/2), K3 = k3 F2r F3t F3p (phi face k+1/2, periodic wrap),
// WV = w Vr Vt Vp -- each product in the association the stencil kernels use, so the
// pass computes bit-identical coefficients; zero where the face is a wall.
__global__ void iso_premul_kernel(Geo G, const double* __restrict__ k1, const double* __restrict__ k2,
                                  const double* __restrict__ k3, const double* __restrict__ w,
                                  double* __restrict__ K1, double* __restrict__ K2, double* __restrict__ K3,
                                  double* __restrict__ WV) {
  // grid: (phi chunks of 256, theta rows, local r planes) -- no index divisions
  const Metrics& M = G.m;
  const bool per = G.periodic3 != 0, kself = per && G.n3 == 1;
  const int k = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, il = blockIdx.z;
  if (k >= G.n3) return;
  const long long e = (long long)il * G.plane + (long long)j * G.n3 + k;
  const int ig = G.i0 + il;
  const bool ip = ig + 1 < G.n1g, jp = j + 1 < G.n2, kp = !kself && (per || k + 1 < G.n3);
  K1[e] = ip ? k1[e] * M.F1r[ig] * (M.F1t[j] * M.F1p[k]) : 0.0;
  K2[e] = jp ? k2[e] * M.F2r[ig] * (M.F2t[j] * M.F2p[k]) : 0.0;
  K3[e] = kp ? k3[e] * M.F2r[ig] * (M.F3t[j] * M.F3p[k]) : 0.0;
  WV[e] = (w ? w[e] : 1.0) * M.Vr[ig] * (M.Vt[j] * M.Vp[k]);
}

void launch_iso_premul(const Geo& G, const double* k1, const double* k2, const double* k3, const double* w,
                       double* K1, double* K2, double* K3, double* WV, cudaStream_t st) {
  if ((long long)G.nl * G.plane == 0) return;
  STS_REQUIRE(G.n2 <= 65535 && G.nl <= 65535, "grid too large for the coefficient pass");
  const dim3 grid((G.n3 + 255) / 256, G.n2, G.nl);
  iso_premul_kernel<<<grid, 256, 0, st>>>(G, k1, k2, k3, w, K1, K2, K3, WV);
  STS_CUDA(cudaGetLastError());
}

void launch_face_kappa(const Geo& G, FieldV T, double* k1, double* k2, double* k3, double kappa0,
                       double T_cut, double fc_r0, double fc_w, const double* x1f_d, const double* x1c_d,
                       cudaStream_t st) {
  if ((long long)G.nl * G.plane == 0) return;
  STS_REQUIRE(G.n2 <= 65535, "grid too large for the face-kappa pass");
  auto a16 = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = G.n3 % 2 == 0 && a16(T.p) && a16(T.hi) && a16(k1) && a16(k2) && a16(k3);
  const int tpb = vec ? FK2_T : FK_T;
  const int nbx = (vec ? G.n3 / 2 + FK2_T - 1 : G.n3 + FK_T - 1) / tpb;
  // ~8 resident blocks per SM x 148 SMs x 4 waves of columns, chunks of >= 8 planes
  // (the vectorised pass: 16 blocks of 128 threads per SM, chunks of >= 16 planes)
  const long long cols = (long long)nbx * G.n2;
  const long long want = vec ? 148LL * 16 * 4 : 148LL * 8 * 4;
  const int minc = vec ? 16 : 8;
  int nch = (int)std::max(1LL, std::min<long long>((want + cols - 1) / cols, (G.nl + minc - 1) / minc));
  nch = std::min(nch, 65535);
  const int ic = (G.nl + nch - 1) / nch;
  nch = (G.nl + ic - 1) / ic;
  if (vec)
    face_kappa2_kernel<<<dim3(nbx, G.n2, nch), FK2_T, 0, st>>>(G, T, k1, k2, k3, kappa0, T_cut, fc_r0, fc_w, x1f_d,
                                                               x1c_d, ic);
  else
    face_kappa_kernel<<<dim3(nbx, G.n2, nch), FK_T, 0, st>>>(G, T, k1, k2, k3, kappa0, T_cut, fc_r0, fc_w, x1f_d,
                                                             x1c_d, ic);
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

// ---- restructured iteration (DESIGN.md §5 "PCG passes"): the x update of Fig. 1
// is deferred to the next p pass, so one iteration is
//   S-pass (stencil): p_k = z_k + beta p_{k-1};  x += alpha_{k-1} p_{k-1};  y = A p_k;  p_k.y
//   U-pass (pointwise): r -= alpha_k y;  z = r d;  r.z
// and one final x += alpha p after convergence.  The kernels below are the
// pointwise pieces (pcg_pnew is the S-pass's pointwise half when the stencil
// has no fused variant).
template <int NC>
__global__ void __launch_bounds__(256) pcg_pnew_kernel(long long n, long long cs, double* __restrict__ pnew,
                                                       const double* __restrict__ z, const double* __restrict__ pold,
                                                       double* __restrict__ x, const PcgScal* __restrict__ sc,
                                                       int first) {
  double beta[NC], ax[NC];
  bool act[NC];
  bool any = false;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    act[q] = !sc[q].done;
    beta[q] = first ? 0.0 : sc[q].beta;
    ax[q] = first ? 0.0 : sc[q].ax;
    any = any || act[q];
  }
  if (!any) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      if (!act[q]) continue;
      const long long o = e + q * cs;
      if (first) {
        pnew[o] = z[o];
      } else {
        const double po = pold[o];
        pnew[o] = fma(beta[q], po, z[o]);
        x[o] = fma(ax[q], po, x[o]);
      }
    }
  }
}

template <int NC>
__global__ void __launch_bounds__(256) pcg_rupdate_kernel(long long n, long long cs, double* __restrict__ r,
                                                          double* __restrict__ z, const double* __restrict__ y,
                                                          const double* __restrict__ d, const PcgScal* __restrict__ sc,
                                                          double* __restrict__ partials, long long pstride,
                                                          FinRed fin) {
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
  // U unrolled elements per thread and trip, every load of a trip issued before any use
  constexpr int U = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; e + (U - 1) * stride < n; e += U * stride) {
    double de[U], rr[NC][U], yy[NC][U];
#pragma unroll
    for (int u = 0; u < U; ++u) de[u] = __ldcs(d + e + u * stride);
#pragma unroll
    for (int q = 0; q < NC; ++q)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long o = e + u * stride + q * cs;
        rr[q][u] = act[q] ? __ldcs(r + o) : 0.0;
        yy[q][u] = act[q] ? __ldcs(y + o) : 0.0;
      }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      if (!act[q]) continue;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long o = e + u * stride + q * cs;
        const double rn = rr[q][u] - alpha[q] * yy[q][u];
        const double zn = rn * de[u];
        __stcs(r + o, rn);
        if (z) __stcs(z + o, zn);
        acc[q] += rn * zn;
      }
    }
  }
  for (; e < n; e += stride) {
    const double de = d[e];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      if (!act[q]) continue;
      const long long o = e + q * cs;
      const double rn = r[o] - alpha[q] * y[o];
      const double zn = rn * de;
      r[o] = rn;
      if (z) z[o] = zn;
      acc[q] += rn * zn;
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
  if (fin.ticket) {
    __shared__ double fred[4 * MAXC * 32];
    __shared__ unsigned flag;
    fused_final_reduce(fin, partials, pstride, gridDim.x, threadIdx.x, blockDim.x, fred, &flag,
                       [] { __syncthreads(); });
  }
}

// 16-byte vectorised variant (n, cs even, arrays 16 B aligned): element pairs, two
// pairs per thread and trip with every load of the trip issued before any use
template <int NC>
__global__ void __launch_bounds__(256) pcg_rupdate_v2_kernel(long long n2, long long cs2, double2* __restrict__ r,
                                                             double2* __restrict__ z, const double2* __restrict__ y,
                                                             const double2* __restrict__ d,
                                                             const PcgScal* __restrict__ sc,
                                                             double* __restrict__ partials, long long pstride,
                                                             FinRed fin) {
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
  constexpr int U = 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  auto one = [&](double2 de, double2 rr, double2 yy, long long o, int q) {
    double2 rn, zn;
    rn.x = rr.x - alpha[q] * yy.x;
    rn.y = rr.y - alpha[q] * yy.y;
    zn.x = rn.x * de.x;
    zn.y = rn.y * de.y;
    __stcs(r + o, rn);
    if (z) __stcs(z + o, zn);
    acc[q] += rn.x * zn.x;
    acc[q] += rn.y * zn.y;
  };
  for (; m + (U - 1) * stride < n2; m += U * stride) {
    double2 de[U], rr[NC][U], yy[NC][U];
#pragma unroll
    for (int u = 0; u < U; ++u) de[u] = __ldcs(d + m + u * stride);
#pragma unroll
    for (int q = 0; q < NC; ++q)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long o = m + u * stride + q * cs2;
        if (act[q]) {
          rr[q][u] = __ldcs(r + o);
          yy[q][u] = __ldcs(y + o);
        }
      }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      if (!act[q]) continue;
#pragma unroll
      for (int u = 0; u < U; ++u) one(de[u], rr[q][u], yy[q][u], m + u * stride + q * cs2, q);
    }
  }
  for (; m < n2; m += stride) {
    const double2 de = d[m];
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (act[q]) one(de, r[m + q * cs2], y[m + q * cs2], m + q * cs2, q);
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
  if (fin.ticket) {
    __shared__ double fred[4 * MAXC * 32];
    __shared__ unsigned flag;
    fused_final_reduce(fin, partials, pstride, gridDim.x, threadIdx.x, blockDim.x, fred, &flag,
                       [] { __syncthreads(); });
  }
}

template <int NC>
__global__ void __launch_bounds__(256) pcg_xfinal_kernel(long long n, long long cs, double* __restrict__ x,
                                                         const double* __restrict__ pk0, const double* __restrict__ pk1,
                                                         const double* __restrict__ pk2, const double* __restrict__ pk3,
                                                         const PcgScal* __restrict__ sc) {
  // what x still owes after the last iteration k = iters (PcgScal::xmf): alpha_k p_k;
  // after a skipped pass also alpha_{k-1} p_{k-1} (X_FIN_TWO), or only that (X_FIN_PREV,
  // a skipped pass that converged on its own r.z: iters = k-1); p_j in pk[j % 4]
  const double* pk[4] = {pk0, pk1, pk2, pk3};
  double ax[NC], axp[NC];
  const double *pp[NC], *pq[NC];
  bool act[NC], two[NC];
  bool any = false;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const int it = sc[q].iters, f = sc[q].xmf;
    act[q] = it > 0 || f == X_FIN_PREV;
    two[q] = f == X_FIN_TWO || f == X_FIN_PREV;
    ax[q] = f == X_FIN_PREV ? 0.0 : sc[q].ax;
    axp[q] = sc[q].axp;
    pp[q] = pk[it & 3];
    pq[q] = (f == X_FIN_PREV) ? pk[it & 3] : pk[(it + 3) & 3];   // p_{k-1}
    any = any || act[q];
  }
  if (!any) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      if (!act[q]) continue;
      const long long o = e + q * cs;
      double xv = x[o];
      if (two[q]) xv = fma(axp[q], pq[q][o], xv);
      x[o] = fma(ax[q], pp[q][o], xv);
    }
  }
}

#define STS_NC_SWITCH(ncomp, KER, ...)                                                  \
  switch (ncomp) {                                                                   \
    case 1: KER<1><<<PW_BLOCKS, 256, 0, st>>>(__VA_ARGS__); break;                   \
    case 2: KER<2><<<PW_BLOCKS, 256, 0, st>>>(__VA_ARGS__); break;                   \
    case 3: KER<3><<<PW_BLOCKS, 256, 0, st>>>(__VA_ARGS__); break;                   \
    default: throw Error{STS_ERR_ARG, "ncomp"};                                      \
  }

void launch_pcg_pnew(int ncomp, long long n, long long cs, double* pnew, const double* z, const double* pold,
                     double* x, const PcgScal* sc, int first, cudaStream_t st) {
  STS_NC_SWITCH(ncomp, pcg_pnew_kernel, n, cs, pnew, z, pold, x, sc, first);
  STS_CUDA(cudaGetLastError());
}

// grid of the U-pass: exactly the resident capacity (blocks per SM x 148, at most
// PW_BLOCKS), so the grid-stride loop has no partial last wave
// (cached per device ordinal: devices may differ in SM count)
template <class K>
static int resident_grid(K kernel) {
  static std::atomic<int> cached[64];
  const int dev = current_device() & 63;
  int v = cached[dev].load(std::memory_order_relaxed);
  if (!v) {
    int per_sm = 0, sms = 148;
    STS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0));
    STS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()));
    v = std::max(1, std::min(PW_BLOCKS, per_sm * sms));
    cached[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

template <int NC>
static int rupdate_nc(long long n, long long cs, double* r, double* z, const double* y, const double* d,
                      const PcgScal* sc, double* partials, long long pstride, FinRed fin, cudaStream_t st) {
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (n % 2 == 0 && cs % 2 == 0 && a16(r) && a16(z) && a16(y) && a16(d)) {
    const int nb = resident_grid(pcg_rupdate_v2_kernel<NC>);
    fin.ntot = nb;
    pcg_rupdate_v2_kernel<NC><<<nb, 256, 0, st>>>(n / 2, cs / 2, reinterpret_cast<double2*>(r),
                                                  reinterpret_cast<double2*>(z), reinterpret_cast<const double2*>(y),
                                                  reinterpret_cast<const double2*>(d), sc, partials, pstride, fin);
    return nb;
  }
  const int nb = resident_grid(pcg_rupdate_kernel<NC>);
  fin.ntot = nb;
  pcg_rupdate_kernel<NC><<<nb, 256, 0, st>>>(n, cs, r, z, y, d, sc, partials, pstride, fin);
  return nb;
}

int launch_pcg_rupdate(int ncomp, long long n, long long cs, double* r, double* z, const double* y, const double* d,
                       const PcgScal* sc, double* partials, long long pstride, const FinRed& fin, cudaStream_t st) {
  int nb = 0;
  switch (ncomp) {
    case 1: nb = rupdate_nc<1>(n, cs, r, z, y, d, sc, partials, pstride, fin, st); break;
    case 2: nb = rupdate_nc<2>(n, cs, r, z, y, d, sc, partials, pstride, fin, st); break;
    case 3: nb = rupdate_nc<3>(n, cs, r, z, y, d, sc, partials, pstride, fin, st); break;
    default: throw Error{STS_ERR_ARG, "ncomp"};
  }
  STS_CUDA(cudaGetLastError());
  return nb;
}

void launch_pcg_xfinal(int ncomp, long long n, long long cs, double* x, const double* const pk[4],
                       const PcgScal* sc, cudaStream_t st) {
  STS_NC_SWITCH(ncomp, pcg_xfinal_kernel, n, cs, x, pk[0], pk[1], pk[2], pk[3], sc);
  STS_CUDA(cudaGetLastError());
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

// Two-level deterministic reduction for large passes: block b sums slice b of every
// row (all rows' loads in flight at once) into l2[row][b]; the last block (ticket)
// sums l2 in a fixed order and runs the scalar phase.  One load round per thread
// instead of the ~100 dependent rounds of a single-block reduction.
constexpr int R2_THREADS = 256, R2_MAXROWS = 4 * MAXC;
__global__ void __launch_bounds__(R2_THREADS) pcg_reduce2_kernel(const double* __restrict__ partials,
                                                                 long long pstride, int nblocks, int ncomp, int nq,
                                                                 double* __restrict__ sums, double* l2,
                                                                 unsigned* ticket, int phase, PcgScal* sc,
                                                                 double rtol2) {
  __shared__ double red[R2_MAXROWS][R2_THREADS / 32];
  __shared__ unsigned flag;
  const int nrows = ncomp * nq, R = gridDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long per = (nblocks + R - 1) / R;
  const long long b0 = blockIdx.x * per, b1 = min((long long)nblocks, b0 + per);
  double v[R2_MAXROWS];
#pragma unroll
  for (int r = 0; r < R2_MAXROWS; ++r) v[r] = 0.0;
  for (long long b = b0 + tid; b < b1; b += R2_THREADS) {
#pragma unroll
    for (int r = 0; r < R2_MAXROWS; ++r)
      if (r < nrows) v[r] += __ldcg(partials + r * pstride + b);
  }
#pragma unroll
  for (int r = 0; r < R2_MAXROWS; ++r) {
    if (r >= nrows) break;
    const double w = warp_sum_d(v[r]);
    if (lane == 0) red[r][wid] = w;
  }
  __syncthreads();
  if (tid < nrows) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < R2_THREADS / 32; ++w) t += red[tid][w];
    l2[tid * R + blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) flag = (atomicAdd(ticket, 1u) == (unsigned)(R - 1)) ? 1u : 0u;
  __syncthreads();
  if (!flag) return;
  __threadfence();
  if (tid < nrows) {
    double t = 0.0;
    for (int b = 0; b < R; ++b) t += __ldcg(l2 + tid * R + b);
    sums[tid] = t;
  }
  __syncthreads();
  if (phase != PH_NONE && tid < ncomp) pcg_phase(sums, tid, nq, phase, sc, rtol2);
  if (tid == 0) *ticket = 0u;
}

void launch_pcg_reduce(const double* partials, long long pstride, int nblocks, int ncomp, int nq, double* sums,
                       int phase, PcgScal* sc, double rtol2, cudaStream_t st, double* l2, unsigned* ticket) {
  const int R = std::min(R2_MAXBLOCKS, (nblocks + R2_THREADS - 1) / R2_THREADS);
  if (l2 && ticket && R >= 2 && ncomp * nq <= R2_MAXROWS) {
    pcg_reduce2_kernel<<<R, R2_THREADS, 0, st>>>(partials, pstride, nblocks, ncomp, nq, sums, l2, ticket, phase, sc,
                                                 rtol2);
  } else {
    pcg_reduce_kernel<<<1, 1024, 0, st>>>(partials, pstride, nblocks, ncomp, nq, sums, phase, sc, rtol2);
  }
  STS_CUDA(cudaGetLastError());
}

void launch_pcg_scalar(const double* sums, int ncomp, int nq, int phase, PcgScal* sc, double rtol2,
                       cudaStream_t st) {
  pcg_scalar_kernel<<<1, 32, 0, st>>>(sums, ncomp, nq, phase, sc, rtol2);
  STS_CUDA(cudaGetLastError());
}

// per-solve initialisation of the PCG scalars: the iteration limit, cleared flags, and
// the counter of executed iteration-pair bodies of the device-driven loop
__global__ void pcg_init_kernel(PcgScal* sc, int ncomp, int kmax, int* body_count) {
  const int c = threadIdx.x;
  if (c < ncomp) {
    sc[c].kmax = kmax;
    sc[c].flags = 0;
    sc[c].done = 0;
    sc[c].iters = 0;
  }
  if (c == 0 && body_count) *body_count = 0;
}

void launch_pcg_init(PcgScal* sc, int ncomp, int kmax, int* body_count, cudaStream_t st) {
  pcg_init_kernel<<<1, 32, 0, st>>>(sc, ncomp, kmax, body_count);
  STS_CUDA(cudaGetLastError());
}

// the loop condition of the device-driven PCG (a WHILE conditional graph node): run
// another iteration pair while any component is neither converged nor stopped
__global__ void pcg_continue_kernel(cudaGraphConditionalHandle h, const PcgScal* sc, int ncomp, int* body_count,
                                    int count) {
  int more = 0;
  for (int c = 0; c < ncomp; ++c) more |= !sc[c].done;
  if (count) *body_count += 1;
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

void launch_pcg_continue(cudaGraphConditionalHandle h, const PcgScal* sc, int ncomp, int* body_count, bool count,
                         cudaStream_t st) {
  pcg_continue_kernel<<<1, 1, 0, st>>>(h, sc, ncomp, body_count, count ? 1 : 0);
  STS_CUDA(cudaGetLastError());
}

// small device results to mapped pinned host memory by SM stores: the host reads
// them after a stream sync without a DMA copy, which would queue behind large
// transfers a caller runs on the copy engines (e.g. the previous result's download)
__global__ void publish_kernel(const double* __restrict__ src, int n, double* dst) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

void launch_publish(const double* src, int n, double* dst_mapped, cudaStream_t st) {
  publish_kernel<<<1, 32, 0, st>>>(src, n, dst_mapped);
  STS_CUDA(cudaGetLastError());
}

}  // namespace sts
