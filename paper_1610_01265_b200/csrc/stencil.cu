// Fused stencil passes of the parabolic operator.
//
//  * aniso_kernel — vertex-centred symmetric scheme for div(kappa b b.grad u)
//    (PAPER.md:173 boxed term, DESIGN R2): per r-plane a CTA stages a
//    (TJ+2) x (TK+2) halo region of u, b and the three face diffusivities in
//    shared memory (2-plane ring), computes every vertex of its tile ONCE
//    (gradient, b_v, kappa_v, V_v -> Q_v = V_v kappa_v (b_v.g_v)), then each
//    cell gathers its 8 vertices.  The CTA marches along r (2.5-D blocking).
//  * iso_kernel   — 7-point div(kappa grad u)/w (PAPER.md:181 boxed viscosity
//    term, :329 test), one thread per (theta, phi) column marching along r with
//    the r-neighbours in registers, ncomp <= 3 components per pass.
//
// Both are templated on an epilogue that fuses the pointwise part of the
// algorithm into the same pass: plain F(u), the RKL2 first stage / stage
// recurrence (Fig. 2), the PCG initial residual + Jacobi diagonal, the
// PCG matvec A p with its p.y partial dot product (Fig. 1), or the
// Gershgorin row sums (App. B).
#include <cfloat>

#include "sts_common.cuh"

namespace sts {

enum { EPI_GERSH = 100 };  // internal: Gershgorin absolute row sums -> atomic max

__device__ __forceinline__ int wrapk(int k, int n3) {
  int r = k % n3;
  return r < 0 ? r + n3 : r;
}

// pointer to local plane il (-1..nl) of component c of a field (nullptr if absent)
__device__ __forceinline__ const double* plane_ptr(const FieldV& f, const Geo& G, int il, int c) {
  if (il < 0) return f.lo ? f.lo + (long long)c * G.plane : nullptr;
  if (il >= G.nl) return f.hi ? f.hi + (long long)c * G.plane : nullptr;
  return f.p + (long long)c * G.cstride + (long long)il * G.plane;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block reduction of NV values per thread -> partials[v][blk]
template <int NV>
__device__ __forceinline__ void block_partials(double (&v)[NV], double* partials, long long pstride,
                                               long long blk) {
  __shared__ double red[NV][NT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = warp_sum(v[q]);
    if (lane == 0) red[q][wid] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[threadIdx.x][w];
    partials[threadIdx.x * pstride + blk] = s;
  }
}

// ============================================================================
// anisotropic vertex-centred kernel
// ============================================================================
// shared-memory layout (doubles)
constexpr int AF_U = 0, AF_B0 = 1, AF_B1 = 2, AF_B2 = 3, AF_K1 = 4, AF_K2 = 5, AF_K3 = 6, AF_N = 7;
constexpr int AV_DR = 0, AV_DT = 1, AV_DP = 2, AV_Q = 3, AV_C = 4, AV_N = 5;
constexpr size_t ANISO_SMEM = (size_t)(2 * AF_N * RC + 2 * AV_N * VC) * sizeof(double);

template <int EPI>
__global__ void __launch_bounds__(NT, 3) aniso_kernel(StencilCall c, int ic, unsigned long long* dmax) {
  extern __shared__ double sm[];
  double* cs = sm;                      // [2][AF_N][RC]
  double* vs = sm + 2 * AF_N * RC;      // [2][AV_N][VC]
  const Geo& G = c.geo;
  const Metrics& M = G.m;
  const int tid = threadIdx.x;
  const int tk = tid % TK, tj = tid / TK;
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * TJ;
  const int ib = c.ib + blockIdx.z * ic;
  const int ie = min(ib + ic, c.ie);
  const long long blk = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
  constexpr bool kNeedU = (EPI != EPI_GERSH);
  constexpr bool kNeedC = (EPI == EPI_PCG_R0 || EPI == EPI_GERSH);

  if constexpr (EPI == EPI_PCG_R0 || EPI == EPI_PCG_AP) {
    if (c.ea.sc && c.ea.sc[0].done) return;
  }

  auto cell = [&](int slot, int f) { return cs + (slot * AF_N + f) * RC; };
  auto vtx = [&](int slot, int f) { return vs + (slot * AV_N + f) * VC; };

  // ---- stage one cell plane (il in [-1, nl]) with its theta/phi halo ----
  auto load_plane = [&](int il, int slot) {
    const double* src[AF_N];
    src[AF_U] = kNeedU ? plane_ptr(c.u, G, il, 0) : nullptr;
    src[AF_B0] = plane_ptr(c.b, G, il, 0);
    src[AF_B1] = plane_ptr(c.b, G, il, 1);
    src[AF_B2] = plane_ptr(c.b, G, il, 2);
    src[AF_K1] = plane_ptr(c.k1, G, il, 0);
    src[AF_K2] = plane_ptr(c.k2, G, il, 0);
    src[AF_K3] = plane_ptr(c.k3, G, il, 0);
    for (int e = tid; e < RC; e += NT) {
      const int row = e / RK, col = e - row * RK;
      const int j = j0 - 1 + row;
      int k = k0 - 1 + col;
      bool ok = (j >= 0 && j < G.n2);
      if (G.periodic3) k = wrapk(k, G.n3);
      else ok = ok && (k >= 0 && k < G.n3);
      const long long off = (long long)j * G.n3 + k;
#pragma unroll
      for (int f = 0; f < AF_N; ++f) {
        double v = 0.0;
        if (ok && src[f]) v = __ldg(src[f] + off);
        cell(slot, f)[e] = v;
      }
    }
  };

  // ---- every vertex (il+1/2, jv+1/2, kv+1/2) of the tile (+ halo ring) ----
  auto vertex_plane = [&](int il, int sl, int sh, int vslot) {
    const int iv = G.i0 + il;  // global r index of the lower cell plane
    const bool ivok = (iv >= 0) && (iv + 1 < G.n1g);
    for (int e = tid; e < VC; e += NT) {
      const int vj = e / VK, vk = e - vj * VK;
      const int jv = j0 - 1 + vj;
      int kv = k0 - 1 + vk;
      bool ok = ivok && jv >= 0 && jv + 1 < G.n2;
      int kvw = kv, kvw1 = kv + 1;
      if (G.periodic3) {
        kvw = wrapk(kv, G.n3);
        kvw1 = wrapk(kv + 1, G.n3);
      } else {
        ok = ok && kv >= 0 && kv + 1 < G.n3;
      }
      double Dr = 0.0, Dt = 0.0, Dp = 0.0, Q = 0.0, C = 0.0;
      if (ok) {
        const int c00 = vj * RK + vk;  // region index of cell (jv, kv)
        const int c01 = c00 + 1, c10 = c00 + RK, c11 = c00 + RK + 1;
        const double* Bl0 = cell(sl, AF_B0); const double* Bh0 = cell(sh, AF_B0);
        const double* Bl1 = cell(sl, AF_B1); const double* Bh1 = cell(sh, AF_B1);
        const double* Bl2 = cell(sl, AF_B2); const double* Bh2 = cell(sh, AF_B2);
        const double br = 0.125 * (Bl0[c00] + Bl0[c01] + Bl0[c10] + Bl0[c11] + Bh0[c00] + Bh0[c01] + Bh0[c10] + Bh0[c11]);
        const double bt = 0.125 * (Bl1[c00] + Bl1[c01] + Bl1[c10] + Bl1[c11] + Bh1[c00] + Bh1[c01] + Bh1[c10] + Bh1[c11]);
        const double bp = 0.125 * (Bl2[c00] + Bl2[c01] + Bl2[c10] + Bl2[c11] + Bh2[c00] + Bh2[c01] + Bh2[c10] + Bh2[c11]);
        const double* K1l = cell(sl, AF_K1);
        const double* K2l = cell(sl, AF_K2); const double* K2h = cell(sh, AF_K2);
        const double* K3l = cell(sl, AF_K3); const double* K3h = cell(sh, AF_K3);
        const double kap = (1.0 / 12.0) * ((K1l[c00] + K1l[c01] + K1l[c10] + K1l[c11]) +
                                           (K2l[c00] + K2l[c01] + K2h[c00] + K2h[c01]) +
                                           (K3l[c00] + K3l[c10] + K3h[c00] + K3h[c10]));
        const double Vv = 0.125 * (M.Vr[iv] + M.Vr[iv + 1]) * (M.Vt[jv] + M.Vt[jv + 1]) * (M.Vp[kvw] + M.Vp[kvw1]);
        C = Vv * kap;
        Dr = 0.25 * br * M.iH1[iv];
        Dt = 0.25 * bt * M.iH2[jv];
        Dp = 0.25 * bp * M.iH3[kvw];
        if constexpr (kNeedU) {
          const double* Ul = cell(sl, AF_U); const double* Uh = cell(sh, AF_U);
          const double ig2l = M.iG2[iv], ig2h = M.iG2[iv + 1];
          const double ig3a = M.iG3[jv], ig3b = M.iG3[jv + 1];
          // 4 differences per direction, each scaled by its own pair's metric
          const double dr = (Uh[c00] - Ul[c00]) + (Uh[c01] - Ul[c01]) + (Uh[c10] - Ul[c10]) + (Uh[c11] - Ul[c11]);
          const double dt = ig2l * ((Ul[c10] - Ul[c00]) + (Ul[c11] - Ul[c01])) +
                            ig2h * ((Uh[c10] - Uh[c00]) + (Uh[c11] - Uh[c01]));
          const double dp = ig2l * (ig3a * (Ul[c01] - Ul[c00]) + ig3b * (Ul[c11] - Ul[c10])) +
                            ig2h * (ig3a * (Uh[c01] - Uh[c00]) + ig3b * (Uh[c11] - Uh[c10]));
          // b_v . g_v with g_a = 1/4 sum(diff)/h_a  ->  Dr*dr + Dt*dt + Dp*dp
          Q = C * (Dr * dr + Dt * dt + Dp * dp);
        }
      }
      vtx(vslot, AV_DR)[e] = Dr;
      vtx(vslot, AV_DT)[e] = Dt;
      vtx(vslot, AV_DP)[e] = Dp;
      vtx(vslot, AV_Q)[e] = Q;
      if constexpr (kNeedC) vtx(vslot, AV_C)[e] = C;
    }
  };

  const int j = j0 + tj, k = k0 + tk;
  const bool own = (j < G.n2) && (k < G.n3);
  const long long coff = (long long)j * G.n3 + k;
  const double ig3c = own ? M.iG3[j] : 0.0;
  double part0 = 0.0, part1 = 0.0;
  double rowmax = 0.0;

  load_plane(ib - 1, (ib - 1) & 1);
  load_plane(ib, ib & 1);
  __syncthreads();
  vertex_plane(ib - 1, (ib - 1) & 1, ib & 1, (ib - 1) & 1);
  __syncthreads();  // the loop's first load overwrites the cell slot just read

  for (int il = ib; il < ie; ++il) {
    load_plane(il + 1, (il + 1) & 1);
    __syncthreads();
    double uc = 0.0;
    if constexpr (kNeedU) uc = cell(il & 1, AF_U)[(tj + 1) * RK + tk + 1];
    vertex_plane(il, il & 1, (il + 1) & 1, il & 1);
    __syncthreads();
    if (!own) continue;
    const int ig = G.i0 + il;
    const double ig2c = M.iG2[ig];
    const double sT = ig2c, sP = ig2c * ig3c;
    double Lu = 0.0, Ld = 0.0;
    // entries of row (cell) for the Gershgorin epilogue: index (di+1)*9+(dj+1)*3+(dk+1)
    double ent[27];
    if constexpr (EPI == EPI_GERSH) {
#pragma unroll
      for (int q = 0; q < 27; ++q) ent[q] = 0.0;
    }
    // periodic n3 == 1: the vertex columns k-1/2 and k+1/2 are the same vertex and
    // the cell occupies both of its phi positions -> its weights add before squaring
    const bool fold1 = G.periodic3 && G.n3 == 1;
#pragma unroll
    for (int up = 0; up < 2; ++up) {         // up=0: vertex plane below (cell at s1=+1)
      const int vsl = (up ? il : il - 1) & 1;
      const double s1 = up ? -1.0 : 1.0;
#pragma unroll
      for (int a = 0; a < 2; ++a) {          // vj = tj + a : a=0 -> vertex j-1/2 (cell at s2=+1)
        double wsum = 0.0, Csum = 0.0;
#pragma unroll
        for (int bq = 0; bq < 2; ++bq) {
          const int e = (tj + a) * VK + tk + bq;
          const double s2 = a ? -1.0 : 1.0, s3 = bq ? -1.0 : 1.0;
          const double Dr = vtx(vsl, AV_DR)[e], Dt = vtx(vsl, AV_DT)[e], Dp = vtx(vsl, AV_DP)[e];
          const double wc = s1 * Dr + s2 * Dt * sT + s3 * Dp * sP;
          if constexpr (kNeedU) Lu -= vtx(vsl, AV_Q)[e] * wc;
          if constexpr (EPI == EPI_PCG_R0) {
            if (fold1) {
              wsum += wc;
              Csum = vtx(vsl, AV_C)[e];
            } else {
              Ld -= vtx(vsl, AV_C)[e] * wc * wc;
            }
          }
          if constexpr (EPI == EPI_GERSH) {
            const double Cv = vtx(vsl, AV_C)[e];
            if (Cv == 0.0) continue;
            // the 8 cells q of this vertex: offsets relative to the vertex base
            // (cell sits at sigma = ((s1+1)/2, (s2+1)/2, (s3+1)/2))
            const int si = up ? 0 : 1, sj = a ? 0 : 1, sk = bq ? 0 : 1;
            const int vig = up ? ig : ig - 1;            // vertex base r index
            const int vjg = j - sj;                      // vertex base theta index
#pragma unroll
            for (int q1 = 0; q1 < 2; ++q1)
#pragma unroll
              for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                for (int q3 = 0; q3 < 2; ++q3) {
                  const double ig2q = M.iG2[vig + q1];
                  const double ig3q = M.iG3[vjg + q2];
                  const double wq = (q1 ? 1.0 : -1.0) * Dr + (q2 ? 1.0 : -1.0) * Dt * ig2q +
                                    (q3 ? 1.0 : -1.0) * Dp * ig2q * ig3q;
                  const int di = q1 - si, dj = q2 - sj, dk = q3 - sk;
                  ent[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)] -= Cv * wc * wq;
                }
          }
        }
        if constexpr (EPI == EPI_PCG_R0) {
          if (fold1) Ld -= Csum * wsum * wsum;
        }
      }
    }
    const double WV = (c.w ? __ldg(c.w + (long long)il * G.plane + coff) : 1.0) * M.Vr[ig] * M.Vt[j] * M.Vp[k];
    const long long gi = (long long)il * G.plane + coff;
    if constexpr (EPI == EPI_F) {
      c.ea.out[gi] = Lu / WV;
    } else if constexpr (EPI == EPI_RKL2_FIRST) {
      const double F = Lu / WV;
      c.ea.out2[gi] = F;
      c.ea.out[gi] = uc + c.ea.c0 * F;
    } else if constexpr (EPI == EPI_RKL2_STAGE) {
      const double F = Lu / WV;
      const double ym2 = c.ea.ym2[gi], y0 = c.ea.y0[gi], m0 = c.ea.m0[gi];
      c.ea.out[gi] = c.ea.mu * uc + c.ea.nu * ym2 + c.ea.c2 * y0 + c.ea.c0 * F + c.ea.c1 * m0;
    } else if constexpr (EPI == EPI_PCG_R0) {
      const double r = c.ea.dt * Lu;
      const double d = 1.0 / (WV - c.ea.dt * Ld);
      const double z = r * d;
      const double bb = WV * uc;
      c.ea.out[gi] = r;
      if (c.ea.out2) c.ea.out2[gi] = uc;
      c.ea.out3[gi] = z;
      c.ea.out4[gi] = d;
      part0 += r * z;
      part1 += bb * bb * d;
    } else if constexpr (EPI == EPI_PCG_AP) {
      const double y = WV * uc - c.ea.dt * Lu;
      c.ea.out[gi] = y;
      part0 += uc * y;
    } else if constexpr (EPI == EPI_GERSH) {
      // sum |L_iq| over distinct cells q: with periodic n3 <= 2 several phi
      // offsets name the same cell and their entries add first
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const double em = ent[3 * q], e0 = ent[3 * q + 1], ep = ent[3 * q + 2];
        if (G.periodic3 && G.n3 == 1) s += fabs(em + e0 + ep);
        else if (G.periodic3 && G.n3 == 2) s += fabs(e0) + fabs(em + ep);
        else s += fabs(em) + fabs(e0) + fabs(ep);
      }
      rowmax = fmax(rowmax, s / WV);
    }
  }

  if constexpr (EPI == EPI_PCG_R0) {
    double v[2] = {part0, part1};
    block_partials<2>(v, c.ea.partials, c.ea.pstride, c.ea.pbase + blk);
  } else if constexpr (EPI == EPI_PCG_AP) {
    double v[1] = {part0};
    block_partials<1>(v, c.ea.partials, c.ea.pstride, c.ea.pbase + blk);
  } else if constexpr (EPI == EPI_GERSH) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rowmax = fmax(rowmax, __shfl_xor_sync(0xffffffffu, rowmax, o));
    if ((tid & 31) == 0 && rowmax > 0.0) atomicMax(dmax, (unsigned long long)__double_as_longlong(rowmax));
  }
}

// ============================================================================
// isotropic 7-point kernel (ncomp components)
// ============================================================================
template <int EPI, int NC>
__global__ void __launch_bounds__(NT, 4) iso_kernel(StencilCall c, int ic, unsigned long long* dmax) {
  const Geo& G = c.geo;
  const Metrics& M = G.m;
  const int tid = threadIdx.x;
  const int tk = tid % TK, tj = tid / TK;
  const int j = blockIdx.y * TJ + tj, k = blockIdx.x * TK + tk;
  const int ib = c.ib + blockIdx.z * ic;
  const int ie = min(ib + ic, c.ie);
  const long long blk = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
  constexpr bool kNeedU = (EPI != EPI_GERSH);
  bool skip[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) skip[q] = false;
  if constexpr (EPI == EPI_PCG_R0 || EPI == EPI_PCG_AP) {
    bool all = true;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      skip[q] = c.ea.sc && c.ea.sc[q].done;
      all = all && skip[q];
    }
    if (all) return;
  }
  double part0[NC], part1[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) part0[q] = part1[q] = 0.0;
  double rowmax = 0.0;
  const bool own = (j < G.n2) && (k < G.n3);
  if (own) {
    const long long coff = (long long)j * G.n3 + k;
    const bool jm = j >= 1, jp = j + 1 < G.n2;
    // periodic n3 == 1: the phi face joins the cell to itself and carries no flux
    const bool kself = G.periodic3 && G.n3 == 1;
    const bool km = !kself && (G.periodic3 || k >= 1), kp = !kself && (G.periodic3 || k + 1 < G.n3);
    const int kmw = G.periodic3 ? wrapk(k - 1, G.n3) : k - 1;
    const int kpw = G.periodic3 ? wrapk(k + 1, G.n3) : k + 1;
    const long long offjm = coff - G.n3, offjp = coff + G.n3;
    const long long offkm = (long long)j * G.n3 + kmw, offkp = (long long)j * G.n3 + kpw;
    // metric pieces that do not depend on r
    const double f1tp = M.F1t[j] * M.F1p[k];
    const double f2tp_p = jp ? M.F2t[j] * M.F2p[k] : 0.0;
    const double f2tp_m = jm ? M.F2t[j - 1] * M.F2p[k] : 0.0;
    const double f3tp_p = kp ? M.F3t[j] * M.F3p[k] : 0.0;
    const double f3tp_m = km ? M.F3t[j] * M.F3p[kmw] : 0.0;
    const double vtp = M.Vt[j] * M.Vp[k];

    double udn[NC], uc[NC], uup[NC];
    const int ig0 = G.i0 + ib;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      uc[q] = udn[q] = 0.0;
      if constexpr (kNeedU) {
        const double* pc = plane_ptr(c.u, G, ib, q);
        uc[q] = __ldg(pc + coff);
        const double* pd = (ig0 >= 1) ? plane_ptr(c.u, G, ib - 1, q) : nullptr;
        udn[q] = pd ? __ldg(pd + coff) : 0.0;
      }
    }
    double kdn = 0.0;
    if (ig0 >= 1) {
      const double* p = plane_ptr(c.k1, G, ib - 1, 0);
      kdn = __ldg(p + coff) * M.F1r[ig0 - 1] * f1tp;
    }
    for (int il = ib; il < ie; ++il) {
      const int ig = G.i0 + il;
      const bool ip = ig + 1 < G.n1g;
      const double* k1p = plane_ptr(c.k1, G, il, 0);
      const double* k2p = plane_ptr(c.k2, G, il, 0);
      const double* k3p = plane_ptr(c.k3, G, il, 0);
      const double f23r = M.F2r[ig];
      const double f3r = M.F3r[ig];
      const double Kup = ip ? __ldg(k1p + coff) * M.F1r[ig] * f1tp : 0.0;
      const double Kjp = jp ? __ldg(k2p + coff) * f23r * f2tp_p : 0.0;
      const double Kjm = jm ? __ldg(k2p + offjm) * f23r * f2tp_m : 0.0;
      const double Kkp = kp ? __ldg(k3p + coff) * f3r * f3tp_p : 0.0;
      const double Kkm = km ? __ldg(k3p + offkm) * f3r * f3tp_m : 0.0;
      const double WV = (c.w ? __ldg(c.w + (long long)il * G.plane + coff) : 1.0) * M.Vr[ig] * vtp;
      const long long gi = (long long)il * G.plane + coff;
      const double Ldiag = -(kdn + Kup + Kjp + Kjm + Kkp + Kkm);
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        double Lu = 0.0;
        if constexpr (kNeedU) {
          const double* pc = plane_ptr(c.u, G, il, q);
          const double* pu = ip ? plane_ptr(c.u, G, il + 1, q) : nullptr;
          uup[q] = pu ? __ldg(pu + coff) : 0.0;
          const double ujm = jm ? __ldg(pc + offjm) : 0.0;
          const double ujp = jp ? __ldg(pc + offjp) : 0.0;
          const double ukm = km ? __ldg(pc + offkm) : 0.0;
          const double ukp = kp ? __ldg(pc + offkp) : 0.0;
          const double u0 = uc[q];
          Lu = kdn * (udn[q] - u0) + Kup * (uup[q] - u0) + Kjm * (ujm - u0) + Kjp * (ujp - u0) +
               Kkm * (ukm - u0) + Kkp * (ukp - u0);
        }
        const long long go = gi + (long long)q * G.cstride;
        if (skip[q]) continue;
        if constexpr (EPI == EPI_F) {
          c.ea.out[go] = Lu / WV;
        } else if constexpr (EPI == EPI_RKL2_FIRST) {
          const double F = Lu / WV;
          c.ea.out2[go] = F;
          c.ea.out[go] = uc[q] + c.ea.c0 * F;
        } else if constexpr (EPI == EPI_RKL2_STAGE) {
          const double F = Lu / WV;
          c.ea.out[go] = c.ea.mu * uc[q] + c.ea.nu * c.ea.ym2[go] + c.ea.c2 * c.ea.y0[go] + c.ea.c0 * F +
                         c.ea.c1 * c.ea.m0[go];
        } else if constexpr (EPI == EPI_PCG_R0) {
          const double r = c.ea.dt * Lu;
          const double d = 1.0 / (WV - c.ea.dt * Ldiag);
          const double z = r * d;
          const double bb = WV * uc[q];
          c.ea.out[go] = r;
          if (c.ea.out2) c.ea.out2[go] = uc[q];
          c.ea.out3[go] = z;
          if (q == 0) c.ea.out4[gi] = d;
          part0[q] += r * z;
          part1[q] += bb * bb * d;
        } else if constexpr (EPI == EPI_PCG_AP) {
          const double y = WV * uc[q] - c.ea.dt * Lu;
          c.ea.out[go] = y;
          part0[q] += uc[q] * y;
        }
      }
      if constexpr (EPI == EPI_GERSH) rowmax = fmax(rowmax, -2.0 * Ldiag / WV);
      kdn = Kup;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        udn[q] = uc[q];
        uc[q] = uup[q];
      }
    }
  }
  if constexpr (EPI == EPI_PCG_R0) {
    double v[2 * NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      v[2 * q] = part0[q];
      v[2 * q + 1] = part1[q];
    }
    block_partials<2 * NC>(v, c.ea.partials, c.ea.pstride, c.ea.pbase + blk);
  } else if constexpr (EPI == EPI_PCG_AP) {
    block_partials<NC>(part0, c.ea.partials, c.ea.pstride, c.ea.pbase + blk);
  } else if constexpr (EPI == EPI_GERSH) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rowmax = fmax(rowmax, __shfl_xor_sync(0xffffffffu, rowmax, o));
    if ((tid & 31) == 0 && rowmax > 0.0) atomicMax(dmax, (unsigned long long)__double_as_longlong(rowmax));
  }
}

// ============================================================================
// launch plumbing
// ============================================================================
int stencil_blocks(const Geo& G, int ib, int ie, int* ic_out) {
  const int nbx = (G.n3 + TK - 1) / TK, nby = (G.n2 + TJ - 1) / TJ;
  const int np = ie - ib;
  if (np <= 0) {
    if (ic_out) *ic_out = 1;
    return 0;
  }
  // enough CTAs for ~4 waves of 148 SMs x 3 resident, but >= 8 planes per chunk
  const long long tiles = (long long)nbx * nby;
  const long long want = 148LL * 3 * 4;
  int ic = (int)((np * tiles + want - 1) / want);
  ic = ic < 8 ? 8 : ic;
  if (ic > np) ic = np;
  const int nbz = (np + ic - 1) / ic;
  if (ic_out) *ic_out = ic;
  return nbx * nby * nbz;
}

template <int EPI>
static void launch_epi(const StencilCall& c, cudaStream_t st, unsigned long long* dmax) {
  int ic = 1;
  stencil_blocks(c.geo, c.ib, c.ie, &ic);
  const int np = c.ie - c.ib;
  if (np <= 0) return;
  dim3 grid((c.geo.n3 + TK - 1) / TK, (c.geo.n2 + TJ - 1) / TJ, (np + ic - 1) / ic);
  if (c.mode == STS_MODE_ANISO) {
    static bool attr_set = false;
    if (!attr_set) {
      STS_CUDA(cudaFuncSetAttribute(aniso_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ANISO_SMEM));
      attr_set = true;
    }
    aniso_kernel<EPI><<<grid, NT, ANISO_SMEM, st>>>(c, ic, dmax);
  } else {
    switch (c.ncomp) {
      case 1: iso_kernel<EPI, 1><<<grid, NT, 0, st>>>(c, ic, dmax); break;
      case 2: iso_kernel<EPI, 2><<<grid, NT, 0, st>>>(c, ic, dmax); break;
      case 3: iso_kernel<EPI, 3><<<grid, NT, 0, st>>>(c, ic, dmax); break;
      default: throw Error{STS_ERR_ARG, "ncomp must be 1..3"};
    }
  }
  STS_CUDA(cudaGetLastError());
}

void launch_stencil(const StencilCall& c, cudaStream_t st) {
  switch (c.epi) {
    case EPI_F: launch_epi<EPI_F>(c, st, nullptr); break;
    case EPI_RKL2_FIRST: launch_epi<EPI_RKL2_FIRST>(c, st, nullptr); break;
    case EPI_RKL2_STAGE: launch_epi<EPI_RKL2_STAGE>(c, st, nullptr); break;
    case EPI_PCG_R0: launch_epi<EPI_PCG_R0>(c, st, nullptr); break;
    case EPI_PCG_AP: launch_epi<EPI_PCG_AP>(c, st, nullptr); break;
    default: throw Error{STS_ERR_ARG, "bad epilogue"};
  }
}

void launch_gershgorin(const StencilCall& c, unsigned long long* d_max, cudaStream_t st) {
  launch_epi<EPI_GERSH>(c, st, d_max);
}

}  // namespace sts
