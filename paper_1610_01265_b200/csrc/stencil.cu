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
      c.ea.out[gi] = c.ea.a0 * uc + c.ea.c0 * F;
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
      if (c.ea.out3) c.ea.out3[gi] = z;
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
// anisotropic operator, fast path (F / RKL2 stages / PCG A p)
// ----------------------------------------------------------------------------
// The vertex coefficients are frozen over an advance (lagged diffusivity,
// PAPER.md:33), so vertex_coef_tiled_kernel folds b, kappa and the metrics into three
// numbers per vertex ONCE per advance:  e_a = sqrt(V_v kappa_v) * b_{v,a} / (4 h_a)
// (h_th, h_ph without their cell-dependent r / sin(theta) factors).  Then
//   Q_v D_a = (e_v . d_v) e_{v,a},   d_v = the 4-difference sums of u,
// and a stage / matvec pass streams only u, e (and the epilogue fields):
// 64 B per cell per RKL2 stage instead of 88, 40 B per PCG matvec instead of 64.
//
// Thread (vj = warp, vk = lane) owns vertex column (j0-1+vj, k0-1+vk) and output
// cell (j0+vj, k0+vk) (vj < 7, vk < 31): 7 x 31 outputs, 8 x 32 vertices, 9 x 33
// staged u cells.  Per r-plane each thread reduces its 2x2 in-plane u box once
// (3 sums kept in registers for the next vertex plane) and each cell reduces its
// 2x2 in-plane vertex box once (3 sums kept for the next cell plane).  u planes
// are staged with cp.async one plane ahead of use.
// ============================================================================
constexpr int FJ = 8, FK = 32;              // vertex rows / cols = warps / lanes
constexpr int FOJ = FJ - 1, FOK = FK - 1;   // output rows / cols
constexpr int FRJ = FJ + 1, FRK = FK + 1;   // staged cell rows / cols
constexpr int FRC = FRJ * FRK;              // 297 staged cells per plane
constexpr int FNT = FJ * FK;                // 256 threads
constexpr size_t FAST_SMEM = (size_t)(2 * FRC + 3 * FNT) * sizeof(double);

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = ok ? 8 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int EPI>
__global__ void __launch_bounds__(FNT, (EPI == EPI_RKL2_STAGE ? 3 : 4)) aniso_fast_kernel(StencilCall c, int ic) {
  extern __shared__ double sm[];
  double* us = sm;                          // [2][FRC] staged u planes
  double* vA = sm + 2 * FRC;                // [FNT] vertex A = Q Dr
  double* vB = vA + FNT;                    //        B = Q Dt
  double* vC = vB + FNT;                    //        C = Q Dp
  const Geo& G = c.geo;
  const Metrics& M = G.m;
  const int tid = threadIdx.x;
  const int vj = tid >> 5, vk = tid & 31;
  const int j0 = blockIdx.y * FOJ, k0 = blockIdx.x * FOK;
  const int ib = c.ib + blockIdx.z * ic;
  const int ie = min(ib + ic, c.ie);
  const long long blk = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);

  if constexpr (EPI == EPI_PCG_AP) {
    if (c.ea.sc && c.ea.sc[0].done) return;
  }

  // ---- staging assignments (fixed for the whole march) ----
  int soff[2];
  bool sok[2];
  bool shas[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int e = tid + q * FNT;
    shas[q] = e < FRC;
    const int row = e / FRK, col = e - (e / FRK) * FRK;
    const int j = j0 - 1 + row;
    int k = k0 - 1 + col;
    bool ok = shas[q] && j >= 0 && j < G.n2;
    if (G.periodic3) k = wrapk(k, G.n3);
    else ok = ok && k >= 0 && k < G.n3;
    sok[q] = ok;
    soff[q] = ok ? j * G.n3 + k : 0;
  }
  auto stage = [&](int il, int slot) {
    const double* src = plane_ptr(c.u, G, il, 0);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!shas[q]) continue;
      const bool ok = sok[q] && src != nullptr;
      cp_async8(us + slot * FRC + tid + q * FNT, ok ? src + soff[q] : c.ev, ok);
    }
    cp_async_commit();
  };

  // ---- per-thread vertex column ----
  const int jv = j0 - 1 + vj;
  int kv = k0 - 1 + vk;
  bool vok = jv >= 0 && jv + 1 < G.n2;
  if (G.periodic3) kv = wrapk(kv, G.n3);
  else vok = vok && kv >= 0 && kv + 1 < G.n3;
  const double ig3a = vok ? M.iG3[jv] : 0.0, ig3b = vok ? M.iG3[jv + 1] : 0.0;
  const long long eoff = vok ? (long long)(jv + 1) * ev_row(G.n3) + kv + 1 : 0;
  const long long epp = ev_plane(G.n2, G.n3);
  const long long es = (long long)(G.nl + 1) * epp;
  const int j = j0 + vj, k = k0 + vk;
  const bool own = vj < FOJ && vk < FOK && j < G.n2 && k < G.n3;
  const long long coff = own ? (long long)j * G.n3 + k : 0;
  const double ig3c = own ? M.iG3[j] : 0.0;
  const double vtpc = own ? M.Vt[j] * M.Vp[k] : 0.0;

  const int c00 = vj * FRK + vk, c01 = c00 + 1, c10 = c00 + FRK, c11 = c10 + 1;
  // in-plane 2x2 u box: sum, theta differences, phi differences (theta-metric weighted)
  auto usums = [&](int slot, double& Su, double& Tu, double& Fu) {
    const double* U = us + slot * FRC;
    const double u00 = U[c00], u01 = U[c01], u10 = U[c10], u11 = U[c11];
    Su = (u00 + u01) + (u10 + u11);
    Tu = (u10 - u00) + (u11 - u01);
    Fu = ig3a * (u01 - u00) + ig3b * (u11 - u10);
  };
  // frozen vertex coefficients of vertex plane il+1/2 (zero if the vertex is missing)
  auto load_e = [&](int il, double& er, double& et, double& ep) {
    const int iv = G.i0 + il;
    er = et = ep = 0.0;
    if (vok && iv >= 0 && iv + 1 < G.n1g && il < ie) {
      const long long o = (long long)(il + 1) * epp + eoff;
      er = __ldg(c.ev + o);
      et = __ldg(c.ev + es + o);
      ep = __ldg(c.ev + 2 * es + o);
    }
  };
  // vertex between cell planes il and il+1
  auto vertex = [&](int il, double er, double et, double ep, double SuL, double TuL, double FuL, double SuH,
                    double TuH, double FuH) {
    const int iv = G.i0 + il;
    double A = 0.0, B = 0.0, C = 0.0;
    if (vok && iv >= 0 && iv + 1 < G.n1g) {
      const double ig2l = M.iG2[iv], ig2h = M.iG2[iv + 1];
      const double q = er * (SuH - SuL) + et * (ig2l * TuL + ig2h * TuH) + ep * (ig2l * FuL + ig2h * FuH);
      A = q * er;
      B = q * et;
      C = q * ep;
    }
    vA[tid] = A;
    vB[tid] = B;
    vC[tid] = C;
  };
  // pointwise epilogue operands of cell plane il (RKL2 stage only)
  auto load_epi = [&](int il, double& ym2, double& y0, double& m0) {
    if constexpr (EPI == EPI_RKL2_STAGE) {
      if (own && il < ie) {
        const long long gi = (long long)il * G.plane + coff;
        ym2 = c.ea.ym2[gi];
        y0 = c.ea.y0[gi];
        m0 = c.ea.m0[gi];
      }
    }
  };
  auto vbox = [&](double& SA, double& DB, double& DC) {
    if (!own) return;
    const double a00 = vA[tid], a01 = vA[tid + 1], a10 = vA[tid + 32], a11 = vA[tid + 33];
    const double b00 = vB[tid], b01 = vB[tid + 1], b10 = vB[tid + 32], b11 = vB[tid + 33];
    const double d00 = vC[tid], d01 = vC[tid + 1], d10 = vC[tid + 32], d11 = vC[tid + 33];
    SA = (a00 + a01) + (a10 + a11);
    DB = (b00 + b01) - (b10 + b11);
    DC = (d00 + d10) - (d01 + d11);
  };

  // ---- prologue: cell planes ib-1, ib -> vertex plane ib-1/2 ----
  double SuL, TuL, FuL, SuH, TuH, FuH;
  double SAl = 0, DBl = 0, DCl = 0;
  double er, et, ep;
  stage(ib - 1, (ib - 1) & 1);
  stage(ib, ib & 1);
  load_e(ib - 1, er, et, ep);
  cp_async_wait_all();
  __syncthreads();
  usums((ib - 1) & 1, SuL, TuL, FuL);
  usums(ib & 1, SuH, TuH, FuH);
  double uc = us[(ib & 1) * FRC + c11];
  vertex(ib - 1, er, et, ep, SuL, TuL, FuL, SuH, TuH, FuH);
  __syncthreads();
  vbox(SAl, DBl, DCl);
  SuL = SuH;
  TuL = TuH;
  FuL = FuH;
  if (ib + 1 <= ie) stage(ib + 1, (ib + 1) & 1);   // overwrites plane ib-1 (all reads done)
  // register prefetch, one plane ahead: e of vertex plane ib+1/2, epilogue operands of cell plane ib
  load_e(ib, er, et, ep);
  double ym2 = 0, y0 = 0, m0 = 0;
  load_epi(ib, ym2, y0, m0);

  double part = 0.0;
  for (int il = ib; il < ie; ++il) {
    const double erc = er, etc = et, epc = ep;
    const double ym2c = ym2, y0c = y0, m0c = m0;
    load_e(il + 1, er, et, ep);                       // in flight during this plane
    load_epi(il + 1, ym2, y0, m0);
    cp_async_wait_all();
    __syncthreads();                                  // plane il+1 staged; vertex smem free
    if (il + 2 <= ie) stage(il + 2, il & 1);          // prefetch: overwrites plane il (in registers)
    usums((il + 1) & 1, SuH, TuH, FuH);
    const double un = us[((il + 1) & 1) * FRC + c11];
    vertex(il, erc, etc, epc, SuL, TuL, FuL, SuH, TuH, FuH);
    __syncthreads();
    double SAh = 0, DBh = 0, DCh = 0;
    vbox(SAh, DBh, DCh);
    if (own) {
      const int ig = G.i0 + il;
      const double ig2c = M.iG2[ig];
      const double Lu = -((SAl - SAh) + ig2c * (DBl + DBh) + ig2c * ig3c * (DCl + DCh));
      const double WV = (c.w ? __ldg(c.w + (long long)il * G.plane + coff) : 1.0) * M.Vr[ig] * vtpc;
      const long long gi = (long long)il * G.plane + coff;
      if constexpr (EPI == EPI_F) {
        c.ea.out[gi] = Lu / WV;
      } else if constexpr (EPI == EPI_RKL2_FIRST) {
        const double F = Lu / WV;
        c.ea.out2[gi] = F;
        c.ea.out[gi] = c.ea.a0 * uc + c.ea.c0 * F;
      } else if constexpr (EPI == EPI_RKL2_STAGE) {
        const double F = Lu / WV;
        c.ea.out[gi] = c.ea.mu * uc + c.ea.nu * ym2c + c.ea.c2 * y0c + c.ea.c0 * F + c.ea.c1 * m0c;
      } else if constexpr (EPI == EPI_PCG_AP) {
        const double y = WV * uc - c.ea.dt * Lu;
        c.ea.out[gi] = y;
        part += uc * y;
      }
    }
    SAl = SAh;
    DBl = DBh;
    DCl = DCh;
    SuL = SuH;
    TuL = TuH;
    FuL = FuH;
    uc = un;
  }
  if constexpr (EPI == EPI_PCG_AP) {
    double v[1] = {part};
    block_partials<1>(v, c.ea.partials, c.ea.pstride, c.ea.pbase + blk);
  }
}

// A CTA owns 8 x 32 padded vertex positions (rows jv+1, cols kv+1) and
// marches along r; each cell plane of b (3 comps) and the three face diffusivities is
// staged once in shared memory (2-plane ring, 9 x 33 cells with halo and periodic wrap)
// and shared by the 8 vertices around every cell (coalesced loads instead of 36
// gathers per vertex).  e for every vertex plane il = -1 .. nl-1 of a slab (vertex
// between cell planes il and il+1) in the padded layout of ev_row/ev_plane
// (sts_common.cuh): column kv+1 holds vertex kv, column 0 the periodic wrap copy of
// kv = n3-1, zero where the vertex has a missing cell.
constexpr int VCJ = 8, VCK = 32, VCR = VCJ + 1, VCC = VCK + 1, VCN = VCR * VCC;   // 9 x 33 cells
__global__ void __launch_bounds__(256) vertex_coef_tiled_kernel(Geo G, FieldV b, FieldV k1, FieldV k2, FieldV k3,
                                                                double* __restrict__ ev, int ic) {
  __shared__ double cs[3][6][VCN];   // cell planes il, il+1 and the one in flight (cp.async)
  const Metrics& M = G.m;
  const int tid = threadIdx.x;
  const int R0 = blockIdx.y * VCJ, C0 = blockIdx.x * VCK;        // padded row / col origin
  const int vlo = -1 + (int)blockIdx.z * ic;                     // vertex planes [vlo, vhi)
  const int vhi = min(vlo + ic, G.nl);
  const long long row = ev_row(G.n3), pp = ev_plane(G.n2, G.n3), es = (long long)(G.nl + 1) * pp;
  // stage cell plane il (-1..nl) into ring slot (il + 3) % 3 asynchronously: cells rows R0-1+r
  // (r < 9), cols C0-1+c (c < 33); missing cells / planes are zero-filled
  auto stage = [&](int il) {
    const int sl = (il + 3) % 3;
    const double* src[6] = {plane_ptr(b, G, il, 0), plane_ptr(b, G, il, 1), plane_ptr(b, G, il, 2),
                            plane_ptr(k1, G, il, 0), plane_ptr(k2, G, il, 0), plane_ptr(k3, G, il, 0)};
    for (int e = tid; e < VCN; e += 256) {
      const int r = e / VCC, cc = e - r * VCC;
      const int j = R0 - 1 + r;
      int k = C0 - 1 + cc;
      bool ok = j >= 0 && j < G.n2;
      if (G.periodic3) k = (k % G.n3 + G.n3) % G.n3;
      else ok = ok && k >= 0 && k < G.n3;
      const long long o = ok ? (long long)j * G.n3 + k : 0;
#pragma unroll
      for (int f = 0; f < 6; ++f) cp_async8(&cs[sl][f][e], (ok && src[f]) ? src[f] + o : ev, ok && src[f]);
    }
    cp_async_commit();
  };
  const int vr = tid >> 5, vc = tid & 31;                        // this thread's padded vertex (R0+vr, C0+vc)
  const int jv = R0 + vr - 1;
  int kv = C0 + vc - 1;
  if (kv == -1 && G.periodic3) kv = G.n3 - 1;
  const bool inrange = (R0 + vr) <= G.n2 && (C0 + vc) < (int)row;
  // cells of the vertex in the staged tile: rows vr, vr+1 ; cols vc, vc+1 (tile col c <-> global C0-1+c)
  const int o00 = vr * VCC + vc, o01 = o00 + 1, o10 = o00 + VCC, o11 = o10 + 1;
  stage(vlo);
  stage(vlo + 1);
  for (int il = vlo; il < vhi; ++il) {
    cp_async_wait_all();   // cell planes il and il+1 have landed (this thread's copies)
    __syncthreads();       // ... everyone's; and plane il-1's slot is no longer read
    if (il + 2 <= vhi) stage(il + 2);   // in flight during this plane's work
    const int iv = G.i0 + il;
    bool ok = inrange && kv >= 0 && kv < G.n3 && iv >= 0 && iv + 1 < G.n1g && jv >= 0 && jv + 1 < G.n2 &&
              (G.periodic3 || kv + 1 < G.n3);
    double er = 0.0, et = 0.0, ep = 0.0;
    if (ok) {
      const int kv1 = (kv + 1 < G.n3) ? kv + 1 : 0;
      const double(&L)[6][VCN] = cs[(il + 3) % 3];
      const double(&H)[6][VCN] = cs[(il + 4) % 3];
      const double br = 0.125 * ((L[0][o00] + L[0][o01]) + (L[0][o10] + L[0][o11]) + ((H[0][o00] + H[0][o01]) + (H[0][o10] + H[0][o11])));
      const double bt = 0.125 * ((L[1][o00] + L[1][o01]) + (L[1][o10] + L[1][o11]) + ((H[1][o00] + H[1][o01]) + (H[1][o10] + H[1][o11])));
      const double bp = 0.125 * ((L[2][o00] + L[2][o01]) + (L[2][o10] + L[2][o11]) + ((H[2][o00] + H[2][o01]) + (H[2][o10] + H[2][o11])));
      const double kap = (1.0 / 12.0) * (((L[3][o00] + L[3][o01]) + (L[3][o10] + L[3][o11])) +
                                         ((L[4][o00] + L[4][o01]) + (L[5][o00] + L[5][o10])) +
                                         ((H[4][o00] + H[4][o01]) + (H[5][o00] + H[5][o10])));
      const double C = 0.125 * (M.Vr[iv] + M.Vr[iv + 1]) * (M.Vt[jv] + M.Vt[jv + 1]) * (M.Vp[kv] + M.Vp[kv1]) * kap;
      const double sq = sqrt(C);
      er = sq * 0.25 * br * M.iH1[iv];
      et = sq * 0.25 * bt * M.iH2[jv];
      ep = sq * 0.25 * bp * M.iH3[kv];
    }
    if (inrange) {
      const long long e = (long long)(il + 1) * pp + (long long)(R0 + vr) * row + (C0 + vc);
      ev[e] = er;
      ev[es + e] = et;
      ev[2 * es + e] = ep;
    }
  }
  cp_async_wait_all();
}

void launch_vertex_coef(const Geo& G, FieldV b, FieldV k1, FieldV k2, FieldV k3, double* ev, cudaStream_t st) {
  const long long nv = (long long)(G.nl + 1) * ev_plane(G.n2, G.n3);
  if (nv == 0) return;
  const int nbx = (int)((ev_row(G.n3) + VCK - 1) / VCK), nby = (G.n2 + 1 + VCJ - 1) / VCJ;
  const int np = G.nl + 1;
  const int ic = choose_chunk((long long)nbx * nby, np, 148LL * 4, 1.0, 4);
  vertex_coef_tiled_kernel<<<dim3(nbx, nby, (np + ic - 1) / ic), 256, 0, st>>>(G, b, k1, k2, k3, ev, ic);
  STS_CUDA(cudaGetLastError());
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
          c.ea.out[go] = c.ea.a0 * uc[q] + c.ea.c0 * F;
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
          if (c.ea.out3) c.ea.out3[go] = z;
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
// isotropic 7-point kernel, fast path (F / RKL2 stages / PCG A p), ncomp <= 3
// ----------------------------------------------------------------------------
// CTA = 8 x 32 (theta x phi) cell columns marching along r.  The u planes (all
// components) and the theta / phi face diffusivities are staged in shared memory
// with cp.async TWO planes ahead (3-slot ring), so the up-neighbour plane is
// resident when a plane is processed and its successor is in flight; the r-face
// diffusivity and w of the own column are register-prefetched one plane ahead.
// ============================================================================
constexpr int IRC = RC;   // (TJ+2) x (TK+2) staged region per field

template <int NC>
struct IsoSmem {
  static constexpr int NF = NC + 2;                       // u comps + k2 + k3
  static constexpr size_t bytes = (size_t)3 * NF * IRC * sizeof(double);
};

__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

template <int EPI, int NC>
__global__ void __launch_bounds__(NT, (NC >= 3 ? 2 : 3)) iso_fast_kernel(StencilCall c, int ic) {
  constexpr int NF = NC + 2;
  extern __shared__ double sm[];
  const Geo& G = c.geo;
  const Metrics& M = G.m;
  const int tid = threadIdx.x;
  const int tk = tid % TK, tj = tid / TK;
  const int j0 = blockIdx.y * TJ, k0 = blockIdx.x * TK;
  const int ib = c.ib + blockIdx.z * ic;
  const int ie = min(ib + ic, c.ie);
  const long long blk = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
  bool skip[NC];
  bool all = true;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    skip[q] = (EPI == EPI_PCG_AP) && c.ea.sc && c.ea.sc[q].done;
    all = all && skip[q];
  }
  if (EPI == EPI_PCG_AP && all) return;

  // staging assignments (fixed)
  int soff[2];
  bool sok[2], shas[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int e = tid + q * NT;
    shas[q] = e < IRC;
    const int row = e / RK, col = e - (e / RK) * RK;
    const int j = j0 - 1 + row;
    int k = k0 - 1 + col;
    bool ok = shas[q] && j >= 0 && j < G.n2;
    if (G.periodic3) k = wrapk(k, G.n3);
    else ok = ok && k >= 0 && k < G.n3;
    sok[q] = ok;
    soff[q] = ok ? j * G.n3 + k : 0;
  }
  auto slot_ptr = [&](int plane, int f) { return sm + ((plane % 3 + 3) % 3 * NF + f) * IRC; };
  auto stage = [&](int il) {   // plane il in [-1, nl] (absent planes -> zeros)
    const double* src[NF];
#pragma unroll
    for (int q = 0; q < NC; ++q) src[q] = plane_ptr(c.u, G, il, q);
    src[NC] = plane_ptr(c.k2, G, il, 0);
    src[NC + 1] = plane_ptr(c.k3, G, il, 0);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!shas[q]) continue;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const bool ok = sok[q] && src[f] != nullptr;
        cp_async8(slot_ptr(il, f) + tid + q * NT, ok ? src[f] + soff[q] : c.k1.p, ok);
      }
    }
    cp_async_commit();
  };

  const int j = j0 + tj, k = k0 + tk;
  const bool own = (j < G.n2) && (k < G.n3);
  const long long coff = own ? (long long)j * G.n3 + k : 0;
  const bool jm = j >= 1, jp = j + 1 < G.n2;
  const bool kself = G.periodic3 && G.n3 == 1;
  const bool km = !kself && (G.periodic3 || k >= 1), kp = !kself && (G.periodic3 || k + 1 < G.n3);
  const int kmw = G.periodic3 ? wrapk(k - 1, G.n3) : k - 1;
  double f1tp = 0, f2p = 0, f2m = 0, f3p = 0, f3m = 0, vtp = 0;
  if (own) {
    f1tp = M.F1t[j] * M.F1p[k];
    f2p = jp ? M.F2t[j] * M.F2p[k] : 0.0;
    f2m = jm ? M.F2t[j - 1] * M.F2p[k] : 0.0;
    f3p = kp ? M.F3t[j] * M.F3p[k] : 0.0;
    f3m = km ? M.F3t[j] * M.F3p[kmw] : 0.0;
    vtp = M.Vt[j] * M.Vp[k];
  }
  const int r0 = (tj + 1) * RK + tk + 1;   // own cell in the staged region

  // prologue: stage planes ib, ib+1 (ib-1 only needed for the own-column u_dn)
  stage(ib);
  stage(ib + 1);
  double udn[NC], uc[NC];
  const int ig0 = G.i0 + ib;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const double* pd = (own && ig0 >= 1) ? plane_ptr(c.u, G, ib - 1, q) : nullptr;
    udn[q] = pd ? __ldg(pd + coff) : 0.0;
  }
  double kdn = 0.0;
  if (own && ig0 >= 1) kdn = __ldg(plane_ptr(c.k1, G, ib - 1, 0) + coff) * M.F1r[ig0 - 1] * f1tp;
  // register prefetch of the own column's r-face diffusivity and w (plane ib)
  double k1n = (own && ig0 + 1 < G.n1g) ? __ldg(plane_ptr(c.k1, G, ib, 0) + coff) : 0.0;
  double wn = (own && c.w) ? __ldg(c.w + (long long)ib * G.plane + coff) : 1.0;
  double part[NC];
  double ym2n[NC], y0n[NC], m0n[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    part[q] = 0.0;
    ym2n[q] = y0n[q] = m0n[q] = 0.0;
    if (EPI == EPI_RKL2_STAGE && own) {
      const long long go = (long long)ib * G.plane + coff + (long long)q * G.cstride;
      ym2n[q] = c.ea.ym2[go];
      y0n[q] = c.ea.y0[go];
      m0n[q] = c.ea.m0[go];
    }
  }
  bool first = true;

  for (int il = ib; il < ie; ++il) {
    const int ig = G.i0 + il;
    const bool ip = ig + 1 < G.n1g;
    if (il + 2 <= ie) stage(il + 2);   // slot of plane il-1 (finished last step)
    else cp_async_commit();            // keep the group count uniform
    const double k1c = k1n, wc = wn;
    if (own && il + 1 < ie) {          // prefetch next plane's column values
      k1n = (ig + 2 < G.n1g) ? __ldg(plane_ptr(c.k1, G, il + 1, 0) + coff) : 0.0;
      wn = c.w ? __ldg(c.w + (long long)(il + 1) * G.plane + coff) : 1.0;
    }
    // epilogue operands: use the ones prefetched last step, prefetch the next plane's
    double ym2[NC], y0v[NC], m0v[NC];
    const long long gi = (long long)il * G.plane + coff;
    if constexpr (EPI == EPI_RKL2_STAGE) {
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        ym2[q] = ym2n[q];
        y0v[q] = y0n[q];
        m0v[q] = m0n[q];
        if (own && il + 1 < ie) {
          const long long go = gi + G.plane + (long long)q * G.cstride;
          ym2n[q] = c.ea.ym2[go];
          y0n[q] = c.ea.y0[go];
          m0n[q] = c.ea.m0[go];
        }
      }
    }
    cp_async_wait_1();                 // planes il and il+1 have landed (own copies)
    __syncthreads();                   // ... and everybody's
    if (own) {
      if (first) {
#pragma unroll
        for (int q = 0; q < NC; ++q) uc[q] = slot_ptr(il, q)[r0];
        first = false;
      }
      const double f23r = M.F2r[ig], f3r = M.F3r[ig];
      const double* K2 = slot_ptr(il, NC);
      const double* K3 = slot_ptr(il, NC + 1);
      const double Kup = ip ? k1c * M.F1r[ig] * f1tp : 0.0;
      const double Kjp = jp ? K2[r0] * f23r * f2p : 0.0;
      const double Kjm = jm ? K2[r0 - RK] * f23r * f2m : 0.0;
      const double Kkp = kp ? K3[r0] * f3r * f3p : 0.0;
      const double Kkm = km ? K3[r0 - 1] * f3r * f3m : 0.0;
      const double WV = wc * M.Vr[ig] * vtp;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const double* U = slot_ptr(il, q);
        const double uup = ip ? slot_ptr(il + 1, q)[r0] : 0.0;
        const double u0 = uc[q];
        const double Lu = kdn * (udn[q] - u0) + Kup * (uup - u0) + Kjm * (U[r0 - RK] - u0) +
                          Kjp * (U[r0 + RK] - u0) + Kkm * (U[r0 - 1] - u0) + Kkp * (U[r0 + 1] - u0);
        const long long go = gi + (long long)q * G.cstride;
        if (!skip[q]) {
          if constexpr (EPI == EPI_F) {
            c.ea.out[go] = Lu / WV;
          } else if constexpr (EPI == EPI_RKL2_FIRST) {
            const double F = Lu / WV;
            c.ea.out2[go] = F;
            c.ea.out[go] = c.ea.a0 * u0 + c.ea.c0 * F;
          } else if constexpr (EPI == EPI_RKL2_STAGE) {
            const double F = Lu / WV;
            c.ea.out[go] = c.ea.mu * u0 + c.ea.nu * ym2[q] + c.ea.c2 * y0v[q] + c.ea.c0 * F + c.ea.c1 * m0v[q];
          } else if constexpr (EPI == EPI_PCG_AP) {
            const double y = WV * u0 - c.ea.dt * Lu;
            c.ea.out[go] = y;
            part[q] += u0 * y;
          }
        }
        udn[q] = u0;
        uc[q] = uup;
      }
      kdn = Kup;
    }
    __syncthreads();                   // slot of plane il is restaged next step
  }
  cp_async_wait_all();
  if constexpr (EPI == EPI_PCG_AP) block_partials<NC>(part, c.ea.partials, c.ea.pstride, c.ea.pbase + blk);
}

// ============================================================================
// launch plumbing
// ============================================================================
static bool use_fast(int mode, int epi) {
  return mode == STS_MODE_ANISO &&
         (epi == EPI_F || epi == EPI_RKL2_FIRST || epi == EPI_RKL2_STAGE || epi == EPI_PCG_AP);
}
bool stencil_uses_vertex_coef(int mode, int epi) { return use_fast(mode, epi); }

// grid of the kernel launch_stencil uses for (mode, epi) on local planes [ib, ie)
static dim3 stencil_grid(int mode, int epi, const Geo& G, int ib, int ie, int* ic_out) {
  const bool fast = use_fast(mode, epi);
  const int tk = fast ? FOK : TK, tj = fast ? FOJ : TJ;
  const int nbx = (G.n3 + tk - 1) / tk, nby = (G.n2 + tj - 1) / tj;
  const int np = ie - ib;
  if (np <= 0) {
    if (ic_out) *ic_out = 1;
    return dim3(0, 0, 0);
  }
  // ~4 waves of 148 SMs x 3 resident CTAs, but >= 8 planes per chunk (each chunk
  // re-stages one extra plane)
  const long long tiles = (long long)nbx * nby;
  const long long want = 148LL * 3 * 4;
  int ic = (int)((np * tiles + want - 1) / want);
  ic = ic < 8 ? 8 : ic;
  if (ic > np) ic = np;
  if (ic_out) *ic_out = ic;
  return dim3(nbx, nby, (np + ic - 1) / ic);
}

int stencil_blocks(int mode, int epi, const Geo& G, int ib, int ie) {
  const dim3 g = stencil_grid(mode, epi, G, ib, ie, nullptr);
  return (int)(g.x * g.y * g.z);
}

template <int EPI, int NC>
static void launch_iso_fast(const StencilCall& c, dim3 grid, int ic, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  ensure_smem_attr(iso_fast_kernel<EPI, NC>, (int)IsoSmem<NC>::bytes, attr);
  iso_fast_kernel<EPI, NC><<<grid, NT, IsoSmem<NC>::bytes, st>>>(c, ic);
}

template <int EPI>
static void launch_epi(const StencilCall& c, cudaStream_t st, unsigned long long* dmax) {
  int ic = 1;
  const dim3 grid = stencil_grid(c.mode, EPI, c.geo, c.ib, c.ie, &ic);
  if (grid.x == 0) return;
  if (c.mode == STS_MODE_ANISO) {
    if constexpr (EPI == EPI_F || EPI == EPI_RKL2_FIRST || EPI == EPI_RKL2_STAGE || EPI == EPI_PCG_AP) {
      static std::atomic<unsigned long long> attr_fast{0};
      ensure_smem_attr(aniso_fast_kernel<EPI>, (int)FAST_SMEM, attr_fast);
      if (!c.ev) throw Error{STS_ERR_STATE, "vertex coefficients missing for the anisotropic fast path"};
      aniso_fast_kernel<EPI><<<grid, FNT, FAST_SMEM, st>>>(c, ic);
    } else {
      static std::atomic<unsigned long long> attr_set{0};
      ensure_smem_attr(aniso_kernel<EPI>, (int)ANISO_SMEM, attr_set);
      aniso_kernel<EPI><<<grid, NT, ANISO_SMEM, st>>>(c, ic, dmax);
    }
  } else {
    if constexpr (EPI == EPI_F || EPI == EPI_RKL2_FIRST || EPI == EPI_RKL2_STAGE || EPI == EPI_PCG_AP) {
      switch (c.ncomp) {
        case 1: launch_iso_fast<EPI, 1>(c, grid, ic, st); break;
        case 2: launch_iso_fast<EPI, 2>(c, grid, ic, st); break;
        case 3: launch_iso_fast<EPI, 3>(c, grid, ic, st); break;
        default: throw Error{STS_ERR_ARG, "ncomp must be 1..3"};
      }
    } else {
      switch (c.ncomp) {
        case 1: iso_kernel<EPI, 1><<<grid, NT, 0, st>>>(c, ic, dmax); break;
        case 2: iso_kernel<EPI, 2><<<grid, NT, 0, st>>>(c, ic, dmax); break;
        case 3: iso_kernel<EPI, 3><<<grid, NT, 0, st>>>(c, ic, dmax); break;
        default: throw Error{STS_ERR_ARG, "ncomp must be 1..3"};
      }
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

// ============================================================================
// Gershgorin row sums from the frozen vertex coefficients (App. B)
// ----------------------------------------------------------------------------
// With e = sqrt(V_v kappa_v) b_v / (4 h) (vertex_coef_tiled_kernel), the weight of the
// cell at corner sigma of vertex v in (b_v . g_v) is
//   g_v(sigma) = s1 e_r + s2 e_t / r_i + s3 e_p / (r_i sin th_j),  s_a = 2 sigma_a - 1,
// (i, j) = the cell's r / theta indices, and E_v = 1/2 (sum_sigma g_v(sigma) u_sigma)^2,
// so L_cq = -sum over the vertices v shared by c and q of g_v(sigma_c) g_v(sigma_q).
// A CTA = 8 warps x 32 lanes = one 8 x 32 block of vertices (vertex row per warp) and
// its 7 x 31 cells; it marches along r.  Per vertex plane each thread computes the 8
// weights of ITS vertex once (e prefetched one plane ahead), stores them for the warp
// below through shared memory (the only CTA barrier of the plane), and takes the
// right-hand neighbours' weights by shuffle: 8 shared loads + 16 shuffles of doubles per
// cell and plane instead of 64 shared loads (the previous version computed all weights
// into shared memory and was shared-memory bound, 0.13 of the copy peak).  A vertex
// plane completes the row of the cell plane below it (entries with the plane above:
// dz = 2, and the rest of its own plane) and opens the row of the cell plane above it
// (entries with the plane below are complete at once, so only their |.| sum and the 9
// own-plane partials are carried).  24 B of e per cell; bound by the FP64 pipe
// (~115 FP64 instructions per cell) and the MIO pipe.  n3 >= 3 (no aliased phi
// neighbours).
constexpr int GJ = 8, GK = 32, GOJ = GJ - 1, GOK = GK - 1;
constexpr int GNT = GJ * GK;

__global__ void __launch_bounds__(GNT, 2) gersh_ev_kernel(Geo G, const double* __restrict__ ev,
                                                          const double* __restrict__ w, int ib0, int ie0, int ic,
                                                          unsigned long long* dmax) {
  __shared__ double gsm[2][8][GNT];
  const Metrics& M = G.m;
  const int tid = threadIdx.x, tj = tid >> 5, tk = tid & 31;
  const int k0 = blockIdx.x * GOK, j0 = blockIdx.y * GOJ;
  const int ib = ib0 + blockIdx.z * ic, ie = min(ib + ic, ie0);
  const long long row = ev_row(G.n3), pp = ev_plane(G.n2, G.n3), es = ev_cstride(G.nl, G.n2, G.n3);
  // this thread's vertex (jv, kv) = (j0 - 1 + tj, k0 - 1 + tk) and cell (j, k) = (j0 + tj, k0 + tk)
  const int jv = j0 - 1 + tj, kv = k0 - 1 + tk;
  const bool vin = jv >= 0 && jv + 1 < G.n2 && kv + 1 <= G.n3;   // (vertex rows between cell rows only)
  const long long vo = (long long)(jv + 1) * row + (kv + 1);
  const double ig3l = vin ? M.iG3[jv] : 0.0, ig3h = vin ? M.iG3[jv + 1] : 0.0;
  const int j = j0 + tj, k = k0 + tk;
  const bool own = tj < GOJ && tk < GOK && j < G.n2 && k < G.n3;
  const double vtp = own ? M.Vt[j] * M.Vp[k] : 0.0;
  auto load_e = [&](int il, double& er, double& et, double& ep) {
    const int iv = G.i0 + il;
    er = et = ep = 0.0;
    if (vin && iv >= 0 && iv + 1 < G.n1g && il + 1 >= 0 && il + 1 <= G.nl) {
      const long long o = (long long)(il + 1) * pp + vo;
      er = __ldg(ev + o);
      et = __ldg(ev + es + o);
      ep = __ldg(ev + 2 * es + o);
    }
  };
  // weights g[s], s = (s1 s2 s3) bits, of this thread's vertex in vertex plane il
  auto weights = [&](int il, double er, double et, double ep, double g[8]) {
    const int iv = G.i0 + il;
    const double g2l = (iv >= 0 && iv < G.n1g) ? M.iG2[iv] : 0.0;
    const double g2h = (iv + 1 >= 0 && iv + 1 < G.n1g) ? M.iG2[iv + 1] : 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int s1 = (s >> 2) & 1, s2 = (s >> 1) & 1, s3 = s & 1;
      const double ig2 = s1 ? g2h : g2l, ig3 = s2 ? ig3h : ig3l;
      g[s] = (s1 ? er : -er) + (s2 ? et : -et) * ig2 + (s3 ? ep : -ep) * (ig2 * ig3);
    }
  };
  double rowmax = 0.0;
  double cmid[9], clow = 0.0;   // the open row of the cell plane above the last vertex plane
#pragma unroll
  for (int q = 0; q < 9; ++q) cmid[q] = 0.0;
  double er, et, ep;
  load_e(ib - 1, er, et, ep);
  for (int il = ib - 1; il < ie; ++il) {   // vertex plane il, between cell planes il and il+1
    double g[8], gn[8];
    weights(il, er, et, ep, g);
    if (il + 1 < ie) load_e(il + 1, er, et, ep);   // prefetch the next plane's e
    double* gp = gsm[il & 1][0];
#pragma unroll
    for (int s = 0; s < 8; ++s) gp[s * GNT + tid] = g[s];
    __syncthreads();
    // the cell's 4 vertices: (a, b) = (0, 0) own, (0, 1) right (shuffle), (1, 0) below
    // (shared memory, the next warp), (1, 1) below-right; the cell sits at octant
    // (c2, c3) = (1 - a, 1 - b) of vertex (a, b)
    double top[9], low[9], nmid[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) top[q] = low[q] = nmid[q] = 0.0;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      if (a == 1) {
#pragma unroll
        for (int s = 0; s < 8; ++s) g[s] = tj + 1 < GJ ? gp[s * GNT + tid + 32] : 0.0;
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) gn[s] = __shfl_down_sync(0xffffffffu, g[s], 1);
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double* gv = b ? gn : g;
        const int c2 = 1 - a, c3 = 1 - b;
        const double glo = gv[(0 << 2) | (c2 << 1) | c3];   // cell il (below the vertex plane): s1 = 0
        const double ghi = gv[(1 << 2) | (c2 << 1) | c3];   // cell il+1 (above): s1 = 1
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int q1 = (q >> 2) & 1, q2 = (q >> 1) & 1, q3 = q & 1;
          const int e9 = (q2 - c2 + 1) * 3 + (q3 - c3 + 1);
          if (q1 == 0) {
            cmid[e9] = fma(glo, gv[q], cmid[e9]);   // cell il, neighbours in plane il
            low[e9] = fma(ghi, gv[q], low[e9]);     // cell il+1, neighbours in plane il
          } else {
            top[e9] = fma(glo, gv[q], top[e9]);     // cell il, neighbours in plane il+1
            nmid[e9] = fma(ghi, gv[q], nmid[e9]);   // cell il+1, neighbours in plane il+1
          }
        }
      }
    }
    if (il >= ib && own) {   // the row of cell (il, j, k) is complete
      double sum = clow;
#pragma unroll
      for (int q = 0; q < 9; ++q) sum += fabs(cmid[q]) + fabs(top[q]);
      const int ig = G.i0 + il;
      const double WV = (w ? __ldg(w + (long long)il * G.plane + (long long)j * G.n3 + k) : 1.0) * M.Vr[ig] * vtp;
      rowmax = fmax(rowmax, sum / WV);
    }
    clow = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      clow += fabs(low[q]);
      cmid[q] = nmid[q];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rowmax = fmax(rowmax, __shfl_xor_sync(0xffffffffu, rowmax, o));
  if ((tid & 31) == 0 && rowmax > 0.0) atomicMax(dmax, (unsigned long long)__double_as_longlong(rowmax));
}

void launch_gershgorin(const StencilCall& c, unsigned long long* d_max, cudaStream_t st) {
  const Geo& G = c.geo;
  if (c.mode == STS_MODE_ANISO && c.ev && G.n3 >= 3) {
    const int nbx = (G.n3 + GOK - 1) / GOK, nby = (G.n2 + GOJ - 1) / GOJ;
    const int np = c.ie - c.ib;
    if (np <= 0) return;
    const int ic = choose_chunk((long long)nbx * nby, np, 148LL * 2, 1.0, 4);
    gersh_ev_kernel<<<dim3(nbx, nby, (np + ic - 1) / ic), GNT, 0, st>>>(G, c.ev, c.w, c.ib, c.ie, ic, d_max);
    STS_CUDA(cudaGetLastError());
    return;
  }
  launch_epi<EPI_GERSH>(c, st, d_max);
}

}  // namespace sts
