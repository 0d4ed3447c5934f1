// TMA + mbarrier pipelined isotropic 7-point stencil pass, ncomp <= 3 (sm_100a).
//
// Operator (R2, PAPER.md:181 boxed viscosity term (1/rho) div(nu rho grad v)
// component-wise, PAPER.md:329 constant-coefficient heat test):
//   (L u)_i = sum_faces K_f (u_nb - u_i),   K_f = kappa_f A_f / h_f,   F = L u / (w V)
// with exactly the arithmetic of iso_fast_kernel (stencil.cu).
//
// Warp-specialised: IJ consumer warps own an IJ x 32 (theta x phi) tile of cell
// columns and march along r; one producer warp streams one "package" per r-plane
// into a ring of shared-memory slots with cp.async.bulk.tensor (TMA):
//   per component of each staged source field: 36 x (IJ+2) box from (k0-2, j0-1)
//        (+ 2-column periodic-wrap boxes on the edge tiles),
//   theta-face coefficient: 32 x (IJ+1) from (k0, j0-1); phi-face: 34 x IJ from
//   (k0-2, j0) (+ wrap), r-face and w: 32 x IJ, epilogue operands: 32 x IJ each.
// Every box origin column is even (16 B aligned, see tma.cuh).  A full mbarrier per
// slot signals "landed", an empty mbarrier (one arrival per consumer warp) signals
// "free"; there is no CTA-wide barrier in the march.
// Tiles (IsoTile / IsoLay): 7 rows at two CTAs per SM for every pass but the
// 3-component merged PCG pass, which runs 13 rows at one CTA per SM with two
// "former" warps (see IsoLay::FORM).
// Epilogues: F, RKL2 first stage / stage recurrence (Fig. 2, also in
// deviation form D_j = Y_j - Y0), the PCG initial residual (R0), the two-pass PCG
// S-pass, and the merged one-pass PCG iteration (Fig. 1 reorganised,
// DESIGN.md §5.3): from staged p_{k-2}, w_{k-1}, p_{k-1},
// z = (p_{k-1} - beta_{k-1} p_{k-2}) - alpha w_{k-1}, p = z + beta p_{k-1}, y = A p,
// w = d y, the four partial sums, x updated every other pass.  Passes other than the merged one take
// the own column's r-neighbours from registers prefetched two planes ahead; the
// merged pass takes the r-up neighbour from the next plane's slot instead.
#include "sts_common.cuh"
#include "tma.cuh"
#include "pcg.cuh"

namespace sts {

using namespace tma;

namespace {

constexpr int IK = 32;                    // tile cols = lanes
constexpr int SBW = 36;                   // staged source box cols
constexpr int rnd16(int n) { return (n + 15) / 16 * 16; }   // 128 B multiples of doubles
constexpr int K2W = 32, K3W = 34;
constexpr int SMEM_1CTA = 232448;         // max dynamic shared memory of one CTA (227 KB)

// Tile geometry of IJ rows: IJ consumer warps own an IJ x 32 (theta x phi) tile
// and one producer warp streams its packages.
//  * IJ = 7, 2 CTAs per SM: 8 warps per CTA -> 4 warps per SM sub-partition, so the
//    64K-register file allows 128 registers per thread (8 consumer warps would drop
//    that to 96 and the 3-component PCG S-pass spills);
//  * ISO_M3_ROWS (13) rows, 1 CTA per SM, for the 3-component merged PCG pass, whose
//    three staged fields make a 7-row slot too large for three ring slots at 2 CTAs
//    per SM: 13 consumer + producer + ISO_FORMERS (2) former warps, 128 registers
//    (the pass reads metric-folded coefficients), three 72 KB slots.  Measured c4
//    fraction of the copy peak by rows (one former warp): 7: 0.79, 8: 0.77, 9: 0.85,
//    11: 0.83, 12: 0.82, 13: 0.86 (14 rows no longer fit three slots); two former
//    warps 0.874 at 13 rows (12 rows with three: 0.874, 11 with three: 0.81).
template <int IJ_>
struct IsoTile {
  static constexpr int IJ = IJ_;
  static constexpr int INT = IJ * IK;               // consumer threads
  static constexpr int SBH = IJ + 2;                // staged source box rows
  static constexpr int S_MAIN = rnd16(SBW * SBH);   // 7 rows: 324 -> 336
  static constexpr int S_W = rnd16(2 * SBH);        // 2 x SBH wrap box
  static constexpr int K2H = IJ + 1, K2SZ = rnd16(K2W * K2H);
  static constexpr int K3H = IJ, K3SZ = rnd16(K3W * K3H);
  static constexpr int K3WR = rnd16(2 * K3H);       // 2 x IJ wrap box
  static constexpr int OWN = IK * IJ;               // 32 x IJ own box
};

// rows of the tile and resident CTAs per SM of one (epilogue, ncomp) variant (host and device)
#ifndef ISO_M3_ROWS
#define ISO_M3_ROWS 13
#endif
#ifndef ISO_RASTER_H     // (theta-first bands measured worse for L2: DESIGN.md §5.4)
#define ISO_RASTER_H 0
#endif
#ifndef ISO_FORM_SPLIT   // one formed barrier per component (consumers start on component 0 earlier; measured neutral: off)
#define ISO_FORM_SPLIT 0
#endif
#ifndef ISO_FORM_UNROLL  // the former warps' loop fully unrolled (measured neutral: off)
#define ISO_FORM_UNROLL 0
#endif
#ifndef ISO_FORM_TRIM    // the former warps form only the staged positions the stencil reads (1: one position
#define ISO_FORM_TRIM 0      // per form; 2: 16-byte aligned pairs); measured slower: off
#endif
#ifndef ISO_M_XG         // merged 3-component PCG: x read per thread from global (issued before the slot
#define ISO_M_XG 0       // wait) instead of staged, so the slot is 1/7 smaller (at 12 rows a 4th slot fits)
#endif
#ifndef ISO_PF           // L2 prefetch distance of the producer in planes (0: none)
#define ISO_PF 0
#endif
#ifndef ISO_D3_ROWS      // rows of the 3-component RKL2 deviation stage (> 7: one CTA per SM)
#define ISO_D3_ROWS 7
#endif
__host__ __device__ constexpr int iso_rows(int epi, int nc) {
  return (epi == EPI_PCG_M && nc == 3) ? ISO_M3_ROWS : ((epi == EPI_RKL2_DSTAGE && nc == 3) ? ISO_D3_ROWS : 7);
}
__host__ __device__ constexpr int iso_minb(int epi, int nc) {
  return (epi == EPI_PCG_M && nc == 3) ? 1 : ((epi == EPI_RKL2_DSTAGE && nc == 3 && ISO_D3_ROWS > 7) ? 1 : 2);
}

template <int EPI, int NC>
struct IsoLay : IsoTile<iso_rows(EPI, NC)> {
  using T = IsoTile<iso_rows(EPI, NC)>;
  static constexpr int MINB = iso_minb(EPI, NC);   // CTAs per SM (launch bounds)
  // merged PCG, one CTA per SM: "former" warps turn each landed slot's zold, wold,
  // pold into z_k = zold - alpha wold (field 0) and p_k = z_k + beta pold (field 1)
  // once per staged position, instead of every consumer re-forming its 5-point
  // neighbourhood; consumers wait on a per-slot "formed" mbarrier (one arrival per
  // former warp)
  static constexpr bool FORM = (EPI == EPI_PCG_M) && MINB == 1;
#ifndef ISO_FORMERS
#define ISO_FORMERS 2
#endif
  static constexpr int NFORM = FORM ? ISO_FORMERS : 0;   // former warps
  static constexpr int THREADS = T::INT + 32 + 32 * NFORM;
  // staged fields: u | PCG S-pass r, pold | merged PCG zold, wold, pold
  static constexpr int nsrcf = (EPI == EPI_PCG_S) ? 2 : (EPI == EPI_PCG_M ? 3 : 1);
  // own-box operands: RKL2 ym2, y0, M0 | S-pass x | merged x (d is recomputed from
  // the staged face coefficients: A_ii = wV - dt L_ii, d = 1 / A_ii as in the R0 pass)
  static constexpr int nepi =
      (EPI == EPI_RKL2_STAGE) ? 3 * NC
                              : (EPI == EPI_RKL2_DSTAGE ? 2 * NC
                                                        : (EPI == EPI_PCG_S ? NC : (EPI == EPI_PCG_M ? (ISO_M_XG && NC == 3 ? 0 : NC) : 0)));
  // one block per staged field: NC main boxes, then the NC x 2 wrap boxes, so a
  // field's cell at any (main or wrap) offset o has its other-field twin at o + FS
  static constexpr int WRP = NC * T::S_MAIN;                          // wrap boxes within a field block
  static constexpr int FS = NC * T::S_MAIN + NC * 2 * T::S_W;         // field block stride
  // PCG S-pass: the Jacobi inverse diagonal d (one component, main + 2 wrap boxes), so
  // z = r d is formed on the fly and the U-pass never stores z
  static constexpr int nd = (EPI == EPI_PCG_S) ? 1 : 0;
  static constexpr int DB = nsrcf * FS;
  static constexpr int K2 = DB + nd * (T::S_MAIN + 2 * T::S_W);
  static constexpr int K3 = K2 + T::K2SZ;
  static constexpr int K3R = K3 + T::K3SZ;
  static constexpr int K1 = K3R + T::K3WR;
  static constexpr int WB = K1 + T::OWN;
  static constexpr int EP = WB + T::OWN;
  static constexpr int MT = EP + nepi * T::OWN;      // per-plane metrics written by the producer
  static constexpr int SLOT = MT + 16;
  static constexpr int FIX = 128;
  // ring slots: as many as MINB CTAs per SM fit (2 CTAs: <= 113 KB each), 2..4 (1 CTA: up to 6)
  static constexpr int NS1 = (SMEM_1CTA - 2048 - FIX) / (SLOT * 8 + 16);   // one CTA per SM: all that fit
  static constexpr int NS2 = (113 * 1024 - FIX) / (SLOT * 8 + 16);   // two CTAs per SM
  static constexpr int NS = (MINB == 2) ? (NS2 > 4 ? 4 : (NS2 < 2 ? 2 : NS2)) : (NS1 > 6 ? 6 : NS1);
  static constexpr size_t SMEM =
      (size_t)NS * SLOT * sizeof(double) + (2 + NC) * NS * sizeof(uint64_t) + 128;
  static_assert(SMEM <= (MINB == 2 ? 113 * 1024 : SMEM_1CTA), "iso TMA slot ring does not fit");
};

}  // namespace

struct IsoTmaArgs {
  CUtensorMap src[3];     // staged sources (u | r, pold | p_{k-2}, w_{k-1}, p_{k-1}), 3D (n3, n2, NC nl), box 36 x (IJ+2)
  CUtensorMap srcw[3];    // their wrap columns, box 2 x (IJ+2)
  CUtensorMap k2, k3, k3w, k1, w;   // boxes 32x8, 34x7, 2x7, 32x7, 32x7
  CUtensorMap epi[3];     // epilogue operands, 3D (n3, n2, NC nl), box 32 x IJ (merged PCG: x)
  CUtensorMap dm, dmw;    // PCG S-pass: d, box 36 x 9 / its wrap columns 2 x 9
  int has_w;
};

// FST: first PCG iteration (p = z, no pold, no x update) -- a template flag so the
// steady-state S-pass carries no per-cell branches on it
// FR: this launch finishes the pass's dot-product reduction in its last CTA (a
// separate instantiation, so the large-grid variant carries none of that code)
template <int EPI, int NC, bool FST, bool FR>
__global__ void __launch_bounds__(IsoLay<EPI, NC>::THREADS, IsoLay<EPI, NC>::MINB)
    iso_tma_kernel(StencilCall c, int ic, const __grid_constant__ IsoTmaArgs ta) {
  using Lay = IsoLay<EPI, NC>;
  constexpr int IJ = Lay::IJ, INT = Lay::INT, SBH = Lay::SBH, S_MAIN = Lay::S_MAIN, S_W = Lay::S_W;
  constexpr int K2H = Lay::K2H, K3H = Lay::K3H, OWN = Lay::OWN;
  constexpr int NS = Lay::NS;
  constexpr bool kS = (EPI == EPI_PCG_S);
  constexpr bool kM = (EPI == EPI_PCG_M);
  constexpr bool kP = (kS || kM) && !FST;   // source = z + beta pold (merged: z = zold - ax wold)
  extern __shared__ __align__(128) double smi[];
  double* ring = smi;
  uint64_t* full = reinterpret_cast<uint64_t*>(smi + NS * Lay::SLOT);
  uint64_t* empty = full + NS;
  uint64_t* formed = empty + NS;     // [NS][NC] (merged PCG with former warps; ISO_FORM_SPLIT: one per component)
  const Geo& G = c.geo;
  const Metrics& M = G.m;
  const int tid = threadIdx.x;
  const Tile3 tl = raster_tile(blockIdx.x, (c.geo.n3 + IK - 1) / IK, (c.geo.n2 + IJ - 1) / IJ, ISO_RASTER_H);
  const int j0 = tl.y * IJ, k0 = tl.x * IK;
  const int ib = c.ib + tl.z * ic;
  const int ie = min(ib + ic, c.ie);
  const long long blk = blockIdx.x;
  const bool per = G.periodic3 != 0;
  const bool wrapL = per && k0 == 0;
  const bool wrapR = per && (k0 + IK >= G.n3);

  bool skip[NC];
  bool all = true;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    skip[q] = (kS || kM) && c.ea.sc && c.ea.sc[q].done;
    all = all && skip[q];
  }
  if ((kS || kM) && all) return;

  // PCG scalars of this iteration, broadcast from shared memory (keeps them out of registers)
  // (merged PCG: each component's x mode of this pass and catch-up coefficients, pcg.cuh)
  __shared__ double sbeta[NC], sax[NC], scxp[NC], scxz[NC], sbp[NC];
  __shared__ int sxm[NC];
  if (tid < NC) {
    sbeta[tid] = kP ? c.ea.sc[tid].beta : 0.0;
    sax[tid] = kP ? c.ea.sc[tid].ax : 0.0;
    sbp[tid] = (kM && kP) ? c.ea.sc[tid].bprev : 0.0;
    scxp[tid] = (kM && kP) ? c.ea.sc[tid].cxp : 0.0;
    scxz[tid] = (kM && kP) ? c.ea.sc[tid].cxz : 0.0;
    sxm[tid] = (kM && kP) ? c.ea.sc[tid].xm : X_NORMAL;
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, IJ);
      for (int q = 0; q < NC; ++q) mbar_init(formed + s * NC + q, Lay::NFORM > 0 ? Lay::NFORM : 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // ======================= producer warp =======================
  constexpr bool kF = Lay::FORM && kP;   // consumers read formed z_k / p_k
  // ======================= former warps (merged PCG) =======================
  if (Lay::FORM && tid >= INT + 32) {
    const int lane = tid & 31;
    const int fl = tid - (INT + 32), fn = 32 * Lay::NFORM;   // this thread among the former warps
    constexpr int NF = 32 * (Lay::NFORM > 0 ? Lay::NFORM : 1);
    // ISO_FORM_TRIM: only the staged positions the 7-point stencil reads are formed -- the
    // own rows 1..IJ at box columns 1..IK+2 (own cells and both phi neighbours) and the two
    // theta-halo rows at the own columns 2..IK+1 -- not the box corners or the alignment
    // columns 0 and IK+3 (2 IK + IJ (IK + 2) = 506 of 540 positions at 13 rows: 8 instead
    // of 9 forms per former thread and component); this thread's offsets, fixed per launch
    // ISO_FORM_TRIM 2: the same set in 16-byte aligned pairs (double2 shared loads / store):
    // the halo rows' own columns as IK/2 pairs, the own rows as SBW/2 pairs (their alignment
    // columns 0 and IK+3 come along), 2 (IK/2) + IJ (SBW/2) = 266 pairs at 13 rows: 5 forms
    // of two positions per former thread and component
    constexpr int PW = (ISO_FORM_TRIM == 2) ? 2 : 1;               // positions per form
    constexpr int HW = IK / PW, OW = (ISO_FORM_TRIM == 2) ? SBW / 2 : IK + 2;
    constexpr int NEED = 2 * HW + IJ * OW;
    constexpr int NT = (NEED + NF - 1) / NF;
    int toff[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const int t = fl + i * NF;
      int o = -1;
      if (t < HW) {
        o = 2 + PW * t;                                              // theta-halo row 0
      } else if (t < HW + IJ * OW) {
        const int u = t - HW;
        o = (1 + u / OW) * SBW + (PW == 2 ? 0 : 1) + PW * (u % OW);  // own rows
      } else if (t < NEED) {
        o = (IJ + 1) * SBW + 2 + PW * (t - HW - IJ * OW);            // theta-halo row IJ+1
      }
      toff[i] = o;
    }
    for (int p = ib; p < ie; ++p) {
      const int slot = (p - ib) % NS;
      mbar_wait(full + slot, (uint32_t)(((p - ib) / NS) & 1));
      double* S = ring + slot * Lay::SLOT;
      // fields p_{k-2}, w_{k-1}, p_{k-1}: z_k = (p_{k-1} - beta_{k-1} p_{k-2}) - alpha_{k-1} w_{k-1},
      // p_k = z_k + beta_k p_{k-1} over w_{k-1}; p_{k-2} stays (the x catch-up reads it), the
      // own cell's z_k = p_k - beta_k p_{k-1} is re-formed by its consumer
      auto form = [&](int o, int q) {
        const double z = fma(-sax[q], S[o + Lay::FS], fma(-sbp[q], S[o], S[o + 2 * Lay::FS]));
        S[o + Lay::FS] = fma(sbeta[q], S[o + 2 * Lay::FS], z);
      };
      // (ISO_FORM_UNROLL: compile-time trip counts, fully unrolled)
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        if constexpr (kF) {
          if constexpr (ISO_FORM_TRIM == 2) {
            // (S_MAIN, FS and the row pitch SBW are even: an even offset is 16-byte aligned)
#pragma unroll
            for (int i = 0; i < NT; ++i)
              if (toff[i] >= 0) {
                const int o = q * S_MAIN + toff[i];
                const double2 pm2 = *reinterpret_cast<const double2*>(S + o);
                const double2 wm1 = *reinterpret_cast<const double2*>(S + o + Lay::FS);
                const double2 pm1 = *reinterpret_cast<const double2*>(S + o + 2 * Lay::FS);
                const double z0 = fma(-sax[q], wm1.x, fma(-sbp[q], pm2.x, pm1.x));
                const double z1 = fma(-sax[q], wm1.y, fma(-sbp[q], pm2.y, pm1.y));
                *reinterpret_cast<double2*>(S + o + Lay::FS) =
                    make_double2(fma(sbeta[q], pm1.x, z0), fma(sbeta[q], pm1.y, z1));
              }
          } else if constexpr (ISO_FORM_TRIM) {
#pragma unroll
            for (int i = 0; i < NT; ++i)
              if (toff[i] >= 0) form(q * S_MAIN + toff[i], q);
          } else if constexpr (ISO_FORM_UNROLL) {
            constexpr int NI = (SBW * SBH + NF - 1) / NF;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              const int o = fl + i * NF;
              if (o < SBW * SBH) form(q * S_MAIN + o, q);
            }
          } else {
            for (int o = fl; o < SBW * SBH; o += fn) form(q * S_MAIN + o, q);
          }
          if (wrapL || wrapR)
            for (int o = fl; o < 2 * S_W; o += fn) form(Lay::WRP + q * 2 * S_W + o, q);
        }
        // release the formed component to the consumers (ISO_FORM_SPLIT: component by
        // component, so the consumers start on component 0 while 1 and 2 are formed)
        if (ISO_FORM_SPLIT || q == NC - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(formed + slot * NC + (ISO_FORM_SPLIT ? q : 0));
        }
      }
    }
    return;
  }
  if (tid >= INT) {   // (the whole warp runs the loop; the elected lane issues)
    constexpr int nsrcf_now = ((kS || kM) && FST) ? 1 : Lay::nsrcf;
    const int cpl = (int)(G.cstride / G.plane);   // planes per component of the (whole local) array
    uint32_t bytes = nsrcf_now * NC * SBW * SBH * 8 + (K2W * K2H + K3W * K3H + OWN) * 8;
    if (wrapL) bytes += nsrcf_now * NC * 2 * SBH * 8 + 2 * K3H * 8;
    if (wrapR) bytes += nsrcf_now * NC * 2 * SBH * 8;
    if (ta.has_w) bytes += OWN * 8;
    // merged PCG: the x box of a component whose x the pass does not touch (first pass,
    // skipped x update) is not loaded
    bool no_x[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) no_x[q] = kM && (!kP || sxm[q] == X_SKIP);
    bytes += Lay::nepi * OWN * 8;
    if constexpr (kM && Lay::nepi > 0)
#pragma unroll
      for (int q = 0; q < NC; ++q)
        if (no_x[q]) bytes -= OWN * 8;
    if (Lay::nd) {
      bytes += SBW * SBH * 8;
      if (wrapL) bytes += 2 * SBH * 8;
      if (wrapR) bytes += 2 * SBH * 8;
    }
    // per-plane metrics, loaded one plane ahead (a load at the top of the iteration put
    // its latency between a slot's release and its TMA issue); F2r == F3r
    double mf1 = 0.0, mf2 = 0.0, mvr = 0.0;
    if (ib < ie) {
      mf1 = M.F1r[G.i0 + ib];
      mf2 = M.F2r[G.i0 + ib];
      mvr = M.Vr[G.i0 + ib];
    }
    for (int p = ib; p < ie; ++p) {
      const int slot = (p - ib) % NS, n = (p - ib) / NS;
      if (n > 0) mbar_wait(empty + slot, (uint32_t)((n - 1) & 1));
      double* S = ring + slot * Lay::SLOT;
      uint64_t* bar = full + slot;
      const double f1 = mf1, f2 = mf2, vr = mvr;
      if (p + 1 < ie) {
        mf1 = M.F1r[G.i0 + p + 1];
        mf2 = M.F2r[G.i0 + p + 1];
        mvr = M.Vr[G.i0 + p + 1];
      }
      if (elect_one()) {
        // (plain stores, released by the arrive below)
        S[Lay::MT + 0] = f1;
        S[Lay::MT + 1] = f2;
        S[Lay::MT + 2] = vr;
        fence_proxy_async();
        mbar_expect_tx(bar, bytes);
#pragma unroll
        for (int f = 0; f < nsrcf_now; ++f)
#pragma unroll
          for (int q = 0; q < NC; ++q) {
            const int pl = q * cpl + p;
            double* F = S + f * Lay::FS;
            tma3(F + q * S_MAIN, &ta.src[f], k0 - 2, j0 - 1, pl, bar);
            if (wrapL) tma3(F + Lay::WRP + (q * 2 + 0) * S_W, &ta.srcw[f], G.n3 - 2, j0 - 1, pl, bar);
            if (wrapR) tma3(F + Lay::WRP + (q * 2 + 1) * S_W, &ta.srcw[f], 0, j0 - 1, pl, bar);
          }
        if (Lay::nd) {
          tma3(S + Lay::DB, &ta.dm, k0 - 2, j0 - 1, p, bar);
          if (wrapL) tma3(S + Lay::DB + S_MAIN, &ta.dmw, G.n3 - 2, j0 - 1, p, bar);
          if (wrapR) tma3(S + Lay::DB + S_MAIN + S_W, &ta.dmw, 0, j0 - 1, p, bar);
        }
        tma3(S + Lay::K2, &ta.k2, k0, j0 - 1, p, bar);
        tma3(S + Lay::K3, &ta.k3, k0 - 2, j0, p, bar);
        if (wrapL) tma3(S + Lay::K3R, &ta.k3w, G.n3 - 2, j0, p, bar);
        tma3(S + Lay::K1, &ta.k1, k0, j0, p, bar);
        if (ta.has_w) tma3(S + Lay::WB, &ta.w, k0, j0, p, bar);
#pragma unroll
        for (int q = 0; q < Lay::nepi; ++q)
          if (!(kM && no_x[q % NC])) tma3(S + Lay::EP + q * OWN, &ta.epi[q / NC], k0, j0, (q % NC) * cpl + p, bar);
        if constexpr (ISO_PF > 0) {
          // L2 prefetch of the package of plane p + PF (main boxes; wrap boxes left to the loads)
          const int pf = p + ISO_PF;
          if (pf < ie) {
#pragma unroll
            for (int f = 0; f < nsrcf_now; ++f)
#pragma unroll
              for (int q = 0; q < NC; ++q) tma3_prefetch(&ta.src[f], k0 - 2, j0 - 1, q * cpl + pf);
            if (Lay::nd) tma3_prefetch(&ta.dm, k0 - 2, j0 - 1, pf);
            tma3_prefetch(&ta.k2, k0, j0 - 1, pf);
            tma3_prefetch(&ta.k3, k0 - 2, j0, pf);
            tma3_prefetch(&ta.k1, k0, j0, pf);
            if (ta.has_w) tma3_prefetch(&ta.w, k0, j0, pf);
#pragma unroll
            for (int q = 0; q < Lay::nepi; ++q)
              if (!(kM && no_x[q % NC])) tma3_prefetch(&ta.epi[q / NC], k0, j0, (q % NC) * cpl + pf);
          }
        }
      }
      __syncwarp();
    }
    return;
  }

  // ======================= consumer warps =======================
  const int tj = tid >> 5, tk = tid & 31;
  const int j = j0 + tj, k = k0 + tk;
  const bool own = (j < G.n2) && (k < G.n3);
  const long long coff = own ? (long long)j * G.n3 + k : 0;
  const bool jm = j >= 1, jp = j + 1 < G.n2;
  const bool kself = per && G.n3 == 1;
  const bool km = !kself && (per || k >= 1), kp = !kself && (per || k + 1 < G.n3);
  const int kmw = per ? (k >= 1 ? k - 1 : G.n3 - 1) : k - 1;
  double cv[6] = {0, 0, 0, 0, 0, 0};   // f1tp, f2p, f2m, f3p, f3m, vtp
  if (own) {
    cv[0] = M.F1t[j] * M.F1p[k];
    cv[1] = jp ? M.F2t[j] * M.F2p[k] : 0.0;
    cv[2] = jm ? M.F2t[j - 1] * M.F2p[k] : 0.0;
    cv[3] = kp ? M.F3t[j] * M.F3p[k] : 0.0;
    cv[4] = km ? M.F3t[j] * M.F3p[kmw] : 0.0;
    cv[5] = M.Vt[j] * M.Vp[k];
  }
  auto CV = [&](int t) -> double { return cv[t]; };   // per-column metric products
  // smem offsets (relative to the slot) of the own cell, its in-plane neighbours per
  // component (periodic phi wrap: cell n3-1 / 0 from the 2-column wrap boxes)
  const int oc = (tj + 1) * SBW + tk + 2;
  const bool kmw_box = per && k == 0, kpw_box = per && k + 1 == G.n3;
  // component q of the k-1 / k+1 neighbour: base + q * stride (main box or wrap box)
  const int okm0 = kmw_box ? Lay::WRP + 0 * S_W + (tj + 1) * 2 + 1 : oc - 1;
  const int okp0 = kpw_box ? Lay::WRP + 1 * S_W + (tj + 1) * 2 : oc + 1;
  const int okms = kmw_box ? 2 * S_W : S_MAIN, okps = kpw_box ? 2 * S_W : S_MAIN;
  const int o8 = tj * IK + tk;
  const int ok2p = Lay::K2 + (tj + 1) * K2W + tk, ok2m = ok2p - K2W;
  const int ok3p = Lay::K3 + tj * K3W + tk + 2;
  const int ok3m = kmw_box ? Lay::K3R + tj * 2 + 1 : ok3p - 1;
  // d offsets of the same five positions (one component)
  const int dc = Lay::DB + oc;
  const int dkm = kmw_box ? Lay::DB + S_MAIN + 0 * S_W + (tj + 1) * 2 + 1 : dc - 1;
  const int dkp = kpw_box ? Lay::DB + S_MAIN + 1 * S_W + (tj + 1) * 2 : dc + 1;
  // merged PCG: z_k at a staged position (field 0 zold, field 1 wold)
  // (fields p_{k-2}, w_{k-1}, p_{k-1}: z_k = (p_{k-1} - beta_{k-1} p_{k-2}) - alpha_{k-1} w_{k-1})
  auto zm = [&](const double* S, int o, int q) {
    if constexpr (kP && !kF) return fma(-sax[q], S[o + Lay::FS], fma(-sbp[q], S[o], S[o + 2 * Lay::FS]));
    return S[o];
  };
  // source value at (field-0 offset o, d offset od): PCG S-pass p = r d + beta pold
  // (first: r d); merged p = zm + beta pold (first: z0); else u
  auto sv = [&](const double* S, int o, int od, int q) {
    if constexpr (kS) {
      const double z = S[o] * S[od];
      if constexpr (kP) return fma(sbeta[q], S[o + Lay::FS], z);
      return z;
    } else if constexpr (kM) {
      if constexpr (kF) return S[o + Lay::FS];
      if constexpr (kP) return fma(sbeta[q], S[o + 2 * Lay::FS], zm(S, o, q));
      return S[o];
    }
    return S[o];
  };
  // own column through global memory (r neighbours, incl. the neighbour slab's halo plane)
  const long long cs = G.cstride, pl = G.plane;
  auto colv = [&](const FieldV& f, int il, int q) -> double {
    if (!own) return 0.0;
    const double* pz;
    if (il >= 0 && il < G.nl) pz = f.p + q * cs + il * pl;
    else if (il == G.nl && f.hi) pz = f.hi + q * pl;
    else if (il == -1 && f.lo) pz = f.lo + q * pl;
    else return 0.0;
    return __ldg(pz + coff);
  };
  // the source value from own-column loads: (z, pold, d) | merged (zold, wold, pold)
  auto comb = [&](double z, double po, double dd, int q) {
    if constexpr (kS) {
      if constexpr (kP) return fma(sbeta[q], po, z * dd);
      return z * dd;
    } else if constexpr (kM) {
      // (z: p_{k-2}, po: p_{k-1}, dd: w_{k-1}) -> p_k = z_k + beta_k p_{k-1}
      if constexpr (kP) return fma(sbeta[q], po, fma(-sax[q], dd, fma(-sbp[q], z, po)));
      return z;
    }
    return z;
  };

  // Register double buffering, unrolled by two (no register moves of in-flight loads,
  // which would make every prefetch wait at the end of its own iteration):
  //   Pre.z/p: own column of plane il+1 (r up-neighbour), loaded one step earlier
  //   (not used by the merged PCG march, which takes it from the next slot);
  struct Pre {
    double z[NC], p[NC], d;
  };
  const int ig0 = G.i0 + ib;
  Pre A, B;
  double udn[NC];
  // merged: own-column fields are u = zold, u2 = wold, u3 = pold
  const FieldV& fP = kM ? c.u3 : c.u2;
  const double ddn = kS ? colv(c.u3, ib - 1, 0) : 1.0;
  A.d = kS ? colv(c.u3, ib + 1, 0) : 1.0;
  B.d = 1.0;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    if constexpr (kM) {
      // (the merged march takes the up neighbour from the next plane's slot, below)
      udn[q] = comb(colv(c.u, ib - 1, q), kP ? colv(fP, ib - 1, q) : 0.0, kP ? colv(c.u2, ib - 1, q) : 0.0, q);
    } else {
      udn[q] = comb(colv(c.u, ib - 1, q), kP ? colv(fP, ib - 1, q) : 0.0, ddn, q);
      A.z[q] = colv(c.u, ib + 1, q);
      A.p[q] = kP ? colv(fP, ib + 1, q) : 0.0;
    }
  }
  double kdn = 0.0;
  if (own && ig0 >= 1) {
    // merged PCG: the local planes of k1 hold the metric-folded K1 (the halo plane is raw)
    if (kM && ib >= 1) kdn = __ldg(c.k1.p + (long long)(ib - 1) * G.plane + coff);
    else kdn = __ldg(plane_ptr(c.k1, G, ib - 1, 0) + coff) * M.F1r[ig0 - 1] * cv[0];
  }
  constexpr int NQ = kM ? 4 : (EPI == EPI_PCG_R0 ? 2 : 1);   // partial sums per component
  double part[NC][NQ];
#pragma unroll
  for (int q = 0; q < NC; ++q)
#pragma unroll
    for (int t = 0; t < NQ; ++t) part[q][t] = 0.0;
  constexpr bool kR0 = (EPI == EPI_PCG_R0);
  // outputs are addressed from the kernel parameters (constant bank) + the cell index,
  // which keeps the pointers out of registers
  double* const o1 = c.ea.out;
  double* const o2 = c.ea.out2;
  double* const o3 = c.ea.out3;
  double* const o4 = c.ea.out4;
  double* const ox = c.ea.x;

  auto body = [&](int il, const Pre& C, Pre& N) {
    const int slot = (il - ib) % NS;
    const double* S = ring + slot * Lay::SLOT;
    const int ig = G.i0 + il;
    const bool ip = ig + 1 < G.n1g;
    // prefetch into the other buffer: own column two planes ahead, metrics one ahead
    const bool more = il + 2 <= ie;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      N.z[q] = more ? colv(c.u, il + 2, q) : 0.0;
      N.p[q] = (kP && more) ? colv(fP, il + 2, q) : 0.0;
    }
    if constexpr (kS) N.d = more ? colv(c.u3, il + 2, 0) : 1.0;
    mbar_wait(full + slot, (uint32_t)(((il - ib) / NS) & 1));
    double Kup = 0.0;
    if (own) {
      const double f1r = S[Lay::MT + 0], f23r = S[Lay::MT + 1], vr = S[Lay::MT + 2];
      Kup = ip ? S[Lay::K1 + o8] * f1r * CV(0) : 0.0;
      const double Kjp = jp ? S[ok2p] * f23r * CV(1) : 0.0;
      const double Kjm = jm ? S[ok2m] * f23r * CV(2) : 0.0;
      const double Kkp = kp ? S[ok3p] * f23r * CV(3) : 0.0;
      const double Kkm = km ? S[ok3m] * f23r * CV(4) : 0.0;
      const double WV = (ta.has_w ? S[Lay::WB + o8] : 1.0) * vr * CV(5);
      const long long gi = (long long)il * pl + coff;
      double dinv = 0.0;
      if constexpr (kR0) {
        // PC1: d = 1/A_ii, A = wV - dt L, L_ii = -(sum of the face coefficients)
        const double Ldiag = -(kdn + Kup + Kjp + Kjm + Kkp + Kkm);
        dinv = rcp_pos(WV - c.ea.dt * Ldiag);   // (the merged pass recomputes it the same way)
        o4[gi] = dinv;
      }
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const int oq = q * S_MAIN + oc;
        const double u0 = sv(S, oq, dc, q);
        const double ujm = sv(S, oq - SBW, dc - SBW, q), ujp = sv(S, oq + SBW, dc + SBW, q);
        const double ukm = sv(S, okm0 + q * okms, dkm, q), ukp = sv(S, okp0 + q * okps, dkp, q);
        const double uup = comb(C.z[q], C.p[q], C.d, q);
        const double Lu = kdn * (udn[q] - u0) + Kup * (uup - u0) + Kjm * (ujm - u0) + Kjp * (ujp - u0) +
                          Kkm * (ukm - u0) + Kkp * (ukp - u0);
        const long long go = gi + q * cs;
        if (!skip[q]) {
          if constexpr (EPI == EPI_F) {
            o1[go] = Lu / WV;
          } else if constexpr (EPI == EPI_RKL2_FIRST) {
            const double F = Lu / WV;
            o2[go] = F;
            o1[go] = c.ea.a0 * u0 + c.ea.c0 * F;
          } else if constexpr (EPI == EPI_RKL2_STAGE) {
            const double F = Lu / WV;
            o1[go] = c.ea.mu * u0 + c.ea.nu * S[Lay::EP + q * OWN + o8] + c.ea.c2 * S[Lay::EP + (NC + q) * OWN + o8] +
                     c.ea.c0 * F + c.ea.c1 * S[Lay::EP + (2 * NC + q) * OWN + o8];
          } else if constexpr (EPI == EPI_RKL2_DSTAGE) {
            const double F = Lu / WV;
            o1[go] = c.ea.mu * u0 + c.ea.nu * S[Lay::EP + q * OWN + o8] + c.ea.c0 * F +
                     c.ea.c1 * S[Lay::EP + (NC + q) * OWN + o8];
          } else if constexpr (kR0) {
            // r0 = b - A x0 = dt L u (x0 = u^n); z0 = r0 d; partials r.z and b.P^-1 b
            const double r = c.ea.dt * Lu;
            const double z = r * dinv;
            const double bb = WV * u0;
            o1[go] = r;
            if (o2) o2[go] = u0;
            if (o3) o3[go] = z;
            part[q][0] += r * z;
            part[q][1] += bb * bb * dinv;
          } else if constexpr (kS) {
            const double y = WV * u0 - c.ea.dt * Lu;
            o1[go] = y;
            o2[go] = u0;                                          // p_k
            if constexpr (kP) ox[go] = fma(sax[q], S[oq + Lay::FS], S[Lay::EP + q * OWN + o8]);
            part[q][0] += u0 * y;
          }
        }
        udn[q] = u0;
      }
    }
    __syncwarp();
    if (tk == 0) mbar_arrive(empty + slot);       // this warp is done with the slot
    kdn = Kup;
  };
  if constexpr (kM) {
    // Merged PCG march with a delayed up neighbour (no own-column loads in the loop):
    // when plane il's slot lands, its p, z, x (and r.z) are final and stored, and its
    // L p is complete except the r-up term; that term needs p at (il+1, own cell),
    // which is the own cell of the NEXT slot, so y, w and the y-partials of plane il
    // are finished one plane later.  The last plane's up neighbour comes from global
    // memory (the neighbour slab's halo plane at a slab boundary).
    // per-plane state carried to the next plane; two sets, unrolled by two (no moves)
    struct St {
      double L[NC], u[NC], z[NC];   // off-diagonal face sum without the r-up term, p, z of the own cell
      double A, dc, K;               // A_ii, d of the own cell, r-up face coefficient
    };
    St SA, SB;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      SA.u[q] = udn[q];              // plane ib-1 (the down neighbour of plane ib)
      SA.L[q] = SA.z[q] = 0.0;
    }
    SA.A = SA.dc = 0.0;
    SA.K = kdn;
    auto finish = [&](int il, const St& P, const double* uup) {   // y-dependent outputs of plane il
      const long long gi = (long long)il * pl + coff;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        if (skip[q]) continue;
        // y = A p = A_ii p - dt sum_f K_f p_f (the matrix row as assembled: diagonal + the
        // six off-diagonal face couplings)
        const double y = P.A * P.u[q] - c.ea.dt * fma(P.K, uup[q], P.L[q]);
        const double wk = P.dc * y;
        __stcs(o3 + gi + q * cs, wk);   // (streaming stores: see the aniso merged pass)
        part[q][1] += P.u[q] * y;
        part[q][2] += P.z[q] * y;
        part[q][3] += wk * y;
      }
    };
    auto mbody = [&](int il, const St& P, St& C) {
      const int slot = (il - ib) % NS;
      const double* S = ring + slot * Lay::SLOT;
      const uint32_t par = (uint32_t)(((il - ib) / NS) & 1);
      constexpr bool kFW = Lay::FORM && Lay::NFORM > 0;   // consumers wait for the former warps
      // (ISO_M_XG: this plane's x of the own cell loaded before the wait, which hides its latency)
      constexpr bool kXG = kP && Lay::nepi == 0;
      double xg[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        xg[q] = 0.0;
        if constexpr (kXG)
          if (own && !skip[q] && sxm[q] != X_SKIP) xg[q] = __ldcs(ox + (long long)il * pl + coff + q * cs);
      }
      mbar_wait(kFW ? formed + slot * NC : full + slot, par);
      if constexpr (kF && Lay::NFORM == 0) {
        // consumer forming (ISO_FORMERS = 0): the consumer warps form the landed slot's
        // p_k at every staged position themselves (the former warps' arithmetic, spread
        // over all consumer threads), then meet at one consumer-only named barrier
        double* SF = ring + slot * Lay::SLOT;
        auto form = [&](int o, int q) {
          const double z = fma(-sax[q], SF[o + Lay::FS], fma(-sbp[q], SF[o], SF[o + 2 * Lay::FS]));
          SF[o + Lay::FS] = fma(sbeta[q], SF[o + 2 * Lay::FS], z);
        };
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          for (int o = tid; o < SBW * SBH; o += INT) form(q * S_MAIN + o, q);
          if (wrapL || wrapR)
            for (int o = tid; o < 2 * S_W; o += INT) form(Lay::WRP + q * 2 * S_W + o, q);
        }
        asm volatile("bar.sync 1, %0;\n" ::"r"(INT) : "memory");
      }
      C.K = 0.0;
      if (own) {
        // metric-folded coefficients (launch_iso_premul: zero on wall faces)
        C.K = S[Lay::K1 + o8];
        const double Kjp = S[ok2p];
        const double Kjm = jm ? S[ok2m] : 0.0;
        const double Kkp = S[ok3p];
        const double Kkm = km ? S[ok3m] : 0.0;
        const double WV = S[Lay::WB + o8];
        // PC1 diagonal of the own cell, the R0 pass's arithmetic (bit-identical d):
        // A_ii = wV - dt L_ii, L_ii = -(sum of the six face coefficients); r.z = z^2 A_ii
        const double Aii = WV - c.ea.dt * -(P.K + C.K + Kjp + Kjm + Kkp + Kkm);
        C.A = Aii;
        C.dc = rcp_pos(Aii);
        const double idcell = Aii;
        const long long gi = (long long)il * pl + coff;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          if (kFW && ISO_FORM_SPLIT && q > 0) mbar_wait(formed + slot * NC + q, par);
          const int oq = q * S_MAIN + oc;
          // (formed slot: field 1 holds p_k, field 0 the raw z_{k-1}: z_k = p_k - beta p_{k-1})
          const double zk = kF ? fma(-sbeta[q], S[oq + 2 * Lay::FS], S[oq + Lay::FS]) : zm(S, oq, q);
          const double u0 = kF ? S[oq + Lay::FS] : (kP ? fma(sbeta[q], S[oq + 2 * Lay::FS], zk) : zk);
          const double ujm = sv(S, oq - SBW, 0, q), ujp = sv(S, oq + SBW, 0, q);
          const double ukm = sv(S, okm0 + q * okms, 0, q), ukp = sv(S, okp0 + q * okps, 0, q);
          C.L[q] = P.K * P.u[q] + Kjm * ujm + Kjp * ujp + Kkm * ukm + Kkp * ukp;
          C.u[q] = u0;
          C.z[q] = zk;
          if (!skip[q]) {
            const long long go = gi + q * cs;
            __stcs(o2 + go, u0);
            if constexpr (kP) {
              // x in pairs (pcg.cuh): x_k = x_{k-1} + alpha_{k-1} p_{k-1}; skipped; or the
              // catch-up x_k = x_{k-2} + alpha_{k-1} p_{k-1} + alpha_{k-2} p_{k-2} (both staged)
              const int m = sxm[q];
              if (m != X_SKIP) {
                double xn = fma(m == X_CATCHUP ? scxp[q] : sax[q], S[oq + 2 * Lay::FS], kXG ? xg[q] : S[Lay::EP + q * OWN + o8]);
                if (m == X_CATCHUP) xn = fma(scxz[q], S[oq], xn);   // + alpha_{k-2} p_{k-2} (field 0)
                __stcs(ox + go, xn);
              }
            }
            part[q][0] += zk * zk * idcell;
          }
        }
        if (il > ib) finish(il - 1, P, C.u);   // plane il-1's up neighbour is this plane's own cell
      }
      __syncwarp();
      if (tk == 0) mbar_arrive(empty + slot);       // this warp is done with the slot
    };
    // the last plane: its up neighbour from global memory (the neighbour slab's halo plane)
    auto tail = [&](const St& P) {
      if (!own || ie <= ib) return;
      double uup[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q)
        uup[q] = comb(colv(c.u, ie, q), kP ? colv(fP, ie, q) : 0.0, kP ? colv(c.u2, ie, q) : 0.0, q);
      finish(ie - 1, P, uup);
    };
    int il = ib;
    for (; il + 1 < ie; il += 2) {
      mbody(il, SA, SB);
      mbody(il + 1, SB, SA);
    }
    if (il < ie) {
      mbody(il, SA, SB);
      tail(SB);
    } else {
      tail(SA);
    }
  } else {
    int il = ib;
    for (; il + 1 < ie; il += 2) {
      body(il, A, B);
      body(il + 1, B, A);
    }
    if (il < ie) body(il, A, B);
  }
  if constexpr (kR0 || kS || kM) {
    // partial rows q*NQ + t (R0: r.z, b.P^-1 b; S: p.y; merged: r.z, p.y, z.y, w.y)
    __shared__ double red[NC * NQ][IJ];
#pragma unroll
    for (int q = 0; q < NC; ++q)
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        double v = part[q][t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (tk == 0) red[q * NQ + t][tj] = v;
      }
    asm volatile("bar.sync 1, %0;\n" ::"r"(INT) : "memory");   // consumer warps only
    if (tid < NC * NQ) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < IJ; ++w) s += red[tid][w];
      c.ea.partials[tid * c.ea.pstride + c.ea.pbase + blk] = s;
    }
    if constexpr (FR && (kS || kM)) {
      __shared__ double fred[4 * MAXC * 32];
      __shared__ unsigned flag;
      fused_final_reduce(c.ea.fin, c.ea.partials, c.ea.pstride,
                         (unsigned long long)gridDim.x, tid, INT, fred, &flag,
                         [] { asm volatile("bar.sync 1, %0;\n" ::"r"(INT) : "memory"); });
    }
  }
}

// ============================================================================
// host side
// ============================================================================
static bool iso_has_tma(int epi) {
  return epi == EPI_F || epi == EPI_RKL2_FIRST || epi == EPI_RKL2_STAGE || epi == EPI_PCG_S || epi == EPI_PCG_R0 ||
         epi == EPI_PCG_M || epi == EPI_RKL2_DSTAGE;
}

bool iso_tma_eligible(const StencilCall& c) {
  if (c.mode != STS_MODE_ISO || c.ncomp < 1 || c.ncomp > 3 || !iso_has_tma(c.epi)) return false;
  const Geo& G = c.geo;
  if (G.n3 % 2 != 0) return false;
  if (!al16(c.u.p) || !al16(c.u2.p) || !al16(c.k1.p) || !al16(c.k2.p) || !al16(c.k3.p) || !al16(c.w)) return false;
  if (!al16(c.ea.ym2) || !al16(c.ea.y0) || !al16(c.ea.m0) || !al16(c.ea.x)) return false;
  if (c.epi == EPI_PCG_S && (!c.u3.p || !al16(c.u3.p))) return false;
  if (c.epi == EPI_PCG_M && (!al16(c.u3.p) || !c.ea.x || !c.ea.out3 || !c.premul || !c.w)) return false;
  if (c.epi == EPI_PCG_R0 && (!c.ea.out4 || c.ea.sc)) return false;
  return true;
}

static dim3 iso_grid(const Geo& G, int ib, int ie, int rows, int minb, int* ic_out) {
  const int nbx = (G.n3 + IK - 1) / IK, nby = (G.n2 + rows - 1) / rows;
  const long long per_sm = minb;   // resident CTAs per SM (IsoLay::MINB)
  const int np = ie - ib;
  if (np <= 0) {
    *ic_out = 1;
    return dim3(0, 0, 0);
  }
  const long long tiles = (long long)nbx * nby;
  // (long marches leave a ragged last wave: cap the chunk at ISO_CHUNK_MAX planes; a chunk
  // costs ISO_CHUNK_EXTRA planes of pipeline fill and r-boundary reads)
#ifndef ISO_CHUNK_EXTRA
#define ISO_CHUNK_EXTRA 0.5
#endif
#ifndef ISO_CHUNK_MAX
#define ISO_CHUNK_MAX 128
#endif
  const int ic = choose_chunk(tiles, np, 148LL * per_sm, ISO_CHUNK_EXTRA, 4, ISO_CHUNK_MAX);
  *ic_out = ic;
  return dim3(nbx, nby, (np + ic - 1) / ic);
}

int iso_tma_blocks(const StencilCall& c) {
  int ic;
  const dim3 g = iso_grid(c.geo, c.ib, c.ie, iso_rows(c.epi, c.ncomp), iso_minb(c.epi, c.ncomp), &ic);
  return (int)(g.x * g.y * g.z);
}

template <int EPI, int NC, bool FST, bool FR>
static void launch_iso_g(const StencilCall& c, dim3 grid, int ic, const IsoTmaArgs& ta, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  ensure_smem_attr(iso_tma_kernel<EPI, NC, FST, FR>, (int)IsoLay<EPI, NC>::SMEM, attr);
  const unsigned nb = grid.x * grid.y * grid.z;
  iso_tma_kernel<EPI, NC, FST, FR><<<dim3(nb), IsoLay<EPI, NC>::THREADS, IsoLay<EPI, NC>::SMEM, st>>>(c, ic, ta);
}

template <int EPI, int NC, bool FST>
static void launch_iso_f(const StencilCall& c, dim3 grid, int ic, const IsoTmaArgs& ta, cudaStream_t st) {
  constexpr bool kPcg = (EPI == EPI_PCG_S || EPI == EPI_PCG_M);
  if (kPcg && c.ea.fin.ticket) launch_iso_g<EPI, NC, FST, kPcg>(c, grid, ic, ta, st);
  else launch_iso_g<EPI, NC, FST, false>(c, grid, ic, ta, st);
}

template <int EPI, int NC>
static void launch_iso_t(const StencilCall& c, dim3 grid, int ic, const IsoTmaArgs& ta, cudaStream_t st) {
  if ((EPI == EPI_PCG_S || EPI == EPI_PCG_M) && c.ea.first) launch_iso_f<EPI, NC, true>(c, grid, ic, ta, st);
  else launch_iso_f<EPI, NC, false>(c, grid, ic, ta, st);
}

template <int EPI>
static void launch_iso_nc(const StencilCall& c, dim3 grid, int ic, const IsoTmaArgs& ta, cudaStream_t st) {
  switch (c.ncomp) {
    case 1: launch_iso_t<EPI, 1>(c, grid, ic, ta, st); break;
    case 2: launch_iso_t<EPI, 2>(c, grid, ic, ta, st); break;
    case 3: launch_iso_t<EPI, 3>(c, grid, ic, ta, st); break;
    default: throw Error{STS_ERR_ARG, "ncomp must be 1..3"};
  }
}

bool launch_iso_tma(const StencilCall& c, cudaStream_t st) {
  if (!iso_tma_eligible(c)) return false;
  const Geo& G = c.geo;
  int ic = 1;
  const int IJ = iso_rows(c.epi, c.ncomp), SBH = IJ + 2, K2H = IJ + 1, K3H = IJ;
  const dim3 grid = iso_grid(G, c.ib, c.ie, IJ, iso_minb(c.epi, c.ncomp), &ic);
  if (grid.x == 0) return true;
  const int NC = c.ncomp;
  // component q of a [ncomp][nl_local][plane] array starts cpl planes after q-1; a virtual
  // slab's base is offset into component 0, so the map spans (NC-1) cpl + nl planes from it
  const int cpl = (int)(G.cstride / G.plane);
  const int npl = (NC - 1) * cpl + G.nl;
  IsoTmaArgs ta;
  memset(&ta, 0, sizeof(ta));
  const double* srcs[3] = {c.u.p, c.u2.p ? c.u2.p : c.u.p, (c.epi == EPI_PCG_M && c.u3.p) ? c.u3.p : c.u.p};
  for (int f = 0; f < 3; ++f) {
    map_plain(&ta.src[f], srcs[f], G, npl, SBW, SBH);
    map_plain(&ta.srcw[f], srcs[f], G, npl, 2, SBH);
  }
  map_plain(&ta.k2, c.k2.p, G, G.nl, K2W, K2H);
  map_plain(&ta.k3, c.k3.p, G, G.nl, K3W, K3H);
  map_plain(&ta.k3w, c.k3.p, G, G.nl, 2, K3H);
  map_plain(&ta.k1, c.k1.p, G, G.nl, IK, IJ);
  map_plain(&ta.w, c.w ? c.w : c.k1.p, G, G.nl, IK, IJ);
  ta.has_w = c.w != nullptr;
  if (c.epi == EPI_RKL2_STAGE) {
    map_plain(&ta.epi[0], c.ea.ym2, G, npl, IK, IJ);
    map_plain(&ta.epi[1], c.ea.y0, G, npl, IK, IJ);
    map_plain(&ta.epi[2], c.ea.m0, G, npl, IK, IJ);
  } else if (c.epi == EPI_RKL2_DSTAGE) {
    map_plain(&ta.epi[0], c.ea.ym2, G, npl, IK, IJ);
    map_plain(&ta.epi[1], c.ea.m0, G, npl, IK, IJ);
  } else if (c.epi == EPI_PCG_S) {
    map_plain(&ta.epi[0], c.ea.x, G, npl, IK, IJ);
    map_plain(&ta.dm, c.u3.p, G, G.nl, SBW, SBH);
    map_plain(&ta.dmw, c.u3.p, G, G.nl, 2, SBH);
  } else if (c.epi == EPI_PCG_M) {
    map_plain(&ta.epi[0], c.ea.x, G, npl, IK, IJ);
  }
  switch (c.epi) {
    case EPI_F: launch_iso_nc<EPI_F>(c, grid, ic, ta, st); break;
    case EPI_RKL2_FIRST: launch_iso_nc<EPI_RKL2_FIRST>(c, grid, ic, ta, st); break;
    case EPI_RKL2_STAGE: launch_iso_nc<EPI_RKL2_STAGE>(c, grid, ic, ta, st); break;
    case EPI_RKL2_DSTAGE: launch_iso_nc<EPI_RKL2_DSTAGE>(c, grid, ic, ta, st); break;
    case EPI_PCG_S: launch_iso_nc<EPI_PCG_S>(c, grid, ic, ta, st); break;
    case EPI_PCG_R0: launch_iso_nc<EPI_PCG_R0>(c, grid, ic, ta, st); break;
    case EPI_PCG_M: launch_iso_nc<EPI_PCG_M>(c, grid, ic, ta, st); break;
    default: return false;
  }
  STS_CUDA(cudaGetLastError());
  return true;
}

}  // namespace sts
