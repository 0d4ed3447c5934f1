// TMA + mbarrier pipelined anisotropic stencil pass (sm_100a).
//
// Same arithmetic as aniso_fast_kernel (stencil.cu: vertex-centred symmetric
// scheme of DESIGN.md R2 / PAPER.md:173 boxed term, with the frozen per-vertex
// coefficients e of the lagged diffusivity), but every operand a CTA
// needs for one r-plane -- the staged source plane(s) with their theta/phi halo,
// the three vertex coefficients, and the pointwise epilogue operands -- arrives
// as ONE "package" of cp.async.bulk.tensor (TMA) boxes completing on one
// mbarrier.  A ring of slots keeps packages in flight while the CTA computes on
// the oldest, so the bytes in flight per SM no longer depend on registers or
// on how far each thread can prefetch (the limit ncu showed for the cp.async
// fast path: 27-29 % of DRAM peak, long-scoreboard bound).
//
// CTA = 8 warps x 32 lanes = 8 x 32 vertex columns -> 7 x 31 output cells.
// Boxes per package Q(p) (cell plane p, global coordinates, OOB -> zeros).  The
// innermost (phi) box origin must be 16 B aligned -- an odd FP64 column origin
// raises an illegal-instruction fault on sm_100a (measured, tools/probe) -- so
// every box starts at the even column at or below the first column it needs and
// the reader adds the shift back:
//   staged source f   : 36 cols x 9 rows from (even(k0-1), j0-1) of plane p
//                       (p = -1 / nl: the library's halo planes of the neighbour slab,
//                        else OOB zeros; the vertices there carry e = 0 anyway)
//   wrap columns      : 2 x 9 from (n3-2, j0-1) and (0, j0-1) (periodic phi, edge tiles)
//   vertex coeffs e   : 34 x 8 per component from (even(k0), j0), vertex plane p-1
//                       (padded e layout: zero row / wrap column built in)
//   epilogue operands : 32 x 7 from (even(k0), j0), cell plane p-1
// Ring depth: 4 slots (3 for the merged PCG pass, whose three staged fields make a
// larger slot; 3 CTAs per SM either way).
// Epilogues: F, RKL2 first stage / stage recurrence (Fig. 2, also in
// deviation form D_j = Y_j - Y0), the PCG initial residual with the Jacobi diagonal,
// the two-pass PCG S-pass  p = z + beta pold, x += ax pold, y = A p, partial p.y, and
// the merged one-pass PCG iteration (from staged p_{k-2}, w_{k-1}, p_{k-1}:
// z = (p_{k-1} - beta_{k-1} p_{k-2}) - ax w_{k-1}, p = z + beta p_{k-1}, y = A p, w = d y,
// four partial sums, x updated every other pass; Fig. 1 reorganised,
// DESIGN.md §5.3).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "sts_common.cuh"
#include "tma.cuh"
#include "pcg.cuh"

namespace sts {

using namespace tma;

namespace {

// register blocking: each consumer thread owns RB vertex rows of its column (the staged
// source rows it shares with its own vertex rows are loaded once, the vertical vertex
// pairs inside the thread are summed in registers; only its first row goes through
// shared memory to the warp above).  NW consumer warps -> XJ = NW RB vertex rows.
#ifndef ANISO_RB
#define ANISO_RB 2
#endif
#ifndef ANISO_NW
#define ANISO_NW 4
#endif
constexpr int RB = ANISO_RB, NW = ANISO_NW;
constexpr int XJ = NW * RB, XK = 32;         // vertex rows / cols
constexpr int XOJ = XJ - 1, XOK = XK - 1;   // output rows / cols
constexpr int XNT = NW * XK;                // consumer threads
constexpr int XTHREADS = XNT + 32;          // + producer warp
// ring slots (packages in flight = slots - 1): TmaLay::NS, 4 (3 for the merged PCG pass)
constexpr int UBW = 36, UBH = XJ + 1;       // staged-source box (cols x rows)
constexpr int EBW = 34;                     // vertex-coefficient box cols
constexpr int MAXSRC = 3;                   // staged sources (PCG S-pass: z, pold; merged: zold, wold, pold)
constexpr int MAXOWN = 4;                   // epilogue operand boxes
constexpr int r16(int n) { return (n + 15) & ~15; }
// slot parts (doubles); every part starts on a 128 B boundary
constexpr int U_MAIN = r16(UBH * UBW);
constexpr int U_WL = r16(2 * UBH), U_WR = r16(2 * UBH);
constexpr int U_FIELD = U_MAIN + U_WL + U_WR;
constexpr int E_COMP = r16(XJ * EBW);
constexpr int E_PART = 3 * E_COMP;
constexpr int O_PART = r16(XOJ * XK);
constexpr int VBUF = 3 * XNT;               // A, B, C of each warp's first vertex row
static_assert(XNT > XJ + 1, "sg3 is loaded by the first XJ + 1 consumer threads");

}  // namespace

// tensor maps of one launch (kernel parameter, __grid_constant__)
struct TmaArgs {
  CUtensorMap src[MAXSRC];    // staged sources, 3D (n3, n2, nl),       box 36 x 9 x 1
  CUtensorMap srch[MAXSRC];   // their halo planes, 3D (n3, n2, 2 MAXC), box 36 x 9 x 1
  CUtensorMap srcw[MAXSRC];   // wrap columns, main planes,             box 2 x 9 x 1
  CUtensorMap srchw[MAXSRC];  // wrap columns, halo planes,             box 2 x 9 x 1
  CUtensorMap e;              // vertex coefficients, 3D (n3+2, n2+1, 3 (nl+1)), box 34 x 8 x 1
                              // (a 4D map with the component as 4th dim faults on sm_100a)
  CUtensorMap own[MAXOWN];    // epilogue operands, 3D (n3, n2, nl),   box 32 x 7 x 1
  int has_lo, has_hi;
};

// resident CTAs per SM and ring slots of the merged PCG pass (compile-time knobs)
#ifndef ANISO_M_MINB
#define ANISO_M_MINB 3
#endif
#ifndef ANISO_M_NS
#define ANISO_M_NS 3
#endif
#ifndef ANISO_M_DREAD    // 0: the merged PCG pass recomputes d from the staged e (8 B/cell fewer)
#define ANISO_M_DREAD 1       // measured 42 % slower (L1 / register bound, spills): reads d
#endif
#ifndef ANISO_RASTER_H   // (theta-first bands measured worse for L2: DESIGN.md §5.4)
#define ANISO_RASTER_H 0
#endif
#ifndef ANISO_LEAN       // own-cell p_{k-1} loaded, z_k re-formed (instead of two more shuffles per row)
#define ANISO_LEAN 1
#endif
#ifndef ANISO_REGS       // PCG scalars and 1/g3 in registers instead of shared-memory operands
#define ANISO_REGS 1
#endif
#ifndef ANISO_PF         // L2 prefetch distance of the producer in planes (0: none)
#define ANISO_PF 0
#endif
#ifndef ANISO_NS         // ring slots of the other passes
#define ANISO_NS 4
#endif
#ifndef ANISO_MINB       // resident CTAs per SM of the other passes
#define ANISO_MINB 3
#endif
constexpr int aniso_minb(int epi) { return epi == EPI_PCG_M ? ANISO_M_MINB : ANISO_MINB; }

// epilogue operand slots
enum { OW_YM2 = 0, OW_Y0 = 1, OW_M0 = 2 };   // RKL2 stage
enum { OW_DM2 = 0, OW_DM0 = 1 };              // RKL2 stage, deviation form
enum { OW_X = 0 };                           // PCG S-pass / merged pass (x)
// slot layout of one (epilogue, has-w) variant
template <int EPI, bool W>
struct TmaLay {
  static constexpr int nsrc = (EPI == EPI_PCG_S) ? 2 : (EPI == EPI_PCG_M ? 3 : 1);
  // (merged PCG pass: x and d; ANISO_M_DREAD = 0 recomputes d from the staged e instead)
  static constexpr int nepi = (EPI == EPI_RKL2_STAGE)
                                  ? 3
                                  : (EPI == EPI_RKL2_DSTAGE || (EPI == EPI_PCG_M && ANISO_M_DREAD)
                                         ? 2
                                         : ((EPI == EPI_PCG_S || EPI == EPI_PCG_M) ? 1 : 0));
  static constexpr int nown = nepi + (W ? 1 : 0);             // w is the last own box
  static constexpr int E = nsrc * U_FIELD;
  static constexpr int O = E + E_PART;
  static constexpr int MT = O + nown * O_PART;       // per-plane metrics written by the producer
  static constexpr int SLOT = MT + 16;
  static constexpr int NS = (EPI == EPI_PCG_M) ? ANISO_M_NS : ANISO_NS;   // (the merged pass has a larger slot)
  static constexpr int MINB = aniso_minb(EPI);
  static constexpr size_t SMEM = (size_t)(NS * SLOT + 2 * VBUF) * sizeof(double) + 2 * NS * sizeof(uint64_t) + 128;
};

// FR: this launch finishes the pass's dot-product reduction in its last CTA
template <int EPI, bool W, bool FR>
__global__ void __launch_bounds__(XTHREADS, TmaLay<EPI, W>::MINB) aniso_tma_kernel(StencilCall c, int ic,
                                                                const __grid_constant__ TmaArgs ta) {
  using Lay = TmaLay<EPI, W>;
  constexpr int XTS = Lay::NS;
  constexpr bool kM = (EPI == EPI_PCG_M);
  extern __shared__ __align__(128) double smx[];
  double* ring = smx;                               // [XTS][SLOT]
  double* vbuf = smx + XTS * Lay::SLOT;             // [2][3][XNT]
  uint64_t* full = reinterpret_cast<uint64_t*>(vbuf + 2 * VBUF);
  uint64_t* empty = full + XTS;
  const Geo& G = c.geo;
  const Metrics& M = G.m;
  const int tid = threadIdx.x;
  const Tile3 tl = raster_tile(blockIdx.x, (c.geo.n3 + XOK - 1) / XOK, (c.geo.n2 + XOJ - 1) / XOJ, ANISO_RASTER_H);
  const int j0 = tl.y * XOJ, k0 = tl.x * XOK;
  const int ib = c.ib + tl.z * ic;
  const int ie = min(ib + ic, c.ie);
  const long long blk = blockIdx.x;

  if constexpr (EPI == EPI_PCG_S || kM) {
    if (c.ea.sc && c.ea.sc[0].done) return;
  }
  const bool first = (EPI == EPI_PCG_S || kM) && c.ea.first;
  const bool per = G.periodic3 != 0;
  const bool wrapL = per && k0 == 0;
  const bool wrapR = per && (k0 + 32 >= G.n3);
  const int ou = (k0 - 1) & ~1;                     // even box origins (floor, also for -1 -> -2)
  const int oe = k0 & ~1, se = k0 - oe;             // e / epilogue boxes and their column shift

  // warp-uniform values in shared memory (broadcast loads instead of registers):
  // 1/g3 of the vertex rows j0-1 .. j0+XJ-1 (row vj of a warp and the one above it)
  // and the PCG scalars beta_k, alpha_{k-1}
  // (merged PCG: the x mode of this pass and its catch-up coefficients, pcg.cuh)
  __shared__ double sg3[XJ + 1], sbx[5];
  __shared__ int sxm;
  if (tid <= XJ) {
    const int r = j0 - 1 + tid;
    sg3[tid] = (r >= 0 && r < G.n2) ? M.iG3[r] : 0.0;
  }
  if (tid == XJ + 1) {
    const bool kPcg = (EPI == EPI_PCG_S || kM) && !first;
    sbx[0] = kPcg ? c.ea.sc[0].beta : 0.0;
    sbx[1] = kPcg ? c.ea.sc[0].ax : 0.0;
    sbx[2] = (kM && kPcg) ? c.ea.sc[0].cxp : 0.0;
    sbx[3] = (kM && kPcg) ? c.ea.sc[0].cxz : 0.0;
    sbx[4] = (kM && kPcg) ? c.ea.sc[0].bprev : 0.0;
    sxm = (kM && kPcg) ? c.ea.sc[0].xm : X_NORMAL;
  }
  if (tid == 0) {
    for (int s = 0; s < XTS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // ======================= producer warp: package Q(p), p = ib-1 .. ie =======================
  if (tid >= XNT) {
    if (tid != XNT) return;
    const int nsrc_now = ((EPI == EPI_PCG_S || kM) && first) ? 1 : Lay::nsrc;
    // merged PCG: no x box when the pass does not touch x (first pass, skipped x update)
    const bool no_x = kM && (first || sxm == X_SKIP);
    for (int p = ib - 1; p <= ie; ++p) {
      const int slot = (p - ib + 1) % XTS, n = (p - ib + 1) / XTS;
      if (n > 0) mbar_wait(empty + slot, (uint32_t)((n - 1) & 1));
      double* S = ring + slot * Lay::SLOT;
      uint64_t* bar = full + slot;
      const bool lo = p < 0, hi = p >= G.nl;
      const bool halo = (lo && ta.has_lo) || (hi && ta.has_hi);
      const int pc = halo ? (lo ? 0 : MAXC) : p;    // no neighbour: OOB plane -> zeros
      const bool has_e = p >= ib, has_own = p >= ib + 1;
      uint32_t bytes = nsrc_now * UBW * UBH * 8;
      if (wrapL) bytes += nsrc_now * 2 * UBH * 8;
      if (wrapR) bytes += nsrc_now * 2 * UBH * 8;
      if (has_e) bytes += 3 * XJ * EBW * 8;   // (E_COMP is padded to 128 B; the box is not)
      // (merged PCG: the x box is of the package's OWN plane p -- the x update uses only
      // values of plane p's slot -- the other epilogue boxes are of plane p-1)
      const bool x_here = kM && !no_x && p >= ib && p < ie;
      if (has_own) bytes += (Lay::nown - (kM ? 1 : 0)) * XOJ * XK * 8;
      if (x_here) bytes += XOJ * XK * 8;
      // per-plane metrics (plain stores: the mbarrier arrive below releases them to the
      // consumers' acquiring wait): iG2 of cell planes p-1 and p, Vr of plane p-1
      {
        const int i = G.i0 + p;
        S[Lay::MT + 0] = (i - 1 >= 0 && i - 1 < G.n1g) ? M.iG2[i - 1] : 0.0;
        S[Lay::MT + 1] = (i >= 0 && i < G.n1g) ? M.iG2[i] : 0.0;
        S[Lay::MT + 2] = (i - 1 >= 0 && i - 1 < G.n1g) ? M.Vr[i - 1] : 0.0;
      }
      fence_proxy_async();
      mbar_expect_tx(bar, bytes);
      for (int f = 0; f < nsrc_now; ++f) {
        double* D = S + f * U_FIELD;
        tma3(D, halo ? &ta.srch[f] : &ta.src[f], ou, j0 - 1, pc, bar);
        if (wrapL) tma3(D + U_MAIN, halo ? &ta.srchw[f] : &ta.srcw[f], G.n3 - 2, j0 - 1, pc, bar);
        if (wrapR) tma3(D + U_MAIN + U_WL, halo ? &ta.srchw[f] : &ta.srcw[f], 0, j0 - 1, pc, bar);
      }
      if (has_e)   // vertex plane p-1 = ev plane index p (row jv+1), one 3D box per component
        for (int a = 0; a < 3; ++a) tma3(S + Lay::E + a * E_COMP, &ta.e, oe, j0, a * (G.nl + 1) + p, bar);
      if (has_own)
#pragma unroll
        for (int q = 0; q < Lay::nown; ++q)
          if (!(kM && q == OW_X)) tma3(S + Lay::O + q * O_PART, &ta.own[q], oe, j0, p - 1, bar);
      if (x_here) tma3(S + Lay::O + OW_X * O_PART, &ta.own[OW_X], oe, j0, p, bar);
      if constexpr (ANISO_PF > 0) {
        // L2 prefetch of package Q(p + PF) (main-array planes only; the wrap columns and
        // halo planes are small and left to the loads)
        const int pf = p + ANISO_PF;
        if (pf <= ie && pf < G.nl) {
          for (int f = 0; f < nsrc_now; ++f) tma3_prefetch(&ta.src[f], ou, j0 - 1, pf);
          for (int a = 0; a < 3; ++a) tma3_prefetch(&ta.e, oe, j0, a * (G.nl + 1) + pf);
#pragma unroll
          for (int q = 0; q < Lay::nown; ++q)
            if (!(kM && q == OW_X)) tma3_prefetch(&ta.own[q], oe, j0, pf - 1);
          if (kM && !no_x && pf < ie) tma3_prefetch(&ta.own[OW_X], oe, j0, pf);
        }
      }
    }
    return;
  }

  // ======================= consumer warps =======================
  // warp vj, lane vk: vertex rows vr = vj RB + t (t < RB) of vertex column vk; the own cell
  // of vertex row vr is cell row j0 + vr, col k0 + vk (between vertex rows vr, vr + 1)
  const int vj = tid >> 5, vk = tid & 31;
  const int vr0 = vj * RB;
  // references into shared memory (read where used; they hold no registers)
#if ANISO_REGS
  // (ANISO_REGS: the warp-uniform scalars and the 1/g3 of the thread's RB+1 rows in
  // registers -- shared-memory operands are re-read after every barrier's memory clobber)
  const double beta = sbx[0], ax = sbx[1], bprev = sbx[4], cxp = sbx[2], cxz = sbx[3];
  double rg3[RB + 1];
#pragma unroll
  for (int r = 0; r <= RB; ++r) rg3[r] = sg3[vr0 + r];
#define G3(r) rg3[r]
#else
  const double& beta = sbx[0];
  const double& ax = sbx[1];
  const double& bprev = sbx[4];
  const double& cxp = sbx[2];
  const double& cxz = sbx[3];
#define G3(r) sg3[vr0 + (r)]
#endif
  const int k = k0 + vk;
  const bool colok = vk < XOK && k < G.n3;
  bool ownr[RB];   // (evaluated once: the march tests it per row and plane)
#pragma unroll
  for (int t = 0; t < RB; ++t) ownr[t] = colok && vr0 + t < XOJ && j0 + vr0 + t < G.n2;
  auto own_t = [&](int t) { return ownr[t]; };
  const long long coff0 = (long long)(j0 + vr0) * G.n3 + k;   // own cell of row t: coff0 + t n3
  double* const xown = kM ? c.ea.x + coff0 : nullptr;          // (merged PCG: x of the own cells)
  double vtpc[RB];
#pragma unroll
  for (int t = 0; t < RB; ++t) vtpc[t] = own_t(t) ? M.Vt[j0 + vr0 + t] * M.Vp[k] : 0.0;
  // offset (within a staged field block) of the cell at tile row r (global j0-1+r) and
  // tile col c (global k0-1+c): base + r * stride (the wrap columns are stored 2 wide)
  auto ubase = [&](int c, int& stride) {
    const int gk = k0 - 1 + c;                        // global phi index
    if (per && gk == -1) { stride = 2; return U_MAIN + 1; }           // periodic wrap: cell n3-1
    if (per && gk == G.n3) { stride = 2; return U_MAIN + U_WL; }      // periodic wrap: cell 0
    stride = UBW;
    return gk - ou;                                   // (non-periodic col -1 / n3: OOB zeros)
  };
  int sa, sb;
  const int ca = ubase(vk, sa), cb = ubase(vk + 1, sb);
  const int oa = ca + vr0 * sa, ob = cb + vr0 * sb;   // tile row vr0, cols vk / vk+1

  // in-plane 2x2 boxes of the source value s (PCG: z + beta pold, else u) of the thread's
  // RB vertex rows: it loads its column's RB+1 source rows once and takes column vk+1 from
  // lane vk+1 by shuffle (lane 31 loads it)
  // merged PCG (kM): fields p_{k-2}, w_{k-1}, p_{k-1}: z_k = (p_{k-1} - beta_{k-1} p_{k-2}) - alpha_{k-1} w_{k-1}
  constexpr bool kP = (EPI == EPI_PCG_S);
  constexpr int PF = kM ? 2 * U_FIELD : U_FIELD;    // pold field offset
  auto zof = [&](const double* S, int o) {
    if (kM && !first) return fma(-ax, S[U_FIELD + o], fma(-bprev, S[o], S[PF + o]));
    return S[o];
  };
  // state of one cell plane carried to the next, per vertex row t: the 2x2 sums of the
  // source, the vertex-pair sums of the vertex plane below it, the own cell's source value
  // (pold, z), and (R0) the L_ii part of the 4 vertices above it.  Two sets, alternated
  // by an unroll by two, so no register moves between planes.
  // R0: L_ii = -sum over the cell's 8 vertices of W^2, W = the cell's weight in q_v =
  // sr er + st et ig2 + sp ep ig2 ig3 (signs from the cell's octant in the vertex)
  struct St {
    double Su[RB], Tu[RB], Fu[RB], SA[RB], DB[RB], DC[RB], u[RB], po[RB], z[RB], ld[RB];
  };
  auto usums = [&](const double* S, St& H) {
    double zl[RB + 1], zr[RB + 1], qr[RB + 1], kr[RB + 1];
#pragma unroll
    for (int r = 0; r <= RB; ++r) {
      double z = zof(S, oa + r * sa);
      const double zk = z;
      double q = 0.0;
      if ((kP || kM) && !first) {
        q = S[PF + oa + r * sa];
        z = fma(beta, q, z);
      }
      zl[r] = z;
      zr[r] = __shfl_down_sync(0xffffffffu, z, 1);
      if constexpr (ANISO_LEAN) {
        // the own cells' p_{k-1} (rows 1..RB, col vk+1) straight from the slot, and their
        // z_k re-formed below as p_k - beta p_{k-1}: one shuffled field instead of three
        (void)zk;
        qr[r] = ((kP || kM) && !first && r > 0) ? S[PF + ob + r * sb] : 0.0;
        kr[r] = 0.0;
        if (vk == XK - 1) zr[r] = zof(S, ob + r * sb);
        if (vk == XK - 1 && (kP || kM) && !first) zr[r] = fma(beta, qr[r] = S[PF + ob + r * sb], zr[r]);
        continue;
      }
      qr[r] = ((kP || kM) && !first) ? __shfl_down_sync(0xffffffffu, q, 1) : 0.0;
      kr[r] = kM ? __shfl_down_sync(0xffffffffu, zk, 1) : 0.0;
      if (vk == XK - 1) {
        double z1 = zof(S, ob + r * sb);
        kr[r] = z1;
        if ((kP || kM) && !first) {
          qr[r] = S[PF + ob + r * sb];
          z1 = fma(beta, qr[r], z1);
        }
        zr[r] = z1;
      }
    }
#pragma unroll
    for (int t = 0; t < RB; ++t) {
      H.Su[t] = (zl[t] + zr[t]) + (zl[t + 1] + zr[t + 1]);
      H.Tu[t] = (zl[t + 1] - zl[t]) + (zr[t + 1] - zr[t]);
      H.Fu[t] = G3(t) * (zr[t] - zl[t]) + G3(t + 1) * (zr[t + 1] - zl[t + 1]);
      H.u[t] = zr[t + 1];    // own cell of this plane
      H.po[t] = qr[t + 1];   // its pold (PCG)
      H.z[t] = ANISO_LEAN ? (kM && !first ? fma(-beta, qr[t + 1], zr[t + 1]) : zr[t + 1])
                          : kr[t + 1];    // its z (merged PCG)
    }
  };

  double part = 0.0, part2 = 0.0, part3 = 0.0, part4 = 0.0;
  constexpr bool kR0 = (EPI == EPI_PCG_R0);
  St SX, SY;
#pragma unroll
  for (int t = 0; t < RB; ++t) {
    SX.Su[t] = SX.Tu[t] = SX.Fu[t] = SX.SA[t] = SX.DB[t] = SX.DC[t] = SX.u[t] = SX.po[t] = SX.z[t] = SX.ld[t] = 0.0;
  }
  SY = SX;
  const int xm = kM ? sxm : X_NORMAL;
  // plane p: Q(p) landed; L = state of cell plane p-1, H receives cell plane p's
  auto body = [&](int p, const St& L, St& H) {
    const int slot = (p - ib + 1) % XTS;
    const double* S = ring + slot * Lay::SLOT;
    mbar_wait(full + slot, (uint32_t)(((p - ib + 1) / XTS) & 1));
    usums(S, H);
    if constexpr (kM) {
      // x of the own cells of plane p, from this slot alone (pcg.cuh "x in pairs"):
      // x_k = x_{k-1} + alpha_{k-1} p_{k-1}, skipped, or the catch-up
      // x_k = x_{k-2} + cxp p_{k-1} - cxz z_{k-1} (raw staged z_{k-1})
      if (!first && xm != X_SKIP && p >= ib && p < ie) {
#pragma unroll
        for (int t = 0; t < RB; ++t) {
          if (!own_t(t)) continue;
          const double* Ox = S + Lay::O + OW_X * O_PART + (vr0 + t) * XK + vk + se;
          double xn = fma(xm == X_CATCHUP ? cxp : ax, H.po[t], *Ox);
          if (xm == X_CATCHUP) xn = fma(cxz, S[ob + (t + 1) * sb], xn);   // + alpha_{k-2} p_{k-2} (field 0)
          __stcs(xown + (long long)p * G.plane + t * G.n3, xn);
        }
      }
    }
    double* vb = vbuf + (p & 1) * VBUF;
#pragma unroll
    for (int t = 0; t < RB; ++t) H.SA[t] = H.DB[t] = H.DC[t] = H.ld[t] = 0.0;
    if (p >= ib) {
      // vertex plane v = p-1, between cell planes p-1 (L) and p (H); e = 0 where a cell is missing
      const double* E = S + Lay::E;
      const double ig2l = S[Lay::MT + 0], ig2h = S[Lay::MT + 1];
      double hA[RB], hB[RB], dC[RB], ldhi[RB];
#pragma unroll
      for (int t = 0; t < RB; ++t) {
        const int ei = (vr0 + t) * EBW + vk + se;
        const double er = E[ei], et = E[E_COMP + ei], ep = E[2 * E_COMP + ei];
        const double q =
            er * (H.Su[t] - L.Su[t]) + et * (ig2l * L.Tu[t] + ig2h * H.Tu[t]) + ep * (ig2l * L.Fu[t] + ig2h * H.Fu[t]);
        ldhi[t] = 0.0;
        if constexpr (kR0 || (kM && !ANISO_M_DREAD)) {
          if (own_t(t)) {
            // this vertex plane is above cell plane p-1 (sr = -1, ig2l) and below plane p (sr = +1, ig2h);
            // the own cell (j, k) sits at (st, sp) = (+,+) in vertex (vr,vk), (+,-) in (vr,vk+1),
            // (-,+) in (vr+1,vk), (-,-) in (vr+1,vk+1)
            const double ig3c = G3(t + 1);
            const int e4[4] = {ei, ei + 1, ei + EBW, ei + EBW + 1};
            const double st4[4] = {1.0, 1.0, -1.0, -1.0}, sp4[4] = {1.0, -1.0, 1.0, -1.0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double r_ = E[e4[u]], t_ = E[E_COMP + e4[u]], p_ = E[2 * E_COMP + e4[u]];
              const double wl = -r_ + st4[u] * t_ * ig2l + sp4[u] * p_ * ig2l * ig3c;
              const double wh = r_ + st4[u] * t_ * ig2h + sp4[u] * p_ * ig2h * ig3c;
              ldhi[t] += wl * wl;
              H.ld[t] += wh * wh;
            }
          }
        }
        // vertex values A, B, C = q e; the horizontal pair sums/differences by shuffle
        const double A = q * er, B = q * et, C = q * ep;
        hA[t] = A + __shfl_down_sync(0xffffffffu, A, 1);
        hB[t] = B + __shfl_down_sync(0xffffffffu, B, 1);
        dC[t] = C - __shfl_down_sync(0xffffffffu, C, 1);
      }
      // the vertical pairs: inside the thread, and through shared memory for the last
      // row (the next vertex row is the first row of the next warp)
      vb[tid] = hA[0];
      vb[XNT + tid] = hB[0];
      vb[2 * XNT + tid] = dC[0];
      // consumer warps only: the vertex plane is complete
      asm volatile("bar.sync 1, %0;\n" ::"r"(XNT) : "memory");
#pragma unroll
      for (int t = 0; t < RB; ++t) {
        if (!own_t(t)) continue;
        const double nA = (t + 1 < RB) ? hA[(t + 1) % RB] : vb[tid + 32];
        const double nB = (t + 1 < RB) ? hB[(t + 1) % RB] : vb[XNT + tid + 32];
        const double nC = (t + 1 < RB) ? dC[(t + 1) % RB] : vb[2 * XNT + tid + 32];
        H.SA[t] = hA[t] + nA;
        H.DB[t] = hB[t] - nB;
        H.DC[t] = dC[t] + nC;
      }
      if (p >= ib + 1) {
        // output cell plane il = p-1 (its own values are L's)
        const int il = p - 1;
        const double ig2c = S[Lay::MT + 0];                   // iG2 of plane p-1
#pragma unroll
        for (int t = 0; t < RB; ++t) {
          if (!own_t(t)) continue;
          const double ig3c = G3(t + 1);
          const double* O = S + Lay::O + (vr0 + t) * XK + vk + se;
          const double Lu = -((L.SA[t] - H.SA[t]) + ig2c * (L.DB[t] + H.DB[t]) + ig2c * ig3c * (L.DC[t] + H.DC[t]));
          const double WV = (W ? O[Lay::nepi * O_PART] : 1.0) * S[Lay::MT + 2] * vtpc[t];
          const long long gi = (long long)il * G.plane + coff0 + (long long)t * G.n3;
          const double uc = L.u[t], poc = L.po[t], zc = L.z[t];
          if constexpr (EPI == EPI_F) {
            c.ea.out[gi] = Lu / WV;
          } else if constexpr (EPI == EPI_RKL2_FIRST) {
            const double F = Lu / WV;
            c.ea.out2[gi] = F;
            c.ea.out[gi] = c.ea.a0 * uc + c.ea.c0 * F;
          } else if constexpr (EPI == EPI_RKL2_STAGE) {
            const double F = Lu / WV;
            c.ea.out[gi] = c.ea.mu * uc + c.ea.nu * O[OW_YM2 * O_PART] + c.ea.c2 * O[OW_Y0 * O_PART] + c.ea.c0 * F +
                           c.ea.c1 * O[OW_M0 * O_PART];
          } else if constexpr (EPI == EPI_RKL2_DSTAGE) {
            const double F = Lu / WV;
            c.ea.out[gi] = c.ea.mu * uc + c.ea.nu * O[OW_DM2 * O_PART] + c.ea.c0 * F + c.ea.c1 * O[OW_DM0 * O_PART];
          } else if constexpr (kR0) {
            // r0 = dt L u (x0 = u^n), d = 1/(wV - dt L_ii) (PC1), z0 = r0 d
            const double Ld = -(L.ld[t] + ldhi[t]);
            const double r = c.ea.dt * Lu;
            const double dinv = rcp_pos(WV - c.ea.dt * Ld);
            const double z = r * dinv;
            const double bb = WV * uc;
            c.ea.out[gi] = r;
            if (c.ea.out2) c.ea.out2[gi] = uc;
            if (c.ea.out3) c.ea.out3[gi] = z;
            c.ea.out4[gi] = dinv;
            part += r * z;
            part2 += bb * bb * dinv;
          } else if constexpr (EPI == EPI_PCG_S) {
            const double y = WV * uc - c.ea.dt * Lu;
            c.ea.out[gi] = y;
            c.ea.out2[gi] = uc;                                   // p_k
            if (!first) c.ea.x[gi] = fma(ax, poc, O[OW_X * O_PART]);   // x_k = x_{k-1} + alpha_{k-1} p_{k-1}
            part += uc * y;
          } else if constexpr (kM) {
            // y_k = A p_k, w_k = d y_k; p_k, w_k to the next buffers (z is not stored);
            // partials r_k.z_k = z_k^2 / d, p_k.y_k, z_k.y_k, w_k.y_k
            const double y = WV * uc - c.ea.dt * Lu;
            // the Jacobi diagonal A_ii = wV - dt L_ii of the R0 pass (same arithmetic), d = 1/A_ii
            const double Aii = ANISO_M_DREAD ? rcp_pos(O[1 * O_PART]) : WV - c.ea.dt * (-(L.ld[t] + ldhi[t]));
            const double dd = ANISO_M_DREAD ? O[1 * O_PART] : rcp_pos(Aii);
            const double wk = dd * y;
            // streaming stores (evict-first in L2): the outputs are read again only by the
            // next pass, after far more than L2 has streamed through; L2 keeps the input
            // halo rows the neighbouring tiles re-read instead
            __stcs(c.ea.out2 + gi, uc);
            __stcs(c.ea.out3 + gi, wk);
            // (x of this plane was updated when its slot landed, above)
            part += zc * zc * Aii;
            part2 += uc * y;
            part3 += zc * y;
            part4 += wk * y;
          }
        }
      }
    }
    __syncwarp();
    if (vk == 0) mbar_arrive(empty + slot);   // this warp is done with the slot of Q(p)
  };
  int p = ib - 1;
  for (; p + 1 <= ie; p += 2) {
    body(p, SX, SY);
    body(p + 1, SY, SX);
  }
  if (p <= ie) body(p, SX, SY);
  if constexpr (kR0) {
    __shared__ double red2[2][XNT / 32];
    double v = part, v2 = part2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_xor_sync(0xffffffffu, v, o);
      v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    if (vk == 0) {
      red2[0][vj] = v;
      red2[1][vj] = v2;
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(XNT) : "memory");
    if (tid < 2) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < XNT / 32; ++w) s += red2[tid][w];
      c.ea.partials[tid * c.ea.pstride + c.ea.pbase + blk] = s;
    }
  }
  if constexpr (EPI == EPI_PCG_S || kM) {
    // partial rows: S-pass p.y; merged r.z, p.y, z.y, w.y
    constexpr int NQ = kM ? 4 : 1;
    __shared__ double red[NQ][XNT / 32];
    double pv[4] = {part, part2, part3, part4};
#pragma unroll
    for (int t = 0; t < NQ; ++t) {
      double v = pv[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (vk == 0) red[t][vj] = v;
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(XNT) : "memory");
    if (tid < NQ) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < XNT / 32; ++w) s += red[tid][w];
      c.ea.partials[tid * c.ea.pstride + c.ea.pbase + blk] = s;
    }
    if constexpr (FR) {
      __shared__ double fred[4 * MAXC * 32];
      __shared__ unsigned flag;
      fused_final_reduce(c.ea.fin, c.ea.partials, c.ea.pstride,
                         (unsigned long long)gridDim.x, tid, XNT, fred, &flag,
                         [] { asm volatile("bar.sync 1, %0;\n" ::"r"(XNT) : "memory"); });
    }
  }
}


#undef G3

// ============================================================================
// host side
// ============================================================================
static bool has_tma(int epi) {
  return epi == EPI_F || epi == EPI_RKL2_FIRST || epi == EPI_RKL2_STAGE || epi == EPI_PCG_S || epi == EPI_PCG_R0 ||
         epi == EPI_PCG_M || epi == EPI_RKL2_DSTAGE;
}

bool aniso_tma_eligible(const StencilCall& c) {
  if (c.mode != STS_MODE_ANISO || c.ncomp != 1 || !has_tma(c.epi) || !c.ev) return false;
  const Geo& G = c.geo;
  if (G.n3 % 2 != 0 || G.n3 < 2) return false;
  if (!al16(c.u.p) || !al16(c.u.lo) || !al16(c.u2.p) || !al16(c.u2.lo) || !al16(c.ev) || !al16(c.w)) return false;
  if (!al16(c.ea.ym2) || !al16(c.ea.y0) || !al16(c.ea.m0) || !al16(c.ea.x)) return false;
  // halo planes come from the library's contiguous [2][MAXC][plane] slot buffers
  if (c.u.lo && c.u.hi && c.u.hi != c.u.lo + (long long)MAXC * G.plane) return false;
  if (c.u2.lo && c.u2.hi && c.u2.hi != c.u2.lo + (long long)MAXC * G.plane) return false;
  if (c.epi == EPI_PCG_M) {
    if (!al16(c.u3.p) || !al16(c.u3.lo) || !c.ea.dinv || !al16(c.ea.dinv) || !c.ea.x || !c.ea.out3) return false;
    if (c.u3.lo && c.u3.hi && c.u3.hi != c.u3.lo + (long long)MAXC * G.plane) return false;
  }
  return true;   // a slab with only a hi halo maps its slot buffer from hi - MAXC*plane
}

static dim3 tma_grid(const Geo& G, int ib, int ie, int minb, int* ic_out) {
  const int nbx = (G.n3 + XOK - 1) / XOK, nby = (G.n2 + XOJ - 1) / XOJ;
  const int np = ie - ib;
  if (np <= 0) {
    *ic_out = 1;
    return dim3(0, 0, 0);
  }
  const long long tiles = (long long)nbx * nby;
  const int ic = choose_chunk(tiles, np, 148LL * minb, 2.0, 6);
  *ic_out = ic;
  return dim3(nbx, nby, (np + ic - 1) / ic);
}

int aniso_tma_blocks(const StencilCall& c) {
  int ic;
  const dim3 g = tma_grid(c.geo, c.ib, c.ie, aniso_minb(c.epi), &ic);
  return (int)(g.x * g.y * g.z);
}

template <int EPI, bool W, bool FR>
static void launch_t(const StencilCall& c, dim3 grid, int ic, const TmaArgs& ta, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  ensure_smem_attr(aniso_tma_kernel<EPI, W, FR>, (int)TmaLay<EPI, W>::SMEM, attr);
  aniso_tma_kernel<EPI, W, FR><<<dim3(grid.x * grid.y * grid.z), XTHREADS, TmaLay<EPI, W>::SMEM, st>>>(c, ic, ta);
}

template <int EPI>
static void launch_w(const StencilCall& c, dim3 grid, int ic, const TmaArgs& ta, cudaStream_t st) {
  constexpr bool kS = (EPI == EPI_PCG_S || EPI == EPI_PCG_M);
  const bool fr = kS && c.ea.fin.ticket;
  if (c.w) {
    if (fr) launch_t<EPI, true, kS>(c, grid, ic, ta, st);
    else launch_t<EPI, true, false>(c, grid, ic, ta, st);
  } else {
    if (fr) launch_t<EPI, false, kS>(c, grid, ic, ta, st);
    else launch_t<EPI, false, false>(c, grid, ic, ta, st);
  }
}

bool launch_aniso_tma(const StencilCall& c, cudaStream_t st) {
  if (!aniso_tma_eligible(c)) return false;
  const Geo& G = c.geo;
  int ic = 1;
  const dim3 grid = tma_grid(G, c.ib, c.ie, aniso_minb(c.epi), &ic);
  if (grid.x == 0) return true;
  TmaArgs ta;
  memset(&ta, 0, sizeof(ta));
  const FieldV* srcs[MAXSRC] = {&c.u, &c.u2, &c.u3};
  const int nsrc = (c.epi == EPI_PCG_S) ? 2 : (c.epi == EPI_PCG_M ? 3 : 1);
  ta.has_lo = c.u.lo != nullptr;
  ta.has_hi = c.u.hi != nullptr;
  for (int f = 0; f < nsrc; ++f) {
    const FieldV& F = *srcs[f];
    const double* pm = F.p ? F.p : c.u.p;   // pold absent on the first PCG iteration: any valid map
    map_plain(&ta.src[f], pm, G, G.nl, UBW, UBH);
    map_plain(&ta.srcw[f], pm, G, G.nl, 2, UBH);
    const double* hb = F.lo ? F.lo : (F.hi ? F.hi - (long long)MAXC * G.plane : nullptr);
    if (hb) {
      map_plain(&ta.srch[f], hb, G, 2 * MAXC, UBW, UBH);
      map_plain(&ta.srchw[f], hb, G, 2 * MAXC, 2, UBH);
    } else {
      ta.srch[f] = ta.src[f];
      ta.srchw[f] = ta.srcw[f];
    }
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)ev_row(G.n3), (cuuint64_t)G.n2 + 1, 3 * ((cuuint64_t)G.nl + 1)};
    const cuuint64_t str[2] = {(cuuint64_t)ev_row(G.n3) * 8, (cuuint64_t)ev_plane(G.n2, G.n3) * 8};
    const cuuint32_t box[3] = {EBW, XJ, 1};
    encode(&ta.e, c.ev, 3, dims, str, box);
  }
  const double* owns[MAXOWN];
  int nown = 0;
  if (c.epi == EPI_RKL2_STAGE) {
    owns[nown++] = c.ea.ym2;
    owns[nown++] = c.ea.y0;
    owns[nown++] = c.ea.m0;
  } else if (c.epi == EPI_RKL2_DSTAGE) {
    owns[nown++] = c.ea.ym2;
    owns[nown++] = c.ea.m0;
  } else if (c.epi == EPI_PCG_S) {
    owns[nown++] = c.ea.x;
  } else if (c.epi == EPI_PCG_M) {
    owns[nown++] = c.ea.x;
    if (ANISO_M_DREAD) owns[nown++] = c.ea.dinv;
  }
  if (c.w) owns[nown++] = c.w;
  for (int q = 0; q < nown; ++q) map_plain(&ta.own[q], owns[q], G, G.nl, XK, XOJ);
  switch (c.epi) {
    case EPI_F: launch_w<EPI_F>(c, grid, ic, ta, st); break;
    case EPI_RKL2_FIRST: launch_w<EPI_RKL2_FIRST>(c, grid, ic, ta, st); break;
    case EPI_RKL2_STAGE: launch_w<EPI_RKL2_STAGE>(c, grid, ic, ta, st); break;
    case EPI_RKL2_DSTAGE: launch_w<EPI_RKL2_DSTAGE>(c, grid, ic, ta, st); break;
    case EPI_PCG_S: launch_w<EPI_PCG_S>(c, grid, ic, ta, st); break;
    case EPI_PCG_R0: launch_w<EPI_PCG_R0>(c, grid, ic, ta, st); break;
    case EPI_PCG_M: launch_w<EPI_PCG_M>(c, grid, ic, ta, st); break;
    default: return false;
  }
  STS_CUDA(cudaGetLastError());
  return true;
}

}  // namespace sts
