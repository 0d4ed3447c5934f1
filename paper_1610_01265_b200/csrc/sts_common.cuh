// Internal declarations of libsts_b200 (not part of the C ABI).
// Product code: shares nothing with oracle/ (DESIGN.md "Boundary").
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <list>
#include <string>
#include <vector>

#include "../../include/sts_b200.h"

namespace sts {

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
void set_error(const std::string& msg);

struct Error {
  int code;
  std::string msg;
};

#define STS_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::sts::Error{STS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                           " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
  } while (0)

#define STS_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw ::sts::Error{STS_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

#define STS_REQUIRE(cond, msg)                                  \
  do {                                                          \
    if (!(cond)) throw ::sts::Error{STS_ERR_ARG, (msg)};        \
  } while (0)

// ----------------------------------------------------------------------------
// tiling constants: a CTA owns a TJ x TK (theta x phi) tile of cell columns and
// marches along r over a chunk of planes (2.5-D blocking, phi contiguous).
// ----------------------------------------------------------------------------
constexpr int TK = 32;            // phi cells per tile  (one warp row, 256 B of FP64)
constexpr int TJ = 8;             // theta cells per tile
constexpr int NT = TK * TJ;       // threads per CTA
constexpr int RJ = TJ + 2;        // cell region rows incl. halo
constexpr int RK = TK + 2;        // cell region cols incl. halo
constexpr int RC = RJ * RK;       // cells in the region
constexpr int VJ = TJ + 1;        // vertex rows
constexpr int VK = TK + 1;        // vertex cols
constexpr int VC = VJ * VK;
constexpr int MAXC = 3;           // max components (velocity)

// Device metric arrays, all indexed by GLOBAL cell index (R1, §5).
//   face coefficient A/h = F{d}r[i] * F{d}t[j] * F{d}p[k]   (ISO operator)
//   volume V            = Vr[i] * Vt[j] * Vp[k]
//   centre distances     h_r = H1[i], h_th = G2[i'] H2[j], h_ph = G2[i'] G3[j'] H3[k]
//   (the "inv" arrays hold reciprocals used by the vertex scheme)
struct Metrics {
  const double *F1r, *F2r, *F3r, *Vr, *iH1, *iG2;   // n1
  const double *F1t, *F2t, *F3t, *Vt, *iH2, *iG3;   // n2
  const double *F1p, *F2p, *F3p, *Vp, *iH3;         // n3
};

// A field as seen by one slab: local planes plus optional halo planes.
struct FieldV {
  const double* p = nullptr;   // [ncomp][nl][plane]
  const double* lo = nullptr;  // [ncomp][plane] : plane il = -1 (nullptr at r_min)
  const double* hi = nullptr;  // [ncomp][plane] : plane il = nl (nullptr at r_max)
};

struct Geo {
  int n1g, n2, n3, periodic3;
  int i0, nl;                  // slab: global planes [i0, i0+nl)
  long long plane;             // n2*n3
  long long cstride;           // nl*plane (component stride of local arrays)
  Metrics m;
};

// ----------------------------------------------------------------------------
// the grid handle
// ----------------------------------------------------------------------------
struct Slab {
  int i0, nl;                  // global planes of this slab
  long long off;               // element offset of the slab in the (virtual) whole array
  // halo buffers owned by the library: [field slot][side][MAXC*plane]
  std::vector<double*> halo_lo, halo_hi;
  bool has_lo, has_hi;
};

// halo planes of the fields the stencils read across slab boundaries.  Per slot
// ONE allocation [2][MAXC][plane]: the lo planes (comp c at c) then the hi planes
// (comp c at MAXC + c), so a single TMA tensor map covers both sides.
enum HaloSlot { H_U = 0, H_K1, H_K2, H_K3, H_B, H_AUX, H_Z, H_P, H_D, H_W, H_NSLOTS };

struct Workspace {
  double* base = nullptr;
  size_t bytes = 0;
};

// Device staging buffer of the host-array path (capi.cu HostIO): free for reuse once
// `ev` (recorded after its last use: the consuming kernels of an input, the download of
// an output) has completed.
struct StageBuf {
  double* p = nullptr;
  size_t bytes = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;     // ev recorded and possibly not complete
  bool claimed = false;     // held by the call being enqueued
  unsigned long long seq = 0;   // release order (oldest first when the pool must wait)
};

// Coefficients of one operator mode kept resident across calls (sts_grid_bind_coeffs):
// the arrays in use (caller device arrays, or library-owned copies of host arrays and
// face-kappa outputs) and the data derived from them once per binding: the frozen vertex
// coefficients (ANISO), the metric-folded face coefficients of the merged PCG pass (ISO)
// and the Gershgorin bound.
struct CoefSlot {
  bool bound = false;
  const double* k[3] = {nullptr, nullptr, nullptr};
  const double* b = nullptr;
  const double* w = nullptr;
  double* own[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};   // k1, k2, k3, b, w copies of host arrays
  size_t own_n[5] = {0, 0, 0, 0, 0};
  double* kfk[3] = {nullptr, nullptr, nullptr};   // face diffusivities written by sts_face_kappa_spitzer
  double* dbuf = nullptr;             // ANISO: vertex coefficients of every slab; ISO: K1, K2, K3, wV
  size_t dbytes = 0;
  // Every call that reads the binding records last_use on its (compute) stream; work
  // that OVERWRITES the binding's arrays on another stream (uploads on the H2D stream,
  // face kappa / derived data on the coefficient stream) waits for it -- exactly the
  // previous binding's readers, not everything enqueued on the compute stream.
  cudaEvent_t last_use = nullptr;
  bool use_set = false;
  bool user_dev = false;              // a bound array is a caller device array (written on the caller's stream)
  bool ev_ok = false, pre_ok = false; // derived data current for the bound arrays
  double lam = -1.0;                  // cached Gershgorin max row sum (< 0: not computed)
};

}  // namespace sts

struct sts_grid {
  int device = 0;
  int geom = 0;
  int n1g = 0, n2 = 0, n3 = 0, periodic3 = 0;
  int i0 = 0, nl = 0;
  int n_virtual = 1;
  long long plane = 0;
  std::vector<double> h_x1f, h_x1c, h_x2f, h_x2c, h_x3f, h_x3c;
  double* d_metrics = nullptr;          // one allocation for all metric arrays
  sts::Metrics m{};
  std::vector<sts::Slab> slabs;         // 1 (real) or n_virtual (emulation)
  // workspace (scratch fields, staging) — grows on demand
  sts::Workspace ws;
  double* d_red = nullptr;              // reduction partials + scalars
  size_t red_bytes = 0;
  unsigned int* d_ticket = nullptr;     // last-block tickets ([0] stencil passes, [1] reductions)
  double* d_red2 = nullptr;             // second level of the multi-block PCG reduction
  double* h_pinned = nullptr;           // small pinned, device-mapped host mailbox
  double* d_pinned = nullptr;           // its device alias (written by launch_publish)
  // multi-GPU
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  long long launches = 0;
  std::atomic<long long> launches_async{0};    // added by completion callbacks of asynchronous solves
  std::atomic<long long> comm_async[2];        // (local, global) likewise
  long long comm_local = 0, comm_global = 0;   // sts_grid_comm_counts
  size_t halo_bytes = 0;
  bool tma = true;                      // TMA pipelined kernels where eligible (sts_grid_set_tma)
  bool graphs = true;                   // CUDA-graph replay of PCG iteration pairs (sts_grid_set_graphs)
  bool pcg_merged = true;               // one-pass PCG iteration where eligible (sts_grid_set_pcg_merged)
  bool rkl2_dev = true;                 // RKL2 stages in deviation form where eligible (sts_grid_set_rkl2_deviation)
  bool halo_overlap = false;            // interior / boundary split of the passes (sts_grid_set_halo_overlap)
  cudaStream_t graph_stream = nullptr;  // non-blocking stream for capture / replay
  cudaEvent_t ev_c = nullptr;
  // per-kernel-class event timing (sts_grid_set_timing)
  bool timing = false;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> free_events;
  double acc_ms[STS_K_NCLASSES] = {};
  long long acc_n[STS_K_NCLASSES] = {};
  // host-array path: copy streams (H2D / D2H engines run concurrently with the compute
  // stream), staging buffers, and the events a caller's stream joins (sts_grid_join)
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  std::list<sts::StageBuf> stage_pool;  // (stable addresses: a call holds pointers into it)
  size_t stage_bytes = 0;
  unsigned long long stage_seq = 0;
  cudaEvent_t ev_h2d_last = nullptr, ev_d2h_last = nullptr;
  bool h2d_used = false, d2h_used = false;
  sts::CoefSlot slot[2];                // resident coefficients per mode (STS_MODE_ISO, STS_MODE_ANISO)
  cudaStream_t coef_stream = nullptr;   // binding work (face kappa, derived data, Gershgorin) of host bindings
  cudaEvent_t ev_coef = nullptr;        // after the last binding work on coef_stream
  cudaEvent_t ev_pos = nullptr;         // scratch: a position on the caller's stream
  double* d_gmax = nullptr;             // Gershgorin maximum (its own word: concurrent with PCG reductions)
  // executable PCG loop graphs still in flight: destroyed once their event has completed
  // (destroying an in-flight executable graph would wait for it)
  std::vector<std::pair<cudaGraphExec_t, cudaEvent_t>> retired_execs;
};

namespace sts {

// pointer to local plane il (-1..nl) of component c of a field (nullptr if absent)
__device__ __forceinline__ const double* plane_ptr(const FieldV& f, const Geo& G, int il, int c) {
  if (il < 0) return f.lo ? f.lo + (long long)c * G.plane : nullptr;
  if (il >= G.nl) return f.hi ? f.hi + (long long)c * G.plane : nullptr;
  return f.p + (long long)c * G.cstride + (long long)il * G.plane;
}

// 1/x for positive normal x (the Jacobi d of a PCG solve): the hardware approximation
// refined by two Newton steps (~1 ulp; no special-case branch, unlike 1.0 / x)
__device__ __forceinline__ double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

Geo slab_geo(const sts_grid* g, const Slab& s);

// CTA rasterisation of the 2.5-D stencil passes (1-D grid of nbx * nby * nchunks CTAs).
// rh == 0: phi tile fastest, then theta, then the r chunk (the plain 3-D grid order).
// rh > 0 : within a chunk the tiles go in bands of rh theta tiles, walked theta-first
// (down a column of the band, then one tile in phi), so theta neighbours start 1 CTA
// apart instead of nbx.  Measured on c4: it RAISES the DRAM reads of
// the merged anisotropic pass from 72 to 98 B/cell (phi neighbours, which share the
// partial 128 B lines at the box edges, move rh CTAs apart), so the passes use rh = 0.
struct Tile3 {
  int x, y, z;
};
__device__ __forceinline__ Tile3 raster_tile(long long lin, int nbx, int nby, int rh) {
  const long long tiles = (long long)nbx * nby;
  Tile3 t;
  t.z = (int)(lin / tiles);
  const int r = (int)(lin - (long long)t.z * tiles);
  if (rh <= 0) {
    t.y = r / nbx;
    t.x = r - t.y * nbx;
    return t;
  }
  const int band = r / (rh * nbx);
  const int hb = min(rh, nby - band * rh);
  const int q = r - band * rh * nbx;
  t.x = q / hb;
  t.y = band * rh + (q - t.x * hb);
  return t;
}

// current CUDA device ordinal (the handle's DeviceGuard has selected it)
inline int current_device() {
  int dev = 0;
  STS_CUDA(cudaGetDevice(&dev));
  return dev;
}

// Once per (call site, device): the >48 KB dynamic shared-memory opt-in of `kernel`.
// `done` is a per-call-site bit mask over device ordinals; setting the attribute twice
// from racing threads is harmless (idempotent), so a lock-free fetch_or suffices.
template <class K>
inline void ensure_smem_attr(K kernel, int bytes, std::atomic<unsigned long long>& done) {
  const unsigned long long bit = 1ull << (current_device() & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  STS_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.fetch_or(bit, std::memory_order_release);
}
double* ws_get(sts_grid* g, size_t bytes);  // scratch of at least `bytes`, reused across calls

// ----------------------------------------------------------------------------
// kernel launchers (stencil.cu)
// ----------------------------------------------------------------------------
// Epilogues of the fused stencil pass (one pass = operator + pointwise update)
enum Epi : int {
  EPI_F = 0,        // out = F(u)
  EPI_RKL2_FIRST,   // M0 = F(u0); y1 = u0 + c0*M0          (c0 = mu~_1 dt)
  EPI_RKL2_STAGE,   // yj = mu*u + nu*ym2 + (1-mu-nu)*y0 + c0*F(u) + c1*M0
  EPI_PCG_R0,       // r = dt*L u; d = 1/(wV - dt L_ii); x = u; z = r d; p = z; partials r.z, b.b d
  EPI_PCG_AP,       // y = wV p - dt L p; partial p.y
  EPI_PCG_S,        // p = z + beta pold; x += ax pold; y = wV p - dt L p; partial p.y  (fused S-pass)
  EPI_PCG_M,        // merged iteration: z = zold - ax wold; p = z + beta pold; x += ax pold;
                    // y = wV p - dt L p; w = d y; partials z.z/d, p.y, z.y, w.y
  EPI_RKL2_DSTAGE,  // deviation form D_j = Y_j - Y0: dj = mu*u + nu*dm2 + c0*F(u) + c1*M0 (no Y0 operand)
};

// PCG per-component scalars (device)
struct PcgScal {
  double rz, rz_old, pAp, alpha, beta, thresh;
  double ax;        // alpha of the last completed iteration, not yet applied to x (deferred x update;
                    // the merged iteration also applies it to z)
  // merged iteration: z is not stored -- the pass forms
  //   p_k = (1 + beta_k) p_{k-1} - bprev p_{k-2} - ax w_{k-1},  bprev = beta_{k-1}
  // -- and x is updated every other pass ("x in pairs"): the pass's x mode xm --
  // X_NORMAL: x_k = x_{k-1} + ax p_{k-1}; X_SKIP: x not touched;
  // X_CATCHUP: x_k = x_{k-2} + cxp p_{k-1} + cxz p_{k-2} (cxp = alpha_{k-1}, cxz = alpha_{k-2});
  // xmf / axp: what the final pass still owes x after the last iteration (X_FIN_*)
  double cxp, cxz, axp, bprev;
  int done, iters;
  int flags;        // PCG_BREAKDOWN (p.A p <= 0 or a non-finite scalar: A not SPD / NaN input), PCG_KMAX
  int kmax;         // iteration limit (set by launch_pcg_init): reaching it stops the component
  int xm, xmf;
  int nskip, ncatch;   // passes run with a skipped x update / a catch-up (instrumentation)
};
enum { X_NORMAL = 0, X_SKIP = 1, X_CATCHUP = 2 };
enum { X_FIN_ONE = 0, X_FIN_TWO = 4, X_FIN_PREV = 5 };   // final x += ax p_k | + axp p_{k-1} | axp p_{k-1} only
// the merged pass skips its x update (then the next one catches up) when beta_{k+1} is at
// least this (the catch-up reads p_{k-2} staged: no division, any beta >= 0 works)
#ifndef STS_X_SKIP_BETA   // (A-B: a value > 1 disables the skipped x updates)
#define STS_X_SKIP_BETA 0.0
#endif
constexpr double X_SKIP_BETA = STS_X_SKIP_BETA;
constexpr int PCG_BREAKDOWN = 1;
constexpr int PCG_KMAX = 2;
static_assert(sizeof(PcgScal) % sizeof(double) == 0, "PcgScal is published as doubles");

// fused final reduction of a PCG pass (pcg.cuh: fused_final_reduce)
struct FinRed {
  unsigned int* ticket = nullptr;   // zeroed counter; null: no fused reduction in this launch
  double* sums = nullptr;
  PcgScal* sc = nullptr;
  int ncomp = 1, nq = 1, phase = 0;
  long long ntot = 0;               // partial slots per row summed by the last CTA
  double rtol2 = 0.0;
};

struct EpiArgs {
  double* out = nullptr;       // primary output   [ncomp][nl][plane]
  double* out2 = nullptr;      // secondary output (M0 / x / ...)
  double* out3 = nullptr;      // (p)
  double* out4 = nullptr;      // (dinv)
  const double* ym2 = nullptr; // Y_{j-2}
  const double* y0 = nullptr;  // Y_0
  const double* m0 = nullptr;  // M0 = F(Y_0)
  double mu = 0, nu = 0, c0 = 0, c1 = 0, c2 = 0, dt = 0;
  double a0 = 1.0;             // EPI_RKL2_FIRST: out = a0*u + c0*F (deviation form: a0 = 0, D_1 = c0 M0)
  double* partials = nullptr;  // [value q][pstride]: per-CTA partial sums
  long long pstride = 0;       // stride between partial-value rows
  long long pbase = 0;         // this launch's first CTA slot
  const PcgScal* sc = nullptr; // per-component PCG scalars (skip components with done set)
  double* x = nullptr;         // EPI_PCG_S: iterate, updated in place (x += ax pold)
  int first = 0;               // EPI_PCG_S: first iteration (p = z, no pold, no x update)
  FinRed fin;                  // fused final reduction (last launch of a single-process pass)
  const double* dinv = nullptr;// EPI_PCG_M: the Jacobi inverse diagonal d (own cells)
};

struct StencilCall {
  int mode;                    // STS_MODE_ISO / STS_MODE_ANISO
  int ncomp;
  int epi;
  Geo geo;
  FieldV u, k1, k2, k3, b;
  FieldV u2;                   // EPI_PCG_S: pold (u = z, or r for the isotropic S-pass); EPI_PCG_M: wold
  FieldV u3;                   // isotropic EPI_PCG_S: the Jacobi inverse diagonal d (z = r d formed on the fly);
                               // EPI_PCG_M: pold
  const double* w;             // [nl][plane] or nullptr
  const double* ev = nullptr;  // ANISO fast path: vertex coefficients [3][nl+1][n2][n3+2] (see ev_pitch)
  int premul = 0;              // ISO EPI_PCG_M: k1.p, k2.p, k3.p, w hold the metric-folded K1, K2, K3, wV
                               // (launch_iso_premul); k1.lo / k1.hi stay the raw halo planes
  EpiArgs ea;
  int ib, ie;                  // local plane range [ib, ie)
};

// number of CTAs launch_stencil will use for (mode, epilogue) on a plane range
// (sizes the per-CTA partial-sum buffers)
int stencil_blocks(int mode, int epi, const Geo& geo, int ib, int ie);
void launch_stencil(const StencilCall& c, cudaStream_t st);

void launch_gershgorin(const StencilCall& c, unsigned long long* d_max, cudaStream_t st);
// e_a = sqrt(V_v kappa_v) b_{v,a} / (4 h_a) for vertex planes -1 .. nl-1 of a slab
void launch_vertex_coef(const Geo& G, FieldV b, FieldV k1, FieldV k2, FieldV k3, double* ev, cudaStream_t st);
bool stencil_uses_vertex_coef(int mode, int epi);
// padded vertex-coefficient layout: vertex (il+1/2, jv+1/2, kv+1/2), il = -1..nl-1,
// jv = -1..n2-1, kv = -1..n3-1, at
//   ev[a*ev_cstride + (il+1)*ev_plane + (jv+1)*ev_row + (kv+1)]
// (row jv = -1 is zeros, column kv = -1 is the periodic wrap copy of kv = n3-1, else
// zeros): every TMA box starts at a non-negative coordinate; the row pitch n3+2 keeps
// rows 16 B aligned for even n3
__host__ __device__ inline long long ev_row(int n3) { return (long long)n3 + 2; }
__host__ __device__ inline long long ev_plane(int n2, int n3) { return (long long)(n2 + 1) * ev_row(n3); }
__host__ __device__ inline long long ev_cstride(int nl, int n2, int n3) { return (long long)(nl + 1) * ev_plane(n2, n3); }

// TMA + mbarrier pipelined anisotropic stencil (stencil_tma.cu).  Returns false (and
// launches nothing) if the call is not eligible (odd n3, misaligned arrays, epilogue
// without a TMA variant); the caller then uses launch_stencil.
bool aniso_tma_eligible(const StencilCall& c);
bool launch_aniso_tma(const StencilCall& c, cudaStream_t st);
int aniso_tma_blocks(const StencilCall& c);
// r-chunk length of a 2.5-D march: minimises (waves of `slots` resident CTAs) x
// (planes a CTA streams = ic + extra), i.e. wave quantisation against the planes
// each extra chunk re-reads (extra = 2 for the vertex scheme, ~0.5 for 7-point)
inline int choose_chunk(long long tiles, int np, long long slots, double extra, int icmin, int icmax = 1 << 30) {
  const int hi = std::max(1, std::min(np, icmax));
  int best = hi;
  double bc = 1e300;
  for (int ic = std::max(1, std::min(icmin, hi)); ic <= hi; ++ic) {
    const long long nch = (np + ic - 1) / ic;
    if (ic != hi && (long long)(np + nch - 1) / nch != ic) continue;   // only distinct chunkings
    const long long ctas = tiles * nch;
    const double cost = (double)((ctas + slots - 1) / slots) * (ic + extra);
    if (cost < bc * (1 - 1e-9)) {
      bc = cost;
      best = ic;
    }
  }
  return best;
}

// the isotropic (ncomp <= 3) counterpart (stencil_tma_iso.cu)
bool iso_tma_eligible(const StencilCall& c);
bool launch_iso_tma(const StencilCall& c, cudaStream_t st);
int iso_tma_blocks(const StencilCall& c);
// PCG pointwise passes of the restructured iteration (aux.cu)
// pnew = z + beta pold (pold unused if first); x += ax pold (not if first)
void launch_pcg_pnew(int ncomp, long long n, long long cstride, double* pnew, const double* z, const double* pold,
                     double* x, const PcgScal* sc, int first, cudaStream_t st);
// r -= alpha y; z = r d; partial r.z  (fin.ticket set: the last CTA also finishes the reduction);
// returns the number of CTAs (partial slots per row) launched
int launch_pcg_rupdate(int ncomp, long long n, long long cstride, double* r, double* z, const double* y,
                        const double* d, const PcgScal* sc, double* partials, long long pstride,
                        const FinRed& fin, cudaStream_t st);
// the final x update (PcgScal::xmf): p_k in pk[k % 4]
void launch_pcg_xfinal(int ncomp, long long n, long long cstride, double* x, const double* const pk[4],
                       const PcgScal* sc, cudaStream_t st);

// pointwise / auxiliary kernels (aux.cu)
// metric-folded isotropic face coefficients and wV of one slab (merged PCG pass)
void launch_iso_premul(const Geo& G, const double* k1, const double* k2, const double* k3, const double* w,
                       double* K1, double* K2, double* K3, double* WV, cudaStream_t st);
void launch_face_kappa(const Geo& geo, FieldV T, double* k1, double* k2, double* k3, double kappa0,
                       double T_cut, double fc_r0, double fc_w, const double* x1f_d, const double* x1c_d,
                       cudaStream_t st);

enum PcgPhase { PH_NONE = 0, PH_R0 = 1, PH_AP = 2, PH_RZ = 3, PH_M = 4 };
constexpr int PW_BLOCKS = 148 * 8;   // grid of the pointwise PCG kernels
// sums[c*nq + q] = sum_b partials[(c*nq+q)*pstride + b], then the phase's scalar update
// (l2 [R2_MAXBLOCKS x 4 MAXC] and a zeroed ticket: the two-level multi-block reduction)
constexpr int R2_MAXBLOCKS = 64;
void launch_pcg_reduce(const double* partials, long long pstride, int nblocks, int ncomp, int nq,
                       double* sums, int phase, PcgScal* sc, double rtol2, cudaStream_t st,
                       double* l2 = nullptr, unsigned* ticket = nullptr);
void launch_pcg_scalar(const double* sums, int ncomp, int nq, int phase, PcgScal* sc, double rtol2,
                       cudaStream_t st);
// per-solve PCG scalar initialisation (iteration limit, flags, loop body counter)
void launch_pcg_init(PcgScal* sc, int ncomp, int kmax, int* body_count, cudaStream_t st);
// condition kernel of the device-driven PCG loop (sets the WHILE node's handle)
void launch_pcg_continue(cudaGraphConditionalHandle h, const PcgScal* sc, int ncomp, int* body_count, bool count,
                         cudaStream_t st);
// copy n doubles to mapped pinned host memory with SM stores (no copy engine)
void launch_publish(const double* src, int n, double* dst_mapped, cudaStream_t st);

}  // namespace sts
