/*
 * sts_b200.h — C ABI of the B200-native parabolic-advance library
 * (libsts_b200.so): RKL2 super time-stepping and backward Euler solved by
 * point-Jacobi preconditioned conjugate gradient, for the anisotropic Spitzer
 * conduction and the artificial-viscosity operators of
 *   Caplan, Mikic, Linker, Lionello, arxiv 1610.01265 ("PAPER.md").
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All floating point is IEEE binary64 (double).
 *  - A grid is logically rectangular, n1 x n2 x n3 cells, (r, theta, phi) or
 *    (x, y, z); a field is a C-contiguous array [n1][n2][n3] (n3 = phi fastest).
 *    When the grid is an r-slab of a distributed grid (sts_comm_init), arrays
 *    hold the LOCAL planes only: [nl][n2][n3].
 *  - Vector fields with ncomp components are stacked [ncomp][nl][n2][n3].
 *  - Face fields use the "+ face" convention: k1[i][j][k] lives on the face
 *    (i+1/2, j, k), k2 on (i, j+1/2, k), k3 on (i, j, k+1/2); entries on faces
 *    that leave the domain are ignored (zero-flux walls, PAPER.md:193 applies
 *    boundary conditions matrix-free).  For periodic dim 3, k3[..][n3-1] is the
 *    wrap face between k = n3-1 and k = 0.
 *  - The unit field b is [3][nl][n2][n3] (components along the grid's own unit
 *    vectors).  w (viscosity: rho) is [nl][n2][n3]; NULL means w = 1.
 *  - Array arguments may be DEVICE pointers (no copy) or HOST pointers.  Host
 *    arrays are staged through device buffers the handle owns: uploads run on the
 *    handle's own host-to-device copy stream and downloads on its device-to-host
 *    copy stream, so the copies of one call overlap the computation of the calls
 *    enqueued before and after it; `stream` waits only for the call's own inputs.
 *      PINNED (page-locked) host arrays make the call asynchronous, like
 *      cudaMemcpyAsync: it returns once the work is enqueued; the caller must not
 *      modify its inputs nor read its outputs before sts_grid_join(g, s) has been
 *      issued on a stream s and s has been synchronized (or sts_grid_synchronize).
 *      PAGEABLE host arrays make the call synchronous: it returns with the outputs
 *      written back.
 *    The caller owns every array it passes; the library never frees caller
 *    pointers, and retains DEVICE coefficient pointers only while they are bound
 *    (sts_grid_bind_coeffs).
 *  - Coefficient arrays (k1, k2, k3, b, w) all NULL: the call uses the coefficients
 *    bound to its mode (sts_grid_bind_coeffs, sts_face_kappa_spitzer with NULL
 *    outputs), and the data the library derives from them -- the frozen vertex
 *    coefficients of STS_MODE_ANISO, the metric-folded face coefficients of the
 *    merged isotropic PCG pass, the Gershgorin bound -- is built once per binding
 *    instead of once per call.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Entry points
 *    that return host-visible values (dt, iteration counts) synchronise the
 *    stream; the others are asynchronous.
 *  - A grid handle owns scratch, halo buffers and reduction counters: calls on one
 *    handle must not run concurrently (from several host threads or on several
 *    streams at once); use one handle per concurrent stream.
 *  - Return value: STS_OK (0) or a negative STS_ERR_* code;
 *    sts_last_error() returns a thread-local message for the last failure.
 *    Calls never abort the process.
 *
 * Operator (Eq. (1), :173 and :181 boxed terms; R2):
 *    F(u) = (L u) / (w V),  (L u)_i = -dE/du_i,
 *    ISO  : E = 1/2 sum_faces kappa_f A_f/h_f (u_R - u_L)^2                 (7-point)
 *    ANISO: E = 1/2 sum_vertices V_v kappa_v (b_v . g_v)^2                 (27-point)
 *  with g_v the vertex gradient (mean of the four differences per direction),
 *  b_v the mean of the 8 surrounding cell b, kappa_v the mean of the 12 faces
 *  around the vertex and V_v the mean of the 8 cell volumes.
 */
#ifndef STS_B200_H
#define STS_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sts_grid sts_grid;

#define STS_OK 0
#define STS_ERR_ARG (-1)          /* invalid argument (size, pointer, mode)          */
#define STS_ERR_CUDA (-2)         /* a CUDA runtime call failed                     */
#define STS_ERR_NCCL (-3)         /* an NCCL call failed                            */
#define STS_ERR_NOT_CONVERGED (-4)/* PCG hit kmax; outputs hold the last iterate    */
#define STS_ERR_STATE (-5)        /* call not valid in the grid's current state     */
#define STS_ERR_ALLOC (-6)        /* device allocation failed                       */
#define STS_ERR_BREAKDOWN (-7)    /* PCG breakdown: p.A p <= 0 or a non-finite scalar
                                     (A not SPD, or NaN / inf input); outputs hold the
                                     last iterate                                   */

#define STS_GEOM_CARTESIAN 0
#define STS_GEOM_SPHERICAL 1

#define STS_MODE_ISO 0            /* div(kappa grad u) / w, ncomp 1..3 (viscosity, heat) */
#define STS_MODE_ANISO 1          /* div(kappa b b.grad u), ncomp 1 (Spitzer conduction) */

#define STS_NCCL_UID_BYTES 128

/* Library version (major*10000 + minor*100 + patch). */
int sts_version(void);

/* Message describing the last error on the calling thread ("" if none). */
const char* sts_last_error(void);

/*
 * sts_grid_create — build a grid handle and its device-resident cell metrics
 * (volumes, face area / centre-distance factors; R1).
 *  geom          STS_GEOM_CARTESIAN or STS_GEOM_SPHERICAL
 *  n1, n2, n3    GLOBAL cell counts (>= 1 each)
 *  x1f[n1+1], x1c[n1]   global face / centre coordinates of dim 1 (r or x), host
 *  x2f[n2+1], x2c[n2]   dim 2 (theta or y), host
 *  x3f[n3+1], x3c[n3]   dim 3 (phi or z), host; if periodic3, the period is
 *                       x3f[n3] - x3f[0]
 *  periodic3     nonzero: dim 3 is periodic
 *  i0, nl        this handle's r-slab: global planes [i0, i0+nl); (0, n1) = whole grid
 *  n_virtual     >= 1. With n_virtual > 1 (whole grid only) the grid is processed
 *                as n_virtual r-slabs inside this process, each reading its
 *                neighbours' boundary planes through halo buffers exactly as the
 *                multi-GPU path does — a single-GPU emulation of the decomposition.
 *  device        CUDA device ordinal the handle's memory lives on
 * Ownership: the coordinates are copied; free the handle with sts_grid_destroy.
 * Errors: STS_ERR_ARG for non-monotone coordinates or bad sizes.
 */
int sts_grid_create(sts_grid** out, int geom, int n1, int n2, int n3,
                    const double* x1f, const double* x1c,
                    const double* x2f, const double* x2c,
                    const double* x3f, const double* x3c,
                    int periodic3, int i0, int nl, int n_virtual, int device);

/* Release every device buffer, stream, event and communicator of the handle. */
int sts_grid_destroy(sts_grid* g);

/* Bytes of device memory currently held by the handle (scratch, halos, host-array
   staging buffers, resident coefficient copies and their derived data). */
int sts_grid_workspace_bytes(const sts_grid* g, size_t* bytes);

/* Number of kernels this handle has launched since creation (instrumentation). */
int sts_grid_kernel_launches(const sts_grid* g, long long* count);

/*
 * Merged-PCG x-update profile of the most recent SYNCHRONOUS be_pcg_solve on the
 * handle (instrumentation; DESIGN.md §5.3 "x in pairs"): per component, the passes
 * that skipped the x update and the passes that caught it up (the others updated x
 * every pass).  ncomp 1..3.
 */
int sts_grid_pcg_xmodes(const sts_grid* g, int ncomp, int* skipped, int* caught_up);

/*
 * Communication profile (Sec. 2.4 and the boxed terms of Figs. 1-2):
 * `local` counts neighbour (halo) exchange events -- one per operator application
 * that reads across slab boundaries -- and `global` counts all-rank reductions
 * (PCG dot products; the convergence test rides on the r.z reduction).  Counted
 * for distributed (NCCL) and virtual-slab grids alike, never for a single slab.
 * RKL2: local = s per super-step, global = 0.  BE+PCG: local = iterations + 1,
 * global = 2 iterations + 1.
 */
int sts_grid_comm_counts(const sts_grid* g, long long* local, long long* global_);

/*
 * Per-kernel-class device timing (instrumentation used by bench.py for the
 * roofline): when enabled, every launch is bracketed by cudaEventRecord on the
 * stream it is launched on.  sts_grid_timing synchronises the recorded events
 * and returns the launch count and summed device milliseconds of one class
 * since the last sts_grid_timing_reset.  Classes:
 */
#define STS_K_FACE_KAPPA 0
#define STS_K_ANISO_F 1
#define STS_K_ANISO_RKL2_FIRST 2
#define STS_K_ANISO_RKL2_STAGE 3
#define STS_K_ANISO_PCG_R0 4
#define STS_K_ANISO_PCG_AP 5
#define STS_K_ANISO_GERSH 6
#define STS_K_ISO_F 7
#define STS_K_ISO_RKL2_FIRST 8
#define STS_K_ISO_RKL2_STAGE 9
#define STS_K_ISO_PCG_R0 10
#define STS_K_ISO_PCG_AP 11
#define STS_K_ISO_GERSH 12
#define STS_K_PCG_UPDATE 13
#define STS_K_PCG_PUPDATE 14
#define STS_K_PCG_REDUCE 15
#define STS_K_HALO 16
#define STS_K_VERTEX_COEF 17
#define STS_K_ANISO_PCG_S 18     /* fused PCG S-pass (p update + x update + A p), TMA path   */
#define STS_K_PCG_XFINAL 19      /* final deferred x += alpha p after convergence            */
#define STS_K_ISO_PCG_S 20       /* fused PCG S-pass of the isotropic operator, TMA path      */
#define STS_K_ANISO_PCG_M 21     /* one-pass (merged) PCG iteration, anisotropic, TMA path    */
#define STS_K_ISO_PCG_M 22       /* one-pass (merged) PCG iteration, isotropic, TMA path      */
#define STS_K_ANISO_RKL2_DSTAGE 23  /* RKL2 stage in deviation form, anisotropic, TMA path */
#define STS_K_ISO_RKL2_DSTAGE 24    /* RKL2 stage in deviation form, isotropic, TMA path    */
#define STS_K_NCLASSES 25
int sts_grid_set_timing(sts_grid* g, int enable);

/*
 * Kernel-path selection (testing / A-B measurement): enable != 0 (the default)
 * lets the anisotropic RKL2 stages and PCG S-passes use the TMA + mbarrier
 * pipelined kernels where eligible (n3 even, 16 B aligned arrays); 0 forces the
 * cp.async kernels everywhere.  Results agree to rounding either way.
 */
int sts_grid_set_tma(sts_grid* g, int enable);

/*
 * enable != 0 (the default): single-process PCG solves run iterations k >= 4 as the
 * body (one iteration pair) of a device-side WHILE loop in a CUDA graph; 0 launches
 * every kernel directly from a host-polled loop.  Graphs are never used while
 * per-launch timing is on or with an NCCL communicator.  The environment variable
 * STS_PCG_HOST_LOOP=1, read at sts_grid_create, selects 0 (profilers such as ncu
 * cannot profile the kernel nodes of a graph with conditional nodes).
 */
int sts_grid_set_graphs(sts_grid* g, int enable);

/*
 * PCG iteration structure of be_pcg_solve (A-B measurement / testing).
 * enable != 0 (the default): where the TMA kernels are eligible, ONE fused pass
 * per iteration (DESIGN.md §5.3 "merged PCG"): it forms z_k = z_{k-1} -
 * alpha_{k-1} d y_{k-1} and p_k = z_k + beta_k p_{k-1} on the fly, applies A,
 * and reduces r_k.z_k, p_k.A p_k, z_k.A p_k and (d A p_k).A p_k together; the
 * next r.z follows from the expansion of (r - alpha y).d(r - alpha y), so one
 * global reduction per iteration replaces Fig. 1's two.  The
 * iterates equal Fig. 1's in exact arithmetic.  0: the two-pass S / U iteration.
 */
int sts_grid_set_pcg_merged(sts_grid* g, int enable);

/*
 * RKL2 stage form (A-B measurement / testing).  enable != 0 (the default): where
 * the TMA kernels are eligible, stages 2..s-1 advance the deviation D_j = Y_j - Y0,
 *   D_j = mu_j D_{j-1} + nu_j D_{j-2} + mu~_j dt M D_{j-1} + (mu~_j + gamma~_j) dt M Y0,
 * D_0 = 0, D_1 = mu~_1 dt M Y0, and the last stage returns Y0 + D_s -- Fig. 2
 * rewritten with M linear, so an intermediate stage streams
 * three solution-sized arrays instead of four.  0: Fig. 2 as printed.
 */
int sts_grid_set_rkl2_deviation(sts_grid* g, int enable);
/*
 * Halo schedule of decomposed grids (virtual slabs or NCCL ranks).
 * enable != 0: every stencil pass computes the interior planes while the neighbour
 * planes are exchanged, then the two boundary planes in their own one-plane launches;
 * 0 (the default): the pass waits for the exchange and is ONE launch per slab (measured
 * faster on B200: a one-plane launch of the TMA pipeline costs more than the exchange).
 */
int sts_grid_set_halo_overlap(sts_grid* g, int enable);
int sts_grid_timing_reset(sts_grid* g);
int sts_grid_timing(sts_grid* g, int kind, long long* count, double* ms);

/*
 * Multi-GPU (one process per GPU, r-slab per rank).
 * sts_nccl_unique_id writes STS_NCCL_UID_BYTES bytes into `out` (rank 0 calls
 * it; the caller broadcasts the bytes, e.g. with torch.distributed).
 * sts_comm_init creates the handle's NCCL communicator; the slab of `rank`
 * must be the rank-th slab in r order (rank 0 holds r_min).  Neighbour
 * exchanges (one theta x phi plane per side) use ncclSend/ncclRecv on an
 * internal communication stream, overlapped with the interior planes of every
 * stencil pass; PCG dot products use ncclAllReduce (one per merged iteration).
 * With a communicator, be_pcg_solve polls convergence from the host in batches
 * sized from the observed convergence rate, and replays iterations k >= 4 as one
 * captured CUDA graph per iteration pair (NCCL calls inside the graph).
 * nranks = 1 is allowed (a one-rank communicator: the NCCL reduction path on one GPU).
 */
int sts_nccl_unique_id(void* out, size_t nbytes);
int sts_comm_init(sts_grid* g, int nranks, int rank, const void* uid, size_t nbytes);

/*
 * Resident coefficients.  sts_grid_bind_coeffs binds the coefficient arrays of one
 * operator mode to the handle (one binding per mode: conduction and viscosity can be
 * resident together).  Each non-NULL array replaces the mode's current one; NULL keeps
 * it.  DEVICE arrays are referenced (the caller keeps them allocated and unchanged
 * while bound); HOST arrays are uploaded into library-owned device copies on the H2D
 * copy stream (two copies per array, used in turn, so an upload overlaps the work still
 * reading the previous binding).  b is STS_MODE_ANISO only; w NULL means w = 1.
 * Calls that pass k1 = k2 = k3 = b = w = NULL then use the binding (see "Coefficient
 * arrays" above).  sts_grid_unbind_coeffs synchronizes the device and releases the
 * mode's binding and library-owned copies.
 * Errors: STS_ERR_ARG for a bad mode; STS_ERR_STATE when a call selects a binding that
 * lacks an array it needs.
 */
int sts_grid_bind_coeffs(sts_grid* g, int mode, const double* k1, const double* k2, const double* k3,
                         const double* b, const double* w, void* stream);
int sts_grid_unbind_coeffs(sts_grid* g, int mode);

/*
 * sts_grid_join makes `stream` wait for every copy the handle has enqueued so far on its
 * copy streams (the uploads and the result downloads of host arrays): after it, work on
 * `stream` -- and a synchronization of `stream` -- also covers the host outputs.
 * sts_grid_synchronize blocks until all of the handle's internal streams are idle.
 */
int sts_grid_join(sts_grid* g, void* stream);
int sts_grid_synchronize(sts_grid* g);

/*
 * A3 — lagged Spitzer face diffusivity (DESIGN R3)
 *   k_d[f] = kappa0 * f_c(r_f) * beta_Tcut(Tf) * Tf^(5/2),  Tf = (T_L + T_R)/2,
 *   beta_Tcut(T) = (T/T_cut)^(5/2) if T < T_cut else 1  (T_cut <= 0: beta = 1),
 *   f_c(r) = 0.5 (1 - tanh((r - fc_r0)/fc_w))            (fc_w <= 0: f_c = 1).
 *  T[nl][n2][n3] (> 0) in; k1, k2, k3 [nl][n2][n3] out (faces leaving the
 *  domain are written as 0).  Distributed grids exchange T's boundary planes.
 *  k1 = k2 = k3 = NULL: the face diffusivities are written into library-owned device
 *  arrays and bound as the STS_MODE_ANISO coefficients (the binding's b is kept).
 */
int sts_face_kappa_spitzer(sts_grid* g, const double* T, double* k1, double* k2, double* k3,
                           double kappa0, double T_cut, double fc_r0, double fc_w,
                           void* stream);

/*
 * A1/A2 — out = F(u) (Eq. 1), component-wise for ncomp > 1.
 *  mode   STS_MODE_ISO (ncomp 1..3, b ignored) or STS_MODE_ANISO (ncomp == 1, b required)
 *  u, out [ncomp][nl][n2][n3]; must not alias.
 */
int sts_op_apply(sts_grid* g, int mode, int ncomp, const double* u, double* out,
                 const double* k1, const double* k2, const double* k3,
                 const double* b, const double* w, void* stream);

/*
 * A4 — explicit Euler limit by the Gershgorin bound of Appendix B
 * (PAPER.md:512 dt = 2/|lambda|_max, :536 |lambda|_max <= max_j sum_i |M_ji|)
 * over the whole (distributed) grid.  *dt_out (host) = +inf if M = 0.
 * Synchronises `stream`.
 */
int sts_dt_euler(sts_grid* g, int mode, const double* k1, const double* k2, const double* k3,
                 const double* b, const double* w, double* dt_out, void* stream);

/*
 * A5 — RKL2 stage count (Eq. 5, DESIGN R5):
 *   s = max(2, ceil((sqrt(9 + 16 dt/dt_exp) - 1)/2)), +1 if force_odd and s even.
 * Returns s (>= 2), or STS_ERR_ARG if dt < 0 or dt_exp <= 0 or non-finite.
 */
int rkl2_num_stages(double dt, double dt_exp, int force_odd);

/*
 * A6 — one RKL2 super-step of du/dt = F(u) (Fig. 2):
 *   Y0 = u0;  M0 = F(Y0);  Y1 = Y0 + mu~_1 dt M0;
 *   Yj = mu_j Y_{j-1} + nu_j Y_{j-2} + (1 - mu_j - nu_j) Y0
 *        + mu~_j dt F(Y_{j-1}) + gamma~_j dt M0,        j = 2..s  (gamma~_j = (b_{j-1}-1) mu~_j)
 *   u1 = Ys.
 * Each stage is ONE fused kernel pass (operator + recurrence).
 *  u0, u1 [ncomp][nl][n2][n3]; u1 may alias u0 (in-place advance).
 *  s >= 2 (from rkl2_num_stages); dt > 0.
 */
int rkl2_advance(sts_grid* g, int mode, int ncomp, const double* u0, double* u1,
                 const double* k1, const double* k2, const double* k3,
                 const double* b, const double* w, double dt, int s, void* stream);

/*
 * A8 — RKL2 with an explicit-Euler prefix and RKL2 sub-cycling, the high-mode
 * remedies PAPER.md:341 (Sec. 6) reports ("sub-cycling explicit Euler steps for ~1/4
 * of the time-step and completing the remainder of the step with RKL2", "sub-cycling
 * the RKL2 method within each large time-step"):
 *   n_euler explicit Euler steps  u <- u + dte F(u),  dte = euler_frac dt / n_euler,
 *   then n_sub RKL2 super-steps of dtr = (1 - euler_frac) dt / n_sub, each with
 *   s = rkl2_num_stages(dtr, dt_exp, 0) stages (Fig. 2).
 *  n_euler < 0 selects the default ceil(euler_frac dt / (dt_exp/2)) (0 if euler_frac = 0):
 *  sub-steps of at most dt_exp/2, the step 1 + (dt_exp/2)(-2/dt_exp) = 0 that annihilates
 *  the highest mode (DESIGN R11).
 *  Requirements: 0 <= euler_frac < 1; n_euler > 0 exactly when euler_frac > 0;
 *  dte <= dt_exp (explicit stability); n_sub >= 1.
 *  stages_out: host int[2] = {n_euler, s} (may be NULL).  u1 may alias u0.
 *  euler_frac = 0, n_sub = 1 is exactly rkl2_advance with s = rkl2_num_stages(dt, dt_exp).
 */
int rkl2_advance_hybrid(sts_grid* g, int mode, int ncomp, const double* u0, double* u1,
                        const double* k1, const double* k2, const double* k3,
                        const double* b, const double* w, double dt, double dt_exp,
                        double euler_frac, int n_euler, int n_sub, int* stages_out, void* stream);

/*
 * A7 — one backward-Euler step (Eqs. 2-4) solved by
 * point-Jacobi PCG (Fig. 1, PC1 of :468-470; DESIGN R7, R8):
 *   (wV - dt L) x = wV un,  x0 = un,  z = r / diag(A),
 *   stop when r.z <= rtol^2 (b . P^-1 b), independently per component.
 *  un, un1 [ncomp][nl][n2][n3] (may alias); iters_out: host int[ncomp] receives
 *  the A p products each component used (may be NULL).  kmax >= 1.
 *  Returns STS_ERR_NOT_CONVERGED (un1 = last iterate) if a component hits kmax,
 *  STS_ERR_BREAKDOWN if a component's p.A p is not positive or a PCG scalar is not
 *  finite (A not SPD, NaN / inf in the inputs; that component stops, un1 = last iterate).
 *  Synchronises `stream` before returning.  Single-process solves run the
 *  iteration loop on the device (a conditional WHILE node of a CUDA graph, one
 *  iteration pair per trip, the condition set by a kernel from the device-side
 *  convergence flags), so the host never polls; with per-launch timing, graphs
 *  disabled or an NCCL communicator the host polls the flags once per batch of
 *  iterations, the batch sized from the observed convergence rate so that at most
 *  one or two no-op iterations follow convergence.  By default each iteration is
 *  one fused stencil pass and one reduction (sts_grid_set_pcg_merged; the
 *  convergence test uses r.z of the next iterate from the expansion of
 *  (r - alpha y).d(r - alpha y), so the count can differ from Fig. 1's by one at
 *  a tie).
 */
int be_pcg_solve(sts_grid* g, int mode, int ncomp, const double* un, double* un1,
                 const double* k1, const double* k2, const double* k3,
                 const double* b, const double* w, double dt, double rtol, int kmax,
                 int* iters_out, void* stream);

/*
 * A7, asynchronous — be_pcg_solve without waiting for the solve: where the loop runs on
 * the device (single process, graphs enabled, per-launch timing off) and no array is in
 * pageable host memory, the call returns once the solve is enqueued; iters_out[ncomp]
 * and *status_out (STS_OK, STS_ERR_NOT_CONVERGED or STS_ERR_BREAKDOWN) are written by the
 * host when `stream` reaches the end of the solve, so both must stay valid until then
 * (either may be NULL).  Otherwise it behaves like be_pcg_solve and writes both before
 * returning.  The return value reports enqueue-time errors only (argument, CUDA, state).
 */
int be_pcg_solve_async(sts_grid* g, int mode, int ncomp, const double* un, double* un1,
                       const double* k1, const double* k2, const double* k3,
                       const double* b, const double* w, double dt, double rtol, int kmax,
                       int* iters_out, int* status_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STS_B200_H */
