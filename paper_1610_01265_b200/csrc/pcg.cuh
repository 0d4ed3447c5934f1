// PCG scalar recurrences and the fused ("last CTA") final reduction, shared by the
// pointwise and the stencil kernels.  Device code only; product path.
#pragma once

#include "sts_common.cuh"

namespace sts {

// stop the component: A is not SPD (p.A p <= 0) or a scalar is not finite (NaN / inf
// input); the host reports STS_ERR_BREAKDOWN, x holds the last iterate
__device__ inline void pcg_breakdown(PcgScal& s) {
  s.done = 1;
  s.flags |= PCG_BREAKDOWN;
  // (a skipped pass still owes x its alpha_{k-1} p_{k-1}: the final pass adds it)
  if (s.xm == X_SKIP) {
    s.xmf = X_FIN_PREV;
    s.axp = s.ax;
  } else {
    s.xmf = X_FIN_ONE;
  }
  s.ax = 0.0;
}

// the iteration limit: a component that has run kmax iterations without converging
// stops (its last alpha still reaches x through the final pass); the host reports
// STS_ERR_NOT_CONVERGED
__device__ inline void pcg_kmax(PcgScal& s) {
  if (!s.done && s.iters >= s.kmax) {
    s.done = 1;
    s.flags |= PCG_KMAX;
  }
}

// scalar recurrences of Fig. 1 (one thread per component)
__device__ inline void pcg_phase(const double* sums, int c, int nq, int phase, PcgScal* sc, double rtol2) {
  PcgScal& s = sc[c];
  if (phase == PH_R0) {
    s.rz = sums[c * nq + 0];
    s.thresh = rtol2 * sums[c * nq + 1];
    s.iters = 0;
    s.flags = 0;                           // (kmax was set by launch_pcg_init)
    s.xm = X_NORMAL;
    s.xmf = X_FIN_ONE;
    s.cxp = s.cxz = s.axp = s.bprev = 0.0;
    s.nskip = s.ncatch = 0;
    s.done = (s.rz <= s.thresh) ? 1 : 0;   // DESIGN R8: already converged -> 0 iterations
    s.beta = 0.0;
    s.ax = 0.0;
    // r.P^-1 r and b.P^-1 b are >= 0 for an SPD Jacobi P (A_ii > 0); NaN fails both tests
    if (!(s.rz >= 0.0) || !(s.thresh >= 0.0) || !isfinite(s.rz) || !isfinite(s.thresh)) pcg_breakdown(s);
  } else if (phase == PH_AP) {
    if (s.done) return;
    s.pAp = sums[c * nq];
    if (!(s.pAp > 0.0) || !isfinite(s.pAp)) return pcg_breakdown(s);
    s.alpha = s.rz / s.pAp;                // alpha_k = r_r / (p_k . y_k)
  } else if (phase == PH_RZ) {
    if (s.done) return;
    s.rz_old = s.rz;
    s.rz = sums[c * nq];                   // r_r = r_{k+1} . z_{k+1}
    s.iters += 1;
    s.ax = s.alpha;                        // x_{k+1} = x_k + alpha_k p_k, applied by the next p pass / final pass
    if (s.rz <= s.thresh) s.done = 1;      // check r_r for convergence
    else s.beta = s.rz / s.rz_old;         // beta_k = r_r / r_old
    pcg_kmax(s);
  } else if (phase == PH_M) {
    // merged iteration k (one pass, one reduction): sums of the pass
    // are r_k.z_k (= z_k^2 / d), p_k.y_k, z_k.y_k and (d y_k).y_k with y_k = A p_k.
    // alpha_k as in Fig. 1; r_{k+1} = r_k - alpha_k y_k gives
    //   r_{k+1}.z_{k+1} = r_k.z_k - 2 alpha_k z_k.y_k + alpha_k^2 (d y_k).y_k
    // (exact in exact arithmetic; r_k.z_k is the pass's own sum, so rounding does
    // not accumulate across iterations).  The pass forms z_{k+1} = z_k - alpha_k d y_k.
    if (s.done) return;
    const int mk = s.xm;                   // x mode of the pass that just ran
    const double rz = sums[c * nq + 0];
    if (rz <= s.thresh) {
      // the pass's own r_k.z_k meets the test: reached only after an extrapolated value
      // below its own rounding (below); x_k is complete unless the pass skipped x
      s.done = 1;
      if (mk == X_SKIP) {
        s.xmf = X_FIN_PREV;
        s.axp = s.ax;
      } else {
        s.xmf = X_FIN_ONE;
      }
      s.ax = 0.0;
      s.rz = rz;
      return;
    }
    s.pAp = sums[c * nq + 1];
    if (!(s.pAp > 0.0) || !isfinite(s.pAp) || !isfinite(rz)) return pcg_breakdown(s);
    const double a_prev = s.ax;            // alpha_{k-1} (used by this pass)
    s.bprev = s.beta;                      // beta_k: the next pass's p_{k-1} coefficient
    s.alpha = rz / s.pAp;
    s.rz_old = rz;
    s.rz = rz - 2.0 * s.alpha * sums[c * nq + 2] + s.alpha * s.alpha * sums[c * nq + 3];
    s.iters += 1;
    s.ax = s.alpha;                        // x_{k+1} = x_k + alpha_k p_k (next pass / final pass)
    // The expansion cancels to ~4 eps r_k.z_k.  A negative value means the true one is
    // below that rounding: it decides convergence only if the rounding itself is under
    // the threshold; otherwise restart the direction (beta = 0) and let the next pass's
    // own r.z sum decide (the test above).
    const double fuzz = 4.0 * 2.220446049250313e-16 * rz;
    if (s.rz < 0.0 && fuzz > s.thresh) s.beta = 0.0;
    else if (s.rz <= s.thresh) s.done = 1;
    else s.beta = s.rz / rz;               // beta_{k+1} = r_{k+1}.z_{k+1} / r_k.z_k
    pcg_kmax(s);
    // x in pairs: after a skipped pass the next one catches up; otherwise the next pass
    // may skip if the catch-up after it divides by a safe beta_{k+1}
    if (s.done) {
      if (mk == X_SKIP) {                  // x still owes alpha_{k-1} p_{k-1} + alpha_k p_k
        s.xmf = X_FIN_TWO;
        s.axp = a_prev;
      } else {
        s.xmf = X_FIN_ONE;
      }
    } else if (mk == X_SKIP) {
      s.xm = X_CATCHUP;
      s.cxp = s.alpha;                     // x_{k+1} = x_{k-1} + alpha_k p_k + alpha_{k-1} p_{k-1}
      s.cxz = a_prev;
      s.ncatch += 1;
    } else if (s.beta >= X_SKIP_BETA) {
      s.xm = X_SKIP;
      s.nskip += 1;
    } else {
      s.xm = X_NORMAL;
      s.cxp = s.alpha;
      s.cxz = 0.0;
    }
  }
}


// Fused final reduction of a PCG pass (single process: no all-reduce between the
// partial sums and the scalar update).  Every CTA of the LAST launch of the pass
// takes a ticket after its partials are visible; the CTA drawing the last ticket
// sums all `ntot` partial slots of every row in a fixed order (deterministic,
// independent of which CTA is last), runs the scalar phase and re-arms the ticket.
// The earlier launches of the pass (interior / boundary planes, virtual slabs) ran
// before this one on the same stream, so their partials are complete.
//   nthr threads participate; sync() is the barrier among them.
template <class Sync>
__device__ inline void fused_final_reduce(const FinRed& f, const double* partials, long long pstride,
                                          unsigned long long nblk, int tid, int nthr, double* red /*[4 MAXC][32]*/,
                                          unsigned* s_flag, Sync sync) {
  constexpr int MAXROWS = 4 * MAXC;
  __threadfence();
  sync();
  if (tid == 0) *s_flag = (atomicAdd(f.ticket, 1u) == (unsigned)(nblk - 1)) ? 1u : 0u;
  sync();
  if (*s_flag == 0u) return;
  __threadfence();
  const int lane = tid & 31, wid = tid >> 5, nw = (nthr + 31) >> 5;
  const int nrows = f.ncomp * f.nq;
  // every row's loads in flight at once (one strided pass over the slots), then a
  // fixed-order combine: deterministic, independent of which CTA is last
  double v[MAXROWS];
#pragma unroll
  for (int r = 0; r < MAXROWS; ++r) v[r] = 0.0;
  for (long long b = tid; b < f.ntot; b += nthr) {
#pragma unroll
    for (int r = 0; r < MAXROWS; ++r)
      if (r < nrows) v[r] += __ldcg(partials + r * pstride + b);
  }
#pragma unroll
  for (int r = 0; r < MAXROWS; ++r) {
    if (r >= nrows) break;
    double a = v[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[r * 32 + wid] = a;
  }
  sync();
  if (tid < nrows) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[tid * 32 + w];
    f.sums[tid] = t;
  }
  sync();
  if (tid < f.ncomp) pcg_phase(f.sums, tid, f.nq, f.phase, f.sc, f.rtol2);
  if (tid == 0) *f.ticket = 0u;
}

}  // namespace sts
