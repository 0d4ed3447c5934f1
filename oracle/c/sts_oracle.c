/*
 * ORACLE (plain C) -- TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT.
 *
 * A plain, slow, obviously-correct CPU implementation in C (BASELINE north_star:
 * "a plain, slow CPU C/C++ implementation of the paper's operators, RKL2
 * coefficients and stage count s, and Jacobi-PCG, sharing no code with the GPU
 * path") of Caplan et al., arxiv 1610.01265 (/root/reference/PAPER.md, cited as
 * PAPER.md:L).  It follows the same readings as oracle/oracle.py (R1-R13)
 * and is pinned against that independently pinned numpy oracle and closed forms in
 * tests/test_oracle_c.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline may load it; it never links, includes or calls paper_1610_01265_b200/.
 *
 * Layout: fields are C-contiguous [n1][n2][n3] (phi fastest); vector fields
 * [ncomp][n1][n2][n3]; face arrays use the "+ face" convention (k_d[i][j][k] is the
 * face between cell (i,j,k) and its +e_d neighbour; faces without one are ignored).
 * Every function loops cell by cell with no blocking or fusion.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int n1, n2, n3, periodic3, spherical;
  const double *x1f, *x1c, *x2f, *x2c, *x3f, *x3c; /* faces n+1, centres n */
} grid_t;

static long idx(const grid_t* g, int i, int j, int k) { return ((long)i * g->n2 + j) * g->n3 + k; }

/* neighbour of (i,j,k) in direction d (+1); returns 0 if it does not exist */
static int plus(const grid_t* g, int d, int i, int j, int k, int* ii, int* jj, int* kk) {
  *ii = i;
  *jj = j;
  *kk = k;
  if (d == 0) {
    if (i + 1 >= g->n1) return 0;
    *ii = i + 1;
  } else if (d == 1) {
    if (j + 1 >= g->n2) return 0;
    *jj = j + 1;
  } else {
    if (k + 1 >= g->n3) {
      if (!g->periodic3) return 0;
      *kk = 0;
    } else {
      *kk = k + 1;
    }
  }
  return 1;
}

/* ---------------------------------------------------------------------------
 * Geometry (Sec. 4.2, DESIGN R1): cell volume, and for the + face of
 * direction d its area A and the distance h between the two centres it separates.
 * ------------------------------------------------------------------------- */
static double volume(const grid_t* g, int i, int j, int k) {
  const double dr = g->x1f[i + 1] - g->x1f[i], dt = g->x2f[j + 1] - g->x2f[j], dp = g->x3f[k + 1] - g->x3f[k];
  if (!g->spherical) return dr * dt * dp;
  const double r3 = (pow(g->x1f[i + 1], 3) - pow(g->x1f[i], 3)) / 3.0;
  return r3 * (cos(g->x2f[j]) - cos(g->x2f[j + 1])) * dp;
}

static double center_gap(const double* xc, const double* xf, int n, int m, int periodic) {
  /* distance from centre m to centre m+1 (wrap for a periodic dimension) */
  if (m + 1 < n) return xc[m + 1] - xc[m];
  if (periodic) return xc[0] + (xf[n] - xf[0]) - xc[m];
  return NAN;
}

static void face_geo(const grid_t* g, int d, int i, int j, int k, double* A, double* h) {
  const double dr = g->x1f[i + 1] - g->x1f[i], dt = g->x2f[j + 1] - g->x2f[j], dp = g->x3f[k + 1] - g->x3f[k];
  if (!g->spherical) {
    if (d == 0) { *A = dt * dp; *h = center_gap(g->x1c, g->x1f, g->n1, i, 0); }
    else if (d == 1) { *A = dr * dp; *h = center_gap(g->x2c, g->x2f, g->n2, j, 0); }
    else { *A = dr * dt; *h = center_gap(g->x3c, g->x3f, g->n3, k, g->periodic3); }
    return;
  }
  const double r2 = 0.5 * (g->x1f[i + 1] * g->x1f[i + 1] - g->x1f[i] * g->x1f[i]);
  if (d == 0) {
    *A = g->x1f[i + 1] * g->x1f[i + 1] * (cos(g->x2f[j]) - cos(g->x2f[j + 1])) * dp;
    *h = center_gap(g->x1c, g->x1f, g->n1, i, 0);
  } else if (d == 1) {
    *A = r2 * sin(g->x2f[j + 1]) * dp;
    *h = g->x1c[i] * center_gap(g->x2c, g->x2f, g->n2, j, 0);
  } else {
    *A = r2 * dt;
    *h = g->x1c[i] * sin(g->x2c[j]) * center_gap(g->x3c, g->x3f, g->n3, k, g->periodic3);
  }
}

/* ---------------------------------------------------------------------------
 * Lagged Spitzer face diffusivity (DESIGN R3):
 * kappa_f = kappa0 f_c(r_f) beta_Tcut(T_f) T_f^(5/2), T_f = (T_L + T_R)/2.
 * ------------------------------------------------------------------------- */
void oc_face_kappa(const grid_t* g, const double* T, double kappa0, double T_cut, double fc_r0, double fc_w,
                   double* k1, double* k2, double* k3) {
  double* K[3] = {k1, k2, k3};
#pragma omp parallel for schedule(static)
  for (int i = 0; i < g->n1; ++i)
    for (int j = 0; j < g->n2; ++j)
      for (int k = 0; k < g->n3; ++k)
        for (int d = 0; d < 3; ++d) {
          int ii, jj, kk;
          double v = 0.0;
          if (plus(g, d, i, j, k, &ii, &jj, &kk)) {
            const double Tf = 0.5 * (T[idx(g, i, j, k)] + T[idx(g, ii, jj, kk)]);
            double beta = 1.0;
            if (T_cut > 0.0 && Tf < T_cut) beta = pow(Tf / T_cut, 2.5);
            v = kappa0 * beta * pow(Tf, 2.5);
            if (g->spherical && fc_w > 0.0) {
              const double rf = (d == 0) ? g->x1f[i + 1] : g->x1c[i];
              v *= 0.5 * (1.0 - tanh((rf - fc_r0) / fc_w));
            }
          }
          K[d][idx(g, i, j, k)] = v;
        }
}

/* ---------------------------------------------------------------------------
 * The operator (DESIGN R2): (L u)_i = -dE/du_i,
 *   isotropic  E = 1/2 sum_faces kappa_f A_f/h_f (u_R - u_L)^2                 (7-point)
 *   anisotropic E = 1/2 sum_vertices V_v kappa_v (b_v . g_v)^2                  (27-point)
 * at every vertex surrounded by 8 existing cells: g_a = 1/4 sum of the 4 differences
 * along a divided by their centre distances, b_v / V_v the means of the 8 cells,
 * kappa_v the mean of the 12 faces around the vertex.  Each vertex is expressed as
 * E_v = 1/2 C_v (sum_p w_p u_p)^2 over its 8 cells p.
 * ------------------------------------------------------------------------- */
typedef struct {
  long id[8];
  double w[8];
  double C;
} vertex_t;

/* vertex at the upper corner of cell (i,j,k); returns 0 if a cell is missing */
static int vertex(const grid_t* g, const double* const kap[3], const double* b, int i, int j, int k, vertex_t* v) {
  const long plane = (long)g->n1 * g->n2 * g->n3;
  int c[8][3];
  for (int s = 0; s < 8; ++s) {
    int ci = i, cj = j, ck = k, ii, jj, kk;
    if (s & 4) { if (!plus(g, 0, ci, cj, ck, &ii, &jj, &kk)) return 0; ci = ii; }
    if (s & 2) { if (!plus(g, 1, ci, cj, ck, &ii, &jj, &kk)) return 0; cj = jj; }
    if (s & 1) { if (!plus(g, 2, ci, cj, ck, &ii, &jj, &kk)) return 0; ck = kk; }
    c[s][0] = ci;
    c[s][1] = cj;
    c[s][2] = ck;
    v->id[s] = idx(g, ci, cj, ck);
  }
  double bv[3] = {0, 0, 0}, Vv = 0.0, kv = 0.0;
  for (int s = 0; s < 8; ++s) {
    for (int a = 0; a < 3; ++a) bv[a] += b[a * plane + v->id[s]] / 8.0;
    Vv += volume(g, c[s][0], c[s][1], c[s][2]) / 8.0;
  }
  /* the 12 faces around the vertex: for direction a, the 4 cells with s_a = 0 */
  for (int a = 0; a < 3; ++a) {
    const int bit = (a == 0) ? 4 : (a == 1) ? 2 : 1;
    for (int s = 0; s < 8; ++s)
      if (!(s & bit)) kv += kap[a][v->id[s]] / 12.0;
  }
  v->C = Vv * kv;
  for (int s = 0; s < 8; ++s) v->w[s] = 0.0;
  for (int a = 0; a < 3; ++a) {
    const int bit = (a == 0) ? 4 : (a == 1) ? 2 : 1;
    for (int s = 0; s < 8; ++s) {
      if (s & bit) continue;
      double A, h;
      face_geo(g, a, c[s][0], c[s][1], c[s][2], &A, &h);
      (void)A;
      v->w[s] -= bv[a] * 0.25 / h;
      v->w[s | bit] += bv[a] * 0.25 / h;
    }
  }
  return 1;
}

/* out = L u  (mode 0: isotropic with face coefficients kappa A/h; mode 1: anisotropic) */
static void apply_L(const grid_t* g, int mode, const double* const kap[3], const double* b, const double* u, double* out) {
  const long n = (long)g->n1 * g->n2 * g->n3;
  for (long q = 0; q < n; ++q) out[q] = 0.0;
  for (int i = 0; i < g->n1; ++i)
    for (int j = 0; j < g->n2; ++j)
      for (int k = 0; k < g->n3; ++k) {
        if (mode == 0) {
          for (int d = 0; d < 3; ++d) {
            int ii, jj, kk;
            if (!plus(g, d, i, j, k, &ii, &jj, &kk)) continue;
            double A, h;
            face_geo(g, d, i, j, k, &A, &h);
            const long L = idx(g, i, j, k), R = idx(g, ii, jj, kk);
            const double K = kap[d][L] * A / h;
            out[L] += K * (u[R] - u[L]);
            out[R] += K * (u[L] - u[R]);
          }
        } else {
          vertex_t v;
          if (!vertex(g, kap, b, i, j, k, &v)) continue;
          double s = 0.0;
          for (int p = 0; p < 8; ++p) s += v.w[p] * u[v.id[p]];
          for (int p = 0; p < 8; ++p) out[v.id[p]] -= v.C * v.w[p] * s;
        }
      }
}

/* F(u) = L u / (w V)  (Eq. 1), component-wise for ncomp > 1 */
void oc_op_apply(const grid_t* g, int mode, int ncomp, const double* k1, const double* k2, const double* k3,
                 const double* b, const double* w, const double* u, double* out) {
  const double* kap[3] = {k1, k2, k3};
  const long n = (long)g->n1 * g->n2 * g->n3;
  for (int c = 0; c < ncomp; ++c) {
    apply_L(g, mode, kap, b, u + c * n, out + c * n);
    for (int i = 0; i < g->n1; ++i)
      for (int j = 0; j < g->n2; ++j)
        for (int k = 0; k < g->n3; ++k) {
          const long q = idx(g, i, j, k);
          out[c * n + q] /= (w ? w[q] : 1.0) * volume(g, i, j, k);
        }
  }
}

/* ---------------------------------------------------------------------------
 * L assembled row by row: for every row at most 27 distinct columns (periodic
 * wrap with n3 <= 2 makes offsets alias one cell; entries of the same column add).
 * ------------------------------------------------------------------------- */
typedef struct {
  long id[27];
  double val[27];
  int cnt;
} row_t;

static void row_add(row_t* r, long col, double v) {
  for (int t = 0; t < r->cnt; ++t)
    if (r->id[t] == col) {
      r->val[t] += v;
      return;
    }
  r->id[r->cnt] = col;
  r->val[r->cnt] = v;
  r->cnt += 1;
}

static row_t* assemble_rows(const grid_t* g, int mode, const double* const kap[3], const double* b) {
  const long n = (long)g->n1 * g->n2 * g->n3;
  row_t* R = calloc(n, sizeof(row_t));
  for (int i = 0; i < g->n1; ++i)
    for (int j = 0; j < g->n2; ++j)
      for (int k = 0; k < g->n3; ++k) {
        if (mode == 0) {
          for (int d = 0; d < 3; ++d) {
            int ii, jj, kk;
            if (!plus(g, d, i, j, k, &ii, &jj, &kk)) continue;
            double A, h;
            face_geo(g, d, i, j, k, &A, &h);
            const long L = idx(g, i, j, k), Rr = idx(g, ii, jj, kk);
            const double K = kap[d][L] * A / h;
            /* E_f = 1/2 K (u_R - u_L)^2  ->  L = -Hessian */
            row_add(&R[L], L, -K);
            row_add(&R[L], Rr, K);
            row_add(&R[Rr], Rr, -K);
            row_add(&R[Rr], L, K);
          }
        } else {
          vertex_t v;
          if (!vertex(g, kap, b, i, j, k, &v)) continue;
          for (int p = 0; p < 8; ++p)
            for (int q = 0; q < 8; ++q) row_add(&R[v.id[p]], v.id[q], -v.C * v.w[p] * v.w[q]);
        }
      }
  return R;
}

static double row_diag(const row_t* r, long i) {
  for (int t = 0; t < r->cnt; ++t)
    if (r->id[t] == i) return r->val[t];
  return 0.0;
}

/* ---------------------------------------------------------------------------
 * Appendix B: dt_Euler = 2 / max_i sum_q |M_iq|, M = L/(wV).
 * ------------------------------------------------------------------------- */
double oc_dt_euler(const grid_t* g, int mode, const double* k1, const double* k2, const double* k3, const double* b,
                   const double* w) {
  const double* kap[3] = {k1, k2, k3};
  row_t* R = assemble_rows(g, mode, kap, b);
  double lam = 0.0;
  for (int i = 0; i < g->n1; ++i)
    for (int j = 0; j < g->n2; ++j)
      for (int k = 0; k < g->n3; ++k) {
        const long q = idx(g, i, j, k);
        double s = 0.0;
        for (int t = 0; t < R[q].cnt; ++t) s += fabs(R[q].val[t]);
        s /= (w ? w[q] : 1.0) * volume(g, i, j, k);
        if (s > lam) lam = s;
      }
  free(R);
  return lam > 0.0 ? 2.0 / lam : INFINITY;
}

/* ---------------------------------------------------------------------------
 * RKL2 (Fig. 2, Eq. 5; DESIGN R5, R6)
 * ------------------------------------------------------------------------- */
int oc_rkl2_num_stages(double dt, double dt_exp) {
  int s = (int)ceil((sqrt(9.0 + 16.0 * dt / dt_exp) - 1.0) / 2.0);
  return s < 2 ? 2 : s;
}

static double bj(int j) { return j <= 2 ? 1.0 / 3.0 : ((double)j * j + j - 2.0) / (2.0 * j * (j + 1.0)); }

void oc_rkl2_advance(const grid_t* g, int mode, int ncomp, const double* k1, const double* k2, const double* k3,
                     const double* b, const double* w, const double* u0, double dt, int s, double* u1) {
  const long n = (long)ncomp * g->n1 * g->n2 * g->n3;
  double* M0 = malloc(n * sizeof(double));
  double* ym1 = malloc(n * sizeof(double));
  double* ym2 = malloc(n * sizeof(double));
  double* yj = malloc(n * sizeof(double));
  double* F = malloc(n * sizeof(double));
  const double ss = (double)s * s + s - 2.0;
  oc_op_apply(g, mode, ncomp, k1, k2, k3, b, w, u0, M0);
  for (long q = 0; q < n; ++q) {
    ym2[q] = u0[q];
    ym1[q] = u0[q] + 4.0 / (3.0 * ss) * dt * M0[q]; /* mu~_1 = b_1 w_1 */
  }
  for (int j = 2; j <= s; ++j) {
    const double mu = (2.0 * j - 1.0) / j * bj(j) / bj(j - 1);
    const double nu = -(j - 1.0) / j * bj(j) / bj(j - 2);
    const double mut = 4.0 * (2.0 * j - 1.0) / (j * ss) * bj(j) / bj(j - 1);
    const double gt = (bj(j - 1) - 1.0) * mut;
    oc_op_apply(g, mode, ncomp, k1, k2, k3, b, w, ym1, F);
    for (long q = 0; q < n; ++q)
      yj[q] = mu * ym1[q] + nu * ym2[q] + (1.0 - mu - nu) * u0[q] + mut * dt * F[q] + gt * dt * M0[q];
    double* t = ym2;
    ym2 = ym1;
    ym1 = yj;
    yj = t;
  }
  memcpy(u1, ym1, n * sizeof(double));
  free(M0);
  free(ym1);
  free(ym2);
  free(yj);
  free(F);
}

/* ---------------------------------------------------------------------------
 * Backward Euler + point-Jacobi PCG (Eqs. 2-4, Fig. 1, PC1 of
 * :468-470; DESIGN R7, R8): (wV - dt L) x = wV u^n, x0 = u^n, z = r / diag,
 * stop when r.z <= rtol^2 b.P^-1 b.  Returns the iterations of the last component.
 * ------------------------------------------------------------------------- */
int oc_be_pcg(const grid_t* g, int mode, int ncomp, const double* k1, const double* k2, const double* k3,
              const double* b, const double* w, const double* un, double dt, double rtol, int kmax, double* x,
              int* iters) {
  const double* kap[3] = {k1, k2, k3};
  const long n = (long)g->n1 * g->n2 * g->n3;
  double* WV = malloc(n * sizeof(double));
  double* diag = malloc(n * sizeof(double));
  double *r = malloc(n * sizeof(double)), *z = malloc(n * sizeof(double)), *p = malloc(n * sizeof(double));
  double *y = malloc(n * sizeof(double)), *Lx = malloc(n * sizeof(double)), *rhs = malloc(n * sizeof(double));
  for (int i = 0; i < g->n1; ++i)
    for (int j = 0; j < g->n2; ++j)
      for (int k = 0; k < g->n3; ++k) {
        const long q = idx(g, i, j, k);
        WV[q] = (w ? w[q] : 1.0) * volume(g, i, j, k);
      }
  /* diag(A) = wV - dt L_ii (PC1: P_ii = A_ii) */
  row_t* R = assemble_rows(g, mode, kap, b);
  for (long q = 0; q < n; ++q) diag[q] = WV[q] - dt * row_diag(&R[q], q);
  free(R);
  int last = 0;
  for (int c = 0; c < ncomp; ++c) {
    const double* u = un + c * n;
    double* xc = x + c * n;
    for (long q = 0; q < n; ++q) {
      xc[q] = u[q];
      rhs[q] = WV[q] * u[q];
    }
    apply_L(g, mode, kap, b, xc, Lx);
    double rz = 0.0, bb = 0.0;
    for (long q = 0; q < n; ++q) {
      r[q] = rhs[q] - (WV[q] * xc[q] - dt * Lx[q]);
      z[q] = r[q] / diag[q];
      p[q] = z[q];
      rz += r[q] * z[q];
      bb += rhs[q] * rhs[q] / diag[q];
    }
    const double thresh = rtol * rtol * bb;
    int kk = 0;
    if (rz > thresh) {
      for (kk = 1; kk <= kmax; ++kk) {
        apply_L(g, mode, kap, b, p, Lx);
        double py = 0.0;
        for (long q = 0; q < n; ++q) {
          y[q] = WV[q] * p[q] - dt * Lx[q];
          py += p[q] * y[q];
        }
        const double alpha = rz / py;
        double rzn = 0.0;
        for (long q = 0; q < n; ++q) {
          xc[q] += alpha * p[q];
          r[q] -= alpha * y[q];
          z[q] = r[q] / diag[q];
          rzn += r[q] * z[q];
        }
        if (rzn <= thresh) break;
        const double beta = rzn / rz;
        rz = rzn;
        for (long q = 0; q < n; ++q) p[q] = beta * p[q] + z[q];
      }
      if (kk > kmax) kk = kmax;
    }
    if (iters) iters[c] = kk;
    last = kk;
  }
  free(WV); free(diag); free(r); free(z); free(p); free(y); free(Lx); free(rhs);
  return last;
}

/* ---------------------------------------------------------------------------
 * Full-grid checker (test infrastructure for the production-size parity tests).
 * Row c of L assembled on its own, matrix-free, from the same vertex / face
 * definitions as assemble_rows (DESIGN R2) -- the "gather" view of the same sum:
 *   anisotropic: L_cq = -sum over the vertices v that contain cell c (the upper
 *                corners of the cells c - (a, b, e), a, b, e in {0, 1}) of
 *                C_v w_{v,p} w_{v,q}, p the slot(s) of c in v;
 *   isotropic  : L_cc = -sum K_f, L_co = +K_f over the faces f between c and o != c.
 * No n x 27 row table is held, so it runs at the 268M-cell configs[4] size, one
 * OpenMP thread per r-plane range (rows are independent; nothing is shared).
 * ------------------------------------------------------------------------- */
static void row_gather(const grid_t* g, int mode, const double* const kap[3], const double* b, int i, int j, int k,
                       row_t* R) {
  const long c = idx(g, i, j, k);
  R->cnt = 0;
  if (mode == 0) {
    for (int d = 0; d < 3; ++d) {
      int ii, jj, kk;
      double A, h;
      /* the + face of c */
      if (plus(g, d, i, j, k, &ii, &jj, &kk) && idx(g, ii, jj, kk) != c) {
        face_geo(g, d, i, j, k, &A, &h);
        const double K = kap[d][c] * A / h;
        row_add(R, c, -K);
        row_add(R, idx(g, ii, jj, kk), K);
      }
      /* the + face of the - neighbour m (whose + neighbour is c) */
      int mi = i, mj = j, mk = k, ok = 1;
      if (d == 0) { if (i == 0) ok = 0; else mi = i - 1; }
      else if (d == 1) { if (j == 0) ok = 0; else mj = j - 1; }
      else { if (k > 0) mk = k - 1; else if (g->periodic3) mk = g->n3 - 1; else ok = 0; }
      if (ok && idx(g, mi, mj, mk) != c) {
        face_geo(g, d, mi, mj, mk, &A, &h);
        const double K = kap[d][idx(g, mi, mj, mk)] * A / h;
        row_add(R, c, -K);
        row_add(R, idx(g, mi, mj, mk), K);
      }
    }
    return;
  }
  long seen[8];
  int nseen = 0;
  for (int s = 0; s < 8; ++s) {
    int bi = i - ((s >> 2) & 1), bj = j - ((s >> 1) & 1), bk = k - (s & 1);
    if (bi < 0 || bj < 0) continue;
    if (bk < 0) {
      if (!g->periodic3) continue;
      bk += g->n3;
    }
    const long base = idx(g, bi, bj, bk);
    int dup = 0;
    for (int t = 0; t < nseen; ++t) dup |= (seen[t] == base);
    if (dup) continue;   /* (n3 = 1 periodic: both phi offsets name the same vertex) */
    seen[nseen++] = base;
    vertex_t v;
    if (!vertex(g, kap, b, bi, bj, bk, &v)) continue;
    for (int p = 0; p < 8; ++p) {
      if (v.id[p] != c) continue;
      for (int q = 0; q < 8; ++q) row_add(R, v.id[q], -v.C * v.w[p] * v.w[q]);
    }
  }
}

/*
 * For the backward-Euler system A = wV - dt L, rhs = wV un (Eq. 4,
 * DESIGN R7) and a candidate solution x, per component c:
 *   out[4c+0] = sum_i r_i^2 / A_ii      (r = rhs - A x; the stopping-test norm of DESIGN R8)
 *   out[4c+1] = sum_i rhs_i^2 / A_ii
 *   out[4c+2] = max_i |r_i| / max_i |rhs_i|
 *   out[4c+3] = 0
 * and *lam = max_i sum_q |L_iq| / (w V)_i (the Appendix B Gershgorin bound).
 * x may be NULL (then only *lam is computed).
 */
void oc_check_full(const grid_t* g, int mode, int ncomp, const double* k1, const double* k2, const double* k3,
                   const double* b, const double* w, const double* un, const double* x, double dt, double* out,
                   double* lam) {
  const double* kap[3] = {k1, k2, k3};
  const long n = (long)g->n1 * g->n2 * g->n3;
  double acc[3][4] = {{0}};
  double lmax = 0.0;
  for (int c = 0; c < ncomp; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.0;
#pragma omp parallel
  {
    double a[3][4] = {{0}};
    double lm = 0.0;
    row_t R;
#pragma omp for schedule(dynamic, 1) collapse(2)
    for (int i = 0; i < g->n1; ++i)
      for (int j = 0; j < g->n2; ++j)
        for (int k = 0; k < g->n3; ++k) {
          const long q = idx(g, i, j, k);
          row_gather(g, mode, kap, b, i, j, k, &R);
          const double wv = (w ? w[q] : 1.0) * volume(g, i, j, k);
          double s = 0.0;
          for (int t = 0; t < R.cnt; ++t) s += fabs(R.val[t]);
          if (s / wv > lm) lm = s / wv;
          if (!x) continue;
          const double Aii = wv - dt * row_diag(&R, q);
          for (int c = 0; c < ncomp; ++c) {
            const double* xc = x + c * n;
            double Lx = 0.0;
            for (int t = 0; t < R.cnt; ++t) Lx += R.val[t] * xc[R.id[t]];
            const double rhs = wv * un[c * n + q];
            const double r = rhs - (wv * xc[q] - dt * Lx);
            a[c][0] += r * r / Aii;
            a[c][1] += rhs * rhs / Aii;
            if (fabs(r) > a[c][2]) a[c][2] = fabs(r);
            if (fabs(rhs) > a[c][3]) a[c][3] = fabs(rhs);
          }
        }
#pragma omp critical
    {
      if (lm > lmax) lmax = lm;
      for (int c = 0; c < ncomp; ++c) {
        acc[c][0] += a[c][0];
        acc[c][1] += a[c][1];
        if (a[c][2] > acc[c][2]) acc[c][2] = a[c][2];
        if (a[c][3] > acc[c][3]) acc[c][3] = a[c][3];
      }
    }
  }
  for (int c = 0; c < ncomp; ++c) {
    out[4 * c + 0] = acc[c][0];
    out[4 * c + 1] = acc[c][1];
    out[4 * c + 2] = acc[c][3] > 0.0 ? acc[c][2] / acc[c][3] : acc[c][2];
    out[4 * c + 3] = 0.0;
  }
  *lam = lmax;
}

/* OpenMP threads of the checker (bench.py's cpu_baseline pins the oracle to 1) */
void oc_set_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oc_max_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
