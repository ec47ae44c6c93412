/*
 * oracle/dg_oracle.c -- O1, the plain fp64 CPU oracle of arXiv 1907.06191.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py
 * (its cpu_baseline leg and --impl reference) may load this library.  The
 * product path (paper_1907_06191_b200/) never imports, links or executes it,
 * and this file shares no code, header, table or constant with that path.
 *
 * What it computes (paper = /root/reference/PAPER.md, "P:<line>"):
 *   - the IBVP u_t = div(k grad u) on a pixel substrate, k = 0 in axons and
 *     k0 = D elsewhere (Eqs. (1)-(5));
 *   - the mixed system q = grad u, u_t = div(k q) (Eq. (6)) in its
 *     element weak form (Eq. (7), read as standard LDG: the printed
 *     "u . grad v" is -int u div(v) and "k q grad . v" is -int k q . grad v;
 *     DESIGN.md reading R4);
 *   - Lagrange P_p elements, w = sum_j w_j N_j (Eq. (8)) on the two
 *     triangles of each square pixel, equispaced nodes (reading R3);
 *   - central u-flux h_u = (u- + u+)/2 n-  and harmonic-mean q-flux
 *     h_q = 2k-k+/(k-+k+) (q- + q+)/2 . n- (P:199-202);
 *   - axon elements are computed too ("null computations"):
 *     their u stays 0 and u+ = 0 enters the neighbour's u-flux (reading R6);
 *   - "a Runge-Kutta method" = SSP-RK3 in increment form (reading R7);
 *   - Dirac Cauchy data at the source pixel centre, L2-projected and
 *     split 1/2, 1/2 between the two triangles sharing the diagonal (R10);
 *   - moments of each density about its source point (R12/R14) and the
 *     mixture covariance Sigma (R15).
 *
 * Everything is done the plain way, element by element: a q pass, then an
 * rhs pass, per stage.  Reference matrices come from Gauss quadrature of the
 * explicit barycentric Lagrange formulas.  No composite stencil, no blocking,
 * no fusion.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define DMAX 10  /* (p+1)(p+2)/2 for p <= 3 ("p+1" is a 1-D typo) */
#define QMAX 8   /* Gauss points per direction */

/* ------------------------------------------------------------------------- */
/* Gauss-Legendre rule on [0,1] (textbook Newton iteration on P_n).           */
/* ------------------------------------------------------------------------- */
static void gauss_legendre01(int n, double *x, double *w) {
  for (int i = 0; i < n; i++) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 200; it++) {
      double p1 = 1.0, p0 = 0.0;
      for (int k = 1; k <= n; k++) {
        double pm = p0;
        p0 = p1;
        p1 = ((2.0 * k - 1.0) * z * p0 - (k - 1.0) * pm) / k;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (fabs(dz) < 1e-17) break;
    }
    {
      double p1 = 1.0, p0 = 0.0;
      for (int k = 1; k <= n; k++) {
        double pm = p0;
        p0 = p1;
        p1 = ((2.0 * k - 1.0) * z * p0 - (k - 1.0) * pm) / k;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
    }
    x[i] = 0.5 * (1.0 - z);
    w[i] = 1.0 / ((1.0 - z * z) * dp * dp); /* = (2/((1-z^2)P'^2)) / 2 */
  }
}

/* ------------------------------------------------------------------------- */
/* Mesh: pixel (i,j) covers [ih,(i+1)h] x [jh,(j+1)h], split by the   */
/* lower-left -> upper-right diagonal (reading R1).  In pixel-local unit      */
/* coordinates (xi, eta):                                                     */
/*   type 0 = L, vertices (0,0),(1,0),(1,1);  type 1 = U, (0,0),(1,1),(0,1). */
/* ------------------------------------------------------------------------- */
static const double VERT[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{0, 0}, {1, 1}, {0, 1}}};

/* barycentric coordinates of (xi,eta) w.r.t. the triangle's vertices, and
 * their constant derivatives d(lambda_k)/d(xi), d(lambda_k)/d(eta)           */
static void barycentric(int t, double xi, double eta, double lam[3], double dlam[3][2]) {
  if (t == 0) { /* L: lam1 = xi - eta, lam2 = eta, lam0 = 1 - xi */
    lam[0] = 1.0 - xi; lam[1] = xi - eta; lam[2] = eta;
    dlam[0][0] = -1; dlam[0][1] = 0;
    dlam[1][0] = 1;  dlam[1][1] = -1;
    dlam[2][0] = 0;  dlam[2][1] = 1;
  } else {      /* U: lam1 = xi, lam2 = eta - xi, lam0 = 1 - eta */
    lam[0] = 1.0 - eta; lam[1] = xi; lam[2] = eta - xi;
    dlam[0][0] = 0;  dlam[0][1] = -1;
    dlam[1][0] = 1;  dlam[1][1] = 0;
    dlam[2][0] = -1; dlam[2][1] = 1;
  }
}

/* Lagrange basis N_j (Eq. (8)) on the equispaced lattice, in the
 * canonical order: vertices v0,v1,v2; edge nodes of v0v1, v1v2, v2v0 (each
 * from its first vertex to its second); interior node.  Values and
 * pixel-local gradients d/dxi, d/deta.                                      */
static void basis(int p, int t, double xi, double eta, double *phi, double (*gphi)[2]) {
  double l[3], dl[3][2];
  barycentric(t, xi, eta, l, dl);
  if (p == 1) {
    for (int k = 0; k < 3; k++) {
      phi[k] = l[k];
      if (gphi) { gphi[k][0] = dl[k][0]; gphi[k][1] = dl[k][1]; }
    }
    return;
  }
  if (p == 2) {
    static const int E[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    for (int k = 0; k < 3; k++) {
      phi[k] = l[k] * (2.0 * l[k] - 1.0);
      if (gphi)
        for (int c = 0; c < 2; c++) gphi[k][c] = (4.0 * l[k] - 1.0) * dl[k][c];
    }
    for (int e = 0; e < 3; e++) {
      int a = E[e][0], b = E[e][1];
      phi[3 + e] = 4.0 * l[a] * l[b];
      if (gphi)
        for (int c = 0; c < 2; c++) gphi[3 + e][c] = 4.0 * (dl[a][c] * l[b] + l[a] * dl[b][c]);
    }
    return;
  }
  /* p == 3 */
  {
    static const int E[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    for (int k = 0; k < 3; k++) {
      double L = l[k];
      phi[k] = 0.5 * L * (3.0 * L - 1.0) * (3.0 * L - 2.0);
      if (gphi) {
        double d = 0.5 * (27.0 * L * L - 18.0 * L + 2.0);
        for (int c = 0; c < 2; c++) gphi[k][c] = d * dl[k][c];
      }
    }
    for (int e = 0; e < 3; e++) {
      int a = E[e][0], b = E[e][1];
      /* node nearer a: lam_a = 2/3, lam_b = 1/3; then node nearer b */
      int order[2][2] = {{a, b}, {b, a}};
      for (int s = 0; s < 2; s++) {
        int m = order[s][0], o = order[s][1];
        int idx = 3 + 2 * e + s;
        phi[idx] = 4.5 * l[m] * l[o] * (3.0 * l[m] - 1.0);
        if (gphi)
          for (int c = 0; c < 2; c++)
            gphi[idx][c] = 4.5 * (dl[m][c] * l[o] * (3.0 * l[m] - 1.0) +
                                  l[m] * dl[o][c] * (3.0 * l[m] - 1.0) +
                                  l[m] * l[o] * 3.0 * dl[m][c]);
      }
    }
    phi[9] = 27.0 * l[0] * l[1] * l[2];
    if (gphi)
      for (int c = 0; c < 2; c++)
        gphi[9][c] = 27.0 * (dl[0][c] * l[1] * l[2] + l[0] * dl[1][c] * l[2] + l[0] * l[1] * dl[2][c]);
  }
}

/* nodes of the lattice in the same canonical order (pixel-local coords) */
static void lattice_nodes(int p, int t, double (*nodes)[2]) {
  const double (*V)[2] = VERT[t];
  int n = 0;
  for (int k = 0; k < 3; k++) { nodes[n][0] = V[k][0]; nodes[n][1] = V[k][1]; n++; }
  static const int E[3][2] = {{0, 1}, {1, 2}, {2, 0}};
  for (int e = 0; e < 3; e++)
    for (int s = 1; s < p; s++) {
      double f = (double)s / p;
      nodes[n][0] = V[E[e][0]][0] + f * (V[E[e][1]][0] - V[E[e][0]][0]);
      nodes[n][1] = V[E[e][0]][1] + f * (V[E[e][1]][1] - V[E[e][0]][1]);
      n++;
    }
  if (p == 3) {
    nodes[n][0] = (V[0][0] + V[1][0] + V[2][0]) / 3.0;
    nodes[n][1] = (V[0][1] + V[1][1] + V[2][1]) / 3.0;
    n++;
  }
}

/* ------------------------------------------------------------------------- */
/* Faces.  Face f of triangle type t: endpoints (local), outward unit normal  */
/* n^- and the neighbour element across it (pixel offset and type).           */
/* ------------------------------------------------------------------------- */
static const double FACE_A[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{1, 1}, {0, 1}, {0, 0}}};
static const double FACE_B[2][3][2] = {{{1, 0}, {1, 1}, {0, 0}}, {{0, 1}, {0, 0}, {1, 1}}};
static const int NB_DI[2][3] = {{0, 1, 0}, {0, -1, 0}};
static const int NB_DJ[2][3] = {{-1, 0, 0}, {1, 0, 0}};

static void face_normal(int t, int f, double n[2]) {
  const double r = 1.0 / sqrt(2.0);
  if (t == 0) {
    if (f == 0) { n[0] = 0; n[1] = -1; }
    else if (f == 1) { n[0] = 1; n[1] = 0; }
    else { n[0] = -r; n[1] = r; }
  } else {
    if (f == 0) { n[0] = 0; n[1] = 1; }
    else if (f == 1) { n[0] = -1; n[1] = 0; }
    else { n[0] = r; n[1] = -r; }
  }
}

/* ------------------------------------------------------------------------- */
/* Reference matrices, physical units (pixel of side h at the origin):        */
/*   M[i][j]      = int_T N_i N_j                                             */
/*   Dc[c][i][j]  = int_T d_c N_i  N_j                                        */
/*   Em[f][i][j]  = int_f N_i^- N_j^-      Ep[f][i][j] = int_f N_i^- N_j^+     */
/* ------------------------------------------------------------------------- */
typedef struct {
  int p, d;
  double h;
  double nodes[2][DMAX][2];
  double M[2][DMAX][DMAX], Minv[2][DMAX][DMAX];
  double Dc[2][2][DMAX][DMAX];
  double Em[2][3][DMAX][DMAX], Ep[2][3][DMAX][DMAX];
  double nrm[2][3][2];
  /* triangle quadrature (pixel-local points, physical weights) */
  int nq;
  double qx[2][QMAX * QMAX][2], qw[2][QMAX * QMAX];
} refel_t;

static void invert(int d, double A[DMAX][DMAX], double X[DMAX][DMAX]) {
  /* Gauss-Jordan with partial pivoting */
  double a[DMAX][2 * DMAX];
  for (int i = 0; i < d; i++)
    for (int j = 0; j < 2 * d; j++) a[i][j] = (j < d) ? A[i][j] : (j - d == i ? 1.0 : 0.0);
  for (int c = 0; c < d; c++) {
    int piv = c;
    for (int r = c + 1; r < d; r++)
      if (fabs(a[r][c]) > fabs(a[piv][c])) piv = r;
    if (piv != c)
      for (int j = 0; j < 2 * d; j++) { double tmp = a[c][j]; a[c][j] = a[piv][j]; a[piv][j] = tmp; }
    double s = 1.0 / a[c][c];
    for (int j = 0; j < 2 * d; j++) a[c][j] *= s;
    for (int r = 0; r < d; r++)
      if (r != c) {
        double f = a[r][c];
        if (f != 0.0)
          for (int j = 0; j < 2 * d; j++) a[r][j] -= f * a[c][j];
      }
  }
  for (int i = 0; i < d; i++)
    for (int j = 0; j < d; j++) X[i][j] = a[i][d + j];
}

static void refel_init(refel_t *R, int p, double h) {
  memset(R, 0, sizeof(*R));
  R->p = p;
  R->d = (p + 1) * (p + 2) / 2;
  R->h = h;
  int d = R->d;
  int n = p + 3; /* collapsed Gauss: exact for total degree <= 2n-2 = 2p+4 */
  double gx[QMAX], gw[QMAX];
  gauss_legendre01(n, gx, gw);
  R->nq = n * n;
  for (int t = 0; t < 2; t++) {
    lattice_nodes(p, t, R->nodes[t]);
    const double *a = VERT[t][0], *b = VERT[t][1], *c = VERT[t][2];
    /* x(u,v) = a + u[(b-a) + v(c-b)],  |J| = u |det(b-a, c-b)|              */
    double det = fabs((b[0] - a[0]) * (c[1] - b[1]) - (b[1] - a[1]) * (c[0] - b[0]));
    int q = 0;
    for (int iu = 0; iu < n; iu++)
      for (int iv = 0; iv < n; iv++, q++) {
        double u = gx[iu], v = gx[iv];
        R->qx[t][q][0] = a[0] + u * ((b[0] - a[0]) + v * (c[0] - b[0]));
        R->qx[t][q][1] = a[1] + u * ((b[1] - a[1]) + v * (c[1] - b[1]));
        R->qw[t][q] = gw[iu] * gw[iv] * u * det * h * h;
      }
    /* volume matrices */
    for (q = 0; q < R->nq; q++) {
      double phi[DMAX], g[DMAX][2];
      basis(p, t, R->qx[t][q][0], R->qx[t][q][1], phi, g);
      double w = R->qw[t][q];
      for (int i = 0; i < d; i++)
        for (int j = 0; j < d; j++) {
          R->M[t][i][j] += w * phi[i] * phi[j];
          for (int cc = 0; cc < 2; cc++) R->Dc[t][cc][i][j] += w * (g[i][cc] / h) * phi[j];
        }
    }
    invert(d, R->M[t], R->Minv[t]);
    /* face matrices: Gauss-Legendre along the face, both elements' basis
     * evaluated at the same physical point                                   */
    for (int f = 0; f < 3; f++) {
      face_normal(t, f, R->nrm[t][f]);
      const double *A = FACE_A[t][f], *B = FACE_B[t][f];
      double len = h * sqrt((B[0] - A[0]) * (B[0] - A[0]) + (B[1] - A[1]) * (B[1] - A[1]));
      int tn = 1 - t; /* neighbour across any face is the other type */
      for (int k = 0; k < n; k++) {
        double xi = A[0] + gx[k] * (B[0] - A[0]);
        double eta = A[1] + gx[k] * (B[1] - A[1]);
        double pm[DMAX], pp[DMAX];
        basis(p, t, xi, eta, pm, NULL);
        basis(p, tn, xi - NB_DI[t][f], eta - NB_DJ[t][f], pp, NULL);
        double w = gw[k] * len;
        for (int i = 0; i < d; i++)
          for (int j = 0; j < d; j++) {
            R->Em[t][f][i][j] += w * pm[i] * pm[j];
            R->Ep[t][f][i][j] += w * pm[i] * pp[j];
          }
      }
    }
  }
}

/* ------------------------------------------------------------------------- */
/* Problem                                                                    */
/* ------------------------------------------------------------------------- */
typedef struct {
  refel_t R;
  int nx, ny;
  double D;
  int outer_bc; /* 0 = REFLECT (reading R9), 1 = ABSORB = Eq. (4) */
  const uint8_t *mask;
} prob_t;

/* diffusivity of pixel (i,j), Eq. (5); out-of-grid = axon under REFLECT */
static double kpix(const prob_t *P, int i, int j) {
  if (i < 0 || j < 0 || i >= P->nx || j >= P->ny) return 0.0;
  return P->mask[(size_t)j * P->nx + i] ? 0.0 : P->D;
}

/* harmonic mean 2k-k+/(k-+k+), defined as 0 when k-+k+ = 0 */
static double harmonic(double km, double kp) {
  if (km + kp == 0.0) return 0.0;
  return 2.0 * km * kp / (km + kp);
}

static inline size_t eidx(const prob_t *P, int i, int j, int t) {
  return (((size_t)j * P->nx + i) * 2 + t) * P->R.d;
}

/* Lu = M^-1 [ rhs of Eq. (7) ] for one source state u.
 * q: scratch of size 2 * nx*ny*2*d (q_x then q_y).                          */
static void apply_L(const prob_t *P, const double *u, double *q, double *Lu) {
  const refel_t *R = &P->R;
  const int d = R->d, nx = P->nx, ny = P->ny;
  const size_t nel = (size_t)nx * ny * 2 * d;
  double *qx = q, *qy = q + nel;
  static const double zero[DMAX] = {0};

  /* q pass: first row of Eq. (7) with the central u-flux:
   * M q_c = -Dc u + sum_f n_c int_f (u- + u+)/2 N_i                         */
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++)
      for (int t = 0; t < 2; t++) {
        const double *uT = u + eidx(P, i, j, t);
        double r[2][DMAX];
        for (int c = 0; c < 2; c++)
          for (int a = 0; a < d; a++) {
            double s = 0.0;
            for (int b = 0; b < d; b++) s -= R->Dc[t][c][a][b] * uT[b];
            r[c][a] = s;
          }
        for (int f = 0; f < 3; f++) {
          int in = i + NB_DI[t][f], jn = j + NB_DJ[t][f];
          int outside = (in < 0 || jn < 0 || in >= nx || jn >= ny);
          if (outside && P->outer_bc == 1) continue; /* ABSORB: ghost u+ = -u-, h_u = 0 */
          /* masked or (REFLECT) out-of-grid neighbour: u+ = 0 (reading R6) */
          const double *un = outside ? zero : u + eidx(P, in, jn, 1 - t);
          for (int a = 0; a < d; a++) {
            double s = 0.0;
            for (int b = 0; b < d; b++) s += R->Em[t][f][a][b] * uT[b] + R->Ep[t][f][a][b] * un[b];
            s *= 0.5;
            r[0][a] += R->nrm[t][f][0] * s;
            r[1][a] += R->nrm[t][f][1] * s;
          }
        }
        double *qxT = qx + eidx(P, i, j, t), *qyT = qy + eidx(P, i, j, t);
        for (int a = 0; a < d; a++) {
          double sx = 0.0, sy = 0.0;
          for (int b = 0; b < d; b++) {
            sx += R->Minv[t][a][b] * r[0][b];
            sy += R->Minv[t][a][b] * r[1][b];
          }
          qxT[a] = sx;
          qyT[a] = sy;
        }
      }

  /* rhs pass: second row of Eq. (7) with the harmonic-mean q-flux
   * (P:199-202): M u_t = -k_T sum_c Dc q_c + sum_f k_f int_f (q-+q+)/2 . n N_i */
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++) {
      double kT = kpix(P, i, j);
      for (int t = 0; t < 2; t++) {
        const double *qT[2] = {qx + eidx(P, i, j, t), qy + eidx(P, i, j, t)};
        double r[DMAX];
        for (int a = 0; a < d; a++) {
          double s = 0.0;
          for (int c = 0; c < 2; c++)
            for (int b = 0; b < d; b++) s += R->Dc[t][c][a][b] * qT[c][b];
          r[a] = -kT * s;
        }
        for (int f = 0; f < 3; f++) {
          int in = i + NB_DI[t][f], jn = j + NB_DJ[t][f];
          int outside = (in < 0 || jn < 0 || in >= nx || jn >= ny);
          if (outside) {
            if (P->outer_bc == 1) { /* ABSORB: q+ = q-, k+ = k-  =>  k_T q- . n */
              for (int a = 0; a < d; a++) {
                double s = 0.0;
                for (int c = 0; c < 2; c++)
                  for (int b = 0; b < d; b++) s += R->nrm[t][f][c] * R->Em[t][f][a][b] * qT[c][b];
                r[a] += kT * s;
              }
            }
            continue; /* REFLECT: k+ = 0 => k_f = 0 */
          }
          double kf = harmonic(kT, kpix(P, in, jn));
          if (kf == 0.0) continue;
          const double *qN[2] = {qx + eidx(P, in, jn, 1 - t), qy + eidx(P, in, jn, 1 - t)};
          for (int a = 0; a < d; a++) {
            double s = 0.0;
            for (int c = 0; c < 2; c++) {
              double sc = 0.0;
              for (int b = 0; b < d; b++) sc += R->Em[t][f][a][b] * qT[c][b] + R->Ep[t][f][a][b] * qN[c][b];
              s += R->nrm[t][f][c] * sc;
            }
            r[a] += kf * 0.5 * s;
          }
        }
        double *LT = Lu + eidx(P, i, j, t);
        for (int a = 0; a < d; a++) {
          double s = 0.0;
          for (int b = 0; b < d; b++) s += R->Minv[t][a][b] * r[b];
          LT[a] = s;
        }
      }
    }
}

/* Dirac Cauchy data at the pixel-local point (xi, eta) of pixel (is,js)
 * (P:241): exact L2 projection M_T u_T = N_T(x_s) on the triangle holding
 * the point (L: eta < xi, U: eta > xi); a point on the shared diagonal (the
 * pixel centre, R10) is split 1/2, 1/2 between L and U.  Sub-pixel points
 * (N4) follow reading R21 (a point on a pixel edge belongs to the pixel
 * floor(x/h), floor(y/h)).                                                  */
static void project_point(const prob_t *P, int is, int js, double xi, double eta, double *u) {
  const refel_t *R = &P->R;
  const int d = R->d;
  memset(u, 0, sizeof(double) * (size_t)P->nx * P->ny * 2 * d);
  for (int t = 0; t < 2; t++) {
    const double w = xi == eta ? 0.5 : ((t == 0) == (eta < xi) ? 1.0 : 0.0);
    if (w == 0.0) continue;
    double phi[DMAX];
    basis(R->p, t, xi, eta, phi, NULL);
    double *uT = u + eidx(P, is, js, t);
    for (int a = 0; a < d; a++) {
      double s = 0.0;
      for (int b = 0; b < d; b++) s += R->Minv[t][a][b] * phi[b];
      uT[a] = w * s;
    }
  }
}

/* the pixel-centre source of P:241 */
static void project_delta(const prob_t *P, int is, int js, double *u) { project_point(P, is, js, 0.5, 0.5, u); }

/* SSP-RK3 in increment form (reading R7):
 *   U1 = u  + dt L(u)
 *   U2 = U1 + 3/4 (u - U1) + 1/4 dt L(U1)
 *   u  = U2 + 1/3 (u - U2) + 2/3 dt L(U2)                                   */
static void ssprk3_step(const prob_t *P, double *u, double *U1, double *U2, double *Lb, double *q,
                        double dt) {
  const size_t n = (size_t)P->nx * P->ny * 2 * P->R.d;
  apply_L(P, u, q, Lb);
  for (size_t k = 0; k < n; k++) U1[k] = u[k] + dt * Lb[k];
  apply_L(P, U1, q, Lb);
  for (size_t k = 0; k < n; k++) U2[k] = U1[k] + 0.75 * (u[k] - U1[k]) + 0.25 * dt * Lb[k];
  apply_L(P, U2, q, Lb);
  for (size_t k = 0; k < n; k++) u[k] = U2[k] + (1.0 / 3.0) * (u[k] - U2[k]) + (2.0 / 3.0) * dt * Lb[k];
}

/* m_ab = int (x-xs)^a (y-ys)^b u_h, (a,b) in {00,10,01,20,11,02}, exact
 * integration of the DG polynomial by quadrature (reading R14), about the
 * source point xs = pixel centre (reading R12).                             */
static void moments_about(const prob_t *P, const double *u, double xs, double ys, double m[6]) {
  const refel_t *R = &P->R;
  const int d = R->d;
  const double h = R->h;
  for (int k = 0; k < 6; k++) m[k] = 0.0;
  for (int j = 0; j < P->ny; j++)
    for (int i = 0; i < P->nx; i++)
      for (int t = 0; t < 2; t++) {
        const double *uT = u + eidx(P, i, j, t);
        int nz = 0;
        for (int a = 0; a < d; a++) nz |= (uT[a] != 0.0);
        if (!nz) continue;
        for (int q = 0; q < R->nq; q++) {
          double phi[DMAX];
          basis(R->p, t, R->qx[t][q][0], R->qx[t][q][1], phi, NULL);
          double val = 0.0;
          for (int a = 0; a < d; a++) val += uT[a] * phi[a];
          double X = (i + R->qx[t][q][0]) * h - xs, Y = (j + R->qx[t][q][1]) * h - ys;
          double w = R->qw[t][q] * val;
          m[0] += w;
          m[1] += w * X;
          m[2] += w * Y;
          m[3] += w * X * X;
          m[4] += w * X * Y;
          m[5] += w * Y * Y;
        }
      }
}

static void moments(const prob_t *P, const double *u, int is, int js, double m[6]) {
  moments_about(P, u, (is + 0.5) * P->R.h, (js + 0.5) * P->R.h, m);
}

/* ------------------------------------------------------------------------- */
/* Exported API (ctypes; see oracle/oracle.py)                                */
/* ------------------------------------------------------------------------- */

/* reference matrices of degree p at pixel size h, canonical order.
 * M, Minv: [2][d][d]; Dc: [2][2][d][d]; Em, Ep: [2][3][d][d]; nrm: [2][3][2];
 * nodes: [2][d][2] (pixel-local)                                            */
int orc_reference(int p, double h, double *M, double *Minv, double *Dc, double *Em, double *Ep,
                  double *nrm, double *nodes) {
  if (p < 1 || p > 3 || !(h > 0)) return 1;
  refel_t *R = (refel_t *)malloc(sizeof(refel_t));
  refel_init(R, p, h);
  int d = R->d;
  for (int t = 0; t < 2; t++) {
    for (int i = 0; i < d; i++) {
      if (nodes) { nodes[(t * d + i) * 2] = R->nodes[t][i][0]; nodes[(t * d + i) * 2 + 1] = R->nodes[t][i][1]; }
      for (int j = 0; j < d; j++) {
        if (M) M[(t * d + i) * d + j] = R->M[t][i][j];
        if (Minv) Minv[(t * d + i) * d + j] = R->Minv[t][i][j];
        for (int c = 0; c < 2; c++)
          if (Dc) Dc[((t * 2 + c) * d + i) * d + j] = R->Dc[t][c][i][j];
        for (int f = 0; f < 3; f++) {
          if (Em) Em[((t * 3 + f) * d + i) * d + j] = R->Em[t][f][i][j];
          if (Ep) Ep[((t * 3 + f) * d + i) * d + j] = R->Ep[t][f][i][j];
        }
      }
    }
    for (int f = 0; f < 3; f++)
      for (int c = 0; c < 2; c++)
        if (nrm) nrm[(t * 3 + f) * 2 + c] = R->nrm[t][f][c];
  }
  free(R);
  return 0;
}

/* basis values at pixel-local points: out[npts][d] */
int orc_basis(int p, int t, int npts, const double *pts, double *out) {
  if (p < 1 || p > 3 || t < 0 || t > 1) return 1;
  int d = (p + 1) * (p + 2) / 2;
  for (int k = 0; k < npts; k++) basis(p, t, pts[2 * k], pts[2 * k + 1], out + (size_t)k * d, NULL);
  return 0;
}

static int setup(prob_t *P, int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc) {
  if (p < 1 || p > 3 || !(h > 0) || !(D > 0) || nx < 1 || ny < 1 || outer_bc < 0 || outer_bc > 1)
    return 1;
  refel_init(&P->R, p, h);
  P->nx = nx;
  P->ny = ny;
  P->D = D;
  P->outer_bc = outer_bc;
  P->mask = mask;
  return 0;
}

/* one evaluation of the semi-discrete operator: Lu = L(u), u: [ny][nx][2][d] */
int orc_apply_L(int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc,
                const double *u, double *Lu) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  if (setup(P, p, h, D, nx, ny, mask, outer_bc)) { free(P); return 1; }
  size_t n = (size_t)nx * ny * 2 * P->R.d;
  double *q = (double *)malloc(sizeof(double) * 2 * n);
  apply_L(P, u, q, Lu);
  free(q);
  free(P);
  return 0;
}

/* advance an arbitrary state nsteps SSP-RK3 steps in place */
int orc_advance(int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc,
                double *u, double dt, int64_t nsteps) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  if (setup(P, p, h, D, nx, ny, mask, outer_bc)) { free(P); return 1; }
  size_t n = (size_t)nx * ny * 2 * P->R.d;
  double *buf = (double *)malloc(sizeof(double) * 5 * n);
  for (int64_t s = 0; s < nsteps; s++) ssprk3_step(P, u, buf, buf + n, buf + 2 * n, buf + 3 * n, dt);
  free(buf);
  free(P);
  return 0;
}

/* moments of an arbitrary state about the centre of pixel (is,js) */
int orc_moments(int p, double h, int nx, int ny, const double *u, int is, int js, double *m) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  static const uint8_t dummy = 0;
  if (setup(P, p, h, 1.0, nx, ny, &dummy, 0)) { free(P); return 1; }
  moments(P, u, is, js, m);
  free(P);
  return 0;
}

/* the Dirac data of one source */
int orc_project_delta(int p, double h, int nx, int ny, int is, int js, double *u) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  static const uint8_t dummy = 0;
  if (setup(P, p, h, 1.0, nx, ny, &dummy, 0)) { free(P); return 1; }
  project_delta(P, is, js, u);
  free(P);
  return 0;
}

/* The first step of the scheme of P:239-243, for n sources: Dirac data at
 * each source, nsteps SSP-RK3 steps of size dt, then the six moments.
 * sources: [n][2] pixel (i,j); mom_out: [n][6]; dens_out: NULL or
 * [n][ny][nx][2][d].  One OpenMP thread per source.
 * Returns 0, 1 (argument), 2 (source on a masked / out-of-grid pixel),
 * 4 (non-finite moments).                                                   */
int orc_solve(int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc,
              const int32_t *sources, int64_t n, double dt, int64_t nsteps, double *mom_out,
              double *dens_out, int nthreads) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  if (setup(P, p, h, D, nx, ny, mask, outer_bc) || n < 0 || nsteps < 0 || !(dt >= 0)) {
    free(P);
    return 1;
  }
  for (int64_t s = 0; s < n; s++) {
    int is = sources[2 * s], js = sources[2 * s + 1];
    if (is < 0 || js < 0 || is >= nx || js >= ny || mask[(size_t)js * nx + is]) { free(P); return 2; }
  }
  const size_t ne = (size_t)nx * ny * 2 * P->R.d;
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
#endif
  for (int64_t s = 0; s < n; s++) {
    double *buf = (double *)malloc(sizeof(double) * 6 * ne);
    double *u = buf;
    int is = sources[2 * s], js = sources[2 * s + 1];
    project_delta(P, is, js, u);
    for (int64_t k = 0; k < nsteps; k++)
      ssprk3_step(P, u, buf + ne, buf + 2 * ne, buf + 3 * ne, buf + 4 * ne, dt);
    double m[6];
    moments(P, u, is, js, m);
    for (int k = 0; k < 6; k++) {
      mom_out[s * 6 + k] = m[k];
      if (!isfinite(m[k])) bad |= 1;
    }
    if (dens_out) memcpy(dens_out + (size_t)s * ne, u, sizeof(double) * ne);
    free(buf);
  }
  free(P);
  return bad ? 4 : 0;
}

/* orc_solve for point sources anywhere in extracellular pixels (N4):
 * points [n][2] physical (x, y); pixel (floor(x/h), floor(y/h)) (R21), the
 * Dirac projected at the point, moments about the point.  Returns as
 * orc_solve.                                                                */
int orc_solve_points(int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc,
                     const double *points, int64_t n, double dt, int64_t nsteps, double *mom_out,
                     double *dens_out, int nthreads) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  if (setup(P, p, h, D, nx, ny, mask, outer_bc) || n < 0 || nsteps < 0 || !(dt >= 0)) {
    free(P);
    return 1;
  }
  for (int64_t s = 0; s < n; s++) {
    double x = points[2 * s] / h, y = points[2 * s + 1] / h;
    if (!(x >= 0 && y >= 0 && x < nx && y < ny)) { free(P); return 2; }
    if (mask[(size_t)(int)floor(y) * nx + (int)floor(x)]) { free(P); return 2; }
  }
  const size_t ne = (size_t)nx * ny * 2 * P->R.d;
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
#endif
  for (int64_t s = 0; s < n; s++) {
    double *buf = (double *)malloc(sizeof(double) * 6 * ne);
    double *u = buf;
    const double x = points[2 * s] / h, y = points[2 * s + 1] / h;
    const int is = (int)floor(x), js = (int)floor(y);
    project_point(P, is, js, x - is, y - js, u);
    for (int64_t k = 0; k < nsteps; k++)
      ssprk3_step(P, u, buf + ne, buf + 2 * ne, buf + 3 * ne, buf + 4 * ne, dt);
    double m[6];
    moments_about(P, u, points[2 * s], points[2 * s + 1], m);
    for (int k = 0; k < 6; k++) {
      mom_out[s * 6 + k] = m[k];
      if (!isfinite(m[k])) bad |= 1;
    }
    if (dens_out) memcpy(dens_out + (size_t)s * ne, u, sizeof(double) * ne);
    free(buf);
  }
  free(P);
  return bad ? 4 : 0;
}

/* Sigma of the mixture from per-source moments, in source order.
 * centering 0: densities shifted by their source point (reading R12);
 * centering 1: by their own mean.  mu may be NULL.
 * Returns 0, 1 (argument), 6 (m00 <= 0), 4 (non-finite).                    */
int orc_sigma(const double *mom, int64_t n, int centering, double *sigma, double *mu) {
  if (n < 1 || centering < 0 || centering > 1) return 1;
  double mx = 0, my = 0, sxx = 0, sxy = 0, syy = 0;
  for (int64_t s = 0; s < n; s++) {
    const double *m = mom + 6 * s;
    if (!(m[0] > 0)) return isfinite(m[0]) ? 6 : 4;
    double ux = m[1] / m[0], uy = m[2] / m[0];          /* centring + normalisation */
    double xx = m[3] / m[0], xy = m[4] / m[0], yy = m[5] / m[0];
    if (centering == 1) { xx -= ux * ux; xy -= ux * uy; yy -= uy * uy; ux = 0; uy = 0; }
    mx += ux; my += uy; sxx += xx; sxy += xy; syy += yy; /* mixture u = (1/m) sum u_i */
  }
  mx /= n; my /= n; sxx /= n; sxy /= n; syy /= n;
  sigma[0] = sxx - mx * mx;                            /* E[(X-mu_x)^2] */
  sigma[1] = sxy - mx * my;
  sigma[2] = sigma[1];
  sigma[3] = syy - my * my;
  if (mu) { mu[0] = mx; mu[1] = my; }
  for (int k = 0; k < 4; k++)
    if (!isfinite(sigma[k])) return 4;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Smooth data for convergence tests: L2 projection of the Gaussian          */
/* g(x) = exp(-|x - x0|^2 / (2 s2)) / (2 pi s2) onto V_h, and the exact L2   */
/* error of a state against it (free-space solution: s2 -> s2 + 2 D t).      */
/* ------------------------------------------------------------------------- */
static double gauss2d(double x, double y, double x0, double y0, double s2) {
  double r2 = (x - x0) * (x - x0) + (y - y0) * (y - y0);
  return exp(-0.5 * r2 / s2) / (2.0 * M_PI * s2);
}

int orc_project_gaussian(int p, double h, int nx, int ny, double x0, double y0, double s2, double *u) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  static const uint8_t dummy = 0;
  if (setup(P, p, h, 1.0, nx, ny, &dummy, 0) || !(s2 > 0)) { free(P); return 1; }
  const refel_t *R = &P->R;
  const int d = R->d;
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++)
      for (int t = 0; t < 2; t++) {
        double b[DMAX] = {0};
        for (int q = 0; q < R->nq; q++) {
          double phi[DMAX];
          basis(p, t, R->qx[t][q][0], R->qx[t][q][1], phi, NULL);
          double g = gauss2d((i + R->qx[t][q][0]) * h, (j + R->qx[t][q][1]) * h, x0, y0, s2);
          for (int a = 0; a < d; a++) b[a] += R->qw[t][q] * g * phi[a];
        }
        double *uT = u + eidx(P, i, j, t);
        for (int a = 0; a < d; a++) {
          double s = 0.0;
          for (int c = 0; c < d; c++) s += R->Minv[t][a][c] * b[c];
          uT[a] = s;
        }
      }
  free(P);
  return 0;
}

int orc_l2_err_gaussian(int p, double h, int nx, int ny, const double *u, double x0, double y0, double s2,
                        double *err) {
  prob_t *P = (prob_t *)malloc(sizeof(prob_t));
  static const uint8_t dummy = 0;
  if (setup(P, p, h, 1.0, nx, ny, &dummy, 0) || !(s2 > 0)) { free(P); return 1; }
  const refel_t *R = &P->R;
  const int d = R->d;
  double e2 = 0.0;
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++)
      for (int t = 0; t < 2; t++) {
        const double *uT = u + eidx(P, i, j, t);
        for (int q = 0; q < R->nq; q++) {
          double phi[DMAX];
          basis(p, t, R->qx[t][q][0], R->qx[t][q][1], phi, NULL);
          double v = 0.0;
          for (int a = 0; a < d; a++) v += uT[a] * phi[a];
          double g = gauss2d((i + R->qx[t][q][0]) * h, (j + R->qx[t][q][1]) * h, x0, y0, s2);
          e2 += R->qw[t][q] * (v - g) * (v - g);
        }
      }
  *err = sqrt(e2);
  free(P);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* The mixture model on the displacement lattice [-R, R]^2 and   */
/* the least-squares residual of Eq. (9) against the Gaussian   */
/* density N(x; mu, Sigma) of P:252.  Node value of source s at (dx, dy):    */
/* the DG solution at the centre of pixel (is+dx, js+dy), taken as the mean  */
/* of the L and U traces there (the centre lies on their shared diagonal,    */
/* DESIGN.md reading R20), divided by m00_s ("centering and normalization",  */
/* P:243).  dens: [n][ny][nx][2][d]; grid: [2R+1][2R+1], dy outer.           */
/* ------------------------------------------------------------------------- */
int orc_mixture(int p, int nx, int ny, const double *dens, const int32_t *sources, const double *mom, int64_t n,
                int R, double *grid) {
  if (p < 1 || p > 3 || n < 1 || R < 0) return 1;
  const int d = (p + 1) * (p + 2) / 2, side = 2 * R + 1;
  double phiL[DMAX], phiU[DMAX];
  basis(p, 0, 0.5, 0.5, phiL, NULL);
  basis(p, 1, 0.5, 0.5, phiU, NULL);
  for (int c = 0; c < side * side; c++) grid[c] = 0.0;
  for (int64_t s = 0; s < n; s++) {
    const double *u = dens + (size_t)s * nx * ny * 2 * d;
    const int is = sources[2 * s], js = sources[2 * s + 1];
    for (int dy = -R; dy <= R; dy++)
      for (int dx = -R; dx <= R; dx++) {
        const int i = is + dx, j = js + dy;
        if (i < 0 || j < 0 || i >= nx || j >= ny) continue;
        const double *uL = u + (((size_t)j * nx + i) * 2 + 0) * d;
        const double *uU = uL + d;
        double vL = 0.0, vU = 0.0;
        for (int a = 0; a < d; a++) { vL += uL[a] * phiL[a]; vU += uU[a] * phiU[a]; }
        grid[(dy + R) * side + (dx + R)] += 0.5 * (vL + vU) / mom[6 * s];
      }
  }
  for (int c = 0; c < side * side; c++) grid[c] /= (double)n;
  return 0;
}

int orc_residual(const double *grid, int R, double h, const double *sigma, const double *mu, double *res) {
  const int side = 2 * R + 1;
  const double sxx = sigma[0], sxy = sigma[1], syy = sigma[3];
  const double det = sxx * syy - sxy * sxy;
  if (!(det > 0)) return 6;
  double r = 0.0;
  for (int dy = -R; dy <= R; dy++)
    for (int dx = -R; dx <= R; dx++) {
      const double x = dx * h - mu[0], y = dy * h - mu[1];
      /* (x, y) Sigma^-1 (x, y)^T */
      const double q = (syy * x * x - 2.0 * sxy * x * y + sxx * y * y) / det;
      const double g = exp(-0.5 * q) / (2.0 * M_PI * sqrt(det));
      const double e = g - grid[(dy + R) * side + (dx + R)];
      r += e * e;
    }
  *res = r;
  return 0;
}

/* ========================================================================= */
/* N4: quadrilateral Q_p elements, one per pixel (SURVEY 8f "Q_p elements on  */
/* one-pixel cells", the north star's "Q2").  The same mixed system, fluxes   */
/* and readings as the triangles (Eq. (7), R4-R7, R9 REFLECT),    */
/* with the tensor-product Lagrange basis N_ab(xi, eta) = l_a(xi) l_b(eta) on */
/* the equispaced nodes (a/p, b/p), dof k = b (p+1) + a, and four faces      */
/* E, W, N, S (bit order of the open-face code).  Written out element by     */
/* element like the triangle oracle: a q pass, then an rhs pass.             */
/* ========================================================================= */
#define QDMAX 16 /* (p+1)^2 for p <= 3 */

typedef struct {
  int p, d;
  double h;
  double M[QDMAX][QDMAX], Minv[QDMAX][QDMAX];
  double Dc[2][QDMAX][QDMAX];
  double Em[4][QDMAX][QDMAX], Ep[4][QDMAX][QDMAX];
  int nq;
  double qx[QMAX * QMAX][2], qw[QMAX * QMAX];
} qref_t;

static const int QNB[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};   /* E W N S */
static const double QNRM[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};

/* 1-D Lagrange basis on s_k = k/p and its derivative */
static void lag1(int p, double s, double *l, double *dl) {
  for (int a = 0; a <= p; a++) {
    double v = 1.0, dv = 0.0;
    for (int k = 0; k <= p; k++) {
      if (k == a) continue;
      const double den = (double)(a - k) / p;
      /* product rule: d(v * (s - s_k)/den) */
      dv = dv * (s - (double)k / p) / den + v / den;
      v *= (s - (double)k / p) / den;
    }
    l[a] = v;
    if (dl) dl[a] = dv;
  }
}

static void qbasis(int p, double xi, double eta, double *phi, double (*g)[2]) {
  double lx[4], dlx[4], ly[4], dly[4];
  lag1(p, xi, lx, dlx);
  lag1(p, eta, ly, dly);
  for (int b = 0; b <= p; b++)
    for (int a = 0; a <= p; a++) {
      const int k = b * (p + 1) + a;
      phi[k] = lx[a] * ly[b];
      if (g) { g[k][0] = dlx[a] * ly[b]; g[k][1] = lx[a] * dly[b]; }
    }
}

static void qinvert(int d, double A[QDMAX][QDMAX], double X[QDMAX][QDMAX]) {
  double a[QDMAX][2 * QDMAX];
  for (int i = 0; i < d; i++)
    for (int j = 0; j < 2 * d; j++) a[i][j] = (j < d) ? A[i][j] : (j - d == i ? 1.0 : 0.0);
  for (int c = 0; c < d; c++) {
    int piv = c;
    for (int r = c + 1; r < d; r++)
      if (fabs(a[r][c]) > fabs(a[piv][c])) piv = r;
    if (piv != c)
      for (int j = 0; j < 2 * d; j++) { double tmp = a[c][j]; a[c][j] = a[piv][j]; a[piv][j] = tmp; }
    double s = 1.0 / a[c][c];
    for (int j = 0; j < 2 * d; j++) a[c][j] *= s;
    for (int r = 0; r < d; r++)
      if (r != c) {
        double f = a[r][c];
        if (f != 0.0)
          for (int j = 0; j < 2 * d; j++) a[r][j] -= f * a[c][j];
      }
  }
  for (int i = 0; i < d; i++)
    for (int j = 0; j < d; j++) X[i][j] = a[i][d + j];
}

static void qref_init(qref_t *R, int p, double h) {
  memset(R, 0, sizeof(*R));
  R->p = p;
  R->d = (p + 1) * (p + 1);
  R->h = h;
  const int d = R->d, n = p + 2;   /* tensor Gauss, exact to degree 2p+2 per direction */
  double gx[QMAX], gw[QMAX];
  gauss_legendre01(n, gx, gw);
  R->nq = n * n;
  for (int iy = 0, q = 0; iy < n; iy++)
    for (int ix = 0; ix < n; ix++, q++) {
      R->qx[q][0] = gx[ix];
      R->qx[q][1] = gx[iy];
      R->qw[q] = gw[ix] * gw[iy] * h * h;
    }
  for (int q = 0; q < R->nq; q++) {
    double phi[QDMAX], g[QDMAX][2];
    qbasis(p, R->qx[q][0], R->qx[q][1], phi, g);
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) {
        R->M[i][j] += R->qw[q] * phi[i] * phi[j];
        for (int c = 0; c < 2; c++) R->Dc[c][i][j] += R->qw[q] * (g[i][c] / h) * phi[j];
      }
  }
  qinvert(d, R->M, R->Minv);
  /* faces: the point s along the face; K's local point and the neighbour's */
  for (int f = 0; f < 4; f++)
    for (int k = 0; k < n; k++) {
      const double s = gx[k];
      double xk, yk;
      if (f == 0) { xk = 1; yk = s; } else if (f == 1) { xk = 0; yk = s; }
      else if (f == 2) { xk = s; yk = 1; } else { xk = s; yk = 0; }
      double pm[QDMAX], pp[QDMAX];
      qbasis(p, xk, yk, pm, NULL);
      qbasis(p, xk - QNB[f][0], yk - QNB[f][1], pp, NULL);
      const double w = gw[k] * h;
      for (int i = 0; i < d; i++)
        for (int j = 0; j < d; j++) {
          R->Em[f][i][j] += w * pm[i] * pm[j];
          R->Ep[f][i][j] += w * pm[i] * pp[j];
        }
    }
}

typedef struct {
  qref_t R;
  int nx, ny;
  double D;
  int outer_bc;   /* 0 = REFLECT (R9), 1 = ABSORB = Eq. (4): ghost u+ = -u-, q+ = q-, k+ = k- */
  const uint8_t *mask;
} qprob_t;

static double qkpix(const qprob_t *P, int i, int j) {
  if (i < 0 || j < 0 || i >= P->nx || j >= P->ny) return 0.0;   /* REFLECT (R9) */
  return P->mask[(size_t)j * P->nx + i] ? 0.0 : P->D;
}

static inline size_t qidx(const qprob_t *P, int i, int j) { return ((size_t)j * P->nx + i) * P->R.d; }

/* Lu = M^-1 [rhs of Eq. (7)] for Q_p: q pass, then rhs pass */
static void q_apply_L(const qprob_t *P, const double *u, double *q, double *Lu) {
  const qref_t *R = &P->R;
  const int d = R->d, nx = P->nx, ny = P->ny;
  const size_t nel = (size_t)nx * ny * d;
  double *qx = q, *qy = q + nel;
  static const double zero[QDMAX] = {0};
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++) {
      const double *uK = u + qidx(P, i, j);
      double r[2][QDMAX];
      for (int c = 0; c < 2; c++)
        for (int a = 0; a < d; a++) {
          double s = 0.0;
          for (int b = 0; b < d; b++) s -= R->Dc[c][a][b] * uK[b];
          r[c][a] = s;
        }
      for (int f = 0; f < 4; f++) {
        const int in = i + QNB[f][0], jn = j + QNB[f][1];
        const int outside = (in < 0 || jn < 0 || in >= nx || jn >= ny);
        if (outside && P->outer_bc == 1) continue;   /* ABSORB: h_u = (u- + u+)/2 = 0 */
        const double *un = outside ? zero : u + qidx(P, in, jn);   /* u+ = 0 outside (R6, R9) */
        for (int a = 0; a < d; a++) {
          double s = 0.0;
          for (int b = 0; b < d; b++) s += R->Em[f][a][b] * uK[b] + R->Ep[f][a][b] * un[b];
          s *= 0.5;
          r[0][a] += QNRM[f][0] * s;
          r[1][a] += QNRM[f][1] * s;
        }
      }
      for (int a = 0; a < d; a++) {
        double sx = 0.0, sy = 0.0;
        for (int b = 0; b < d; b++) {
          sx += R->Minv[a][b] * r[0][b];
          sy += R->Minv[a][b] * r[1][b];
        }
        qx[qidx(P, i, j) + a] = sx;
        qy[qidx(P, i, j) + a] = sy;
      }
    }
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++) {
      const double kK = qkpix(P, i, j);
      const double *qK[2] = {qx + qidx(P, i, j), qy + qidx(P, i, j)};
      double r[QDMAX];
      for (int a = 0; a < d; a++) {
        double s = 0.0;
        for (int c = 0; c < 2; c++)
          for (int b = 0; b < d; b++) s += R->Dc[c][a][b] * qK[c][b];
        r[a] = -kK * s;
      }
      for (int f = 0; f < 4; f++) {
        const int in = i + QNB[f][0], jn = j + QNB[f][1];
        if ((in < 0 || jn < 0 || in >= nx || jn >= ny) && P->outer_bc == 1) {
          /* ABSORB: q+ = q-, k+ = k-  =>  h_q = k_K q- . n */
          for (int a = 0; a < d; a++) {
            double sc = 0.0;
            for (int c = 0; c < 2; c++)
              for (int b = 0; b < d; b++) sc += QNRM[f][c] * R->Em[f][a][b] * qK[c][b];
            r[a] += kK * sc;
          }
          continue;
        }
        const double kf = harmonic(kK, qkpix(P, in, jn));
        if (kf == 0.0) continue;
        const double *qN[2] = {qx + qidx(P, in, jn), qy + qidx(P, in, jn)};
        for (int a = 0; a < d; a++) {
          double s = 0.0;
          for (int c = 0; c < 2; c++) {
            double sc = 0.0;
            for (int b = 0; b < d; b++) sc += R->Em[f][a][b] * qK[c][b] + R->Ep[f][a][b] * qN[c][b];
            s += QNRM[f][c] * sc;
          }
          r[a] += kf * 0.5 * s;
        }
      }
      for (int a = 0; a < d; a++) {
        double s = 0.0;
        for (int b = 0; b < d; b++) s += R->Minv[a][b] * r[b];
        Lu[qidx(P, i, j) + a] = s;
      }
    }
}

static void q_ssprk3_step(const qprob_t *P, double *u, double *U1, double *U2, double *Lb, double *q, double dt) {
  const size_t n = (size_t)P->nx * P->ny * P->R.d;
  q_apply_L(P, u, q, Lb);
  for (size_t k = 0; k < n; k++) U1[k] = u[k] + dt * Lb[k];
  q_apply_L(P, U1, q, Lb);
  for (size_t k = 0; k < n; k++) U2[k] = U1[k] + 0.75 * (u[k] - U1[k]) + 0.25 * dt * Lb[k];
  q_apply_L(P, U2, q, Lb);
  for (size_t k = 0; k < n; k++) u[k] = U2[k] + (1.0 / 3.0) * (u[k] - U2[k]) + (2.0 / 3.0) * dt * Lb[k];
}

/* Dirac at the centre of pixel (is, js): M u_K = N(1/2, 1/2) (interior point:
 * no split) */
static void q_project_delta(const qprob_t *P, int is, int js, double *u) {
  const qref_t *R = &P->R;
  memset(u, 0, sizeof(double) * (size_t)P->nx * P->ny * R->d);
  double phi[QDMAX];
  qbasis(R->p, 0.5, 0.5, phi, NULL);
  double *uK = u + qidx(P, is, js);
  for (int a = 0; a < R->d; a++) {
    double s = 0.0;
    for (int b = 0; b < R->d; b++) s += R->Minv[a][b] * phi[b];
    uK[a] = s;
  }
}

/* sub-pixel point (xi, eta) of pixel (is, js) (N4, reading R21): M u_K = N(xi, eta) */
static void q_project_point(const qprob_t *P, int is, int js, double xi, double eta, double *u) {
  const qref_t *R = &P->R;
  memset(u, 0, sizeof(double) * (size_t)P->nx * P->ny * R->d);
  double phi[QDMAX];
  qbasis(R->p, xi, eta, phi, NULL);
  double *uK = u + qidx(P, is, js);
  for (int a = 0; a < R->d; a++) {
    double s = 0.0;
    for (int b = 0; b < R->d; b++) s += R->Minv[a][b] * phi[b];
    uK[a] = s;
  }
}

static void q_moments_about(const qprob_t *P, const double *u, double xs, double ys, double m[6]);

static void q_moments(const qprob_t *P, const double *u, int is, int js, double m[6]) {
  q_moments_about(P, u, (is + 0.5) * P->R.h, (js + 0.5) * P->R.h, m);
}

static void q_moments_about(const qprob_t *P, const double *u, double xs, double ys, double m[6]) {
  const qref_t *R = &P->R;
  const double h = R->h;
  for (int k = 0; k < 6; k++) m[k] = 0.0;
  for (int j = 0; j < P->ny; j++)
    for (int i = 0; i < P->nx; i++) {
      const double *uK = u + qidx(P, i, j);
      int nz = 0;
      for (int a = 0; a < R->d; a++) nz |= (uK[a] != 0.0);
      if (!nz) continue;
      for (int q = 0; q < R->nq; q++) {
        double phi[QDMAX];
        qbasis(R->p, R->qx[q][0], R->qx[q][1], phi, NULL);
        double val = 0.0;
        for (int a = 0; a < R->d; a++) val += uK[a] * phi[a];
        const double X = (i + R->qx[q][0]) * h - xs, Y = (j + R->qx[q][1]) * h - ys, w = R->qw[q] * val;
        m[0] += w;
        m[1] += w * X;
        m[2] += w * Y;
        m[3] += w * X * X;
        m[4] += w * X * Y;
        m[5] += w * Y * Y;
      }
    }
}

static int q_setup(qprob_t *P, int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc) {
  if (p < 1 || p > 3 || !(h > 0) || !(D > 0) || nx < 1 || ny < 1 || !mask || outer_bc < 0 || outer_bc > 1) return 1;
  qref_init(&P->R, p, h);
  P->nx = nx;
  P->ny = ny;
  P->D = D;
  P->outer_bc = outer_bc;
  P->mask = mask;
  return 0;
}

/* reference matrices: M, Minv [d][d]; Dc [2][d][d]; Em, Ep [4][d][d] */
int orc_q_reference(int p, double h, double *M, double *Minv, double *Dc, double *Em, double *Ep) {
  if (p < 1 || p > 3) return 1;
  qref_t *R = (qref_t *)malloc(sizeof(qref_t));
  qref_init(R, p, h);
  const int d = R->d;
  for (int i = 0; i < d; i++)
    for (int j = 0; j < d; j++) {
      M[i * d + j] = R->M[i][j];
      Minv[i * d + j] = R->Minv[i][j];
      for (int c = 0; c < 2; c++) Dc[(c * d + i) * d + j] = R->Dc[c][i][j];
      for (int f = 0; f < 4; f++) {
        Em[(f * d + i) * d + j] = R->Em[f][i][j];
        Ep[(f * d + i) * d + j] = R->Ep[f][i][j];
      }
    }
  free(R);
  return 0;
}

/* u, out: [ny][nx][(p+1)^2] */
int orc_q_apply_L(int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc, const double *u,
                  double *out) {
  qprob_t *P = (qprob_t *)malloc(sizeof(qprob_t));
  if (q_setup(P, p, h, D, nx, ny, mask, outer_bc)) { free(P); return 1; }
  double *q = (double *)malloc(sizeof(double) * 2 * (size_t)nx * ny * P->R.d);
  q_apply_L(P, u, q, out);
  free(q);
  free(P);
  return 0;
}

/* as orc_solve, for Q_p (REFLECT or ABSORB); dens_out: NULL or [n][ny][nx][(p+1)^2] */
int orc_q_solve(int p, double h, double D, int nx, int ny, const uint8_t *mask, int outer_bc, const int32_t *sources,
                int64_t n, double dt, int64_t nsteps, double *mom_out, double *dens_out, int nthreads) {
  qprob_t *P = (qprob_t *)malloc(sizeof(qprob_t));
  if (q_setup(P, p, h, D, nx, ny, mask, outer_bc) || n < 0 || nsteps < 0 || !(dt >= 0)) { free(P); return 1; }
  for (int64_t s = 0; s < n; s++) {
    int is = sources[2 * s], js = sources[2 * s + 1];
    if (is < 0 || js < 0 || is >= nx || js >= ny || mask[(size_t)js * nx + is]) { free(P); return 2; }
  }
  const size_t ne = (size_t)nx * ny * P->R.d;
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
#endif
  for (int64_t s = 0; s < n; s++) {
    double *buf = (double *)malloc(sizeof(double) * 6 * ne);
    double *u = buf;
    const int is = sources[2 * s], js = sources[2 * s + 1];
    q_project_delta(P, is, js, u);
    for (int64_t k = 0; k < nsteps; k++)
      q_ssprk3_step(P, u, buf + ne, buf + 2 * ne, buf + 3 * ne, buf + 4 * ne, dt);
    double m[6];
    q_moments(P, u, is, js, m);
    for (int k = 0; k < 6; k++) {
      mom_out[s * 6 + k] = m[k];
      if (!isfinite(m[k])) bad |= 1;
    }
    if (dens_out) memcpy(dens_out + (size_t)s * ne, u, sizeof(double) * ne);
    free(buf);
  }
  free(P);
  return bad ? 4 : 0;
}

/* orc_q_solve for physical point sources (N4; R21): pixel (floor(x/h),
 * floor(y/h)), Dirac projected at the point, moments about the point */
int orc_q_solve_points(int p, double h, double D, int nx, int ny, const uint8_t *mask, const double *points,
                       int64_t n, double dt, int64_t nsteps, double *mom_out, double *dens_out, int nthreads) {
  qprob_t *P = (qprob_t *)malloc(sizeof(qprob_t));
  if (q_setup(P, p, h, D, nx, ny, mask, 0) || n < 0 || nsteps < 0 || !(dt >= 0)) { free(P); return 1; }
  for (int64_t s = 0; s < n; s++) {
    const double x = points[2 * s] / h, y = points[2 * s + 1] / h;
    if (!(x >= 0 && y >= 0 && x < nx && y < ny)) { free(P); return 2; }
    if (mask[(size_t)(int)floor(y) * nx + (int)floor(x)]) { free(P); return 2; }
  }
  const size_t ne = (size_t)nx * ny * P->R.d;
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
#endif
  for (int64_t s = 0; s < n; s++) {
    double *buf = (double *)malloc(sizeof(double) * 6 * ne);
    double *u = buf;
    const double x = points[2 * s] / h, y = points[2 * s + 1] / h;
    const int is = (int)floor(x), js = (int)floor(y);
    q_project_point(P, is, js, x - is, y - js, u);
    for (int64_t k = 0; k < nsteps; k++)
      q_ssprk3_step(P, u, buf + ne, buf + 2 * ne, buf + 3 * ne, buf + 4 * ne, dt);
    double m[6];
    q_moments_about(P, u, points[2 * s], points[2 * s + 1], m);
    for (int k = 0; k < 6; k++) {
      mom_out[s * 6 + k] = m[k];
      if (!isfinite(m[k])) bad |= 1;
    }
    if (dens_out) memcpy(dens_out + (size_t)s * ne, u, sizeof(double) * ne);
    free(buf);
  }
  free(P);
  return bad ? 4 : 0;
}
