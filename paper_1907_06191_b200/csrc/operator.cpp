// operator.cpp -- K0: host precompute of the composite 5-point DG operator.
//
// Derivation: the element weak form Eq. (7) (LDG
// reading) with Lagrange P_p elements (Eq. (8)) on the two
// triangles of each pixel, central u-flux and
// harmonic-mean q-flux.  Eliminating q = grad u (Eq. (6),
// P:131-137) leaves, for every extracellular pixel, a linear map from the u of
// the pixel and of its four face neighbours to du/dt.  Because
// k_f is either k0 or 0 (axon neighbour or outer square, R6/R9), the
// map depends only on the pixel's 4-bit open-face code: 16 variants.
//
// Everything is computed in exact rational arithmetic (__int128), in units
// D/h^2 (h = D = 1), so the table can be checked to be dyadic and is then exact
// in both fp64 and fp32.  dt and the RK weights are applied as
// scalars by the kernels.  This file shares no code with oracle/.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "operator.h"

namespace dgop {

typedef __int128 i128;

static i128 gcd(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

struct Q {
  i128 n, d;
  Q(i128 n_ = 0, i128 d_ = 1) : n(n_), d(d_) { norm(); }
  void norm() {
    if (d == 0) throw std::runtime_error("rational: zero denominator");
    if (d < 0) { n = -n; d = -d; }
    i128 g = gcd(n, d);
    if (g > 1) { n /= g; d /= g; }
    const i128 lim = (i128)1 << 110;
    if (n > lim || n < -lim || d > lim) throw std::runtime_error("rational: overflow");
  }
  bool zero() const { return n == 0; }
  double to_double() const { return (double)n / (double)d; }
};
static Q operator+(Q a, Q b) { i128 g = gcd(a.d, b.d); return Q(a.n * (b.d / g) + b.n * (a.d / g), a.d / g * b.d); }
static Q operator-(Q a) { return Q(-a.n, a.d); }
static Q operator-(Q a, Q b) { return a + (-b); }
static Q operator*(Q a, Q b) {
  i128 g1 = gcd(a.n, b.d), g2 = gcd(b.n, a.d);
  if (g1 == 0) g1 = 1;
  if (g2 == 0) g2 = 1;
  return Q((a.n / g1) * (b.n / g2), (a.d / g2) * (b.d / g1));
}
static Q operator/(Q a, Q b) { return a * Q(b.d, b.n); }
static Q &operator+=(Q &a, Q b) { a = a + b; return a; }

typedef std::vector<std::vector<Q>> Mat;
static Mat zeros(int r, int c) { return Mat(r, std::vector<Q>(c, Q(0))); }
static Mat mul(const Mat &A, const Mat &B) {
  int r = A.size(), k = B.size(), c = B[0].size();
  Mat C = zeros(r, c);
  for (int i = 0; i < r; i++)
    for (int l = 0; l < k; l++) {
      if (A[i][l].zero()) continue;
      for (int j = 0; j < c; j++)
        if (!B[l][j].zero()) C[i][j] += A[i][l] * B[l][j];
    }
  return C;
}
static void axpy(Mat &Y, Q a, const Mat &X) {  // Y += a X
  for (size_t i = 0; i < Y.size(); i++)
    for (size_t j = 0; j < Y[0].size(); j++)
      if (!X[i][j].zero()) Y[i][j] += a * X[i][j];
}
static Mat inverse(Mat A) {
  int n = A.size();
  Mat X = zeros(n, n);
  for (int i = 0; i < n; i++) X[i][i] = Q(1);
  for (int c = 0; c < n; c++) {
    int piv = c;
    while (piv < n && A[piv][c].zero()) piv++;
    if (piv == n) throw std::runtime_error("singular matrix");
    std::swap(A[c], A[piv]);
    std::swap(X[c], X[piv]);
    Q s = Q(1) / A[c][c];
    for (int j = 0; j < n; j++) { A[c][j] = A[c][j] * s; X[c][j] = X[c][j] * s; }
    for (int r = 0; r < n; r++)
      if (r != c && !A[r][c].zero()) {
        Q f = A[r][c];
        for (int j = 0; j < n; j++) {
          A[r][j] = A[r][j] - f * A[c][j];
          X[r][j] = X[r][j] - f * X[c][j];
        }
      }
  }
  return X;
}

// ---- polynomials in (xi, eta): P[a][b] coefficient of xi^a eta^b ----------
typedef std::vector<std::vector<Q>> Poly2;
typedef std::vector<Q> Poly1;

static Q qpow(Q x, int k) { Q r(1); for (int i = 0; i < k; i++) r = r * x; return r; }

// int over the unit-pixel triangle t of xi^a eta^b
// t = 0 (L = {0 < eta < xi < 1}): 1/((b+1)(a+b+2)); t = 1 (U): 1/((a+1)(a+b+2))
static Q tri_int(int t, int a, int b) { return t == 0 ? Q(1, (b + 1) * (a + b + 2)) : Q(1, (a + 1) * (a + b + 2)); }

static Q integrate2(int t, const Poly2 &P) {
  Q s(0);
  for (size_t a = 0; a < P.size(); a++)
    for (size_t b = 0; b < P[a].size(); b++)
      if (!P[a][b].zero()) s += P[a][b] * tri_int(t, a, b);
  return s;
}
static Poly2 pmul(const Poly2 &A, const Poly2 &B) {
  Poly2 C(A.size() + B.size() - 1, std::vector<Q>(A[0].size() + B[0].size() - 1, Q(0)));
  for (size_t a = 0; a < A.size(); a++)
    for (size_t b = 0; b < A[a].size(); b++)
      if (!A[a][b].zero())
        for (size_t c = 0; c < B.size(); c++)
          for (size_t e = 0; e < B[c].size(); e++)
            if (!B[c][e].zero()) C[a + c][b + e] += A[a][b] * B[c][e];
  return C;
}
static Poly2 pderiv(const Poly2 &P, int var) {
  Poly2 D(P.size(), std::vector<Q>(P[0].size(), Q(0)));
  for (size_t a = 0; a < P.size(); a++)
    for (size_t b = 0; b < P[a].size(); b++) {
      if (P[a][b].zero()) continue;
      if (var == 0 && a > 0) D[a - 1][b] += P[a][b] * Q(a);
      if (var == 1 && b > 0) D[a][b - 1] += P[a][b] * Q(b);
    }
  return D;
}
static Q peval(const Poly2 &P, Q x, Q y) {
  Q s(0);
  for (size_t a = 0; a < P.size(); a++)
    for (size_t b = 0; b < P[a].size(); b++)
      if (!P[a][b].zero()) s += P[a][b] * qpow(x, a) * qpow(y, b);
  return s;
}
static Poly1 p1mul(const Poly1 &A, const Poly1 &B) {
  Poly1 C(A.size() + B.size() - 1, Q(0));
  for (size_t i = 0; i < A.size(); i++)
    for (size_t j = 0; j < B.size(); j++) C[i + j] += A[i] * B[j];
  return C;
}
// restrict P to the line (x0 + s dx, y0 + s dy), s in [0, 1]
static Poly1 restrict_line(const Poly2 &P, Q x0, Q dx, Q y0, Q dy) {
  Poly1 out(1, Q(0));
  for (size_t a = 0; a < P.size(); a++)
    for (size_t b = 0; b < P[a].size(); b++) {
      if (P[a][b].zero()) continue;
      Poly1 term(1, P[a][b]);
      for (size_t k = 0; k < a; k++) term = p1mul(term, Poly1{x0, dx});
      for (size_t k = 0; k < b; k++) term = p1mul(term, Poly1{y0, dy});
      if (term.size() > out.size()) out.resize(term.size(), Q(0));
      for (size_t k = 0; k < term.size(); k++) out[k] += term[k];
    }
  return out;
}
static Q integrate1(const Poly1 &P) {
  Q s(0);
  for (size_t k = 0; k < P.size(); k++) s += P[k] * Q(1, k + 1);
  return s;
}

// ---- reference element -----------------------------------------------------
// triangle vertices (pixel-local): t=0 L (0,0),(1,0),(1,1); t=1 U (0,0),(1,1),(0,1)
static const int VX[2][3] = {{0, 1, 1}, {0, 1, 0}};
static const int VY[2][3] = {{0, 0, 1}, {0, 1, 1}};
// faces: start, end; scaled outward normal nu = n |f| / h; neighbour pixel offset
static const int FA[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{1, 1}, {0, 1}, {0, 0}}};
static const int FB[2][3][2] = {{{1, 0}, {1, 1}, {0, 0}}, {{0, 1}, {0, 0}, {1, 1}}};
static const int NU[2][3][2] = {{{0, -1}, {1, 0}, {-1, 1}}, {{0, 1}, {-1, 0}, {1, -1}}};
static const int NDI[2][3] = {{0, 1, 0}, {0, -1, 0}};
static const int NDJ[2][3] = {{-1, 0, 0}, {1, 0, 0}};
// which of the pixel's 4 faces (code bit) a triangle face is: -1 = internal diagonal
// bit0 E, bit1 W, bit2 N, bit3 S
static const int FACEBIT[2][3] = {{3, 0, -1}, {2, 1, -1}};

struct RefEl {
  int p, d;
  std::vector<Poly2> phi[2];
  Mat M[2], Minv[2], Dc[2][2], Em[2][3], Ep[2][3];
};

static void build_ref(RefEl &R, int p) {
  R.p = p;
  R.d = (p + 1) * (p + 2) / 2;
  int d = R.d;
  std::vector<std::pair<int, int>> mons;
  for (int a = 0; a <= p; a++)
    for (int b = 0; a + b <= p; b++) mons.push_back({a, b});
  for (int t = 0; t < 2; t++) {
    // equispaced lattice nodes, canonical order
    std::vector<std::pair<Q, Q>> nodes;
    for (int k = 0; k < 3; k++) nodes.push_back({Q(VX[t][k]), Q(VY[t][k])});
    const int E[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    for (int e = 0; e < 3; e++)
      for (int s = 1; s < p; s++) {
        Q f(s, p);
        int a = E[e][0], b = E[e][1];
        nodes.push_back({Q(VX[t][a]) + f * Q(VX[t][b] - VX[t][a]), Q(VY[t][a]) + f * Q(VY[t][b] - VY[t][a])});
      }
    if (p == 3) nodes.push_back({Q(VX[t][0] + VX[t][1] + VX[t][2], 3), Q(VY[t][0] + VY[t][1] + VY[t][2], 3)});
    Mat V = zeros(d, d);
    for (int n = 0; n < d; n++)
      for (int m = 0; m < d; m++) V[n][m] = qpow(nodes[n].first, mons[m].first) * qpow(nodes[n].second, mons[m].second);
    Mat C = inverse(V);  // N_j = sum_m C[m][j] mono_m
    R.phi[t].assign(d, Poly2(p + 1, std::vector<Q>(p + 1, Q(0))));
    for (int j = 0; j < d; j++)
      for (int m = 0; m < d; m++) R.phi[t][j][mons[m].first][mons[m].second] = C[m][j];
    // check nodality (the construction guarantees it; keeps the table honest)
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) {
        Q v = peval(R.phi[t][j], nodes[i].first, nodes[i].second);
        if (!((i == j && v.n == 1 && v.d == 1) || (i != j && v.zero()))) throw std::runtime_error("basis not nodal");
      }
    R.M[t] = zeros(d, d);
    R.Dc[t][0] = zeros(d, d);
    R.Dc[t][1] = zeros(d, d);
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) {
        R.M[t][i][j] = integrate2(t, pmul(R.phi[t][i], R.phi[t][j]));
        for (int c = 0; c < 2; c++) R.Dc[t][c][i][j] = integrate2(t, pmul(pderiv(R.phi[t][i], c), R.phi[t][j]));
      }
    R.Minv[t] = inverse(R.M[t]);
  }
  for (int t = 0; t < 2; t++)
    for (int f = 0; f < 3; f++) {
      R.Em[t][f] = zeros(d, d);
      R.Ep[t][f] = zeros(d, d);
      Q x0(FA[t][f][0]), y0(FA[t][f][1]);
      Q dx(FB[t][f][0] - FA[t][f][0]), dy(FB[t][f][1] - FA[t][f][1]);
      std::vector<Poly1> pm(d), pn(d);
      for (int i = 0; i < d; i++) {
        pm[i] = restrict_line(R.phi[t][i], x0, dx, y0, dy);
        pn[i] = restrict_line(R.phi[1 - t][i], x0 - Q(NDI[t][f]), dx, y0 - Q(NDJ[t][f]), dy);
      }
      for (int i = 0; i < d; i++)
        for (int j = 0; j < d; j++) {
          R.Em[t][f][i][j] = integrate1(p1mul(pm[i], pm[j]));
          R.Ep[t][f][i][j] = integrate1(p1mul(pm[i], pn[j]));
        }
    }
}

// ---- composite operator over a 3x3 pixel patch ------------------------------
static int tri_index(int di, int dj, int t) { return ((dj + 1) * 3 + (di + 1)) * 2 + t; }

static bool dyadic(const Q &q) { return (q.d & (q.d - 1)) == 0; }

// outer: faces of the centre pixel that lie on the outer square under the
// absorbing condition Eq. (4) (ghost u+ = -u-, q+ = q-, k+ = k-):
// they contribute h_u = 0 to its q and the full k_T q- . n to its rhs.
static void build_table(const RefEl &R, int code, Mat &out /* 2d x 18d */, int outer = 0) {
  const int d = R.d, N = 18 * d;
  // q_c of a triangle of the patch as a d x N matrix (first row of Eq. (7),
  // central u-flux; any neighbour's u may be nonzero)
  auto qmat = [&](int di, int dj, int t, int c) {
    Mat rhs = zeros(d, N);
    int T = tri_index(di, dj, t);
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) rhs[i][T * d + j] = -R.Dc[t][c][i][j];
    for (int f = 0; f < 3; f++) {
      if (di == 0 && dj == 0 && FACEBIT[t][f] >= 0 && ((outer >> FACEBIT[t][f]) & 1)) continue;  // h_u = 0
      int ni = di + NDI[t][f], nj = dj + NDJ[t][f];
      if (ni < -1 || ni > 1 || nj < -1 || nj > 1) throw std::runtime_error("patch too small");
      int Tn = tri_index(ni, nj, 1 - t);
      Q w = Q(NU[t][f][c], 2);
      if (w.zero()) continue;
      for (int i = 0; i < d; i++)
        for (int j = 0; j < d; j++) {
          rhs[i][T * d + j] += w * R.Em[t][f][i][j];
          rhs[i][Tn * d + j] += w * R.Ep[t][f][i][j];
        }
    }
    return mul(R.Minv[t], rhs);
  };
  out = zeros(2 * d, N);
  for (int t = 0; t < 2; t++) {
    Mat q0[2] = {qmat(0, 0, t, 0), qmat(0, 0, t, 1)};
    Mat r = zeros(d, N);
    // volume: -k_T sum_c Dc q_c (k_T = 1: the pixel is extracellular)
    for (int c = 0; c < 2; c++) axpy(r, Q(-1), mul(R.Dc[t][c], q0[c]));
    // faces: k_f 1/2 sum_c nu_c (E- q_c + E+ q_c^nb), k_f = 1 if open else 0
    for (int f = 0; f < 3; f++) {
      int bit = FACEBIT[t][f];
      if (bit >= 0 && ((outer >> bit) & 1)) {   // absorbing outer face: k_T q- . n, full weight
        for (int c = 0; c < 2; c++) {
          Q w = Q(NU[t][f][c]);
          if (!w.zero()) axpy(r, w, mul(R.Em[t][f], q0[c]));
        }
        continue;
      }
      if (bit >= 0 && !((code >> bit) & 1)) continue;
      int ni = NDI[t][f], nj = NDJ[t][f];
      for (int c = 0; c < 2; c++) {
        Q w = Q(NU[t][f][c], 2);
        if (w.zero()) continue;
        Mat qn = qmat(ni, nj, 1 - t, c);
        axpy(r, w, mul(R.Em[t][f], q0[c]));
        axpy(r, w, mul(R.Ep[t][f], qn));
      }
    }
    Mat du = mul(R.Minv[t], r);
    for (int i = 0; i < d; i++) out[t * d + i] = du[i];
  }
}

Table build(int p) {
  if (p < 1 || p > 3) throw std::runtime_error("degree must be 1..3");
  RefEl R;
  build_ref(R, p);
  const int d = R.d, D2 = 2 * d;
  Table T;
  T.p = p;
  T.d = d;
  T.A.assign((size_t)16 * 5 * D2 * D2, 0.0);
  T.W.assign((size_t)2 * 6 * d, 0.0);
  T.init.assign((size_t)2 * d, 0.0);
  T.nnz.assign((size_t)16 * 5, 0);
  const int OFF[5][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  for (int code = 0; code < 16; code++) {
    Mat full;
    build_table(R, code, full);
    for (int dj = -1; dj <= 1; dj++)
      for (int di = -1; di <= 1; di++) {
        int o = -1;
        for (int k = 0; k < 5; k++)
          if (OFF[k][0] == di && OFF[k][1] == dj) o = k;
        // a closed neighbour holds u = 0: its block is never applied
        bool used = (o == 0) || (o > 0 && ((code >> (o - 1)) & 1));
        for (int r = 0; r < D2; r++)
          for (int t = 0; t < 2; t++)
            for (int j = 0; j < d; j++) {
              const Q &q = full[r][tri_index(di, dj, t) * d + j];
              if (o < 0) {
                if (!q.zero()) throw std::runtime_error("corner coupling is not zero");
                continue;
              }
              if (!used) continue;
              // P1/P2 entries are dyadic (exact in fp32 and fp64); P3 entries are
              // not and are rounded to the nearest double (fp32: float)
              if (p <= 2 && !dyadic(q)) throw std::runtime_error("composite entry is not dyadic");
              T.A[(((size_t)code * 5 + o) * D2 + r) * D2 + t * d + j] = q.to_double();
              if (!q.zero()) T.nnz[code * 5 + o]++;
            }
      }
  }
  // moment weights W[t][ab][j] = int_T xi^a eta^b N_j (unit pixel)
  const int AB[6][2] = {{0, 0}, {1, 0}, {0, 1}, {2, 0}, {1, 1}, {0, 2}};
  for (int t = 0; t < 2; t++)
    for (int q = 0; q < 6; q++)
      for (int j = 0; j < d; j++) {
        Poly2 m(AB[q][0] + 1, std::vector<Q>(AB[q][1] + 1, Q(0)));
        m[AB[q][0]][AB[q][1]] = Q(1);
        T.W[(t * 6 + q) * d + j] = integrate2(t, pmul(m, R.phi[t][j])).to_double();
      }
  // Dirac at the pixel centre, L2-projected, split 1/2 - 1/2 (R10):
  // u_T = 1/2 M_T^-1 N_T(1/2, 1/2)   (units 1/h^2)
  for (int t = 0; t < 2; t++)
    for (int i = 0; i < d; i++) {
      Q s(0);
      for (int j = 0; j < d; j++) s += R.Minv[t][i][j] * peval(R.phi[t][j], Q(1, 2), Q(1, 2));
      T.init[t * d + i] = (s * Q(1, 2)).to_double();
    }
  // node value at the pixel centre (the diagonal's midpoint, shared by L and U)
  T.cw.assign((size_t)2 * d, 0.0);
  for (int t = 0; t < 2; t++)
    for (int j = 0; j < d; j++) T.cw[t * d + j] = peval(R.phi[t][j], Q(1, 2), Q(1, 2)).to_double();
  // M^-1 and the monomial coefficients of the basis, for sub-pixel Diracs
  T.minv.assign((size_t)2 * d * d, 0.0);
  T.phic.assign((size_t)2 * d * (p + 1) * (p + 1), 0.0);
  for (int t = 0; t < 2; t++)
    for (int i = 0; i < d; i++) {
      for (int j = 0; j < d; j++) T.minv[((size_t)t * d + i) * d + j] = R.Minv[t][i][j].to_double();
      for (int a = 0; a <= p; a++)
        for (int b = 0; b <= p; b++)
          T.phic[(((size_t)t * d + i) * (p + 1) + a) * (p + 1) + b] = R.phi[t][i][a][b].to_double();
    }
  return T;
}

// ---- N4: quadrilateral Q_p elements ----------------------------------------
struct QuadRef;
static void quad_ref(int p, QuadRef &R);

QuadTable build_quad(int p) {
  if (p < 1 || p > 2) throw std::runtime_error("quadrilateral elements: degree must be 1 or 2");
  const int d = (p + 1) * (p + 1);
  // tensor Lagrange basis from the nodal Vandermonde on (a/p, b/p), dof k = b (p+1) + a
  std::vector<std::pair<int, int>> mons;
  for (int b = 0; b <= p; b++)
    for (int a = 0; a <= p; a++) mons.push_back({a, b});
  Mat V = zeros(d, d);
  for (int n = 0; n < d; n++)
    for (int m = 0; m < d; m++)
      V[n][m] = qpow(Q(mons[n].first, p), mons[m].first) * qpow(Q(mons[n].second, p), mons[m].second);
  Mat C = inverse(V);
  std::vector<Poly2> phi(d, Poly2(p + 1, std::vector<Q>(p + 1, Q(0))));
  for (int k = 0; k < d; k++)
    for (int m = 0; m < d; m++) phi[k][mons[m].first][mons[m].second] = C[m][k];
  auto sq = [&](const Poly2 &P) {   // int over the unit square
    Q s(0);
    for (size_t a = 0; a < P.size(); a++)
      for (size_t b = 0; b < P[a].size(); b++)
        if (!P[a][b].zero()) s += P[a][b] * Q(1, (i128)(a + 1) * (i128)(b + 1));
    return s;
  };
  Mat M = zeros(d, d), Dc[2] = {zeros(d, d), zeros(d, d)};
  for (int i = 0; i < d; i++)
    for (int j = 0; j < d; j++) {
      M[i][j] = sq(pmul(phi[i], phi[j]));
      for (int c = 0; c < 2; c++) Dc[c][i][j] = sq(pmul(pderiv(phi[i], c), phi[j]));
    }
  Mat Mi = inverse(M);
  // faces E W N S: K-local segment A -> B, neighbour offset, normal
  const int FA[4][2] = {{1, 0}, {0, 0}, {0, 1}, {0, 0}}, FB[4][2] = {{1, 1}, {0, 1}, {1, 1}, {1, 0}};
  const int OFF[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}}, NRM[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  const int OPP[4] = {1, 0, 3, 2};
  Mat Em[4], Ep[4];
  for (int f = 0; f < 4; f++) {
    Em[f] = zeros(d, d);
    Ep[f] = zeros(d, d);
    Q x0(FA[f][0]), y0(FA[f][1]), dx(FB[f][0] - FA[f][0]), dy(FB[f][1] - FA[f][1]);
    std::vector<Poly1> pm(d), pn(d);
    for (int i = 0; i < d; i++) {
      pm[i] = restrict_line(phi[i], x0, dx, y0, dy);
      pn[i] = restrict_line(phi[i], x0 - Q(OFF[f][0]), dx, y0 - Q(OFF[f][1]), dy);
    }
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) {
        Em[f][i][j] = integrate1(p1mul(pm[i], pm[j]));
        Ep[f][i][j] = integrate1(p1mul(pm[i], pn[j]));
      }
  }
  // q of an element: S0_c (its own u, all four faces' E^- terms: u+ = 0 at
  // walls keeps them) and P_f,c (the neighbour across face f)
  Mat S0[2], Pf[4][2];
  for (int c = 0; c < 2; c++) {
    Mat t = zeros(d, d);
    axpy(t, Q(-1), Dc[c]);
    for (int f = 0; f < 4; f++)
      if (NRM[f][c]) axpy(t, Q(NRM[f][c], 2), Em[f]);
    S0[c] = mul(Mi, t);
    for (int f = 0; f < 4; f++) {
      Mat e = zeros(d, d);
      if (NRM[f][c]) axpy(e, Q(NRM[f][c], 2), Ep[f]);
      Pf[f][c] = mul(Mi, e);
    }
  }
  QuadTable T;
  T.p = p;
  T.d = d;
  T.blocks.assign((size_t)28 * d * d, 0.0);
  auto put = [&](int b, const Mat &A) {
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) T.blocks[((size_t)b * d + i) * d + j] = A[i][j].to_double();
  };
  // rhs_K = M^-1 [ sum_c T_c q_Kc + sum_{f open} 1/2 n_fc Ep_f q_{N_f,c} ],
  // T_c = -Dc + sum_{f open} 1/2 n_fc Em_f (k = D on open faces, units D = 1);
  // the perpendicular neighbours of N_f drop out exactly (n_f . n_perp = 0)
  auto Tc = [&](int code, int c) {
    Mat t = zeros(d, d);
    axpy(t, Q(-1), Dc[c]);
    for (int f = 0; f < 4; f++)
      if (((code >> f) & 1) && NRM[f][c]) axpy(t, Q(NRM[f][c], 2), Em[f]);
    return t;
  };
  for (int code = 0; code < 16; code++) {
    Mat A = zeros(d, d);
    for (int c = 0; c < 2; c++) {
      Mat t = mul(Tc(code, c), S0[c]);
      for (int f = 0; f < 4; f++)
        if (((code >> f) & 1) && NRM[f][c]) axpy(t, Q(NRM[f][c], 2), mul(Ep[f], Pf[OPP[f]][c]));
      for (int i = 0; i < d; i++)
        for (int j = 0; j < d; j++) A[i][j] += t[i][j];
    }
    put(code, mul(Mi, A));
  }
  for (int f = 0; f < 4; f++)
    for (int oo = 0; oo < 2; oo++) {   // opposite face open (oo = 1) or closed
      const int code = (1 << f) | (oo ? (1 << OPP[f]) : 0);
      Mat A = zeros(d, d);
      for (int c = 0; c < 2; c++) {
        Mat t = mul(Tc(code, c), Pf[f][c]);
        if (NRM[f][c]) axpy(t, Q(NRM[f][c], 2), mul(Ep[f], S0[c]));
        for (int i = 0; i < d; i++)
          for (int j = 0; j < d; j++) A[i][j] += t[i][j];
      }
      put(oo ? 16 + f : 20 + f, mul(Mi, A));
    }
  for (int f = 0; f < 4; f++) {
    Mat A = zeros(d, d);
    for (int c = 0; c < 2; c++)
      if (NRM[f][c]) axpy(A, Q(NRM[f][c], 2), mul(Ep[f], Pf[f][c]));
    put(24 + f, mul(Mi, A));
  }
  const int AB[6][2] = {{0, 0}, {1, 0}, {0, 1}, {2, 0}, {1, 1}, {0, 2}};
  T.W.assign((size_t)6 * d, 0.0);
  for (int q = 0; q < 6; q++)
    for (int k = 0; k < d; k++) {
      Poly2 m(AB[q][0] + 1, std::vector<Q>(AB[q][1] + 1, Q(0)));
      m[AB[q][0]][AB[q][1]] = Q(1);
      T.W[(size_t)q * d + k] = sq(pmul(m, phi[k])).to_double();
    }
  T.init.assign(d, 0.0);
  T.cw.assign(d, 0.0);
  for (int i = 0; i < d; i++) {
    Q s(0);
    for (int j = 0; j < d; j++) s += Mi[i][j] * peval(phi[j], Q(1, 2), Q(1, 2));
    T.init[i] = s.to_double();
    T.cw[i] = peval(phi[i], Q(1, 2), Q(1, 2)).to_double();
  }
  T.minv.assign((size_t)d * d, 0.0);
  T.phic.assign((size_t)d * (p + 1) * (p + 1), 0.0);
  for (int i = 0; i < d; i++) {
    for (int j = 0; j < d; j++) T.minv[(size_t)i * d + j] = Mi[i][j].to_double();
    for (int a = 0; a <= p; a++)
      for (int b = 0; b <= p; b++) T.phic[((size_t)i * (p + 1) + a) * (p + 1) + b] = phi[i][a][b].to_double();
  }
  return T;
}

// ---- quads under ABSORB (Eq. (4)) ----------------------------------------------
// outer faces: h_u = 0 (no u-flux term at all) and h_q = k q- . n (full, not
// halved).  Layout: self [16 code][16 outer][d][d], then N [4 f][3 opposite
// state: 0 closed, 1 open, 2 outer][2 far face outer][d][d], then NN [4][d][d].
struct QuadRef {
  int d = 0;
  Mat Mi, Dc[2], Em[4], Ep[4];
};

static void quad_ref(int p, QuadRef &R) {
  const int d = (p + 1) * (p + 1);
  std::vector<std::pair<int, int>> mons;
  for (int b = 0; b <= p; b++)
    for (int a = 0; a <= p; a++) mons.push_back({a, b});
  Mat V = zeros(d, d);
  for (int n = 0; n < d; n++)
    for (int m = 0; m < d; m++)
      V[n][m] = qpow(Q(mons[n].first, p), mons[m].first) * qpow(Q(mons[n].second, p), mons[m].second);
  Mat C = inverse(V);
  std::vector<Poly2> phi(d, Poly2(p + 1, std::vector<Q>(p + 1, Q(0))));
  for (int k = 0; k < d; k++)
    for (int m = 0; m < d; m++) phi[k][mons[m].first][mons[m].second] = C[m][k];
  auto sq = [&](const Poly2 &P) {
    Q s(0);
    for (size_t a = 0; a < P.size(); a++)
      for (size_t b = 0; b < P[a].size(); b++)
        if (!P[a][b].zero()) s += P[a][b] * Q(1, (i128)(a + 1) * (i128)(b + 1));
    return s;
  };
  Mat M = zeros(d, d);
  R.Dc[0] = zeros(d, d);
  R.Dc[1] = zeros(d, d);
  for (int i = 0; i < d; i++)
    for (int j = 0; j < d; j++) {
      M[i][j] = sq(pmul(phi[i], phi[j]));
      for (int c = 0; c < 2; c++) R.Dc[c][i][j] = sq(pmul(pderiv(phi[i], c), phi[j]));
    }
  R.Mi = inverse(M);
  const int FA[4][2] = {{1, 0}, {0, 0}, {0, 1}, {0, 0}}, FB[4][2] = {{1, 1}, {0, 1}, {1, 1}, {1, 0}};
  const int OFF[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  for (int f = 0; f < 4; f++) {
    R.Em[f] = zeros(d, d);
    R.Ep[f] = zeros(d, d);
    Q x0(FA[f][0]), y0(FA[f][1]), dx(FB[f][0] - FA[f][0]), dy(FB[f][1] - FA[f][1]);
    std::vector<Poly1> pm(d), pn(d);
    for (int i = 0; i < d; i++) {
      pm[i] = restrict_line(phi[i], x0, dx, y0, dy);
      pn[i] = restrict_line(phi[i], x0 - Q(OFF[f][0]), dx, y0 - Q(OFF[f][1]), dy);
    }
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) {
        R.Em[f][i][j] = integrate1(p1mul(pm[i], pm[j]));
        R.Ep[f][i][j] = integrate1(p1mul(pm[i], pn[j]));
      }
  }
  R.d = d;
}

std::vector<double> build_quad_absorb(int p) {
  if (p < 1 || p > 2) throw std::runtime_error("quadrilateral elements: degree must be 1 or 2");
  QuadRef R;
  quad_ref(p, R);
  const int d = R.d, NRM[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}}, OPP[4] = {1, 0, 3, 2};
  // q of an element with outer face set `out`: S0 (own u) and P_f (across face f)
  auto S0 = [&](int out, int c) {
    Mat t = zeros(d, d);
    axpy(t, Q(-1), R.Dc[c]);
    for (int f = 0; f < 4; f++)
      if (!((out >> f) & 1) && NRM[f][c]) axpy(t, Q(NRM[f][c], 2), R.Em[f]);
    return mul(R.Mi, t);
  };
  auto Pf = [&](int f, int c) {
    Mat e = zeros(d, d);
    if (NRM[f][c]) axpy(e, Q(NRM[f][c], 2), R.Ep[f]);
    return mul(R.Mi, e);
  };
  auto Tc = [&](int code, int out, int c) {
    Mat t = zeros(d, d);
    axpy(t, Q(-1), R.Dc[c]);
    for (int f = 0; f < 4; f++) {
      if (!NRM[f][c]) continue;
      if ((code >> f) & 1) axpy(t, Q(NRM[f][c], 2), R.Em[f]);
      if ((out >> f) & 1) axpy(t, Q(NRM[f][c]), R.Em[f]);   // ABSORB q-flux: k q- . n
    }
    return t;
  };
  std::vector<double> T((size_t)(256 + 24 + 4) * d * d, 0.0);
  auto put = [&](size_t b, const Mat &A) {
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) T[(b * d + i) * d + j] = A[i][j].to_double();
  };
  for (int code = 0; code < 16; code++)
    for (int out = 0; out < 16; out++) {
      if (code & out) continue;
      Mat A = zeros(d, d);
      for (int c = 0; c < 2; c++) {
        Mat t = mul(Tc(code, out, c), S0(out, c));
        for (int f = 0; f < 4; f++)
          if (((code >> f) & 1) && NRM[f][c]) axpy(t, Q(NRM[f][c], 2), mul(R.Ep[f], Pf(OPP[f], c)));
        for (int i = 0; i < d; i++)
          for (int j = 0; j < d; j++) A[i][j] += t[i][j];
      }
      put((size_t)code * 16 + out, mul(R.Mi, A));
    }
  for (int f = 0; f < 4; f++)
    for (int os = 0; os < 3; os++)
      for (int far = 0; far < 2; far++) {
        const int code = (1 << f) | (os == 1 ? 1 << OPP[f] : 0), out = os == 2 ? 1 << OPP[f] : 0;
        const int nout = far ? 1 << f : 0;   // the neighbour's far face on the outer square
        Mat A = zeros(d, d);
        for (int c = 0; c < 2; c++) {
          Mat t = mul(Tc(code, out, c), Pf(f, c));
          if (NRM[f][c]) axpy(t, Q(NRM[f][c], 2), mul(R.Ep[f], S0(nout, c)));
          for (int i = 0; i < d; i++)
            for (int j = 0; j < d; j++) A[i][j] += t[i][j];
        }
        put(256 + ((size_t)f * 3 + os) * 2 + far, mul(R.Mi, A));
      }
  for (int f = 0; f < 4; f++) {
    Mat A = zeros(d, d);
    for (int c = 0; c < 2; c++)
      if (NRM[f][c]) axpy(A, Q(NRM[f][c], 2), mul(R.Ep[f], Pf(f, c)));
    put(280 + f, mul(R.Mi, A));
  }
  return T;
}

void point_init_quad(const QuadTable &T, double xi, double eta, double *out) {
  const int p = T.p, d = T.d;
  double phi[16];
  for (int k = 0; k < d; k++) {
    double s = 0.0, xa = 1.0;
    for (int a = 0; a <= p; a++, xa *= xi) {
      double yb = 1.0;
      for (int b = 0; b <= p; b++, yb *= eta) s += T.phic[((size_t)k * (p + 1) + a) * (p + 1) + b] * xa * yb;
    }
    phi[k] = s;
  }
  for (int i = 0; i < d; i++) {
    double s = 0.0;
    for (int j = 0; j < d; j++) s += T.minv[(size_t)i * d + j] * phi[j];
    out[i] = s;
  }
}

void point_init(const Table &T, double xi, double eta, double *out) {
  const int p = T.p, d = T.d;
  const double wt[2] = {eta < xi ? 1.0 : eta > xi ? 0.0 : 0.5, eta > xi ? 1.0 : eta < xi ? 0.0 : 0.5};
  for (int t = 0; t < 2; t++) {
    double phi[16];
    for (int j = 0; j < d; j++) {
      double s = 0.0, xa = 1.0;
      for (int a = 0; a <= p; a++, xa *= xi) {
        double yb = 1.0;
        for (int b = 0; b <= p; b++, yb *= eta) s += T.phic[(((size_t)t * d + j) * (p + 1) + a) * (p + 1) + b] * xa * yb;
      }
      phi[j] = s;
    }
    for (int i = 0; i < d; i++) {
      double s = 0.0;
      for (int j = 0; j < d; j++) s += T.minv[((size_t)t * d + i) * d + j] * phi[j];
      out[t * d + i] = wt[t] * s;
    }
  }
}

std::vector<double> build_absorb(int p) {
  if (p < 1 || p > 3) throw std::runtime_error("absorbing table: degree must be 1..3");
  RefEl R;
  build_ref(R, p);
  const int d = R.d, D2 = 2 * d;
  const int OFF[5][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  std::vector<double> A((size_t)16 * 16 * 5 * D2 * D2, 0.0);
  for (int code = 0; code < 16; code++)
    for (int outer = 1; outer < 16; outer++) {
      if (code & outer) continue;                    // a face is open or outer, not both
      Mat full;
      build_table(R, code, full, outer);
      for (int dj = -1; dj <= 1; dj++)
        for (int di = -1; di <= 1; di++) {
          int o = -1;
          for (int k = 0; k < 5; k++)
            if (OFF[k][0] == di && OFF[k][1] == dj) o = k;
          bool used = (o == 0) || (o > 0 && ((code >> (o - 1)) & 1));
          for (int r = 0; r < D2; r++)
            for (int t = 0; t < 2; t++)
              for (int j = 0; j < d; j++) {
                const Q &q = full[r][tri_index(di, dj, t) * d + j];
                if (o < 0 || !used) {
                  if (o < 0 && !q.zero()) throw std::runtime_error("absorbing: corner coupling is not zero");
                  continue;
                }
                A[((((size_t)code * 16 + outer) * 5 + o) * D2 + r) * D2 + t * d + j] = q.to_double();
              }
        }
    }
  return A;
}

}  // namespace dgop
