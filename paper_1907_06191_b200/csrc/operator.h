// operator.h -- K0 host precompute (see operator.cpp).
#pragma once
#include <vector>

namespace dgop {

struct Table {
  int p = 0, d = 0;
  std::vector<double> A;    // [16][5][2d][2d], units D/h^2, exact dyadic
  std::vector<double> W;    // [2][6][d] moment weights on the unit pixel
  std::vector<double> init; // [2][d] projected Dirac at the pixel centre, units 1/h^2
  std::vector<int> nnz;     // [16][5] structural non-zeros per block
  std::vector<double> cw;   // [2][d] N_j at the pixel centre (1/2, 1/2) (mixture node values)
  std::vector<double> minv; // [2][d][d] M_T^-1 on the unit pixel (rounded from exact)
  std::vector<double> phic; // [2][d][p+1][p+1] monomial coefficients of N_j (xi^a eta^b)
};

// Projected Dirac at the pixel-local point (xi, eta) in [0,1)^2 (N4 sub-pixel
// sources; generalises reading R10): u_T = w_T M_T^-1 N_T(xi, eta), w = 1 on
// the triangle containing the point (L: eta < xi, U: eta > xi), 1/2 on each
// if it lies on the diagonal.  out[2][d], units 1/h^2.
void point_init(const Table &T, double xi, double eta, double *out);

// Throws std::runtime_error on failure (unsupported degree, non-dyadic entry,
// non-zero corner coupling, rational overflow).
Table build(int p);

// N4: quadrilateral Q_p elements, one per pixel (p = 1, 2).  The composite
// operator (q eliminated) is a 9-point cross: after exact elimination
//   A[code][self]                 16 variants (open-face code of the pixel)
//   A[f] = N_f[opposite face open] 2 variants per face (the opposite face's
//                                  E^- term meets the lifted jump of face f)
//   A[ff] = NN_f                   fixed (the neighbour's far face)
// blocks[28][d][d], ids 0..15 self[code], 16+f N_f (opposite open), 20+f N_f
// (opposite closed), 24+f NN_f; units D/h^2; d = (p+1)^2, dof b (p+1) + a
// for the node (a/p, b/p).  Corner couplings vanish exactly (checked).
struct QuadTable {
  int p = 0, d = 0;
  std::vector<double> blocks;  // [28][d][d]
  std::vector<double> W;       // [6][d] moment weights on the unit pixel
  std::vector<double> init;    // [d] projected central Dirac, units 1/h^2
  std::vector<double> cw;      // [d] N_k(1/2, 1/2)
  std::vector<double> minv;    // [d][d] M^-1 on the unit pixel
  std::vector<double> phic;    // [d][p+1][p+1] coefficients of xi^a eta^b in N_k
};
QuadTable build_quad(int p);
// quads under ABSORB (Eq. (4)): self [16 code][16 outer][d][d], then N [4 f][3
// opposite-face state: 0 closed, 1 open, 2 outer][2 far face outer][d][d],
// then NN [4][d][d]; units D/h^2
std::vector<double> build_quad_absorb(int p);
// projected Dirac at the pixel-local point (xi, eta): u = M^-1 N(xi, eta), out[d]
void point_init_quad(const QuadTable &T, double xi, double eta, double *out);

// Composite blocks of pixels with absorbing outer faces (outer_bc = ABSORB,
// Eq. (4)): A[code][outer][5][2d][2d] (outer = faces on the outer square; zero
// unless code & outer == 0 and outer != 0), units D/h^2.
std::vector<double> build_absorb(int p);

}  // namespace dgop
