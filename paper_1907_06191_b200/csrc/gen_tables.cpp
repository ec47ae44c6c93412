// gen_tables.cpp -- build-time generator: runs K0 (operator.cpp) and writes
// tables.inc, the composite operator as compile-time constants for the
// kernels.  Because k_f enters Eq. (7) linearly and each neighbour
// block only exists when its face is open, the 16 code variants decompose
// exactly as
//     A[code][self] = V + sum_{f open} F_f,    A[code][f] = N_f  (f open)
// (checked here entry by entry: exactly on the dyadic P1/P2 values, to 1e-12
// on the rounded P3 values).
// Block ids: 0 = V, 1..4 = F_E, F_W, F_N, F_S, 5..8 = N_E, N_W, N_N, N_S,
// 9 + code = the full self block A[code][self] of that open-face code (used
// by the kernels through a warp-uniform switch: 116 MACs per P1 pixel).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "operator.h"

static int emit(FILE *f, int p) {
  dgop::Table T = dgop::build(p);
  const int D2 = 2 * T.d;
  auto A = [&](int code, int o, int r, int c) { return T.A[(((size_t)code * 5 + o) * D2 + r) * D2 + c]; };
  const int NB = 9 + 16;
  std::vector<double> blk((size_t)NB * D2 * D2, 0.0);
  for (int r = 0; r < D2; r++)
    for (int c = 0; c < D2; c++) {
      blk[(0 * D2 + r) * D2 + c] = A(0, 0, r, c);
      for (int fb = 0; fb < 4; fb++) {
        blk[((1 + fb) * D2 + r) * D2 + c] = A(1 << fb, 0, r, c) - A(0, 0, r, c);
        blk[((5 + fb) * D2 + r) * D2 + c] = A(15, 1 + fb, r, c);
      }
      for (int code = 0; code < 16; code++) blk[((9 + code) * D2 + r) * D2 + c] = A(code, 0, r, c);
    }
  // verify the decomposition for every code (exact: dyadic values, short mantissas)
  for (int code = 0; code < 16; code++)
    for (int r = 0; r < D2; r++)
      for (int c = 0; c < D2; c++) {
        double s = blk[(0 * D2 + r) * D2 + c];
        for (int fb = 0; fb < 4; fb++)
          if ((code >> fb) & 1) s += blk[((1 + fb) * D2 + r) * D2 + c];
        // exact for the dyadic P1/P2 values; P3 values are rounded doubles
        const double tol = p <= 2 ? 0.0 : 1e-12 * (1.0 + std::fabs(A(code, 0, r, c)));
        if (std::fabs(s - A(code, 0, r, c)) > tol) {
          fprintf(stderr, "p%d code %d self (%d,%d) not linear\n", p, code, r, c);
          return 1;
        }
        for (int fb = 0; fb < 4; fb++) {
          double want = ((code >> fb) & 1) ? blk[((5 + fb) * D2 + r) * D2 + c] : 0.0;
          if (A(code, 1 + fb, r, c) != want) { fprintf(stderr, "p%d code %d nb %d not fixed\n", p, code, fb); return 1; }
        }
      }
  fprintf(f, "// P%d: blocks of %dx%d (0 V, 1-4 F_E..F_S, 5-8 N_E..N_S, 9+code self[code]), units D/h^2\n", p, D2, D2);
  if (p == 3) {
    // P3 (400-entry blocks): a constexpr array (a switch of this size makes
    // the device compiler's constant folding explode)
    fprintf(f, "#define DGK_TAB_P3_DATA \\\n");
    int nnz = 0;
    for (size_t i = 0; i < blk.size(); i++) {
      fprintf(f, "%a,%s", blk[i], (i % 8 == 7) ? " \\\n" : " ");
      nnz += blk[i] != 0.0;
    }
    fprintf(f, "\nconstexpr double TAB_P3_H[%d] = {DGK_TAB_P3_DATA};\n", NB * D2 * D2);
    fprintf(f, "__device__ constexpr double TAB_P3_D[%d] = {DGK_TAB_P3_DATA};\n", NB * D2 * D2);
    fprintf(f, "__host__ __device__ constexpr double tab_p3(int b, int r, int c) {\n#ifdef __CUDA_ARCH__\n"
               "  return TAB_P3_D[(b * %d + r) * %d + c];\n#else\n  return TAB_P3_H[(b * %d + r) * %d + c];\n#endif\n}\n",
            D2, D2, D2, D2);
    fprintf(f, "// nnz(P3) = %d\n\n", nnz);
    return 0;
  }
  fprintf(f, "__host__ __device__ constexpr double tab_p%d(int b, int r, int c) {\n  switch ((b * %d + r) * %d + c) {\n", p, D2, D2);
  int nnz = 0;
  for (int b = 0; b < NB; b++)
    for (int r = 0; r < D2; r++)
      for (int c = 0; c < D2; c++) {
        double v = blk[((size_t)b * D2 + r) * D2 + c];
        if (v != 0.0) {
          fprintf(f, "    case %d: return %a;\n", (b * D2 + r) * D2 + c, v);
          nnz++;
        }
      }
  fprintf(f, "    default: return 0.0;\n  }\n}\n");
  fprintf(f, "// nnz(P%d) = %d\n\n", p, nnz);
  return 0;
}

// N4 quads: 28 blocks of (p+1)^2 (0..15 self[code], 16+f N_f opposite open,
// 20+f N_f opposite closed, 24+f NN_f), as tab_q<p>(b, r, c)
static int emit_quad(FILE *f, int p) {
  dgop::QuadTable T = dgop::build_quad(p);
  const int d = T.d;
  fprintf(f, "// Q%d: 28 blocks of %dx%d (0-15 self[code], 16+f N_f opp. open, 20+f N_f opp. closed, 24+f NN_f)\n", p, d, d);
  fprintf(f, "__host__ __device__ constexpr double tab_q%d(int b, int r, int c) {\n  switch ((b * %d + r) * %d + c) {\n", p, d, d);
  int nnz = 0;
  for (int b = 0; b < 28; b++)
    for (int r = 0; r < d; r++)
      for (int c = 0; c < d; c++) {
        const double v = T.blocks[((size_t)b * d + r) * d + c];
        if (v != 0.0) {
          fprintf(f, "    case %d: return %a;\n", (b * d + r) * d + c, v);
          nnz++;
        }
      }
  fprintf(f, "    default: return 0.0;\n  }\n}\n// nnz(Q%d) = %d\n\n", p, nnz);
  return 0;
}

int main(int argc, char **argv) {
  if (argc < 2) { fprintf(stderr, "usage: gen_tables out.inc\n"); return 2; }
  FILE *f = fopen(argv[1], "w");
  if (!f) return 2;
  fprintf(f, "// tables.inc -- GENERATED at build time by gen_tables (K0, operator.cpp). Do not edit.\n#pragma once\n\n");
  int rc = emit(f, 1) || emit(f, 2) || emit(f, 3) || emit_quad(f, 1) || emit_quad(f, 2);
  fclose(f);
  return rc;
}
