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
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "operator.h"

// P3 column form for the ring kernel (round 2): the same V, F_f, N_f values as
// TAB_P3 laid out column by column, so the kernel applies each block as a
// short runtime loop over its non-zero columns (one broadcast shared-memory
// load per two coefficients, all rows of a column at once) instead of ~100 KB
// of straight-line code that overflows the instruction cache.  Layout:
//   V            [D2 cols][D2 rows]
//   per face f:  F_f [NCF][RF rows]  over columns P3COL_CF[f][] and the RF
//                contiguous rows from P3COL_R0F[f] (F_f only touches the
//                triangle that owns face f: checked here),
//                N_f [NCN][D2 rows]  over columns P3COL_CN[f][]
// Lists shorter than NCF / NCN are padded with column 0 and zero coefficients.
static int emit_p3_columns(FILE *f, const std::vector<double> &blk, int D2) {
  auto B = [&](int b, int r, int c) { return blk[((size_t)b * D2 + r) * D2 + c]; };
  const int RF = D2 / 2;
  std::vector<int> cf[4], cn[4];
  int r0f[4], ncf = 0, ncn = 0;
  for (int fb = 0; fb < 4; fb++) {
    int rlo = D2, rhi = -1;
    for (int c = 0; c < D2; c++) {
      bool nzf = false, nzn = false;
      for (int r = 0; r < D2; r++) {
        if (B(1 + fb, r, c) != 0.0) { nzf = true; rlo = std::min(rlo, r); rhi = std::max(rhi, r); }
        if (B(5 + fb, r, c) != 0.0) nzn = true;
      }
      if (nzf) cf[fb].push_back(c);
      if (nzn) cn[fb].push_back(c);
    }
    r0f[fb] = rlo < RF ? 0 : RF;
    if (rhi >= r0f[fb] + RF || rlo < r0f[fb]) {
      fprintf(stderr, "p3 F_%d rows [%d, %d] not within one triangle\n", fb, rlo, rhi);
      return 1;
    }
    ncf = std::max(ncf, (int)cf[fb].size());
    ncn = std::max(ncn, (int)cn[fb].size());
  }
  if (ncf % 2) ncf++;   // the kernel's column loop is unrolled by two
  if (ncn % 2) ncn++;
  std::vector<double> col;
  for (int c = 0; c < D2; c++)
    for (int r = 0; r < D2; r++) col.push_back(B(0, r, c));
  for (int fb = 0; fb < 4; fb++) {
    for (int k = 0; k < ncf; k++)
      for (int r = 0; r < RF; r++) col.push_back(k < (int)cf[fb].size() ? B(1 + fb, r0f[fb] + r, cf[fb][k]) : 0.0);
    for (int k = 0; k < ncn; k++)
      for (int r = 0; r < D2; r++) col.push_back(k < (int)cn[fb].size() ? B(5 + fb, r, cn[fb][k]) : 0.0);
  }
  fprintf(f, "// P3 column form (V, then per face F_f over NCF columns x %d rows and N_f over NCN columns x %d rows)\n",
          RF, D2);
  fprintf(f, "constexpr int P3COL_NCF = %d, P3COL_NCN = %d, P3COL_RF = %d, P3COL_N = %zu;\n", ncf, ncn, RF, col.size());
  fprintf(f, "constexpr int P3COL_R0F[4] = {%d, %d, %d, %d};\n", r0f[0], r0f[1], r0f[2], r0f[3]);
  for (int pass = 0; pass < 2; pass++) {
    fprintf(f, "__device__ const unsigned char P3COL_%s[4][%d] = {", pass ? "CN" : "CF", pass ? ncn : ncf);
    for (int fb = 0; fb < 4; fb++) {
      const std::vector<int> &v = pass ? cn[fb] : cf[fb];
      const int n = pass ? ncn : ncf;
      fprintf(f, "{");
      for (int k = 0; k < n; k++) fprintf(f, "%d%s", k < (int)v.size() ? v[k] : 0, k + 1 < n ? ", " : "");
      fprintf(f, "}%s", fb < 3 ? ", " : "");
    }
    fprintf(f, "};\n");
  }
  fprintf(f, "#define DGK_P3COL_DATA \\\n");
  for (size_t i = 0; i < col.size(); i++) fprintf(f, "%a,%s", col[i], (i % 8 == 7) ? " \\\n" : " ");
  fprintf(f, "\n__device__ const double P3COL_D[%zu] = {DGK_P3COL_DATA};\n\n", col.size());
  return 0;
}

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
    return emit_p3_columns(f, blk, D2);
  }
  // the transposed operator L^T (adjoint moments, opts.adjoint) has the same
  // structure: self blocks transposed, and the block across open face f is the
  // transposed neighbour block of the OPPOSITE face, (N_opp(f))^T
  for (int tr = 0; tr < 2; tr++) {
    fprintf(f, "__host__ __device__ constexpr double tab_p%d%s(int b, int r, int c) {\n  switch ((b * %d + r) * %d + c) {\n",
            p, tr ? "t" : "", D2, D2);
    int nnz = 0;
    for (int b = 0; b < NB; b++)
      for (int r = 0; r < D2; r++)
        for (int c = 0; c < D2; c++) {
          const int bs = (tr && b >= 5 && b <= 8) ? 5 + ((b - 5) ^ 1) : b;   // E<->W, N<->S
          double v = tr ? blk[((size_t)bs * D2 + c) * D2 + r] : blk[((size_t)b * D2 + r) * D2 + c];
          if (v != 0.0) {
            fprintf(f, "    case %d: return %a;\n", (b * D2 + r) * D2 + c, v);
            nnz++;
          }
        }
    fprintf(f, "    default: return 0.0;\n  }\n}\n");
    fprintf(f, "// nnz(P%d%s) = %d\n\n", p, tr ? "t" : "", nnz);
  }
  return 0;
}

// N4 quads: 28 blocks of (p+1)^2 (0..15 self[code], 16+f N_f opposite open,
// 20+f N_f opposite closed, 24+f NN_f), as tab_q<p>(b, r, c)
static int emit_quad(FILE *f, int p) {
  dgop::QuadTable T = dgop::build_quad(p);
  const int d = T.d;
  fprintf(f, "// Q%d: 28 blocks of %dx%d (0-15 self[code], 16+f N_f opp. open, 20+f N_f opp. closed, 24+f NN_f)\n", p, d, d);
  // tr = 1: the transposed operator L^T (adjoint moments): self blocks
  // transposed; the blocks of face f and of the far pixel in direction f are
  // the transposed blocks of the OPPOSITE direction (variant ids kept: the
  // kernel picks the face variant by the far pixel's state under L^T)
  for (int tr = 0; tr < 2; tr++) {
    fprintf(f, "__host__ __device__ constexpr double tab_q%d%s(int b, int r, int c) {\n  switch ((b * %d + r) * %d + c) {\n",
            p, tr ? "t" : "", d, d);
    int nnz = 0;
    for (int b = 0; b < 28; b++)
      for (int r = 0; r < d; r++)
        for (int c = 0; c < d; c++) {
          const int bs = (tr && b >= 16) ? 16 + ((b - 16) / 4) * 4 + (((b - 16) % 4) ^ 1) : b;   // E<->W, N<->S
          const double v = tr ? T.blocks[((size_t)bs * d + c) * d + r] : T.blocks[((size_t)b * d + r) * d + c];
          if (v != 0.0) {
            fprintf(f, "    case %d: return %a;\n", (b * d + r) * d + c, v);
            nnz++;
          }
        }
    fprintf(f, "    default: return 0.0;\n  }\n}\n// nnz(Q%d%s) = %d\n\n", p, tr ? "t" : "", nnz);
  }
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
