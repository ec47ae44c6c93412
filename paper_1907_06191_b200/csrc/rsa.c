/*
 * rsa.c -- random sequential adsorption of disks (input generation only; see
 * paper_1907_06191_b200/substrate.py).  No DG arithmetic lives here.
 *
 * rsa_place: try to place each radius (in the given order) at the next
 * candidate centres taken from `uniforms` (pairs in [0,1), consumed in order,
 * shared across radii), rejecting candidates that overlap an already placed
 * disk; rasterise every accepted disk into `mask` (pixel centre in the closed
 * disk, reading R16).  Stops when the mask count reaches `target` or the
 * uniforms run out; *radii_done = radii consumed (a radius cut short by the
 * end of the uniforms counts as consumed).  Returns the number of disks placed; *consumed is the
 * number of uniform pairs used; *masked is updated.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct { double x, y, r; int next; } disk_t;

int64_t rsa_place(const double *radii, int64_t nr, double Lx, double Ly, double cell, int max_attempts,
                  const double *uniforms, int64_t nuni, int64_t *consumed,
                  uint8_t *mask, int nx, int ny, double h, int64_t *masked, int64_t target,
                  double *out_xyr, int64_t out_cap,
                  /* existing disks (from earlier calls) */ const double *prev_xyr, int64_t nprev, int64_t *radii_done) {
  int ncx = (int)ceil(Lx / cell), ncy = (int)ceil(Ly / cell);
  int *head = (int *)malloc(sizeof(int) * (size_t)ncx * ncy);
  for (int64_t k = 0; k < (int64_t)ncx * ncy; k++) head[k] = -1;
  int64_t cap = nprev + nr;
  disk_t *D = (disk_t *)malloc(sizeof(disk_t) * (size_t)(cap > 0 ? cap : 1));
  int64_t nd = 0;
  for (int64_t k = 0; k < nprev; k++) {
    double x = prev_xyr[3 * k], y = prev_xyr[3 * k + 1];
    int ci = (int)(x / cell), cj = (int)(y / cell);
    if (ci >= ncx) ci = ncx - 1;
    if (cj >= ncy) cj = ncy - 1;
    D[nd].x = x; D[nd].y = y; D[nd].r = prev_xyr[3 * k + 2];
    D[nd].next = head[cj * ncx + ci];
    head[cj * ncx + ci] = (int)nd;
    nd++;
  }
  int64_t u = *consumed, placed = 0, k = 0;
  for (; k < nr && *masked < target && u < nuni; k++) {
    double r = radii[k];
    for (int a = 0; a < max_attempts && u < nuni; a++, u++) {
      double x = uniforms[2 * u] * Lx, y = uniforms[2 * u + 1] * Ly;
      int ci = (int)(x / cell), cj = (int)(y / cell);
      if (ci >= ncx) ci = ncx - 1;
      if (cj >= ncy) cj = ncy - 1;
      int clear = 1;
      for (int jj = (cj > 0 ? cj - 1 : 0); clear && jj <= (cj + 1 < ncy ? cj + 1 : ncy - 1); jj++)
        for (int ii = (ci > 0 ? ci - 1 : 0); clear && ii <= (ci + 1 < ncx ? ci + 1 : ncx - 1); ii++)
          for (int e = head[jj * ncx + ii]; e >= 0; e = D[e].next) {
            double dx = x - D[e].x, dy = y - D[e].y, rr = r + D[e].r;
            if (dx * dx + dy * dy < rr * rr) { clear = 0; break; }
          }
      if (!clear) continue;
      D[nd].x = x; D[nd].y = y; D[nd].r = r;
      D[nd].next = head[cj * ncx + ci];
      head[cj * ncx + ci] = (int)nd;
      nd++;
      if (placed < out_cap) {
        out_xyr[3 * placed] = x; out_xyr[3 * placed + 1] = y; out_xyr[3 * placed + 2] = r;
      }
      placed++;
      /* rasterise: pixel centres (i+1/2)h within the closed disk */
      int i0 = (int)floor((x - r) / h - 0.5), i1 = (int)ceil((x + r) / h - 0.5);
      int j0 = (int)floor((y - r) / h - 0.5), j1 = (int)ceil((y + r) / h - 0.5);
      if (i0 < 0) i0 = 0;
      if (j0 < 0) j0 = 0;
      if (i1 > nx - 1) i1 = nx - 1;
      if (j1 > ny - 1) j1 = ny - 1;
      for (int j = j0; j <= j1; j++)
        for (int i = i0; i <= i1; i++) {
          double px = (i + 0.5) * h - x, py = (j + 0.5) * h - y;
          if (px * px + py * py <= r * r && !mask[(size_t)j * nx + i]) {
            mask[(size_t)j * nx + i] = 1;
            (*masked)++;
          }
        }
      u++;
      break;
    }
  }
  *consumed = u;
  *radii_done = k;
  free(D);
  free(head);
  return placed;
}
