/*
 * dgdiff.h -- C-ABI of the B200-native hot path of arXiv 1907.06191
 * ("DG-CUDA" diffusion covariance).  Paper = PAPER.md, cited as P:<line>.
 *
 * The library advances a batch of independent Dirac point sources
 * by explicit SSP-RK3 steps of the paper's DG discretisation (Eq. (7),
 * P:160-169; fluxes P:192-204; pixel mesh P:211) on a masked pixel substrate
 * (axon pixels = k 0, Eq. (5)), reduces every density to its mass,
 * first and second moments about its source point and combines them
 * into the 2x2 covariance Sigma of the averaged Gaussian.
 *
 * Conventions (all functions):
 *  - grid units are the caller's: pixel side h, diffusivity D, time dt;
 *    pixel (i, j) covers [ih, (i+1)h] x [jh, (j+1)h]; arrays [ny][nx] are
 *    row-major with i (x) fastest;
 *  - every pointer argument is a HOST pointer; the library copies inputs and
 *    writes outputs into caller buffers; the caller keeps ownership;
 *  - a handle owns all of its device memory and, when nranks > 1, its NCCL
 *    communicator; a handle is not thread-safe; separate handles are
 *    independent;
 *  - nothing throws across the ABI; every fallible call returns a
 *    dgdiff_status and leaves a message for dgdiff_last_error();
 *  - there is no CPU fallback: without a CUDA device dgdiff_create fails
 *    with DGDIFF_E_CUDA.
 */
#ifndef DGDIFF_H
#define DGDIFF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dgdiff_s *dgdiff_t; /* opaque */

typedef enum {
  DGDIFF_OK = 0,
  DGDIFF_E_ARG = 1,        /* bad argument (sizes, degree, NULL, unsupported option) */
  DGDIFF_E_SOURCE = 2,     /* a source pixel is outside the grid or masked */
  DGDIFF_E_UNSTABLE = 3,   /* dt > dgdiff_dt_max(degree, h, D) */
  DGDIFF_E_NONFINITE = 4,  /* NaN/Inf in the moments */
  DGDIFF_E_STATE = 5,      /* call out of order, or delta != nsteps*dt */
  DGDIFF_E_DEGENERATE = 6, /* a density with m00 <= 0 */
  DGDIFF_E_CUDA = 7,       /* CUDA runtime error / no device */
  DGDIFF_E_NCCL = 8,       /* NCCL missing or failed */
  DGDIFF_E_NOMEM = 9       /* device allocation failed */
} dgdiff_status;

typedef struct {
  int32_t precision;      /* 64 (default) or 32: arithmetic type of the state and
                             of the stencil sum; moments always accumulate in fp64 */
  int32_t outer_bc;       /* 0 = REFLECT (default): the outer square acts as an
                             axon wall (reading R9).  1 = ABSORB, Eq. (4)
                             (P:67-70): u = 0 on the outer square (ghost u+ = -u-);
                             mass leaves the grid.  ABSORB runs on the default
                             ring kernel only (kernel 1/2 or temporal_steps 2 ->
                             E_ARG), for every element type */
  int32_t centering;      /* 0 = shift each density by its source point (default,
                             reading R12); 1 = by its own mean */
  int32_t temporal_steps; /* 0 = library choice (K2); 1 = one launch per RK
                             stage (K2); 2 = fused step (K3: one whole SSP-RK3
                             step per launch, temporal blocking over the 3
                             stages, lock-step rows; P1 triangles); 3 = fused
                             step with decoupled warp roles (K3b, fp64 P1,
                             bit-identical to K2); 4 = wavefront step (K3c:
                             one launch per step, the K2 items of all three
                             stages ordered as a skewed wavefront with
                             per-item completion counters; P1/P2 triangles,
                             fp64/fp32, bit-identical to K2); 5 = stage pair
                             (K3d: stage 1 on K2, stages 2 and 3 fused in one
                             launch with U2 kept in shared memory: 5 state
                             passes per step instead of 8; P1/P2 triangles,
                             fp64/fp32, bit-identical to K2).  Other degrees /
                             elements use K2; 2..5 exclude ABSORB, windows,
                             quads, P3; 4 and 5 need kernel 0 */
  int32_t device;         /* CUDA device ordinal; -1 = current device */
  int32_t rank, nranks;   /* source sharding: rank takes the contiguous block
                             [rank*n/nranks, (rank+1)*n/nranks) of every batch
                             (with windows != 0: that block of the batch in
                             Morton order, so every rank's sources stay
                             spatially compact; every rank sorts the same list) */
  const void *nccl_id;    /* ncclUniqueId* (128 bytes): the handle joins an
                             NCCL communicator of nranks ranks (with nranks == 1
                             a one-rank communicator).  NULL with nranks > 1 =
                             LOGICAL rank: no communicator; the handle solves
                             its shard only and its [n][6] moment table holds
                             zeros in the other ranks' rows; dgdiff_covariance
                             then fails with E_STATE and the caller sums the
                             ranks' tables (dgdiff_source_moments) and calls
                             dgdiff_covariance_table (the same sum NCCL would
                             do: exact, so Sigma is bitwise that of nranks = 1) */
  int32_t keep_density;   /* 1: keep the final states of the last source chunk for
                             dgdiff_get_density (tests); 0 (default) */
  int32_t max_chunk;      /* max sources resident per chunk; 0 = fit device memory */
  void *stream;           /* cudaStream_t to launch on; NULL = a library stream */
  int32_t kernel;         /* stage kernel variant: 0 = default (= 3); 1 = v1,
                             operator table in global memory, global loads;
                             2 = v2, operator as compile-time immediates, global
                             loads; 3 = v3, row-marching shared-memory ring fed
                             by bulk TMA.  Results agree to rounding; the
                             state layout (and so the source-group size) differs:
                             v1/v2 16-byte lanes; v3 16-byte lanes for P1,
                             8-byte lanes for P2, P3 and the quadrilaterals.
                             v1/v2 exist for the P1/P2 triangles only */
  int32_t mixture_radius; /* R > 0: accumulate the mixture density grid
                             on the displacement lattice [-R, R]^2 (pixel
                             units) during dgdiff_solve_batch, for
                             dgdiff_mixture; 0 (default) = off */
  int32_t windows;        /* N1 active windows ("the outer
                             boundary is not reached"): 1 = sort the batch
                             spatially (Morton order) before sharding, into
                             source groups, and, at every RK stage, compute only the
                             rows / column strips inside each group's source
                             box grown by one pixel per stage so far.  Exact:
                             the 5-point operator spreads support by one pixel
                             per stage, so everything outside is identically
                             zero (results agree with windows = 0 to
                             rounding; moments are returned in input order).
                             Ring kernel only (kernel 1/2, temporal_steps 2 ->
                             E_ARG).  2 = the same, with each box's growth
                             also capped at K sigma = K sqrt(2 D t) / h
                             (+ one stencil reach), K = 20 (P1), 25 (Q1), 30 (P2),
                             40 (Q2), 45 (P3): the DG density's tails are
                             below fp64 rounding there (DESIGN R23),
                             so results agree with the whole-grid solve to
                             ~1e-14 but are no longer bitwise equal.
                             0 (default) = whole grid */
  int32_t element;        /* 0 (default) = two P_p triangles per pixel;
                             1 = one Q_p quadrilateral per pixel (N4, the north
                             star's "Q2"; degree 1 or 2): tensor Lagrange basis
                             on (a/p, b/p), dof b (p+1) + a, same fluxes; the
                             composite operator is a 9-point cross.  Default
                             ring kernel only (REFLECT or ABSORB); densities
                             are [ny][nx][(p+1)^2] */
  int32_t adjoint;        /* 1 = moments by the adjoint (round 2): for the
                             linear scheme m_s = w_s^T P(dt L)^N u0_s =
                             (P(dt L^T)^N w_s)^T u0_s, and the moment weights
                             w_s about the source point are combinations of the
                             six weight fields of 1, x, y, x^2, xy, y^2 about a
                             nearby origin; so dgdiff_solve_batch evolves those
                             fields (30 origins on a lattice over the sources'
                             box: 3 groups of 64 lanes for P1, 6 of 32 for P2)
                             with the transposed composite operator (ring
                             kernel with transposed tables over the sources'
                             domain of dependence; kernel = 1: the v1 table
                             kernel) and reads every source's moments from
                             them at its pixel: a few groups of work for any
                             number of sources.  Same Sigma as the
                             per-source solve up to rounding (the centring
                             subtraction loses ~log10(box^2 / m_20) digits).
                             Pixel sources and N4 sub-pixel points.  The
                             fields are fp64 also on fp32 handles (ring kernel).
                             P1/P2 triangles or Q1/Q2 (ring kernel), REFLECT,
                             no windows, mixture, temporal blocking or
                             densities (E_ARG);
                             0 (default) = per-source forward solves */
} dgdiff_opts;

/* Fill *o with the defaults above. */
void dgdiff_opts_default(dgdiff_opts *o);

/* Create a solver for one substrate.
 *  mask   [ny][nx] uint8, 1 = axon pixel (k = 0, Eq. (5)), 0 = extracellular
 *         (k = D); copied.
 *  h, D   pixel side and extracellular diffusivity k0 (> 0).
 *  degree Lagrange degree p of the triangle elements (Eq. (8); "p <= 3
 *         suffices"): 1, 2 or 3 (P3: default ring kernel only; its
 *         non-dyadic operator entries are rounded once to the state type).
 * Builds the operator tables (host), the open-face code of every pixel and the
 * active-pixel index, copies them to the device; when nranks > 1 initialises
 * NCCL from opts->nccl_id.  On failure *out is NULL. */
dgdiff_status dgdiff_create(dgdiff_t *out, const uint8_t *mask, int32_t nx, int32_t ny, double h,
                            double D, int32_t degree, const dgdiff_opts *opts);

/* Step 1 of the scheme of P:239-243 for a batch of sources.
 *  sources [n][2] int32 pixel indices (i, j); the Dirac sits at the pixel
 *          centre ((i+1/2)h, (j+1/2)h); every rank passes the full list.
 *  dt, nsteps  SSP-RK3 step and step count; the solve horizon is
 *          Delta = nsteps*dt.  dt > dgdiff_dt_max -> E_UNSTABLE.
 * On return (stream-ordered; the call itself does not synchronise with the
 * device except for its host->device source copy) the per-source moments of
 * this rank's shard are in the device moment table. */
dgdiff_status dgdiff_solve_batch(dgdiff_t, const int32_t *sources, int64_t n, double dt,
                                 int64_t nsteps);

/* N4: as dgdiff_solve_batch, for point sources anywhere in the extracellular
 * pixels ("m points chosen uniformly in Omega_e").
 *  points [n][2] (x, y) in physical units, 0 <= x < nx*h, 0 <= y < ny*h;
 *         copied.  The point belongs to pixel (floor(x/h), floor(y/h)) (a
 *         point on a pixel edge goes to the pixel above / right of it:
 *         DESIGN.md reading R21); its Dirac is L2-projected onto the triangle
 *         containing it (L: eta < xi, U: eta > xi; on the diagonal split 1/2 -
 *         1/2 as for pixel centres, R10) -- for quadrilaterals (element = 1)
 *         onto the pixel's single element -- and its moments are taken about
 *         the point itself (R12).  A point at a pixel centre reproduces
 *         dgdiff_solve_batch exactly.  E_SOURCE: non-finite, outside the grid
 *         or in an axon pixel.  The mixture lattice (dgdiff_mixture) is not
 *         accumulated for point sources (-> E_STATE there). */
dgdiff_status dgdiff_solve_batch_points(dgdiff_t, const double *points, int64_t n, double dt,
                                        int64_t nsteps);

/* Steps 2-4 of P:243-265: centre + normalise each density, mix, and return
 * the mixture's covariance.  delta must equal nsteps*dt of the last solve
 * (relative 1e-12) -> else E_STATE.  When nranks > 1 this is the only
 * collective: one ncclAllReduce(sum, fp64) of the zero-padded [n][6] moment
 * table, after which every rank reduces the table in source order, so Sigma
 * is bitwise identical for every nranks.  sigma[4] row-major (exactly
 * symmetric), mu[2] (nullable) the mixture mean.  Synchronises. */
dgdiff_status dgdiff_covariance(dgdiff_t, double delta, double sigma[4], double mu[2]);

/* K5 alone: Sigma and mu (as dgdiff_covariance, the handle's centering) of a
 * caller-provided moment table mom [n][6] (host, copied), e.g. the sum of
 * the zero-padded tables of the logical ranks of one batch.  Errors:
 * E_ARG (NULL, n < 1), E_DEGENERATE, E_NONFINITE.  Synchronises. */
dgdiff_status dgdiff_covariance_table(dgdiff_t, const double *mom, int64_t n, double sigma[4], double mu[2]);

/* The mixture model u = (1/m) sum_i u_i of the centred, normalised densities
 * sampled at the displacement nodes (dx, dy) in [-R, R]^2 (pixel
 * units, R = opts.mixture_radius): u_i(dx, dy) = value of the DG solution of
 * source i at the centre of pixel (i_s + dx, j_s + dy) (the mean of the two
 * triangles' traces there; 0 on axon pixels and outside the grid), divided
 * by its m00; and the least-squares residual of Eq. (9)
 *   residual = sum_{dx,dy} [ N((dx h, dy h); mu, Sigma) - u(dx, dy) ]^2
 * with N the Gaussian density of the last dgdiff_covariance.
 * grid [(2R+1)][(2R+1)] row-major (dy outer), either pointer nullable.
 * Needs mixture_radius > 0 at create and dgdiff_covariance -> else E_STATE.
 * When nranks > 1 the grid is all-reduced (NCCL) first.  Synchronises. */
dgdiff_status dgdiff_mixture(dgdiff_t, double *grid, double *residual);

/* Monte-Carlo cross-check (the paper's MC comparison): K walkers
 * per source start at the source pixel centres and take nsteps steps of
 * length l = sqrt(4 D delta / nsteps) in uniform directions; a step
 * whose segment enters an axon pixel or leaves the grid is rejected (the
 * walker stays).  Needs l < h (nsteps >= 4 D delta / h^2) -> else E_ARG.
 * Philox4x32-10 counter-based randomness keyed by (seed, walker): runs are
 * reproducible.  Walker w belongs to source w mod n.  sigma[4] (row-major,
 * symmetric) and mu[2] of the pooled displacements, se[3] the standard errors
 * of sxx, sxy, syy from 32 batches of walkers (each batch spans all sources);
 * disp (nullable) [n*K][2] the displacements in pixel units.  Synchronises. */
dgdiff_status dgdiff_mc_covariance(dgdiff_t, const int32_t *sources, int64_t n, int32_t walkers_per_source,
                                   int64_t nsteps, double delta, uint32_t seed, double sigma[4], double mu[2],
                                   double se[3], double *disp);

/* Per-source moments [n][6] = m00 m10 m01 m20 m11 m02 of the last solve,
 * about each source point; rows of other ranks' shards are zero until
 * dgdiff_covariance has run.  Synchronises. */
dgdiff_status dgdiff_source_moments(dgdiff_t, double *out);

/* Final state of source `src` of the last solve, in the canonical fp64 layout
 * [ny][nx][2][d] (triangle 0 = L (0,0),(1,0),(1,1); 1 = U (0,0),(1,1),(0,1);
 * nodes: vertices, then edge nodes of v0v1, v1v2, v2v0, then interior);
 * quadrilaterals: [ny][nx][(p+1)^2], dof b (p+1) + a at the node (a/p, b/p).
 * Requires keep_density and src in this rank's last chunk -> else E_STATE. */
dgdiff_status dgdiff_get_density(dgdiff_t, int64_t src, double *out);

/* Largest stable SSP-RK3 step for the triangle elements: 2.5127453 / rho_p *
 * h^2 / D with rho_1 = 60, rho_2 = 192.7953, rho_3 = 462.37 (DESIGN.md
 * reading R8; pinned against the assembled operator's spectrum); 0 for an
 * unsupported degree.  The quadrilaterals use rho_Q1 = 32, rho_Q2 = 130.7
 * (R22) inside dgdiff_solve_batch. */
double dgdiff_dt_max(int32_t degree, double h, double D);

/* Thread-local message of the last failing call ("" if none). */
const char *dgdiff_last_error(void);

/* NULL-safe. */
void dgdiff_destroy(dgdiff_t);

/* ---- host-only introspection (no device needed) ------------------------ */

/* The composite stencil of the semi-discrete operator after eliminating q,
 * in units of D/h^2, for degree p (1, 2):  A [16][5][2d][2d] with
 * code bit0 = E open, bit1 = W, bit2 = N, bit3 = S and offsets
 * 0 self, 1 E (+1,0), 2 W (-1,0), 3 N (0,+1), 4 S (0,-1); rows = outputs,
 * columns = the neighbour's dofs in canonical order (triangle-major).
 *  W    [2][6][d]: int over the unit pixel's triangle of xi^a eta^b N_j,
 *       (a,b) = 00,10,01,20,11,02.
 *  init [2][d]:  the projected Dirac at the pixel centre times h^2.
 * Any pointer may be NULL. */
dgdiff_status dgdiff_operator_table(int32_t degree, double *A, double *W, double *init);

/* Composite blocks of pixels with absorbing outer faces (outer_bc = 1,
 * Eq. (4)): A [16][16][5][2d][2d] indexed [code][outer] with outer the 4-bit
 * set of the pixel's faces on the outer square (same bit order as code); only
 * entries with code & outer == 0 and outer != 0 are used.  Units D/h^2. */
dgdiff_status dgdiff_absorb_table(int32_t degree, double *A);

/* Values at the pixel centre (1/2, 1/2) of the unit pixel's basis functions,
 * cw [2][d] (triangle-major, canonical order): the mixture node weights. */
dgdiff_status dgdiff_centre_weights(int32_t degree, double *cw);

/* N4 quadrilateral Q_p elements (degree 1 or 2, host K0, exact rationals
 * rounded once): the 9-point-cross composite operator, blocks [28][d][d],
 * d = (p+1)^2 (dof b (p+1) + a at the node (a/p, b/p)); ids 0..15 the self
 * block of open-face code c, 16+f the face-f neighbour block when the
 * opposite face is open, 20+f when it is closed, 24+f the block of the pixel
 * two steps away in direction f (f = E, W, N, S).  Units D/h^2. */
dgdiff_status dgdiff_quad_table(int32_t degree, double *blocks);

/* Source shard of `rank` out of `nranks` for a batch of n sources. */
void dgdiff_shard(int64_t n, int32_t rank, int32_t nranks, int64_t *begin, int64_t *end);

typedef struct {
  int64_t launches;        /* kernels launched by this handle so far */
  int64_t stage_launches;  /* of which RK-stage (or temporal-blocked) launches */
  double stage_ms;         /* summed device time of those launches (CUDA events on
                              the launch stream), if timing is enabled */
  double stage_bytes;      /* algorithmic HBM bytes of those launches */
  double stage_flops;      /* algorithmic flops of those launches (structural MACs) */
  int64_t n_active;        /* extracellular pixels */
  int64_t chunk;           /* sources per chunk of the last solve */
  int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by the last solve+covariance */
  int64_t env_overrides;   /* tuning knobs taken from the environment (always 0
                              in product builds: they ignore the environment) */
  int64_t tuning_build;    /* 1 if the library was built with -DDGDIFF_TUNING */
  double dom_ms;           /* the dominant kernel alone (K2: every stage launch;
                              K3d: the stage-pair launches): summed device time
                              (timing enabled), algorithmic HBM bytes, launches */
  double dom_bytes;
  int64_t dom_launches;
} dgdiff_stats_t;

/* Enable (1) / disable (0) CUDA-event timing of the stage launches. */
dgdiff_status dgdiff_set_timing(dgdiff_t, int32_t enable);
dgdiff_status dgdiff_get_stats(dgdiff_t, dgdiff_stats_t *out);
dgdiff_status dgdiff_reset_stats(dgdiff_t);

#ifdef __cplusplus
}
#endif
#endif /* DGDIFF_H */
