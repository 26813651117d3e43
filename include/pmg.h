/*
 * pmg.h -- C ABI of libpmg.so, the B200 (sm_100a) implementation of the
 * pressure-correction solve path of arXiv:1307.2036 (reference package
 * `panelmg`, /root/reference/pkg/src/panelmg).
 *
 * Every entry point takes plain pointers and sizes; device pointers are
 * CUDA global-memory addresses, `stream` is a cudaStream_t passed as
 * void* (NULL = legacy default stream).  Every call returns 0 on success
 * or a negative status; pmg_last_error() returns the message of the most
 * recent failure on the calling thread.  Calls are stream-ordered and
 * never synchronise the host, except where a scalar is returned to a
 * HOST pointer (documented per call).
 *
 * Field layout on the device (one "part" = the columns one worker owns):
 * red/black split, horizontal index fastest.  Cell (i, j, k) of a part
 * with local i in [-1, nx], j in [-1, ny] (-1 and nx/ny are halo) lives at
 *
 *   field[c * cstride + (j + 1) * nz * plane + k * plane + PMG_OFF + (i >> 1)]
 *   with colour c = (i + j + parity) & 1, parity = (i0 + j0) & 1,
 *   plane = pitch = roundup(PMG_OFF + nx/2 + 1, 8), cstride = (ny+2)*nz*plane,
 *
 * i.e. red cells ((i+j) even in GLOBAL indices, reference smoother.py:66)
 * and black cells are two separate [ny+2][nz][pitch] arrays (rows j
 * slowest, then vertical levels k, then the horizontal index).  Use
 * pmg_level_layout() for pitch/plane/cstride and pmg_level_field_doubles()
 * (= 2 * cstride) for the allocation size.
 */
#ifndef PMG_H
#define PMG_H

#ifdef __cplusplus
extern "C" {
#endif

#define PMG_OK 0
#define PMG_ERR_VALUE -1    /* maps to ValueError (shape / layout / config)     */
#define PMG_ERR_CUDA -2     /* CUDA runtime failure -> RuntimeError              */
#define PMG_ERR_PIVOT -3    /* zero pivot -> ZeroPivotError (tridiag.py:20)      */
#define PMG_ERR_INTERNAL -4
#define PMG_ERR_BREAKDOWN -5 /* CG breakdown -> BreakdownError (krylov.py:29)    */

#define PMG_OFF 4           /* offset (doubles) of h = 0 inside a row            */

typedef struct pmg_level pmg_level;   /* opaque */

/*
 * One grid level of one part.  Replaces the coefficient set-up of
 * PanelOperator.__init__ (stencil.py:90-114), GridFactors/build_factors
 * (geometry.py:141-240) and the pivot factorisation of _Block
 * (smoother.py:89-99).  2-D factor arrays are HOST pointers covering the
 * part's owned columns, stored with j (y) slowest:
 *   wx   [ny][nx+1]   wx[j][i]  = face between local columns i-1 and i
 *   wy   [ny+1][nx]   wy[j][i]  = face between local rows j-1 and j
 *   av, vh, sumw [ny][nx]
 * 1-D arrays: dr[nz], vprof[nz+1], volprof[nz].  Arrays are copied; if
 * every 2-D array is constant the level runs the uniform-coefficient
 * kernels (1-D diagonal / pivot tables, reference arithmetic order).
 */
typedef struct pmg_level_desc {
    int nx, ny, nz;            /* owned columns of this part, vertical cells   */
    int i0, j0;                /* global origin of the part                    */
    double omega2;             /* omega^2                  (stencil.py:101)   */
    double vcoef;              /* omega^2 * lambda^2       (stencil.py:102)   */
    const double *dr, *vprof, *volprof;
    const double *wx, *wy, *av, *vh, *sumw;
} pmg_level_desc;

int pmg_version(void);
/* number of kernel launches this library has issued (or recorded into a
 * CUDA graph) since load; launchers with a reduction count two. */
long long pmg_launch_count(void);
/* tracing mode (the reference times the iteration
 * loop with wall time only, multigrid.py:321,329): while on (1), the
 * drivers push NVTX ranges -- solve, cycle / CG iteration, level, halo
 * exchange (level ranges mark the cycle graph's capture) -- and time every
 * cycle's graph replay on the device with a CUDA event pair
 * (pmg_hier_cycle_times / pmg_phier_cycle_times).  Off (0) by default. */
int pmg_set_tracing(int on);
int pmg_get_tracing(void);
const char *pmg_last_error(void);
int pmg_device_sm_count(int device, int *out);

int pmg_level_create(const pmg_level_desc *desc, pmg_level **out);
/* owned columns and vertical cells of a level */
int pmg_level_dims(const pmg_level *lvl, int *nx, int *ny, int *nz);
int pmg_level_destroy(pmg_level *lvl);
long long pmg_level_field_doubles(const pmg_level *lvl);
int pmg_level_layout(const pmg_level *lvl, int *pitch, long long *plane,
                     long long *cstride, int *parity, int *uniform);
/* copy of the 1-D tables the uniform kernels use (diag[nz], band[nz+1],
 * invd[nz]); fails with PMG_ERR_VALUE on a variable-coefficient level. */
int pmg_level_tables(const pmg_level *lvl, double *diag, double *band, double *invd);
/* pivot table of a variable-coefficient level: computes the per-column
 * invd of smoother.py:93-99 into the level (device, field layout).
 * Called automatically on first use; exposed for set-up timing. */
int pmg_level_prepare(pmg_level *lvl, void *stream);

/* ---- layout conversion: reference (nx, ny, nz) C-order, k fastest
 *      (field.py:3-10 owned block) <-> device split layout -------------- */
int pmg_from_ref_layout(const pmg_level *lvl, const double *src_dev, double *field,
                        void *stream);
int pmg_to_ref_layout(const pmg_level *lvl, const double *field, double *dst_dev,
                      void *stream);
/* the same for the columns i0 <= i < i1 only: i is the slowest index of the
 * reference block, so the slab is the contiguous range [i0 ny nz, i1 ny nz)
 * of src_dev / dst_dev (which still point at the whole block) -- a host
 * transfer can be converted slab by slab while the next slab is in flight
 * (pipeline.py). */
int pmg_from_ref_layout_slab(const pmg_level *lvl, const double *src_dev, double *field, int i0,
                             int i1, void *stream);
int pmg_to_ref_layout_slab(const pmg_level *lvl, const double *field, double *dst_dev, int i0,
                           int i1, void *stream);

/* host (nx, ny, nz) reference-layout block <-> device field through a
 * device staging buffer of nx*ny*nz doubles (Field upload / download of
 * SURVEY 8b; scatter_owned / gather_owned per part, partition.py:243-264).
 * Stream-ordered; the host buffer should be pinned for asynchrony. */
int pmg_field_upload(const pmg_level *lvl, const double *host, double *field,
                     double *staging_dev, void *stream);
int pmg_field_download(const pmg_level *lvl, const double *field, double *host,
                       double *staging_dev, void *stream);
/* Device field of a level (both colour arrays, halo ring and padding:
 * pmg_level_field_doubles() doubles), zero-filled; pmg_field_free releases
 * it (NULL is a no-op).  Callers may equally pass their own allocations
 * (e.g. torch tensors) of that size to every entry point. */
int pmg_field_alloc(const pmg_level *lvl, double **out);
int pmg_field_free(double *field);
/* whole allocation (halo included): fill with a value / copy
 * (DistField.fill / copy, partition.py:128-137) */
int pmg_fill(const pmg_level *lvl, double *field, double value, void *stream);
int pmg_copy(const pmg_level *lvl, double *dst, const double *src, void *stream);
/* copy a w x h block of columns (all k) between two parts, e.g. the
 * coarse-level folding of collect / distribute (partition.py:194-240):
 * dst (di + i, dj + j, k) = src (si + i, sj + j, k), local indices, the halo
 * ring (-1, nx / ny) included; colours follow each part's global parity. */
int pmg_copy_block(const pmg_level *src_lvl, const double *src, const pmg_level *dst_lvl,
                   double *dst, int si, int sj, int di, int dj, int w, int h, void *stream);

/* ---- operator: PanelOperator.apply / residual (stencil.py:127-165) --- */
/* out = A u on owned cells; u halo must be current. */
int pmg_apply(const pmg_level *lvl, const double *u, double *out, void *stream);
/* r = f - A u.  r may be NULL (norm only).  If norm2_dev != NULL,
 * norm2_dev[0] = sum of r^2 over owned cells (fixed reduction order;
 * scratch holds pmg_partials_size() doubles). */
int pmg_residual(const pmg_level *lvl, const double *f, const double *u, double *r,
                 double *scratch, double *norm2_dev, void *stream);
/* q = A p and dot_dev[0] = p.q over owned cells (CG, krylov.py:139-140). */
int pmg_apply_dot(const pmg_level *lvl, const double *p, double *q, double *scratch,
                  double *dot_dev, void *stream);
/* residual fused with the children-sum restriction (multigrid.py:278-282):
 * coarse_f = R (f - A u), r never stored. */
int pmg_residual_restrict(const pmg_level *fine, const pmg_level *coarse,
                          const double *f, const double *u, double *coarse_f,
                          void *stream);
/* the same right after a black half-sweep with exact line solves and
 * rho = 1 (the V-cycle's pre-smoothing): the black residual is then zero,
 * so only the red children are summed -- 14 N bytes instead of 18 N.
 * Fast mode, uniform coefficients, nx a multiple of 4; PMG_ERR_VALUE
 * otherwise.  Equal to pmg_residual_restrict up to the black cells'
 * rounding-level residual. */
int pmg_residual_restrict_red(const pmg_level *fine, const pmg_level *coarse,
                              const double *f, const double *u, double *coarse_f,
                              void *stream);
int pmg_residual_restrict_red_ok(const pmg_level *fine);
/* norm2_dev[0] = sum over the RED owned cells of (f - A u)^2 (the
 * convergence norm after an exact black half-sweep, rho = 1, whose black
 * residual is zero); same eligibility as pmg_residual_restrict_red. */
int pmg_red_residual_norm(const pmg_level *lvl, const double *f, const double *u,
                          double *scratch, double *norm2_dev, void *stream);

/* ---- line smoother: LineSmoother.half_sweep (smoother.py:122-182) ---- */
/* mode 0 (default): fast k-segmented column solve (uniform levels; agrees
 * with the sequential Thomas algorithm to ~1e-15 relative); mode 1: exact
 * sequential Thomas recurrence, bit-identical to the reference.  Levels
 * with variable coefficients always use the exact solver. */
int pmg_set_smoother_mode(int mode);
int pmg_get_smoother_mode(void);
int pmg_half_sweep(const pmg_level *lvl, double *u, const double *f, int color,
                   double rho, int zero_start, int neighbors_zero, double post_scale,
                   void *stream);
/* the same half-sweep restricted to a tile region: the 32-cell strips
 * rx0 + s * rxs (s < rxn) of the relaxed colour's rows and the rows
 * ry0 + t * rys (t < ryn).  A boundary-first multi-part sweep relaxes the
 * strips and rows that hold the part's boundary columns first, exchanges
 * their halos while the interior region relaxes, with the
 * same values as one whole-part call.  Fast smoother mode, on uniform
 * levels or on variable levels the band kernel runs (nz = 128, rows of a
 * multiple of 64 cells, eight rows or more; rows must then be consecutive,
 * rys = 1, and neighbors_zero needs rho = 1 without zero_start) --
 * pmg_half_sweep_region_ok -- else PMG_ERR_VALUE. */
int pmg_half_sweep_region_ok(const pmg_level *lvl);
int pmg_half_sweep_region(const pmg_level *lvl, double *u, const double *f, int color, double rho,
                          int zero_start, int neighbors_zero, double post_scale, int rx0, int rxs,
                          int rxn, int ry0, int rys, int ryn, void *stream);
/* red half sweep (rho = 1) fused with the convergence residual of the
 * iterate it relaxes: reads u, writes the relaxed red values into the red
 * array of u_new (u_new's black array is not touched; u_new != u), and
 * norm2_dev[0] = sum over u's RED owned cells of (f - A u)^2 (fixed order,
 * scratch: pmg_partials_size() doubles).  After a V-cycle whose last
 * half-sweep relaxed black lines exactly (rho = 1) the black residual is
 * zero, so this is the next cycle's first half-sweep and the previous
 * cycle's ||f - A u||^2 in one pass (multigrid.py:322-324 + smoother.py:
 * 184-186).  Fast mode, uniform coefficients, nz a multiple of 16
 * (<= 128); PMG_ERR_VALUE otherwise. */
int pmg_half_sweep_res(const pmg_level *lvl, const double *u, double *u_new, const double *f,
                       double *scratch, double *norm2_dev, void *stream);
int pmg_half_sweep_res_ok(const pmg_level *lvl);

/* z = M^-1 r, symmetric red-black block SSOR from zero for a part that is
 * its own neighbour (LineSmoother.ssor_apply, smoother.py:224-244): red
 * (zero start, no neighbours), black (zero start, x (2 - rho)), red, each
 * followed by pmg_halo_self.  If rz_dev != NULL also rz_dev[0] = <r, z>
 * (scratch: pmg_partials_size() doubles). */
int pmg_ssor_apply(const pmg_level *lvl, const double *r, double *z, double rho,
                   int periodic_x, int periodic_y, double *scratch, double *rz_dev,
                   void *stream);

/* ---- transfers (multigrid.py:209-268) ------------------------------- */
/* coarse = weight * sum of the 4 children (weight 1: V-cycle, 0.25: mean) */
int pmg_restrict(const pmg_level *fine, const pmg_level *coarse, const double *fine_f,
                 double *coarse_f, double weight, void *stream);
/* fine (+)= P coarse (9-3-3-1 bilinear); coarse halo incl. corners current.
 * add = 0: overwrite owned cells, add = 1: u += P e (multigrid.py:287-290). */
int pmg_prolong(const pmg_level *fine, const pmg_level *coarse, const double *coarse_u,
                double *fine_u, int add, void *stream);
/* fine += P coarse: pmg_prolong with add = 1 (SURVEY 8b's pmg_prolong_add) */
int pmg_prolong_add(const pmg_level *fine, const pmg_level *coarse, const double *coarse_u,
                    double *fine_u, void *stream);
/* same, restricted to the colours in color_mask (1 red, 2 black, 3 both):
 * with rho = 1 the post-smoothing red half-sweep overwrites every red cell
 * without reading it, so the V-cycle prolongs into black cells only. */
int pmg_prolong_colors(const pmg_level *fine, const pmg_level *coarse, const double *coarse_u,
                       double *fine_u, int add, int color_mask, void *stream);


/* ---- halos (partition.py:158-191) ----------------------------------- */
/* Fill the whole halo ring of a part that is its own neighbour (one worker
 * per direction): periodic_x/y wrap, otherwise mirror the adjacent owned
 * value.  Two-phase semantics incl. corners. */
int pmg_halo_self(const pmg_level *lvl, double *field, int periodic_x, int periodic_y,
                  void *stream);
/* Pack / unpack one face strip (both colours, all k) for an exchange with
 * another part.  face: 0 = -x (i = 0), 1 = +x (i = nx-1), 2 = -y (j = 0),
 * 3 = +y (j = ny-1).  x faces span j in [0, ny); y faces span i in
 * [-1, nx] (extended range: corners, phase 2 of partition.py:181-190).
 * Buffer length: pmg_face_doubles(). unpack writes the halo strip on the
 * same side (face 0 -> i = -1, ...); mirror = 1 copies the part's own
 * adjacent owned strip instead of buf (physical boundary). */
long long pmg_face_doubles(const pmg_level *lvl, int face);
int pmg_pack_face(const pmg_level *lvl, const double *field, int face, double *buf,
                  void *stream);
int pmg_unpack_face(const pmg_level *lvl, double *field, int face, const double *buf,
                    int mirror, void *stream);

/* ---- reductions and vector updates (partition.py:138-155, 267-286) -- */
/* scratch size (doubles) every reduction entry point may use */
long long pmg_partials_size(void);
/* out_dev[0] = ||a||^2 over owned cells (pmg_dot(a, a)) */
int pmg_norm2(const pmg_level *lvl, const double *a, double *scratch, double *out_dev,
              void *stream);
/* out_dev[0] = a.b over owned cells (deterministic order) */
int pmg_dot(const pmg_level *lvl, const double *a, const double *b, double *scratch,
            double *out_dev, void *stream);
/* full-allocation BLAS-1 (halo included, like DistField.add_scaled):
 * y = y + a x ; y = x + b y */
int pmg_axpy(long long n, double a, const double *x, double *y, void *stream);
int pmg_xpby(long long n, const double *x, double b, double *y, void *stream);
/* CG update (krylov.py:143-146) fused: u += alpha p (skipped if u is NULL);
 * r -= alpha q (full allocation) and rr_dev[0] = ||r||^2 over owned cells.  alpha is
 * read from DEVICE memory as alpha_num[0] / alpha_den[0] so the step
 * needs no host round trip. */
int pmg_cg_update(const pmg_level *lvl, const double *alpha_num, const double *alpha_den,
                  const double *p, const double *q, double *u, double *r,
                  double *scratch, double *rr_dev, void *stream);
/* u += (alpha_num/alpha_den) p; p = z + (beta_num/beta_den) p in one pass
 * (full allocation): the iterate update of CG iteration k deferred into the
 * direction update of iteration k+1.  z = NULL: only u += alpha p. */
int pmg_cg_step(long long n, const double *alpha_num, const double *alpha_den,
                const double *beta_num, const double *beta_den, const double *z, double *p,
                double *u, void *stream);
/* p = z + (beta_num[0]/beta_den[0]) p over the full allocation. */
int pmg_cg_direction(long long n, const double *beta_num, const double *beta_den,
                     const double *z, double *p, void *stream);

/* ---- batched tridiagonal solves (paper Alg. 3; reference tridiag.py:59-100) --
 * nsys independent systems of n unknowns, stored system-fastest (element k
 * of system s at k * nsys + s; device pointers): diagonal a, superdiagonal
 * b and subdiagonal c (n - 1 rows used; may be NULL when n = 1), right-hand
 * side f, solution x.  work: pmg_thomas_work_doubles(n, nsys) device
 * doubles.  One thread per system, the reference's operation order
 * (bit-identical to its scalar solve).  PMG_ERR_PIVOT when a pivot falls
 * below 1e-300 in magnitude (tridiag.py:79-90); *bad_row is the first such
 * row over all systems, else -1.  Synchronises the stream. */
int pmg_thomas_batch(int n, long long nsys, const double *a, const double *b, const double *c,
                     const double *f, double *x, double *work, int *bad_row, void *stream);
long long pmg_thomas_work_doubles(int n, long long nsys);

/* ---- device-resident drivers (multigrid.py:271-330, krylov.py:88-167) --
 * For one part that is its own neighbour in both directions (one GPU per
 * process; halos periodic or mirror per axis).  The hierarchy keeps the
 * level handles (not owned; they must outlive it) and allocates the coarse
 * iterates / right-hand sides and reduction scratch.  Same operation
 * sequence as the Python drivers (bit-identical results). */
typedef struct pmg_hier pmg_hier;     /* opaque */
typedef struct pmg_mg_desc {
    int nu_pre, nu_post;       /* V(nu_pre, nu_post)           (multigrid.py:54-84) */
    int coarse_sweeps;         /* red-black sweeps on the coarsest level             */
    double rho;                /* overrelaxation weight, (0, 2)                      */
    int periodic_x, periodic_y;
    /* 1: lagged convergence norm -- each cycle's ||f - A u|| is summed by
     * the next cycle's first red half-sweep (pmg_half_sweep_res; the new
     * red values go to a second red array, so the converged iterate is
     * never touched).  Needs rho = 1, nu_pre, nu_post >= 1, two levels and
     * pmg_half_sweep_res_ok(levels[0]); ignored otherwise.  Same iterates
     * bit for bit; the history omits the black cells' rounding-level
     * residual. */
    int lagged_norm;
    /* 1: the pre-smoothed residual is restricted from its red cells only
     * (pmg_residual_restrict_red) where the level allows it; needs rho = 1
     * and nu_pre >= 1, ignored otherwise. */
    int red_restrict;
} pmg_mg_desc;
/* levels[0] finest ... levels[nlev-1] coarsest, each halving nx and ny.
 * PMG_ERR_VALUE for a periodic axis along which some level is one column
 * wide: every cell is then its own neighbour through the wrap, and the
 * red-black identities this driver's cycle rests on (no zero fill of the
 * coarse iterates, black-only prolongation, red-only restriction, the lagged
 * norm) do not hold -- use fewer levels, or the Python driver, which runs
 * the reference's plain op sequence on such hierarchies.  The multi-part
 * pmg_phier_create refuses them likewise. */
int pmg_hier_create(const pmg_level *const *levels, int nlev, const pmg_mg_desc *desc,
                    pmg_hier **out);
int pmg_hier_destroy(pmg_hier *hier);
/* one V-cycle on u (halo current) for right-hand side f (multigrid.py:271-294);
 * first = 1: u is zero on entry but unfilled (rho = 1, nu_pre >= 1) */
int pmg_vcycle(pmg_hier *hier, double *u, const double *f, int first, void *stream);
/* u = 0; V-cycles until ||f - A u|| / ||f|| < eps or maxiter (multigrid.py:297-330).
 * hist[0..iters] (HOST, maxiter + 1 doubles) receives the residual norms;
 * non-convergence is reported in *converged, not as an error.  Synchronises
 * the stream once per cycle; the cycle + norm replays as a CUDA graph. */
int pmg_mg_solve(pmg_hier *hier, const double *f, double *u, double eps, int maxiter,
                 double *hist, int *iters, int *converged, void *stream);
/* kernels per replay of the cycle graph captured for (f, u, first); -1 if
 * none (launch accounting: graph replays issue no host-side launches) */
long long pmg_hier_graph_launches(const pmg_hier *hier, const double *f, const double *u,
                                  int first);
/* cumulative kernels issued by this hierarchy's graph replays */
long long pmg_hier_replayed_launches(const pmg_hier *hier);
/* device milliseconds of each V-cycle of the last pmg_mg_solve run with
 * tracing on: copies min(count, cap) values to ms, returns the count (0 when
 * that solve ran untraced), -1 on a null handle */
int pmg_hier_cycle_times(const pmg_hier *hier, double *ms, int cap);
/* preconditioned CG from u = 0 (krylov.py:88-167): precond 1 = SSOR(rho),
 * 0 = identity; tau as the reference (tiny-residual cut-off).  work: device
 * buffer of pmg_pcg_work_doubles() doubles; hist as pmg_mg_solve.
 * PMG_ERR_BREAKDOWN on <p, A p> <= 0 or <r, z> <= 0. */
long long pmg_pcg_work_doubles(const pmg_level *lvl);
int pmg_pcg_solve(const pmg_level *lvl, const double *f, double *u, double eps, int maxiter,
                  double tau, int precond, double rho, int periodic_x, int periodic_y,
                  double *work, double *hist, int *iters, int *converged, void *stream);

/* ---- multi-part drivers (multigrid.py:271-330 over a px x py
 * decomposition; partition.py:158-191 halo exchange, partition.py:267-286
 * reductions) ------------------------------------------------------------
 * A hierarchy over the parts this process owns: all parts of the
 * decomposition (in-process, one device: the exchange is a device copy
 * between parts), or exactly one part per rank with a communicator (the
 * exchange is ncclSend / ncclRecv, the reductions an ncclAllGather of the
 * per-part sums, added in worker order -- the in-process order, so results
 * do not depend on the transport).  Each V-cycle + convergence norm is one
 * CUDA graph replay (halo exchanges and reductions inside it) and one
 * 8-byte host read.  overlap_nx > 0: levels whose parts are at least that
 * wide (and >= 256 columns) relax boundary-first -- the frame regions
 * (pmg_half_sweep_region), then the frame's halo exchange on a second
 * stream while the interior relaxes; same values bit for
 * bit.  Same operation sequence as the Python multi-part driver
 * (multigrid.v_cycle, fused path). */
typedef struct pmg_comm pmg_comm;     /* opaque: an NCCL communicator */
typedef struct pmg_phier pmg_phier;   /* opaque */
typedef struct pmg_part_desc {
    int worker;   /* worker id; with a communicator: this rank */
    int nbr[4];   /* worker across the W, E, S, N face; -1: physical boundary (mirror) */
    int diag[4];  /* worker across the SW, SE, NW, NE corner; >= 0 exactly where both
                   * adjacent faces have a neighbour (the y neighbour of the x neighbour) */
} pmg_part_desc;
/* 1 if libnccl.so.2 can be loaded (resolved at run time; no link dependency) */
int pmg_comm_available(void);
/* NCCL unique id (128 bytes) on one rank, to be broadcast to the others */
int pmg_comm_unique_id(void *id128);
/* communicator of nranks ranks on the current device (ncclCommInitRank) */
int pmg_comm_create(const void *id128, int nranks, int rank, pmg_comm **out);
int pmg_comm_destroy(pmg_comm *comm);
/* The multi-part drivers' halo exchange is ONE phase: the four face strips
 * (the y strips over the extended range, whose end columns carry the
 * sender's mirrored boundary column at a physical x boundary) and the four
 * corner columns from the diagonal parts travel in one NCCL group, between
 * one pack and one unpack launch; the ring then holds what the two-phase
 * exchange of partition.py:158-191 leaves there, bit for bit.
 * pmg_exchange_plan8: its ordered message plan for a part with neighbours
 * nbr8[8] = W, E, S, N, SW, SE, NW, NE (-1 none): ops[3 * n] = 0 send /
 * 1 receive, ops[3 * n + 1] = direction (side of the part), ops[3 * n + 2] =
 * peer worker; at most 16 ops.  Per direction d [send d, recv opposite(d)]:
 * the messages two parts exchange pair up under NCCL's in-order matching per
 * peer for every grid.  Host only.
 * pmg_exchange_plan: one phase of the two-phase plan the Python multi-rank
 * path posts (phase 0: W/E faces, 1: S/N faces including the corners; at
 * most 4 ops, [send a, recv b, send b, recv a]).  Host only. */
int pmg_exchange_plan8(const int *nbr8, int *ops, int *nops);
int pmg_exchange_plan(const int *nbr, int phase, int *ops, int *nops);
/* levels[p * nlev + c]: part p (ascending worker order), level c (finest
 * first, halving nx and ny) */
int pmg_phier_create(const pmg_level *const *levels, int nlev, int nparts,
                     const pmg_part_desc *parts, const pmg_mg_desc *desc, pmg_comm *comm,
                     int overlap_nx, pmg_phier **out);
int pmg_phier_destroy(pmg_phier *hier);
/* mg_solve over every part: f[p], u[p] the parts' fields (multigrid.py:297-330) */
int pmg_phier_mg_solve(pmg_phier *hier, const double *const *f, double *const *u, double eps,
                       int maxiter, double *hist, int *iters, int *converged, void *stream);
/* preconditioned CG from u = 0 over every part (krylov.py:88-167): precond
 * 1 = line SSOR(rho) with the halo exchanges of smoother.py:224-244, 0 =
 * identity; dots added in worker order across parts and ranks; one host
 * read per iteration.  Uses level 0 of the hierarchy (a one-level
 * hierarchy is enough).  PMG_ERR_BREAKDOWN on <p, A p> <= 0 or <r, z> <= 0. */
int pmg_phier_pcg_solve(pmg_phier *hier, const double *const *f, double *const *u, double eps,
                        int maxiter, double tau, int precond, double rho, double *hist, int *iters,
                        int *converged, void *stream);
/* one V-cycle (u halos current; first = 1: u zero on entry, unfilled) */
int pmg_phier_vcycle(pmg_phier *hier, double *const *u, const double *const *f, int first,
                     void *stream);
/* halo exchange of level `level`'s fields (partition.py:158-191) */
int pmg_phier_halo_exchange(pmg_phier *hier, int level, double *const *fields, void *stream);
/* owned-cell dot over every part and rank into *out (device or host-mapped) */
int pmg_phier_dot(pmg_phier *hier, int level, const double *const *a, const double *const *b,
                  double *out, void *stream);
long long pmg_phier_replayed_launches(const pmg_phier *hier);
/* as pmg_hier_cycle_times, for the last pmg_phier_mg_solve */
int pmg_phier_cycle_times(const pmg_phier *hier, double *ms, int cap);
long long pmg_phier_exchanges(const pmg_phier *hier);

#ifdef __cplusplus
}
#endif
#endif /* PMG_H */
