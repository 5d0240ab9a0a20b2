/* mgrit_b200.h — C ABI of the B200-native MGRIT semi-Lagrangian hot path.
 *
 * The reference (mgrit_advect, pure Python + one numba kernel) has no C ABI:
 * its plug-in surface is the Python `Level` operator protocol plus the driver
 * functions.  Each entry point below replaces one reference
 * operation and is cited as  file:line  relative to
 * /root/reference/pkg/src/mgrit_advect/.  The Python mirror of the reference
 * API (paper_2203_13382_b200/) binds these with ctypes; INTEGRATION.md shows
 * the binding a reference maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every `double*` / `int*` argument that is
 *    not documented as "host" is DEVICE memory (cudaMalloc / torch tensor).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - All work is stream-ordered; no entry point synchronises the device.
 *  - Return value: MGRIT_OK, or MGRIT_EINVAL (bad argument, nothing launched)
 *    or MGRIT_ECUDA (launch error; text in mgrit_last_error()).
 *  - Non-finite data seen by a GMRES solve sets *status = 1 (sticky device
 *    flag) and writes a NaN row, mirroring _kernels.py:123-128; the Python
 *    layer raises ValueError -> solve status "diverged" (mgrit.py:363-366).
 *  - State arrays are row-major (n_rows, n_points) fp64, 2D flat index
 *    j*n_x + i (x fastest), exactly as the reference (core.py:51-82).
 */
#ifndef MGRIT_B200_H
#define MGRIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGRIT_ABI_VERSION 3

enum { MGRIT_OK = 0, MGRIT_EINVAL = 2, MGRIT_ECUDA = 3 };
/* launch policy of corrected 1D phases / sweeps: AUTO picks the cluster-split
 * kernels when the level has too few row chains to fill the GPU */
enum { MGRIT_LAUNCH_AUTO = 0, MGRIT_LAUNCH_CTA = 1, MGRIT_LAUNCH_CLUSTER = 2,
       MGRIT_LAUNCH_AUTO_ONE = 3, /* AUTO without the two-CTAs-per-SM phase form */
       /* cluster kernels of exactly 2 / 4 / 8 / 16 CTAs wherever eligible */
       MGRIT_LAUNCH_CLUSTER2 = 4, MGRIT_LAUNCH_CLUSTER4 = 5, MGRIT_LAUNCH_CLUSTER8 = 6,
       MGRIT_LAUNCH_CLUSTER16 = 7 };

/* operator kinds (mgrit.py:34).  MGRIT_KIND_SL covers "fine" and
 * "rediscretized" (plain semi-Lagrangian step); "ideal" is composed on the
 * host from the finer level's operator (mgrit.py:137-141). */
enum { MGRIT_KIND_SL = 0, MGRIT_KIND_CORRECTED = 1, MGRIT_KIND_FORWARD_EULER = 2 };

/* wave speeds traced on the device: reference catalog C1..C5 (core.py:130-153)
 * and BASELINE.json's B2 (1D configs 2-3) / B4 (2D configs 4-5). */
enum { MGRIT_SPEED_C1 = 1, MGRIT_SPEED_C2, MGRIT_SPEED_C3, MGRIT_SPEED_C4,
       MGRIT_SPEED_C5, MGRIT_SPEED_B2, MGRIT_SPEED_B4 };

/* One level's device-resident operator data (replaces Level, mgrit.py:89-167).
 * Departure records are stored as the scaled periodic coordinate
 *     s = mod(x_dep - x_lo, L) / h                    (semi_lagrangian.py:125)
 * from which the east index and eps are re-derived bit-exactly on every
 * application (decompose, semi_lagrangian.py:118-137): 8 B/node/axis instead
 * of the reference's 16 B (int64 east + f64 eps). */
typedef struct mgrit_level_desc {
    int32_t dim;            /* 1 or 2 */
    int32_t n_x;            /* nodes per direction */
    int32_t p;              /* interpolation degree 1, 3, 5 */
    int32_t kind;           /* MGRIT_KIND_* */
    int32_t shared;         /* 1: a single record set for all steps */
    int32_t n_steps;        /* steps on this level */
    int64_t n_points;       /* n_x^dim */
    const double *s_x;      /* [S][n_points]  S = shared ? 1 : n_steps */
    const double *s_y;      /* 2D only, else NULL */
    const double *sig_x;    /* corrected / forward_euler: sigma per step [S][n_points] */
    const double *sig_y;    /* 2D only */
    int32_t gmres_max_iters;/* GmresConfig.max_iters (coarse_correction.py:157-170) */
    int32_t stencil_numba;  /* 1: numba grouping of the D stencil sum (_kernels.py:18-31) */
    double gmres_tol;       /* < 0 : fixed iteration count (tol None) */
    int32_t gmres_lowsync;  /* 0: classic MGS (the reference's loop, default);
                               1: low-synchronisation MGS -- same coefficients in
                               exact arithmetic, one cluster all-reduce per
                               Arnoldi step instead of k+1 (1D cluster kernels;
                               the one-CTA kernels always run classic MGS, whose
                               block reductions are cheaper there) */
    int32_t launch_policy;  /* MGRIT_LAUNCH_*: corrected 1D levels may run one
                               thread-block cluster (2-16 SMs) per row chain */
    int32_t sl2d_separable; /* 2D: set ONLY from mgrit_records_separable() on these
                               very record arrays.  1 = s_x does not depend on the
                               mesh row and s_y not on the column (bitwise), so a
                               plain SL step reads one x-record per column (mesh
                               row 0) and one y-record per row (column 0) instead
                               of 16 B per node, and shares each source row's
                               x-interpolation down a column (bit-identical rows).
                               0 = every node's own records are read. */
    int32_t pad_;
} mgrit_level_desc;

/* ERK tableau for departure tracing (semi_lagrangian.py:46-72); built on the
 * host with the reference's exact double constants. */
typedef struct mgrit_erk_tableau {
    int32_t n_stages;
    int32_t pad;
    double a[6][6];
    double b[6];
    double c[6];
} mgrit_erk_tableau;

int mgrit_abi_version(void);
const char *mgrit_last_error(void);
/* bytes of device scratch the GMRES paths need for `rows` concurrent systems */
int64_t mgrit_gmres_scratch_bytes(const mgrit_level_desc *L, int64_t rows);
/* number of row-systems the batched kernels keep resident at once (their
 * persistent grid size); size GMRES scratch for min(B, this) rows */
int64_t mgrit_resident_rows(const mgrit_level_desc *L);

/* ---------------------------------------------------------------- setup --- */

/* Fine-level departures for steps k = set_first .. set_first+n_sets-1:
 * one backward ERK step from every node over [k*dt, (k+1)*dt]
 * (erk_departures / erk_trace_back, semi_lagrangian.py:75-115, 208-217).
 * With n_sub > 1 the step composes n_sub sub-steps of size dt_sub
 * (departure_policy "erk_substeps", mgrit.py:203-213); t_start = k*dt.
 * Outputs s_x/s_y (see above) and disp = arrival - departure, [n_sets][n_points]. */
int mgrit_erk_departures(int32_t dim, int32_t n_x, int32_t speed_id,
                         const mgrit_erk_tableau *tab, int64_t set_first,
                         int64_t n_sets, double dt, int32_t n_sub, double dt_sub,
                         double *s_x, double *s_y, double *disp_x, double *disp_y,
                         void *stream);

/* Departure coordinates supplied by the caller (any tracing scheme) ->
 * records (DepartureSet*.from_coords, semi_lagrangian.py:175-205). */
int mgrit_departures_from_coords(int32_t dim, int32_t n_x, int64_t n_sets,
                                 const double *cx, const double *cy,
                                 double *s_x, double *s_y, double *disp_x,
                                 double *disp_y, void *stream);

/* Coarse departures by backtracking through m child steps
 * (backtrack_1d/2d, backtracking.py:21-86).  Child k of coarse set n is
 * fine set (child_shared ? 0 : n*m + k). */
int mgrit_backtrack(int32_t dim, int32_t n_x, int32_t m, int64_t n_sets,
                    int32_t child_shared, const double *child_disp_x,
                    const double *child_disp_y, double *s_x, double *s_y,
                    double *disp_x, double *disp_y, void *stream);

/* 2D: *flag (device int32) = 1 iff in every one of the n_sets record sets s_x is
 * bitwise independent of the mesh row and s_y of the mesh column -- true when
 * the x-speed depends on (x, t) only and the y-speed on (y, t) only, as for
 * BASELINE's 2D speed: erk_trace_back (semi_lagrangian.py:75-115) then traces
 * every row / column with identical operands.  Every record is compared.  The
 * only valid source of mgrit_level_desc::sl2d_separable. */
int mgrit_records_separable(int32_t n_x, int64_t n_sets, const double *s_x,
                            const double *s_y, int32_t *flag, void *stream);

/* sigma = phi(eps_coarse, eps_children) [+ sum_k sigma_child_k]
 * (phi_field / sigma_accumulate, coarse_correction.py:92-127; mgrit.py:249-256).
 * child_sig_* NULL on the first coarse level. */
int mgrit_phi_sigma(int32_t dim, int32_t n_x, int32_t p, int32_t m, int64_t n_sets,
                    int32_t child_shared, const double *s_x, const double *s_y,
                    const double *child_s_x, const double *child_s_y,
                    const double *child_sig_x, const double *child_sig_y,
                    double *sig_x, double *sig_y, void *stream);

/* numpy default_rng(seed).random() stream (PCG64 XSL-RR + 53-bit doubles),
 * element k = draw k after the given 128-bit state; pm1 maps to 2x-1
 * (mgrit.py:350-353; BASELINE config 1).  state/inc as hi/lo 64-bit words. */
int mgrit_pcg64_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, int64_t count, int32_t pm1, double *out,
                     void *stream);

/* ------------------------------------------------------------ hot path --- */

/* Batched step operator on B rows (Level.step_batch mgrit.py:152-167,
 * Level.step 135-150, sl_step semi_lagrangian.py:220-253,
 * corrected_coarse_step coarse_correction.py:231-240):
 *   S_b   = Phi_{t_b} U_in[b]          (t_b = t_idx ? t_idx[b] : t_first + b*t_stride)
 *   relax form    (U_sub == NULL): out[b] = S_b + G[b]           (G NULL => + 0.0)
 *   residual form (U_sub != NULL): out[b] = (G[b] + S_b) - U_sub[b]
 * row_sumsq (nullable, [B]): sum of out[b]^2 per row (fixed order);
 *   out may be NULL when row_sumsq is given (norms only, no rows written).
 * gmres_iters (nullable, [B]): Arnoldi steps per corrected row.
 * scratch: >= mgrit_gmres_scratch_bytes(L, B) bytes for corrected levels. */
int mgrit_apply_rows(const mgrit_level_desc *L, int64_t B, const int64_t *t_idx,
                     int64_t t_first, int64_t t_stride,
                     const double *U_in, int64_t ld_in,
                     const double *G, int64_t ld_g,
                     const double *U_sub, int64_t ld_sub,
                     double *out, int64_t ld_out, double *row_sumsq,
                     int32_t *gmres_iters, void *scratch, int64_t scratch_bytes,
                     int32_t *status, void *stream);

/* Fused per-level MGRIT phases over whole C-intervals (f_relax / c_relax /
 * residual / restriction / injection, mgrit.py:276-299, 317-334).  One CTA
 * (1D) walks each C-interval's m-1 dependent F-steps with the state on chip.
 * Interval c spans global steps [c*m, (c+1)*m]; U row of global step t is
 * U + (t - u_row0)*ldu; Cbuf/Uc/Gc rows and partial[] are indexed by the
 * global C index minus c_row0.  Modes:
 *   MGRIT_PHASE_FC      : F-relax from U[cm], C-relax -> Cbuf[c+1]
 *   MGRIT_PHASE_F_RES   : (after FC) U[cm] <- Cbuf[c] (c>0), F-relax,
 *                         U[(c+1)m] <- Cbuf[c+1], and the C-point residual
 *                         r = G + Phi U[(c+1)m-1] - Cbuf[c+1] -> Gc[c+1],
 *                         partial[c] = sum r^2
 *   MGRIT_PHASE_FONLY_RES: F-relax from U[cm], Cbuf[c+1] <- U[(c+1)m], residual as above
 *   MGRIT_PHASE_INJ_F   : U[cm] <- Cbuf[c] + Uc[c] (c=0: U[0] + Uc[0]), F-relax,
 *                         last interval also U[N] <- Cbuf[N/m] + Uc[N/m];
 *                         with partial != NULL also the fine residual at (c+1)m.
 * zero_init: this level's U starts at zero (coarse levels, mgrit.py:331); C
 * rows are treated as 0 and written as 0 instead of being read. */
enum { MGRIT_PHASE_FC = 0, MGRIT_PHASE_F_RES = 1, MGRIT_PHASE_FONLY_RES = 2,
       MGRIT_PHASE_INJ_F = 3 };

typedef struct mgrit_phase_args {
    int32_t phase;
    int32_t m;
    int64_t c_begin, c_count;   /* global C-interval range handled */
    int64_t n_intervals;        /* global number of intervals on the level (N/m) */
    double *U; int64_t ldu; int64_t u_row0;
    const double *G; int64_t ldg; int64_t g_row0;   /* G NULL => zero forcing */
    double *Cbuf; const double *Uc; double *Gc; int64_t c_row0;
    double *partial; int64_t partial0;
    int32_t zero_init;
    int32_t f_relaxed;          /* MGRIT_PHASE_FC on a 2D level: 1 = the F-points already
                                   hold the F-relaxation of the current C-points (the
                                   previous V-cycle ended with it, mgrit.py:334, and
                                   nothing changed since), so the phase runs only its
                                   C-step; the skipped F-steps would rewrite the same
                                   bits.  The 1D phase kernels ignore it (they carry the
                                   interval through shared memory anyway). */
} mgrit_phase_args;

int mgrit_level_phase(const mgrit_level_desc *L, const mgrit_phase_args *A,
                      void *scratch, int64_t scratch_bytes, int32_t *status,
                      void *stream);

/* Sequential time stepping of a whole level on one SM cluster/CTA
 * (solve_sequential mgrit.py:302-314, numba _kernels.py:104-131,
 * sequential_reference mgrit.py:381-390):
 *   U[t+1] = Phi_t U[t] + G[t+1],  t = 0 .. n_steps-1  (G NULL => + 0.0).
 * zero_init: U[0] := 0 (coarsest level of a V-cycle). */
int mgrit_sequential_sweep(const mgrit_level_desc *L, double *U, int64_t ldu,
                           const double *G, int64_t ldg, int32_t zero_init,
                           int32_t *gmres_iters, void *scratch,
                           int64_t scratch_bytes, int32_t *status, void *stream);

/* Deterministic fixed-order sum of n doubles (pairwise tree over the index):
 * out[0] = sum x[i].  Used for the space-time norm (core.py:173-181). */
int mgrit_sum(const double *x, int64_t n, double *out, void *stream);

/* U[rows] += X[rows] (generic injection U[::m] += Uc, mgrit.py:333). */
int mgrit_axpy_rows(double *U, int64_t ldu, int64_t u_stride_rows,
                    const double *X, int64_t ldx, int64_t rows, int64_t n,
                    void *stream);

/* ------------------------------------------- device-resident solve loop --- */

/* The iteration loop of solve() (mgrit.py:355-373) as one CUDA graph: a WHILE
 * node whose body is the captured V-cycle (the caller's launches between
 * mgrit_loop_begin and mgrit_loop_end on `stream`) followed by the stop test
 * (mgrit_loop_check).  Per solve: mgrit_loop_init (r0 from the initial
 * residual's sum of squares), mgrit_loop_launch, one host sync, then read
 *   ctrl[0] = iterations, ctrl[1] = MGRIT_LOOP_* state, hist[0..ctrl[0]].
 * Stop rule, in the reference's order: non-finite GMRES input (status != 0)
 * -> history NaN, diverged; r = sqrt(sumsq); !finite(r) or
 * r >= divergence_factor*r0 -> diverged; r <= rtol*r0 -> converged;
 * iterations == max_iters -> max_iters.
 * ctrl: device int32[4]; par: device double[2] (written by mgrit_loop_init);
 * hist: device double[max_iters + 1].  `stream` must not be the legacy
 * default stream (it cannot be captured). */
enum { MGRIT_LOOP_RUNNING = 0, MGRIT_LOOP_CONVERGED = 1, MGRIT_LOOP_DIVERGED = 2,
       MGRIT_LOOP_MAX_ITERS = 3 };

int mgrit_loop_begin(void *stream, void **loop_out);
int mgrit_loop_check(void *loop, const double *sumsq, const int32_t *status,
                     double *hist, int32_t *ctrl, const double *par, void *stream);
int mgrit_loop_end(void *loop, void *stream);
int mgrit_loop_init(const double *r0_sumsq, double *hist, int32_t *ctrl, double *par,
                    double rtol, double divergence_factor, int32_t max_iters,
                    void *stream);
int mgrit_loop_launch(void *loop, void *stream);
void mgrit_loop_destroy(void *loop);
/* kernel nodes of the captured body (one V-cycle + stop test); -1 on error */
int64_t mgrit_loop_body_kernels(void *loop);

/* -------------------------------------- operator-level API below Level --- */

/* decompose(grid, coords) (semi_lagrangian.py:118-137): east index (int64,
 * wrapped into [0, n_x)) and offset eps in [0, 1) of `count` coordinates on
 * a periodic [-1, 1) axis of n_x nodes, with the reference's rounding guards. */
int mgrit_decompose(int32_t n_x, int64_t count, const double *coords, int64_t *east,
                    double *eps, void *stream);

/* interp_weights(p, eps) (semi_lagrangian.py:140-161): w[count][p+1], the
 * reference's products and (correctly rounded) divisions. */
int mgrit_interp_weights(int32_t p, int64_t count, const double *eps, double *w,
                         void *stream);

/* Records from a reference DepartureSet (DepartureSet1D.east/eps,
 * DepartureSet2D.east_x/eps and east_y/nu; semi_lagrangian.py:164-205): the
 * scaled coordinate s = E - eps (E = east, or n_x for east == 0), from which
 * the device re-derives exactly the given (east, eps) — a records-based entry
 * for callers that hold DepartureSets instead of coordinates. */
int mgrit_records_from_east_eps(int32_t n_x, int64_t count, const int64_t *east,
                                const double *eps, double *s, void *stream);

/* apply_ImSD(field, derivative_stencil(p), v, grid) (coarse_correction.py:
 * 130-149) on `rows` vectors sharing one field: out = (I - diag(sx) Dx
 * [- diag(sy) Dy]) v, the reference's grouping, separately rounded. */
int mgrit_apply_imsd(int32_t dim, int32_t n_x, int32_t p, int64_t rows,
                     const double *sig_x, const double *sig_y, const double *v,
                     int64_t ldv, double *out, int64_t ldo, void *stream);

/* Level.step_batch with the GMRES residual history of every corrected row
 * (gmres_solve's (x, res_hist) return, coarse_correction.py:173-228):
 * out[b] = Phi_{t_b} U_in[b]; gmres_hist[b][0..iters[b]] = beta, |g_1|, ...
 * (gmres_hist: [B][gmres_max_iters + 1], nullable). */
int mgrit_apply_rows_hist(const mgrit_level_desc *L, int64_t B, const int64_t *t_idx,
                          int64_t t_first, int64_t t_stride, const double *U_in,
                          int64_t ld_in, double *out, int64_t ld_out,
                          int32_t *gmres_iters, double *gmres_hist, void *scratch,
                          int64_t scratch_bytes, int32_t *status, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MGRIT_B200_H */
