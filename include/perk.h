/*
 * perk.h -- C ABI of libperk_b200.so: one Paired-Explicit Runge-Kutta (P-ERK) multirate step
 * on a DGSEM (N = 3) semidiscretisation partitioned by AMR refinement level, on one B200.
 *
 * Source of every operation: /root/reference/PAPER.md ("P:l.N" = line N), readings in
 * SURVEY.md §8(c) and DESIGN.md §2.
 *   - problem U'(t) = F(t, U), DOFs partitioned by cell level into R partitions
 *     (P:l.192-205, eq. PartitionedODESys; mask matrices I^(r), P:l.289-301)
 *   - stage update K_i^(r) = F^(r)(U_n + dt sum_j sum_k a_ij^(k) K_j^(k)), U_{n+1} = U_n + dt sum b_i K_i
 *     (P:l.209-218, eq. PartitionedRKSystem) with the P-ERK2 pattern: shared c, b = e_S, two nonzeros
 *     a_{i,1}, a_{i,i-1} per row, member E evaluates stages {1} u {S-E+2..S}
 *     (P:l.407-436, eq. PERK_ButcherTableauClassic; a_{i,1} = c_i - a_{i,i-1}, P:l.533)
 *   - coefficients a_{i,i-1} from the stability polynomial (P:l.1048-1064, eqs. PERK2_StabPnom,
 *     PERKCoeffsConstruction)
 *   - per-level element / boundary / interface / mortar index lists; interfaces by common level,
 *     mortars by the fine side (P:l.1243-1256); level -> member fill rule (P:l.1276-1279)
 *
 * Conventions (all calls):
 *   - return 0 (PERK_OK) or a negative PERK_E* code; no exception crosses the ABI;
 *     perk_last_error(ctx) gives a text for the last failure.
 *   - pointers named *_dev are CUDA device pointers (e.g. torch.Tensor.data_ptr() of a cuda tensor),
 *     pointers named *_host are host pointers; the library never frees caller memory and never
 *     retains a caller pointer past the call, except U_dev inside the captured step graph, which is
 *     re-captured whenever perk_step sees a different U_dev or dt.
 *   - all device work is ordered on the context stream (perk_set_stream; default: the legacy
 *     stream 0).  Calls documented "asynchronous" do not synchronise; device-side errors
 *     (capacity overflow, unbalanced level map) latch a device flag reported by the next
 *     synchronising call (perk_sync and every introspection call).
 *   - one context per host thread at a time; contexts are independent.
 */
#ifndef PERK_B200_PERK_H
#define PERK_B200_PERK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PERK_OK = 0,
    PERK_EINVAL = -1,       /* invalid argument (null pointer, bad enum, S/R/E out of range, ...) */
    PERK_EUNBALANCED = -2,  /* level map not block-aligned, or 2:1 face balance violated */
    PERK_ECAPACITY = -3,    /* more cells / faces than the capacity given at perk_init */
    PERK_ECUDA = -4,        /* a CUDA runtime call failed */
    PERK_ENOTINIT = -5,     /* context null or destroyed */
    PERK_EUNSUPPORTED = -6  /* combination not implemented (e.g. Navier-Stokes with non-periodic faces) */
};

enum { PERK_EQ_ADVECTION = 0, PERK_EQ_EULER = 1, PERK_EQ_NAVIER_STOKES = 2 };
enum { PERK_VOL_WEAK = 0, PERK_VOL_FLUXDIFF = 1 };               /* weak form (1D), Ranocha flux differencing (2D) */
enum { PERK_FLUX_UPWIND = 0, PERK_FLUX_RUSANOV = 1, PERK_FLUX_HLL = 2 };
enum { PERK_KIND_ELEMENTS = 0, PERK_KIND_INTERFACES = 1, PERK_KIND_MORTARS = 2, PERK_KIND_BOUNDARIES = 3 };

#define PERK_MAX_STAGES 64
#define PERK_MAX_MEMBERS 8
#define PERK_NUM_KERNEL_KINDS 7   /* profile slots: 0 surface flux, 1 volume+stage, 2 mesh rebuild, 3 transfer,
                                    4 BR1 gradient traces, 5 BR1 gradients + viscous-flux traces,
                                    6 shock-capturing blending factors (+ smoothing) */

/* Problem description.  DG degree N = 3 (LGL nodes) is fixed.
 *   dim            1 or 2
 *   n_base[2]      base cells per direction (n_base[1] ignored in 1D); square cells required in 2D
 *   max_level      maximum allowed refinement level L (finest grid = n_base << L per direction)
 *   periodic[2]    1 = periodic, 0 = weakly imposed Dirichlet state bc_state on that direction's faces
 *   domain_lo/hi   physical box ([lo, hi] per direction)
 *   gamma          ratio of specific heats (Euler / NS)
 *   prandtl, mu    Navier-Stokes parameters (equation 2, 2D only, periodic only): viscosity mu, Prandtl
 *                  number; heat conductivity kappa = mu gamma / ((gamma - 1) Pr), T = p / rho.  The
 *                  viscous terms are BR1 (P:l.1419-1420; D7)
 *   adv_velocity   1D linear advection speed a (equation 0)
 *   bc_state[4]    conserved ghost state for non-periodic faces
 *   max_cells      capacity (cells) for all buffers; the caller's U_dev must hold max_cells rows */
typedef struct perk_problem {
    int32_t dim;
    int32_t equation;
    int32_t volume;
    int32_t surface;
    int32_t n_base[2];
    int32_t max_level;
    int32_t periodic[2];
    int32_t _pad;
    double domain_lo[2];
    double domain_hi[2];
    double gamma;
    double prandtl;
    double mu;
    double adv_velocity;
    double bc_state[4];
    int64_t max_cells;
} perk_problem;

/* P-ERK family: S stages, R members with E[0] < ... < E[R-1] <= S (E[r] >= 2).
 * Stage pattern (which stages member r evaluates): active[r] bit i-1 = stage i.  All zero = the
 * standard pattern {1} u {S-E_r+2..S} (P:l.407-436); otherwise every member's set must hold stages 1
 * and S and E[r] stages in total, e.g. the alternating and early-shared patterns of P:l.642-700.
 * c[i-1] = c_i; a_sub[r][i-1] = a_{i,p(i)} of member r, the coefficient of K_{p(i)} in stage i's
 * state, where p(i) is the member's previous evaluated stage > 1 (= i-1 in the standard pattern);
 * it may be nonzero only at evaluated stages that have such a predecessor.  a_{i,1} = c_i - a_sub is
 * derived.  Non-standard patterns: 1D / 2D Euler / Navier-Stokes (NS launches the superset member
 * prefix of each stage).
 * Shared weights b[i-1] = b_i, nonzero only at i = 1, S-1, S:
 *   P-ERK2: b = e_S (P:l.423; perk_tableau_p2 fills it);
 *   P-ERK3: b_1 = b_{S-1} = 1/6, b_S = 4/6 (Shu-Osher base, P:l.870-883), c_{S-1} = 1, c_S = 1/2,
 *           coefficients computed offline (P:l.1067-1090) and passed in by the caller; requires
 *           E[0] >= 3.  The final update U_n + dt (b_1 K_1 + b_{S-1} K_{S-1} + b_S K_S) is formed as
 *           W = U_n + dt (b_1 K_1 + b_{S-1} K_{S-1}) in the stage S-1 epilogue, U_{n+1} = W + dt b_S K_S.
 * Member r is assigned to level l by r = clamp(R-1-(L-l), 0, R-1). */
typedef struct perk_tableau {
    int32_t S;
    int32_t R;
    int32_t E[PERK_MAX_MEMBERS];
    double c[PERK_MAX_STAGES];
    double b[PERK_MAX_STAGES];
    double a_sub[PERK_MAX_MEMBERS][PERK_MAX_STAGES];
    uint64_t active[PERK_MAX_MEMBERS];
} perk_tableau;

typedef struct perk_ctx perk_ctx;

/* Host only.  Taylor rule of BASELINE.json cfg 1: alpha[k] = 1/k!, k = 0..E (alpha has E+1 entries). */
int perk_alpha_taylor(int32_t E, double *alpha_host);

/* Host only.  Build a P-ERK2 family (b = e_S) from stability-polynomial coefficients:
 * alpha_host is R rows of (S+1) doubles, row r = alpha_0..alpha_S of member r (entries above E[r]
 * ignored).  c_i = (i-1)/(2(S-1)) (P:l.439-442); a_{i,i-1} by the recursion of P:l.1062 for
 * i = 0..E-3, all other a_{i,i-1} = 0.  EINVAL on bad sizes or a zero pivot. */
int perk_tableau_p2(int32_t S, int32_t R, const int32_t *E_host, const double *alpha_host, perk_tableau *out);
/* Host only.  perk_tableau_p2 generalised: stage pattern active_host[R] (NULL or
 * all zero = standard) and abscissa c_S (0.5 = the standard midpoint choice; 1 = Heun, 2/3 = Ralston,
 * P:l.439-442): c_i = c_S (i-1)/(S-1), b_S = 1/(2 c_S), b_1 = 1 - b_S.  Along member r's evaluated
 * stages after 1, s_1 < ... < s_{E-1} = S, the row coefficients a_k of stage s_k follow
 * a_{E-1-i} = alpha_{3+i} / (b_S c_{s_{E-2-i}} prod_{m<i} a_{E-1-m}), i = 0..E-3 (the recursion of
 * P:l.1058-1064 along the chain).  EINVAL on bad sizes, patterns or a zero pivot. */
int perk_tableau_p2_ex(int32_t S, int32_t R, const int32_t *E_host, const double *alpha_host,
                       const uint64_t *active_host, double c_S, perk_tableau *out);

/* Host only.  Evaluated-stage set of a member with E evaluations in an S-stage method, as the bit
 * mask perk_tableau_p2_ex / perk_tableau.active take (bit i-1 = stage i):
 *   kind PERK_PATTERN_STANDARD    {1} u {S-E+2, ..., S}          (P:l.407-436, eq. PERK_ButcherTableauClassic)
 *   kind PERK_PATTERN_EARLY       {1, ..., E-1} u {S}            (P:l.683-700: S = 6, E = 4 -> {1,2,3,6})
 *   kind PERK_PATTERN_ALTERNATING {1} u {S - floor((E-1-k)(S-1)/(E-1) + 1/2) : k = 1..E-1}
 *                                 (P:l.655-675: S = 6, E = 4 -> {1,3,4,6}; general rule DESIGN.md F1)
 *   kind PERK_PATTERN_EXPLICIT    the n_stages stage numbers in stages_host (1-based, must hold 1
 *                                 and S, no duplicates, n_stages == E)
 * EINVAL on 2 > E, E > S, S > PERK_MAX_STAGES, an unknown kind or an invalid explicit set. */
enum { PERK_PATTERN_STANDARD = 0, PERK_PATTERN_EARLY = 1, PERK_PATTERN_ALTERNATING = 2, PERK_PATTERN_EXPLICIT = 3 };
int perk_pattern_mask(int32_t S, int32_t E, int32_t kind, const int32_t *stages_host, int32_t n_stages,
                      uint64_t *mask_out);

/* Create a context: validates prob/tab (EINVAL, EUNSUPPORTED), uploads the tableau, allocates
 * capacity-sized device buffers and builds the mesh and per-member lists on the device from the
 * finest-grid level map level_map_dev (uint8, (n_base[0] << L) x (n_base[1] << L) entries, x
 * fastest; not retained).  Synchronises once at the end: EUNBALANCED / ECAPACITY are reported here.
 * stream: a cudaStream_t (NULL = legacy stream).
 * Ownership: unless out / prob / level_map_dev / tab is NULL (EINVAL, *out untouched), *out receives
 * the context on EVERY return, including errors: read perk_last_error(*out), then release it with
 * perk_destroy (it frees whatever was allocated before the failure).
 * Environment read here (schedule knobs; none changes a result bit): PERK_VOL_BLOCKS / PERK_GRAD_BLOCKS /
 * PERK_SURF_BLOCKS cap the persistent grids (race tests); PERK_SWEEP=0 makes every 2D stage kernel walk
 * its lists forward instead of alternating the direction from launch to launch (DESIGN.md §5 item 4). */
int perk_init(perk_ctx **out, const perk_problem *prob, const uint8_t *level_map_dev, const perk_tableau *tab,
              void *stream);
int perk_destroy(perk_ctx *ctx);
int perk_set_stream(perk_ctx *ctx, void *stream);

/* One P-ERK step in place, asynchronous.  U_dev: fp64 [max_cells][nv][(N+1)^dim], cells in the
 * canonical (Morton) order of perk_get_leaves, variables conserved, nodes x fastest.  The step is
 * a CUDA graph captured on first use (and re-captured when U_dev or dt change). */
int perk_step(perk_ctx *ctx, double *U_dev, double dt);

/* Same step with HOST buffers: copies U_host (n_cells rows) to the device, runs nsteps steps,
 * copies the result back and synchronises.  End-to-end API used by bench.py's e2e number. */
int perk_run_host(perk_ctx *ctx, double *U_host, double dt, int64_t nsteps);

/* Re-mesh, asynchronous: rebuild leaves, faces, per-member lists and stage prefix tables from a new
 * level map on the device (no host round trip), and transfer U_dev in place (refine: interpolation,
 * coarsen: exact L2 projection; |level change| <= 1 per finest cell required).  2D only (1D meshes
 * are static: EUNSUPPORTED).  An unbalanced / misaligned map (EUNBALANCED), a level jump > 1
 * (EUNBALANCED) or more cells than max_cells (ECAPACITY) latch the device error flag and are
 * reported by the next synchronising call; U_dev and the mesh are then undefined. */
int perk_repartition(perk_ctx *ctx, const uint8_t *level_map_dev, double *U_dev);

/* dU = sum_{r in mask} I^(r) F(U) (P:l.289-301): zero on cells of unmasked members.  Asynchronous.
 * U_dev read only; dU_dev caller-owned, same layout as U. */
int rhs_eval(perk_ctx *ctx, const double *U_dev, uint32_t partition_mask, double *dU_dev);

/* ---- indicator-driven AMR (A1-A6), 2D Euler / Navier-Stokes ----
 * The paper refines by indicators it cites but does not define: Loehner on v_x (P:l.1440-1441),
 * Hennemann-Gassner on rho or rho*p (P:l.1548, l.1731, l.1886), and defines the enstrophy
 * eps = 0.5 rho w.w with a refinement threshold (P:l.1615-1622, eq. Enstrophy).
 *   indicator   PERK_IND_*; variable PERK_VAR_* (the indicator quantity at each node; ignored by
 *               the enstrophy indicator)
 *   controller  target level = base_level if indicator <= med_threshold, med_level if
 *               indicator <= max_threshold, else max_level; each adaptation moves a leaf one level
 *               toward its target; a leaf coarsens only together with its three siblings; the
 *               result is made 2:1 face balanced by further refinement.
 *               0 <= base_level <= med_level <= max_level <= perk_problem.max_level <= 7.
 *   alpha_max, alpha_min   Hennemann-Gassner clipping (alpha < alpha_min -> 0, > 1 - alpha_min -> 1,
 *               then min(alpha, alpha_max)); f_wave   Loehner noise filter (e.g. 0.2). */
enum { PERK_IND_HENNEMANN_GASSNER = 0, PERK_IND_LOHNER = 1, PERK_IND_ENSTROPHY = 2 };
enum { PERK_VAR_DENSITY = 0, PERK_VAR_PRESSURE = 1, PERK_VAR_DENSITY_PRESSURE = 2, PERK_VAR_VX = 3, PERK_VAR_VY = 4 };
typedef struct perk_amr {
    int32_t indicator;
    int32_t variable;
    int32_t base_level;
    int32_t med_level;
    int32_t max_level;
    int32_t _pad;
    double med_threshold;
    double max_threshold;
    double alpha_max;
    double alpha_min;
    double f_wave;
} perk_amr;

/* Per-leaf indicator of the state U_dev (layout of perk_step) into ind_dev (fp64, >= n_cells
 * entries, canonical leaf order).  Asynchronous.  EUNSUPPORTED for 1D / advection, EINVAL for bad
 * parameters. */
int perk_amr_indicator(perk_ctx *ctx, const double *U_dev, const perk_amr *amr, double *ind_dev);
/* Indicator + controller + 2:1 balance: writes the next finest-grid level map (uint8, layout of
 * perk_init's level map) to level_map_dev, asynchronous and without a host round trip; pass it to
 * perk_repartition(ctx, level_map_dev, U_dev) to re-mesh.  The current mesh is not changed. */
int perk_amr_adapt(perk_ctx *ctx, const double *U_dev, const perk_amr *amr, uint8_t *level_map_dev);
/* Number of kernel launches one perk_amr_adapt performs (max_level + 3). */
int perk_amr_launches(perk_ctx *ctx, int32_t *launches);

/* ---- subcell shock capturing ----
 * The paper's inviscid applications use the Hennemann-Gassner shock capturing (P:l.964, l.1729,
 * l.1795-1799; A7-A9): per element and stage the flux-differencing volume integral V_DG is
 * replaced by (1 - alpha) V_DG + alpha V_FV, V_FV the first-order finite-volume divergence on the
 * element's LGL subcells (widths w_i h / 2) with the problem's surface flux between neighbouring
 * nodes.  alpha = alpha_fixed if alpha_fixed >= 0, else the Hennemann-Gassner indicator of
 * `variable` (PERK_VAR_*) on the element's stage state, 0 below alpha_min, 1 above 1 - alpha_min,
 * clipped to alpha_max; smooth != 0: alpha_e = max(alpha_e, alpha_n / 2) over face neighbours n.
 * Each P-ERK stage then launches 1 more kernel (the blending factors) before its surface flux, which
 * also applies the smoothing (env PERK_SC_FUSED=0 at this call: a separate smoothing launch). */
typedef struct perk_shock_capturing {
    int32_t variable;
    int32_t smooth;
    double alpha_max;
    double alpha_min;
    double alpha_fixed;
} perk_shock_capturing;

/* Switch shock capturing on (sc != NULL; parameters copied) or off (sc = NULL) for the following
 * steps and rhs_eval calls; re-mesh keeps it.  Synchronises the context stream.  Any stage pattern
 * (non-standard ones evaluate alpha on every element at every stage).  EUNSUPPORTED for 1D /
 * advection problems; EINVAL for parameters out of range (0 <= alpha_min <= 1/2,
 * 0 <= alpha_max <= 1, alpha_fixed <= 1, variable in 0..4). */
int perk_set_shock_capturing(perk_ctx *ctx, const perk_shock_capturing *sc);
/* Blending factors of the state U_dev (raw indicator and smoothed) into device arrays of >= n_cells
 * doubles, canonical leaf order.  Asynchronous; EINVAL if shock capturing is off. */
int perk_sc_alpha(perk_ctx *ctx, const double *U_dev, double *raw_dev, double *smoothed_dev);

/* ---- introspection (synchronising) ---- */
int perk_num_cells(perk_ctx *ctx, int64_t *n_cells);
int perk_num_faces(perk_ctx *ctx, int64_t *counts3);            /* interfaces, mortars, boundaries */
/* physical node coordinates, device array [n_cells][dim][(N+1)^dim] (asynchronous) */
int perk_node_coords(perk_ctx *ctx, double *xy_dev);
/* leaf origins on the finest grid, level and member, host arrays of >= n_cells entries */
int perk_get_leaves(perk_ctx *ctx, int32_t *fx_host, int32_t *fy_host, uint8_t *level_host, int32_t *member_host,
                    int64_t cap);
/* face records (host): interfaces [n][3] = low elem, high elem, orientation; mortars [n][5] = large,
 * small_lo, small_hi, orientation, large_side (0: large element on the low side); boundaries [n][2] =
 * elem, face (0 +x, 1 -x, 2 +y, 3 -y); member_host[n] = the partition of each record. */
int perk_get_faces(perk_ctx *ctx, int32_t kind, int32_t *rec_host, int32_t *member_host, int64_t cap, int64_t *len);
/* per-member compacted list of `kind` (item indices), segments by descending member; seg_host[R+1] */
int perk_get_list(perk_ctx *ctx, int32_t kind, int32_t *list_host, int64_t cap, int64_t *seg_host);
/* count_active_host[i-1] = number of `kind` items evaluated at stage i, i = 1..S */
int perk_get_count_active(perk_ctx *ctx, int32_t kind, int32_t *count_active_host);
/* BR1 / shock-capturing halo per stage (Navier-Stokes or shock capturing contexts; zeros otherwise):
 * halo_host[kind][i-1] for kind 0 elements, 1 interfaces, 2 mortars, i = 1..S = number of halo
 * items the stage-i BR1 / indicator launches process besides the active ones (the large elements of
 * the active mortars whose fine side is another member, and their faces; D7).  Synchronising. */
int perk_get_halo_counts(perk_ctx *ctx, int32_t *halo_host);
/* per element face neighbours of the fused BR1 gradient pass (Navier-Stokes contexts built with
 * BR1_FUSED; EUNSUPPORTED otherwise): table_host[e][face][2], face 0 +x, 1 -x, 2 +y, 3 -y:
 * conforming {nb, -1}; small side of a mortar {large, -2 (lower half) / -3 (upper half)}; large side
 * {small_lo, small_hi}; boundary {-1, -4}.  Cells only (the member bits of the device table are
 * stripped).  cap >= 8 n_cells entries.  Synchronising. */
int perk_get_face_table(perk_ctx *ctx, int32_t *table_host, int64_t cap);
/* element-RHS evaluations (sum over steps of sum_r E_r N_C(r), P:l.1282-1289) and steps taken */
int perk_get_counters(perk_ctx *ctx, int64_t *elem_rhs_evals, int64_t *steps);
int perk_sync(perk_ctx *ctx);
const char *perk_last_error(perk_ctx *ctx);

/* Profiling (synchronising): run one step eagerly (no graph) with CUDA events around every launch
 * on the context stream; ms_host[k] += device time of kernel kind k, launches_host[k] += launches. */
int perk_profile_step(perk_ctx *ctx, double *U_dev, double dt, float *ms_host, int32_t *launches_host);
/* Device time per step of only the kernels of the kinds in kind_mask (bit k = kind k above), launched
 * exactly as perk_step launches them (captured graph, programmatic dependent launches): one warm-up
 * replay, then CUDA events around `reps` replays on the context stream.  The other kinds' kernels are
 * left out of the graph, so the state is NOT a valid P-ERK evolution afterwards (timing only).
 * Synchronising. */
int perk_time_kernels(perk_ctx *ctx, double *U_dev, double dt, uint32_t kind_mask, int32_t reps, float *ms_per_step);
/* perk_time_kernels with an L2 flush between replays: before each of the reps replays (outside its
 * event pair) flush_bytes of the caller's device buffer flush_dev are overwritten (use more than the
 * 126 MB L2); ms_per_step = mean of the per-replay event times.  flush_bytes = 0: no flush. */
int perk_time_kernels_ex(perk_ctx *ctx, double *U_dev, double dt, uint32_t kind_mask, int32_t reps,
                         void *flush_dev, int64_t flush_bytes, float *ms_per_step);
/* Same for one repartition (kinds 2 and 3). */
int perk_profile_repartition(perk_ctx *ctx, const uint8_t *level_map_dev, double *U_dev, float *ms_host,
                             int32_t *launches_host);
/* Build configuration of the library (no context): bit 0 = BR1_DV (k_grad2d forms the viscous volume
 * term), bit 1 = BR1_FUSED (k_grad2d forms the BR1 central traces from the face neighbours: kernel
 * kind 4, k_gsurf2d, is never launched).  Pure, never fails. */
int perk_build_flags(void);
/* Number of kernel launches one perk_step performs (graph nodes). */
int perk_launches_per_step(perk_ctx *ctx, int32_t *launches);
/* Race exposure, debug library only (libperk_debug.so, -DPERK_DEBUG; EUNSUPPORTED otherwise): seed != 0
 * makes every thread of the staged kernels (k_vol2d, k_grad2d) sleep a pseudo-random 0..4 us at
 * each warp barrier / asynchronous-copy wait, for all contexts of the current device; seed 0 turns it
 * off.  Results must be bitwise those of an unjittered run (tests/test_gpu_races.py). */
int perk_debug_jitter(uint32_t seed);

/* ------------------------------------------------------------------------------------------------
 * Spatial domain decomposition over ranks.  The paper's
 * partitioning is by level only and "no additional data exchange is required compared to standard
 * Runge-Kutta methods" (P:l.1258-1263, §6.3): across GPUs each rank owns a contiguous Morton range of
 * leaves, balanced in the per-step work sum_leaves E_member (the E-weighted split below), keeps its
 * owned elements and the faces with an owned side, and receives per stage the blocks its ghost cells
 * (face neighbours owned elsewhere) changed.  2D, standard stage pattern, no shock capturing.
 * ------------------------------------------------------------------------------------------------ */

/* Host only.  The E-weighted split of n leaves in Morton order with per-leaf weights w_k (the stage
 * evaluations E of the leaf's member): owner_k = min(P-1, floor(P (2 prefix_k + w_k) / (2 W))),
 * prefix_k = sum_{j<k} w_j, W = sum w (all owners 0 when W = 0).  Owners are non-decreasing in k
 * (contiguous ranges); the device mesh pipeline computes the same owners.  EINVAL on n < 0,
 * NULL arrays with n > 0, negative weights, nranks outside 1..8. */
int perk_dd_split(int64_t n, const int32_t *weights_host, int32_t nranks, int32_t *owner_host);

/* Create sub-domain `rank` of an nranks-way decomposition: like perk_init (every rank passes the same
 * problem, level map and tableau and builds the same global mesh), then keeps the owned part.  The
 * state U_dev is still [max_cells][nv][npe] in global cell order: rows of owned cells are this rank's,
 * rows of its ghost cells are kept current by the exchange, other rows are not used.  nranks = 1 is
 * perk_init.  EINVAL on rank / nranks, EUNSUPPORTED for 1D or a non-standard stage pattern.  A
 * sub-domain context does not take perk_step (EUNSUPPORTED); perk_repartition and perk_amr_* need the
 * complete state on every rank (gather the owned ranges first, perk_dd_info). */
int perk_init_dd(perk_ctx **out, const perk_problem *prob, const uint8_t *level_map_dev, const perk_tableau *tab,
                 void *stream, int32_t rank, int32_t nranks);
/* rank, nranks and the owned cells [first, first + count) of the current mesh (synchronising) */
int perk_dd_info(perk_ctx *ctx, int32_t *rank, int32_t *nranks, int64_t *first, int64_t *count);
/* Per stage i = 1..S, the number of cell blocks this rank sends to / receives from `peer` for
 * `what` (0: state blocks, 1: Navier-Stokes viscous-flux traces; see perk_dd_pack).  Synchronising. */
int perk_dd_counts(perk_ctx *ctx, int32_t peer, int32_t what, int32_t *send_host, int32_t *recv_host);
/* The send (dir 0: owned cells that are ghosts of peer) or receive (dir 1: peer's cells that are ghosts
 * here) list, member-sorted by descending E; synchronising. */
int perk_dd_get_list(perk_ctx *ctx, int32_t peer, int32_t dir, int32_t *list_host, int64_t cap, int64_t *len);
/* Asynchronous stage launches of a sub-domain: part 0 = the BR1 passes of stage `stage`
 * (Navier-Stokes; nothing otherwise), part 1 = surface flux + volume / stage epilogue.  A stage is
 * part 0, exchange what = 1, part 1, exchange what = 0. */
int perk_dd_stage(perk_ctx *ctx, double *U_dev, double dt, int32_t stage, int32_t part);
/* Asynchronous, on the context stream: gather (pack) into buf_dev / scatter (unpack) from buf_dev the
 * blocks of stage `stage` exchanged with `peer`, in list order: what 0 = the blocks the stage's volume
 * epilogue wrote (K_1 at stage 1, the next stage state at 1 < i < S, U_{n+1} = U_dev at stage S;
 * nv * (N+1)^2 doubles per cell) of the cells active at the stage; what 1 = Vt (48 doubles per cell)
 * of the active cells and of the member below (the BR1 halo).  buf_dev holds the perk_dd_counts
 * number of blocks; the transport between ranks (NCCL send / recv) is the caller's. */
int perk_dd_pack(perk_ctx *ctx, double *U_dev, int32_t stage, int32_t what, int32_t peer, double *buf_dev);
int perk_dd_unpack(perk_ctx *ctx, double *U_dev, int32_t stage, int32_t what, int32_t peer, const double *buf_dev);
/* In-process exchange between two sub-domains of one split (on one device, or on devices with peer
 * access): src's blocks for dst go straight into the same rows of dst's arrays, one kernel on src's
 * stream (the caller orders dst's stream after it). */
int perk_dd_exchange(perk_ctx *src, perk_ctx *dst, double *U_src_dev, double *U_dst_dev, int32_t stage, int32_t what);
/* One P-ERK step of all n sub-domains of a split held by this process (ctxs[p] = rank p, sharing one
 * stream): per stage the parts and exchanges above, in order.  Asynchronous. */
int perk_dd_group_step(perk_ctx **ctxs, int32_t n, double **U_dev, double dt);

#ifdef __cplusplus
}
#endif
#endif /* PERK_B200_PERK_H */
