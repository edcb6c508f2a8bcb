/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation (C99, fp64, built with
 * -O2 -ffp-contract=off, no fast-math) of what the P-ERK multirate hot path
 * computes.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant generator with paper_2403_05144_b200/ (the CUDA path).
 *
 * Citations: "P:l.N" = /root/reference/PAPER.md line N (section/equation given),
 * "SURVEY §8(c) Ox" = the reading recorded in SURVEY.md and DESIGN.md §2.
 *
 * Contents
 *   1. DGSEM N=3 basis (LGL nodes/weights, derivative matrix, mortar
 *      interpolation and exact-L2 projection)
 *   2. Mesh from a finest-grid level map: Morton leaves, 2:1 check, faces,
 *      partition (member) assignment, per-member lists   P:l.1243-1256, l.1276-1279
 *   3. Numerical fluxes (upwind, Rusanov, HLL, Ranocha EC two-point flux)
 *   4. RHS F(U) (weak form 1D, flux differencing 2D; 4b: BR1 viscous terms for
 *      Navier-Stokes), "reference" (full F then
 *      mask I^(r), P:l.299) and "restricted" (active lists only) modes
 *   5. Partitioned P-ERK step, materialised stage states   P:l.209-218, l.407-436
 *   6. Re-mesh solution transfer (refine = interpolation, coarsen = exact L2)
 *   7. FV Godunov testbed (linear advection / Burgers)     P:l.479-520
 *   8. AMR indicators (Hennemann-Gassner, Loehner, enstrophy) and the level
 *      controller with 2:1 balance     P:l.1440-1441, l.1548, l.1615-1622
 *   9. Subcell shock capturing (Hennemann-Gassner blending of the flux-differencing
 *      volume integral with a first-order subcell finite-volume one)
 *                                                          P:l.964, l.1729, l.1795-1799
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py; the
 * Navier-Stokes BR1 operator (section 4b) by tests/test_oracle_ns.py (free stream,
 * conservation, manufactured viscous terms term by term, restricted == reference);
 * section 8 by tests/test_oracle_amr.py (closed-form modal energies, hand-computed Loehner
 * ratios, exact vorticity of polynomial fields, brute-force minimal balanced trees); section 9 by
 * tests/test_oracle_sc.py (alpha = 1 equals an independent global first-order finite-volume scheme
 * on the subcell grid, alpha = 0 is bitwise the unblended operator, free stream, conservation with
 * mortars, smoothing against geometric brute-force neighbours, restricted == reference).
 */
#include <math.h>
#include <stdint.h>
/* Optional OpenMP (ORACLE_OMP=1 -> liboracle_omp.so, only for long full-run parity checks): every parallel loop
   below writes disjoint per-element / per-face-slot outputs and has no reduction, so the results are
   bitwise identical for any thread count; the default build has no -fopenmp and runs
   the same loops serially. */
#define OMP_FOR _Pragma("omp parallel for schedule(static)")
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NP 4        /* N + 1 LGL nodes per direction, N = 3 (BASELINE.json configs) */
#define MAXV 4      /* at most 4 conserved variables (2D Euler) */
#define MAXS 64
#define MAXR 8

/* ------------------------------------------------------------------------- */
/* public structs (mirrored by ctypes in oracle/oracle.py)                   */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t dim;          /* 1 or 2 */
    int32_t equation;     /* 0 advection, 1 euler, 2 navier-stokes (2D, BR1) */
    int32_t volume;       /* 0 weak form, 1 flux differencing (Ranocha) */
    int32_t surface;      /* 0 upwind, 1 Rusanov, 2 HLL, 3 Ranocha EC (2D Euler; entropy pin only) */
    int32_t nbx, nby;     /* base cells per direction (nby = 1 in 1D) */
    int32_t max_level;
    int32_t periodic[2];
    double lo[2], hi[2];
    double gamma, prandtl, mu, adv;
    double bc_state[MAXV];/* Dirichlet ghost state (conserved) on non-periodic faces */
} OraProblem;

typedef struct {
    int32_t S, R;
    int32_t E[MAXR];            /* ascending; member r has E[r] RHS evaluations */
    double c[MAXS];             /* c_i, index i-1 */
    double b[MAXS];             /* b_i, index i-1 (P-ERK2: e_S; P-ERK3: 1/6, 0.., 1/6, 4/6) */
    double a1[MAXR][MAXS];      /* a_{i,1}^{(r)}   (index i-1) */
    double asub[MAXR][MAXS];    /* a_{i,p(i)}^{(r)} (index i-1): the coefficient of K_{p(i)}, p(i) = the
                                   member's previous evaluated stage > 1 (= i-1 in the standard pattern) */
    uint64_t active[MAXR];      /* bit i-1: member r evaluates stage i; 0 = the standard pattern
                                   {1} u {S-E+2..S} (P:l.428); other patterns P:l.642-700 */
} OraTableau;

/* subcell shock capturing (section 9) */
typedef struct {
    int32_t variable;           /* indicator variable: 0 rho, 1 p, 2 rho*p, 3 v_x, 4 v_y */
    int32_t smooth;             /* 1: alpha_e = max(alpha_e, alpha_nbr / 2) over face neighbours */
    double alpha_max, alpha_min;
    double alpha_fixed;         /* >= 0: this blending factor for every element (no indicator) */
} OraSC;

/* stage i (1-based) is evaluated by member r: standard pattern i == 1 or i >= S - E_r + 2
   (P:l.407-436, eq. PERK_ButcherTableauClassic: member E evaluates K_1 and the last E-1 stages),
   or the member's explicit stage set (alternating / early-shared patterns, P:l.642-700) */
static int tab_active(const OraTableau *t, int r, int i)
{
    if (t->active[r]) return (int)((t->active[r] >> (i - 1)) & 1u);
    return i == 1 || i >= t->S - t->E[r] + 2;
}

/* ------------------------------------------------------------------------- */
/* 1. basis                                                                  */
/* ------------------------------------------------------------------------- */
typedef struct {
    double xi[NP], w[NP];
    double D[NP][NP];       /* D_ij = l_j'(xi_i) */
    double Dhat[NP][NP];    /* weak form: Dhat_ij = w_j D_ji / w_i */
    double Dsplit[NP][NP];  /* flux differencing: 2D, D00 += 1/w0, DNN -= 1/wN */
    double Plo[NP][NP], Pup[NP][NP];  /* l_j((xi_i -/+ 1)/2) */
    double Rlo[NP][NP], Rup[NP][NP];  /* exact L2 projection of a half onto the whole */
} Basis;

static double lagrange(const double *xi, int j, double x)
{
    double v = 1.0;
    for (int k = 0; k < NP; ++k)
        if (k != j) v *= (x - xi[k]) / (xi[j] - xi[k]);
    return v;
}

/* l_j'(x) = sum_{m != j} 1/(xi_j - xi_m) prod_{k != j,m} (x - xi_k)/(xi_j - xi_k)  (product rule) */
static double lagrange_deriv(const double *xi, int j, double x)
{
    double s = 0.0;
    for (int m = 0; m < NP; ++m) {
        if (m == j) continue;
        double t = 1.0 / (xi[j] - xi[m]);
        for (int k = 0; k < NP; ++k)
            if (k != j && k != m) t *= (x - xi[k]) / (xi[j] - xi[k]);
        s += t;
    }
    return s;
}

static void solve4(double A[NP][NP], double *b)  /* Gaussian elimination with partial pivoting */
{
    double M[NP][NP + 1];
    for (int i = 0; i < NP; ++i) { for (int j = 0; j < NP; ++j) M[i][j] = A[i][j]; M[i][NP] = b[i]; }
    for (int c = 0; c < NP; ++c) {
        int p = c;
        for (int r = c + 1; r < NP; ++r) if (fabs(M[r][c]) > fabs(M[p][c])) p = r;
        for (int j = 0; j <= NP; ++j) { double t = M[c][j]; M[c][j] = M[p][j]; M[p][j] = t; }
        for (int r = c + 1; r < NP; ++r) {
            double f = M[r][c] / M[c][c];
            for (int j = c; j <= NP; ++j) M[r][j] -= f * M[c][j];
        }
    }
    for (int i = NP - 1; i >= 0; --i) {
        double s = M[i][NP];
        for (int j = i + 1; j < NP; ++j) s -= M[i][j] * b[j];
        b[i] = s / M[i][i];
    }
}

static void basis_init(Basis *b)
{
    /* LGL nodes and weights for N = 3: xi = -1, -1/sqrt5, 1/sqrt5, 1; w = 1/6, 5/6, 5/6, 1/6 */
    double s5 = 1.0 / sqrt(5.0);
    b->xi[0] = -1.0; b->xi[1] = -s5; b->xi[2] = s5; b->xi[3] = 1.0;
    b->w[0] = 1.0 / 6.0; b->w[1] = 5.0 / 6.0; b->w[2] = 5.0 / 6.0; b->w[3] = 1.0 / 6.0;
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j)
            b->D[i][j] = lagrange_deriv(b->xi, j, b->xi[i]);
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j) {
            b->Dhat[i][j] = b->w[j] * b->D[j][i] / b->w[i];
            b->Dsplit[i][j] = 2.0 * b->D[i][j];
        }
    b->Dsplit[0][0] += 1.0 / b->w[0];
    b->Dsplit[NP - 1][NP - 1] -= 1.0 / b->w[NP - 1];
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j) {
            b->Plo[i][j] = lagrange(b->xi, j, 0.5 * (b->xi[i] - 1.0));
            b->Pup[i][j] = lagrange(b->xi, j, 0.5 * (b->xi[i] + 1.0));
        }
    /* exact L2 projection: M R = B, M_ik = int_{-1}^{1} l_i l_k, B_ij = int_{half} l_i(x) l_j(child coord) dx,
       with 4-point Gauss-Legendre (exact for degree 7 >= 6). */
    double g[4], gw[4];
    double a = sqrt(3.0 / 7.0 - 2.0 / 7.0 * sqrt(6.0 / 5.0));
    double c = sqrt(3.0 / 7.0 + 2.0 / 7.0 * sqrt(6.0 / 5.0));
    g[0] = -c; g[1] = -a; g[2] = a; g[3] = c;
    gw[0] = (18.0 - sqrt(30.0)) / 36.0; gw[1] = (18.0 + sqrt(30.0)) / 36.0;
    gw[2] = gw[1]; gw[3] = gw[0];
    double M[NP][NP];
    for (int i = 0; i < NP; ++i)
        for (int k = 0; k < NP; ++k) {
            double s = 0.0;
            for (int q = 0; q < 4; ++q) s += gw[q] * lagrange(b->xi, i, g[q]) * lagrange(b->xi, k, g[q]);
            M[i][k] = s;
        }
    for (int half = 0; half < 2; ++half) {
        for (int j = 0; j < NP; ++j) {
            double col[NP];
            for (int i = 0; i < NP; ++i) {
                double s = 0.0;
                for (int q = 0; q < 4; ++q) {
                    /* x in the half [-1,0] (lower) or [0,1] (upper); child coordinate eta = 2x +/- 1 */
                    double x = half == 0 ? 0.5 * (g[q] - 1.0) : 0.5 * (g[q] + 1.0);
                    double eta = half == 0 ? 2.0 * x + 1.0 : 2.0 * x - 1.0;
                    s += 0.5 * gw[q] * lagrange(b->xi, i, x) * lagrange(b->xi, j, eta);
                }
                col[i] = s;
            }
            solve4(M, col);
            for (int i = 0; i < NP; ++i) {
                if (half == 0) b->Rlo[i][j] = col[i]; else b->Rup[i][j] = col[i];
            }
        }
    }
}

void ora_get_basis(double *out)  /* xi, w, D, Dhat, Dsplit, Plo, Pup, Rlo, Rup (row-major) */
{
    Basis b; basis_init(&b);
    double *o = out;
    memcpy(o, b.xi, sizeof b.xi); o += NP;
    memcpy(o, b.w, sizeof b.w); o += NP;
    memcpy(o, b.D, sizeof b.D); o += NP * NP;
    memcpy(o, b.Dhat, sizeof b.Dhat); o += NP * NP;
    memcpy(o, b.Dsplit, sizeof b.Dsplit); o += NP * NP;
    memcpy(o, b.Plo, sizeof b.Plo); o += NP * NP;
    memcpy(o, b.Pup, sizeof b.Pup); o += NP * NP;
    memcpy(o, b.Rlo, sizeof b.Rlo); o += NP * NP;
    memcpy(o, b.Rup, sizeof b.Rup);
}

/* ------------------------------------------------------------------------- */
/* 2. mesh                                                                   */
/* ------------------------------------------------------------------------- */
typedef struct {
    OraProblem prob;
    OraTableau tab;
    Basis B;
    int nv, npe;            /* conserved variables, nodes per element */
    int nfx, nfy;           /* finest grid */
    int n;                  /* leaves */
    int32_t *fx, *fy;       /* leaf origin on the finest grid */
    uint8_t *lev;
    int32_t *member;
    int32_t *cell_of;       /* finest cell -> leaf id */
    /* faces */
    int n_if; int32_t *ifc;   /* [n_if][3]: low elem, high elem, orientation */
    int n_mo; int32_t *mor;   /* [n_mo][5]: large, small_lo, small_hi, orientation, large_side */
    int n_bd; int32_t *bnd;   /* [n_bd][2]: elem, face (0 +x, 1 -x, 2 +y, 3 -y) */
    int32_t *if_member, *mo_member, *bd_member;
    /* per-member lists, segments by descending member (finest first) */
    int32_t *list[4]; int64_t seg[4][MAXR + 1];
    /* scratch */
    double *Fs;               /* surface flux per element face: [n][4][nv][NP] */
    double *Gs;               /* BR1: central gradient-variable trace w* per element face, [n][4][4][NP] */
    double *Q;                /* BR1: gradients of w = (rho, v1, v2, T), [n][2 (x, y)][4][NP*NP] */
    double *Fv;               /* BR1: central viscous face flux per element face, [n][4][4][NP] */
    int64_t elem_rhs_count;   /* element-RHS evaluations (counter, P:l.1282-1289) */
    int sc_on; OraSC sc;      /* subcell shock capturing (section 9) */
    double *alpha_raw, *alpha;/* per element: indicator blending factor, after neighbour smoothing */
} Ora;

static uint64_t morton2(uint32_t x, uint32_t y)
{
    uint64_t m = 0;
    for (int b = 0; b < 32; ++b) {
        m |= (uint64_t)((x >> b) & 1u) << (2 * b);
        m |= (uint64_t)((y >> b) & 1u) << (2 * b + 1);
    }
    return m;
}

static uint64_t *g_sort_keys;
static int cmp_key(const void *a, const void *b)
{
    uint64_t ka = g_sort_keys[*(const int32_t *)a], kb = g_sort_keys[*(const int32_t *)b];
    return ka < kb ? -1 : (ka > kb ? 1 : 0);
}

/* member(l) = clamp(R-1-(Lmax-l), 0, R-1): finest allowed level -> highest E, the next levels the
   next members, all coarser levels the lowest E (P:l.1276-1279). */
static int member_of_level(const Ora *o, int l)
{
    int m = o->tab.R - 1 - (o->prob.max_level - l);
    if (m < 0) m = 0;
    if (m > o->tab.R - 1) m = o->tab.R - 1;
    return m;
}

/* stage i (1-based) is evaluated by member r (tab_active above) */
static int member_active(const Ora *o, int r, int i) { return tab_active(&o->tab, r, i); }

static int wrapi(int v, int n) { return ((v % n) + n) % n; }

/* finest cell (x, y) -> leaf id, or -1 outside a non-periodic domain */
static int cell_at(const Ora *o, int x, int y)
{
    if (x < 0 || x >= o->nfx) { if (!o->prob.periodic[0]) return -1; x = wrapi(x, o->nfx); }
    if (y < 0 || y >= o->nfy) { if (!o->prob.periodic[1]) return -1; y = wrapi(y, o->nfy); }
    return o->cell_of[(int64_t)y * o->nfx + x];
}

static void build_lists(Ora *o, int kind, int nitems, const int32_t *mem)
{
    int R = o->tab.R;
    o->list[kind] = (int32_t *)malloc(sizeof(int32_t) * (nitems > 0 ? nitems : 1));
    int64_t pos = 0;
    for (int r = R - 1, s = 0; r >= 0; --r, ++s) {
        o->seg[kind][s] = pos;
        for (int k = 0; k < nitems; ++k)
            if (mem[k] == r) o->list[kind][pos++] = k;
    }
    o->seg[kind][R] = pos;
}

void ora_destroy(void *p)
{
    Ora *o = (Ora *)p;
    if (!o) return;
    free(o->fx); free(o->fy); free(o->lev); free(o->member); free(o->cell_of);
    free(o->ifc); free(o->mor); free(o->bnd);
    free(o->if_member); free(o->mo_member); free(o->bd_member);
    for (int k = 0; k < 4; ++k) free(o->list[k]);
    free(o->Fs); free(o->Gs); free(o->Q); free(o->Fv);
    free(o->alpha_raw); free(o->alpha);
    free(o);
}

/* Build the mesh from a finest-grid level map (x fastest).  Returns NULL and fills err on an
   invalid map (not block-aligned) or a violation of 2:1 face balance. */
void *ora_create(const OraProblem *prob, const uint8_t *lmap, const OraTableau *tab, char *err, int errlen)
{
    Ora *o = (Ora *)calloc(1, sizeof(Ora));
    o->prob = *prob;
    o->tab = *tab;
    basis_init(&o->B);
    int dim = prob->dim, L = prob->max_level;
    o->nv = prob->equation == 0 ? 1 : (dim == 1 ? 3 : 4);
    o->npe = dim == 1 ? NP : NP * NP;
    o->nfx = prob->nbx << L;
    o->nfy = dim == 1 ? 1 : (prob->nby << L);
    int64_t nf = (int64_t)o->nfx * o->nfy;
    /* validity: every finest cell is covered by exactly one leaf, the one at its own level */
    for (int64_t c = 0; c < nf; ++c) {
        int x = (int)(c % o->nfx), y = (int)(c / o->nfx);
        int lc = lmap[c], covers = 0, ok_own = 0;
        if (lc > L) { snprintf(err, errlen, "level %d > max_level at cell %lld", lc, (long long)c); ora_destroy(o); return NULL; }
        for (int l = 0; l <= L; ++l) {
            int s = 1 << (L - l);
            int ox = x - x % s, oy = dim == 1 ? 0 : y - y % s;
            if (lmap[(int64_t)oy * o->nfx + ox] == l) { covers++; if (l == lc) ok_own = 1; }
        }
        if (covers != 1 || !ok_own) {
            snprintf(err, errlen, "level map not block-aligned at finest cell (%d,%d)", x, y);
            ora_destroy(o); return NULL;
        }
    }
    /* leaves = block origins, sorted by Morton code of the origin (x bit lowest); 1D: left to right */
    int cap = 0;
    for (int64_t c = 0; c < nf; ++c) {
        int x = (int)(c % o->nfx), y = (int)(c / o->nfx);
        int s = 1 << (L - lmap[c]);
        if (x % s == 0 && (dim == 1 || y % s == 0)) cap++;
    }
    o->n = cap;
    int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * cap);
    int32_t *tx = (int32_t *)malloc(sizeof(int32_t) * cap), *ty = (int32_t *)malloc(sizeof(int32_t) * cap);
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * cap);
    int k = 0;
    for (int64_t c = 0; c < nf; ++c) {
        int x = (int)(c % o->nfx), y = (int)(c / o->nfx);
        int s = 1 << (L - lmap[c]);
        if (x % s == 0 && (dim == 1 || y % s == 0)) {
            tx[k] = x; ty[k] = y; idx[k] = k;
            key[k] = dim == 1 ? (uint64_t)x : morton2((uint32_t)x, (uint32_t)y);
            k++;
        }
    }
    g_sort_keys = key;
    qsort(idx, cap, sizeof(int32_t), cmp_key);
    o->fx = (int32_t *)malloc(sizeof(int32_t) * cap);
    o->fy = (int32_t *)malloc(sizeof(int32_t) * cap);
    o->lev = (uint8_t *)malloc(cap);
    o->member = (int32_t *)malloc(sizeof(int32_t) * cap);
    for (int e = 0; e < cap; ++e) {
        o->fx[e] = tx[idx[e]]; o->fy[e] = ty[idx[e]];
        o->lev[e] = lmap[(int64_t)o->fy[e] * o->nfx + o->fx[e]];
        o->member[e] = member_of_level(o, o->lev[e]);
    }
    free(idx); free(tx); free(ty); free(key);
    o->cell_of = (int32_t *)malloc(sizeof(int32_t) * nf);
    for (int e = 0; e < cap; ++e) {
        int s = 1 << (L - o->lev[e]);
        for (int dy = 0; dy < (dim == 1 ? 1 : s); ++dy)
            for (int dx = 0; dx < s; ++dx)
                o->cell_of[(int64_t)(o->fy[e] + dy) * o->nfx + o->fx[e] + dx] = e;
    }
    /* faces (P:l.1253-1256), per leaf in canonical order, directions (+x, -x, +y, -y) */
    int nd = dim == 1 ? 2 : 4;
    o->ifc = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)(2 * cap + 1));
    o->mor = (int32_t *)malloc(sizeof(int32_t) * 5 * (size_t)(4 * cap + 1));
    o->bnd = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)(4 * cap + 1));
    o->if_member = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * cap + 1));
    o->mo_member = (int32_t *)malloc(sizeof(int32_t) * (size_t)(4 * cap + 1));
    o->bd_member = (int32_t *)malloc(sizeof(int32_t) * (size_t)(4 * cap + 1));
    for (int e = 0; e < cap; ++e) {
        int l = o->lev[e], s = 1 << (L - l);
        for (int d = 0; d < nd; ++d) {
            int orient = d / 2, plus = (d % 2 == 0);
            int nx, ny;
            if (orient == 0) { nx = plus ? o->fx[e] + s : o->fx[e] - 1; ny = o->fy[e]; }
            else { nx = o->fx[e]; ny = plus ? o->fy[e] + s : o->fy[e] - 1; }
            int nb = cell_at(o, nx, ny);
            if (nb < 0) {  /* domain boundary, weakly imposed Dirichlet state */
                o->bnd[2 * o->n_bd] = e; o->bnd[2 * o->n_bd + 1] = d;
                o->bd_member[o->n_bd] = o->member[e];
                o->n_bd++;
                continue;
            }
            int ln = o->lev[nb];
            if (ln > l + 1 || ln < l - 1) {
                snprintf(err, errlen, "2:1 face balance violated between leaves %d (level %d) and %d (level %d)", e, l, nb, ln);
                ora_destroy(o); return NULL;
            }
            if (dim == 1) {
                /* 1D: every cell emits its right interface; member of the fine side */
                if (plus) {
                    int32_t *f = o->ifc + 3 * o->n_if;
                    f[0] = e; f[1] = nb; f[2] = 0;
                    o->if_member[o->n_if] = member_of_level(o, ln > l ? ln : l);
                    o->n_if++;
                }
                continue;
            }
            if (ln == l) {
                if (plus) {
                    int32_t *f = o->ifc + 3 * o->n_if;
                    f[0] = e; f[1] = nb; f[2] = orient;
                    o->if_member[o->n_if] = o->member[e];   /* common level */
                    o->n_if++;
                }
            } else if (ln == l + 1) {
                /* mortar owned by the large element; small elements ordered along the face */
                int h = s / 2, a0x, a0y, a1x, a1y;
                if (orient == 0) { a0x = nx; a0y = o->fy[e]; a1x = nx; a1y = o->fy[e] + h; }
                else { a0x = o->fx[e]; a0y = ny; a1x = o->fx[e] + h; a1y = ny; }
                int s0 = cell_at(o, a0x, a0y), s1 = cell_at(o, a1x, a1y);
                if (o->lev[s0] != l + 1 || o->lev[s1] != l + 1) {
                    snprintf(err, errlen, "2:1 face balance violated at mortar of leaf %d", e);
                    ora_destroy(o); return NULL;
                }
                int32_t *m = o->mor + 5 * o->n_mo;
                m[0] = e; m[1] = s0; m[2] = s1; m[3] = orient; m[4] = plus ? 0 : 1;
                o->mo_member[o->n_mo] = member_of_level(o, l + 1);  /* fine side (P:l.1256) */
                o->n_mo++;
            }
        }
    }
    build_lists(o, 0, o->n, o->member);
    build_lists(o, 1, o->n_if, o->if_member);
    build_lists(o, 2, o->n_mo, o->mo_member);
    build_lists(o, 3, o->n_bd, o->bd_member);
    o->Fs = (double *)calloc((size_t)o->n * 4 * o->nv * NP, sizeof(double));
    if (prob->equation == 2) {
        if (dim != 2 || prob->volume != 1) {
            snprintf(err, errlen, "Navier-Stokes (BR1) is implemented for 2D flux differencing only");
            ora_destroy(o); return NULL;
        }
        if (o->n_bd > 0) {
            snprintf(err, errlen, "Navier-Stokes (BR1) needs a periodic domain (no viscous boundary fluxes)");
            ora_destroy(o); return NULL;
        }
        o->Gs = (double *)calloc((size_t)o->n * 4 * 4 * NP, sizeof(double));
        o->Q = (double *)calloc((size_t)o->n * 2 * 4 * NP * NP, sizeof(double));
        o->Fv = (double *)calloc((size_t)o->n * 4 * 4 * NP, sizeof(double));
    }
    return o;
}

int ora_num_cells(void *p) { return ((Ora *)p)->n; }
void ora_face_counts(void *p, int64_t *out) { Ora *o = (Ora *)p; out[0] = o->n_if; out[1] = o->n_mo; out[2] = o->n_bd; }

void ora_get_leaves(void *p, int32_t *fx, int32_t *fy, uint8_t *lev, int32_t *member)
{
    Ora *o = (Ora *)p;
    for (int e = 0; e < o->n; ++e) { fx[e] = o->fx[e]; fy[e] = o->fy[e]; lev[e] = o->lev[e]; member[e] = o->member[e]; }
}

void ora_get_faces(void *p, int kind, int32_t *out, int32_t *mem)
{
    Ora *o = (Ora *)p;
    if (kind == 1) { memcpy(out, o->ifc, sizeof(int32_t) * 3 * o->n_if); memcpy(mem, o->if_member, sizeof(int32_t) * o->n_if); }
    if (kind == 2) { memcpy(out, o->mor, sizeof(int32_t) * 5 * o->n_mo); memcpy(mem, o->mo_member, sizeof(int32_t) * o->n_mo); }
    if (kind == 3) { memcpy(out, o->bnd, sizeof(int32_t) * 2 * o->n_bd); memcpy(mem, o->bd_member, sizeof(int32_t) * o->n_bd); }
}

/* kind: 0 elements, 1 interfaces, 2 mortars, 3 boundaries.  seg[s] = start of the s-th segment,
   segments ordered by descending member (finest / highest E first). */
void ora_get_list(void *p, int kind, int32_t *list, int64_t *seg)
{
    Ora *o = (Ora *)p;
    int64_t len = o->seg[kind][o->tab.R];
    memcpy(list, o->list[kind], sizeof(int32_t) * len);
    memcpy(seg, o->seg[kind], sizeof(int64_t) * (o->tab.R + 1));
}

/* number of items of `kind` whose member is active at stage i, i = 1..S  (out[i-1]) */
void ora_count_active(void *p, int kind, int32_t *out)
{
    Ora *o = (Ora *)p;
    int n = kind == 0 ? o->n : kind == 1 ? o->n_if : kind == 2 ? o->n_mo : o->n_bd;
    const int32_t *mem = kind == 0 ? o->member : kind == 1 ? o->if_member : kind == 2 ? o->mo_member : o->bd_member;
    for (int i = 1; i <= o->tab.S; ++i) {
        int c = 0;
        for (int k = 0; k < n; ++k) c += member_active(o, mem[k], i);
        out[i - 1] = c;
    }
}

static double finest_h(const Ora *o) { return (o->prob.hi[0] - o->prob.lo[0]) / o->nfx; }
static double cell_h(const Ora *o, int e) { return finest_h(o) * (double)(1 << (o->prob.max_level - o->lev[e])); }

/* physical node coordinates, [n][dim][npe]: x = x_left + (h/2)(xi + 1) */
void ora_node_coords(void *p, double *xy)
{
    Ora *o = (Ora *)p;
    double hf = finest_h(o);
    for (int e = 0; e < o->n; ++e) {
        double h = cell_h(o, e);
        double x0 = o->prob.lo[0] + o->fx[e] * hf, y0 = o->prob.lo[1] + o->fy[e] * hf;
        for (int q = 0; q < o->npe; ++q) {
            int i = q % NP, j = q / NP;
            if (o->prob.dim == 1) {
                xy[(size_t)e * o->npe + q] = x0 + 0.5 * h * (o->B.xi[i] + 1.0);
            } else {
                xy[((size_t)e * 2 + 0) * o->npe + q] = x0 + 0.5 * h * (o->B.xi[i] + 1.0);
                xy[((size_t)e * 2 + 1) * o->npe + q] = y0 + 0.5 * h * (o->B.xi[j] + 1.0);
            }
        }
    }
}

/* ------------------------------------------------------------------------- */
/* 3. fluxes                                                                 */
/* ------------------------------------------------------------------------- */
/* physical flux of the equation in direction `orient` */
static void phys_flux(const Ora *o, const double *u, int orient, double *f)
{
    double g = o->prob.gamma;
    if (o->prob.equation == 0) { f[0] = o->prob.adv * u[0]; return; }
    if (o->prob.dim == 1) {
        double rho = u[0], v = u[1] / rho, p = (g - 1.0) * (u[2] - 0.5 * rho * v * v);
        f[0] = rho * v; f[1] = rho * v * v + p; f[2] = (u[2] + p) * v;
        return;
    }
    double rho = u[0], v1 = u[1] / rho, v2 = u[2] / rho;
    double p = (g - 1.0) * (u[3] - 0.5 * rho * (v1 * v1 + v2 * v2));
    double vn = orient == 0 ? v1 : v2;
    f[0] = rho * vn;
    f[1] = rho * v1 * vn + (orient == 0 ? p : 0.0);
    f[2] = rho * v2 * vn + (orient == 1 ? p : 0.0);
    f[3] = (u[3] + p) * vn;
}

/* normal velocity and sound speed */
static void vn_c(const Ora *o, const double *u, int orient, double *vn, double *c)
{
    double g = o->prob.gamma;
    if (o->prob.dim == 1) {
        double rho = u[0], v = u[1] / rho, p = (g - 1.0) * (u[2] - 0.5 * rho * v * v);
        *vn = v; *c = sqrt(g * p / rho); return;
    }
    double rho = u[0], v1 = u[1] / rho, v2 = u[2] / rho;
    double p = (g - 1.0) * (u[3] - 0.5 * rho * (v1 * v1 + v2 * v2));
    *vn = orient == 0 ? v1 : v2; *c = sqrt(g * p / rho);
}

void ora_flux_ranocha(const double *uL, const double *uR, int orient, double g, double *f);

/* numerical flux f*(uL, uR) with uL on the low side of the face */
static void num_flux(const Ora *o, const double *uL, const double *uR, int orient, double *f)
{
    int nv = o->nv;
    if (o->prob.surface == 0) {          /* upwind for linear advection */
        if (o->prob.adv >= 0) f[0] = o->prob.adv * uL[0]; else f[0] = o->prob.adv * uR[0];
        return;
    }
    if (o->prob.surface == 3) { ora_flux_ranocha(uL, uR, orient, o->prob.gamma, f); return; }
    double fL[MAXV], fR[MAXV], vL, cL, vR, cR;
    phys_flux(o, uL, orient, fL); phys_flux(o, uR, orient, fR);
    vn_c(o, uL, orient, &vL, &cL); vn_c(o, uR, orient, &vR, &cR);
    if (o->prob.surface == 1) {          /* Rusanov / local Lax-Friedrichs */
        double lam = fmax(fabs(vL) + cL, fabs(vR) + cR);
        for (int v = 0; v < nv; ++v) f[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * lam * (uR[v] - uL[v]);
        return;
    }
    /* HLL with Davis wave-speed estimates */
    double sL = fmin(vL - cL, vR - cR), sR = fmax(vL + cL, vR + cR);
    if (sL >= 0.0) { for (int v = 0; v < nv; ++v) f[v] = fL[v]; return; }
    if (sR <= 0.0) { for (int v = 0; v < nv; ++v) f[v] = fR[v]; return; }
    for (int v = 0; v < nv; ++v)
        f[v] = (sR * fL[v] - sL * fR[v] + sL * sR * (uR[v] - uL[v])) / (sR - sL);
}

/* logarithmic mean (b - a) / (ln b - ln a), series in u = ((b-a)/(b+a))^2 near a = b
    */
double ora_ln_mean(double a, double b)
{
    double f = (b - a) / (b + a), u = f * f;
    if (u < 1e-4) return (a + b) / (2.0 + u * (2.0 / 3.0 + u * (2.0 / 5.0 + u * (2.0 / 7.0))));
    return (b - a) / log(b / a);
}

/* Ranocha's entropy-conserving and kinetic-energy-preserving two-point flux (cited by P:l.964,
   l.1437, l.1729), 2D Euler, direction `orient`. */
void ora_flux_ranocha(const double *uL, const double *uR, int orient, double g, double *f)
{
    double rL = uL[0], v1L = uL[1] / rL, v2L = uL[2] / rL, pL = (g - 1.0) * (uL[3] - 0.5 * rL * (v1L * v1L + v2L * v2L));
    double rR = uR[0], v1R = uR[1] / rR, v2R = uR[2] / rR, pR = (g - 1.0) * (uR[3] - 0.5 * rR * (v1R * v1R + v2R * v2R));
    double rho_hat = ora_ln_mean(rL, rR);
    double beta_hat = ora_ln_mean(rL / pL, rR / pR);
    double v1a = 0.5 * (v1L + v1R), v2a = 0.5 * (v2L + v2R), pa = 0.5 * (pL + pR);
    double vnL = orient == 0 ? v1L : v2L, vnR = orient == 0 ? v1R : v2R, vna = 0.5 * (vnL + vnR);
    double frho = rho_hat * vna;
    f[0] = frho;
    f[1] = frho * v1a + (orient == 0 ? pa : 0.0);
    f[2] = frho * v2a + (orient == 1 ? pa : 0.0);
    f[3] = frho * (0.5 * (v1L * v1R + v2L * v2R) + 1.0 / ((g - 1.0) * beta_hat)) + 0.5 * (pL * vnR + pR * vnL);
}

void ora_num_flux_pub(void *p, const double *uL, const double *uR, int orient, double *f)
{
    num_flux((Ora *)p, uL, uR, orient, f);
}

/* ------------------------------------------------------------------------- */
/* 4. RHS                                                                    */
/* ------------------------------------------------------------------------- */
#define UIDX(o, e, v, q) (((size_t)(e) * (o)->nv + (v)) * (o)->npe + (q))
#define FIDX(o, e, face, v, k) ((((size_t)(e) * 4 + (face)) * (o)->nv + (v)) * NP + (k))

/* node index of the k-th node on face `face` (0 +x, 1 -x, 2 +y, 3 -y); 1D: single node */
static int face_node(const Ora *o, int face, int k)
{
    if (o->prob.dim == 1) return face == 0 ? NP - 1 : 0;
    switch (face) {
    case 0: return k * NP + (NP - 1);
    case 1: return k * NP;
    case 2: return (NP - 1) * NP + k;
    default: return k;
    }
}

static void trace(const Ora *o, const double *U, int e, int face, int k, double *u)
{
    int q = face_node(o, face, k);
    for (int v = 0; v < o->nv; ++v) u[v] = U[UIDX(o, e, v, q)];
}

static void interface_flux(Ora *o, const double *U, int f)
{
    int eL = o->ifc[3 * f], eR = o->ifc[3 * f + 1], orient = o->ifc[3 * f + 2];
    int nk = o->prob.dim == 1 ? 1 : NP;
    for (int k = 0; k < nk; ++k) {
        double uL[MAXV], uR[MAXV], fl[MAXV];
        trace(o, U, eL, 2 * orient, k, uL);       /* +orient face of the low element */
        trace(o, U, eR, 2 * orient + 1, k, uR);   /* -orient face of the high element */
        num_flux(o, uL, uR, orient, fl);
        for (int v = 0; v < o->nv; ++v) {
            o->Fs[FIDX(o, eL, 2 * orient, v, k)] = fl[v];
            o->Fs[FIDX(o, eR, 2 * orient + 1, v, k)] = fl[v];
        }
    }
}

/* L2 mortar: interpolate the large trace to both halves (P_lower, P_upper), two numerical fluxes,
   the small elements take them directly, the large element gets R_lower f_lo + R_upper f_hi. */
static void mortar_flux(Ora *o, const double *U, int m)
{
    const int32_t *M = o->mor + 5 * m;
    int eL = M[0], orient = M[3], side = M[4];
    int large_face = 2 * orient + (side == 0 ? 0 : 1);   /* side 0: large element is the low side */
    int small_face = 2 * orient + (side == 0 ? 1 : 0);
    double ul[NP][MAXV];
    for (int k = 0; k < NP; ++k) trace(o, U, eL, large_face, k, ul[k]);
    double fh[2][NP][MAXV];
    for (int h = 0; h < 2; ++h) {
        int es = M[1 + h];
        for (int k = 0; k < NP; ++k) {
            double ui[MAXV], us[MAXV];
            for (int v = 0; v < o->nv; ++v) {
                double s = 0.0;
                for (int j = 0; j < NP; ++j) s += (h == 0 ? o->B.Plo[k][j] : o->B.Pup[k][j]) * ul[j][v];
                ui[v] = s;
            }
            trace(o, U, es, small_face, k, us);
            if (side == 0) num_flux(o, ui, us, orient, fh[h][k]);
            else num_flux(o, us, ui, orient, fh[h][k]);
            for (int v = 0; v < o->nv; ++v) o->Fs[FIDX(o, es, small_face, v, k)] = fh[h][k][v];
        }
    }
    for (int k = 0; k < NP; ++k)
        for (int v = 0; v < o->nv; ++v) {
            double s = 0.0;
            for (int j = 0; j < NP; ++j) s += o->B.Rlo[k][j] * fh[0][j][v] + o->B.Rup[k][j] * fh[1][j][v];
            o->Fs[FIDX(o, eL, large_face, v, k)] = s;
        }
}

static void boundary_flux(Ora *o, const double *U, int b)
{
    int e = o->bnd[2 * b], face = o->bnd[2 * b + 1], orient = face / 2, plus = face % 2 == 0;
    int nk = o->prob.dim == 1 ? 1 : NP;
    for (int k = 0; k < nk; ++k) {
        double ui[MAXV], fl[MAXV];
        trace(o, U, e, face, k, ui);
        if (plus) num_flux(o, ui, o->prob.bc_state, orient, fl);
        else num_flux(o, o->prob.bc_state, ui, orient, fl);
        for (int v = 0; v < o->nv; ++v) o->Fs[FIDX(o, e, face, v, k)] = fl[v];
    }
}

static void sc_subcell_volume(Ora *o, const double *U, int e, int i, int j, double *fv);

/* element RHS.  1D weak form (cfg 1-2):
     du_i = (2/h) [ sum_j Dhat_ij f(u_j) + (delta_i0 f*_L - delta_iN f*_R) / w_i ]
   2D flux differencing (cfg 3-5), per direction:
     du_ij -= (2/h) [ sum_k Dsplit_ik f#(u_ij, u_kj) + (delta_iN f*_R - delta_i0 f*_L) / w_i ]
   with shock capturing the volume part sum_k ... is blended with the subcell FV one (section 9) */
static void element_rhs(Ora *o, const double *U, int e, double *dU)
{
    double h = cell_h(o, e), J = 2.0 / h;
    int nv = o->nv;
    if (o->prob.dim == 1) {
        double f[NP][MAXV];
        for (int j = 0; j < NP; ++j) {
            double u[MAXV];
            for (int v = 0; v < nv; ++v) u[v] = U[UIDX(o, e, v, j)];
            phys_flux(o, u, 0, f[j]);
        }
        for (int i = 0; i < NP; ++i)
            for (int v = 0; v < nv; ++v) {
                double s = 0.0;
                for (int j = 0; j < NP; ++j) s += o->B.Dhat[i][j] * f[j][v];
                if (i == 0) s += o->Fs[FIDX(o, e, 1, v, 0)] / o->B.w[0];
                if (i == NP - 1) s -= o->Fs[FIDX(o, e, 0, v, 0)] / o->B.w[NP - 1];
                dU[UIDX(o, e, v, i)] = J * s;
            }
        return;
    }
    double g = o->prob.gamma;
    for (int j = 0; j < NP; ++j)
        for (int i = 0; i < NP; ++i) {
            double acc[MAXV] = {0, 0, 0, 0};
            double ui[MAXV];
            for (int v = 0; v < nv; ++v) ui[v] = U[UIDX(o, e, v, j * NP + i)];
            for (int k = 0; k < NP; ++k) {       /* x direction, line j */
                double uk[MAXV], f[MAXV];
                for (int v = 0; v < nv; ++v) uk[v] = U[UIDX(o, e, v, j * NP + k)];
                ora_flux_ranocha(ui, uk, 0, g, f);
                for (int v = 0; v < nv; ++v) acc[v] += o->B.Dsplit[i][k] * f[v];
            }
            for (int k = 0; k < NP; ++k) {       /* y direction, line i */
                double uk[MAXV], f[MAXV];
                for (int v = 0; v < nv; ++v) uk[v] = U[UIDX(o, e, v, k * NP + i)];
                ora_flux_ranocha(ui, uk, 1, g, f);
                for (int v = 0; v < nv; ++v) acc[v] += o->B.Dsplit[j][k] * f[v];
            }
            if (o->sc_on) {   /* section 9: (1 - alpha) V_DG + alpha V_FV */
                double fv[MAXV];
                sc_subcell_volume(o, U, e, i, j, fv);
                double a = o->alpha[e];
                for (int v = 0; v < nv; ++v) acc[v] = (1.0 - a) * acc[v] + a * fv[v];
            }
            for (int v = 0; v < nv; ++v) {
                double s = acc[v];
                if (i == NP - 1) s += o->Fs[FIDX(o, e, 0, v, j)] / o->B.w[NP - 1];
                if (i == 0) s -= o->Fs[FIDX(o, e, 1, v, j)] / o->B.w[0];
                if (j == NP - 1) s += o->Fs[FIDX(o, e, 2, v, i)] / o->B.w[NP - 1];
                if (j == 0) s -= o->Fs[FIDX(o, e, 3, v, i)] / o->B.w[0];
                dU[UIDX(o, e, v, j * NP + i)] = -J * s;
            }
        }
}


/* ------------------------------------------------------------------------- */
/* 4b. Navier-Stokes viscous terms, BR1 (P:l.1419-1420 cites Bassi-Rebay 1;  */
/*     the paper does not define it: SURVEY §8(c) O3 "BR1", D5; D7) */
/*   U_t + div F^a(U) = div F^v(U, grad w),  w = (rho, v1, v2, T = p/rho)     */
/*   1. q = grad w by the weak-form DG derivative with the central trace      */
/*      w* = (w_L + w_R)/2 (mortars: halves (P w_large + w_small)/2, large    */
/*      side = R_lower w*_lo + R_upper w*_hi)                                 */
/*   2. F^v(u, q) at the nodes: tau = mu (grad v + grad v^T - 2/3 div v I),   */
/*      heat flux kappa grad T, kappa = mu gamma / ((gamma - 1) Pr)           */
/*   3. central viscous face flux (F^v_L + F^v_R)/2 (mortars as in step 1,    */
/*      applied to the normal viscous flux traces)                            */
/*   4. du += (2/h) [ -Dhat F^v_x - Dhat F^v_y + surface lift ]  (weak form)  */
/* ------------------------------------------------------------------------- */
#define GIDX(o, e, face, v, k) ((((size_t)(e) * 4 + (face)) * 4 + (v)) * NP + (k))
#define QIDX(o, e, d, v, q) ((((size_t)(e) * 2 + (d)) * 4 + (v)) * (NP * NP) + (q))

/* gradient variables w = (rho, v1, v2, T), T = p / rho */
static void prim_w(const Ora *o, const double *u, double *w)
{
    double g = o->prob.gamma;
    double rho = u[0], v1 = u[1] / rho, v2 = u[2] / rho;
    double p = (g - 1.0) * (u[3] - 0.5 * rho * (v1 * v1 + v2 * v2));
    w[0] = rho; w[1] = v1; w[2] = v2; w[3] = p / rho;
}

/* viscous flux F^v_orient(u, q), q = (dw/dx, dw/dy) */
static void visc_flux(const Ora *o, const double *u, const double *qx, const double *qy, int orient, double *f)
{
    double mu = o->prob.mu, g = o->prob.gamma;
    double kappa = mu * g / ((g - 1.0) * o->prob.prandtl);
    double v1 = u[1] / u[0], v2 = u[2] / u[0];
    double v1x = qx[1], v2x = qx[2], Tx = qx[3];
    double v1y = qy[1], v2y = qy[2], Ty = qy[3];
    double t11 = mu * (4.0 / 3.0 * v1x - 2.0 / 3.0 * v2y);
    double t22 = mu * (4.0 / 3.0 * v2y - 2.0 / 3.0 * v1x);
    double t12 = mu * (v1y + v2x);
    f[0] = 0.0;
    if (orient == 0) {
        f[1] = t11; f[2] = t12; f[3] = v1 * t11 + v2 * t12 + kappa * Tx;
    } else {
        f[1] = t12; f[2] = t22; f[3] = v1 * t12 + v2 * t22 + kappa * Ty;
    }
}

static void trace_w(const Ora *o, const double *U, int e, int face, int k, double *w)
{
    double u[MAXV];
    trace(o, U, e, face, k, u);
    prim_w(o, u, w);
}

/* normal viscous flux at face node k of element e (orientation of the face) */
static void trace_fv(const Ora *o, const double *U, int e, int face, int k, double *f)
{
    int q = face_node(o, face, k);
    double u[MAXV], qx[4], qy[4];
    for (int v = 0; v < 4; ++v) {
        u[v] = U[UIDX(o, e, v, q)];
        qx[v] = o->Q[QIDX(o, e, 0, v, q)];
        qy[v] = o->Q[QIDX(o, e, 1, v, q)];
    }
    visc_flux(o, u, qx, qy, face / 2, f);
}

typedef void (*trace_fn)(const Ora *o, const double *U, int e, int face, int k, double *val);

/* central face value of a BR1 quantity (w for the gradient, F^v_n for the viscous flux) into the
   per-element face slots `out` ([n][4][4][NP]) */
static void central_interface(Ora *o, const double *U, int f, trace_fn tr, double *out)
{
    int eL = o->ifc[3 * f], eR = o->ifc[3 * f + 1], orient = o->ifc[3 * f + 2];
    for (int k = 0; k < NP; ++k) {
        double a[4], b[4];
        tr(o, U, eL, 2 * orient, k, a);
        tr(o, U, eR, 2 * orient + 1, k, b);
        for (int v = 0; v < 4; ++v) {
            double c = 0.5 * (a[v] + b[v]);
            out[GIDX(o, eL, 2 * orient, v, k)] = c;
            out[GIDX(o, eR, 2 * orient + 1, v, k)] = c;
        }
    }
}

static void central_mortar(Ora *o, const double *U, int m, trace_fn tr, double *out)
{
    const int32_t *M = o->mor + 5 * m;
    int eL = M[0], orient = M[3], side = M[4];
    int large_face = 2 * orient + (side == 0 ? 0 : 1);
    int small_face = 2 * orient + (side == 0 ? 1 : 0);
    double al[NP][4], ch[2][NP][4];
    for (int k = 0; k < NP; ++k) tr(o, U, eL, large_face, k, al[k]);
    for (int h = 0; h < 2; ++h) {
        int es = M[1 + h];
        for (int k = 0; k < NP; ++k) {
            double ai[4], as[4];
            for (int v = 0; v < 4; ++v) {
                double s = 0.0;
                for (int j = 0; j < NP; ++j) s += (h == 0 ? o->B.Plo[k][j] : o->B.Pup[k][j]) * al[j][v];
                ai[v] = s;
            }
            tr(o, U, es, small_face, k, as);
            for (int v = 0; v < 4; ++v) {
                ch[h][k][v] = 0.5 * (ai[v] + as[v]);
                out[GIDX(o, es, small_face, v, k)] = ch[h][k][v];
            }
        }
    }
    for (int k = 0; k < NP; ++k)
        for (int v = 0; v < 4; ++v) {
            double s = 0.0;
            for (int j = 0; j < NP; ++j) s += o->B.Rlo[k][j] * ch[0][j][v] + o->B.Rup[k][j] * ch[1][j][v];
            out[GIDX(o, eL, large_face, v, k)] = s;
        }
}

/* q = grad w of element e (weak form with the central traces in Gs):
     q_x[i,j] = (2/h) [ -sum_k Dhat_ik w[k,j] + (delta_iN w*_{+x}[j] - delta_i0 w*_{-x}[j]) / w_i ] */
static void element_grad(Ora *o, const double *U, int e)
{
    double J = 2.0 / cell_h(o, e);
    double w[NP * NP][4];
    for (int q = 0; q < NP * NP; ++q) {
        double u[MAXV];
        for (int v = 0; v < 4; ++v) u[v] = U[UIDX(o, e, v, q)];
        prim_w(o, u, w[q]);
    }
    for (int j = 0; j < NP; ++j)
        for (int i = 0; i < NP; ++i)
            for (int v = 0; v < 4; ++v) {
                double sx = 0.0, sy = 0.0;
                for (int k = 0; k < NP; ++k) {
                    sx -= o->B.Dhat[i][k] * w[j * NP + k][v];
                    sy -= o->B.Dhat[j][k] * w[k * NP + i][v];
                }
                if (i == NP - 1) sx += o->Gs[GIDX(o, e, 0, v, j)] / o->B.w[NP - 1];
                if (i == 0) sx -= o->Gs[GIDX(o, e, 1, v, j)] / o->B.w[0];
                if (j == NP - 1) sy += o->Gs[GIDX(o, e, 2, v, i)] / o->B.w[NP - 1];
                if (j == 0) sy -= o->Gs[GIDX(o, e, 3, v, i)] / o->B.w[0];
                o->Q[QIDX(o, e, 0, v, j * NP + i)] = J * sx;
                o->Q[QIDX(o, e, 1, v, j * NP + i)] = J * sy;
            }
}

/* du += (2/h) [ -sum_k Dhat_ik F^v_x[k,j] - sum_k Dhat_jk F^v_y[i,k] + viscous surface lift ] */
static void element_visc(Ora *o, const double *U, int e, double *dU)
{
    double J = 2.0 / cell_h(o, e);
    double fx[NP * NP][4], fy[NP * NP][4];
    for (int q = 0; q < NP * NP; ++q) {
        double u[MAXV], qx[4], qy[4];
        for (int v = 0; v < 4; ++v) {
            u[v] = U[UIDX(o, e, v, q)];
            qx[v] = o->Q[QIDX(o, e, 0, v, q)];
            qy[v] = o->Q[QIDX(o, e, 1, v, q)];
        }
        visc_flux(o, u, qx, qy, 0, fx[q]);
        visc_flux(o, u, qx, qy, 1, fy[q]);
    }
    for (int j = 0; j < NP; ++j)
        for (int i = 0; i < NP; ++i)
            for (int v = 0; v < 4; ++v) {
                double s = 0.0;
                for (int k = 0; k < NP; ++k) {
                    s -= o->B.Dhat[i][k] * fx[j * NP + k][v];
                    s -= o->B.Dhat[j][k] * fy[k * NP + i][v];
                }
                if (i == NP - 1) s += o->Fv[GIDX(o, e, 0, v, j)] / o->B.w[NP - 1];
                if (i == 0) s -= o->Fv[GIDX(o, e, 1, v, j)] / o->B.w[0];
                if (j == NP - 1) s += o->Fv[GIDX(o, e, 2, v, i)] / o->B.w[NP - 1];
                if (j == 0) s -= o->Fv[GIDX(o, e, 3, v, i)] / o->B.w[0];
                dU[UIDX(o, e, v, j * NP + i)] += J * s;
            }
}

/* dU = sum_{r in mask} I^(r) F(U) (P:l.289-301).
   mode 0 "reference": evaluate every face and element, then zero the unmasked elements.
   mode 1 "restricted": loop over the members in mask only, through the per-member lists;
   a mortar is evaluated whenever its (fine-side) member is in the mask (P:l.1256). */
static void sc_alpha(Ora *o, const double *U);

int ora_rhs(void *p, const double *U, uint32_t mask, double *dU, int mode)
{
    Ora *o = (Ora *)p;
    int R = o->tab.R;
    int ns = o->prob.equation == 2;
    if (o->sc_on) sc_alpha(o, U);   /* blending factors of every element from the stage state U */
    if (mode == 1) {
        /* the restricted loops are only equivalent to I^(r)F for upward-closed masks (every member
           finer than a masked one is masked too), which is what every P-ERK stage uses (P:l.428):
           a coarse element's mortar faces belong to the finer member (P:l.1256). */
        for (int r = 0; r + 1 < R; ++r)
            if (((mask >> r) & 1u) && !((mask >> (r + 1)) & 1u)) return -1;
        memset(o->Fs, 0, sizeof(double) * (size_t)o->n * 4 * o->nv * NP);
    }
    if (mode == 0) {
        if (ns) {   /* BR1 step 1: gradients everywhere */
            OMP_FOR
            for (int f = 0; f < o->n_if; ++f) central_interface(o, U, f, trace_w, o->Gs);
            OMP_FOR
            for (int m = 0; m < o->n_mo; ++m) central_mortar(o, U, m, trace_w, o->Gs);
            OMP_FOR
            for (int e = 0; e < o->n; ++e) element_grad(o, U, e);
        }
        OMP_FOR
        for (int f = 0; f < o->n_if; ++f) interface_flux(o, U, f);
        OMP_FOR
        for (int m = 0; m < o->n_mo; ++m) mortar_flux(o, U, m);
        OMP_FOR
        for (int b = 0; b < o->n_bd; ++b) boundary_flux(o, U, b);
        if (ns) {
            OMP_FOR
            for (int f = 0; f < o->n_if; ++f) central_interface(o, U, f, trace_fv, o->Fv);
            OMP_FOR
            for (int m = 0; m < o->n_mo; ++m) central_mortar(o, U, m, trace_fv, o->Fv);
        }
        OMP_FOR
        for (int e = 0; e < o->n; ++e) {
            element_rhs(o, U, e, dU);
            if (ns) element_visc(o, U, e, dU);
        }
        OMP_FOR
        for (int e = 0; e < o->n; ++e)
            if (!((mask >> o->member[e]) & 1u))
                for (int v = 0; v < o->nv; ++v)
                    for (int q = 0; q < o->npe; ++q) dU[UIDX(o, e, v, q)] = 0.0;
        return 0;
    }
    memset(dU, 0, sizeof(double) * (size_t)o->n * o->nv * o->npe);
    if (ns) {
        /* BR1 gradients are needed on the active elements and on their face neighbours across
           active mortars, which belong to the next coarser member: evaluate them over the members
           of mask | (mask >> 1).  Every face of such an element has a member in that set (a face
           belongs to its finer side, P:l.1256), so these gradients equal the full-F ones. */
        uint32_t ext = mask | (mask >> 1);
        for (int s = 0; s < R; ++s) {
            int r = R - 1 - s;
            if (!((ext >> r) & 1u)) continue;
            OMP_FOR
            for (int64_t t = o->seg[1][s]; t < o->seg[1][s + 1]; ++t) central_interface(o, U, o->list[1][t], trace_w, o->Gs);
            OMP_FOR
            for (int64_t t = o->seg[2][s]; t < o->seg[2][s + 1]; ++t) central_mortar(o, U, o->list[2][t], trace_w, o->Gs);
        }
        for (int s = 0; s < R; ++s) {
            int r = R - 1 - s;
            if (!((ext >> r) & 1u)) continue;
            OMP_FOR
            for (int64_t t = o->seg[0][s]; t < o->seg[0][s + 1]; ++t) element_grad(o, U, o->list[0][t]);
        }
    }
    for (int s = 0; s < R; ++s) {
        int r = R - 1 - s;
        if (!((mask >> r) & 1u)) continue;
        OMP_FOR
        for (int64_t t = o->seg[1][s]; t < o->seg[1][s + 1]; ++t) interface_flux(o, U, o->list[1][t]);
        OMP_FOR
        for (int64_t t = o->seg[2][s]; t < o->seg[2][s + 1]; ++t) mortar_flux(o, U, o->list[2][t]);
        OMP_FOR
        for (int64_t t = o->seg[3][s]; t < o->seg[3][s + 1]; ++t) boundary_flux(o, U, o->list[3][t]);
        if (ns) {
            OMP_FOR
            for (int64_t t = o->seg[1][s]; t < o->seg[1][s + 1]; ++t) central_interface(o, U, o->list[1][t], trace_fv, o->Fv);
            OMP_FOR
            for (int64_t t = o->seg[2][s]; t < o->seg[2][s + 1]; ++t) central_mortar(o, U, o->list[2][t], trace_fv, o->Fv);
        }
    }
    for (int s = 0; s < R; ++s) {
        int r = R - 1 - s;
        if (!((mask >> r) & 1u)) continue;
        OMP_FOR
        for (int64_t t = o->seg[0][s]; t < o->seg[0][s + 1]; ++t) {
            element_rhs(o, U, o->list[0][t], dU);
            if (ns) element_visc(o, U, o->list[0][t], dU);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 5. P-ERK step (materialised), P:l.209-218 and eq. PERK_ButcherTableauClassic  */
/* ------------------------------------------------------------------------- */
typedef void (*rhs_fn)(void *ctx, const double *U, uint32_t mask, double *dU);

/* Generic partitioned P-ERK step over `nunits` units of `usize` doubles, unit u in member[u]
   (P:l.209-218, eq. PartitionedRKSystem, with the two-nonzero rows of the P-ERK tableaux):
     K_1 = F(U_n)
     U^(i)|_r = U_n|_r + dt (a_{i,1}^(r) K_1|_r + a_{i,p(i)}^(r) K_{p(i)}|_r),  i = 2..S
        p(i) = the member's previous evaluated stage > 1 (= i-1 in the standard pattern; the
        alternating / early-shared rows of P:l.655-700); the row has no other nonzero a_{i,j}
     K_i|_r = I^(r) F(U^(i))  for the members r active at stage i (others: 0, never used)
     U_{n+1} = U_n + dt sum_i b_i K_i   (shared b: P-ERK2 b = e_S, P:l.423; Heun / Ralston b_1, b_S,
                                         P:l.439-442; P-ERK3 Shu-Osher b = (1/6, 0, .., 0, 1/6, 4/6),
                                         P:l.872-883)
   Kp holds, per unit, K of its member's most recent evaluated stage > 1 (zero before the first),
   which is K_{p(i)} when stage i is evaluated.  The weighted sum is accumulated stage by stage in
   the order i = 1..S (terms with b_i = 0 add an exact zero, so b = e_S gives U_n + dt K_S
   bitwise).                                                                                  */
static int64_t perk_step_generic(const OraTableau *t, int nunits, int usize, const int32_t *member,
                                 double *U, double dt, rhs_fn F, void *ctx)
{
    size_t nd = (size_t)nunits * usize;
    double *K1 = (double *)malloc(sizeof(double) * nd);
    double *Kp = (double *)malloc(sizeof(double) * nd);
    double *Kn = (double *)malloc(sizeof(double) * nd);
    double *Us = (double *)malloc(sizeof(double) * nd);
    double *Ksum = (double *)malloc(sizeof(double) * nd);
    int64_t evals = 0;
    uint32_t all = (t->R >= 32) ? 0xffffffffu : ((1u << t->R) - 1u);
    F(ctx, U, all, K1);
    evals += nunits;
    memset(Kp, 0, sizeof(double) * nd);
    for (size_t d = 0; d < nd; ++d) Ksum[d] = 0.0 + t->b[0] * K1[d];
    for (int i = 2; i <= t->S; ++i) {
        OMP_FOR
        for (int u = 0; u < nunits; ++u) {
            int r = member[u];
            double a1 = t->a1[r][i - 1], as = t->asub[r][i - 1];
            for (int q = 0; q < usize; ++q) {
                size_t d = (size_t)u * usize + q;
                Us[d] = U[d] + dt * (a1 * K1[d] + as * Kp[d]);
            }
        }
        uint32_t mask = 0;
        for (int r = 0; r < t->R; ++r)
            if (tab_active(t, r, i)) mask |= 1u << r;
        F(ctx, Us, mask, Kn);
        for (int u = 0; u < nunits; ++u) {
            size_t d0 = (size_t)u * usize;
            if ((mask >> member[u]) & 1u) {
                evals++;
                for (int q = 0; q < usize; ++q) Kp[d0 + q] = Kn[d0 + q];
            } else {
                for (int q = 0; q < usize; ++q) Kn[d0 + q] = 0.0;   /* K_i^(r) = 0: I^(r) mask */
            }
        }
        for (size_t d = 0; d < nd; ++d) Ksum[d] = Ksum[d] + t->b[i - 1] * Kn[d];
    }
    for (size_t d = 0; d < nd; ++d) U[d] = U[d] + dt * Ksum[d];
    free(K1); free(Kp); free(Kn); free(Us); free(Ksum);
    return evals;
}

static int g_rhs_mode;
/* restricted mode needs an upward-closed member mask (every standard-pattern stage); the stage masks of
   other patterns can be any set, and fall back to the definition (full F, then the mask) */
static void dg_rhs_cb(void *ctx, const double *U, uint32_t mask, double *dU)
{
    if (ora_rhs(ctx, U, mask, dU, g_rhs_mode) != 0) (void)ora_rhs(ctx, U, mask, dU, 0);
}

/* one P-ERK step of the DG system; returns element-RHS evaluations of this step */
int64_t ora_step(void *p, double *U, double dt, int mode)
{
    Ora *o = (Ora *)p;
    g_rhs_mode = mode;
    int64_t ev = perk_step_generic(&o->tab, o->n, o->nv * o->npe, o->member, U, dt, dg_rhs_cb, o);
    o->elem_rhs_count += ev;
    return ev;
}

int64_t ora_steps(void *p, double *U, double dt, int nsteps, int mode)
{
    int64_t ev = 0;
    for (int s = 0; s < nsteps; ++s) ev += ora_step(p, U, dt, mode);
    return ev;
}

/* ------------------------------------------------------------------------- */
/* 6. re-mesh transfer: new leaf at the same level -> copy; finer -> interpolate the parent to the   */
/*    child's nodes (tensor P_lower/P_upper); coarser -> exact L2 projection of the 4 children.      */
/* ------------------------------------------------------------------------- */
int ora_transfer(void *pold, void *pnew, const double *Uold, double *Unew)
{
    Ora *a = (Ora *)pold, *b = (Ora *)pnew;
    int L = b->prob.max_level, nv = b->nv;
    if (b->prob.dim != 2) return -1;
    for (int e = 0; e < b->n; ++e) {
        int l = b->lev[e], s = 1 << (L - l);
        int eo = a->cell_of[(int64_t)b->fy[e] * a->nfx + b->fx[e]];
        int lo_ = a->lev[eo];
        if (lo_ == l) {
            for (int v = 0; v < nv; ++v)
                for (int q = 0; q < NP * NP; ++q) Unew[UIDX(b, e, v, q)] = Uold[UIDX(a, eo, v, q)];
        } else if (lo_ == l - 1) {
            int sp = 2 * s;
            int cx = ((b->fx[e] - a->fx[eo]) / s) & 1, cy = ((b->fy[e] - a->fy[eo]) / s) & 1;
            (void)sp;
            const double (*Px)[NP] = cx ? b->B.Pup : b->B.Plo;
            const double (*Py)[NP] = cy ? b->B.Pup : b->B.Plo;
            for (int v = 0; v < nv; ++v)
                for (int j = 0; j < NP; ++j)
                    for (int i = 0; i < NP; ++i) {
                        double sum = 0.0;
                        for (int l2 = 0; l2 < NP; ++l2)
                            for (int k = 0; k < NP; ++k)
                                sum += Py[j][l2] * Px[i][k] * Uold[UIDX(a, eo, v, l2 * NP + k)];
                        Unew[UIDX(b, e, v, j * NP + i)] = sum;
                    }
        } else if (lo_ == l + 1) {
            int h = s / 2;
            for (int v = 0; v < nv; ++v)
                for (int q = 0; q < NP * NP; ++q) Unew[UIDX(b, e, v, q)] = 0.0;
            for (int cy = 0; cy < 2; ++cy)
                for (int cx = 0; cx < 2; ++cx) {
                    int ec = a->cell_of[(int64_t)(b->fy[e] + cy * h) * a->nfx + b->fx[e] + cx * h];
                    if (a->lev[ec] != l + 1) return -2;
                    const double (*Rx)[NP] = cx ? b->B.Rup : b->B.Rlo;
                    const double (*Ry)[NP] = cy ? b->B.Rup : b->B.Rlo;
                    for (int v = 0; v < nv; ++v)
                        for (int j = 0; j < NP; ++j)
                            for (int i = 0; i < NP; ++i) {
                                double sum = 0.0;
                                for (int l2 = 0; l2 < NP; ++l2)
                                    for (int k = 0; k < NP; ++k)
                                        sum += Ry[j][l2] * Rx[i][k] * Uold[UIDX(a, ec, v, l2 * NP + k)];
                                Unew[UIDX(b, e, v, j * NP + i)] += sum;
                            }
                }
        } else {
            return -3;  /* |level change| > 1 */
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 7. FV Godunov testbed (P:l.479-520, eq. UpwindFullSystem): du_j = -(F_{j+1/2} - F_{j-1/2})/dx_j, */
/*    periodic; kind 0 linear advection with speed a > 0 (F = a u_left), kind 1 Burgers (exact     */
/*    Godunov flux for f = u^2/2).                                                                 */
/* ------------------------------------------------------------------------- */
typedef struct { int n; const double *dx; int kind; double a; } FvCtx;

static double godunov_burgers(double uL, double uR)
{
    if (uL > uR) {                       /* shock, speed (uL + uR)/2 */
        double s = 0.5 * (uL + uR);
        return s > 0.0 ? 0.5 * uL * uL : 0.5 * uR * uR;
    }
    if (uL > 0.0) return 0.5 * uL * uL;  /* rarefaction */
    if (uR < 0.0) return 0.5 * uR * uR;
    return 0.0;                          /* sonic point */
}

void ora_fv_rhs(int n, const double *dx, const double *U, double *dU, int kind, double a)
{
    for (int j = 0; j < n; ++j) {
        int jm = (j - 1 + n) % n, jp = (j + 1) % n;
        double Fm, Fp;
        if (kind == 0) { Fm = a * U[jm]; Fp = a * U[j]; }
        else { Fm = godunov_burgers(U[jm], U[j]); Fp = godunov_burgers(U[j], U[jp]); }
        dU[j] = -(Fp - Fm) / dx[j];
    }
}

static void fv_rhs_cb(void *ctx, const double *U, uint32_t mask, double *dU)
{
    FvCtx *c = (FvCtx *)ctx;
    (void)mask;  /* full F; the stepper only uses the masked components (reference mode) */
    ora_fv_rhs(c->n, c->dx, U, dU, c->kind, c->a);
}

void ora_fv_step(int n, const double *dx, const int32_t *member, const OraTableau *t,
                 double *U, double dt, int kind, double a)
{
    FvCtx c = {n, dx, kind, a};
    perk_step_generic(t, n, 1, member, U, dt, fv_rhs_cb, &c);
}

/* ------------------------------------------------------------------------- */
/* 8. AMR indicators and the level controller (A1-A6).  2D, Euler / NS.  */
/*    The paper uses indicator-driven AMR (Loehner on v_x, P:l.1440-1441; Hennemann-Gassner on rho  */
/*    or rho*p, P:l.1548, l.1731, l.1886; enstrophy eps = 0.5 rho w.w with a threshold, P:l.1615-   */
/*    1622, eq. Enstrophy) but defines neither the cited indicators nor the controller: the         */
/*    readings below restate the cited published methods and are listed in DESIGN.md.              */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t indicator;      /* 0 Hennemann-Gassner, 1 Loehner, 2 enstrophy */
    int32_t variable;       /* 0 rho, 1 p, 2 rho*p, 3 v_x, 4 v_y (ignored by enstrophy) */
    int32_t base_level, med_level, max_level, _pad;
    double med_threshold, max_threshold;
    double alpha_max, alpha_min;   /* Hennemann-Gassner */
    double f_wave;                 /* Loehner */
} OraAmr;

/* indicator variable at one node from the conserved state (rho, rho v1, rho v2, E) */
static double amr_variable(const Ora *o, const double *u, int var)
{
    double rho = u[0], vx = u[1] / rho, vy = u[2] / rho;
    double p = (o->prob.gamma - 1.0) * (u[3] - 0.5 * rho * (vx * vx + vy * vy));
    switch (var) {
    case 0: return rho;
    case 1: return p;
    case 2: return rho * p;
    case 3: return vx;
    default: return vy;
    }
}

/* orthonormal Legendre polynomial Ptilde_k(x) = sqrt((2k+1)/2) P_k(x), Bonnet's recursion */
static double legendre_orthonormal(int k, double x)
{
    double p0 = 1.0, p1 = x;
    if (k == 0) return sqrt(0.5);
    for (int m = 1; m < k; ++m) {
        double p2 = ((2.0 * m + 1.0) * x * p1 - m * p0) / (m + 1.0);
        p0 = p1;
        p1 = p2;
    }
    return sqrt((2.0 * k + 1.0) / 2.0) * p1;
}

/* A1 Hennemann-Gassner (cited at P:l.1548): modal coefficients m_kl of the nodal values in the
   orthonormal Legendre basis (u(x,y) = sum_kl m_kl Ptilde_k(x) Ptilde_l(y) interpolates the nodes);
   energy fractions of the highest mode and of the second-highest mode:
     E = max((sum_all - sum_{k,l<=N-1}) / sum_all, (sum_{k,l<=N-1} - sum_{k,l<=N-2}) / sum_{k,l<=N-1})
   (a quotient with a zero denominator counts as 0); threshold T = 0.5 10^(-1.8 (N+1)^(1/4)),
   sharpness s = ln((1 - 1e-4) / 1e-4), alpha = 1 / (1 + exp(-(s / T)(E - T))); alpha < alpha_min -> 0,
   alpha > 1 - alpha_min -> 1; alpha = min(alpha, alpha_max). */
static double indicator_hg(const Ora *o, const double *val, const OraAmr *a)
{
    double V[NP][NP], Vinv[NP][NP];
    for (int i = 0; i < NP; ++i)
        for (int k = 0; k < NP; ++k) V[i][k] = legendre_orthonormal(k, o->B.xi[i]);
    for (int c = 0; c < NP; ++c) {      /* column c of V^-1: solve V x = e_c */
        double col[NP] = {0, 0, 0, 0};
        col[c] = 1.0;
        solve4(V, col);
        for (int k = 0; k < NP; ++k) Vinv[k][c] = col[k];
    }
    double tot = 0.0, clip1 = 0.0, clip2 = 0.0;
    for (int l = 0; l < NP; ++l)
        for (int k = 0; k < NP; ++k) {
            double m = 0.0;
            for (int j = 0; j < NP; ++j)
                for (int i = 0; i < NP; ++i) m += Vinv[k][i] * Vinv[l][j] * val[j * NP + i];
            double m2 = m * m;
            tot += m2;
            if (k <= NP - 2 && l <= NP - 2) clip1 += m2;
            if (k <= NP - 3 && l <= NP - 3) clip2 += m2;
        }
    double e1 = tot > 0.0 ? (tot - clip1) / tot : 0.0;
    double e2 = clip1 > 0.0 ? (clip1 - clip2) / clip1 : 0.0;
    double E = e1 > e2 ? e1 : e2;
    double T = 0.5 * pow(10.0, -1.8 * pow((double)NP, 0.25));
    double s = log((1.0 - 0.0001) / 0.0001);
    double alpha = 1.0 / (1.0 + exp(-(s / T) * (E - T)));
    if (alpha < a->alpha_min) alpha = 0.0;
    else if (alpha > 1.0 - a->alpha_min) alpha = 1.0;
    return alpha < a->alpha_max ? alpha : a->alpha_max;
}

/* A2 Loehner (cited at P:l.1440-1441, LGL adaptation of P:l.1441): along every x and y node line,
   at every interior node: |u+ - 2 u0 + u-| / (|u+ - u0| + |u0 - u-| + f_wave (|u+| + 2|u0| + |u-|)),
   0 where the denominator vanishes; the element value is the maximum. */
static double lohner_estimate(double um, double u0, double up, double fw)
{
    double num = fabs(up - 2.0 * u0 + um);
    double den = fabs(up - u0) + fabs(u0 - um) + fw * (fabs(up) + 2.0 * fabs(u0) + fabs(um));
    return den > 0.0 ? num / den : 0.0;
}

static double indicator_lohner(const double *val, const OraAmr *a)
{
    double mx = 0.0;
    for (int j = 0; j < NP; ++j)
        for (int i = 1; i < NP - 1; ++i) {
            double ex = lohner_estimate(val[j * NP + i - 1], val[j * NP + i], val[j * NP + i + 1], a->f_wave);
            double ey = lohner_estimate(val[(i - 1) * NP + j], val[i * NP + j], val[(i + 1) * NP + j], a->f_wave);
            if (ex > mx) mx = ex;
            if (ey > mx) mx = ey;
        }
    return mx;
}

/* A3 enstrophy eps = 0.5 rho w.w (P:l.1615-1622, eq. Enstrophy), 2D vorticity w = dv_y/dx - dv_x/dy
   of the nodal interpolant (D_ij = l_j'(xi_i), times 2/h); the element value is the maximum over
   its nodes. */
static double indicator_enstrophy(const Ora *o, const double *U, int e)
{
    double J = 2.0 / cell_h(o, e), mx = 0.0;
    double vx[NP * NP], vy[NP * NP];
    for (int q = 0; q < NP * NP; ++q) {
        vx[q] = U[UIDX(o, e, 1, q)] / U[UIDX(o, e, 0, q)];
        vy[q] = U[UIDX(o, e, 2, q)] / U[UIDX(o, e, 0, q)];
    }
    for (int j = 0; j < NP; ++j)
        for (int i = 0; i < NP; ++i) {
            double dvydx = 0.0, dvxdy = 0.0;
            for (int k = 0; k < NP; ++k) {
                dvydx += o->B.D[i][k] * vy[j * NP + k];
                dvxdy += o->B.D[j][k] * vx[k * NP + i];
            }
            double w = J * dvydx - J * dvxdy;
            double eps = 0.5 * U[UIDX(o, e, 0, j * NP + i)] * w * w;
            if (eps > mx) mx = eps;
        }
    return mx;
}

static int amr_check(const Ora *o, const OraAmr *a)
{
    if (o->prob.dim != 2 || o->prob.equation == 0) return -2;
    if (a->indicator < 0 || a->indicator > 2 || a->variable < 0 || a->variable > 4) return -1;
    if (a->base_level < 0 || a->base_level > a->med_level || a->med_level > a->max_level ||
        a->max_level > o->prob.max_level || !(a->med_threshold <= a->max_threshold)) return -1;
    return 0;
}

int ora_amr_indicator(void *p, const double *U, const OraAmr *a, double *ind)
{
    Ora *o = (Ora *)p;
    int rc = amr_check(o, a);
    if (rc) return rc;
    for (int e = 0; e < o->n; ++e) {
        if (a->indicator == 2) { ind[e] = indicator_enstrophy(o, U, e); continue; }
        double val[NP * NP];
        for (int q = 0; q < NP * NP; ++q) {
            double u[MAXV];
            for (int v = 0; v < 4; ++v) u[v] = U[UIDX(o, e, v, q)];
            val[q] = amr_variable(o, u, a->variable);
        }
        ind[e] = a->indicator == 0 ? indicator_hg(o, val, a) : indicator_lohner(val, a);
    }
    return 0;
}

/* A4-A6 controller (three levels) and 2:1 balance, writing the new finest-grid level map:
   A4 target(e) = base_level if ind <= med_threshold, med_level if ind <= max_threshold, else
      max_level; a leaf moves at most one level per adaptation toward its target;
   A5 a leaf coarsens only together with its three siblings (all four leaves at the same level,
      all four wanting to coarsen);
   A6 2:1 face balance (the condition perk_init / perk_repartition check) is restored by refining:
      while some leaf has a face neighbour two or more levels finer, split that leaf. */
int ora_amr_adapt_ind(void *p, const double *ind, const OraAmr *a, uint8_t *lmap);

int ora_amr_adapt(void *p, const double *U, const OraAmr *a, uint8_t *lmap)
{
    Ora *o = (Ora *)p;
    int rc = amr_check(o, a);
    if (rc) return rc;
    double *ind = (double *)malloc(sizeof(double) * o->n);
    ora_amr_indicator(p, U, a, ind);
    rc = ora_amr_adapt_ind(p, ind, a, lmap);
    free(ind);
    return rc;
}

/* the controller + balance alone, on a given per-leaf indicator (tests: the same decisions from
   another implementation's indicator values) */
int ora_amr_adapt_ind(void *p, const double *ind, const OraAmr *a, uint8_t *lmap)
{
    Ora *o = (Ora *)p;
    int rc = amr_check(o, a);
    if (rc) return rc;
    int L = o->prob.max_level;
    int *want = (int *)malloc(sizeof(int) * o->n);
    for (int e = 0; e < o->n; ++e) {
        int target = ind[e] <= a->med_threshold ? a->base_level
                   : (ind[e] <= a->max_threshold ? a->med_level : a->max_level);
        int l = o->lev[e];
        want[e] = target > l ? l + 1 : (target < l ? l - 1 : l);
    }
    for (int e = 0; e < o->n; ++e) {
        int l = o->lev[e], s = 1 << (L - l), newl = want[e];
        if (want[e] < l) {              /* A5: the four children of the parent block */
            int px = o->fx[e] - o->fx[e] % (2 * s), py = o->fy[e] - o->fy[e] % (2 * s);
            for (int cy = 0; cy < 2; ++cy)
                for (int cx = 0; cx < 2; ++cx) {
                    int c = o->cell_of[(int64_t)(py + cy * s) * o->nfx + px + cx * s];
                    if (o->lev[c] != l || want[c] >= l) newl = l;
                }
        }
        for (int y = 0; y < s; ++y)
            for (int x = 0; x < s; ++x) lmap[(int64_t)(o->fy[e] + y) * o->nfx + o->fx[e] + x] = (uint8_t)newl;
    }
    int changed = 1;
    while (changed) {               /* A6 */
        changed = 0;
        for (int y = 0; y < o->nfy; ++y)
            for (int x = 0; x < o->nfx; ++x) {
                int l = lmap[(int64_t)y * o->nfx + x];
                for (int d = 0; d < 4; ++d) {
                    int nx = x + (d == 0) - (d == 1), ny = y + (d == 2) - (d == 3);
                    if (nx < 0 || nx >= o->nfx) { if (!o->prob.periodic[0]) continue; nx = wrapi(nx, o->nfx); }
                    if (ny < 0 || ny >= o->nfy) { if (!o->prob.periodic[1]) continue; ny = wrapi(ny, o->nfy); }
                    if (lmap[(int64_t)ny * o->nfx + nx] >= l + 2) {   /* split the leaf holding (x, y) */
                        int s = 1 << (L - l), ox = x - x % s, oy = y - y % s;
                        for (int yy = 0; yy < s; ++yy)
                            for (int xx = 0; xx < s; ++xx) lmap[(int64_t)(oy + yy) * o->nfx + ox + xx] = (uint8_t)(l + 1);
                        changed = 1;
                        break;
                    }
                }
            }
    }
    free(want);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 9. subcell shock capturing (Hennemann & Gassner 2021, cited by the paper   */
/*    for every inviscid application: P:l.964, l.1729, l.1795-1799, l.1856)   */
/*    DESIGN.md readings A7-A9.  Per element:                                 */
/*      V = (1 - alpha) V_DG + alpha V_FV                                     */
/*    V_DG = sum_k Dsplit_ik f#(u_i, u_k) (flux differencing, section 4);     */
/*    V_FV = (F_{i+1/2} - F_{i-1/2}) / w_i along each node line, with the     */
/*    subcell fluxes F_{i+1/2} = f*(u_i, u_{i+1}) (the surface flux of the    */
/*    problem) between neighbouring LGL nodes and F_{-1/2} = F_{N+1/2} = 0:   */
/*    with the unchanged surface term (f*_R at node N, f*_L at node 0) this   */
/*    is the first-order FV scheme on the subcells of widths w_i h / 2.       */
/*    alpha: Hennemann-Gassner indicator (section 8, A1) of the chosen        */
/*    variable on the element's stage state, then optional smoothing         */
/*    alpha_e = max(alpha_e, alpha_n / 2) over the face neighbours n (across  */
/*    interfaces and mortars, raw neighbour values).                          */
/* ------------------------------------------------------------------------- */
static void sc_subcell_volume(Ora *o, const double *U, int e, int i, int j, double *fv)
{
    int nv = o->nv;
    for (int v = 0; v < nv; ++v) fv[v] = 0.0;
    for (int d = 0; d < 2; ++d) {              /* d = 0: x line j, node i; d = 1: y line i, node j */
        int a = d == 0 ? i : j;
        double u[NP][MAXV];
        for (int k = 0; k < NP; ++k) {
            int q = d == 0 ? j * NP + k : k * NP + i;
            for (int v = 0; v < nv; ++v) u[k][v] = U[UIDX(o, e, v, q)];
        }
        double Fr[MAXV] = {0, 0, 0, 0}, Fl[MAXV] = {0, 0, 0, 0};
        if (a < NP - 1) num_flux(o, u[a], u[a + 1], d, Fr);
        if (a > 0) num_flux(o, u[a - 1], u[a], d, Fl);
        for (int v = 0; v < nv; ++v) fv[v] += (Fr[v] - Fl[v]) / o->B.w[a];
    }
}

static void sc_alpha(Ora *o, const double *U)
{
    OraAmr a;
    memset(&a, 0, sizeof(a));
    a.variable = o->sc.variable;
    a.alpha_max = o->sc.alpha_max;
    a.alpha_min = o->sc.alpha_min;
    OMP_FOR
    for (int e = 0; e < o->n; ++e) {
        if (o->sc.alpha_fixed >= 0.0) { o->alpha_raw[e] = o->sc.alpha_fixed; continue; }
        double val[NP * NP];
        for (int q = 0; q < NP * NP; ++q) {
            double u[MAXV];
            for (int v = 0; v < 4; ++v) u[v] = U[UIDX(o, e, v, q)];
            val[q] = amr_variable(o, u, a.variable);
        }
        o->alpha_raw[e] = indicator_hg(o, val, &a);
    }
    for (int e = 0; e < o->n; ++e) o->alpha[e] = o->alpha_raw[e];
    if (!o->sc.smooth) return;
    for (int f = 0; f < o->n_if; ++f) {
        int eL = o->ifc[3 * f], eR = o->ifc[3 * f + 1];
        o->alpha[eL] = fmax(o->alpha[eL], 0.5 * o->alpha_raw[eR]);
        o->alpha[eR] = fmax(o->alpha[eR], 0.5 * o->alpha_raw[eL]);
    }
    for (int m = 0; m < o->n_mo; ++m) {
        const int32_t *M = o->mor + 5 * m;
        for (int h = 0; h < 2; ++h) {
            o->alpha[M[0]] = fmax(o->alpha[M[0]], 0.5 * o->alpha_raw[M[1 + h]]);
            o->alpha[M[1 + h]] = fmax(o->alpha[M[1 + h]], 0.5 * o->alpha_raw[M[0]]);
        }
    }
}

/* sc = NULL switches shock capturing off.  -2: not a 2D Euler / Navier-Stokes flux-differencing
   problem; -1: invalid parameters */
int ora_set_shock_capturing(void *p, const OraSC *sc)
{
    Ora *o = (Ora *)p;
    if (!sc) { o->sc_on = 0; return 0; }
    if (o->prob.dim != 2 || o->prob.equation == 0 || o->prob.volume != 1) return -2;
    if (sc->variable < 0 || sc->variable > 4 || !(sc->alpha_min >= 0.0) || !(sc->alpha_max >= 0.0) ||
        !(sc->alpha_max <= 1.0) || !(sc->alpha_fixed <= 1.0)) return -1;
    o->sc = *sc;
    if (!o->alpha) {
        o->alpha_raw = (double *)calloc((size_t)o->n, sizeof(double));
        o->alpha = (double *)calloc((size_t)o->n, sizeof(double));
    }
    o->sc_on = 1;
    return 0;
}

/* blending factors of U (raw indicator and smoothed), canonical leaf order; -1 if off */
int ora_sc_alpha(void *p, const double *U, double *raw, double *smoothed)
{
    Ora *o = (Ora *)p;
    if (!o->sc_on) return -1;
    sc_alpha(o, U);
    memcpy(raw, o->alpha_raw, sizeof(double) * (size_t)o->n);
    memcpy(smoothed, o->alpha, sizeof(double) * (size_t)o->n);
    return 0;
}
