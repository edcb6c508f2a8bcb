// common.cuh -- shared device definitions of libperk_b200 (sm_100a, fp64).
//
// Layouts:
//   U, K1, Ubuf : [cell][var][node], node = j*4 + i (x fastest); 2D Euler cell = 64 doubles = 512 B
//   Fs          : [cell][face 0..3 = +x,-x,+y,-y][var][k], k = node along the face; 512 B per 2D cell
//   interfaces  : int4 {low elem, high elem, orientation, member}
//   mortars     : int4 {large, small_lo, small_hi, orientation | side << 1 | member << 8}
//   boundaries  : int2 {elem, face | member << 8}
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace perk {

constexpr int NP = 4;          // N + 1 LGL nodes per direction (N = 3)
constexpr int MAXV = 4;
constexpr int MAXS = 64;
constexpr int MAXR = 8;
constexpr int SM_COUNT_B200 = 148;

enum Kind { KIND_EL = 0, KIND_IF = 1, KIND_MO = 2, KIND_BD = 3 };
// count_active[EXT_OFF + kind * MAXS + i - 1]: items of the active members at stage i plus the next
// coarser member (BR1 gradients are needed one element beyond the active set across mortars)
constexpr int EXT_OFF = 4 * MAXS;
enum Mode { MODE_STAGE = 0, MODE_RHS = 1 };
enum ErrBits { ERR_UNBALANCED = 1, ERR_CAPACITY = 2, ERR_TRANSFER = 4 };

// DGSEM N=3 tables, generated on the host by basis.cuh and uploaded once per process.
struct BasisTables {
    double xi[NP], w[NP], invw[NP];
    double Dhat[NP][NP];    // weak form
    double Dsplit[NP][NP];  // flux differencing (2D - boundary corrections)
    double Plo[NP][NP], Pup[NP][NP];
    double Rlo[NP][NP], Rup[NP][NP];
};
__constant__ BasisTables cB;

// Device-resident mesh state.  All counts live in device memory so that captured graphs
// stay valid across repartitions.
struct MeshDev {
    int dim, nv, npe, max_level, nfx, nfy;
    int periodic[2];
    int equation, surface;
    double lo[2], hf;            // domain origin, finest cell size
    double gamma, adv;
    double mu, kappa;            // Navier-Stokes: viscosity, heat conductivity mu gamma / ((gamma - 1) Pr)
    double bc[MAXV];
    int cap;                     // cell capacity
    // device pointers
    int *n;                      // [4]: cells, interfaces, mortars, boundaries
    int *count_active;           // [4][MAXS] stage prefix counts, then [4][MAXS] BR1 gradient prefixes (EXT_OFF)
    int *seg;                    // [4][MAXR+1]
    int *err;                    // error flag bits
    unsigned long long *evals;   // element-RHS evaluation counter
    int *list[4];                // per-kind member-sorted item lists
    int *fx, *fy;                // leaf origin (finest grid)
    uint8_t *lev, *mem;          // leaf level, member
    int *cell_of;                // finest cell -> leaf
    int4 *ifc; int4 *mor; int2 *bnd;
};

// Per-launch stage parameters (kernel argument, graph-captured).
struct StageParams {
    int stage;                   // 1..S
    int S;
    int R;
    int mode;                    // MODE_STAGE / MODE_RHS
    unsigned mask;               // rhs_eval partition mask
    double dt;
    double c_stage;              // c_i (lazy state U_n + dt c_i K_1)
    int first[MAXR];             // f(r) = S - E_r + 2: first active stage after 1
    double a1_next[MAXR];        // a_{i+1,1}^{(r)}
    double asub_next[MAXR];      // a_{i+1,i}^{(r)}
};

// Which buffer holds element e's stage-i state (SURVEY §7 rule):
//   i == 1: U_n;  i > f(e): Ubuf;  2 <= i <= f(e): U_n + dt c_i K_1 (formed on the fly)
enum StateSrc { SRC_UN = 0, SRC_BUF = 1, SRC_LAZY = 2, SRC_IN = 3 };

__device__ __forceinline__ int state_src(const StageParams &sp, int member)
{
    if (sp.mode == MODE_RHS) return SRC_IN;
    if (sp.stage == 1) return SRC_UN;
    return sp.stage > sp.first[member] ? SRC_BUF : SRC_LAZY;
}

struct StateBufs {
    const double *Un;
    const double *Ubuf;
    const double *K1;
    const double *Uin;
};

__device__ __forceinline__ double load_state(const StateBufs &sb, int src, double dtc, size_t idx)
{
    switch (src) {
    case SRC_UN: return __ldg(sb.Un + idx);
    case SRC_BUF: return __ldg(sb.Ubuf + idx);
    case SRC_LAZY: return fma(dtc, __ldg(sb.K1 + idx), __ldg(sb.Un + idx));
    default: return __ldg(sb.Uin + idx);
    }
}

// node index of the k-th node on face f (0 +x, 1 -x, 2 +y, 3 -y)
__device__ __forceinline__ int face_node2d(int face, int k)
{
    switch (face) {
    case 0: return k * NP + (NP - 1);
    case 1: return k * NP;
    case 2: return (NP - 1) * NP + k;
    default: return k;
    }
}

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// fast fp64 reciprocal: MUFU approximation + two Newton steps (<= 1 ulp from the IEEE result)
__device__ __forceinline__ double rcp64(double x)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// fast fp64 square root: MUFU reciprocal-sqrt approximation + Newton steps (<= 1 ulp off IEEE)
__device__ __forceinline__ double sqrt64(double x)
{
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * fma(-0.5 * x * r, r, 1.5);
    r = r * fma(-0.5 * x * r, r, 1.5);
    double s = x * r;
    return fma(0.5 * r, fma(-s, s, x), s);
}

}  // namespace perk
