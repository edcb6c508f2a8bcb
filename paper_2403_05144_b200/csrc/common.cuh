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

// Device-side bounds checks of the gather indices (build with -DPERK_DEBUG; compute-sanitizer is not
// available on this GPU pool): a violated check prints its location and traps the kernel.
#ifdef PERK_DEBUG
#include <cstdio>
#define PERK_DASSERT(c)                                                                   \
    do {                                                                                  \
        if (!(c)) {                                                                       \
            printf("PERK_DASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);           \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define PERK_DASSERT(c) \
    do {                \
    } while (0)
#endif

namespace perk {

// Race exposure (debug builds only; compute-sanitizer's racecheck is closed on this GPU pool): with
// perk_debug_jitter(seed != 0) every thread sleeps a pseudo-random 0..4 us at the marked points of
// the staged kernels (before each warp barrier / wait and before reading staged data), so threads of
// a warp drift apart.  A missing __syncwarp / cp.async wait then reads stale shared memory and the
// result differs from the unjittered run (tests/test_gpu_races.py compares them bitwise).
#ifdef PERK_DEBUG
__device__ unsigned g_jitter_seed;
__device__ __forceinline__ void perk_jitter(unsigned site)
{
    const unsigned s = g_jitter_seed;
    if (!s) return;
    unsigned h = s ^ (blockIdx.x * 0x9E3779B9u) ^ (threadIdx.x * 0x85EBCA6Bu) ^ (site * 0xC2B2AE35u) ^
                 (unsigned)clock();
    h ^= h >> 16;
    h *= 0x7FEB352Du;
    h ^= h >> 15;
    __nanosleep(h & 4095u);
}
#define PERK_JITTER(site) perk_jitter(site)
#else
#define PERK_JITTER(site) \
    do {                  \
    } while (0)
#endif

constexpr int NP = 4;          // N + 1 LGL nodes per direction (N = 3)
constexpr int MAXV = 4;
constexpr int MAXS = 64;
constexpr int MAXR = 8;
constexpr int SM_COUNT_B200 = 148;

enum Kind { KIND_EL = 0, KIND_IF = 1, KIND_MO = 2, KIND_BD = 3 };
enum Mode { MODE_STAGE = 0, MODE_RHS = 1 };
enum ErrBits { ERR_UNBALANCED = 1, ERR_CAPACITY = 2, ERR_TRANSFER = 4 };

// DGSEM N=3 tables, generated on the host by basis.cuh and uploaded once per process.
struct BasisTables {
    double xi[NP], w[NP], invw[NP];
    double Dhat[NP][NP];    // weak form
    double Dsplit[NP][NP];  // flux differencing (2D - boundary corrections)
    double Plo[NP][NP], Pup[NP][NP];
    double Rlo[NP][NP], Rup[NP][NP];
    double D[NP][NP];       // D_ij = l_j'(xi_i) (AMR enstrophy indicator)
    double Vinv[NP][NP];    // nodal -> orthonormal-Legendre modal coefficients (AMR Hennemann-Gassner)
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
    int *count_active;           // [4][MAXS] stage prefix counts
    int *seg;                    // [4][MAXR+1]
    int *err;                    // error flag bits
    unsigned long long *evals;   // [3]: element-RHS evaluations, steps, evaluations per step
    int *list[4];                // per-kind member-sorted item lists
    int *fx, *fy;                // leaf origin (finest grid)
    uint8_t *lev, *mem;          // leaf level, member
    int *cell_of;                // finest cell -> leaf
    int4 *ifc; int4 *mor; int2 *bnd;
    // hot-path copies in list (member-sorted) order, so a stage kernel reaches its item with one load:
    int *elpk;                   // elements: e | member << 24 | level << 27 (PK_* below)
    int4 *ifcs; int4 *mors;      // interface / mortar records in list order
    // BR1 halo (Navier-Stokes): the gradients of an active element's neighbours across mortars are
    // needed; those neighbours are the LARGE sides of mortars of the finer member.  halo[e] = 1 for
    // such elements; per member, halo element / interface / mortar lists (faces of halo elements
    // that belong to the halo's own member); hrng[kind][stage] = {start, count} of the halo lists
    // a stage needs (the halo of the lowest active member; empty at stage 1).
    uint8_t *halo;
    int *hlist[3];               // elements, interfaces, mortars (member-sorted, descending)
    int *hseg;                   // [3][MAXR + 1]
    int2 *hrng;                  // [3][MAXS]
    int *hpk;                    // packed entries of hlist[KIND_EL]
    // per element and face (+x, -x, +y, -y), the face neighbours (Navier-Stokes, the fused BR1 gradient
    // kernel; rebuilt with the face records): {x, y} with x, y packed (cell | member << 24):
    // conforming {nb, FNB_CONF}; small side of a mortar {large, FNB_SMALL_LO / FNB_SMALL_HI};
    // large side {small_lo, small_hi}; no neighbour (boundary) {-1, FNB_NONE}
    int2 *fnb;
};
constexpr int FNB_CONF = -1, FNB_SMALL_LO = -2, FNB_SMALL_HI = -3, FNB_NONE = -4;

// 2/h of a cell at level lev without a division per element: 2 / (hf 2^(L - lev)) = (2 / hf) 2^(lev - L),
// and the power-of-two scaling is exact, so this is bitwise 2.0 / (hf * (1 << (L - lev))) (two_over_hf =
// 2.0 / md.hf, formed once per thread)
__device__ __forceinline__ double two_over_h(double two_over_hf, int lev, int max_level)
{
    return two_over_hf * __hiloint2double((1023 + lev - max_level) << 20, 0);
}

// packed element entry of md.elpk (cells < 2^24, members < 8, levels < 16)
constexpr int PK_EBITS = 24;
__device__ __forceinline__ int pk_elem(int pk) { return pk & ((1 << PK_EBITS) - 1); }
__device__ __forceinline__ int pk_member(int pk) { return (pk >> PK_EBITS) & 7; }
__device__ __forceinline__ int pk_level(int pk) { return (pk >> (PK_EBITS + 3)) & 15; }

// Per-launch stage parameters (kernel argument, graph-captured).
struct StageParams {
    int stage;                   // 1..S
    int S;
    int R;
    int mode;                    // MODE_STAGE / MODE_RHS
    unsigned mask;               // rhs_eval partition mask
    double dt;
    double c_stage;              // c_i (lazy state U_n + dt c_i K_1)
    unsigned actmask;            // members evaluating this stage (the launch covers a superset prefix)
    unsigned bufmask;            // members whose stage state is in Ubuf (evaluated, with an earlier
                                 // evaluated stage > 1); the others form U_n + dt c_i K_1 on the fly
    double a1_next[MAXR];        // a_{n,1}^{(r)}, n = the member's next evaluated stage after this one
    double asub_next[MAXR];      // a_{n,i}^{(r)} (standard pattern: n = i + 1)
    double bS;                   // b_S: U_{n+1} = W + dt b_S K_S (W = U_n when b = e_S)
    double wb1, wbS1;            // b_1, b_{S-1}: W = U_n + dt (b_1 K_1 + b_{S-1} K_{S-1}) ...
    int wmode;                   // ... written by the stage S-1 epilogue when wmode = 1 (P-ERK3)
    int fin_k1;                  // stage S with b_1 != 0 and b_{S-1} = 0 (Heun / Ralston weights, P:l.439-442):
                                 // U_{n+1} = U_n + dt (b_1 K_1 + b_S K_S), no W buffer
    int rev;                     // 1: this launch walks its lists from the end (the stage kernels of a step
                                 // alternate direction, so a launch starts on the data its predecessor
                                 // touched last, which is what the L2 still holds; results do not depend on it)
};
// list position of the t-th item of a launch over n items
__device__ __forceinline__ int sweep_idx(const StageParams &sp, int t, int n) { return sp.rev ? n - 1 - t : t; }

// Subcell shock capturing parameters (sc.cuh, k_vol2d<., ., true>)
struct ScParams {
    int variable, smooth;
    double alpha_max, alpha_min, alpha_fixed;   // alpha_fixed >= 0: no indicator
    double hg_T, hg_sT;                         // threshold T and s / T (host-computed, as AmrParams)
    int epi;                                    // k_vol2d computes the next stage's alpha of the elements
                                                // whose next stage state its epilogue writes (stages 2..S-1)
    int all;                                    // non-standard stage patterns: alpha of every element at
                                                // every stage (no nested halo lists exist for them)
};

// Which buffer holds element e's stage-i state (SURVEY §7 rule):
//   i == 1: U_n;  i evaluated after an earlier evaluated stage > 1 (standard: i > f(e) = S - E + 2):
//   Ubuf;  otherwise U_n + dt c_i K_1 (formed on the fly)
enum StateSrc { SRC_UN = 0, SRC_BUF = 1, SRC_LAZY = 2, SRC_IN = 3 };

__device__ __forceinline__ int state_src(const StageParams &sp, int member)
{
    if (sp.mode == MODE_RHS) return SRC_IN;
    if (sp.stage == 1) return SRC_UN;
    return ((sp.bufmask >> member) & 1u) ? SRC_BUF : SRC_LAZY;
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
    double e = fma(-x, y, 1.0);      // |e| <~ 2^-22 from the MUFU seed; two Newton steps reach 2^-88
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// natural logarithm of a positive, finite, normal double without branches (the libm log has
// special-case control flow that serialises the hot loop): x = 2^k m, m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh(t) = 2 t (1 + t^2/3 + ... + t^20/21), t = (m-1)/(m+1), |t| <= 0.1716 (truncation
// < 1e-17 relative); <= 3 ulp against the correctly rounded result in a 40k-sample host check.
__device__ __forceinline__ double log_pos(double x)
{
    const long long ix = __double_as_longlong(x);
    const long long k = (ix - 0x3FE6A09E667F3BCDll) >> 52;          // sqrt(1/2) = 0x3FE6A09E667F3BCD
    const double m = __longlong_as_double(ix - (k << 52));
    const double f = m - 1.0;
    const double t = f * rcp64(2.0 + f);
    const double t2 = t * t;
    double q = 1.0 / 21.0;
    q = fma(q, t2, 1.0 / 19.0);
    q = fma(q, t2, 1.0 / 17.0);
    q = fma(q, t2, 1.0 / 15.0);
    q = fma(q, t2, 1.0 / 13.0);
    q = fma(q, t2, 1.0 / 11.0);
    q = fma(q, t2, 1.0 / 9.0);
    q = fma(q, t2, 1.0 / 7.0);
    q = fma(q, t2, 1.0 / 5.0);
    q = fma(q, t2, 1.0 / 3.0);
    q = fma(q, t2, 1.0);
    const double kd = (double)k;
    return fma(kd, 6.93147180369123816490e-01, fma(2.0 * t, q, kd * 1.90821492927058770002e-10));
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

// ---------------------------------------------------------------------------------------------
// Blackwell bulk-copy (TMA engine, SASS UBLKCP) + mbarrier helpers: a 512 B element block is one
// cp.async.bulk global -> shared copy whose completion is counted in bytes on an mbarrier.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order this thread's earlier generic-proxy shared-memory accesses before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Programmatic dependent launch (sm_90+): the stage kernels are launched with programmatic stream
// serialisation and wait for their predecessor's completion and memory (griddepcontrol.wait) only
// before touching stage data, so the successor's launch and index prologue overlap the
// predecessor's tail (cfg 3: 0.587 -> 0.570 ms/step).  No explicit launch_dependents trigger: the
// implicit trigger at CTA exit measured faster than triggering at kernel start (0.615 ms/step), where
// early-resident waiting CTAs of the successor crowd the predecessor's last waves.  No-op without
// the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// a load the compiler cannot merge with an earlier one (re-reading a value instead of keeping it live)
__device__ __forceinline__ int ld_volatile(const int *p) { return *reinterpret_cast<const volatile int *>(p); }

// L1 prefetch of the line holding p (no register, no scoreboard entry)
__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Ampere-style asynchronous copies (SASS LDGSTS): no registers, per-thread commit groups
__device__ __forceinline__ void cp_async16(void *dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// L2 eviction hints for data that is dead once this launch has read it (face fluxes, the viscous volume
// term, the viscous-flux traces; U_n and K_1, whose next reader is several launches away): with the
// alternating sweep (StageParams::rev) what the next launch finds in the L2 is what its predecessor left
// there, so dead lines are offered for eviction first.  L2_HINTS = 0: plain loads; 1: Fs and Dv; 2: also U_n and
// K_1 (cfg 3, whose working set is about the size of the L2: 0.5407 / 0.5386 / 0.5243 ms per step; cfg 5:
// 5.873 / 5.861 / 5.859; profiles/r02_ab_l2_hints2.json).
#ifndef L2_HINTS
#define L2_HINTS 2
#endif
__device__ __forceinline__ unsigned long long l2_evict_first_policy()
{
    unsigned long long p = 0;
#if L2_HINTS
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}
__device__ __forceinline__ void cp_async16_dead(void *dst, const void *src, unsigned long long pol)
{
#if L2_HINTS
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "l"(pol) : "memory");
#else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
#endif
}
__device__ __forceinline__ double2 ldg2_dead(const double2 *p, unsigned long long pol)
{
#if L2_HINTS
    double2 r;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ double ldg_dead(const double *p, unsigned long long pol)
{
#if L2_HINTS
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace perk
