// sc.cuh -- subcell shock capturing (A7-A9), 2D Euler / Navier-Stokes.
//
// The paper runs its inviscid applications with the Hennemann-Gassner shock capturing (P:l.964,
// l.1729, l.1795-1799): per element the flux-differencing volume integral V_DG is blended with the
// first-order subcell finite-volume one, V = (1 - alpha) V_DG + alpha V_FV.  The blend itself lives
// in k_vol2d<., ., true> (per node line, from the primitives it already holds in shared memory);
// this file computes alpha per stage, before the stage's surface and volume launches:
//
//   k_sc_alpha  : Hennemann-Gassner indicator (the modal energy and logistic of the AMR indicator,
//                 amr.cuh / DESIGN.md A1) on the elements the stage needs -- the active elements and their
//                 neighbours across active mortars (the BR1 halo lists, mesh.cuh) -- from the
//                 element's stage state (U_n, the stage buffer, or U_n + dt c_i K_1 formed on the
//                 fly); writes alpha_raw and alpha.  With ScParams::epi (Euler default) the elements
//                 whose state the previous stage's k_vol2d wrote to the stage buffer already have
//                 theirs (computed in that epilogue) and are skipped
//   smoothing   : alpha_e = max(alpha_e, alpha_raw_n / 2) over the stage's active interfaces and
//                 mortars (atomicMax on the fp64 bit pattern, exact for alpha >= 0, so the result does
//                 not depend on the order); every face of an active element is active, so every
//                 active element sees all its neighbours.  Done by lane 0 of each face inside
//                 k_surf2d<., ., true> (no extra launch); k_sc_smooth is the stand-alone version
//                 (PERK_SC_FUSED=0, used by the tests to cross-check the fused one bitwise)
#pragma once
#include "common.cuh"
#include "amr.cuh"

namespace perk {


// One 16-lane group per element (lane q = node q) forms the indicator variable and its orthonormal
// Legendre modal coefficients with width-16 shuffles (as k_amr_indicator), reduces the three energy
// sums, and leaves them in a per-warp shared-memory buffer; every 8 iterations (16 elements) the
// warp runs the scalar tail (two quotients, the logistic's exp, the clipping) once, one lane per
// element, instead of the 16-fold replicated tail of the per-group form (warp-synchronous: a
// per-CTA tail behind __syncthreads made barrier waits the top stall).  The next iteration's state (U_n and K_1 raw for a
// lazy state) is loaded into registers before the current one is processed, so two elements per
// group are in flight (ncu of the unpipelined form: 1.1 TB/s, 47 % issue-active, latency bound);
// the Vandermonde rows come from shared memory to leave the registers to the prefetch.
template <int MODE>
__global__ void __launch_bounds__(AMR_T) k_sc_alpha(MeshDev md, StageParams sp, ScParams scp,
                                                    const double *__restrict__ Un, const double *__restrict__ Ubuf,
                                                    const double *__restrict__ K1, const double *__restrict__ Uin,
                                                    double *__restrict__ alpha_raw, double *__restrict__ alpha)
{
    constexpr int PER = AMR_T / 16;    // elements per CTA and iteration
    constexpr int NW = AMR_T / 32;     // warps per CTA
    __shared__ double sE[NW][3][16];   // per warp: tot, clip1, clip2 of up to 16 buffered elements
    __shared__ int sEl[NW][16];        // element id (-1: no element)
    __shared__ double sV[NP][NP];      // Vinv
    const int q = threadIdx.x & 15, g = threadIdx.x >> 4, wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hg = g & 1;              // group within the warp
    int nb = 0;                        // elements buffered by this warp (warp-uniform)
    const unsigned gm = 0xffffffffu;   // converged full-mask shuffles (width 16), as in k_amr_indicator
    const int i = q & 3, j = q >> 2;
    if (threadIdx.x < NP * NP) sV[threadIdx.x >> 2][threadIdx.x & 3] = cB.Vinv[threadIdx.x >> 2][threadIdx.x & 3];
    __syncthreads();
    pdl_wait();
    // items: [active elements | halo elements of the member below the lowest active one].  With
    // scp.epi the previous stage's k_vol2d epilogue already wrote alpha for the elements whose stage
    // state it wrote to the stage buffer -- the elements active at stage i - 1 >= 2, a prefix of the
    // member-sorted list -- so only the rest (first-time active, lazy states) and the halo remain.
    // Non-standard stage patterns (scp.all): every element, in the member-sorted list (an inactive
    // member's stage state is the lazy U_n + dt c_i K_1, state_src).
    const bool part = MODE == MODE_STAGE && !scp.all;
    const int skip = (part && scp.epi && scp.alpha_fixed < 0.0 && sp.stage >= 3)
                         ? md.count_active[KIND_EL * MAXS + sp.stage - 2] : 0;
    const int n_el_a = (part ? md.count_active[KIND_EL * MAXS + sp.stage - 1] : md.n[0]) - skip;
    const int2 hel = part ? md.hrng[KIND_EL * MAXS + sp.stage - 1] : make_int2(0, 0);
    const int n_items = n_el_a + hel.y;
    const int *elpk = md.elpk + skip;
    const double dtc = sp.dt * sp.c_stage;
    const double gm1 = md.gamma - 1.0;
    if (scp.alpha_fixed >= 0.0) {
        for (int t = blockIdx.x * PER + g; t < n_items; t += gridDim.x * PER) {
            if (q) continue;
            const int e = MODE == MODE_STAGE ? pk_elem(t < n_el_a ? elpk[t] : md.hpk[hel.x + t - n_el_a]) : t;
            alpha_raw[e] = scp.alpha_fixed;
            alpha[e] = scp.alpha_fixed;
        }
        return;
    }
    // element of slot t (clamped into range) and its state source
    auto element_at = [&](int t, int &e, int &src) {
        const int tt = t < n_items ? t : n_items - 1;
        if (MODE == MODE_STAGE) {
            const int pk = tt < n_el_a ? elpk[tt] : md.hpk[hel.x + tt - n_el_a];
            e = pk_elem(pk);
            src = state_src(sp, pk_member(pk));
        } else {
            e = tt;
            src = SRC_IN;
        }
        PERK_DASSERT(e >= 0 && e < md.n[0]);
    };
    // raw loads of one element's node values: a[v] (U_n, stage buffer or U_in), k[v] (K_1, lazy only)
    auto issue = [&](int e, int src, double a[4], double k[4]) {
        const size_t b = (size_t)e * 64 + q;
        const double *base = src == SRC_BUF ? Ubuf : (src == SRC_IN ? Uin : Un);
#pragma unroll
        for (int v = 0; v < 4; ++v) a[v] = __ldg(base + b + 16 * v);
        if (src == SRC_LAZY) {
#pragma unroll
            for (int v = 0; v < 4; ++v) k[v] = __ldg(K1 + b + 16 * v);
        }
    };
    int base = blockIdx.x * PER;
    if (base >= n_items) return;
    int e, src;
    element_at(base + g, e, src);
    double ca[4], ck[4] = {0.0, 0.0, 0.0, 0.0};
    issue(e, src, ca, ck);
    for (; base < n_items; base += gridDim.x * PER) {   // CTA-uniform trip count
        const int t = base + g;
        const bool has_next = base + gridDim.x * PER < n_items;
        int e_n = 0, src_n = SRC_UN;
        double na[4], nk[4] = {0.0, 0.0, 0.0, 0.0};
        if (has_next) {
            element_at(t + gridDim.x * PER, e_n, src_n);
            issue(e_n, src_n, na, nk);
        }
        double u[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) u[v] = src == SRC_LAZY ? fma(dtc, ck[v], ca[v]) : ca[v];
        const double rho = u[0], mx = u[1], my = u[2], En = u[3];
        const double irho = rcp64(rho);
        const double vx = mx * irho, vy = my * irho;
        const double p = gm1 * (En - 0.5 * rho * (vx * vx + vy * vy));
        double val;
        switch (scp.variable) {
        case 0: val = rho; break;
        case 1: val = p; break;
        case 2: val = rho * p; break;
        case 3: val = vx; break;
        default: val = vy; break;
        }
        // m_kl = sum_ij Vinv[k][i] Vinv[l][j] val_ij; lane (k, l) = (i, j) ends with m_kl
        double tq = 0.0;
#pragma unroll
        for (int a = 0; a < NP; ++a) tq = fma(sV[i][a], __shfl_sync(gm, val, j * 4 + a, 16), tq);
        double m = 0.0;
#pragma unroll
        for (int c = 0; c < NP; ++c) m = fma(sV[j][c], __shfl_sync(gm, tq, c * 4 + i, 16), m);
        const double mm = m * m;
        const double tot = sum16(gm, mm);
        const double c1 = sum16(gm, (i <= NP - 2 && j <= NP - 2) ? mm : 0.0);
        const double c2 = sum16(gm, (i <= NP - 3 && j <= NP - 3) ? mm : 0.0);
        if (q == 0) {
            sE[wi][0][nb + hg] = tot;
            sE[wi][1][nb + hg] = c1;
            sE[wi][2][nb + hg] = c2;
            sEl[wi][nb + hg] = t < n_items ? e : -1;
        }
        nb += 2;
        if (nb == 16 || !has_next) {   // warp-uniform
            __syncwarp();
            if (lane < nb) {   // tail: one lane per element
                const int ee = sEl[wi][lane];
                if (ee >= 0) {
                    const double T0 = sE[wi][0][lane], T1 = sE[wi][1][lane], T2 = sE[wi][2][lane];
                    const double e1 = T0 > 0.0 ? (T0 - T1) / T0 : 0.0;
                    const double e2 = T1 > 0.0 ? (T1 - T2) / T1 : 0.0;
                    const double E = fmax(e1, e2);
                    double a = 1.0 / (1.0 + exp(-scp.hg_sT * (E - scp.hg_T)));
                    if (a < scp.alpha_min) a = 0.0;
                    else if (a > 1.0 - scp.alpha_min) a = 1.0;
                    a = fmin(a, scp.alpha_max);
                    alpha_raw[ee] = a;
                    alpha[ee] = a;
                }
            }
            __syncwarp();
            nb = 0;
        }
        e = e_n;
        src = src_n;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            ca[v] = na[v];
            ck[v] = nk[v];
        }
    }
}

__device__ __forceinline__ void atomic_max_nonneg(double *p, double v)
{
    atomicMax(reinterpret_cast<unsigned long long *>(p), (unsigned long long)__double_as_longlong(v));
}

template <int MODE>
__global__ void __launch_bounds__(256) k_sc_smooth(MeshDev md, StageParams sp, const double *__restrict__ alpha_raw,
                                                   double *__restrict__ alpha)
{
    pdl_wait();
    const int n_if = MODE == MODE_STAGE ? md.count_active[KIND_IF * MAXS + sp.stage - 1] : md.n[1];
    const int n_mo = MODE == MODE_STAGE ? md.count_active[KIND_MO * MAXS + sp.stage - 1] : md.n[2];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_if + n_mo; t += gridDim.x * blockDim.x) {
        if (t < n_if) {
            const int4 I = MODE == MODE_STAGE ? md.ifcs[t] : md.ifc[t];
            atomic_max_nonneg(alpha + I.x, 0.5 * __ldg(alpha_raw + I.y));
            atomic_max_nonneg(alpha + I.y, 0.5 * __ldg(alpha_raw + I.x));
        } else {
            const int4 M = MODE == MODE_STAGE ? md.mors[t - n_if] : md.mor[t - n_if];
            const double al = 0.5 * __ldg(alpha_raw + M.x);
            atomic_max_nonneg(alpha + M.x, 0.5 * fmax(__ldg(alpha_raw + M.y), __ldg(alpha_raw + M.z)));
            atomic_max_nonneg(alpha + M.y, al);
            atomic_max_nonneg(alpha + M.z, al);
        }
    }
}

}  // namespace perk
