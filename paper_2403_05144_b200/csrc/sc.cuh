// sc.cuh -- subcell shock capturing (A7-A9), 2D Euler / Navier-Stokes.
//
// The paper runs its inviscid applications with the Hennemann-Gassner shock capturing (P:l.964,
// l.1729, l.1795-1799): per element the flux-differencing volume integral V_DG is blended with the
// first-order subcell finite-volume one, V = (1 - alpha) V_DG + alpha V_FV.  The blend itself lives
// in k_vol2d<., ., true> (per node line, from the primitives it already holds in shared memory);
// this file computes alpha per stage, before the stage's surface and volume launches:
//
//   k_sc_alpha  : Hennemann-Gassner indicator (amr.cuh, the same modal energy and logistic as the
//                 AMR indicator) on the elements the stage needs -- the active elements and their
//                 neighbours across active mortars (the BR1 halo lists, mesh.cuh) -- from the
//                 element's stage state (U_n, the stage buffer, or U_n + dt c_i K_1 formed on the
//                 fly); writes alpha_raw and alpha
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

struct ScParams {
    int variable, smooth;
    double alpha_max, alpha_min, alpha_fixed;   // alpha_fixed >= 0: no indicator
    double hg_T, hg_sT;                         // threshold T and s / T (host-computed, as AmrParams)
};

template <int MODE>
__global__ void __launch_bounds__(AMR_T) k_sc_alpha(MeshDev md, StageParams sp, ScParams scp,
                                                    const double *__restrict__ Un, const double *__restrict__ Ubuf,
                                                    const double *__restrict__ K1, const double *__restrict__ Uin,
                                                    double *__restrict__ alpha_raw, double *__restrict__ alpha)
{
    const int q = threadIdx.x & 15, g = threadIdx.x >> 4;
    const unsigned gm = 0xffffffffu;   // converged full-mask shuffles (width 16), as in k_amr_indicator
    double Ri[NP], Rj[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        Ri[k] = cB.Vinv[q & 3][k];
        Rj[k] = cB.Vinv[q >> 2][k];
    }
    AmrParams ap;
    ap.indicator = IND_HG;
    ap.variable = scp.variable;
    ap.base_level = ap.med_level = ap.max_level = 0;
    ap.med_thr = ap.max_thr = 0.0;
    ap.alpha_max = scp.alpha_max;
    ap.alpha_min = scp.alpha_min;
    ap.hg_T = scp.hg_T;
    ap.hg_sT = scp.hg_sT;
    ap.f_wave = 0.0;
    pdl_wait();
    // items: [active elements | halo elements of the member below the lowest active one]
    const int n_el_a = MODE == MODE_STAGE ? md.count_active[KIND_EL * MAXS + sp.stage - 1] : md.n[0];
    const int2 hel = MODE == MODE_STAGE ? md.hrng[KIND_EL * MAXS + sp.stage - 1] : make_int2(0, 0);
    const int n_items = n_el_a + hel.y;
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const double dtc = sp.dt * sp.c_stage;
    const int per = AMR_T / 16;
    for (int base = blockIdx.x * per; base < n_items; base += gridDim.x * per) {   // CTA-uniform trip count
        const int t = base + g;
        const int tt = t < n_items ? t : base;
        int e, src;
        if (MODE == MODE_STAGE) {
            const int pk = tt < n_el_a ? md.elpk[tt] : md.hpk[hel.x + tt - n_el_a];
            e = pk_elem(pk);
            src = state_src(sp, pk_member(pk));
        } else {
            e = tt;
            src = SRC_IN;
        }
        PERK_DASSERT(e >= 0 && e < md.n[0]);
        double a;
        if (scp.alpha_fixed >= 0.0) {
            a = scp.alpha_fixed;
        } else {
            const size_t b = (size_t)e * 64 + q;
            const double u0 = load_state(sb, src, dtc, b), u1 = load_state(sb, src, dtc, b + 16);
            const double u2 = load_state(sb, src, dtc, b + 32), u3 = load_state(sb, src, dtc, b + 48);
            a = amr_element_indicator<IND_HG>(md, ap, 0, u0, u1, u2, u3, Ri, Rj, gm, q);
        }
        if (q == 0 && t < n_items) {
            alpha_raw[e] = a;
            alpha[e] = a;
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
