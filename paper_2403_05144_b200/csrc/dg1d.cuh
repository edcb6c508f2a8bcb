// dg1d.cuh -- 1D DGSEM (N = 3) weak-form kernels of one P-ERK stage (BASELINE cfg 1-2).
//
// k_surf1d : one thread per active interface / boundary: upwind (linear advection) or Rusanov
//            (Euler) flux of the two stage-i traces, written to both elements' face slots.
//            A level-jump interface belongs to the fine side's member; its coarse side may be
//            inactive, so each side's trace follows its own member's state rule.
// k_vol1d  : one thread per active element: du_i = (2/h)[sum_j Dhat_ij f(u_j) + (d_i0 f*_L - d_iN f*_R)/w_i]
//             fused with the stage epilogue (as k_vol2d).
// Fs layout in 1D: [cell][face 0 = +x, 1 = -x][var].
#pragma once
#include "common.cuh"

namespace perk {

template <int NV>
__device__ __forceinline__ void phys_flux1d(const double u[NV], double g, double a, double f[NV])
{
    if (NV == 1) {
        f[0] = a * u[0];
    } else {
        const double v = u[1] / u[0];
        const double p = (g - 1.0) * (u[2] - 0.5 * u[1] * v);
        f[0] = u[1];
        f[1] = u[1] * v + p;
        f[2] = (u[2] + p) * v;
    }
}

template <int NV>
__device__ __forceinline__ void numflux1d(const double uL[NV], const double uR[NV], double g, double a, double f[NV])
{
    if (NV == 1) {   // upwind
        f[0] = a >= 0.0 ? a * uL[0] : a * uR[0];
        return;
    }
    double fL[NV], fR[NV];
    phys_flux1d<NV>(uL, g, a, fL);
    phys_flux1d<NV>(uR, g, a, fR);
    const double vL = uL[1] / uL[0], vR = uR[1] / uR[0];
    const double pL = (g - 1.0) * (uL[2] - 0.5 * uL[1] * vL), pR = (g - 1.0) * (uR[2] - 0.5 * uR[1] * vR);
    const double lam = fmax(fabs(vL) + sqrt(g * pL / uL[0]), fabs(vR) + sqrt(g * pR / uR[0]));
#pragma unroll
    for (int v = 0; v < NV; ++v) f[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * lam * (uR[v] - uL[v]);
}

template <int NV, int MODE>
__global__ void __launch_bounds__(256) k_surf1d(MeshDev md, StageParams sp, const double *__restrict__ Un,
                                               const double *__restrict__ Ubuf, const double *__restrict__ K1,
                                               const double *__restrict__ Uin, double *__restrict__ Fs)
{
    int nif, nbd;
    if (MODE == MODE_STAGE) {
        nif = md.count_active[KIND_IF * MAXS + sp.stage - 1];
        nbd = md.count_active[KIND_BD * MAXS + sp.stage - 1];
    } else {
        nif = md.n[1]; nbd = md.n[3];
    }
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const double dtc = sp.dt * sp.c_stage;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < nif + nbd; it += gridDim.x * blockDim.x) {
        double uL[NV], uR[NV], f[NV];
        if (it < nif) {
            const int fi = MODE == MODE_STAGE ? md.list[KIND_IF][it] : it;
            const int4 I = md.ifc[fi];
            PERK_DASSERT(I.x >= 0 && I.x < md.n[0] && I.y >= 0 && I.y < md.n[0]);
            const int sL = state_src(sp, md.mem[I.x]), sR = state_src(sp, md.mem[I.y]);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                uL[v] = load_state(sb, sL, dtc, ((size_t)I.x * NV + v) * NP + (NP - 1));
                uR[v] = load_state(sb, sR, dtc, ((size_t)I.y * NV + v) * NP);
            }
            numflux1d<NV>(uL, uR, md.gamma, md.adv, f);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                Fs[((size_t)I.x * 2 + 0) * NV + v] = f[v];
                Fs[((size_t)I.y * 2 + 1) * NV + v] = f[v];
            }
        } else {
            const int q = it - nif;
            const int bi = MODE == MODE_STAGE ? md.list[KIND_BD][q] : q;
            const int2 B = md.bnd[bi];
            PERK_DASSERT(B.x >= 0 && B.x < md.n[0]);
            const int face = B.y & 7;
            const int s = state_src(sp, B.y >> 8);
            double u[NV], gst[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                u[v] = load_state(sb, s, dtc, ((size_t)B.x * NV + v) * NP + (face == 0 ? NP - 1 : 0));
                gst[v] = md.bc[v];
            }
            if (face == 0) numflux1d<NV>(u, gst, md.gamma, md.adv, f);
            else numflux1d<NV>(gst, u, md.gamma, md.adv, f);
#pragma unroll
            for (int v = 0; v < NV; ++v) Fs[((size_t)B.x * 2 + face) * NV + v] = f[v];
        }
    }
}

template <int NV, int MODE>
__global__ void __launch_bounds__(128) k_vol1d(MeshDev md, StageParams sp, double *__restrict__ Un,
                                              double *__restrict__ Ubuf, double *__restrict__ K1,
                                              const double *__restrict__ Fs, const double *__restrict__ Uin,
                                              double *__restrict__ dU, double *__restrict__ Wb)
{
    const int n_act = MODE == MODE_STAGE ? md.count_active[KIND_EL * MAXS + sp.stage - 1] : md.n[0];
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const double dtc = sp.dt * sp.c_stage;
    if (MODE == MODE_STAGE && sp.stage == sp.S && blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(md.evals, md.evals[2]);           // sum_r E_r N_C(r), set by the mesh pipeline
        atomicAdd(md.evals + 1, 1ull);
    }
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_act; t += gridDim.x * blockDim.x) {
        const int e = MODE == MODE_STAGE ? md.list[KIND_EL][t] : t;
        const int m = md.mem[e];
        if (MODE == MODE_STAGE && !((sp.actmask >> m) & 1u)) continue;   // surplus member of the prefix
        const int src = state_src(sp, m);
        const size_t eb = (size_t)e * NV * NP;
        double u[NP][NV], f[NP][NV];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
#pragma unroll
            for (int v = 0; v < NV; ++v) u[j][v] = load_state(sb, src, dtc, eb + v * NP + j);
            phys_flux1d<NV>(u[j], md.gamma, md.adv, f[j]);
        }
        const double J = 2.0 / (md.hf * (double)(1 << (md.max_level - md.lev[e])));
        double fR[NV], fLf[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            fR[v] = Fs[((size_t)e * 2 + 0) * NV + v];
            fLf[v] = Fs[((size_t)e * 2 + 1) * NV + v];
        }
#pragma unroll
        for (int i = 0; i < NP; ++i) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < NP; ++j) s = fma(cB.Dhat[i][j], f[j][v], s);
                if (i == 0) s = fma(fLf[v], cB.invw[0], s);
                if (i == NP - 1) s = fma(-fR[v], cB.invw[NP - 1], s);
                const double K = J * s;
                const size_t idx = eb + v * NP + i;
                if (MODE == MODE_RHS) {
                    dU[idx] = ((sp.mask >> m) & 1u) ? K : 0.0;
                } else if (sp.stage == 1) {
                    K1[idx] = K;
                } else if (sp.stage == sp.S) {
                    if (sp.fin_k1) Un[idx] = fma(sp.dt, fma(sp.wb1, K1[idx], sp.bS * K), Un[idx]);
                    else Un[idx] = fma(sp.dt * sp.bS, K, Wb ? Wb[idx] : Un[idx]);
                } else {
                    const double un = Un[idx], k1 = K1[idx];
                    Ubuf[idx] = fma(sp.dt, fma(sp.a1_next[m], k1, sp.asub_next[m] * K), un);
                    if (sp.wmode) Wb[idx] = fma(sp.dt, fma(sp.wb1, k1, sp.wbS1 * K), un);
                }
            }
        }
    }
}

}  // namespace perk
