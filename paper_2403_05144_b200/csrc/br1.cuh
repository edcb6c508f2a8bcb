// br1.cuh -- Navier-Stokes BR1 passes of one P-ERK stage (D7).
//
// The paper cites BR1 (P:l.1419-1420) without defining it.  Per stage, before the inviscid+viscous
// surface kernel (k_surf2d<.., NS>) and the volume kernel (k_vol2d<.., NS>):
//   k_gsurf2d : central traces w* = (w_L + w_R)/2 of the gradient variables w = (v1, v2, T) on the
//               interfaces and mortars of the EXTENDED prefix (active members + the next coarser
//               member: the coarse neighbours across active mortars need gradients too); mortars:
//               halves (P w_large + w_small)/2, the large side gets R_lower w*_lo + R_upper w*_hi.
//   k_grad2d  : on the elements of the extended prefix, q = grad w (weak form with w*), then the
//               normal viscous flux F^v_n(u, q) at the 12 face nodes -> Vt, read by k_surf2d.
// The volume kernel recomputes q from the state and w* (cheaper than storing 16 x 6 gradients).
#pragma once
#include "dg2d.cuh"

namespace perk {

template <int MODE>
__global__ void __launch_bounds__(256, 3) k_gsurf2d(MeshDev md, StageParams sp, const double *__restrict__ Un,
                                                const double *__restrict__ Ubuf, const double *__restrict__ K1,
                                                const double *__restrict__ Uin, double *__restrict__ Gs)
{
    pdl_wait();
    int nif, nmo;
    if (MODE == MODE_STAGE) {
        nif = md.count_active[EXT_OFF + KIND_IF * MAXS + sp.stage - 1];
        nmo = md.count_active[EXT_OFF + KIND_MO * MAXS + sp.stage - 1];
    } else {
        nif = md.n[1]; nmo = md.n[2];
    }
    const int total = 4 * (nif + nmo);
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const double dtc = sp.dt * sp.c_stage;
    const double gm1 = md.gamma - 1.0;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = 0xFu << (lane & ~3);
    for (int gt = blockIdx.x * blockDim.x + threadIdx.x; gt < total; gt += gridDim.x * blockDim.x) {
        const int item = gt >> 2, k = gt & 3;
        if (item < nif) {
            const int f = MODE == MODE_STAGE ? md.list[KIND_IF][item] : item;
            const int4 I = md.ifc[f];
            const int o = I.z;
            const int src = state_src(sp, I.w);
            double uL[4], uR[4], wL[GV], wR[GV];
            trace2d(sb, src, dtc, I.x, 2 * o, k, uL);
            trace2d(sb, src, dtc, I.y, 2 * o + 1, k, uR);
            prim_vT(uL, gm1, wL);
            prim_vT(uR, gm1, wR);
#pragma unroll
            for (int c = 0; c < GV; ++c) {
                const double w = 0.5 * (wL[c] + wR[c]);
                Gs[gidx2d(I.x, 2 * o, c, k)] = w;
                Gs[gidx2d(I.y, 2 * o + 1, c, k)] = w;
            }
        } else {
            const int q = item - nif;
            const int mo = MODE == MODE_STAGE ? md.list[KIND_MO][q] : q;
            const int4 M = md.mor[mo];
            const int o = M.w & 1, side = (M.w >> 1) & 1, mfine = M.w >> 8;
            const int lf = 2 * o + side, sf = 2 * o + 1 - side;
            double ul[4], us0[4], us1[4], wl[GV], ws0[GV], ws1[GV];
            trace2d(sb, state_src(sp, md.mem[M.x]), dtc, M.x, lf, k, ul);
            const int srcS = state_src(sp, mfine);
            trace2d(sb, srcS, dtc, M.y, sf, k, us0);
            trace2d(sb, srcS, dtc, M.z, sf, k, us1);
            prim_vT(ul, gm1, wl);
            prim_vT(us0, gm1, ws0);
            prim_vT(us1, gm1, ws1);
            double clo[GV], chi[GV];
#pragma unroll
            for (int c = 0; c < GV; ++c) {
                double il = 0.0, ih = 0.0;
#pragma unroll
                for (int j = 0; j < NP; ++j) {
                    const double wj = __shfl_sync(gmask, wl[c], j, 4);
                    il = fma(cB.Plo[k][j], wj, il);
                    ih = fma(cB.Pup[k][j], wj, ih);
                }
                clo[c] = 0.5 * (il + ws0[c]);
                chi[c] = 0.5 * (ih + ws1[c]);
                Gs[gidx2d(M.y, sf, c, k)] = clo[c];
                Gs[gidx2d(M.z, sf, c, k)] = chi[c];
            }
#pragma unroll
            for (int c = 0; c < GV; ++c) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < NP; ++j) {
                    s = fma(cB.Rlo[k][j], __shfl_sync(gmask, clo[c], j, 4), s);
                    s = fma(cB.Rup[k][j], __shfl_sync(gmask, chi[c], j, 4), s);
                }
                Gs[gidx2d(M.x, lf, c, k)] = s;
            }
        }
    }
}

// 8 threads per element as in k_vol2d: gradients along the x-lines and y-lines, exchanged through
// shared memory, then the normal viscous flux at the two end nodes of every line = the face nodes.
constexpr int GRAD2D_LS = VOL2D_LS;

template <int MODE>
__global__ void __launch_bounds__(128) k_grad2d(MeshDev md, StageParams sp, const double *__restrict__ Un,
                                                const double *__restrict__ Ubuf, const double *__restrict__ K1,
                                                const double *__restrict__ Uin, const double *__restrict__ Gs,
                                                double *__restrict__ Vt)
{
    // field slots follow k_vol2d's numbering (F_V1, F_V2, F_T; gradients in 4..6)
    __shared__ double sm[8][2][GRAD2D_LS];
    pdl_wait();
    const int t8 = threadIdx.x & 7, le = threadIdx.x >> 3;
    const int n_act = MODE == MODE_STAGE ? md.count_active[EXT_OFF + KIND_EL * MAXS + sp.stage - 1] : md.n[0];
    const double gm1 = md.gamma - 1.0;
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const double dtc = sp.dt * sp.c_stage;
    const int q0 = 2 * t8;
    const int o = t8 >> 2, ln = t8 & 3;
    const int eo = le * 17, yo = 2;
    for (int base = blockIdx.x * VOL2D_EPB; base < n_act; base += gridDim.x * VOL2D_EPB) {
        const int t = base + le;
        const bool valid = t < n_act;
        const int tt = valid ? t : base;
        const int e = MODE == MODE_STAGE ? md.list[KIND_EL][tt] : tt;
        const int src = state_src(sp, md.mem[e]);
        const size_t eb = (size_t)e * 64;
        const double hcell = md.hf * (double)(1 << (md.max_level - md.lev[e]));
        {
            double2 u[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) u[v] = load_state2(sb, src, dtc, eb + v * 16 + q0);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int q = q0 + h, i = q & 3, j = q >> 2;
                const double uu[4] = {h ? u[0].y : u[0].x, h ? u[1].y : u[1].x, h ? u[2].y : u[2].x, h ? u[3].y : u[3].x};
                double w[GV];
                prim_vT(uu, gm1, w);
                const int fld[GV] = {F_V1, F_V2, F_T};
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    sm[fld[c]][0][eo + 4 * j + i] = w[c];
                    sm[fld[c]][1][yo + eo + 4 * i + j] = w[c];
                }
            }
        }
        __syncwarp();
        const int lo = o == 0 ? eo + 4 * ln : yo + eo + 4 * ln;
        double q[GV][NP];
        const int fld[GV] = {F_V1, F_V2, F_T};
        const double sc[GV] = {1.0, 1.0, 1.0};
        line_gradient<GRAD2D_LS>(sm, o, lo, e, ln, Gs, 2.0 / hcell, fld, sc, q);
#pragma unroll
        for (int c = 0; c < GV; ++c)
#pragma unroll
            for (int a = 0; a < NP; ++a) sm[4 + c][o][lo + a] = q[c][a];
        __syncwarp();
        if (valid) {
#pragma unroll
            for (int end = 0; end < 2; ++end) {
                const int a = end ? NP - 1 : 0;
                const int oi = o == 0 ? yo + eo + 4 * a + ln : eo + 4 * a + ln;
                double qo[GV], qs[GV], fv[GV];
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    qs[c] = q[c][a];
                    qo[c] = sm[4 + c][1 - o][oi];
                }
                const double v1 = sm[F_V1][o][lo + a], v2 = sm[F_V2][o][lo + a];
                if (o == 0) visc_flux2d(v1, v2, qs, qo, 0, md.mu, md.kappa, fv);
                else visc_flux2d(v1, v2, qo, qs, 1, md.mu, md.kappa, fv);
                const int face = 2 * o + (end ? 0 : 1);      // a = N: +o face, a = 0: -o face
#pragma unroll
                for (int c = 0; c < GV; ++c) Vt[gidx2d(e, face, c, ln)] = fv[c];
            }
        }
        __syncwarp();
    }
}

}  // namespace perk
