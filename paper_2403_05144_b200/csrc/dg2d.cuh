// dg2d.cuh -- 2D compressible Euler DGSEM (N = 3) kernels of one P-ERK stage.
//
// k_surf2d : one launch per stage over the active prefixes of the interface, mortar and boundary
//            lists (4 threads per face, one per face node): gathers the two traces of the stage-i
//            state (U_n, the stage buffer, or U_n + dt c_i K_1 formed on the fly), HLL flux,
//            writes the per-element face-flux slots Fs.  Mortars interpolate the large trace to the
//            two halves (P_lower/P_upper) and project the two half fluxes back (exact-L2 R), with
//            the 4-node exchanges done by warp shuffles inside the 4-lane group.
// k_vol2d  : one launch per stage over the active element prefix, 8 threads per element (4 x-lines
//            + 4 y-lines): primitives and logarithms per node once (shared memory), 48 symmetric
//            Ranocha two-point fluxes (6 per line), surface lift (1/w) and Jacobian (-2/h), then the
//            stage epilogue in registers: K_1 (stage 1), the state of the member's next evaluated
//            stage n, U^(n) = U_n + dt (a_{n,1} K_1 + a_{n,i} K_i) (standard pattern: n = i + 1), or
//            U_{n+1} = W + dt b_S K_S (W = U_n, or the P-ERK3 / Heun-Ralston combination).
#pragma once
#include "common.cuh"

namespace perk {

// ---------------------------------------------------------------------------------------------
// fluxes
// ---------------------------------------------------------------------------------------------
struct Prim {
    double rho, v1, v2, p, lrho, beta, lbeta;
};

// logarithmic mean as a quotient N / D (no division here): (b - a) / (ln b - ln a), or near a = b
// the series (a + b) / (2 + u (2/3 + u (2/5 + u 2/7))), u = ((b - a)/(b + a))^2 < 1e-4
// (SURVEY §8(c) D3), multiplied through by (a + b)^6.
__device__ __forceinline__ void ln_mean_nd(double a, double b, double la, double lb, double &N, double &D)
{
    const double s = a + b, d = b - a;
    const double s2 = s * s, d2 = d * d;
    const bool series = d2 < 1e-4 * s2;
    const double s4 = s2 * s2, s6 = s4 * s2;
    const double Ds = fma(2.0, s6, d2 * fma(2.0 / 3.0, s4, d2 * fma(2.0 / 5.0, s2, d2 * (2.0 / 7.0))));
    N = series ? s6 * s : d;
    D = series ? Ds : lb - la;
}

// Ranocha entropy-conserving two-point flux in direction o:
// f_rho = rho_hat vbar_n, f_m = f_rho vbar + pbar n, f_E = f_rho (1/2 vL.vR + 1/((g-1) beta_hat)) + 1/2 (pL vnR + pR vnL)
__device__ __forceinline__ void flux_ranocha(const Prim &L, const Prim &R, int o, double inv_gm1, double f[4])
{
    double Nr, Dr, Nb, Db;
    ln_mean_nd(L.rho, R.rho, L.lrho, R.lrho, Nr, Dr);
    ln_mean_nd(L.beta, R.beta, L.lbeta, R.lbeta, Nb, Db);
    const double q = rcp64(Dr * Nb);
    const double rho_hat = Nr * Nb * q;          // Nr / Dr
    const double inv_beta_hat = Db * Dr * q;     // Db / Nb
    const double v1a = 0.5 * (L.v1 + R.v1), v2a = 0.5 * (L.v2 + R.v2), pa = 0.5 * (L.p + R.p);
    const double vnL = o == 0 ? L.v1 : L.v2, vnR = o == 0 ? R.v1 : R.v2;
    const double frho = rho_hat * 0.5 * (vnL + vnR);
    f[0] = frho;
    f[1] = fma(frho, v1a, o == 0 ? pa : 0.0);
    f[2] = fma(frho, v2a, o == 1 ? pa : 0.0);
    f[3] = fma(frho, fma(0.5, fma(L.v1, R.v1, L.v2 * R.v2), inv_beta_hat * inv_gm1), 0.5 * fma(L.p, vnR, R.p * vnL));
}

// The same flux in line coordinates, as the volume kernel evaluates it: per node the layout of the
// line's direction stores rho, hvn = v_n / 2, hvt = v_t / 2, hp = p / 2 (n = the line direction, t
// the other one), so the flux needs no orientation selects and the averages are single additions:
// f = (rho_hat vbar_n, rho_hat vbar_n^2 + pbar, rho_hat vbar_n vbar_t,
//      rho_hat vbar_n (2 (hvn_L hvn_R + hvt_L hvt_R) + 1/((g-1) beta_hat)) + 2 (hp_L hvn_R + hp_R hvn_L))
struct LinePrim {
    double rho, hvn, hvt, hp, lrho, beta, lbeta;
};

__device__ __forceinline__ void flux_ranocha_line(const LinePrim &L, const LinePrim &R, double inv_gm1, double f[4])
{
    double Nr, Dr, Nb, Db;
    ln_mean_nd(L.rho, R.rho, L.lrho, R.lrho, Nr, Dr);
    ln_mean_nd(L.beta, R.beta, L.lbeta, R.lbeta, Nb, Db);
    const double q = rcp64(Dr * Nb);
    const double rho_hat = Nr * Nb * q;          // Nr / Dr
    const double inv_beta_hat = Db * Dr * q;     // Db / Nb
    const double vna = L.hvn + R.hvn, vta = L.hvt + R.hvt, pa = L.hp + R.hp;
    const double frho = rho_hat * vna;
    f[0] = frho;
    f[1] = fma(frho, vna, pa);
    f[2] = frho * vta;
    f[3] = fma(frho, fma(2.0, fma(L.hvn, R.hvn, L.hvt * R.hvt), inv_beta_hat * inv_gm1),
               2.0 * fma(L.hp, R.hvn, R.hp * L.hvn));
}

__device__ __forceinline__ void euler_flux2d(const double u[4], double p, double vn, int o, double f[4])
{
    f[0] = u[0] * vn;
    f[1] = u[1] * vn + (o == 0 ? p : 0.0);
    f[2] = u[2] * vn + (o == 1 ? p : 0.0);
    f[3] = (u[3] + p) * vn;
}

// HLL with Davis wave-speed estimates; Rusanov as the alternative
__device__ __forceinline__ void numflux2d(const double uL[4], const double uR[4], int o, double g, int surface,
                                          double f[4])
{
    const double gm1 = g - 1.0;
    const double irL = rcp64(uL[0]), irR = rcp64(uR[0]);
    const double v1L = uL[1] * irL, v2L = uL[2] * irL;
    const double v1R = uR[1] * irR, v2R = uR[2] * irR;
    const double pL = gm1 * (uL[3] - 0.5 * (uL[1] * v1L + uL[2] * v2L));
    const double pR = gm1 * (uR[3] - 0.5 * (uR[1] * v1R + uR[2] * v2R));
    const double cL = sqrt64(g * pL * irL), cR = sqrt64(g * pR * irR);
    const double vnL = o == 0 ? v1L : v2L, vnR = o == 0 ? v1R : v2R;
    double fL[4], fR[4];
    euler_flux2d(uL, pL, vnL, o, fL);
    euler_flux2d(uR, pR, vnR, o, fR);
    if (surface == 1) {   // Rusanov
        const double lam = fmax(fabs(vnL) + cL, fabs(vnR) + cR);
#pragma unroll
        for (int v = 0; v < 4; ++v) f[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * lam * (uR[v] - uL[v]);
        return;
    }
    // HLL with Davis wave-speed estimates
    const double sL = fmin(vnL - cL, vnR - cR), sR = fmax(vnL + cL, vnR + cR);
    if (sL >= 0.0) {
#pragma unroll
        for (int v = 0; v < 4; ++v) f[v] = fL[v];
    } else if (sR <= 0.0) {
#pragma unroll
        for (int v = 0; v < 4; ++v) f[v] = fR[v];
    } else {
        const double inv = rcp64(sR - sL);
#pragma unroll
        for (int v = 0; v < 4; ++v) f[v] = (sR * fL[v] - sL * fR[v] + sL * sR * (uR[v] - uL[v])) * inv;
    }
}

// ---------------------------------------------------------------------------------------------
// Navier-Stokes BR1 helpers (D7): gradient variables w = (rho, v1, v2,
// T = p/rho); the gradient, viscous-flux and face arrays hold the 3 components (v1, v2, T) /
// (momentum x, momentum y, energy) -- the density gradient and the viscous mass flux are unused / 0.
// ---------------------------------------------------------------------------------------------
constexpr int GV = 3;

__device__ __forceinline__ void prim_vT(const double u[4], double gm1, double w[GV])
{
    const double ir = rcp64(u[0]);
    const double v1 = u[1] * ir, v2 = u[2] * ir;
    const double p = gm1 * (u[3] - 0.5 * fma(u[1], v1, u[2] * v2));
    w[0] = v1;
    w[1] = v2;
    w[2] = p * ir;
}

// viscous flux in direction o from the velocities and q_x = (v1_x, v2_x, T_x), q_y = (...)_y:
// tau = mu (grad v + grad v^T - 2/3 div v I), heat flux kappa grad T; returns the momentum-x,
// momentum-y and energy components
__device__ __forceinline__ void visc_flux2d(double v1, double v2, const double qx[GV], const double qy[GV], int o,
                                            double mu, double kappa, double f[GV])
{
    const double t11 = mu * ((4.0 / 3.0) * qx[0] - (2.0 / 3.0) * qy[1]);
    const double t22 = mu * ((4.0 / 3.0) * qy[1] - (2.0 / 3.0) * qx[0]);
    const double t12 = mu * (qy[0] + qx[1]);
    if (o == 0) {
        f[0] = t11;
        f[1] = t12;
        f[2] = fma(v1, t11, fma(v2, t12, kappa * qx[2]));
    } else {
        f[0] = t12;
        f[1] = t22;
        f[2] = fma(v1, t12, fma(v2, t22, kappa * qy[2]));
    }
}

// the same flux for a line thread of direction o without a branch on o (the x- and y-line threads of an
// element share a warp, so `if (o == 0)` ran both bodies): qs = the gradient along the line (direction
// o), qo = along the other direction; components swapped into line coordinates (normal, tangential),
// the o = 0 formula, swapped back to (momentum x, momentum y, energy)
__device__ __forceinline__ void visc_flux2d_line(int o, double v1, double v2, const double qs[GV], const double qo[GV],
                                                 double mu, double kappa, double f[GV])
{
    const bool y = o != 0;
    const double vn = y ? v2 : v1, vt = y ? v1 : v2;
    const double sn = y ? qs[1] : qs[0], st = y ? qs[0] : qs[1];   // d v_n / d n, d v_t / d n
    const double on = y ? qo[1] : qo[0], ot = y ? qo[0] : qo[1];   // d v_n / d t, d v_t / d t
    const double tnn = mu * ((4.0 / 3.0) * sn - (2.0 / 3.0) * ot);
    const double tnt = mu * (on + st);
    const double fe = fma(vn, tnn, fma(vt, tnt, kappa * qs[2]));
    f[0] = y ? tnt : tnn;
    f[1] = y ? tnn : tnt;
    f[2] = fe;
}

// BR1 face arrays Gs (central w*), Vt (normal viscous flux trace): [cell][face][GV][k]
__device__ __forceinline__ size_t gidx2d(int e, int face, int c, int k) { return (((size_t)e * 4 + face) * GV + c) * NP + k; }
// Vt with VT_CF = 1: [cell][GV][face][k] -- a component's four face traces share one 128 B line, so a
// warp-wide trace store of k_grad2d (fixed c and line end; the x- and y-line threads of an element write
// faces {0, 2} or {1, 3}) touches one line per element instead of two.  Time-neutral on cfg 5 (gradients
// 1.989 vs 1.992 ms/step); kept because k_grad2d's allocation then fits its 128 registers without a spill.
#ifndef VT_CF
#define VT_CF 1
#endif
__device__ __forceinline__ size_t vidx2d(int e, int face, int c, int k)
{
    return VT_CF ? (((size_t)e * GV + c) * 4 + face) * NP + k : gidx2d(e, face, c, k);
}
// ---------------------------------------------------------------------------------------------
// surface kernel
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ const double *state_base(const StateBufs &sb, int src)
{
    return src == SRC_BUF ? sb.Ubuf : (src == SRC_IN ? sb.Uin : sb.Un);
}

// the 4 conserved variables of face node k of element e in the stage state given by src; all loads
// are issued before any use (the K_1 loads only when the state is formed lazily)
__device__ __forceinline__ void trace2d(const StateBufs &sb, int src, double dtc, int e, int face, int k, double u[4])
{
    const size_t b = (size_t)e * 64 + face_node2d(face, k);
    const double *P = state_base(sb, src);
#pragma unroll
    for (int v = 0; v < 4; ++v) u[v] = __ldg(P + b + v * 16);
    if (src == SRC_LAZY) {
        double kk[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) kk[v] = __ldg(sb.K1 + b + v * 16);
#pragma unroll
        for (int v = 0; v < 4; ++v) u[v] = fma(dtc, kk[v], u[v]);
    }
}

__device__ __forceinline__ void store_face2d(double *Fs, int e, int face, int k, const double f[4])
{
    const size_t b = ((size_t)e * 4 + face) * 16 + k;
#pragma unroll
    for (int v = 0; v < 4; ++v) Fs[b + v * 4] = f[v];
}

// NS: the face flux is HLL(u_L, u_R) - (F^v_L + F^v_R)/2 (central BR1 viscous flux from the
// normal viscous-flux traces Vt of k_grad2d), so the volume kernel lifts one combined flux.
#ifndef SURF2D_MINB
#define SURF2D_MINB 3
#endif
// SCS: the shock-capturing neighbour smoothing (sc.cuh) rides along, in a pass over the faces after the
// fluxes (one thread per interface / mortar) -- formerly lane k = 0 of every interface /
// mortar raises alpha of both sides to half the other side's raw value (k_sc_alpha ran before).
__device__ __forceinline__ void sc_amax(double *p, double v)
{
    atomicMax(reinterpret_cast<unsigned long long *>(p), (unsigned long long)__double_as_longlong(v));
}

template <int MODE, bool NS, bool SCS = false>
__global__ void __launch_bounds__(256, SURF2D_MINB) k_surf2d(MeshDev md, StageParams sp, const double *__restrict__ Un,
                                               const double *__restrict__ Ubuf, const double *__restrict__ K1,
                                               const double *__restrict__ Uin, double *__restrict__ Fs,
                                               const double *__restrict__ Vt, const double *__restrict__ alpha_raw,
                                               double *alpha)
{
    int nif, nmo, nbd;
    if (MODE == MODE_STAGE) {
        nif = md.count_active[KIND_IF * MAXS + sp.stage - 1];
        nmo = md.count_active[KIND_MO * MAXS + sp.stage - 1];
        nbd = md.count_active[KIND_BD * MAXS + sp.stage - 1];
    } else {
        nif = md.n[1]; nmo = md.n[2]; nbd = md.n[3];
    }
    const int total = 4 * (nif + nmo + nbd);
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const double dtc = sp.dt * sp.c_stage;
    const double g = md.gamma;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = 0xFu << (lane & ~3);
    const int GS = gridDim.x * blockDim.x;
    const int nI = 4 * nif;
    int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int4 *__restrict__ IR = MODE == MODE_STAGE ? md.ifcs : md.ifc;
#ifndef L2_HINTS_SURF
#define L2_HINTS_SURF 2     // Vt is dead once read: 2 = streaming loads (ld.global.cs, evict-first, no extra register;
                            // cfg 5 surface 1.424 -> 1.411 ms/step); 1 = a cache-hint policy operand, which pushes the
                            // Navier-Stokes instantiation over its 80 registers (spills, slower); 0 = plain loads
#endif
    const unsigned long long pol_dead = NS && L2_HINTS_SURF == 1 ? l2_evict_first_policy() : 0ull;   // Vt is dead after this launch
    auto ldg_vt = [&](const double *p) { return L2_HINTS_SURF == 2 ? __ldcs(p) : (L2_HINTS_SURF ? ldg_dead(p, pol_dead) : __ldg(p)); };
    pdl_wait();
    // two interface face nodes per iteration while both are interfaces: twice the loads in flight
    // per thread (the kernel is bound by the latency of the record -> trace gathers).  (Tried: the next
    // iteration's records prefetched into registers (spills at 80 registers), into L1, or the first
    // records into L1 before the dependency wait: cfg 3 surface 0.1847 -> 0.1854 / 0.1838 ms/step, noise)
    for (; gt + GS < nI; gt += 2 * GS) {
        const int ka = gt & 3, kb = (gt + GS) & 3;
        const int4 Ia = IR[sweep_idx(sp, gt >> 2, nif)];
        const int4 Ib = IR[sweep_idx(sp, (gt + GS) >> 2, nif)];
        PERK_DASSERT(Ia.x >= 0 && Ia.x < md.n[0] && Ia.y >= 0 && Ia.y < md.n[0] && Ib.x >= 0 && Ib.x < md.n[0] &&
                     Ib.y >= 0 && Ib.y < md.n[0]);
        const int srca = state_src(sp, Ia.w), srcb = state_src(sp, Ib.w);
        double uLa[4], uRa[4], uLb[4], uRb[4], fa[4], fb[4];
        trace2d(sb, srca, dtc, Ia.x, 2 * Ia.z, ka, uLa);
        trace2d(sb, srca, dtc, Ia.y, 2 * Ia.z + 1, ka, uRa);
        trace2d(sb, srcb, dtc, Ib.x, 2 * Ib.z, kb, uLb);
        trace2d(sb, srcb, dtc, Ib.y, 2 * Ib.z + 1, kb, uRb);
        numflux2d(uLa, uRa, Ia.z, g, md.surface, fa);
        numflux2d(uLb, uRb, Ib.z, g, md.surface, fb);
        if (NS) {
#pragma unroll
            for (int c = 0; c < GV; ++c) {
                fa[1 + c] -= 0.5 * (ldg_vt(Vt + vidx2d(Ia.x, 2 * Ia.z, c, ka)) + ldg_vt(Vt + vidx2d(Ia.y, 2 * Ia.z + 1, c, ka)));
                fb[1 + c] -= 0.5 * (ldg_vt(Vt + vidx2d(Ib.x, 2 * Ib.z, c, kb)) + ldg_vt(Vt + vidx2d(Ib.y, 2 * Ib.z + 1, c, kb)));
            }
        }
        store_face2d(Fs, Ia.x, 2 * Ia.z, ka, fa);
        store_face2d(Fs, Ia.y, 2 * Ia.z + 1, ka, fa);
        store_face2d(Fs, Ib.x, 2 * Ib.z, kb, fb);
        store_face2d(Fs, Ib.y, 2 * Ib.z + 1, kb, fb);
    }
    for (; gt < total; gt += GS) {
        const int item = gt >> 2, k = gt & 3;
        if (item < nif) {
            const int4 I = IR[sweep_idx(sp, item, nif)];
            PERK_DASSERT(I.x >= 0 && I.x < md.n[0] && I.y >= 0 && I.y < md.n[0]);
            const int o = I.z;
            const int src = state_src(sp, I.w);    // conforming: both sides share the member
            double uL[4], uR[4], fl[4];

            trace2d(sb, src, dtc, I.x, 2 * o, k, uL);
            trace2d(sb, src, dtc, I.y, 2 * o + 1, k, uR);
            numflux2d(uL, uR, o, g, md.surface, fl);
            if (NS) {
#pragma unroll
                for (int c = 0; c < GV; ++c)
                    fl[1 + c] -= 0.5 * (ldg_vt(Vt + vidx2d(I.x, 2 * o, c, k)) + ldg_vt(Vt + vidx2d(I.y, 2 * o + 1, c, k)));
            }
            store_face2d(Fs, I.x, 2 * o, k, fl);
            store_face2d(Fs, I.y, 2 * o + 1, k, fl);
        } else if (item < nif + nmo) {
            const int q = sweep_idx(sp, item - nif, nmo);
            const int4 M = MODE == MODE_STAGE ? md.mors[q] : md.mor[q];
            PERK_DASSERT(M.x >= 0 && M.x < md.n[0] && M.y >= 0 && M.y < md.n[0] && M.z >= 0 && M.z < md.n[0]);
            const int o = M.w & 1, side = (M.w >> 1) & 1, mfine = M.w >> 8;
            const int lf = 2 * o + side, sf = 2 * o + 1 - side;
            const int srcL = state_src(sp, md.mem[M.x]);
            const int srcS = state_src(sp, mfine);
            double ul[4];
            trace2d(sb, srcL, dtc, M.x, lf, k, ul);
            double uil[4] = {0, 0, 0, 0}, uih[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                const double plo = cB.Plo[k][j], pup = cB.Pup[k][j];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const double uj = __shfl_sync(gmask, ul[v], j, 4);
                    uil[v] = fma(plo, uj, uil[v]);
                    uih[v] = fma(pup, uj, uih[v]);
                }
            }
            double flo[4], fhi[4];
            {
                double us[4];
                trace2d(sb, srcS, dtc, M.y, sf, k, us);
                if (side == 0) numflux2d(uil, us, o, g, md.surface, flo);
                else numflux2d(us, uil, o, g, md.surface, flo);
            }
            {
                double us[4];
                trace2d(sb, srcS, dtc, M.z, sf, k, us);
                if (side == 0) numflux2d(uih, us, o, g, md.surface, fhi);
                else numflux2d(us, uih, o, g, md.surface, fhi);
            }
            if (NS) {   // central viscous flux on each half: (P F^v_large + F^v_small) / 2
                double vl[GV];
#pragma unroll
                for (int c = 0; c < GV; ++c) vl[c] = ldg_vt(Vt + vidx2d(M.x, lf, c, k));
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    double il = 0.0, ih = 0.0;
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        const double vj = __shfl_sync(gmask, vl[c], j, 4);
                        il = fma(cB.Plo[k][j], vj, il);
                        ih = fma(cB.Pup[k][j], vj, ih);
                    }
                    flo[1 + c] -= 0.5 * (il + ldg_vt(Vt + vidx2d(M.y, sf, c, k)));
                    fhi[1 + c] -= 0.5 * (ih + ldg_vt(Vt + vidx2d(M.z, sf, c, k)));
                }
            }
            store_face2d(Fs, M.y, sf, k, flo);
            store_face2d(Fs, M.z, sf, k, fhi);
            double fl[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                const double rlo = cB.Rlo[k][j], rup = cB.Rup[k][j];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const double a = __shfl_sync(gmask, flo[v], j, 4);
                    const double b = __shfl_sync(gmask, fhi[v], j, 4);
                    fl[v] = fma(rup, b, fma(rlo, a, fl[v]));
                }
            }
            store_face2d(Fs, M.x, lf, k, fl);
        } else {
            const int q = item - nif - nmo;
            const int bi = MODE == MODE_STAGE ? md.list[KIND_BD][q] : q;
            const int2 B = md.bnd[bi];
            PERK_DASSERT(B.x >= 0 && B.x < md.n[0]);
            const int face = B.y & 7, o = face >> 1;
            const int src = state_src(sp, B.y >> 8);
            double u[4], fl[4];
            trace2d(sb, src, dtc, B.x, face, k, u);
            if ((face & 1) == 0) numflux2d(u, md.bc, o, g, md.surface, fl);
            else numflux2d(md.bc, u, o, g, md.surface, fl);
            store_face2d(Fs, B.x, face, k, fl);
        }
    }
    if (SCS) {   // shock-capturing smoothing: one thread per face after the fluxes (kept out of the flux
                 // loops, whose 80-register budget of 3 CTAs per SM it would exceed); counts re-read
        const int nif2 = MODE == MODE_STAGE ? ld_volatile(md.count_active + KIND_IF * MAXS + sp.stage - 1) : md.n[1];
        const int nmo2 = MODE == MODE_STAGE ? ld_volatile(md.count_active + KIND_MO * MAXS + sp.stage - 1) : md.n[2];
        for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nif2 + nmo2; t += gridDim.x * blockDim.x) {
            if (t < nif2) {
                const int4 I = MODE == MODE_STAGE ? md.ifcs[t] : md.ifc[t];
                sc_amax(alpha + I.x, 0.5 * __ldg(alpha_raw + I.y));
                sc_amax(alpha + I.y, 0.5 * __ldg(alpha_raw + I.x));
            } else {
                const int4 M = MODE == MODE_STAGE ? md.mors[t - nif2] : md.mor[t - nif2];
                const double al = 0.5 * __ldg(alpha_raw + M.x);
                sc_amax(alpha + M.x, 0.5 * fmax(__ldg(alpha_raw + M.y), __ldg(alpha_raw + M.z)));
                sc_amax(alpha + M.y, al);
                sc_amax(alpha + M.z, al);
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// volume + surface lift + Jacobian + stage epilogue
// ---------------------------------------------------------------------------------------------
constexpr int VOL2D_EPB = 16;   // elements per 128-thread block (8 threads per element)
// Shared-memory layout (bank-conflict free): every field is stored twice, in
// x-line order (index 16 le + 4j + i) and in y-line order (index 20 le + 4i + j, shifted by 2), in
// the 2 LS doubles of the field; the x-line and y-line threads of an element hit disjoint banks in
// the 16 B line loads, and the two elements of a half-warp hit disjoint banks in the scalar y-layout
// stores / loads.  The accumulators alias the first 4 fields; the BR1 gradients (NS) alias fields
// 4..6 once the two-point fluxes have consumed them.
constexpr int VOL2D_LS = 288;   // half of the doubles per field (x part 16 EPB, y part 20 EPB + 2 < 2 LS)
// k_vol2d fields (layout o = line direction): rho, v_n/2, v_t/2, p/2, ln rho, beta = rho/p, ln beta (+ T)
constexpr int F_RHO = 0, F_HVN = 1, F_HVT = 2, F_HP = 3, F_LRHO = 4, F_BETA = 5, F_LBETA = 6, F_T = 7;
// k_grad2d fields (both layouts): v1, v2, T
constexpr int F_V1 = 1, F_V2 = 2;

__device__ __forceinline__ double2 load_state2(const StateBufs &sb, int src, double dtc, size_t idx)
{
    switch (src) {
    case SRC_UN: return __ldg(reinterpret_cast<const double2 *>(sb.Un + idx));
    case SRC_BUF: return __ldg(reinterpret_cast<const double2 *>(sb.Ubuf + idx));
    case SRC_LAZY: {
        const double2 a = __ldg(reinterpret_cast<const double2 *>(sb.Un + idx));
        const double2 k = __ldg(reinterpret_cast<const double2 *>(sb.K1 + idx));
        return make_double2(fma(dtc, k.x, a.x), fma(dtc, k.y, a.y));
    }
    default: return __ldg(reinterpret_cast<const double2 *>(sb.Uin + idx));
    }
}

// BR1 gradient of (v1, v2, T) along this thread's line (direction o, line ln), weak form with the
// central traces Gs:  q[c][a] = (2/h) [ -sum_k Dhat_ak w_c[k] + (delta_a3 w*_{+o} - delta_a0 w*_{-o}) / w_a ].
// Component c is read from field fld[c] of layout o, which holds w_c / sc[c] (sc = 1 or 2: the volume
// kernel stores half velocities; scaling by 2 is exact, so q is bitwise the unscaled result).
// Ge = the element's 48 central traces ([face][c][k], e.g. a shared-memory staged copy).
template <int LS>
__device__ __forceinline__ void line_gradient(const double (*sm)[2][LS], int o, int lo, int ln,
                                              const double *Ge, double Jq, const int fld[GV],
                                              const double sc[GV], double q[GV][NP])
{
#pragma unroll
    for (int c = 0; c < GV; ++c) {
        double w[NP];
        {   // the line is contiguous and 16 B aligned in either layout: two 16 B loads (one element per
            // quarter-warp, conflict-free) instead of four scalar ones
            const double2 w01 = *reinterpret_cast<const double2 *>(&sm[fld[c]][o][lo]);
            const double2 w23 = *reinterpret_cast<const double2 *>(&sm[fld[c]][o][lo + 2]);
            w[0] = w01.x; w[1] = w01.y; w[2] = w23.x; w[3] = w23.y;
        }
        const double isc = 1.0 / sc[c];
        const double ghi = Ge[gidx2d(0, 2 * o, c, ln)] * isc;
        const double glo = Ge[gidx2d(0, 2 * o + 1, c, ln)] * isc;
#pragma unroll
        for (int a = 0; a < NP; ++a) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < NP; ++k) t = fma(-cB.Dhat[a][k], w[k], t);
            if (a == NP - 1) t = fma(ghi, cB.invw[NP - 1], t);
            if (a == 0) t = fma(-glo, cB.invw[0], t);
            q[c][a] = (Jq * sc[c]) * t;
        }
    }
    PERK_JITTER(8);
}

// the same gradient with the two end traces given in registers (fused BR1 gradient kernel; sc = 1):
// ghi[c] = w*_c at the +o face node of the line, glo[c] at the -o face node
template <int LS>
__device__ __forceinline__ void line_gradient_g(const double (*sm)[2][LS], int o, int lo, const double ghi[GV],
                                                const double glo[GV], double Jq, const int fld[GV], double q[GV][NP])
{
#pragma unroll
    for (int c = 0; c < GV; ++c) {
        double w[NP];
        {
            const double2 w01 = *reinterpret_cast<const double2 *>(&sm[fld[c]][o][lo]);
            const double2 w23 = *reinterpret_cast<const double2 *>(&sm[fld[c]][o][lo + 2]);
            w[0] = w01.x; w[1] = w01.y; w[2] = w23.x; w[3] = w23.y;
        }
#pragma unroll
        for (int a = 0; a < NP; ++a) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < NP; ++k) t = fma(-cB.Dhat[a][k], w[k], t);
            if (a == NP - 1) t = fma(ghi[c], cB.invw[NP - 1], t);
            if (a == 0) t = fma(-glo[c], cB.invw[0], t);
            q[c][a] = Jq * t;
        }
    }
    PERK_JITTER(8);
}

// the same with the line's values in registers
__device__ __forceinline__ void line_gradient_w(const double w[GV][NP], const double ghi[GV], const double glo[GV],
                                                double Jq, double q[GV][NP])
{
#pragma unroll
    for (int c = 0; c < GV; ++c) {
#pragma unroll
        for (int a = 0; a < NP; ++a) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < NP; ++k) t = fma(-cB.Dhat[a][k], w[c][k], t);
            if (a == NP - 1) t = fma(ghi[c], cB.invw[NP - 1], t);
            if (a == 0) t = fma(-glo[c], cB.invw[0], t);
            q[c][a] = Jq * t;
        }
    }
    PERK_JITTER(8);
}

// NS volume contribution (MODE_STAGE and MODE_RHS): adds sum_a Dhat_ia F^v_o(node a) to acc (in line
// coordinates: acc[.][1] normal, acc[.][2] tangential momentum), i.e. -(2/h)(...) of the weak-form
// viscous divergence after the common -2/h scaling.  Fields 4..6 are overwritten with the gradients.
template <int LS>
__device__ __forceinline__ void visc_volume(double (*sm)[2][LS], int o, int lo, int eox, int eoy, int yo, int ln,
                                            const double *Ge, double Jq, double mu, double kappa,
                                            double acc[NP][4])
{
    const int fld[GV] = {o == 0 ? F_HVN : F_HVT, o == 0 ? F_HVT : F_HVN, F_T};   // v1/2, v2/2, T
    const double sc[GV] = {2.0, 2.0, 1.0};
    double q[GV][NP];
    line_gradient<LS>(sm, o, lo, ln, Ge, Jq, fld, sc, q);
    __syncwarp();   // every thread of the element is done with fields 4..6 (two-point fluxes)
#pragma unroll
    for (int c = 0; c < GV; ++c) {   // contiguous, 16 B aligned line: two 16 B stores
        *reinterpret_cast<double2 *>(&sm[4 + c][o][lo]) = make_double2(q[c][0], q[c][1]);
        *reinterpret_cast<double2 *>(&sm[4 + c][o][lo + 2]) = make_double2(q[c][2], q[c][3]);
    }
    __syncwarp();
    // the line's own half velocities: contiguous, two 16 B loads per field (scalar reads of the x layout
    // were 2-way bank conflicts between the two elements of a half-warp)
    double hv1[NP], hv2[NP];
    {
        const double2 a01 = *reinterpret_cast<const double2 *>(&sm[fld[0]][o][lo]);
        const double2 a23 = *reinterpret_cast<const double2 *>(&sm[fld[0]][o][lo + 2]);
        const double2 b01 = *reinterpret_cast<const double2 *>(&sm[fld[1]][o][lo]);
        const double2 b23 = *reinterpret_cast<const double2 *>(&sm[fld[1]][o][lo + 2]);
        hv1[0] = a01.x; hv1[1] = a01.y; hv1[2] = a23.x; hv1[3] = a23.y;
        hv2[0] = b01.x; hv2[1] = b01.y; hv2[2] = b23.x; hv2[3] = b23.y;
    }
#pragma unroll
    for (int a = 0; a < NP; ++a) {
        // the other direction's gradient at this node: node (a, ln) of an x-line lives at y-layout
        // index yo + eoy + 4a + ln; node (ln, a) of a y-line at x-layout index eox + 4a + ln
        const int oi = o == 0 ? yo + eoy + 4 * a + ln : eox + 4 * a + ln;
        double qo[GV], qs[GV];
#pragma unroll
        for (int c = 0; c < GV; ++c) {
            qs[c] = q[c][a];
            qo[c] = sm[4 + c][1 - o][oi];
        }
        const double v1 = 2.0 * hv1[a], v2 = 2.0 * hv2[a];
        double f[GV];
        if (o == 0) visc_flux2d(v1, v2, qs, qo, 0, mu, kappa, f);
        else visc_flux2d(v1, v2, qo, qs, 1, mu, kappa, f);
        // (momentum x, momentum y, energy) -> line coordinates (normal, tangential, energy), applied to
        // every node at once (same per-node summation order over a as a separate contraction, without
        // holding the 12 fluxes of the line)
        const double fl[GV] = {o == 0 ? f[0] : f[1], o == 0 ? f[1] : f[0], f[2]};
#pragma unroll
        for (int i = 0; i < NP; ++i)
#pragma unroll
            for (int c = 0; c < GV; ++c) acc[i][1 + c] = fma(cB.Dhat[i][a], fl[c], acc[i][1 + c]);
    }
}

// BR1_DV = 1: k_grad2d, which holds the element's gradients anyway, also forms the viscous volume
// term Dv = -(2/h) sum_a Dhat_ia F^v(node a) (x + y lines, 384 B per element) and the volume kernel
// adds it in its epilogue instead of recomputing the gradients from Gs (same bytes staged: Dv instead
// of Gs; the Navier-Stokes volume kernel becomes the Euler one plus one 16 B shared load per variable).
// BR1_DV = 0: the volume kernel recomputes q from the state and Gs (visc_volume).
#ifndef BR1_DV
#define BR1_DV 1
#endif

// Dynamic shared memory of k_vol2d (bytes): field arrays, own-state staging, epilogue staging.
__host__ __device__ constexpr int vol2d_nf(bool ns) { return ns && !BR1_DV ? 8 : 7; }
// U_n / K_1 operands of the stage epilogue: 1 = staged in shared memory with the Fs fluxes,
// 2 = loaded into registers before the two-point-flux loop.  Measured (cfg 3 / cfg 5 volume ms/step):
// Euler 1: 0.361, 2: 0.378; Navier-Stokes 1: 3.60, 2: 3.52 (its 16 KB smaller footprint fits 3
// instead of 2 CTAs per SM); read from global memory in the epilogue instead: Euler 0.406
// Navier-Stokes, mode 2: issue the register loads of U_n / K_1 after the two-point fluxes (in flight
// during the BR1 part) instead of before them, so they do not occupy 32 registers across the flux loop
#ifndef VOL2D_PRELOAD_LATE
#define VOL2D_PRELOAD_LATE 0
#endif
#ifndef VOL2D_EPI_MODE_EULER
#define VOL2D_EPI_MODE_EULER 1
#endif
#ifndef VOL2D_EPI_MODE_NS
#define VOL2D_EPI_MODE_NS 2
#endif
__host__ __device__ constexpr int vol2d_epi_mode(bool ns) { return ns ? VOL2D_EPI_MODE_NS : VOL2D_EPI_MODE_EULER; }
constexpr int EPI_UN = 0, EPI_K1 = 1;                                   // (mode 1 only)
__host__ __device__ constexpr int vol2d_epi_fs(bool ns) { return vol2d_epi_mode(ns) == 1 ? 2 : 0; }
__host__ __device__ constexpr int vol2d_epi_slots(bool ns) { return (vol2d_epi_mode(ns) == 1 ? 3 : 1) + (ns ? 1 : 0); }   // (U_n, K_1,) Fs (+ Gs)
// Staged face fluxes: face stride 18 doubles (instead of 16) and an element block == 8 mod 16, so that
// the lift's scalar reads of the x-line threads (faces 0/1) and y-line threads (faces 2/3) of the two
// elements of a half-warp fall into 4 disjoint bank groups (unpadded they were 4-way conflicts).
#ifndef VOL2D_FS_PAD
#define VOL2D_FS_PAD 1
#endif
__host__ __device__ constexpr int vol2d_fs_face(bool) { return VOL2D_FS_PAD ? 18 : 16; }
// element block: [U_n 64][K_1 64] (mode 1) [Fs 4 x face stride] [Gs 48 (NS)]; Euler 200 doubles,
// Navier-Stokes (mode 2) 72 + 48 = 120, both == 8 mod 16 with the padded faces
__host__ __device__ constexpr int vol2d_epi_stride(bool ns)
{
    return (vol2d_epi_mode(ns) == 1 ? 128 : 0) + 4 * vol2d_fs_face(ns) + (ns ? 4 * GV * NP : 0);
}
// elements per CTA: 16 (Euler: 4.5 KB of shared memory per element, 3 CTAs = 48 elements per SM).
// Navier-Stokes needs 5.4 KB per element: 16 per CTA fit 2 CTAs (32 elements) per SM, 8 per CTA
// fit 5 (40 elements) but measured no faster (cfg 5 volume 3.66 vs 3.62 ms/step), so 16 stays
#ifndef VOL2D_EPB_NS
#define VOL2D_EPB_NS 16
#endif
__host__ __device__ constexpr int vol2d_epb(bool ns) { return ns ? VOL2D_EPB_NS : VOL2D_EPB; }
__host__ __device__ constexpr int vol2d_ls(bool ns) { return 18 * vol2d_epb(ns); }   // == 0 mod 16 for 8 | EPB
__host__ __device__ constexpr int vol2d_threads(bool ns) { return 8 * vol2d_epb(ns); }
__host__ __device__ constexpr size_t vol2d_smem_bytes(bool ns)
{
    return sizeof(double) * ((size_t)vol2d_nf(ns) * 2 * vol2d_ls(ns) + vol2d_epb(ns) * 2 * 64 +
                             vol2d_epb(ns) * vol2d_epi_stride(ns));
}

// Volume + surface lift + Jacobian + stage epilogue.  Persistent grid-stride loop over groups of 16
// active elements per 128-thread CTA; each element's 512 B blocks are staged into shared memory with
// cp.async (16 B per thread and copy, coalesced, no registers), in two commit groups per iteration:
//   stg[le][0..1] : the stage state of the NEXT group (U_n | stage buffer | U_in, or U_n and K_1 for a
//                   lazy state), issued as soon as the current group's state has been read (phase 1)
//   epi[le][0..2] : U_n, K_1 and the face fluxes Fs of the CURRENT group, issued before the two-point
//                   flux loop and consumed after it (lift + epilogue)
// so neither the state gather nor the epilogue reads expose memory latency.  (A first version used
// cp.async.bulk on mbarriers; issuing the per-element bulk copies through the uniform datapath cost
// about a quarter of the kernel's issue slots.)
//
// SC (shock capturing, sc.cuh): the element's inviscid volume part becomes (1 - alpha) V_DG + alpha V_FV,
// V_FV[a] = (F_{a+1/2} - F_{a-1/2}) / w_a along the line with the subcell fluxes F_{a+1/2} = f*(u_a,
// u_{a+1}) of the problem's surface flux (F_{-1/2} = F_{N+1/2} = 0), evaluated in line coordinates
// from the primitives the line already holds; alpha = 0 elements skip it.
template <int MODE, bool NS, bool SC = false>
// (Navier-Stokes + shock capturing: 2 CTAs per SM -- at 3 the 168-register budget spilled 44 B and the
//  kernel was slower, cfg 5 SC volume 4.48 vs 4.18 ms/step; NSSC_MINB=3 builds that variant)
#ifndef NSSC_MINB
#define NSSC_MINB 2
#endif
__global__ void __launch_bounds__(vol2d_threads(NS), NS ? (VOL2D_EPB_NS == 8 ? 5 : (SC ? NSSC_MINB : 3)) : 3)
k_vol2d(MeshDev md, StageParams sp, double *__restrict__ Un,
                                                 double *__restrict__ Ubuf, double *__restrict__ K1,
                                                 const double *__restrict__ Fs, const double *__restrict__ Uin,
                                                 double *__restrict__ dU, const double *__restrict__ Gs,
                                                 double *__restrict__ Wb, double *alpha, double *alpha_raw,
                                                 ScParams scp)
{
    constexpr int NF = vol2d_nf(NS);          // rho, v_n/2, v_t/2, p/2, ln rho, beta, ln beta (+ T)
    constexpr int EPB = vol2d_epb(NS), LS = vol2d_ls(NS);
    extern __shared__ __align__(16) unsigned char smraw[];
    double (*sm)[2][LS] = reinterpret_cast<double (*)[2][LS]>(smraw);
    double (*stg)[2][64] = reinterpret_cast<double (*)[2][64]>(smraw + sizeof(double) * NF * 2 * LS);
    constexpr int NEPI = vol2d_epi_slots(NS);
    constexpr int EM = vol2d_epi_mode(NS), EPI_FS = vol2d_epi_fs(NS), EPI_GS = EPI_FS + 1;
    constexpr int FSF = vol2d_fs_face(NS), EPS = vol2d_epi_stride(NS);
    static_assert(EPS >= (EM == 1 ? 128 : 0) + 4 * FSF + (NS ? 4 * GV * NP : 0), "epilogue block");
    double *epi_all = reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(stg) + sizeof(double) * EPB * 2 * 64);
    const int t8 = threadIdx.x & 7, le = threadIdx.x >> 3;
    // slot base of this element: U_n, K_1 (64 each, mode 1), Fs (4 faces x FSF), Gs (NS) right after Fs
    auto EP = [&](int slot) {
        return epi_all + (size_t)le * EPS + (slot <= EPI_FS ? slot * 64 : EPI_FS * 64 + 4 * FSF);
    };
    const int n_act = MODE == MODE_STAGE ? md.count_active[KIND_EL * MAXS + sp.stage - 1] : md.n[0];
    const double g = md.gamma, gm1 = g - 1.0, inv_gm1 = 1.0 / gm1;
    const double dtc = sp.dt * sp.c_stage;
    const double two_hf = 2.0 / md.hf;
    const int q0 = 2 * t8;
    const int o = t8 >> 2, ln = t8 & 3;
    // element offsets: x layout 16 per element, y layout 20 per element starting 2 doubles into the
    // second half of the field's 2 LS doubles (yo < 0 indexes from [k][1] back into that half): the
    // x-line and y-line threads of one element hit disjoint banks in the line loads (y - x == 2 mod 4)
    // and the two elements of a half-warp hit disjoint banks in the scalar y-layout stores / loads
    // (20 == 4 mod 8); with 18 / 18 and +2 the latter were 2-way conflicts
    const int eox = le * 16, eoy = le * 20;
    const int yo = 2 - 2 * EPB;
    static_assert(16 * EPB + 20 * (EPB - 1) + 2 + 16 <= 2 * LS, "field layout");
    const int stride = gridDim.x * EPB;

    int base = blockIdx.x * EPB;
    // SC epilogue indicator: Vandermonde rows in shared memory (lane-indexed __constant__ reads would
    // serialise) and a per-warp buffer of the energy sums of up to 16 elements, whose scalar tail
    // (quotients, exp, clipping) runs once per element on one lane
    __shared__ double sVv[SC ? NP * NP : 1];
    __shared__ double sTail[SC ? EPB / 4 : 1][3][SC ? 16 : 1];
    __shared__ int sTe[SC ? EPB / 4 : 1][SC ? 16 : 1];
    int nbuf = 0;                                    // elements buffered by this warp (warp-uniform)
    if (SC) {
        if (threadIdx.x < NP * NP) sVv[threadIdx.x] = cB.Vinv[threadIdx.x >> 2][threadIdx.x & 3];
        __syncthreads();
    }
    // prologue before the dependency wait: indices only (lists are rebuilt by the mesh pipeline,
    // which completed before the step started)
    const int pk0 = base < n_act ? (MODE == MODE_STAGE ? md.elpk[sweep_idx(sp, base + le < n_act ? base + le : base, n_act)] : 0) : 0;
    pdl_wait();
    if (MODE == MODE_STAGE && sp.stage == sp.S && blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(md.evals, md.evals[2]);           // sum_r E_r N_C(r), set by the mesh pipeline
        atomicAdd(md.evals + 1, 1ull);
    }
    if (base >= n_act) return;

    // packed entry (element | member | level) of this thread's slot in the group starting at b
    auto entry_at = [&](int b) {
        const int t = b + le;
        const int tt = sweep_idx(sp, t < n_act ? t : b, n_act);
        if (MODE == MODE_STAGE) return md.elpk[tt];
        return tt | ((int)md.mem[tt] << PK_EBITS) | ((int)md.lev[tt] << (PK_EBITS + 3));
    };
    // the element's 8 threads copy a 512 B block: 16 B chunks t8, t8 + 8, t8 + 16, t8 + 24
    auto copy_block = [&](double *dst, const double *src) {
#pragma unroll
        for (int r = 0; r < 4; ++r) cp_async16(dst + 2 * (t8 + 8 * r), src + 2 * (t8 + 8 * r));
    };
    const unsigned long long pol_dead = l2_evict_first_policy();   // Fs, Dv, U_n, K_1: not read again soon
    auto copy_block_dead = [&](double *dst, const double *src) {
#pragma unroll
        for (int r = 0; r < 4; ++r) cp_async16_dead(dst + 2 * (t8 + 8 * r), src + 2 * (t8 + 8 * r), pol_dead);
    };
    // U_n and K_1 come back at the next stage (L2_HINTS = 2 marks them too)
    auto copy_block_far = [&](double *dst, const double *src) {
        if (L2_HINTS >= 2) copy_block_dead(dst, src);
        else copy_block(dst, src);
    };
    auto ldg2_far = [&](const double2 *p) { return L2_HINTS >= 2 ? ldg2_dead(p, pol_dead) : __ldg(p); };
    auto issue_state = [&](int pkx) {
        const size_t off = (size_t)pk_elem(pkx) * 64;
        const int srce = state_src(sp, pk_member(pkx));
        copy_block(stg[le][0], (srce == SRC_UN || srce == SRC_LAZY ? Un : (srce == SRC_BUF ? Ubuf : Uin)) + off);
        if (srce == SRC_LAZY) copy_block(stg[le][1], K1 + off);
        cp_async_commit();
    };
    int pk = MODE == MODE_STAGE ? pk0 : entry_at(base);
    // packed entries run two groups ahead: the next group's entry is needed right after phase 1 (to
    // issue its state copy), too soon for a load issued at the top of the same iteration (ncu: 15 %
    // of the Navier-Stokes kernel's stall samples waited on it)
    int pk_ahead = base + stride < n_act ? entry_at(base + stride) : 0;
    issue_state(pk);

    for (; base < n_act; base += stride) {
        const bool valid = base + le < n_act;
        const bool has_next = base + stride < n_act;     // uniform across the CTA
        const int pk_next = pk_ahead;                     // consumed after phase 1
        pk_ahead = base + 2 * stride < n_act ? entry_at(base + 2 * stride) : 0;
        const int e = pk_elem(pk);
        PERK_DASSERT(!valid || (e >= 0 && e < md.n[0]));
        const int m = pk_member(pk);
        const int src = state_src(sp, m);
        const size_t eb = (size_t)e * 64;
        const double j2h = two_over_h(two_hf, pk_level(pk), md.max_level);   // 2 / h
        double2 pre_un[4], pre_k1[4];          // epilogue operands held in registers (EM == 2)
        const double al = SC ? alpha[e] : 0.0;   // read before this element's next-stage alpha is written

        // phase 1: nodes q0, q0+1 -> primitives + logs, stored in x-line and y-line layouts
        PERK_JITTER(1);
        cp_async_wait<0>();
        __syncwarp();
        PERK_JITTER(2);
        {
            double2 u[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                u[v] = *reinterpret_cast<const double2 *>(&stg[le][0][v * 16 + q0]);
                if (src == SRC_LAZY) {
                    const double2 k = *reinterpret_cast<const double2 *>(&stg[le][1][v * 16 + q0]);
                    u[v] = make_double2(fma(dtc, k.x, u[v].x), fma(dtc, k.y, u[v].y));
                }
            }
            double fx[2][8], fy[2][8];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double r = h ? u[0].y : u[0].x;
                const double m1 = h ? u[1].y : u[1].x, m2 = h ? u[2].y : u[2].x, E = h ? u[3].y : u[3].x;
                const double ir = rcp64(r);
                const double v1 = m1 * ir, v2 = m2 * ir;
                const double p = gm1 * (E - 0.5 * fma(m1, v1, m2 * v2));
                const double beta = r * rcp64(p);
                const double lr = log_pos(r), lb = lr - log_pos(p);   // ln beta = ln rho - ln p
                const double hv1 = 0.5 * v1, hv2 = 0.5 * v2, hp = 0.5 * p;
                // x layout: normal = x; y layout: normal = y
                const double ax[8] = {r, hv1, hv2, hp, lr, beta, lb, p * ir};
                const double ay[8] = {r, hv2, hv1, hp, lr, beta, lb, p * ir};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    fx[h][k] = ax[k];
                    fy[h][k] = ay[k];
                }
            }
            // nodes q0 = (i0, j0), q0 + 1 = (i0 + 1, j0): adjacent in the x layout (one 16 B store),
            // 4 apart in the y layout
            const int i0 = q0 & 3, j0 = q0 >> 2;
#pragma unroll
            for (int k = 0; k < NF; ++k) {
                *reinterpret_cast<double2 *>(&sm[k][0][eox + 4 * j0 + i0]) = make_double2(fx[0][k], fx[1][k]);
                sm[k][1][yo + eoy + 4 * i0 + j0] = fy[0][k];
                sm[k][1][yo + eoy + 4 * (i0 + 1) + j0] = fy[1][k];
            }
        }
        PERK_JITTER(3);
        __syncwarp();   // the warp has read stg: refill it (next group) and stage this group's epilogue operands
        {
            const bool need_un = MODE == MODE_STAGE && sp.stage > 1;
            const bool need_k1 = MODE == MODE_STAGE && sp.stage > 1 && (sp.stage < sp.S || sp.fin_k1);
            if (FSF == 18) {   // padded face layout: chunk c of the 512 B block -> 2c + 2 (c / 8)
#pragma unroll
                for (int r = 0; r < 4; ++r) cp_async16_dead(EP(EPI_FS) + 2 * (t8 + 8 * r) + 2 * r, Fs + eb + 2 * (t8 + 8 * r), pol_dead);
            } else {
                copy_block_dead(EP(EPI_FS), Fs + eb);
            }
            // stage S combines with W (P-ERK3) or U_n
            if (EM == 2) {
                if (valid && !(NS && VOL2D_PRELOAD_LATE)) {
                    const double *usrc = (Wb && sp.stage == sp.S) ? Wb : Un;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        if (need_un) pre_un[v] = ldg2_far(reinterpret_cast<const double2 *>(usrc + eb + v * 16 + q0));
                        if (need_k1) pre_k1[v] = ldg2_far(reinterpret_cast<const double2 *>(K1 + eb + v * 16 + q0));
                    }
                }
            } else {
                if (need_un) copy_block_far(EP(EPI_UN), (Wb && sp.stage == sp.S ? Wb : Un) + eb);
                if (need_k1) copy_block_far(EP(EPI_K1), K1 + eb);
            }
            if (NS) {   // the element's 48 BR1 central traces, or (BR1_DV) its viscous volume term (384 B = 24 chunks)
#pragma unroll
                for (int r = 0; r < 3; ++r)
                    cp_async16_dead(EP(EPI_GS) + 2 * (t8 + 8 * r), Gs + (size_t)e * 4 * GV * NP + 2 * (t8 + 8 * r), pol_dead);
            }
            cp_async_commit();
        }
        if (has_next) issue_state(pk_next);

        // phase 2: 6 symmetric two-point fluxes along this thread's line (x-line j = ln, or y-line i = ln)
        const int lo = o == 0 ? eox + 4 * ln : yo + eoy + 4 * ln;   // line start in layout o
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[a][v] = 0.0;
        // the line's 4 nodes x 7 fields, loaded once with 16 B shared loads (the line is contiguous)
        LinePrim P[4];
        {
            const double *L0 = &sm[0][o][lo];   // field k of line node a: L0[k * 2 * LS + a]
            double fv[7][4];
#pragma unroll
            for (int k = 0; k < 7; ++k) {
                const double2 x01 = *reinterpret_cast<const double2 *>(L0 + k * 2 * LS);
                const double2 x23 = *reinterpret_cast<const double2 *>(L0 + k * 2 * LS + 2);
                fv[k][0] = x01.x;
                fv[k][1] = x01.y;
                fv[k][2] = x23.x;
                fv[k][3] = x23.y;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) P[a] = LinePrim{fv[0][a], fv[1][a], fv[2][a], fv[3][a], fv[4][a], fv[5][a], fv[6][a]};
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
#pragma unroll
            for (int b = a + 1; b < 4; ++b) {
                double f[4];
                flux_ranocha_line(P[a], P[b], inv_gm1, f);
                const double dab = cB.Dsplit[a][b], dba = cB.Dsplit[b][a];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    acc[a][v] = fma(dab, f[v], acc[a][v]);
                    acc[b][v] = fma(dba, f[v], acc[b][v]);
                }
            }
        }
        if (SC && al != 0.0) {   // blend with the subcell finite-volume divergence
            double Fp[3][4];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                double uL[4], uR[4];
                const LinePrim &A = P[a], &B = P[a + 1];
                const double vnA = 2.0 * A.hvn, vtA = 2.0 * A.hvt, vnB = 2.0 * B.hvn, vtB = 2.0 * B.hvt;
                uL[0] = A.rho; uL[1] = A.rho * vnA; uL[2] = A.rho * vtA;
                uL[3] = 2.0 * A.hp * inv_gm1 + 0.5 * A.rho * (vnA * vnA + vtA * vtA);
                uR[0] = B.rho; uR[1] = B.rho * vnB; uR[2] = B.rho * vtB;
                uR[3] = 2.0 * B.hp * inv_gm1 + 0.5 * B.rho * (vnB * vnB + vtB * vtB);
                numflux2d(uL, uR, 0, g, md.surface, Fp[a]);   // line coordinates: normal first
            }
            const double bl = 1.0 - al;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const double fr = a < 3 ? Fp[a][v] : 0.0, fl = a > 0 ? Fp[a - 1][v] : 0.0;
                    acc[a][v] = fma(al, (fr - fl) * cB.invw[a], bl * acc[a][v]);
                }
        }
        // NS: + sum_a Dhat_ia F^v(node a) along the line (BR1 gradients recomputed from Gs)
        if (NS && EM == 2 && VOL2D_PRELOAD_LATE && valid) {   // the epilogue operands, in flight during the BR1 part
            const bool need_un = MODE == MODE_STAGE && sp.stage > 1;
            const bool need_k1 = MODE == MODE_STAGE && sp.stage > 1 && (sp.stage < sp.S || sp.fin_k1);
            const double *usrc = (Wb && sp.stage == sp.S) ? Wb : Un;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                if (need_un) pre_un[v] = ldg2_far(reinterpret_cast<const double2 *>(usrc + eb + v * 16 + q0));
                if (need_k1) pre_k1[v] = ldg2_far(reinterpret_cast<const double2 *>(K1 + eb + v * 16 + q0));
            }
        }
        if (NS && !BR1_DV) {
            PERK_JITTER(4);
            if (has_next) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncwarp();
            visc_volume<LS>(sm, o, lo, eox, eoy, yo, ln, EP(EPI_GS), j2h, md.mu, md.kappa, acc);
        }
        // surface lift: + f*_hi / w_N at the last node, - f*_lo / w_0 at the first node
        // line coordinates (normal, tangential) -> (momentum x, momentum y)
        if (o == 1) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const double t = acc[a][1];
                acc[a][1] = acc[a][2];
                acc[a][2] = t;
            }
        }
        PERK_JITTER(5);
        if (has_next) cp_async_wait<1>();    // this group's epilogue operands (the next state may still fly)
        else cp_async_wait<0>();
        __syncwarp();
        {
            const double *Fhi = EP(EPI_FS) + (2 * o) * FSF + ln;
            const double *Flo = EP(EPI_FS) + (2 * o + 1) * FSF + ln;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                acc[3][v] = fma(Fhi[v * 4], cB.invw[3], acc[3][v]);
                acc[0][v] = fma(-Flo[v * 4], cB.invw[0], acc[0][v]);
            }
        }
        double2 nu[4];   // SC: the next stage state of nodes q0, q0 + 1 written to the stage buffer
        // stage epilogue of one node pair (qq, qq + 1) of variable v (K = the pair's RHS values)
        auto epilogue = [&](int v, int qq, double2 K) {
            const size_t idx = eb + v * 16 + qq;
            if (MODE == MODE_RHS) {
                const bool on = (sp.mask >> m) & 1u;
                *reinterpret_cast<double2 *>(dU + idx) = on ? K : make_double2(0.0, 0.0);
            } else if (sp.stage == 1) {
                *reinterpret_cast<double2 *>(K1 + idx) = K;
            } else if (sp.stage == sp.S) {
                const double2 w = EM == 2 ? pre_un[v]
                                          : *reinterpret_cast<const double2 *>(EP(EPI_UN) + v * 16 + qq);   // W or U_n
                if (sp.fin_k1) {
                    const double2 k1 = EM == 2 ? pre_k1[v] : *reinterpret_cast<const double2 *>(EP(EPI_K1) + v * 16 + qq);
                    *reinterpret_cast<double2 *>(Un + idx) =
                        make_double2(fma(sp.dt, fma(sp.wb1, k1.x, sp.bS * K.x), w.x),
                                     fma(sp.dt, fma(sp.wb1, k1.y, sp.bS * K.y), w.y));
                } else {
                    const double db = sp.dt * sp.bS;
                    *reinterpret_cast<double2 *>(Un + idx) = make_double2(fma(db, K.x, w.x), fma(db, K.y, w.y));
                }
            } else {
                const double2 un = EM == 2 ? pre_un[v] : *reinterpret_cast<const double2 *>(EP(EPI_UN) + v * 16 + qq);
                const double2 k1 = EM == 2 ? pre_k1[v] : *reinterpret_cast<const double2 *>(EP(EPI_K1) + v * 16 + qq);
                const double a1 = sp.a1_next[m], as = sp.asub_next[m];
                const double2 nxt = make_double2(fma(sp.dt, fma(a1, k1.x, as * K.x), un.x), fma(sp.dt, fma(a1, k1.y, as * K.y), un.y));
                *reinterpret_cast<double2 *>(Ubuf + idx) = nxt;
                if (SC) nu[v] = nxt;
                if (sp.wmode)
                    *reinterpret_cast<double2 *>(Wb + idx) =
                        make_double2(fma(sp.dt, fma(sp.wb1, k1.x, sp.wbS1 * K.x), un.x),
                                     fma(sp.dt, fma(sp.wb1, k1.y, sp.wbS1 * K.y), un.y));
            }
        };
        // members in the launch's prefix that do not evaluate this stage (non-standard patterns) write nothing
        const bool writes = valid && (MODE == MODE_RHS || ((sp.actmask >> m) & 1u));
        const double J = -j2h;
        PERK_JITTER(6);
        __syncwarp();   // all primitives consumed: reuse sm[v][o] as the accumulator arrays
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            *reinterpret_cast<double2 *>(&sm[v][o][lo]) = make_double2(acc[0][v], acc[1][v]);
            *reinterpret_cast<double2 *>(&sm[v][o][lo + 2]) = make_double2(acc[2][v], acc[3][v]);
        }
        PERK_JITTER(7);
        __syncwarp();

        // phase 3: K = -(2/h) (x + y contributions), stage epilogue for nodes q0, q0+1
        if (writes) {
            const int i0 = q0 & 3, j0 = q0 >> 2;   // q0 + 1 has i0 + 1
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const double2 sx = *reinterpret_cast<const double2 *>(&sm[v][0][eox + q0]);
                const double s0 = sx.x + sm[v][1][yo + eoy + 4 * i0 + j0];
                const double s1 = sx.y + sm[v][1][yo + eoy + 4 * (i0 + 1) + j0];
                double2 K = make_double2(J * s0, J * s1);
                if (NS && BR1_DV && v > 0) {   // + the viscous volume term of k_grad2d (staged in the Gs slot)
                    const double2 d = *reinterpret_cast<const double2 *>(EP(EPI_GS) + (v - 1) * 16 + q0);
                    K = make_double2(K.x + d.x, K.y + d.y);
                }
                epilogue(v, q0, K);
            }
        }
        if (SC && MODE == MODE_STAGE && scp.epi && scp.alpha_fixed < 0.0 && sp.stage > 1 && sp.stage < sp.S) {
            // Hennemann-Gassner indicator of the next stage state just written (the blend factor the
            // next stage needs; k_sc_alpha skips these elements).  The element's 8 threads hold nodes
            // (i0, j0), (i0 + 1, j0): the modal transform runs as width-8 shuffles (warp-converged).
            const int i0 = q0 & 3, j0 = q0 >> 2, par = t8 & 1;
            double vq[2] = {1.0, 1.0};
            if (writes) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double r = h ? nu[0].y : nu[0].x, m1 = h ? nu[1].y : nu[1].x;
                    const double m2 = h ? nu[2].y : nu[2].x, En = h ? nu[3].y : nu[3].x;
                    const double ir = rcp64(r), v1 = m1 * ir, v2 = m2 * ir;
                    const double p = gm1 * (En - 0.5 * r * (v1 * v1 + v2 * v2));
                    vq[h] = scp.variable == 0 ? r : scp.variable == 1 ? p : scp.variable == 2 ? r * p
                          : scp.variable == 3 ? v1 : v2;
                }
            }
            const double o0 = __shfl_xor_sync(0xffffffffu, vq[0], 1, 8), o1 = __shfl_xor_sync(0xffffffffu, vq[1], 1, 8);
            const double row[4] = {par ? o0 : vq[0], par ? o1 : vq[1], par ? vq[0] : o0, par ? vq[1] : o1};
            double tk0 = 0.0, tk1 = 0.0;   // x transform of row j0, modes k = i0, i0 + 1
#pragma unroll
            for (int a = 0; a < NP; ++a) {
                tk0 = fma(sVv[i0 * NP + a], row[a], tk0);
                tk1 = fma(sVv[(i0 + 1) * NP + a], row[a], tk1);
            }
            double m0 = 0.0, m1 = 0.0;     // y transform: modes (i0, j0), (i0 + 1, j0)
#pragma unroll
            for (int b = 0; b < NP; ++b) {
                const double vb = sVv[j0 * NP + b];
                m0 = fma(vb, __shfl_sync(0xffffffffu, tk0, 2 * b + par, 8), m0);
                m1 = fma(vb, __shfl_sync(0xffffffffu, tk1, 2 * b + par, 8), m1);
            }
            const double mm0 = m0 * m0, mm1 = m1 * m1;
            double tot = mm0 + mm1;
            double c1 = (j0 <= NP - 2 ? (i0 <= NP - 2 ? mm0 : 0.0) + (i0 + 1 <= NP - 2 ? mm1 : 0.0) : 0.0);
            double c2 = (j0 <= NP - 3 ? (i0 <= NP - 3 ? mm0 : 0.0) + (i0 + 1 <= NP - 3 ? mm1 : 0.0) : 0.0);
#pragma unroll
            for (int off = 4; off > 0; off >>= 1) {
                tot += __shfl_xor_sync(0xffffffffu, tot, off, 8);
                c1 += __shfl_xor_sync(0xffffffffu, c1, off, 8);
                c2 += __shfl_xor_sync(0xffffffffu, c2, off, 8);
            }
            const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31, slot = nbuf + (lane >> 3);
            if (t8 == 0) {
                sTail[wi][0][slot] = tot;
                sTail[wi][1][slot] = c1;
                sTail[wi][2][slot] = c2;
                sTe[wi][slot] = writes ? e : -1;
            }
            nbuf += 4;
            if (nbuf == 16 || !has_next) {   // CTA-uniform
                __syncwarp();
                if (lane < nbuf && sTe[wi][lane] >= 0) {
                    const double T0 = sTail[wi][0][lane], T1 = sTail[wi][1][lane], T2 = sTail[wi][2][lane];
                    const double e1 = T0 > 0.0 ? (T0 - T1) / T0 : 0.0;
                    const double e2 = T1 > 0.0 ? (T1 - T2) / T1 : 0.0;
                    double a = 1.0 / (1.0 + exp(-scp.hg_sT * (fmax(e1, e2) - scp.hg_T)));
                    if (a < scp.alpha_min) a = 0.0;
                    else if (a > 1.0 - scp.alpha_min) a = 1.0;
                    a = fmin(a, scp.alpha_max);
                    alpha_raw[sTe[wi][lane]] = a;
                    alpha[sTe[wi][lane]] = a;
                }
                __syncwarp();
                nbuf = 0;
            }
        }
        __syncwarp();
        pk = pk_next;
    }
}

}  // namespace perk
