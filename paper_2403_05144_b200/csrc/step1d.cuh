// step1d.cuh -- a whole P-ERK step of a small 1D mesh in ONE single-CTA launch (BASELINE cfg 1/2:
// 48 / 352 cells, SURVEY §7 "tiny configs are latency-bound").
//
// The state (U_n, K_1, the stage buffer, the current K and the face fluxes; W for P-ERK3) lives in
// shared memory for the whole step; the S stages are separated by __syncthreads instead of kernel
// boundaries.  Per stage the threads loop over the ACTIVE prefixes only (interfaces, boundaries, then
// element nodes), so a stage costs ceil(active / blockDim) passes: the multirate saving shows up in
// wall time, which it cannot with two ~3 us launches per stage.  Same arithmetic as k_surf1d /
// k_vol1d (weak form, upwind / Rusanov, lazy first-order states, fused stage combination).
#pragma once
#include "dg1d.cuh"

namespace perk {

struct StepTab1D {
    int S, R;
    unsigned actmask[MAXS];      // stage i (index i-1): members evaluating it
    unsigned bufmask[MAXS];      // stage i: members whose stage state is in the stage buffer
    double c[MAXS];
    double b1, bS1, bS;          // shared weights at stages 1, S-1, S
    double a1n[MAXR][MAXS];      // after evaluating stage i (index i-1): a_{n,1}^{(r)} of the next
    double asubn[MAXR][MAXS];    // evaluated stage n, and a_{n,i}^{(r)} (standard pattern: n = i+1)
};

// threads per CTA: the per-stage cost is ceil(active / blockDim) dependent passes; measured best
// (B200, mesh data staged in shared memory): 256 for advection (cfg 1: 0.0205 ms/step; 512 the same,
// 128 0.024), 1024 for Euler (cfg 2: 0.0655 ms/step; 512 0.0676, 256 0.086)
#ifndef STEP1D_T1
#define STEP1D_T1 256
#endif
#ifndef STEP1D_T3
#define STEP1D_T3 1024
#endif
__host__ __device__ constexpr int step1d_threads(int nv) { return nv == 1 ? STEP1D_T1 : STEP1D_T3; }

// state (U_n, K_1, stage buffer, K_i, W) + face fluxes, then the step's read-only mesh data staged once
// per step so the per-stage loops never wait on global memory: 2/h per element, interface pairs packed
// with their members (list order, <= n), boundaries (<= 2), the element list packed with the members
__host__ __device__ inline size_t step1d_smem_bytes(int n, int nv, bool use_w)
{
    return sizeof(double) * ((size_t)n * nv * NP * (use_w ? 4 : 3) + (size_t)n * 2 * nv + (size_t)n) +
           (size_t)n * 8 + 16 + (size_t)n * 4;
}

template <int NV>
__global__ void __launch_bounds__(step1d_threads(NV)) k_step1d(MeshDev md, const StepTab1D *__restrict__ tb,
                                                            double *__restrict__ U, double dt, int use_w)
{
    extern __shared__ __align__(16) double sh[];
    __shared__ StepTab1D T;
    __shared__ int sCnt[3][MAXS];   // active interfaces / boundaries / elements per stage (no global load per stage)
    __shared__ double sD[NP][NP];   // Dhat: row j = the node's lane-dependent index (__constant__ reads would serialise)
    const int n = md.n[0];
    const int rowd = NV * NP;
    double *sUn = sh, *sK1 = sUn + (size_t)n * rowd, *sUb = sK1 + (size_t)n * rowd;
    double *sW = sUb + (size_t)n * rowd;
    double *sFs = use_w ? sW + (size_t)n * rowd : sW;
    double *sJ = sFs + (size_t)n * 2 * NV;                       // 2 / h per element (no division per stage)
    int2 *sIf = reinterpret_cast<int2 *>(sJ + n);                // interface sides packed with their members
    int2 *sBd = sIf + n;
    int *sEl = reinterpret_cast<int *>(sBd + 2);                 // element list packed with the members
    const int tid = threadIdx.x, nt = blockDim.x;
    {
        const int *src = reinterpret_cast<const int *>(tb);
        int *dst = reinterpret_cast<int *>(&T);
        for (int k = tid; k < (int)(sizeof(StepTab1D) / sizeof(int)); k += nt) dst[k] = src[k];
    }
    for (int k = tid; k < n * rowd; k += nt) sUn[k] = U[k];
    {
        const int nif_all = md.n[1], nbd_all = md.n[3];
        for (int k = tid; k < nif_all; k += nt) {
            const int4 I = md.ifcs[k];
            PERK_DASSERT(I.x >= 0 && I.x < n && I.y >= 0 && I.y < n);
            sIf[k] = make_int2(I.x | ((int)md.mem[I.x] << PK_EBITS), I.y | ((int)md.mem[I.y] << PK_EBITS));
        }
        for (int k = tid; k < nbd_all && k < 2; k += nt) sBd[k] = md.bnd[md.list[KIND_BD][k]];
        if (tid < NP * NP) sD[tid / NP][tid % NP] = cB.Dhat[tid / NP][tid % NP];
        for (int k = tid; k < 3 * MAXS; k += nt) {
            const int kind = k / MAXS == 0 ? KIND_IF : (k / MAXS == 1 ? KIND_BD : KIND_EL);
            sCnt[k / MAXS][k % MAXS] = md.count_active[kind * MAXS + k % MAXS];
        }
        for (int k = tid; k < n; k += nt) {
            const int e = md.list[KIND_EL][k];
            sEl[k] = e | ((int)md.mem[e] << PK_EBITS);
            sJ[k] = 2.0 / (md.hf * (double)(1 << (md.max_level - md.lev[k])));
        }
    }
    __syncthreads();
    const int S = T.S;
    for (int i = 1; i <= S; ++i) {
        const int nif = sCnt[0][i - 1], nbd = sCnt[1][i - 1], nel = sCnt[2][i - 1];
        const double dtc = dt * T.c[i - 1];
        const unsigned bufm = T.bufmask[i - 1];
        // the stage-i state of element e (member m), variable v, node j (SURVEY §7 rule)
        auto state = [&](int e, int m, int v, int j) {
            const size_t x = ((size_t)e * NV + v) * NP + j;
            if (i == 1) return sUn[x];
            if ((bufm >> m) & 1u) return sUb[x];
            return fma(dtc, sK1[x], sUn[x]);
        };
        // surface fluxes over the active interfaces and boundaries
        for (int t = tid; t < nif + nbd; t += nt) {
            double uL[NV], uR[NV], f[NV];
            if (t < nif) {
                const int2 I = sIf[t];
                const int eL = pk_elem(I.x), eR = pk_elem(I.y), mL = I.x >> PK_EBITS, mR = I.y >> PK_EBITS;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    uL[v] = state(eL, mL, v, NP - 1);
                    uR[v] = state(eR, mR, v, 0);
                }
                numflux1d<NV>(uL, uR, md.gamma, md.adv, f);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    sFs[((size_t)eL * 2 + 0) * NV + v] = f[v];
                    sFs[((size_t)eR * 2 + 1) * NV + v] = f[v];
                }
            } else {
                const int2 B = sBd[t - nif];
                const int face = B.y & 7;
                double u[NV], gst[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    u[v] = state(B.x, B.y >> 8, v, face == 0 ? NP - 1 : 0);
                    gst[v] = md.bc[v];
                }
                if (face == 0) numflux1d<NV>(u, gst, md.gamma, md.adv, f);
                else numflux1d<NV>(gst, u, md.gamma, md.adv, f);
#pragma unroll
                for (int v = 0; v < NV; ++v) sFs[((size_t)B.x * 2 + face) * NV + v] = f[v];
            }
        }
        __syncthreads();
        // K_i at the active element nodes (one thread per node; an element's 4 node threads are
        // consecutive lanes of one warp) and, once the element's stage state has been read by all
        // four (__syncwarp), the stage combination from registers; surplus members of the prefix skip
        const unsigned act = T.actmask[i - 1];
        const int tot = NP * nel;
        for (int t0 = 0; t0 < tot; t0 += nt) {
            const int t = t0 + tid;
            bool on = t < tot;
            int e = 0, j = 0, m = 0;
            if (on) {
                const int pe = sEl[t / NP];
                e = pk_elem(pe);
                j = t % NP;
                m = pe >> PK_EBITS;
                on = (act >> m) & 1u;
            }
            double K[NV];
            if (on) {
                double f[NP][NV];
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    double u[NV];
#pragma unroll
                    for (int v = 0; v < NV; ++v) u[v] = state(e, m, v, k);
                    phys_flux1d<NV>(u, md.gamma, md.adv, f[k]);
                }
                const double J = sJ[e];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < NP; ++k) s = fma(sD[j][k], f[k][v], s);
                    if (j == 0) s = fma(sFs[((size_t)e * 2 + 1) * NV + v], cB.invw[0], s);
                    if (j == NP - 1) s = fma(-sFs[((size_t)e * 2 + 0) * NV + v], cB.invw[NP - 1], s);
                    K[v] = J * s;
                }
            }
            __syncwarp();
            if (on) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const size_t x = ((size_t)e * NV + v) * NP + j;
                    if (i == 1) {
                        sK1[x] = K[v];
                    } else if (i == S) {
                        if (!use_w && T.b1 != 0.0) sUn[x] = fma(dt, fma(T.b1, sK1[x], T.bS * K[v]), sUn[x]);   // Heun / Ralston
                        else sUn[x] = fma(dt * T.bS, K[v], use_w ? sW[x] : sUn[x]);
                    } else {
                        const double un = sUn[x], k1 = sK1[x];
                        sUb[x] = fma(dt, fma(T.a1n[m][i - 1], k1, T.asubn[m][i - 1] * K[v]), un);   // next evaluated stage
                        if (use_w && i == S - 1) sW[x] = fma(dt, fma(T.b1, k1, T.bS1 * K[v]), un);
                    }
                }
            }
        }
        __syncthreads();
    }
    for (int k = tid; k < n * rowd; k += nt) U[k] = sUn[k];
    if (tid == 0) {
        atomicAdd(md.evals, md.evals[2]);
        atomicAdd(md.evals + 1, 1ull);
    }
}

}  // namespace perk
