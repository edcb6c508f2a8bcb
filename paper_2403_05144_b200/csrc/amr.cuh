// amr.cuh -- indicator-driven AMR on the device, 2D Euler / Navier-Stokes.
//
//   U (current mesh) --k_amr_indicator--> per-leaf indicator + wanted level (one level per adapt)
//   --k_amr_coarsen--> new level per leaf (a leaf coarsens only with its three siblings)
//   --k_amr_balance<true>, k_amr_balance<false> x L--> 2:1-balanced finest-grid level map
//
// The map is the input of perk_repartition: adapt + repartition run back to back on the context
// stream with the cell count kept on the device (no host round trip).  Indicators (DESIGN.md
// A1-A3): Hennemann-Gassner modal energy (cited at P:l.1548, l.1731, l.1886), Loehner's normalised
// second difference (cited at P:l.1440-1441), enstrophy 0.5 rho w.w (P:l.1615-1622, eq. Enstrophy);
// controller and balance: DESIGN.md A4-A6.
//
// Layout: one 16-lane group per element (lane q = i + 4 j owns node (i, j)), so the state loads are
// 128-byte coalesced rows of the [cell][var][node] layout, and the line operations (modal
// transform, second differences, derivatives) are shuffles inside the group.  The balance works on
// one base cell per CTA: the 4^L finest cells of a base cell are held in shared memory in Morton
// order, where every level-l block is a contiguous range, so the block maxima form a pyramid.
#pragma once
#include "common.cuh"
#include "mesh.cuh"

namespace perk {

enum { IND_HG = 0, IND_LOHNER = 1, IND_ENSTROPHY = 2 };

struct AmrParams {
    int indicator, variable;
    int base_level, med_level, max_level;
    double med_thr, max_thr;
    double alpha_max, alpha_min;   // Hennemann-Gassner
    double hg_T, hg_sT;            // threshold T = 0.5 10^(-1.8 (N+1)^(1/4)) and s / T (host-computed)
    double f_wave;                 // Loehner
};

constexpr int AMR_T = 256;         // threads per CTA of the per-element kernels (16 elements)

__device__ __forceinline__ double sum16(unsigned gm, double v)
{
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(gm, v, o, 16);
    return v;
}

__device__ __forceinline__ double max16(unsigned gm, double v)
{
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(gm, v, o, 16));
    return v;
}

__device__ __forceinline__ double lohner_est(double um, double u0, double up, double fw)
{
    const double num = fabs(up - 2.0 * u0 + um);
    const double den = fabs(up - u0) + fabs(u0 - um) + fw * (fabs(up) + 2.0 * fabs(u0) + fabs(um));
    return den > 0.0 ? num / den : 0.0;
}

// indicator of element e, computed by its 16-lane group; every lane returns the value
__device__ __forceinline__ double amr_element_indicator(const MeshDev &md, const AmrParams &ap,
                                                        const double *__restrict__ U, int e, unsigned gm, int q)
{
    const int i = q & 3, j = q >> 2;
    const double *u = U + (size_t)e * 4 * 16 + q;
    const double rho = __ldg(u), mx = __ldg(u + 16), my = __ldg(u + 32), En = __ldg(u + 48);
    const double vx = mx / rho, vy = my / rho;
    if (ap.indicator == IND_ENSTROPHY) {
        const double J = 2.0 / (md.hf * (double)(1 << (md.max_level - md.lev[e])));
        double dvydx = 0.0, dvxdy = 0.0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            dvydx = fma(cB.D[i][k], __shfl_sync(gm, vy, j * 4 + k, 16), dvydx);
            dvxdy = fma(cB.D[j][k], __shfl_sync(gm, vx, k * 4 + i, 16), dvxdy);
        }
        const double w = J * dvydx - J * dvxdy;
        return max16(gm, 0.5 * rho * w * w);
    }
    const double p = (md.gamma - 1.0) * (En - 0.5 * rho * (vx * vx + vy * vy));
    double val;
    switch (ap.variable) {
    case 0: val = rho; break;
    case 1: val = p; break;
    case 2: val = rho * p; break;
    case 3: val = vx; break;
    default: val = vy; break;
    }
    if (ap.indicator == IND_LOHNER) {
        // x lines: neighbours q -/+ 1; y lines: q -/+ 4 (clamped source lanes, used only inside)
        const double xm = __shfl_sync(gm, val, i > 0 ? q - 1 : q, 16);
        const double xp = __shfl_sync(gm, val, i < 3 ? q + 1 : q, 16);
        const double ym = __shfl_sync(gm, val, j > 0 ? q - 4 : q, 16);
        const double yp = __shfl_sync(gm, val, j < 3 ? q + 4 : q, 16);
        double est = 0.0;
        if (i == 1 || i == 2) est = lohner_est(xm, val, xp, ap.f_wave);
        if (j == 1 || j == 2) est = fmax(est, lohner_est(ym, val, yp, ap.f_wave));
        return max16(gm, est);
    }
    // Hennemann-Gassner: m_kl = sum_ij Vinv[k][i] Vinv[l][j] val_ij, lane (k, l) ends with m_kl
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < NP; ++a) t = fma(cB.Vinv[i][a], __shfl_sync(gm, val, j * 4 + a, 16), t);   // t_{k=i, j}
    double m = 0.0;
#pragma unroll
    for (int b = 0; b < NP; ++b) m = fma(cB.Vinv[j][b], __shfl_sync(gm, t, b * 4 + i, 16), m);     // m_{i, l=j}
    const double mm = m * m;
    const double tot = sum16(gm, mm);
    const double c1 = sum16(gm, (i <= NP - 2 && j <= NP - 2) ? mm : 0.0);
    const double c2 = sum16(gm, (i <= NP - 3 && j <= NP - 3) ? mm : 0.0);
    const double e1 = tot > 0.0 ? (tot - c1) / tot : 0.0;
    const double e2 = c1 > 0.0 ? (c1 - c2) / c1 : 0.0;
    const double E = fmax(e1, e2);
    double alpha = 1.0 / (1.0 + exp(-ap.hg_sT * (E - ap.hg_T)));
    if (alpha < ap.alpha_min) alpha = 0.0;
    else if (alpha > 1.0 - ap.alpha_min) alpha = 1.0;
    return fmin(alpha, ap.alpha_max);
}

// per leaf: indicator (ind may be null), controller target -> wanted level (one step toward it)
__global__ void __launch_bounds__(AMR_T) k_amr_indicator(MeshDev md, AmrParams ap, const double *__restrict__ U,
                                                         double *__restrict__ ind, uint8_t *__restrict__ want)
{
    const int q = threadIdx.x & 15;
    const unsigned gm = 0xffffu << (threadIdx.x & 16);
    const int n = md.n[0];
    const int per_cta = AMR_T / 16;
    for (int e = blockIdx.x * per_cta + (threadIdx.x >> 4); e < n; e += gridDim.x * per_cta) {
        const double v = amr_element_indicator(md, ap, U, e, gm, q);
        if (q == 0) {
            const int target = v <= ap.med_thr ? ap.base_level : (v <= ap.max_thr ? ap.med_level : ap.max_level);
            const int l = md.lev[e];
            want[e] = (uint8_t)(target > l ? l + 1 : (target < l ? l - 1 : l));
            if (ind) ind[e] = v;
        }
    }
}

// per leaf: new level; coarsening only if the 4 children of the parent are leaves that all want it
__global__ void k_amr_coarsen(MeshDev md, const uint8_t *__restrict__ want, uint8_t *__restrict__ newlev)
{
    const int n = md.n[0];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int l = md.lev[e], w = want[e];
        int nl = w;
        if (w < l) {
            const int s = 1 << (md.max_level - l);
            const int px = md.fx[e] & ~(2 * s - 1), py = md.fy[e] & ~(2 * s - 1);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = md.cell_of[(size_t)(py + (k >> 1) * s) * md.nfx + px + (k & 1) * s];
                if (md.lev[c] != l || want[c] >= l) nl = l;
            }
        }
        newlev[e] = (uint8_t)nl;
    }
}

__host__ __device__ inline size_t amr_balance_smem(int L)
{
    size_t tot = 0;
    for (int l = 0; l <= L; ++l) tot += (size_t)1 << (2 * l);
    return tot;
}

// one balance iteration on one base cell (blockIdx.x = base cell, x fastest):
//   T(c) = max(M(c), max over the 4 face neighbours M(n) - 1)          (the 2:1 requirement)
//   M'(c) = min { l : max of T over the level-l block holding c <= l }   (smallest valid tree >= T)
// FIRST: M(c) = newlev[leaf of c] (rasterisation of the controller's decision).  L + 1 iterations
// reach the fixed point: cells raised in iteration k get levels <= L - k (A6).
template <bool FIRST>
__global__ void __launch_bounds__(AMR_T) k_amr_balance(MeshDev md, const uint8_t *__restrict__ newlev,
                                                       const uint8_t *__restrict__ Min, uint8_t *__restrict__ Mout)
{
    extern __shared__ uint8_t pyr[];            // level l block maxima at offset (4^l - 1) / 3
    const int L = md.max_level, side = 1 << L, ncell = side * side;
    const int nbx = md.nfx >> L;
    const int bx = blockIdx.x % nbx, by = blockIdx.x / nbx;
    auto M = [&](int x, int y) -> int {
        const size_t c = (size_t)y * md.nfx + x;
        return FIRST ? newlev[md.cell_of[c]] : Min[c];
    };
    uint8_t *T = pyr + (((size_t)1 << (2 * L)) - 1) / 3;
    for (int m = threadIdx.x; m < ncell; m += blockDim.x) {
        const int x = bx * side + (int)compact_bits((unsigned long long)m);
        const int y = by * side + (int)compact_bits((unsigned long long)m >> 1);
        int t = M(x, y);
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            int nx = x + (d == 0) - (d == 1), ny = y + (d == 2) - (d == 3);
            if (nx < 0 || nx >= md.nfx) { if (!md.periodic[0]) continue; nx = wrapi(nx, md.nfx); }
            if (ny < 0 || ny >= md.nfy) { if (!md.periodic[1]) continue; ny = wrapi(ny, md.nfy); }
            t = max(t, M(nx, ny) - 1);
        }
        T[m] = (uint8_t)t;
    }
    __syncthreads();
    for (int l = L - 1; l >= 0; --l) {
        uint8_t *P = pyr + (((size_t)1 << (2 * l)) - 1) / 3;
        const uint8_t *C = pyr + (((size_t)1 << (2 * (l + 1))) - 1) / 3;
        for (int b = threadIdx.x; b < (1 << (2 * l)); b += blockDim.x)
            P[b] = max(max(C[4 * b], C[4 * b + 1]), max(C[4 * b + 2], C[4 * b + 3]));
        __syncthreads();
    }
    for (int m = threadIdx.x; m < ncell; m += blockDim.x) {
        int lv = L;
        for (int l = 0; l < L; ++l)
            if (pyr[(((size_t)1 << (2 * l)) - 1) / 3 + (m >> (2 * (L - l)))] <= l) { lv = l; break; }
        const int x = bx * side + (int)compact_bits((unsigned long long)m);
        const int y = by * side + (int)compact_bits((unsigned long long)m >> 1);
        Mout[(size_t)y * md.nfx + x] = (uint8_t)lv;
    }
}

}  // namespace perk
