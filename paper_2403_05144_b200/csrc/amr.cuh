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

// indicator of element e (level lev), computed by its 16-lane group from the node's conserved state
// (rho, mx, my, En); every lane returns the value
// Ri / Rj: row i and row j (i = q & 3, j = q >> 2) of D (enstrophy) or of Vinv (Hennemann-Gassner),
// held in registers: lane-dependent indices into __constant__ tables would serialise
template <int IND>
__device__ __forceinline__ double amr_element_indicator(const MeshDev &md, const AmrParams &ap, int lev,
                                                        double rho, double mx, double my, double En,
                                                        const double (&Ri)[NP], const double (&Rj)[NP],
                                                        unsigned gm, int q)
{
    const int i = q & 3, j = q >> 2;
    const double irho = rcp64(rho);
    const double vx = mx * irho, vy = my * irho;
    if (IND == IND_ENSTROPHY) {
        const double J = 2.0 / (md.hf * (double)(1 << (md.max_level - lev)));
        double dvydx = 0.0, dvxdy = 0.0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            dvydx = fma(Ri[k], __shfl_sync(gm, vy, j * 4 + k, 16), dvydx);
            dvxdy = fma(Rj[k], __shfl_sync(gm, vx, k * 4 + i, 16), dvxdy);
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
    if (IND == IND_LOHNER) {
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
    for (int a = 0; a < NP; ++a) t = fma(Ri[a], __shfl_sync(gm, val, j * 4 + a, 16), t);   // t_{k=i, j}
    double m = 0.0;
#pragma unroll
    for (int b = 0; b < NP; ++b) m = fma(Rj[b], __shfl_sync(gm, t, b * 4 + i, 16), m);     // m_{i, l=j}
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

// per leaf: indicator (ind may be null), controller target -> wanted level (one step toward it).
// Persistent grid over tiles of AMR_TILE consecutive elements: a tile is one contiguous 8 KB block of
// U, fetched by one bulk copy (TMA engine) into a 3-stage shared-memory ring, so each SM keeps up to
// 4 CTAs x 3 x 8 KB of HBM reads in flight while the 16-lane groups (one element each) work on the
// oldest stage.
constexpr int AMR_TILE = AMR_T / 16;
constexpr int AMR_STAGES = 3;

template <int IND>
__global__ void __launch_bounds__(AMR_T) k_amr_indicator(MeshDev md, AmrParams ap, const double *__restrict__ U,
                                                         double *__restrict__ ind, uint8_t *__restrict__ want)
{
    __shared__ __align__(128) double tile[AMR_STAGES][AMR_TILE * 64];
    __shared__ __align__(8) unsigned long long bar[AMR_STAGES];
    const int q = threadIdx.x & 15, g = threadIdx.x >> 4;
    // the shuffles run warp-converged with the full mask (width 16 keeps them inside each group):
    // a partial mask in divergent code would compile to WARPSYNC / collective loops
    const unsigned gm = 0xffffffffu;
    double Ri[NP], Rj[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        Ri[k] = IND == IND_HG ? cB.Vinv[q & 3][k] : (IND == IND_ENSTROPHY ? cB.D[q & 3][k] : 0.0);
        Rj[k] = IND == IND_HG ? cB.Vinv[q >> 2][k] : (IND == IND_ENSTROPHY ? cB.D[q >> 2][k] : 0.0);
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < AMR_STAGES; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();
    const int n = md.n[0];
    const int ntiles = (n + AMR_TILE - 1) / AMR_TILE;
    auto issue = [&](int t, int s) {
        const int e0 = t * AMR_TILE;
        const unsigned bytes = (unsigned)min(AMR_TILE, n - e0) * 64u * 8u;
        mbar_arrive_expect_tx(&bar[s], bytes);
        bulk_g2s(tile[s], U + (size_t)e0 * 64, bytes, &bar[s]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < AMR_STAGES; ++s) {
            const int t = blockIdx.x + s * gridDim.x;
            if (t < ntiles) issue(t, s);
        }
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % AMR_STAGES;
        const int e = t * AMR_TILE + g;
        const int l = e < n ? md.lev[e] : 0;
        mbar_wait(&bar[s], (unsigned)(k / AMR_STAGES) & 1u);
        {
            // groups past the last element compute on stale tile data and store nothing
            const double *u = tile[s] + g * 64 + q;
            const double v = amr_element_indicator<IND>(md, ap, l, u[0], u[16], u[32], u[48], Ri, Rj, gm, q);
            if (q == 0 && e < n) {
                const int target = v <= ap.med_thr ? ap.base_level : (v <= ap.max_thr ? ap.med_level : ap.max_level);
                want[e] = (uint8_t)(target > l ? l + 1 : (target < l ? l - 1 : l));
                if (ind) ind[e] = v;
            }
        }
        __syncthreads();                                // stage s consumed by every group
        if (threadIdx.x == 0) {
            const int tn = t + AMR_STAGES * gridDim.x;
            if (tn < ntiles) {
                fence_proxy_async_smem();
                issue(tn, s);
            }
        }
    }
}

// per leaf: new level; coarsening only if the 4 children of the parent are leaves that all want it
__global__ void k_amr_coarsen(MeshDev md, const uint8_t *__restrict__ want, uint8_t *__restrict__ newlev)
{
    pdl_wait();
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
                PERK_DASSERT(c >= 0 && c < md.n[0]);
                if (md.lev[c] != l || want[c] >= l) nl = l;
            }
        }
        newlev[e] = (uint8_t)nl;
    }
}

// per base cell, the block maxima of levels 0..L-1: level l at offset (4^l - 1) / 3
__host__ __device__ inline int amr_pyramid_bytes(int L) { return ((1 << (2 * L)) - 1) / 3; }

// base cells per balance CTA (L >= 1): one 2x2 quad of finest cells per thread
__host__ __device__ inline int amr_base_per_cta(int L)
{
    const int qpb = 1 << (2 * (L - 1));            // quads per base cell
    return qpb >= AMR_T ? 1 : AMR_T / qpb;
}

__device__ __forceinline__ unsigned compact16(unsigned m)   // even bits of m (< 2^16 used) -> low bits
{
    m &= 0x55555555u;
    m = (m | (m >> 1)) & 0x33333333u;
    m = (m | (m >> 2)) & 0x0f0f0f0fu;
    m = (m | (m >> 4)) & 0x00ff00ffu;
    m = (m | (m >> 8)) & 0x0000ffffu;
    return m;
}

// one balance iteration (max_level L >= 1); each CTA owns amr_base_per_cta(L) consecutive base cells
// (row-major base grid), each thread one 2x2 quad (4 Morton-consecutive finest cells):
//   T(c) = max(M(c), max over the 4 face neighbours M(n) - 1)          (the 2:1 requirement)
//   M'(c) = min { l : max of T over the level-l block holding c <= l }   (smallest valid tree >= T)
// The quad's maximum is its level-(L-1) block maximum (the base of the shared-memory pyramid), and
// the quad's four cells share one answer.
// FIRST: M(c) = newlev[leaf of c] (rasterisation of the controller's decision).  L + 1 iterations
// reach the fixed point: cells raised in iteration k get levels <= L - k (A6).
//
// flags[k] (k = 1..L) records whether iteration k changed any cell; iteration k >= 2 whose
// predecessor changed nothing has reached the fixed point and only copies Min to Mout.
template <bool FIRST>
__global__ void __launch_bounds__(AMR_T) k_amr_balance(MeshDev md, const uint8_t *__restrict__ newlev,
                                                       const uint8_t *__restrict__ Min, uint8_t *__restrict__ Mout,
                                                       int *__restrict__ flags, int it)
{
    pdl_wait();
    extern __shared__ uint8_t pyr_all[];
    if (FIRST) {
        if (blockIdx.x == 0 && threadIdx.x <= md.max_level) flags[threadIdx.x] = 0;
    } else if (it >= 2 && flags[it - 1] == 0) {
        const size_t nvec = (size_t)md.nfx * md.nfy / 16;
        if (((size_t)md.nfx * md.nfy) % 16 == 0 && (((uintptr_t)Min | (uintptr_t)Mout) & 15) == 0) {
            const uint4 *src = reinterpret_cast<const uint4 *>(Min);
            uint4 *dst = reinterpret_cast<uint4 *>(Mout);
            for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < nvec; k += (size_t)gridDim.x * blockDim.x)
                dst[k] = src[k];
        } else {
            for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < (size_t)md.nfx * md.nfy;
                 k += (size_t)gridDim.x * blockDim.x)
                Mout[k] = Min[k];
        }
        return;
    }
    const int L = md.max_level, side = 1 << L, nfx = md.nfx, nfy = md.nfy;
    const int nbx = nfx >> L, nbase = nbx * (nfy >> L);
    const int bpc = amr_base_per_cta(L);
    const int b0 = blockIdx.x * bpc;
    const int nb = min(bpc, nbase - b0);
    const int qsh = 2 * (L - 1), qpb = 1 << qsh;   // quads per base cell
    const int psz = amr_pyramid_bytes(L);
    const bool px = md.periodic[0], py = md.periodic[1];
    auto M = [&](int x, int y) -> int {
        const size_t c = (size_t)y * nfx + x;
        return FIRST ? newlev[md.cell_of[c]] : Min[c];
    };
    // neighbour value, or -1 outside a non-periodic domain (never raises T)
    auto Mn = [&](int x, int y) -> int {
        if (x < 0) { if (!px) return -1; x += nfx; }
        if (x >= nfx) { if (!px) return -1; x -= nfx; }
        if (y < 0) { if (!py) return -1; y += nfy; }
        if (y >= nfy) { if (!py) return -1; y -= nfy; }
        return M(x, y);
    };
    const int nq = nb * qpb;
    const int offq = ((1 << qsh) - 1) / 3;         // pyramid offset of level L-1 (one entry per quad)
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
        const int b = b0 + (q >> qsh), mq = q & (qpb - 1);
        const int x0 = (b % nbx) * side + 2 * (int)compact16((unsigned)mq);
        const int y0 = (b / nbx) * side + 2 * (int)compact16((unsigned)mq >> 1);
        const int a00 = M(x0, y0), a10 = M(x0 + 1, y0), a01 = M(x0, y0 + 1), a11 = M(x0 + 1, y0 + 1);
        const int t0 = max(a00, max(max(a10, a01), max(Mn(x0 - 1, y0), Mn(x0, y0 - 1))) - 1);
        const int t1 = max(a10, max(max(a00, a11), max(Mn(x0 + 2, y0), Mn(x0 + 1, y0 - 1))) - 1);
        const int t2 = max(a01, max(max(a11, a00), max(Mn(x0 - 1, y0 + 1), Mn(x0, y0 + 2))) - 1);
        const int t3 = max(a11, max(max(a01, a10), max(Mn(x0 + 2, y0 + 1), Mn(x0 + 1, y0 + 2))) - 1);
        pyr_all[(q >> qsh) * psz + offq + mq] = (uint8_t)max(max(t0, t1), max(t2, t3));
    }
    __syncthreads();
    for (int l = L - 2; l >= 0; --l) {
        const int offl = ((1 << (2 * l)) - 1) / 3, offc = ((1 << (2 * (l + 1))) - 1) / 3;
        const int per = 1 << (2 * l);
        for (int k = threadIdx.x; k < nb * per; k += blockDim.x) {
            uint8_t *P = pyr_all + (k >> (2 * l)) * psz;
            const int bb = k & (per - 1);
            const uint8_t *C = P + offc + 4 * bb;
            P[offl + bb] = max(max(C[0], C[1]), max(C[2], C[3]));
        }
        __syncthreads();
    }
    int changed = 0;
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
        const int b = b0 + (q >> qsh), mq = q & (qpb - 1);
        const int x0 = (b % nbx) * side + 2 * (int)compact16((unsigned)mq);
        const int y0 = (b / nbx) * side + 2 * (int)compact16((unsigned)mq >> 1);
        const uint8_t *P = pyr_all + (q >> qsh) * psz;
        // the four cells share every block of level <= L-1; at level L each cell is its own block,
        // where max T = T(c) <= L always holds
        int lq = L;
        for (int l = 0; l <= L - 1; ++l)
            if (P[((1 << (2 * l)) - 1) / 3 + (mq >> (2 * (L - 1 - l)))] <= l) { lq = l; break; }
        const uint8_t o = (uint8_t)lq;
        if (!FIRST) {
            const uchar2 r0 = *reinterpret_cast<const uchar2 *>(Min + (size_t)y0 * nfx + x0);
            const uchar2 r1 = *reinterpret_cast<const uchar2 *>(Min + (size_t)(y0 + 1) * nfx + x0);
            changed |= (r0.x != o) | (r0.y != o) | (r1.x != o) | (r1.y != o);
        }
        *reinterpret_cast<uchar2 *>(Mout + (size_t)y0 * nfx + x0) = make_uchar2(o, o);
        *reinterpret_cast<uchar2 *>(Mout + (size_t)(y0 + 1) * nfx + x0) = make_uchar2(o, o);
    }
    if (!FIRST && __syncthreads_or(changed) && threadIdx.x == 0) atomicOr(flags + it, 1);
}

}  // namespace perk
