// transfer.cuh -- solution transfer on re-mesh, 2D, N = 3.
// A new leaf with the same level as the old leaf at its origin copies it; one level finer
// (refined) interpolates the parent polynomial at its own LGL nodes (P_lower / P_upper per
// direction); one level coarser (coarsened) is the exact L2 projection of its 4 children
// (R_lower / R_upper per direction).  |level change| > 1 latches ERR_TRANSFER.
#pragma once
#include "common.cuh"

namespace perk {

struct OldMesh {
    const int *n_old;
    const int *cell_of;
    const uint8_t *lev;
    const int *fx, *fy;
};

// copy n rows (n read from device) of `row` doubles (row even: 16 B vectors)
__global__ void k_copy_rows(const int *__restrict__ n_ptr, int row, const double *__restrict__ src, double *__restrict__ dst)
{
    const int total = (*n_ptr) * (row / 2);                     // < 2^24 * 32
    const double2 *s2 = reinterpret_cast<const double2 *>(src);
    double2 *d2 = reinterpret_cast<double2 *>(dst);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) d2[i] = __ldg(s2 + i);
}

__global__ void k_save_old(MeshDev md, int *n_old, int *cell_of_old, uint8_t *lev_old, int *fx_old, int *fy_old)
{
    const size_t nf = (size_t)md.nfx * md.nfy;
    const int n = md.n[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_old = n;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += (size_t)gridDim.x * blockDim.x) {
        cell_of_old[i] = md.cell_of[i];
        if (i < (size_t)n) {
            lev_old[i] = md.lev[i];
            fx_old[i] = md.fx[i];
            fy_old[i] = md.fy[i];
        }
    }
}

// One 16-lane group per new element (lane = node q = i + 4 j, all 4 variables): every source block
// (the old leaf, its parent, or each of its 4 children) is read once with coalesced 128 B rows into
// the group's shared-memory slot, and the tensor-product operators (P_lower / P_upper, R_lower /
// R_upper, held in shared memory because lane-dependent indices into __constant__ tables
// serialise) are applied from there.  Uold is a copy of the pre-remesh state; 2D states have nv = 4.
__global__ void __launch_bounds__(256) k_transfer2d(MeshDev md, OldMesh om, int nv, const double *__restrict__ Uold,
                                                   double *__restrict__ Unew)
{
    __shared__ double Pm[4][NP][NP];          // Plo, Pup, Rlo, Rup
    __shared__ __align__(16) double blk[16][64];   // per group: one source block [var][node]
    for (int t = threadIdx.x; t < 4 * NP * NP; t += blockDim.x) {
        const int m = t / (NP * NP), r = (t / NP) % NP, k = t % NP;
        Pm[m][r][k] = m == 0 ? cB.Plo[r][k] : (m == 1 ? cB.Pup[r][k] : (m == 2 ? cB.Rlo[r][k] : cB.Rup[r][k]));
    }
    __syncthreads();
    const int npe = NP * NP;
    const int q = threadIdx.x & 15, i = q % NP, j = q / NP, g = threadIdx.x >> 4;
    const unsigned gm = 0xffffu << (threadIdx.x & 16);
    double *B = blk[g];
    const int n = md.n[0];
    const int per_cta = blockDim.x / 16;
    // out[v] += (Ry (x) Rx) applied to the block in B, at this lane's node
    auto apply = [&](const double (*Mx)[NP], const double (*My)[NP], double out[4]) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            double o = out[v];
#pragma unroll
            for (int l2 = 0; l2 < NP; ++l2) {
                double row = 0.0;
#pragma unroll
                for (int k = 0; k < NP; ++k) row = fma(Mx[i][k], B[v * 16 + l2 * NP + k], row);
                o = fma(My[j][l2], row, o);
            }
            out[v] = o;
        }
    };
    auto stage = [&](int src) {
        __syncwarp(gm);                    // the group is done with the previous block
#pragma unroll
        for (int v = 0; v < 4; ++v) B[v * 16 + q] = __ldg(Uold + ((size_t)src * 4 + v) * npe + q);
        __syncwarp(gm);
    };
    for (int e = blockIdx.x * per_cta + g; e < n; e += gridDim.x * per_cta) {
        const int L = md.max_level, l = md.lev[e], s = 1 << (L - l);
        const int fx = md.fx[e], fy = md.fy[e];
        const int eo = om.cell_of[(size_t)fy * md.nfx + fx];
        if (eo < 0) { atomicOr(md.err, ERR_CAPACITY); continue; }   // the old mesh had overflowed
        PERK_DASSERT(eo >= 0 && eo < *om.n_old);
        const int lo = om.lev[eo];
        double out[4] = {0.0, 0.0, 0.0, 0.0};
        if (lo == l) {
#pragma unroll
            for (int v = 0; v < 4; ++v) out[v] = __ldg(Uold + ((size_t)eo * 4 + v) * npe + q);
        } else if (lo == l - 1) {
            const int cx = ((fx - om.fx[eo]) / s) & 1, cy = ((fy - om.fy[eo]) / s) & 1;
            stage(eo);
            apply(Pm[cx], Pm[cy], out);
        } else if (lo == l + 1) {
            const int h = s >> 1;
            for (int c = 0; c < 4; ++c) {
                const int cx = c & 1, cy = c >> 1;
                const int ec = om.cell_of[(size_t)(fy + cy * h) * md.nfx + fx + cx * h];
                if (ec < 0) { atomicOr(md.err, ERR_CAPACITY); continue; }
                PERK_DASSERT(ec >= 0 && ec < *om.n_old);
                if (om.lev[ec] != l + 1) { atomicOr(md.err, ERR_TRANSFER); continue; }
                stage(ec);
                apply(Pm[2 + cx], Pm[2 + cy], out);
            }
        } else {
            atomicOr(md.err, ERR_TRANSFER);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) Unew[((size_t)e * 4 + v) * npe + q] = out[v];
    }
}

}  // namespace perk
