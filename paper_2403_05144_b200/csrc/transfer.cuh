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

// copy n rows (n read from device) of `row` doubles
__global__ void k_copy_rows(const int *__restrict__ n_ptr, int row, const double *__restrict__ src, double *__restrict__ dst)
{
    const size_t total = (size_t)(*n_ptr) * row;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
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

// one thread per (new element, variable, node); Uold is a copy of the pre-remesh state
__global__ void __launch_bounds__(256) k_transfer2d(MeshDev md, OldMesh om, int nv, const double *__restrict__ Uold,
                                                   double *__restrict__ Unew)
{
    const int npe = NP * NP;
    const size_t total = (size_t)md.n[0] * nv * npe;
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
        const int q = (int)(g % npe);
        const int v = (int)((g / npe) % nv);
        const int e = (int)(g / ((size_t)npe * nv));
        const int i = q % NP, j = q / NP;
        const int L = md.max_level, l = md.lev[e], s = 1 << (L - l);
        const int fx = md.fx[e], fy = md.fy[e];
        const int eo = om.cell_of[(size_t)fy * md.nfx + fx];
        const int lo = om.lev[eo];
        double out = 0.0;
        if (lo == l) {
            out = Uold[((size_t)eo * nv + v) * npe + q];
        } else if (lo == l - 1) {
            const int cx = ((fx - om.fx[eo]) / s) & 1, cy = ((fy - om.fy[eo]) / s) & 1;
            const double *ub = Uold + ((size_t)eo * nv + v) * npe;
#pragma unroll
            for (int l2 = 0; l2 < NP; ++l2) {
                const double py = cy ? cB.Pup[j][l2] : cB.Plo[j][l2];
                double row = 0.0;
#pragma unroll
                for (int k = 0; k < NP; ++k) row = fma(cx ? cB.Pup[i][k] : cB.Plo[i][k], ub[l2 * NP + k], row);
                out = fma(py, row, out);
            }
        } else if (lo == l + 1) {
            const int h = s >> 1;
            for (int cy = 0; cy < 2; ++cy)
                for (int cx = 0; cx < 2; ++cx) {
                    const int ec = om.cell_of[(size_t)(fy + cy * h) * md.nfx + fx + cx * h];
                    if (om.lev[ec] != l + 1) { atomicOr(md.err, ERR_TRANSFER); continue; }
                    const double *ub = Uold + ((size_t)ec * nv + v) * npe;
#pragma unroll
                    for (int l2 = 0; l2 < NP; ++l2) {
                        const double ry = cy ? cB.Rup[j][l2] : cB.Rlo[j][l2];
                        double row = 0.0;
#pragma unroll
                        for (int k = 0; k < NP; ++k) row = fma(cx ? cB.Rup[i][k] : cB.Rlo[i][k], ub[l2 * NP + k], row);
                        out = fma(ry, row, out);
                    }
                }
        } else {
            atomicOr(md.err, ERR_TRANSFER);
        }
        Unew[g] = out;
    }
}

}  // namespace perk
