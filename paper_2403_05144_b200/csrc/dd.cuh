// dd.cuh -- spatial domain decomposition of the P-ERK step over ranks.
//
// The paper partitions the ODE system by refinement level only and notes that the per-partition
// lists are local, so "no additional data exchange is required compared to standard Runge-Kutta
// methods" (P:l.1258-1263, §6.3).  Across GPUs the mesh is split into contiguous Morton ranges of
// leaves; a leaf's work per step is E_r (the stage evaluations of its member), so the ranges are
// balanced in sum_leaves E_member (an equal-cell split is unbalanced under multirate):
//
//   w_k = E[member(k)],  W = sum_k w_k,  owner(k) = min(P - 1, floor(P (2 prefix_k + w_k) / (2 W)))
//
// (prefix_k = sum_{j<k} w_j, the midpoint rule; monotone in k, so every rank owns a contiguous range
// of cells).  Every rank builds the same global mesh on its device (cheap: a1-a3 are list rebuilds),
// then keeps the elements it owns and the faces with an owned side; the cells across those faces are
// its ghosts.  Per stage the owner sends the blocks its stage-i volume epilogue wrote (K_1 at stage 1,
// the next stage state at 1 < i < S, U_{n+1} at stage S) for the active cells on another rank's
// ghost layer, and, for Navier-Stokes, the normal viscous-flux traces Vt after the gradient pass.
// Face fluxes of faces between two ranks are computed by both with identical inputs, so every
// owned cell's result is bitwise the single-domain one.
#pragma once
#include "common.cuh"
#include "partition.cuh"

namespace perk {

constexpr int DD_MAXP = 8;          // ranks per decomposition (one node)
constexpr int DD_SCAN_T = 1024;

// per-leaf weight E[member] and per-block sums
__global__ void __launch_bounds__(DD_SCAN_T) k_dd_block_sums(MeshDev md, ActiveDesc ad, long long *bsum)
{
    __shared__ int wsum[32];
    const int n = md.n[0];
    const int k = blockIdx.x * DD_SCAN_T + threadIdx.x;
    const int w = k < n ? ad.E[md.mem[k]] : 0;
    int tot;
    block_incl_scan(w, wsum, tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// one block: exclusive scan of the block sums (in place) and the total W in bsum[nblocks]
__global__ void __launch_bounds__(DD_SCAN_T) k_dd_scan_blocks(const int *n_ptr, long long *bsum)
{
    __shared__ long long part[DD_SCAN_T];
    const int nb = (*n_ptr + DD_SCAN_T - 1) / DD_SCAN_T;
    long long base = 0;
    for (int c = 0; c < nb; c += DD_SCAN_T) {
        const int b = c + threadIdx.x;
        const long long v = b < nb ? bsum[b] : 0;
        part[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < DD_SCAN_T; o <<= 1) {      // Hillis-Steele (64-bit, few thousand blocks)
            const long long y = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
            __syncthreads();
            part[threadIdx.x] += y;
            __syncthreads();
        }
        if (b < nb) bsum[b] = base + part[threadIdx.x] - v;
        base += part[DD_SCAN_T - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nb] = base;
}

// owner of every leaf; owned range [first, first + count) in range[0..1] (range preset to {n, 0})
__global__ void __launch_bounds__(DD_SCAN_T) k_dd_owner(MeshDev md, ActiveDesc ad, const long long *bsum, int P,
                                                     int rank, uint8_t *owner, int *range)
{
    __shared__ int wsum[32];
    const int n = md.n[0];
    const int nb = (n + DD_SCAN_T - 1) / DD_SCAN_T;
    const int k = blockIdx.x * DD_SCAN_T + threadIdx.x;
    const int w = k < n ? ad.E[md.mem[k]] : 0;
    int tot;
    const int incl = block_incl_scan(w, wsum, tot);
    if (k >= n) return;
    const long long pre = bsum[blockIdx.x] + (incl - w);
    const long long W = bsum[nb];
    long long o = W > 0 ? ((long long)P * (2 * pre + w)) / (2 * W) : 0;
    if (o > P - 1) o = P - 1;
    owner[k] = (uint8_t)o;
    if (o == rank) {
        atomicMin(range + 0, k);
        atomicAdd(range + 1, 1);
    }
}

__global__ void k_dd_range_init(const int *n_ptr, int *range)
{
    range[0] = *n_ptr;
    range[1] = 0;
}

// ownership-filtered partition keys (the unfiltered keys of partition.cuh, -1 when not kept)
struct KeyOwnEl {
    const uint8_t *mem, *owner;
    int rank;
    __device__ int operator()(int i) const { return owner[i] == rank ? (int)mem[i] : -1; }
};
struct KeyOwnIfc {
    const int4 *a;
    const uint8_t *owner;
    int rank;
    __device__ int operator()(int i) const
    {
        const int4 I = a[i];
        return (owner[I.x] == rank || owner[I.y] == rank) ? I.w : -1;
    }
};
struct KeyOwnMor {
    const int4 *a;
    const uint8_t *owner;
    int rank;
    __device__ int operator()(int i) const
    {
        const int4 M = a[i];
        return (owner[M.x] == rank || owner[M.y] == rank || owner[M.z] == rank) ? (M.w >> 8) : -1;
    }
};
struct KeyOwnBnd {
    const int2 *a;
    const uint8_t *owner;
    int rank;
    __device__ int operator()(int i) const { return owner[a[i].x] == rank ? (a[i].y >> 8) : -1; }
};
// BR1 halo restricted to owned halo elements (their gradients are this rank's to compute) and the
// faces those elements need
struct KeyOwnHaloEl {
    const uint8_t *halo, *mem, *owner;
    int rank;
    __device__ int operator()(int i) const { return (halo[i] && owner[i] == rank) ? (int)mem[i] : -1; }
};
struct KeyOwnHaloIf {
    const int4 *a;
    const uint8_t *halo, *owner;
    int rank;
    __device__ int operator()(int i) const
    {
        const int4 I = a[i];
        return ((halo[I.x] && owner[I.x] == rank) || (halo[I.y] && owner[I.y] == rank)) ? I.w : -1;
    }
};
struct KeyOwnHaloMo {
    const int4 *a;
    const uint8_t *halo, *owner;
    int rank;
    __device__ int operator()(int i) const
    {
        const int4 M = a[i];
        return ((halo[M.y] && owner[M.y] == rank) || (halo[M.z] && owner[M.z] == rank)) ? (M.w >> 8) : -1;
    }
};
// send / receive lists: cells flagged for one peer, by member (descending) so that every stage's
// active cells are a prefix
struct KeyFlagMem {
    const uint8_t *flag, *mem;
    __device__ int operator()(int i) const { return flag[i] ? (int)mem[i] : -1; }
};

// flags[(2 q + 0) cap + c] = cell c (owned here) is a ghost of rank q; flags[(2 q + 1) cap + c] =
// cell c (owned by q) is a ghost here.  Interfaces and mortars of the global face records.
__device__ __forceinline__ void dd_mark(uint8_t *flags, int cap, const uint8_t *owner, int rank, int a, int b)
{
    const int oa = owner[a], ob = owner[b];
    if (oa == ob) return;
    if (oa == rank) {
        flags[(size_t)(2 * ob) * cap + a] = 1;
        flags[(size_t)(2 * ob + 1) * cap + b] = 1;
    } else if (ob == rank) {
        flags[(size_t)(2 * oa) * cap + b] = 1;
        flags[(size_t)(2 * oa + 1) * cap + a] = 1;
    }
}

__global__ void k_dd_flags(MeshDev md, const uint8_t *owner, int rank, uint8_t *flags)
{
    const int nif = md.n[1], nmo = md.n[2];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nif + nmo; t += gridDim.x * blockDim.x) {
        if (t < nif) {
            const int4 I = md.ifc[t];
            dd_mark(flags, md.cap, owner, rank, I.x, I.y);
        } else {
            const int4 M = md.mor[t - nif];
            dd_mark(flags, md.cap, owner, rank, M.x, M.y);
            dd_mark(flags, md.cap, owner, rank, M.x, M.z);
        }
    }
}

// per stage i: cnt[0][i-1] = cells of the members active at stage i (state exchange after the
// volume kernel), cnt[1][i-1] = the same plus the member just below (Navier-Stokes: viscous-flux
// traces of the active cells and of the BR1 halo, whose large elements belong to that member)
__global__ void k_dd_counts(const int *seg, ActiveDesc ad, int *cnt)
{
    const int t = threadIdx.x;
    if (t >= ad.S) return;
    const int k = active_segments(ad, t + 1);
    cnt[t] = seg[k];
    cnt[MAXS + t] = seg[k + 1 <= ad.R ? k + 1 : ad.R];
}

// pack (row doubles of each listed cell, in list order) / unpack / direct copy into a peer's array
__global__ void k_dd_pack(const int *__restrict__ list, const int *__restrict__ cnt, int row,
                          const double *__restrict__ src, double *__restrict__ buf)
{
    const int n = *cnt;
    const int h = row / 2;
    const double2 *s2 = reinterpret_cast<const double2 *>(src);
    double2 *b2 = reinterpret_cast<double2 *>(buf);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)n * h;
         t += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(t / h), c = (int)(t % h);
        b2[t] = s2[(size_t)list[j] * h + c];
        (void)j;
    }
}

__global__ void k_dd_unpack(const int *__restrict__ list, const int *__restrict__ cnt, int row,
                            const double *__restrict__ buf, double *__restrict__ dst)
{
    const int n = *cnt;
    const int h = row / 2;
    const double2 *b2 = reinterpret_cast<const double2 *>(buf);
    double2 *d2 = reinterpret_cast<double2 *>(dst);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)n * h;
         t += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(t / h), c = (int)(t % h);
        d2[(size_t)list[j] * h + c] = b2[t];
    }
}

// in-process exchange (sub-domains of one process, on one device or on peer-accessible devices):
// the owner's blocks go straight into the same global rows of the peer's array (no staging buffer)
__global__ void k_dd_copy(const int *__restrict__ list, const int *__restrict__ cnt, int row,
                          const double *__restrict__ src, double *__restrict__ dst)
{
    const int n = *cnt;
    const int h = row / 2;
    const double2 *s2 = reinterpret_cast<const double2 *>(src);
    double2 *d2 = reinterpret_cast<double2 *>(dst);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)n * h;
         t += (long long)gridDim.x * blockDim.x) {
        const size_t idx = (size_t)list[(int)(t / h)] * h + (int)(t % h);
        d2[idx] = s2[idx];
    }
}

}  // namespace perk
