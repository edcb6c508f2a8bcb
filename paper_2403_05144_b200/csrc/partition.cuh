// partition.cuh -- device stream compaction: stable multi-bucket partition by a small key
// (warp ballot + block scan), the primitive behind every list rebuild.
//
// Items i in [0, n) (n read from device memory, times `mult`) with key(i) in [0, R) are written
// to out[] grouped by DESCENDING key (segment s holds key R-1-s), order-preserving inside a
// bucket.  Three launches: per-block bucket counts (ballot + popc) -> one-block scan of the
// block counts in segment order -> scatter (ballot prefix within the warp + warp offsets).
#pragma once
#include "common.cuh"

namespace perk {

constexpr int PART_T = 1024;   // items per block (one per thread)

struct KeyU8 {
    const uint8_t *a;
    __device__ int operator()(int i) const { return a[i]; }
};
struct KeyIfc {
    const int4 *a;
    __device__ int operator()(int i) const { return a[i].w; }
};
struct KeyMor {
    const int4 *a;
    __device__ int operator()(int i) const { return a[i].w >> 8; }
};
struct KeyBnd {
    const int2 *a;
    __device__ int operator()(int i) const { return a[i].y >> 8; }
};
// BR1 halo keys: the member for flagged items, -1 (not partitioned) otherwise
struct KeyHaloEl {
    const uint8_t *halo, *mem;
    __device__ int operator()(int i) const { return halo[i] ? (int)mem[i] : -1; }
};
struct KeyHaloIf {
    const int4 *a;
    const uint8_t *halo;
    __device__ int operator()(int i) const { const int4 I = a[i]; return (halo[I.x] | halo[I.y]) ? I.w : -1; }
};
struct KeyHaloMo {
    const int4 *a;
    const uint8_t *halo;
    __device__ int operator()(int i) const { const int4 M = a[i]; return (halo[M.y] | halo[M.z]) ? (M.w >> 8) : -1; }
};

// Per-stage item lists for non-nested stage patterns (2D): key 0 = the item is needed at the stage
// (an element / interface / boundary of an evaluating member, a mortar with an evaluating fine or
// coarse side), -1 = dropped.  Items are positions in the member-sorted hot arrays.
struct KeyStageEl {
    const int *elpk;
    unsigned mask;
    __device__ int operator()(int t) const { return ((mask >> ((elpk[t] >> 24) & 7)) & 1u) ? 0 : -1; }
};
struct KeyStageIf {
    const int4 *a;
    unsigned mask;
    __device__ int operator()(int t) const { return ((mask >> a[t].w) & 1u) ? 0 : -1; }
};
struct KeyStageMo {
    const int4 *a;
    const uint8_t *mem;
    unsigned mask;
    __device__ int operator()(int t) const
    {
        const int4 M = a[t];
        return (((mask >> (M.w >> 8)) | (mask >> mem[M.x])) & 1u) ? 0 : -1;
    }
};
struct KeyStageBd {
    const int *list;
    const int2 *bnd;
    unsigned mask;
    __device__ int operator()(int t) const { return ((mask >> (bnd[list[t]].y >> 8)) & 1u) ? 0 : -1; }
};

// Stage-activity description for the count_active table (P:l.428: member r evaluates stage i iff
// i == 1 or E_r >= S - i + 2).
struct ActiveDesc {
    int S, R;
    int E[MAXR];
    unsigned long long act[MAXR];   // evaluated stages of member r (bit i-1), standard or not
};

// members are sorted by descending E in the lists; the stage-i launch covers the segments of every
// member from the top down to the lowest-index member evaluating stage i (standard pattern: exactly
// the evaluating members, a prefix; other patterns: a superset whose surplus members are skipped)
__device__ __forceinline__ int active_segments(const ActiveDesc &ad, int i)
{
    int rmin = ad.R;
    for (int r = ad.R - 1; r >= 0; --r)
        if ((ad.act[r] >> (i - 1)) & 1ull) rmin = r;
    return ad.R - rmin;
}

template <class KeyFn>
__global__ void __launch_bounds__(PART_T) k_part_count(KeyFn kf, const int *n_ptr, int mult, int R, int *blockcnt)
{
    __shared__ int cnt[MAXR];
    const int n = *n_ptr * mult;
    const int i = blockIdx.x * PART_T + threadIdx.x;
    if (threadIdx.x < MAXR) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int key = i < n ? kf(i) : -1;
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < R; ++r) {
        unsigned b = __ballot_sync(0xffffffffu, key == r);
        if (lane == 0 && b) atomicAdd(&cnt[r], __popc(b));
    }
    __syncthreads();
    if (threadIdx.x < MAXR) blockcnt[blockIdx.x * MAXR + threadIdx.x] = cnt[threadIdx.x];
}

__device__ __forceinline__ int block_incl_scan(int v, int *wsum, int &total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    x += warp > 0 ? wsum[warp - 1] : 0;
    total = wsum[nw - 1];
    __syncthreads();
    return x;
}

// One block.  blockoff[b][r] = start of block b's bucket-r items; seg[s] = start of segment s
// (key R-1-s), seg[R] = total.  Optionally: *total_out = total, and count_active[i-1] for the
// member partitions (active members are the top ones, i.e. a prefix of the segments).
constexpr int PART_OFF_T = 1024;   // k_part_offsets block: 4x fewer sequential chunk scans than PART_T
__global__ void __launch_bounds__(PART_OFF_T) k_part_offsets(const int *blockcnt, int nblocks, int R, int *blockoff, int *seg,
                                                        int *total_out, ActiveDesc ad, int *count_active,
                                                        unsigned long long *evals_per_step = nullptr)
{
    __shared__ int wsum[32];
    int base = 0;
    for (int s = 0; s < R; ++s) {
        const int r = R - 1 - s;
        if (threadIdx.x == 0) seg[s] = base;
        for (int chunk = 0; chunk < nblocks; chunk += blockDim.x) {
            const int b = chunk + threadIdx.x;
            const int v = b < nblocks ? blockcnt[b * MAXR + r] : 0;
            int tot;
            const int incl = block_incl_scan(v, wsum, tot);
            if (b < nblocks) blockoff[b * MAXR + r] = base + incl - v;
            base += tot;
        }
    }
    if (threadIdx.x == 0) {
        seg[R] = base;
        if (total_out) *total_out = base;
    }
    __syncthreads();
    if (count_active && threadIdx.x < ad.S) {
        const int i = threadIdx.x + 1;
        count_active[i - 1] = seg[active_segments(ad, i)];
    }
    if (evals_per_step && threadIdx.x == 0) {      // sum_r E_r N_C(r) (P:l.1282-1289)
        unsigned long long tot = 0;
        for (int r = 0; r < ad.R; ++r)
            tot += (unsigned long long)ad.E[r] * (unsigned long long)(seg[R - r] - seg[R - 1 - r]);
        *evals_per_step = tot;
    }
}

template <class KeyFn>
__global__ void __launch_bounds__(PART_T) k_part_scatter(KeyFn kf, const int *n_ptr, int mult, int R, const int *blockoff,
                                                        int *out, int *rank)
{
    __shared__ int wcnt[PART_T / 32][MAXR];
    const int n = *n_ptr * mult;
    const int i = blockIdx.x * PART_T + threadIdx.x;
    const int key = i < n ? kf(i) : -1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    int myprefix = 0;
    for (int r = 0; r < R; ++r) {
        unsigned b = __ballot_sync(0xffffffffu, key == r);
        if (lane == 0) wcnt[warp][r] = __popc(b);
        if (key == r) myprefix = __popc(b & lt);
    }
    __syncthreads();
    if (threadIdx.x < R) {
        int acc = 0;
        for (int w = 0; w < PART_T / 32; ++w) {
            int t = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = acc;
            acc += t;
        }
    }
    __syncthreads();
    if (key >= 0) {
        const int pos = blockoff[blockIdx.x * MAXR + key] + wcnt[warp][key] + myprefix;
        out[pos] = i;
        if (rank) rank[i] = pos;
    }
}

}  // namespace perk
