// mesh.cuh -- device-side mesh + partition pipeline, no host round trip.
//
//   level map (uint8, finest grid)  --k_leaf_flags-->  leaf-origin flag per Morton index
//   --stable partition-->  leaves in Morton order (+ rank of every origin)
//   --k_leaf_fill / k_cell_of-->  leaf origin, level, member; finest cell -> leaf
//   --k_classify-->  class of every (leaf, direction) slot: interface / mortar / boundary / none
//   --stable partition by class-->  canonical face order  --k_face_records-->  int4/int2 records
//   --stable partition by member (x4 kinds)-->  per-member lists + stage prefix tables count_active
//
// Conventions (paper silent): Morton order of leaf origins (x bit lowest);
// faces per leaf in direction order (+x, -x, +y, -y); interface emitted by the low side when the
// neighbour has the same level; mortar owned by the large element; 1D: every cell emits its +x
// interface and a level-jump interface belongs to the fine side's member.
#pragma once
#include "common.cuh"
#include "partition.cuh"

namespace perk {

__device__ __forceinline__ unsigned compact_bits(unsigned long long m)   // even bits -> low 32 bits
{
    m &= 0x5555555555555555ull;
    m = (m | (m >> 1)) & 0x3333333333333333ull;
    m = (m | (m >> 2)) & 0x0f0f0f0f0f0f0f0full;
    m = (m | (m >> 4)) & 0x00ff00ff00ff00ffull;
    m = (m | (m >> 8)) & 0x0000ffff0000ffffull;
    m = (m | (m >> 16)) & 0x00000000ffffffffull;
    return (unsigned)m;
}

__device__ __forceinline__ unsigned long long spread_bits(unsigned x)
{
    unsigned long long m = x;
    m = (m | (m << 16)) & 0x0000ffff0000ffffull;
    m = (m | (m << 8)) & 0x00ff00ff00ff00ffull;
    m = (m | (m << 4)) & 0x0f0f0f0f0f0f0f0full;
    m = (m | (m << 2)) & 0x3333333333333333ull;
    m = (m | (m << 1)) & 0x5555555555555555ull;
    return m;
}

__device__ __forceinline__ long long morton_of(const MeshDev &md, int x, int y)
{
    return md.dim == 1 ? (long long)x : (long long)(spread_bits(x) | (spread_bits(y) << 1));
}

// member(l) = clamp(R-1-(L-l), 0, R-1)  (P:l.1276-1279)
__device__ __forceinline__ int member_of_level(int R, int L, int l)
{
    int m = R - 1 - (L - l);
    return m < 0 ? 0 : (m > R - 1 ? R - 1 : m);
}

// flag[m] = 1 iff the finest cell with Morton index m is the origin of a leaf; validates that every
// finest cell is covered by exactly one aligned block, the one of its own level.
__global__ void k_leaf_flags(MeshDev md, const uint8_t *__restrict__ lmap, long long nmorton, uint8_t *flag)
{
    const long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= nmorton) return;
    int x, y;
    if (md.dim == 1) { x = (int)m; y = 0; }
    else { x = (int)compact_bits(m); y = (int)compact_bits(m >> 1); }
    if (x >= md.nfx || y >= md.nfy) { flag[m] = 0; return; }
    const int L = md.max_level;
    const int lc = lmap[(size_t)y * md.nfx + x];
    int covers = 0, own = 0;
    if (lc > L) { atomicOr(md.err, ERR_UNBALANCED); flag[m] = 0; return; }
    for (int l = 0; l <= L; ++l) {
        const int s = 1 << (L - l);
        const int ox = x - x % s, oy = md.dim == 1 ? 0 : y - y % s;
        if (lmap[(size_t)oy * md.nfx + ox] == l) { ++covers; if (l == lc) own = 1; }
    }
    if (covers != 1 || !own) atomicOr(md.err, ERR_UNBALANCED);
    const int s = 1 << (L - lc);
    flag[m] = (x % s == 0 && (md.dim == 1 || y % s == 0)) ? 1 : 0;
}

constexpr int CELL_OVERFLOW = -2;

__global__ void k_check_capacity(MeshDev md)
{
    if (md.n[0] > md.cap) { atomicOr(md.err, ERR_CAPACITY); md.n[0] = md.cap; }
}

// leaf k <- Morton index morton_list[k]
__global__ void k_leaf_fill(MeshDev md, const uint8_t *__restrict__ lmap, const int *__restrict__ morton_list, int R)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= md.n[0]) return;
    const long long m = morton_list[k];
    int x, y;
    if (md.dim == 1) { x = (int)m; y = 0; }
    else { x = (int)compact_bits(m); y = (int)compact_bits(m >> 1); }
    const int l = lmap[(size_t)y * md.nfx + x];
    md.fx[k] = x;
    md.fy[k] = y;
    md.lev[k] = (uint8_t)l;
    md.mem[k] = (uint8_t)member_of_level(R, md.max_level, l);
}

// finest cell -> leaf id (the rank of its block origin among the leaf origins)
__global__ void k_cell_of(MeshDev md, const uint8_t *__restrict__ lmap, const int *__restrict__ rank)
{
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (long long)md.nfx * md.nfy) return;
    const int x = (int)(c % md.nfx), y = (int)(c / md.nfx);
    const int s = 1 << (md.max_level - lmap[c]);
    const int ox = x - x % s, oy = md.dim == 1 ? 0 : y - y % s;
    int r = rank[morton_of(md, ox, oy)];
    // leaves beyond the capacity (md.n[0] was clamped to cap by k_check_capacity) have no storage:
    // mark them -2 so that no later kernel indexes a cap-sized array with them
    if (r >= md.n[0]) { atomicOr(md.err, ERR_CAPACITY); r = CELL_OVERFLOW; }
    md.cell_of[c] = r;
}

// finest cell (x, y) -> leaf, -1 outside a non-periodic domain, CELL_OVERFLOW past the capacity
__device__ __forceinline__ int cell_at(const MeshDev &md, int x, int y)
{
    if (x < 0 || x >= md.nfx) { if (!md.periodic[0]) return -1; x = wrapi(x, md.nfx); }
    if (y < 0 || y >= md.nfy) { if (!md.periodic[1]) return -1; y = wrapi(y, md.nfy); }
    return md.cell_of[(size_t)y * md.nfx + x];
}

enum SlotClass { SLOT_NONE = 0, SLOT_BND = 1, SLOT_MOR = 2, SLOT_IF = 3 };

struct SlotInfo {
    int cls, nb, s0, s1;
};

__device__ __forceinline__ SlotInfo classify_slot(const MeshDev &md, int e, int d, bool check)
{
    SlotInfo r{SLOT_NONE, -1, -1, -1};
    const int L = md.max_level, l = md.lev[e], s = 1 << (L - l);
    const int orient = d >> 1;
    const bool plus = (d & 1) == 0;
    int nx, ny;
    if (orient == 0) { nx = plus ? md.fx[e] + s : md.fx[e] - 1; ny = md.fy[e]; }
    else { nx = md.fx[e]; ny = plus ? md.fy[e] + s : md.fy[e] - 1; }
    const int nb = cell_at(md, nx, ny);
    if (nb == CELL_OVERFLOW) return r;     // capacity error already latched; no face
    if (nb < 0) { r.cls = SLOT_BND; return r; }
    const int ln = md.lev[nb];
    r.nb = nb;
    if (ln > l + 1 || ln < l - 1) {
        if (check) atomicOr(md.err, ERR_UNBALANCED);
        return r;
    }
    if (md.dim == 1) { r.cls = plus ? SLOT_IF : SLOT_NONE; return r; }
    if (ln == l) { r.cls = plus ? SLOT_IF : SLOT_NONE; return r; }
    if (ln == l + 1) {
        const int h = s >> 1;
        int a0x, a0y, a1x, a1y;
        if (orient == 0) { a0x = nx; a0y = md.fy[e]; a1x = nx; a1y = md.fy[e] + h; }
        else { a0x = md.fx[e]; a0y = ny; a1x = md.fx[e] + h; a1y = ny; }
        r.s0 = cell_at(md, a0x, a0y);
        r.s1 = cell_at(md, a1x, a1y);
        if (r.s0 < 0 || r.s1 < 0) return r;   // CELL_OVERFLOW (capacity error latched)
        if (md.lev[r.s0] != l + 1 || md.lev[r.s1] != l + 1) {
            if (check) atomicOr(md.err, ERR_UNBALANCED);
            return r;
        }
        r.cls = SLOT_MOR;
    }
    return r;
}

__global__ void k_classify(MeshDev md, uint8_t *slot_class)
{
    const int nd = md.dim == 1 ? 2 : 4;
    const int sl = blockIdx.x * blockDim.x + threadIdx.x;
    if (sl >= md.n[0] * nd) return;
    slot_class[sl] = (uint8_t)classify_slot(md, sl / nd, sl % nd, true).cls;
}

// seg = class-partition segments: [0] interfaces, [1] mortars, [2] boundaries, [3] none
__global__ void k_face_counts(MeshDev md, const int *seg, int cap_faces)
{
    int nif = seg[1] - seg[0], nmo = seg[2] - seg[1], nbd = seg[3] - seg[2];
    if (nif > cap_faces || nmo > cap_faces || nbd > cap_faces) {
        atomicOr(md.err, ERR_CAPACITY);
        nif = min(nif, cap_faces); nmo = min(nmo, cap_faces); nbd = min(nbd, cap_faces);
    }
    md.n[1] = nif; md.n[2] = nmo; md.n[3] = nbd;
}

__global__ void k_face_records(MeshDev md, const int *__restrict__ slot_list, const int *__restrict__ seg, int R)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int nd = md.dim == 1 ? 2 : 4;
    const int nif = md.n[1], nmo = md.n[2], nbd = md.n[3];
    if (p >= nif + nmo + nbd) return;
    const int L = md.max_level;
    if (p < nif) {
        const int sl = slot_list[seg[0] + p];
        const int e = sl / nd, d = sl % nd;
        const SlotInfo si = classify_slot(md, e, d, false);
        const int l = md.lev[e], ln = md.lev[si.nb];
        const int mem = member_of_level(R, L, max(l, ln));   // 2D: equal levels; 1D: the fine side
        md.ifc[p] = make_int4(e, si.nb, d >> 1, mem);
    } else if (p < nif + nmo) {
        const int q = p - nif;
        const int sl = slot_list[seg[1] + q];
        const int e = sl / nd, d = sl % nd;
        const SlotInfo si = classify_slot(md, e, d, false);
        const int side = (d & 1);                              // 0: large element on the low side
        const int mem = member_of_level(R, L, md.lev[e] + 1);  // the fine side (P:l.1256)
        md.mor[q] = make_int4(e, si.s0, si.s1, (d >> 1) | (side << 1) | (mem << 8));
    } else {
        const int q = p - nif - nmo;
        const int sl = slot_list[seg[2] + q];
        const int e = sl / nd, d = sl % nd;
        md.bnd[q] = make_int2(e, d | ((int)md.mem[e] << 8));
    }
}

// per element face neighbours (MeshDev::fnb) from the face records (grid-stride over all records)
__global__ void k_face_table(MeshDev md)
{
    const int nif = md.n[1], nmo = md.n[2], nbd = md.n[3];
    auto pkn = [&](int e) { return e | ((int)md.mem[e] << PK_EBITS); };
    auto ok = [&](int e) { return e >= 0 && e < md.cap; };   // (a latched capacity error leaves no valid mesh)
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nif + nmo + nbd; p += gridDim.x * blockDim.x) {
        if (p >= nif + nmo) {
            const int2 B = md.bnd[p - nif - nmo];
            if (ok(B.x)) md.fnb[(size_t)B.x * 4 + (B.y & 7)] = make_int2(-1, FNB_NONE);
        } else if (p < nif) {
            const int4 I = md.ifc[p];                      // low side's face 2o, high side's face 2o + 1
            if (!ok(I.x) || !ok(I.y)) continue;
            md.fnb[(size_t)I.x * 4 + 2 * I.z] = make_int2(pkn(I.y), FNB_CONF);
            md.fnb[(size_t)I.y * 4 + 2 * I.z + 1] = make_int2(pkn(I.x), FNB_CONF);
        } else {
            const int4 M = md.mor[p - nif];
            if (!ok(M.x) || !ok(M.y) || !ok(M.z)) continue;
            const int o = M.w & 1, side = (M.w >> 1) & 1;
            const int lf = 2 * o + side, sf = 2 * o + 1 - side;
            md.fnb[(size_t)M.x * 4 + lf] = make_int2(pkn(M.y), pkn(M.z));
            md.fnb[(size_t)M.y * 4 + sf] = make_int2(pkn(M.x), FNB_SMALL_LO);
            md.fnb[(size_t)M.z * 4 + sf] = make_int2(pkn(M.x), FNB_SMALL_HI);
        }
    }
}

// physical node coordinates [n][dim][npe]
// hot-path copies in list order: packed element entries, interface and mortar records
// (list lengths = the partition totals seg[kind][R]: all items, or the owned ones of a sub-domain)
__global__ void k_hot_lists(MeshDev md, int R)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < md.seg[KIND_EL * (MAXR + 1) + R]) {
        const int e = md.list[KIND_EL][t];
        md.elpk[t] = e | ((int)md.mem[e] << PK_EBITS) | ((int)md.lev[e] << (PK_EBITS + 3));
    }
    if (t < md.seg[KIND_IF * (MAXR + 1) + R]) md.ifcs[t] = md.ifc[md.list[KIND_IF][t]];
    if (t < md.seg[KIND_MO * (MAXR + 1) + R]) md.mors[t] = md.mor[md.list[KIND_MO][t]];
}

// BR1 halo flags: the large side of a mortar whose fine side belongs to another member
// gather the per-stage hot arrays: out position j <- hot-array position idx[j] (count from seg[1])
__global__ void k_stage_gather(const int *__restrict__ seg, const int *__restrict__ idx, int kind, MeshDev md,
                               int *el_out, int4 *f4_out, int *bd_out)
{
    const int n = seg[1];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int t = idx[j];
        if (kind == KIND_EL) el_out[j] = md.elpk[t];
        else if (kind == KIND_IF) f4_out[j] = md.ifcs[t];
        else if (kind == KIND_MO) f4_out[j] = md.mors[t];
        else bd_out[j] = md.list[KIND_BD][t];
    }
}

__global__ void k_halo_clear(MeshDev md)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < md.cap) md.halo[e] = 0;
}
__global__ void k_halo_flags(MeshDev md)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= md.n[2]) return;
    const int4 M = md.mor[q];
    if ((int)md.mem[M.x] != (M.w >> 8)) md.halo[M.x] = 1;
}
// per stage, the halo lists of the member just below the lowest active one; packed halo entries
__global__ void k_halo_ranges(MeshDev md, ActiveDesc ad)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < 3 * ad.S) {
        const int kind = t / ad.S, i = t % ad.S + 1;
        const int k = active_segments(ad, i);    // Navier-Stokes runs the standard pattern only
        const int *sg = md.hseg + kind * (MAXR + 1);
        md.hrng[kind * MAXS + i - 1] = k < ad.R ? make_int2(sg[k], sg[k + 1] - sg[k]) : make_int2(0, 0);
    }
    const int total = md.hseg[KIND_EL * (MAXR + 1) + ad.R];
    for (int h = t; h < total; h += gridDim.x * blockDim.x) {
        const int e = md.hlist[KIND_EL][h];
        md.hpk[h] = e | ((int)md.mem[e] << PK_EBITS) | ((int)md.lev[e] << (PK_EBITS + 3));
    }
}

__global__ void k_node_coords(MeshDev md, double *xy)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= md.n[0]) return;
    const double h = md.hf * (double)(1 << (md.max_level - md.lev[e]));
    const double x0 = md.lo[0] + md.fx[e] * md.hf, y0 = md.lo[1] + md.fy[e] * md.hf;
    for (int q = 0; q < md.npe; ++q) {
        const int i = q % NP, j = q / NP;
        if (md.dim == 1) {
            xy[(size_t)e * md.npe + q] = x0 + 0.5 * h * (cB.xi[i] + 1.0);
        } else {
            xy[((size_t)e * 2 + 0) * md.npe + q] = x0 + 0.5 * h * (cB.xi[i] + 1.0);
            xy[((size_t)e * 2 + 1) * md.npe + q] = y0 + 0.5 * h * (cB.xi[j] + 1.0);
        }
    }
}

}  // namespace perk
