// br1.cuh -- Navier-Stokes BR1 passes of one P-ERK stage (D7).
//
// The paper cites BR1 (P:l.1419-1420) without defining it.  Per stage, before the inviscid+viscous
// surface kernel (k_surf2d<.., NS>) and the volume kernel (k_vol2d<.., NS>):
//   k_grad2d  : on the active elements and the halo (the large elements of the active mortars, which
//               belong to the next coarser member and whose gradients the active viscous face fluxes
//               need; MeshDev::halo): the central traces w* = (w_L + w_R)/2 of the gradient variables
//               w = (v1, v2, T) on the element's own faces, formed from the face neighbours' traces
//               (BR1_FUSED, MeshDev::fnb; mortars: halves (P w_large + w_small)/2, the large side
//               R_lower w*_lo + R_upper w*_hi), q = grad w (weak form with w*), then the viscous flux at
//               the line nodes: the normal one at the 12 face nodes -> Vt, read by k_surf2d, and the
//               viscous volume term Dv = -(2/h) sum_a Dhat_ia F^v(node a) (BR1_DV), read by k_vol2d.
//   k_gsurf2d : (BR1_FUSED = 0 only) the central traces as a separate pass over the active interfaces /
//               mortars and the halo faces -> Gs, staged by k_grad2d.
// (The oracle evaluates gradients on the whole next coarser member instead; both give the same
// gradients on every element whose viscous face flux is used.)
#pragma once
#include "dg2d.cuh"

namespace perk {

template <int MODE>
__global__ void __launch_bounds__(256, 3) k_gsurf2d(MeshDev md, StageParams sp, const double *__restrict__ Un,
                                                const double *__restrict__ Ubuf, const double *__restrict__ K1,
                                                const double *__restrict__ Uin, double *__restrict__ Gs)
{
    pdl_wait();
    // items: [active interfaces | halo interfaces | active mortars | halo mortars]
    int nif_a, nmo_a;
    int2 hif = make_int2(0, 0), hmo = make_int2(0, 0);
    if (MODE == MODE_STAGE) {
        nif_a = md.count_active[KIND_IF * MAXS + sp.stage - 1];
        nmo_a = md.count_active[KIND_MO * MAXS + sp.stage - 1];
        hif = md.hrng[KIND_IF * MAXS + sp.stage - 1];
        hmo = md.hrng[KIND_MO * MAXS + sp.stage - 1];
    } else {
        nif_a = md.n[1]; nmo_a = md.n[2];
    }
    const int nif = nif_a + hif.y, nmo = nmo_a + hmo.y;
    const int total = 4 * (nif + nmo);
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const double dtc = sp.dt * sp.c_stage;
    const double gm1 = md.gamma - 1.0;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = 0xFu << (lane & ~3);
    for (int gt = blockIdx.x * blockDim.x + threadIdx.x; gt < total; gt += gridDim.x * blockDim.x) {
        const int item = gt >> 2, k = gt & 3;
        if (item < nif) {
            const int4 I = MODE == MODE_RHS ? md.ifc[item]
                                            : (item < nif_a ? md.ifcs[item] : md.ifc[md.hlist[KIND_IF][hif.x + item - nif_a]]);
            PERK_DASSERT(I.x >= 0 && I.x < md.n[0] && I.y >= 0 && I.y < md.n[0]);
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
            const int4 M = MODE == MODE_RHS ? md.mor[q] : (q < nmo_a ? md.mors[q] : md.mor[md.hlist[KIND_MO][hmo.x + q - nmo_a]]);
            PERK_DASSERT(M.x >= 0 && M.x < md.n[0] && M.y >= 0 && M.y < md.n[0] && M.z >= 0 && M.z < md.n[0]);
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
// Persistent CTAs of 16 elements; the element's stage state (and, unfused, its 48 central traces) is
// staged with cp.async one group ahead (commit groups as in k_vol2d); packed entries two groups ahead.
//
// BR1_FUSED = 1: no k_gsurf2d pass and no Gs array -- each element forms the central traces w* of its
// own faces from the face neighbours' stage-state traces (MeshDev::fnb), gathered at the top of the
// iteration while its own state is turned into primitives: conforming 1/2 (w + w_nb); small side of a
// mortar 1/2 (P w_large + w); large side R_lo 1/2 (P_lo w + w_s0) + R_up 1/2 (P_up w + w_s1), the
// interpolations / projections as 4-lane shuffles over the face's nodes, in exactly k_gsurf2d's
// operation order (so w* is bitwise the same number on both sides of every face).  Saves the Gs write
// and read (768 B per element-stage) and one launch per stage; the trace gathers move here.
#ifndef BR1_FUSED
#define BR1_FUSED 1
#endif
// 2/h by the exact power-of-two scaling of common.cuh two_over_h (0) or by a division (1).  The division
// (inline reciprocal iteration + guarded slow-path call, ~25 issued instructions per warp and group in a
// kernel that is issue-bound) costs cfg 5 gradients 1.89 vs 1.77 ms/step (profiles/r02_ab_grad_l1.json);
// before GRAD2D_LG freed registers the scaling variant spilled at the 128-register cap (2.25).
#ifndef VISC_LINE
#define VISC_LINE 1
#endif
#ifndef GRAD2D_DIV
#define GRAD2D_DIV 0
#endif
static_assert(!BR1_FUSED || BR1_DV, "the fused BR1 gradient kernel leaves no Gs for the volume kernel");
// shared-memory field layout.  GRAD2D_SX = 16: k_vol2d's (x part 16 le + 4j + i, y part 258 + 20 le + 4i + j);
// the cross-direction gradient reads (scalar, fixed node a: the y-line threads read 16 le + 4a + ln) then
// hit the same banks for all four elements of a warp (ncu: 6 instead of 2 wavefronts per load, 22 % of
// the kernel's shared-memory wavefronts; bank conflicts per stage-30 launch 4.7M -> 1.3M, cfg 5
// gradients 1.80 -> 1.77 ms/step).  20: both parts with element stride 20 (x part 20 le + 4j + i,
// y part 318 + 20 le + 4i + j): (4 le + 4a + ln) mod 16 is distinct over the warp's 16 lanes of either
// direction, the two directions 14 apart; line loads / stores stay conflict-free (4 (le + ln) mod 16).
#ifndef GRAD2D_SX
#define GRAD2D_SX 20
#endif
constexpr int GRAD2D_LS = GRAD2D_SX == 16 ? VOL2D_LS : 320;
constexpr int GRAD2D_NF = 5;   // fields: v1, v2, T, d v1, d v2 (the T gradient stays in registers)
constexpr int G_V1 = 0, G_V2 = 1, G_T = 2, G_Q = 3;     // shared fields: v1, v2, T, velocity gradients (2)
// staged central traces per element (unfused): 48 doubles padded to 52 (== 4 mod 16), so that the
// scalar trace reads of the x-line threads (faces 0/1) and y-line threads (faces 2/3) of the two
// elements of a half-warp fall into disjoint banks (with 48 the two elements collided).  (Loading each
// thread's 6 end traces into registers one group ahead instead, which frees this buffer: 1.33 vs
// 1.23 ms/step on cfg 5, slower.)
constexpr int GST_STRIDE = 4 * GV * NP + 4;
// staging slots per element: 2 = the state and, for a lazily formed state, K_1 (cp.async one group
// ahead); 1 = the state only, K_1 of a lazy state read directly (8 KB less shared memory per CTA, so
// more L1 for the neighbour gathers: cfg 5 gradients 2.046 -> 2.019 ms/step); 0 (default, fused only) = no
// staging: the thread's two nodes (and K_1 of a lazy state) are loaded into registers together with the
// neighbour gathers, whose latency the iteration waits for anyway -- no cp.async address loop, no staging
// round trip through shared memory (cfg 5 step 6.07 -> 5.99 ms; gradients alone 1.82 -> 1.77)
#ifndef GRAD2D_STG
#define GRAD2D_STG 0
#endif
static_assert(GRAD2D_STG > 0 || BR1_FUSED, "unstaged state loads are written for the fused kernel");
__host__ __device__ constexpr size_t grad2d_smem_bytes()
{
    return sizeof(double) * ((size_t)GRAD2D_NF * 2 * GRAD2D_LS + VOL2D_EPB * GRAD2D_STG * 64 + (BR1_FUSED ? 0 : VOL2D_EPB * GST_STRIDE));
}
#ifndef GRAD2D_MINB
#define GRAD2D_MINB 4
#endif
// the line's own (v1, v2, T) loaded once into registers (ncu: l1tex throughput 92 %, 218 shared-memory
// wavefronts per warp and group): 1 = its end nodes serve as the own face traces (6 scalar shared loads
// less per thread), 2 = also the velocities of the viscous flux (cfg 5 gradients 1.81 -> 1.77 ms/step)
#ifndef GRAD2D_WREG
#define GRAD2D_WREG 2
#endif
// 1 = the whole warp skips the (if-converted) lazy-state K_1 loads when no lane has a lazy state: measured
// slower than the predicated code (1.94 vs 1.89 ms/step), off
#ifndef GRAD2D_LAZYVOTE
#define GRAD2D_LAZYVOTE 0
#endif
// 1 = only the x-line threads finalise Dv (half the shared-memory traffic of the x + y sum, idle y-line
// threads): slower (1.99 vs 1.95 ms/step), off
// 1 = Dv is stored with the streaming policy (st.global.cs): its reader, the volume kernel, runs after the
// surface kernel has streamed several hundred MB through the L2, so the lines are offered for eviction
// first and the L2 keeps Vt and the stage state for the surface kernel (cfg 5 step 5.798 -> 5.755 ms
// together with the streaming Vt loads of k_surf2d, profiles/r02_ab_cs.json)
#ifndef GRAD2D_DVCS
#define GRAD2D_DVCS 1
#endif
#ifndef GRAD2D_DVX
#define GRAD2D_DVX 0
#endif
// 1 = the second small element of a large mortar side is gathered inside the large-side branch (below)
#ifndef GRAD2D_LG
#define GRAD2D_LG 1
#endif

// (the rhs_eval instantiation, off the hot path, takes 3 CTAs per SM: at 4 it spilled 12 B)
template <int MODE>
__global__ void __launch_bounds__(128, MODE == MODE_RHS ? 3 : GRAD2D_MINB) k_grad2d(MeshDev md, StageParams sp, const double *__restrict__ Un,
                                                   const double *__restrict__ Ubuf, const double *__restrict__ K1,
                                                   const double *__restrict__ Uin, const double *__restrict__ Gs,
                                                   double *__restrict__ Vt, double *__restrict__ Dv)
{
    constexpr bool FUSED = BR1_FUSED;
    extern __shared__ __align__(16) unsigned char smraw[];
    double (*sm)[2][GRAD2D_LS] = reinterpret_cast<double (*)[2][GRAD2D_LS]>(smraw);
    double (*stg)[GRAD2D_STG ? GRAD2D_STG : 1][64] = reinterpret_cast<double (*)[GRAD2D_STG ? GRAD2D_STG : 1][64]>(smraw + sizeof(double) * GRAD2D_NF * 2 * GRAD2D_LS);
    double (*gst)[GST_STRIDE] = reinterpret_cast<double (*)[GST_STRIDE]>(reinterpret_cast<unsigned char *>(stg) +
                                                                         sizeof(double) * VOL2D_EPB * GRAD2D_STG * 64);
    const int t8 = threadIdx.x & 7, le = threadIdx.x >> 3;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = 0xFu << (lane & ~3);      // the 4 lanes of one line direction of one element
    // items: [active elements | halo elements of the member below the lowest active one]
    const int n_el_a = MODE == MODE_STAGE ? md.count_active[KIND_EL * MAXS + sp.stage - 1] : md.n[0];
    const int2 hel = MODE == MODE_STAGE ? md.hrng[KIND_EL * MAXS + sp.stage - 1] : make_int2(0, 0);
    const int n_act = n_el_a + hel.y;
    const double gm1 = md.gamma - 1.0;
    const double dtc = sp.dt * sp.c_stage;
    const double two_hf = 2.0 / md.hf;
    const StateBufs sb{Un, Ubuf, K1, Uin};
    const int q0 = 2 * t8;
    const int o = t8 >> 2, ln = t8 & 3;
    const int eox = le * GRAD2D_SX, eoy = le * 20, yo = GRAD2D_SX == 16 ? 2 - 2 * VOL2D_EPB : -2;
    const int stride = gridDim.x * VOL2D_EPB;
    int base = blockIdx.x * VOL2D_EPB;
    auto entry_at = [&](int b) {
        const int t = b + le;
        const int tt = sweep_idx(sp, t < n_act ? t : b, n_act);
        if (MODE == MODE_STAGE) return tt < n_el_a ? md.elpk[tt] : md.hpk[hel.x + tt - n_el_a];
        return tt | ((int)md.mem[tt] << PK_EBITS) | ((int)md.lev[tt] << (PK_EBITS + 3));
    };
    auto copy_chunks = [&](double *dst, const double *src, int nchunks) {   // 16 B chunks over 8 threads
        for (int c = t8; c < nchunks; c += 8) cp_async16(dst + 2 * c, src + 2 * c);
    };
    auto issue_state = [&](int pkx) {
        if (GRAD2D_STG == 0) return;
        const size_t off = (size_t)pk_elem(pkx) * 64;
        const int srce = state_src(sp, pk_member(pkx));
        copy_chunks(stg[le][0], (srce == SRC_UN || srce == SRC_LAZY ? Un : (srce == SRC_BUF ? Ubuf : Uin)) + off, 32);
        if (GRAD2D_STG == 2 && srce == SRC_LAZY) copy_chunks(stg[le][GRAD2D_STG ? GRAD2D_STG - 1 : 0], K1 + off, 32);
    };
    auto issue_gs = [&](int pkx) { copy_chunks(gst[le], Gs + (size_t)pk_elem(pkx) * 4 * GV * NP, 4 * GV * NP / 2); };
    // face-neighbour entries of this thread's two faces (2o: the line's a = N end, 2o + 1: a = 0)
    auto faces_of = [&](int pkx, int2 f[2]) {
        const int2 *F = md.fnb + (size_t)pk_elem(pkx) * 4 + 2 * o;
        f[0] = F[0];
        f[1] = F[1];
    };
    const int pk0 = base < n_act ? entry_at(base) : 0;
    int pk_ahead = base + stride < n_act ? entry_at(base + stride) : 0;   // entries two groups ahead
    pdl_wait();
    if (base >= n_act) return;
    int pk = pk0;
    int2 fn[2] = {make_int2(-1, FNB_NONE), make_int2(-1, FNB_NONE)};
    if (FUSED) faces_of(pk, fn);
    issue_state(pk);
    if (!FUSED) issue_gs(pk);
    cp_async_commit();
    for (; base < n_act; base += stride) {
        const bool valid = base + le < n_act;
        const bool has_next = base + stride < n_act;
        const int pk_next = pk_ahead;
        pk_ahead = base + 2 * stride < n_act ? entry_at(base + 2 * stride) : 0;
        const int e = pk_elem(pk);
        PERK_DASSERT(e >= 0 && e < md.n[0]);
        const int src = state_src(sp, pk_member(pk));
#if GRAD2D_DIV
        const double j2h = 2.0 / (md.hf * (double)(1 << (md.max_level - pk_level(pk))));
#else
        const double j2h = two_over_h(two_hf, pk_level(pk), md.max_level);   // 2 / h
#endif
        // fused: the neighbours' traces at this thread's two face nodes (a large side needs both smalls),
        // every load issued before any is used; lazy states formed after the loads.  (Tried and slower,
        // cfg 5 gradients ms/step: the line's own velocities as 16 B loads 2.11 -> 2.12; the cross reads
        // in a skewed node order (3 -> 2 wavefronts per half-warp on paper) 2.16; the first neighbour's
        // traces staged one group ahead by 8 B cp.async, face entries two groups ahead, 2.62 -- the
        // entry -> face-table chain stalled every iteration and shared-memory conflicts doubled; the next
        // group's neighbour traces prefetched into L2 / L1 after the gradients, 2.42; 3 CTAs/SM, 2.19;
        // the next group's first-neighbour traces loaded into registers after this group's phase 1
        // (entries three groups ahead, 3 CTAs/SM for the registers), 2.14 vs 2.07; again after the
        // instruction diet, when these gathers had become the top stall: the next group's neighbour AND own
        // loads issued after the gradients into the registers the central traces release, 168 registers at
        // 3 CTAs/SM: 1.99 vs 1.77 at 4 CTAs/SM -- 3 CTAs/SM alone costs 1.97, profiles/r02_ab_grad_pf.json)
#if GRAD2D_LG
        // the second small element of a large mortar side (rare: 1-2 % of the elements have such a face) is
        // gathered inside the large-side branch below, not here: 16 registers less at the top
        double un[2][1][4];
        constexpr int NH = 1;
#else
        double un[2][2][4];
        constexpr int NH = 2;
#endif
        if (FUSED) {
            int xe[2][NH], xs[2][NH];
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                const int p0 = fn[f].x >= 0 ? fn[f].x : pk;
                xe[f][0] = pk_elem(p0);
                xs[f][0] = state_src(sp, pk_member(p0));
                if (NH == 2) {
                    const int p1 = fn[f].y >= 0 ? fn[f].y : p0;
                    xe[f][NH - 1] = pk_elem(p1);
                    xs[f][NH - 1] = state_src(sp, pk_member(p1));
                }
            }
#pragma unroll
            for (int f = 0; f < 2; ++f)
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    if (h == 1 && fn[f].y < 0) continue;
                    const double *P = state_base(sb, xs[f][h]) + (size_t)xe[f][h] * 64 + face_node2d((2 * o + f) ^ 1, ln);
#pragma unroll
                    for (int v = 0; v < 4; ++v) un[f][h][v] = __ldg(P + v * 16);
                }
            // lazily formed neighbour states: skipped by the whole warp when none of its lanes has one (the
            // if-converted K_1 loads and FMAs were ~9 % of the kernel's issued instructions at the stages
            // where no state is lazy); the warp is converged here
            bool nlazy = false;
#pragma unroll
            for (int f = 0; f < 2; ++f)
#pragma unroll
                for (int h = 0; h < NH; ++h) nlazy |= !(h == 1 && fn[f].y < 0) && xs[f][h] == SRC_LAZY;
            if (!GRAD2D_LAZYVOTE || __any_sync(0xffffffffu, nlazy)) {
#pragma unroll
                for (int f = 0; f < 2; ++f)
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        if ((h == 1 && fn[f].y < 0) || xs[f][h] != SRC_LAZY) continue;
                        const double *P = K1 + (size_t)xe[f][h] * 64 + face_node2d((2 * o + f) ^ 1, ln);
                        double kk[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v) kk[v] = __ldg(P + v * 16);
#pragma unroll
                        for (int v = 0; v < 4; ++v) un[f][h][v] = fma(dtc, kk[v], un[f][h][v]);
                    }
            }
        }
        double2 u[4];
        const bool olazy_any = !GRAD2D_LAZYVOTE || __any_sync(0xffffffffu, src == SRC_LAZY);
        if (GRAD2D_STG == 0) {   // the element's own two nodes, issued with the neighbour gathers
            const double *Ps = state_base(sb, src) + (size_t)e * 64 + q0;
#pragma unroll
            for (int v = 0; v < 4; ++v) u[v] = __ldg(reinterpret_cast<const double2 *>(Ps + v * 16));
            if (olazy_any && src == SRC_LAZY) {
                double2 k[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) k[v] = __ldg(reinterpret_cast<const double2 *>(K1 + (size_t)e * 64 + v * 16 + q0));
#pragma unroll
                for (int v = 0; v < 4; ++v) u[v] = make_double2(fma(dtc, k[v].x, u[v].x), fma(dtc, k[v].y, u[v].y));
            }
        }
        PERK_JITTER(11);
        cp_async_wait<0>();
        __syncwarp();
        PERK_JITTER(12);
        {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                if (GRAD2D_STG) u[v] = *reinterpret_cast<const double2 *>(&stg[le][0][v * 16 + q0]);
                if (GRAD2D_STG && olazy_any && src == SRC_LAZY) {
                    const double2 k = GRAD2D_STG == 2 ? *reinterpret_cast<const double2 *>(&stg[le][GRAD2D_STG ? GRAD2D_STG - 1 : 0][v * 16 + q0])
                                                      : __ldg(reinterpret_cast<const double2 *>(K1 + (size_t)e * 64 + v * 16 + q0));
                    u[v] = make_double2(fma(dtc, k.x, u[v].x), fma(dtc, k.y, u[v].y));
                }
            }
            const int i0 = q0 & 3, j0 = q0 >> 2;
            double w[2][GV];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double uu[4] = {h ? u[0].y : u[0].x, h ? u[1].y : u[1].x, h ? u[2].y : u[2].x, h ? u[3].y : u[3].x};
                prim_vT(uu, gm1, w[h]);
            }
#pragma unroll
            for (int c = 0; c < GV; ++c) {
                *reinterpret_cast<double2 *>(&sm[G_V1 + c][0][eox + 4 * j0 + i0]) = make_double2(w[0][c], w[1][c]);
                sm[G_V1 + c][1][yo + eoy + 4 * i0 + j0] = w[0][c];
                sm[G_V1 + c][1][yo + eoy + 4 * (i0 + 1) + j0] = w[1][c];
            }
        }
        PERK_JITTER(13);
        __syncwarp();
        if (has_next) issue_state(pk_next);       // stg consumed
        cp_async_commit();
        const int lo = o == 0 ? eox + 4 * ln : yo + eoy + 4 * ln;
        double q[GV][NP];
        const int fld[GV] = {G_V1, G_V2, G_T};
        const double sc[GV] = {1.0, 1.0, 1.0};
#if GRAD2D_WREG
        double wl[GV][NP];   // the line's own (v1, v2, T): its end nodes are the own face traces
#pragma unroll
        for (int c = 0; c < GV; ++c) {
            const double2 w01 = *reinterpret_cast<const double2 *>(&sm[G_V1 + c][o][lo]);
            const double2 w23 = *reinterpret_cast<const double2 *>(&sm[G_V1 + c][o][lo + 2]);
            wl[c][0] = w01.x; wl[c][1] = w01.y; wl[c][2] = w23.x; wl[c][3] = w23.y;
        }
#endif
        if (FUSED) {
            // central traces w* at this thread's nodes of faces 2o (g[0]) and 2o + 1 (g[1])
            double g[2][GV];
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                const int a = f == 0 ? NP - 1 : 0;
                double wo[GV], wn[GV];
#pragma unroll
                for (int c = 0; c < GV; ++c) {
#if GRAD2D_WREG
                    wo[c] = wl[c][a];
#else
                    wo[c] = sm[G_V1 + c][o][lo + a];
#endif
                }
                prim_vT(un[f][0], gm1, wn);
                const int ty = fn[f].y;
                if (ty == FNB_CONF) {
#pragma unroll
                    for (int c = 0; c < GV; ++c) g[f][c] = 0.5 * (wo[c] + wn[c]);
                } else if (ty == FNB_SMALL_LO || ty == FNB_SMALL_HI) {   // wn: the large side's node ln
#pragma unroll
                    for (int c = 0; c < GV; ++c) {
                        double il = 0.0;
#pragma unroll
                        for (int j = 0; j < NP; ++j) {
                            const double wj = __shfl_sync(gmask, wn[c], j, 4);
                            il = fma(ty == FNB_SMALL_LO ? cB.Plo[ln][j] : cB.Pup[ln][j], wj, il);
                        }
                        g[f][c] = 0.5 * (il + wo[c]);
                    }
                } else if (ty >= 0) {                                     // large side: wn, wn1 the smalls
                    double wn1[GV];
#if GRAD2D_LG
                    {
                        double u1[4];
                        trace2d(sb, state_src(sp, pk_member(ty)), dtc, pk_elem(ty), (2 * o + f) ^ 1, ln, u1);
                        prim_vT(u1, gm1, wn1);
                    }
#else
                    prim_vT(un[f][1], gm1, wn1);
#endif
#pragma unroll
                    for (int c = 0; c < GV; ++c) {
                        double il = 0.0, ih = 0.0;
#pragma unroll
                        for (int j = 0; j < NP; ++j) {
                            const double wj = __shfl_sync(gmask, wo[c], j, 4);
                            il = fma(cB.Plo[ln][j], wj, il);
                            ih = fma(cB.Pup[ln][j], wj, ih);
                        }
                        const double clo = 0.5 * (il + wn[c]), chi = 0.5 * (ih + wn1[c]);
                        double s = 0.0;
#pragma unroll
                        for (int j = 0; j < NP; ++j) {
                            s = fma(cB.Rlo[ln][j], __shfl_sync(gmask, clo, j, 4), s);
                            s = fma(cB.Rup[ln][j], __shfl_sync(gmask, chi, j, 4), s);
                        }
                        g[f][c] = s;
                    }
                } else {                                                  // no neighbour (unsupported for BR1)
#pragma unroll
                    for (int c = 0; c < GV; ++c) g[f][c] = wo[c];
                }
            }
#if GRAD2D_WREG
            line_gradient_w(wl, g[0], g[1], j2h, q);
#else
            line_gradient_g<GRAD2D_LS>(sm, o, lo, g[0], g[1], j2h, fld, q);
#endif
        } else {
            line_gradient<GRAD2D_LS>(sm, o, lo, ln, gst[le], j2h, fld, sc, q);
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {    // the line is contiguous and 16 B aligned: two 16 B stores; only the
                                         // velocity gradients cross directions (the flux takes T's along its line)
            *reinterpret_cast<double2 *>(&sm[G_Q + c][o][lo]) = make_double2(q[c][0], q[c][1]);
            *reinterpret_cast<double2 *>(&sm[G_Q + c][o][lo + 2]) = make_double2(q[c][2], q[c][3]);
        }
        PERK_JITTER(14);
        __syncwarp();
        if (!FUSED && has_next) issue_gs(pk_next);          // gst consumed
        cp_async_commit();
        if (FUSED && has_next) faces_of(pk_next, fn);       // the next group's face entries (used at its top)
        if (BR1_DV) {
            // viscous flux in direction o at the line's 4 nodes: the end nodes' go to Vt (face traces),
            // all four into dv[i] = sum_a Dhat_ia F^v_o(node a); x + y lines summed through shared memory
            // (fields v1, v2, T, free once every thread has read its line's velocities) -> Dv = -(2/h) dv
            double dv[NP][GV];
#pragma unroll
            for (int i = 0; i < NP; ++i)
#pragma unroll
                for (int c = 0; c < GV; ++c) dv[i][c] = 0.0;
#pragma unroll
            for (int a = 0; a < NP; ++a) {
                const int oi = o == 0 ? yo + eoy + 4 * a + ln : eox + 4 * a + ln;
                double qo[GV], qs[GV], fv[GV];
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    qs[c] = q[c][a];
                    qo[c] = c < 2 ? sm[G_Q + c][1 - o][oi] : 0.0;   // T's cross gradient is not used
                }
#if GRAD2D_WREG == 2
                const double v1 = wl[0][a], v2 = wl[1][a];
#else
                const double v1 = sm[G_V1][o][lo + a], v2 = sm[G_V2][o][lo + a];
#endif
#if VISC_LINE
                visc_flux2d_line(o, v1, v2, qs, qo, md.mu, md.kappa, fv);
#else
                if (o == 0) visc_flux2d(v1, v2, qs, qo, 0, md.mu, md.kappa, fv);
                else visc_flux2d(v1, v2, qo, qs, 1, md.mu, md.kappa, fv);
#endif
                if (valid && (a == 0 || a == NP - 1)) {
                    const int face = 2 * o + (a == NP - 1 ? 0 : 1);   // a = N: +o face, a = 0: -o face
#pragma unroll
                    for (int c = 0; c < GV; ++c) Vt[vidx2d(e, face, c, ln)] = fv[c];
                }
#pragma unroll
                for (int i = 0; i < NP; ++i)
#pragma unroll
                    for (int c = 0; c < GV; ++c) dv[i][c] = fma(cB.Dhat[i][a], fv[c], dv[i][c]);
            }
            PERK_JITTER(15);
            __syncwarp();
#if GRAD2D_DVX
            // the y-line threads hand their sums over in the y layout; the x-line threads add their own
            // (x + y, as before) and write their line's 4 nodes (half the shared-memory traffic of both
            // directions storing and every thread summing two nodes)
            if (o == 1) {
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    *reinterpret_cast<double2 *>(&sm[G_V1 + c][1][lo]) = make_double2(dv[0][c], dv[1][c]);
                    *reinterpret_cast<double2 *>(&sm[G_V1 + c][1][lo + 2]) = make_double2(dv[2][c], dv[3][c]);
                }
            }
            PERK_JITTER(16);
            __syncwarp();
            if (o == 0 && valid && sweep_idx(sp, base + le, n_act) < n_el_a) {   // halo elements (their member is inactive) need no Dv
                const double J = -j2h;
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    double s4[NP];
#pragma unroll
                    for (int a = 0; a < NP; ++a) s4[a] = J * (dv[a][c] + sm[G_V1 + c][1][yo + eoy + 4 * a + ln]);
                    double *D = Dv + (size_t)e * (GV * 16) + c * 16 + 4 * ln;
                    *reinterpret_cast<double2 *>(D) = make_double2(s4[0], s4[1]);
                    *reinterpret_cast<double2 *>(D + 2) = make_double2(s4[2], s4[3]);
                }
            }
#else
#pragma unroll
            for (int c = 0; c < GV; ++c) {
                *reinterpret_cast<double2 *>(&sm[G_V1 + c][o][lo]) = make_double2(dv[0][c], dv[1][c]);
                *reinterpret_cast<double2 *>(&sm[G_V1 + c][o][lo + 2]) = make_double2(dv[2][c], dv[3][c]);
            }
            PERK_JITTER(16);
            __syncwarp();
            if (valid && sweep_idx(sp, base + le, n_act) < n_el_a) {   // halo elements (their member is inactive) need no Dv
                const int i0 = q0 & 3, j0 = q0 >> 2;
                const double J = -j2h;
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    const double2 sx = *reinterpret_cast<const double2 *>(&sm[G_V1 + c][0][eox + q0]);
                    const double s0 = sx.x + sm[G_V1 + c][1][yo + eoy + 4 * i0 + j0];
                    const double s1 = sx.y + sm[G_V1 + c][1][yo + eoy + 4 * (i0 + 1) + j0];
#if GRAD2D_DVCS
                    __stcs(reinterpret_cast<double2 *>(Dv + (size_t)e * (GV * 16) + c * 16 + q0), make_double2(J * s0, J * s1));
#else
                    *reinterpret_cast<double2 *>(Dv + (size_t)e * (GV * 16) + c * 16 + q0) = make_double2(J * s0, J * s1);
#endif
                }
            }
#endif
        } else if (valid) {
#pragma unroll
            for (int end = 0; end < 2; ++end) {
                const int a = end ? NP - 1 : 0;
                const int oi = o == 0 ? yo + eoy + 4 * a + ln : eox + 4 * a + ln;
                double qo[GV], qs[GV], fv[GV];
#pragma unroll
                for (int c = 0; c < GV; ++c) {
                    qs[c] = q[c][a];
                    qo[c] = c < 2 ? sm[G_Q + c][1 - o][oi] : 0.0;   // T's cross gradient is not used
                }
                const double v1 = sm[G_V1][o][lo + a], v2 = sm[G_V2][o][lo + a];
#if VISC_LINE
                visc_flux2d_line(o, v1, v2, qs, qo, md.mu, md.kappa, fv);
#else
                if (o == 0) visc_flux2d(v1, v2, qs, qo, 0, md.mu, md.kappa, fv);
                else visc_flux2d(v1, v2, qo, qs, 1, md.mu, md.kappa, fv);
#endif
                const int face = 2 * o + (end ? 0 : 1);      // a = N: +o face, a = 0: -o face
#pragma unroll
                for (int c = 0; c < GV; ++c) Vt[vidx2d(e, face, c, ln)] = fv[c];
            }
        }
        __syncwarp();
        pk = pk_next;
    }
    cp_async_wait<0>();
}

}  // namespace perk
