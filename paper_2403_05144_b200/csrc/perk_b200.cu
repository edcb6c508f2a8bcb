// perk_b200.cu -- libperk_b200.so: the C ABI of include/perk.h (host side) + all device kernels.
//
// Host-side responsibilities: argument validation, tableau construction (P:l.1062; stage patterns
// and Heun / Ralston weights), capacity-sized allocations, launching the device mesh pipeline
// (mesh.cuh; captured as one graph per re-mesh), capturing one CUDA graph per P-ERK step (2 launches
// per stage: k_surf*, k_vol*; + 2 BR1 launches for Navier-Stokes; one k_step1d launch for small 1D
// meshes), the device AMR adapt (amr.cuh), profiling hooks.  No step of the method runs on the host:
// after perk_init the host never reads mesh data except in introspection calls.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "perk.h"
#include "common.cuh"
#include "basis.cuh"
#include "partition.cuh"
#include "mesh.cuh"
#include "dg1d.cuh"
#include "dg2d.cuh"
#include "br1.cuh"
#include "step1d.cuh"
#include "transfer.cuh"
#include "amr.cuh"
#include "sc.cuh"
#include "dd.cuh"

using namespace perk;

struct Prof {
    float ms[PERK_NUM_KERNEL_KINDS];
    int launches[PERK_NUM_KERNEL_KINDS];
    std::vector<cudaEvent_t> ev;
    std::vector<int> kind;
};

struct perk_ctx {
    perk_problem prob;
    perk_tableau tab;
    MeshDev md;
    int nv = 0, npe = 0, nd = 0;
    long long nmorton = 0;
    size_t nf = 0;
    int cap = 0, cap_faces = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t cap_stream = nullptr;
    double *K1 = nullptr, *Ubuf = nullptr, *Fs = nullptr, *Utmp = nullptr, *Uhost_dev = nullptr;
    double *Gs = nullptr, *Vt = nullptr;   // BR1 (Navier-Stokes): central w* and viscous-flux traces
    double *Dv = nullptr;                  // BR1_DV: viscous volume term of k_grad2d, read by k_vol2d
    double *Wb = nullptr;                  // P-ERK3: W = U_n + dt (b_1 K_1 + b_{S-1} K_{S-1})
    bool ns = false;
    bool sc = false;                       // subcell shock capturing (sc.cuh): per-stage alpha, blended volume
    ScParams scp{};
    double *alpha_raw = nullptr, *alpha = nullptr;
    bool halo_alloc = false;               // BR1 / shock-capturing halo lists allocated
    bool sc_fused = true;                  // smoothing inside k_surf2d (PERK_SC_FUSED=0: k_sc_smooth launch)
    unsigned long long act[MAXR] = {};     // evaluated stages per member (bit i-1), standard or given
    bool std_pattern = true;
    // non-nested stage patterns (2D): per-stage hot arrays [S][capacity] (elements, interfaces,
    // mortars, boundary list), so every launch covers exactly the items its stage needs
    bool stage_lists = false;
    int *st_el = nullptr, *st_bd = nullptr, *st_idx = nullptr;
    int4 *st_if = nullptr, *st_mo = nullptr;
    uint8_t *lmap = nullptr, *keys = nullptr;
    int *items = nullptr, *rank = nullptr, *blockcnt = nullptr, *blockoff = nullptr, *segtmp = nullptr;
    int *dconst = nullptr;     // [0] = nmorton
    int *n_old = nullptr, *cell_of_old = nullptr, *fx_old = nullptr, *fy_old = nullptr;
    uint8_t *lev_old = nullptr;
    double *amr_ind = nullptr;                         // AMR scratch: indicator, wanted / new level per leaf,
    uint8_t *amr_want = nullptr, *amr_newlev = nullptr;  // ping-pong finest-grid maps of the balance
    uint8_t *amr_map[2] = {nullptr, nullptr};
    int *amr_flags = nullptr;                            // balance: iteration k changed a cell
    int vol_blocks = 0, vol_blocks_sc = 0, surf_blocks = 0, grad_blocks = 0;
    int sweep = 1;               // alternate the list direction of consecutive stage kernels (PERK_SWEEP=0: off)
    unsigned kind_mask = ~0u;              // kernel kinds launch_step issues (perk_time_kernels)
    bool step1d = false;                   // small 1D mesh: whole step in one single-CTA launch
    StepTab1D *tb1d = nullptr;
    size_t step1d_smem = 0;
    cudaGraphExec_t gexec = nullptr;
    cudaGraphExec_t rexec = nullptr;       // re-mesh graph (mesh pipeline + transfer), keyed on U
    double *rU = nullptr;
    double *gU = nullptr;
    double gdt = 0.0;
    // spatial domain decomposition (dd.cuh): this context is sub-domain dd_rank of
    // dd_P; dd_P == 1 is the undecomposed path
    int dd_rank = 0, dd_P = 1;
    uint8_t *dd_owner = nullptr, *dd_flags = nullptr;  // owner rank per leaf; [2P][cap] send / ghost flags
    long long *dd_bsum = nullptr;                       // per-block weight sums (E-weighted split)
    int *dd_range = nullptr;                            // owned cells [first, first + count)
    int *dd_list[DD_MAXP][2] = {};                      // per peer: send (owned ghosts of the peer), recv lists
    int *dd_seg[DD_MAXP][2] = {};                       // their member segments
    int *dd_cnt[DD_MAXP][2] = {};                       // [2][MAXS] per-stage prefix counts (k_dd_counts)
    std::vector<void *> allocs;
    std::string err;
};

// __constant__ basis tables are per device: one upload per device a context is created on
static std::mutex g_basis_mutex;
static unsigned long long g_basis_uploaded = 0;   // bit d: uploaded on device d

static int set_err(perk_ctx *c, int code, const std::string &msg)
{
    if (c) c->err = msg;
    return code;
}

#define CU(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return set_err(c, PERK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
    } while (0)

template <class T>
static cudaError_t dalloc(perk_ctx *c, T **p, size_t n)
{
    cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (n ? n : 1));
    if (e == cudaSuccess) {
        c->allocs.push_back((void *)*p);
        cudaMemset(*p, 0, sizeof(T) * (n ? n : 1));
    }
    return e;
}

// ----------------------------------------------------------------------------------------------
// tableau
// ----------------------------------------------------------------------------------------------
extern "C" int perk_alpha_taylor(int32_t E, double *alpha)
{
    if (!alpha || E < 0 || E > PERK_MAX_STAGES) return PERK_EINVAL;
    double f = 1.0;
    alpha[0] = 1.0;
    for (int k = 1; k <= E; ++k) {
        f *= k;
        alpha[k] = 1.0 / f;
    }
    return PERK_OK;
}

extern "C" int perk_tableau_p2_ex(int32_t S, int32_t R, const int32_t *E, const double *alpha,
                                  const uint64_t *active, double c_S, perk_tableau *out)
{
    if (!E || !alpha || !out || S < 2 || S > PERK_MAX_STAGES || R < 1 || R > PERK_MAX_MEMBERS) return PERK_EINVAL;
    if (!(c_S > 0.0) || !(c_S <= 1.0)) return PERK_EINVAL;
    bool any = false;
    for (int r = 0; r < R; ++r) {
        if (E[r] < 2 || E[r] > S) return PERK_EINVAL;
        if (r > 0 && E[r] <= E[r - 1]) return PERK_EINVAL;
        if (active && active[r]) any = true;
    }
    memset(out, 0, sizeof(*out));
    out->S = S;
    out->R = R;
    const double bS = 1.0 / (2.0 * c_S);
    out->b[S - 1] = bS;                        // b = e_S for c_S = 1/2 (P:l.423); Heun / Ralston (P:l.439-442)
    out->b[0] += 1.0 - bS;
    for (int i = 1; i <= S; ++i)
        out->c[i - 1] = c_S == 0.5 ? (double)(i - 1) / (double)(2 * (S - 1)) : c_S * (double)(i - 1) / (double)(S - 1);
    for (int r = 0; r < R; ++r) {
        out->E[r] = E[r];
        unsigned long long act = 1ull;
        if (any) {
            act = active[r];
            const unsigned long long allowed = S == 64 ? ~0ull : ((1ull << S) - 1ull);
            if ((act & ~allowed) || !(act & 1ull) || !((act >> (S - 1)) & 1ull) || __builtin_popcountll(act) != E[r])
                return PERK_EINVAL;
            out->active[r] = act;
        } else {
            for (int i = S - E[r] + 2; i <= S; ++i) act |= 1ull << (i - 1);
        }
        // chain of evaluated stages after 1: s[1] < ... < s[E-1] = S
        int st[PERK_MAX_STAGES + 1], ns = 0;
        for (int i = 2; i <= S; ++i)
            if ((act >> (i - 1)) & 1ull) st[++ns] = i;
        const double *al = alpha + (size_t)r * (S + 1);
        double a[PERK_MAX_STAGES + 1] = {0};   // chain position k -> a_k
        // a_{E-1-i} = alpha_{3+i} / (b_S c_{s_{E-2-i}} prod_{m<i} a_{E-1-m}),  i = 0..E-3   (P:l.1058-1064)
        for (int i = 0; i <= E[r] - 3; ++i) {
            const int k = E[r] - 1 - i;
            double prod = 1.0;
            for (int m = E[r] - 1; m >= k + 1; --m) prod *= a[m];
            const double den = bS * out->c[st[k - 1] - 1] * prod;
            if (den == 0.0) return PERK_EINVAL;
            a[k] = al[3 + i] / den;
        }
        for (int k = 2; k <= E[r] - 1; ++k) out->a_sub[r][st[k] - 1] = a[k];
    }
    return PERK_OK;
}

extern "C" int perk_pattern_mask(int32_t S, int32_t E, int32_t kind, const int32_t *stages, int32_t n_stages,
                                 uint64_t *mask_out)
{
    if (!mask_out || S < 2 || S > PERK_MAX_STAGES || E < 2 || E > S) return PERK_EINVAL;
    unsigned long long m = 0;
    switch (kind) {
    case PERK_PATTERN_STANDARD:
        m = 1ull;
        for (int i = S - E + 2; i <= S; ++i) m |= 1ull << (i - 1);
        break;
    case PERK_PATTERN_EARLY:
        for (int i = 1; i <= E - 1; ++i) m |= 1ull << (i - 1);
        m |= 1ull << (S - 1);
        break;
    case PERK_PATTERN_ALTERNATING:
        // S - floor((E-1-k)(S-1)/(E-1) + 1/2) in integers: floor((2(E-1-k)(S-1) + (E-1)) / (2(E-1)))
        m = 1ull;
        for (int k = 1; k <= E - 1; ++k) {
            const long long num = 2ll * (E - 1 - k) * (S - 1) + (E - 1);
            m |= 1ull << (S - (int)(num / (2ll * (E - 1))) - 1);
        }
        break;
    case PERK_PATTERN_EXPLICIT:
        if (!stages || n_stages != E) return PERK_EINVAL;
        for (int k = 0; k < n_stages; ++k) {
            const int i = stages[k];
            if (i < 1 || i > S || ((m >> (i - 1)) & 1ull)) return PERK_EINVAL;
            m |= 1ull << (i - 1);
        }
        if (!(m & 1ull) || !((m >> (S - 1)) & 1ull)) return PERK_EINVAL;
        break;
    default:
        return PERK_EINVAL;
    }
    if (__builtin_popcountll(m) != E) return PERK_EINVAL;   // e.g. an alternating rule collision
    *mask_out = m;
    return PERK_OK;
}

extern "C" int perk_tableau_p2(int32_t S, int32_t R, const int32_t *E, const double *alpha, perk_tableau *out)
{
    return perk_tableau_p2_ex(S, R, E, alpha, nullptr, 0.5, out);
}

// ----------------------------------------------------------------------------------------------
// partition launcher
// ----------------------------------------------------------------------------------------------
static ActiveDesc active_desc(const perk_ctx *c)
{
    ActiveDesc ad;
    ad.S = c->tab.S;
    ad.R = c->tab.R;
    for (int r = 0; r < MAXR; ++r) {
        ad.E[r] = r < c->tab.R ? c->tab.E[r] : 0;
        ad.act[r] = r < c->tab.R ? c->act[r] : 0ull;
    }
    return ad;
}

static void prof_mark(Prof *p, cudaStream_t s, int kind)
{
    if (!p) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    p->ev.push_back(e);
    p->kind.push_back(kind);
}

template <class KeyFn>
static void partition(perk_ctx *c, cudaStream_t s, KeyFn kf, const int *n_ptr, int mult, long long max_items, int R,
                      int *out, int *rank, int *seg, int *total_out, int *count_active,
                      unsigned long long *evals_per_step = nullptr)
{
    int nb = (int)((max_items + PART_T - 1) / PART_T);
    if (nb < 1) nb = 1;
    k_part_count<<<nb, PART_T, 0, s>>>(kf, n_ptr, mult, R, c->blockcnt);
    k_part_offsets<<<1, PART_OFF_T, 0, s>>>(c->blockcnt, nb, R, c->blockoff, seg, total_out, active_desc(c), count_active,
                                        evals_per_step);
    k_part_scatter<<<nb, PART_T, 0, s>>>(kf, n_ptr, mult, R, c->blockoff, out, rank);
}

__global__ void k_set_count(int *dst, const int *seg, int idx) { *dst = seg[idx + 1] - seg[idx]; }

// launch with programmatic stream serialisation (PDL): the kernels call pdl_wait() (common.cuh)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, args...);
}

static int blocks_for(long long n, int t)
{
    long long b = (n + t - 1) / t;
    return (int)(b < 1 ? 1 : b);
}

// level map (device) -> leaves, faces, per-member lists, stage prefix tables; all asynchronous
static void build_mesh(perk_ctx *c, cudaStream_t s, const uint8_t *lmap)
{
    MeshDev &md = c->md;
    const int R = c->tab.R;
    k_leaf_flags<<<blocks_for(c->nmorton, 256), 256, 0, s>>>(md, lmap, c->nmorton, c->keys);
    partition(c, s, KeyU8{c->keys}, c->dconst, 1, c->nmorton, 2, c->items, c->rank, c->segtmp, nullptr, nullptr);
    k_set_count<<<1, 1, 0, s>>>(md.n, c->segtmp, 0);
    k_check_capacity<<<1, 1, 0, s>>>(md);
    k_leaf_fill<<<blocks_for(c->cap, 256), 256, 0, s>>>(md, lmap, c->items, R);
    k_cell_of<<<blocks_for((long long)c->nf, 256), 256, 0, s>>>(md, lmap, c->rank);
    const bool dd = c->dd_P > 1;
    const int ddr = c->dd_rank;
    if (dd) {   // E-weighted contiguous Morton ranges (dd.cuh)
        const int nb = blocks_for(c->cap, DD_SCAN_T);
        k_dd_block_sums<<<nb, DD_SCAN_T, 0, s>>>(md, active_desc(c), c->dd_bsum);
        k_dd_scan_blocks<<<1, DD_SCAN_T, 0, s>>>(md.n, c->dd_bsum);
        k_dd_range_init<<<1, 1, 0, s>>>(md.n, c->dd_range);
        k_dd_owner<<<nb, DD_SCAN_T, 0, s>>>(md, active_desc(c), c->dd_bsum, c->dd_P, ddr, c->dd_owner, c->dd_range);
    }
    k_classify<<<blocks_for((long long)c->nd * c->cap, 256), 256, 0, s>>>(md, c->keys);
    partition(c, s, KeyU8{c->keys}, md.n, c->nd, (long long)c->nd * c->cap, 4, c->items, nullptr, c->segtmp, nullptr,
              nullptr);
    k_face_counts<<<1, 1, 0, s>>>(md, c->segtmp, c->cap_faces);
    k_face_records<<<blocks_for((long long)c->nd * c->cap, 256), 256, 0, s>>>(md, c->items, c->segtmp, R);
    if (md.fnb) k_face_table<<<SM_COUNT_B200 * 8, 256, 0, s>>>(md);   // fused BR1 (Navier-Stokes)
    if (dd) {   // a sub-domain keeps its owned elements and the faces with an owned side
        const uint8_t *ow = c->dd_owner;
        partition(c, s, KeyOwnEl{md.mem, ow, ddr}, md.n + 0, 1, c->cap, R, md.list[KIND_EL], nullptr,
                  md.seg + 0 * (MAXR + 1), nullptr, md.count_active + KIND_EL * MAXS, md.evals + 2);
        partition(c, s, KeyOwnIfc{md.ifc, ow, ddr}, md.n + 1, 1, c->cap_faces, R, md.list[KIND_IF], nullptr,
                  md.seg + 1 * (MAXR + 1), nullptr, md.count_active + KIND_IF * MAXS);
        partition(c, s, KeyOwnMor{md.mor, ow, ddr}, md.n + 2, 1, c->cap_faces, R, md.list[KIND_MO], nullptr,
                  md.seg + 2 * (MAXR + 1), nullptr, md.count_active + KIND_MO * MAXS);
        partition(c, s, KeyOwnBnd{md.bnd, ow, ddr}, md.n + 3, 1, c->cap_faces, R, md.list[KIND_BD], nullptr,
                  md.seg + 3 * (MAXR + 1), nullptr, md.count_active + KIND_BD * MAXS);
    } else {
        partition(c, s, KeyU8{md.mem}, md.n + 0, 1, c->cap, R, md.list[KIND_EL], nullptr, md.seg + 0 * (MAXR + 1),
                  nullptr, md.count_active + KIND_EL * MAXS, md.evals + 2);
        partition(c, s, KeyIfc{md.ifc}, md.n + 1, 1, c->cap_faces, R, md.list[KIND_IF], nullptr,
                  md.seg + 1 * (MAXR + 1), nullptr, md.count_active + KIND_IF * MAXS);
        partition(c, s, KeyMor{md.mor}, md.n + 2, 1, c->cap_faces, R, md.list[KIND_MO], nullptr,
                  md.seg + 2 * (MAXR + 1), nullptr, md.count_active + KIND_MO * MAXS);
        partition(c, s, KeyBnd{md.bnd}, md.n + 3, 1, c->cap_faces, R, md.list[KIND_BD], nullptr,
                  md.seg + 3 * (MAXR + 1), nullptr, md.count_active + KIND_BD * MAXS);
    }
    k_hot_lists<<<blocks_for(c->cap_faces, 256), 256, 0, s>>>(md, R);
    if (dd) {   // ghost layers: per peer the owned cells it reads (send) and its cells read here (recv)
        cudaMemsetAsync(c->dd_flags, 0, (size_t)2 * c->dd_P * c->cap, s);
        k_dd_flags<<<SM_COUNT_B200 * 4, 256, 0, s>>>(md, c->dd_owner, ddr, c->dd_flags);
        for (int q = 0; q < c->dd_P; ++q) {
            if (q == ddr) continue;
            for (int d = 0; d < 2; ++d) {
                partition(c, s, KeyFlagMem{c->dd_flags + (size_t)(2 * q + d) * c->cap, md.mem}, md.n + 0, 1, c->cap, R,
                          c->dd_list[q][d], nullptr, c->dd_seg[q][d], nullptr, nullptr);
                k_dd_counts<<<1, MAXS, 0, s>>>(c->dd_seg[q][d], active_desc(c), c->dd_cnt[q][d]);
            }
        }
    }
    if (c->stage_lists) {   // per-stage lists (non-nested patterns): stable compaction per (stage, kind)
        for (int i = 1; i <= c->tab.S; ++i) {
            unsigned mask = 0;
            for (int r = 0; r < R; ++r)
                if ((c->act[r] >> (i - 1)) & 1ull) mask |= 1u << r;
            const size_t oc = (size_t)(i - 1) * c->cap, of = (size_t)(i - 1) * c->cap_faces;
            int *ca = md.count_active;
            partition(c, s, KeyStageEl{md.elpk, mask}, md.n + 0, 1, c->cap, 1, c->st_idx, nullptr, c->segtmp, nullptr, nullptr);
            k_stage_gather<<<blocks_for(c->cap, 256), 256, 0, s>>>(c->segtmp, c->st_idx, KIND_EL, md, c->st_el + oc, nullptr, nullptr);
            k_set_count<<<1, 1, 0, s>>>(ca + KIND_EL * MAXS + i - 1, c->segtmp, 0);
            partition(c, s, KeyStageIf{md.ifcs, mask}, md.n + 1, 1, c->cap_faces, 1, c->st_idx, nullptr, c->segtmp, nullptr, nullptr);
            k_stage_gather<<<blocks_for(c->cap_faces, 256), 256, 0, s>>>(c->segtmp, c->st_idx, KIND_IF, md, nullptr, c->st_if + of, nullptr);
            k_set_count<<<1, 1, 0, s>>>(ca + KIND_IF * MAXS + i - 1, c->segtmp, 0);
            partition(c, s, KeyStageMo{md.mors, md.mem, mask}, md.n + 2, 1, c->cap_faces, 1, c->st_idx, nullptr, c->segtmp, nullptr, nullptr);
            k_stage_gather<<<blocks_for(c->cap_faces, 256), 256, 0, s>>>(c->segtmp, c->st_idx, KIND_MO, md, nullptr, c->st_mo + of, nullptr);
            k_set_count<<<1, 1, 0, s>>>(ca + KIND_MO * MAXS + i - 1, c->segtmp, 0);
            partition(c, s, KeyStageBd{md.list[KIND_BD], md.bnd, mask}, md.n + 3, 1, c->cap_faces, 1, c->st_idx, nullptr, c->segtmp, nullptr, nullptr);
            k_stage_gather<<<blocks_for(c->cap_faces, 256), 256, 0, s>>>(c->segtmp, c->st_idx, KIND_BD, md, nullptr, nullptr, c->st_bd + of);
            k_set_count<<<1, 1, 0, s>>>(ca + KIND_BD * MAXS + i - 1, c->segtmp, 0);
        }
    }
    if (c->halo_alloc) {   // BR1 / shock-capturing halo lists (see MeshDev::halo)
        k_halo_clear<<<blocks_for(c->cap, 256), 256, 0, s>>>(md);
        k_halo_flags<<<blocks_for(c->cap_faces, 256), 256, 0, s>>>(md);
        if (dd) {   // the halo elements this sub-domain owns (others' gradients arrive with Vt)
            partition(c, s, KeyOwnHaloEl{md.halo, md.mem, c->dd_owner, ddr}, md.n + 0, 1, c->cap, R, md.hlist[KIND_EL],
                      nullptr, md.hseg + KIND_EL * (MAXR + 1), nullptr, nullptr);
            partition(c, s, KeyOwnHaloIf{md.ifc, md.halo, c->dd_owner, ddr}, md.n + 1, 1, c->cap_faces, R,
                      md.hlist[KIND_IF], nullptr, md.hseg + KIND_IF * (MAXR + 1), nullptr, nullptr);
            partition(c, s, KeyOwnHaloMo{md.mor, md.halo, c->dd_owner, ddr}, md.n + 2, 1, c->cap_faces, R,
                      md.hlist[KIND_MO], nullptr, md.hseg + KIND_MO * (MAXR + 1), nullptr, nullptr);
        } else {
            partition(c, s, KeyHaloEl{md.halo, md.mem}, md.n + 0, 1, c->cap, R, md.hlist[KIND_EL], nullptr,
                      md.hseg + KIND_EL * (MAXR + 1), nullptr, nullptr);
            partition(c, s, KeyHaloIf{md.ifc, md.halo}, md.n + 1, 1, c->cap_faces, R, md.hlist[KIND_IF], nullptr,
                      md.hseg + KIND_IF * (MAXR + 1), nullptr, nullptr);
            partition(c, s, KeyHaloMo{md.mor, md.halo}, md.n + 2, 1, c->cap_faces, R, md.hlist[KIND_MO], nullptr,
                      md.hseg + KIND_MO * (MAXR + 1), nullptr, nullptr);
        }
        k_halo_ranges<<<SM_COUNT_B200, 256, 0, s>>>(md, active_desc(c));
    }
}

// ----------------------------------------------------------------------------------------------
// stage launches
// ----------------------------------------------------------------------------------------------
static StageParams stage_params(const perk_ctx *c, int i, double dt, int mode, unsigned mask)
{
    StageParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.stage = i;
    sp.S = c->tab.S;
    sp.R = c->tab.R;
    sp.mode = mode;
    sp.mask = mask;
    sp.dt = dt;
    sp.c_stage = c->tab.c[i - 1];
    sp.bS = c->tab.b[c->tab.S - 1];
    sp.wb1 = c->tab.b[0];
    sp.wbS1 = c->tab.b[c->tab.S - 2];
    sp.wmode = (c->Wb && i == c->tab.S - 1) ? 1 : 0;
    sp.fin_k1 = (!c->Wb && i == c->tab.S && c->tab.b[0] != 0.0) ? 1 : 0;
    for (int r = 0; r < c->tab.R; ++r) {
        const unsigned long long a = c->act[r];
        if ((a >> (i - 1)) & 1ull) sp.actmask |= 1u << r;
        // stage i state in Ubuf: evaluated at i and at some stage in (1, i)
        if (i > 1 && ((a >> (i - 1)) & 1ull) && (a & (((1ull << (i - 1)) - 1ull) & ~1ull))) sp.bufmask |= 1u << r;
        // after evaluating stage i: the state of the next evaluated stage n,
        // U^(n) = U_n + dt (a_{n,1} K_1 + a_{n,i} K_i)   (standard pattern: n = i + 1)
        int n = 0;
        for (int j = i + 1; j <= c->tab.S; ++j)
            if ((a >> (j - 1)) & 1ull) { n = j; break; }
        if (n) {
            sp.asub_next[r] = c->tab.a_sub[r][n - 1];
            sp.a1_next[r] = c->tab.c[n - 1] - c->tab.a_sub[r][n - 1];
        }
    }
    return sp;
}

// the mesh view of one launch: for non-nested stage patterns, a stage launch reads the stage's own
// hot arrays (count_active then holds their lengths); otherwise the shared member-sorted arrays
static MeshDev stage_mesh(const perk_ctx *c, const StageParams &sp)
{
    MeshDev md = c->md;
    if (c->stage_lists && sp.mode == MODE_STAGE) {
        const size_t oc = (size_t)(sp.stage - 1) * c->cap, of = (size_t)(sp.stage - 1) * c->cap_faces;
        md.elpk = c->st_el + oc;
        md.ifcs = c->st_if + of;
        md.mors = c->st_mo + of;
        md.list[KIND_BD] = c->st_bd + of;
    }
    return md;
}

static void launch_surface(perk_ctx *c, cudaStream_t s, const StageParams &sp, const double *Un, const double *Uin)
{
    const MeshDev md = stage_mesh(c, sp);
    if (c->prob.dim == 2) {
        const bool st = sp.mode == MODE_STAGE;
        const bool scs = c->sc && c->scp.smooth && c->sc_fused;   // shock-capturing smoothing rides along
        const double *vt = c->ns ? c->Vt : nullptr;
        const double *ar = c->alpha_raw;
        double *al = c->alpha;
        if (c->ns)   // (Navier-Stokes smooths in k_sc_smooth: fused, the 80-register budget spilled)
            launch_pdl(st ? k_surf2d<MODE_STAGE, true> : k_surf2d<MODE_RHS, true>, c->surf_blocks, 256, 0, s, md, sp, Un, (const double *)c->Ubuf, (const double *)c->K1, Uin, c->Fs, vt, ar, al);
        else if (scs)
            launch_pdl(st ? k_surf2d<MODE_STAGE, false, true> : k_surf2d<MODE_RHS, false, true>, c->surf_blocks, 256, 0, s, md, sp, Un, (const double *)c->Ubuf, (const double *)c->K1, Uin, c->Fs, vt, ar, al);
        else
            launch_pdl(st ? k_surf2d<MODE_STAGE, false> : k_surf2d<MODE_RHS, false>, c->surf_blocks, 256, 0, s, md, sp, Un, (const double *)c->Ubuf, (const double *)c->K1, Uin, c->Fs, vt, ar, al);
    } else if (c->nv == 1) {
        if (sp.mode == MODE_STAGE)
            k_surf1d<1, MODE_STAGE><<<c->surf_blocks, 256, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, Uin, c->Fs);
        else
            k_surf1d<1, MODE_RHS><<<c->surf_blocks, 256, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, Uin, c->Fs);
    } else {
        if (sp.mode == MODE_STAGE)
            k_surf1d<3, MODE_STAGE><<<c->surf_blocks, 256, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, Uin, c->Fs);
        else
            k_surf1d<3, MODE_RHS><<<c->surf_blocks, 256, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, Uin, c->Fs);
    }
}

static void launch_volume(perk_ctx *c, cudaStream_t s, const StageParams &sp, double *Un, const double *Uin, double *dU)
{
    const MeshDev md = stage_mesh(c, sp);
    if (c->prob.dim == 2) {
        double *al = c->alpha;
        const bool st = sp.mode == MODE_STAGE;
        const int tn = vol2d_threads(c->ns);
        const size_t sm = vol2d_smem_bytes(c->ns);
        if (c->ns && c->sc)
            launch_pdl(st ? k_vol2d<MODE_STAGE, true, true> : k_vol2d<MODE_RHS, true, true>, c->vol_blocks_sc, tn, sm, s, md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, (const double *)(BR1_DV ? c->Dv : c->Gs), c->Wb, al, c->alpha_raw, c->scp);
        else if (c->ns)
            launch_pdl(st ? k_vol2d<MODE_STAGE, true> : k_vol2d<MODE_RHS, true>, c->vol_blocks, tn, sm, s, md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, (const double *)(BR1_DV ? c->Dv : c->Gs), c->Wb, al, c->alpha_raw, c->scp);
        else if (c->sc)
            launch_pdl(st ? k_vol2d<MODE_STAGE, false, true> : k_vol2d<MODE_RHS, false, true>, c->vol_blocks_sc, tn, sm, s, md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, (const double *)nullptr, c->Wb, al, c->alpha_raw, c->scp);
        else
            launch_pdl(st ? k_vol2d<MODE_STAGE, false> : k_vol2d<MODE_RHS, false>, c->vol_blocks, tn, sm, s, md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, (const double *)nullptr, c->Wb, al, c->alpha_raw, c->scp);
    } else if (c->nv == 1) {
        if (sp.mode == MODE_STAGE)
            k_vol1d<1, MODE_STAGE><<<c->vol_blocks, 128, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, c->Wb);
        else
            k_vol1d<1, MODE_RHS><<<c->vol_blocks, 128, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, c->Wb);
    } else {
        if (sp.mode == MODE_STAGE)
            k_vol1d<3, MODE_STAGE><<<c->vol_blocks, 128, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, c->Wb);
        else
            k_vol1d<3, MODE_RHS><<<c->vol_blocks, 128, 0, s>>>(md, sp, Un, c->Ubuf, c->K1, c->Fs, Uin, dU, c->Wb);
    }
}

// shock capturing (sc.cuh): blending factors of the stage's elements, then neighbour smoothing
static void launch_sc(perk_ctx *c, cudaStream_t s, const StageParams &sp, const double *Un, const double *Uin, Prof *p,
                      bool smooth_kernel = false)
{
    prof_mark(p, s, 6);
    if (!((c->kind_mask >> 6) & 1u)) return;
    const int ga = std::min(blocks_for(c->cap, AMR_T / 16), SM_COUNT_B200 * 4);   // persistent: 4 CTAs per SM
    if (sp.mode == MODE_STAGE)
        launch_pdl(k_sc_alpha<MODE_STAGE>, ga, AMR_T, 0, s, c->md, sp, c->scp, Un, (const double *)c->Ubuf, (const double *)c->K1, Uin, c->alpha_raw, c->alpha);
    else
        launch_pdl(k_sc_alpha<MODE_RHS>, ga, AMR_T, 0, s, c->md, sp, c->scp, Un, (const double *)c->Ubuf, (const double *)c->K1, Uin, c->alpha_raw, c->alpha);
    if (!c->scp.smooth || (c->sc_fused && !smooth_kernel)) return;   // fused: k_surf2d smooths
    prof_mark(p, s, 6);                   // the smoothing kernel: its own segment (one launch each)
    const int gs = std::min(blocks_for(c->cap_faces, 256), SM_COUNT_B200 * 8);
    if (sp.mode == MODE_STAGE)
        launch_pdl(k_sc_smooth<MODE_STAGE>, gs, 256, 0, s, c->md, sp, (const double *)c->alpha_raw, c->alpha);
    else
        launch_pdl(k_sc_smooth<MODE_RHS>, gs, 256, 0, s, c->md, sp, (const double *)c->alpha_raw, c->alpha);
}

// BR1 passes (Navier-Stokes): central gradient traces, then gradients + viscous-flux traces
static void launch_br1(perk_ctx *c, cudaStream_t s, const StageParams &sp, const double *Un, const double *Uin, Prof *p)
{
    const MeshDev &md = c->md;
    if (!BR1_FUSED) prof_mark(p, s, 4);   // (the profile counts one launch per marked segment)
    if (BR1_FUSED || !((c->kind_mask >> 4) & 1u)) {   // fused: k_grad2d forms the central traces itself
    } else if (sp.mode == MODE_STAGE)
        launch_pdl(k_gsurf2d<MODE_STAGE>, c->surf_blocks, 256, 0, s, md, sp, Un, c->Ubuf, c->K1, Uin, c->Gs);
    else
        launch_pdl(k_gsurf2d<MODE_RHS>, c->surf_blocks, 256, 0, s, md, sp, Un, c->Ubuf, c->K1, Uin, c->Gs);
    prof_mark(p, s, 5);
    if (!((c->kind_mask >> 5) & 1u)) {
    } else if (sp.mode == MODE_STAGE)
        launch_pdl(k_grad2d<MODE_STAGE>, c->grad_blocks, 128, grad2d_smem_bytes(), s, md, sp, Un, c->Ubuf, c->K1, Uin, c->Gs, c->Vt, c->Dv);
    else
        launch_pdl(k_grad2d<MODE_RHS>, c->grad_blocks, 128, grad2d_smem_bytes(), s, md, sp, Un, c->Ubuf, c->K1, Uin, c->Gs, c->Vt, c->Dv);
}

static void launch_step(perk_ctx *c, cudaStream_t s, double *U, double dt, Prof *p)
{
    if (c->step1d) {
        prof_mark(p, s, 1);
        if ((c->kind_mask >> 1) & 1u) {
            if (c->nv == 1) k_step1d<1><<<1, step1d_threads(1), c->step1d_smem, s>>>(c->md, c->tb1d, U, dt, c->Wb != nullptr);
            else k_step1d<3><<<1, step1d_threads(3), c->step1d_smem, s>>>(c->md, c->tb1d, U, dt, c->Wb != nullptr);
        }
        prof_mark(p, s, -1);
        return;
    }
    // alternating sweep direction (StageParams::rev): every gradient / surface / volume launch of the step
    // walks its lists opposite to the launch before it, so it starts where the L2 is still warm
    // (graphs restricted to one kernel kind -- perk_time_kernels -- keep every launch forward: consecutive
    // launches of one kind re-read the same arrays, and sweeping them back and forth would show a reuse
    // the step does not have)
    int k = 0;
    const bool sweep = c->sweep && (c->kind_mask & 3u) == 3u;
    auto dir = [&](StageParams sp) { sp.rev = sweep ? (k++ & 1) : 0; return sp; };
    for (int i = 1; i <= c->tab.S; ++i) {
        const StageParams sp = stage_params(c, i, dt, MODE_STAGE, 0u);
        if (c->sc) launch_sc(c, s, sp, U, nullptr, p);
        if (c->ns) launch_br1(c, s, dir(sp), U, nullptr, p);
        prof_mark(p, s, 0);
        if ((c->kind_mask >> 0) & 1u) launch_surface(c, s, dir(sp), U, nullptr);
        prof_mark(p, s, 1);
        if ((c->kind_mask >> 1) & 1u) launch_volume(c, s, dir(sp), U, nullptr, nullptr);
        prof_mark(p, s, -1);
    }
}

// halo lists (MeshDev::halo): BR1 gradients and shock-capturing blending factors of the neighbours
// of active elements across mortars
static int alloc_halo(perk_ctx *c)
{
    if (c->halo_alloc) return PERK_OK;
    MeshDev &md = c->md;
    CU(dalloc(c, &md.halo, c->cap));
    CU(dalloc(c, &md.hlist[KIND_EL], c->cap));
    CU(dalloc(c, &md.hlist[KIND_IF], c->cap_faces));
    CU(dalloc(c, &md.hlist[KIND_MO], c->cap_faces));
    CU(dalloc(c, &md.hseg, 3 * (MAXR + 1)));
    CU(dalloc(c, &md.hrng, 3 * MAXS));
    CU(dalloc(c, &md.hpk, c->cap));
    c->halo_alloc = true;
    return PERK_OK;
}

static int check_device_err(perk_ctx *c)
{
    CU(cudaStreamSynchronize(c->stream));
    int e = 0;
    CU(cudaMemcpy(&e, c->md.err, sizeof(int), cudaMemcpyDeviceToHost));
    if (e) {
        int z = 0;
        CU(cudaMemcpy(c->md.err, &z, sizeof(int), cudaMemcpyHostToDevice));
        // capacity first: an overflowing mesh is truncated, which the later checks then also flag
        if (e & ERR_CAPACITY) return set_err(c, PERK_ECAPACITY, "cell / face capacity exceeded");
        if (e & ERR_UNBALANCED) return set_err(c, PERK_EUNBALANCED, "level map not block-aligned or not 2:1 face balanced");
        if (e & ERR_TRANSFER) return set_err(c, PERK_EUNBALANCED, "re-mesh changed a level by more than one");
    }
    return PERK_OK;
}

// ----------------------------------------------------------------------------------------------
// C ABI
// ----------------------------------------------------------------------------------------------
static int validate(perk_ctx *c, const perk_problem *p, const perk_tableau *t)
{
    if (p->dim != 1 && p->dim != 2) return set_err(c, PERK_EINVAL, "dim must be 1 or 2");
    if (p->n_base[0] < 1 || (p->dim == 2 && p->n_base[1] < 1)) return set_err(c, PERK_EINVAL, "n_base");
    if (p->max_level < 0 || p->max_level > 12) return set_err(c, PERK_EINVAL, "max_level");
    if (p->max_cells < 1 || p->max_cells > (1ll << 24)) return set_err(c, PERK_EINVAL, "max_cells must be in [1, 2^24]");
    if (p->dim == 1) {
        if (p->equation == PERK_EQ_ADVECTION) {
            if (p->surface != PERK_FLUX_UPWIND) return set_err(c, PERK_EUNSUPPORTED, "1D advection uses the upwind flux");
        } else if (p->equation == PERK_EQ_EULER) {
            if (p->surface != PERK_FLUX_RUSANOV) return set_err(c, PERK_EUNSUPPORTED, "1D Euler uses the Rusanov flux");
        } else {
            return set_err(c, PERK_EUNSUPPORTED, "1D supports advection and Euler");
        }
        if (p->volume != PERK_VOL_WEAK) return set_err(c, PERK_EUNSUPPORTED, "1D uses the weak form");
    } else {
        if (p->equation == PERK_EQ_NAVIER_STOKES) {
            if (!p->periodic[0] || !p->periodic[1])
                return set_err(c, PERK_EUNSUPPORTED, "Navier-Stokes (BR1) needs a periodic domain (no viscous boundary fluxes)");
            if (!(p->mu >= 0.0) || !(p->prandtl > 0.0)) return set_err(c, PERK_EINVAL, "mu >= 0 and prandtl > 0 required");
        } else if (p->equation != PERK_EQ_EULER) {
            return set_err(c, PERK_EUNSUPPORTED, "2D supports Euler and Navier-Stokes");
        }
        if (p->volume != PERK_VOL_FLUXDIFF) return set_err(c, PERK_EUNSUPPORTED, "2D uses flux differencing");
        if (p->surface != PERK_FLUX_HLL && p->surface != PERK_FLUX_RUSANOV) return set_err(c, PERK_EUNSUPPORTED, "2D surface flux");
        const double hx = (p->domain_hi[0] - p->domain_lo[0]) / p->n_base[0];
        const double hy = (p->domain_hi[1] - p->domain_lo[1]) / p->n_base[1];
        if (!(hx > 0) || std::fabs(hx - hy) > 1e-12 * hx) return set_err(c, PERK_EINVAL, "2D cells must be square");
    }
    if (!(p->domain_hi[0] > p->domain_lo[0])) return set_err(c, PERK_EINVAL, "domain");
    if (t->S < 2 || t->S > PERK_MAX_STAGES || t->R < 1 || t->R > PERK_MAX_MEMBERS) return set_err(c, PERK_EINVAL, "S/R");
    for (int r = 0; r < t->R; ++r) {
        if (t->E[r] < 2 || t->E[r] > t->S || (r > 0 && t->E[r] <= t->E[r - 1]))
            return set_err(c, PERK_EINVAL, "E must be ascending in [2, S]");
    }
    // shared weights: nonzero only at stages 1, S-1, S, summing to 1 (b^T 1 = 1, P:l.236)
    double bsum = 0.0;
    for (int i = 0; i < t->S; ++i) {
        if (t->b[i] != 0.0 && i != 0 && i != t->S - 2 && i != t->S - 1)
            return set_err(c, PERK_EUNSUPPORTED, "b may be nonzero only at stages 1, S-1, S");
        bsum += t->b[i];
    }
    if (std::fabs(bsum - 1.0) > 1e-14) return set_err(c, PERK_EINVAL, "b must sum to 1");
    // stage patterns: all zero = standard, else every member's set holds 1 and S and E[r] stages
    bool any = false;
    for (int r = 0; r < t->R; ++r) any |= t->active[r] != 0;
    unsigned long long act[MAXR] = {};
    for (int r = 0; r < t->R; ++r) {
        if (!any) {
            act[r] = 1ull;
            for (int i = t->S - t->E[r] + 2; i <= t->S; ++i) act[r] |= 1ull << (i - 1);
        } else {
            act[r] = t->active[r];
            const unsigned long long allowed = t->S == 64 ? ~0ull : ((1ull << t->S) - 1ull);
            if ((act[r] & ~allowed) || !(act[r] & 1ull) || !((act[r] >> (t->S - 1)) & 1ull) ||
                __builtin_popcountll(act[r]) != t->E[r])
                return set_err(c, PERK_EINVAL, "active[r] must hold stages 1 and S and E[r] stages in [1, S]");
        }
        for (int i = 1; i <= t->S; ++i) {       // a_{i,p(i)} only at evaluated stages with a predecessor > 1
            const bool ok = i > 1 && ((act[r] >> (i - 1)) & 1ull) && (act[r] & (((1ull << (i - 1)) - 1ull) & ~1ull));
            if (t->a_sub[r][i - 1] != 0.0 && !ok)
                return set_err(c, PERK_EINVAL, "a_sub[r][i-1] != 0 at a stage without an evaluated predecessor > 1");
        }
    }
    // b_{S-1} != 0 (P-ERK3): W = U_n + dt (b_1 K_1 + b_{S-1} K_{S-1}) is formed in the stage S-1 epilogue;
    // b_1 alone (Heun / Ralston) is added at stage S
    if (t->S >= 3 && t->b[t->S - 2] != 0.0)
        for (int r = 0; r < t->R; ++r)
            if (!((act[r] >> (t->S - 2)) & 1ull))
                return set_err(c, PERK_EINVAL, "b_{S-1} != 0 needs every member to evaluate stage S-1");
    if (c) {
        for (int r = 0; r < MAXR; ++r) c->act[r] = r < t->R ? act[r] : 0ull;
        c->std_pattern = !any;
    }
    return PERK_OK;
}

extern "C" int perk_init(perk_ctx **out, const perk_problem *prob, const uint8_t *level_map_dev, const perk_tableau *tab,
                         void *stream)
{
    return perk_init_dd(out, prob, level_map_dev, tab, stream, 0, 1);
}

extern "C" int perk_init_dd(perk_ctx **out, const perk_problem *prob, const uint8_t *level_map_dev,
                            const perk_tableau *tab, void *stream, int32_t rank, int32_t nranks)
{
    if (!out || !prob || !level_map_dev || !tab) return PERK_EINVAL;
    *out = nullptr;
    perk_ctx *c = new perk_ctx();
    // the handle is returned on every path from here on, so that a caller can read perk_last_error
    // and release the partially built context (streams, device buffers) with perk_destroy
    *out = c;
    int rc = validate(c, prob, tab);
    if (rc) return rc;
    if (nranks < 1 || nranks > DD_MAXP || rank < 0 || rank >= nranks)
        return set_err(c, PERK_EINVAL, "need 1 <= nranks <= 8 and 0 <= rank < nranks");
    if (nranks > 1 && (prob->dim != 2 || !c->std_pattern))
        return set_err(c, PERK_EUNSUPPORTED, "domain decomposition: 2D problems with the standard stage pattern");
    c->dd_rank = rank;
    c->dd_P = nranks;
    c->prob = *prob;
    c->tab = *tab;
    c->stream = (cudaStream_t)stream;
    const int dim = prob->dim, L = prob->max_level;
    c->nv = prob->equation == PERK_EQ_ADVECTION ? 1 : (dim == 1 ? 3 : 4);
    c->npe = dim == 1 ? NP : NP * NP;
    c->nd = dim == 1 ? 2 : 4;
    c->cap = (int)prob->max_cells;
    c->cap_faces = c->nd * c->cap;
    MeshDev &md = c->md;
    memset(&md, 0, sizeof(md));
    md.dim = dim;
    md.nv = c->nv;
    md.npe = c->npe;
    md.max_level = L;
    md.nfx = prob->n_base[0] << L;
    md.nfy = dim == 1 ? 1 : (prob->n_base[1] << L);
    md.periodic[0] = prob->periodic[0];
    md.periodic[1] = dim == 1 ? 1 : prob->periodic[1];
    md.equation = prob->equation;
    md.surface = prob->surface;
    md.lo[0] = prob->domain_lo[0];
    md.lo[1] = prob->domain_lo[1];
    md.hf = (prob->domain_hi[0] - prob->domain_lo[0]) / md.nfx;
    md.gamma = prob->gamma;
    md.adv = prob->adv_velocity;
    c->ns = dim == 2 && prob->equation == PERK_EQ_NAVIER_STOKES;
    md.mu = c->ns ? prob->mu : 0.0;
    md.kappa = c->ns ? prob->mu * prob->gamma / ((prob->gamma - 1.0) * prob->prandtl) : 0.0;
    for (int v = 0; v < MAXV; ++v) md.bc[v] = prob->bc_state[v];
    md.cap = c->cap;
    c->nf = (size_t)md.nfx * md.nfy;
    if (dim == 1) {
        c->nmorton = md.nfx;
    } else {
        long long P = 1;
        while (P < md.nfx || P < md.nfy) P <<= 1;
        c->nmorton = P * P;
    }
    if (c->nmorton > (1ll << 30)) { *out = c; return set_err(c, PERK_EINVAL, "finest grid too large"); }

    CU(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    {
        int dev = 0;
        CU(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lock(g_basis_mutex);
        if (dev >= 64 || !((g_basis_uploaded >> dev) & 1ull)) {
            BasisTables B;
            build_basis(B);
            CU(cudaMemcpyToSymbol(cB, &B, sizeof(B)));
            if (dev < 64) g_basis_uploaded |= 1ull << dev;
        }
    }
    const size_t rowd = (size_t)c->nv * c->npe;
    const long long max_items = c->nmorton > (long long)c->nd * c->cap ? c->nmorton : (long long)c->nd * c->cap;
    const int nb_max = (int)((max_items + PART_T - 1) / PART_T) + 1;
    CU(dalloc(c, &md.n, 4));
    CU(dalloc(c, &md.count_active, 4 * MAXS));
    CU(dalloc(c, &md.seg, 4 * (MAXR + 1)));
    CU(dalloc(c, &md.err, 1));
    CU(dalloc(c, &md.evals, 3));
    CU(dalloc(c, &md.list[KIND_EL], c->cap));
    for (int k = 1; k < 4; ++k) CU(dalloc(c, &md.list[k], c->cap_faces));
    CU(dalloc(c, &md.fx, c->cap));
    CU(dalloc(c, &md.fy, c->cap));
    CU(dalloc(c, &md.lev, c->cap));
    CU(dalloc(c, &md.mem, c->cap));
    CU(dalloc(c, &md.cell_of, c->nf));
    CU(dalloc(c, &md.ifc, c->cap_faces));
    CU(dalloc(c, &md.mor, c->cap_faces));
    CU(dalloc(c, &md.bnd, c->cap_faces));
    CU(dalloc(c, &md.elpk, c->cap));
    CU(dalloc(c, &md.ifcs, c->cap_faces));
    CU(dalloc(c, &md.mors, c->cap_faces));
    CU(dalloc(c, &c->K1, (size_t)c->cap * rowd));
    CU(dalloc(c, &c->Ubuf, (size_t)c->cap * rowd));
    CU(dalloc(c, &c->Fs, (size_t)c->cap * (dim == 1 ? 2 * c->nv : 4 * c->nv * NP)));
    if (tab->S >= 3 && tab->b[tab->S - 2] != 0.0) CU(dalloc(c, &c->Wb, (size_t)c->cap * rowd));   // P-ERK3
    if (c->ns) {
        rc = alloc_halo(c);
        if (rc) { *out = c; return rc; }
        if (!BR1_FUSED) CU(dalloc(c, &c->Gs, (size_t)c->cap * 4 * GV * NP));
        else CU(dalloc(c, &c->md.fnb, (size_t)c->cap * 4));
        CU(dalloc(c, &c->Vt, (size_t)c->cap * 4 * GV * NP));
        if (BR1_DV) CU(dalloc(c, &c->Dv, (size_t)c->cap * GV * 16));
    }
    CU(dalloc(c, &c->lmap, c->nf));
    CU(dalloc(c, &c->keys, (size_t)max_items));
    CU(dalloc(c, &c->items, (size_t)max_items));
    CU(dalloc(c, &c->rank, (size_t)c->nmorton));
    CU(dalloc(c, &c->blockcnt, (size_t)nb_max * MAXR));
    CU(dalloc(c, &c->blockoff, (size_t)nb_max * MAXR));
    CU(dalloc(c, &c->segtmp, 16));
    CU(dalloc(c, &c->dconst, 4));
    if (c->dd_P > 1) {
        CU(dalloc(c, &c->dd_owner, c->cap));
        CU(dalloc(c, &c->dd_flags, (size_t)2 * c->dd_P * c->cap));
        CU(dalloc(c, &c->dd_bsum, (size_t)blocks_for(c->cap, DD_SCAN_T) + 1));
        CU(dalloc(c, &c->dd_range, 2));
        for (int q = 0; q < c->dd_P; ++q) {
            if (q == c->dd_rank) continue;
            for (int d = 0; d < 2; ++d) {
                CU(dalloc(c, &c->dd_list[q][d], c->cap));
                CU(dalloc(c, &c->dd_seg[q][d], MAXR + 1));
                CU(dalloc(c, &c->dd_cnt[q][d], 2 * MAXS));
            }
        }
    }
    int h_const[4] = {(int)c->nmorton, 0, 0, 0};
    CU(cudaMemcpy(c->dconst, h_const, sizeof(h_const), cudaMemcpyHostToDevice));

    int occ = 0;
    if (dim == 2) {
        CU(cudaFuncSetAttribute(k_vol2d<MODE_STAGE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(true)));
        CU(cudaFuncSetAttribute(k_vol2d<MODE_RHS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(true)));
        CU(cudaFuncSetAttribute(k_vol2d<MODE_STAGE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(false)));
        CU(cudaFuncSetAttribute(k_vol2d<MODE_RHS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(false)));
        CU(cudaFuncSetAttribute(k_vol2d<MODE_STAGE, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(true)));
        CU(cudaFuncSetAttribute(k_vol2d<MODE_RHS, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(true)));
        CU(cudaFuncSetAttribute(k_vol2d<MODE_STAGE, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(false)));
        CU(cudaFuncSetAttribute(k_vol2d<MODE_RHS, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vol2d_smem_bytes(false)));
        if (c->ns) CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_vol2d<MODE_STAGE, true>, vol2d_threads(true), vol2d_smem_bytes(true)));
        else CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_vol2d<MODE_STAGE, false>, vol2d_threads(false), vol2d_smem_bytes(false)));
        const int want = (c->cap + vol2d_epb(c->ns) - 1) / vol2d_epb(c->ns);
        c->vol_blocks = std::min(want, SM_COUNT_B200 * std::max(occ, 1));
        // test hooks: PERK_VOL_BLOCKS / PERK_GRAD_BLOCKS / PERK_SURF_BLOCKS cap the persistent grids (a grid
        // of 1 CTA sends every element group through one CTA's staging rings; results must not change)
        auto cap_env = [](const char *name, int v) {
            const char *e = std::getenv(name);
            const int k = e ? std::atoi(e) : 0;
            return k > 0 ? std::min(v, k) : v;
        };
        c->vol_blocks = cap_env("PERK_VOL_BLOCKS", c->vol_blocks);
        int occ_sc = 0;   // the shock-capturing variant has its own register budget (NS: 2 CTAs per SM)
        if (c->ns) CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sc, k_vol2d<MODE_STAGE, true, true>, vol2d_threads(true), vol2d_smem_bytes(true)));
        else CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sc, k_vol2d<MODE_STAGE, false, true>, vol2d_threads(false), vol2d_smem_bytes(false)));
        c->vol_blocks_sc = cap_env("PERK_VOL_BLOCKS", std::min(want, SM_COUNT_B200 * std::max(occ_sc, 1)));
        int occg = 0;
        CU(cudaFuncSetAttribute(k_grad2d<MODE_STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grad2d_smem_bytes()));
        CU(cudaFuncSetAttribute(k_grad2d<MODE_RHS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grad2d_smem_bytes()));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occg, k_grad2d<MODE_STAGE>, 128, grad2d_smem_bytes()));
        c->grad_blocks = cap_env("PERK_GRAD_BLOCKS", std::min(want, SM_COUNT_B200 * std::max(occg, 1)));
        int occf = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf, k_surf2d<MODE_STAGE, false>, 256, 0));
        c->surf_blocks = std::min(blocks_for(4ll * c->cap_faces, 256), SM_COUNT_B200 * std::max(occf, 1));
        c->surf_blocks = cap_env("PERK_SURF_BLOCKS", c->surf_blocks);
        if (const char *e = std::getenv("PERK_SWEEP")) c->sweep = std::atoi(e) != 0;
        // re-mesh (transfer double buffer, old-mesh copy) and AMR scratch, allocated up front so that
        // no cudaMalloc / memset lands inside a timed re-mesh
        CU(dalloc(c, &c->Utmp, (size_t)c->cap * c->nv * c->npe));
        CU(dalloc(c, &c->n_old, 1));
        CU(dalloc(c, &c->cell_of_old, c->nf));
        CU(dalloc(c, &c->lev_old, c->cap));
        CU(dalloc(c, &c->fx_old, c->cap));
        CU(dalloc(c, &c->fy_old, c->cap));
        if (prob->equation != PERK_EQ_ADVECTION) {
            CU(dalloc(c, &c->amr_ind, c->cap));
            CU(dalloc(c, &c->amr_want, c->cap));
            CU(dalloc(c, &c->amr_newlev, c->cap));
            CU(dalloc(c, &c->amr_map[0], c->nf));
            CU(dalloc(c, &c->amr_map[1], c->nf));
            CU(dalloc(c, &c->amr_flags, 16));
        }
    } else {
        c->vol_blocks = std::min(blocks_for(c->cap, 128), SM_COUNT_B200 * 8);
        c->surf_blocks = std::min(blocks_for(c->cap_faces, 256), SM_COUNT_B200 * 8);
    }
    if (dim == 2 && !c->std_pattern) {   // per-stage lists for non-nested stage patterns
        bool nested = true;                // every stage's evaluating members form a prefix of the order?
        for (int i = 1; i <= tab->S && nested; ++i) {
            int rmin = tab->R;
            for (int r = tab->R - 1; r >= 0; --r)
                if ((c->act[r] >> (i - 1)) & 1ull) rmin = r;
            for (int r = rmin; r < tab->R; ++r)
                if (!((c->act[r] >> (i - 1)) & 1ull)) nested = false;
        }
        // per-stage arrays cost S x (4 B per cell + 36 B per face slot); beyond 8 GB keep the superset
        // prefix (correct, surplus members skipped) instead
        const double bytes = (double)tab->S * ((double)c->cap * 4.0 + (double)c->cap_faces * 36.0);
        const char *env = std::getenv("PERK_STAGE_LISTS");   // "0": force the superset path (tests)
        // Navier-Stokes keeps the superset prefix: its BR1 halo lists (the neighbours of the launch's
        // members across mortars) are defined for member prefixes; surplus members of the prefix see
        // their lazy stage state, so their gradients are the definition's
        if (!nested && bytes <= 8.0e9 && !(env && env[0] == '0') && !c->ns) {
            c->stage_lists = true;
            const size_t S = (size_t)tab->S;
            CU(dalloc(c, &c->st_el, S * c->cap));
            CU(dalloc(c, &c->st_if, S * c->cap_faces));
            CU(dalloc(c, &c->st_mo, S * c->cap_faces));
            CU(dalloc(c, &c->st_bd, S * c->cap_faces));
            CU(dalloc(c, &c->st_idx, (size_t)std::max(c->cap, c->cap_faces)));
        }
    }
    CU(cudaMemcpyAsync(c->lmap, level_map_dev, c->nf, cudaMemcpyDeviceToDevice, c->stream));
    build_mesh(c, c->stream, c->lmap);
    CU(cudaGetLastError());
    rc = check_device_err(c);
    *out = c;
    if (rc == PERK_OK && dim == 1) {
        // small 1D meshes (static: 1D has no re-mesh): one single-CTA launch per step if the whole
        // state fits in shared memory
        int n = 0;
        CU(cudaMemcpy(&n, md.n, sizeof(int), cudaMemcpyDeviceToHost));
        const size_t sh = step1d_smem_bytes(n, c->nv, c->Wb != nullptr);
        if (sh <= 200u * 1024u) {
            StepTab1D h;
            memset(&h, 0, sizeof(h));
            h.S = tab->S;
            h.R = tab->R;
            for (int i = 1; i <= tab->S; ++i) {
                const StageParams sp = stage_params(c, i, 0.0, MODE_STAGE, 0u);
                h.actmask[i - 1] = sp.actmask;
                h.bufmask[i - 1] = sp.bufmask;
                for (int r = 0; r < tab->R; ++r) {
                    h.a1n[r][i - 1] = sp.a1_next[r];
                    h.asubn[r][i - 1] = sp.asub_next[r];
                }
            }
            for (int i = 0; i < tab->S; ++i) h.c[i] = tab->c[i];
            h.b1 = tab->b[0];
            h.bS1 = tab->S >= 2 ? tab->b[tab->S - 2] : 0.0;
            h.bS = tab->b[tab->S - 1];
            CU(dalloc(c, &c->tb1d, 1));
            CU(cudaMemcpy(c->tb1d, &h, sizeof(h), cudaMemcpyHostToDevice));
            CU(cudaFuncSetAttribute(k_step1d<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            CU(cudaFuncSetAttribute(k_step1d<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            c->step1d_smem = sh;
            c->step1d = true;
        }
    }
    return rc;
}

extern "C" int perk_destroy(perk_ctx *c)
{
    if (!c) return PERK_ENOTINIT;
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->rexec) cudaGraphExecDestroy(c->rexec);
    cudaDeviceSynchronize();
    for (void *p : c->allocs) cudaFree(p);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    delete c;
    return PERK_OK;
}

extern "C" int perk_set_stream(perk_ctx *c, void *stream)
{
    if (!c) return PERK_ENOTINIT;
    c->stream = (cudaStream_t)stream;
    return PERK_OK;
}

static int ensure_graph(perk_ctx *c, double *U, double dt)
{
    if (c->gexec && c->gU == U && c->gdt == dt) return PERK_OK;
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    cudaGraph_t g;
    CU(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    launch_step(c, c->cap_stream, U, dt, nullptr);
    CU(cudaStreamEndCapture(c->cap_stream, &g));
    CU(cudaGraphInstantiate(&c->gexec, g, 0));
    cudaGraphDestroy(g);
    c->gU = U;
    c->gdt = dt;
    return PERK_OK;
}

extern "C" int perk_step(perk_ctx *c, double *U, double dt)
{
    if (!c) return PERK_ENOTINIT;
    if (!U) return set_err(c, PERK_EINVAL, "U_dev is null");
    if (c->dd_P > 1)
        return set_err(c, PERK_EUNSUPPORTED, "a sub-domain steps with perk_dd_group_step or perk_dd_stage + exchange");
    int rc = ensure_graph(c, U, dt);
    if (rc) return rc;
    CU(cudaGraphLaunch(c->gexec, c->stream));
    return PERK_OK;
}

extern "C" int perk_launches_per_step(perk_ctx *c, int32_t *launches)
{
    if (!c) return PERK_ENOTINIT;
    if (!launches) return PERK_EINVAL;
    // per stage: surface + volume (+ the BR1 pass(es): k_grad2d, and k_gsurf2d unless fused) (+ shock capturing)
    *launches = c->step1d ? 1 : ((c->ns ? (BR1_FUSED ? 3 : 4) : 2) + (c->sc ? ((c->scp.smooth && !c->sc_fused) ? 2 : 1) : 0)) * c->tab.S;
    return PERK_OK;
}

extern "C" int perk_num_cells(perk_ctx *c, int64_t *n)
{
    if (!c) return PERK_ENOTINIT;
    if (!n) return PERK_EINVAL;
    int rc = check_device_err(c);
    if (rc) return rc;
    int h = 0;
    CU(cudaMemcpy(&h, c->md.n, sizeof(int), cudaMemcpyDeviceToHost));
    *n = h;
    return PERK_OK;
}

extern "C" int perk_num_faces(perk_ctx *c, int64_t *counts3)
{
    if (!c) return PERK_ENOTINIT;
    if (!counts3) return PERK_EINVAL;
    int rc = check_device_err(c);
    if (rc) return rc;
    int h[4];
    CU(cudaMemcpy(h, c->md.n, sizeof(h), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 3; ++k) counts3[k] = h[k + 1];
    return PERK_OK;
}

extern "C" int perk_run_host(perk_ctx *c, double *U_host, double dt, int64_t nsteps)
{
    if (!c) return PERK_ENOTINIT;
    if (!U_host || nsteps < 0) return set_err(c, PERK_EINVAL, "U_host / nsteps");
    int64_t n = 0;
    int rc = perk_num_cells(c, &n);
    if (rc) return rc;
    const size_t bytes = (size_t)n * c->nv * c->npe * sizeof(double);
    if (!c->Uhost_dev) CU(dalloc(c, &c->Uhost_dev, (size_t)c->cap * c->nv * c->npe));
    CU(cudaMemcpyAsync(c->Uhost_dev, U_host, bytes, cudaMemcpyHostToDevice, c->stream));
    for (int64_t s = 0; s < nsteps; ++s) {
        rc = perk_step(c, c->Uhost_dev, dt);
        if (rc) return rc;
    }
    CU(cudaMemcpyAsync(U_host, c->Uhost_dev, bytes, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return PERK_OK;
}

// the re-mesh after the level map has been copied into c->lmap: old-mesh snapshot, mesh pipeline,
// transfer (about 30 small launches)
static void remesh_launches(perk_ctx *c, cudaStream_t s, double *U, Prof *p)
{
    k_save_old<<<SM_COUNT_B200 * 4, 256, 0, s>>>(c->md, c->n_old, c->cell_of_old, c->lev_old, c->fx_old, c->fy_old);
    k_copy_rows<<<SM_COUNT_B200 * 4, 256, 0, s>>>(c->md.n, c->nv * c->npe, U, c->Utmp);
    build_mesh(c, s, c->lmap);
    prof_mark(p, s, 3);
    OldMesh om{c->n_old, c->cell_of_old, c->lev_old, c->fx_old, c->fy_old};
    k_transfer2d<<<std::min(blocks_for(c->cap, 16), SM_COUNT_B200 * 8), 256, 0, s>>>(c->md, om, c->nv, c->Utmp, U);
}

static int do_repartition(perk_ctx *c, const uint8_t *lmap, double *U, Prof *p)
{
    if (c->prob.dim != 2) return set_err(c, PERK_EUNSUPPORTED, "repartition with solution transfer is 2D only");
    cudaStream_t s = c->stream;
    prof_mark(p, s, 2);
    CU(cudaMemcpyAsync(c->lmap, lmap, c->nf, cudaMemcpyDeviceToDevice, s));
    if (p) {                       // profiling: eager launches with events between the kinds
        remesh_launches(c, s, U, p);
        prof_mark(p, s, -1);
    } else {                       // one graph launch instead of ~30 host-side kernel launches
        if (!c->rexec || c->rU != U) {
            if (c->rexec) {
                cudaGraphExecDestroy(c->rexec);
                c->rexec = nullptr;
            }
            cudaGraph_t g;
            CU(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
            remesh_launches(c, c->cap_stream, U, nullptr);
            CU(cudaStreamEndCapture(c->cap_stream, &g));
            CU(cudaGraphInstantiate(&c->rexec, g, 0));
            cudaGraphDestroy(g);
            c->rU = U;
        }
        CU(cudaGraphLaunch(c->rexec, s));
    }
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_repartition(perk_ctx *c, const uint8_t *lmap, double *U)
{
    if (!c) return PERK_ENOTINIT;
    if (!lmap || !U) return set_err(c, PERK_EINVAL, "null pointer");
    return do_repartition(c, lmap, U, nullptr);
}

// ----------------------------------------------------------------------------------------------
// indicator-driven AMR (amr.cuh)
// ----------------------------------------------------------------------------------------------
static int amr_setup(perk_ctx *c, const double *U, const perk_amr *a, AmrParams &ap)
{
    if (!c) return PERK_ENOTINIT;
    if (!U || !a) return set_err(c, PERK_EINVAL, "null pointer");
    if (c->prob.dim != 2 || c->prob.equation == PERK_EQ_ADVECTION)
        return set_err(c, PERK_EUNSUPPORTED, "AMR indicators need a 2D Euler / Navier-Stokes problem");
    if (c->prob.max_level > 7) return set_err(c, PERK_EUNSUPPORTED, "AMR balance supports max_level <= 7");
    if (a->indicator < 0 || a->indicator > 2 || a->variable < 0 || a->variable > 4)
        return set_err(c, PERK_EINVAL, "bad indicator / variable");
    if (a->base_level < 0 || a->base_level > a->med_level || a->med_level > a->max_level ||
        a->max_level > c->prob.max_level)
        return set_err(c, PERK_EINVAL, "need 0 <= base_level <= med_level <= max_level <= problem max_level");
    if (!(a->med_threshold <= a->max_threshold))
        return set_err(c, PERK_EINVAL, "need med_threshold <= max_threshold");
    if (a->indicator == PERK_IND_HENNEMANN_GASSNER &&
        !(a->alpha_min >= 0.0 && a->alpha_min <= 0.5 && a->alpha_max >= 0.0 && a->alpha_max <= 1.0))
        return set_err(c, PERK_EINVAL, "need 0 <= alpha_min <= 1/2, 0 <= alpha_max <= 1");
    if (a->indicator == PERK_IND_LOHNER && !(a->f_wave >= 0.0))
        return set_err(c, PERK_EINVAL, "need f_wave >= 0");
    ap.indicator = a->indicator;
    ap.variable = a->variable;
    ap.base_level = a->base_level;
    ap.med_level = a->med_level;
    ap.max_level = a->max_level;
    ap.med_thr = a->med_threshold;
    ap.max_thr = a->max_threshold;
    ap.alpha_max = a->alpha_max;
    ap.alpha_min = a->alpha_min;
    ap.f_wave = a->f_wave;
    ap.hg_T = 0.5 * std::pow(10.0, -1.8 * std::pow((double)NP, 0.25));
    ap.hg_sT = std::log((1.0 - 0.0001) / 0.0001) / ap.hg_T;
    return PERK_OK;
}

// persistent indicator grid: 4 CTAs per SM (24 KB shared memory each), at most one tile per CTA
static int amr_indicator_blocks(const perk_ctx *c)
{
    return std::min(blocks_for((long long)c->cap, AMR_TILE), SM_COUNT_B200 * 4);
}

static void launch_amr_indicator(perk_ctx *c, cudaStream_t s, const AmrParams &ap, const double *U, double *ind)
{
    const int g = amr_indicator_blocks(c);
    switch (ap.indicator) {
    case IND_HG: launch_pdl(k_amr_indicator<IND_HG>, g, AMR_T, 0, s, c->md, ap, U, ind, c->amr_want); break;
    case IND_LOHNER: launch_pdl(k_amr_indicator<IND_LOHNER>, g, AMR_T, 0, s, c->md, ap, U, ind, c->amr_want); break;
    default: launch_pdl(k_amr_indicator<IND_ENSTROPHY>, g, AMR_T, 0, s, c->md, ap, U, ind, c->amr_want); break;
    }
}

extern "C" int perk_amr_indicator(perk_ctx *c, const double *U, const perk_amr *a, double *ind)
{
    AmrParams ap;
    int rc = amr_setup(c, U, a, ap);
    if (rc) return rc;
    if (!ind) return set_err(c, PERK_EINVAL, "null pointer");
    launch_amr_indicator(c, c->stream, ap, U, ind);
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_amr_adapt(perk_ctx *c, const double *U, const perk_amr *a, uint8_t *lmap)
{
    AmrParams ap;
    int rc = amr_setup(c, U, a, ap);
    if (rc) return rc;
    if (!lmap) return set_err(c, PERK_EINVAL, "null pointer");
    cudaStream_t s = c->stream;
    const int L = c->prob.max_level;
    if (L == 0) {   // no refinement allowed: the only map is all zeros
        CU(cudaMemsetAsync(lmap, 0, c->nf, s));
        return PERK_OK;
    }
    const int nbase = c->prob.n_base[0] * c->prob.n_base[1];
    const int bpc = amr_base_per_cta(L);
    const int bal_blocks = (nbase + bpc - 1) / bpc;
    const size_t smem = (size_t)bpc * amr_pyramid_bytes(L);
    const uint8_t *none = nullptr;
    launch_amr_indicator(c, s, ap, U, c->amr_ind);
    launch_pdl(k_amr_coarsen, blocks_for(c->cap, 256), 256, 0, s, c->md, (const uint8_t *)c->amr_want, c->amr_newlev);
    // L + 1 balance iterations, the last one into the caller's map
    uint8_t *out = c->amr_map[0];
    launch_pdl(k_amr_balance<true>, bal_blocks, AMR_T, smem, s, c->md, (const uint8_t *)c->amr_newlev, none, out,
               c->amr_flags, 0);
    for (int it = 1; it <= L; ++it) {
        const uint8_t *in = out;
        out = it == L ? lmap : c->amr_map[it & 1];
        launch_pdl(k_amr_balance<false>, bal_blocks, AMR_T, smem, s, c->md, none, in, out, c->amr_flags, it);
    }
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_amr_launches(perk_ctx *c, int32_t *launches)
{
    if (!c) return PERK_ENOTINIT;
    if (!launches) return set_err(c, PERK_EINVAL, "null pointer");
    *launches = c->prob.max_level + 3;
    return PERK_OK;
}

// ----------------------------------------------------------------------------------------------
// subcell shock capturing (sc.cuh)
// ----------------------------------------------------------------------------------------------
extern "C" int perk_set_shock_capturing(perk_ctx *c, const perk_shock_capturing *sc)
{
    if (!c) return PERK_ENOTINIT;
    if (sc && c->dd_P > 1) return set_err(c, PERK_EUNSUPPORTED, "shock capturing with domain decomposition");
    if (sc) {
        if (c->prob.dim != 2 || c->prob.equation == PERK_EQ_ADVECTION)
            return set_err(c, PERK_EUNSUPPORTED, "shock capturing needs a 2D Euler / Navier-Stokes problem");
        if (sc->variable < 0 || sc->variable > 4 || !(sc->alpha_min >= 0.0 && sc->alpha_min <= 0.5) ||
            !(sc->alpha_max >= 0.0 && sc->alpha_max <= 1.0) || !(sc->alpha_fixed <= 1.0))
            return set_err(c, PERK_EINVAL, "need variable in 0..4, 0 <= alpha_min <= 1/2, 0 <= alpha_max <= 1, alpha_fixed <= 1");
    }
    // the captured step and re-mesh graphs change shape: capture again on next use
    CU(cudaStreamSynchronize(c->stream));
    if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }
    if (c->rexec) { cudaGraphExecDestroy(c->rexec); c->rexec = nullptr; }
    if (!sc) { c->sc = false; return PERK_OK; }
    if (!c->alpha) {
        CU(dalloc(c, &c->alpha_raw, c->cap));
        CU(dalloc(c, &c->alpha, c->cap));
    }
    if (!c->halo_alloc) {   // halo lists of the current mesh (build_mesh keeps them up to date from now on)
        int rc = alloc_halo(c);
        if (rc) return rc;
        const MeshDev &md = c->md;
        const int R = c->tab.R;
        cudaStream_t s = c->stream;
        k_halo_clear<<<blocks_for(c->cap, 256), 256, 0, s>>>(md);
        k_halo_flags<<<blocks_for(c->cap_faces, 256), 256, 0, s>>>(md);
        partition(c, s, KeyHaloEl{md.halo, md.mem}, md.n + 0, 1, c->cap, R, md.hlist[KIND_EL], nullptr,
                  md.hseg + KIND_EL * (MAXR + 1), nullptr, nullptr);
        partition(c, s, KeyHaloIf{md.ifc, md.halo}, md.n + 1, 1, c->cap_faces, R, md.hlist[KIND_IF], nullptr,
                  md.hseg + KIND_IF * (MAXR + 1), nullptr, nullptr);
        partition(c, s, KeyHaloMo{md.mor, md.halo}, md.n + 2, 1, c->cap_faces, R, md.hlist[KIND_MO], nullptr,
                  md.hseg + KIND_MO * (MAXR + 1), nullptr, nullptr);
        k_halo_ranges<<<SM_COUNT_B200, 256, 0, s>>>(md, active_desc(c));
        CU(cudaGetLastError());
    }
    const char *fenv = std::getenv("PERK_SC_FUSED");
    // fused smoothing (a pass over the faces at the end of k_surf2d) for Euler; Navier-Stokes uses the
    // separate k_sc_smooth launch (A/B on one box, cfg 5 SC: 8.29 vs 8.31 ms/step fused, whose variant of
    // the Navier-Stokes surface kernel spilled at the 80-register budget of 3 CTAs per SM)
    c->sc_fused = !(fenv && fenv[0] == '0') && !c->ns;
    // next-stage alpha in the k_vol2d epilogue (cfg 3: 0.764 -> 0.719 ms/step, cfg 5: 8.68 -> 8.54 with
    // the batched tail; before it, the Navier-Stokes kernel got slower, 8.93).  PERK_SC_EPI=0: off.
    const char *eenv = std::getenv("PERK_SC_EPI");
    c->scp.epi = (eenv && eenv[0] == '0') || !c->std_pattern ? 0 : 1;
    c->scp.all = c->std_pattern ? 0 : 1;   // non-standard patterns: alpha of every element per stage
    c->scp.variable = sc->variable;
    c->scp.smooth = sc->smooth ? 1 : 0;
    c->scp.alpha_max = sc->alpha_max;
    c->scp.alpha_min = sc->alpha_min;
    c->scp.alpha_fixed = sc->alpha_fixed;
    c->scp.hg_T = 0.5 * std::pow(10.0, -1.8 * std::pow((double)NP, 0.25));
    c->scp.hg_sT = std::log((1.0 - 0.0001) / 0.0001) / c->scp.hg_T;
    c->sc = true;
    return PERK_OK;
}

extern "C" int perk_sc_alpha(perk_ctx *c, const double *U, double *raw, double *smoothed)
{
    if (!c) return PERK_ENOTINIT;
    if (!U || !raw || !smoothed) return set_err(c, PERK_EINVAL, "null pointer");
    if (!c->sc) return set_err(c, PERK_EINVAL, "shock capturing is off");
    const StageParams sp = stage_params(c, 1, 0.0, MODE_RHS, ~0u);
    launch_sc(c, c->stream, sp, nullptr, U, nullptr, true);
    int64_t n = 0;
    int rc = perk_num_cells(c, &n);
    if (rc) return rc;
    CU(cudaMemcpyAsync(raw, c->alpha_raw, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemcpyAsync(smoothed, c->alpha, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int rhs_eval(perk_ctx *c, const double *U, uint32_t mask, double *dU)
{
    if (!c) return PERK_ENOTINIT;
    if (!U || !dU) return set_err(c, PERK_EINVAL, "null pointer");
    const StageParams sp = stage_params(c, 1, 0.0, MODE_RHS, mask);
    if (c->sc) launch_sc(c, c->stream, sp, nullptr, U, nullptr);
    if (c->ns) launch_br1(c, c->stream, sp, nullptr, U, nullptr);
    launch_surface(c, c->stream, sp, nullptr, U);
    launch_volume(c, c->stream, sp, nullptr, U, dU);
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_node_coords(perk_ctx *c, double *xy)
{
    if (!c) return PERK_ENOTINIT;
    if (!xy) return PERK_EINVAL;
    k_node_coords<<<blocks_for(c->cap, 128), 128, 0, c->stream>>>(c->md, xy);
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_get_leaves(perk_ctx *c, int32_t *fx, int32_t *fy, uint8_t *lev, int32_t *mem, int64_t cap)
{
    int64_t n = 0;
    int rc = perk_num_cells(c, &n);
    if (rc) return rc;
    if (cap < n || !fx || !fy || !lev || !mem) return set_err(c, PERK_EINVAL, "host arrays too small");
    std::vector<uint8_t> m8(n);
    CU(cudaMemcpy(fx, c->md.fx, n * sizeof(int), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(fy, c->md.fy, n * sizeof(int), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(lev, c->md.lev, n, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(m8.data(), c->md.mem, n, cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < n; ++k) mem[k] = m8[k];
    return PERK_OK;
}

extern "C" int perk_get_faces(perk_ctx *c, int32_t kind, int32_t *rec, int32_t *mem, int64_t cap, int64_t *len)
{
    if (!c) return PERK_ENOTINIT;
    if (kind < 1 || kind > 3 || !len) return set_err(c, PERK_EINVAL, "kind");
    int64_t cnt[3];
    int rc = perk_num_faces(c, cnt);
    if (rc) return rc;
    const int64_t n = cnt[kind - 1];
    *len = n;
    if (!rec || !mem || cap < n) return set_err(c, PERK_EINVAL, "host arrays too small");
    if (kind == 1) {
        std::vector<int4> h(n);
        CU(cudaMemcpy(h.data(), c->md.ifc, n * sizeof(int4), cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < n; ++k) {
            rec[3 * k] = h[k].x; rec[3 * k + 1] = h[k].y; rec[3 * k + 2] = h[k].z; mem[k] = h[k].w;
        }
    } else if (kind == 2) {
        std::vector<int4> h(n);
        CU(cudaMemcpy(h.data(), c->md.mor, n * sizeof(int4), cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < n; ++k) {
            rec[5 * k] = h[k].x; rec[5 * k + 1] = h[k].y; rec[5 * k + 2] = h[k].z;
            rec[5 * k + 3] = h[k].w & 1; rec[5 * k + 4] = (h[k].w >> 1) & 1; mem[k] = h[k].w >> 8;
        }
    } else {
        std::vector<int2> h(n);
        CU(cudaMemcpy(h.data(), c->md.bnd, n * sizeof(int2), cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < n; ++k) {
            rec[2 * k] = h[k].x; rec[2 * k + 1] = h[k].y & 7; mem[k] = h[k].y >> 8;
        }
    }
    return PERK_OK;
}

extern "C" int perk_get_list(perk_ctx *c, int32_t kind, int32_t *list, int64_t cap, int64_t *seg)
{
    if (!c) return PERK_ENOTINIT;
    if (kind < 0 || kind > 3 || !seg) return set_err(c, PERK_EINVAL, "kind");
    int rc = check_device_err(c);
    if (rc) return rc;
    int hs[MAXR + 1];
    CU(cudaMemcpy(hs, c->md.seg + kind * (MAXR + 1), sizeof(hs), cudaMemcpyDeviceToHost));
    const int R = c->tab.R;
    for (int s = 0; s <= R; ++s) seg[s] = hs[s];
    const int64_t n = hs[R];
    if (!list || cap < n) return set_err(c, PERK_EINVAL, "host array too small");
    CU(cudaMemcpy(list, c->md.list[kind], n * sizeof(int), cudaMemcpyDeviceToHost));
    return PERK_OK;
}

extern "C" int perk_get_count_active(perk_ctx *c, int32_t kind, int32_t *out)
{
    if (!c) return PERK_ENOTINIT;
    if (kind < 0 || kind > 3 || !out) return set_err(c, PERK_EINVAL, "kind");
    int rc = check_device_err(c);
    if (rc) return rc;
    CU(cudaMemcpy(out, c->md.count_active + kind * MAXS, c->tab.S * sizeof(int), cudaMemcpyDeviceToHost));
    return PERK_OK;
}

extern "C" int perk_get_face_table(perk_ctx *c, int32_t *table, int64_t cap)
{
    if (!c) return PERK_ENOTINIT;
    if (!c->md.fnb) return set_err(c, PERK_EUNSUPPORTED, "no face table (Navier-Stokes with BR1_FUSED only)");
    int rc = check_device_err(c);
    if (rc) return rc;
    int n = 0;
    CU(cudaMemcpy(&n, c->md.n, sizeof(int), cudaMemcpyDeviceToHost));
    if (!table || cap < 8 * (int64_t)n) return set_err(c, PERK_EINVAL, "host array too small");
    std::vector<int2> h((size_t)4 * n);
    CU(cudaMemcpy(h.data(), c->md.fnb, sizeof(int2) * 4 * (size_t)n, cudaMemcpyDeviceToHost));
    const int mask = (1 << PK_EBITS) - 1;
    for (size_t k = 0; k < h.size(); ++k) {
        table[2 * k] = h[k].x >= 0 ? (h[k].x & mask) : h[k].x;
        table[2 * k + 1] = h[k].y >= 0 ? (h[k].y & mask) : h[k].y;
    }
    return PERK_OK;
}

extern "C" int perk_get_halo_counts(perk_ctx *c, int32_t *out)
{
    if (!c) return PERK_ENOTINIT;
    if (!out) return set_err(c, PERK_EINVAL, "null pointer");
    int rc = check_device_err(c);
    if (rc) return rc;
    const int S = c->tab.S;
    for (int k = 0; k < 3 * S; ++k) out[k] = 0;
    if (!c->halo_alloc) return PERK_OK;
    std::vector<int2> h((size_t)3 * MAXS);
    CU(cudaMemcpy(h.data(), c->md.hrng, sizeof(int2) * 3 * MAXS, cudaMemcpyDeviceToHost));
    for (int kind = 0; kind < 3; ++kind)
        for (int i = 0; i < S; ++i) out[kind * S + i] = h[(size_t)kind * MAXS + i].y;
    return PERK_OK;
}

extern "C" int perk_get_counters(perk_ctx *c, int64_t *evals, int64_t *steps)
{
    if (!c) return PERK_ENOTINIT;
    int rc = check_device_err(c);
    if (rc) return rc;
    unsigned long long h[2];
    CU(cudaMemcpy(h, c->md.evals, sizeof(h), cudaMemcpyDeviceToHost));
    if (evals) *evals = (int64_t)h[0];
    if (steps) *steps = (int64_t)h[1];
    return PERK_OK;
}

extern "C" int perk_sync(perk_ctx *c)
{
    if (!c) return PERK_ENOTINIT;
    return check_device_err(c);
}

extern "C" const char *perk_last_error(perk_ctx *c)
{
    if (!c) return "null context";
    return c->err.c_str();
}

static int finish_prof(perk_ctx *c, Prof &p, float *ms, int32_t *launches)
{
    CU(cudaStreamSynchronize(c->stream));
    for (size_t k = 0; k + 1 < p.ev.size(); ++k) {
        const int kind = p.kind[k];
        if (kind >= 0) {
            float t = 0.f;
            cudaEventElapsedTime(&t, p.ev[k], p.ev[k + 1]);
            if (ms) ms[kind] += t;
            if (launches) launches[kind] += 1;
        }
    }
    for (auto e : p.ev) cudaEventDestroy(e);
    return PERK_OK;
}

extern "C" int perk_profile_step(perk_ctx *c, double *U, double dt, float *ms, int32_t *launches)
{
    if (!c) return PERK_ENOTINIT;
    if (!U) return set_err(c, PERK_EINVAL, "U_dev is null");
    Prof p;
    launch_step(c, c->stream, U, dt, &p);
    CU(cudaGetLastError());
    return finish_prof(c, p, ms, launches);
}

extern "C" int perk_time_kernels_ex(perk_ctx *c, double *U, double dt, uint32_t kind_mask, int32_t reps,
                                    void *flush_dev, int64_t flush_bytes, float *ms_per_step)
{
    if (!c) return PERK_ENOTINIT;
    if (!U || !ms_per_step || reps < 1 || reps > 1000 || (flush_bytes > 0 && !flush_dev))
        return set_err(c, PERK_EINVAL, "U_dev / ms / reps / flush buffer");
    cudaGraph_t g;
    cudaGraphExec_t ge;
    c->kind_mask = kind_mask;
    cudaError_t ce = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (ce == cudaSuccess) {
        launch_step(c, c->cap_stream, U, dt, nullptr);
        ce = cudaStreamEndCapture(c->cap_stream, &g);
    }
    c->kind_mask = ~0u;
    if (ce != cudaSuccess) return set_err(c, PERK_ECUDA, std::string("capture: ") + cudaGetErrorString(ce));
    CU(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    std::vector<cudaEvent_t> ev(2 * (size_t)reps);
    for (auto &e : ev) CU(cudaEventCreate(&e));
    CU(cudaGraphLaunch(ge, c->stream));   // warm-up
    for (int r = 0; r < reps; ++r) {
        // L2 flush between replays (outside the events): the replays then see the cache state of a
        // step inside a timed P-ERK run, not the previous replay's leftovers
        if (flush_bytes > 0) CU(cudaMemsetAsync(flush_dev, r & 0xff, (size_t)flush_bytes, c->stream));
        CU(cudaEventRecord(ev[2 * r], c->stream));
        CU(cudaGraphLaunch(ge, c->stream));
        CU(cudaEventRecord(ev[2 * r + 1], c->stream));
    }
    CU(cudaEventSynchronize(ev.back()));
    float tot = 0.f;
    for (int r = 0; r < reps; ++r) {
        float t = 0.f;
        CU(cudaEventElapsedTime(&t, ev[2 * r], ev[2 * r + 1]));
        tot += t;
    }
    *ms_per_step = tot / reps;
    for (auto &e : ev) cudaEventDestroy(e);
    cudaGraphExecDestroy(ge);
    return check_device_err(c);
}

extern "C" int perk_time_kernels(perk_ctx *c, double *U, double dt, uint32_t kind_mask, int32_t reps, float *ms_per_step)
{
    return perk_time_kernels_ex(c, U, dt, kind_mask, reps, nullptr, 0, ms_per_step);
}

extern "C" int perk_build_flags(void) { return (BR1_DV ? 1 : 0) | (BR1_FUSED ? 2 : 0); }

extern "C" int perk_profile_repartition(perk_ctx *c, const uint8_t *lmap, double *U, float *ms, int32_t *launches)
{
    if (!c) return PERK_ENOTINIT;
    if (!lmap || !U) return set_err(c, PERK_EINVAL, "null pointer");
    Prof p;
    int rc = do_repartition(c, lmap, U, &p);
    if (rc) return rc;
    return finish_prof(c, p, ms, launches);
}

// ----------------------------------------------------------------------------------------------
// spatial domain decomposition (dd.cuh)
// ----------------------------------------------------------------------------------------------
extern "C" int perk_dd_split(int64_t n, const int32_t *weights, int32_t nranks, int32_t *owner)
{
    if (n < 0 || (n > 0 && (!weights || !owner)) || nranks < 1 || nranks > DD_MAXP) return PERK_EINVAL;
    long long W = 0;
    for (int64_t k = 0; k < n; ++k) {
        if (weights[k] < 0) return PERK_EINVAL;
        W += weights[k];
    }
    long long pre = 0;
    for (int64_t k = 0; k < n; ++k) {
        long long o = W > 0 ? ((long long)nranks * (2 * pre + weights[k])) / (2 * W) : 0;
        owner[k] = (int32_t)(o > nranks - 1 ? nranks - 1 : o);
        pre += weights[k];
    }
    return PERK_OK;
}

static int dd_check(perk_ctx *c)
{
    if (!c) return PERK_ENOTINIT;
    if (c->dd_P < 2) return set_err(c, PERK_EINVAL, "not a sub-domain context (perk_init_dd with nranks > 1)");
    return PERK_OK;
}

extern "C" int perk_dd_info(perk_ctx *c, int32_t *rank, int32_t *nranks, int64_t *first, int64_t *count)
{
    if (!c) return PERK_ENOTINIT;
    if (!rank || !nranks || !first || !count) return set_err(c, PERK_EINVAL, "null pointer");
    *rank = c->dd_rank;
    *nranks = c->dd_P;
    int rc = check_device_err(c);
    if (rc) return rc;
    if (c->dd_P < 2) {
        int n = 0;
        CU(cudaMemcpy(&n, c->md.n, sizeof(int), cudaMemcpyDeviceToHost));
        *first = 0;
        *count = n;
        return PERK_OK;
    }
    int h[2];
    CU(cudaMemcpy(h, c->dd_range, sizeof(h), cudaMemcpyDeviceToHost));
    *first = h[1] > 0 ? h[0] : 0;
    *count = h[1];
    return PERK_OK;
}

extern "C" int perk_dd_counts(perk_ctx *c, int32_t peer, int32_t what, int32_t *send_host, int32_t *recv_host)
{
    int rc = dd_check(c);
    if (rc) return rc;
    if (peer < 0 || peer >= c->dd_P || peer == c->dd_rank || what < 0 || what > 1 || !send_host || !recv_host)
        return set_err(c, PERK_EINVAL, "peer / what / null pointer");
    rc = check_device_err(c);
    if (rc) return rc;
    const int S = c->tab.S;
    CU(cudaMemcpy(send_host, c->dd_cnt[peer][0] + what * MAXS, S * sizeof(int), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(recv_host, c->dd_cnt[peer][1] + what * MAXS, S * sizeof(int), cudaMemcpyDeviceToHost));
    return PERK_OK;
}

extern "C" int perk_dd_get_list(perk_ctx *c, int32_t peer, int32_t dir, int32_t *list_host, int64_t cap, int64_t *len)
{
    int rc = dd_check(c);
    if (rc) return rc;
    if (peer < 0 || peer >= c->dd_P || peer == c->dd_rank || dir < 0 || dir > 1 || !len)
        return set_err(c, PERK_EINVAL, "peer / dir / null pointer");
    rc = check_device_err(c);
    if (rc) return rc;
    int seg[MAXR + 1];
    CU(cudaMemcpy(seg, c->dd_seg[peer][dir], sizeof(seg), cudaMemcpyDeviceToHost));
    *len = seg[c->tab.R];
    if (!list_host || cap < *len) return set_err(c, PERK_EINVAL, "host array too small");
    CU(cudaMemcpy(list_host, c->dd_list[peer][dir], (size_t)*len * sizeof(int), cudaMemcpyDeviceToHost));
    return PERK_OK;
}

// the array a stage's exchange carries (what 0: the blocks the stage-i volume epilogue wrote; 1: Vt)
static double *dd_array(perk_ctx *c, double *U, int stage, int what, int &row)
{
    if (what == 1) {
        row = 4 * GV * NP;
        return c->Vt;
    }
    row = c->nv * c->npe;
    return stage == 1 ? c->K1 : (stage == c->tab.S ? U : c->Ubuf);
}

static int dd_args(perk_ctx *c, double *U, int32_t stage, int32_t what)
{
    int rc = dd_check(c);
    if (rc) return rc;
    if (!U || stage < 1 || stage > c->tab.S || what < 0 || what > 1) return set_err(c, PERK_EINVAL, "U / stage / what");
    if (what == 1 && !c->ns) return set_err(c, PERK_EINVAL, "Vt exchange needs a Navier-Stokes context");
    return PERK_OK;
}

extern "C" int perk_dd_stage(perk_ctx *c, double *U, double dt, int32_t stage, int32_t part)
{
    int rc = dd_check(c);
    if (rc) return rc;
    if (!U || stage < 1 || stage > c->tab.S || part < 0 || part > 1) return set_err(c, PERK_EINVAL, "U / stage / part");
    const StageParams sp = stage_params(c, stage, dt, MODE_STAGE, 0u);
    if (part == 0) {
        if (c->ns) launch_br1(c, c->stream, sp, U, nullptr, nullptr);
    } else {
        launch_surface(c, c->stream, sp, U, nullptr);
        launch_volume(c, c->stream, sp, U, nullptr, nullptr);
    }
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_dd_pack(perk_ctx *c, double *U, int32_t stage, int32_t what, int32_t peer, double *buf)
{
    int rc = dd_args(c, U, stage, what);
    if (rc) return rc;
    if (peer < 0 || peer >= c->dd_P || peer == c->dd_rank || !buf) return set_err(c, PERK_EINVAL, "peer / buffer");
    int row;
    const double *a = dd_array(c, U, stage, what, row);
    k_dd_pack<<<SM_COUNT_B200 * 2, 256, 0, c->stream>>>(c->dd_list[peer][0], c->dd_cnt[peer][0] + what * MAXS + stage - 1,
                                                       row, a, buf);
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_dd_unpack(perk_ctx *c, double *U, int32_t stage, int32_t what, int32_t peer, const double *buf)
{
    int rc = dd_args(c, U, stage, what);
    if (rc) return rc;
    if (peer < 0 || peer >= c->dd_P || peer == c->dd_rank || !buf) return set_err(c, PERK_EINVAL, "peer / buffer");
    int row;
    double *a = dd_array(c, U, stage, what, row);
    k_dd_unpack<<<SM_COUNT_B200 * 2, 256, 0, c->stream>>>(c->dd_list[peer][1], c->dd_cnt[peer][1] + what * MAXS + stage - 1,
                                                         row, buf, a);
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_dd_exchange(perk_ctx *src, perk_ctx *dst, double *U_src, double *U_dst, int32_t stage, int32_t what)
{
    int rc = dd_args(src, U_src, stage, what);
    if (rc) return rc;
    rc = dd_args(dst, U_dst, stage, what);
    if (rc) return rc;
    if (src->dd_P != dst->dd_P || src->dd_rank == dst->dd_rank) return set_err(src, PERK_EINVAL, "not two sub-domains of one split");
    perk_ctx *c = src;
    int row;
    const double *a = dd_array(src, U_src, stage, what, row);
    double *b = dd_array(dst, U_dst, stage, what, row);
    k_dd_copy<<<SM_COUNT_B200 * 2, 256, 0, src->stream>>>(src->dd_list[dst->dd_rank][0],
                                                         src->dd_cnt[dst->dd_rank][0] + what * MAXS + stage - 1, row, a, b);
    CU(cudaGetLastError());
    return PERK_OK;
}

extern "C" int perk_dd_group_step(perk_ctx **ctxs, int32_t n, double **U, double dt)
{
    if (!ctxs || !U || n < 2 || n > DD_MAXP) return PERK_EINVAL;
    for (int p = 0; p < n; ++p) {
        int rc = dd_check(ctxs[p]);
        if (rc) return rc;
        if (ctxs[p]->dd_P != n || ctxs[p]->dd_rank != p || !U[p])
            return set_err(ctxs[p], PERK_EINVAL, "ctxs[p] must be sub-domain p of an n-way split, U[p] non-null");
        if (ctxs[p]->stream != ctxs[0]->stream || ctxs[p]->tab.S != ctxs[0]->tab.S)
            return set_err(ctxs[p], PERK_EINVAL, "the sub-domains of a group share one stream and one tableau");
    }
    const int S = ctxs[0]->tab.S;
    const bool ns = ctxs[0]->ns;
    for (int i = 1; i <= S; ++i) {
        if (ns) {
            for (int p = 0; p < n; ++p) {
                int rc = perk_dd_stage(ctxs[p], U[p], dt, i, 0);
                if (rc) return rc;
            }
            for (int p = 0; p < n; ++p)
                for (int q = 0; q < n; ++q)
                    if (q != p) {
                        int rc = perk_dd_exchange(ctxs[p], ctxs[q], U[p], U[q], i, 1);
                        if (rc) return rc;
                    }
        }
        for (int p = 0; p < n; ++p) {
            int rc = perk_dd_stage(ctxs[p], U[p], dt, i, 1);
            if (rc) return rc;
        }
        for (int p = 0; p < n; ++p)
            for (int q = 0; q < n; ++q)
                if (q != p) {
                    int rc = perk_dd_exchange(ctxs[p], ctxs[q], U[p], U[q], i, 0);
                    if (rc) return rc;
                }
    }
    return PERK_OK;
}

// ----------------------------------------------------------------------------------------------
// race exposure (debug builds)
// ----------------------------------------------------------------------------------------------
extern "C" int perk_debug_jitter(uint32_t seed)
{
#ifdef PERK_DEBUG
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return PERK_ECUDA;
    if (cudaMemcpyToSymbol(g_jitter_seed, &seed, sizeof(seed)) != cudaSuccess) return PERK_ECUDA;
    return PERK_OK;
#else
    (void)seed;
    return PERK_EUNSUPPORTED;
#endif
}
