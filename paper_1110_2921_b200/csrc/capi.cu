// capi.cu -- the C ABI of include/vfmm.h: context, workspace, and the evaluate pipeline
//   keys -> radix sort -> leaf ranges -> gather -> P2M -> M2M -> periodic -> (L2L, M2L)
//   per level -> P2P -> L2P + combine + un-permute
// (section 3.1; the step list is DESIGN.md "Hot path").  Every step is a kernel
// on the caller's stream; the host only validates parameters and enqueues.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "dist.h"
#include "vfmm_internal.h"

using namespace vfmm;

// reinitialization workspace (vfmm_reinit): trees of the old and new particles, Krylov basis
struct RbfWs {
    int64_t cap_old = 0, cap_new = 0;
    int cap_depth = -1, cap_m = -1;
    uint32_t *ok[2] = {nullptr, nullptr}, *ov[2] = {nullptr, nullptr};
    uint32_t *nk[2] = {nullptr, nullptr}, *nv[2] = {nullptr, nullptr};
    void *otmp = nullptr, *ntmp = nullptr;
    float *o6 = nullptr, *n6 = nullptr;
    int *ols = nullptr, *nls = nullptr;
    float *V = nullptr, *w = nullptr, *x = nullptr, *om = nullptr;
    double *part = nullptr, *dots = nullptr, *coef = nullptr;
    void release() {
        for (void* p : {(void*)ok[0], (void*)ok[1], (void*)ov[0], (void*)ov[1], (void*)nk[0],
                        (void*)nk[1], (void*)nv[0], (void*)nv[1], otmp, ntmp, (void*)o6, (void*)n6,
                        (void*)ols, (void*)nls, (void*)V, (void*)w, (void*)x, (void*)om,
                        (void*)part, (void*)dots, (void*)coef})
            if (p) cudaFree(p);
        *this = RbfWs();
    }
};

struct vfmm_ctx {
    vfmm_params prm{};
    int device = 0;
    std::string err;
    // operators
    int ops_p = -1, ops_levels = -1;
    HostOps hops;
    float *d_m2m = nullptr, *d_l2l = nullptr, *d_m2l = nullptr, *d_per = nullptr;
    float *d_tc_hi = nullptr, *d_tc_lo = nullptr;  // tensor-core M2L operators (3xTF32)
    uint16_t *d_h16_hi = nullptr, *d_h16_lo = nullptr;  // balanced 3xFP16 operators
    float *d_h16_rs = nullptr, *d_h16_cs = nullptr;     // their row / column scales
    uint32_t* d_tcmax = nullptr;                        // [32] per-level staging max (f16)
    float *g_hi = nullptr, *g_lo = nullptr;        // tensor-core M2L staged source grid
    size_t g_cap = 0;
    float *g2_hi = nullptr, *g2_lo = nullptr;      // staging for the side stream (levels < L)
    size_t g2_cap = 0;
    cudaStream_t side = nullptr;                   // coarse M2L levels run here, joined by events
    cudaStream_t far_st = nullptr;  // co-resident mode: the far-field chain (high priority)
    cudaEvent_t ev_tree = nullptr, ev_far = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_gamma = nullptr;  // evaluate_host: strengths copied on the side stream
    bool gamma_pending = false;      // the next evaluate waits for ev_gamma before the gather
    int* d_slots = nullptr;  // [8][189]
    int* d_groups = nullptr; // [8][72][4] offset groups (tensor-core M2L y-windows)
    float* m2m_scratch = nullptr;  // coarse-level op-split partials (M2M, SIMT M2L): main stream
    float* side_scratch = nullptr; // the same for the side stream's SIMT M2L levels
    size_t m2m_scratch_floats = 0, side_scratch_floats = 0;
    int *d_l2p_rowptr = nullptr, *d_l2p_pairs = nullptr;  // L2P derivative map (CSR)
    // workspace
    int64_t cap_n = 0;
    int cap_depth = -1, cap_p = -1;
    uint32_t *keys[2] = {nullptr, nullptr}, *vals[2] = {nullptr, nullptr};
    void* radix_tmp = nullptr;
    size_t radix_tmp_bytes = 0;
    float *sorted6 = nullptr, *near6 = nullptr;
    int* leaf_start = nullptr;
    float *Mall = nullptr, *Lall = nullptr;
    int* d_err = nullptr;
    unsigned long long* d_pairs = nullptr;  // P2P pair counter of the last evaluate
    // vfmm_evaluate_tree: adaptive leaves (level, cell), their count, interaction counters
    int2* tree_groups = nullptr;
    size_t tree_groups_cap = 0;
    int* d_tree_ng = nullptr;
    unsigned long long* d_tree_cnt = nullptr;
    bool tree_last = false;  // the last evaluate was a treecode one (stats)
    // VFMM_MODE_HYBRID: the choice between the FMM and the treecode, by timing, cached per
    // (n, p, image_levels, depth parameter)
    int64_t hyb_n = -1;
    int hyb_p = -1, hyb_levels = -1, hyb_depth = -2;
    int hyb_choice = 0;  // 0: FMM; k = 1..3: treecode with n_crit = 16 << k (32, 64, 128)
    float hyb_ms[4] = {0, 0, 0, 0};
    // host-API staging
    int64_t cap_host_n = 0;
    float* hbuf = nullptr;  // 12 x n
    RbfWs rbf;
    int64_t cap_at_n = 0;
    float* at_buf = nullptr;    // vfmm_evaluate_at: sources + targets, 12 x (n_src + n_tgt)
    int64_t cap_step_n = 0;
    int64_t cap_sig_n = 0;
    float* sorted_sig = nullptr;  // vfmm_evaluate_sigma: per-particle sigma in Morton order
    float* step_buf = nullptr;  // vfmm_step: u and dgamma/dt when the caller passes no buffers
    cudaStream_t own_stream = nullptr;
    // last evaluate
    cudaStream_t last_stream = nullptr;
    bool have_last = false;  // ev[NEV-1] marks the end of an earlier evaluate
    // depth = -1: depth chosen by timing ("automatically choosing the number
    // of particles per box"), cached per (n, p, mode, image_levels)
    int64_t tuned_n = -1;
    int tuned_p = -1, tuned_mode = -1, tuned_levels = -1, tuned_depth = 0;
    float tuned_ms[3] = {0, 0, 0};
    uint32_t *keys_sorted = nullptr, *perm = nullptr;
    int64_t last_n = 0;
    int last_depth = 0;
    bool have_tree = false, have_exp = false;
    vfmm_stats stats{};
    // distributed state (dist: NCCL context, this process = rank `rank` of R; logical mode:
    // one RankState per logical rank)
    int R = 1, rank = 0;
    bool dist = false;
    void* comm = nullptr;
    std::vector<vfmm::RankState*> ranks;
    static constexpr int NEV = 10;
    cudaEvent_t ev[NEV] = {};
    // distributed contexts: communication stream (all NCCL calls) and exchange timing events
    cudaStream_t comm_st = nullptr;
    static constexpr int NCE = 20;
    cudaEvent_t evc[NCE] = {};
    bool comm_timed = false;  // evc hold the exchanges of the last evaluate
    bool comm_overlap = false;  // NCCL mode: X2 / X3 overlapped (exposed part from evc 11-16)
};

namespace {

// VFMM_M2L selects the M2L engine: "simt" (FP32 CUDA cores), "tf32" (tcgen05 3xTF32), default
// (or "f16") tcgen05 scaled 3xFP16.  0 = simt, 1 = tf32, 2 = f16
int m2l_env_mode() {
    const char* e = getenv("VFMM_M2L");
    if (e && strcmp(e, "simt") == 0) return 0;
    if (e && strcmp(e, "tf32") == 0) return 1;
    return 2;
}

L2PMap l2p_map(const vfmm_ctx* c) {
    L2PMap m;
    m.rowptr = c->d_l2p_rowptr;
    m.terms = reinterpret_cast<const uint4*>(c->d_l2p_pairs);
    return m;
}

TcOps tc_ops(const vfmm_ctx* c) {
    TcOps t;
    t.groups = reinterpret_cast<const int4*>(c->d_groups);
    if (m2l_env_mode() == 2 && c->d_h16_hi) {
        t.hi = c->d_h16_hi;
        t.lo = c->d_h16_lo;
        t.rs = c->d_h16_rs;
        t.cs = c->d_h16_cs;
        t.f16 = true;
        t.nr = c->hops.h16_nr;
        t.kp = c->hops.h16_kp;
    } else {
        t.hi = c->d_tc_hi;
        t.lo = c->d_tc_lo;
    }
    return t;
}

vfmm_status cuda_fail(vfmm_ctx* c, cudaError_t e, const char* where) {
    if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? VFMM_ENOMEM : VFMM_ECUDA;
}

#define CK(call, where)                                    \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, where); \
    } while (0)

bool finite_pos(float x) { return std::isfinite(x) && x > 0.f; }

vfmm_status validate(const vfmm_params* p) {
    if (!p) return VFMM_EINVAL;
    if (p->p < 1 || p->p > VFMM_PMAX) return VFMM_EINVAL;
    if (p->depth < -1 || p->depth > 10) return VFMM_EINVAL;
    if (p->image_levels < 0 || p->image_levels > 6) return VFMM_EINVAL;
    if (p->scheme != 0 && p->scheme != 1) return VFMM_EINVAL;
    if (p->mode < 0 || p->mode > 4) return VFMM_EINVAL;
    if (!finite_pos(p->sigma) || !finite_pos(p->box_len) || !std::isfinite(p->box_lo))
        return VFMM_EINVAL;
    return VFMM_OK;
}

int auto_depth(const vfmm_params& p, int64_t n) {
    int L = (int)std::lround(std::log((double)n / 64.0) / std::log(8.0));
    if (L < 1) L = 1;
    if (L > 10) L = 10;
    // far field omits the cutoff: keep the leaf width >= 4 sigma (reading R3)
    while (L > 1 && (double)p.box_len / (double)(1 << L) < 4.0 * (double)p.sigma * (1.0 - 1e-6))
        --L;
    return L;
}

template <class T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

vfmm_status ensure_ops(vfmm_ctx* c) {
    if (c->ops_p == c->prm.p && c->ops_levels == c->prm.image_levels) return VFMM_OK;
    // nothing may throw across the C ABI: host table construction allocates (bad_alloc) and
    // checks its own invariants (runtime_error)
    try {
        build_host_ops(c->prm.p, c->prm.image_levels, &c->hops);
    } catch (const std::bad_alloc&) {
        c->err = "host operator tables: out of memory";
        return VFMM_ENOMEM;
    } catch (const std::exception& ex) {
        c->err = std::string("host operator tables: ") + ex.what();
        return VFMM_ESTATE;
    }
    dfree(c->d_m2m);
    dfree(c->d_l2l);
    dfree(c->d_m2l);
    dfree(c->d_per);
    auto up = [&](const std::vector<float>& h, float** d) -> cudaError_t {
        cudaError_t e = cudaMalloc((void**)d, h.size() * sizeof(float));
        if (e != cudaSuccess) return e;
        return cudaMemcpy(*d, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice);
    };
    CK(up(c->hops.m2m, &c->d_m2m), "upload m2m");
    CK(up(c->hops.l2l, &c->d_l2l), "upload l2l");
    CK(up(c->hops.m2l, &c->d_m2l), "upload m2l");
    CK(up(c->hops.per, &c->d_per), "upload periodic");
    dfree(c->d_l2p_rowptr);
    dfree(c->d_l2p_pairs);
    dfree(c->m2m_scratch);
    dfree(c->side_scratch);
    {
        // largest op-split partial set: M2M of < 296 x 32 parents (< 2 tiles per SM) x 8
        // children (main stream only), or a SIMT M2L level with < 296 tiles (slices x 8
        // children x parents; main stream for level L, side stream for the coarse levels)
        size_t need_m2l = 0;
        for (int64_t pc = 1; pc <= 4096; pc *= 8) {
            const int64_t tiles = 8 * ((pc + 31) / 32) * (c->hops.NR / 128);
            const int64_t os = tiles >= 296 ? 1 : std::min<int64_t>(27, (296 + tiles - 1) / tiles);
            if (os > 1) need_m2l = std::max(need_m2l, (size_t)(os * 8 * pc));
        }
        c->m2m_scratch_floats = std::max<size_t>((size_t)8 * 4096, need_m2l) * 3 * c->hops.nc;
        c->side_scratch_floats = std::max<size_t>(need_m2l, 1) * 3 * c->hops.nc;
    }
    CK(cudaMalloc((void**)&c->m2m_scratch, c->m2m_scratch_floats * sizeof(float)),
       "alloc op-split scratch");
    CK(cudaMalloc((void**)&c->side_scratch, c->side_scratch_floats * sizeof(float)),
       "alloc op-split scratch");
    {
        auto upi = [&](const std::vector<int>& h, int** d) -> cudaError_t {
            cudaError_t e = cudaMalloc((void**)d, std::max<size_t>(h.size(), 1) * sizeof(int));
            if (e != cudaSuccess || h.empty()) return e;
            return cudaMemcpy(*d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice);
        };
        CK(upi(c->hops.l2p_rowptr, &c->d_l2p_rowptr), "upload l2p map");
        std::vector<int> terms(c->hops.l2p_src.size());
        for (size_t t = 0; t < c->hops.l2p_src.size(); ++t) {
            const float cf = c->hops.l2p_coef[t];
            const __half h = __float2half_rn(cf);
            if (__half2float(h) != cf || c->hops.l2p_src[t] > 0xffff) {
                c->err = "L2P derivative map coefficient not exact in half";
                return VFMM_ESTATE;
            }
            uint16_t hb;
            memcpy(&hb, &h, 2);
            terms[t] = (int)((uint32_t)c->hops.l2p_src[t] | ((uint32_t)hb << 16));
        }
        CK(upi(terms, &c->d_l2p_pairs), "upload l2p map");
    }
    dfree(c->d_tc_hi);
    dfree(c->d_tc_lo);
    dfree(c->d_h16_hi);
    dfree(c->d_h16_lo);
    dfree(c->d_h16_rs);
    dfree(c->d_h16_cs);
    if (!c->hops.m2l_tc_hi.empty()) {
        CK(up(c->hops.m2l_tc_hi, &c->d_tc_hi), "upload m2l tc hi");
        CK(up(c->hops.m2l_tc_lo, &c->d_tc_lo), "upload m2l tc lo");
    }
    if (!c->hops.m2l_h16_hi.empty()) {
        auto up16 = [&](const std::vector<uint16_t>& h, uint16_t** d) -> cudaError_t {
            cudaError_t e = cudaMalloc((void**)d, h.size() * sizeof(uint16_t));
            if (e != cudaSuccess) return e;
            return cudaMemcpy(*d, h.data(), h.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
        };
        CK(up16(c->hops.m2l_h16_hi, &c->d_h16_hi), "upload m2l f16 hi");
        CK(up16(c->hops.m2l_h16_lo, &c->d_h16_lo), "upload m2l f16 lo");
        CK(up(c->hops.h16_rs, &c->d_h16_rs), "upload m2l f16 scales");
        CK(up(c->hops.h16_cs, &c->d_h16_cs), "upload m2l f16 scales");
    }
    if (!c->d_tcmax) CK(cudaMalloc((void**)&c->d_tcmax, 32 * sizeof(uint32_t)), "alloc tc max");
    if (!c->d_slots) {
        // interaction list per parity: o_a in {-2-b_a .. 3-b_a}, minus |o|inf <= 1 (189 cells)
        std::vector<int> slots;
        for (int par = 0; par < 8; ++par) {
            const int bx = par & 1, by = (par >> 1) & 1, bz = (par >> 2) & 1;
            int cnt = 0;
            for (int ox = -2 - bx; ox <= 3 - bx; ++ox)
                for (int oy = -2 - by; oy <= 3 - by; ++oy)
                    for (int oz = -2 - bz; oz <= 3 - bz; ++oz) {
                        if (std::abs(ox) <= 1 && std::abs(oy) <= 1 && std::abs(oz) <= 1) continue;
                        slots.push_back(m2l_slot(ox, oy, oz));
                        ++cnt;
                    }
            if (cnt != 189) return VFMM_EINVAL;
        }
        CK(cudaMalloc((void**)&c->d_slots, slots.size() * sizeof(int)), "alloc slots");
        CK(cudaMemcpy(c->d_slots, slots.data(), slots.size() * sizeof(int),
                      cudaMemcpyHostToDevice),
           "upload slots");
        const std::vector<int> groups = m2l_groups();
        CK(cudaMalloc((void**)&c->d_groups, groups.size() * sizeof(int)), "alloc groups");
        CK(cudaMemcpy(c->d_groups, groups.data(), groups.size() * sizeof(int),
                      cudaMemcpyHostToDevice),
           "upload groups");
    }
    c->ops_p = c->prm.p;
    c->ops_levels = c->prm.image_levels;
    return VFMM_OK;
}

vfmm_status ensure_ws(vfmm_ctx* c, int64_t n, int depth) {
    if (n > c->cap_n) {
        for (int b = 0; b < 2; ++b) {
            dfree(c->keys[b]);
            dfree(c->vals[b]);
        }
        dfree(c->sorted6);
        dfree(c->near6);
        dfree(c->radix_tmp);
        c->cap_n = 0;
        for (int b = 0; b < 2; ++b) {
            CK(cudaMalloc((void**)&c->keys[b], n * sizeof(uint32_t)), "alloc keys");
            CK(cudaMalloc((void**)&c->vals[b], n * sizeof(uint32_t)), "alloc vals");
        }
        CK(cudaMalloc((void**)&c->sorted6, 6 * n * sizeof(float)), "alloc sorted");
        CK(cudaMalloc((void**)&c->near6, 6 * n * sizeof(float)), "alloc near");
        c->radix_tmp_bytes = radix_temp_bytes(n);
        CK(cudaMalloc(&c->radix_tmp, c->radix_tmp_bytes), "alloc radix");
        c->cap_n = n;
    }
    if (depth != c->cap_depth || c->prm.p != c->cap_p) {
        dfree(c->leaf_start);
        dfree(c->Mall);
        dfree(c->Lall);
        c->cap_depth = -1;
        const int64_t nleaf = (int64_t)1 << (3 * depth);
        const int64_t cells = level_offset(depth + 1);
        const int nc = ncoef(c->prm.p);
        CK(cudaMalloc((void**)&c->leaf_start, (nleaf + 1) * sizeof(int)), "alloc leaf_start");
        CK(cudaMalloc((void**)&c->Mall, cells * 3 * nc * sizeof(float)), "alloc M");
        CK(cudaMalloc((void**)&c->Lall, cells * 3 * nc * sizeof(float)), "alloc L");
        c->cap_depth = depth;
        c->cap_p = c->prm.p;
    }
    return VFMM_OK;
}

DistShared make_shared(vfmm_ctx* c, int R) {
    DistShared D;
    D.prm = c->prm;
    D.depth = c->prm.depth;
    D.R = R;
    D.m2m = c->d_m2m;
    D.l2l = c->d_l2l;
    D.m2l = c->d_m2l;
    D.per = c->d_per;
    D.tc = tc_ops(c);
    D.l2p = l2p_map(c);
    D.m2m_scratch = c->m2m_scratch;
    D.m2m_scratch_floats = c->m2m_scratch_floats;
    D.slots = c->d_slots;
    D.KP = c->hops.KP;
    D.NR = c->hops.NR;
    D.allow_tc = m2l_env_mode() != 0;
    return D;
}

bool valid_R(int R) { return R == 1 || R == 2 || R == 4 || R == 8; }

void ensure_rank_states(vfmm_ctx* c, int R, int first_rank, int count) {
    while ((int)c->ranks.size() < count) c->ranks.push_back(new RankState());
    for (int i = 0; i < count; ++i) {
        RankState* S = c->ranks[i];
        S->rank = first_rank + i;
        const int per = c->prm.image_levels > 0;
        if (S->plan.L != c->prm.depth || S->plan.R != R || S->plan.rank != S->rank ||
            S->plan.periodic != per || S->plan.p_send.empty()) {
            build_dist_plan(c->prm.depth, R, S->rank, per, &S->plan);
            S->plan_dirty = true;
        }
    }
}

vfmm_status dist_sticky(vfmm_ctx* c, RankState* S) {
    int flag = 0;
    if (!S->d_err) return VFMM_OK;
    CK(cudaMemcpy(&flag, S->d_err, sizeof(int), cudaMemcpyDeviceToHost), "read flag");
    if (flag) {
        CK(cudaMemset(S->d_err, 0, sizeof(int)), "clear flag");
        c->err = "a particle lies outside the box (or is not finite)";
        return VFMM_EDOMAIN;
    }
    return VFMM_OK;
}

}  // namespace

extern "C" {

vfmm_status vfmm_partition(int depth, int nranks, int rank, int64_t* leaf_lo, int64_t* leaf_hi) {
    if (!valid_R(nranks) || rank < 0 || rank >= nranks || depth < 1 || depth > 10)
        return VFMM_EINVAL;
    const int64_t nleaf = (int64_t)1 << (3 * depth);
    if (leaf_lo) *leaf_lo = nleaf / nranks * rank;
    if (leaf_hi) *leaf_hi = nleaf / nranks * (rank + 1);
    return VFMM_OK;
}

vfmm_status vfmm_dist_plan(int depth, int nranks, int rank, int periodic, int kind, int dir,
                           int peer, int32_t* out, int64_t cap, int64_t* count) {
    if (!valid_R(nranks) || rank < 0 || rank >= nranks || peer < 0 || peer >= nranks ||
        depth < 2 || depth > 8 || !count || (kind != 0 && (kind < 2 || kind > depth)) ||
        (dir != 0 && dir != 1))
        return VFMM_EINVAL;
    DistPlan P;
    build_dist_plan(depth, nranks, rank, periodic ? 1 : 0, &P);
    const std::vector<int>& v = kind == 0 ? (dir == 0 ? P.p_recv[peer] : P.p_send[peer])
                                          : (dir == 0 ? P.m_recv[kind][peer] : P.m_send[kind][peer]);
    *count = (int64_t)v.size();
    if (out)
        for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)v.size()); ++i) out[i] = v[i];
    return VFMM_OK;
}

vfmm_status vfmm_nccl_get_unique_id(void* out128) {
    if (!out128) return VFMM_EINVAL;
    return nccl_unique_id(out128);
}

vfmm_status vfmm_create_nccl(vfmm_ctx** out, const vfmm_params* prm, int device,
                             const void* nccl_id128, int nranks, int rank) {
    if (!out || !nccl_id128 || !prm || !valid_R(nranks) || rank < 0 || rank >= nranks)
        return VFMM_EINVAL;
    if (prm->depth < 2 || prm->mode == VFMM_MODE_DIRECT || prm->mode == VFMM_MODE_HYBRID)
        return VFMM_EINVAL;
    vfmm_status s = vfmm_create(out, prm, device);
    if (s != VFMM_OK) return s;
    vfmm_ctx* c = *out;
    c->R = nranks;
    c->rank = rank;
    // every NCCL context runs the distributed phases, also with one rank (a 1-rank
    // communicator: the all-gathers degenerate to copies), so the NCCL plumbing is exercised
    c->dist = true;
    if (cudaStreamCreateWithFlags(&c->comm_st, cudaStreamNonBlocking) != cudaSuccess) {
        vfmm_destroy(c);
        *out = nullptr;
        return VFMM_ECUDA;
    }
    {
        s = nccl_init(&c->comm, nranks, rank, nccl_id128);
        if (s != VFMM_OK) {
            c->err = "ncclCommInitRank failed";
            vfmm_destroy(c);
            *out = nullptr;
            return s;
        }
    }
    return VFMM_OK;
}

vfmm_status vfmm_evaluate_logical(vfmm_ctx* c, int nranks, const int64_t* n,
                                  const float* const* pos, const float* const* gamma,
                                  float* const* vel, float* const* dgamma, void* stream) {
    if (!c || !valid_R(nranks) || !n || !pos || !gamma || !vel || !dgamma) return VFMM_EINVAL;
    if (c->prm.depth < 2 || c->prm.mode == VFMM_MODE_DIRECT || c->prm.mode == VFMM_MODE_HYBRID)
        return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    (void)cudaGetLastError();
    cudaStream_t st = (cudaStream_t)stream;
    if (c->last_stream != st && c->have_last)
        CK(cudaStreamWaitEvent(st, c->ev[vfmm_ctx::NEV - 1], 0), "order after last evaluate");
    c->have_last = true;
    ensure_rank_states(c, nranks, 0, nranks);
    CK(cudaEventRecord(c->ev[0], st), "event");
    DistShared D = make_shared(c, nranks);
    std::vector<RankState*> S(c->ranks.begin(), c->ranks.begin() + nranks);
    for (int r = 0; r < nranks; ++r) {
        if (n[r] < 0 || (n[r] > 0 && (!pos[r] || !gamma[r] || !vel[r] || !dgamma[r])))
            return VFMM_EINVAL;
        S[r]->n_in = n[r];
        S[r]->in_pos = pos[r];
        S[r]->in_gam = gamma[r];
        S[r]->in_vel = vel[r];
        S[r]->in_dg = dgamma[r];
    }
    vfmm_status s;
    int ce = 0;  // exchange timing events: (start, end) pairs on the one stream
    auto phase = [&](vfmm_status (*f)(RankState&, const DistShared&, cudaStream_t, std::string*)) {
        for (int r = 0; r < nranks; ++r) {
            vfmm_status t = f(*S[r], D, st, &c->err);
            if (t != VFMM_OK) return t;
        }
        return VFMM_OK;
    };
    auto xchg = [&](vfmm_status (*f)(std::vector<RankState*>&, const DistShared&, cudaStream_t)) {
        cudaEventRecord(c->evc[ce++], st);
        vfmm_status t = f(S, D, st);
        cudaEventRecord(c->evc[ce++], st);
        return t;
    };
    if ((s = phase(dist_phase0a)) != VFMM_OK) return s;
    if ((s = xchg(logical_x0a)) != VFMM_OK) return s;
    if ((s = phase(dist_phase0b)) != VFMM_OK) return s;
    if ((s = xchg(logical_x0b)) != VFMM_OK) return s;
    if ((s = phase(dist_phase0c)) != VFMM_OK) return s;
    if ((s = phase(dist_phase1)) != VFMM_OK) return s;
    if ((s = xchg(logical_x1)) != VFMM_OK) return s;
    if ((s = phase(dist_phase2)) != VFMM_OK) return s;
    if ((s = xchg(logical_x2)) != VFMM_OK) return s;
    if ((s = phase(dist_unpack_halo)) != VFMM_OK) return s;
    if ((s = phase(dist_phase3)) != VFMM_OK) return s;
    if ((s = xchg(logical_x3)) != VFMM_OK) return s;
    if ((s = phase(dist_unpack_let)) != VFMM_OK) return s;
    if ((s = phase(dist_phase4_far)) != VFMM_OK) return s;
    if ((s = phase(dist_phase4_near)) != VFMM_OK) return s;
    if ((s = phase(dist_phase5a)) != VFMM_OK) return s;
    if ((s = xchg(logical_x5)) != VFMM_OK) return s;
    if ((s = phase(dist_phase5b)) != VFMM_OK) return s;
    for (int i = 1; i < vfmm_ctx::NEV; ++i) CK(cudaEventRecord(c->ev[i], st), "event");
    c->last_stream = st;
    c->have_tree = false;
    c->have_exp = false;
    c->comm_timed = true;
    c->comm_overlap = false;
    memset(&c->stats, 0, sizeof(c->stats));
    c->stats.depth_used = c->prm.depth;
    for (int r = 0; r < nranks; ++r) {
        c->stats.bytes_sent += S[r]->bytes_sent;
        c->stats.bytes_recv += S[r]->bytes_recv;
    }
    CK(cudaStreamSynchronize(st), "sync");
    for (int r = 0; r < nranks; ++r)
        if ((s = dist_sticky(c, S[r])) != VFMM_OK) return s;
    return VFMM_OK;
}

vfmm_status vfmm_route_counts(int depth, int nranks, int64_t n, const float* pos_h, float box_lo,
                              float box_len, int64_t* counts) {
    if (!valid_R(nranks) || depth < 1 || depth > 10 || n < 0 || !counts || (n > 0 && !pos_h) ||
        !(box_len > 0.f))
        return VFMM_EINVAL;
    const int64_t per = ((int64_t)1 << (3 * depth)) / nranks;
    for (int q = 0; q < nranks; ++q) counts[q] = 0;
    bool all_in = true;
    for (int64_t i = 0; i < n; ++i) {
        bool in = true;
        const int64_t leaf = host_leaf_of(pos_h[i], pos_h[n + i], pos_h[2 * n + i], depth, box_lo,
                                          box_len, &in);
        all_in &= in;
        counts[leaf / per] += 1;
    }
    return all_in ? VFMM_OK : VFMM_EDOMAIN;
}

int32_t vfmm_abi_version(void) { return VFMM_ABI_VERSION; }

void vfmm_params_default(vfmm_params* prm) {
    if (!prm) return;
    prm->p = 10;
    prm->depth = 0;
    prm->image_levels = 3;
    prm->scheme = VFMM_STRETCH_CLASSICAL;
    prm->mode = VFMM_MODE_FMM;
    prm->sigma = (float)(2.0 * M_PI / 256.0);
    prm->box_lo = (float)(-M_PI);
    prm->box_len = (float)(2.0 * M_PI);
}

const char* vfmm_strerror(vfmm_status s) {
    switch (s) {
        case VFMM_OK: return "VFMM_OK";
        case VFMM_EINVAL: return "VFMM_EINVAL: invalid parameter";
        case VFMM_EDOMAIN: return "VFMM_EDOMAIN: position outside the box or non-finite input";
        case VFMM_ENOMEM: return "VFMM_ENOMEM: device allocation failed";
        case VFMM_ECUDA: return "VFMM_ECUDA: CUDA error";
        case VFMM_ENCCL: return "VFMM_ENCCL: NCCL error";
        case VFMM_ESTATE: return "VFMM_ESTATE: invalid state";
    }
    return "unknown vfmm_status";
}

const char* vfmm_last_error_message(const vfmm_ctx* c) { return c ? c->err.c_str() : ""; }

vfmm_status vfmm_create(vfmm_ctx** out, const vfmm_params* prm, int device) {
    if (!out) return VFMM_EINVAL;
    *out = nullptr;
    vfmm_status s = validate(prm);
    if (s != VFMM_OK) return s;
    vfmm_ctx* c = new vfmm_ctx();
    c->prm = *prm;
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete c;
        return VFMM_ECUDA;
    }
    s = ensure_ops(c);
    if (s == VFMM_OK) {
        cudaError_t e2 = cudaMalloc((void**)&c->d_err, sizeof(int));
        if (e2 == cudaSuccess) e2 = cudaMalloc((void**)&c->d_pairs, sizeof(unsigned long long));
        if (e2 == cudaSuccess) e2 = cudaMemset(c->d_err, 0, sizeof(int));
        if (e2 == cudaSuccess) e2 = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
        // the side stream (coarse M2L levels, latency-bound chains of few CTAs) gets the
        // highest priority, so its CTAs take SMs as soon as level-L CTAs retire and the coarse
        // levels run under the level-L kernel instead of after it
        int prio_least = 0, prio_greatest = 0;
        if (e2 == cudaSuccess) e2 = cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest);
        if (e2 == cudaSuccess)
            e2 = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_greatest);
        if (e2 == cudaSuccess)
            e2 = cudaStreamCreateWithPriority(&c->far_st, cudaStreamNonBlocking, prio_greatest);
        if (e2 == cudaSuccess) e2 = cudaEventCreateWithFlags(&c->ev_tree, cudaEventDisableTiming);
        if (e2 == cudaSuccess) e2 = cudaEventCreateWithFlags(&c->ev_far, cudaEventDisableTiming);
        if (e2 == cudaSuccess) e2 = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
        if (e2 == cudaSuccess) e2 = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
        if (e2 == cudaSuccess) e2 = cudaEventCreateWithFlags(&c->ev_gamma, cudaEventDisableTiming);
        for (int i = 0; i < vfmm_ctx::NEV && e2 == cudaSuccess; ++i) e2 = cudaEventCreate(&c->ev[i]);
        for (int i = 0; i < vfmm_ctx::NCE && e2 == cudaSuccess; ++i) e2 = cudaEventCreate(&c->evc[i]);
        if (e2 != cudaSuccess) s = cuda_fail(c, e2, "create");
    }
    if (s != VFMM_OK) {
        vfmm_destroy(c);
        return s;
    }
    *out = c;
    return VFMM_OK;
}

vfmm_status vfmm_set_params(vfmm_ctx* c, const vfmm_params* prm) {
    if (!c) return VFMM_EINVAL;
    vfmm_status s = validate(prm);
    if (s != VFMM_OK) return s;
    CK(cudaSetDevice(c->device), "set device");
    if (c->last_stream) CK(cudaStreamSynchronize(c->last_stream), "sync");
    c->prm = *prm;
    c->have_exp = false;
    return ensure_ops(c);
}

static vfmm_status evaluate_impl(vfmm_ctx* c, int64_t n, const float* pos, const float* gamma,
                                 const float* sig, float* vel, float* dgamma, void* stream);

vfmm_status vfmm_evaluate(vfmm_ctx* c, int64_t n, const float* pos, const float* gamma,
                          float* vel, float* dgamma, void* stream) {
    return evaluate_impl(c, n, pos, gamma, nullptr, vel, dgamma, stream);
}

vfmm_status vfmm_evaluate_sigma(vfmm_ctx* c, int64_t n, const float* pos, const float* gamma,
                                const float* sigma, float* vel, float* dgamma, void* stream) {
    if (!c || !sigma || c->dist) return VFMM_EINVAL;
    return evaluate_impl(c, n, pos, gamma, sigma, vel, dgamma, stream);
}

static vfmm_status evaluate_impl(vfmm_ctx* c, int64_t n, const float* pos, const float* gamma,
                                 const float* sig, float* vel, float* dgamma, void* stream) {
    if (!c || n < 0 || (n == 0 && !c->dist)) return VFMM_EINVAL;
    if (n > 0 && (!pos || !gamma || !vel || !dgamma)) return VFMM_EINVAL;
    if (n > ((int64_t)1 << 31) - 1) return VFMM_EINVAL;
    // outputs must not alias inputs or each other
    auto overlap = [n](const void* a, const void* b) {
        const char* x = (const char*)a;
        const char* y = (const char*)b;
        const size_t L = 3 * (size_t)n * sizeof(float);
        return x < y + L && y < x + L;
    };
    if (overlap(vel, dgamma) || overlap(vel, pos) || overlap(vel, gamma) ||
        overlap(dgamma, pos) || overlap(dgamma, gamma))
        return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    (void)cudaGetLastError();  // drop stale non-sticky errors of unrelated earlier calls
    cudaStream_t st = (cudaStream_t)stream;
    // the workspace is shared by every evaluate of this context: work on a new stream waits
    // for the previous evaluate (its last event) before touching it
    if (c->last_stream != st && c->have_last)
        CK(cudaStreamWaitEvent(st, c->ev[vfmm_ctx::NEV - 1], 0), "order after last evaluate");
    c->have_last = true;
    c->tree_last = false;
    if (c->dist) {  // distributed evaluation over NCCL (this process = one rank)
        ensure_rank_states(c, c->R, c->rank, 1);
        DistShared D = make_shared(c, c->R);
        RankState& R0 = *c->ranks[0];
        R0.n_in = n;
        R0.in_pos = pos;
        R0.in_gam = gamma;
        R0.in_vel = vel;
        R0.in_dg = dgamma;
        cudaStream_t cs = c->comm_st;
        cudaEvent_t* E = c->evc;
        vfmm_status s;
        // every NCCL call runs on the communication stream cs, ordered by events; X0/X1/X5
        // are waited for at once, X2 (halo particles) overlaps P2M / M2M / M2L and X3 (LET
        // multipoles) overlaps the LET packing tail until the M2L needs it
        auto to_comm = [&](int e_ready) {
            CK(cudaEventRecord(E[e_ready], st), "event");
            CK(cudaStreamWaitEvent(cs, E[e_ready], 0), "wait");
            CK(cudaEventRecord(E[e_ready + 1], cs), "event");
            return VFMM_OK;
        };
        CK(cudaEventRecord(c->ev[0], st), "event");
        NvtxRange nv("vfmm/dist/redistribute");
        if ((s = dist_phase0a(R0, D, st, &c->err)) != VFMM_OK) return s;
        if ((s = to_comm(0)) != VFMM_OK) return s;
        if ((s = nccl_x0a(R0, D, c->comm, cs)) != VFMM_OK) return s;
        CK(cudaEventRecord(E[2], cs), "event");
        CK(cudaStreamWaitEvent(st, E[2], 0), "wait");
        if ((s = dist_phase0b(R0, D, st, &c->err)) != VFMM_OK) return s;
        if ((s = to_comm(3)) != VFMM_OK) return s;
        if ((s = nccl_x0b(R0, D, c->comm, cs)) != VFMM_OK) return s;
        CK(cudaEventRecord(E[5], cs), "event");
        CK(cudaStreamWaitEvent(st, E[5], 0), "wait");
        if ((s = dist_phase0c(R0, D, st, &c->err)) != VFMM_OK) return s;
        if ((s = dist_phase1(R0, D, st, &c->err)) != VFMM_OK) return s;
        if ((s = to_comm(6)) != VFMM_OK) return s;
        if ((s = nccl_x1(R0, D, c->comm, cs)) != VFMM_OK) return s;
        CK(cudaEventRecord(E[8], cs), "event");
        CK(cudaStreamWaitEvent(st, E[8], 0), "wait");
        nv.next("vfmm/dist/halo_let");
        if ((s = dist_phase2(R0, D, st, &c->err)) != VFMM_OK) return s;
        if ((s = to_comm(9)) != VFMM_OK) return s;
        if ((s = nccl_x2(R0, D, c->comm, cs)) != VFMM_OK) return s;
        if ((s = dist_unpack_halo(R0, D, cs, &c->err)) != VFMM_OK) return s;
        CK(cudaEventRecord(E[11], cs), "event");
        if ((s = dist_phase3(R0, D, st, &c->err)) != VFMM_OK) return s;
        if ((s = to_comm(12)) != VFMM_OK) return s;
        if ((s = nccl_x3(R0, D, c->comm, cs)) != VFMM_OK) return s;
        if ((s = dist_unpack_let(R0, D, cs, &c->err)) != VFMM_OK) return s;
        CK(cudaEventRecord(E[14], cs), "event");
        CK(cudaEventRecord(E[15], st), "event");  // compute stream ready for the LET
        CK(cudaStreamWaitEvent(st, E[14], 0), "wait");
        nv.next("vfmm/dist/evaluate");
        if ((s = dist_phase4_far(R0, D, st, &c->err)) != VFMM_OK) return s;
        CK(cudaEventRecord(E[16], st), "event");  // compute stream ready for the halo
        CK(cudaStreamWaitEvent(st, E[11], 0), "wait");
        if ((s = dist_phase4_near(R0, D, st, &c->err)) != VFMM_OK) return s;
        nv.next("vfmm/dist/return");
        if ((s = dist_phase5a(R0, D, st, &c->err)) != VFMM_OK) return s;
        if ((s = to_comm(17)) != VFMM_OK) return s;
        if ((s = nccl_x5(R0, D, c->comm, cs)) != VFMM_OK) return s;
        CK(cudaEventRecord(E[19], cs), "event");
        CK(cudaStreamWaitEvent(st, E[19], 0), "wait");
        if ((s = dist_phase5b(R0, D, st, &c->err)) != VFMM_OK) return s;
        for (int i = 1; i < vfmm_ctx::NEV; ++i) CK(cudaEventRecord(c->ev[i], st), "event");
        memset(&c->stats, 0, sizeof(c->stats));
        c->stats.bytes_sent = R0.bytes_sent;
        c->stats.bytes_recv = R0.bytes_recv;
        c->stats.depth_used = c->prm.depth;
        c->last_stream = st;
        c->have_tree = false;
        c->have_exp = false;
        c->comm_timed = true;
        c->comm_overlap = true;
        return VFMM_OK;
    }
    if (c->prm.mode == VFMM_MODE_HYBRID) {
        // "a properly implemented FMM [...] always selects the least expensive option"
        // (PAPER.md:150): the first evaluate of a new (n, p, image_levels, depth) times the
        // FMM (cell-cell) and the treecode (cell-particle, theta = 0.5) at n_crit = 32, 64, 128
        // particles per leaf ("automatically choosing the number of particles per box",
        // PAPER.md:152) and keeps the fastest; per-particle sigma always takes the FMM
        auto run = [&](int k) -> vfmm_status {
            if (k > 0)
                return vfmm_evaluate_tree(c, n, pos, gamma, vel, dgamma, 0.5f, 16 << k, stream);
            c->prm.mode = VFMM_MODE_FMM;
            const vfmm_status r = evaluate_impl(c, n, pos, gamma, sig, vel, dgamma, stream);
            c->prm.mode = VFMM_MODE_HYBRID;
            return r;
        };
        if (sig) return run(0);
        if (!(c->hyb_n == n && c->hyb_p == c->prm.p && c->hyb_levels == c->prm.image_levels &&
              c->hyb_depth == c->prm.depth)) {
            cudaEvent_t t0, t1;
            CK(cudaEventCreate(&t0), "event");
            CK(cudaEventCreate(&t1), "event");
            int best = 0;
            for (int k = 0; k < 4; ++k) {
                vfmm_status r = run(k);  // warm-up (and the depth tuning for depth = -1)
                if (r == VFMM_OK) {
                    cudaEventRecord(t0, st);
                    r = run(k);
                    cudaEventRecord(t1, st);
                }
                if (r != VFMM_OK) {
                    cudaEventDestroy(t0);
                    cudaEventDestroy(t1);
                    return r;
                }
                CK(cudaEventSynchronize(t1), "sync");
                cudaEventElapsedTime(&c->hyb_ms[k], t0, t1);
                if (c->hyb_ms[k] < c->hyb_ms[best]) best = k;
            }
            cudaEventDestroy(t0);
            cudaEventDestroy(t1);
            c->hyb_choice = best;
            c->hyb_n = n;
            c->hyb_p = c->prm.p;
            c->hyb_levels = c->prm.image_levels;
            c->hyb_depth = c->prm.depth;
        }
        return run(c->hyb_choice);
    }
    const vfmm_params& P = c->prm;
    vfmm_stats& S = c->stats;
    memset(&S, 0, sizeof(S));
    c->comm_timed = false;
    c->last_stream = st;
    c->last_n = n;
    const KernelConsts kc = make_kernel_consts(P.sigma);
    CK(cudaEventRecord(c->ev[0], st), "event");
    if (P.mode == VFMM_MODE_DIRECT) {
        if (c->gamma_pending) {
            CK(cudaStreamWaitEvent(st, c->ev_gamma, 0), "wait h2d");
            c->gamma_pending = false;
        }
        if (sig)
            launch_direct_sigma(pos, gamma, sig, n, P.box_len, P.image_levels, P.scheme, vel,
                                dgamma, st);
        else
            launch_direct(pos, gamma, n, P.box_len, P.image_levels, P.scheme, kc, vel, dgamma, st);
        CK(cudaGetLastError(), "direct kernel");
        for (int i = 1; i < vfmm_ctx::NEV; ++i) CK(cudaEventRecord(c->ev[i], st), "event");
        int m = 0;
        for (int l = 0; l < P.image_levels; ++l) m = 3 * m + 1;
        S.n_p2p_pairs = n * n * (int64_t)((2 * m + 1) * (2 * m + 1) * (2 * m + 1));
        S.n_kernel_launches = 1;
        c->have_tree = false;
        c->have_exp = false;
        return VFMM_OK;
    }
    // a cached choice stays valid while its leaf width keeps >= 4 sigma (reading R3; sigma
    // grows by core spreading in vfmm_step)
    const bool tuned_valid =
        c->tuned_n == n && c->tuned_p == P.p && c->tuned_mode == P.mode &&
        c->tuned_levels == P.image_levels &&
        (double)P.box_len / (double)(1 << c->tuned_depth) >= 4.0 * (double)P.sigma * (1.0 - 1e-6);
    if (P.depth == -1 && !tuned_valid) {
        // time the default depth and its two neighbours once (the paper's auto-tuning picks
        // the particles per box by measurement), keep the fastest
        const int L0 = auto_depth(P, n);
        float best = 1e30f;
        int bestL = L0;
        cudaEvent_t t0, t1;
        CK(cudaEventCreate(&t0), "event");
        CK(cudaEventCreate(&t1), "event");
        for (int k = 0; k < 3; ++k) {
            const int L = L0 - 1 + k;
            c->tuned_ms[k] = 0.f;
            if (L < 1 || L > 10) continue;
            if ((double)P.box_len / (double)(1 << L) < 4.0 * (double)P.sigma * (1.0 - 1e-6)) continue;
            if (((int64_t)1 << (3 * L)) > 64 * n + 8) continue;  // hardly any particle per leaf
            c->prm.depth = L;
            vfmm_status s0 = evaluate_impl(c, n, pos, gamma, sig, vel, dgamma, stream);  // warm-up
            if (s0 == VFMM_OK) {
                cudaEventRecord(t0, st);
                s0 = evaluate_impl(c, n, pos, gamma, sig, vel, dgamma, stream);
                cudaEventRecord(t1, st);
            }
            c->prm.depth = -1;
            if (s0 != VFMM_OK) {
                cudaEventDestroy(t0);
                cudaEventDestroy(t1);
                return s0;
            }
            CK(cudaEventSynchronize(t1), "sync");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t0, t1);
            c->tuned_ms[k] = ms;
            if (ms < best) {
                best = ms;
                bestL = L;
            }
        }
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        c->tuned_n = n;
        c->tuned_p = P.p;
        c->tuned_mode = P.mode;
        c->tuned_levels = P.image_levels;
        c->tuned_depth = bestL;
    }
    const int depth = P.depth > 0 ? P.depth : (P.depth == -1 ? c->tuned_depth : auto_depth(P, n));
    vfmm_status s = ensure_ws(c, n, depth);
    if (s != VFMM_OK) return s;
    c->last_depth = depth;
    S.depth_used = depth;
    Geom g{P.box_lo, P.box_len, (double)P.box_lo, (double)P.box_len, depth, P.image_levels > 0};
    const float a = (float)((double)P.box_len / (double)(1 << depth));  // exact in float
    int nl = 0;
    // ---- tree ----
    NvtxRange nv("vfmm/tree");
    launch_keys(pos, n, g, c->keys[0], c->vals[0], c->d_err, st);
    ++nl;
    CK(cudaEventRecord(c->ev[1], st), "event");
    launch_radix_sort(c->keys[0], c->vals[0], c->keys[1], c->vals[1], n, 3 * depth, c->radix_tmp,
                      st, &c->keys_sorted, &c->perm, &nl);
    CK(cudaEventRecord(c->ev[2], st), "event");
    launch_leaf_ranges(c->keys_sorted, n, depth, c->leaf_start, st);
    if (c->gamma_pending) {  // evaluate_host: the strengths arrive on the side stream
        CK(cudaStreamWaitEvent(st, c->ev_gamma, 0), "wait h2d");
        c->gamma_pending = false;
    }
    launch_gather(pos, gamma, c->perm, c->keys_sorted, n, g, c->sorted6, n, 0, st);
    nl += 2;
    CK(cudaGetLastError(), "tree kernels");
    CK(cudaEventRecord(c->ev[3], st), "event");
    c->have_tree = true;
    const bool use_far = P.mode == VFMM_MODE_FMM || P.mode == VFMM_MODE_FAR_ONLY;
    const bool use_near = P.mode == VFMM_MODE_FMM || P.mode == VFMM_MODE_NEAR_ONLY;
    const int p = P.p, nc = ncoef(p);
    const HostOps& H = c->hops;
    auto Mlev = [&](int l) { return c->Mall + level_offset(l) * 3 * nc; };
    auto Llev = [&](int l) { return c->Lall + level_offset(l) * 3 * nc; };
    // Co-resident mode (VFMM_CORES=1): the near field (FP32 pipe) runs on the caller's stream
    // concurrently with the far-field chain (tensor pipe) on a high-priority stream; the lean
    // kernel variants (P2P 61.5 KB, tcgen05 M2L 161 KB / 192 threads) let one block of each
    // share an SM.  Otherwise everything runs in sequence on the caller's stream.
    const char* cores_env = getenv("VFMM_CORES");
    const bool cores = cores_env && cores_env[0] == '1' && use_far && use_near && !sig;
    cudaStream_t fs = st;  // stream of the far-field chain
    if (cores) {
        CK(cudaEventRecord(c->ev_tree, st), "event");
        CK(cudaStreamWaitEvent(c->far_st, c->ev_tree, 0), "fork far field");
        fs = c->far_st;
        CK(cudaMemsetAsync(c->d_pairs, 0, sizeof(unsigned long long), st), "memset pairs");
        launch_p2p(c->sorted6, n, c->leaf_start, depth, a, P.image_levels > 0, P.scheme, kc,
                   c->near6, c->d_pairs, 0, (int64_t)1 << (3 * (depth - 1)), st, true);
        ++nl;
        CK(cudaGetLastError(), "p2p kernel");
    }
    // ---- upward pass ----
    nv.next("vfmm/upward");
    if (use_far) {
        launch_p2m(c->sorted6, n, c->leaf_start, p, 1.f / a, Mlev(depth), 0,
                   (int64_t)1 << (3 * depth), fs);
        ++nl;
    }
    CK(cudaEventRecord(c->ev[4], st), "event");
    if (use_far) {
        for (int l = depth - 1; l >= 0; --l) {
            nl += launch_m2m(c->d_m2m, p, H.KP, H.NR, Mlev(l + 1), Mlev(l), l, 0,
                             (int64_t)1 << (3 * l), c->m2m_scratch, c->m2m_scratch_floats, fs);
            S.n_m2m += (int64_t)8 << (3 * l);
        }
        CK(cudaGetLastError(), "upward kernels");
    }
    CK(cudaEventRecord(c->ev[5], fs), "event");
    // ---- M2L at every level (writes L_l), then periodic images + L2L top-down (adds) ----
    // The levels are independent: levels 1..L-1 (few CTAs each, latency bound) and the
    // periodic-image operator run on a side stream concurrently with level L (fork/join by
    // events), each stream with its own tensor-core staging buffer.
    nv.next("vfmm/m2l");
    if (use_far) {
        TcOps tco = tc_ops(c);
        tco.lean = cores;
        const bool allow_tc = m2l_env_mode() != 0 && tco.hi;
        CK(cudaMemsetAsync(c->d_tcmax, 0, 32 * sizeof(uint32_t), fs), "memset tc max");
        CK(cudaEventRecord(c->ev_fork, fs), "fork");
        CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0), "fork");
        for (int l = depth; l >= 1; --l) {
            cudaStream_t sl = l == depth ? fs : c->side;
            float** ghi = l == depth ? &c->g_hi : &c->g2_hi;
            float** glo = l == depth ? &c->g_lo : &c->g2_lo;
            size_t* gcap = l == depth ? &c->g_cap : &c->g2_cap;
            const int box[6] = {0, 0, 0, 1 << (l - 1), 1 << (l - 1), 1 << (l - 1)};
            if (allow_tc && m2l_tc_supported(p, l) && m2l_tc_shape_ok(box, p)) {
                const size_t need = m2l_tc_grid_floats(l);
                if (need > *gcap) {
                    CK(cudaStreamSynchronize(sl), "sync before grid realloc");
                    dfree(*ghi);
                    dfree(*glo);
                    *gcap = 0;
                    CK(cudaMalloc((void**)ghi, need * sizeof(float)), "alloc m2l grid");
                    CK(cudaMalloc((void**)glo, need * sizeof(float)), "alloc m2l grid");
                    *gcap = need;
                }
                const int rc = launch_m2l_tc(tco, c->d_slots, p, Mlev(l), Llev(l), l,
                                             P.image_levels > 0, *ghi, *glo, c->d_tcmax + l, box,
                                             sl);
                if (rc != 0) {
                    c->err = "tensor-map encode failed for tcgen05 M2L";
                    return VFMM_ECUDA;
                }
                nl += tco.f16 ? 3 : 2;
            } else {
                nl += launch_m2l(c->d_m2l, c->d_slots, p, H.KP, H.NR, Mlev(l), Llev(l), l,
                                 P.image_levels > 0, 0, (int64_t)1 << (3 * (l - 1)),
                                 l == depth ? c->m2m_scratch : c->side_scratch,
                                 l == depth ? c->m2m_scratch_floats : c->side_scratch_floats, sl);
            }
            S.n_m2l += (int64_t)189 << (3 * l);
        }
        if (P.image_levels >= 2) {
            launch_periodic(c->d_per, p, H.KP, H.NR, Mlev(0), Llev(0), c->side);
            ++nl;
        } else {
            CK(cudaMemsetAsync(Llev(0), 0, 3 * nc * sizeof(float), c->side), "memset L0");
        }
        CK(cudaEventRecord(c->ev_join, c->side), "join");
        CK(cudaStreamWaitEvent(fs, c->ev_join, 0), "join");
        CK(cudaGetLastError(), "m2l kernels");
    }
    CK(cudaEventRecord(c->ev[6], fs), "event");
    nv.next("vfmm/downward");
    if (use_far) {
        for (int l = 1; l <= depth; ++l) {
            launch_l2l(c->d_l2l, p, H.KP, H.NR, Llev(l - 1), Llev(l), l, 0,
                       (int64_t)1 << (3 * (l - 1)), fs);
            ++nl;
            S.n_l2l += (int64_t)1 << (3 * l);
        }
        CK(cudaGetLastError(), "downward kernels");
        c->have_exp = true;
    }
    CK(cudaEventRecord(c->ev[7], fs), "event");
    if (cores) {  // join the far-field chain
        CK(cudaEventRecord(c->ev_far, fs), "event");
        CK(cudaStreamWaitEvent(st, c->ev_far, 0), "join far field");
    }
    if (getenv("VFMM_DEBUG_SYNC")) CK(cudaStreamSynchronize(st), "debug sync");
    // ---- near field ----
    nv.next("vfmm/p2p");
    if (use_near && !cores) {
        CK(cudaMemsetAsync(c->d_pairs, 0, sizeof(unsigned long long), st), "memset pairs");
        if (sig) {  // per-particle core radius: sigma into Morton order, the sigma_j P2P
            if (n > c->cap_sig_n) {
                dfree(c->sorted_sig);
                c->cap_sig_n = 0;
                CK(cudaMalloc((void**)&c->sorted_sig, n * sizeof(float)), "alloc sorted sigma");
                c->cap_sig_n = n;
            }
            launch_gather1(sig, c->perm, n, c->sorted_sig, st);
            launch_p2p_sigma(c->sorted6, c->sorted_sig, n, c->leaf_start, depth, a,
                             P.image_levels > 0, P.scheme, c->near6, c->d_pairs, 0,
                             (int64_t)1 << (3 * (depth - 1)), st);
            nl += 2;
        } else
        launch_p2p(c->sorted6, n, c->leaf_start, depth, a, P.image_levels > 0, P.scheme, kc,
                   c->near6, c->d_pairs, 0, (int64_t)1 << (3 * (depth - 1)), st);
        ++nl;
        CK(cudaGetLastError(), "p2p kernel");
    }
    CK(cudaEventRecord(c->ev[8], st), "event");
    nv.next("vfmm/l2p");
    launch_l2p_combine(l2p_map(c), c->sorted6, c->near6, c->perm, n, c->leaf_start, p, a, Llev(depth),
                       P.scheme, use_near, use_far, vel, dgamma, 0, (int64_t)1 << (3 * depth), 0, n,
                       st);
    ++nl;
    CK(cudaGetLastError(), "l2p kernel");
    CK(cudaEventRecord(c->ev[9], st), "event");
    S.n_kernel_launches = nl;
    return VFMM_OK;
}

vfmm_status vfmm_evaluate_tree(vfmm_ctx* c, int64_t n, const float* pos, const float* gamma,
                               float* vel, float* dgamma, float theta, int32_t n_crit,
                               void* stream) {
    if (!c || n < 1 || !pos || !gamma || !vel || !dgamma) return VFMM_EINVAL;
    if (c->dist || !(theta >= 0.f && theta < 1.f) || n_crit < 1) return VFMM_EINVAL;
    if (n > ((int64_t)1 << 31) - 1) return VFMM_EINVAL;
    auto overlap = [n](const void* a, const void* b) {
        const char* x = (const char*)a;
        const char* y = (const char*)b;
        const size_t L = 3 * (size_t)n * sizeof(float);
        return x < y + L && y < x + L;
    };
    if (overlap(vel, dgamma) || overlap(vel, pos) || overlap(vel, gamma) ||
        overlap(dgamma, pos) || overlap(dgamma, gamma))
        return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    (void)cudaGetLastError();
    cudaStream_t st = (cudaStream_t)stream;
    if (c->last_stream != st && c->have_last)
        CK(cudaStreamWaitEvent(st, c->ev[vfmm_ctx::NEV - 1], 0), "order after last evaluate");
    c->have_last = true;
    const vfmm_params& P = c->prm;
    vfmm_stats& S = c->stats;
    memset(&S, 0, sizeof(S));
    c->comm_timed = false;
    c->last_stream = st;
    c->last_n = n;
    c->tree_last = true;
    const KernelConsts kc = make_kernel_consts(P.sigma);
    // finest level: the context's depth, else the FMM's automatic one (leaf width >= 4 sigma,
    // so every cell-particle interaction the MAC accepts is far outside the cores, reading R3)
    const int depth = P.depth > 0 ? P.depth : auto_depth(P, n);
    vfmm_status s = ensure_ws(c, n, depth);
    if (s != VFMM_OK) return s;
    const size_t gcap = tree_groups_cap(n, depth);
    if (gcap > c->tree_groups_cap || !c->d_tree_ng) {
        if (c->last_stream) CK(cudaStreamSynchronize(c->last_stream), "sync");
        dfree(c->tree_groups);
        c->tree_groups_cap = 0;
        CK(cudaMalloc((void**)&c->tree_groups, gcap * sizeof(int2)), "alloc tree groups");
        c->tree_groups_cap = gcap;
        if (!c->d_tree_ng) CK(cudaMalloc((void**)&c->d_tree_ng, sizeof(int)), "alloc");
        if (!c->d_tree_cnt)
            CK(cudaMalloc((void**)&c->d_tree_cnt, 2 * sizeof(unsigned long long)), "alloc");
    }
    c->last_depth = depth;
    S.depth_used = depth;
    Geom g{P.box_lo, P.box_len, (double)P.box_lo, (double)P.box_len, depth, P.image_levels > 0};
    const float a = (float)((double)P.box_len / (double)(1 << depth));
    const int p = P.p, nc = ncoef(p);
    const HostOps& H = c->hops;
    auto Mlev = [&](int l) { return c->Mall + level_offset(l) * 3 * nc; };
    auto Llev = [&](int l) { return c->Lall + level_offset(l) * 3 * nc; };
    int nl = 0;
    NvtxRange nv("vfmm/tree");
    CK(cudaEventRecord(c->ev[0], st), "event");
    launch_keys(pos, n, g, c->keys[0], c->vals[0], c->d_err, st);
    CK(cudaEventRecord(c->ev[1], st), "event");
    launch_radix_sort(c->keys[0], c->vals[0], c->keys[1], c->vals[1], n, 3 * depth, c->radix_tmp,
                      st, &c->keys_sorted, &c->perm, &nl);
    CK(cudaEventRecord(c->ev[2], st), "event");
    launch_leaf_ranges(c->keys_sorted, n, depth, c->leaf_start, st);
    launch_gather(pos, gamma, c->perm, c->keys_sorted, n, g, c->sorted6, n, 0, st);
    nl += 3;
    CK(cudaGetLastError(), "tree kernels");
    CK(cudaEventRecord(c->ev[3], st), "event");
    c->have_tree = true;
    // multipoles of every cell (Eq. 10 about the cell centres): P2M + M2M, as in the FMM
    nv.next("vfmm/upward");
    launch_p2m(c->sorted6, n, c->leaf_start, p, 1.f / a, Mlev(depth), 0, (int64_t)1 << (3 * depth),
               st);
    ++nl;
    CK(cudaEventRecord(c->ev[4], st), "event");
    for (int l = depth - 1; l >= 0; --l)
        nl += launch_m2m(c->d_m2m, p, H.KP, H.NR, Mlev(l + 1), Mlev(l), l, 0, (int64_t)1 << (3 * l),
                         c->m2m_scratch, c->m2m_scratch_floats, st);
    CK(cudaGetLastError(), "upward kernels");
    CK(cudaEventRecord(c->ev[5], st), "event");
    // images outside the near 3^3 block: root local expansion, L2L to the leaves
    const bool rings = P.image_levels >= 2;
    nv.next("vfmm/m2l");
    if (rings) {
        launch_periodic(c->d_per, p, H.KP, H.NR, Mlev(0), Llev(0), st);
        CK(cudaMemsetAsync(Llev(1), 0, (level_offset(depth + 1) - 1) * 3 * nc * sizeof(float), st),
           "memset L");
        ++nl;
    }
    CK(cudaEventRecord(c->ev[6], st), "event");
    nv.next("vfmm/downward");
    if (rings) {
        for (int l = 1; l <= depth; ++l) {
            launch_l2l(c->d_l2l, p, H.KP, H.NR, Llev(l - 1), Llev(l), l, 0,
                       (int64_t)1 << (3 * (l - 1)), st);
            ++nl;
        }
        CK(cudaGetLastError(), "downward kernels");
    }
    CK(cudaEventRecord(c->ev[7], st), "event");
    // the traversal: cell-particle and particle-particle interactions into near6
    nv.next("vfmm/p2p");
    launch_tree(c->sorted6, n, c->keys_sorted, c->leaf_start, depth, a, P.image_levels > 0,
                P.scheme, p, n_crit, theta, c->Mall, kc, c->tree_groups, c->d_tree_ng,
                c->d_tree_cnt, c->near6, st);
    nl += 2;
    CK(cudaGetLastError(), "tree traversal");
    CK(cudaEventRecord(c->ev[8], st), "event");
    nv.next("vfmm/l2p");
    launch_l2p_combine(l2p_map(c), c->sorted6, c->near6, c->perm, n, c->leaf_start, p, a,
                       Llev(depth), P.scheme, true, rings, vel, dgamma, 0,
                       (int64_t)1 << (3 * depth), 0, n, st);
    ++nl;
    CK(cudaGetLastError(), "l2p kernel");
    CK(cudaEventRecord(c->ev[9], st), "event");
    S.n_kernel_launches = nl;
    c->have_exp = false;
    return VFMM_OK;
}

vfmm_status vfmm_evaluate_at(vfmm_ctx* c, int64_t n_src, const float* pos, const float* gamma,
                             int64_t n_tgt, const float* tpos, float* tvel, void* stream) {
    if (!c || n_src < 0 || n_tgt < 0 || (n_src > 0 && (!pos || !gamma)) ||
        (n_tgt > 0 && (!tpos || !tvel)))
        return VFMM_EINVAL;
    const int64_t N = n_src + n_tgt;
    if (N == 0 && !c->dist) return VFMM_EINVAL;
    if (N > ((int64_t)1 << 31) - 1) return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    cudaStream_t st = (cudaStream_t)stream;
    if (c->last_stream != st && c->have_last)  // at_buf may still be read by the last evaluate
        CK(cudaStreamWaitEvent(st, c->ev[vfmm_ctx::NEV - 1], 0), "order after last evaluate");
    if (N > c->cap_at_n) {
        if (c->last_stream) CK(cudaStreamSynchronize(c->last_stream), "sync");
        dfree(c->at_buf);
    c->rbf.release();
        c->cap_at_n = 0;
        CK(cudaMalloc((void**)&c->at_buf, 12 * std::max<int64_t>(N, 1) * sizeof(float)),
           "alloc target buffers");
        c->cap_at_n = N;
    }
    float* P = c->at_buf;        // positions: sources then targets, per component
    float* G = P + 3 * N;        // strengths: targets carry zero strength
    float* V = G + 3 * N;
    float* S = V + 3 * N;
    for (int a = 0; a < 3; ++a) {
        if (n_src) {
            CK(cudaMemcpyAsync(P + a * N, pos + a * n_src, n_src * 4, cudaMemcpyDeviceToDevice, st), "copy");
            CK(cudaMemcpyAsync(G + a * N, gamma + a * n_src, n_src * 4, cudaMemcpyDeviceToDevice, st), "copy");
        }
        if (n_tgt) {
            CK(cudaMemcpyAsync(P + a * N + n_src, tpos + a * n_tgt, n_tgt * 4, cudaMemcpyDeviceToDevice, st), "copy");
            CK(cudaMemsetAsync(G + a * N + n_src, 0, n_tgt * 4, st), "zero");
        }
    }
    vfmm_status s = vfmm_evaluate(c, N, P, G, V, S, stream);
    if (s != VFMM_OK) return s;
    for (int a = 0; a < 3 && n_tgt; ++a)
        CK(cudaMemcpyAsync(tvel + a * n_tgt, V + a * N + n_src, n_tgt * 4, cudaMemcpyDeviceToDevice, st),
           "copy");
    return VFMM_OK;
}

vfmm_status vfmm_reinit(vfmm_ctx* c, int64_t n_old, const float* pos_old,
                        const float* gamma_old, float sigma_old, int64_t n_new,
                        const float* pos_new, float sigma_new, float tol, int32_t max_iter,
                        int32_t restart, float* gamma_new, float* omega_new,
                        vfmm_reinit_info* info, void* stream) {
    if (!c || c->dist || n_old < 1 || n_new < 1 || !pos_old || !gamma_old || !pos_new ||
        !gamma_new || !finite_pos(sigma_old) || !finite_pos(sigma_new) || !(tol > 0.f) ||
        !std::isfinite(tol) || max_iter < 1 || restart < 1 || restart > 200)
        return VFMM_EINVAL;
    if (n_old > ((int64_t)1 << 31) - 1 || n_new > ((int64_t)1 << 31) - 1) return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    (void)cudaGetLastError();
    cudaStream_t st = (cudaStream_t)stream;
    if (c->last_stream != st && c->have_last)
        CK(cudaStreamWaitEvent(st, c->ev[vfmm_ctx::NEV - 1], 0), "order after last evaluate");
    const vfmm_params& P = c->prm;
    const int depth = P.depth > 0 ? P.depth : auto_depth(P, n_new);
    const int64_t nleaf = (int64_t)1 << (3 * depth);
    const float a = (float)((double)P.box_len / (double)(1 << depth));
    const int periodic = P.image_levels > 0;
    const int ws_old = rbf_ws(a, sigma_old), ws_new = rbf_ws(a, sigma_new);
    // (a neighbour cube wider than the periodic box visits further images of the same leaves:
    // each offset is a distinct image, so the truncated periodic sum stays exact)
    const int m = restart;
    RbfWs& W = c->rbf;
    const int64_t n = n_new;
    // ---- workspace ----
    if (n_old > W.cap_old) {
        for (int b = 0; b < 2; ++b) {
            dfree(W.ok[b]);
            dfree(W.ov[b]);
        }
        dfree(W.otmp);
        dfree(W.o6);
        W.cap_old = 0;
        for (int b = 0; b < 2; ++b) {
            CK(cudaMalloc((void**)&W.ok[b], n_old * 4), "alloc rbf");
            CK(cudaMalloc((void**)&W.ov[b], n_old * 4), "alloc rbf");
        }
        CK(cudaMalloc(&W.otmp, radix_temp_bytes(n_old)), "alloc rbf");
        CK(cudaMalloc((void**)&W.o6, 6 * n_old * sizeof(float)), "alloc rbf");
        W.cap_old = n_old;
    }
    if (n_new > W.cap_new || m > W.cap_m) {
        for (int b = 0; b < 2; ++b) {
            dfree(W.nk[b]);
            dfree(W.nv[b]);
        }
        dfree(W.ntmp);
        dfree(W.n6);
        dfree(W.V);
        dfree(W.w);
        dfree(W.x);
        dfree(W.om);
        dfree(W.part);
        dfree(W.dots);
        dfree(W.coef);
        W.cap_new = 0;
        W.cap_m = -1;
        const int64_t nn = std::max(n_new, W.cap_new);
        for (int b = 0; b < 2; ++b) {
            CK(cudaMalloc((void**)&W.nk[b], nn * 4), "alloc rbf");
            CK(cudaMalloc((void**)&W.nv[b], nn * 4), "alloc rbf");
        }
        CK(cudaMalloc(&W.ntmp, radix_temp_bytes(nn)), "alloc rbf");
        CK(cudaMalloc((void**)&W.n6, 6 * nn * sizeof(float)), "alloc rbf");
        CK(cudaMalloc((void**)&W.V, (size_t)(m + 1) * 3 * nn * sizeof(float)), "alloc Krylov basis");
        CK(cudaMalloc((void**)&W.w, 3 * nn * sizeof(float)), "alloc rbf");
        CK(cudaMalloc((void**)&W.x, 3 * nn * sizeof(float)), "alloc rbf");
        CK(cudaMalloc((void**)&W.om, 3 * nn * sizeof(float)), "alloc rbf");
        CK(cudaMalloc((void**)&W.part, rbf_dot_part_doubles(m + 1) * sizeof(double)), "alloc rbf");
        CK(cudaMalloc((void**)&W.dots, 3 * (m + 1) * sizeof(double)), "alloc rbf");
        CK(cudaMalloc((void**)&W.coef, 3 * (m + 1) * sizeof(double)), "alloc rbf");
        W.cap_new = nn;
        W.cap_m = m;
    }
    if (depth != W.cap_depth) {
        dfree(W.ols);
        dfree(W.nls);
        W.cap_depth = -1;
        CK(cudaMalloc((void**)&W.ols, (nleaf + 1) * 4), "alloc rbf");
        CK(cudaMalloc((void**)&W.nls, (nleaf + 1) * 4), "alloc rbf");
        W.cap_depth = depth;
    }
    CK(cudaEventRecord(c->ev[0], st), "event");
    // ---- trees of the old and the new particles (same depth) ----
    Geom g{P.box_lo, P.box_len, (double)P.box_lo, (double)P.box_len, depth, periodic};
    int nl = 0;
    uint32_t *oks = nullptr, *operm = nullptr, *nks = nullptr, *nperm = nullptr;
    launch_keys(pos_old, n_old, g, W.ok[0], W.ov[0], c->d_err, st);
    launch_radix_sort(W.ok[0], W.ov[0], W.ok[1], W.ov[1], n_old, 3 * depth, W.otmp, st, &oks,
                      &operm, &nl);
    launch_leaf_ranges(oks, n_old, depth, W.ols, st);
    launch_gather(pos_old, gamma_old, operm, oks, n_old, g, W.o6, n_old, 0, st);
    launch_keys(pos_new, n_new, g, W.nk[0], W.nv[0], c->d_err, st);
    launch_radix_sort(W.nk[0], W.nv[0], W.nk[1], W.nv[1], n_new, 3 * depth, W.ntmp, st, &nks,
                      &nperm, &nl);
    launch_leaf_ranges(nks, n_new, depth, W.nls, st);
    // the new particles carry no strength yet: the gather's strength rows are unused
    launch_gather(pos_new, pos_new, nperm, nks, n_new, g, W.n6, n_new, 0, st);
    CK(cudaGetLastError(), "reinit tree kernels");
    // ---- right-hand side: omega at the new points (Eq. 3), initial guess omega dx^3 ----
    launch_gauss(W.n6, n, W.nls, W.o6, n_old, W.ols, nullptr, depth, a, periodic, ws_old,
                 sigma_old, W.om, st);
    const double dx3 = (double)P.box_len * (double)P.box_len * (double)P.box_len / (double)n_new;
    {
        const double al[3] = {dx3, dx3, dx3}, be[3] = {0, 0, 0};
        launch_scale3(W.om, nullptr, W.x, n, al, be, st);
    }
    CK(cudaGetLastError(), "reinit rhs kernels");
    // ---- GMRES(m), the three components in lockstep (same matrix) ----
    auto matvec = [&](const float* v, float* out) {  // out = A v
        launch_gauss(W.n6, n, W.nls, W.n6, n, W.nls, v, depth, a, periodic, ws_new, sigma_new, out,
                     st);
    };
    std::vector<double> hd(3 * (m + 1));
    auto dots = [&](const float* X, int nv, const float* Y) -> vfmm_status {
        launch_multidot(X, 3 * n, nv, Y, n, W.part, W.dots, st);
        CK(cudaMemcpyAsync(hd.data(), W.dots, 3 * nv * sizeof(double), cudaMemcpyDeviceToHost, st),
           "copy dots");
        CK(cudaStreamSynchronize(st), "sync dots");
        return VFMM_OK;
    };
    double beta0[3] = {0, 0, 0}, res[3] = {0, 0, 0};
    int total = 0;
    bool conv = false;
    std::vector<double> H(3 * (size_t)(m + 1) * m), gv(3 * (m + 1)), cs(3 * m), sn(3 * m);
    auto Hc = [&](int c, int i, int k) -> double& { return H[((size_t)c * (m + 1) + i) * m + k]; };
    vfmm_status sres;
    for (int cycle = 0;; ++cycle) {
        // r = omega - A x -> V_0
        matvec(W.x, W.w);
        {
            const double al[3] = {1, 1, 1}, be[3] = {-1, -1, -1};
            launch_scale3(W.om, W.w, W.V, n, al, be, st);
        }
        if ((sres = dots(W.V, 1, W.V)) != VFMM_OK) return sres;
        double beta[3];
        bool done[3];
        for (int cc = 0; cc < 3; ++cc) {
            beta[cc] = std::sqrt(std::max(hd[cc], 0.0));
            if (cycle == 0) beta0[cc] = beta[cc];
            res[cc] = beta0[cc] > 0 ? beta[cc] / beta0[cc] : 0.0;
            done[cc] = beta0[cc] == 0 || beta[cc] <= (double)tol * beta0[cc];
        }
        conv = done[0] && done[1] && done[2];
        if (conv || total >= max_iter) break;
        {
            double al[3], be[3] = {0, 0, 0};
            for (int cc = 0; cc < 3; ++cc) al[cc] = done[cc] ? 0.0 : 1.0 / beta[cc];
            launch_scale3(W.V, nullptr, W.V, n, al, be, st);
        }
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(gv.begin(), gv.end(), 0.0);
        for (int cc = 0; cc < 3; ++cc) gv[cc * (m + 1)] = done[cc] ? 0.0 : beta[cc];
        bool active[3] = {!done[0], !done[1], !done[2]};
        int kused = 0;
        for (int k = 0; k < m && total < max_iter; ++k) {
            float* vk = W.V + (size_t)k * 3 * n;
            matvec(vk, W.w);
            ++total;
            for (int pass = 0; pass < 2; ++pass) {  // classical Gram-Schmidt, twice
                if ((sres = dots(W.V, k + 1, W.w)) != VFMM_OK) return sres;
                std::vector<double> coef(3 * (k + 1));
                for (int i = 0; i <= k; ++i)
                    for (int cc = 0; cc < 3; ++cc) {
                        const double h = active[cc] ? hd[i * 3 + cc] : 0.0;
                        Hc(cc, i, k) += h;
                        coef[i * 3 + cc] = -h;
                    }
                CK(cudaMemcpyAsync(W.coef, coef.data(), coef.size() * sizeof(double),
                                   cudaMemcpyHostToDevice, st),
                   "copy coef");
                launch_multiaxpy(W.V, 3 * n, k + 1, W.coef, W.w, n, st);
                CK(cudaStreamSynchronize(st), "sync coef");  // coef (host) reused next pass
            }
            if ((sres = dots(W.w, 1, W.w)) != VFMM_OK) return sres;
            double al[3], be[3] = {0, 0, 0};
            bool all = true;
            for (int cc = 0; cc < 3; ++cc) {
                const double hn = std::sqrt(std::max(hd[cc], 0.0));
                al[cc] = 0.0;
                if (!active[cc]) continue;
                Hc(cc, k + 1, k) = hn;
                al[cc] = hn > 1e-300 ? 1.0 / hn : 0.0;
                // Givens rotations on column k
                double* csc = &cs[cc * m];
                double* snc = &sn[cc * m];
                for (int i = 0; i < k; ++i) {
                    const double t = csc[i] * Hc(cc, i, k) + snc[i] * Hc(cc, i + 1, k);
                    Hc(cc, i + 1, k) = -snc[i] * Hc(cc, i, k) + csc[i] * Hc(cc, i + 1, k);
                    Hc(cc, i, k) = t;
                }
                const double hk = Hc(cc, k, k), hk1 = Hc(cc, k + 1, k);
                const double r = std::hypot(hk, hk1);
                csc[k] = r > 0 ? hk / r : 1.0;
                snc[k] = r > 0 ? hk1 / r : 0.0;
                Hc(cc, k, k) = r;
                Hc(cc, k + 1, k) = 0.0;
                double* gc = &gv[cc * (m + 1)];
                gc[k + 1] = -snc[k] * gc[k];
                gc[k] = csc[k] * gc[k];
                res[cc] = std::fabs(gc[k + 1]) / beta0[cc];
                if (res[cc] <= (double)tol || hn <= 1e-300) active[cc] = false;
                all = all && !active[cc];
            }
            launch_scale3(W.w, nullptr, W.V + (size_t)(k + 1) * 3 * n, n, al, be, st);
            kused = k + 1;
            if (all) break;
        }
        // x += V y, H y = g (upper triangular, per component)
        std::vector<double> coef(3 * kused, 0.0);
        for (int cc = 0; cc < 3; ++cc) {
            if (done[cc]) continue;
            std::vector<double> y(kused, 0.0);
            for (int i = kused - 1; i >= 0; --i) {
                double t = gv[cc * (m + 1) + i];
                for (int j = i + 1; j < kused; ++j) t -= Hc(cc, i, j) * y[j];
                y[i] = Hc(cc, i, i) != 0 ? t / Hc(cc, i, i) : 0.0;
            }
            for (int i = 0; i < kused; ++i) coef[i * 3 + cc] = y[i];
        }
        if (kused) {
            CK(cudaMemcpyAsync(W.coef, coef.data(), coef.size() * sizeof(double),
                               cudaMemcpyHostToDevice, st),
               "copy coef");
            launch_multiaxpy(W.V, 3 * n, kused, W.coef, W.x, n, st);
            CK(cudaStreamSynchronize(st), "sync coef");
        }
    }
    // ---- outputs in the input order of the new particles ----
    launch_unpermute3(W.x, nperm, n, gamma_new, st);
    if (omega_new) launch_unpermute3(W.om, nperm, n, omega_new, st);
    CK(cudaGetLastError(), "reinit kernels");
    for (int i = 1; i < vfmm_ctx::NEV; ++i) CK(cudaEventRecord(c->ev[i], st), "event");
    CK(cudaStreamSynchronize(st), "sync");
    c->last_stream = st;
    c->have_last = true;
    c->have_tree = false;
    c->have_exp = false;
    c->prm.sigma = sigma_new;
    if (info) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[vfmm_ctx::NEV - 1]);
        info->iterations = total;
        info->converged = conv ? 1 : 0;
        for (int cc = 0; cc < 3; ++cc) info->rel_residual[cc] = res[cc];
        info->ms = ms;
        info->depth_used = depth;
        info->ws_old = ws_old;
        info->ws_new = ws_new;
    }
    int flag = 0;
    CK(cudaMemcpy(&flag, c->d_err, sizeof(int), cudaMemcpyDeviceToHost), "read flag");
    if (flag) {
        CK(cudaMemset(c->d_err, 0, sizeof(int)), "clear flag");
        c->err = "reinit: a position outside the box or non-finite";
        return VFMM_EDOMAIN;
    }
    return VFMM_OK;
}

vfmm_status vfmm_step(vfmm_ctx* c, int64_t n, float* pos, float* gamma, float dt, float nu,
                      float* vel, float* dgamma, float* sigma_out, void* stream) {
    if (!c || !std::isfinite(dt) || !std::isfinite(nu) || !(nu >= 0.f)) return VFMM_EINVAL;
    if (n < 0 || (n == 0 && !c->dist) || (n > 0 && (!pos || !gamma))) return VFMM_EINVAL;
    const double s2 = (double)c->prm.sigma * (double)c->prm.sigma + 2.0 * (double)nu * (double)dt;
    if (!(s2 > 0.0) || !std::isfinite((float)std::sqrt(s2))) return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    float* v = vel;
    float* s = dgamma;
    if (n > 0 && (!v || !s)) {
        if (n > c->cap_step_n) {
            dfree(c->step_buf);
    dfree(c->at_buf);
    dfree(c->sorted_sig);
            c->cap_step_n = 0;
            CK(cudaMalloc((void**)&c->step_buf, 6 * n * sizeof(float)), "alloc step buffers");
            c->cap_step_n = n;
        }
        if (!v) v = c->step_buf;
        if (!s) s = c->step_buf + 3 * n;
    }
    vfmm_status st = vfmm_evaluate(c, n, pos, gamma, v, s, stream);
    if (st != VFMM_OK) return st;
    if (n > 0) {
        launch_euler_update(pos, gamma, v, s, n, dt, c->prm.box_lo, c->prm.box_len,
                            c->prm.image_levels > 0, (cudaStream_t)stream);
        CK(cudaGetLastError(), "euler update kernel");
        c->stats.n_kernel_launches += 1;
    }
    c->prm.sigma = (float)std::sqrt(s2);  // core spreading, uniform core (Eq. 9)
    if (sigma_out) *sigma_out = c->prm.sigma;
    return VFMM_OK;
}

vfmm_status vfmm_evaluate_host(vfmm_ctx* c, int64_t n, const float* pos_h, const float* gamma_h,
                               float* vel_h, float* dgamma_h) {
    if (!c || n < 1 || !pos_h || !gamma_h || !vel_h || !dgamma_h) return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    if (n > c->cap_host_n) {
        dfree(c->hbuf);
        c->cap_host_n = 0;
        CK(cudaMalloc((void**)&c->hbuf, 12 * n * sizeof(float)), "alloc host staging");
        c->cap_host_n = n;
    }
    float* dp = c->hbuf;
    float* dg = dp + 3 * n;
    float* dv = dg + 3 * n;
    float* ds = dv + 3 * n;
    cudaStream_t st = c->own_stream;
    CK(cudaMemcpyAsync(dp, pos_h, 3 * n * sizeof(float), cudaMemcpyHostToDevice, st), "h2d");
    // the strengths are first needed by the gather (after keys, sort and leaf ranges): copy
    // them on the side stream so the copy overlaps the tree build (single-context path)
    const bool overlap = !c->dist;
    if (overlap) {
        CK(cudaStreamWaitEvent(c->side, c->ev_join, 0), "order");  // previous evaluation done
        CK(cudaMemcpyAsync(dg, gamma_h, 3 * n * sizeof(float), cudaMemcpyHostToDevice, c->side),
           "h2d");
        CK(cudaEventRecord(c->ev_gamma, c->side), "event");
        c->gamma_pending = true;
    } else {
        CK(cudaMemcpyAsync(dg, gamma_h, 3 * n * sizeof(float), cudaMemcpyHostToDevice, st), "h2d");
    }
    vfmm_status s = vfmm_evaluate(c, n, dp, dg, dv, ds, st);
    c->gamma_pending = false;
    if (s != VFMM_OK) {
        // the caller's buffers may still be read by queued H2D copies: drain before returning
        cudaStreamSynchronize(st);
        cudaStreamSynchronize(c->side);
        return s;
    }
    CK(cudaMemcpyAsync(vel_h, dv, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, st), "d2h");
    CK(cudaMemcpyAsync(dgamma_h, ds, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, st), "d2h");
    return vfmm_sync_status(c);
}

vfmm_status vfmm_sync_status(vfmm_ctx* c) {
    if (!c) return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    CK(cudaStreamSynchronize(c->last_stream), "sync");
    if (c->dist) {
        vfmm_status s = nccl_async_error(c->comm, &c->err);
        if (s != VFMM_OK) return s;
    }
    if (c->dist && !c->ranks.empty()) {
        vfmm_status s = dist_sticky(c, c->ranks[0]);
        if (s != VFMM_OK) return s;
    }
    int flag = 0;
    CK(cudaMemcpy(&flag, c->d_err, sizeof(int), cudaMemcpyDeviceToHost), "read flag");
    if (flag) {
        CK(cudaMemset(c->d_err, 0, sizeof(int)), "clear flag");
        c->err = "input position outside [lo, lo+len)^3 or non-finite";
        return VFMM_EDOMAIN;
    }
    return VFMM_OK;
}

vfmm_status vfmm_get_stats(vfmm_ctx* c, vfmm_stats* out) {
    if (!c || !out) return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    CK(cudaStreamSynchronize(c->last_stream), "sync");
    vfmm_stats& S = c->stats;
    float ms[vfmm_ctx::NEV] = {0};
    for (int i = 1; i < vfmm_ctx::NEV; ++i)
        CK(cudaEventElapsedTime(&ms[i], c->ev[i - 1], c->ev[i]), "elapsed");
    S.ms_keys = ms[1];
    S.ms_sort = ms[2];
    S.ms_tree = ms[3];  // leaf ranges + gather
    S.ms_p2m = ms[4];
    S.ms_m2m = ms[5];
    S.ms_m2l = ms[6];
    S.ms_l2l = ms[7];   // periodic images + L2L
    S.ms_p2p = ms[8];
    S.ms_l2p = ms[9];   // L2P + near/far combine + un-permute
    float tot = 0;
    CK(cudaEventElapsedTime(&tot, c->ev[0], c->ev[vfmm_ctx::NEV - 1]), "elapsed");
    S.ms_total = tot;
    if (c->comm_timed) {
        auto el = [&](int a, int b) {
            float t = 0.f;
            return cudaEventElapsedTime(&t, c->evc[a], c->evc[b]) == cudaSuccess ? (double)t : 0.0;
        };
        if (c->comm_overlap) {  // NCCL: (start, end) of X0a, X0b, X1, X2, X3, X5 on the comm stream
            const double x0a = el(1, 2), x0b = el(4, 5), x1 = el(7, 8), x2 = el(10, 11),
                         x3 = el(13, 14), x5 = el(18, 19);
            S.ms_comm = x0a + x0b + x1 + x2 + x3 + x5;
            S.ms_comm_exposed = x0a + x0b + x1 + x5 + std::max(0.0, el(15, 14)) +
                                std::max(0.0, el(16, 11));
        } else {  // logical ranks: six (start, end) pairs on the one stream, all exposed
            double t = 0;
            for (int i = 0; i < 12; i += 2) t += el(i, i + 1);
            S.ms_comm = S.ms_comm_exposed = t;
        }
    }
    if (c->tree_last) {  // treecode: P2P pairs and M2P cell-particle interactions
        unsigned long long cnt[2] = {0, 0};
        CK(cudaMemcpy(cnt, c->d_tree_cnt, sizeof(cnt), cudaMemcpyDeviceToHost), "copy counts");
        S.n_p2p_pairs = (int64_t)cnt[0];
        S.n_m2l = (int64_t)cnt[1];
    } else if (c->prm.mode == VFMM_MODE_FMM || c->prm.mode == VFMM_MODE_NEAR_ONLY ||
               c->prm.mode == VFMM_MODE_HYBRID) {
        unsigned long long pairs = 0;
        CK(cudaMemcpy(&pairs, c->d_pairs, sizeof(pairs), cudaMemcpyDeviceToHost), "copy pairs");
        S.n_p2p_pairs = (int64_t)pairs;
    }
    *out = S;
    return VFMM_OK;
}

vfmm_status vfmm_debug_tree(vfmm_ctx* c, uint32_t* keys_sorted, uint32_t* perm,
                            int32_t* leaf_start) {
    if (!c) return VFMM_EINVAL;
    if (!c->have_tree) return VFMM_ESTATE;
    CK(cudaSetDevice(c->device), "set device");
    CK(cudaStreamSynchronize(c->last_stream), "sync");
    const int64_t n = c->last_n;
    if (keys_sorted)
        CK(cudaMemcpy(keys_sorted, c->keys_sorted, n * 4, cudaMemcpyDeviceToHost), "copy keys");
    if (perm) CK(cudaMemcpy(perm, c->perm, n * 4, cudaMemcpyDeviceToHost), "copy perm");
    if (leaf_start)
        CK(cudaMemcpy(leaf_start, c->leaf_start, (((int64_t)1 << (3 * c->last_depth)) + 1) * 4,
                      cudaMemcpyDeviceToHost),
           "copy leaf_start");
    return VFMM_OK;
}

vfmm_status vfmm_debug_expansions(vfmm_ctx* c, int kind, int level, float* out) {
    if (!c || !out || (kind != 0 && kind != 1)) return VFMM_EINVAL;
    if (!c->have_exp) return VFMM_ESTATE;
    if (level < 0 || level > c->last_depth) return VFMM_EINVAL;
    CK(cudaSetDevice(c->device), "set device");
    CK(cudaStreamSynchronize(c->last_stream), "sync");
    const int nc = ncoef(c->prm.p);
    const float* base = (kind == 0 ? c->Mall : c->Lall) + level_offset(level) * 3 * nc;
    CK(cudaMemcpy(out, base, ((size_t)1 << (3 * level)) * 3 * nc * sizeof(float),
                  cudaMemcpyDeviceToHost),
       "copy expansions");
    return VFMM_OK;
}

void vfmm_destroy(vfmm_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->last_stream) cudaStreamSynchronize(c->last_stream);
    dfree(c->tree_groups);
    dfree(c->d_tree_ng);
    dfree(c->d_tree_cnt);
    dfree(c->d_m2m);
    dfree(c->d_l2l);
    dfree(c->d_m2l);
    dfree(c->d_per);
    dfree(c->d_slots);
    dfree(c->d_groups);
    dfree(c->d_l2p_rowptr);
    dfree(c->d_l2p_pairs);
    dfree(c->m2m_scratch);
    dfree(c->side_scratch);
    dfree(c->d_tc_hi);
    dfree(c->d_tc_lo);
    dfree(c->d_h16_hi);
    dfree(c->d_h16_lo);
    dfree(c->d_h16_rs);
    dfree(c->d_h16_cs);
    dfree(c->d_tcmax);
    dfree(c->g_hi);
    dfree(c->g_lo);
    for (int b = 0; b < 2; ++b) {
        dfree(c->keys[b]);
        dfree(c->vals[b]);
    }
    dfree(c->radix_tmp);
    dfree(c->sorted6);
    dfree(c->near6);
    dfree(c->leaf_start);
    dfree(c->Mall);
    dfree(c->Lall);
    dfree(c->d_err);
    dfree(c->d_pairs);
    dfree(c->hbuf);
    dfree(c->step_buf);
    for (int i = 0; i < vfmm_ctx::NEV; ++i)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    for (int i = 0; i < vfmm_ctx::NCE; ++i)
        if (c->evc[i]) cudaEventDestroy(c->evc[i]);
    if (c->comm_st) cudaStreamDestroy(c->comm_st);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->far_st) cudaStreamDestroy(c->far_st);
    if (c->ev_tree) cudaEventDestroy(c->ev_tree);
    if (c->ev_far) cudaEventDestroy(c->ev_far);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_gamma) cudaEventDestroy(c->ev_gamma);
    dfree(c->g2_hi);
    dfree(c->g2_lo);
    for (auto* s : c->ranks) delete s;
    c->ranks.clear();
    if (c->comm) nccl_destroy(c->comm);
    delete c;
}

}  // extern "C"
