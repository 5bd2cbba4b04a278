// dist.h -- distributed (multi-GPU / logical-rank) FMM state and plans (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "vfmm_internal.h"

namespace vfmm {

// Static exchange plan of one rank for (depth L, R ranks, periodic).
struct DistPlan {
    int L = 0, R = 1, rank = 0, periodic = 1;
    std::vector<std::vector<int>> p_recv, p_send;               // [peer] -> halo leaves
    std::vector<std::vector<std::vector<int>>> m_recv, m_send;  // [level][peer] -> cells (l >= 2)
};
void build_dist_plan(int L, int R, int rank, int periodic, DistPlan* P);

// contiguous run of particles (rank-local compact sorted index) and its message offset
struct Seg {
    int64_t src;
    int64_t cnt;
    int64_t off;
};

// Per-rank device state of the distributed pipeline.
//
// C1 (redistribution): the caller's n_in particles (anywhere in the box) are Morton-sorted
// locally, cut at the rank boundaries and sent to their owners; the owner's n_own received
// particles (peer order, each peer's run in Morton order) are what the FMM phases evaluate.
// The results travel back the same way (reverse trip) and are scattered to the caller's order.
//
// Particle arrays are compact: only the rank's owned leaves and its halo leaves hold particles
// (leaf_start has zero-length ranges elsewhere), so they are sized owned + halo.  Expansion
// arrays keep the whole tree (M2L kernels address cells by global Morton index; 0.87 GB at
// c4 p = 10, < 0.5 % of HBM), written only where the rank owns or receives cells.
struct RankState {
    int rank = 0;
    DistPlan plan;
    bool plan_dirty = true;  // static device tables (need mask, LET cell lists) to upload
    // ---- C1: caller's particles ----
    int64_t n_in = 0, cap_in = 0;
    const float* in_pos = nullptr;
    const float* in_gam = nullptr;
    float* in_vel = nullptr;
    float* in_dg = nullptr;
    uint32_t *ikeys[2] = {nullptr, nullptr}, *ivals[2] = {nullptr, nullptr};
    void* itmp = nullptr;
    uint32_t *ikeys_sorted = nullptr, *iperm = nullptr;
    float* isend = nullptr;      // 6 x n_in AoS, local Morton order; reverse trip: results
    int* d_crow = nullptr;       // R particles per destination rank (this rank's row)
    int* d_cmat = nullptr;       // R x R, row = sender, column = receiver
    std::vector<int> h_cmat;
    std::vector<int64_t> c1_send_off, c1_send_cnt, c1_recv_off, c1_recv_cnt;  // particles
    int64_t n_own = 0, cap_own = 0;
    float* irecv = nullptr;      // 6 x n_own AoS, received order; reverse trip: results
    float* own = nullptr;        // 12 x n_own SoA: pos 3, gamma 3, vel 3, dgamma 3 (received order)
    // ---- the FMM phases on the owned particles ----
    int64_t n_local = 0, cap_local = 0;
    const float* pos = nullptr;
    const float* gam = nullptr;
    float* vel = nullptr;
    float* dg = nullptr;
    uint32_t *keys[2] = {nullptr, nullptr}, *vals[2] = {nullptr, nullptr};
    void* radix_tmp = nullptr;
    uint32_t *keys_sorted = nullptr, *perm = nullptr;
    int* lstart = nullptr;      // local leaf_start (8^L + 1)
    int* counts_own = nullptr;  // owned leaf counts (sized 8^L: any R)
    int* counts_all = nullptr;  // all leaf counts (8^L), all-gathered
    int* gstart = nullptr;      // compact leaf_start (8^L + 1): owned + halo leaves only
    uint8_t* d_need = nullptr;  // per leaf: 1 if owned or halo of this rank
    std::vector<int> hstart;    // host copy of gstart
    int64_t n_total = 0, cap_total = 0, gbase = 0;  // owned + halo particles; owned offset
    float *sorted6 = nullptr, *near6 = nullptr;
    float *Mall = nullptr, *Lall = nullptr;
    int cap_depth = -1, cap_p = -1, cap_R = -1;
    // messages
    float *sendbuf = nullptr, *recvbuf = nullptr;    // halo particles (AoS, 6 floats)
    size_t cap_send = 0, cap_recv = 0;               // floats
    float *msend = nullptr, *mrecv = nullptr;        // LET multipoles
    size_t cap_msend = 0, cap_mrecv = 0;             // floats
    int n_send_segs = 0;
    std::vector<Seg> h_segs;   // host copy (kept alive: the upload may still be reading it)
    Seg* d_segs = nullptr;
    int* d_cells = nullptr;    // LET cell ids: send lists then receive lists (static)
    size_t cap_segs = 0, cap_cells = 0;
    std::vector<int64_t> p_send_off, p_send_cnt, p_recv_off, p_recv_cnt;  // particles per peer
    std::vector<int64_t> m_send_off, m_send_cnt, m_recv_off, m_recv_cnt;  // floats per peer
    int64_t p_recv_total = 0, m_recv_floats = 0;
    int n_recv_segs = 0, n_recv_cells_off = 0, n_recv_cells = 0;
    int* d_err = nullptr;
    unsigned long long* d_pairs = nullptr;
    float *g_hi = nullptr, *g_lo = nullptr;  // tcgen05 M2L staging
    size_t g_cap = 0;
    uint32_t* tcmax = nullptr;  // [32] per-level f16 staging max
    int64_t bytes_sent = 0, bytes_recv = 0;
    ~RankState();
    void release();
};

// Read-only context data the distributed phases need (operators, parameters).
struct DistShared {
    vfmm_params prm;
    int depth = 0, R = 1;
    const float *m2m = nullptr, *l2l = nullptr, *m2l = nullptr, *per = nullptr;
    TcOps tc;  // tensor-core M2L operators (3xTF32 or 3xFP16)
    L2PMap l2p;  // L2P derivative map
    float* m2m_scratch = nullptr;  // coarse-level M2M op-split partials (used on the stream of
    size_t m2m_scratch_floats = 0; // the phase; logical ranks run their phases in sequence)
    const int* slots = nullptr;
    int KP = 0, NR = 0;
    bool allow_tc = true;
};

// Phases of one distributed evaluation (see dist.cu); exchanges happen between them.
//  0a input keys + sort + destination counts | X0a counts matrix | 0b offsets (host sync), pack
//  | X0b particles to owners | 0c unpack | 1 owned keys + sort + leaf counts | X1 leaf counts
//  | 2 compact leaf starts (host sync), gather, pack halo | X2 halo particles | unpack_halo
//  | 3 P2M, M2M, pack LET | X3 level-1 all-gather + LET multipoles | unpack_let
//  | 4far root M2M, M2L, periodic, L2L | 4near P2P, L2P | 5a pack results | X5 results back
//  | 5b scatter to the caller's order
vfmm_status dist_phase0a(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase0b(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase0c(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase1(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase2(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_unpack_halo(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase3(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_unpack_let(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase4_far(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase4_near(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase5a(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase5b(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
// exchanges, logical ranks (all ranks in this process, device copies)
vfmm_status logical_x0a(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
vfmm_status logical_x0b(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
vfmm_status logical_x1(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
vfmm_status logical_x2(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
vfmm_status logical_x3(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
vfmm_status logical_x5(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
// exchanges over NCCL (this rank), comm = ncclComm_t; every call checks every NCCL result
vfmm_status nccl_x0a(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
vfmm_status nccl_x0b(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
vfmm_status nccl_x1(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
vfmm_status nccl_x2(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
vfmm_status nccl_x3(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
vfmm_status nccl_x5(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
bool nccl_available();
vfmm_status nccl_unique_id(void* out128);
vfmm_status nccl_init(void** comm, int nranks, int rank, const void* id128);
vfmm_status nccl_async_error(void* comm, std::string* err);  // ncclCommGetAsyncError
void nccl_destroy(void* comm);

// host: Morton leaf of a float position triple at depth L (the keys kernel's arithmetic)
int64_t host_leaf_of(float x, float y, float z, int depth, float lo, float len, bool* inside);

}  // namespace vfmm
