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

// contiguous run of particles (global sorted index) or cells, and its message offset
struct Seg {
    int64_t src;
    int64_t cnt;
    int64_t off;
};

// Per-rank device state of the distributed pipeline.
struct RankState {
    int rank = 0;
    DistPlan plan;
    // local particles (this rank's input)
    int64_t n_local = 0, cap_local = 0;
    const float* pos = nullptr;
    const float* gam = nullptr;
    float* vel = nullptr;
    float* dg = nullptr;
    uint32_t *keys[2] = {nullptr, nullptr}, *vals[2] = {nullptr, nullptr};
    void* radix_tmp = nullptr;
    uint32_t *keys_sorted = nullptr, *perm = nullptr;
    int* lstart = nullptr;      // local leaf_start (8^L + 1)
    int* counts_own = nullptr;  // owned leaf counts (8^L / R)
    int* counts_all = nullptr;  // all leaf counts (8^L), all-gathered
    int* gstart = nullptr;      // global leaf_start (8^L + 1)
    std::vector<int> hstart;    // host copy of gstart
    // global-order particle arrays (owned + halo filled) and expansions (full tree size)
    int64_t n_total = 0, cap_total = 0, gbase = 0;
    float *sorted6 = nullptr, *near6 = nullptr;
    float *Mall = nullptr, *Lall = nullptr;
    int cap_depth = -1, cap_p = -1;
    // messages
    float *sendbuf = nullptr, *recvbuf = nullptr;    // halo particles (AoS, 6 floats)
    size_t cap_send = 0, cap_recv = 0;               // floats
    float *msend = nullptr, *mrecv = nullptr;        // LET multipoles
    size_t cap_msend = 0, cap_mrecv = 0;             // floats
    int n_send_segs = 0;
    Seg* d_segs = nullptr;
    int* d_cells = nullptr;
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
vfmm_status dist_phase1(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase2(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase3(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
vfmm_status dist_phase4(RankState& S, const DistShared& D, cudaStream_t st, std::string* err);
// exchanges, logical ranks (all ranks in this process, device copies)
vfmm_status logical_x1(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
vfmm_status logical_x2(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
vfmm_status logical_x3(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st);
// exchanges over NCCL (this rank), comm = ncclComm_t
vfmm_status nccl_x1(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
vfmm_status nccl_x2(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
vfmm_status nccl_x3(RankState& S, const DistShared& D, void* comm, cudaStream_t st);
bool nccl_available();
vfmm_status nccl_unique_id(void* out128);
vfmm_status nccl_init(void** comm, int nranks, int rank, const void* id128);
void nccl_destroy(void* comm);

}  // namespace vfmm
