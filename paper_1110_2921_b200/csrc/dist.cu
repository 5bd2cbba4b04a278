// dist.cu -- multi-GPU FMM: Morton-range spatial decomposition with a local-essential-tree
// (LET) exchange (SURVEY.md section 8(e); the paper's scaling runs, PAPER.md:41, :366-367,
// used MPI across 4096 GPUs -- here NCCL over NVLink/NVSwitch, one process per GPU).
//
// Rank r of R (R in {1, 2, 4, 8}) owns the contiguous Morton range of leaves
// [r 8^L/R, (r+1) 8^L/R), i.e. 8/R whole octants; at every level >= 1 its cells form a box.
// One evaluation:
//   1  local Morton keys + stable sort of the rank's particles (which must lie in its range)
//   X1 all-gather of owned leaf counts -> global leaf_start on every rank (+ one D2H copy so
//      the host knows halo message sizes)
//   2  owned particles -> their global sorted positions; pack halo leaves for the peers
//   X2 halo particle exchange (leaves within one leaf of a peer's range, periodic)
//   3  P2M, M2M over owned cells (levels L-1 .. 1); pack halo multipoles
//   X3 all-gather of level-1 multipoles + LET multipole exchange for levels 2..L (cells in a
//      peer's 189-cell interaction lists)
//   4  root M2M, periodic images and L2L redundantly on every rank; M2L, L2L, P2P, L2P for
//      owned cells; results back to the caller's input order on the same rank.
// The exchange plans are static for (L, R, periodic) and built once on the host.
// Transport: NCCL (grouped ncclSend/ncclRecv, ncclAllGather on the compute stream, library
// loaded with dlopen -- the same libnccl.so.2 torch uses), or "logical ranks": all R ranks'
// phases run on one GPU in lockstep and exchanges are device-to-device copies (tests).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "dist.h"

namespace vfmm {

// ---------------------------------------------------------------------------------------
// NCCL via dlopen
// ---------------------------------------------------------------------------------------
namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
        Send = (decltype(Send))dlsym(h, "ncclSend");
        Recv = (decltype(Recv))dlsym(h, "ncclRecv");
        AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        return GetUniqueId && CommInitRank && CommDestroy && GroupStart && GroupEnd && Send &&
               Recv && AllGather;
    }
};
NcclApi g_nccl;

// ---- kernels -------------------------------------------------------------------------

// exclusive scan of counts[0..m) -> start[0..m]; one block (small m, once per evaluation)
__global__ void scan_counts_kernel(const int* __restrict__ counts, int64_t m, int* __restrict__ start) {
    __shared__ int wsum[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t b = 0; b < m; b += blockDim.x) {
        const int64_t i = b + threadIdx.x;
        const int v = i < m ? counts[i] : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        int pre = 0, tot = 0;
        for (int k = 0; k < nw; ++k) {
            if (k < w) pre += wsum[k];
            tot += wsum[k];
        }
        const int c0 = carry;
        if (i < m) start[i] = c0 + pre + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry = c0 + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) start[m] = carry;
}

// owned leaf counts from the local leaf_start (all leaves) of the rank's particles; flags
// particles outside the owned range
__global__ void owned_counts_kernel(const int* __restrict__ lstart, int64_t leaf_lo,
                                    int64_t nown, int64_t nleaf, int64_t nlocal,
                                    int* __restrict__ counts, int* __restrict__ err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nown;
         i += (int64_t)gridDim.x * blockDim.x)
        counts[i] = lstart[leaf_lo + i + 1] - lstart[leaf_lo + i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // every local particle must fall in [leaf_lo, leaf_lo + nown)
        if (lstart[leaf_lo] != 0 || lstart[leaf_lo + nown] != nlocal) atomicOr(err, 2);
        (void)nleaf;
    }
}

// copy rows of a 6-component SoA array (stride n6) in [src, src+cnt) to an AoS buffer
__global__ void pack_particles_kernel(const float* __restrict__ s6, int64_t n6,
                                      const Seg* __restrict__ segs, int nseg,
                                      float* __restrict__ buf) {
    for (int s = blockIdx.x; s < nseg; s += gridDim.x) {
        const Seg g = segs[s];
        for (int64_t k = threadIdx.x; k < g.cnt * 6; k += blockDim.x) {
            const int64_t j = k / 6;
            const int c = (int)(k - j * 6);
            buf[(g.off + j) * 6 + c] = s6[c * n6 + g.src + j];
        }
    }
}
__global__ void unpack_particles_kernel(float* __restrict__ s6, int64_t n6,
                                        const Seg* __restrict__ segs, int nseg,
                                        const float* __restrict__ buf) {
    for (int s = blockIdx.x; s < nseg; s += gridDim.x) {
        const Seg g = segs[s];
        for (int64_t k = threadIdx.x; k < g.cnt * 6; k += blockDim.x) {
            const int64_t j = k / 6;
            const int c = (int)(k - j * 6);
            s6[c * n6 + g.src + j] = buf[(g.off + j) * 6 + c];
        }
    }
}
// cells: contiguous 3*nc floats each
__global__ void pack_cells_kernel(const float* __restrict__ M, int cellsz,
                                  const int* __restrict__ cells, int ncell, float* __restrict__ buf) {
    const int64_t total = (int64_t)ncell * cellsz;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = k / cellsz;
        buf[k] = M[(int64_t)cells[c] * cellsz + (k - c * cellsz)];
    }
}
__global__ void unpack_cells_kernel(float* __restrict__ M, int cellsz, const int* __restrict__ cells,
                                    int ncell, const float* __restrict__ buf) {
    const int64_t total = (int64_t)ncell * cellsz;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = k / cellsz;
        M[(int64_t)cells[c] * cellsz + (k - c * cellsz)] = buf[k];
    }
}

template <class T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

int64_t enc3(int x, int y, int z, int l) {
    int64_t k = 0;
    for (int b = 0; b < l; ++b)
        k |= ((int64_t)((x >> b) & 1) << (3 * b)) | ((int64_t)((y >> b) & 1) << (3 * b + 1)) |
             ((int64_t)((z >> b) & 1) << (3 * b + 2));
    return k;
}
void dec3(int64_t k, int l, int* x, int* y, int* z) {
    *x = *y = *z = 0;
    for (int b = 0; b < l; ++b) {
        *x |= (int)((k >> (3 * b)) & 1) << b;
        *y |= (int)((k >> (3 * b + 1)) & 1) << b;
        *z |= (int)((k >> (3 * b + 2)) & 1) << b;
    }
}

}  // namespace

// ---------------------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------------------

// cells at `level` that rank `r`'s owned targets need from other ranks, per owner:
// kind 0 = particle halo at the leaf level (27 neighbours), kind 1 = M2L sources (189 list)
static void needs(int level, int R, int r, int periodic, int kind,
                  std::vector<std::vector<int>>& per_owner) {
    const int side = 1 << level;
    const int64_t ncell = (int64_t)1 << (3 * level);
    const int64_t per = ncell / R;
    per_owner.assign(R, {});
    std::vector<uint8_t> mark(ncell, 0);
    for (int64_t t = r * per; t < (r + 1) * per; ++t) {
        int tx, ty, tz;
        dec3(t, level, &tx, &ty, &tz);
        auto visit = [&](int sx, int sy, int sz) {
            if (!periodic && (sx < 0 || sy < 0 || sz < 0 || sx >= side || sy >= side || sz >= side))
                return;
            sx &= side - 1;
            sy &= side - 1;
            sz &= side - 1;
            const int64_t s = enc3(sx, sy, sz, level);
            if (s / per != r) mark[s] = 1;
        };
        if (kind == 0) {
            for (int o = 0; o < 27; ++o) visit(tx + o % 3 - 1, ty + (o / 3) % 3 - 1, tz + o / 9 - 1);
        } else {
            const int px = tx >> 1, py = ty >> 1, pz = tz >> 1;
            for (int sx = 2 * px - 2; sx < 2 * px + 4; ++sx)
                for (int sy = 2 * py - 2; sy < 2 * py + 4; ++sy)
                    for (int sz = 2 * pz - 2; sz < 2 * pz + 4; ++sz) {
                        if (std::abs(sx - tx) <= 1 && std::abs(sy - ty) <= 1 && std::abs(sz - tz) <= 1)
                            continue;
                        visit(sx, sy, sz);
                    }
        }
    }
    for (int64_t s = 0; s < ncell; ++s)
        if (mark[s]) per_owner[s / per].push_back((int)s);
}

void build_dist_plan(int L, int R, int rank, int periodic, DistPlan* P) {
    P->L = L;
    P->R = R;
    P->rank = rank;
    P->periodic = periodic;
    P->p_recv.clear();
    P->p_send.assign(R, {});
    needs(L, R, rank, periodic, 0, P->p_recv);
    for (int q = 0; q < R; ++q) {
        if (q == rank) continue;
        std::vector<std::vector<int>> theirs;
        needs(L, R, q, periodic, 0, theirs);
        P->p_send[q] = theirs[rank];
    }
    P->m_recv.assign(L + 1, {});
    P->m_send.assign(L + 1, {});
    for (int l = 2; l <= L; ++l) {
        needs(l, R, rank, periodic, 1, P->m_recv[l]);
        P->m_send[l].assign(R, {});
        for (int q = 0; q < R; ++q) {
            if (q == rank) continue;
            std::vector<std::vector<int>> theirs;
            needs(l, R, q, periodic, 1, theirs);
            P->m_send[l][q] = theirs[rank];
        }
    }
}

// ---------------------------------------------------------------------------------------
// rank state
// ---------------------------------------------------------------------------------------

RankState::~RankState() { release(); }

void RankState::release() {
    for (int b = 0; b < 2; ++b) {
        dfree(keys[b]);
        dfree(vals[b]);
    }
    dfree(radix_tmp);
    dfree(lstart);
    dfree(counts_own);
    dfree(counts_all);
    dfree(gstart);
    dfree(sorted6);
    dfree(near6);
    dfree(Mall);
    dfree(Lall);
    dfree(sendbuf);
    dfree(recvbuf);
    dfree(msend);
    dfree(mrecv);
    cap_msend = cap_mrecv = 0;
    dfree(d_segs);
    dfree(d_cells);
    dfree(d_err);
    dfree(d_pairs);
    dfree(g_hi);
    dfree(g_lo);
    dfree(tcmax);
    cap_local = cap_total = 0;
    cap_send = cap_recv = 0;
    cap_segs = cap_cells = 0;
    g_cap = 0;
}

// ---------------------------------------------------------------------------------------
// phases
// ---------------------------------------------------------------------------------------
namespace {

#define DCK(call, what)                                                          \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            if (err) *err = std::string(what) + ": " + cudaGetErrorString(e_);   \
            return e_ == cudaErrorMemoryAllocation ? VFMM_ENOMEM : VFMM_ECUDA;   \
        }                                                                        \
    } while (0)

template <class T>
cudaError_t grow(T*& p, size_t& cap, size_t need) {
    if (need <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc((void**)&p, (need ? need : 1) * sizeof(T));
    if (e == cudaSuccess) cap = need;
    return e;
}

int grid_of(int64_t work, int bs = 256) {
    int64_t g = (work + bs - 1) / bs;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

int64_t owned_lo(int l, int R, int r) { return ((int64_t)r << (3 * l)) / R; }
int64_t owned_cnt(int l, int R) { return ((int64_t)1 << (3 * l)) / R; }

}  // namespace

vfmm_status dist_phase1(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R;
    const int64_t n = S.n_local;
    const int64_t nleaf = (int64_t)1 << (3 * L);
    if (n > S.cap_local) {
        for (int b = 0; b < 2; ++b) {
            dfree(S.keys[b]);
            dfree(S.vals[b]);
        }
        dfree(S.radix_tmp);
        S.cap_local = 0;
        for (int b = 0; b < 2; ++b) {
            DCK(cudaMalloc((void**)&S.keys[b], std::max<int64_t>(n, 1) * 4), "alloc keys");
            DCK(cudaMalloc((void**)&S.vals[b], std::max<int64_t>(n, 1) * 4), "alloc vals");
        }
        DCK(cudaMalloc(&S.radix_tmp, radix_temp_bytes(std::max<int64_t>(n, 1))), "alloc radix");
        S.cap_local = n;
    }
    if (S.cap_depth != L) {
        dfree(S.lstart);
        dfree(S.counts_own);
        dfree(S.counts_all);
        dfree(S.gstart);
        DCK(cudaMalloc((void**)&S.lstart, (nleaf + 1) * 4), "alloc lstart");
        // sized for R = 1 (the largest owned range): R may change between calls at one depth
        DCK(cudaMalloc((void**)&S.counts_own, nleaf * 4), "alloc counts");
        DCK(cudaMalloc((void**)&S.counts_all, nleaf * 4), "alloc counts");
        DCK(cudaMalloc((void**)&S.gstart, (nleaf + 1) * 4), "alloc gstart");
    }
    if (!S.d_err) {
        DCK(cudaMalloc((void**)&S.d_err, sizeof(int)), "alloc err");
        DCK(cudaMemset(S.d_err, 0, sizeof(int)), "memset err");
        DCK(cudaMalloc((void**)&S.d_pairs, sizeof(unsigned long long)), "alloc pairs");
    }
    const vfmm_params& P = D.prm;
    Geom g{P.box_lo, P.box_len, (double)P.box_lo, (double)P.box_len, L, P.image_levels > 0};
    int nl = 0;
    if (n > 0) {
        launch_keys(S.pos, n, g, S.keys[0], S.vals[0], S.d_err, st);
        launch_radix_sort(S.keys[0], S.vals[0], S.keys[1], S.vals[1], n, 3 * L, S.radix_tmp, st,
                          &S.keys_sorted, &S.perm, &nl);
        launch_leaf_ranges(S.keys_sorted, n, L, S.lstart, st);
    } else {
        DCK(cudaMemsetAsync(S.lstart, 0, (nleaf + 1) * 4, st), "memset lstart");
    }
    owned_counts_kernel<<<grid_of(nleaf / R), 256, 0, st>>>(S.lstart, owned_lo(L, R, S.rank),
                                                            nleaf / R, nleaf, n, S.counts_own,
                                                            S.d_err);
    DCK(cudaGetLastError(), "phase1 kernels");
    return VFMM_OK;
}

vfmm_status dist_phase2(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int64_t nleaf = (int64_t)1 << (3 * L);
    scan_counts_kernel<<<1, 1024, 0, st>>>(S.counts_all, nleaf, S.gstart);
    S.hstart.resize(nleaf + 1);
    DCK(cudaMemcpyAsync(S.hstart.data(), S.gstart, (nleaf + 1) * 4, cudaMemcpyDeviceToHost, st),
        "copy gstart");
    DCK(cudaStreamSynchronize(st), "sync gstart");
    S.n_total = S.hstart[nleaf];
    S.gbase = S.hstart[owned_lo(L, R, r)];
    const int nc = ncoef(D.prm.p);
    if (S.n_total > S.cap_total || S.cap_depth != L || S.cap_p != D.prm.p) {
        dfree(S.sorted6);
        dfree(S.near6);
        dfree(S.Mall);
        dfree(S.Lall);
        S.cap_total = 0;
        const int64_t nt = std::max<int64_t>(S.n_total, 1);
        DCK(cudaMalloc((void**)&S.sorted6, 6 * nt * 4), "alloc sorted6");
        DCK(cudaMalloc((void**)&S.near6, 6 * nt * 4), "alloc near6");
        const int64_t cells = level_offset(L + 1);
        DCK(cudaMalloc((void**)&S.Mall, cells * 3 * nc * 4), "alloc M");
        DCK(cudaMalloc((void**)&S.Lall, cells * 3 * nc * 4), "alloc L");
        DCK(cudaMemset(S.Mall, 0, cells * 3 * nc * 4), "memset M");
        S.cap_total = S.n_total;
        S.cap_depth = L;
        S.cap_p = D.prm.p;
    }
    const vfmm_params& P = D.prm;
    Geom g{P.box_lo, P.box_len, (double)P.box_lo, (double)P.box_len, L, P.image_levels > 0};
    if (S.n_local > 0)
        launch_gather(S.pos, S.gam, S.perm, S.keys_sorted, S.n_local, g, S.sorted6, S.n_total,
                      S.gbase, st);
    // ---- pack halo particles for every peer ----
    std::vector<Seg> segs;
    S.p_send_off.assign(R, 0);
    S.p_send_cnt.assign(R, 0);
    int64_t off = 0;
    for (int q = 0; q < R; ++q) {
        S.p_send_off[q] = off;
        for (int leaf : S.plan.p_send[q]) {
            const int64_t c = S.hstart[leaf + 1] - S.hstart[leaf];
            if (c) segs.push_back({S.hstart[leaf], c, off});
            off += c;
        }
        S.p_send_cnt[q] = off - S.p_send_off[q];
    }
    const int nsend_segs = (int)segs.size();
    S.n_send_segs = nsend_segs;
    S.p_recv_off.assign(R, 0);
    S.p_recv_cnt.assign(R, 0);
    int64_t roff = 0;
    for (int q = 0; q < R; ++q) {
        S.p_recv_off[q] = roff;
        for (int leaf : S.plan.p_recv[q]) {
            const int64_t c = S.hstart[leaf + 1] - S.hstart[leaf];
            if (c) segs.push_back({S.hstart[leaf], c, roff});
            roff += c;
        }
        S.p_recv_cnt[q] = roff - S.p_recv_off[q];
    }
    S.p_recv_total = roff;
    S.n_recv_segs = (int)segs.size() - nsend_segs;
    DCK(grow(S.d_segs, S.cap_segs, segs.size()), "alloc segs");
    if (!segs.empty())
        DCK(cudaMemcpyAsync(S.d_segs, segs.data(), segs.size() * sizeof(Seg), cudaMemcpyHostToDevice,
                            st),
            "copy segs");
    DCK(grow(S.sendbuf, S.cap_send, (size_t)std::max<int64_t>(off * 6, 1)), "alloc send");
    DCK(grow(S.recvbuf, S.cap_recv, (size_t)std::max<int64_t>(roff * 6, 1)), "alloc recv");
    if (nsend_segs)
        pack_particles_kernel<<<std::min(nsend_segs, 148 * 8), 256, 0, st>>>(
            S.sorted6, S.n_total, S.d_segs, nsend_segs, S.sendbuf);
    // the host segment vector must stay alive until the async copy is done
    DCK(cudaStreamSynchronize(st), "sync segs");
    DCK(cudaGetLastError(), "phase2 kernels");
    S.bytes_sent = off * 24;
    S.bytes_recv = roff * 24;
    return VFMM_OK;
}

vfmm_status dist_phase3(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int p = D.prm.p, nc = ncoef(p);
    const int cellsz = 3 * nc;
    const int64_t nleaf = (int64_t)1 << (3 * L);
    // halo particles into their global positions
    if (S.n_recv_segs)
        unpack_particles_kernel<<<std::min(S.n_recv_segs, 148 * 8), 256, 0, st>>>(
            S.sorted6, S.n_total, S.d_segs + S.n_send_segs, S.n_recv_segs, S.recvbuf);
    (void)nleaf;
    const float a = (float)((double)D.prm.box_len / (double)(1 << L));
    auto Mlev = [&](int l) { return S.Mall + level_offset(l) * cellsz; };
    launch_p2m(S.sorted6, S.n_total, S.gstart, p, 1.f / a, Mlev(L), owned_lo(L, R, r),
               owned_cnt(L, R), st);
    for (int l = L - 1; l >= 1; --l)
        launch_m2m(D.m2m, p, D.KP, D.NR, Mlev(l + 1), Mlev(l), l, owned_lo(l, R, r),
                   owned_cnt(l, R), D.m2m_scratch, D.m2m_scratch_floats, st);
    // ---- pack LET multipoles (levels 2..L) per peer ----
    std::vector<int> cells;
    S.m_send_off.assign(R, 0);
    S.m_send_cnt.assign(R, 0);
    int64_t off = 0;  // floats
    std::vector<std::pair<int, int>> send_runs;  // (level, count) in order, for the pack launch
    for (int q = 0; q < R; ++q) {
        S.m_send_off[q] = off;
        for (int l = 2; l <= L; ++l) {
            const auto& v = S.plan.m_send[l][q];
            for (int cidx : v) cells.push_back(cidx);
            send_runs.push_back({l, (int)v.size()});
            off += (int64_t)v.size() * cellsz;
        }
        S.m_send_cnt[q] = off - S.m_send_off[q];
    }
    const int nsend_cells = (int)cells.size();
    S.m_recv_off.assign(R, 0);
    S.m_recv_cnt.assign(R, 0);
    int64_t roff = 0;
    for (int q = 0; q < R; ++q) {
        S.m_recv_off[q] = roff;
        for (int l = 2; l <= L; ++l) {
            const auto& v = S.plan.m_recv[l][q];
            for (int cidx : v) cells.push_back(cidx);
            roff += (int64_t)v.size() * cellsz;
        }
        S.m_recv_cnt[q] = roff - S.m_recv_off[q];
    }
    S.m_recv_floats = roff;
    S.n_recv_cells_off = nsend_cells;
    S.n_recv_cells = (int)cells.size() - nsend_cells;
    DCK(grow(S.d_cells, S.cap_cells, cells.size()), "alloc cells");
    if (!cells.empty())
        DCK(cudaMemcpyAsync(S.d_cells, cells.data(), cells.size() * sizeof(int),
                            cudaMemcpyHostToDevice, st),
            "copy cells");
    DCK(grow(S.msend, S.cap_msend, (size_t)std::max<int64_t>(off, 1)), "alloc msend");
    DCK(grow(S.mrecv, S.cap_mrecv, (size_t)std::max<int64_t>(roff, 1)), "alloc mrecv");
    int64_t coff = 0, boff = 0;
    for (int q = 0; q < R; ++q)
        for (int l = 2; l <= L; ++l) {
            const int cnt = (int)S.plan.m_send[l][q].size();
            if (cnt)
                pack_cells_kernel<<<grid_of((int64_t)cnt * cellsz), 256, 0, st>>>(
                    Mlev(l), cellsz, S.d_cells + coff, cnt, S.msend + boff);
            coff += cnt;
            boff += (int64_t)cnt * cellsz;
        }
    DCK(cudaStreamSynchronize(st), "sync cells");
    DCK(cudaGetLastError(), "phase3 kernels");
    S.bytes_sent += off * 4;
    S.bytes_recv += roff * 4;
    return VFMM_OK;
}

vfmm_status dist_phase4(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int p = D.prm.p, nc = ncoef(p);
    const int cellsz = 3 * nc;
    const vfmm_params& P = D.prm;
    const int periodic = P.image_levels > 0;
    auto Mlev = [&](int l) { return S.Mall + level_offset(l) * cellsz; };
    auto Llev = [&](int l) { return S.Lall + level_offset(l) * cellsz; };
    // LET multipoles into place
    int64_t coff = S.n_recv_cells_off, boff = 0;
    for (int q = 0; q < R; ++q)
        for (int l = 2; l <= L; ++l) {
            const int cnt = (int)S.plan.m_recv[l][q].size();
            if (cnt)
                unpack_cells_kernel<<<grid_of((int64_t)cnt * cellsz), 256, 0, st>>>(
                    Mlev(l), cellsz, S.d_cells + coff, cnt, S.mrecv + boff);
            coff += cnt;
            boff += (int64_t)cnt * cellsz;
        }
    // root multipole (every rank, from the all-gathered level 1)
    launch_m2m(D.m2m, p, D.KP, D.NR, Mlev(1), Mlev(0), 0, 0, 1, D.m2m_scratch,
               D.m2m_scratch_floats, st);
    // M2L for owned targets (level 1: all 8 cells -- sources are global there)
    for (int l = 1; l <= L; ++l) {
        const int64_t plo = l == 1 ? 0 : owned_lo(l - 1, R, r);
        const int64_t pcnt = l == 1 ? 1 : owned_cnt(l - 1, R);
        // owned box of parents at level l-1 (8/R whole octants)
        const int nP = 1 << (l - 1);
        int box[6] = {0, 0, 0, nP, nP, nP};
        if (l >= 2) {
            const int k = 8 / R;  // octants per rank: 8, 4, 2, 1
            const int o0 = r * k;
            const int half = nP / 2;
            box[0] = (k >= 2 ? 0 : (o0 & 1) * half);
            box[1] = (k >= 4 ? 0 : ((o0 >> 1) & 1) * half);
            box[2] = (k >= 8 ? 0 : ((o0 >> 2) & 1) * half);
            box[3] = k >= 2 ? nP : half;
            box[4] = k >= 4 ? nP : half;
            box[5] = k >= 8 ? nP : half;
        }
        if (D.allow_tc && D.tc.hi && m2l_tc_supported(p, l) && m2l_tc_shape_ok(box)) {
            const size_t need = m2l_tc_grid_floats(l);
            if (need > S.g_cap) {
                dfree(S.g_hi);
                dfree(S.g_lo);
                S.g_cap = 0;
                DCK(cudaMalloc((void**)&S.g_hi, need * 4), "alloc m2l grid");
                DCK(cudaMalloc((void**)&S.g_lo, need * 4), "alloc m2l grid");
                S.g_cap = need;
            }
            if (!S.tcmax) {
                DCK(cudaMalloc((void**)&S.tcmax, 32 * sizeof(uint32_t)), "alloc tc max");
            }
            DCK(cudaMemsetAsync(S.tcmax + l, 0, sizeof(uint32_t), st), "memset tc max");
            if (launch_m2l_tc(D.tc, D.slots, p, Mlev(l), Llev(l), l, periodic, S.g_hi, S.g_lo,
                              S.tcmax + l, box, st) != 0) {
                if (err) *err = "tensor-map encode failed";
                return VFMM_ECUDA;
            }
        } else {
            launch_m2l(D.m2l, D.slots, p, D.KP, D.NR, Mlev(l), Llev(l), l, periodic, plo, pcnt,
                       D.m2m_scratch, D.m2m_scratch_floats, st);
        }
    }
    if (P.image_levels >= 2) launch_periodic(D.per, p, D.KP, D.NR, Mlev(0), Llev(0), st);
    else DCK(cudaMemsetAsync(Llev(0), 0, cellsz * 4, st), "memset L0");
    for (int l = 1; l <= L; ++l) {
        const int64_t plo = l == 1 ? 0 : owned_lo(l - 1, R, r);
        const int64_t pcnt = l == 1 ? 1 : owned_cnt(l - 1, R);
        launch_l2l(D.l2l, p, D.KP, D.NR, Llev(l - 1), Llev(l), l, plo, pcnt, st);
    }
    const KernelConsts kc = make_kernel_consts(P.sigma);
    const float a = (float)((double)P.box_len / (double)(1 << L));
    const bool use_far = P.mode == VFMM_MODE_FMM || P.mode == VFMM_MODE_FAR_ONLY;
    const bool use_near = P.mode == VFMM_MODE_FMM || P.mode == VFMM_MODE_NEAR_ONLY;
    DCK(cudaMemsetAsync(S.d_pairs, 0, sizeof(unsigned long long), st), "memset pairs");
    if (use_near)
        launch_p2p(S.sorted6, S.n_total, S.gstart, L, a, periodic, P.scheme, kc, S.near6, S.d_pairs,
                   owned_lo(L - 1, R, r), owned_cnt(L - 1, R), st);
    if (S.n_local > 0)
        launch_l2p_combine(D.l2p, S.sorted6, S.near6, S.perm, S.n_total, S.gstart, p, a, Llev(L), P.scheme,
                           use_near, use_far, S.vel, S.dg, owned_lo(L, R, r), owned_cnt(L, R),
                           S.gbase, S.n_local, st);
    DCK(cudaGetLastError(), "phase4 kernels");
    return VFMM_OK;
}

// ---------------------------------------------------------------------------------------
// exchanges: logical ranks (device copies within one process)
// ---------------------------------------------------------------------------------------
vfmm_status logical_x1(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st) {
    const int R = D.R;
    const int64_t per = ((int64_t)1 << (3 * D.depth)) / R;
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < R; ++q)
            if (cudaMemcpyAsync(S[r]->counts_all + q * per, S[q]->counts_own, per * 4,
                                cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return VFMM_ECUDA;
    return VFMM_OK;
}
vfmm_status logical_x2(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st) {
    const int R = D.R;
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < R; ++q) {
            if (q == r) continue;
            const int64_t c = S[r]->p_recv_cnt[q];
            if (c != S[q]->p_send_cnt[r]) return VFMM_ESTATE;  // plans must agree
            if (c && cudaMemcpyAsync(S[r]->recvbuf + S[r]->p_recv_off[q] * 6,
                                     S[q]->sendbuf + S[q]->p_send_off[r] * 6, c * 24,
                                     cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return VFMM_ECUDA;
        }
    return VFMM_OK;
}
vfmm_status logical_x3(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st) {
    const int R = D.R;
    const int cellsz = 3 * ncoef(D.prm.p);
    const int64_t per1 = 8 / R;
    // all-gather of level-1 multipoles (level-1 cells start at offset 1 in the level arrays)
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < R; ++q) {
            if (q == r) continue;
            const int64_t o = (level_offset(1) + q * per1) * cellsz;
            if (cudaMemcpyAsync(S[r]->Mall + o, S[q]->Mall + o, per1 * cellsz * 4,
                                cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return VFMM_ECUDA;
        }
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < R; ++q) {
            if (q == r) continue;
            const int64_t c = S[r]->m_recv_cnt[q];
            if (c != S[q]->m_send_cnt[r]) return VFMM_ESTATE;
            if (c && cudaMemcpyAsync(S[r]->mrecv + S[r]->m_recv_off[q],
                                     S[q]->msend + S[q]->m_send_off[r], c * 4,
                                     cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return VFMM_ECUDA;
        }
    return VFMM_OK;
}

// ---------------------------------------------------------------------------------------
// exchanges: NCCL (grouped point-to-point + all-gather on the compute stream)
// ---------------------------------------------------------------------------------------
bool nccl_available() { return g_nccl.load(); }

vfmm_status nccl_unique_id(void* out128) {
    if (!g_nccl.load()) return VFMM_ENCCL;
    ncclUniqueId id;
    if (g_nccl.GetUniqueId(&id) != ncclSuccess) return VFMM_ENCCL;
    memcpy(out128, &id, sizeof(id));
    return VFMM_OK;
}
vfmm_status nccl_init(void** comm, int nranks, int rank, const void* id128) {
    if (!g_nccl.load()) return VFMM_ENCCL;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    if (g_nccl.CommInitRank(&c, nranks, id, rank) != ncclSuccess) return VFMM_ENCCL;
    *comm = (void*)c;
    return VFMM_OK;
}
void nccl_destroy(void* comm) {
    if (comm && g_nccl.h) g_nccl.CommDestroy((ncclComm_t)comm);
}
vfmm_status nccl_x1(RankState& S, const DistShared& D, void* comm, cudaStream_t st) {
    const int64_t per = ((int64_t)1 << (3 * D.depth)) / D.R;
    if (g_nccl.AllGather(S.counts_own, S.counts_all, per, ncclInt32, (ncclComm_t)comm, st) !=
        ncclSuccess)
        return VFMM_ENCCL;
    return VFMM_OK;
}
vfmm_status nccl_x2(RankState& S, const DistShared& D, void* comm, cudaStream_t st) {
    const int R = D.R;
    if (g_nccl.GroupStart() != ncclSuccess) return VFMM_ENCCL;
    for (int q = 0; q < R; ++q) {
        if (q == S.rank) continue;
        if (S.p_send_cnt[q])
            g_nccl.Send(S.sendbuf + S.p_send_off[q] * 6, S.p_send_cnt[q] * 6, ncclFloat32, q,
                        (ncclComm_t)comm, st);
        if (S.p_recv_cnt[q])
            g_nccl.Recv(S.recvbuf + S.p_recv_off[q] * 6, S.p_recv_cnt[q] * 6, ncclFloat32, q,
                        (ncclComm_t)comm, st);
    }
    if (g_nccl.GroupEnd() != ncclSuccess) return VFMM_ENCCL;
    return VFMM_OK;
}
vfmm_status nccl_x3(RankState& S, const DistShared& D, void* comm, cudaStream_t st) {
    const int R = D.R;
    const int cellsz = 3 * ncoef(D.prm.p);
    const int64_t per1 = 8 / R;
    float* l1 = S.Mall + level_offset(1) * cellsz;
    if (g_nccl.GroupStart() != ncclSuccess) return VFMM_ENCCL;
    g_nccl.AllGather(l1 + S.rank * per1 * cellsz, l1, per1 * cellsz, ncclFloat32,
                     (ncclComm_t)comm, st);  // in place
    for (int q = 0; q < R; ++q) {
        if (q == S.rank) continue;
        if (S.m_send_cnt[q])
            g_nccl.Send(S.msend + S.m_send_off[q], S.m_send_cnt[q], ncclFloat32, q,
                        (ncclComm_t)comm, st);
        if (S.m_recv_cnt[q])
            g_nccl.Recv(S.mrecv + S.m_recv_off[q], S.m_recv_cnt[q], ncclFloat32, q,
                        (ncclComm_t)comm, st);
    }
    if (g_nccl.GroupEnd() != ncclSuccess) return VFMM_ENCCL;
    return VFMM_OK;
}

}  // namespace vfmm
