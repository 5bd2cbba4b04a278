// dist.cu -- multi-GPU FMM: Morton-range spatial decomposition with a local-essential-tree
// (LET) exchange (SURVEY.md section 8(e); the paper's scaling runs, PAPER.md:41, :366-367,
// used MPI across 4096 GPUs -- here NCCL over NVLink/NVSwitch, one process per GPU).
//
// Rank r of R (R in {1, 2, 4, 8}) owns the contiguous Morton range of leaves
// [r 8^L/R, (r+1) 8^L/R), i.e. 8/R whole octants; at every level >= 1 its cells form a box.
// Each rank passes any particles (anywhere in the box).  One evaluation:
//   0  C1: Morton keys + stable sort of the caller's particles, cut at the rank boundaries;
//      X0 counts matrix all-gather (one D2H copy: message sizes) and the particles to their
//      owners (grouped send/recv); the owner evaluates them in received order
//   1  keys + stable sort of the owned particles (ties: sender rank, then the sender's input
//      order = the global input order of the concatenated per-rank inputs)
//   X1 all-gather of owned leaf counts -> compact leaf_start over the rank's owned + halo
//      leaves (+ one D2H copy so the host knows halo message sizes)
//   2  owned particles -> their compact sorted positions; pack halo leaves for the peers
//   X2 halo particle exchange (leaves within one leaf of a peer's range, periodic)
//   3  P2M, M2M over owned cells (levels L-1 .. 1); pack halo multipoles
//   X3 all-gather of level-1 multipoles + LET multipole exchange for levels 2..L (cells in a
//      peer's 189-cell interaction lists)
//   4  root M2M, periodic images and L2L redundantly on every rank; M2L, L2L for owned cells
//      (after X3), P2P (after X2), L2P
//   5  results back to their senders (reverse trip of X0) and to the caller's input order.
// The exchange plans are static for (L, R, periodic) and built once on the host; the static
// device tables (halo leaf mask, LET cell lists) are uploaded once per plan.
// Transport: NCCL (grouped ncclSend/ncclRecv and ncclAllGather on a communication stream,
// X2 overlapping P2M / M2M / M2L and X3 overlapping the M2L-independent work; library loaded
// with dlopen -- the same libnccl.so.2 torch uses), or "logical ranks": all R ranks' phases run
// on one GPU in lockstep and exchanges are device-to-device copies (tests).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
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
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
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
        CommGetAsyncError = (decltype(CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        return GetUniqueId && CommInitRank && CommDestroy && GroupStart && GroupEnd && Send &&
               Recv && AllGather;
    }
};
NcclApi g_nccl;

// ---- kernels -------------------------------------------------------------------------

// exclusive scan of counts[0..m) (times need[i] if given) -> start[0..m]; one block (small m,
// once per evaluation)
__global__ void scan_counts_kernel(const int* __restrict__ counts, const uint8_t* __restrict__ need,
                                   int64_t m, int* __restrict__ start) {
    __shared__ int wsum[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t b = 0; b < m; b += blockDim.x) {
        const int64_t i = b + threadIdx.x;
        const int v = i < m ? (need && !need[i] ? 0 : counts[i]) : 0;
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

// C1: particles per destination rank from the sorted keys (lower bounds of the rank
// boundaries); one thread per rank
__global__ void dest_counts_kernel(const uint32_t* __restrict__ keys, int64_t n, int R,
                                   int64_t nleaf, int* __restrict__ crow) {
    const int q = threadIdx.x;
    if (q >= R) return;
    auto lb = [&](int64_t c) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)keys[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    const int64_t a = lb(nleaf / R * q), b = q == R - 1 ? n : lb(nleaf / R * (q + 1));
    crow[q] = (int)(b - a);
}
// AoS6 [k] = (a[perm[k]], b[perm[k]]) for SoA3 a, b of length n (perm null: identity)
__global__ void pack_aos6_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                 int64_t n, const uint32_t* __restrict__ perm,
                                 float* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = perm ? (int64_t)perm[k] : k;
        float* o = out + k * 6;
        o[0] = a[i];
        o[1] = a[n + i];
        o[2] = a[2 * n + i];
        o[3] = b[i];
        o[4] = b[n + i];
        o[5] = b[2 * n + i];
    }
}
// SoA3 a[perm[k]], b[perm[k]] = AoS6 [k] (perm null: identity)
__global__ void unpack_aos6_kernel(const float* __restrict__ in, int64_t n,
                                   const uint32_t* __restrict__ perm, float* __restrict__ a,
                                   float* __restrict__ b) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = perm ? (int64_t)perm[k] : k;
        const float* v = in + k * 6;
        a[i] = v[0];
        a[n + i] = v[1];
        a[2 * n + i] = v[2];
        b[i] = v[3];
        b[n + i] = v[4];
        b[2 * n + i] = v[5];
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
        dfree(ikeys[b]);
        dfree(ivals[b]);
    }
    dfree(radix_tmp);
    dfree(itmp);
    dfree(isend);
    dfree(irecv);
    dfree(own);
    dfree(d_crow);
    dfree(d_cmat);
    dfree(lstart);
    dfree(counts_own);
    dfree(counts_all);
    dfree(gstart);
    dfree(d_need);
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
    cap_in = cap_own = cap_local = cap_total = 0;
    cap_send = cap_recv = 0;
    cap_segs = cap_cells = 0;
    g_cap = 0;
    cap_depth = cap_p = cap_R = -1;
    plan_dirty = true;
}

int64_t host_leaf_of(float x, float y, float z, int depth, float lo, float len, bool* inside) {
    const int side = 1 << depth;
    const float inv = (float)((double)side / (double)len);
    const float hi = lo + len;
    const float v[3] = {x, y, z};
    int64_t key = 0;
    bool in = true;
    for (int a = 0; a < 3; ++a) {
        if (!(v[a] >= lo && v[a] < hi)) in = false;
        volatile float d = v[a] - lo;  // single RN subtract, single RN multiply
        volatile float s = d * inv;
        const float fl = std::floor((float)s);
        int q = fl >= 0.f ? (int)fl : 0;
        if (q > side - 1) q = side - 1;
        for (int b = 0; b < depth; ++b) key |= (int64_t)((q >> b) & 1) << (3 * b + a);
    }
    if (inside) *inside = in;
    return key;
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
template <class T>
cudaError_t grow64(T*& p, int64_t& cap, int64_t need, size_t per) {
    if (need <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc((void**)&p, (size_t)std::max<int64_t>(need, 1) * per * sizeof(T));
    if (e == cudaSuccess) cap = need;
    return e;
}

int grid_of(int64_t work, int bs = 256) {
    int64_t g = (work + bs - 1) / bs;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

int64_t owned_lo(int l, int R, int r) { return ((int64_t)r << (3 * l)) / R; }
int64_t owned_cnt(int l, int R) { return ((int64_t)1 << (3 * l)) / R; }

Geom geom_of(const DistShared& D) {
    const vfmm_params& P = D.prm;
    return Geom{P.box_lo, P.box_len, (double)P.box_lo, (double)P.box_len, D.depth,
                P.image_levels > 0};
}

}  // namespace

// ---- 0: C1 redistribution of the caller's particles ------------------------------------

vfmm_status dist_phase0a(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R;
    const int64_t n = S.n_in;
    if (n > S.cap_in) {
        for (int b = 0; b < 2; ++b) {
            dfree(S.ikeys[b]);
            dfree(S.ivals[b]);
        }
        dfree(S.itmp);
        dfree(S.isend);
        S.cap_in = 0;
        for (int b = 0; b < 2; ++b) {
            DCK(cudaMalloc((void**)&S.ikeys[b], n * 4), "alloc keys");
            DCK(cudaMalloc((void**)&S.ivals[b], n * 4), "alloc vals");
        }
        DCK(cudaMalloc(&S.itmp, radix_temp_bytes(n)), "alloc radix");
        DCK(cudaMalloc((void**)&S.isend, 6 * n * sizeof(float)), "alloc c1 send");
        S.cap_in = n;
    }
    if (!S.d_err) {
        DCK(cudaMalloc((void**)&S.d_err, sizeof(int)), "alloc err");
        DCK(cudaMemset(S.d_err, 0, sizeof(int)), "memset err");
        DCK(cudaMalloc((void**)&S.d_pairs, sizeof(unsigned long long)), "alloc pairs");
    }
    if (S.cap_R != R) {
        dfree(S.d_crow);
        dfree(S.d_cmat);
        DCK(cudaMalloc((void**)&S.d_crow, R * sizeof(int)), "alloc counts");
        DCK(cudaMalloc((void**)&S.d_cmat, R * R * sizeof(int)), "alloc counts");
        S.cap_R = R;
    }
    const int64_t nleaf = (int64_t)1 << (3 * L);
    if (n > 0) {
        int nl = 0;
        launch_keys(S.in_pos, n, geom_of(D), S.ikeys[0], S.ivals[0], S.d_err, st);
        launch_radix_sort(S.ikeys[0], S.ivals[0], S.ikeys[1], S.ivals[1], n, 3 * L, S.itmp, st,
                          &S.ikeys_sorted, &S.iperm, &nl);
        dest_counts_kernel<<<1, 32, 0, st>>>(S.ikeys_sorted, n, R, nleaf, S.d_crow);
    } else {
        DCK(cudaMemsetAsync(S.d_crow, 0, R * sizeof(int), st), "memset counts");
    }
    DCK(cudaGetLastError(), "phase0a kernels");
    return VFMM_OK;
}

vfmm_status dist_phase0b(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int R = D.R, r = S.rank;
    S.h_cmat.resize((size_t)R * R);
    DCK(cudaMemcpyAsync(S.h_cmat.data(), S.d_cmat, R * R * sizeof(int), cudaMemcpyDeviceToHost,
                        st),
        "copy counts");
    DCK(cudaStreamSynchronize(st), "sync counts");  // host sync 1 of 2: C1 message sizes
    S.c1_send_off.assign(R, 0);
    S.c1_send_cnt.assign(R, 0);
    S.c1_recv_off.assign(R, 0);
    S.c1_recv_cnt.assign(R, 0);
    int64_t so = 0, ro = 0;
    for (int q = 0; q < R; ++q) {
        S.c1_send_off[q] = so;
        S.c1_send_cnt[q] = S.h_cmat[(size_t)r * R + q];
        so += S.c1_send_cnt[q];
        S.c1_recv_off[q] = ro;
        S.c1_recv_cnt[q] = S.h_cmat[(size_t)q * R + r];
        ro += S.c1_recv_cnt[q];
    }
    if (so != S.n_in) {
        if (err) *err = "C1 counts do not add up to the rank's particles";
        return VFMM_ESTATE;
    }
    S.n_own = ro;
    if (S.n_own > S.cap_own) {
        dfree(S.irecv);
        dfree(S.own);
        S.cap_own = 0;
        DCK(cudaMalloc((void**)&S.irecv, 6 * S.n_own * sizeof(float)), "alloc c1 recv");
        DCK(cudaMalloc((void**)&S.own, 12 * S.n_own * sizeof(float)), "alloc owned");
        S.cap_own = S.n_own;
    }
    if (S.n_in > 0)
        pack_aos6_kernel<<<grid_of(S.n_in), 256, 0, st>>>(S.in_pos, S.in_gam, S.n_in, S.iperm,
                                                          S.isend);
    DCK(cudaGetLastError(), "phase0b kernels");
    S.bytes_sent = (so - S.c1_send_cnt[r]) * 24;
    S.bytes_recv = (ro - S.c1_recv_cnt[r]) * 24;
    return VFMM_OK;
}

vfmm_status dist_phase0c(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    (void)D;
    const int64_t m = S.n_own;
    if (m > 0)
        unpack_aos6_kernel<<<grid_of(m), 256, 0, st>>>(S.irecv, m, nullptr, S.own, S.own + 3 * m);
    DCK(cudaGetLastError(), "phase0c kernels");
    S.n_local = m;
    S.pos = S.own;
    S.gam = S.own + 3 * m;
    S.vel = S.own + 6 * m;
    S.dg = S.own + 9 * m;
    return VFMM_OK;
}

// ---- 1-4: the FMM on the owned particles ----------------------------------------------

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
            DCK(cudaMalloc((void**)&S.keys[b], n * 4), "alloc keys");
            DCK(cudaMalloc((void**)&S.vals[b], n * 4), "alloc vals");
        }
        DCK(cudaMalloc(&S.radix_tmp, radix_temp_bytes(n)), "alloc radix");
        S.cap_local = n;
    }
    if (S.cap_depth != L) {
        dfree(S.lstart);
        dfree(S.counts_own);
        dfree(S.counts_all);
        dfree(S.gstart);
        dfree(S.d_need);
        DCK(cudaMalloc((void**)&S.lstart, (nleaf + 1) * 4), "alloc lstart");
        // sized for R = 1 (the largest owned range): R may change between calls at one depth
        DCK(cudaMalloc((void**)&S.counts_own, nleaf * 4), "alloc counts");
        DCK(cudaMalloc((void**)&S.counts_all, nleaf * 4), "alloc counts");
        DCK(cudaMalloc((void**)&S.gstart, (nleaf + 1) * 4), "alloc gstart");
        DCK(cudaMalloc((void**)&S.d_need, nleaf), "alloc need mask");
        S.plan_dirty = true;
    }
    int nl = 0;
    if (n > 0) {
        launch_keys(S.pos, n, geom_of(D), S.keys[0], S.vals[0], S.d_err, st);
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

// static device tables of the plan: the need mask (owned + halo leaves) and the LET cell lists
static vfmm_status upload_plan(RankState& S, const DistShared& D, cudaStream_t st,
                               std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int64_t nleaf = (int64_t)1 << (3 * L);
    std::vector<uint8_t> need(nleaf, 0);
    for (int64_t c = owned_lo(L, R, r); c < owned_lo(L, R, r) + owned_cnt(L, R); ++c) need[c] = 1;
    for (int q = 0; q < R; ++q)
        for (int leaf : S.plan.p_recv[q]) need[leaf] = 1;
    std::vector<int> cells;
    for (int q = 0; q < R; ++q)
        for (int l = 2; l <= L; ++l)
            for (int cidx : S.plan.m_send[l][q]) cells.push_back(cidx);
    const int nsend_cells = (int)cells.size();
    for (int q = 0; q < R; ++q)
        for (int l = 2; l <= L; ++l)
            for (int cidx : S.plan.m_recv[l][q]) cells.push_back(cidx);
    S.n_recv_cells_off = nsend_cells;
    S.n_recv_cells = (int)cells.size() - nsend_cells;
    DCK(grow(S.d_cells, S.cap_cells, cells.size()), "alloc cells");
    // synchronous uploads (once per plan): the host vectors die at return
    DCK(cudaStreamSynchronize(st), "sync before plan upload");
    DCK(cudaMemcpy(S.d_need, need.data(), nleaf, cudaMemcpyHostToDevice), "upload need mask");
    if (!cells.empty())
        DCK(cudaMemcpy(S.d_cells, cells.data(), cells.size() * sizeof(int), cudaMemcpyHostToDevice),
            "upload cells");
    S.plan_dirty = false;
    return VFMM_OK;
}

vfmm_status dist_phase2(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int64_t nleaf = (int64_t)1 << (3 * L);
    if (S.plan_dirty) {
        vfmm_status s = upload_plan(S, D, st, err);
        if (s != VFMM_OK) return s;
    }
    scan_counts_kernel<<<1, 1024, 0, st>>>(S.counts_all, S.d_need, nleaf, S.gstart);
    S.hstart.resize(nleaf + 1);
    DCK(cudaMemcpyAsync(S.hstart.data(), S.gstart, (nleaf + 1) * 4, cudaMemcpyDeviceToHost, st),
        "copy gstart");
    DCK(cudaStreamSynchronize(st), "sync gstart");  // host sync 2 of 2: halo message sizes
    S.n_total = S.hstart[nleaf];
    S.gbase = S.hstart[owned_lo(L, R, r)];
    const int nc = ncoef(D.prm.p);
    if (S.n_total > S.cap_total) {
        dfree(S.sorted6);
        dfree(S.near6);
        S.cap_total = 0;
        const int64_t nt = std::max<int64_t>(S.n_total, 1);
        DCK(cudaMalloc((void**)&S.sorted6, 6 * nt * 4), "alloc sorted6");
        DCK(cudaMalloc((void**)&S.near6, 6 * nt * 4), "alloc near6");
        S.cap_total = S.n_total;
    }
    if (S.cap_depth != L || S.cap_p != D.prm.p) {
        dfree(S.Mall);
        dfree(S.Lall);
        const int64_t cells = level_offset(L + 1);
        DCK(cudaMalloc((void**)&S.Mall, cells * 3 * nc * 4), "alloc M");
        DCK(cudaMalloc((void**)&S.Lall, cells * 3 * nc * 4), "alloc L");
        DCK(cudaMemset(S.Mall, 0, cells * 3 * nc * 4), "memset M");
        S.cap_depth = L;
        S.cap_p = D.prm.p;
    }
    if (S.n_local > 0)
        launch_gather(S.pos, S.gam, S.perm, S.keys_sorted, S.n_local, geom_of(D), S.sorted6,
                      S.n_total, S.gbase, st);
    // ---- pack halo particles for every peer (segments in compact sorted order) ----
    S.h_segs.clear();
    S.p_send_off.assign(R, 0);
    S.p_send_cnt.assign(R, 0);
    int64_t off = 0;
    for (int q = 0; q < R; ++q) {
        S.p_send_off[q] = off;
        for (int leaf : S.plan.p_send[q]) {
            const int64_t c = S.hstart[leaf + 1] - S.hstart[leaf];
            if (c) S.h_segs.push_back({S.hstart[leaf], c, off});
            off += c;
        }
        S.p_send_cnt[q] = off - S.p_send_off[q];
    }
    const int nsend_segs = (int)S.h_segs.size();
    S.n_send_segs = nsend_segs;
    S.p_recv_off.assign(R, 0);
    S.p_recv_cnt.assign(R, 0);
    int64_t roff = 0;
    for (int q = 0; q < R; ++q) {
        S.p_recv_off[q] = roff;
        for (int leaf : S.plan.p_recv[q]) {
            const int64_t c = S.hstart[leaf + 1] - S.hstart[leaf];
            if (c) S.h_segs.push_back({S.hstart[leaf], c, roff});
            roff += c;
        }
        S.p_recv_cnt[q] = roff - S.p_recv_off[q];
    }
    S.p_recv_total = roff;
    S.n_recv_segs = (int)S.h_segs.size() - nsend_segs;
    DCK(grow(S.d_segs, S.cap_segs, S.h_segs.size()), "alloc segs");
    // pageable upload: staged before the call returns, and h_segs outlives it anyway
    if (!S.h_segs.empty())
        DCK(cudaMemcpyAsync(S.d_segs, S.h_segs.data(), S.h_segs.size() * sizeof(Seg),
                            cudaMemcpyHostToDevice, st),
            "copy segs");
    DCK(grow(S.sendbuf, S.cap_send, (size_t)std::max<int64_t>(off * 6, 1)), "alloc send");
    DCK(grow(S.recvbuf, S.cap_recv, (size_t)std::max<int64_t>(roff * 6, 1)), "alloc recv");
    if (nsend_segs)
        pack_particles_kernel<<<std::min(nsend_segs, 148 * 8), 256, 0, st>>>(
            S.sorted6, S.n_total, S.d_segs, nsend_segs, S.sendbuf);
    DCK(cudaGetLastError(), "phase2 kernels");
    S.bytes_sent += off * 24;
    S.bytes_recv += roff * 24;
    return VFMM_OK;
}

vfmm_status dist_unpack_halo(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    (void)D;
    if (S.n_recv_segs)
        unpack_particles_kernel<<<std::min(S.n_recv_segs, 148 * 8), 256, 0, st>>>(
            S.sorted6, S.n_total, S.d_segs + S.n_send_segs, S.n_recv_segs, S.recvbuf);
    DCK(cudaGetLastError(), "halo unpack");
    return VFMM_OK;
}

vfmm_status dist_phase3(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int p = D.prm.p, nc = ncoef(p);
    const int cellsz = 3 * nc;
    const float a = (float)((double)D.prm.box_len / (double)(1 << L));
    auto Mlev = [&](int l) { return S.Mall + level_offset(l) * cellsz; };
    launch_p2m(S.sorted6, S.n_total, S.gstart, p, 1.f / a, Mlev(L), owned_lo(L, R, r),
               owned_cnt(L, R), st);
    for (int l = L - 1; l >= 1; --l)
        launch_m2m(D.m2m, p, D.KP, D.NR, Mlev(l + 1), Mlev(l), l, owned_lo(l, R, r),
                   owned_cnt(l, R), D.m2m_scratch, D.m2m_scratch_floats, st);
    // ---- pack LET multipoles (levels 2..L) per peer (cell lists uploaded with the plan) ----
    S.m_send_off.assign(R, 0);
    S.m_send_cnt.assign(R, 0);
    int64_t off = 0;  // floats
    for (int q = 0; q < R; ++q) {
        S.m_send_off[q] = off;
        for (int l = 2; l <= L; ++l) off += (int64_t)S.plan.m_send[l][q].size() * cellsz;
        S.m_send_cnt[q] = off - S.m_send_off[q];
    }
    S.m_recv_off.assign(R, 0);
    S.m_recv_cnt.assign(R, 0);
    int64_t roff = 0;
    for (int q = 0; q < R; ++q) {
        S.m_recv_off[q] = roff;
        for (int l = 2; l <= L; ++l) roff += (int64_t)S.plan.m_recv[l][q].size() * cellsz;
        S.m_recv_cnt[q] = roff - S.m_recv_off[q];
    }
    S.m_recv_floats = roff;
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
    DCK(cudaGetLastError(), "phase3 kernels");
    S.bytes_sent += off * 4;
    S.bytes_recv += roff * 4;
    return VFMM_OK;
}

vfmm_status dist_unpack_let(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R;
    const int cellsz = 3 * ncoef(D.prm.p);
    auto Mlev = [&](int l) { return S.Mall + level_offset(l) * cellsz; };
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
    DCK(cudaGetLastError(), "LET unpack");
    return VFMM_OK;
}

vfmm_status dist_phase4_far(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int p = D.prm.p, nc = ncoef(p);
    const int cellsz = 3 * nc;
    const vfmm_params& P = D.prm;
    const int periodic = P.image_levels > 0;
    auto Mlev = [&](int l) { return S.Mall + level_offset(l) * cellsz; };
    auto Llev = [&](int l) { return S.Lall + level_offset(l) * cellsz; };
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
        if (D.allow_tc && D.tc.hi && m2l_tc_supported(p, l) && m2l_tc_shape_ok(box, p)) {
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
    DCK(cudaGetLastError(), "phase4 far kernels");
    return VFMM_OK;
}

vfmm_status dist_phase4_near(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    const int L = D.depth, R = D.R, r = S.rank;
    const int p = D.prm.p;
    const vfmm_params& P = D.prm;
    const int periodic = P.image_levels > 0;
    const KernelConsts kc = make_kernel_consts(P.sigma);
    const float a = (float)((double)P.box_len / (double)(1 << L));
    const bool use_far = P.mode == VFMM_MODE_FMM || P.mode == VFMM_MODE_FAR_ONLY;
    const bool use_near = P.mode == VFMM_MODE_FMM || P.mode == VFMM_MODE_NEAR_ONLY;
    const int cellsz = 3 * ncoef(p);
    DCK(cudaMemsetAsync(S.d_pairs, 0, sizeof(unsigned long long), st), "memset pairs");
    if (use_near)
        launch_p2p(S.sorted6, S.n_total, S.gstart, L, a, periodic, P.scheme, kc, S.near6, S.d_pairs,
                   owned_lo(L - 1, R, r), owned_cnt(L - 1, R), st);
    if (S.n_local > 0)
        launch_l2p_combine(D.l2p, S.sorted6, S.near6, S.perm, S.n_total, S.gstart, p, a,
                           S.Lall + level_offset(L) * cellsz, P.scheme, use_near, use_far, S.vel,
                           S.dg, owned_lo(L, R, r), owned_cnt(L, R), S.gbase, S.n_local, st);
    DCK(cudaGetLastError(), "phase4 near kernels");
    return VFMM_OK;
}

// ---- 5: results back to the caller ----------------------------------------------------

vfmm_status dist_phase5a(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    (void)D;
    const int64_t m = S.n_own;  // results in received order -> AoS for the return trip
    if (m > 0)
        pack_aos6_kernel<<<grid_of(m), 256, 0, st>>>(S.vel, S.dg, m, nullptr, S.irecv);
    DCK(cudaGetLastError(), "phase5a kernels");
    return VFMM_OK;
}

vfmm_status dist_phase5b(RankState& S, const DistShared& D, cudaStream_t st, std::string* err) {
    (void)D;
    const int64_t n = S.n_in;  // isend now holds the results in local Morton order
    if (n > 0)
        unpack_aos6_kernel<<<grid_of(n), 256, 0, st>>>(S.isend, n, S.iperm, S.in_vel, S.in_dg);
    DCK(cudaGetLastError(), "phase5b kernels");
    S.bytes_sent += (S.n_own - S.c1_recv_cnt[S.rank]) * 24;
    S.bytes_recv += (S.n_in - S.c1_send_cnt[S.rank]) * 24;
    return VFMM_OK;
}

// ---------------------------------------------------------------------------------------
// exchanges: logical ranks (device copies within one process)
// ---------------------------------------------------------------------------------------
vfmm_status logical_x0a(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st) {
    const int R = D.R;
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < R; ++q)
            if (cudaMemcpyAsync(S[r]->d_cmat + q * R, S[q]->d_crow, R * sizeof(int),
                                cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return VFMM_ECUDA;
    return VFMM_OK;
}
vfmm_status logical_x0b(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st) {
    const int R = D.R;
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < R; ++q) {  // q sends its run for r
            const int64_t c = S[r]->c1_recv_cnt[q];
            if (c != S[q]->c1_send_cnt[r]) return VFMM_ESTATE;
            if (c && cudaMemcpyAsync(S[r]->irecv + S[r]->c1_recv_off[q] * 6,
                                     S[q]->isend + S[q]->c1_send_off[r] * 6, c * 24,
                                     cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return VFMM_ECUDA;
        }
    return VFMM_OK;
}
vfmm_status logical_x5(std::vector<RankState*>& S, const DistShared& D, cudaStream_t st) {
    const int R = D.R;
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < R; ++q) {  // r returns q's results
            const int64_t c = S[r]->c1_recv_cnt[q];
            if (c && cudaMemcpyAsync(S[q]->isend + S[q]->c1_send_off[r] * 6,
                                     S[r]->irecv + S[r]->c1_recv_off[q] * 6, c * 24,
                                     cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return VFMM_ECUDA;
        }
    return VFMM_OK;
}
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
// exchanges: NCCL (grouped point-to-point + all-gather on the given stream)
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
vfmm_status nccl_async_error(void* comm, std::string* err) {
    if (!comm || !g_nccl.CommGetAsyncError) return VFMM_OK;
    ncclResult_t a = ncclSuccess;
    if (g_nccl.CommGetAsyncError((ncclComm_t)comm, &a) != ncclSuccess || a != ncclSuccess) {
        if (err)
            *err = std::string("NCCL asynchronous error: ") +
                   (g_nccl.GetErrorString ? g_nccl.GetErrorString(a) : "unknown");
        return VFMM_ENCCL;
    }
    return VFMM_OK;
}
void nccl_destroy(void* comm) {
    if (comm && g_nccl.h) g_nccl.CommDestroy((ncclComm_t)comm);
}

namespace {
// grouped point-to-point exchange: send[q] / recv[q] = (pointer, floats); every return code
// is checked, and the group is always closed
vfmm_status nccl_p2p_group(int R, int self, const std::vector<std::pair<const float*, int64_t>>& snd,
                           const std::vector<std::pair<float*, int64_t>>& rcv, ncclComm_t comm,
                           cudaStream_t st, const float* ag_send = nullptr, float* ag_recv = nullptr,
                           int64_t ag_count = 0) {
    if (g_nccl.GroupStart() != ncclSuccess) return VFMM_ENCCL;
    ncclResult_t r = ncclSuccess;
    if (ag_recv && r == ncclSuccess)
        r = g_nccl.AllGather(ag_send, ag_recv, (size_t)ag_count, ncclFloat32, comm, st);
    for (int q = 0; q < R && r == ncclSuccess; ++q) {
        if (q == self) continue;
        if (snd[q].second && r == ncclSuccess)
            r = g_nccl.Send(snd[q].first, (size_t)snd[q].second, ncclFloat32, q, comm, st);
        if (rcv[q].second && r == ncclSuccess)
            r = g_nccl.Recv(rcv[q].first, (size_t)rcv[q].second, ncclFloat32, q, comm, st);
    }
    const ncclResult_t e = g_nccl.GroupEnd();
    return (r == ncclSuccess && e == ncclSuccess) ? VFMM_OK : VFMM_ENCCL;
}
}  // namespace

vfmm_status nccl_x0a(RankState& S, const DistShared& D, void* comm, cudaStream_t st) {
    if (g_nccl.AllGather(S.d_crow, S.d_cmat, (size_t)D.R, ncclInt32, (ncclComm_t)comm, st) !=
        ncclSuccess)
        return VFMM_ENCCL;
    return VFMM_OK;
}
vfmm_status nccl_x0b(RankState& S, const DistShared& D, void* comm, cudaStream_t st) {
    const int R = D.R, r = S.rank;
    std::vector<std::pair<const float*, int64_t>> snd(R);
    std::vector<std::pair<float*, int64_t>> rcv(R);
    for (int q = 0; q < R; ++q) {
        snd[q] = {S.isend + S.c1_send_off[q] * 6, S.c1_send_cnt[q] * 6};
        rcv[q] = {S.irecv + S.c1_recv_off[q] * 6, S.c1_recv_cnt[q] * 6};
    }
    // the rank's own run stays local
    if (S.c1_send_cnt[r] &&
        cudaMemcpyAsync(rcv[r].first, snd[r].first, S.c1_send_cnt[r] * 24,
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return VFMM_ECUDA;
    return nccl_p2p_group(R, r, snd, rcv, (ncclComm_t)comm, st);
}
vfmm_status nccl_x5(RankState& S, const DistShared& D, void* comm, cudaStream_t st) {
    const int R = D.R, r = S.rank;
    std::vector<std::pair<const float*, int64_t>> snd(R);
    std::vector<std::pair<float*, int64_t>> rcv(R);
    for (int q = 0; q < R; ++q) {  // reverse of X0b
        snd[q] = {S.irecv + S.c1_recv_off[q] * 6, S.c1_recv_cnt[q] * 6};
        rcv[q] = {S.isend + S.c1_send_off[q] * 6, S.c1_send_cnt[q] * 6};
    }
    if (S.c1_send_cnt[r] &&
        cudaMemcpyAsync(rcv[r].first, snd[r].first, S.c1_send_cnt[r] * 24,
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return VFMM_ECUDA;
    return nccl_p2p_group(R, r, snd, rcv, (ncclComm_t)comm, st);
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
    std::vector<std::pair<const float*, int64_t>> snd(R);
    std::vector<std::pair<float*, int64_t>> rcv(R);
    for (int q = 0; q < R; ++q) {
        snd[q] = {S.sendbuf + S.p_send_off[q] * 6, S.p_send_cnt[q] * 6};
        rcv[q] = {S.recvbuf + S.p_recv_off[q] * 6, S.p_recv_cnt[q] * 6};
    }
    return nccl_p2p_group(R, S.rank, snd, rcv, (ncclComm_t)comm, st);
}
vfmm_status nccl_x3(RankState& S, const DistShared& D, void* comm, cudaStream_t st) {
    const int R = D.R;
    const int cellsz = 3 * ncoef(D.prm.p);
    const int64_t per1 = 8 / R;
    float* l1 = S.Mall + level_offset(1) * cellsz;
    std::vector<std::pair<const float*, int64_t>> snd(R);
    std::vector<std::pair<float*, int64_t>> rcv(R);
    for (int q = 0; q < R; ++q) {
        snd[q] = {S.msend + S.m_send_off[q], S.m_send_cnt[q]};
        rcv[q] = {S.mrecv + S.m_recv_off[q], S.m_recv_cnt[q]};
    }
    // level-1 multipoles all-gathered in place, in the same group as the LET exchange
    return nccl_p2p_group(R, S.rank, snd, rcv, (ncclComm_t)comm, st, l1 + S.rank * per1 * cellsz,
                          l1, per1 * cellsz);
}

}  // namespace vfmm
