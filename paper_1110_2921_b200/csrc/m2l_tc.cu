// m2l_tc.cu -- M2L (Eq. 11; operators of Cheng et al.) on the
// 5th-generation tensor cores with a 3-term split (A_hi B_hi + A_hi B_lo + A_lo B_hi) so the
// result keeps ~FP32 accuracy, operands staged by TMA (SWIZZLE_128B, K-major), accumulators in
// TMEM.  Two operand formats (same 10+1-bit significand, so the same split accuracy):
//   * 3xTF32 (tcgen05.mma kind::tf32): hi = v with the low 13 mantissa bits cleared.
//   * 3xFP16 (kind::f16, twice the tensor rate and half the operand bytes): the operator is
//     balanced by power-of-2 row/column scales, Ahat = T / (rs[r] cs[k]) (|Ahat| <= 1), and the
//     multipoles are staged as Mhat_k = M_k cs[k] s with one power-of-2 s per level chosen from
//     the level's max |cs[k] M_k| (max |Mhat| < 2^14, far from the half overflow); the epilogue
//     multiplies row r by rs[r] / s.  Every scale is exact, so apart from the half range
//     (entries below 2^-14 of the scaled max lose significand bits) the split is bit-for-bit
//     the TF32 one.
//
// The M2L of level l is a batch of dense GEMMs, one per (target parity pi, offset o):
//   D[r][(px,c)] += sum_k T_o[r][k] * Msrc[(px + dx, c)][k]
// A = T_o (128 output coefficients r x 128 input coefficients k, zero padded, one per slot),
// B = a "slab" of source multipoles: one x-row of XT <= 16 parent cells x 3 strength
// components = N <= 48 rows, read from a parity-major, halo-padded copy of the level's
// multipoles (stage kernels) so every (target row, offset) maps to one TMA box row.
// A CTA owns T target rows (Py .. Py+T-1, Pz) of one parity; their slabs are stacked so a
// single MMA (N' = T N <= 192) serves all T rows (T accumulator tiles side by side in TMEM).
// y-windows: the 189 offsets of a parity fall into 72 groups (source parent dx, dz, source
// parity) of <= 3 offsets dy = -1, 0, 1.  One TMA box of T + 2 consecutive y-slabs per group
// and K chunk serves all of them -- the B operand of offset dy is the window shifted by
// (dy + 1) N rows -- cutting the slab traffic to (T+2)/(2.6 T) of one load per offset.
//
// Accuracy: the tensor core accumulates with truncation, so a TMEM chain over all
// 189 offsets x 16 K-steps x 3 products (~9000 accumulations) drifts by ~1e-4.  The chain is
// therefore cut after every (offset group, K chunk) -- at p = 10 with the order split
// (launch_m2l_tc) <= 3 offsets x 10 MMAs: the MMA warp alternates between two TMEM buffers
// and the epilogue warps add each finished buffer into FP32 registers (round-to-nearest,
// packed f32x2 adds), so the result keeps ~FP32 accuracy (scripts/m2l_precision.py models the
// truncation; VFMM_M2L_CHAIN=1 cuts after every offset: 15 % less rounding in the coarse
// local expansions, 0.7 ms slower at c4, u and dgamma/dt unchanged).
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM alloc + MMA issuer,
// warps 2-9 = epilogue (TMEM -> FP32 register sums -> L in Morton order).
// CTA order: parity fastest, then 8x8 tiles of row groups, so co-resident CTAs share the
// source slabs they stream (L2 reuse).  CTAs run in 2-CTA clusters (same parity, adjacent
// row groups): each loads one half (hi or lo) of an operator chunk with TMA multicast into
// both CTAs, halving operator traffic; operator stages are released by both MMA warps.
#include <cuda.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "vfmm_internal.h"

namespace vfmm {

namespace {

// K chunks of 128 B: 4 x 32 tf32 or 2 x 64 halves (K = 128)
template <bool F16> __host__ __device__ constexpr int tc_ke() { return F16 ? 64 : 32; }
// A (operator) pipeline stages: TC_AST = 2 (template default), or 4 in the deep variant (the
// lean layout with T = 2 rows per CTA, 225 KB)
constexpr int TC_BST = 2;      // B pipeline stages (each holds one y-window of T + 2 slabs)
// MT = output row tiles of 128 (1: (p+1)^2 <= 128; 2: <= 256, f16 only)
constexpr int A_TILE = 128 * 128;  // one K chunk of 128 operator rows, one half (hi or lo): 16 KB
template <int MT> __host__ __device__ constexpr int a_bytes() { return MT * A_TILE; }
// max window rows (T + 2) N: MT = 1 up to 288 rows (36 KB), MT = 2 up to 192 (24 KB)
template <int MT> __host__ __device__ constexpr int b_wrows() { return MT == 1 ? 288 : 192; }
template <int MT> __host__ __device__ constexpr int b_bytes() { return b_wrows<MT>() * 128; }
// Epilogue warps: 8 (2 per TMEM lane quarter, the warp pair splits the T tiles) or, in the
// LEAN variant, 4 (one per quarter, T = 2 row tiles of N = 48: 96 columns each) with 192-row
// y-windows -- 161 KB of shared memory and 192 threads, so one P2P block (62 KB) fits beside
// it on the same SM (tensor pipe and FP32 pipe busy at once, capi.cu "co-resident mode")
template <bool LEAN> __host__ __device__ constexpr int tc_epi() { return LEAN ? 4 : 8; }
// warps: 0 operator producer, 1 MMA issuer, 2 .. 1 + tc_epi epilogue, 2 + tc_epi window producer
// (LEAN: warp 0 produces both, to stay within its register budget)
template <bool LEAN> __host__ __device__ constexpr int tc_threads() {
    return (LEAN ? 64 : 96) + 32 * tc_epi<LEAN>();
}
// window stage bytes: LEAN 192 rows; the 3-stage variant (AST = 3, XT = 8 / T = 8 layout)
// 240 rows (30 KB), which leaves room for a third operator stage
template <int MT, bool LEAN = false, int AST = 2> __host__ __device__ constexpr int b_bytes_v() {
    return LEAN ? 192 * 128 : (AST == 3 ? 240 * 128 : b_bytes<MT>());
}
template <int MT, bool LEAN = false, int AST = 2>
constexpr size_t tc_smem() {
    return 1024 + (size_t)AST * 2 * a_bytes<MT>() + (size_t)TC_BST * 2 * b_bytes_v<MT, LEAN, AST>() + 512;
}
static_assert(tc_smem<1, true, 4>() <= 232448, "deep variant exceeds 227 KB");
static_assert(tc_smem<2>() <= 232448, "MT = 2 stages exceed 227 KB");
static_assert(tc_smem<1, false, 3>() <= 232448, "3-stage variant exceeds 227 KB");
static_assert(tc_smem<1, true>() <= 166 * 1024, "LEAN stages exceed 166 KB");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    uint32_t done = 0;
    uint32_t spins = 0;
    while (!done) {
        if (++spins == (1u << 30)) asm volatile("trap;");  // watchdog: never hang the GPU
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, int c2, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// Warp-wide issue: the whole (converged) warp executes these, one elected lane issues.  The
// operands are then warp-uniform values, so no per-instruction elect/broadcast loop is needed
// to move them into uniform registers (as for an issue under `if (lane == 0)`).
__device__ __forceinline__ void mma_w(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                      uint32_t accumulate, bool f16) {
    if (f16)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_w(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::
            "r"(bar)
        : "memory");
}
__device__ __forceinline__ void commit_mc_w(uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n\t}" ::"r"(bar),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row atoms of 1024 B
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
    const uint64_t addr = smem_u32(p);
    uint64_t d = (addr >> 4) & 0x3FFFull;  // start address
    d |= 1ull << 16;                        // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;       // SBO = 1024 B between 8-row groups
    d |= 1ull << 46;                        // version (sm_100)
    d |= 2ull << 61;                        // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ uint32_t spread3t(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

struct TcParams {
    int nP;     // parent cells per axis at this level (2^(l-1))
    int XT;     // parents per B tile row (<= 32)
    int ntx;    // x tiles per row (nP / XT)
    int N;      // MMA N = 3 XT rounded up to a multiple of 16 (extra rows are discarded)
    int NV;     // valid columns = 3 * XT
    int T;      // target rows per CTA (accumulator tiles), T N <= 192
    int rows;   // target rows per parity = nP * nP * ntx
    int nc;     // (p+1)^2 <= 128 MT
    int nkc;    // K chunks of 128 B (64 halves / 32 tf32) covering nc
    int level;
    int bx0, by0, bz0, bny;  // owned box of target parents (origin; y extent)
    const int* slots;  // [8][189] M2L slot per target parity
    float* L;          // local expansions of this level, Morton [cell][3][nc]
    const float* rs;   // f16: row scales [128]
    const uint32_t* maxbits;  // f16: the level's max |cs[k] M_k| (float bits)
    const int4* groups;  // [8][72] offset groups per target parity (see m2l_groups)
    // bit s of full[mt]: K step s (MMA K = 16 halves / 8 tf32) of row tile mt takes the whole
    // 3-product split; otherwise hi x hi alone (see launch_m2l_tc: low-order terms only)
    uint32_t full[2];
    int chain;  // offsets per TMEM chain of a full-split K chunk (VFMM_M2L_CHAIN, default 3)
    int dbg;  // VFMM_M2L_DBG (measurement only, wrong results): 1 no TMEM drain, 2 no A, 4 no B loads
};

// f16 staging scale s = 2^(14 - e) for the level max m = f 2^e (f in [0.5, 1)): max |Mhat| < 2^14
__device__ __forceinline__ int h16_scale_exp(uint32_t bits) {
    const float m = __uint_as_float(bits);
    if (!(m > 0.f) || !isfinite(m)) return 0;
    int e;
    frexpf(m, &e);
    return min(14 - e, 120);
}

// row group g of a CTA -> (x tile, first target row y, row z) inside the owned box;
// groups are visited in 8x8 tiles of (y group, z) so co-resident CTAs share source rows
__device__ __forceinline__ void group_rows(const TcParams& P, int g, int* tx, int* py0, int* pz) {
    *tx = g % P.ntx;
    const int gg = g / P.ntx;
    const int GY = P.bny / P.T, GZ = P.rows / (P.ntx * P.bny);  // groups along y, rows in z
    int gy, gz;
    if (GY % 8 == 0 && GZ % 8 == 0) {
        const int tile = gg / 64, w = gg % 64;
        gy = (tile % (GY / 8)) * 8 + (w & 7);
        gz = (tile / (GY / 8)) * 8 + (w >> 3);
    } else {
        gy = gg % GY;
        gz = gg / GY;
    }
    *py0 = P.by0 + gy * P.T;
    *pz = P.bz0 + gz;
}

// VFMM_M2L_DBG & 8 (measurement only): clock64 timeline of cluster 0 (CTAs 0 and 1) of a
// launch with >= 1024 CTAs; the next launch prints a summary to stderr.  Events per CTA:
// 0 producer past a_empty (per operator load), 1 MMA past a_full, 2 MMA past its commits,
// 3 epilogue warp 2 past acc_full, 4 MMA past acc_empty (per chain); meta: kernel start,
// MMA loop end, epilogue stores end
constexpr int TR_N = 1024;
__device__ long long g_m2l_trace[2][5][TR_N];
__device__ long long g_m2l_meta[2][4];

__device__ __forceinline__ long long clk() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}

template <bool F16, int MT, bool LEAN = false, int TC_AST = 2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc_threads<LEAN>(), LEAN ? 2 : 1)
    m2l_tc_kernel(const __grid_constant__ CUtensorMap tmA_hi, const __grid_constant__ CUtensorMap tmA_lo,
                  const __grid_constant__ CUtensorMap tmB_hi, const __grid_constant__ CUtensorMap tmB_lo,
                  TcParams P) {
    extern __shared__ uint8_t tc_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>(((uintptr_t)tc_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* Abuf = sm;                                  // [AST][hi|lo][16 KB]
    constexpr int A_BYTES = a_bytes<MT>(), B_BYTES = b_bytes_v<MT, LEAN, TC_AST>();
    uint8_t* Bbuf = sm + TC_AST * 2 * A_BYTES;           // [BST][hi|lo][B_BYTES]
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bbuf + TC_BST * 2 * B_BYTES);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + TC_AST;
    uint64_t* b_full = bars + 2 * TC_AST;
    uint64_t* b_empty = bars + 2 * TC_AST + TC_BST;
    uint64_t* acc_full = bars + 2 * TC_AST + 2 * TC_BST;  // [2]
    uint64_t* acc_empty = acc_full + 2;                  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // 2-CTA clusters: both CTAs take the same parity (same operator sequence) and adjacent row
    // groups; each loads one half (hi / lo) of every operator chunk and multicasts it to both
    const uint32_t crank = cluster_rank();
    const int cidx = blockIdx.x >> 1;
    const int pi = cidx & 7;  // target parity fastest (co-resident clusters share slabs)
    const int g = ((cidx >> 3) << 1) | (int)crank;
    const int pix = pi & 1, piy = (pi >> 1) & 1, piz = (pi >> 2) & 1;
    int gtx, gpy0, gpz;
    group_rows(P, g, &gtx, &gpy0, &gpz);
    constexpr uint32_t tmem_cols = 512;  // 2 buffers x 256 columns

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < TC_AST; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 2);  // both CTAs' MMA warps release a shared operator stage
        }
        for (int i = 0; i < TC_BST; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], tc_epi<LEAN>());
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // peer barriers initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const bool tr = (P.dbg & 8) && blockIdx.x < 2 && gridDim.x >= 1024;
    const int tb = blockIdx.x & 1;
    if (tr && threadIdx.x == 0) g_m2l_meta[tb][0] = clk();

    if (warp == 0 || (!LEAN && warp == 2 + tc_epi<LEAN>())) {
        // ===================== TMA producers =====================
        // per offset group (dx, dz, source parity): one y-window of T + 2 slabs (rows
        // gpy0 - 1 .. gpy0 + T) per K chunk serves the group's <= 3 offsets dy = -1, 0, 1
        // (window producer, the last warp); the operator chunk of each valid offset, shared
        // with the peer CTA (operator producer, warp 0).  Two threads, so neither stream waits
        // behind the other's free slots.
        const bool doA = warp == 0, doB = LEAN || warp != 0;
        if (lane == 0) {
            int sa = 0, sb = 0, nload = 0;
            uint32_t pa = 0, pb = 0;
            const uint32_t b_tx = 2u * (uint32_t)((P.T + 2) * P.N) * 128u;
            for (int gi = 0; gi < 72; ++gi) {
                const int4 G = P.groups[pi * 72 + gi];
                const int mask = G.x & 7;
                if (!mask) continue;
                const int dx = ((G.x >> 4) & 3) - 1, dz = ((G.x >> 6) & 3) - 1, pis = (G.x >> 8) & 7;
                const int c1 = 3 * (2 + P.bx0 + gtx * P.XT + dx);
                const int c2 = 1 + gpy0, c3 = 2 + gpz + dz;
                for (int kc = 0; kc < P.nkc; ++kc) {
                    // the lo halves are loaded only for K chunks with a full-split step
                    const bool need_lo = (((P.full[0] | (MT == 2 ? P.full[1] : 0u)) >> (4 * kc)) & 15u) != 0;
                    if (doB) {
                    mbar_wait(&b_empty[sb], pb ^ 1);
                    if (P.dbg & 4) {
                        mbar_arrive(&b_full[sb]);
                    } else {
                    mbar_expect_tx(&b_full[sb], need_lo ? b_tx : b_tx / 2);
                    tma_load_5d(Bbuf + (sb * 2 + 0) * B_BYTES, &tmB_hi, &b_full[sb], kc * tc_ke<F16>(),
                                c1, c2, c3, pis);
                    if (need_lo)
                        tma_load_5d(Bbuf + (sb * 2 + 1) * B_BYTES, &tmB_lo, &b_full[sb],
                                    kc * tc_ke<F16>(), c1, c2, c3, pis);
                    }
                    if (++sb == TC_BST) {
                        sb = 0;
                        pb ^= 1;
                    }
                    }
                    if (!doA) continue;
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        if (!((mask >> d) & 1)) continue;
                        const int slot = d == 0 ? G.y : (d == 1 ? G.z : G.w);
                        mbar_wait(&a_empty[sa], pa ^ 1);
                        if (tr && nload < TR_N) g_m2l_trace[tb][0][nload] = clk();
                        ++nload;
                        if (P.dbg & 2) {
                            mbar_arrive(&a_full[sa]);
                        } else if (need_lo) {  // hi from rank 0, lo from rank 1
                            mbar_expect_tx(&a_full[sa], 2u * A_BYTES);
                            if (crank == 0)
                                tma_load_3d_mc(Abuf + (sa * 2 + 0) * A_BYTES, &tmA_hi, &a_full[sa],
                                               kc * tc_ke<F16>(), 0, slot, (uint16_t)3);
                            else
                                tma_load_3d_mc(Abuf + (sa * 2 + 1) * A_BYTES, &tmA_lo, &a_full[sa],
                                               kc * tc_ke<F16>(), 0, slot, (uint16_t)3);
                        } else {  // hi only, the ranks take turns
                            mbar_expect_tx(&a_full[sa], (uint32_t)A_BYTES);
                            if ((int)crank == ((gi + d) & 1))
                                tma_load_3d_mc(Abuf + (sa * 2 + 0) * A_BYTES, &tmA_hi, &a_full[sa],
                                               kc * tc_ke<F16>(), 0, slot, (uint16_t)3);
                        }
                        if (++sa == TC_AST) {
                            sa = 0;
                            pa ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        // instruction descriptor: D f32, A/B tf32 (2) or f16 (0), both K-major, N, M = 128
        // one MMA covers all T rows: N' = T N columns (tile t at columns [t N, (t+1) N)); the
        // B operand of offset dy starts (dy + 1) N rows into the y-window.  One TMEM
        // accumulation chain per group (<= 3 offsets x K x 3 products), then flushed to FP32
        const uint32_t ab_fmt = F16 ? 0u : 2u;
        const uint32_t idesc = (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) |
                               ((uint32_t)((P.T * P.N) >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t slab_step = (uint64_t)((P.N * 128) >> 4);  // descriptor units (16 B)
        int sa = 0, sb = 0;
        uint32_t pa = 0, pb = 0;
        // One TMEM accumulation chain per P.chain offsets of a group and K chunk (<= 4 K steps
        // x 3 products each), or, for a K chunk without full-split steps (hi x hi alone, high
        // orders only), per (offset group, K chunk): <= 3 offsets x 4 single MMAs.
        int chain = 0;
        // issue one chain segment: K steps [0, nks) of every row tile, the first nf[mt] steps
        // with the whole split; first = this segment opens the TMEM chain
        auto issue = [&](uint32_t d, uint64_t ahi, uint64_t alo, uint64_t bhi, uint64_t blo,
                         int nks, int nf0, int nf1, bool first) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {  // row tile mt: rows 128 mt ..
                const uint32_t dm = d + (uint32_t)(mt * P.T * P.N);
                const uint64_t am = (uint64_t)(mt * (A_TILE >> 4));
                const int nf = mt == 0 ? nf0 : nf1;
                for (int ks = 0; ks < nks; ++ks) {  // K = 8 tf32 / 16 f16 = 32 B per MMA
                    const uint64_t adv = (uint64_t)(ks * 2);
                    const uint32_t acc = (first && ks == 0) ? 0u : 1u;
                    mma_w(dm, ahi + am + adv, bhi + adv, idesc, acc, F16);
                    if (ks < nf) {
                        mma_w(dm, ahi + am + adv, blo + adv, idesc, 1u, F16);
                        mma_w(dm, alo + am + adv, bhi + adv, idesc, 1u, F16);
                    }
                }
            }
        };
        for (int gi = 0; gi < 72; ++gi) {
            const int mask = P.groups[pi * 72 + gi].x & 7;
            if (!mask) continue;
            const int last_dd = 31 - __clz(mask);
            for (int kc = 0; kc < P.nkc; ++kc) {
                // K steps holding real coefficients: the last chunk of a padded K
                // (e.g. (p+1)^2 = 196 in 4 chunks of 64) skips its all-zero steps
                const int kleft = P.nc - kc * tc_ke<F16>();
                const int nks = min(4, (kleft + tc_ke<F16>() / 4 - 1) / (tc_ke<F16>() / 4));
                // leading full-split steps of this chunk per row tile (a prefix by construction)
                const int nf0 = __popc((P.full[0] >> (4 * kc)) & 15u);
                const int nf1 = MT == 2 ? __popc((P.full[1] >> (4 * kc)) & 15u) : 0;
                const bool merged = nf0 == 0 && nf1 == 0;
                mbar_wait(&b_full[sb], pb);
                tc_fence_after();
                const uint64_t bhi = sw128_desc(Bbuf + (sb * 2 + 0) * B_BYTES);
                const uint64_t blo = sw128_desc(Bbuf + (sb * 2 + 1) * B_BYTES);
#pragma unroll
                for (int dd = 0; dd < 3; ++dd) {
                    if (!((mask >> dd) & 1)) continue;
                    const int buf = chain & 1;
                    // position of this offset among the group's offsets; a full chunk's chain
                    // spans P.chain consecutive offsets, a hi-only chunk's the whole group
                    const int pos = __popc(mask & ((1 << dd) - 1));
                    const bool opens = merged ? pos == 0 : pos % P.chain == 0;
                    const bool closes = dd == last_dd || (!merged && pos % P.chain == P.chain - 1);
                    if (opens) {
                        mbar_wait(&acc_empty[buf], ((chain >> 1) & 1) ^ 1);  // epilogue drained it
                        if (tr && lane == 0 && chain < TR_N) g_m2l_trace[tb][4][chain] = clk();
                    }
                    mbar_wait(&a_full[sa], pa);
                    if (tr && lane == 0 && chain < TR_N) g_m2l_trace[tb][1][chain] = clk();
                    tc_fence_after();
                    const uint32_t d = tmem + (uint32_t)(buf * 256);
                    const uint64_t ahi = sw128_desc(Abuf + (sa * 2 + 0) * A_BYTES);
                    const uint64_t alo = sw128_desc(Abuf + (sa * 2 + 1) * A_BYTES);
                    const uint64_t bsh = (uint64_t)dd * slab_step;
                    __syncwarp();
                    issue(d, ahi, alo, bhi + bsh, blo + bsh, nks, nf0, nf1, opens);
                    commit_mc_w(smem_u32(&a_empty[sa]), (uint16_t)3);  // release in both CTAs
                    if (closes) {
                        commit_w(smem_u32(&acc_full[buf]));
                        if (tr && lane == 0 && chain < TR_N) g_m2l_trace[tb][2][chain] = clk();
                    }
                    __syncwarp();
                    if (closes) ++chain;
                    if (++sa == TC_AST) {
                        sa = 0;
                        pa ^= 1;
                    }
                }
                __syncwarp();
                commit_w(smem_u32(&b_empty[sb]));
                if (++sb == TC_BST) {
                    sb = 0;
                    pb ^= 1;
                }
            }
        }
    } else {
        // ===================== epilogue: TMEM groups -> FP32 register sums -> L =====================
        const int e = warp - 2;
        const int quarter = warp & 3;  // TMEM lanes [32 quarter, 32 quarter + 32)
        const int half = LEAN ? 0 : e >> 2;  // this warp owns tiles [half T/2, (half+1) T/2)
        const int tpw = LEAN ? P.T : P.T / 2;  // tiles per warp
        const int ncol = tpw * P.N;    // columns per warp and row tile: MT * ncol <= 96
        const int col0 = half * ncol;
        const int r = quarter * 32 + lane;
        // each finished chain (one offset x one K chunk, <= 12 MMAs per row tile: truncating TMEM
        // accumulation) is added into FP32 registers with round-to-nearest, packed two at a time
        unsigned long long acc2[48];
#pragma unroll
        for (int j = 0; j < 48; ++j) acc2[j] = 0ull;
        // chains: one per (offset, K chunk), or one per (group, K chunk) for a chunk without
        // full-split steps (see the MMA issuer)
        int nchains = 0;
        for (int gi = 0; gi < 72; ++gi) {
            const int m = P.groups[pi * 72 + gi].x & 7;
            if (!m) continue;
            for (int kc = 0; kc < P.nkc; ++kc) {
                const bool merged = ((P.full[0] | (MT == 2 ? P.full[1] : 0u)) >> (4 * kc) & 15u) == 0;
                nchains += merged ? 1 : (__popc(m) + P.chain - 1) / P.chain;
            }
        }
        for (int ch = 0; ch < nchains; ++ch) {
            const int buf = ch & 1;
            mbar_wait(&acc_full[buf], (ch >> 1) & 1);
            if (tr && e == 0 && lane == 0 && ch < TR_N) g_m2l_trace[tb][3][ch] = clk();
            tc_fence_after();
            if (P.dbg & 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[buf]);
                continue;
            }
            // two halves of 48 accumulator columns (MT = 1: the warp's 96 columns; MT = 2: one
            // row tile each), three 16-column loads in flight, one wait each
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                uint32_t w[48];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int col = MT == 1 ? (hh * 3 + c) * 16 : c * 16;
                    const int tcol = MT == 1 ? col0 + col : hh * P.T * P.N + col0 + col;
                    if (col < ncol) {
                        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) +
                                               (uint32_t)(buf * 256 + tcol);
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, "
                            "%7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
                            : "=r"(w[c * 16 + 0]), "=r"(w[c * 16 + 1]), "=r"(w[c * 16 + 2]),
                              "=r"(w[c * 16 + 3]), "=r"(w[c * 16 + 4]), "=r"(w[c * 16 + 5]),
                              "=r"(w[c * 16 + 6]), "=r"(w[c * 16 + 7]), "=r"(w[c * 16 + 8]),
                              "=r"(w[c * 16 + 9]), "=r"(w[c * 16 + 10]), "=r"(w[c * 16 + 11]),
                              "=r"(w[c * 16 + 12]), "=r"(w[c * 16 + 13]), "=r"(w[c * 16 + 14]),
                              "=r"(w[c * 16 + 15])
                            : "r"(taddr));
                    }
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int col = MT == 1 ? (hh * 3 + c) * 16 : c * 16;
                    if (col < ncol) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            unsigned long long v;
                            asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(w[c * 16 + 2 * j]),
                                "r"(w[c * 16 + 2 * j + 1]));
                            const int a = (hh * 3 + c) * 8 + j;
                            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc2[a]) : "l"(acc2[a]), "l"(v));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
        if (tr && e == 0 && lane == 0) g_m2l_meta[tb][1] = clk();
        float acc[96];
#pragma unroll
        for (int j = 0; j < 48; ++j)
            asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[2 * j]), "=f"(acc[2 * j + 1]) : "l"(acc2[j]));
        const float sinv = F16 ? ldexpf(1.f, -h16_scale_exp(*P.maxbits)) : 1.f;
        const uint32_t cz = spread3t(2 * gpz + piz) << 2;
        // Stage the scaled sums through shared memory (the operand buffers are idle once the
        // last chain is drained: every MMA has read them and every load, the peer's multicasts
        // included, has landed) so the scatter into L is one short loop -- 96 unrolled address
        // computations made a ~9000-instruction tail that missed the instruction cache
        float* stg = reinterpret_cast<float*>(sm) + e * (96 * 32);
        constexpr int CPT = 96 / MT;  // accumulator columns per row tile
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int rr = r + 128 * mt;
            const float fsc = (F16 && rr < P.nc) ? P.rs[rr] * sinv : 1.f;  // undo the balancing
#pragma unroll
            for (int jj = 0; jj < CPT; ++jj) stg[(mt * CPT + jj) * 32 + lane] = acc[mt * CPT + jj] * fsc;
        }
        __syncwarp();
        for (int mt = 0; mt < MT; ++mt) {
            const int rr = r + 128 * mt;
            if (rr >= P.nc) continue;
            for (int jj = 0; jj < ncol; ++jj) {
                const int t = half * tpw + jj / P.N, cj = jj % P.N;
                if (cj >= P.NV) continue;
                const int py = gpy0 + t;
                const int px = P.bx0 + gtx * P.XT + cj / 3, comp = cj % 3;
                const uint32_t cell = spread3t(2 * px + pix) | (spread3t(2 * py + piy) << 1) | cz;
                P.L[((int64_t)cell * 3 + comp) * P.nc + rr] = stg[(mt * CPT + jj) * 32 + lane];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tr && threadIdx.x == 0) g_m2l_meta[tb][2] = clk();
    cluster_sync();  // the peer may still multicast into / arrive on this CTA until here
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(tmem_cols));
}

// Morton level multipoles -> parity-major halo-padded grid (hi = tf32 part, lo = rest):
// grid[pi'][Z][Y][X][comp][128], parent coords (X-2, Y-2, Z-2) wrapped (periodic) or zero.
__global__ void m2l_stage_kernel(const float* __restrict__ M, int nP, int periodic, int nc,
                                 float* __restrict__ ghi, float* __restrict__ glo) {
    const int Xp = nP + 4;
    const int64_t total = (int64_t)8 * Xp * Xp * Xp * 3 * 128;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i & 127);
        int64_t q = i >> 7;
        const int comp = (int)(q % 3);
        q /= 3;
        const int X = (int)(q % Xp);
        q /= Xp;
        const int Y = (int)(q % Xp);
        q /= Xp;
        const int Z = (int)(q % Xp);
        const int ps = (int)(q / Xp);
        int px = X - 2, py = Y - 2, pz = Z - 2;
        float v = 0.f;
        const bool inside = px >= 0 && px < nP && py >= 0 && py < nP && pz >= 0 && pz < nP;
        if (k < nc && (periodic || inside)) {
            px = (px + nP) % nP;
            py = (py + nP) % nP;
            pz = (pz + nP) % nP;
            const uint32_t cell = spread3t(2 * px + (ps & 1)) | (spread3t(2 * py + ((ps >> 1) & 1)) << 1) |
                                  (spread3t(2 * pz + ((ps >> 2) & 1)) << 2);
            v = M[((int64_t)cell * 3 + comp) * nc + k];
        }
        const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
        ghi[i] = hi;
        glo[i] = v - hi;
    }
}

// f16 staging, two passes over the same padded grid.  One block per (pi', Z, Y) x-row of the
// grid (blockDim = (128 k, 4)); the 4 thread rows walk its 3 (Xp) (X, comp) rows, so the
// Morton bits of (Y, Z, pi') are computed once per block.
// MAXPASS: max |cs[k] M_k| of the staged values -> atomicMax on the float bits (non-negative);
// else:    grid[pi'][Z][Y][X][comp][128] = half split of M_k cs[k] s, s = 2^h16_scale_exp(max)
template <bool MAXPASS>
__global__ void __launch_bounds__(512) m2l_stage16_kernel(const float* __restrict__ M, int nP,
                                                          int periodic, int nc,
                                                          const float* __restrict__ cs,
                                                          uint32_t* __restrict__ maxbits,
                                                          __half* __restrict__ ghi,
                                                          __half* __restrict__ glo) {
    const int Xp = nP + 4;
    const int k = threadIdx.x;
    const float ck = k < nc ? cs[k] : 0.f;
    const float s = MAXPASS ? 1.f : ldexpf(1.f, h16_scale_exp(*maxbits));
    const int Y = blockIdx.x % Xp, Z = (blockIdx.x / Xp) % Xp, ps = blockIdx.x / (Xp * Xp);
    int py = Y - 2, pz = Z - 2;
    const bool yz_in = py >= 0 && py < nP && pz >= 0 && pz < nP;
    py = (py + nP) & (nP - 1);
    pz = (pz + nP) & (nP - 1);
    const uint32_t cyz = (spread3t(2 * py + ((ps >> 1) & 1)) << 1) |
                         (spread3t(2 * pz + ((ps >> 2) & 1)) << 2);
    const bool kin = k < nc && (periodic || yz_in);
    const int64_t row0 = (int64_t)blockIdx.x * Xp * 3;  // grid row of (X = 0, comp = 0)
    float mx = 0.f;
    for (int rr = threadIdx.y; rr < 3 * Xp; rr += blockDim.y) {
        const int X = rr / 3, comp = rr - 3 * X;
        const int px = X - 2;
        float v = 0.f;
        if (kin && (periodic || (px >= 0 && px < nP))) {
            const uint32_t cell = spread3t(2 * ((px + nP) & (nP - 1)) + (ps & 1)) | cyz;
            v = M[((int64_t)cell * 3 + comp) * nc + k];
        }
        if (MAXPASS) {
            mx = fmaxf(mx, fabsf(v * ck));
        } else {
            const float x = v * ck * s;
            const __half h = __float2half_rn(x);
            const __half l = __float2half_rn(x - __half2float(h));
            ghi[(row0 + rr) * blockDim.x + k] = h;  // row length = padded K (128 or 256)
            glo[(row0 + rr) * blockDim.x + k] = l;
        }
    }
    if (MAXPASS) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0 && mx > 0.f) atomicMax(maxbits, __float_as_uint(mx));
    }
}

// the level's max |cs[k] M_k| straight over the Morton array (every cell once, coalesced;
// the halo copies of the staged grid repeat these values or are zero)
__global__ void __launch_bounds__(256) m2l_max_kernel(const float* __restrict__ M, int64_t count,
                                                      int nc, const float* __restrict__ cs,
                                                      uint32_t* __restrict__ maxbits) {
    float mx = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        mx = fmaxf(mx, fabsf(M[i] * cs[(int)(i % nc)]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ float wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float b = 0.f;
        for (int w = 0; w < 8; ++w) b = fmaxf(b, wm[w]);
        if (b > 0.f) atomicMax(maxbits, __float_as_uint(b));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

}  // namespace

// rows per CTA for a box: the largest T in {8, 4, 2} with MT T N <= 192 (MT = 2: T N <= 128)
// and (T + 2) N within the window stage, T | bny and an even number of CTAs (2-CTA clusters);
// 0 if none
// parents per slab row: 16 (N = 48, T = 4) or VFMM_M2L_XT=8 (N = 24, T = 8: same MMA N', a
// 240-row window instead of 288)
static int pick_XT(const int box[6]) {
    int xt = 16;
    if (const char* e = getenv("VFMM_M2L_XT")) xt = atoi(e) == 8 ? 8 : 16;
    return box[3] < xt ? box[3] : xt;
}
// slab rows N: 3 XT rounded up to 16, or exactly 24 for XT = 8 (a multiple of the 8-row
// swizzle atom; the MMA N' = T N stays a multiple of 16 for even T)
static int slab_N(int XT) { return XT == 8 ? 24 : (3 * XT + 15) / 16 * 16; }
static int pick_T(const int box[6], int MT, bool lean = false) {
    const int bnx = box[3], bny = box[4], bnz = box[5];
    const int XT = pick_XT(box);
    if (bnx % XT != 0) return 0;
    const int N = slab_N(XT);
    const int rows = bny * bnz * (bnx / XT);
    const int wrows = lean ? 192 : (MT == 1 ? b_wrows<1>() : b_wrows<2>());
    for (int T = 8; T >= 2; T /= 2) {
        // accumulator columns per epilogue warp (its tiles x N x row tiles) fit its 96
        // registers; one TMEM buffer (MT T N columns) fits half of the 512 columns
        const int warp_cols = (lean ? T : T / 2) * N * MT;
        if (warp_cols <= 96 && MT * T * N <= 256 && (T + 2) * N <= wrows && (T * N) % 16 == 0 &&
            bny % T == 0 && (rows / T) % 2 == 0)
            return T;
    }
    return 0;
}

// lowest term degree run as hi x hi alone (VFMM_M2L_SPLIT=<degree>; "full" keeps the
// 3-product split for every term)
int m2l_split_degree() {
    const char* e = getenv("VFMM_M2L_SPLIT");
    if (e && e[0]) {
        if (!strcmp(e, "full")) return 1 << 20;
        const int v = atoi(e);
        if (v > 0) return v;
    }
    return 6;
}

bool m2l_tc_shape_ok(const int box[6], int p) {
    return pick_T(box, (p + 1) * (p + 1) > 128 ? 2 : 1) != 0;
}

// (p+1)^2 <= 128: 3xTF32 or 3xFP16; (p+1)^2 <= 256 (p <= 15): 3xFP16 with two row tiles
bool m2l_tc_supported(int p, int level) {
    return (p + 1) * (p + 1) <= 256 && level >= 2 && get_encode() != nullptr;
}

size_t m2l_tc_grid_floats(int level) {  // floats: 128 tf32 or 256 halves per grid row
    const int64_t nP = (int64_t)1 << (level - 1), Xp = nP + 4;
    return (size_t)(8 * Xp * Xp * Xp * 3 * 128);
}

int launch_m2l_tc(const TcOps& ops, const int* il_slots, int p, const float* M_l, float* L_l,
                  int level, int periodic, float* ghi, float* glo, uint32_t* maxbits,
                  const int box[6], cudaStream_t st) {
    const int nc = (p + 1) * (p + 1);
    const int nP = 1 << (level - 1);
    const int Xp = nP + 4;
    const bool f16 = ops.f16;
    const int MT = ops.nr / 128;   // output row tiles
    const int KPG = ops.kp;        // padded K of the operators and of the staged grid rows
    if (nc > ops.nr || nc > KPG || (MT == 2 && !f16) || MT < 1 || MT > 2) return -5;
    const int nkc = (nc + (f16 ? 63 : 31)) / (f16 ? 64 : 32);
    const size_t esz = f16 ? 2 : 4;
    const CUtensorMapDataType dt = f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const cuuint32_t ke = f16 ? 64 : 32;  // K elements per 128-byte chunk
    // 1) stage the level's multipoles into the halo-padded parity-major grid
    {
        const int64_t total = (int64_t)8 * Xp * Xp * Xp * 3 * 128;
        if (f16) {
            const int64_t blocks = (int64_t)8 * Xp * Xp;  // one per (pi', Z, Y) x-row
            const dim3 blk(KPG, 512 / KPG);
            const int64_t cnt = ((int64_t)1 << (3 * level)) * 3 * nc;
            const int64_t mb = std::min<int64_t>((cnt + 255) / 256, 148 * 8);
            m2l_max_kernel<<<(unsigned)mb, 256, 0, st>>>(M_l, cnt, nc, ops.cs, maxbits);
            m2l_stage16_kernel<false><<<(unsigned)blocks, blk, 0, st>>>(
                M_l, nP, periodic, nc, ops.cs, maxbits, reinterpret_cast<__half*>(ghi),
                reinterpret_cast<__half*>(glo));
        } else {
            int64_t blocks = (total + 255) / 256;
            if (blocks > 148 * 64) blocks = 148 * 64;
            m2l_stage_kernel<<<(unsigned)blocks, 256, 0, st>>>(M_l, nP, periodic, nc, ghi, glo);
        }
    }
    // 2) tensor maps
    auto enc = get_encode();
    if (!enc) return -1;
    CUtensorMap mAh, mAl, mBh, mBl;
    {
        cuuint64_t dims[3] = {(cuuint64_t)KPG, (cuuint64_t)ops.nr, 343};
        cuuint64_t strides[2] = {KPG * esz, (cuuint64_t)KPG * ops.nr * esz};
        cuuint32_t bx[3] = {ke, (cuuint32_t)ops.nr, 1};
        cuuint32_t es[3] = {1, 1, 1};
        if (enc(&mAh, dt, 3, const_cast<void*>(ops.hi), dims, strides, bx, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -2;
        if (enc(&mAl, dt, 3, const_cast<void*>(ops.lo), dims, strides, bx, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -2;
    }
    // owned box of target parents: origin box[0..2], extents box[3..5] (whole level: 0, nP)
    const int bnx = box[3], bny = box[4], bnz = box[5];
    const int XT = pick_XT(box);
    const int NV = 3 * XT;
    // VFMM_M2L_DEEP=1: the lean layout (T = 2) with 4 operator stages for the plain pipeline
    const char* deep_env = getenv("VFMM_M2L_DEEP");
    const bool deep = deep_env && deep_env[0] == '1' && !ops.lean && MT == 1 && f16 &&
                      pick_T(box, 1, true) != 0;
    const bool lean = (ops.lean || deep) && MT == 1 && f16 && pick_T(box, 1, true) != 0;
    const int T = pick_T(box, MT, lean);
    if (T == 0) return -4;
    const int N = slab_N(XT);  // slab rows (T N: the MMA N, a multiple of 16 for M = 128)
    {
        const cuuint64_t row = (cuuint64_t)KPG * esz;
        cuuint64_t dims[5] = {(cuuint64_t)KPG, (cuuint64_t)3 * Xp, (cuuint64_t)Xp, (cuuint64_t)Xp, 8};
        cuuint64_t strides[4] = {row, (cuuint64_t)3 * Xp * row, (cuuint64_t)Xp * 3 * Xp * row,
                                 (cuuint64_t)Xp * Xp * 3 * Xp * row};
        cuuint32_t bx[5] = {ke, (cuuint32_t)N, (cuuint32_t)(T + 2), 1, 1};  // y-window
        cuuint32_t es[5] = {1, 1, 1, 1, 1};
        if (enc(&mBh, dt, 5, (void*)ghi, dims, strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -3;
        if (enc(&mBl, dt, 5, (void*)glo, dims, strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -3;
    }
    static PerDeviceOnce once;
    once([] {
        cudaFuncSetAttribute(m2l_tc_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_smem<1>());
        cudaFuncSetAttribute(m2l_tc_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_smem<1>());
        cudaFuncSetAttribute(m2l_tc_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_smem<2>());
        cudaFuncSetAttribute(m2l_tc_kernel<true, 1, false, 3>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem<1, false, 3>());
        cudaFuncSetAttribute(m2l_tc_kernel<true, 1, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem<1, true>());
        cudaFuncSetAttribute(m2l_tc_kernel<true, 1, true, 4>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_smem<1, true, 4>());
    });
    TcParams P;
    P.nP = nP;
    P.XT = XT;
    P.ntx = bnx / XT;
    P.N = N;
    P.NV = NV;
    P.rows = bny * bnz * P.ntx;
    P.bx0 = box[0];
    P.by0 = box[1];
    P.bz0 = box[2];
    P.bny = bny;
    P.nc = nc;
    P.nkc = nkc;
    P.level = level;
    P.slots = il_slots;
    P.L = L_l;
    P.rs = ops.rs;
    P.maxbits = maxbits;
    P.T = T;
    P.groups = ops.groups;
    {
        const char* d = getenv("VFMM_M2L_DBG");
        P.dbg = d ? atoi(d) : 0;
        const char* ch = getenv("VFMM_M2L_CHAIN");
        P.chain = ch ? std::max(1, std::min(3, atoi(ch))) : 3;
        static bool traced = false;
        if ((P.dbg & 8) && traced) {  // summary of the previous traced launch
            static long long T[2][5][TR_N], Mt[2][4];
            cudaStreamSynchronize(st);
            cudaMemcpyFromSymbol(T, g_m2l_trace, sizeof(T));
            cudaMemcpyFromSymbol(Mt, g_m2l_meta, sizeof(Mt));
            for (int b = 0; b < 2; ++b) {
                const long long t0 = Mt[b][0];
                int nch = 0;
                while (nch < TR_N && T[b][3][nch] > t0) ++nch;
                double per = 0, ia = 0, ex = 0, pr = 0;
                int cnt = 0;
                for (int c = 20; c + 2 < nch - 20; ++c, ++cnt) {
                    per += (double)(T[b][3][c + 1] - T[b][3][c]);  // chain completion period
                    ia += (double)(T[b][1][c] - T[b][4][c]);       // acc_empty -> a_full
                    ex += (double)(T[b][3][c] - T[b][2][c]);       // commit issued -> complete
                    pr += (double)(T[b][1][c + 2] - T[b][3][c]);   // c done -> c+2 issuable
                }
                if (cnt) {
                    fprintf(stderr,
                            "[m2l trace] cta %d: kernel %lld cyc, chains %d, MMA loop %lld, "
                            "stores %lld; per chain: period %.0f, acc_empty->a_full %.0f, "
                            "issue->complete %.0f, complete(c)->a_full(c+2) %.0f\n",
                            b, Mt[b][2] - t0, nch, Mt[b][1] - t0, Mt[b][2] - Mt[b][1], per / cnt,
                            ia / cnt, ex / cnt, pr / cnt);
                    if (P.dbg & 16)  // every chain of this CTA
                        for (int c = 0; c < nch; ++c)
                            fprintf(stderr, "T %d %d %lld %lld %lld %lld %lld\n", b, c,
                                    T[b][4][c] - t0, T[b][1][c] - t0, T[b][2][c] - t0,
                                    T[b][3][c] - t0, T[b][0][c] - t0);
                    for (int c = 100; c < 106 && c < nch; ++c)
                        fprintf(stderr, "  chain %d: acc_empty %lld a_full %lld committed %lld "
                                "epi %lld (load %lld)\n", c, T[b][4][c] - t0, T[b][1][c] - t0,
                                T[b][2][c] - t0, T[b][3][c] - t0, T[b][0][c] - t0);
                }
            }
        }
        if ((P.dbg & 8) && (int)(8 * (bny * bnz * (bnx / XT) / T)) >= 1024) traced = true;
    }
    // Split by term order.  Term (r, k) of a translation couples local degree j(r) with
    // multipole degree n(k); its share of the field falls geometrically with j + n (the p sweep
    // in DESIGN.md 7: ~0.43 per degree), so the A_hi B_lo + A_lo B_hi correction (2^-11 of a
    // term) matters only for the low orders.  K step s of row tile mt takes the full split iff
    // both the tile's lowest row degree and the step's lowest column degree are below
    // m2l_split_degree(); the others run hi x hi alone (DESIGN.md 6b "order-split M2L").
    {
        const int n0 = m2l_split_degree();
        const int kstep = f16 ? 16 : 8;  // coefficients per MMA K step
        auto deg = [](int k) { int n = 0; while ((n + 1) * (n + 1) <= k) ++n; return n; };
        for (int mt = 0; mt < 2; ++mt) {
            P.full[mt] = 0u;
            if (mt >= MT) continue;
            const int jmin = deg(128 * mt);
            for (int s = 0; s < 4 * nkc && s < 32; ++s)
                if (jmin < n0 && deg(s * kstep) < n0) P.full[mt] |= 1u << s;
        }
    }
    const unsigned grid = (unsigned)(8 * (P.rows / P.T));
    if (f16 && MT == 2)
        m2l_tc_kernel<true, 2><<<grid, tc_threads<false>(), tc_smem<2>(), st>>>(mAh, mAl, mBh, mBl, P);
    else if (deep)
        m2l_tc_kernel<true, 1, true, 4><<<grid, tc_threads<true>(), tc_smem<1, true, 4>(), st>>>(
            mAh, mAl, mBh, mBl, P);
    else if (lean)
        m2l_tc_kernel<true, 1, true><<<grid, tc_threads<true>(), tc_smem<1, true>(), st>>>(
            mAh, mAl, mBh, mBl, P);
    else if (f16 && (T + 2) * N <= 240 && getenv("VFMM_M2L_AST3"))  // three operator stages
        m2l_tc_kernel<true, 1, false, 3><<<grid, tc_threads<false>(), tc_smem<1, false, 3>(), st>>>(
            mAh, mAl, mBh, mBl, P);
    else if (f16)
        m2l_tc_kernel<true, 1><<<grid, tc_threads<false>(), tc_smem<1>(), st>>>(mAh, mAl, mBh, mBl, P);
    else
        m2l_tc_kernel<false, 1><<<grid, tc_threads<false>(), tc_smem<1>(), st>>>(mAh, mAl, mBh, mBl, P);
    return 0;
}

}  // namespace vfmm
