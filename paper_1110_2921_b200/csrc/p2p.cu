// p2p.cu -- exact near field ("calculated by solving Eq. (5) exactly") and
// the all-pairs DIRECT test mode.  FP32 FMA/SFU pipes (the paper runs FP32).
//
// Per ordered pair (target i, source j), d = x_i - x_j (periodic image), r = |d|:
//   f = g(r) / (4 pi r^3),        g = erf(rho) - 2/sqrt(pi) rho e^{-rho^2}, rho = r/(sqrt2 sigma)
//   q = f'/r = (zeta - 3 f)/r^2,  zeta = (2 pi sigma^2)^{-3/2} e^{-rho^2}
//   u_i += f (gamma_j x d)                                        Eq. (5)
//   classical: A_i += f gamma_j, B_i += q (gamma_i . d)(gamma_j x d);
//              sdot_i = A_i x gamma_i + B_i                          Eq. (8)
//   transpose: B_i += q (gamma_i . (gamma_j x d)) d; sdot_i = gamma_i x A_i + B_i
// rho^2 < 1/4: Taylor series in rho^2 (exact r -> 0 limits, no cancellation);
// otherwise 1 - g = e^{-rho^2} (erfcx(rho) + 2 rho/sqrt(pi)) with erfcx from a degree-4
// polynomial in t = 1/(1 + rho/2) (scripts/fit_cutoff_poly.py): 3 MUFU (rsqrt, ex2, rcp).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "vfmm_internal.h"

namespace vfmm {

// erfcx(rho) / (4 pi) ~= sum_k ERFCX_Ck t^k, t = 1/(1 + rho/2), degree 4
// (scripts/fit_cutoff_poly.py 4: relative error of g <= 4.8e-7 over rho in [0.5, 10], below
// the 1.4e-6 FP32 evaluation floor near rho = 0.5; degree 5 reached 1.6e-8 for one more FFMA2)
constexpr float ERFCX_C0 = -2.582819305e-03f, ERFCX_C1 = 4.079926104e-02f,
                ERFCX_C2 = -2.760024571e-02f, ERFCX_C3 = 8.149271438e-02f,
                ERFCX_C4 = -1.250394818e-02f;

KernelConsts make_kernel_consts(float sigma) {
    const double s = (double)sigma;
    KernelConsts k;
    k.inv2s2 = (float)(1.0 / (2.0 * s * s));
    k.neg_l2e_inv2s2 = (float)(-1.4426950408889634 / (2.0 * s * s));
    k.inv_s_sqrt2 = (float)(1.0 / (std::sqrt(2.0) * s));
    const double z0 = std::pow(2.0 * M_PI * s * s, -1.5);
    k.zeta0 = (float)z0;
    k.zeta0_over_s2 = (float)(z0 / (s * s));
    k.r2_series = (float)(0.5 * s * s);
    k.t_scale = (float)(1.0 / (2.0 * std::sqrt(2.0) * s));
    k.q_scale = (float)(2.0 / (4.0 * M_PI * std::sqrt(M_PI)) / (std::sqrt(2.0) * s));
    // packed path: the erfcx/(4 pi) polynomial (ERFCX_C0..4, ascending in t) scaled by -1/zeta0
    // (folds the zeta0 factor of the exponential into the ex2 argument and a negation)
    k.ez_off = (float)std::log2(z0);
    k.qn_scale = (float)(-(2.0 / (4.0 * M_PI * std::sqrt(M_PI)) / (std::sqrt(2.0) * s)) / z0);
    const float c[5] = {ERFCX_C0, ERFCX_C1, ERFCX_C2, ERFCX_C3, ERFCX_C4};
    for (int i = 0; i < 5; ++i) k.en[i] = (float)(-(double)c[i] / z0);
    k.en[5] = 0.f;  // unused (degree 4)
    return k;
}

namespace {

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct Acc {
    float u0, u1, u2, a0, a1, a2, b0, b1, b2;
};

// ---- packed FP32x2 (Blackwell FFMA2 / FMUL2 / FADD2): lane's two targets in .lo / .hi ----
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2 bc(float a) { return pk(a, a); }
__device__ __forceinline__ void upk(f2 v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
struct Acc2 {
    f2 u0, u1, u2, a0, a1, a2, b0, b1, b2;
};
// classical scheme with source cross products s_j = gamma_j x x_j staged per source: with
// d = x_i - x_j, sum f (gamma_j x d) = A x x_i - V and sum w (gamma_j x d) = Wg x x_i - Ws,
// so no per-pair cross product is formed (A = sum f gamma_j, V = sum f s_j, Wg = sum w gamma_j,
// Ws = sum w s_j, w = q (gamma_i . d))
struct Acc2S {
    f2 a0, a1, a2, v0, v1, v2, wg0, wg1, wg2, ws0, ws1, ws2;
};

// f, q by the Taylor series (rho^2 < 1/4, incl. r = 0)
__device__ __forceinline__ void fq_series(float r2, const KernelConsts& kc, float& f, float& q) {
    // f = zeta0 sum (-s)^k/(k!(2k+3)),  q = zeta0/sigma^2 sum_{k>=1} (-1)^k s^{k-1}/((k-1)!(2k+3))
    const float s = r2 * kc.inv2s2;  // rho^2
    float pf = 1.f / 10800.f;
    pf = fmaf(pf, s, -1.f / 1560.f);
    pf = fmaf(pf, s, 1.f / 264.f);
    pf = fmaf(pf, s, -1.f / 54.f);
    pf = fmaf(pf, s, 1.f / 14.f);
    pf = fmaf(pf, s, -1.f / 5.f);
    pf = fmaf(pf, s, 1.f / 3.f);
    float pq = -1.f / 12240.f;
    pq = fmaf(pq, s, 1.f / 1800.f);
    pq = fmaf(pq, s, -1.f / 312.f);
    pq = fmaf(pq, s, 1.f / 66.f);
    pq = fmaf(pq, s, -1.f / 18.f);
    pq = fmaf(pq, s, 1.f / 7.f);
    pq = fmaf(pq, s, -1.f / 5.f);
    f = kc.zeta0 * pf;
    q = kc.zeta0_over_s2 * pq;
}

// f, q in closed form (rho^2 >= 1/4): (1/4pi)(1 - g) = e^{-rho^2} (erfcx(rho) + 2 rho/sqrt(pi))/(4pi)
__device__ __forceinline__ void fq_closed(float r2, const KernelConsts& kc, float& f, float& q) {
    const float rinv = rsqrt_approx(r2);
    const float e = ex2_approx(r2 * kc.neg_l2e_inv2s2);
    const float r = r2 * rinv;
    const float t = rcp_approx(fmaf(kc.t_scale, r, 1.f));
    float E = ERFCX_C4;  // erfcx(rho)/(4 pi), polynomial in t
    E = fmaf(E, t, ERFCX_C3);
    E = fmaf(E, t, ERFCX_C2);
    E = fmaf(E, t, ERFCX_C1);
    E = fmaf(E, t, ERFCX_C0);
    const float Q = fmaf(kc.q_scale, r, E);
    const float g4pi = fmaf(-e, Q, 0.0795774715459476679f);  // g / (4 pi)
    const float rinv2 = rinv * rinv;
    f = g4pi * (rinv2 * rinv);
    q = fmaf(kc.zeta0, e, -3.f * f) * rinv2;
}

// f, q for two pairs at once (closed form), in the scaled form of KernelConsts::en:
//   e_z = zeta0 e^{-rho^2},  f = (1/(4 pi) + e_z Qn) / r^3,  q = (e_z - 3 f) / r^2
__device__ __forceinline__ void fq_closed2(f2 r2, const KernelConsts& kc, f2& f, f2& q) {
    float ra, rb;
    upk(r2, ra, rb);
    const f2 rinv = pk(rsqrt_approx(ra), rsqrt_approx(rb));
    float ea, eb;
    upk(fma2(r2, bc(kc.neg_l2e_inv2s2), bc(kc.ez_off)), ea, eb);
    const f2 ez = pk(ex2_approx(ea), ex2_approx(eb));
    const f2 r = mul2(r2, rinv);
    float da, db;
    upk(fma2(r, bc(kc.t_scale), bc(1.f)), da, db);
    const f2 t = pk(rcp_approx(da), rcp_approx(db));
    // Horner (Estrin's depth-3 form measured 4% slower for its extra instruction)
    f2 E = fma2(bc(kc.en[4]), t, bc(kc.en[3]));
    E = fma2(E, t, bc(kc.en[2]));
    E = fma2(E, t, bc(kc.en[1]));
    E = fma2(E, t, bc(kc.en[0]));
    const f2 Qn = fma2(bc(kc.qn_scale), r, E);
    const f2 g4pi = fma2(ez, Qn, bc(0.0795774715459476679f));  // g / (4 pi)
    const f2 rinv2 = mul2(rinv, rinv);
    f = mul2(g4pi, mul2(rinv2, rinv));
    q = mul2(fma2(bc(-3.f), f, ez), rinv2);
}

// c = gamma_j x d with the negated products folded into FMUL2 operand modifiers
__device__ __forceinline__ void cross2(float gjx, float gjy, float gjz, f2 dx, f2 dy, f2 dz,
                                       f2& cx, f2& cy, f2& cz) {
    cx = fma2(bc(gjy), dz, mul2(bc(-gjz), dy));
    cy = fma2(bc(gjz), dx, mul2(bc(-gjx), dz));
    cz = fma2(bc(gjx), dy, mul2(bc(-gjy), dx));
}

template <int SCHEME>
__device__ __forceinline__ void accumulate2(f2 dx, f2 dy, f2 dz, f2 f, f2 q, float gjx,
                                            float gjy, float gjz, f2 gix, f2 giy, f2 giz,
                                            Acc2& acc) {
    f2 cx, cy, cz;  // gamma_j x d
    cross2(gjx, gjy, gjz, dx, dy, dz, cx, cy, cz);
    acc.u0 = fma2(f, cx, acc.u0);
    acc.u1 = fma2(f, cy, acc.u1);
    acc.u2 = fma2(f, cz, acc.u2);
    acc.a0 = fma2(f, bc(gjx), acc.a0);
    acc.a1 = fma2(f, bc(gjy), acc.a1);
    acc.a2 = fma2(f, bc(gjz), acc.a2);
    if (SCHEME == 0) {
        const f2 w = mul2(q, fma2(gix, dx, fma2(giy, dy, mul2(giz, dz))));
        acc.b0 = fma2(w, cx, acc.b0);
        acc.b1 = fma2(w, cy, acc.b1);
        acc.b2 = fma2(w, cz, acc.b2);
    } else {
        const f2 w = mul2(q, fma2(gix, cx, fma2(giy, cy, mul2(giz, cz))));
        acc.b0 = fma2(w, dx, acc.b0);
        acc.b1 = fma2(w, dy, acc.b1);
        acc.b2 = fma2(w, dz, acc.b2);
    }
}

__device__ __forceinline__ void accumulate2s(f2 dx, f2 dy, f2 dz, f2 f, f2 q, float gjx,
                                             float gjy, float gjz, float sjx, float sjy,
                                             float sjz, f2 gix, f2 giy, f2 giz, Acc2S& acc) {
    acc.a0 = fma2(f, bc(gjx), acc.a0);
    acc.a1 = fma2(f, bc(gjy), acc.a1);
    acc.a2 = fma2(f, bc(gjz), acc.a2);
    acc.v0 = fma2(f, bc(sjx), acc.v0);
    acc.v1 = fma2(f, bc(sjy), acc.v1);
    acc.v2 = fma2(f, bc(sjz), acc.v2);
    const f2 w = mul2(q, fma2(gix, dx, fma2(giy, dy, mul2(giz, dz))));
    acc.wg0 = fma2(w, bc(gjx), acc.wg0);
    acc.wg1 = fma2(w, bc(gjy), acc.wg1);
    acc.wg2 = fma2(w, bc(gjz), acc.wg2);
    acc.ws0 = fma2(w, bc(sjx), acc.ws0);
    acc.ws1 = fma2(w, bc(sjy), acc.ws1);
    acc.ws2 = fma2(w, bc(sjz), acc.ws2);
}

template <int SCHEME>
__device__ __forceinline__ void accumulate(float dx, float dy, float dz, float f, float q,
                                           float gjx, float gjy, float gjz, float gix, float giy,
                                           float giz, Acc& acc) {
    // c = gamma_j x d
    const float cx = fmaf(gjy, dz, -gjz * dy);
    const float cy = fmaf(gjz, dx, -gjx * dz);
    const float cz = fmaf(gjx, dy, -gjy * dx);
    acc.u0 = fmaf(f, cx, acc.u0);
    acc.u1 = fmaf(f, cy, acc.u1);
    acc.u2 = fmaf(f, cz, acc.u2);
    acc.a0 = fmaf(f, gjx, acc.a0);
    acc.a1 = fmaf(f, gjy, acc.a1);
    acc.a2 = fmaf(f, gjz, acc.a2);
    if (SCHEME == 0) {
        const float w = q * fmaf(gix, dx, fmaf(giy, dy, giz * dz));
        acc.b0 = fmaf(w, cx, acc.b0);
        acc.b1 = fmaf(w, cy, acc.b1);
        acc.b2 = fmaf(w, cz, acc.b2);
    } else {
        const float w = q * fmaf(gix, cx, fmaf(giy, cy, giz * cz));
        acc.b0 = fmaf(w, dx, acc.b0);
        acc.b1 = fmaf(w, dy, acc.b1);
        acc.b2 = fmaf(w, dz, acc.b2);
    }
}

template <int SCHEME>
__device__ __forceinline__ void pair(float dx, float dy, float dz, float gjx, float gjy, float gjz,
                                     float gix, float giy, float giz, const KernelConsts& kc,
                                     Acc& acc) {
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    float f, q;
    if (r2 < kc.r2_series) fq_series(r2, kc, f, q);
    else fq_closed(r2, kc, f, q);
    accumulate<SCHEME>(dx, dy, dz, f, q, gjx, gjy, gjz, gix, giy, giz, acc);
}

template <int SCHEME>
__device__ __forceinline__ void finish(const Acc& a, float gx, float gy, float gz, float out[6]) {
    out[0] = a.u0;
    out[1] = a.u1;
    out[2] = a.u2;
    if (SCHEME == 0) {  // A x gamma_i + B
        out[3] = fmaf(a.a1, gz, -a.a2 * gy) + a.b0;
        out[4] = fmaf(a.a2, gx, -a.a0 * gz) + a.b1;
        out[5] = fmaf(a.a0, gy, -a.a1 * gx) + a.b2;
    } else {  // gamma_i x A + B
        out[3] = fmaf(gy, a.a2, -gz * a.a1) + a.b0;
        out[4] = fmaf(gz, a.a0, -gx * a.a2) + a.b1;
        out[5] = fmaf(gx, a.a1, -gy * a.a0) + a.b2;
    }
}

__device__ __forceinline__ uint32_t spread3p(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ uint32_t compact3p(uint32_t v) {
    v &= 0x09249249u;
    v = (v ^ (v >> 2)) & 0x030C30C3u;
    v = (v ^ (v >> 4)) & 0x0300F00Fu;
    v = (v ^ (v >> 8)) & 0x030000FFu;
    v = (v ^ (v >> 16)) & 0x000003FFu;
    return v;
}

// One block (256 threads = 8 warps) per level-(L-1) cell: its 8 child leaves are the
// targets (warp w <-> child w, 2 targets per lane), the 4x4x4 leaves around them are the
// sources, staged once in shared memory (x, y, z, gx | gy, gz), positions relative to the
// parent-cell centre: s = d_j + (r - 3/2) a, t = d_i + (b - 1/2) a, exact leaf-centre
// offsets (reading R8).  If the 64 source leaves exceed the shared-memory capacity they are
// staged in passes of consecutive region leaves.
constexpr int P2P_THREADS = 256;
// sources per pass at 2 blocks / SM: 24 B per source (x y z gx | gy gz) or, with the staged
// cross products, 36 B (x y z gx | gy gz sx sy | sz)
// MINB = 1: the lean variant (2 blocks / SM on their own, 2560 sources = 61.5 KB of shared
// memory so one block fits beside a lean tensor-core M2L block, capi.cu co-resident mode)
template <bool SJ, int MINB = 2> constexpr int p2p_cap() {
    return MINB == 1 ? (SJ ? 1664 : 2560) : MINB >= 3 ? (SJ ? 1920 : 2816) : (SJ ? 3072 : 4352);
}
constexpr int P2P_PAD = 4;     // slack after each staged array (keeps the arrays 16-byte aligned)

// SJ (classical scheme only): accumulate with the staged source cross products s_j (Acc2S:
// 38 instead of 41 FP32 instructions per pair, rounding ~1.4x larger since the sums carry
// |x_j| instead of |d|); otherwise the per-pair cross product gamma_j x d
template <int SCHEME, bool SJ, int MINB = 2, int UNR = 2>
__global__ void __launch_bounds__(P2P_THREADS, MINB == 1 ? 2 : MINB) p2p_kernel(
    const float* __restrict__ s6, int64_t n, const int* __restrict__ leaf_start, int depth,
    float a, int periodic, KernelConsts kc, float* __restrict__ near6,
    unsigned long long* __restrict__ npairs, int64_t plo) {
    extern __shared__ float4 p2p_sm[];
    constexpr int P2P_CAP = p2p_cap<SJ, MINB>();
    float4* S4 = p2p_sm;                         // x, y, z, gx
    // SJ: gy, gz, sx, sy (s_j = gamma_j x x_j) and sz; else gy, gz
    float4* S4b = S4 + P2P_CAP + P2P_PAD;
    float* S1 = reinterpret_cast<float*>(S4b + P2P_CAP + P2P_PAD);
    float2* S2 = reinterpret_cast<float2*>(S4 + P2P_CAP + P2P_PAD);
    __shared__ int rstart[65], rend[64], rcnt[64], rsrc[64];
    __shared__ int wsplit;
    // bounding box of each staged leaf's real sources in the current window (min xyz, max xyz):
    // a target chunk and a source leaf whose boxes are further apart than the series threshold
    // have no close pair, so that leaf runs the pair loop without the per-iteration test
    __shared__ float sbox[64][6];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t parent = (uint32_t)(plo + blockIdx.x);
    const int side = 1 << depth;
    const int px = (int)compact3p(parent), py = (int)compact3p(parent >> 1),
              pz = (int)compact3p(parent >> 2);
    // ---- region table: leaf (rx,ry,rz) in [0,4)^3 <-> global (2p - 1 + r) ----
    if (tid < 64) {
        const int rx = tid & 3, ry = (tid >> 2) & 3, rz = tid >> 4;
        int gx = 2 * px - 1 + rx, gy = 2 * py - 1 + ry, gz = 2 * pz - 1 + rz;
        int cnt = 0, st = 0;
        if (periodic || (gx >= 0 && gx < side && gy >= 0 && gy < side && gz >= 0 && gz < side)) {
            gx &= side - 1;
            gy &= side - 1;
            gz &= side - 1;
            const uint32_t lf = spread3p(gx) | (spread3p(gy) << 1) | (spread3p(gz) << 2);
            st = leaf_start[lf];
            cnt = leaf_start[lf + 1] - st;
        }
        rcnt[tid] = cnt;
        rsrc[tid] = st;
    }
    __syncthreads();
    if (tid == 0) {  // staged offsets: every leaf padded to an even count (see staging)
        // z-layers in the order 1, 2, 0, 3: every warp's 27 neighbours span the two middle
        // layers plus one outer layer, so a region staged in two windows (middle | outer)
        // gives every warp 18 + 9 leaves -- balanced windows, short barrier waits
        int run = 0;
        for (int li = 0; li < 4; ++li) {
            const int rz = li == 0 ? 1 : li == 1 ? 2 : li == 2 ? 0 : 3;
            if (li == 2) wsplit = run;
            for (int i = 16 * rz; i < 16 * rz + 16; ++i) {
                rstart[i] = run;
                run += (rcnt[i] + 1) & ~1;
                rend[i] = run;
            }
        }
        rstart[64] = run;
    }
    __syncthreads();
    // ---- this warp's target leaf (child w of the parent) ----
    const int bx = w & 1, by = (w >> 1) & 1, bz = (w >> 2) & 1;
    const uint32_t tleaf = (parent << 3) | (uint32_t)w;
    const int ts = leaf_start[tleaf], te = leaf_start[tleaf + 1];
    const float tox = (bx - 0.5f) * a, toy = (by - 0.5f) * a, toz = (bz - 0.5f) * a;
    const int total = rstart[64];
    if (lane == 0) {  // ordered near-field pairs of this warp's leaf (stats)
        int ns = 0;
        for (int nb = 0; nb < 27; ++nb)
            ns += rcnt[(bx + nb % 3) + 4 * (by + (nb / 3) % 3) + 16 * (bz + nb / 9)];
        if (te > ts) atomicAdd(npairs, (unsigned long long)(te - ts) * (unsigned long long)ns);
    }
    // target chunks of 64 (2 per lane) -- loop outermost only when a leaf has > 64 particles
    const int nchunk = (te - ts + 63) / 64;
    // all warps must take part in every staging pass: iterate chunks up to the block max
    __shared__ int maxchunk;
    if (tid == 0) maxchunk = 0;
    __syncthreads();
    atomicMax(&maxchunk, nchunk);
    __syncthreads();
    const int nch = maxchunk;
    for (int ch = 0; ch < nch; ++ch) {
        const int i0 = ts + ch * 64 + lane, i1 = i0 + 32;
        const bool a0 = i0 < te, a1 = i1 < te;
        float x0 = 0, y0 = 0, z0 = 0, g0x = 0, g0y = 0, g0z = 0;
        float x1 = 0, y1 = 0, z1 = 0, g1x = 0, g1y = 0, g1z = 0;
        if (a0) {
            x0 = s6[i0] + tox; y0 = s6[n + i0] + toy; z0 = s6[2 * n + i0] + toz;
            g0x = s6[3 * n + i0]; g0y = s6[4 * n + i0]; g0z = s6[5 * n + i0];
        }
        if (a1) {
            x1 = s6[i1] + tox; y1 = s6[n + i1] + toy; z1 = s6[2 * n + i1] + toz;
            g1x = s6[3 * n + i1]; g1y = s6[4 * n + i1]; g1z = s6[5 * n + i1];
        }
        // the warp's target box (warp-uniform after the reduction)
        float tb[6];
        tb[0] = fminf(a0 ? x0 : 1e30f, a1 ? x1 : 1e30f);
        tb[1] = fminf(a0 ? y0 : 1e30f, a1 ? y1 : 1e30f);
        tb[2] = fminf(a0 ? z0 : 1e30f, a1 ? z1 : 1e30f);
        tb[3] = fmaxf(a0 ? x0 : -1e30f, a1 ? x1 : -1e30f);
        tb[4] = fmaxf(a0 ? y0 : -1e30f, a1 ? y1 : -1e30f);
        tb[5] = fmaxf(a0 ? z0 : -1e30f, a1 ? z1 : -1e30f);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                tb[c] = fminf(tb[c], __shfl_xor_sync(0xffffffffu, tb[c], o));
                tb[c + 3] = fmaxf(tb[c + 3], __shfl_xor_sync(0xffffffffu, tb[c + 3], o));
            }
        }
        // targets (i0, i1) packed in the two halves of f2 registers
        const f2 X = pk(x0, x1), Y = pk(y0, y1), Z = pk(z0, z1);
        const f2 GX = pk(g0x, g1x), GY = pk(g0y, g1y), GZ = pk(g0z, g1z);
        const f2 z2 = pk(0.f, 0.f);
        Acc2 C = {z2, z2, z2, z2, z2, z2, z2, z2, z2};
        Acc2S CS = {z2, z2, z2, z2, z2, z2, z2, z2, z2, z2, z2, z2};
        const f2 thr = bc(kc.r2_series);
        (void)thr;
        // windows [w0, w1) of the concatenated region sources, P2P_CAP at a time (a warp idle
        // at a window barrier leaves the pipes to the SM's other block; balanced two-phase
        // staging by source layers measured 1.5% slower for its 25% extra staging)
        // windows: the whole region, or middle | outer layers when each fits, else P2P_CAP
        // chunks (dense leaves)
        const bool split2 = total > P2P_CAP && wsplit <= P2P_CAP && total - wsplit <= P2P_CAP;
        for (int w0 = 0, w1 = 0; w0 < total; w0 = w1) {
            w1 = split2 ? (w0 == 0 ? wsplit : total) : min(w0 + P2P_CAP, total);
            __syncthreads();
            for (int rl = w; rl < 64; rl += P2P_THREADS / 32) {
                const int lo = max(rstart[rl], w0), hi = min(rend[rl], w1);
                if (lo >= hi) continue;
                const int src = rsrc[rl] + (lo - rstart[rl]);
                const float ox = ((rl & 3) - 1.5f) * a, oy = (((rl >> 2) & 3) - 1.5f) * a,
                            oz = ((rl >> 4) - 1.5f) * a;
                float bmin[3] = {1e30f, 1e30f, 1e30f}, bmax[3] = {-1e30f, -1e30f, -1e30f};
                for (int k = lane; k < hi - lo; k += 32) {
                    // an odd leaf ends with a padding source: far away, zero strength (exact 0
                    // contribution), so the pair loop runs over whole pairs of sources
                    const int j = src + k;
                    const bool real = lo - rstart[rl] + k < rcnt[rl];
                    const float x = real ? s6[j] + ox : 1e4f, y = real ? s6[n + j] + oy : 1e4f,
                                z = real ? s6[2 * n + j] + oz : 1e4f;
                    if (real) {
                        bmin[0] = fminf(bmin[0], x);
                        bmin[1] = fminf(bmin[1], y);
                        bmin[2] = fminf(bmin[2], z);
                        bmax[0] = fmaxf(bmax[0], x);
                        bmax[1] = fmaxf(bmax[1], y);
                        bmax[2] = fmaxf(bmax[2], z);
                    }
                    const float gx = real ? s6[3 * n + j] : 0.f, gy = real ? s6[4 * n + j] : 0.f,
                                gz = real ? s6[5 * n + j] : 0.f;
                    S4[lo - w0 + k] = make_float4(x, y, z, gx);
                    if (SJ) {
                        S4b[lo - w0 + k] = make_float4(gy, gz, gy * z - gz * y, gz * x - gx * z);
                        S1[lo - w0 + k] = gx * y - gy * x;
                    } else {
                        S2[lo - w0 + k] = make_float2(gy, gz);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        bmin[c] = fminf(bmin[c], __shfl_xor_sync(0xffffffffu, bmin[c], o));
                        bmax[c] = fmaxf(bmax[c], __shfl_xor_sync(0xffffffffu, bmax[c], o));
                    }
                }
                if (lane == 0) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        sbox[rl][c] = bmin[c];
                        sbox[rl][c + 3] = bmax[c];
                    }
                }
            }
            __syncthreads();
            for (int nb = 0; nb < 27; ++nb) {
                const int rx = bx + nb % 3, ry = by + (nb / 3) % 3, rz = bz + nb / 9;
                const int rl = rx + 4 * ry + 16 * rz;
                const int js = max(rstart[rl], w0) - w0, je = min(rend[rl], w1) - w0;
                if (js >= je) continue;  // leaf not in this window
                // two sources per iteration; each source x two targets = one packed pair
                // (SJ: the 4-wide second record; else the 2-wide one, zero-extended).  Loads
                // are left to the compiler's schedule (an explicit one-iteration prefetch
                // measured 43.5 vs 43.1 ms)
                auto rec2 = [&](int jj) {
                    if (SJ) return S4b[jj];
                    const float2 t = S2[jj];
                    return make_float4(t.x, t.y, 0.f, 0.f);
                };
                // the source leaf's box apart from the target box by more than the series
                // threshold: no close pair, no per-iteration test (warp-uniform decision)
                const float th = kc.r2_series;
                const float gx_ = fmaxf(0.f, fmaxf(sbox[rl][0] - tb[3], tb[0] - sbox[rl][3]));
                const float gy_ = fmaxf(0.f, fmaxf(sbox[rl][1] - tb[4], tb[1] - sbox[rl][4]));
                const float gz_ = fmaxf(0.f, fmaxf(sbox[rl][2] - tb[5], tb[2] - sbox[rl][5]));
                const bool apart = gx_ * gx_ + gy_ * gy_ + gz_ * gz_ >= th;
                auto pairs = [&](auto check_tag) {
                constexpr bool CHECK = decltype(check_tag)::value;
                // unrolled by 2 (c4 P2P: 43.1 ms; 49.6 without unrolling, 44.0 unrolled by 4)
#pragma unroll UNR
                for (int j = js; j < je; j += 2) {  // js, je even (padded leaves, even CAP)
                    const float4 pa = S4[j];
                    const float4 qa = rec2(j);
                    const float4 pb = S4[j + 1];
                    const float4 qb = rec2(j + 1);
                    const float sza = SJ ? S1[j] : 0.f, szb = SJ ? S1[j + 1] : 0.f;
                    const float gbx = pb.w;
                    const f2 dxa = sub2(X, bc(pa.x)), dya = sub2(Y, bc(pa.y)), dza = sub2(Z, bc(pa.z));
                    const f2 dxb = sub2(X, bc(pb.x)), dyb = sub2(Y, bc(pb.y)), dzb = sub2(Z, bc(pb.z));
                    const f2 r2a = fma2(dxa, dxa, fma2(dya, dya, mul2(dza, dza)));
                    const f2 r2b = fma2(dxb, dxb, fma2(dyb, dyb, mul2(dzb, dzb)));
                    float ra0, ra1, rb0, rb1;
                    upk(r2a, ra0, ra1);
                    upk(r2b, rb0, rb1);
                    const bool close = CHECK && ((a0 && (ra0 < th || rb0 < th)) ||
                                                 (a1 && (ra1 < th || rb1 < th)));
                    f2 fa, qa2, fb, qb2;
                    if (!CHECK) {
                        fq_closed2(r2a, kc, fa, qa2);
                        fq_closed2(r2b, kc, fb, qb2);
                    } else if (SJ) {
                        // closed form for all pairs, outside the branch (schedules with the
                        // other unrolled iteration); the rare close pairs (self pairs, rho^2 <
                        // 1/4) then get the Taylor series in place (41.9 ms; 42.7 with the
                        // cross variant's form below)
                        fq_closed2(r2a, kc, fa, qa2);
                        fq_closed2(r2b, kc, fb, qb2);
                        if (__any_sync(0xffffffffu, close)) {
                            float f0, q0, f1, q1;
                            upk(fa, f0, f1);
                            upk(qa2, q0, q1);
                            if (ra0 < th) fq_series(ra0, kc, f0, q0);
                            if (ra1 < th) fq_series(ra1, kc, f1, q1);
                            fa = pk(f0, f1);
                            qa2 = pk(q0, q1);
                            upk(fb, f0, f1);
                            upk(qb2, q0, q1);
                            if (rb0 < th) fq_series(rb0, kc, f0, q0);
                            if (rb1 < th) fq_series(rb1, kc, f1, q1);
                            fb = pk(f0, f1);
                            qb2 = pk(q0, q1);
                        }
                    } else if (__any_sync(0xffffffffu, close)) {
                        // rare path (self pairs, close particles): per pair, series or closed
                        // form (this branch form schedules best for the cross variant: 43.1 ms)
                        float f0, q0, f1, q1;
                        if (ra0 < th) fq_series(ra0, kc, f0, q0); else fq_closed(ra0, kc, f0, q0);
                        if (ra1 < th) fq_series(ra1, kc, f1, q1); else fq_closed(ra1, kc, f1, q1);
                        fa = pk(f0, f1);
                        qa2 = pk(q0, q1);
                        if (rb0 < th) fq_series(rb0, kc, f0, q0); else fq_closed(rb0, kc, f0, q0);
                        if (rb1 < th) fq_series(rb1, kc, f1, q1); else fq_closed(rb1, kc, f1, q1);
                        fb = pk(f0, f1);
                        qb2 = pk(q0, q1);
                    } else {
                        fq_closed2(r2a, kc, fa, qa2);
                        fq_closed2(r2b, kc, fb, qb2);
                    }
                    if (SJ) {
                        accumulate2s(dxa, dya, dza, fa, qa2, pa.w, qa.x, qa.y, qa.z, qa.w, sza, GX,
                                     GY, GZ, CS);
                        accumulate2s(dxb, dyb, dzb, fb, qb2, gbx, qb.x, qb.y, qb.z, qb.w, szb, GX,
                                     GY, GZ, CS);
                    } else {
                        accumulate2<SCHEME>(dxa, dya, dza, fa, qa2, pa.w, qa.x, qa.y, GX, GY, GZ, C);
                        accumulate2<SCHEME>(dxb, dyb, dzb, fb, qb2, gbx, qb.x, qb.y, GX, GY, GZ, C);
                    }
                }
                };
                if (apart) pairs(std::false_type{});
                else pairs(std::true_type{});
            }
        }
        if (SJ) {  // u = A x x_i - V, B = Wg x x_i - Ws
            C.a0 = CS.a0;
            C.a1 = CS.a1;
            C.a2 = CS.a2;
            C.u0 = sub2(sub2(mul2(CS.a1, Z), mul2(CS.a2, Y)), CS.v0);
            C.u1 = sub2(sub2(mul2(CS.a2, X), mul2(CS.a0, Z)), CS.v1);
            C.u2 = sub2(sub2(mul2(CS.a0, Y), mul2(CS.a1, X)), CS.v2);
            C.b0 = sub2(sub2(mul2(CS.wg1, Z), mul2(CS.wg2, Y)), CS.ws0);
            C.b1 = sub2(sub2(mul2(CS.wg2, X), mul2(CS.wg0, Z)), CS.ws1);
            C.b2 = sub2(sub2(mul2(CS.wg0, Y), mul2(CS.wg1, X)), CS.ws2);
        }
        Acc c0, c1;
        upk(C.u0, c0.u0, c1.u0);
        upk(C.u1, c0.u1, c1.u1);
        upk(C.u2, c0.u2, c1.u2);
        upk(C.a0, c0.a0, c1.a0);
        upk(C.a1, c0.a1, c1.a1);
        upk(C.a2, c0.a2, c1.a2);
        upk(C.b0, c0.b0, c1.b0);
        upk(C.b1, c0.b1, c1.b1);
        upk(C.b2, c0.b2, c1.b2);
        float o[6];
        if (a0) {
            finish<SCHEME>(c0, g0x, g0y, g0z, o);
#pragma unroll
            for (int k = 0; k < 6; ++k) near6[k * n + i0] = o[k];
        }
        if (a1) {
            finish<SCHEME>(c1, g1x, g1y, g1z, o);
#pragma unroll
            for (int k = 0; k < 6; ++k) near6[k * n + i1] = o[k];
        }
    }
}

// ---- per-particle core radius sigma_j (Eq. 6 as written: the source's sigma, NEXT-4) ----
// With rt = r / sigma_j, rho = rt / sqrt2 and ez' = zeta0(1) e^{-rho^2} (sigma-independent
// offset), the closed form of fq_closed2 becomes f = (1/4pi + ez' Qn(rt)) / r^3 with the
// sigma = 1 polynomial (kc1: make_kernel_consts(1)), q = (ez' / sigma_j^3 - 3 f) / r^2.
// Per source staged: c_j = -log2(e) / (2 sigma_j^2), 1/sigma_j, 1/sigma_j^3, sigma_j^2 / 2.
__device__ __forceinline__ void fq_closed2_sig(f2 r2, float cj, float isig, float isig3,
                                               const KernelConsts& kc1, f2& f, f2& q) {
    float ra, rb;
    upk(r2, ra, rb);
    const f2 rinv = pk(rsqrt_approx(ra), rsqrt_approx(rb));
    float ea, eb;
    upk(fma2(r2, bc(cj), bc(kc1.ez_off)), ea, eb);
    const f2 ez = pk(ex2_approx(ea), ex2_approx(eb));
    const f2 rt = mul2(mul2(r2, rinv), bc(isig));
    float da, db;
    upk(fma2(rt, bc(kc1.t_scale), bc(1.f)), da, db);
    const f2 t = pk(rcp_approx(da), rcp_approx(db));
    f2 E = fma2(bc(kc1.en[4]), t, bc(kc1.en[3]));
    E = fma2(E, t, bc(kc1.en[2]));
    E = fma2(E, t, bc(kc1.en[1]));
    E = fma2(E, t, bc(kc1.en[0]));
    const f2 Qn = fma2(bc(kc1.qn_scale), rt, E);
    const f2 g4pi = fma2(ez, Qn, bc(0.0795774715459476679f));
    const f2 rinv2 = mul2(rinv, rinv);
    f = mul2(g4pi, mul2(rinv2, rinv));
    q = mul2(fma2(bc(-3.f), f, mul2(ez, bc(isig3))), rinv2);
}
// the Taylor series for rho^2 < 1/4 with sigma_j (exact r -> 0 limits)
__device__ __forceinline__ void fq_series_sig(float r2, float isig, float isig3,
                                              const KernelConsts& kc1, float& f, float& q) {
    KernelConsts k = kc1;  // sigma = 1 constants rescaled to sigma_j
    k.inv2s2 = 0.5f * isig * isig;
    k.zeta0 = kc1.zeta0 * isig3;
    k.zeta0_over_s2 = kc1.zeta0 * isig3 * isig * isig;
    fq_series(r2, k, f, q);
}

template <int SCHEME>
__global__ void __launch_bounds__(P2P_THREADS, 2) p2p_sig_kernel(
    const float* __restrict__ s6, const float* __restrict__ ssig, int64_t n,
    const int* __restrict__ leaf_start, int depth, float a, int periodic, KernelConsts kc1,
    float* __restrict__ near6, unsigned long long* __restrict__ npairs, int64_t plo) {
    constexpr int CAP = 1024;             // staged sources per window (40 B each)
    __shared__ float4 S4[CAP], S4b[CAP];  // (x, y, z, gx), (gy, gz, c_j, 1/sigma_j)
    extern __shared__ float2 p2ps_sm[];
    float2* S2 = p2ps_sm;                  // (1/sigma_j^3, sigma_j^2 / 2)
    __shared__ int rstart[65], rcnt[64], rsrc[64];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t parent = (uint32_t)(plo + blockIdx.x);
    const int side = 1 << depth;
    const int px = (int)compact3p(parent), py = (int)compact3p(parent >> 1),
              pz = (int)compact3p(parent >> 2);
    if (tid < 64) {
        const int rx = tid & 3, ry = (tid >> 2) & 3, rz = tid >> 4;
        int gx = 2 * px - 1 + rx, gy = 2 * py - 1 + ry, gz = 2 * pz - 1 + rz;
        int cnt = 0, st = 0;
        if (periodic || (gx >= 0 && gx < side && gy >= 0 && gy < side && gz >= 0 && gz < side)) {
            gx &= side - 1;
            gy &= side - 1;
            gz &= side - 1;
            const uint32_t lf = spread3p(gx) | (spread3p(gy) << 1) | (spread3p(gz) << 2);
            st = leaf_start[lf];
            cnt = leaf_start[lf + 1] - st;
        }
        rcnt[tid] = cnt;
        rsrc[tid] = st;
    }
    __syncthreads();
    if (tid == 0) {
        int run = 0;
        for (int i = 0; i < 64; ++i) {
            rstart[i] = run;
            run += rcnt[i];
        }
        rstart[64] = run;
    }
    __syncthreads();
    const int bx = w & 1, by = (w >> 1) & 1, bz = (w >> 2) & 1;
    const uint32_t tleaf = (parent << 3) | (uint32_t)w;
    const int ts = leaf_start[tleaf], te = leaf_start[tleaf + 1];
    const float tox = (bx - 0.5f) * a, toy = (by - 0.5f) * a, toz = (bz - 0.5f) * a;
    const int total = rstart[64];
    if (lane == 0) {
        int ns = 0;
        for (int nb = 0; nb < 27; ++nb)
            ns += rcnt[(bx + nb % 3) + 4 * (by + (nb / 3) % 3) + 16 * (bz + nb / 9)];
        if (te > ts) atomicAdd(npairs, (unsigned long long)(te - ts) * (unsigned long long)ns);
    }
    const int nchunk = (te - ts + 63) / 64;
    __shared__ int maxchunk;
    if (tid == 0) maxchunk = 0;
    __syncthreads();
    atomicMax(&maxchunk, nchunk);
    __syncthreads();
    const int nch = maxchunk;
    for (int ch = 0; ch < nch; ++ch) {
        const int i0 = ts + ch * 64 + lane, i1 = i0 + 32;
        const bool a0 = i0 < te, a1 = i1 < te;
        float x0 = 0, y0 = 0, z0 = 0, g0x = 0, g0y = 0, g0z = 0;
        float x1 = 0, y1 = 0, z1 = 0, g1x = 0, g1y = 0, g1z = 0;
        if (a0) {
            x0 = s6[i0] + tox; y0 = s6[n + i0] + toy; z0 = s6[2 * n + i0] + toz;
            g0x = s6[3 * n + i0]; g0y = s6[4 * n + i0]; g0z = s6[5 * n + i0];
        }
        if (a1) {
            x1 = s6[i1] + tox; y1 = s6[n + i1] + toy; z1 = s6[2 * n + i1] + toz;
            g1x = s6[3 * n + i1]; g1y = s6[4 * n + i1]; g1z = s6[5 * n + i1];
        }
        const f2 X = pk(x0, x1), Y = pk(y0, y1), Z = pk(z0, z1);
        const f2 GX = pk(g0x, g1x), GY = pk(g0y, g1y), GZ = pk(g0z, g1z);
        const f2 z2 = pk(0.f, 0.f);
        Acc2 C = {z2, z2, z2, z2, z2, z2, z2, z2, z2};
        for (int w0 = 0; w0 < total; w0 += CAP) {
            const int w1 = min(w0 + CAP, total);
            __syncthreads();
            for (int rl = w; rl < 64; rl += P2P_THREADS / 32) {
                const int lo = max(rstart[rl], w0), hi = min(rstart[rl + 1], w1);
                if (lo >= hi) continue;
                const int src = rsrc[rl] + (lo - rstart[rl]);
                const float ox = ((rl & 3) - 1.5f) * a, oy = (((rl >> 2) & 3) - 1.5f) * a,
                            oz = ((rl >> 4) - 1.5f) * a;
                for (int k = lane; k < hi - lo; k += 32) {
                    const int j = src + k;
                    const float sg = ssig[j], isg = 1.f / sg;
                    S4[lo - w0 + k] = make_float4(s6[j] + ox, s6[n + j] + oy, s6[2 * n + j] + oz,
                                                  s6[3 * n + j]);
                    S4b[lo - w0 + k] = make_float4(s6[4 * n + j], s6[5 * n + j],
                                                   -1.4426950408889634f * 0.5f * isg * isg, isg);
                    S2[lo - w0 + k] = make_float2(isg * isg * isg, 0.5f * sg * sg);
                }
            }
            __syncthreads();
            for (int nb = 0; nb < 27; ++nb) {
                const int rx = bx + nb % 3, ry = by + (nb / 3) % 3, rz = bz + nb / 9;
                const int rl = rx + 4 * ry + 16 * rz;
                const int js = max(rstart[rl], w0) - w0, je = min(rstart[rl + 1], w1) - w0;
                for (int j = js; j < je; ++j) {
                    const float4 pa = S4[j], qa = S4b[j];
                    const float2 sa = S2[j];
                    const f2 dx = sub2(X, bc(pa.x)), dy = sub2(Y, bc(pa.y)), dz = sub2(Z, bc(pa.z));
                    const f2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
                    float r0, r1;
                    upk(r2, r0, r1);
                    f2 f, q;
                    const bool close = (a0 && r0 < sa.y) || (a1 && r1 < sa.y);
                    if (__any_sync(0xffffffffu, close)) {
                        float f0, q0, f1, q1;
                        fq_closed2_sig(r2, qa.z, qa.w, sa.x, kc1, f, q);
                        upk(f, f0, f1);
                        upk(q, q0, q1);
                        if (r0 < sa.y) fq_series_sig(r0, qa.w, sa.x, kc1, f0, q0);
                        if (r1 < sa.y) fq_series_sig(r1, qa.w, sa.x, kc1, f1, q1);
                        f = pk(f0, f1);
                        q = pk(q0, q1);
                    } else {
                        fq_closed2_sig(r2, qa.z, qa.w, sa.x, kc1, f, q);
                    }
                    accumulate2<SCHEME>(dx, dy, dz, f, q, pa.w, qa.x, qa.y, GX, GY, GZ, C);
                }
            }
        }
        Acc c0, c1;
        upk(C.u0, c0.u0, c1.u0);
        upk(C.u1, c0.u1, c1.u1);
        upk(C.u2, c0.u2, c1.u2);
        upk(C.a0, c0.a0, c1.a0);
        upk(C.a1, c0.a1, c1.a1);
        upk(C.a2, c0.a2, c1.a2);
        upk(C.b0, c0.b0, c1.b0);
        upk(C.b1, c0.b1, c1.b1);
        upk(C.b2, c0.b2, c1.b2);
        float o[6];
        if (a0) {
            finish<SCHEME>(c0, g0x, g0y, g0z, o);
#pragma unroll
            for (int k = 0; k < 6; ++k) near6[k * n + i0] = o[k];
        }
        if (a1) {
            finish<SCHEME>(c1, g1x, g1y, g1z, o);
#pragma unroll
            for (int k = 0; k < 6; ++k) near6[k * n + i1] = o[k];
        }
    }
}

// DIRECT mode with per-source sigma_j: scalar pair of the same building blocks
template <int SCHEME>
__global__ void __launch_bounds__(128) direct_sig_kernel(const float* __restrict__ pos,
                                                         const float* __restrict__ gam,
                                                         const float* __restrict__ sig,
                                                         int64_t n, double len, int m,
                                                         KernelConsts kc1,
                                                         float* __restrict__ vel,
                                                         float* __restrict__ dgam) {
    __shared__ double sx[128], sy[128], sz[128];
    __shared__ float sgx[128], sgy[128], sgz[128], ss[128];
    const int64_t i = blockIdx.x * (int64_t)128 + threadIdx.x;
    const bool act = i < n;
    double xi = 0, yi = 0, zi = 0;
    float gix = 0, giy = 0, giz = 0;
    if (act) {
        xi = pos[i];
        yi = pos[n + i];
        zi = pos[2 * n + i];
        gix = gam[i];
        giy = gam[n + i];
        giz = gam[2 * n + i];
    }
    double tot[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const int side = 2 * m + 1;
    for (int64_t sb = 0; sb < n; sb += 128) {
        __syncthreads();
        const int64_t j = sb + threadIdx.x;
        if (j < n) {
            sx[threadIdx.x] = pos[j];
            sy[threadIdx.x] = pos[n + j];
            sz[threadIdx.x] = pos[2 * n + j];
            sgx[threadIdx.x] = gam[j];
            sgy[threadIdx.x] = gam[n + j];
            sgz[threadIdx.x] = gam[2 * n + j];
            ss[threadIdx.x] = sig[j];
        }
        __syncthreads();
        const int cnt = (int)min((int64_t)128, n - sb);
        if (!act) continue;
        for (int im = 0; im < side * side * side; ++im) {
            const double shx = (im / (side * side) - m) * len;
            const double shy = ((im / side) % side - m) * len;
            const double shz = (im % side - m) * len;
            Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            for (int qq = 0; qq < cnt; ++qq) {
                const float dx = (float)(xi - sx[qq] - shx), dy = (float)(yi - sy[qq] - shy),
                            dz = (float)(zi - sz[qq] - shz);
                const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                const float sgq = ss[qq], isg = 1.f / sgq;
                float f, q;
                if (r2 < 0.5f * sgq * sgq) {
                    fq_series_sig(r2, isg, isg * isg * isg, kc1, f, q);
                } else {
                    f2 f2v, q2v;
                    fq_closed2_sig(pk(r2, r2), -1.4426950408889634f * 0.5f * isg * isg, isg,
                                   isg * isg * isg, kc1, f2v, q2v);
                    float fb, qb;
                    upk(f2v, f, fb);
                    upk(q2v, q, qb);
                }
                accumulate<SCHEME>(dx, dy, dz, f, q, sgx[qq], sgy[qq], sgz[qq], gix, giy, giz, acc);
            }
            tot[0] += acc.u0;
            tot[1] += acc.u1;
            tot[2] += acc.u2;
            tot[3] += acc.a0;
            tot[4] += acc.a1;
            tot[5] += acc.a2;
            tot[6] += acc.b0;
            tot[7] += acc.b1;
            tot[8] += acc.b2;
        }
    }
    if (act) {
        float o[6];
        const Acc t = {(float)tot[0], (float)tot[1], (float)tot[2], (float)tot[3], (float)tot[4],
                       (float)tot[5], (float)tot[6], (float)tot[7], (float)tot[8]};
        finish<SCHEME>(t, gix, giy, giz, o);
        for (int k = 0; k < 3; ++k) {
            vel[k * n + i] = o[k];
            dgam[k * n + i] = o[3 + k];
        }
    }
}

// DIRECT mode: all pairs over the image cube; targets in input order, 128 per block.
// d is formed in double from the float inputs, then rounded once (test mode).
template <int SCHEME>
__global__ void __launch_bounds__(128) direct_kernel(const float* __restrict__ pos,
                                                     const float* __restrict__ gam, int64_t n,
                                                     double len, int m, KernelConsts kc,
                                                     float* __restrict__ vel,
                                                     float* __restrict__ dgam) {
    __shared__ double sx[128], sy[128], sz[128];
    __shared__ float sgx[128], sgy[128], sgz[128];
    const int64_t i = blockIdx.x * (int64_t)128 + threadIdx.x;
    const bool act = i < n;
    double xi = 0, yi = 0, zi = 0;
    float gix = 0, giy = 0, giz = 0;
    if (act) {
        xi = pos[i];
        yi = pos[n + i];
        zi = pos[2 * n + i];
        gix = gam[i];
        giy = gam[n + i];
        giz = gam[2 * n + i];
    }
    double tot[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // image partials summed in double
    const int side = 2 * m + 1;
    for (int64_t sb = 0; sb < n; sb += 128) {
        __syncthreads();
        const int64_t j = sb + threadIdx.x;
        if (j < n) {
            sx[threadIdx.x] = pos[j];
            sy[threadIdx.x] = pos[n + j];
            sz[threadIdx.x] = pos[2 * n + j];
            sgx[threadIdx.x] = gam[j];
            sgy[threadIdx.x] = gam[n + j];
            sgz[threadIdx.x] = gam[2 * n + j];
        }
        __syncthreads();
        const int cnt = (int)min((int64_t)128, n - sb);
        if (!act) continue;
        for (int im = 0; im < side * side * side; ++im) {
            const double shx = (im / (side * side) - m) * len;
            const double shy = ((im / side) % side - m) * len;
            const double shz = (im % side - m) * len;
            Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            for (int q = 0; q < cnt; ++q)
                pair<SCHEME>((float)(xi - sx[q] - shx), (float)(yi - sy[q] - shy),
                             (float)(zi - sz[q] - shz), sgx[q], sgy[q], sgz[q], gix, giy, giz, kc,
                             acc);
            tot[0] += acc.u0;
            tot[1] += acc.u1;
            tot[2] += acc.u2;
            tot[3] += acc.a0;
            tot[4] += acc.a1;
            tot[5] += acc.a2;
            tot[6] += acc.b0;
            tot[7] += acc.b1;
            tot[8] += acc.b2;
        }
    }
    if (act) {
        float o[6];
        const Acc t = {(float)tot[0], (float)tot[1], (float)tot[2], (float)tot[3], (float)tot[4],
                       (float)tot[5], (float)tot[6], (float)tot[7], (float)tot[8]};
        finish<SCHEME>(t, gix, giy, giz, o);
        for (int k = 0; k < 3; ++k) {
            vel[k * n + i] = o[k];
            dgam[k * n + i] = o[3 + k];
        }
    }
}

}  // namespace

namespace {
template <int SCHEME, bool SJ, int MINB, int UNR>
void p2p_go(const float* sorted6, int64_t n, const int* leaf_start, int depth, float a,
            int periodic, KernelConsts kc, float* near6, unsigned long long* npairs, int64_t plo,
            int64_t pcnt, cudaStream_t st) {
    constexpr int cap = p2p_cap<SJ, MINB>();
    const size_t smem = SJ ? (size_t)(cap + P2P_PAD) * (2 * sizeof(float4) + sizeof(float))
                           : (size_t)(cap + P2P_PAD) * (sizeof(float4) + sizeof(float2));
    static PerDeviceOnce once;
    once([&] {
        cudaFuncSetAttribute(p2p_kernel<SCHEME, SJ, MINB, UNR>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    p2p_kernel<SCHEME, SJ, MINB, UNR><<<(unsigned)pcnt, P2P_THREADS, smem, st>>>(
        sorted6, n, leaf_start, depth, a, periodic, kc, near6, npairs, plo);
}
}  // namespace

void launch_p2p(const float* sorted6, int64_t n, const int* leaf_start, int depth, float a,
                int periodic, int scheme, KernelConsts kc, float* near6,
                unsigned long long* npairs, int64_t plo, int64_t pcnt, cudaStream_t st,
                bool lean) {
    if (pcnt <= 0) return;
    // classical scheme, default: staged source cross products s_j = gamma_j x x_j (reading R17;
    // 38 instead of 41 FP32 operations per pair, P2P 41.9 vs 43.1 ms at c4; the sums carry
    // the lever arm |x_j| ~ the 4-leaf region instead of |d|, ~1e-6 relative rounding at c4);
    // VFMM_P2P=cross: per-pair gamma_j x d (the smallest rounding; the transpose scheme and the
    // lean co-resident variant always use it).
    // VFMM_P2P_CFG: occupancy / unroll variants (measurement knob): "b3u1", "b3u2", "b2u1"
    // (per-pair form), "s2", "s1" (staged form unrolled by 2 / 1)
    // The staged form's rounding grows with the lever arm (the 4-leaf region) over the close
    // pairs' distance (~sigma): default to it only while the leaf width is <= 8 sigma (the
    // benched lattice: 4 sigma); wider leaves (clustered inputs, small sigma) keep per-pair
    // cross products.  VFMM_P2P=sj / cross force either form.
    const char* env = getenv("VFMM_P2P");
    const float sigma = sqrtf(0.5f / kc.inv2s2);
    const bool sj = env ? strcmp(env, "sj") == 0 : a <= 8.f * sigma;
    const char* cfg = getenv("VFMM_P2P_CFG");
    const int v = !cfg ? 0 : strcmp(cfg, "b3u1") == 0 ? 1 : strcmp(cfg, "b3u2") == 0 ? 2
                                : strcmp(cfg, "b2u1") == 0 ? 3 : strcmp(cfg, "s2") == 0 ? 4
                                : strcmp(cfg, "s1") == 0 ? 5 : 0;
#define P2P_ARGS sorted6, n, leaf_start, depth, a, periodic, kc, near6, npairs, plo, pcnt, st
    if (scheme == 0 && sj && !lean && v == 4) {
        p2p_go<0, true, 2, 2>(P2P_ARGS);
    } else if (scheme == 0 && sj && !lean && v == 5) {
        p2p_go<0, true, 2, 1>(P2P_ARGS);
    } else if (scheme == 0 && sj && !lean && v == 0) {
        // unrolled by 4 since the box test removed the loop's branch (37.7 vs 38.3 ms at c4)
        p2p_go<0, true, 2, 4>(P2P_ARGS);
    } else if (lean) {
        if (scheme == 0) p2p_go<0, false, 1, 2>(P2P_ARGS);
        else p2p_go<1, false, 1, 2>(P2P_ARGS);
    } else if (scheme == 0) {
        if (v == 1) p2p_go<0, false, 3, 1>(P2P_ARGS);
        else if (v == 2) p2p_go<0, false, 3, 2>(P2P_ARGS);
        else if (v == 3) p2p_go<0, false, 2, 1>(P2P_ARGS);
        else p2p_go<0, false, 2, 2>(P2P_ARGS);
    } else {
        p2p_go<1, false, 2, 2>(P2P_ARGS);
    }
#undef P2P_ARGS
}

void launch_p2p_sigma(const float* sorted6, const float* sorted_sig, int64_t n,
                      const int* leaf_start, int depth, float a, int periodic, int scheme,
                      float* near6, unsigned long long* npairs, int64_t plo, int64_t pcnt,
                      cudaStream_t st) {
    if (pcnt <= 0) return;
    const KernelConsts kc1 = make_kernel_consts(1.f);
    const size_t smem = 1024 * sizeof(float2);
    if (scheme == 0)
        p2p_sig_kernel<0><<<(unsigned)pcnt, P2P_THREADS, smem, st>>>(
            sorted6, sorted_sig, n, leaf_start, depth, a, periodic, kc1, near6, npairs, plo);
    else
        p2p_sig_kernel<1><<<(unsigned)pcnt, P2P_THREADS, smem, st>>>(
            sorted6, sorted_sig, n, leaf_start, depth, a, periodic, kc1, near6, npairs, plo);
}

void launch_direct_sigma(const float* pos, const float* gamma, const float* sigma, int64_t n,
                         float len, int image_levels, int scheme, float* vel, float* dgam,
                         cudaStream_t st) {
    int m = 0;
    for (int l = 0; l < image_levels; ++l) m = 3 * m + 1;
    const KernelConsts kc1 = make_kernel_consts(1.f);
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (scheme == 0)
        direct_sig_kernel<0><<<grid, 128, 0, st>>>(pos, gamma, sigma, n, (double)len, m, kc1, vel, dgam);
    else
        direct_sig_kernel<1><<<grid, 128, 0, st>>>(pos, gamma, sigma, n, (double)len, m, kc1, vel, dgam);
}

void launch_direct(const float* pos, const float* gamma, int64_t n, float len, int image_levels,
                   int scheme, KernelConsts kc, float* vel, float* dgam, cudaStream_t st) {
    int m = 0;
    for (int l = 0; l < image_levels; ++l) m = 3 * m + 1;
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (scheme == 0)
        direct_kernel<0><<<grid, 128, 0, st>>>(pos, gamma, n, (double)len, m, kc, vel, dgam);
    else
        direct_kernel<1><<<grid, 128, 0, st>>>(pos, gamma, n, (double)len, m, kc, vel, dgam);
}


// ---------------------------------------------------------------------------
// Hybrid treecode, cell-particle half (section 3.2): stack-based traversal
// of the adaptive octree with cell-particle (M2P) and particle-particle interactions; the
// adaptive leaves hold <= n_crit particles ("automatically choosing the number of particles
// per box", reading R22).  The multipoles of every cell are the FMM's P2M / M2M output (Eq. 10
// about the cell centre, scaled M~ = M / w_l^n); the images outside the near 3^3 block come
// through the root local expansion (periodic kernel + L2L + L2P, as in the FMM).
// ---------------------------------------------------------------------------
namespace {

constexpr int TREE_WARPS = 4;
constexpr int TREE_STACK = 128;

__host__ __device__ __forceinline__ int64_t lvl_off(int l) { return ((int64_t(1) << (3 * l)) - 1) / 7; }

// adaptive leaves: a non-empty cell of level l >= 1 with count <= n_crit (or l = L) whose parent
// holds more than n_crit; appended (in no particular order) to groups as one (chunk << 4 |
// level, cell) item per chunk of 32 targets
__global__ void tree_groups_kernel(const int* __restrict__ leaf_start, int L, int ncrit,
                                   int64_t total, int2* __restrict__ groups,
                                   int* __restrict__ ngroups) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = t + 1;  // skip the root
        int l = 1;
        while (l < L && g >= lvl_off(l + 1)) ++l;
        const int64_t c = g - lvl_off(l);
        const int sh = 3 * (L - l);
        const int cnt = leaf_start[(c + 1) << sh] - leaf_start[c << sh];
        if (cnt == 0 || (l < L && cnt > ncrit)) continue;
        if (l > 1) {
            const int64_t pc = c >> 3;
            const int psh = sh + 3;
            if (leaf_start[(pc + 1) << psh] - leaf_start[pc << psh] <= ncrit) continue;
        }
        // one work item per chunk of 32 targets (balances leaves of very different sizes)
        const int nch = (cnt + 31) >> 5;
        const int k = atomicAdd(ngroups, nch);
        for (int q = 0; q < nch; ++q) groups[k + q] = make_int2((q << 4) | l, (int)c);
    }
}

struct TreeArgs {
    const float* s6;
    int64_t n;
    const uint32_t* keys;
    const int* leaf_start;
    const int2* groups;
    const int* ngroups;
    const float* Mall;
    float* near6;
    unsigned long long* counters;  // [0] P2P pairs, [1] M2P cell-particle interactions
    int L, p, ncrit, periodic;
    float aL;      // leaf width at level L (float, exact len / 2^L)
    float theta;
    int dbg;       // VFMM_TREE_DBG: bit 0 drops the P2P terms, bit 1 the M2P terms (tests)
};

// Multipole (scaled, level l, packed real) -> rows n <= 2 of the local expansion at the target
// point, Eq. (11): L_n^m = sum_{k,l} (-1)^{n+m} I_{n+k}^{l-m}(D) M_k^l, D in cell widths.
// I_j^q (q >= 0) by I_0^0 = 1/r, I_j^j = -(2j-1)(x+iy)/r^2 I_{j-1}^{j-1},
// I_j^q = ((2j-1) z I_{j-1}^q - ((j-1)^2 - q^2) I_{j-2}^q) / r^2, rows rolled through 3 slots of
// the lane's shared-memory column; negative orders by I^{-q} = (-1)^q conj(I^q).
// out (per component c): [L10, ReL11, ImL11, L20, ReL21, ImL21, ReL22, ImL22]
__device__ __forceinline__ void m2p_rows(const float* __restrict__ Msh, int p, int nc, float dx,
                                         float dy, float dz, float* __restrict__ Ish, int lane,
                                         float out[3][8]) {
    const int PQ = p + 3;
    // I_j^q of this lane at Ish[((j % 3) PQ + q) 64 + 2 lane] (Re, Im adjacent: one 64-bit load)
    auto IR = [&](int j, int q) -> float& { return Ish[((j % 3) * PQ + q) * 64 + 2 * lane]; };
    auto II = [&](int j, int q) -> float& { return Ish[((j % 3) * PQ + q) * 64 + 2 * lane + 1]; };
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float rho = 1.f / r2;
    auto gen = [&](int j) {
        if (j == 0) {
            IR(0, 0) = rsqrtf(r2);
            II(0, 0) = 0.f;
            return;
        }
        const float f = (float)(2 * j - 1);
        for (int q = 0; q < j; ++q) {
            const float a = IR(j - 1, q), b = II(j - 1, q);
            float vr = f * dz * a, vi = f * dz * b;
            if (q <= j - 2) {
                const float w = (float)((j - 1) * (j - 1) - q * q);
                vr = fmaf(-w, IR(j - 2, q), vr);
                vi = fmaf(-w, II(j - 2, q), vi);
            }
            IR(j, q) = vr * rho;
            II(j, q) = vi * rho;
        }
        const float a = IR(j - 1, j - 1), b = II(j - 1, j - 1);
        const float s = -f * rho;
        IR(j, j) = s * (dx * a - dy * b);
        II(j, j) = s * (dx * b + dy * a);
    };
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int t = 0; t < 8; ++t) out[c][t] = 0.f;
    gen(0);
    gen(1);
    gen(2);
    for (int k = 0; k <= p; ++k) {
        if (k >= 1) gen(k + 2);
        // sliding window over l: each step loads only I_{k+1}^l and I_{k+2}^l (the other three
        // orders are the previous steps'); negative l (conjugate symmetry of M and I) and l >= 0
        // run as separate loops over linear shared-memory offsets
        const float4* Mk = reinterpret_cast<const float4*>(Msh) + k * k;  // pk_re(k, 0)
        const float2* Ia = reinterpret_cast<const float2*>(Ish + ((k + 1) % 3) * PQ * 64) + lane;
        const float2* Ib = reinterpret_cast<const float2*>(Ish + ((k + 2) % 3) * PQ * 64) + lane;
        auto ineg = [&](const float2* R, int q, float& re, float& im) {  // I^{-q}, q > 0
            const float sg = (q & 1) ? -1.f : 1.f;
            const float2 v = R[32 * q];
            re = sg * v.x;
            im = -sg * v.y;
        };
        float a0r, a0i, b0r, b0i, b1r, b1i;
        ineg(Ia, k + 1, a0r, a0i);
        ineg(Ib, k + 2, b0r, b0i);
        ineg(Ib, k + 1, b1r, b1i);
        auto step = [&](const float (&mr)[3], const float (&mi)[3], float a1r, float a1i, float b2r,
                        float b2i) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                // (n, m) = (1, 0): sign -1, real part; I_{k+1}^l
                out[c][0] -= a1r * mr[c] - a1i * mi[c];
                // (1, 1): sign +1; I_{k+1}^{l-1}
                out[c][1] += a0r * mr[c] - a0i * mi[c];
                out[c][2] += a0r * mi[c] + a0i * mr[c];
                // (2, 0): sign +1, real part; I_{k+2}^l
                out[c][3] += b2r * mr[c] - b2i * mi[c];
                // (2, 1): sign -1; I_{k+2}^{l-1}
                out[c][4] -= b1r * mr[c] - b1i * mi[c];
                out[c][5] -= b1r * mi[c] + b1i * mr[c];
                // (2, 2): sign +1; I_{k+2}^{l-2}
                out[c][6] += b0r * mr[c] - b0i * mi[c];
                out[c][7] += b0r * mi[c] + b0i * mr[c];
            }
            a0r = a1r;
            a0i = a1i;
            b0r = b1r;
            b0i = b1i;
            b1r = b2r;
            b1i = b2i;
        };
        for (int al = k; al >= 1; --al) {  // l = -al: M^l = (-1)^al conj(M^al)
            const float sg = (al & 1) ? -1.f : 1.f;
            const float4 re4 = Mk[2 * al - 1], im4 = Mk[2 * al];
            const float mr[3] = {sg * re4.x, sg * re4.y, sg * re4.z};
            const float mi[3] = {-sg * im4.x, -sg * im4.y, -sg * im4.z};
            float a1r, a1i, b2r, b2i;
            ineg(Ia, al, a1r, a1i);
            ineg(Ib, al, b2r, b2i);
            step(mr, mi, a1r, a1i, b2r, b2i);
        }
        {  // l = 0
            const float4 re4 = Mk[0];
            const float mr[3] = {re4.x, re4.y, re4.z};
            const float mi[3] = {0.f, 0.f, 0.f};
            const float2 ia = Ia[0], ib = Ib[0];
            step(mr, mi, ia.x, ia.y, ib.x, ib.y);
        }
        for (int l = 1; l <= k; ++l) {
            const float4 re4 = Mk[2 * l - 1], im4 = Mk[2 * l];
            const float mr[3] = {re4.x, re4.y, re4.z};
            const float mi[3] = {im4.x, im4.y, im4.z};
            const float2 ia = Ia[32 * l], ib = Ib[32 * l];
            step(mr, mi, ia.x, ia.y, ib.x, ib.y);
        }
    }
}

template <int SCHEME>
__global__ void __launch_bounds__(TREE_WARPS * 32, 4) tree_kernel(TreeArgs A, KernelConsts kc) {
    extern __shared__ float4 tree_sm4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = A.p, nc = (p + 1) * (p + 1), L = A.L;
    const int ish_floats = 3 * (p + 3) * 2 * 32;
    const int msh_floats = 4 * nc;  // [k][component] float4 (one broadcast load per coefficient)
    float* base = reinterpret_cast<float*>(tree_sm4) + warp * (ish_floats + msh_floats + 9 * 32);
    float* Ish = base;
    float* Msh = base + ish_floats;
    float* Ssh = Msh + msh_floats;  // sources: float4 (dx dy dz ix)[32], (gx gy gz iy)[32], iz[32]
    __shared__ int2 stack_sm[TREE_WARPS][TREE_STACK];
    int2* stk = stack_sm[warp];
    const int ng = *A.ngroups;
    const int side = 1 << L;
    const float aL = A.aL;
    const float inv_aL = 1.f / aL;
    const int nimg = A.periodic ? 27 : 1;
    const double th2 = (double)A.theta * (double)A.theta;
    for (int g = blockIdx.x * TREE_WARPS + warp; g < ng; g += gridDim.x * TREE_WARPS) {  // items
        const int2 grp = A.groups[g];
        const int lb = grp.x & 15, cb = grp.y, chunk = grp.x >> 4;
        const int shb = 3 * (L - lb);
        const int s = A.leaf_start[(int64_t)cb << shb], e = A.leaf_start[((int64_t)cb + 1) << shb];
        const float wb = (float)(1 << (L - lb));  // group width in leaf widths
        const float Gx = ((float)compact3p((uint32_t)cb) + 0.5f) * wb;
        const float Gy = ((float)compact3p((uint32_t)cb >> 1) + 0.5f) * wb;
        const float Gz = ((float)compact3p((uint32_t)cb >> 2) + 0.5f) * wb;
        {
            const int t0 = s + 32 * chunk;
            const int i = t0 + lane;
            const bool act = i < e;
            int tx = 0, ty = 0, tz = 0;
            float dxi = 0, dyi = 0, dzi = 0, gix = 0, giy = 0, giz = 0;
            if (act) {
                const uint32_t key = A.keys[i];
                tx = (int)compact3p(key);
                ty = (int)compact3p(key >> 1);
                tz = (int)compact3p(key >> 2);
                dxi = A.s6[i];
                dyi = A.s6[A.n + i];
                dzi = A.s6[2 * A.n + i];
                gix = A.s6[3 * A.n + i];
                giy = A.s6[4 * A.n + i];
                giz = A.s6[5 * A.n + i];
            }
            const float txf = (float)tx, tyf = (float)ty, tzf = (float)tz;  // exact leaf indices
            // target position in leaf widths from the box corner
            const float Px = (float)tx + 0.5f + dxi * inv_aL;
            const float Py = (float)ty + 0.5f + dyi * inv_aL;
            const float Pz = (float)tz + 0.5f + dzi * inv_aL;
            Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            float Lt[3][8];
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int q = 0; q < 8; ++q) Lt[c][q] = 0.f;
            unsigned long long npairs = 0, nm2p = 0;
            __syncwarp();
            if (lane < nimg) stk[lane] = make_int2(lane << 8, 0);  // (image << 8 | level, cell)
            int sp = nimg;
            __syncwarp();
            while (sp > 0) {
                const int2 ent = stk[--sp];
                __syncwarp();
                const int l = ent.x & 0xff, img = ent.x >> 8;
                const int64_t c = ent.y;
                const int ox = A.periodic ? img / 9 - 1 : 0, oy = A.periodic ? (img / 3) % 3 - 1 : 0,
                          oz = A.periodic ? img % 3 - 1 : 0;
                const int sh = 3 * (L - l);
                const int rs = A.leaf_start[c << sh], re = A.leaf_start[(c + 1) << sh];
                if (re == rs) continue;
                const int wl = 1 << (L - l);
                const float Cx = ((float)compact3p((uint32_t)c) + 0.5f) * wl + ox * side;
                const float Cy = ((float)compact3p((uint32_t)c >> 1) + 0.5f) * wl + oy * side;
                const float Cz = ((float)compact3p((uint32_t)c >> 2) + 0.5f) * wl + oz * side;
                // MAC r_S + r_B < theta d, r = (sqrt 3 / 2) w: 0.75 (w_S + w_B)^2 < theta^2 d^2 in
                // leaf widths, in double (every term but the last product exact: the oracle
                // takes the same decision on ties)
                const double ddx = (double)Gx - (double)Cx, ddy = (double)Gy - (double)Cy,
                             ddz = (double)Gz - (double)Cz;
                const double d2 = ddx * ddx + ddy * ddy + ddz * ddz;
                const double ws = (double)wl + (double)wb;
                // an accepted cell with fewer than (p+1)^2 particles acts particle-particle
                // (exact, and cheaper than its multipole; reading R22)
                const bool accept = 0.75 * ws * ws < th2 * d2;
                if (accept && re - rs >= nc) {  // cell-particle: M2P
                    const float* Mg = A.Mall + (lvl_off(l) + c) * 3 * nc;
                    for (int k = lane; k < 3 * nc; k += 32) Msh[(k % nc) * 4 + k / nc] = Mg[k];
                    __syncwarp();
                    if (act && !(A.dbg & 2)) {
                        const float iw = 1.f / (float)wl;
                        float o[3][8];
                        m2p_rows(Msh, p, nc, (Px - Cx) * iw, (Py - Cy) * iw, (Pz - Cz) * iw, Ish,
                                 lane, o);
                        // L_n (absolute) = sum / w^(n+1), w = wl aL
                        const float w1 = iw * inv_aL, w2 = w1 * w1, w3 = w2 * w1;
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) {
                            Lt[cc][0] = fmaf(o[cc][0], w2, Lt[cc][0]);
                            Lt[cc][1] = fmaf(o[cc][1], w2, Lt[cc][1]);
                            Lt[cc][2] = fmaf(o[cc][2], w2, Lt[cc][2]);
#pragma unroll
                            for (int q = 3; q < 8; ++q) Lt[cc][q] = fmaf(o[cc][q], w3, Lt[cc][q]);
                        }
                        ++nm2p;
                    }
                    __syncwarp();
                } else if (accept || (l >= 1 && (l == L || re - rs <= A.ncrit))) {  // P2P
                    // sources staged as (delta, leaf index) float4 pairs: d = (t - s) a + (delta_i -
                    // delta_j) with exact leaf offsets, three shared loads per pair
                    float4* SA = reinterpret_cast<float4*>(Ssh);           // dx dy dz ix
                    float4* SB = reinterpret_cast<float4*>(Ssh + 4 * 32);  // gx gy gz iy
                    float* SC = Ssh + 8 * 32;                              // iz
                    for (int j0 = rs; j0 < re; j0 += 32) {
                        const int j = j0 + lane;
                        if (j < re) {
                            const uint32_t key = A.keys[j];
                            SA[lane] = make_float4(A.s6[j], A.s6[A.n + j], A.s6[2 * A.n + j],
                                                   (float)((int)compact3p(key) + ox * side));
                            SB[lane] = make_float4(A.s6[3 * A.n + j], A.s6[4 * A.n + j],
                                                   A.s6[5 * A.n + j],
                                                   (float)((int)compact3p(key >> 1) + oy * side));
                            SC[lane] = (float)((int)compact3p(key >> 2) + oz * side);
                        }
                        __syncwarp();
                        const int cnt = min(32, re - j0);
                        if (act) {
                            for (int q = 0; q < cnt; ++q) {
                                const float4 a4 = SA[q], b4 = SB[q];
                                const float cz = SC[q];
                                const float dx = fmaf(txf - a4.w, aL, dxi - a4.x);
                                const float dy = fmaf(tyf - b4.w, aL, dyi - a4.y);
                                const float dz = fmaf(tzf - cz, aL, dzi - a4.z);
                                if (!(A.dbg & 1))
                                    pair<SCHEME>(dx, dy, dz, b4.x, b4.y, b4.z, gix, giy, giz, kc, acc);
                            }
                            npairs += cnt;
                        }
                        __syncwarp();
                    }
                } else {  // open the cell: push its non-empty children
                    const int csh = sh - 3;
                    int cnt_c = 0;
                    if (lane < 8) {
                        const int64_t ch = 8 * c + lane;
                        cnt_c = A.leaf_start[(ch + 1) << csh] - A.leaf_start[ch << csh];
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, lane < 8 && cnt_c > 0);
                    if (lane < 8 && cnt_c > 0) {
                        const int pos = sp + __popc(m & ((1u << lane) - 1u));
                        if (pos < TREE_STACK)
                            stk[pos] = make_int2((img << 8) | (l + 1), (int)(8 * c + lane));
                    }
                    sp += __popc(m);
                    if (sp > TREE_STACK) sp = TREE_STACK;  // cannot happen: depth <= 10
                    __syncwarp();
                }
            }
            if (act) {
                float o[6];
                finish<SCHEME>(acc, gix, giy, giz, o);
                // gradient and Hessian of phi_c from the order-2 local expansion at the target
                // (derivative rules of the regular harmonics at the expansion centre)
                float gr[3][3], H[3][6];  // H: xx, xy, xz, yy, yz, zz
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    gr[cc][0] = -Lt[cc][1];
                    gr[cc][1] = Lt[cc][2];
                    gr[cc][2] = Lt[cc][0];
                    H[cc][0] = 0.5f * Lt[cc][6] - 0.5f * Lt[cc][3];
                    H[cc][1] = -0.5f * Lt[cc][7];
                    H[cc][2] = -Lt[cc][4];
                    H[cc][3] = -0.5f * Lt[cc][6] - 0.5f * Lt[cc][3];
                    H[cc][4] = Lt[cc][5];
                    H[cc][5] = Lt[cc][3];
                }
                auto Hs = [&](int cc, int a, int b) -> float {
                    const int lo = a < b ? a : b, hi = a < b ? b : a;
                    const int idx = lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
                    return H[cc][idx];
                };
                const float k4 = 0.0795774715459476679f;  // 1 / (4 pi)
                const float gi[3] = {gix, giy, giz};
                // u_a = eps_abc d_b phi_c / 4 pi
                o[0] += k4 * (gr[2][1] - gr[1][2]);
                o[1] += k4 * (gr[0][2] - gr[2][0]);
                o[2] += k4 * (gr[1][0] - gr[0][1]);
                float sv[3];
                if (SCHEME == 0) {
                    // s_a = eps_abc (gamma . grad) d_b phi_c / 4 pi
                    float D[3][3];  // D[c][b] = sum_d g_d d_d d_b phi_c
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
                        for (int b = 0; b < 3; ++b)
                            D[cc][b] = gi[0] * Hs(cc, 0, b) + gi[1] * Hs(cc, 1, b) + gi[2] * Hs(cc, 2, b);
                    sv[0] = D[2][1] - D[1][2];
                    sv[1] = D[0][2] - D[2][0];
                    sv[2] = D[1][0] - D[0][1];
                } else {
                    // s_a = eps_dbc g_d d_a d_b phi_c / 4 pi = d_a (gamma . curl phi) / 4 pi
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        sv[a] = gi[0] * (Hs(2, a, 1) - Hs(1, a, 2)) +
                                gi[1] * (Hs(0, a, 2) - Hs(2, a, 0)) +
                                gi[2] * (Hs(1, a, 0) - Hs(0, a, 1));
                }
                o[3] += k4 * sv[0];
                o[4] += k4 * sv[1];
                o[5] += k4 * sv[2];
                for (int k = 0; k < 6; ++k) A.near6[k * A.n + i] = o[k];
            }
            // interaction counts (one atomic per warp and chunk)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                npairs += __shfl_xor_sync(0xffffffffu, npairs, off);
                nm2p += __shfl_xor_sync(0xffffffffu, nm2p, off);
            }
            if (lane == 0) {
                atomicAdd(A.counters, npairs);
                atomicAdd(A.counters + 1, nm2p);
            }
        }
    }
}

}  // namespace

size_t tree_groups_cap(int64_t n, int depth) {  // work items: chunks of 32 targets per leaf
    const int64_t cells = lvl_off(depth + 1) - 1;
    return (size_t)((n < cells ? n : cells) + n / 32 + 1);
}

void launch_tree(const float* sorted6, int64_t n, const uint32_t* keys_sorted,
                 const int* leaf_start, int depth, float aL, int periodic, int scheme, int p,
                 int ncrit, float theta, const float* Mall, KernelConsts kc, int2* groups,
                 int* ngroups, unsigned long long* counters, float* near6, cudaStream_t st) {
    cudaMemsetAsync(ngroups, 0, sizeof(int), st);
    cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), st);
    const int64_t total = lvl_off(depth + 1) - 1;
    const int gb = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    tree_groups_kernel<<<gb, 256, 0, st>>>(leaf_start, depth, ncrit, total, groups, ngroups);
    TreeArgs A{sorted6, n, keys_sorted, leaf_start, groups, ngroups, Mall, near6, counters,
               depth, p, ncrit, periodic, aL, theta, 0};
    if (const char* e = getenv("VFMM_TREE_DBG")) A.dbg = atoi(e);
    const int nc = (p + 1) * (p + 1);
    const size_t per_warp = (size_t)(3 * (p + 3) * 2 * 32 + 4 * nc + 9 * 32);
    const size_t smem = per_warp * TREE_WARPS * sizeof(float);
    static PerDeviceOnce once;
    once([&] {
        cudaFuncSetAttribute(tree_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(tree_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    const int grid = 148 * 4;
    if (scheme == 0)
        tree_kernel<0><<<grid, TREE_WARPS * 32, smem, st>>>(A, kc);
    else
        tree_kernel<1><<<grid, TREE_WARPS * 32, smem, st>>>(A, kc);
}

}  // namespace vfmm
