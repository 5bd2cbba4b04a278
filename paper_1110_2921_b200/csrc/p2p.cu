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
// otherwise 1 - g = e^{-rho^2} (erfcx(rho) + 2 rho/sqrt(pi)) with erfcx from a degree-7
// polynomial in t = 1/(1 + rho/2) (scripts/fit_cutoff_poly.py): 3 MUFU (rsqrt, ex2, rcp).
#include <cuda_runtime.h>

#include <cmath>

#include "vfmm_internal.h"

namespace vfmm {

KernelConsts make_kernel_consts(float sigma) {
    const double s = (double)sigma;
    KernelConsts k;
    k.inv2s2 = (float)(1.0 / (2.0 * s * s));
    k.neg_l2e_inv2s2 = (float)(-1.4426950408889634 / (2.0 * s * s));
    k.inv_s_sqrt2 = (float)(1.0 / (std::sqrt(2.0) * s));
    const double z0 = std::pow(2.0 * M_PI * s * s, -1.5);
    k.zeta0 = (float)z0;
    k.zeta0_over_s2 = (float)(z0 / (s * s));
    return k;
}

namespace {

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
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

template <int SCHEME>
__device__ __forceinline__ void pair(float dx, float dy, float dz, float gjx, float gjy, float gjz,
                                     float gix, float giy, float giz, const KernelConsts& kc,
                                     Acc& acc) {
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float s = r2 * kc.inv2s2;  // rho^2
    float f, q;
    if (s < 0.25f) {
        // f = zeta0 sum (-s)^k/(k!(2k+3)),  q = zeta0/sigma^2 sum_{k>=1} (-1)^k s^{k-1}/((k-1)!(2k+3))
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
    } else {
        const float rinv = rsqrtf(r2);
        const float e = ex2_approx(r2 * kc.neg_l2e_inv2s2);
        const float rho = r2 * rinv * kc.inv_s_sqrt2;
        const float t = rcp_approx(fmaf(0.5f, rho, 1.f)) - 0.5f;
        float E = 7.796925861e-02f;
        E = fmaf(E, t, -2.091334887e-02f);
        E = fmaf(E, t, -2.338621977e-01f);
        E = fmaf(E, t, 6.124646918e-02f);
        E = fmaf(E, t, 6.317173519e-01f);
        E = fmaf(E, t, 9.666348646e-01f);
        E = fmaf(E, t, 8.543718279e-01f);
        E = fmaf(E, t, 2.553956723e-01f);
        const float Q = fmaf(1.1283791670955126f, rho, E);  // + 2 rho / sqrt(pi)
        const float g = fmaf(-e, Q, 1.f);
        const float rinv2 = rinv * rinv;
        f = g * rinv2 * rinv * 0.0795774715459476679f;
        q = fmaf(kc.zeta0, e, -3.f * f) * rinv2;
    }
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

// one block (64 threads) per target leaf; sources = the 27 neighbour leaves (periodic
// images), staged through shared memory in chunks of 64, positions relative to the target
// leaf centre (s = d_j + o a, exact leaf-centre differences; reading R8).
template <int SCHEME>
__global__ void __launch_bounds__(64) p2p_kernel(const float* __restrict__ s6, int64_t n,
                                                 const int* __restrict__ leaf_start, int depth,
                                                 float a, int periodic, KernelConsts kc,
                                                 float* __restrict__ near6) {
    __shared__ float sx[64], sy[64], sz[64], sgx[64], sgy[64], sgz[64];
    const uint32_t leaf = blockIdx.x;
    const int side = 1 << depth;
    const int tx = (int)compact3p(leaf), ty = (int)compact3p(leaf >> 1),
              tz = (int)compact3p(leaf >> 2);
    const int st = leaf_start[leaf], et = leaf_start[leaf + 1];
    for (int tb = st; tb < et; tb += 64) {
        const int i = tb + threadIdx.x;
        const bool act = i < et;
        float xi = 0.f, yi = 0.f, zi = 0.f, gix = 0.f, giy = 0.f, giz = 0.f;
        if (act) {
            xi = s6[i];
            yi = s6[n + i];
            zi = s6[2 * n + i];
            gix = s6[3 * n + i];
            giy = s6[4 * n + i];
            giz = s6[5 * n + i];
        }
        Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int nb = 0; nb < 27; ++nb) {
            const int ox = nb % 3 - 1, oy = (nb / 3) % 3 - 1, oz = nb / 9 - 1;
            int nx = tx + ox, ny = ty + oy, nz = tz + oz;
            if (!periodic && (nx < 0 || nx >= side || ny < 0 || ny >= side || nz < 0 || nz >= side))
                continue;
            nx &= side - 1;
            ny &= side - 1;
            nz &= side - 1;
            const uint32_t sc = spread3p(nx) | (spread3p(ny) << 1) | (spread3p(nz) << 2);
            const int ss = leaf_start[sc], es = leaf_start[sc + 1];
            const float offx = ox * a, offy = oy * a, offz = oz * a;
            for (int sb = ss; sb < es; sb += 64) {
                __syncthreads();
                const int j = sb + threadIdx.x;
                if (j < es) {
                    sx[threadIdx.x] = s6[j] + offx;
                    sy[threadIdx.x] = s6[n + j] + offy;
                    sz[threadIdx.x] = s6[2 * n + j] + offz;
                    sgx[threadIdx.x] = s6[3 * n + j];
                    sgy[threadIdx.x] = s6[4 * n + j];
                    sgz[threadIdx.x] = s6[5 * n + j];
                }
                __syncthreads();
                const int cnt = min(64, es - sb);
                if (act) {
                    for (int q = 0; q < cnt; ++q)
                        pair<SCHEME>(xi - sx[q], yi - sy[q], zi - sz[q], sgx[q], sgy[q], sgz[q],
                                     gix, giy, giz, kc, acc);
                }
            }
        }
        if (act) {
            float o[6];
            finish<SCHEME>(acc, gix, giy, giz, o);
#pragma unroll
            for (int k = 0; k < 6; ++k) near6[k * n + i] = o[k];
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
    Acc tot = {0, 0, 0, 0, 0, 0, 0, 0, 0};
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
            tot.u0 += acc.u0;
            tot.u1 += acc.u1;
            tot.u2 += acc.u2;
            tot.a0 += acc.a0;
            tot.a1 += acc.a1;
            tot.a2 += acc.a2;
            tot.b0 += acc.b0;
            tot.b1 += acc.b1;
            tot.b2 += acc.b2;
        }
    }
    if (act) {
        float o[6];
        finish<SCHEME>(tot, gix, giy, giz, o);
        for (int k = 0; k < 3; ++k) {
            vel[k * n + i] = o[k];
            dgam[k * n + i] = o[3 + k];
        }
    }
}

}  // namespace

void launch_p2p(const float* sorted6, int64_t n, const int* leaf_start, int depth, float a,
                int periodic, int scheme, KernelConsts kc, float* near6, cudaStream_t st) {
    const int64_t nleaf = (int64_t)1 << (3 * depth);
    if (scheme == 0)
        p2p_kernel<0><<<(unsigned)nleaf, 64, 0, st>>>(sorted6, n, leaf_start, depth, a, periodic,
                                                      kc, near6);
    else
        p2p_kernel<1><<<(unsigned)nleaf, 64, 0, st>>>(sorted6, n, leaf_start, depth, a, periodic,
                                                      kc, near6);
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

}  // namespace vfmm
