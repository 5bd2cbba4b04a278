// rbf.cu -- NEXT-2: reinitialization of the particles onto a lattice by RBF interpolation
// (PAPER.md:113-114, :191, :272-277).
//
//   omega_i = sum_j gamma_j zeta_sigma_old(x_i - x_j)            Eq. (3) at the new points x_i
//   solve   sum_j gamma'_j zeta_sigma_new(x_i - x_j) = omega_i    for gamma' (the RBF system)
//
// "matrix-vector multiplications are done in matrix-free form by calculating Eq. (3) ... we
// use the FMM neighbor list to calculate Eq. (3) between neighboring particles only"
// (PAPER.md:114), GMRES with the initial guess gamma' = omega (dx)^3 and the exit tolerance
// measured as the relative drop of the residual from that guess.  Everything
// runs on the device: Morton trees of the old and the new particles (tree.cu), the Gaussian
// sums over the neighbour leaves (gauss_kernel), and GMRES in lockstep for the three strength
// components (Krylov basis in HBM, deterministic multi-dot reductions, CGS2 orthogonalisation;
// only the (m+1) x m Hessenberg recurrences run on the host).
//
// Neighbour list (reading R18): the leaves within ws of the target leaf, ws the
// smallest integer with ws a >= 6 sigma (a = leaf width), so the Gaussian is truncated below
// e^{-18} = 1.5e-8 of its peak (the paper's 27-leaf list, ws = 1, truncates at e^{-8} when
// a = 4 sigma -- the 64-per-leaf tree with sigma = h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "vfmm_internal.h"

namespace vfmm {

namespace {

__device__ __forceinline__ float ex2_approx_r(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t spread3r(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ uint32_t compact3r(uint32_t v) {
    v &= 0x09249249u;
    v = (v ^ (v >> 2)) & 0x030C30C3u;
    v = (v ^ (v >> 4)) & 0x0300F00Fu;
    v = (v ^ (v >> 8)) & 0x030000FFu;
    v = (v ^ (v >> 16)) & 0x000003FFu;
    return v;
}

constexpr int G_THREADS = 64;
constexpr int G_CAP = 1024;  // staged sources per pass

// out[c][i] = zeta0 sum_{j in the (2 ws + 1)^3 neighbour leaves of i's leaf} g_j,c
//             2^(c2 |x_i - x_j|^2),   c2 = -log2(e) / (2 sigma^2)
// t6 / s6: sorted [dx dy dz gx gy gz] (d = x - exact leaf centre), leaf starts tls / sls at the
// same depth; sg (3 x ns, sorted order) overrides the source strengths when not null.
// One block per target leaf; targets in chunks of 64, sources staged per neighbour leaf.
__global__ void __launch_bounds__(G_THREADS) gauss_kernel(
    const float* __restrict__ t6, int64_t nt, const int* __restrict__ tls,
    const float* __restrict__ s6, int64_t ns, const int* __restrict__ sls,
    const float* __restrict__ sg, int depth, float a, int periodic, int ws, float c2, float zeta0,
    float* __restrict__ out) {
    __shared__ float4 sp[G_CAP];
    __shared__ float2 sq[G_CAP];
    const uint32_t leaf = blockIdx.x;
    const int ts = tls[leaf], te = tls[leaf + 1];
    if (ts >= te) return;
    const int side = 1 << depth;
    const int tx = (int)compact3r(leaf), ty = (int)compact3r(leaf >> 1), tz = (int)compact3r(leaf >> 2);
    const float* gsrc = sg ? sg : s6 + 3 * ns;
    const int64_t gstride = sg ? ns : ns;
    for (int c0 = ts; c0 < te; c0 += G_THREADS) {
        const int i = c0 + threadIdx.x;
        const bool act = i < te;
        const float xi = act ? t6[i] : 0.f, yi = act ? t6[nt + i] : 0.f, zi = act ? t6[2 * nt + i] : 0.f;
        float ax = 0.f, ay = 0.f, az = 0.f;
        for (int oz = -ws; oz <= ws; ++oz)
            for (int oy = -ws; oy <= ws; ++oy)
                for (int ox = -ws; ox <= ws; ++ox) {
                    int sx = tx + ox, sy = ty + oy, sz = tz + oz;
                    if (!periodic && (sx < 0 || sy < 0 || sz < 0 || sx >= side || sy >= side || sz >= side))
                        continue;
                    sx = (sx + side) & (side - 1);
                    sy = (sy + side) & (side - 1);
                    sz = (sz + side) & (side - 1);
                    const uint32_t sl = spread3r(sx) | (spread3r(sy) << 1) | (spread3r(sz) << 2);
                    const int ss = sls[sl], se = sls[sl + 1];
                    // source positions relative to the target leaf centre: d_j + o a (exact offset)
                    const float offx = ox * a, offy = oy * a, offz = oz * a;
                    for (int w0 = ss; w0 < se; w0 += G_CAP) {
                        const int cnt = min(G_CAP, se - w0);
                        __syncthreads();
                        for (int k = threadIdx.x; k < cnt; k += G_THREADS) {
                            const int j = w0 + k;
                            sp[k] = make_float4(s6[j] + offx, s6[ns + j] + offy, s6[2 * ns + j] + offz,
                                                gsrc[j]);
                            sq[k] = make_float2(gsrc[gstride + j], gsrc[2 * gstride + j]);
                        }
                        __syncthreads();
                        if (act) {
#pragma unroll 4
                            for (int k = 0; k < cnt; ++k) {
                                const float4 p = sp[k];
                                const float dx = xi - p.x, dy = yi - p.y, dz = zi - p.z;
                                const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                                const float e = ex2_approx_r(r2 * c2);
                                const float2 q = sq[k];
                                ax = fmaf(e, p.w, ax);
                                ay = fmaf(e, q.x, ay);
                                az = fmaf(e, q.y, az);
                            }
                        }
                    }
                }
        if (act) {
            out[i] = zeta0 * ax;
            out[nt + i] = zeta0 * ay;
            out[2 * nt + i] = zeta0 * az;
        }
    }
}

// ---- deterministic BLAS-1 over 3-component vectors (3 x n SoA) ----
constexpr int D_BLOCKS = 296;
constexpr int D_THREADS = 256;

// part[b][v][c] = block b's share of <x_v, y> for component c, v < nv (x_v = X + v xs)
__global__ void __launch_bounds__(D_THREADS) multidot_kernel(const float* __restrict__ X,
                                                             int64_t xs, int nv,
                                                             const float* __restrict__ Y,
                                                             int64_t n, double* __restrict__ part) {
    __shared__ double red[D_THREADS / 32];
    for (int v = 0; v < nv; ++v)
        for (int c = 0; c < 3; ++c) {
            const float* x = X + v * xs + c * n;
            const float* y = Y + c * n;
            double s = 0.0;
            for (int64_t i = blockIdx.x * (int64_t)D_THREADS + threadIdx.x; i < n;
                 i += (int64_t)gridDim.x * D_THREADS)
                s += (double)x[i] * (double)y[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
            __syncthreads();
            if (threadIdx.x == 0) {
                double t = 0.0;
                for (int w = 0; w < D_THREADS / 32; ++w) t += red[w];
                part[((int64_t)blockIdx.x * nv + v) * 3 + c] = t;
            }
            __syncthreads();
        }
}
// out[v][c] = sum over blocks in order
__global__ void multidot_finish_kernel(const double* __restrict__ part, int nb, int nvc,
                                       double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nvc) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(int64_t)b * nvc + k];
    out[k] = s;
}
// Y[c] += sum_v coef[v][c] X_v[c]   (coef in device memory, float64)
__global__ void multiaxpy_kernel(const float* __restrict__ X, int64_t xs, int nv,
                                 const double* __restrict__ coef, float* __restrict__ Y,
                                 int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / n);
        double s = Y[i];
        for (int v = 0; v < nv; ++v) s += coef[v * 3 + c] * (double)X[v * xs + i];
        Y[i] = (float)s;
    }
}
// Y[c] = alpha[c] * X[c] + beta[c] * Z[c]  (alpha, beta host values)
__global__ void scale_kernel(const float* __restrict__ X, const float* __restrict__ Z,
                             float* __restrict__ Y, int64_t n, float a0, float a1, float a2,
                             float b0, float b1, float b2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / n);
        const float al = c == 0 ? a0 : (c == 1 ? a1 : a2);
        const float be = c == 0 ? b0 : (c == 1 ? b1 : b2);
        Y[i] = al * X[i] + (Z ? be * Z[i] : 0.f);
    }
}
// out[c][perm[k]] = in[c][k] (sorted -> input order)
__global__ void unpermute3_kernel(const float* __restrict__ in, const uint32_t* __restrict__ perm,
                                  int64_t n, float* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = perm[k];
        out[i] = in[k];
        out[n + i] = in[n + k];
        out[2 * n + i] = in[2 * n + k];
    }
}

int grid_n(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

}  // namespace

// ---------------------------------------------------------------------------------------

void launch_gauss(const float* t6, int64_t nt, const int* tls, const float* s6, int64_t ns,
                  const int* sls, const float* sg, int depth, float a, int periodic, int ws,
                  float sigma, float* out, cudaStream_t st) {
    const double s = sigma;
    const float c2 = (float)(-1.4426950408889634 / (2.0 * s * s));
    const float z0 = (float)std::pow(2.0 * M_PI * s * s, -1.5);
    const unsigned nleaf = 1u << (3 * depth);
    gauss_kernel<<<nleaf, G_THREADS, 0, st>>>(t6, nt, tls, s6, ns, sls, sg, depth, a, periodic,
                                              ws, c2, z0, out);
}

int rbf_ws(float a, float sigma) {
    return std::max(1, (int)std::ceil(6.0 * (double)sigma / (double)a - 1e-9));
}

size_t rbf_dot_part_doubles(int nv) { return (size_t)D_BLOCKS * nv * 3; }

// dots[v][c] = <X_v, Y>_c for v < nv; part: rbf_dot_part_doubles(nv) doubles, dots: 3 nv
void launch_multidot(const float* X, int64_t xs, int nv, const float* Y, int64_t n, double* part,
                     double* dots, cudaStream_t st) {
    multidot_kernel<<<D_BLOCKS, D_THREADS, 0, st>>>(X, xs, nv, Y, n, part);
    multidot_finish_kernel<<<(3 * nv + 127) / 128, 128, 0, st>>>(part, D_BLOCKS, 3 * nv, dots);
}
void launch_multiaxpy(const float* X, int64_t xs, int nv, const double* coef, float* Y, int64_t n,
                      cudaStream_t st) {
    multiaxpy_kernel<<<grid_n(3 * n), 256, 0, st>>>(X, xs, nv, coef, Y, n);
}
void launch_scale3(const float* X, const float* Z, float* Y, int64_t n, const double al[3],
                   const double be[3], cudaStream_t st) {
    scale_kernel<<<grid_n(3 * n), 256, 0, st>>>(X, Z, Y, n, (float)al[0], (float)al[1],
                                                (float)al[2], (float)be[0], (float)be[1],
                                                (float)be[2]);
}
void launch_unpermute3(const float* in, const uint32_t* perm, int64_t n, float* out,
                       cudaStream_t st) {
    unpermute3_kernel<<<grid_n(n), 256, 0, st>>>(in, perm, n, out);
}

}  // namespace vfmm
