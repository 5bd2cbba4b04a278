// tree.cu -- Morton keys, stable LSD radix sort, leaf ranges and the sorted gather.
//
// The paper builds its octree on the CPU with an auto-tuned leaf size
// (PAPER.md:152); here the uniform octree of depth L is built on the GPU.  Contract
// (bit-exact):
//   i_a = clamp((int)floorf(__fmul_rn(__fsub_rn(x_a, lo), inv)), 0, 2^L - 1),
//   inv = (float)(2^L / (double)len);  key bit 3b+a = bit b of i_a;
//   stable sort of (key, input index); leaf_start[c] = #keys < c.
#include <cuda_runtime.h>

#include "vfmm_internal.h"

namespace vfmm {

namespace {

__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> every 3rd bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__device__ __forceinline__ uint32_t compact3(uint32_t v) {
    v &= 0x09249249u;
    v = (v ^ (v >> 2)) & 0x030C30C3u;
    v = (v ^ (v >> 4)) & 0x0300F00Fu;
    v = (v ^ (v >> 8)) & 0x030000FFu;
    v = (v ^ (v >> 16)) & 0x000003FFu;
    return v;
}

__global__ void keys_kernel(const float* __restrict__ pos, int64_t n, float lo, float hi,
                            float inv, int side, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals, int* __restrict__ err) {
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float x = __ldg(pos + i + a * n);
            if (!(x >= lo && x < hi)) bad = 1;  // also NaN
            const float s = __fmul_rn(__fsub_rn(x, lo), inv);
            const float fl = floorf(s);
            int q = fl >= 0.f ? (int)fl : 0;
            if (!(fl >= 0.f)) q = 0;
            q = q > side - 1 ? side - 1 : q;
            c[a] = (uint32_t)q;
        }
        keys[i] = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
        vals[i] = (uint32_t)i;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1);
}

// ---- LSD radix sort: 8-bit digits, tiles of 4096 keys (8 warps x 16 chunks x 32) ----
// digit width per pass <= RB (9 bits): the key bits are split into equal-width passes
// (18-bit keys at depth 6: 2 passes of 9 bits instead of 3 of 8)
constexpr int RB = 9;
constexpr int RBINS = 1 << RB;  // bins of the widest digit
constexpr int RWARPS = 8;
constexpr int RCHUNK = 16;
constexpr int RTILE = RWARPS * RCHUNK * 32;  // 4096

__global__ void __launch_bounds__(256) radix_count(const uint32_t* __restrict__ keys, int64_t n,
                                                   int shift, int nbins,
                                                   uint32_t* __restrict__ counts, int nblocks) {
    __shared__ uint32_t h[RBINS];
    for (int d = threadIdx.x; d < nbins; d += 256) h[d] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RTILE;
    for (int i = threadIdx.x; i < RTILE; i += 256) {
        const int64_t k = base + i;
        if (k < n) atomicAdd(&h[(keys[k] >> shift) & (nbins - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nbins; d += 256) counts[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

// one block per digit: exclusive scan of its row over blocks; row total -> totals[d]
__global__ void __launch_bounds__(256) radix_scan_rows(uint32_t* __restrict__ counts, int nblocks,
                                                       uint32_t* __restrict__ totals) {
    __shared__ uint32_t wsum[8];
    __shared__ uint32_t carry;
    uint32_t* row = counts + (int64_t)blockIdx.x * nblocks;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b0 = 0; b0 < nblocks; b0 += 256) {
        const int b = b0 + threadIdx.x;
        const uint32_t v = b < nblocks ? row[b] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
        for (int i = 0; i < 8; ++i) {
            if (i < w) wpre += wsum[i];
            tot += wsum[i];
        }
        const uint32_t c0 = carry;
        if (b < nblocks) row[b] = c0 + wpre + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry = c0 + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(256) radix_scan_totals(uint32_t* __restrict__ totals, int nbins) {
    __shared__ uint32_t s[RBINS];
    for (int d = threadIdx.x; d < nbins; d += blockDim.x) s[d] = totals[d];
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int d = 0; d < nbins; ++d) {
            const uint32_t t = s[d];
            s[d] = run;
            run += t;
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nbins; d += blockDim.x) totals[d] = s[d];
}

__global__ void __launch_bounds__(256) radix_scatter(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, int64_t n, int shift,
    int nbins, const uint32_t* __restrict__ counts, const uint32_t* __restrict__ digit_base,
    int nblocks, uint32_t* __restrict__ kout, uint32_t* __restrict__ vout) {
    __shared__ uint32_t wh[RWARPS][RBINS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RWARPS * RBINS; i += 256) (&wh[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RTILE + (int64_t)w * RCHUNK * 32;
    uint32_t key[RCHUNK], val[RCHUNK], lpos[RCHUNK];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int c = 0; c < RCHUNK; ++c) {
        const int64_t k = base + c * 32 + lane;
        const bool ok = k < n;
        key[c] = ok ? kin[k] : 0u;
        val[c] = ok ? vin[k] : 0u;
        const uint32_t d = ok ? ((key[c] >> shift) & (nbins - 1)) : (uint32_t)RBINS;  // RBINS: none
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lt);
        const uint32_t before = (d < RBINS) ? wh[w][d] : 0u;
        lpos[c] = before + rank;
        __syncwarp();
        if (d < RBINS && rank == 0) wh[w][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nbins; d += 256) {  // exclusive prefix over warps per digit
        uint32_t run = digit_base[d] + counts[(int64_t)d * nblocks + blockIdx.x];
        for (int i = 0; i < RWARPS; ++i) {
            const uint32_t t = wh[i][d];
            wh[i][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < RCHUNK; ++c) {
        const int64_t k = base + c * 32 + lane;
        if (k < n) {
            const uint32_t d = (key[c] >> shift) & (nbins - 1);
            const uint32_t o = wh[w][d] + lpos[c];
            kout[o] = key[c];
            vout[o] = val[c];
        }
    }
}

__global__ void leaf_ranges_kernel(const uint32_t* __restrict__ keys, int64_t n, int64_t nleaf,
                                   int* __restrict__ leaf_start) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i < n ? (int64_t)keys[i] : nleaf;
        const int64_t kp = i > 0 ? (int64_t)keys[i - 1] : -1;
        for (int64_t c = kp + 1; c <= k; ++c) leaf_start[c] = (int)i;
    }
}

// sorted6 = [dx | dy | dz | gx | gy | gz], d = x - (exact leaf centre), each n floats
__global__ void gather_kernel(const float* __restrict__ pos, const float* __restrict__ gam,
                              const uint32_t* __restrict__ perm,
                              const uint32_t* __restrict__ keys, int64_t n, double lo,
                              double a, float* __restrict__ out, int64_t ostride, int64_t ooff) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = perm[k];
        const uint32_t key = keys[k];
        const uint32_t c[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const double ctr = lo + ((double)c[ax] + 0.5) * a;
            out[ax * ostride + ooff + k] = (float)((double)__ldg(pos + ax * n + i) - ctr);
            out[(3 + ax) * ostride + ooff + k] = __ldg(gam + ax * n + i);
        }
    }
}

int grid_for(int64_t n, int bs) {
    int64_t g = (n + bs - 1) / bs;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace

void launch_keys(const float* pos, int64_t n, Geom g, uint32_t* keys, uint32_t* vals,
                 int* err_flag, cudaStream_t st) {
    const int side = 1 << g.depth;
    const float inv = (float)((double)side / (double)g.len);
    const float hi = g.lo + g.len;
    keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(pos, n, g.lo, hi, inv, side, keys, vals,
                                                  err_flag);
}

size_t radix_temp_bytes(int64_t n) {
    const int64_t nb = (n + RTILE - 1) / RTILE;
    return sizeof(uint32_t) * ((size_t)nb * RBINS + RBINS);
}

void launch_radix_sort(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                       int64_t n, int key_bits, void* temp, cudaStream_t st,
                       uint32_t** keys_out, uint32_t** vals_out, int* n_launch) {
    const int nb = (int)((n + RTILE - 1) / RTILE);
    uint32_t* counts = (uint32_t*)temp;
    uint32_t* totals = counts + (size_t)nb * RBINS;
    uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
    const int passes = key_bits <= 0 ? 1 : (key_bits + RB - 1) / RB;
    const int width = key_bits <= 0 ? 1 : (key_bits + passes - 1) / passes;  // <= RB
    for (int shift = 0, pass = 0; pass < passes; shift += width, ++pass) {
        const int nbins = 1 << width;
        radix_count<<<nb, 256, 0, st>>>(ki, n, shift, nbins, counts, nb);
        radix_scan_rows<<<nbins, 256, 0, st>>>(counts, nb, totals);
        radix_scan_totals<<<1, 256, 0, st>>>(totals, nbins);
        radix_scatter<<<nb, 256, 0, st>>>(ki, vi, n, shift, nbins, counts, totals, nb, ko, vo);
        *n_launch += 4;
        uint32_t* t = ki;
        ki = ko;
        ko = t;
        t = vi;
        vi = vo;
        vo = t;
    }
    *keys_out = ki;
    *vals_out = vi;
}

void launch_leaf_ranges(const uint32_t* keys_sorted, int64_t n, int depth, int* leaf_start,
                        cudaStream_t st) {
    leaf_ranges_kernel<<<grid_for(n + 1, 256), 256, 0, st>>>(keys_sorted, n,
                                                            (int64_t)1 << (3 * depth), leaf_start);
}

namespace {
__global__ void gather1_kernel(const float* __restrict__ in, const uint32_t* __restrict__ perm,
                               int64_t n, float* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        out[k] = in[perm[k]];
}
}  // namespace

void launch_gather1(const float* in, const uint32_t* perm, int64_t n, float* out,
                    cudaStream_t st) {
    gather1_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, perm, n, out);
}

void launch_gather(const float* pos, const float* gamma, const uint32_t* perm,
                   const uint32_t* keys_sorted, int64_t n, Geom g, float* sorted6,
                   int64_t ostride, int64_t ooff, cudaStream_t st) {
    const double a = g.len_d / (double)(1 << g.depth);
    gather_kernel<<<grid_for(n, 256), 256, 0, st>>>(pos, gamma, perm, keys_sorted, n, g.lo_d, a,
                                                    sorted6, ostride, ooff);
}

}  // namespace vfmm
