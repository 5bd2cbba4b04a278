// vfmm_internal.h -- internal declarations of libvfmm (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/vfmm.h"

namespace vfmm {

constexpr int kPMax = VFMM_PMAX;

inline int ncoef(int p) { return (p + 1) * (p + 1); }

// Runs f() once per CUDA device (the current one), thread-safe.  Kernel attributes such as
// cudaFuncAttributeMaxDynamicSharedMemorySize are per device, so a process driving several
// devices must set them on each.
struct PerDeviceOnce {
    std::mutex m;
    uint64_t done = 0;
    template <class F>
    void operator()(F&& f) {
        int d = 0;
        cudaGetDevice(&d);
        std::lock_guard<std::mutex> g(m);
        if (d < 0 || d > 63 || ((done >> d) & 1)) return;
        f();
        done |= uint64_t(1) << d;
    }
};

// Named NVTX range over the host-side enqueue of one pipeline phase, so that profilers
// attribute the phase's kernel launches to it (nsys timeline, `ncu --nvtx --nvtx-include
// "vfmm/p2p/"`).  With no profiler attached, push and pop return at once.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
    void next(const char* name) {
        nvtxRangePop();
        nvtxRangePushA(name);
    }
};

// Packed real coefficient index:
// Re(n,0) -> n^2 ; Re(n,m) -> n^2 + 2m - 1 ; Im(n,m) -> n^2 + 2m   (m >= 1)
__host__ __device__ inline int pk_re(int n, int m) { return n * n + (m == 0 ? 0 : 2 * m - 1); }
__host__ __device__ inline int pk_im(int n, int m) { return n * n + 2 * m; }

// cells at level l start at (8^l - 1) / 7 in the concatenated per-level arrays
inline int64_t level_offset(int l) { return ((int64_t(1) << (3 * l)) - 1) / 7; }

// ---------------------------------------------------------------------------
// host operator tables (ops_host.cpp), double precision, packed real form
// ---------------------------------------------------------------------------
struct HostOps {
    int p = 0, nc = 0;
    int KP = 0;  // K padded to a multiple of 16
    int NR = 0;  // rows padded to a multiple of 128
    // all matrices stored transposed+padded: T[k * NR + r] = A[r][k]  (float32 upload)
    std::vector<float> m2m;  // 8 child matrices   [8][KP][NR]
    std::vector<float> l2l;  // 8 child matrices   [8][KP][NR]
    std::vector<float> m2l;  // 343 offset slots   [343][KP][NR] (|o|inf <= 1 slots zero)
    std::vector<float> per;  // periodic operator  [1][KP][NR]
    std::vector<double> per_d;  // periodic operator row-major [nc][nc] (double, for tests)
    // tensor-core M2L operands (nc <= 128): row-major [343][128 r][128 k], 3xTF32 split
    std::vector<float> m2l_tc_hi, m2l_tc_lo;
    // 3xFP16 split of the balanced operators Ahat = T / (rs[r] cs[k]) (rs, cs powers of 2,
    // |Ahat| <= 1), IEEE half bit patterns, row-major [343][h16_nr][h16_kp]: 128 x 128 for
    // nc <= 128, else 256 rows x (64 ceil(nc / 64)) columns (p <= 15)
    std::vector<uint16_t> m2l_h16_hi, m2l_h16_lo;
    std::vector<float> h16_rs, h16_cs;  // [h16_nr] row / [h16_kp] column scales
    int h16_nr = 128, h16_kp = 128;
    // L2P: D[k][q] = sum_t coef[t] L[src[t]] for t in [rowptr[k 12 + q], rowptr[k 12 + q + 1]),
    // src indexing the 3 nc packed coefficients of a leaf (q: curl psi 3, grad u 9; k < p^2);
    // rows padded to multiples of 4 terms with zeros (uploaded as 32-bit terms: src in the low
    // 16 bits, the coefficient -- sums of +-2^-k, exact in half -- in the high 16 bits)
    std::vector<int> l2p_rowptr, l2p_src;
    std::vector<float> l2p_coef;
};

// Build all operator tables for order p and image_levels (periodic operator is zero for
// image_levels < 2).  Deterministic, double precision.
void build_host_ops(int p, int image_levels, HostOps* out);

// M2L offset slot of o in {-3..3}^3
__host__ __device__ inline int m2l_slot(int ox, int oy, int oz) {
    return ((ox + 3) * 7 + (oy + 3)) * 7 + (oz + 3);
}

// ---------------------------------------------------------------------------
// kernels' launch wrappers (defined in .cu files); all async on `st`
// ---------------------------------------------------------------------------
struct Geom {
    float lo, len;   // box
    double lo_d, len_d;
    int depth;       // L
    int periodic;    // image_levels > 0
};

// tree.cu
void launch_keys(const float* pos, int64_t n, Geom g, uint32_t* keys, uint32_t* vals,
                 int* err_flag, cudaStream_t st);
size_t radix_temp_bytes(int64_t n);
void launch_radix_sort(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                       int64_t n, int key_bits, void* temp, cudaStream_t st,
                       uint32_t** keys_out, uint32_t** vals_out, int* n_launch);
void launch_leaf_ranges(const uint32_t* keys_sorted, int64_t n, int depth, int* leaf_start,
                        cudaStream_t st);
void launch_gather(const float* pos, const float* gamma, const uint32_t* perm,
                   const uint32_t* keys_sorted, int64_t n, Geom g, float* sorted6,
                   int64_t ostride, int64_t ooff, cudaStream_t st);

// out[k] = in[perm[k]] (one float per particle into Morton order)
void launch_gather1(const float* in, const uint32_t* perm, int64_t n, float* out,
                    cudaStream_t st);

// expansions.cu  (ranges: the owned part of the tree; whole tree for one rank)
void launch_p2m(const float* sorted6, int64_t n, const int* leaf_start, int p, float inv_a,
                float* M_leaf, int64_t leaf_lo, int64_t leaf_cnt, cudaStream_t st);
// returns the number of kernels launched; scratch (>= 8 x 3 nc x parents floats) enables the
// deterministic op split at coarse levels (< 296 tiles of 32 parents)
int launch_m2m(const float* ops_m2m, int p, int KP, int NR, const float* M_child, float* M_par,
               int level_par, int64_t plo, int64_t pcnt, float* scratch, size_t scratch_floats,
               cudaStream_t st);
void launch_l2l(const float* ops_l2l, int p, int KP, int NR, const float* L_par, float* L_child,
                int level_child, int64_t plo, int64_t pcnt, cudaStream_t st);
// returns the number of kernels launched; the scratch (if large enough) makes the coarse
// levels' op split deterministic (partials + zsum) instead of atomic
int launch_m2l(const float* ops_m2l, const int* il_slots, int p, int KP, int NR,
               const float* M_l, float* L_l, int level, int periodic, int64_t plo, int64_t pcnt,
               float* scratch, size_t scratch_floats, cudaStream_t st);
void launch_periodic(const float* ops_per, int p, int KP, int NR, const float* M0, float* L0,
                     cudaStream_t st);
struct L2PMap {
    const int* rowptr = nullptr;   // [12 p^2 + 1], multiples of 4
    const uint4* terms = nullptr;  // four terms per entry, each (src | half(coef) << 16)
};
void launch_l2p_combine(const L2PMap& map, const float* sorted6, const float* near6, const uint32_t* perm,
                        int64_t n, const int* leaf_start, int p, float a, const float* L_leaf,
                        int scheme, int use_near, int use_far, float* vel, float* dgam,
                        int64_t leaf_lo, int64_t leaf_cnt, int64_t gbase, int64_t nout,
                        cudaStream_t st);

// m2l_tc.cu (tcgen05: 3xTF32 or scaled 3xFP16)
struct TcOps {
    const void* hi = nullptr;  // [343][128][128] operator hi parts (float tf32 / half)
    const void* lo = nullptr;  // remainders
    const float* rs = nullptr; // f16: row scales [128]
    const float* cs = nullptr; // f16: column scales [128]
    const int4* groups = nullptr;  // [8][72] offset groups per target parity (m2l_groups)
    bool f16 = false;
    int nr = 128, kp = 128;  // operator layout [343][nr][kp] (f16 with (p+1)^2 > 128: 256 rows)
    bool lean = false;       // f16, (p+1)^2 <= 128: the 161 KB / 192-thread variant (T = 2)
};
// The 189 M2L offsets of target parity pi grouped by (source parent dx, dz, source parity):
// entry [pi][((dx+1) 3 + (dz+1)) 8 + pis] = {mask (bit dy+1 set if offset (dx, dy, dz, pis) is
// in the list) | (dx+1) << 4 | (dz+1) << 6 | pis << 8, slot(dy=-1), slot(0), slot(1)}
std::vector<int> m2l_groups();
bool m2l_tc_supported(int p, int level);
bool m2l_tc_shape_ok(const int box[6], int p);
int m2l_split_degree();  // lowest term degree run as hi x hi alone (m2l_tc.cu)
size_t m2l_tc_grid_floats(int level);
// maxbits: one zeroed uint32 per launch (f16: the level's max |cs[k] M_k|, as float bits)
int launch_m2l_tc(const TcOps& ops, const int* il_slots, int p, const float* M_l, float* L_l,
                  int level, int periodic, float* ghi, float* glo, uint32_t* maxbits,
                  const int box[6], cudaStream_t st);

// p2p.cu
struct KernelConsts {
    float inv2s2;        // 1 / (2 sigma^2)
    float neg_l2e_inv2s2;// -log2(e) / (2 sigma^2)
    float inv_s_sqrt2;   // 1 / (sqrt(2) sigma)
    float zeta0;         // (2 pi sigma^2)^(-3/2)
    float zeta0_over_s2; // zeta0 / sigma^2
    float r2_series;     // r^2 below which the Taylor series is used (rho^2 < 1/4)
    float t_scale;       // 1 / (2 sqrt(2) sigma): t = 1 / (1 + r t_scale) = 1/(1 + rho/2)
    float q_scale;       // 2 / (4 pi sqrt(pi) sqrt(2) sigma): rho term of (1 - g)/(4 pi)
    // packed fast path (p2p.cu fq_closed2): e_z = zeta0 e^{-rho^2} = 2^(r^2 neg_l2e_inv2s2 +
    // ez_off); (1 - g)/(4 pi) = -e_z Qn with Qn = qn_scale r + sum_k en[k] t^k (the erfcx
    // polynomial expanded in powers of t and scaled by -1/zeta0)
    float ez_off;        // log2(zeta0)
    float qn_scale;      // -q_scale / zeta0
    float en[6];
};
KernelConsts make_kernel_consts(float sigma);
void launch_p2p(const float* sorted6, int64_t n, const int* leaf_start, int depth, float a,
                int periodic, int scheme, KernelConsts kc, float* near6,
                unsigned long long* npairs, int64_t plo, int64_t pcnt, cudaStream_t st,
                bool lean = false);
// hybrid treecode, cell-particle half (p2p.cu)
size_t tree_groups_cap(int64_t n, int depth);
void launch_tree(const float* sorted6, int64_t n, const uint32_t* keys_sorted,
                 const int* leaf_start, int depth, float aL, int periodic, int scheme, int p,
                 int ncrit, float theta, const float* Mall, KernelConsts kc, int2* groups,
                 int* ngroups, unsigned long long* counters, float* near6, cudaStream_t st);
// rbf.cu (reinitialization): Gaussian sums over the ws-neighbour leaves, BLAS-1 for GMRES
void launch_gauss(const float* t6, int64_t nt, const int* tls, const float* s6, int64_t ns,
                  const int* sls, const float* sg, int depth, float a, int periodic, int ws,
                  float sigma, float* out, cudaStream_t st);
int rbf_ws(float a, float sigma);
size_t rbf_dot_part_doubles(int nv);
void launch_multidot(const float* X, int64_t xs, int nv, const float* Y, int64_t n, double* part,
                     double* dots, cudaStream_t st);
void launch_multiaxpy(const float* X, int64_t xs, int nv, const double* coef, float* Y, int64_t n,
                      cudaStream_t st);
void launch_scale3(const float* X, const float* Z, float* Y, int64_t n, const double al[3],
                   const double be[3], cudaStream_t st);
void launch_unpermute3(const float* in, const uint32_t* perm, int64_t n, float* out,
                       cudaStream_t st);

// step.cu: x += u dt (wrapped into the box when periodic), gamma += dgamma dt
void launch_euler_update(float* pos, float* gamma, const float* vel, const float* dgamma,
                         int64_t n, float dt, float lo, float len, int periodic, cudaStream_t st);
// per-particle core radius (Eq. 6's sigma_j): near field and DIRECT mode
void launch_p2p_sigma(const float* sorted6, const float* sorted_sig, int64_t n,
                      const int* leaf_start, int depth, float a, int periodic, int scheme,
                      float* near6, unsigned long long* npairs, int64_t plo, int64_t pcnt,
                      cudaStream_t st);
void launch_direct_sigma(const float* pos, const float* gamma, const float* sigma, int64_t n,
                         float len, int image_levels, int scheme, float* vel, float* dgam,
                         cudaStream_t st);
void launch_direct(const float* pos, const float* gamma, int64_t n, float len, int image_levels,
                   int scheme, KernelConsts kc, float* vel, float* dgam, cudaStream_t st);

}  // namespace vfmm
