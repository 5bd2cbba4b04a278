/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, double-precision CPU oracle for the periodic regularized
 * Biot-Savart velocity and vortex-stretching sums of Yokota & Barba,
 * arXiv:1110.2921.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product in paper_1110_2921_b200/ (which must never call it).
 *
 * What it computes (the plain definition):
 *   d = x_i - x_j - n*len,  r = |d|,  rho = r / (sqrt(2) sigma)
 *   zeta(r) = (2 pi sigma^2)^(-3/2) exp(-rho^2)              PAPER.md:76  Eq.(4)
 *   g(r)    = erf(rho) - (2/sqrt(pi)) rho exp(-rho^2)          PAPER.md:86  Eq.(6)
 *   G = 1/(4 pi r)
 *   f(r) = g/(4 pi r^3)   [gamma_j x grad G g = f gamma_j x d, physical sign: reading R1]
 *   q(r) = f'(r)/r = (zeta - 3 f)/r^2                          (g' = 4 pi r^2 zeta)
 *   u_i      = sum_n sum_j f (gamma_j x d)                      PAPER.md:81  Eq.(5)
 *   dgamma_i = sum_n sum_j [ f (gamma_j x gamma_i)
 *                          + q (gamma_i . d)(gamma_j x d) ]     PAPER.md:100 Eq.(8), classical (R2)
 *   transpose scheme (scheme=1): f (gamma_i x gamma_j) + q (gamma_i . (gamma_j x d)) d
 *   images n in the cube {-m..m}^3, m = (3^L - 1)/2, L = image_levels
 *   (L = 3 -> 27^3 boxes = "3^3 x 3^3 x 3^3 - 1" images); L = 0 -> free space.
 *
 * Kernel evaluation branches (all exact up to double rounding):
 *   r == 0        : limits f(0) = zeta0/3, q(0) = -zeta0/(5 sigma^2)
 *   rho < 0.25    : 8-term Taylor series in rho^2 (the closed form cancels there)
 *   r >= 12 sigma : g = 1, zeta = 0 to double precision (1-g < 1e-32)
 *   otherwise     : closed form with erf()/exp() from libm
 *
 * Also: vfmm_oracle_morton, the plain definition of the Morton-ordered
 * uniform octree (quantize, interleave, stable sort, leaf ranges), to be
 * compared bit-exactly.  Compiled with -ffp-contract=off (no FMA contraction)
 * so FP32 quantization is a single RN-even subtract and multiply.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846264338327950288

/* ---- scalar kernels ------------------------------------------------------ */

/* zeta, g, f, q at distance r (r >= 0) for core radius sigma > 0, given
   zeta0 = (2 pi sigma^2)^(-3/2) (hoisted out of the pair loops: the same double value). */
static inline void or_kernels(double r, double sigma, double zeta0, double* zeta, double* g,
                              double* f, double* q)
{
    const double rho2 = r * r / (2.0 * sigma * sigma);
    const double rho = sqrt(rho2);
    if (r == 0.0) {
        *zeta = zeta0;
        *g = 0.0;
        *f = zeta0 / 3.0;
        *q = -zeta0 / (5.0 * sigma * sigma);
        return;
    }
    if (rho < 0.25) {
        /* f = zeta0 sum_{k>=0} (-rho^2)^k / (k! (2k+3))
           q = (zeta0/sigma^2) sum_{k>=1} (-1)^k rho^(2k-2) / ((k-1)! (2k+3)) */
        double sf = 0.0, sq = 0.0, term = 1.0; /* term = (-rho^2)^k / k! */
        for (int k = 0; k < 8; ++k) {
            sf += term / (2.0 * k + 3.0);
            term *= -rho2 / (double)(k + 1);
        }
        term = -1.0; /* (-1)^k rho^(2k-2)/(k-1)! at k = 1 */
        for (int k = 1; k <= 8; ++k) {
            sq += term / (2.0 * k + 3.0);
            term *= -rho2 / (double)k;
        }
        *zeta = zeta0 * exp(-rho2);
        *f = zeta0 * sf;
        *q = zeta0 / (sigma * sigma) * sq;
        *g = (*f) * 4.0 * OR_PI * r * r * r;
        return;
    }
    if (r >= 12.0 * sigma) {
        *zeta = 0.0;
        *g = 1.0;
        *f = 1.0 / (4.0 * OR_PI * r * r * r);
        *q = -3.0 * (*f) / (r * r);
        return;
    }
    const double e = exp(-rho2);
    *zeta = zeta0 * e;
    *g = erf(rho) - 2.0 / sqrt(OR_PI) * rho * e;
    *f = (*g) / (4.0 * OR_PI * r * r * r);
    *q = (*zeta - 3.0 * (*f)) / (r * r);
}

static double or_zeta0(double sigma) { return pow(2.0 * OR_PI * sigma * sigma, -1.5); }

/* Returns zeta, g, f, q at distance r (r >= 0) for core radius sigma > 0. */
void vfmm_oracle_kernels(double r, double sigma, double* zeta, double* g, double* f, double* q)
{
    or_kernels(r, sigma, or_zeta0(sigma), zeta, g, f, q);
}

/* ---- direct sum ----------------------------------------------------------- */
/* One source-target pair's contribution (PAPER.md:81 Eq. 5, :100 Eq. 8):
   c = gamma_j x d;  u += f c;
   classical (scheme 0): s += f (gamma_j x gamma_i) + q (gamma_i . d) c
   transpose (scheme 1): s += f (gamma_i x gamma_j) + q (gamma_i . c) d */
static inline void or_pair(int scheme, double f, double q, double d0, double d1, double d2,
                           double gj0, double gj1, double gj2, const double gi[3], double u[3],
                           double s[3])
{
    const double c0 = gj1 * d2 - gj2 * d1;
    const double c1 = gj2 * d0 - gj0 * d2;
    const double c2 = gj0 * d1 - gj1 * d0;
    u[0] += f * c0;
    u[1] += f * c1;
    u[2] += f * c2;
    if (scheme == 0) {
        const double gd = gi[0] * d0 + gi[1] * d1 + gi[2] * d2;
        s[0] += f * (gj1 * gi[2] - gj2 * gi[1]) + q * gd * c0;
        s[1] += f * (gj2 * gi[0] - gj0 * gi[2]) + q * gd * c1;
        s[2] += f * (gj0 * gi[1] - gj1 * gi[0]) + q * gd * c2;
    } else {
        const double gc = gi[0] * c0 + gi[1] * c1 + gi[2] * c2;
        s[0] += f * (gi[1] * gj2 - gi[2] * gj1) + q * gc * d0;
        s[1] += f * (gi[2] * gj0 - gi[0] * gj2) + q * gc * d1;
        s[2] += f * (gi[0] * gj1 - gi[1] * gj0) + q * gc * d2;
    }
}


/*
 * n_src sources (SoA 3 x n_src doubles: x[0..n), y[..], z[..]).
 * Targets: if tgt_idx != NULL, target t is source tgt_idx[t] (its position and gamma);
 *          else target t is the probe (tgt_pos[t + k n_tgt], tgt_gam[...]).
 * vel, dgam: SoA 3 x n_tgt, overwritten.
 * Returns 0, or -1 on bad parameters.
 */
/* The direct sum with the core radius of every source given (sig_src[j], Eq. 6 has sigma_j,
   PAPER.md:86; zeta0 per source) or uniform (sig_src == NULL: sigma). */
static int or_eval(int64_t n_src, const double* src_pos, const double* src_gam,
                   double sigma, const double* sig_src, double box_lo, double box_len,
                   int image_levels, int scheme, int64_t n_tgt, const int64_t* tgt_idx,
                   const double* tgt_pos, const double* tgt_gam, double* vel, double* dgam,
                   int nthreads)
{
    (void)box_lo; /* only differences of positions enter the sum */
    if (n_src < 1 || !(sigma > 0.0) || !(box_len > 0.0) || image_levels < 0 ||
        image_levels > 6 || (scheme != 0 && scheme != 1) || n_tgt < 0)
        return -1;
    double* z0_src = NULL;
    if (sig_src) {
        for (int64_t j = 0; j < n_src; ++j)
            if (!(sig_src[j] > 0.0)) return -1;
        z0_src = (double*)malloc(sizeof(double) * (size_t)n_src);
        if (!z0_src) return -2;
        for (int64_t j = 0; j < n_src; ++j) z0_src[j] = or_zeta0(sig_src[j]);
    }
    if (tgt_idx == NULL && (tgt_pos == NULL || tgt_gam == NULL)) return -1;
    int m = 0;
    for (int l = 0; l < image_levels; ++l) m = 3 * m + 1; /* m = (3^L - 1)/2 */
    if (image_levels == 0) m = 0;
    const int side = 2 * m + 1;
    const int64_t n_img = (int64_t)side * side * side;
    const int periodic = image_levels > 0;
    const double zeta0 = or_zeta0(sigma);

#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n_tgt; ++t) {
        double xi[3], gi[3];
        for (int k = 0; k < 3; ++k) {
            if (tgt_idx) {
                xi[k] = src_pos[tgt_idx[t] + k * n_src];
                gi[k] = src_gam[tgt_idx[t] + k * n_src];
            } else {
                xi[k] = tgt_pos[t + k * n_tgt];
                gi[k] = tgt_gam[t + k * n_tgt];
            }
        }
        double U[3] = {0, 0, 0}, S[3] = {0, 0, 0};
        for (int64_t im = 0; im < (periodic ? n_img : 1); ++im) {
            /* lexicographic image order: nx slowest */
            const int nx = periodic ? (int)(im / ((int64_t)side * side)) - m : 0;
            const int ny = periodic ? (int)((im / side) % side) - m : 0;
            const int nz = periodic ? (int)(im % side) - m : 0;
            const double sx = nx * box_len, sy = ny * box_len, sz = nz * box_len;
            double u[3] = {0, 0, 0}, s[3] = {0, 0, 0};
            for (int64_t j = 0; j < n_src; ++j) {
                const double d0 = xi[0] - src_pos[j] - sx;
                const double d1 = xi[1] - src_pos[j + n_src] - sy;
                const double d2 = xi[2] - src_pos[j + 2 * n_src] - sz;
                const double r = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
                double zeta, g, f, q;
                if (sig_src)
                    or_kernels(r, sig_src[j], z0_src[j], &zeta, &g, &f, &q);
                else
                    or_kernels(r, sigma, zeta0, &zeta, &g, &f, &q);
                or_pair(scheme, f, q, d0, d1, d2, src_gam[j], src_gam[j + n_src],
                        src_gam[j + 2 * n_src], gi, u, s);
            }
            for (int k = 0; k < 3; ++k) {
                U[k] += u[k];
                S[k] += s[k];
            }
        }
        for (int k = 0; k < 3; ++k) {
            vel[t + k * n_tgt] = U[k];
            dgam[t + k * n_tgt] = S[k];
        }
    }
    free(z0_src);
    return 0;
}

int vfmm_oracle_eval(int64_t n_src, const double* src_pos, const double* src_gam,
                     double sigma, double box_lo, double box_len, int image_levels, int scheme,
                     int64_t n_tgt, const int64_t* tgt_idx, const double* tgt_pos,
                     const double* tgt_gam, double* vel, double* dgam, int nthreads)
{
    return or_eval(n_src, src_pos, src_gam, sigma, NULL, box_lo, box_len, image_levels, scheme,
                   n_tgt, tgt_idx, tgt_pos, tgt_gam, vel, dgam, nthreads);
}

/* Per-particle core radius sigma_j of the source (Eq. 6 as written, sigma_j; NEXT-4):
   sig_src[n_src] > 0; otherwise as vfmm_oracle_eval. */
int vfmm_oracle_eval_sigma(int64_t n_src, const double* src_pos, const double* src_gam,
                           const double* sig_src, double box_lo, double box_len,
                           int image_levels, int scheme, int64_t n_tgt, const int64_t* tgt_idx,
                           const double* tgt_pos, const double* tgt_gam, double* vel,
                           double* dgam, int nthreads)
{
    if (!sig_src) return -1;
    return or_eval(n_src, src_pos, src_gam, 1.0, sig_src, box_lo, box_len, image_levels, scheme,
                   n_tgt, tgt_idx, tgt_pos, tgt_gam, vel, dgam, nthreads);
}

/*
 * Same sum, same result bit for bit, loops reordered for large sampled-target runs
 * (tests/golden reference values at 27^3 images): targets go in batches of OR_TB; for each
 * image (in parallel) one pass over the sources serves the whole batch, each target keeping
 * its own per-image partial sums in the same j order as vfmm_oracle_eval; the per-image
 * partials are then added in the same lexicographic image order.  Only the loop nest differs,
 * so every floating-point operation and its order per target is vfmm_oracle_eval's
 * (tests/test_oracle_pins.py::test_batched_oracle_is_bitwise_the_plain_one).
 * Same arguments and return value as vfmm_oracle_eval; -2 if the partials cannot be allocated.
 */
#define OR_TB 16
int vfmm_oracle_eval_batched(int64_t n_src, const double* src_pos, const double* src_gam,
                             double sigma, double box_lo, double box_len, int image_levels,
                             int scheme, int64_t n_tgt, const int64_t* tgt_idx,
                             const double* tgt_pos, const double* tgt_gam, double* vel,
                             double* dgam, int nthreads)
{
    (void)box_lo;
    if (n_src < 1 || !(sigma > 0.0) || !(box_len > 0.0) || image_levels < 0 ||
        image_levels > 6 || (scheme != 0 && scheme != 1) || n_tgt < 0)
        return -1;
    if (tgt_idx == NULL && (tgt_pos == NULL || tgt_gam == NULL)) return -1;
    int m = 0;
    for (int l = 0; l < image_levels; ++l) m = 3 * m + 1;
    if (image_levels == 0) m = 0;
    const int side = 2 * m + 1;
    const int periodic = image_levels > 0;
    const int64_t n_img = periodic ? (int64_t)side * side * side : 1;
    const double zeta0 = or_zeta0(sigma);
    const double far_r = 12.0 * sigma;
    double* part = (double*)malloc(sizeof(double) * 6 * OR_TB * (size_t)n_img);
    if (!part) return -2;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t t0 = 0; t0 < n_tgt; t0 += OR_TB) {
        const int nb = (int)((n_tgt - t0) < OR_TB ? (n_tgt - t0) : OR_TB);
        double xi[3][OR_TB], gi[3][OR_TB];
        for (int b = 0; b < OR_TB; ++b) { /* unused lanes repeat the batch's first target */
            const int64_t t = t0 + (b < nb ? b : 0);
            for (int k = 0; k < 3; ++k) {
                xi[k][b] = tgt_idx ? src_pos[tgt_idx[t] + k * n_src] : tgt_pos[t + k * n_tgt];
                gi[k][b] = tgt_idx ? src_gam[tgt_idx[t] + k * n_src] : tgt_gam[t + k * n_tgt];
            }
        }
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t im = 0; im < n_img; ++im) {
            const int nx = periodic ? (int)(im / ((int64_t)side * side)) - m : 0;
            const int ny = periodic ? (int)((im / side) % side) - m : 0;
            const int nz = periodic ? (int)(im % side) - m : 0;
            const double sx = nx * box_len, sy = ny * box_len, sz = nz * box_len;
            double u[OR_TB][3], s[OR_TB][3];
            memset(u, 0, sizeof u);
            memset(s, 0, sizeof s);
            for (int64_t j = 0; j < n_src; ++j) {
                const double xj0 = src_pos[j], xj1 = src_pos[j + n_src], xj2 = src_pos[j + 2 * n_src];
                const double gj0 = src_gam[j], gj1 = src_gam[j + n_src], gj2 = src_gam[j + 2 * n_src];
                double d0[OR_TB], d1[OR_TB], d2[OR_TB], r[OR_TB];
                int n_far = 0;
                for (int b = 0; b < OR_TB; ++b) {
                    d0[b] = xi[0][b] - xj0 - sx;
                    d1[b] = xi[1][b] - xj1 - sy;
                    d2[b] = xi[2][b] - xj2 - sz;
                    r[b] = sqrt(d0[b] * d0[b] + d1[b] * d1[b] + d2[b] * d2[b]);
                    n_far += r[b] >= far_r;
                }
                if (n_far == OR_TB) { /* or_kernels' r >= 12 sigma branch, for every lane */
                    for (int b = 0; b < OR_TB; ++b) {
                        const double f = 1.0 / (4.0 * OR_PI * r[b] * r[b] * r[b]);
                        const double q = -3.0 * f / (r[b] * r[b]);
                        const double g3[3] = {gi[0][b], gi[1][b], gi[2][b]};
                        or_pair(scheme, f, q, d0[b], d1[b], d2[b], gj0, gj1, gj2, g3, u[b], s[b]);
                    }
                } else {
                    for (int b = 0; b < OR_TB; ++b) {
                        double zeta, g, f, q;
                        or_kernels(r[b], sigma, zeta0, &zeta, &g, &f, &q);
                        const double g3[3] = {gi[0][b], gi[1][b], gi[2][b]};
                        or_pair(scheme, f, q, d0[b], d1[b], d2[b], gj0, gj1, gj2, g3, u[b], s[b]);
                    }
                }
            }
            double* P = part + (size_t)im * 6 * OR_TB;
            for (int b = 0; b < OR_TB; ++b)
                for (int k = 0; k < 3; ++k) {
                    P[b * 6 + k] = u[b][k];
                    P[b * 6 + 3 + k] = s[b][k];
                }
        }
        for (int b = 0; b < nb; ++b) {
            double U[3] = {0, 0, 0}, S[3] = {0, 0, 0};
            for (int64_t im = 0; im < n_img; ++im) /* lexicographic image order */
                for (int k = 0; k < 3; ++k) {
                    U[k] += part[(size_t)im * 6 * OR_TB + b * 6 + k];
                    S[k] += part[(size_t)im * 6 * OR_TB + b * 6 + 3 + k];
                }
            for (int k = 0; k < 3; ++k) {
                vel[t0 + b + k * n_tgt] = U[k];
                dgam[t0 + b + k * n_tgt] = S[k];
            }
        }
    }
    free(part);
    return 0;
}

/* ---- Morton-ordered uniform octree (bit-exact contract) ------------------ */

typedef struct {
    uint32_t key;
    uint32_t idx;
} or_kv;

static int or_cmp(const void* a, const void* b)
{
    const or_kv* x = (const or_kv*)a;
    const or_kv* y = (const or_kv*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0); /* ties keep input order */
}

/*
 * Quantize each axis: i = (int)floorf((x - lo) * inv), inv = (float)(2^L / (double)len),
 * clamped to [0, 2^L - 1]; key bit 3b = bit b of ix, 3b+1 = iy, 3b+2 = iz.
 * keys_sorted, perm: n entries; leaf_start: 8^L + 1 entries (leaf_start[c] = #keys < c).
 * Returns 0, -1 bad params, -2 a position outside [lo, lo+len) or non-finite.
 */
int vfmm_oracle_morton(int64_t n, const float* pos, int depth, float lo, float len,
                       uint32_t* keys_sorted, uint32_t* perm, int32_t* leaf_start)
{
    if (n < 0 || depth < 1 || depth > 10 || !(len > 0.0f)) return -1;
    const uint32_t side = 1u << depth;
    const float inv = (float)((double)side / (double)len);
    const float hi = lo + len;
    or_kv* kv = (or_kv*)malloc(sizeof(or_kv) * (size_t)(n > 0 ? n : 1));
    if (!kv) return -1;
    int err = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t c[3];
        for (int a = 0; a < 3; ++a) {
            const float x = pos[i + a * n];
            if (!(x >= lo && x < hi)) err = 1; /* also catches NaN */
            volatile float dx = x - lo;        /* single RN-even subtract */
            volatile float sx = dx * inv;      /* single RN-even multiply */
            float fl = floorf(sx);
            int32_t q = (fl >= 0.0f) ? (int32_t)fl : 0;
            if (!(fl >= 0.0f)) q = 0;
            if (q > (int32_t)side - 1) q = (int32_t)side - 1;
            c[a] = (uint32_t)q;
        }
        uint32_t key = 0;
        for (int b = 0; b < depth; ++b) {
            key |= ((c[0] >> b) & 1u) << (3 * b);
            key |= ((c[1] >> b) & 1u) << (3 * b + 1);
            key |= ((c[2] >> b) & 1u) << (3 * b + 2);
        }
        kv[i].key = key;
        kv[i].idx = (uint32_t)i;
    }
    qsort(kv, (size_t)n, sizeof(or_kv), or_cmp);
    for (int64_t i = 0; i < n; ++i) {
        keys_sorted[i] = kv[i].key;
        perm[i] = kv[i].idx;
    }
    const int64_t nleaf = (int64_t)1 << (3 * depth);
    int64_t k = 0;
    for (int64_t c = 0; c <= nleaf; ++c) { /* lower_bound */
        while (k < n && (int64_t)kv[k].key < c) ++k;
        leaf_start[c] = (int32_t)k;
    }
    free(kv);
    return err ? -2 : 0;
}
