// ops_host.cpp -- translation operators of the FMM, built once per context in double
// precision on the host ("nomenclature of Cheng et al."; Eqs. (10)-(11),
// PAPER.md:123-128), then rounded to float32 and uploaded.
//
// Solid harmonics, complex, m >= 0, by recurrence:
//   R_0^0 = 1, R_m^m = -(x+iy)/(2m) R_{m-1}^{m-1}, R_{m+1}^m = z R_m^m,
//   (n+m)(n-m) R_n^m = (2n-1) z R_{n-1}^m - r^2 R_{n-2}^m
//   I_0^0 = 1/r, I_m^m = -(2m-1)(x+iy)/r^2 I_{m-1}^{m-1}, I_{m+1}^m = (2m+1) z/r^2 I_m^m,
//   r^2 I_n^m = (2n-1) z I_{n-1}^m - (n-1-m)(n-1+m) I_{n-2}^m
//   R_n^{-m} = (-1)^m conj(R_n^m), I_n^{-m} = (-1)^m conj(I_n^m)
// with 1/|x-y| = sum conj(R_n^m(y)) I_n^m(x) (Eq. 10's M_j = rho^n Y_n^{-m}, S = r^{-n-1} Y_n^m).
//
// Scaled (level-independent) operators, cell width a:  Mt = M / a^n, Lt = L a^(n+1)
//   M2M (child c' -> parent c, d = (c'-c)/a_p):   Mt_p[n,m] = sum conj(R_k^l(d)) 2^-(n-k) Mt_c[n-k,m-l]
//   M2L (source at c_t + o a):                   Lt[n,m]   = sum (-1)^(n+m) I_{n+k}^{l-m}(-o) Mt[k,l]
//   L2L (parent c -> child c', d = (c'-c)/a_p):   Lt_c[n,m] = sum_{k>=n} 2^-(n+1) R_{k-n}^{l-m}(d) Lt_p[k,l]
//   periodic (unit box, rings of 3x supercells): see build_periodic below.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <complex>
#include <map>
#include <stdexcept>
#include <utility>
#include <vector>

#include "vfmm_internal.h"

namespace vfmm {
namespace {

using cd = std::complex<double>;

inline int fidx(int n, int m) { return n * n + n + m; }  // full complex index, |m| <= n

// regular solid harmonics R_n^m(x) for all |m| <= n <= p
void solid_R(double x, double y, double z, int p, std::vector<cd>& out) {
    out.assign((p + 1) * (p + 1), cd(0, 0));
    const double r2 = x * x + y * y + z * z;
    const cd xy(x, y);
    cd diag(1.0, 0.0);  // R_m^m
    for (int m = 0; m <= p; ++m) {
        if (m > 0) diag = -xy / (2.0 * m) * diag;
        cd rm2 = diag, rm1(0, 0);
        out[fidx(m, m)] = diag;
        if (m + 1 <= p) {
            rm1 = z * diag;
            out[fidx(m + 1, m)] = rm1;
        }
        for (int n = m + 2; n <= p; ++n) {
            cd rn = ((2.0 * n - 1.0) * z * rm1 - r2 * rm2) / double((n + m) * (n - m));
            out[fidx(n, m)] = rn;
            rm2 = rm1;
            rm1 = rn;
        }
    }
    for (int n = 1; n <= p; ++n)
        for (int m = 1; m <= n; ++m)
            out[fidx(n, -m)] = ((m & 1) ? -1.0 : 1.0) * std::conj(out[fidx(n, m)]);
}

// irregular solid harmonics I_n^m(x) for all |m| <= n <= p
void solid_I(double x, double y, double z, int p, std::vector<cd>& out) {
    out.assign((p + 1) * (p + 1), cd(0, 0));
    const double r2 = x * x + y * y + z * z;
    const double ir2 = 1.0 / r2;
    const cd xy(x, y);
    cd diag(1.0 / std::sqrt(r2), 0.0);  // I_m^m
    for (int m = 0; m <= p; ++m) {
        if (m > 0) diag = -(2.0 * m - 1.0) * xy * ir2 * diag;
        cd im2 = diag, im1(0, 0);
        out[fidx(m, m)] = diag;
        if (m + 1 <= p) {
            im1 = (2.0 * m + 1.0) * z * ir2 * diag;
            out[fidx(m + 1, m)] = im1;
        }
        for (int n = m + 2; n <= p; ++n) {
            cd in = ((2.0 * n - 1.0) * z * im1 - double((n - 1 - m) * (n - 1 + m)) * im2) * ir2;
            out[fidx(n, m)] = in;
            im2 = im1;
            im1 = in;
        }
    }
    for (int n = 1; n <= p; ++n)
        for (int m = 1; m <= n; ++m)
            out[fidx(n, -m)] = ((m & 1) ? -1.0 : 1.0) * std::conj(out[fidx(n, m)]);
}

// A: full complex matrix (nc x nc, row-major, acting on full coefficient vectors).
// Returns the packed real matrix P (nc x nc row-major): P = pack o A o unpack.
std::vector<double> pack_matrix(const std::vector<cd>& A, int p) {
    const int nc = (p + 1) * (p + 1);
    std::vector<double> P((size_t)nc * nc, 0.0);
    for (int n = 0; n <= p; ++n) {
        for (int m = 0; m <= n; ++m) {
            // unpacked images of the packed basis vectors (Re / Im of coefficient (n,m))
            for (int part = 0; part < (m == 0 ? 1 : 2); ++part) {
                const int j = part == 0 ? pk_re(n, m) : pk_im(n, m);
                std::vector<cd> col(nc, cd(0, 0));
                const double sg = (m & 1) ? -1.0 : 1.0;
                for (int r = 0; r < nc; ++r) {
                    cd v = A[(size_t)r * nc + fidx(n, m)] * (part == 0 ? cd(1, 0) : cd(0, 1));
                    if (m > 0)
                        v += A[(size_t)r * nc + fidx(n, -m)] * sg * (part == 0 ? cd(1, 0) : cd(0, -1));
                    col[r] = v;
                }
                for (int nn = 0; nn <= p; ++nn) {
                    P[(size_t)pk_re(nn, 0) * nc + j] = col[fidx(nn, 0)].real();
                    for (int mm = 1; mm <= nn; ++mm) {
                        P[(size_t)pk_re(nn, mm) * nc + j] = col[fidx(nn, mm)].real();
                        P[(size_t)pk_im(nn, mm) * nc + j] = col[fidx(nn, mm)].imag();
                    }
                }
            }
        }
    }
    return P;
}

// full complex M2M matrix: M_parent[n,m] += conj(R_k^l(d)) s^(n-k) M_child[n-k, m-l]
std::vector<cd> m2m_full(double dx, double dy, double dz, int p, double s) {
    const int nc = (p + 1) * (p + 1);
    std::vector<cd> R;
    solid_R(dx, dy, dz, p, R);
    std::vector<cd> A((size_t)nc * nc, cd(0, 0));
    for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m)
            for (int k = 0; k <= n; ++k)
                for (int l = -k; l <= k; ++l) {
                    const int nn = n - k, mm = m - l;
                    if (std::abs(mm) > nn) continue;
                    A[(size_t)fidx(n, m) * nc + fidx(nn, mm)] +=
                        std::conj(R[fidx(k, l)]) * std::pow(s, nn);
                }
    return A;
}

// full complex M2L matrix: L[n,m] = sum (-1)^(n+m) I_{n+k}^{l-m}(D) M[k,l]
std::vector<cd> m2l_full(double Dx, double Dy, double Dz, int p) {
    const int nc = (p + 1) * (p + 1);
    std::vector<cd> I;
    solid_I(Dx, Dy, Dz, 2 * p, I);
    std::vector<cd> A((size_t)nc * nc, cd(0, 0));
    for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
            const double sg = ((n + m) & 1) ? -1.0 : 1.0;
            for (int k = 0; k <= p; ++k)
                for (int l = -k; l <= k; ++l)
                    A[(size_t)fidx(n, m) * nc + fidx(k, l)] = sg * I[fidx(n + k, l - m)];
        }
    return A;
}

// full complex L2L matrix: L_child[n,m] = sum_{k>=n} s^(n+1) R_{k-n}^{l-m}(d) L_parent[k,l]
std::vector<cd> l2l_full(double dx, double dy, double dz, int p, double s) {
    const int nc = (p + 1) * (p + 1);
    std::vector<cd> R;
    solid_R(dx, dy, dz, p, R);
    std::vector<cd> A((size_t)nc * nc, cd(0, 0));
    for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m)
            for (int k = n; k <= p; ++k)
                for (int l = -k; l <= k; ++l) {
                    const int j = k - n, t = l - m;
                    if (std::abs(t) > j) continue;
                    A[(size_t)fidx(n, m) * nc + fidx(k, l)] += std::pow(s, n + 1) * R[fidx(j, t)];
                }
    return A;
}

std::vector<double> matmul(const std::vector<double>& A, const std::vector<double>& B, int nc) {
    std::vector<double> C((size_t)nc * nc, 0.0);
    for (int i = 0; i < nc; ++i)
        for (int k = 0; k < nc; ++k) {
            const double a = A[(size_t)i * nc + k];
            if (a == 0.0) continue;
            for (int j = 0; j < nc; ++j) C[(size_t)i * nc + j] += a * B[(size_t)k * nc + j];
        }
    return C;
}

// Periodic far-field operator in unit-box scaled form: Lt_0 += P Mt_0, covering all
// images of the image cube {-m..m}^3 outside the near 3^3 block (reading R5):
//   ring k = 0..levels-2: supercells of width 3^k at offsets 3^k n, n in {-4..4}^3 \ {-1..1}^3
//   supercell_{k+1} = sum over d in {-1,0,1}^3 of M2M(shift d 3^k) supercell_k
std::vector<double> build_periodic(int p, int levels) {
    const int nc = (p + 1) * (p + 1);
    std::vector<double> P((size_t)nc * nc, 0.0);
    if (levels < 2) return P;
    std::vector<double> S((size_t)nc * nc, 0.0);  // supercell_k = S * Mt_0
    for (int i = 0; i < nc; ++i) S[(size_t)i * nc + i] = 1.0;
    for (int k = 0; k <= levels - 2; ++k) {
        const double w = std::pow(3.0, k);
        std::vector<double> ring((size_t)nc * nc, 0.0);
        for (int a = -4; a <= 4; ++a)
            for (int b = -4; b <= 4; ++b)
                for (int c = -4; c <= 4; ++c) {
                    if (std::max(std::abs(a), std::max(std::abs(b), std::abs(c))) <= 1) continue;
                    auto T = pack_matrix(m2l_full(-a * w, -b * w, -c * w, p), p);
                    for (size_t i = 0; i < T.size(); ++i) ring[i] += T[i];
                }
        auto RS = matmul(ring, S, nc);
        for (size_t i = 0; i < P.size(); ++i) P[i] += RS[i];
        if (k == levels - 2) break;
        std::vector<double> up((size_t)nc * nc, 0.0);
        for (int a = -1; a <= 1; ++a)
            for (int b = -1; b <= 1; ++b)
                for (int c = -1; c <= 1; ++c) {
                    auto T = pack_matrix(m2m_full(a * w, b * w, c * w, p, 1.0), p);
                    for (size_t i = 0; i < T.size(); ++i) up[i] += T[i];
                }
        S = matmul(up, S, nc);
    }
    return P;
}

// store a packed row-major matrix A (nc x nc) transposed + padded at slot `slot`
// row-major [slot][128][128] tf32 hi part (low 13 mantissa bits cleared) and FP32 remainder
void store_tc(std::vector<float>& hi, std::vector<float>& lo, int slot,
              const std::vector<double>& A, int nc) {
    float* H = hi.data() + (size_t)slot * 128 * 128;
    float* Lo = lo.data() + (size_t)slot * 128 * 128;
    for (int r = 0; r < nc; ++r)
        for (int k = 0; k < nc; ++k) {
            const float v = (float)A[(size_t)r * nc + k];
            uint32_t u;
            memcpy(&u, &v, 4);
            u &= 0xFFFFE000u;
            float h;
            memcpy(&h, &u, 4);
            H[(size_t)r * 128 + k] = h;
            Lo[(size_t)r * 128 + k] = v - h;
        }
}

// 3xFP16 operands: balance the operators by power-of-2 column scales cs[k] (max over slots and
// rows of |T[r][k]|) and row scales rs[r] (max of |T[r][k]| / cs[k]), so Ahat = T / (rs cs)
// has |Ahat| <= 1 and no overflow in half; hi = half(Ahat), lo = half(Ahat - hi)
void store_h16(const std::vector<std::pair<int, std::vector<double>>>& ops, int nc, HostOps* out) {
    auto pow2_ceil = [](double v) { return v > 0 ? std::exp2(std::ceil(std::log2(v))) : 1.0; };
    const int NRh = nc <= 128 ? 128 : 256, KPh = nc <= 128 ? 128 : (nc + 63) / 64 * 64;
    out->h16_nr = NRh;
    out->h16_kp = KPh;
    std::vector<double> cs(KPh, 1.0), rs(NRh, 1.0);
    for (int k = 0; k < nc; ++k) {
        double m = 0;
        for (const auto& so : ops)
            for (int r = 0; r < nc; ++r) m = std::max(m, std::fabs(so.second[(size_t)r * nc + k]));
        cs[k] = pow2_ceil(m);
    }
    for (int r = 0; r < nc; ++r) {
        double m = 0;
        for (const auto& so : ops)
            for (int k = 0; k < nc; ++k)
                m = std::max(m, std::fabs(so.second[(size_t)r * nc + k]) / cs[k]);
        rs[r] = pow2_ceil(m);
    }
    out->m2l_h16_hi.assign((size_t)343 * NRh * KPh, 0);
    out->m2l_h16_lo.assign((size_t)343 * NRh * KPh, 0);
    for (const auto& so : ops) {
        uint16_t* H = out->m2l_h16_hi.data() + (size_t)so.first * NRh * KPh;
        uint16_t* Lo = out->m2l_h16_lo.data() + (size_t)so.first * NRh * KPh;
        for (int r = 0; r < nc; ++r)
            for (int k = 0; k < nc; ++k) {
                const double v = so.second[(size_t)r * nc + k] / (rs[r] * cs[k]);
                const __half h = __double2half(v);
                const __half l = __double2half(v - (double)__half2float(h));
                memcpy(&H[(size_t)r * KPh + k], &h, 2);
                memcpy(&Lo[(size_t)r * KPh + k], &l, 2);
            }
    }
    out->h16_rs.assign(rs.begin(), rs.end());
    out->h16_cs.assign(cs.begin(), cs.end());
}

void store_t(std::vector<float>& dst, int slot, const std::vector<double>& A, int nc, int KP,
             int NR) {
    float* base = dst.data() + (size_t)slot * KP * NR;
    for (int r = 0; r < nc; ++r)
        for (int k = 0; k < nc; ++k) base[(size_t)k * NR + r] = (float)A[(size_t)r * nc + k];
}

}  // namespace

// ---- L2P: the 12 derivative combinations of a leaf's local expansion as a sparse map ----
// Symbolic replay of the device's derivative rules (expansions.cu deriv_expansion / getc):
// every entry of an expansion is a sparse vector over the 3 nc packed inputs of L.
namespace {
using SV = std::vector<std::pair<int, double>>;
SV sv_axpy(const SV& a, double ca, const SV& b, double cb) {
    std::map<int, double> m;
    for (const auto& t : a) m[t.first] += ca * t.second;
    for (const auto& t : b) m[t.first] += cb * t.second;
    SV r;
    for (const auto& t : m)
        if (t.second != 0.0) r.emplace_back(t.first, t.second);
    return r;
}
struct CSV {
    SV re, im;
};
CSV getc_sym(const std::vector<SV>& E, int n, int m) {
    if (m > n || -m > n || n < 0) return {};
    if (m == 0) return {E[pk_re(n, 0)], {}};
    const int am = m < 0 ? -m : m;
    CSV v{E[pk_re(n, am)], E[pk_im(n, am)]};
    if (m < 0) {  // (-1)^m conj
        v.im = sv_axpy(v.im, -1.0, {}, 0.0);
        if (am & 1) {
            v.re = sv_axpy(v.re, -1.0, {}, 0.0);
            v.im = sv_axpy(v.im, -1.0, {}, 0.0);
        }
    }
    return v;
}
std::vector<SV> deriv_sym(const std::vector<SV>& E, int pin, int axis) {
    std::vector<SV> out((size_t)pin * pin);
    for (int k = 0; k < pin * pin; ++k) {
        int n = 0;
        while ((n + 1) * (n + 1) <= k) ++n;
        const int j = k - n * n, m = (j + 1) >> 1;
        const bool isim = j > 0 && (j & 1) == 0;
        CSV v;
        if (axis == 2) {
            v = getc_sym(E, n + 1, m);
        } else {
            const CSV up = getc_sym(E, n + 1, m + 1), dn = getc_sym(E, n + 1, m - 1);
            if (axis == 0) v = {sv_axpy(dn.re, 0.5, up.re, -0.5), sv_axpy(dn.im, 0.5, up.im, -0.5)};
            else v = {sv_axpy(up.im, 0.5, dn.im, 0.5), sv_axpy(up.re, -0.5, dn.re, -0.5)};
        }
        out[k] = isim ? v.im : v.re;
    }
    return out;
}
}  // namespace

void build_l2p_map(int p, HostOps* out) {
    // Two stages, both rows of D[k][q] (k < p^2, 12 columns):
    //  q < 3:  u_q = (curl phi)_q expansion, terms over the leaf's L (src = c nc + i);
    //  q >= 3: J[a][kk] = d_kk u_a, terms over the stage-1 rows (src = k' 12 + a, i.e. D itself)
    // (second derivatives as first derivatives of u: 2.6x fewer terms than from L directly)
    const int nc = (p + 1) * (p + 1), ng = p * p, nh = (p - 1) * (p - 1);
    std::vector<SV> Lc[3];
    for (int c = 0; c < 3; ++c) {
        Lc[c].resize(nc);
        for (int i = 0; i < nc; ++i) Lc[c][i] = {{c * nc + i, 1.0}};
    }
    std::vector<SV> G[3][3];
    for (int c = 0; c < 3; ++c)
        for (int ax = 0; ax < 3; ++ax) G[c][ax] = deriv_sym(Lc[c], p, ax);
    std::vector<SV> U[3], J[3][3];
    for (int a = 0; a < 3; ++a) {
        U[a].resize(ng);
        for (int k = 0; k < ng; ++k) U[a][k] = {{k * 12 + a, 1.0}};
        if (p >= 2)
            for (int kk = 0; kk < 3; ++kk) J[a][kk] = deriv_sym(U[a], p - 1, kk);
    }
    out->l2p_rowptr.assign(1, 0);
    out->l2p_src.clear();
    out->l2p_coef.clear();
    for (int k = 0; k < ng; ++k)
        for (int q = 0; q < 12; ++q) {
            SV v;
            if (q == 0) v = sv_axpy(G[2][1][k], 1.0, G[1][2][k], -1.0);
            else if (q == 1) v = sv_axpy(G[0][2][k], 1.0, G[2][0][k], -1.0);
            else if (q == 2) v = sv_axpy(G[1][0][k], 1.0, G[0][1][k], -1.0);
            else if (k < nh) v = J[(q - 3) / 3][(q - 3) % 3][k];
            for (const auto& t : v) {
                out->l2p_src.push_back(t.first);
                out->l2p_coef.push_back((float)t.second);
            }
            // every row has <= 4 terms (curl: two first-derivative entries of <= 2 terms each;
            // grad u: one first-derivative entry): one 16-byte record per row
            if (v.size() > 4) throw std::runtime_error("L2P map row with more than 4 terms");
            for (size_t t = v.size(); t < 4; ++t) {  // exactly 4 slots: record e at 4 e
                out->l2p_src.push_back(0);
                out->l2p_coef.push_back(0.f);
            }
            out->l2p_rowptr.push_back((int)out->l2p_src.size());
        }
}

std::vector<int> m2l_groups() {
    std::vector<int> g((size_t)8 * 72 * 4, 0);
    for (int pi = 0; pi < 8; ++pi) {
        for (int i = 0; i < 72; ++i) {
            int* e = &g[((size_t)pi * 72 + i) * 4];
            const int dx = i / 24 - 1, dz = (i / 8) % 3 - 1, pis = i % 8;
            e[0] = ((dx + 1) << 4) | ((dz + 1) << 6) | (pis << 8);
            e[1] = e[2] = e[3] = -1;
        }
        const int bx = pi & 1, by = (pi >> 1) & 1, bz = (pi >> 2) & 1;
        int cnt = 0;
        for (int ox = -2 - bx; ox <= 3 - bx; ++ox)
            for (int oy = -2 - by; oy <= 3 - by; ++oy)
                for (int oz = -2 - bz; oz <= 3 - bz; ++oz) {
                    if (std::abs(ox) <= 1 && std::abs(oy) <= 1 && std::abs(oz) <= 1) continue;
                    const int sx = bx + ox, sy = by + oy, sz = bz + oz;  // source child coords
                    const int dx = sx >> 1, dy = sy >> 1, dz = sz >> 1;   // floor division
                    const int pis = (sx & 1) | ((sy & 1) << 1) | ((sz & 1) << 2);
                    const int i = ((dx + 1) * 3 + (dz + 1)) * 8 + pis;
                    int* e = &g[((size_t)pi * 72 + i) * 4];
                    e[0] |= 1 << (dy + 1);
                    e[1 + dy + 1] = m2l_slot(ox, oy, oz);
                    ++cnt;
                }
        (void)cnt;  // 189 per parity (checked with the slot table in capi.cu)
    }
    return g;
}

void build_host_ops(int p, int image_levels, HostOps* out) {
    const int nc = (p + 1) * (p + 1);
    out->p = p;
    out->nc = nc;
    out->KP = (nc + 15) / 16 * 16;
    out->NR = (nc + 127) / 128 * 128;
    const size_t msz = (size_t)out->KP * out->NR;
    out->m2m.assign(8 * msz, 0.f);
    out->l2l.assign(8 * msz, 0.f);
    out->m2l.assign(343 * msz, 0.f);
    out->per.assign(msz, 0.f);
    const bool tc = nc <= 128;        // 3xTF32 operators
    const bool h16 = nc <= 256;       // 3xFP16 operators (two row tiles above 128)
    out->m2l_tc_hi.assign(tc ? (size_t)343 * 128 * 128 : 0, 0.f);
    out->m2l_tc_lo.assign(tc ? (size_t)343 * 128 * 128 : 0, 0.f);
    std::vector<std::pair<int, std::vector<double>>> tc_ops;  // (slot, packed operator)
    for (int ch = 0; ch < 8; ++ch) {
        const double dx = (((ch >> 0) & 1) - 0.5) * 0.5;
        const double dy = (((ch >> 1) & 1) - 0.5) * 0.5;
        const double dz = (((ch >> 2) & 1) - 0.5) * 0.5;
        store_t(out->m2m, ch, pack_matrix(m2m_full(dx, dy, dz, p, 0.5), p), nc, out->KP, out->NR);
        store_t(out->l2l, ch, pack_matrix(l2l_full(dx, dy, dz, p, 0.5), p), nc, out->KP, out->NR);
    }
    for (int ox = -3; ox <= 3; ++ox)
        for (int oy = -3; oy <= 3; ++oy)
            for (int oz = -3; oz <= 3; ++oz) {
                if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) <= 1) continue;
                const auto T = pack_matrix(m2l_full(-ox, -oy, -oz, p), p);
                store_t(out->m2l, m2l_slot(ox, oy, oz), T, nc, out->KP, out->NR);
                if (tc) store_tc(out->m2l_tc_hi, out->m2l_tc_lo, m2l_slot(ox, oy, oz), T, nc);
                if (h16) tc_ops.emplace_back(m2l_slot(ox, oy, oz), T);
            }
    if (h16) store_h16(tc_ops, nc, out);
    build_l2p_map(p, out);
    out->per_d = build_periodic(p, image_levels);
    store_t(out->per, 0, out->per_d, nc, out->KP, out->NR);
}

}  // namespace vfmm
