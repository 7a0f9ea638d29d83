// Quadratic case M = N (paper Section "The quadratic case", P:344-489,
// adjoint Remark P:576-584): the inverse NFFT by the Lagrange relation
//   g_l = a_l sum_j f_j b_j (cot(pi (x_l - y_j)) - i)                     (eq. lagrange_formula)
// at equispaced targets x_l = -1/2 + l/N + delta, then fcheck = (1/N) E^* g by one FFT
// (Alg. "Fast inverse NFFT - quadratic case" step 6), and its adjoint
//   f_j = b_j sum_l a_l v_l (cot(pi (x_l - y_j)) + i),  v = (1/N) E h   (eq. lagrange_formula_adjoint).
// a_l = prod_n sin(pi (x_l - y_n)) and b_j = prod_{n != j} 1/sin(pi (y_j - y_n)) (eq. coeff_ab)
// are formed in the log domain with counted signs and the balancing shift s
// (Remark P:431-449, reading A22).
//
// B200 design: the three sums (ln|sin| for a and b, the cotangent sum per RHS) run by the
// NFFT-based fast summation the paper uses (see "fast summation" below): far field
// through this library's own plain NFFT at the nodes (bandwidth 4N, sigma_2 = 2, m_2 = 8) and
// one length-N FFT for the equispaced targets, near field (|t - s| < 8/N) directly from the
// sorted nodes; O(N log N).  Below N = 512 (or with INFT_QUAD_DIRECT=1) the sums are evaluated
// directly and exactly by tiled kernels (one thread per target, sources through shared
// memory, one sin/cos per pair reused for 16 right-hand sides); both paths are deterministic.
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "inft_internal.cuh"

namespace inft {
namespace quad {

constexpr int kTile = 256;  // sources per shared-memory tile
constexpr int kRG = 16;     // right-hand sides per cotangent-sum block

static int64_t nb(int64_t n, int t = 256) { return (n + t - 1) / t; }

// logsum[t] = sgn * sum_{n (!= t if self)} ln|sin(pi (tgt_t - src_n))|, neg[t] = #{n: factor < 0};
// *bad set if a factor is exactly zero (coincident nodes).
__global__ void k_logsum(const double* __restrict__ tgt, int64_t nt, const double* __restrict__ src, int64_t ns,
                         int self, double sgn, double* __restrict__ logsum, int* __restrict__ negs,
                         int* __restrict__ bad) {
    __shared__ double ys[kTile];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const double xt = t < nt ? tgt[t] : 0.0;
    double acc = 0.0;
    int neg = 0, zero = 0;
    for (int64_t n0 = 0; n0 < ns; n0 += kTile) {
        const int cnt = (int)(ns - n0 < kTile ? ns - n0 : kTile);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) ys[i] = src[n0 + i];
        __syncthreads();
        if (t >= nt) continue;
        for (int i = 0; i < cnt; ++i) {
            if (self && n0 + i == t) continue;
            const double d = xt - ys[i];  // in (-1, 1): sin(pi d) < 0 iff d < 0
            const double sv = sinpi(d);
            zero |= sv == 0.0;
            neg += d < 0.0;
            acc += log(fabs(sv));
        }
    }
    if (t < nt) {
        logsum[t] = sgn * acc;
        negs[t] = neg;
        if (zero) atomicOr(bad, 1);
    }
}

// s = (max btilde - max atilde) / 2 (reading A22), one block, fixed reduction order
__global__ void k_shift(const double* __restrict__ at, const double* __restrict__ bt, int64_t N,
                        double* __restrict__ s) {
    __shared__ double ma[256], mb[256];
    double a = -INFINITY, b = -INFINITY;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        a = fmax(a, at[i]);
        b = fmax(b, bt[i]);
    }
    ma[threadIdx.x] = a;
    mb[threadIdx.x] = b;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            ma[threadIdx.x] = fmax(ma[threadIdx.x], ma[threadIdx.x + o]);
            mb[threadIdx.x] = fmax(mb[threadIdx.x], mb[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *s = 0.5 * (mb[0] - ma[0]);
}

// a_l = (-1)^neg e^{atilde + s},  b_j = (-1)^neg e^{btilde - s}   (Alg. steps 2-3)
__global__ void k_signed(const double* __restrict__ lg, const int* __restrict__ negs, int64_t N,
                         const double* __restrict__ s, double ssgn, double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double v = exp(lg[i] + ssgn * *s);
    out[i] = (negs[i] & 1) ? -v : v;
}

// out[r][t] = sum_s cf[r][s] cot(pi (tgt_t - src_s)), r in this block's group of kRG
__global__ void __launch_bounds__(128) k_cotsum(const double* __restrict__ tgt, int64_t nt,
                                                const double* __restrict__ src, int64_t ns,
                                                const double2* __restrict__ cf, int64_t R,
                                                double2* __restrict__ out) {
    __shared__ double ys[128];
    __shared__ double2 cs[kRG][128];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.y * kRG;
    const int nr = (int)(R - r0 < kRG ? R - r0 : kRG);
    const double xt = t < nt ? tgt[t] : 0.0;
    double ax[kRG], ay[kRG];
#pragma unroll
    for (int q = 0; q < kRG; ++q) ax[q] = ay[q] = 0.0;
    for (int64_t n0 = 0; n0 < ns; n0 += 128) {
        const int cnt = (int)(ns - n0 < 128 ? ns - n0 : 128);
        __syncthreads();
        if ((int)threadIdx.x < cnt) ys[threadIdx.x] = src[n0 + threadIdx.x];
        for (int q = 0; q < kRG; ++q)
            cs[q][threadIdx.x] = (q < nr && (int)threadIdx.x < cnt) ? cf[(r0 + q) * ns + n0 + threadIdx.x]
                                                                    : make_double2(0.0, 0.0);
        __syncthreads();
        for (int i = 0; i < cnt; ++i) {
            double sn, cn;
            sincospi(xt - ys[i], &sn, &cn);
            const double ct = cn / sn;
#pragma unroll
            for (int q = 0; q < kRG; ++q) {
                ax[q] = fma(cs[q][i].x, ct, ax[q]);
                ay[q] = fma(cs[q][i].y, ct, ay[q]);
            }
        }
    }
    if (t < nt)
        for (int q = 0; q < nr; ++q) out[(r0 + q) * nt + t] = make_double2(ax[q], ay[q]);
}

// sums[r] = sum_i v[r][i] (one block per row, fixed order)
__global__ void k_rowsum(const double2* __restrict__ v, int64_t n, double2* __restrict__ sums) {
    __shared__ double sx[256], sy[256];
    double x = 0.0, y = 0.0;
    const double2* row = v + (int64_t)blockIdx.x * n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        x += row[i].x;
        y += row[i].y;
    }
    sx[threadIdx.x] = x;
    sy[threadIdx.x] = y;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sx[threadIdx.x] += sx[threadIdx.x + o];
            sy[threadIdx.x] += sy[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[blockIdx.x] = make_double2(sx[0], sy[0]);
}

// c[r][j] = f[r][j] * w[j]  (real weights)
__global__ void k_scale(const double2* __restrict__ f, const double* __restrict__ w, int64_t n, int64_t total,
                        double2* __restrict__ c) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const double s = w[i % n];
    c[i] = make_double2(f[i].x * s, f[i].y * s);
}

// g[r][l] = a_l (gt[r][l] - i S_r)   (eq. coeff_g)
__global__ void k_glue_inv(const double2* __restrict__ gt, const double* __restrict__ a, const double2* __restrict__ S,
                           int64_t N, int64_t total, double2* __restrict__ g) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, l = i - r * N;
    const double2 v = gt[i], s = S[r];
    // (v - i s) = (v.x + s.y, v.y - s.x)
    g[i] = make_double2(a[l] * (v.x + s.y), a[l] * (v.y - s.x));
}

// fcheck[r][k + N/2] = (1/N) (-1)^k e^{-2 pi i k delta} G[r][k mod N]   (Alg. step 6 with
// x_l = -1/2 + l/N + delta: e^{-2 pi i k x_l} = (-1)^k e^{-2 pi i k delta} e^{-2 pi i k l/N})
__global__ void k_post_inv(const double2* __restrict__ G, int64_t N, int64_t total, double delta,
                           double2* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, c = i - r * N;
    const int64_t k = c - N / 2;
    const double2 v = G[r * N + (k < 0 ? k + N : k)];
    double sn, cs;
    sincospi(-2.0 * ((double)k * delta), &sn, &cs);
    const double sg = (k & 1) ? -1.0 / (double)N : 1.0 / (double)N;
    out[i] = make_double2(sg * (v.x * cs - v.y * sn), sg * (v.x * sn + v.y * cs));
}

// u[r][k mod N] = (1/N) (-1)^k e^{2 pi i k delta} h[r][k + N/2]; the inverse FFT then gives
// v_l = (1/N) sum_k h_k e^{2 pi i k x_l}
__global__ void k_pre_adj(const double2* __restrict__ h, int64_t N, int64_t total, double delta,
                          double2* __restrict__ u) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, c = i - r * N;
    const int64_t k = c - N / 2;
    const double2 v = h[i];
    double sn, cs;
    sincospi(2.0 * ((double)k * delta), &sn, &cs);
    const double sg = (k & 1) ? -1.0 / (double)N : 1.0 / (double)N;
    u[r * N + (k < 0 ? k + N : k)] = make_double2(sg * (v.x * cs - v.y * sn), sg * (v.x * sn + v.y * cs));
}

// f[r][j] = b_j (-ct[r][j] + i W_r), ct = sum_l w_l cot(pi (y_j - x_l)) = -sum_l w_l cot(pi (x_l - y_j))
__global__ void k_glue_adj(const double2* __restrict__ ct, const double* __restrict__ b, const double2* __restrict__ W,
                           int64_t N, int64_t total, double2* __restrict__ f) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, j = i - r * N;
    const double2 v = ct[i], w = W[r];
    // -v + i w = (-v.x - w.y, -v.y + w.x)
    f[i] = make_double2(b[j] * (-v.x - w.y), b[j] * (-v.y + w.x));
}

// ------------------------------------------------------------------ fast summation
// The three sums sum_j c_j K(t - s_j), K in {cot(pi x), ln|sin(pi x)|} (1-periodic, singular
// only at x = 0), by the NFFT-based fast summation the paper uses (Potts-Steidl):
// K = K_R + K_NE with K_R = K outside |x| < eps and, inside, the two-point Taylor (Hermite)
// interpolant T of degree 2p-1 matching K^(r)(+-eps), r < p, so K_R is C^(p-1) and periodic;
//   far  field  sum_{|k| < n/2} b_k e^{2 pi i k t} chat_k,  b_k = Fourier coefficients of K_R,
//               chat_k = sum_j c_j e^{-2 pi i k s_j}  (adjoint NFFT / FFT for the equispaced x),
//               evaluated by an FFT (equispaced targets x_l) or an NFFT (targets y_j);
//   near field  sum_{|t - s_j| < eps} c_j (K - T)(t - s_j)  directly (sorted sources).
// eps = kFsA / N, n = kFsOver N: the truncation error ~ p! / (pi n eps)^(p+1) ~ 1e-16.
constexpr int kFsP = 10;
constexpr double kFsA = 8.0;
constexpr int kFsOver = 4;
struct FsPoly {
    double t[2 * kFsP];  // T(x) = sum_i t_i (x / eps)^i on |x| < eps
};

__device__ __forceinline__ double fs_poly(const FsPoly& T, double u) {
    double v = T.t[2 * kFsP - 1];
#pragma unroll
    for (int i = 2 * kFsP - 2; i >= 0; --i) v = fma(v, u, T.t[i]);
    return v;
}
// kind 0: cot(pi x), kind 1: ln|sin(pi x)|
__device__ __forceinline__ double fs_k(int kind, double d) {
    double sn, cs;
    sincospi(d, &sn, &cs);
    return kind == 0 ? cs / sn : log(fabs(sn));
}
__device__ __forceinline__ double fs_near(int kind, const FsPoly& T, double eps, double d) {
    return fs_k(kind, d) - fs_poly(T, d / eps);
}

// samples of K_R at x_i = -1/2 + i / nf
__global__ void k_fs_sample(int kind, FsPoly T, double eps, int64_t nf, double2* __restrict__ s) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const double x = -0.5 + (double)i / (double)nf;
    const double v = fabs(x) < eps ? fs_poly(T, x / eps) : (i == 0 ? fs_k(kind, -0.5) : fs_k(kind, x));
    s[i] = make_double2(v, 0.0);
}
// b_k = (1/nf) sum_i K_R(x_i) e^{-2 pi i k x_i} = (-1)^k / nf * S[k mod nf], k = -n/2..n/2-1 at k + n/2
__global__ void k_fs_coef(const double2* __restrict__ S, int64_t nf, int64_t n, double2* __restrict__ b) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    const int64_t k = c - n / 2;
    const double2 v = S[k < 0 ? k + nf : k];
    const double sg = ((k & 1) ? -1.0 : 1.0) / (double)nf;
    b[c] = make_double2(sg * v.x, sg * v.y);
}

// equispaced targets: U[r][kappa] = sum_{k = kappa mod N} b_k chat[r][k] (-1)^k e^{2 pi i k delta}
// (then sum_kappa U e^{2 pi i kappa l / N} = sum_k b_k chat_k e^{2 pi i k x_l})
__global__ void k_fs_fold(const double2* __restrict__ chat, const double2* __restrict__ b, int64_t n, int64_t N,
                          int64_t R, double delta, double2* __restrict__ U) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= R * N) return;
    const int64_t r = i / N, kap = i - r * N;
    double ax = 0.0, ay = 0.0;
    // k = kap + t N in [-n/2, n/2)
    int64_t k = kap - ((kap + n / 2) / N) * N;
    for (; k < n / 2; k += N) {
        const int64_t c = k + n / 2;
        const double2 v = chat[r * n + c], w = b[c];
        const double px = v.x * w.x - v.y * w.y, py = v.x * w.y + v.y * w.x;
        double sn, cs;
        sincospi(2.0 * ((double)k * delta), &sn, &cs);
        const double sg = (k & 1) ? -1.0 : 1.0;
        ax += sg * (px * cs - py * sn);
        ay += sg * (px * sn + py * cs);
    }
    U[i] = make_double2(ax, ay);
}

// equispaced sources: u[r][k] = b_k chat_k with chat_k = sum_l w_l e^{-2 pi i k x_l}
// = (-1)^k e^{-2 pi i k delta} W[r][k mod N], W = forward FFT of w
__global__ void k_fs_pre(const double2* __restrict__ W, const double2* __restrict__ b, int64_t n, int64_t N,
                         int64_t R, double delta, double2* __restrict__ u) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= R * n) return;
    const int64_t r = i / n, c = i - r * n;
    const int64_t k = c - n / 2;
    int64_t km = k % N;
    if (km < 0) km += N;
    const double2 v = W[r * N + km], w = b[c];
    double sn, cs;
    sincospi(-2.0 * ((double)k * delta), &sn, &cs);
    const double sg = (k & 1) ? -1.0 : 1.0;
    const double cx = sg * (v.x * cs - v.y * sn), cy = sg * (v.x * sn + v.y * cs);
    u[i] = make_double2(cx * w.x - cy * w.y, cx * w.y + cy * w.x);
}

// u[r][k] = b_k chat[r][k]
__global__ void k_fs_mulb(const double2* __restrict__ chat, const double2* __restrict__ b, int64_t n, int64_t total,
                          double2* __restrict__ u) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const double2 v = chat[i], w = b[i % n];
    u[i] = make_double2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
}

__device__ __forceinline__ int64_t lower_bound_d(const double* __restrict__ a, int64_t n, double v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// near field, sources = sorted nodes ys (caller index idx[s]), targets tgt (N_t), coefficients
// cf[r][caller index] (or 1 if cf == nullptr); self = exclude the source whose caller index is
// the target index.  out[r][t] += sum (K - T)(wrap(t - s)) c.
__global__ void k_fs_near_sorted(int kind, FsPoly T, double eps, const double* __restrict__ tgt, int64_t nt,
                                 const double* __restrict__ ys, const int32_t* __restrict__ idx, int64_t ns,
                                 const double2* __restrict__ cf, int64_t R, int self, double2* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= R * nt) return;
    const int64_t r = i / nt, t = i - r * nt;
    const double x = tgt[t];
    double ax = 0.0, ay = 0.0;
    // window [x - eps, x + eps] on the circle: up to two ranges of the sorted sources
    double lo = x - eps, hi = x + eps;
    double rl[2][2];
    int nr = 0;
    if (lo < -0.5) {
        rl[nr][0] = lo + 1.0; rl[nr][1] = 0.5; ++nr;
        rl[nr][0] = -0.5; rl[nr][1] = hi; ++nr;
    } else if (hi >= 0.5) {
        rl[nr][0] = lo; rl[nr][1] = 0.5; ++nr;
        rl[nr][0] = -0.5; rl[nr][1] = hi - 1.0; ++nr;
    } else {
        rl[nr][0] = lo; rl[nr][1] = hi; ++nr;
    }
    for (int q = 0; q < nr; ++q) {
        for (int64_t s = lower_bound_d(ys, ns, rl[q][0]); s < ns && ys[s] < rl[q][1]; ++s) {
            const int64_t j = idx[s];
            if (self && j == t) continue;
            double d = x - ys[s];
            d -= rint(d);
            if (fabs(d) >= eps) continue;
            const double kv = fs_near(kind, T, eps, d);
            if (cf) {
                const double2 c = cf[r * ns + j];
                ax = fma(c.x, kv, ax);
                ay = fma(c.y, kv, ay);
            } else {
                ax += kv;
            }
        }
    }
    double2 o = out[i];
    out[i] = make_double2(o.x + ax, o.y + ay);
}

// near field, sources = equispaced x_l = -1/2 + l/N + delta with coefficients w[r][l], targets y_j
__global__ void k_fs_near_equi(int kind, FsPoly T, double eps, const double* __restrict__ tgt, int64_t nt, int64_t N,
                               double delta, const double2* __restrict__ w, int64_t R, double2* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= R * nt) return;
    const int64_t r = i / nt, t = i - r * nt;
    const double y = tgt[t];
    const int64_t l0 = (int64_t)ceil((y - eps + 0.5 - delta) * (double)N) - 1;
    const int64_t l1 = (int64_t)floor((y + eps + 0.5 - delta) * (double)N) + 1;
    double ax = 0.0, ay = 0.0;
    for (int64_t L = l0; L <= l1; ++L) {
        int64_t l = L % N;
        if (l < 0) l += N;
        double d = y - (-0.5 + (double)l / (double)N + delta);
        d -= rint(d);
        if (fabs(d) >= eps) continue;
        const double kv = fs_near(kind, T, eps, d);
        const double2 c = w[r * N + l];
        ax = fma(c.x, kv, ax);
        ay = fma(c.y, kv, ay);
    }
    double2 o = out[i];
    out[i] = make_double2(o.x + ax, o.y + ay);
}

__global__ void k_fs_addconst(double2* __restrict__ v, int64_t n, double c) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i].x += c;
}
__global__ void k_fs_real(const double2* __restrict__ v, int64_t n, double sgn, double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = sgn * v[i].x;
}
__global__ void k_fs_ones(double2* __restrict__ v, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = make_double2(1.0, 0.0);
}

// host: D^r K at x, r < nd, for cot(pi x) (kind 0) or ln|sin(pi x)| (kind 1).
// D^r cot(pi x) = pi^r P_r(cot(pi x)), P_0(c) = c, P_{r+1}(c) = -(1 + c^2) P_r'(c);
// D ln|sin(pi x)| = pi cot(pi x).
static void fs_derivs(int kind, long double x, int nd, long double* out) {
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double c = cosl(pi * x) / sinl(pi * x);
    std::vector<long double> P{0.0L, 1.0L};  // P_0(c) = c
    std::vector<long double> cot(nd + 1);
    long double pw = 1.0L;
    for (int r = 0; r <= nd; ++r) {
        long double v = 0.0L;
        for (int i = (int)P.size() - 1; i >= 0; --i) v = v * c + P[i];
        cot[r] = pw * v;
        // P_{r+1} = -(1 + c^2) P_r'
        std::vector<long double> d(P.size() > 1 ? P.size() - 1 : 1, 0.0L);
        for (size_t i = 1; i < P.size(); ++i) d[i - 1] = (long double)i * P[i];
        std::vector<long double> nx(d.size() + 2, 0.0L);
        for (size_t i = 0; i < d.size(); ++i) {
            nx[i] -= d[i];
            nx[i + 2] -= d[i];
        }
        P = nx;
        pw *= pi;
    }
    for (int r = 0; r < nd; ++r) {
        if (kind == 0) out[r] = cot[r];
        else out[r] = r == 0 ? logl(fabsl(sinl(pi * x))) : pi * cot[r - 1];
    }
}

// host: two-point Taylor interpolant T(u) = sum_i t_i u^i, u = x / eps, T^(r)(+-1) = eps^r K^(r)(+-eps)
static FsPoly fs_poly_build(int kind, double eps) {
    const int p = kFsP, n = 2 * p;
    long double Kp[kFsP], Km[kFsP];
    fs_derivs(kind, (long double)eps, p, Kp);
    fs_derivs(kind, -(long double)eps, p, Km);
    std::vector<long double> A((size_t)n * n, 0.0L), b(n);
    long double er = 1.0L;
    for (int r = 0; r < p; ++r) {
        for (int side = 0; side < 2; ++side) {
            const int row = 2 * r + side;
            const long double u = side ? -1.0L : 1.0L;
            for (int i = r; i < n; ++i) {
                long double f = 1.0L;
                for (int q = 0; q < r; ++q) f *= (long double)(i - q);
                long double up = 1.0L;
                for (int q = 0; q < i - r; ++q) up *= u;
                A[(size_t)row * n + i] = f * up;
            }
            b[row] = er * (side ? Km[r] : Kp[r]);
        }
        er *= (long double)eps;
    }
    // Gaussian elimination, partial pivoting
    for (int c = 0; c < n; ++c) {
        int pv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabsl(A[(size_t)r * n + c]) > fabsl(A[(size_t)pv * n + c])) pv = r;
        if (pv != c) {
            for (int i = 0; i < n; ++i) std::swap(A[(size_t)c * n + i], A[(size_t)pv * n + i]);
            std::swap(b[c], b[pv]);
        }
        for (int r = c + 1; r < n; ++r) {
            const long double f = A[(size_t)r * n + c] / A[(size_t)c * n + c];
            if (f == 0.0L) continue;
            for (int i = c; i < n; ++i) A[(size_t)r * n + i] -= f * A[(size_t)c * n + i];
            b[r] -= f * b[c];
        }
    }
    FsPoly T;
    std::vector<long double> t(n);
    for (int r = n - 1; r >= 0; --r) {
        long double v = b[r];
        for (int i = r + 1; i < n; ++i) v -= A[(size_t)r * n + i] * t[i];
        t[r] = v / A[(size_t)r * n + r];
    }
    for (int i = 0; i < n; ++i) T.t[i] = (double)t[i];
    return T;
}

struct QPlan {
    int64_t N = 0;
    int device = 0;
    double delta = 0.0;
    DevBuf x, y, a, b, s;
    DevBuf w1, w2, w3, sums;  // per-apply workspaces ([R][N] complex x 3, [R] complex)
    int64_t wsR = 0;
    std::map<int64_t, cufftHandle> fft;  // batch -> plan
    int64_t launches = 0;
    // fast summation (N >= kFsMinN unless INFT_QUAD_DIRECT=1)
    bool fast = false;
    double eps = 0.0;
    int64_t nfs = 0;           // far-field bandwidth n
    FsPoly Tcot, Tlog;
    DevBuf bcot, blog;         // [n] Fourier coefficients of the regularised kernels
    DevBuf ys, yidx;           // nodes sorted, caller index of each
    inft_plan_t nfft = nullptr;  // plain NFFT at the nodes, bandwidth n (A, A^* approximations)
    DevBuf wfs;                  // far-field workspace [R][n] complex
    int64_t wfsR = 0;
    void ensure_wfs(int64_t R) {
        if (R <= wfsR) return;
        wfs.alloc(sizeof(double2) * (size_t)R * (size_t)nfs);
        wfsR = R;
    }
    ~QPlan() {
        for (auto& kv : fft) cufftDestroy(kv.second);
        if (nfft) inft_destroy(nfft);
    }
    cufftHandle plan_for(int64_t R, cudaStream_t st) {
        auto it = fft.find(R);
        cufftHandle h;
        if (it == fft.end()) {
            int n[1] = {(int)N};
            INFT_CUFFT(cufftPlanMany(&h, 1, n, nullptr, 1, (int)N, nullptr, 1, (int)N, CUFFT_Z2Z, (int)R));
            fft[R] = h;
        } else {
            h = it->second;
        }
        cufftSetStream(h, st);
        return h;
    }
    void ensure_ws(int64_t R) {
        if (R <= wsR) return;
        const size_t bytes = sizeof(double2) * (size_t)R * (size_t)N;
        w1.alloc(bytes);
        w2.alloc(bytes);
        w3.alloc(bytes);
        sums.alloc(sizeof(double2) * (size_t)R);
        wsR = R;
    }
};

constexpr int64_t kFsMinN = 512;  // below: direct sums

static void check_status(inft_status st, const char* what) {
    if (st != INFT_OK) {
        set_error(std::string("quadratic case, fast summation: ") + what + " failed");
        throw Fail{st};
    }
}

// Fourier coefficients b_k (k = -n/2..n/2-1) of the regularised kernel (kind 0 cot, 1 log)
static void fs_coefficients(QPlan& q, int kind, const FsPoly& T, DevBuf& out, cudaStream_t st) {
    const int64_t n = q.nfs, nf = 4 * n;
    DevBuf smp;
    smp.alloc(sizeof(double2) * (size_t)nf);
    k_fs_sample<<<(unsigned)nb(nf), 256, 0, st>>>(kind, T, q.eps, nf, smp.as<double2>());
    INFT_CHECK_LAUNCH();
    cufftHandle h;
    INFT_CUFFT(cufftPlan1d(&h, (int)nf, CUFFT_Z2Z, 1));
    cufftSetStream(h, st);
    const cufftResult r = cufftExecZ2Z(h, (cufftDoubleComplex*)smp.p, (cufftDoubleComplex*)smp.p, CUFFT_FORWARD);
    cufftDestroy(h);
    if (r != CUFFT_SUCCESS) {
        set_error("cufftExecZ2Z (fast summation coefficients) failed");
        throw Fail{INFT_ERR_CUFFT};
    }
    out.alloc(sizeof(double2) * (size_t)n);
    k_fs_coef<<<(unsigned)nb(n), 256, 0, st>>>(smp.as<double2>(), nf, n, out.as<double2>());
    INFT_CHECK_LAUNCH();
    q.launches += 2;
    INFT_CUDA(cudaStreamSynchronize(st));
}

// steps 1-3 by the fast summation: atilde (targets x), btilde (targets y, self excluded), signs
// by ranks in the sorted nodes (#{n: y_n > x_l}, #{n: y_n > y_j})
static void build_fast(QPlan& q, const std::vector<double>& yh, const std::vector<double>& xh, DevBuf& la,
                       DevBuf& lb, DevBuf& na, DevBuf& nbn, cudaStream_t st) {
    const int64_t N = q.N;
    std::vector<int32_t> order(N);
    for (int64_t j = 0; j < N; ++j) order[j] = (int32_t)j;
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return yh[a] < yh[b]; });
    std::vector<double> ysh(N);
    for (int64_t s = 0; s < N; ++s) ysh[s] = yh[order[s]];
    for (int64_t s = 1; s < N; ++s)
        if (ysh[s] == ysh[s - 1]) {
            set_error("quadratic case: coincident nodes (a node equals another node)");
            throw Fail{INFT_ERR_NODE_RANGE};
        }
    std::vector<int> nah(N), nbh(N);
    for (int64_t l = 0; l < N; ++l) {
        const int64_t ub = std::upper_bound(ysh.begin(), ysh.end(), xh[l]) - ysh.begin();
        if (ub > 0 && ysh[ub - 1] == xh[l]) {
            set_error("quadratic case: coincident nodes (a node equals a target x_l)");
            throw Fail{INFT_ERR_NODE_RANGE};
        }
        nah[l] = (int)(N - ub);
    }
    for (int64_t s = 0; s < N; ++s) nbh[order[s]] = (int)(N - 1 - s);
    q.ys.alloc(sizeof(double) * N);
    q.yidx.alloc(sizeof(int32_t) * N);
    INFT_CUDA(cudaMemcpyAsync(q.ys.p, ysh.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    INFT_CUDA(cudaMemcpyAsync(q.yidx.p, order.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
    INFT_CUDA(cudaMemcpyAsync(na.p, nah.data(), sizeof(int) * N, cudaMemcpyHostToDevice, st));
    INFT_CUDA(cudaMemcpyAsync(nbn.p, nbh.data(), sizeof(int) * N, cudaMemcpyHostToDevice, st));
    q.eps = kFsA / (double)N;
    q.nfs = kFsOver * N;
    q.Tcot = fs_poly_build(0, q.eps);
    q.Tlog = fs_poly_build(1, q.eps);
    fs_coefficients(q, 0, q.Tcot, q.bcot, st);
    fs_coefficients(q, 1, q.Tlog, q.blog, st);
    // plain NFFT at the nodes with bandwidth n (inner sigma_2 = 2, Kaiser-Bessel m_2 = 8)
    const int64_t nn = q.nfs;
    check_status(inft_plan(&q.nfft, 1, &nn, N, q.y.as<double>(), 2.0, 8, INFT_KAISER_BESSEL, INFT_C128, q.device,
                           (inft_stream_t)st), "inner NFFT plan");
    check_status(inft_precompute(q.nfft, INFT_PLAIN_NFFT, INFT_WEIGHTS_REAL, 0.0, (inft_stream_t)st),
                 "inner NFFT window");
    // atilde_l = sum_n ln|sin(pi (x_l - y_n))|: far field at x by fold + FFT, near field direct
    DevBuf ones, chat, far;
    ones.alloc(sizeof(double2) * N);
    chat.alloc(sizeof(double2) * nn);
    far.alloc(sizeof(double2) * N);
    k_fs_ones<<<(unsigned)nb(N), 256, 0, st>>>(ones.as<double2>(), N);
    INFT_CHECK_LAUNCH();
    check_status(inft_apply(q.nfft, ones.p, chat.p, 1, (inft_stream_t)st), "inner adjoint NFFT");
    k_fs_fold<<<(unsigned)nb(N), 256, 0, st>>>(chat.as<double2>(), q.blog.as<double2>(), nn, N, 1, q.delta,
                                               far.as<double2>());
    INFT_CHECK_LAUNCH();
    cufftHandle h1 = q.plan_for(1, st);
    if (cufftExecZ2Z(h1, (cufftDoubleComplex*)far.p, (cufftDoubleComplex*)far.p, CUFFT_INVERSE) != CUFFT_SUCCESS) {
        set_error("cufftExecZ2Z (fast summation, far field) failed");
        throw Fail{INFT_ERR_CUFFT};
    }
    k_fs_near_sorted<<<(unsigned)nb(N), 256, 0, st>>>(1, q.Tlog, q.eps, q.x.as<double>(), N, q.ys.as<double>(),
                                                      q.yidx.as<int32_t>(), N, nullptr, 1, 0, far.as<double2>());
    INFT_CHECK_LAUNCH();
    k_fs_real<<<(unsigned)nb(N), 256, 0, st>>>(far.as<double2>(), N, 1.0, la.as<double>());
    INFT_CHECK_LAUNCH();
    // btilde_j = -sum_{n != j} ln|sin(pi (y_j - y_n))|: far field at y by the NFFT, minus the
    // self pair's T(0), near field without the self pair
    DevBuf u;
    u.alloc(sizeof(double2) * nn);
    k_fs_mulb<<<(unsigned)nb(nn), 256, 0, st>>>(chat.as<double2>(), q.blog.as<double2>(), nn, nn, u.as<double2>());
    INFT_CHECK_LAUNCH();
    check_status(inft_adjoint_apply(q.nfft, u.p, far.p, 1, (inft_stream_t)st), "inner NFFT");
    k_fs_addconst<<<(unsigned)nb(N), 256, 0, st>>>(far.as<double2>(), N, -q.Tlog.t[0]);
    k_fs_near_sorted<<<(unsigned)nb(N), 256, 0, st>>>(1, q.Tlog, q.eps, q.y.as<double>(), N, q.ys.as<double>(),
                                                      q.yidx.as<int32_t>(), N, nullptr, 1, 1, far.as<double2>());
    k_fs_real<<<(unsigned)nb(N), 256, 0, st>>>(far.as<double2>(), N, -1.0, lb.as<double>());
    INFT_CHECK_LAUNCH();
    q.launches += 8;
    INFT_CUDA(cudaStreamSynchronize(st));
}

static void build(QPlan& q, const double* nodes_host_or_dev, cudaStream_t st) {
    const int64_t N = q.N;
    std::vector<double> yh(N), xh(N);
    if (is_device_pointer(nodes_host_or_dev)) {
        INFT_CUDA(cudaMemcpyAsync(yh.data(), nodes_host_or_dev, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        INFT_CUDA(cudaStreamSynchronize(st));
    } else {
        std::memcpy(yh.data(), nodes_host_or_dev, sizeof(double) * N);
    }
    for (int64_t j = 0; j < N; ++j)
        if (!std::isfinite(yh[j]) || yh[j] < -0.5 || yh[j] >= 0.5) {
            set_error("quadratic case: node outside [-1/2, 1/2)");
            throw Fail{INFT_ERR_NODE_RANGE};
        }
    for (int64_t l = 0; l < N; ++l) xh[l] = -0.5 + (double)l / (double)N + q.delta;
    q.x.alloc(sizeof(double) * N);
    q.y.alloc(sizeof(double) * N);
    q.a.alloc(sizeof(double) * N);
    q.b.alloc(sizeof(double) * N);
    q.s.alloc(sizeof(double));
    INFT_CUDA(cudaMemcpyAsync(q.x.p, xh.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    INFT_CUDA(cudaMemcpyAsync(q.y.p, yh.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    DevBuf la, lb, na, nbn, bad;
    la.alloc(sizeof(double) * N);
    lb.alloc(sizeof(double) * N);
    na.alloc(sizeof(int) * N);
    nbn.alloc(sizeof(int) * N);
    bad.alloc(sizeof(int));
    INFT_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    const char* ed = getenv("INFT_QUAD_DIRECT");
    q.fast = N >= kFsMinN && !(ed && atoi(ed));
    if (q.fast) {
        build_fast(q, yh, xh, la, lb, na, nbn, st);
    } else {
    // step 1: atilde_l = sum_n ln|sin(pi(x_l - y_n))|, btilde_j = -sum_{n != j} ln|sin(pi(y_j - y_n))|
    k_logsum<<<(unsigned)nb(N), 256, 0, st>>>(q.x.as<double>(), N, q.y.as<double>(), N, 0, 1.0, la.as<double>(),
                                              na.as<int>(), bad.as<int>());
    INFT_CHECK_LAUNCH();
    k_logsum<<<(unsigned)nb(N), 256, 0, st>>>(q.y.as<double>(), N, q.y.as<double>(), N, 1, -1.0, lb.as<double>(),
                                              nbn.as<int>(), bad.as<int>());
    INFT_CHECK_LAUNCH();
    }
    // steps 2-3: shift, exponentials, signs
    k_shift<<<1, 256, 0, st>>>(la.as<double>(), lb.as<double>(), N, q.s.as<double>());
    INFT_CHECK_LAUNCH();
    k_signed<<<(unsigned)nb(N), 256, 0, st>>>(la.as<double>(), na.as<int>(), N, q.s.as<double>(), 1.0, q.a.as<double>());
    INFT_CHECK_LAUNCH();
    k_signed<<<(unsigned)nb(N), 256, 0, st>>>(lb.as<double>(), nbn.as<int>(), N, q.s.as<double>(), -1.0,
                                              q.b.as<double>());
    INFT_CHECK_LAUNCH();
    q.launches += 5;
    int hb = 0;
    INFT_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    if (hb) {
        set_error("quadratic case: coincident nodes (a node equals a target x_l or another node)");
        throw Fail{INFT_ERR_NODE_RANGE};
    }
}

// in/out: device or host [R][N] complex128 (host data staged synchronously)
template <typename Body>
static void with_device_io(QPlan& q, const void* in, void* out, int64_t R, cudaStream_t st, Body&& body) {
    const size_t bytes = sizeof(double2) * (size_t)R * (size_t)q.N;
    const bool din = is_device_pointer(in), dout = is_device_pointer(out);
    DevBuf ti, to;
    const double2* di = static_cast<const double2*>(in);
    double2* dov = static_cast<double2*>(out);
    if (!din) {
        ti.alloc(bytes);
        INFT_CUDA(cudaMemcpyAsync(ti.p, in, bytes, cudaMemcpyHostToDevice, st));
        di = ti.as<double2>();
    }
    if (!dout) {
        to.alloc(bytes);
        dov = to.as<double2>();
    }
    body(di, dov);
    if (!dout) {
        INFT_CUDA(cudaMemcpyAsync(out, dov, bytes, cudaMemcpyDeviceToHost, st));
    }
    if (!din || !dout) INFT_CUDA(cudaStreamSynchronize(st));
}

static void apply_inverse(QPlan& q, const double2* f, double2* fhat, int64_t R, cudaStream_t st) {
    const int64_t N = q.N, tot = R * N;
    q.ensure_ws(R);
    double2 *c = q.w1.as<double2>(), *gt = q.w2.as<double2>(), *g = q.w3.as<double2>();
    k_scale<<<(unsigned)nb(tot), 256, 0, st>>>(f, q.b.as<double>(), N, tot, c);  // f_j b_j
    k_rowsum<<<(unsigned)R, 256, 0, st>>>(c, N, q.sums.as<double2>());          // sum_j f_j b_j
    if (q.fast) {  // eq. coeff_g_tilde by the fast summation: far field (NFFT^*, fold, FFT) + near field
        q.ensure_wfs(R);
        check_status(inft_apply(q.nfft, c, q.wfs.p, R, (inft_stream_t)st), "inner adjoint NFFT");
        k_fs_fold<<<(unsigned)nb(tot), 256, 0, st>>>(q.wfs.as<double2>(), q.bcot.as<double2>(), q.nfs, N, R, q.delta,
                                                     gt);
        INFT_CHECK_LAUNCH();
        cufftHandle hf = q.plan_for(R, st);
        if (cufftExecZ2Z(hf, (cufftDoubleComplex*)gt, (cufftDoubleComplex*)gt, CUFFT_INVERSE) != CUFFT_SUCCESS) {
            set_error("cufftExecZ2Z (fast summation, far field) failed");
            throw Fail{INFT_ERR_CUFFT};
        }
        k_fs_near_sorted<<<(unsigned)nb(tot), 256, 0, st>>>(0, q.Tcot, q.eps, q.x.as<double>(), N, q.ys.as<double>(),
                                                            q.yidx.as<int32_t>(), N, c, R, 0, gt);
        q.launches += 2;
    } else {
    dim3 grid((unsigned)nb(N, 128), (unsigned)nb(R, kRG));
    k_cotsum<<<grid, 128, 0, st>>>(q.x.as<double>(), N, q.y.as<double>(), N, c, R, gt);  // eq. coeff_g_tilde
    }
    k_glue_inv<<<(unsigned)nb(tot), 256, 0, st>>>(gt, q.a.as<double>(), q.sums.as<double2>(), N, tot, g);
    INFT_CHECK_LAUNCH();
    cufftHandle h = q.plan_for(R, st);
    if (cufftExecZ2Z(h, (cufftDoubleComplex*)g, (cufftDoubleComplex*)gt, CUFFT_FORWARD) != CUFFT_SUCCESS) {
        set_error("cufftExecZ2Z (quadratic case, step 6) failed");
        throw Fail{INFT_ERR_CUFFT};
    }
    k_post_inv<<<(unsigned)nb(tot), 256, 0, st>>>(gt, N, tot, q.delta, fhat);
    INFT_CHECK_LAUNCH();
    q.launches += 5;
}

static void apply_adjoint(QPlan& q, const double2* h, double2* f, int64_t R, cudaStream_t st) {
    const int64_t N = q.N, tot = R * N;
    q.ensure_ws(R);
    double2 *u = q.w1.as<double2>(), *v = q.w2.as<double2>(), *ct = q.w3.as<double2>();
    k_pre_adj<<<(unsigned)nb(tot), 256, 0, st>>>(h, N, tot, q.delta, u);
    INFT_CHECK_LAUNCH();
    cufftHandle hp = q.plan_for(R, st);
    if (cufftExecZ2Z(hp, (cufftDoubleComplex*)u, (cufftDoubleComplex*)v, CUFFT_INVERSE) != CUFFT_SUCCESS) {
        set_error("cufftExecZ2Z (quadratic case, adjoint) failed");
        throw Fail{INFT_ERR_CUFFT};
    }
    k_scale<<<(unsigned)nb(tot), 256, 0, st>>>(v, q.a.as<double>(), N, tot, u);  // w_l = a_l v_l
    k_rowsum<<<(unsigned)R, 256, 0, st>>>(u, N, q.sums.as<double2>());          // sum_l w_l
    if (q.fast) {  // sum_l w_l cot(pi (y_j - x_l)): far field (FFT, pre, NFFT) + near field
        q.ensure_wfs(R);
        cufftHandle hf = q.plan_for(R, st);
        if (cufftExecZ2Z(hf, (cufftDoubleComplex*)u, (cufftDoubleComplex*)v, CUFFT_FORWARD) != CUFFT_SUCCESS) {
            set_error("cufftExecZ2Z (fast summation, far field) failed");
            throw Fail{INFT_ERR_CUFFT};
        }
        k_fs_pre<<<(unsigned)nb(R * q.nfs), 256, 0, st>>>(v, q.bcot.as<double2>(), q.nfs, N, R, q.delta,
                                                          q.wfs.as<double2>());
        INFT_CHECK_LAUNCH();
        check_status(inft_adjoint_apply(q.nfft, q.wfs.p, ct, R, (inft_stream_t)st), "inner NFFT");
        k_fs_near_equi<<<(unsigned)nb(tot), 256, 0, st>>>(0, q.Tcot, q.eps, q.y.as<double>(), N, N, q.delta, u, R, ct);
        q.launches += 2;
    } else {
    dim3 grid((unsigned)nb(N, 128), (unsigned)nb(R, kRG));
    k_cotsum<<<grid, 128, 0, st>>>(q.y.as<double>(), N, q.x.as<double>(), N, u, R, ct);
    }
    k_glue_adj<<<(unsigned)nb(tot), 256, 0, st>>>(ct, q.b.as<double>(), q.sums.as<double2>(), N, tot, f);
    INFT_CHECK_LAUNCH();
    q.launches += 5;
}

}  // namespace quad
}  // namespace inft

using inft::Fail;

#define INFT_Q_TRY try {
#define INFT_Q_CATCH                                          \
    }                                                         \
    catch (const Fail& f_) {                                  \
        return f_.st;                                         \
    }                                                         \
    catch (const std::bad_alloc&) {                           \
        inft::set_error("host allocation failed");            \
        return INFT_ERR_OOM;                                  \
    }                                                         \
    catch (...) {                                             \
        inft::set_error("unexpected C++ exception");          \
        return INFT_ERR_CUDA;                                 \
    }                                                         \
    return INFT_OK;

extern "C" {

inft_status inft_quad_plan(inft_quad_t* out, int64_t N, const double* nodes, double delta, int device,
                           inft_stream_t stream) {
    if (!out) return INFT_ERR_INVALID_ARG;
    *out = nullptr;
    if (N < 2 || (N & 1) || !nodes || N > (int64_t(1) << 30)) return INFT_ERR_INVALID_ARG;
    if (delta == 0.0) delta = 0.5 / (double)N;  // reading A23
    if (!(delta > 0.0 && delta < 1.0 / (double)N)) return INFT_ERR_INVALID_ARG;
    INFT_Q_TRY
    inft::DeviceGuard g(device);
    auto* q = new inft::quad::QPlan();
    q->N = N;
    q->device = device;
    q->delta = delta;
    try {
        inft::quad::build(*q, nodes, (cudaStream_t)stream);
    } catch (...) {
        delete q;
        throw;
    }
    *out = reinterpret_cast<inft_quad_t>(q);
    INFT_Q_CATCH
}

inft_status inft_quad_apply(inft_quad_t plan, const void* f, void* fhat, int64_t R, inft_stream_t stream) {
    if (!plan || R < 0) return INFT_ERR_INVALID_ARG;
    if (R == 0) return INFT_OK;
    if (!f || !fhat) return INFT_ERR_INVALID_ARG;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    const cudaStream_t st = (cudaStream_t)stream;
    inft::quad::with_device_io(*q, f, fhat, R, st, [&](const double2* di, double2* dout) {
        inft::quad::apply_inverse(*q, di, dout, R, st);
    });
    INFT_Q_CATCH
}

inft_status inft_quad_adjoint_apply(inft_quad_t plan, const void* h, void* f, int64_t R, inft_stream_t stream) {
    if (!plan || R < 0) return INFT_ERR_INVALID_ARG;
    if (R == 0) return INFT_OK;
    if (!h || !f) return INFT_ERR_INVALID_ARG;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    const cudaStream_t st = (cudaStream_t)stream;
    inft::quad::with_device_io(*q, h, f, R, st, [&](const double2* di, double2* dout) {
        inft::quad::apply_adjoint(*q, di, dout, R, st);
    });
    INFT_Q_CATCH
}

inft_status inft_quad_get_coeffs(inft_quad_t plan, double* x, double* a, double* b, double* s) {
    if (!plan) return INFT_ERR_INVALID_ARG;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    INFT_CUDA(cudaDeviceSynchronize());
    const size_t bytes = sizeof(double) * (size_t)q->N;
    if (x) INFT_CUDA(cudaMemcpy(x, q->x.p, bytes, cudaMemcpyDeviceToHost));
    if (a) INFT_CUDA(cudaMemcpy(a, q->a.p, bytes, cudaMemcpyDeviceToHost));
    if (b) INFT_CUDA(cudaMemcpy(b, q->b.p, bytes, cudaMemcpyDeviceToHost));
    if (s) INFT_CUDA(cudaMemcpy(s, q->s.p, sizeof(double), cudaMemcpyDeviceToHost));
    INFT_Q_CATCH
}

inft_status inft_quad_kernel_launches(inft_quad_t plan, int64_t* count) {
    if (!plan || !count) return INFT_ERR_INVALID_ARG;
    *count = reinterpret_cast<inft::quad::QPlan*>(plan)->launches;
    return INFT_OK;
}

inft_status inft_quad_destroy(inft_quad_t plan) {
    if (!plan) return INFT_OK;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    delete q;
    INFT_Q_CATCH
}

}  // extern "C"
