// Setup stage: B_opt on the GPU.
//
// INFT_ALG2_GRIDWISE -- Alg. "Fast optimization of the matrix B".
//   For every grid point l the column b~_l of B_opt minimises ||L_l b - e_l||_2
//   over real b, L_l = F D H_l (eq. matrix_Ll).
//   Because F^* F = M_sigma I_M (M <= M_sigma) the normal equations are
//     Re(G(x_j - x_j')) b = Re(K+(x_j - l/M_sigma)),  j, j' in I(l)
//   with G(x) = (1/M_sigma) sum_k e^{2 pi i k x}/what(k)^2 and
//   K+(x) = (1/M_sigma) sum_k e^{2 pi i k x}/what(k).
//   Only |x| <= (2m+1)/M_sigma is ever needed, where both kernels are smooth
//   (<= ~m/sigma oscillations): they are tabulated once as piecewise Chebyshev
//   interpolants of degree 16 whose samples are exact direct sums over k.
//   2-D (reading A12): G = G1 G2, K+ = K+1 K+2 (separable; the unpaired
//   k = -M/2 term makes the factors complex, Re is taken of the product).
// INFT_ALG1_NODEWISE -- Alg. "Fast optimization of the matrix B*".
//   K = A D^* F^* (eq. matrix_K) is formed row by row with one M_sigma-point
//   FFT per node (batched cuFFT), then per node j the normal equations
//   Re(K_j^* K_j) b = M Re(K_j^* e_j) (eq. solution_ansatz1).
// Every small symmetric system is solved by cyclic Jacobi (one CTA per column,
// parallel round-robin rotations) with the minimum-norm cutoff of reading A6:
// eigenvalues below tau^2 lambda_max are dropped (tau on singular values).
// INFT_PLAIN_NFFT -- the window matrix B (eq. matrix_B), KB window (reading A7).
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <vector>

#include "inft_internal.cuh"

namespace inft {

static constexpr double kPi = 3.141592653589793238462643383279502884;
static constexpr int kChebDeg = 16;  // Chebyshev degree per piece

static inline unsigned nblk(int64_t n, int bs = 256) { return (unsigned)std::max<int64_t>(1, ceil_div(n, bs)); }

__device__ __forceinline__ int64_t md(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

// ------------------------------------------------------------------ sorted node copies
__global__ void k_sorted_nodes(const double* __restrict__ x, const int32_t* __restrict__ l0,
                               const int32_t* __restrict__ perm, int64_t N, int d, double* __restrict__ xs,
                               int32_t* __restrict__ l0s) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int64_t j = perm[i];
    for (int k = 0; k < d; k++) {
        xs[i * d + k] = x[j * d + k];
        l0s[i * d + k] = l0[j * d + k];
    }
}

// Is slot t of a node (coordinate x, base l0) in the support: |Ms x - (l0 + t)| <= m.
// Same arithmetic as the oracle: one rounded product, then subtraction.
__device__ __forceinline__ bool in_support(double x, int64_t l0, int64_t t, int64_t Ms, int m) {
    double v = __dmul_rn((double)Ms, x) - (double)(l0 + t);
    return v >= -(double)m && v <= (double)m;
}

// First in-support slot t of the node on grid point n (mod Ms), or -1.  Later
// in-support slots congruent mod Ms are aliases (reading A5) and not unknowns.
__device__ __forceinline__ int64_t live_slot(int64_t n, int64_t n0, double x, int64_t l0, int P, int64_t Ms, int m) {
    for (int64_t t = md(n - n0, Ms); t < P; t += Ms)
        if (in_support(x, l0, t, Ms, m)) return t;
    return -1;
}

// Visit every (sorted node i, slot t) of column n = (n1, n2) (eq. set_l).  F(i, t).
struct ColCtx {
    const int32_t* seg_start;
    const int32_t* n0s;
    const double* xs;
    const int32_t* l0s;
    int d, m, P1, S1, S2;
    int64_t Ms1, Ms2, nseg2;
};

template <typename Fn>
__device__ void for_column(const ColCtx& c, int64_t n, int lane, int nlanes, Fn&& fn) {
    int64_t n1 = c.d == 2 ? n / c.Ms2 : n;
    int64_t n2 = c.d == 2 ? n - (n / c.Ms2) * c.Ms2 : 0;
    const int64_t nseg1 = (c.Ms1 + c.S1 - 1) / c.S1;
    for_segments(n1, std::min<int64_t>(c.P1, c.Ms1), c.Ms1, c.S1, nseg1, [&](int64_t s1) {
        if (c.d == 1) {
            for (int64_t i = c.seg_start[s1] + lane; i < c.seg_start[s1 + 1]; i += nlanes) {
                int64_t t = live_slot(n1, c.n0s[i], c.xs[i], c.l0s[i], c.P1, c.Ms1, c.m);
                if (t >= 0) fn(i, t);
            }
        } else {
            for_segments(n2, std::min<int64_t>(c.P1, c.Ms2), c.Ms2, c.S2, c.nseg2, [&](int64_t s2) {
                int64_t tile = s1 * c.nseg2 + s2;
                for (int64_t i = c.seg_start[tile] + lane; i < c.seg_start[tile + 1]; i += nlanes) {
                    int64_t t1 = live_slot(n1, c.n0s[2 * i], c.xs[2 * i], c.l0s[2 * i], c.P1, c.Ms1, c.m);
                    if (t1 < 0) continue;
                    int64_t t2 = live_slot(n2, c.n0s[2 * i + 1], c.xs[2 * i + 1], c.l0s[2 * i + 1], c.P1, c.Ms2, c.m);
                    if (t2 < 0) continue;
                    fn(i, t1 * c.P1 + t2);
                }
            });
        }
    });
}

__global__ void k_col_count(ColCtx c, int64_t ncol, int32_t* __restrict__ cnt) {
    int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= ncol) return;
    int k = 0;
    for_column(c, n, 0, 1, [&](int64_t, int64_t) { k++; });
    cnt[n] = k;
}

// ------------------------------------------------------------------ kernel tables
// 1/(M_sigma what(k)) = 1/I0(m sqrt(b^2 - (2 pi k/Ms)^2)) for k = 0..M/2 (even window).
__global__ void k_inv_what(double* __restrict__ iw, int64_t M, int64_t Ms, int m, double sigma, int window) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k > M / 2) return;
    if (window == INFT_DIRICHLET) {  // what = 1; the unpaired frequency (stored at k = M/2) zeroed (reading A21)
        iw[k] = k == M / 2 ? 0.0 : 1.0 / (double)Ms;
        return;
    }
    if (window == INFT_BSPLINE) {  // 1/(M_sigma what(k)) = sinc(pi k/M_sigma)^{-2m} (reading A24)
        const double t = (double)k / (double)Ms;
        const double sc = k == 0 ? 1.0 : sinpi(t) / (kPi * t);
        iw[k] = 1.0 / pow(sc, 2.0 * m);
        return;
    }
    double b = kPi * (2.0 - 1.0 / sigma);
    double u = 2.0 * kPi * (double)k / (double)Ms;
    iw[k] = 1.0 / cyl_bessel_i0((double)m * sqrt(fmax(__dsub_rn(__dmul_rn(b, b), __dmul_rn(u, u)), 0.0)));
}

// Exact samples of Re G and Re K+ at the Chebyshev points of every piece:
//   Re G(x)  = Ms [iw0^2 + 2 sum_{k=1}^{M/2-1} iw_k^2 cos(2 pi k x) + iw_{M/2}^2 cos(pi M x)]
//   Re K+(x) =     iw0   + 2 sum_{k=1}^{M/2-1} iw_k   cos(2 pi k x) + iw_{M/2}   cos(pi M x)
// (G = (1/Ms) sum_k e^{..}/what^2 = Ms sum_k iw_k^2 e^{..} since iw = 1/(Ms what)).
__global__ void k_cheb_samples(const double* __restrict__ iw, int64_t M, int64_t Ms, double X, double pw, int npc,
                               double* __restrict__ sampG, double* __restrict__ sampK) {
    const int sidx = blockIdx.x;  // piece * (deg+1) + node
    const int pc = sidx / (kChebDeg + 1), q = sidx % (kChebDeg + 1);
    const double tq = cos(kPi * (q + 0.5) / (kChebDeg + 1));
    const double x = -X + pc * pw + 0.5 * pw * (tq + 1.0);
    double sg = 0.0, sk = 0.0;
    for (int64_t k = 1 + threadIdx.x; k < M / 2; k += blockDim.x) {
        double c = cospi(2.0 * (double)k * x);
        sg += iw[k] * iw[k] * c;
        sk += iw[k] * c;
    }
    __shared__ double rg[256], rk[256];
    rg[threadIdx.x] = sg;
    rk[threadIdx.x] = sk;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            rg[threadIdx.x] += rg[threadIdx.x + o];
            rk[threadIdx.x] += rk[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double ch = cospi((double)M * x);
        double h = iw[M / 2];
        sampG[sidx] = (double)Ms * (iw[0] * iw[0] + 2.0 * rg[0] + h * h * ch);
        sampK[sidx] = iw[0] + 2.0 * rk[0] + h * ch;
    }
}

// Chebyshev coefficients c_j = (2/(D+1)) sum_q f(t_q) cos(pi j (q+1/2)/(D+1)), c_0 halved.
__global__ void k_cheb_coef(const double* __restrict__ samp, int npc, double* __restrict__ coef) {
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= npc * (kChebDeg + 1)) return;
    int pc = idx / (kChebDeg + 1), j = idx % (kChebDeg + 1);
    double s = 0.0;
    for (int q = 0; q <= kChebDeg; q++)
        s += samp[pc * (kChebDeg + 1) + q] * cos(kPi * j * (q + 0.5) / (kChebDeg + 1));
    s *= 2.0 / (kChebDeg + 1);
    if (j == 0) s *= 0.5;
    coef[idx] = s;
}

struct KTab {
    double X, pw;
    int npc;
    const double* cG;
    const double* cK;
    double Msd, Md, imG, imK;  // Im G(x) = -imG sin(pi M x), Im K+(x) = -imK sin(pi M x)
};

__device__ __forceinline__ double cheb_eval(const double* __restrict__ c, double t) {
    double b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int j = kChebDeg; j >= 1; j--) {
        double b0 = fma(2.0 * t, b1, c[j] - b2);
        b2 = b1;
        b1 = b0;
    }
    return fma(t, b1, c[0] - b2);
}

__device__ __forceinline__ double tab_eval(const KTab& T, const double* coef, double x) {
    double u = (x + T.X) / T.pw;
    int pc = (int)floor(u);
    pc = pc < 0 ? 0 : (pc >= T.npc ? T.npc - 1 : pc);
    double t = 2.0 * (u - pc) - 1.0;
    return cheb_eval(coef + pc * (kChebDeg + 1), t);
}

__device__ __forceinline__ double wrapd(double a) { return a - floor(a + 0.5); }

// Gram entry and right-hand side of column n for unknowns (i, i'), 1-D or 2-D.
struct GramCtx {
    KTab t1, t2;
    int d;
    const double* xs;
};

__device__ __forceinline__ double gram_entry(const GramCtx& g, int64_t a, int64_t b) {
    if (g.d == 1) return tab_eval(g.t1, g.t1.cG, wrapd(g.xs[a] - g.xs[b]));
    double d1 = wrapd(g.xs[2 * a] - g.xs[2 * b]);
    double d2 = wrapd(g.xs[2 * a + 1] - g.xs[2 * b + 1]);
    double r1 = tab_eval(g.t1, g.t1.cG, d1), r2 = tab_eval(g.t2, g.t2.cG, d2);
    double i1 = -g.t1.imG * sinpi(g.t1.Md * d1), i2 = -g.t2.imG * sinpi(g.t2.Md * d2);
    return r1 * r2 - i1 * i2;
}

__device__ __forceinline__ double rhs_entry(const GramCtx& g, int64_t a, int64_t n) {
    if (g.d == 1) return tab_eval(g.t1, g.t1.cK, wrapd(g.xs[a] - (double)n / g.t1.Msd));
    int64_t Ms2 = (int64_t)g.t2.Msd;
    int64_t n1 = n / Ms2, n2 = n - (n / Ms2) * Ms2;
    double d1 = wrapd(g.xs[2 * a] - (double)n1 / g.t1.Msd);
    double d2 = wrapd(g.xs[2 * a + 1] - (double)n2 / g.t2.Msd);
    double r1 = tab_eval(g.t1, g.t1.cK, d1), r2 = tab_eval(g.t2, g.t2.cK, d2);
    double i1 = -g.t1.imK * sinpi(g.t1.Md * d1), i2 = -g.t2.imK * sinpi(g.t2.Md * d2);
    return r1 * r2 - i1 * i2;
}

// ------------------------------------------------------------------ Jacobi eigen-solver
// Cyclic two-sided Jacobi with the round-robin (circle) ordering: n'/2
// disjoint rotations per step, all threads of the CTA cooperate.  A (n x n,
// leading dimension ld) is overwritten by its eigenvalues on the diagonal, V
// by the eigenvectors (columns).  Rotation (Golub-Van Loan, symmetric Schur):
// tau = (a_qq - a_pp)/(2 a_pq), t = sign(tau)/(|tau| + sqrt(1 + tau^2)),
// c = 1/sqrt(1 + t^2), s = t c; A <- J^T A J with J_pp = J_qq = c, J_pq = s, J_qp = -s.
// sweep statistics (INFT_SETUP_DEBUG=1 prints them after Alg. 2): total sweeps, calls, max
__device__ unsigned long long g_jac_stats[3];
// large-column solver phase cycles (thread 0 of each CTA): collect+sort, diag, pivoted
// Cholesky, C = L^T L, Jacobi, back-substitution
__device__ unsigned long long g_lr_cycles[6];

__device__ void jacobi_eig(double* A, double* V, int n, int ld, double* cs, int* pq, int* flag) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int np = (n + 1) & ~1;
    const int half = np / 2;
    for (int idx = tid; idx < n * n; idx += nt) {
        int i = idx / n, j = idx % n;
        V[i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
    __shared__ double s_tol;
    if (tid == 0) {
        double mx = 0.0;
        for (int i = 0; i < n; i++) mx = fmax(mx, fabs(A[i * ld + i]));
        // off-diagonal entries below 1e-15 of the largest diagonal entry are rounding noise
        // (two-sided rotations cannot push the entries next to a large diagonal entry lower);
        // they move eigenvalues by at most that much (Weyl), i.e. within the min-norm cutoff's
        // tau^2 lambda_max = 1e-12 lambda_max by a factor 1e-3
        s_tol = 1e-15 * mx;
    }
    __syncthreads();
    const double tol = s_tol;
    for (int sweep = 0; sweep < 60; sweep++) {
        if (tid == 0) *flag = 0;
        __syncthreads();
        for (int r = 0; r < np - 1; r++) {
            for (int k = tid; k < half; k += nt) {
                int pa = k == 0 ? 0 : ((k - 1 + r) % (np - 1)) + 1;
                int kb = np - 1 - k;
                int pb = ((kb - 1 + r) % (np - 1)) + 1;
                int p = min(pa, pb), q = max(pa, pb);
                double c = 1.0, s = 0.0;
                if (q < n) {
                    double apq = A[p * ld + q];
                    if (fabs(apq) > tol) {
                        double app = A[p * ld + p], aqq = A[q * ld + q];
                        double tau = (aqq - app) / (2.0 * apq);
                        double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                        *flag = 1;
                    }
                }
                cs[2 * k] = c;
                cs[2 * k + 1] = s;
                pq[2 * k] = p;
                pq[2 * k + 1] = q;
            }
            __syncthreads();
            // rows: A <- J^T A
            for (int idx = tid; idx < half * n; idx += nt) {
                int k = idx / n, j = idx % n;
                double s = cs[2 * k + 1];
                if (s == 0.0) continue;
                double c = cs[2 * k];
                int p = pq[2 * k], q = pq[2 * k + 1];
                double a = A[p * ld + j], b = A[q * ld + j];
                A[p * ld + j] = c * a - s * b;
                A[q * ld + j] = s * a + c * b;
            }
            __syncthreads();
            // columns: A <- A J, V <- V J
            for (int idx = tid; idx < half * n; idx += nt) {
                int k = idx / n, i = idx % n;
                double s = cs[2 * k + 1];
                if (s == 0.0) continue;
                double c = cs[2 * k];
                int p = pq[2 * k], q = pq[2 * k + 1];
                double a = A[i * ld + p], b = A[i * ld + q];
                A[i * ld + p] = c * a - s * b;
                A[i * ld + q] = s * a + c * b;
                double va = V[i * ld + p], vb = V[i * ld + q];
                V[i * ld + p] = c * va - s * vb;
                V[i * ld + q] = s * va + c * vb;
            }
            __syncthreads();
        }
        if (*flag == 0) {
            if (tid == 0) {
                atomicAdd(&g_jac_stats[0], (unsigned long long)(sweep + 1));
                atomicAdd(&g_jac_stats[1], 1ull);
                atomicMax(&g_jac_stats[2], (unsigned long long)(sweep + 1));
            }
            break;
        }
        __syncthreads();
        if (sweep == 59 && tid == 0) {
            atomicAdd(&g_jac_stats[0], 60ull);
            atomicAdd(&g_jac_stats[1], 1ull);
            atomicMax(&g_jac_stats[2], 60ull);
        }
    }
}

// Jacobi for the large-column solver, without eigenvectors: the rotations are (a) applied to the
// vector t on the fly (t <- J^T t, so t ends as V^T t) and (b) logged per round in `log`
// ([round][np] (c, s) pairs, at most max_rounds rounds) so that V u can be formed afterwards
// (jacobi_apply_v).  Returns the number of logged rounds.
// Storage: A holds the upper triangle of an
// np x np symmetric matrix (np = n rounded up to even; the pad row/column is zero), element
// (i, j), i <= j, at pidx(i, j).  One round applies all disjoint rotations of the round-robin
// ordering at once, A <- J^T A J, as independent 2 x 2 block updates: for rotation pairs
// (p, q) and (p', q') the block A[{p, q}][{p', q'}] becomes R^T B R' with R = [[c, s], [-s, c]]
// (the same rotation as jacobi_eig).  One read and one write per element and one barrier per
// round, so the k x k problem of a big column fits shared memory in packed form (k <= 230).
__device__ __forceinline__ int pidx(int i, int j, int np) {
    if (i > j) {
        const int t = i;
        i = j;
        j = t;
    }
    return i * np - (i * (i - 1)) / 2 + (j - i);
}

__host__ __device__ inline size_t packed_doubles(int n) {
    const size_t np = (size_t)((n + 1) & ~1);
    return np * (np + 1) / 2;
}

__device__ int jacobi_packed_log(double* A, int n, double* t, double* log, int max_rounds, double* cs, int* pq,
                                 int* flag) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int np = (n + 1) & ~1;
    const int half = np / 2;
    __shared__ double s_tol;
    if (tid == 0) {
        double mx = 0.0;
        for (int i = 0; i < n; i++) mx = fmax(mx, fabs(A[pidx(i, i, np)]));
        s_tol = 1e-15 * mx;  // as jacobi_eig
    }
    __syncthreads();
    const double tol = s_tol;
    int g = 0, sweeps = 0;
    for (int sweep = 0; g + np - 1 <= max_rounds; sweep++) {
        if (tid == 0) *flag = 0;
        __syncthreads();
        for (int r = 0; r < np - 1; r++, g++) {
            for (int k = tid; k < half; k += nt) {
                int pa = k == 0 ? 0 : ((k - 1 + r) % (np - 1)) + 1;
                int kb = np - 1 - k;
                int pb = ((kb - 1 + r) % (np - 1)) + 1;
                int p = min(pa, pb), q = max(pa, pb);
                double c = 1.0, s = 0.0;
                if (q < n) {
                    double apq = A[pidx(p, q, np)];
                    if (fabs(apq) > tol) {
                        double app = A[pidx(p, p, np)], aqq = A[pidx(q, q, np)];
                        double tau = (aqq - app) / (2.0 * apq);
                        double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + tt * tt);
                        s = tt * c;
                        *flag = 1;
                        const double a = t[p], b = t[q];
                        t[p] = c * a - s * b;
                        t[q] = s * a + c * b;
                    }
                }
                cs[2 * k] = c;
                cs[2 * k + 1] = s;
                pq[2 * k] = p;
                pq[2 * k + 1] = q;
                log[(size_t)g * np + 2 * k] = c;
                log[(size_t)g * np + 2 * k + 1] = s;
            }
            __syncthreads();
            for (int a = warp; a < half; a += nw) {
                const double ca = cs[2 * a], sa = cs[2 * a + 1];
                const int p = pq[2 * a], q = pq[2 * a + 1];
                for (int b = a + lane; b < half; b += 32) {
                    const double cb = cs[2 * b], sb = cs[2 * b + 1];
                    if (sa == 0.0 && sb == 0.0) continue;
                    const int p2 = pq[2 * b], q2 = pq[2 * b + 1];
                    if (b == a) {  // diagonal block [[app, apq], [apq, aqq]]
                        const int ipp = pidx(p, p, np), ipq = pidx(p, q, np), iqq = pidx(q, q, np);
                        const double app = A[ipp], apq = A[ipq], aqq = A[iqq];
                        // R^T M R with R = [[c, s], [-s, c]]
                        const double m00 = ca * app - sa * apq, m01 = ca * apq - sa * aqq;
                        const double m10 = sa * app + ca * apq, m11 = sa * apq + ca * aqq;
                        A[ipp] = ca * m00 - sa * m01;
                        A[ipq] = sa * m00 + ca * m01;
                        A[iqq] = sa * m10 + ca * m11;
                    } else {
                        const int i00 = pidx(p, p2, np), i01 = pidx(p, q2, np), i10 = pidx(q, p2, np),
                                  i11 = pidx(q, q2, np);
                        const double x00 = A[i00], x01 = A[i01], x10 = A[i10], x11 = A[i11];
                        // rows: R_a^T; columns: R_b
                        const double y00 = ca * x00 - sa * x10, y01 = ca * x01 - sa * x11;
                        const double y10 = sa * x00 + ca * x10, y11 = sa * x01 + ca * x11;
                        A[i00] = cb * y00 - sb * y01;
                        A[i01] = sb * y00 + cb * y01;
                        A[i10] = cb * y10 - sb * y11;
                        A[i11] = sb * y10 + cb * y11;
                    }
                }
            }
            __syncthreads();
        }
        sweeps = sweep + 1;
        if (*flag == 0) break;
        __syncthreads();
    }
    if (tid == 0) {
        atomicAdd(&g_jac_stats[0], (unsigned long long)sweeps);
        atomicAdd(&g_jac_stats[1], 1ull);
        atomicMax(&g_jac_stats[2], (unsigned long long)sweeps);
    }
    __syncthreads();
    return g;
}

// v <- V v for the V of jacobi_packed_log (V = J_1 J_2 ... J_G, the rounds' rotations in
// order): rounds applied in reverse order.
__device__ void jacobi_apply_v(double* v, int n, const double* log, int rounds) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int np = (n + 1) & ~1;
    const int half = np / 2;
    for (int g = rounds - 1; g >= 0; g--) {
        const int r = g % (np - 1);
        for (int k = tid; k < half; k += nt) {
            const double s = log[(size_t)g * np + 2 * k + 1];
            if (s == 0.0) continue;
            const double c = log[(size_t)g * np + 2 * k];
            int pa = k == 0 ? 0 : ((k - 1 + r) % (np - 1)) + 1;
            int kb = np - 1 - k;
            int pb = ((kb - 1 + r) % (np - 1)) + 1;
            int p = min(pa, pb), q = max(pa, pb);
            const double a = v[p], b = v[q];
            v[p] = c * a + s * b;
            v[q] = -s * a + c * b;
        }
        __syncthreads();
    }
}

// b = V diag(1/lambda) V^T y over eigenvalues lambda > tau^2 lambda_max; returns #dropped.
__device__ int minnorm_from_eig(const double* A, const double* V, int n, int ld, const double* y, double* u,
                                double* b, double tau2) {
    const int tid = threadIdx.x, nt = blockDim.x;
    __shared__ double s_lmax;
    __shared__ int s_drop;
    if (tid == 0) {
        double mx = 0.0;
        for (int i = 0; i < n; i++) mx = fmax(mx, A[i * ld + i]);
        s_lmax = mx;
        int dr = 0;
        for (int i = 0; i < n; i++) dr += !(A[i * ld + i] > tau2 * mx);
        s_drop = dr;
    }
    __syncthreads();
    const double cut = tau2 * s_lmax;
    for (int k = tid; k < n; k += nt) {
        double lam = A[k * ld + k];
        double s = 0.0;
        if (lam > cut && s_lmax > 0.0)
            for (int i = 0; i < n; i++) s += V[i * ld + k] * y[i];
        u[k] = (lam > cut && s_lmax > 0.0) ? s / lam : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < n; i += nt) {
        double s = 0.0;
        for (int k = 0; k < n; k++) s += V[i * ld + k] * u[k];
        b[i] = s;
    }
    __syncthreads();
    return s_drop;
}

// ------------------------------------------------------------------ Alg. 2 column solve
// One CTA per column.  Unknown list, Gram matrix and eigenvectors live in
// shared memory (nmax <= smem limit) or in a global scratch slice per CTA.
__global__ void k_alg2_solve(ColCtx cc, GramCtx gc, const int64_t* __restrict__ cols, int64_t ncols,
                             const int32_t* __restrict__ cnt, int nmax, int use_global, double* __restrict__ scratch,
                             double tau2, int P, double* __restrict__ w64, unsigned long long* __restrict__ ndrop) {
    extern __shared__ double sm[];
    const int ld = nmax + 1;
    double *A, *V, *y, *u, *b;
    size_t slot = (size_t)blockIdx.x;
    double* base = use_global ? scratch + slot * (size_t)(2 * nmax * ld + 3 * nmax) : sm;
    A = base;
    V = A + (size_t)nmax * ld;
    y = V + (size_t)nmax * ld;
    u = y + nmax;
    b = u + nmax;
    // small per-CTA lists in shared memory after the matrices (smem case) or at the start (global case)
    int64_t* li = reinterpret_cast<int64_t*>(use_global ? sm : (double*)(b + nmax));
    int* lt = reinterpret_cast<int*>(li + nmax);
    double* cs = reinterpret_cast<double*>(lt + nmax + (nmax & 1));
    int* pq = reinterpret_cast<int*>(cs + nmax + 2);
    int* cntr = pq + nmax + 2;
    for (int64_t ci = blockIdx.x; ci < ncols; ci += gridDim.x) {
        const int64_t n = cols[ci];
        const int nc = cnt[n];
        if (threadIdx.x == 0) *cntr = 0;
        __syncthreads();
        // collect unknowns (order fixed afterwards by sorting on (i, t) for determinism)
        for_column(cc, n, threadIdx.x, blockDim.x, [&](int64_t i, int64_t t) {
            int k = atomicAdd(cntr, 1);
            if (k < nmax) {
                li[k] = i;
                lt[k] = (int)t;
            }
        });
        __syncthreads();
        if (threadIdx.x == 0) {  // insertion sort by (i, t): deterministic unknown order
            for (int a = 1; a < nc; a++) {
                int64_t vi = li[a];
                int vt = lt[a];
                int q = a - 1;
                while (q >= 0 && (li[q] > vi || (li[q] == vi && lt[q] > vt))) {
                    li[q + 1] = li[q];
                    lt[q + 1] = lt[q];
                    q--;
                }
                li[q + 1] = vi;
                lt[q + 1] = vt;
            }
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) {
            int a = idx / nc, c = idx % nc;
            if (c >= a) {
                double g = gram_entry(gc, li[a], li[c]);
                A[a * ld + c] = g;
                A[c * ld + a] = g;
            }
        }
        for (int a = threadIdx.x; a < nc; a += blockDim.x) y[a] = rhs_entry(gc, li[a], n);
        __syncthreads();
        jacobi_eig(A, V, nc, ld, cs, pq, cntr);
        __syncthreads();
        int dropped = minnorm_from_eig(A, V, nc, ld, y, u, b, tau2);
        for (int a = threadIdx.x; a < nc; a += blockDim.x) w64[li[a] * P + lt[a]] = b[a];
        if (threadIdx.x == 0 && dropped > 0) atomicAdd(ndrop, 1ull);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ Alg. 2, large columns
// Block-wide argmax over v[0, n) (ties -> smallest index); every thread gets the result.
__device__ void block_argmax(const double* v, int n, double& vmax, int& imax, double* rv, int* ri) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double x = v[i];
        if (x > bv) {
            bv = x;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, bv, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    const int warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        rv[warp] = bv;
        ri[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; w++)
            if (rv[w] > rv[0] || (rv[w] == rv[0] && ri[w] < ri[0])) {
                rv[0] = rv[w];
                ri[0] = ri[w];
            }
    }
    __syncthreads();
    vmax = rv[0];
    imax = ri[0];
    __syncthreads();
}

// Large columns (|I(l)| > 64).  The Gram matrix G of a big column has a small numerical rank
// (config 4: n = 3528 unknowns, rank ~180-250 above 1e-15 of its diagonal), so instead of an
// O(n^3) eigensolve per column:
//   1. pivoted Cholesky G ~ L L^T (L: n x r, greedy largest-residual-diagonal pivots, columns of G
//      evaluated on demand, stop when every residual diagonal <= rel * max diag(G): far below the
//      tau^2 lambda_max cutoff since lambda_max >= max diag);
//   2. the r x r eigenproblem C = L^T L = W Lambda W^T (Jacobi; its nonzero eigenvalues are those of
//      L L^T), then the same min-norm cut as the small columns:
//      b = L W Lambda^{-2} W^T L^T y over lambda > tau^2 lambda_max  (= V Lambda^{-1} V^T y).
// Unknowns are put in canonical (i, t) order by rank counting (deterministic result).
struct LrScratch {
    double *L, *dg, *y, *C, *log, *z, *u;
    int64_t* li;
    int* lt;
    int64_t* li0;
    int* lt0;
};

constexpr int kLrSweeps = 24;  // rotation-log capacity in sweeps (config 4: <= 15 needed)

__host__ __device__ inline size_t lr_log_doubles(int rmax) { return (size_t)kLrSweeps * (rmax + 1) * (rmax + 2); }

__device__ LrScratch lr_slices(double* base, int nmax, int rmax) {
    LrScratch S;
    S.L = base;
    S.dg = S.L + (size_t)rmax * nmax;
    S.y = S.dg + nmax;
    S.C = S.y + nmax;
    S.log = S.C + (size_t)rmax * (rmax + 1);
    S.z = S.log + lr_log_doubles(rmax);
    S.u = S.z + rmax;
    S.li = reinterpret_cast<int64_t*>(S.u + rmax);
    S.li0 = S.li + nmax;
    S.lt = reinterpret_cast<int*>(S.li0 + nmax);
    S.lt0 = S.lt + nmax;
    return S;
}

__host__ __device__ inline size_t lr_scratch_doubles(int nmax, int rmax) {
    return (size_t)rmax * nmax + 2 * (size_t)nmax + (size_t)rmax * (rmax + 1) + lr_log_doubles(rmax) +
           2 * (size_t)rmax + 2 * (size_t)nmax /* li, li0 */ + (size_t)nmax /* lt, lt0 */ + 8;
}

__global__ void __launch_bounds__(256) k_alg2_solve_lr(ColCtx cc, GramCtx gc, const int64_t* __restrict__ cols,
                                                       int64_t ncols, const int32_t* __restrict__ cnt, int nmax,
                                                       int rmax, int ksm, double* __restrict__ scratch, double tau2,
                                                       double rel, int P, double* __restrict__ w64,
                                                       unsigned long long* __restrict__ ndrop,
                                                       int* __restrict__ rank_max) {
    __shared__ double rv[32];
    __shared__ int ri[32];
    __shared__ int cntr;
    // dynamic: packed C for k <= ksm, then the rotation lists cs[rmax + 2], pq[rmax + 2]
    extern __shared__ double smx[];
    double* Csm = smx;
    double* cs = Csm + packed_doubles(ksm);
    int* pq = reinterpret_cast<int*>(cs + rmax + 2);
    LrScratch S = lr_slices(scratch + (size_t)blockIdx.x * lr_scratch_doubles(nmax, rmax), nmax, rmax);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    for (int64_t ci = blockIdx.x; ci < ncols; ci += gridDim.x) {
        const int64_t n = cols[ci];
        const int nc = min(cnt[n], nmax);
        long long tph = clock64();
        auto phase = [&](int w) {
            if (tid == 0) {
                const long long now = clock64();
                atomicAdd(&g_lr_cycles[w], (unsigned long long)(now - tph));
                tph = now;
            }
        };
        if (tid == 0) cntr = 0;
        __syncthreads();
        for_column(cc, n, tid, nt, [&](int64_t i, int64_t t) {
            const int k = atomicAdd(&cntr, 1);
            if (k < nmax) {
                S.li0[k] = i;
                S.lt0[k] = (int)t;
            }
        });
        __syncthreads();
        // canonical order: position = number of smaller (i, t) keys (keys are distinct)
        for (int a = tid; a < nc; a += nt) {
            const int64_t ia = S.li0[a];
            const int ta = S.lt0[a];
            int r = 0;
            for (int c = 0; c < nc; c++) {
                const int64_t ic = S.li0[c];
                r += (ic < ia) || (ic == ia && S.lt0[c] < ta);
            }
            S.li[r] = ia;
            S.lt[r] = ta;
        }
        __syncthreads();
        phase(0);
        for (int a = tid; a < nc; a += nt) {
            S.dg[a] = gram_entry(gc, S.li[a], S.li[a]);
            S.y[a] = rhs_entry(gc, S.li[a], n);
        }
        __syncthreads();
        double c0;
        int ignore;
        block_argmax(S.dg, nc, c0, ignore, rv, ri);
        phase(1);
        // 1. pivoted Cholesky
        int k = 0;
        while (k < rmax) {
            double v;
            int piv;
            block_argmax(S.dg, nc, v, piv, rv, ri);
            if (!(v > rel * c0)) break;
            const double sq = sqrt(v);
            const int64_t lp = S.li[piv];
            double* Lk = S.L + (size_t)k * nmax;
            for (int i = tid; i < nc; i += nt) {
                double acc = 0.0;
                for (int j = 0; j < k; j++) acc = fma(S.L[(size_t)j * nmax + i], S.L[(size_t)j * nmax + piv], acc);
                Lk[i] = (gram_entry(gc, S.li[i], lp) - acc) / sq;
            }
            __syncthreads();
            for (int i = tid; i < nc; i += nt) S.dg[i] = (i == piv) ? 0.0 : S.dg[i] - Lk[i] * Lk[i];
            __syncthreads();
            k++;
        }
        phase(2);
        // 2. C = L^T L (k x k, packed upper triangle; shared memory when it fits) and z = L^T y:
        //    one warp per entry, lanes over the unknowns
        double* C = k <= ksm ? Csm : S.C;
        const int npk = (k + 1) & ~1;
        for (size_t e = tid; e < packed_doubles(k); e += nt) C[e] = 0.0;
        __syncthreads();
        for (int e = warp; e < k * (k + 1) / 2 + k; e += nw) {
            int a, c;
            const double* vb;
            if (e < k * (k + 1) / 2) {
                a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
                while ((a + 1) * (a + 2) / 2 <= e) a++;
                while (a * (a + 1) / 2 > e) a--;
                c = e - a * (a + 1) / 2;  // c <= a
                vb = S.L + (size_t)c * nmax;
            } else {
                a = e - k * (k + 1) / 2;
                c = -1;
                vb = S.y;
            }
            const double* va = S.L + (size_t)a * nmax;
            double acc = 0.0;
            for (int i = lane; i < nc; i += 32) acc = fma(va[i], vb[i], acc);
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
            if (lane == 0) {
                if (c >= 0)
                    C[pidx(c, a, npk)] = acc;
                else
                    S.z[a] = acc;
            }
        }
        __syncthreads();
        int dropped = nc - k;
        phase(3);
        if (k > 0) {
            // 3. eigenvalues of C; z <- W^T z on the fly, rotations logged for W u
            const int rounds = jacobi_packed_log(C, k, S.z, S.log, kLrSweeps * (k + 1), cs, pq, &cntr);
            if (tid == 0) {
                double mx = 0.0;
                int dr = 0;
                for (int a = 0; a < k; a++) mx = fmax(mx, C[pidx(a, a, npk)]);
                for (int a = 0; a < k; a++) dr += !(C[pidx(a, a, npk)] > tau2 * mx && mx > 0.0);
                rv[0] = mx;
                cntr = dr;
            }
            __syncthreads();
            const double cut = tau2 * rv[0];
            for (int a = tid; a < k; a += nt) {
                const double lam = C[pidx(a, a, npk)];
                S.u[a] = (lam > cut && rv[0] > 0.0) ? S.z[a] / (lam * lam) : 0.0;
            }
            dropped += cntr;
            __syncthreads();
            jacobi_apply_v(S.u, k, S.log, rounds);  // u <- W u
        }
        phase(4);
        for (int i = tid; i < nc; i += nt) {
            double b = 0.0;
            for (int a = 0; a < k; a++) b = fma(S.L[(size_t)a * nmax + i], S.u[a], b);
            w64[S.li[i] * P + S.lt[i]] = b;
        }
        if (tid == 0) {
            if (dropped > 0) atomicAdd(ndrop, 1ull);
            atomicMax(rank_max, k);
        }
        __syncthreads();
        phase(5);
    }
}

// ------------------------------------------------------------------ Alg. 1 (node-wise)
// Row h of K = A D^* F^*: K[h][l] = sum_k e^{2 pi i k x_h} iw_k e^{-2 pi i k l/Ms}
// = forward DFT over q = k mod Ms of a_q = iw_k e^{2 pi i k x_h}; build a_q here.
__global__ void k_alg1_rows(const double* __restrict__ xs, const double* __restrict__ iw, int64_t N, int64_t M,
                            int64_t Ms, double2* __restrict__ out) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= N * Ms) return;
    int64_t h = idx / Ms, q = idx - (idx / Ms) * Ms;
    int64_t k = q < Ms / 2 ? q : q - Ms;
    double2 v = make_double2(0.0, 0.0);
    if (k >= -M / 2 && k < M / 2) {
        // phase k x_h reduced exactly: hi + lo = k * x_h (two-product), frac(hi) + lo
        double x = xs[h];
        double hi = (double)k * x;
        double lo = fma((double)k, x, -hi);
        double ph = (hi - rint(hi)) + lo;
        double sn, c;
        sincospi(2.0 * ph, &sn, &c);
        double a = iw[k < 0 ? -k : k];
        v = make_double2(a * c, a * sn);
    }
    out[idx] = v;
}

// Per node j (one CTA): Gram Re(K_j^* K_j) over all rows h, rhs M Re(K[j][l]), solve.
__global__ void k_alg1_solve(const double2* __restrict__ K, const int32_t* __restrict__ n0s,
                             const int32_t* __restrict__ l0s, const double* __restrict__ xs, int64_t N, int64_t Ms,
                             int m, int P, double Mscale, double tau2, double* __restrict__ w64,
                             unsigned long long* __restrict__ ndrop) {
    extern __shared__ double sm[];
    const int nmax = P;
    const int ld = nmax + 1;
    double* A = sm;
    double* V = A + nmax * ld;
    double* y = V + nmax * ld;
    double* u = y + nmax;
    double* b = u + nmax;
    int* lt = reinterpret_cast<int*>(b + nmax);
    double* cs = reinterpret_cast<double*>(lt + nmax + (nmax & 1));
    int* pq = reinterpret_cast<int*>(cs + nmax + 2);
    int* cntr = pq + nmax + 2;
    for (int64_t j = blockIdx.x; j < N; j += gridDim.x) {
        if (threadIdx.x == 0) {
            int k = 0;
            for (int t = 0; t < P; t++) {
                // live slots of node j (alias-free: first congruent in-support slot)
                bool live = in_support(xs[j], l0s[j], t, Ms, m);
                for (int t2 = t - (int)Ms; live && t2 >= 0; t2 -= (int)Ms)
                    if (in_support(xs[j], l0s[j], t2, Ms, m)) live = false;
                if (live) lt[k++] = t;
            }
            *cntr = k;
        }
        __syncthreads();
        const int nc = *cntr;
        for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) {
            int a = idx / nc, c = idx % nc;
            if (c < a) continue;
            int64_t la = md(n0s[j] + lt[a], Ms), lc = md(n0s[j] + lt[c], Ms);
            double s = 0.0;
            for (int64_t h = 0; h < N; h++) {
                double2 ka = K[h * Ms + la], kc = K[h * Ms + lc];
                s += ka.x * kc.x + ka.y * kc.y;  // Re(conj(ka) kc)
            }
            A[a * ld + c] = s;
            A[c * ld + a] = s;
        }
        for (int a = threadIdx.x; a < nc; a += blockDim.x) {
            int64_t la = md(n0s[j] + lt[a], Ms);
            y[a] = Mscale * K[j * Ms + la].x;  // M Re(conj(K[j][l])) = M Re K[j][l]
        }
        __syncthreads();
        jacobi_eig(A, V, nc, ld, cs, pq, cntr);
        __syncthreads();
        int dropped = minnorm_from_eig(A, V, nc, ld, y, u, b, tau2);
        // B_opt^* column j holds b; B_opt = conj -> real: same values (reading A4)
        for (int a = threadIdx.x; a < nc; a += blockDim.x) w64[j * P + lt[a]] = b[a];
        if (threadIdx.x == 0 && dropped > 0) atomicAdd(ndrop, 1ull);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ Alg. 1, Gram by grid pairs
// The normal equations of node j need Re(K_j^* K_j) and M Re K_j^* e_j with
// K_j = (K(x_h - l/Ms))_{h, l in I(x_j)} and K(t) = sum_k c_k e^{2 pi i k t}, c_k = iw_|k|
// (= 1/(Ms what(k)); k = -M/2 uses iw_{M/2}).  The Gram entry of two slots depends only on
// their grid columns l, l + delta (delta = 0..2m), not on the node:
//   Gam(l, delta) = Re sum_h conj K(x_h - l/Ms) K(x_h - (l + delta)/Ms)
//                 = Re sum_{|q| < M} Sp(q) C_delta(q) e^{-2 pi i q l / Ms},
//   Sp(q) = sum_h e^{2 pi i q x_h},   C_delta(q) = sum_k c_{k-q} c_k e^{-2 pi i k delta / Ms}
// (expand both sums, q = k' - k).  So every node's Gram matrix comes from one node sum Sp
// (O(N M)), 2m+1 correlations C_delta (FFTs of length 2M) and 2m+1 FFTs of length Ms, instead
// of forming every K_j (O(N^2)).  The right-hand side
// M Re K(x_j - l/Ms) comes from the piecewise-Chebyshev table of Re K+ that Alg. 2 uses.
constexpr int kSpQ = 32;  // consecutive frequencies per thread (phase recurrence length)
__global__ void __launch_bounds__(128) k_alg1_sp(const double* __restrict__ xs, int64_t N, int64_t M,
                                                 double2* __restrict__ sp) {
    __shared__ double xt[1024];
    const int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kSpQ;
    double ax[kSpQ], ay[kSpQ];
#pragma unroll
    for (int u = 0; u < kSpQ; ++u) ax[u] = ay[u] = 0.0;
    for (int64_t h0 = 0; h0 < N; h0 += 1024) {
        const int nh = (int)(N - h0 < 1024 ? N - h0 : 1024);
        __syncthreads();
        for (int i = threadIdx.x; i < nh; i += blockDim.x) xt[i] = xs[h0 + i];
        __syncthreads();
        if (q0 >= M) continue;
        for (int i = 0; i < nh; ++i) {
            const double x = xt[i];
            // e^{2 pi i q0 x}: the phase q0 x reduced exactly (two-product), then the
            // recurrence z <- z e^{2 pi i x} over the next kSpQ - 1 frequencies
            const double hi = (double)q0 * x;
            const double lo = fma((double)q0, x, -hi);
            double zs, zc, s1, c1;
            sincospi(2.0 * ((hi - rint(hi)) + lo), &zs, &zc);
            sincospi(2.0 * x, &s1, &c1);
#pragma unroll
            for (int u = 0; u < kSpQ; ++u) {
                ax[u] += zc;
                ay[u] += zs;
                const double nc = fma(zc, c1, -zs * s1);
                zs = fma(zc, s1, zs * c1);
                zc = nc;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kSpQ; ++u)
        if (q0 + u < M) sp[q0 + u] = make_double2(ax[u], ay[u]);
}

// rows delta < P: U_delta[n] = c_k e^{-2 pi i k delta / Ms}; row P: V[n] = c_k (k = n - M/2,
// n < M; zero padded to L = 2M)
__global__ void k_alg1_corr_in(const double* __restrict__ iw, int64_t M, int64_t Ms, int P, int64_t L,
                               double2* __restrict__ buf) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)(P + 1) * L) return;
    const int r = (int)(idx / L);
    const int64_t n = idx - (int64_t)r * L;
    double2 v = make_double2(0.0, 0.0);
    if (n < M) {
        const int64_t k = n - M / 2;
        const double c = iw[k < 0 ? -k : k];
        if (r == P) {
            v.x = c;
        } else {
            // e^{-2 pi i k delta / Ms}, k delta reduced mod Ms in integers (exact)
            const int64_t e = ((k * r) % Ms + Ms) % Ms;
            double sn, cs;
            sincospi(-2.0 * (double)e / (double)Ms, &sn, &cs);
            v = make_double2(c * cs, c * sn);
        }
    }
    buf[idx] = v;
}

// U_delta^ <- U_delta^ conj(V^) / L  (then the inverse FFT gives C_delta(q) at q mod L)
__global__ void k_alg1_corr_mul(int P, int64_t L, double2* __restrict__ buf) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)P * L) return;
    const int64_t nu = idx % L;
    const double2 u = buf[idx], v = buf[(int64_t)P * L + nu];
    const double s = 1.0 / (double)L;
    buf[idx] = make_double2((u.x * v.x + u.y * v.y) * s, (u.y * v.x - u.x * v.y) * s);
}

// Z_delta[l] = sum_{q = l mod Ms, |q| < M} Sp(q) C_delta(q)   (Sp(-q) = conj Sp(q))
__global__ void k_alg1_fold(const double2* __restrict__ sp, const double2* __restrict__ corr, int64_t M, int64_t Ms,
                            int64_t L, int P, double2* __restrict__ z) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)P * Ms) return;
    const int r = (int)(idx / Ms);
    const int64_t l = idx - (int64_t)r * Ms;
    double ax = 0.0, ay = 0.0;
    // q = l + t Ms over -M < q < M
    int64_t q = l - ((l + M - 1) / Ms) * Ms;
    for (; q < M; q += Ms) {
        if (q <= -M) continue;
        double2 s = sp[q < 0 ? -q : q];
        if (q < 0) s.y = -s.y;
        const double2 c = corr[(int64_t)r * L + (q < 0 ? q + L : q)];
        ax += s.x * c.x - s.y * c.y;
        ay += s.x * c.y + s.y * c.x;
    }
    z[idx] = make_double2(ax, ay);
}

// Per node j (one CTA): Gram from Gam (real parts of the transformed Z rows), rhs from the
// Re K+ table, then the same min-norm eigen-solve as k_alg1_solve.
__global__ void k_alg1_solve_gam(const double2* __restrict__ gam, KTab tab, const int32_t* __restrict__ n0s,
                                 const int32_t* __restrict__ l0s, const double* __restrict__ xs, int64_t N,
                                 int64_t Ms, int m, int P, double Mscale, double tau2, double* __restrict__ w64,
                                 unsigned long long* __restrict__ ndrop) {
    extern __shared__ double sm[];
    const int nmax = P;
    const int ld = nmax + 1;
    double* A = sm;
    double* V = A + nmax * ld;
    double* y = V + nmax * ld;
    double* u = y + nmax;
    double* b = u + nmax;
    int* lt = reinterpret_cast<int*>(b + nmax);
    double* cs = reinterpret_cast<double*>(lt + nmax + (nmax & 1));
    int* pq = reinterpret_cast<int*>(cs + nmax + 2);
    int* cntr = pq + nmax + 2;
    for (int64_t j = blockIdx.x; j < N; j += gridDim.x) {
        if (threadIdx.x == 0) {
            int k = 0;
            for (int t = 0; t < P; t++) {
                bool live = in_support(xs[j], l0s[j], t, Ms, m);
                for (int t2 = t - (int)Ms; live && t2 >= 0; t2 -= (int)Ms)
                    if (in_support(xs[j], l0s[j], t2, Ms, m)) live = false;
                if (live) lt[k++] = t;
            }
            *cntr = k;
        }
        __syncthreads();
        const int nc = *cntr;
        for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) {
            const int a = idx / nc, c = idx % nc;
            if (c < a) continue;
            const int64_t la = md(n0s[j] + lt[a], Ms);
            const double s = gam[(int64_t)(lt[c] - lt[a]) * Ms + la].x;
            A[a * ld + c] = s;
            A[c * ld + a] = s;
        }
        for (int a = threadIdx.x; a < nc; a += blockDim.x) {
            const int64_t la = md(n0s[j] + lt[a], Ms);
            y[a] = Mscale * tab_eval(tab, tab.cK, wrapd(xs[j] - (double)la / (double)Ms));
        }
        __syncthreads();
        jacobi_eig(A, V, nc, ld, cs, pq, cntr);
        __syncthreads();
        int dropped = minnorm_from_eig(A, V, nc, ld, y, u, b, tau2);
        for (int a = threadIdx.x; a < nc; a += blockDim.x) w64[j * P + lt[a]] = b[a];
        if (threadIdx.x == 0 && dropped > 0) atomicAdd(ndrop, 1ull);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ plain window B
// w[i][t] = w~_m(x - l/Ms) = sum_z w_m(x - l/Ms + z) on live slots (eq. matrix_B, A7).
// centred cardinal B-spline of order n (support [-n/2, n/2]) at v: N_n(v + n/2) by the
// recursion N_k(u) = (u N_{k-1}(u) + (k - u) N_{k-1}(u - 1)) / (k - 1), N_1 = chi_[0, 1)
__device__ double bspline_centred(double v, int n) {
    const double u = v + 0.5 * n;
    if (!(u >= 0.0 && u < (double)n)) return 0.0;
    double c[33];  // c[j] = N_k(u - j), j = 0..n
    for (int j = 0; j <= n; ++j) c[j] = (u - j >= 0.0 && u - j < 1.0) ? 1.0 : 0.0;
    for (int k = 2; k <= n; ++k)
        for (int j = 0; j < n; ++j) c[j] = ((u - j) * c[j] + (k - (u - j)) * c[j + 1]) / (k - 1);
    return c[0];
}

__global__ void k_window_weights(const double* __restrict__ xs, const int32_t* __restrict__ l0s, int64_t N, int d,
                                 int64_t Ms1, int64_t Ms2, int m, double sigma, int P1, int window,
                                 double* __restrict__ w64) {
    const int P = d == 2 ? P1 * P1 : P1;
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= N * P) return;
    int64_t i = idx / P;
    int t = (int)(idx - i * P);
    const double b = kPi * (2.0 - 1.0 / sigma);
    double val = 1.0;
    for (int k = 0; k < d; k++) {
        int tk = d == 2 ? (k == 0 ? t / P1 : t % P1) : t;
        int64_t Ms = k == 0 ? Ms1 : Ms2;
        double x = xs[i * d + k];
        int64_t l0 = l0s[i * d + k];
        bool live = in_support(x, l0, tk, Ms, m);
        for (int t2 = tk - (int)Ms; live && t2 >= 0; t2 -= (int)Ms)
            if (in_support(x, l0, t2, Ms, m)) live = false;
        if (!live) {
            val = 0.0;
            break;
        }
        double v = __dmul_rn((double)Ms, x) - (double)(l0 + tk);  // Ms (x - l/Ms)
        double acc = 0.0;
        for (int z = -1; z <= 1; z++) {
            double vz = v + (double)z * (double)Ms;
            if (fabs(vz) <= (double)m) {
                if (window == INFT_BSPLINE) {
                    acc += bspline_centred(vz, 2 * m);  // w(x) = M_2m(M_sigma x)
                } else {
                    double r2 = (double)m * m - vz * vz;
                    acc += (r2 > 0.0 ? sinh(b * sqrt(r2)) / sqrt(r2) : b) / kPi;
                }
            }
        }
        val *= acc;
    }
    w64[idx] = val;
}

// ------------------------------------------------------------------ host driver
struct Tables {
    DevBuf iw, cG, cK, samp;
    KTab tab;
};

static void build_tables(Plan& p, int dim, Tables& T, double X, cudaStream_t st) {
    const int64_t M = p.M[dim], Ms = p.Ms[dim];
    T.iw.alloc(sizeof(double) * (M / 2 + 1));
    k_inv_what<<<nblk(M / 2 + 1), 256, 0, st>>>(T.iw.as<double>(), M, Ms, p.m, p.sigma,
                                                 (int)p.window);
    INFT_CHECK_LAUNCH();
    p.launches++;
    // piece width 2h with (pi M) h <= 1: |phase change| <= 1 rad per half piece
    double pw = 2.0 / (kPi * (double)M);
    int npc = (int)std::max<double>(1.0, std::ceil(2.0 * X / pw));
    pw = 2.0 * X / npc;
    T.samp.alloc(sizeof(double) * 2 * npc * (kChebDeg + 1));
    T.cG.alloc(sizeof(double) * npc * (kChebDeg + 1));
    T.cK.alloc(sizeof(double) * npc * (kChebDeg + 1));
    double* sG = T.samp.as<double>();
    double* sK = sG + npc * (kChebDeg + 1);
    k_cheb_samples<<<npc * (kChebDeg + 1), 256, 0, st>>>(T.iw.as<double>(), M, Ms, X, pw, npc, sG, sK);
    INFT_CHECK_LAUNCH();
    k_cheb_coef<<<nblk(npc * (kChebDeg + 1)), 256, 0, st>>>(sG, npc, T.cG.as<double>());
    INFT_CHECK_LAUNCH();
    k_cheb_coef<<<nblk(npc * (kChebDeg + 1)), 256, 0, st>>>(sK, npc, T.cK.as<double>());
    INFT_CHECK_LAUNCH();
    p.launches += 3;
    // Im parts from the unpaired k = -M/2 term: iw_{M/2} on host
    double iwh = 0.0;
    INFT_CUDA(cudaMemcpyAsync(&iwh, T.iw.as<double>() + M / 2, sizeof(double), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    T.tab.X = X;
    T.tab.pw = pw;
    T.tab.npc = npc;
    T.tab.cG = T.cG.as<double>();
    T.tab.cK = T.cK.as<double>();
    T.tab.Msd = (double)Ms;
    T.tab.Md = (double)M;
    T.tab.imG = (double)Ms * iwh * iwh;
    T.tab.imK = iwh;
}

static size_t alg2_smem_bytes(int nmax) {
    size_t ld = nmax + 1;
    size_t dbl = 2 * (size_t)nmax * ld + 3 * nmax;
    size_t lists = sizeof(int64_t) * nmax + sizeof(int) * (nmax + 1) + sizeof(double) * (nmax + 2) +
                   sizeof(int) * (nmax + 2) + sizeof(int) * 4;
    return sizeof(double) * dbl + lists + 64;
}

static void alg2(Plan& p, double tau, DevBuf& w64, cudaStream_t st) {
    const int d = p.d;
    const int64_t N = p.N;
    DevBuf xs, l0s;
    xs.alloc(sizeof(double) * std::max<int64_t>(1, N * d));
    l0s.alloc(sizeof(int32_t) * std::max<int64_t>(1, N * d));
    if (N > 0) {
        k_sorted_nodes<<<nblk(N), 256, 0, st>>>(p.nodes.as<double>(), p.l0.as<int32_t>(), p.perm.as<int32_t>(), N, d,
                                                xs.as<double>(), l0s.as<int32_t>());
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    ColCtx cc;
    cc.seg_start = p.seg_start.as<int32_t>();
    cc.n0s = p.n0s.as<int32_t>();
    cc.xs = xs.as<double>();
    cc.l0s = l0s.as<int32_t>();
    cc.d = d;
    cc.m = p.m;
    cc.P1 = p.P1;
    cc.S1 = p.S[0];
    cc.S2 = p.S[1];
    cc.Ms1 = p.Ms[0];
    cc.Ms2 = d == 2 ? p.Ms[1] : 1;
    cc.nseg2 = p.nseg[1];
    const int64_t ncol = p.Mstot;
    DevBuf cnt;
    cnt.alloc(sizeof(int32_t) * ncol);
    k_col_count<<<nblk(ncol), 256, 0, st>>>(cc, ncol, cnt.as<int32_t>());
    INFT_CHECK_LAUNCH();
    p.launches++;
    std::vector<int32_t> hc(ncol);
    INFT_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, sizeof(int32_t) * ncol, cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    // kernel tables: differences up to (2m+1)/Ms per dim (whole period if the support wraps)
    Tables T1, T2;
    for (int k = 0; k < d; k++) {
        double X = std::min(1.0, (2.0 * p.m + 1.0) / (double)p.Ms[k]);
        build_tables(p, k, k == 0 ? T1 : T2, X, st);
    }
    GramCtx gc;
    gc.t1 = T1.tab;
    gc.t2 = d == 2 ? T2.tab : T1.tab;
    gc.d = d;
    gc.xs = xs.as<double>();
    // size classes
    std::vector<int64_t> cls[3];
    int64_t empty = 0, mx = 0;
    for (int64_t n = 0; n < ncol; n++) {
        int c = hc[n];
        mx = std::max<int64_t>(mx, c);
        if (c == 0) {
            empty++;
            continue;
        }
        cls[c <= 32 ? 0 : (c <= 64 ? 1 : 2)].push_back(n);
    }
    p.n_empty_cols = empty;
    p.max_col_size = mx;
    DevBuf ndrop;
    ndrop.alloc(sizeof(unsigned long long));
    INFT_CUDA(cudaMemsetAsync(ndrop.p, 0, sizeof(unsigned long long), st));
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int limits[3] = {32, 64, (int)mx};
    const int threads[3] = {32, 128, 256};
    DevBuf rank_max;
    rank_max.alloc(sizeof(int));
    INFT_CUDA(cudaMemsetAsync(rank_max.p, 0, sizeof(int), st));
    for (int k = 0; k < 3; k++) {
        if (cls[k].empty()) continue;
        if (k == 2) {  // large columns: pivoted Cholesky + small eigenproblem (k_alg2_solve_lr)
            const int nmax = (int)mx;
            const int rmax = std::min(nmax, 384);
            const int ksm = std::min(rmax, 231);  // packed C in shared memory up to k = 231 (216 KB)
            DevBuf cols;
            cols.alloc(sizeof(int64_t) * cls[k].size());
            INFT_CUDA(cudaMemcpyAsync(cols.p, cls[k].data(), sizeof(int64_t) * cls[k].size(), cudaMemcpyHostToDevice,
                                      st));
            const size_t per = sizeof(double) * lr_scratch_doubles(nmax, rmax);
            const size_t budget = (size_t)8 << 30;
            const unsigned grid = (unsigned)std::max<int64_t>(
                1, std::min<int64_t>((int64_t)cls[k].size(), std::min<int64_t>((int64_t)nsm, budget / per)));
            DevBuf scratch;
            scratch.alloc(per * grid);
            const size_t smem = sizeof(double) * (packed_doubles(ksm) + rmax + 2) + sizeof(int) * (rmax + 2) + 16;
            ensure_smem_attr((const void*)k_alg2_solve_lr, smem);
            k_alg2_solve_lr<<<grid, 256, smem, st>>>(cc, gc, cols.as<int64_t>(), (int64_t)cls[k].size(),
                                                     cnt.as<int32_t>(), nmax, rmax, ksm, scratch.as<double>(), tau * tau,
                                                     1e-15, p.P, w64.as<double>(), ndrop.as<unsigned long long>(),
                                                     rank_max.as<int>());
            INFT_CHECK_LAUNCH();
            p.launches++;
            INFT_CUDA(cudaStreamSynchronize(st));
            continue;
        }
        int nmax = limits[k];
        DevBuf cols;
        cols.alloc(sizeof(int64_t) * cls[k].size());
        INFT_CUDA(cudaMemcpyAsync(cols.p, cls[k].data(), sizeof(int64_t) * cls[k].size(), cudaMemcpyHostToDevice, st));
        size_t smem = alg2_smem_bytes(nmax);
        int use_global = 0;
        DevBuf scratch;
        unsigned grid = (unsigned)std::min<int64_t>((int64_t)cls[k].size(), (int64_t)nsm * 64);
        if (smem > 200 * 1024) {
            use_global = 1;
            size_t per = sizeof(double) * (2 * (size_t)nmax * (nmax + 1) + 3 * (size_t)nmax);
            size_t budget = (size_t)8 << 30;
            grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)cls[k].size(),
                                                                    std::min<int64_t>(nsm * 2, budget / per)));
            scratch.alloc(per * grid);
            smem = sizeof(int64_t) * nmax + sizeof(int) * (nmax + 1) + sizeof(double) * (nmax + 2) +
                   sizeof(int) * (nmax + 2) + sizeof(int) * 4 + 64;
        }
        ensure_smem_attr((const void*)k_alg2_solve, smem);
        k_alg2_solve<<<grid, threads[k], smem, st>>>(cc, gc, cols.as<int64_t>(), (int64_t)cls[k].size(),
                                                     cnt.as<int32_t>(), nmax, use_global,
                                                     use_global ? scratch.as<double>() : nullptr, tau * tau, p.P,
                                                     w64.as<double>(), ndrop.as<unsigned long long>());
        INFT_CHECK_LAUNCH();
        p.launches++;
        INFT_CUDA(cudaStreamSynchronize(st));
    }
    unsigned long long nd = 0;
    int rk = 0;
    INFT_CUDA(cudaMemcpyAsync(&nd, ndrop.p, sizeof(nd), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaMemcpyAsync(&rk, rank_max.p, sizeof(rk), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    p.n_rank_deficient = (int64_t)nd;
    p.max_lowrank_rank = rk;
    if (getenv("INFT_SETUP_DEBUG")) {
        unsigned long long js[3];
        INFT_CUDA(cudaMemcpyFromSymbol(js, g_jac_stats, sizeof(js)));
        unsigned long long lc[6];
        INFT_CUDA(cudaMemcpyFromSymbol(lc, g_lr_cycles, sizeof(lc)));
        fprintf(stderr, "alg2: classes %zu/%zu/%zu cols, jacobi calls %llu mean sweeps %.2f max %llu\n",
                cls[0].size(), cls[1].size(), cls[2].size(), js[1], js[1] ? (double)js[0] / js[1] : 0.0, js[2]);
        fprintf(stderr, "alg2 large columns, Gcycles per phase: collect %.2f diag %.2f pchol %.2f gram %.2f "
                "jacobi %.2f back %.2f\n", lc[0] * 1e-9, lc[1] * 1e-9, lc[2] * 1e-9, lc[3] * 1e-9, lc[4] * 1e-9,
                lc[5] * 1e-9);
    }
}

// Alg. 1 normal equations: dense K (INFT_ALG1=dense; N * M_sigma <= 2^28) or Gram by grid
// pairs (INFT_ALG1=gram; default once N * M_sigma > 2^24, see k_alg1_sp)
static bool alg1_use_gram(const Plan& p) {
    const char* e = getenv("INFT_ALG1");
    if (e && !strcmp(e, "gram")) return true;
    if (e && !strcmp(e, "dense")) return false;
    return (double)p.N * (double)p.Ms[0] > (double)(1ll << 24);
}

static void cufft_z2z_many(int64_t n, int batch, double2* data, int dir, cudaStream_t st, const char* what) {
    cufftHandle h;
    int nn[1] = {(int)n};
    INFT_CUFFT(cufftPlanMany(&h, 1, nn, nullptr, 1, (int)n, nullptr, 1, (int)n, CUFFT_Z2Z, batch));
    cufftSetStream(h, st);
    const cufftResult r = cufftExecZ2Z(h, (cufftDoubleComplex*)data, (cufftDoubleComplex*)data, dir);
    cufftDestroy(h);
    if (r != CUFFT_SUCCESS) {
        set_error(std::string("cufftExecZ2Z failed: ") + what);
        throw Fail{INFT_ERR_CUFFT};
    }
}

static void alg1_gram(Plan& p, DevBuf& xs, DevBuf& l0s, DevBuf& iw, double tau, size_t solve_smem, DevBuf& w64,
                      DevBuf& ndrop, cudaStream_t st) {
    const int64_t N = p.N, M = p.M[0], Ms = p.Ms[0];
    const int P = p.P;
    // Sp(q) = sum_h e^{2 pi i q x_h}, q in [0, M)
    DevBuf sp, cb, zb;
    sp.alloc(sizeof(double2) * M);
    const int64_t nthr = ceil_div(M, (int64_t)kSpQ);
    k_alg1_sp<<<(unsigned)ceil_div(nthr, (int64_t)128), 128, 0, st>>>(xs.as<double>(), N, M, sp.as<double2>());
    INFT_CHECK_LAUNCH();
    // C_delta(q), |q| < M: correlations by FFTs of length L = 2M (no wrap)
    const int64_t L = 2 * M;
    cb.alloc(sizeof(double2) * (size_t)(P + 1) * L);
    k_alg1_corr_in<<<nblk((int64_t)(P + 1) * L), 256, 0, st>>>(iw.as<double>(), M, Ms, P, L, cb.as<double2>());
    INFT_CHECK_LAUNCH();
    cufft_z2z_many(L, P + 1, cb.as<double2>(), CUFFT_FORWARD, st, "Alg. 1 correlation (forward)");
    k_alg1_corr_mul<<<nblk((int64_t)P * L), 256, 0, st>>>(P, L, cb.as<double2>());
    INFT_CHECK_LAUNCH();
    cufft_z2z_many(L, P, cb.as<double2>(), CUFFT_INVERSE, st, "Alg. 1 correlation (inverse)");
    // Gam(l, delta) = Re FFT_l[ sum_{q = l mod Ms} Sp(q) C_delta(q) ]
    zb.alloc(sizeof(double2) * (size_t)P * Ms);
    k_alg1_fold<<<nblk((int64_t)P * Ms), 256, 0, st>>>(sp.as<double2>(), cb.as<double2>(), M, Ms, L, P,
                                                          zb.as<double2>());
    INFT_CHECK_LAUNCH();
    cufft_z2z_many(Ms, P, zb.as<double2>(), CUFFT_FORWARD, st, "Alg. 1 Gram table");
    // rhs table: Re K+ on |x| <= (2m+1)/Ms
    Tables T;
    build_tables(p, 0, T, std::min(1.0, (2.0 * p.m + 1.0) / (double)Ms), st);
    ensure_smem_attr((const void*)k_alg1_solve_gam, solve_smem);
    k_alg1_solve_gam<<<(unsigned)std::min<int64_t>(N, 148 * 16), 64, solve_smem, st>>>(
        zb.as<double2>(), T.tab, p.n0s.as<int32_t>(), l0s.as<int32_t>(), xs.as<double>(), N, Ms, p.m, P,
        (double)M, tau * tau, w64.as<double>(), ndrop.as<unsigned long long>());
    INFT_CHECK_LAUNCH();
    p.launches += 5;
    INFT_CUDA(cudaStreamSynchronize(st));  // the buffers above die here
}

// dense form: K = A D^* F^* row by row (one FFT of length Ms per node), Gram sums over all rows
static void alg1_dense(Plan& p, DevBuf& xs, DevBuf& l0s, DevBuf& iw, double tau, size_t solve_smem, DevBuf& w64,
                       DevBuf& ndrop, cudaStream_t st) {
    const int64_t N = p.N, M = p.M[0], Ms = p.Ms[0];
    const int P = p.P;
    DevBuf K;
    K.alloc(sizeof(double2) * N * Ms);
    k_alg1_rows<<<nblk(N * Ms), 256, 0, st>>>(xs.as<double>(), iw.as<double>(), N, M, Ms, K.as<double2>());
    INFT_CHECK_LAUNCH();
    p.launches += 3;
    cufftHandle h;
    int n[1] = {(int)Ms};
    INFT_CUFFT(cufftPlanMany(&h, 1, n, nullptr, 1, (int)Ms, nullptr, 1, (int)Ms, CUFFT_Z2Z, (int)N));
    cufftSetStream(h, st);
    cufftResult fr = cufftExecZ2Z(h, (cufftDoubleComplex*)K.p, (cufftDoubleComplex*)K.p, CUFFT_FORWARD);
    cufftDestroy(h);
    if (fr != CUFFT_SUCCESS) {
        set_error("cufftExecZ2Z (Alg. 1 kernel matrix) failed");
        throw Fail{INFT_ERR_CUFFT};
    }
    ensure_smem_attr((const void*)k_alg1_solve, solve_smem);
    k_alg1_solve<<<(unsigned)std::min<int64_t>(N, 148 * 16), 64, solve_smem, st>>>(
        K.as<double2>(), p.n0s.as<int32_t>(), l0s.as<int32_t>(), xs.as<double>(), N, Ms, p.m, P, (double)M,
        tau * tau, w64.as<double>(), ndrop.as<unsigned long long>());
    INFT_CHECK_LAUNCH();
    p.launches++;
    INFT_CUDA(cudaStreamSynchronize(st));  // K dies here
}

static void alg1(Plan& p, double tau, DevBuf& w64, cudaStream_t st) {
    if (p.d != 1) {
        set_error("Alg. 1 (node-wise) is implemented for d = 1");
        throw Fail{INFT_ERR_UNSUPPORTED};
    }
    const int64_t N = p.N, M = p.M[0], Ms = p.Ms[0];
    const bool gram = alg1_use_gram(p);
    if (!gram && (double)N * (double)Ms > (double)(1ll << 28)) {
        set_error("Alg. 1 dense form (INFT_ALG1=dense) needs N * M_sigma <= 2^28");
        throw Fail{INFT_ERR_UNSUPPORTED};
    }
    if (N == 0) return;
    DevBuf xs, l0s, iw;
    xs.alloc(sizeof(double) * N);
    l0s.alloc(sizeof(int32_t) * N);
    k_sorted_nodes<<<nblk(N), 256, 0, st>>>(p.nodes.as<double>(), p.l0.as<int32_t>(), p.perm.as<int32_t>(), N, 1,
                                            xs.as<double>(), l0s.as<int32_t>());
    iw.alloc(sizeof(double) * (M / 2 + 1));
    k_inv_what<<<nblk(M / 2 + 1), 256, 0, st>>>(iw.as<double>(), M, Ms, p.m, p.sigma,
                                                 (int)p.window);
    DevBuf ndrop;
    ndrop.alloc(sizeof(unsigned long long));
    INFT_CUDA(cudaMemsetAsync(ndrop.p, 0, sizeof(unsigned long long), st));
    const int P = p.P;
    const size_t solve_smem = sizeof(double) * (2 * (size_t)P * (P + 1) + 3 * P) + sizeof(int) * (P + 1) +
                              sizeof(double) * (P + 2) + sizeof(int) * (P + 2) + sizeof(int) * 4 + 64;
    if (gram) {
        alg1_gram(p, xs, l0s, iw, tau, solve_smem, w64, ndrop, st);
    } else {
        alg1_dense(p, xs, l0s, iw, tau, solve_smem, w64, ndrop, st);
    }
    unsigned long long nd = 0;
    INFT_CUDA(cudaMemcpyAsync(&nd, ndrop.p, sizeof(nd), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    p.n_rank_deficient = (int64_t)nd;
    p.max_lowrank_rank = 0;
    p.n_empty_cols = 0;
    p.max_col_size = p.P;
}

void precompute(Plan& p, inft_method method, inft_weights wt, double tau, cudaStream_t st) {
    if (method == INFT_AUTO) method = (p.Mtot >= p.N) ? INFT_ALG1_NODEWISE : INFT_ALG2_GRIDWISE;
    if (wt == INFT_WEIGHTS_COMPLEX && method != INFT_PLAIN_NFFT) {
        set_error("complex-weight optimisation is not implemented on the GPU (use inft_set_bopt)");
        throw Fail{INFT_ERR_UNSUPPORTED};
    }
    wt = INFT_WEIGHTS_REAL;
    DevBuf w64;
    w64.alloc(sizeof(double) * std::max<int64_t>(1, p.N * p.P));
    INFT_CUDA(cudaMemsetAsync(w64.p, 0, sizeof(double) * std::max<int64_t>(1, p.N * p.P), st));
    p.n_rank_deficient = p.n_empty_cols = p.max_col_size = 0;
    p.tau = tau;
    if (method == INFT_PLAIN_NFFT) {
        if (p.window == INFT_DIRICHLET) {
            set_error("INFT_PLAIN_NFFT needs a window function in space (Kaiser-Bessel or B-spline)");
            throw Fail{INFT_ERR_INVALID_ARG};
        }
        if (p.N > 0) {
            DevBuf xs, l0s;
            xs.alloc(sizeof(double) * p.N * p.d);
            l0s.alloc(sizeof(int32_t) * p.N * p.d);
            k_sorted_nodes<<<nblk(p.N), 256, 0, st>>>(p.nodes.as<double>(), p.l0.as<int32_t>(), p.perm.as<int32_t>(),
                                                      p.N, p.d, xs.as<double>(), l0s.as<int32_t>());
            k_window_weights<<<nblk(p.N * p.P), 256, 0, st>>>(xs.as<double>(), l0s.as<int32_t>(), p.N, p.d, p.Ms[0],
                                                              p.d == 2 ? p.Ms[1] : 1, p.m, p.sigma, p.P1,
                                                              (int)p.window, w64.as<double>());
            INFT_CHECK_LAUNCH();
            p.launches += 2;
            INFT_CUDA(cudaStreamSynchronize(st));
        }
        p.max_col_size = p.P;
    } else if (method == INFT_ALG2_GRIDWISE) {
        alg2(p, tau, w64, st);
    } else {
        alg1(p, tau, w64, st);
    }
    install_weights_from_device(p, w64.as<double>(), method, wt, st);
    INFT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace inft
