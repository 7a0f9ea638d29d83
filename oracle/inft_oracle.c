/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * implementation of the apply stage of Kircheis & Potts' direct inverse NFFT
 * (arXiv:1811.05335).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file's library.  It
 * shares no code, header or table with the CUDA path
 * (paper_1811_05335_b200/csrc).  Citations: P:<n> = PAPER.md line n.
 *
 * Every routine follows the paper's factorisation literally, in fp64:
 *   inverse NFFT            fhat = s * D^* F^* B_opt^* f
 *   inverse adjoint NFFT    f    = s * B_opt F D h
 * with D = diag(1/(M_sigma what(k))) (eq. matrix_D), the truncated
 * Fourier matrix F_{l,k} = e^{2 pi i k l / M_sigma} (eq. matrix_F)
 * and the (2m+1)-sparse B_opt stored per node as slot weights w[j][t] =
 * B_opt[j, l0_j + t] with l0_j = ceil(M_sigma x_j) - m (index set).
 * The caller passes d[k] = s / (M_sigma what(k)) (scale s folded in, A2).
 *
 * Grid vectors are held in "FFT order" n = l mod M_sigma; because every factor
 * of F is M_sigma-periodic in l this is the same sum as the paper's
 * l = -M_sigma/2 .. M_sigma/2-1 (A9).  Spectral vectors are stored
 * centered: entry k + M/2 holds index k.
 *
 * Complex numbers are interleaved (re, im) doubles.  The DFT is an iterative
 * radix-2 FFT for power-of-two lengths with every twiddle computed directly by
 * cos/sin of an exactly reduced angle, and a plain O(n^2) DFT otherwise.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double TWO_PI = 6.283185307179586476925286766559;

static int64_t mod_i64(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

static int is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

/* In-place DFT of length n with stride 1:  X_q = sum_n x_n e^{sign 2 pi i q n / len}.
 * sign = -1: forward (the F^* step); sign = +1: unnormalised inverse (the F step). */
static void dft_inplace(double* x, int64_t n, int sign, double* scratch) {
    if (n <= 1) return;
    if (is_pow2(n)) {
        /* bit reversal permutation */
        int64_t j = 0;
        for (int64_t i = 1; i < n; i++) {
            int64_t bit = n >> 1;
            for (; j & bit; bit >>= 1) j ^= bit;
            j ^= bit;
            if (i < j) {
                double tr = x[2 * i], ti = x[2 * i + 1];
                x[2 * i] = x[2 * j]; x[2 * i + 1] = x[2 * j + 1];
                x[2 * j] = tr; x[2 * j + 1] = ti;
            }
        }
        /* butterflies; twiddle e^{sign 2 pi i k / len} computed directly */
        for (int64_t len = 2; len <= n; len <<= 1) {
            int64_t half = len >> 1;
            for (int64_t k = 0; k < half; k++) {
                double ang = sign * TWO_PI * (double)k / (double)len;
                double wr = cos(ang), wi = sin(ang);
                for (int64_t s = 0; s < n; s += len) {
                    double* a = x + 2 * (s + k);
                    double* b = x + 2 * (s + k + half);
                    double br = b[0] * wr - b[1] * wi;
                    double bi = b[0] * wi + b[1] * wr;
                    b[0] = a[0] - br; b[1] = a[1] - bi;
                    a[0] = a[0] + br; a[1] = a[1] + bi;
                }
            }
        }
    } else {
        /* plain DFT with the phase index reduced exactly: (q * t) mod n */
        for (int64_t q = 0; q < n; q++) {
            double sr = 0.0, si = 0.0;
            for (int64_t t = 0; t < n; t++) {
                double ang = sign * TWO_PI * (double)mod_i64(q * t, n) / (double)n;
                double c = cos(ang), s = sin(ang);
                sr += x[2 * t] * c - x[2 * t + 1] * s;
                si += x[2 * t] * s + x[2 * t + 1] * c;
            }
            scratch[2 * q] = sr; scratch[2 * q + 1] = si;
        }
        memcpy(x, scratch, (size_t)(2 * n) * sizeof(double));
    }
}

/* 2-D DFT of an n1 x n2 row-major array: rows then columns. */
static void dft2_inplace(double* x, int64_t n1, int64_t n2, int sign, double* scratch, double* col) {
    for (int64_t a = 0; a < n1; a++) dft_inplace(x + 2 * a * n2, n2, sign, scratch);
    for (int64_t b = 0; b < n2; b++) {
        for (int64_t a = 0; a < n1; a++) { col[2 * a] = x[2 * (a * n2 + b)]; col[2 * a + 1] = x[2 * (a * n2 + b) + 1]; }
        dft_inplace(col, n1, sign, scratch);
        for (int64_t a = 0; a < n1; a++) { x[2 * (a * n2 + b)] = col[2 * a]; x[2 * (a * n2 + b) + 1] = col[2 * a + 1]; }
    }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------- 1-D ---- */

/* Inverse NFFT (modified adjoint NFFT), P:631 / P:1279:
 *   g_n   = sum_j sum_t [n == (l0_j + t) mod Msig] conj(w[j][t]) f_j     (B_opt^* f)
 *   ghat_q = sum_n g_n e^{-2 pi i q n / Msig}                           (F^*)
 *   fhat_k = d_k ghat_{k mod Msig},  k = -M/2..M/2-1                     (D^*, truncation) */
int oracle_inverse_1d(int64_t N, int64_t M, int64_t Msig, int P, const int64_t* l0,
                      const double* w_re, const double* w_im, const double* d,
                      const double* f, double* fhat, int64_t R, int nthreads) {
    if (N < 0 || M <= 0 || Msig < M || P <= 0 || R < 0) return 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* g = (double*)malloc((size_t)(2 * Msig) * sizeof(double));
        double* scratch = is_pow2(Msig) ? NULL : (double*)malloc((size_t)(2 * Msig) * sizeof(double));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t r = 0; r < R; r++) {
            const double* fr = f + 2 * r * N;
            memset(g, 0, (size_t)(2 * Msig) * sizeof(double));
            for (int64_t j = 0; j < N; j++) {
                for (int t = 0; t < P; t++) {
                    double wr = w_re[j * P + t];
                    double wi = w_im ? w_im[j * P + t] : 0.0;
                    int64_t n = mod_i64(l0[j] + t, Msig);
                    /* conj(w) * f */
                    g[2 * n] += wr * fr[2 * j] + wi * fr[2 * j + 1];
                    g[2 * n + 1] += wr * fr[2 * j + 1] - wi * fr[2 * j];
                }
            }
            dft_inplace(g, Msig, -1, scratch);
            double* out = fhat + 2 * r * M;
            for (int64_t k = -M / 2; k < M / 2; k++) {
                int64_t q = mod_i64(k, Msig);
                out[2 * (k + M / 2)] = d[k + M / 2] * g[2 * q];
                out[2 * (k + M / 2) + 1] = d[k + M / 2] * g[2 * q + 1];
            }
        }
        free(g);
        free(scratch);
    }
    return 0;
}

/* Inverse adjoint NFFT (modified NFFT), P:1116 / P:1522:
 *   ghat_{k mod Msig} = d_k h_k, zero elsewhere                          (D, zero pad)
 *   g_n = sum_q ghat_q e^{+2 pi i q n / Msig}                            (F)
 *   f_j = sum_t w[j][t] g_{(l0_j + t) mod Msig}                          (B_opt) */
int oracle_adjoint_1d(int64_t N, int64_t M, int64_t Msig, int P, const int64_t* l0,
                      const double* w_re, const double* w_im, const double* d,
                      const double* h, double* f, int64_t R, int nthreads) {
    if (N < 0 || M <= 0 || Msig < M || P <= 0 || R < 0) return 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* g = (double*)malloc((size_t)(2 * Msig) * sizeof(double));
        double* scratch = is_pow2(Msig) ? NULL : (double*)malloc((size_t)(2 * Msig) * sizeof(double));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t r = 0; r < R; r++) {
            const double* hr = h + 2 * r * M;
            memset(g, 0, (size_t)(2 * Msig) * sizeof(double));
            for (int64_t k = -M / 2; k < M / 2; k++) {
                int64_t q = mod_i64(k, Msig);
                g[2 * q] = d[k + M / 2] * hr[2 * (k + M / 2)];
                g[2 * q + 1] = d[k + M / 2] * hr[2 * (k + M / 2) + 1];
            }
            dft_inplace(g, Msig, +1, scratch);
            double* out = f + 2 * r * N;
            for (int64_t j = 0; j < N; j++) {
                double sr = 0.0, si = 0.0;
                for (int t = 0; t < P; t++) {
                    double wr = w_re[j * P + t];
                    double wi = w_im ? w_im[j * P + t] : 0.0;
                    int64_t n = mod_i64(l0[j] + t, Msig);
                    sr += wr * g[2 * n] - wi * g[2 * n + 1];
                    si += wr * g[2 * n + 1] + wi * g[2 * n];
                }
                out[2 * j] = sr;
                out[2 * j + 1] = si;
            }
        }
        free(g);
        free(scratch);
    }
    return 0;
}

/* ---------------------------------------------------------------- 2-D ---- */
/* Tensor-product reading (A12): slots (t1, t2) -> t = t1*P2 + t2,
 * grid n = n1*Msig2 + n2, spectrum (k1 + M1/2)*M2 + (k2 + M2/2),
 * d_k = d1[k1] d2[k2]. */
int oracle_inverse_2d(int64_t N, const int64_t* M, const int64_t* Msig, const int* P,
                      const int64_t* l0, const double* w_re, const double* w_im,
                      const double* d1, const double* d2, const double* f, double* fhat,
                      int64_t R, int nthreads) {
    int64_t M1 = M[0], M2 = M[1], S1 = Msig[0], S2 = Msig[1];
    int P1 = P[0], P2 = P[1], PP = P[0] * P[1];
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* g = (double*)malloc((size_t)(2 * S1 * S2) * sizeof(double));
        int64_t mx = S1 > S2 ? S1 : S2;
        double* scratch = (double*)malloc((size_t)(2 * mx) * sizeof(double));
        double* col = (double*)malloc((size_t)(2 * S1) * sizeof(double));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t r = 0; r < R; r++) {
            const double* fr = f + 2 * r * N;
            memset(g, 0, (size_t)(2 * S1 * S2) * sizeof(double));
            for (int64_t j = 0; j < N; j++) {
                for (int t1 = 0; t1 < P1; t1++) {
                    int64_t n1 = mod_i64(l0[2 * j] + t1, S1);
                    for (int t2 = 0; t2 < P2; t2++) {
                        int64_t n2 = mod_i64(l0[2 * j + 1] + t2, S2);
                        int64_t t = (int64_t)t1 * P2 + t2;
                        double wr = w_re[j * PP + t];
                        double wi = w_im ? w_im[j * PP + t] : 0.0;
                        int64_t n = n1 * S2 + n2;
                        g[2 * n] += wr * fr[2 * j] + wi * fr[2 * j + 1];
                        g[2 * n + 1] += wr * fr[2 * j + 1] - wi * fr[2 * j];
                    }
                }
            }
            dft2_inplace(g, S1, S2, -1, scratch, col);
            double* out = fhat + 2 * r * M1 * M2;
            for (int64_t k1 = -M1 / 2; k1 < M1 / 2; k1++) {
                int64_t q1 = mod_i64(k1, S1);
                for (int64_t k2 = -M2 / 2; k2 < M2 / 2; k2++) {
                    int64_t q2 = mod_i64(k2, S2);
                    double dk = d1[k1 + M1 / 2] * d2[k2 + M2 / 2];
                    int64_t o = (k1 + M1 / 2) * M2 + (k2 + M2 / 2);
                    out[2 * o] = dk * g[2 * (q1 * S2 + q2)];
                    out[2 * o + 1] = dk * g[2 * (q1 * S2 + q2) + 1];
                }
            }
        }
        free(g);
        free(scratch);
        free(col);
    }
    return 0;
}

int oracle_adjoint_2d(int64_t N, const int64_t* M, const int64_t* Msig, const int* P,
                      const int64_t* l0, const double* w_re, const double* w_im,
                      const double* d1, const double* d2, const double* h, double* f,
                      int64_t R, int nthreads) {
    int64_t M1 = M[0], M2 = M[1], S1 = Msig[0], S2 = Msig[1];
    int P1 = P[0], P2 = P[1], PP = P[0] * P[1];
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* g = (double*)malloc((size_t)(2 * S1 * S2) * sizeof(double));
        int64_t mx = S1 > S2 ? S1 : S2;
        double* scratch = (double*)malloc((size_t)(2 * mx) * sizeof(double));
        double* col = (double*)malloc((size_t)(2 * S1) * sizeof(double));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t r = 0; r < R; r++) {
            const double* hr = h + 2 * r * M1 * M2;
            memset(g, 0, (size_t)(2 * S1 * S2) * sizeof(double));
            for (int64_t k1 = -M1 / 2; k1 < M1 / 2; k1++) {
                int64_t q1 = mod_i64(k1, S1);
                for (int64_t k2 = -M2 / 2; k2 < M2 / 2; k2++) {
                    int64_t q2 = mod_i64(k2, S2);
                    double dk = d1[k1 + M1 / 2] * d2[k2 + M2 / 2];
                    int64_t o = (k1 + M1 / 2) * M2 + (k2 + M2 / 2);
                    g[2 * (q1 * S2 + q2)] = dk * hr[2 * o];
                    g[2 * (q1 * S2 + q2) + 1] = dk * hr[2 * o + 1];
                }
            }
            dft2_inplace(g, S1, S2, +1, scratch, col);
            double* out = f + 2 * r * N;
            for (int64_t j = 0; j < N; j++) {
                double sr = 0.0, si = 0.0;
                for (int t1 = 0; t1 < P1; t1++) {
                    int64_t n1 = mod_i64(l0[2 * j] + t1, S1);
                    for (int t2 = 0; t2 < P2; t2++) {
                        int64_t n2 = mod_i64(l0[2 * j + 1] + t2, S2);
                        int64_t t = (int64_t)t1 * P2 + t2;
                        double wr = w_re[j * PP + t];
                        double wi = w_im ? w_im[j * PP + t] : 0.0;
                        int64_t n = n1 * S2 + n2;
                        sr += wr * g[2 * n] - wi * g[2 * n + 1];
                        si += wr * g[2 * n + 1] + wi * g[2 * n];
                    }
                }
                out[2 * j] = sr;
                out[2 * j + 1] = si;
            }
        }
        free(g);
        free(scratch);
        free(col);
    }
    return 0;
}

/* Standalone DFT entry (tests pin this against the DFT definition). */
int oracle_dft(double* x, int64_t n, int sign) {
    double* scratch = (double*)malloc((size_t)(2 * (n > 0 ? n : 1)) * sizeof(double));
    dft_inplace(x, n, sign, scratch);
    free(scratch);
    return 0;
}

/* ------------------------------------------------------ trigonometric sums ---- */

/* e^{2 pi i k x} from the exactly reduced phase frac(k x): the product k x is split into
 * p + e by one fma (two-product), so |k| up to 2^21 keeps ~1e-16 phase accuracy. */
static void unit_phase(double k, double x, double* c, double* s) {
    double p = k * x;
    double e = fma(k, x, -p);
    double fr = p - floor(p);
    fr += e;
    fr -= floor(fr);
    *c = cos(TWO_PI * fr);
    *s = sin(TWO_PI * fr);
}

/* out[r][i] = sum_{k=-M/2}^{M/2-1} c[r][k + M/2] e^{2 pi i k x_i}, r < R, i < n (direct sum;
 * c and out interleaved complex).  Used for the kernels G(x), K+(x) of the Gram form of
 * Alg. "Fast optimization of the matrix B" (coefficients 1/(M_sigma what(k)^2), 1/(M_sigma
 * what(k)); reading A6) and for the NDFT f = A fhat (eq. nfft).
 * e^{2 pi i k x} is stepped by the angle-addition recurrence z_{k+1} = z_k e^{2 pi i x} and
 * restarted from unit_phase() every 32 terms (<= 32 roundings between restarts). */
/* One coefficient vector, eight x at a time (eight independent recurrences). */
static void trig_sum_x8(int64_t M, const double* c, const double* x, int nb, double* out) {
    enum { BLK = 32, XB = 8 };
    double sc[XB], ss[XB], zr[XB], zi[XB], ar[XB], ai[XB];
    for (int b = 0; b < XB; b++) {
        unit_phase(1.0, x[b < nb ? b : 0], &sc[b], &ss[b]);
        ar[b] = ai[b] = 0.0;
    }
    for (int64_t k0 = -M / 2; k0 < M / 2; k0 += BLK) {
        for (int b = 0; b < XB; b++) unit_phase((double)k0, x[b < nb ? b : 0], &zr[b], &zi[b]);
        const int64_t k1 = k0 + BLK < M / 2 ? k0 + BLK : M / 2;
        for (int64_t k = k0; k < k1; k++) {
            const double cr = c[2 * (k + M / 2)], ci = c[2 * (k + M / 2) + 1];
            for (int b = 0; b < XB; b++) {
                ar[b] += cr * zr[b] - ci * zi[b];
                ai[b] += cr * zi[b] + ci * zr[b];
                const double t = zr[b] * sc[b] - zi[b] * ss[b];
                zi[b] = zr[b] * ss[b] + zi[b] * sc[b];
                zr[b] = t;
            }
        }
    }
    for (int b = 0; b < nb; b++) {
        out[2 * b] = ar[b];
        out[2 * b + 1] = ai[b];
    }
}

int oracle_trig_sum(int64_t M, int64_t R, const double* c, int64_t n, const double* x, double* out,
                    int nthreads) {
    enum { BLK = 32 };
    if (R == 1) {
#ifdef _OPENMP
        if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
        for (int64_t i = 0; i < n; i += 8) trig_sum_x8(M, c, x + i, (int)(n - i < 8 ? n - i : 8), out + 2 * i);
        return 0;
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int64_t i = 0; i < n; i++) {
        double sc, ss;
        unit_phase(1.0, x[i], &sc, &ss);
        double* acc = (double*)calloc((size_t)(2 * (R > 0 ? R : 1)), sizeof(double));
        for (int64_t k0 = -M / 2; k0 < M / 2; k0 += BLK) {
            double zr, zi;
            unit_phase((double)k0, x[i], &zr, &zi);
            const int64_t k1 = k0 + BLK < M / 2 ? k0 + BLK : M / 2;
            for (int64_t k = k0; k < k1; k++) {
                const double* ck = c + 2 * (k + M / 2);
                for (int64_t r = 0; r < R; r++) {
                    const double cr = ck[2 * r * M], ci = ck[2 * r * M + 1];
                    acc[2 * r] += cr * zr - ci * zi;
                    acc[2 * r + 1] += cr * zi + ci * zr;
                }
                const double t = zr * sc - zi * ss;
                zi = zr * ss + zi * sc;
                zr = t;
            }
        }
        for (int64_t r = 0; r < R; r++) {
            out[2 * (r * n + i)] = acc[2 * r];
            out[2 * (r * n + i) + 1] = acc[2 * r + 1];
        }
        free(acc);
    }
    return 0;
}
