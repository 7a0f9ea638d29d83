// Fused four-step FFT for the 1-D apply (SURVEY 8(a) a3+a4 and a5+a6).
//
// N = M_sigma = N1 * N2 (powers of two).  With n = N2*n1 + n2 and k = k1 + N1*k2,
//   X[k1 + N1 k2] = sum_{n2} w_{N2}^{n2 k2} [ w_N^{n2 k1} sum_{n1} x[N2 n1 + n2] w_{N1}^{n1 k1} ]
// (w = e^{sign 2 pi i / .}).  Pass A does the N1-point column transforms of a tile of TA
// columns and applies the twiddle w_N^{n2 k1}; pass B does the N2-point row transforms of a
// tile of TB rows.  Inside a CTA the transform is a Stockham autosort FFT (radix 16/8/4/2):
// the first stage reads global memory straight into registers and the last stage writes
// global memory from registers; only the stages in between exchange through shared memory.
//
// Fusions (each removes a full pass over the grid):
//   inverse NFFT  (a3+a4): pass A in place on the spread grid, pass B writes only the kept
//                 frequencies k in [-M/2, M/2) multiplied by d_k straight into fhat;
//   inverse adjoint (a5+a6): pass A reads h directly (d_k h_k inside the band, zero
//                 elsewhere -- no padded grid is materialised), pass B writes the natural-
//                 order grid and its 2m halo for the gather.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "inft_internal.cuh"

namespace inft {
namespace fft {

// ------------------------------------------------------------------ complex helpers
template <typename T>
__device__ __forceinline__ C2<T> cadd(C2<T> a, C2<T> b) { return mk<T>(a.x + b.x, a.y + b.y); }
template <typename T>
__device__ __forceinline__ C2<T> csub(C2<T> a, C2<T> b) { return mk<T>(a.x - b.x, a.y - b.y); }
template <typename T>
__device__ __forceinline__ C2<T> cmul(C2<T> a, C2<T> b) {
    return mk<T>(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// cos(pi m / 8), m = 0..15 (exact to double rounding)
__device__ __forceinline__ constexpr double c16(int m) {
    constexpr double t[16] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                              -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173,
                              0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613};
    return t[m & 15];
}

// a * e^{SIGN 2 pi i E / 16} with E a compile-time exponent (multiples of 4 are exact swaps)
template <typename T, int SIGN, int E>
__device__ __forceinline__ C2<T> rot16(C2<T> a) {
    constexpr int e = ((E % 16) + 16) % 16;
    if constexpr (e == 0) return a;
    if constexpr (e == 8) return mk<T>(-a.x, -a.y);
    if constexpr (e == 4) return SIGN > 0 ? mk<T>(-a.y, a.x) : mk<T>(a.y, -a.x);   // * (SIGN i)
    if constexpr (e == 12) return SIGN > 0 ? mk<T>(a.y, -a.x) : mk<T>(-a.y, a.x);  // * (-SIGN i)
    // cos(2 pi e/16) = cos(pi e/8) = c16(e);  sin(2 pi e/16) = cos(pi (4 - e)/8) = c16(4 - e)
    const T co = (T)c16(e);
    const T si = (T)(SIGN * c16(4 - e));
    return mk<T>(fma(a.x, co, -a.y * si), fma(a.x, si, a.y * co));
}

// a * e^{SIGN 2 pi i e / 16} for an exponent e that is a constant after unrolling
template <typename T, int SIGN>
__device__ __forceinline__ C2<T> rot16rt(C2<T> v, int e) {
    switch (e & 15) {
        case 0: return v;
        case 1: return rot16<T, SIGN, 1>(v);
        case 2: return rot16<T, SIGN, 2>(v);
        case 3: return rot16<T, SIGN, 3>(v);
        case 4: return rot16<T, SIGN, 4>(v);
        case 5: return rot16<T, SIGN, 5>(v);
        case 6: return rot16<T, SIGN, 6>(v);
        case 7: return rot16<T, SIGN, 7>(v);
        case 8: return rot16<T, SIGN, 8>(v);
        case 9: return rot16<T, SIGN, 9>(v);
        case 10: return rot16<T, SIGN, 10>(v);
        case 11: return rot16<T, SIGN, 11>(v);
        case 12: return rot16<T, SIGN, 12>(v);
        case 13: return rot16<T, SIGN, 13>(v);
        case 14: return rot16<T, SIGN, 14>(v);
        default: return rot16<T, SIGN, 15>(v);
    }
}

// DFT4 in place: X_k = sum_n x_n (SIGN i)^{nk}
template <typename T, int SIGN>
__device__ __forceinline__ void dft4(C2<T>& x0, C2<T>& x1, C2<T>& x2, C2<T>& x3) {
    const C2<T> u0 = cadd<T>(x0, x2), u1 = csub<T>(x0, x2), u2 = cadd<T>(x1, x3);
    const C2<T> u3 = rot16<T, SIGN, 4>(csub<T>(x1, x3));
    x0 = cadd<T>(u0, u2);
    x2 = csub<T>(u0, u2);
    x1 = cadd<T>(u1, u3);
    x3 = csub<T>(u1, u3);
}

// In-register DFT of size R (2, 4, 8, 16): a[k] <- sum_n a[n] e^{SIGN 2 pi i n k / R}.
// R = P*Q with n = n1 + P n2, k = Q k1 + k2:
//   X[Q k1 + k2] = sum_{n1} w_P^{n1 k1} w_R^{n1 k2} sum_{n2} x[n1 + P n2] w_Q^{n2 k2}
// (Q = 4 inner DFT4s, twiddles, P-point outer DFTs); every index is static.
template <typename T, int SIGN, int R>
__device__ __forceinline__ void dft_reg(C2<T> (&a)[R]) {
    if constexpr (R == 2) {
        const C2<T> t = a[0];
        a[0] = cadd<T>(t, a[1]);
        a[1] = csub<T>(t, a[1]);
    } else if constexpr (R == 4) {
        dft4<T, SIGN>(a[0], a[1], a[2], a[3]);
    } else {
        constexpr int P = R / 4;  // 2 or 4
        C2<T> y[P][4];
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) {
#pragma unroll
            for (int n2 = 0; n2 < 4; ++n2) y[n1][n2] = a[n1 + P * n2];
            dft4<T, SIGN>(y[n1][0], y[n1][1], y[n1][2], y[n1][3]);
#pragma unroll
            for (int k2 = 1; k2 < 4; ++k2) y[n1][k2] = rot16rt<T, SIGN>(y[n1][k2], n1 * k2 * (16 / R));
        }
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
            if constexpr (P == 4) {
                C2<T> z0 = y[0][k2], z1 = y[1][k2], z2 = y[2][k2], z3 = y[3][k2];
                dft4<T, SIGN>(z0, z1, z2, z3);
                a[k2] = z0;
                a[4 + k2] = z1;
                a[8 + k2] = z2;
                a[12 + k2] = z3;
            } else {
                a[k2] = cadd<T>(y[0][k2], y[1][k2]);
                a[4 + k2] = csub<T>(y[0][k2], y[1][k2]);
            }
        }
    }
}

// shared-memory layout of TF transforms: [f][L + 2] (row stride = 2 mod 8 complex, so the
// 8 lanes of a quarter warp -- 2 positions x 4 transforms -- fall on distinct banks)
__device__ __forceinline__ int sidx(int f, int pos, int L) { return f * (L + 2) + pos; }

// ------------------------------------------------------------------ kernel parameters
template <typename T>
struct Args {
    C2<T>* grid;          // [R][GS]
    C2<T>* ybuf;          // [R][N]  (adjoint pass A output)
    const C2<T>* hin;     // [R][M]  (adjoint input h)
    C2<T>* fhat;          // [R][M]  (inverse output)
    const T* dk;          // [M] deconvolution (s folded)
    const C2<T>* tw1;     // [N1]  e^{-2 pi i e / N1}
    const C2<T>* tw2;     // [N2]  e^{-2 pi i e / N2}
    const C2<T>* tlo;     // [2^LB]     e^{-2 pi i e / N}
    const C2<T>* thi;     // [N >> LB]  e^{-2 pi i e 2^LB / N}
    int64_t N, GS, M;
    int N1, N2, LB, H;
    int nst1, nst2;       // number of radix stages for N1 / N2
    int rad1[8], rad2[8]; // radix per stage (first to last)
};

template <typename T, int SIGN>
__device__ __forceinline__ C2<T> twid(const C2<T>* __restrict__ tab, int e) {
    C2<T> w = __ldg(tab + e);
    if (SIGN > 0) w.y = -w.y;
    return w;
}

// One Stockham stage on registers: given a[m] = data[j + m L/R] (already loaded), multiply
// by e^{SIGN 2 pi i m (j mod Ns) / (Ns R)} (table entry m (j mod Ns) L/(Ns R) of length L),
// DFT_R; outputs a[m] belong at index (j / Ns) Ns R + (j mod Ns) + m Ns.
template <typename T, int SIGN, int R>
__device__ __forceinline__ void stage_regs(C2<T> (&a)[R], int j, int Ns, int L, const C2<T>* __restrict__ tw) {
    if (Ns > 1) {
        const int k = j % Ns;
        // one table load, the other powers by multiplication (depth <= 4, a few ulps)
        C2<T> w[R];
        w[1] = twid<T, SIGN>(tw, k * (L / (Ns * R)));
#pragma unroll
        for (int m = 2; m < R; ++m) {
            if ((m & (m - 1)) == 0)
                w[m] = cmul<T>(w[m / 2], w[m / 2]);
            else {
                const int hi = 1 << (31 - __clz(m));  // largest power of two below m
                w[m] = cmul<T>(w[hi], w[m - hi]);
            }
        }
#pragma unroll
        for (int m = 1; m < R; ++m) a[m] = cmul<T>(a[m], w[m]);
    }
    dft_reg<T, SIGN, R>(a);
}

// ------------------------------------------------------------------ generic CTA transform
// TF independent length-L transforms, thread t -> (f = t % TF, butterfly index b = t / TF).
// LOAD(f, n) -> value of element n of transform f; STORE(f, k, v) writes output k.
// sm: shared scratch of sp(L * TF) complex.  All threads of the CTA participate.
template <typename T, int SIGN, int R, typename Load, typename Store>
__device__ __forceinline__ void run_stage(int si, int nst, int L, int TF, int Ns, const C2<T>* tw, C2<T>* sm,
                                          Load&& load, Store&& store) {
    const int nbut = L / R;
    const int total = nbut * TF;
    // read phase (all butterflies of this thread) then write phase: each thread handles
    // `per` butterflies; registers hold them all between the two phases.
    constexpr int MAXPER = 16 / R;
    C2<T> a[MAXPER][R];
    const int per = (total + blockDim.x - 1) / blockDim.x;
#pragma unroll
    for (int p = 0; p < MAXPER; ++p) {
        if (p >= per) break;
        const int t = threadIdx.x + p * blockDim.x;
        if (t >= total) break;
        const int f = t % TF, j = t / TF;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int n = j + m * nbut;
            a[p][m] = (si == 0) ? load(f, n) : sm[sidx(f, n, L)];
        }
    }
    if (si > 0) __syncthreads();  // everyone has read the shared buffer
#pragma unroll
    for (int p = 0; p < MAXPER; ++p) {
        if (p >= per) break;
        const int t = threadIdx.x + p * blockDim.x;
        if (t >= total) break;
        const int f = t % TF, j = t / TF;
        stage_regs<T, SIGN, R>(a[p], j, Ns, L, tw);
        const int base = (j / Ns) * Ns * R + (j % Ns);
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int k = base + m * Ns;
            if (si == nst - 1)
                store(f, k, a[p][m]);
            else
                sm[sidx(f, k, L)] = a[p][m];
        }
    }
    if (si < nst - 1) __syncthreads();  // writes visible to the next stage
}

// Static radix plan for L = 2^K: a first stage of radix 2^(K mod 4) (if any), then radix-16.
template <typename T, int SIGN, int L, typename Load, typename Store>
__device__ __forceinline__ void cta_fft(int TF, const C2<T>* tw, C2<T>* sm, Load&& load, Store&& store) {
    constexpr int K = __builtin_ctz(L);
    constexpr int R0 = 1 << (K % 4);
    constexpr int N16 = K / 4;
    constexpr int NST = N16 + (R0 > 1 ? 1 : 0);
    int Ns = 1, si = 0;
    if constexpr (R0 > 1) {
        run_stage<T, SIGN, R0>(si, NST, L, TF, Ns, tw, sm, load, store);
        Ns *= R0;
        ++si;
    }
#pragma unroll 1
    for (int s16 = 0; s16 < N16; ++s16) {
        run_stage<T, SIGN, 16>(si, NST, L, TF, Ns, tw, sm, load, store);
        Ns *= 16;
        ++si;
    }
}

// ------------------------------------------------------------------ pass A (columns)
// MODE 0: inverse, in place on the grid (x = grid[r][n]);  MODE 1: adjoint, x = d_k h_k in
// the band (zero elsewhere), output to ybuf.
template <typename T, int SIGN, int MODE, int L>
__global__ void __launch_bounds__(256) k_pass_a(Args<T> A, int TA) {
    extern __shared__ __align__(16) unsigned char smraw[];
    C2<T>* sm = reinterpret_cast<C2<T>*>(smraw);
    const int64_t r = blockIdx.y;
    const int col0 = blockIdx.x * TA;
    const int N1 = A.N1, N2 = A.N2;
    C2<T>* grow = A.grid + r * A.GS;
    C2<T>* yrow = A.ybuf + r * A.N;
    const C2<T>* hrow = A.hin + r * A.M;
    auto load = [&](int f, int n1) -> C2<T> {
        const int64_t n = (int64_t)N2 * n1 + col0 + f;
        if (MODE == 0) return grow[n];
        // adjoint: ghat_q = d_k h_k for k = q (q < M/2) or q - N (q >= N - M/2)
        const int64_t half = A.M / 2;
        int64_t c;
        if (n < half)
            c = n + half;
        else if (n >= A.N - half)
            c = n - (A.N - half);
        else
            return mk<T>(T(0), T(0));
        const C2<T> v = hrow[c];
        const T d = A.dk[c];
        return mk<T>(d * v.x, d * v.y);
    };
    auto store = [&](int f, int k1, C2<T> v) {
        const int n2 = col0 + f;
        const int e = n2 * k1;  // < N
        const C2<T> w = cmul<T>(twid<T, SIGN>(A.tlo, e & ((1 << A.LB) - 1)), twid<T, SIGN>(A.thi, e >> A.LB));
        v = cmul<T>(v, w);
        const int64_t o = (int64_t)k1 * N2 + n2;
        if (MODE == 0)
            grow[o] = v;
        else
            yrow[o] = v;
    };
    cta_fft<T, SIGN, L>(TA, A.tw1, sm, load, store);
}

// ------------------------------------------------------------------ pass B (rows)
// MODE 0: inverse, input grid rows, output fhat (kept band times d_k);
// MODE 1: adjoint, input ybuf rows, output grid (natural order) + halo.
template <typename T, int SIGN, int MODE, int L>
__global__ void __launch_bounds__(256) k_pass_b(Args<T> A, int TB) {
    extern __shared__ __align__(16) unsigned char smraw[];
    C2<T>* sm = reinterpret_cast<C2<T>*>(smraw);
    const int64_t r = blockIdx.y;
    const int row0 = blockIdx.x * TB;
    const int N1 = A.N1, N2 = A.N2;
    const C2<T>* src = (MODE == 0) ? (A.grid + r * A.GS) : (A.ybuf + r * A.N);
    C2<T>* grow = A.grid + r * A.GS;
    C2<T>* frow = A.fhat + r * A.M;
    auto load = [&](int f, int n2) -> C2<T> { return src[(int64_t)(row0 + f) * N2 + n2]; };
    auto store = [&](int f, int k2, C2<T> v) {
        const int64_t k = (int64_t)(row0 + f) + (int64_t)N1 * k2;
        if (MODE == 0) {
            const int64_t half = A.M / 2;
            int64_t c;
            if (k < half)
                c = k + half;
            else if (k >= A.N - half)
                c = k - (A.N - half);
            else
                return;
            const T d = A.dk[c];
            frow[c] = mk<T>(d * v.x, d * v.y);
        } else {
            grow[k] = v;
            if (k < A.H) grow[A.N + k] = v;
        }
    };
    cta_fft<T, SIGN, L>(TB, A.tw2, sm, load, store);
}

}  // namespace fft

// =========================================================================== host
static void radix_plan(int L, int* rad, int& nst) {
    nst = 0;
    int rem = L;
    while (rem > 1) {
        int R = rem >= 16 ? 16 : rem;
        rad[nst++] = R;
        rem /= R;
    }
    // put the smallest radix first (its stage reads global memory)
    std::reverse(rad, rad + nst);
}

template <typename T>
__global__ void k_twiddle_table(C2<T>* out, int64_t count, int64_t denom, int64_t mult) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    // e^{-2 pi i (i*mult)/denom}, angle reduced exactly in integers
    const int64_t e = (i * mult) % denom;
    double s, c;
    sincospi(-2.0 * (double)e / (double)denom, &s, &c);
    out[i] = mk<T>((T)c, (T)s);
}

struct FftState {
    bool ready = false;
    int N1 = 0, N2 = 0, LB = 0;
    DevBuf tw1, tw2, tlo, thi;
    DevBuf ybuf;
    int64_t y_rhs = 0;
};

static std::map<const Plan*, FftState*>& fft_states() {
    static std::map<const Plan*, FftState*> m;
    return m;
}

bool fused_fft_available(const Plan& p) {
    if (p.d != 1) return false;
    const int64_t N = p.Ms[0];
    if (N < 256 || (N & (N - 1)) || N > (int64_t(1) << 24)) return false;
    if (p.GS < N) return false;
    return true;
}

template <typename T>
static FftState& fft_state(Plan& p, cudaStream_t st) {
    auto& m = fft_states();
    FftState*& s = m[&p];
    if (!s) s = new FftState();
    if (s->ready) return *s;
    const int64_t N = p.Ms[0];
    int lg = 0;
    while ((int64_t(1) << lg) < N) lg++;
    s->N1 = 1 << (lg / 2);       // strided pass (columns)
    s->N2 = (int)(N / s->N1);    // contiguous pass (rows), N2 >= N1
    s->LB = (lg + 1) / 2;
    const size_t cs = sizeof(C2<T>);
    s->tw1.alloc(cs * s->N1);
    s->tw2.alloc(cs * s->N2);
    s->tlo.alloc(cs * ((size_t)1 << s->LB));
    s->thi.alloc(cs * (size_t)(N >> s->LB));
    k_twiddle_table<T><<<(unsigned)ceil_div(s->N1, 256), 256, 0, st>>>(s->tw1.as<C2<T>>(), s->N1, s->N1, 1);
    k_twiddle_table<T><<<(unsigned)ceil_div(s->N2, 256), 256, 0, st>>>(s->tw2.as<C2<T>>(), s->N2, s->N2, 1);
    k_twiddle_table<T><<<(unsigned)ceil_div((int64_t)1 << s->LB, 256), 256, 0, st>>>(s->tlo.as<C2<T>>(),
                                                                                      (int64_t)1 << s->LB, N, 1);
    k_twiddle_table<T><<<(unsigned)ceil_div(N >> s->LB, 256), 256, 0, st>>>(s->thi.as<C2<T>>(), N >> s->LB, N,
                                                                             (int64_t)1 << s->LB);
    INFT_CHECK_LAUNCH();
    p.launches += 4;
    s->ready = true;
    return *s;
}

void release_fft_state(const Plan* p) {
    auto& m = fft_states();
    auto it = m.find(p);
    if (it != m.end()) {
        delete it->second;
        m.erase(it);
    }
}

template <typename T>
static fft::Args<T> make_args(Plan& p, FftState& s) {
    fft::Args<T> A{};
    A.N = p.Ms[0];
    A.GS = p.GS;
    A.M = p.M[0];
    A.N1 = s.N1;
    A.N2 = s.N2;
    A.LB = s.LB;
    A.H = (int)(p.GS - p.Ms[0]);
    radix_plan(s.N1, A.rad1, A.nst1);
    radix_plan(s.N2, A.rad2, A.nst2);
    A.tw1 = s.tw1.as<C2<T>>();
    A.tw2 = s.tw2.as<C2<T>>();
    A.tlo = s.tlo.as<C2<T>>();
    A.thi = s.thi.as<C2<T>>();
    return A;
}

static int tile_for(int L, size_t cs) {
    // ~64 KB of shared memory per CTA (3 CTAs per SM), at least one transform
    int t = (int)std::max<size_t>(1, (size_t)(64 * 1024) / ((size_t)L * cs));
    t = std::min(t, 8);
    while (t > 1 && (t & (t - 1))) t--;
    return t;
}

template <typename T, int L>
static void (*pick_L(int which, int mode))(fft::Args<T>, int) {
    // mode 0 = inverse NFFT (forward sign), mode 1 = inverse adjoint (inverse sign)
    if (which == 0) return mode == 0 ? fft::k_pass_a<T, -1, 0, L> : fft::k_pass_a<T, 1, 1, L>;
    return mode == 0 ? fft::k_pass_b<T, -1, 0, L> : fft::k_pass_b<T, 1, 1, L>;
}

template <typename T>
static void (*pick_kernel(int which, int mode, int L))(fft::Args<T>, int) {
    switch (L) {
        case 16: return pick_L<T, 16>(which, mode);
        case 32: return pick_L<T, 32>(which, mode);
        case 64: return pick_L<T, 64>(which, mode);
        case 128: return pick_L<T, 128>(which, mode);
        case 256: return pick_L<T, 256>(which, mode);
        case 512: return pick_L<T, 512>(which, mode);
        case 1024: return pick_L<T, 1024>(which, mode);
        case 2048: return pick_L<T, 2048>(which, mode);
        case 4096: return pick_L<T, 4096>(which, mode);
    }
    return nullptr;
}

template <typename T>
static void launch_pass(Plan& p, fft::Args<T>& A, int which, int mode, int sign, int64_t R, cudaStream_t st) {
    const int L = which == 0 ? A.N1 : A.N2;
    const int other = which == 0 ? A.N2 : A.N1;
    // TF transforms per CTA: ~64 KB of shared memory, <= 256 threads (TF * L / 16)
    const int TF = std::max(1, std::min({tile_for(L, sizeof(C2<T>)), other, std::max(1, 4096 / L)}));
    const size_t smem = sizeof(C2<T>) * (size_t)((L + 2) * TF);
    int threads = TF * (L / 16);
    threads = std::max(32, std::min(256, threads));
    dim3 g((unsigned)(other / TF), (unsigned)R);
    void (*kern)(fft::Args<T>, int) = pick_kernel<T>(which, mode, L);
    if (!kern) {
        set_error("fused FFT: unsupported factor length");
        throw Fail{INFT_ERR_UNSUPPORTED};
    }
    INFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<g, threads, smem, st>>>(A, TF);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

template <typename T>
const T* dtab_for(const Plan& p);
template <>
const double* dtab_for<double>(const Plan& p) { return p.dk.as<double>(); }
template <>
const float* dtab_for<float>(const Plan& p) { return p.dkf.as<float>(); }

// inverse: grid (spread output, rows GS) -> fhat  (F^* then truncate, times d)
template <typename T>
static void fused_inverse_t(Plan& p, void* grid, void* fhat, int64_t R, cudaStream_t st) {
    FftState& s = fft_state<T>(p, st);
    fft::Args<T> A = make_args<T>(p, s);
    A.grid = static_cast<C2<T>*>(grid);
    A.fhat = static_cast<C2<T>*>(fhat);
    A.dk = dtab_for<T>(p);
    launch_pass<T>(p, A, 0, 0, -1, R, st);
    launch_pass<T>(p, A, 1, 0, -1, R, st);
}

// adjoint: h -> grid (D, zero pad, F), natural order with halo
template <typename T>
static void fused_adjoint_t(Plan& p, const void* h, void* grid, int64_t R, cudaStream_t st) {
    FftState& s = fft_state<T>(p, st);
    if (s.y_rhs < R) {
        s.ybuf.alloc(sizeof(C2<T>) * (size_t)p.Ms[0] * R);
        s.y_rhs = R;
    }
    fft::Args<T> A = make_args<T>(p, s);
    A.grid = static_cast<C2<T>*>(grid);
    A.ybuf = s.ybuf.as<C2<T>>();
    A.hin = static_cast<const C2<T>*>(h);
    A.dk = dtab_for<T>(p);
    launch_pass<T>(p, A, 0, 1, +1, R, st);
    launch_pass<T>(p, A, 1, 1, +1, R, st);
}

void fused_fft_inverse(Plan& p, void* grid, void* fhat, int64_t R, cudaStream_t st) {
    if (p.prec == INFT_C128)
        fused_inverse_t<double>(p, grid, fhat, R, st);
    else
        fused_inverse_t<float>(p, grid, fhat, R, st);
}

void fused_fft_adjoint(Plan& p, const void* h, void* grid, int64_t R, cudaStream_t st) {
    if (p.prec == INFT_C128)
        fused_adjoint_t<double>(p, h, grid, R, st);
    else
        fused_adjoint_t<float>(p, h, grid, R, st);
}

}  // namespace inft
