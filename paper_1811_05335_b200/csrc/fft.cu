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
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "inft_internal.cuh"
#include "tma.cuh"

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

// cos(pi m / 16), m = 0..31
__device__ __forceinline__ constexpr double c32(int m) {
    constexpr double t[32] = {1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
                              0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173,
                              0.19509032201612826785, 0.0, -0.19509032201612826785, -0.38268343236508977173,
                              -0.55557023301960222474, -0.70710678118654752440, -0.83146961230254523708,
                              -0.92387953251128675613, -0.98078528040323044913, -1.0, -0.98078528040323044913,
                              -0.92387953251128675613, -0.83146961230254523708, -0.70710678118654752440,
                              -0.55557023301960222474, -0.38268343236508977173, -0.19509032201612826785, 0.0,
                              0.19509032201612826785, 0.38268343236508977173, 0.55557023301960222474,
                              0.70710678118654752440, 0.83146961230254523708, 0.92387953251128675613,
                              0.98078528040323044913};
    return t[m & 31];
}

// a * e^{SIGN 2 pi i E / 32} (even exponents reduce to rot16)
template <typename T, int SIGN, int E>
__device__ __forceinline__ C2<T> rot32(C2<T> a) {
    constexpr int e = ((E % 32) + 32) % 32;
    if constexpr (e % 2 == 0) {
        return rot16<T, SIGN, e / 2>(a);
    } else {
        // cos(2 pi e / 32) = cos(pi e / 16);  sin(2 pi e / 32) = cos(pi (8 - e) / 16)
        const T co = (T)c32(e);
        const T si = (T)(SIGN * c32(8 - e));
        return mk<T>(fma(a.x, co, -a.y * si), fma(a.x, si, a.y * co));
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

// DFT4 of the first-level sub-transforms; Z: inputs x1 = x2 = 0 (the zero band of the adjoint's
// first stage, see run_stage_ip): X = (x0 + x3, x0 - SIGN i x3, x0 - x3, x0 + SIGN i x3)
template <typename T, int SIGN, bool Z>
__device__ __forceinline__ void dft4g(C2<T>& x0, C2<T>& x1, C2<T>& x2, C2<T>& x3) {
    if constexpr (Z) {
        const C2<T> u3 = rot16<T, SIGN, 4>(mk<T>(-x3.x, -x3.y));
        const C2<T> a = x0, b = x3;
        x0 = cadd<T>(a, b);
        x2 = csub<T>(a, b);
        x1 = cadd<T>(a, u3);
        x3 = csub<T>(a, u3);
    } else {
        dft4<T, SIGN>(x0, x1, x2, x3);
    }
}

// In-register DFT of size R (2, 4, 8, 16): a[k] <- sum_n a[n] e^{SIGN 2 pi i n k / R}.
// R = P*Q with n = n1 + P n2, k = Q k1 + k2:
//   X[Q k1 + k2] = sum_{n1} w_P^{n1 k1} w_R^{n1 k2} sum_{n2} x[n1 + P n2] w_Q^{n2 k2}
// (Q = 4 inner DFT4s, twiddles, P-point outer DFTs); every index is static.
// Z: a[m] = 0 for m in [R/4, 3R/4) (inputs n2 = 1, 2 of every inner DFT4), the zeros never read.
template <typename T, int SIGN, int R, bool Z = false>
__device__ __forceinline__ void dft_reg(C2<T> (&a)[R]);

// 32-point DFT as 8 x 4: n = n1 + 8 n2, k = 4 k1 + k2:
//   X[4 k1 + k2] = sum_{n1} w_8^{n1 k1} w_32^{n1 k2} sum_{n2} x[n1 + 8 n2] w_4^{n2 k2}
template <typename T, int SIGN, bool Z = false>
__device__ __forceinline__ void dft32(C2<T> (&a)[32]) {
    C2<T> y[8][4];
#pragma unroll
    for (int n1 = 0; n1 < 8; ++n1) {
        C2<T> x0 = a[n1], x1 = a[n1 + 8], x2 = a[n1 + 16], x3 = a[n1 + 24];
        dft4g<T, SIGN, Z>(x0, x1, x2, x3);
        y[n1][0] = x0;
        y[n1][1] = x1;
        y[n1][2] = x2;
        y[n1][3] = x3;
    }
#define INFT_R32_TW(N1, K2) y[N1][K2] = rot32<T, SIGN, (N1) * (K2)>(y[N1][K2]);
#define INFT_R32_ROW(N1) INFT_R32_TW(N1, 1) INFT_R32_TW(N1, 2) INFT_R32_TW(N1, 3)
    INFT_R32_ROW(1) INFT_R32_ROW(2) INFT_R32_ROW(3) INFT_R32_ROW(4) INFT_R32_ROW(5) INFT_R32_ROW(6) INFT_R32_ROW(7)
#undef INFT_R32_ROW
#undef INFT_R32_TW
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
        C2<T> z[8];
#pragma unroll
        for (int n1 = 0; n1 < 8; ++n1) z[n1] = y[n1][k2];
        dft_reg<T, SIGN, 8>(z);
#pragma unroll
        for (int k1 = 0; k1 < 8; ++k1) a[4 * k1 + k2] = z[k1];
    }
}

template <typename T, int SIGN, int R, bool Z>
__device__ __forceinline__ void dft_reg(C2<T> (&a)[R]) {
    if constexpr (R == 32) {
        dft32<T, SIGN, Z>(a);
    } else if constexpr (R == 2) {
        const C2<T> t = a[0];
        a[0] = cadd<T>(t, a[1]);
        a[1] = csub<T>(t, a[1]);
    } else if constexpr (R == 4) {
        dft4g<T, SIGN, Z>(a[0], a[1], a[2], a[3]);
    } else {
        constexpr int P = R / 4;  // 2 or 4
        C2<T> y[P][4];
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) {
#pragma unroll
            for (int n2 = 0; n2 < 4; ++n2) y[n1][n2] = a[n1 + P * n2];
            dft4g<T, SIGN, Z>(y[n1][0], y[n1][1], y[n1][2], y[n1][3]);
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
};

// table entry e of a forward-sign twiddle table, conjugated for SIGN > 0 (any state space)
template <typename T, int SIGN>
__device__ __forceinline__ C2<T> twid(const C2<T>* tab, int e) {
    C2<T> w = tab[e];
    if (SIGN > 0) w.y = -w.y;
    return w;
}

template <typename T, int SIGN>
__device__ __forceinline__ C2<T> twid_g(const C2<T>* __restrict__ tab, int e) {
    C2<T> w = __ldg(tab + e);
    if (SIGN > 0) w.y = -w.y;
    return w;
}

// One Stockham stage on registers: given a[m] = data[j + m L/R] (already loaded), multiply
// by e^{SIGN 2 pi i m (j mod Ns) / (Ns R)} (table entry m (j mod Ns) L/(Ns R) of length L),
// DFT_R; outputs a[m] belong at index (j / Ns) Ns R + (j mod Ns) + m Ns.
#ifndef INFT_R32_BLOCKTW
#define INFT_R32_BLOCKTW 1
#endif
#ifndef INFT_R16_BLOCKTW
#define INFT_R16_BLOCKTW 1
#endif
// Stage twiddle table (in-place radix-16 passes, stages with a span NS <= 8): the stage has only
// NS distinct twiddle sets, so all R - 1 powers of each sit in a small shared table [R - 1][NS]
// (built once per CTA) and are loaded (a warp touches <= 8 consecutive entries: one wavefront)
// instead of derived from one table entry by 14 complex products per butterfly.
#ifndef INFT_FFT_STAGE_TAB
#define INFT_FFT_STAGE_TAB 1
#endif
constexpr bool kStageTab = INFT_FFT_STAGE_TAB != 0;
constexpr int kStageTabNS = 8;                         // largest span served by the table
constexpr int kStageTabElems = 15 * kStageTabNS;       // entries (radix 16)
template <int R, int NS>
constexpr bool stage_tab() { return kStageTab && R == 16 && NS > 1 && NS <= kStageTabNS; }

template <typename T, int SIGN, int R, int L, int NS, bool Z = false, bool TAB = false>
__device__ __forceinline__ void stage_regs(C2<T> (&a)[R], int j, const C2<T>* __restrict__ tw,
                                           const C2<T>* __restrict__ tw2 = nullptr) {
    if constexpr (TAB) {
        const int k = j % NS;
#pragma unroll
        for (int m = 1; m < R; ++m) a[m] = cmul<T>(a[m], twid<T, SIGN>(tw2, (m - 1) * NS + k));
    } else if constexpr (NS > 1 && ((R == 32 && INFT_R32_BLOCKTW) || (R == 16 && INFT_R16_BLOCKTW))) {
        // radix 32: twiddles in blocks of four, a[4b + i] *= w^i w^{4b} with w^{4b} by a running
        // product (depth <= 8): six live twiddles instead of 31 (the full table held ~120
        // registers of the 246 the radix-32 passes used)
        const int k = j % NS;
        const C2<T> w1 = twid<T, SIGN>(tw, k * (L / (NS * R)));
        const C2<T> w2 = cmul<T>(w1, w1);
        const C2<T> w3 = cmul<T>(w2, w1);
        const C2<T> w4 = cmul<T>(w2, w2);
        C2<T> wb = w4;
#pragma unroll
        for (int b = 0; b < R / 4; ++b) {
            if (b > 0) a[4 * b] = cmul<T>(a[4 * b], wb);
            a[4 * b + 1] = cmul<T>(a[4 * b + 1], b > 0 ? cmul<T>(wb, w1) : w1);
            a[4 * b + 2] = cmul<T>(a[4 * b + 2], b > 0 ? cmul<T>(wb, w2) : w2);
            a[4 * b + 3] = cmul<T>(a[4 * b + 3], b > 0 ? cmul<T>(wb, w3) : w3);
            if (b > 0 && b + 1 < R / 4) wb = cmul<T>(wb, w4);
        }
    } else if constexpr (NS > 1) {
        const int k = j % NS;
        // one table load, the other powers by multiplication (depth <= 4, a few ulps)
        C2<T> w[R];
        w[1] = twid<T, SIGN>(tw, k * (L / (NS * R)));
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
    dft_reg<T, SIGN, R, Z>(a);
}

// ------------------------------------------------------------------ CTA transform geometry
// kRB: radix of the bulk Stockham stages (16: 16 elements per thread, 8: twice the threads
// per tile at half the registers per thread)
#ifndef INFT_FFT_RADIX
#define INFT_FFT_RADIX 16
#endif
constexpr int kRB = INFT_FFT_RADIX;
// elements per tile (4096: 64 KB at complex128, one CTA per SM; 2048: two CTAs per SM)
#ifndef INFT_FFT_TILE
#define INFT_FFT_TILE 4096
#endif
constexpr int kTileElems = INFT_FFT_TILE;
// complex64 tiles (elements): 8192 = 64 KB like a complex128 tile, 512 threads at <= 128
// registers (config 5 c64: 4096 -> 3.55 ms/step, 8192 -> 3.06)
#ifndef INFT_FFT_TILE_F
#define INFT_FFT_TILE_F 8192
#endif
constexpr int kTileElemsF = INFT_FFT_TILE_F;
// in-place kernels: 4096-element tiles at both precisions (256 threads, <= 128 registers at two
// CTAs per SM; complex64's 8192-element tiles would need 512 threads at 64 registers)
constexpr int kTileIP = 4096;
// in-place kernels: L2 prefetch of the next tile at the start of the current one
// experiment (timing only, wrong results): INFT_EXP_NOLOAD=1 -- the in-place passes skip their
// tile loads (compute + stores only)
#ifndef INFT_EXP_NOLOAD
#define INFT_EXP_NOLOAD 0
#endif
constexpr bool kNoLoad = INFT_EXP_NOLOAD != 0;
#ifndef INFT_FFT_PREFETCH
#define INFT_FFT_PREFETCH 1
#endif
constexpr bool kPrefetch = INFT_FFT_PREFETCH != 0;
// in-place pass B of the adjoint (INFT_FFT_IP_B1=1): plain stores of the grid from registers
// (1) or staged TMA store boxes (0)
#ifndef INFT_FFT_PLAIN_B1
#define INFT_FFT_PLAIN_B1 1
#endif
constexpr bool kPlainB1 = INFT_FFT_PLAIN_B1 != 0;
// pass A, L2 prefetch of the next tile at the start of the current one: on for the adjoint
// (MODE 1: band rows of h; config 5: 0.742 -> 0.720 ms), off for the inverse (MODE 0: the whole
// strided column tile; 0.826 -> 0.96 ms with it)
#ifndef INFT_FFT_PREFETCH_A
#define INFT_FFT_PREFETCH_A 0
#endif
#ifndef INFT_FFT_PREFETCH_A1
#define INFT_FFT_PREFETCH_A1 1
#endif
constexpr bool kPrefetchA = INFT_FFT_PREFETCH_A != 0;
constexpr bool kPrefetchA1 = INFT_FFT_PREFETCH_A1 != 0;
template <typename T>
constexpr int tile_elems() { return sizeof(T) == 8 ? kTileElems : kTileElemsF; }
constexpr int kLgRB = kRB == 32 ? 5 : (kRB == 16 ? 4 : (kRB == 8 ? 3 : 2));
// TF independent length-L transforms per tile (compile-time: ~64 KB of shared memory, at
// most 256 threads = TF L / 16, at most 8), thread t -> (f = t % TF, butterfly j = t / TF).
// Static radix plan for L = 2^K: a first stage of radix 2^(K mod 4) (if any), then radix-16.
template <typename T, int L, int TE_ = 0, int RB_ = kRB>
struct Geo {
    static constexpr int RB = RB_;  // radix of the bulk stages
    static constexpr int LgRB = RB == 32 ? 5 : (RB == 16 ? 4 : (RB == 8 ? 3 : 2));
    static constexpr int TE = TE_ > 0 ? TE_ : tile_elems<T>();
    static constexpr int TF = L >= TE / 8 ? (TE / L > 0 ? TE / L : 1) : 8;
    static constexpr int NT = TF * L / RB < 32 ? 32 : TF * L / RB;  // threads per CTA
    // row padding of the [f][L + PAD] layout: the lanes of one 128-byte shared wavefront cover
    // TF transforms x (wavefront / TF) consecutive positions
    static constexpr int WAVE = (int)(128 / sizeof(C2<T>));
    static constexpr int PAD = WAVE / TF > 1 ? WAVE / TF : 1;
    static constexpr int ST = L + PAD;  // row stride of pass B's bulk-copied tile rows
    static constexpr int K = __builtin_ctz(L);
    static constexpr int R0 = 1 << (K % LgRB);
    static constexpr int RF = R0 > 1 ? R0 : RB;  // radix of the first stage
    static constexpr int PER0 = RB / RF;         // butterflies per thread in the first stage
    static constexpr int NST = K / LgRB + (R0 > 1 ? 1 : 0);
    static constexpr int LR = L / RB;            // span of the last stage = twiddle table size
    // work buffer rows: position p lives at p + p / SKD with SKD = RF (one skew slot per
    // first-stage butterfly, so the first stage's strided writes RF j + m spread over the
    // banks) when one wavefront spans several butterflies of a transform (PAD > 1); row
    // stride SW = PAD (mod WAVE) like ST
    // (radix-8 build: one slot per 8 positions -- conflict-free for first-stage radices 2..8
    //  at 12.5 % extra rows, which keeps pass B of M_sigma = 2^21 inside 227 KB)
    static constexpr int SKD = RB == 8 ? (PAD > 1 ? 8 : L) : ((PAD > 1 && RF >= 4) ? RF : L);  // skew divisor (L: none)
    static constexpr int SW0 = L + L / SKD;
    static constexpr int SW = SW0 + ((PAD - SW0 % WAVE) % WAVE + WAVE) % WAVE;
};

// shared-memory layout of the TF transforms: [f][S]
template <typename G>
__device__ __forceinline__ int sidx(int f, int pos) { return f * G::SW + pos + pos / G::SKD; }

// One stage SI (radix R, span NS) of TF transforms.  LOAD(f, n, p, m) -> element n of
// transform f (the first stage's butterfly p, leg m of this thread); STORE(f, k, v, m) writes
// output k (leg m of the last stage's single butterfly of this thread, legs in increasing m).
// sm: [TF][S] shared scratch;  tw: table e^{-2 pi i e / L}, e < L / 16 (the entries the
// radix-16 stages use).
template <typename T, int SIGN, typename G, int R, int NS, int SI, typename Load, typename Store>
__device__ __forceinline__ void run_stage(const C2<T>* tw, C2<T>* sm, Load&& load, Store&& store) {
    constexpr int L = G::ST - G::PAD;
    constexpr int TF = G::TF;
    constexpr int nbut = L / R;
    constexpr int total = nbut * TF;
    constexpr int per = (total + G::NT - 1) / G::NT;
    constexpr bool last = SI == G::NST - 1;
    C2<T> a[per][R];
#pragma unroll
    for (int p = 0; p < per; ++p) {
        const int t = threadIdx.x + p * G::NT;
        if (total % G::NT != 0 && t >= total) break;
        const int f = t % TF, j = t / TF;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int n = j + m * nbut;
            if constexpr (SI == 0)
                a[p][m] = load(f, n, p, m);
            else
                a[p][m] = sm[sidx<G>(f, n)];
        }
    }
    // everyone has read the shared buffer (also for a single-stage transform: its outputs are
    // staged in the buffer its inputs came from)
    if constexpr (SI > 0 || last) __syncthreads();
#pragma unroll
    for (int p = 0; p < per; ++p) {
        const int t = threadIdx.x + p * G::NT;
        if (total % G::NT != 0 && t >= total) break;
        const int f = t % TF, j = t / TF;
        stage_regs<T, SIGN, R, L, NS>(a[p], j, tw);
        const int base = (j / NS) * NS * R + (j % NS);
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int k = base + m * NS;
            if constexpr (last)
                store(f, k, a[p][m], m);
            else
                sm[sidx<G>(f, k)] = a[p][m];
        }
    }
    if constexpr (!last) __syncthreads();  // writes visible to the next stage
}

template <typename T, int SIGN, typename G, int SI, int NS, typename Load, typename Store>
__device__ __forceinline__ void fft_stages(const C2<T>* tw, C2<T>* sm, Load&& load, Store&& store) {
    if constexpr (SI < G::NST) {
        constexpr int R = (SI == 0) ? G::RF : kRB;
        run_stage<T, SIGN, G, R, NS, SI>(tw, sm, load, store);
        fft_stages<T, SIGN, G, SI + 1, NS * R>(tw, sm, load, store);
    }
}

template <typename T, int SIGN, int L, typename Load, typename Store>
__device__ __forceinline__ void cta_fft(const C2<T>* tw, C2<T>* sm, Load&& load, Store&& store) {
    fft_stages<T, SIGN, Geo<T, L>, 0, 1>(tw, sm, load, store);
}

// In-place variant (experiment, INFT_FFT_IP): the tile buffer is also the work buffer, so a
// CTA needs one ~80 KB buffer and two CTAs share an SM; stage 0 reads the landed tile, waits
// for every thread, then writes the skewed work layout into the same buffer; after the last
// stage has read the buffer, on_free() (thread 0) issues the next tile's copy into it.
// HZ (first stage of the adjoint's pass A when the band is L/4 rows on each side, sigma = 2):
// rows [L/4, 3L/4) are zero and, with a first-stage radix RF >= 4, they are exactly the legs
// m in [RF/4, 3RF/4) of every butterfly -- never loaded, and the inner DFT4s skip them.
template <typename T, int SIGN, typename G, int R, int NS, int SI, bool HZ, typename Load, typename Store,
          typename Free>
__device__ __forceinline__ void run_stage_ip(const C2<T>* tw, const C2<T>* tw2, C2<T>* sm, Load&& load, Store&& store,
                                             Free&& on_free) {
    constexpr bool Z = HZ && SI == 0 && R >= 4;
    constexpr int L = G::ST - G::PAD;
    constexpr int TF = G::TF;
    constexpr int nbut = L / R;
    constexpr int total = nbut * TF;
    constexpr int per = (total + G::NT - 1) / G::NT;
    constexpr bool last = SI == G::NST - 1;
    C2<T> a[per][R];
#pragma unroll
    for (int p = 0; p < per; ++p) {
        const int t = threadIdx.x + p * G::NT;
        if (total % G::NT != 0 && t >= total) break;
        const int f = t % TF, j = t / TF;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int n = j + m * nbut;
            if constexpr (Z) {
                if (m >= R / 4 && m < 3 * R / 4) continue;
            }
            if constexpr (SI == 0)
                a[p][m] = load(f, n, p, m);
            else
                a[p][m] = sm[sidx<G>(f, n)];
        }
    }
    if constexpr (last) fence_proxy_async();  // generic reads before the next tile's TMA
    __syncthreads();  // every read of the shared buffer done (the writes below reuse it)
    if constexpr (last) on_free();
#pragma unroll
    for (int p = 0; p < per; ++p) {
        const int t = threadIdx.x + p * G::NT;
        if (total % G::NT != 0 && t >= total) break;
        const int f = t % TF, j = t / TF;
        stage_regs<T, SIGN, R, L, NS, Z, stage_tab<R, NS>()>(a[p], j, tw, tw2);
        const int base = (j / NS) * NS * R + (j % NS);
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int k = base + m * NS;
            if constexpr (last)
                store(f, k, a[p][m], m);
            else
                sm[sidx<G>(f, k)] = a[p][m];
        }
    }
    if constexpr (!last) __syncthreads();
}

template <typename T, int SIGN, typename G, int SI, int NS, bool HZ, typename Load, typename Store, typename Free>
__device__ __forceinline__ void fft_stages_ip(const C2<T>* tw, const C2<T>* tw2, C2<T>* sm, Load&& load, Store&& store,
                                              Free&& on_free) {
    if constexpr (SI < G::NST) {
        constexpr int R = (SI == 0) ? G::RF : G::RB;
        run_stage_ip<T, SIGN, G, R, NS, SI, HZ>(tw, tw2, sm, load, store, on_free);
        fft_stages_ip<T, SIGN, G, SI + 1, NS * R, HZ>(tw, tw2, sm, load, store, on_free);
    }
}

// The in-place kernels keep the stage twiddle table in the LAST kStageTabElems entries of their
// dynamic shared memory (the host adds the room); it serves the stage whose span is RF, the
// first-stage radix (the only stage with 1 < NS <= 8 in a radix-16 plan).
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t v;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
    return v;
}
template <typename T, typename G>
__device__ __forceinline__ const C2<T>* stage_tab_fill(unsigned char* smraw, const C2<T>* __restrict__ gtab) {
    constexpr int L = G::ST - G::PAD;
    constexpr int NS = G::RF;  // span of the stage after the first one
    C2<T>* t2 = reinterpret_cast<C2<T>*>(smraw + dyn_smem_bytes() - sizeof(C2<T>) * kStageTabElems);
    if constexpr (stage_tab<G::RB, NS>() && G::NST >= 2) {
        for (int i = threadIdx.x; i < 15 * NS; i += blockDim.x) {
            const int m = i / NS + 1, k = i % NS;
            t2[i] = gtab[m * k * (L / (NS * 16))];
        }
    }
    return t2;
}

// byte offset of pass B's deconvolution tile: after tile[2] | work | twiddles, 128-aligned
template <typename T>
__host__ __device__ constexpr size_t d_offset(int L, int ST, int SW, int TB) {
    return ((sizeof(C2<T>) * (size_t)(2 * ST * TB + SW * TB + L / kRB)) + 127) / 128 * 128;
}

// ------------------------------------------------------------------ persistent tiled passes
// Each pass is a persistent kernel (one CTA per SM) walking a list of tiles; the next tile
// is copied into the other half of a double buffer by the Tensor Memory Accelerator (pass A:
// 3-D tensor-map boxes of the strided columns; pass B: 1-D bulk copies of whole rows) while
// the CTA transforms the current one, so HBM reads overlap the arithmetic.  The first
// Stockham stage reads the landed tile, the stages in between use the work buffer, the last
// stage applies the epilogue and writes global memory from registers.
//
// Shared memory: tile[2] | work | mbarrier[2].
//
// Pass A (columns, length L = N1, TF = TA columns per tile, tile layout [n1][TA]):
//   MODE 0 (inverse): x = grid[r][N2 n1 + n2], output in place (twiddled);
//   MODE 1 (adjoint): x = d_c h[r][c] on the band rows (the TMA boxes fetch only those rows,
//                     the other rows are zero and never read), output to ybuf.
template <typename T, int SIGN, int MODE, int L>
__global__ void __launch_bounds__(Geo<T, L>::NT, 1)
    k_pass_a(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap dmap, Args<T> A, int BR,
             int ntiles) {
    extern __shared__ __align__(128) unsigned char smraw[];
    constexpr int CE = (int)(sizeof(C2<T>) / 8);
    using G = Geo<T, L>;
    constexpr int TA = G::TF, S = G::SW;
    C2<T>* tile = reinterpret_cast<C2<T>*>(smraw);
    C2<T>* work = tile + 2 * L * TA;
    C2<T>* tws = work + S * TA;  // stage twiddles, L / 16 entries
    uint64_t* bars = reinterpret_cast<uint64_t*>(tws + L / kRB);
    const int N2 = A.N2;
    const int tiles_per_rhs = N2 / TA;
    const int B = (int)(A.M / 2 / N2);  // band rows on each side (MODE 1)
    // MODE 1: the deconvolution factors of the band rows land in the unused middle rows of the
    // tile buffer, as [2B][DW] (rows: d rows [B, 2B) then [0, B); DW >= TA columns)
    constexpr int DW = (int)(16 / sizeof(T)) > TA ? (int)(16 / sizeof(T)) : TA;
    const uint32_t tile_bytes = (uint32_t)(MODE == 0 ? sizeof(C2<T>) * TA * L
                                                     : sizeof(C2<T>) * TA * 2 * B + sizeof(T) * DW * 2 * B);
    if (threadIdx.x == 0) {
        prefetch_tmap(&map);
        if (MODE == 1) prefetch_tmap(&dmap);
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < L / kRB; i += blockDim.x) tws[i] = A.tw1[i];
    __syncthreads();
    auto issue = [&](int id, int b) {
        const int r = id / tiles_per_rhs, c0 = (id % tiles_per_rhs) * TA * CE;
        C2<T>* dst = tile + b * L * TA;
        mbar_arrive_expect_tx(&bars[b], tile_bytes);
        if (MODE == 0) {
            for (int q = 0; q < L; q += BR) tma_load_3d(dst + q * TA, &map, c0, q, r, &bars[b]);
        } else {
            // tile rows [0, B) <- h rows [B, 2B);  tile rows [L - B, L) <- h rows [0, B)
            T* dsm = reinterpret_cast<T*>(dst + B * TA);
            const int dc0 = ((id % tiles_per_rhs) * TA) & ~(DW - 1);  // 16-byte aligned box start
            for (int q = 0; q < B; q += BR) {
                tma_load_3d(dst + q * TA, &map, c0, B + q, r, &bars[b]);
                tma_load_3d(dst + (L - B + q) * TA, &map, c0, q, r, &bars[b]);
                tma_load_3d(dsm + q * DW, &dmap, dc0, B + q, 0, &bars[b]);
                tma_load_3d(dsm + (B + q) * DW, &dmap, dc0, q, 0, &bars[b]);
            }
        }
    };
    // this thread's single butterfly of the last stage: transform fl, outputs k1 = jl + m L/16
    const int fl = threadIdx.x % TA, jl = threadIdx.x < TA * (L / kRB) ? threadIdx.x / TA : 0;
    const int lmask = (1 << A.LB) - 1;
    int it = 0;
    if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++it) {
        const int b = it & 1;
        if (threadIdx.x == 0 && id + (int)gridDim.x < ntiles) issue(id + gridDim.x, b ^ 1);
        const int64_t r = id / tiles_per_rhs;
        const int col0 = (id % tiles_per_rhs) * TA;
        // loads independent of the tile data, issued before waiting for it:
        // four-step twiddles w_N^{n2 k1} = w_N^{n2 jl} (w_N^{n2 L/16})^m ...
        const int n2l = col0 + fl;
        const int e0 = n2l * jl, eq = n2l * (L / kRB);
        const C2<T> t0a = twid_g<T, SIGN>(A.tlo, e0 & lmask), t0b = twid_g<T, SIGN>(A.thi, e0 >> A.LB);
        const C2<T> tqa = twid_g<T, SIGN>(A.tlo, eq & lmask), tqb = twid_g<T, SIGN>(A.thi, eq >> A.LB);
        mbar_wait(&bars[b], (it >> 1) & 1);
        const C2<T>* tl = tile + b * L * TA;
        const T* dsm = reinterpret_cast<const T*>(tl + B * TA);
        auto load = [&](int f, int n1, int, int) -> C2<T> {
            if (MODE == 0) return tl[n1 * TA + f];
            if (n1 >= B && n1 < L - B) return mk<T>(T(0), T(0));
            const C2<T> v = tl[n1 * TA + f];
            const T d = dsm[(n1 < B ? n1 : n1 - (L - 2 * B)) * DW + (col0 & (DW - 1)) + f];
            return mk<T>(d * v.x, d * v.y);
        };
        // the twiddle products are formed at the first store (last stage), so the table loads
        // issued above complete under the earlier stages instead of stalling here
        C2<T> wq, wcur;
        // plain stores from registers: staging the outputs in tile[b] and storing them by TMA
        // boxes (as pass B does) was slower here -- the boxes are only TA columns (64 B) wide
        // (config 5: 0.944 vs 0.886 ms)
        C2<T>* orow = (MODE == 0) ? A.grid + r * A.GS : A.ybuf + r * A.N;
        auto store = [&](int f, int k1, C2<T> v, int m) {
            if (m == 0) {
                wq = cmul<T>(tqa, tqb);
                wcur = cmul<T>(t0a, t0b);
            } else {
                wcur = cmul<T>(wcur, wq);
            }
            orow[(int64_t)k1 * N2 + col0 + f] = cmul<T>(v, wcur);
        };
        cta_fft<T, SIGN, L>(tws, work, load, store);
        fence_proxy_async();  // this thread's reads of tile[b] precede the next TMA into it
        __syncthreads();      // tile[b] and work free for the next iteration
    }
}

// Pass A in place (MODE 0 inverse, MODE 1 adjoint; same data flow as k_pass_a): one buffer
// of max(L TA, SW TA) elements per CTA, two CTAs per SM (config 5 pass A MODE 0: 0.886 ->
// 0.826 ms against the double-buffered one-CTA kernel).
#ifndef INFT_R32_MINB
#define INFT_R32_MINB 2
#endif
// HZ (MODE 1 only): the band is exactly L/4 rows on each side (sigma = 2), so the first stage
// skips the zero rows at compile time (run_stage_ip); the host picks it when M / 2 / N2 == L / 4.
template <typename T, int SIGN, int MODE, int L, int TE = kTileIP, int RB = kRB, bool HZ = false>
// (complex64 adjoint, 8192-element radix-32 tiles: ONE 256-thread CTA per SM with all the registers
//  it wants (246, no spills) instead of two at 128 with spills -- config 5 c64: 0.444 -> 0.375 ms;
//  the inverse's pass A is the other way round, 0.400 -> 0.500 ms.  -DINFT_C64_A1_MINB=2: two CTAs)
#ifndef INFT_C64_A1_MINB
#define INFT_C64_A1_MINB 1
#endif
__global__ void __launch_bounds__(Geo<T, L, TE, RB>::NT, TE == kTileIP ? (RB == 32 ? INFT_R32_MINB : 2) : (TE < kTileIP ? 4 : (sizeof(T) == 4 && MODE == 1 ? INFT_C64_A1_MINB : 2)))
    k_pass_a_ip(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap dmap, Args<T> A, int BR,
                int ntiles) {
    extern __shared__ __align__(128) unsigned char smraw[];
    constexpr int CE = (int)(sizeof(C2<T>) / 8);
    using G = Geo<T, L, TE, RB>;
    constexpr int TA = G::TF, S = G::SW;
    constexpr int BUF = (L * TA > S * TA ? L * TA : S * TA);
    C2<T>* buf = reinterpret_cast<C2<T>*>(smraw);
    C2<T>* tws = buf + BUF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(tws + L / RB);
    const int N2 = A.N2;
    const int tiles_per_rhs = N2 / TA;
    const int B = (int)(A.M / 2 / N2);  // band rows on each side (MODE 1)
    constexpr int DW = (int)(16 / sizeof(T)) > TA ? (int)(16 / sizeof(T)) : TA;
    const uint32_t tile_bytes = (uint32_t)(MODE == 0 ? sizeof(C2<T>) * TA * L
                                                     : sizeof(C2<T>) * TA * 2 * B + sizeof(T) * DW * 2 * B);
    if (threadIdx.x == 0) {
        prefetch_tmap(&map);
        if (MODE == 1) prefetch_tmap(&dmap);
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < L / RB; i += blockDim.x) tws[i] = A.tw1[i];
    const C2<T>* tws2 = stage_tab_fill<T, G>(smraw, A.tw1);
    __syncthreads();
    // L2 prefetch of a tile's boxes (INFT_FFT_PREFETCH_A, off: slower here, see kPrefetchA): the
    // in-place buffer can only take the next tile after the last stage has read it
    auto prefetch = [&](int id) {
        const int r = id / tiles_per_rhs, c0 = (id % tiles_per_rhs) * TA * CE;
        if (MODE == 0) {
            for (int q = 0; q < L; q += BR) tma_prefetch_3d(&map, c0, q, r);
        } else {
            for (int q = 0; q < B; q += BR) {
                tma_prefetch_3d(&map, c0, B + q, r);
                tma_prefetch_3d(&map, c0, q, r);
            }
        }
    };
    auto issue = [&](int id) {
        const int r = id / tiles_per_rhs, c0 = (id % tiles_per_rhs) * TA * CE;
        mbar_arrive_expect_tx(bar, tile_bytes);
        if (MODE == 0) {
            for (int q = 0; q < L; q += BR) tma_load_3d(buf + q * TA, &map, c0, q, r, bar);
        } else {
            T* dsm = reinterpret_cast<T*>(buf + B * TA);
            const int dc0 = ((id % tiles_per_rhs) * TA) & ~(DW - 1);
            for (int q = 0; q < B; q += BR) {
                tma_load_3d(buf + q * TA, &map, c0, B + q, r, bar);
                tma_load_3d(buf + (L - B + q) * TA, &map, c0, q, r, bar);
                tma_load_3d(dsm + q * DW, &dmap, dc0, B + q, 0, bar);
                tma_load_3d(dsm + (B + q) * DW, &dmap, dc0, q, 0, bar);
            }
        }
    };
    const int fl = threadIdx.x % TA, jl = threadIdx.x < TA * (L / RB) ? threadIdx.x / TA : 0;
    const int lmask = (1 << A.LB) - 1;
    int it = 0;
    if (!kNoLoad && threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x);
    for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++it) {
        const int64_t r = id / tiles_per_rhs;
        const int col0 = (id % tiles_per_rhs) * TA;
        const int n2l = col0 + fl;
        const int e0 = n2l * jl, eq = n2l * (L / RB);
        const C2<T> t0a = twid_g<T, SIGN>(A.tlo, e0 & lmask), t0b = twid_g<T, SIGN>(A.thi, e0 >> A.LB);
        const C2<T> tqa = twid_g<T, SIGN>(A.tlo, eq & lmask), tqb = twid_g<T, SIGN>(A.thi, eq >> A.LB);
        if ((MODE == 1 ? kPrefetchA1 : kPrefetchA) && threadIdx.x == 0 && id + (int)gridDim.x < ntiles)
            prefetch(id + (int)gridDim.x);
        if (!kNoLoad) mbar_wait(bar, it & 1);
        const T* dsm = reinterpret_cast<const T*>(buf + B * TA);
        auto load = [&](int f, int n1, int, int) -> C2<T> {
            if (MODE == 0) return buf[n1 * TA + f];
            if (n1 >= B && n1 < L - B) return mk<T>(T(0), T(0));
            const C2<T> v = buf[n1 * TA + f];
            const T d = dsm[(n1 < B ? n1 : n1 - (L - 2 * B)) * DW + (col0 & (DW - 1)) + f];
            return mk<T>(d * v.x, d * v.y);
        };
        C2<T> wq, wcur;
        C2<T>* orow = (MODE == 0) ? A.grid + r * A.GS : A.ybuf + r * A.N;
        auto store = [&](int f, int k1, C2<T> v, int m) {
            if (m == 0) {
                wq = cmul<T>(tqa, tqb);
                wcur = cmul<T>(t0a, t0b);
            } else {
                wcur = cmul<T>(wcur, wq);
            }
            orow[(int64_t)k1 * N2 + col0 + f] = cmul<T>(v, wcur);
        };
        const int nxt = id + (int)gridDim.x;
        auto on_free = [&]() {
            if (!kNoLoad && threadIdx.x == 0 && nxt < ntiles) issue(nxt);
        };
        fft_stages_ip<T, SIGN, G, 0, 1, MODE == 1 && HZ>(tws, tws2, buf, load, store, on_free);
    }
}

// Pass B (rows, length L = N2, TF = TB rows per tile, tile layout [f][S]):
//   MODE 0 (inverse): input grid rows, output fhat (kept band times d_c);
//   MODE 1 (adjoint): input ybuf rows, output grid (natural order) + halo.
template <typename T, int SIGN, int MODE, int L>
__global__ void __launch_bounds__(Geo<T, L>::NT, 1)
    k_pass_b(const __grid_constant__ CUtensorMap dmap, const __grid_constant__ CUtensorMap omap, Args<T> A, int BRd,
             int BRo, int ntiles) {
#ifndef INFT_STAGE_B_F
#define INFT_STAGE_B_F 0
#endif
    constexpr bool kStageB = sizeof(T) == 8 || INFT_STAGE_B_F;  // see the store lambda
    extern __shared__ __align__(128) unsigned char smraw[];
    using G = Geo<T, L>;
    constexpr int TB = G::TF, S = G::ST, SW = G::SW;
    constexpr int CE = (int)(sizeof(C2<T>) / 8);
    // MODE 0: the deconvolution factors of the tile's kept outputs, [2 B2][DW] (rows: k2 in
    // [0, B2), then k2 in [N2 - B2, N2)), fetched by TMA while the first stages run
    constexpr int DW = (int)(16 / sizeof(T)) > TB ? (int)(16 / sizeof(T)) : TB;
    const int N1 = A.N1;
    const int64_t half = A.M / 2;
    const int B2 = (int)(half / N1);  // kept k2 rows: [0, B2) and [N2 - B2, N2)
    C2<T>* tile = reinterpret_cast<C2<T>*>(smraw);
    C2<T>* work = tile + 2 * S * TB;
    C2<T>* tws = work + SW * TB;
    T* dsm = reinterpret_cast<T*>(smraw + d_offset<T>(L, S, SW, TB));
    uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + (MODE == 0 ? 2 * B2 * DW : 0));
    const int tiles_per_rhs = N1 / TB;
    const C2<T>* src = (MODE == 0) ? A.grid : A.ybuf;
    const int64_t src_stride = (MODE == 0) ? A.GS : A.N;
    if (threadIdx.x == 0) {
        if (MODE == 0) prefetch_tmap(&dmap);
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < L / kRB; i += blockDim.x) tws[i] = A.tw2[i];
    __syncthreads();
    auto issue = [&](int id, int b) {
        const int64_t r = id / tiles_per_rhs;
        const int row0 = (id % tiles_per_rhs) * TB;
        mbar_arrive_expect_tx(&bars[b], (uint32_t)(sizeof(C2<T>) * L * TB));
        for (int f = 0; f < TB; ++f)
            bulk_g2s(tile + b * S * TB + f * S, src + r * src_stride + (int64_t)(row0 + f) * L,
                     (uint32_t)(sizeof(C2<T>) * L), &bars[b]);
    };
    int it = 0;
    if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++it) {
        const int b = it & 1;
        const int64_t r = id / tiles_per_rhs;
        const int row0 = (id % tiles_per_rhs) * TB;
        if (threadIdx.x == 0) {
            if (id + (int)gridDim.x < ntiles) {
                if (kStageB) bulk_wait_read<0>();  // the previous tile's output store has left b ^ 1
                issue(id + gridDim.x, b ^ 1);
            }
            if (MODE == 0) {
                // d rows [B2, 2 B2) (k2 < B2) and [0, B2) (k2 >= N2 - B2), columns row0 ..
                // the box's inner start must be 16-byte aligned (an unaligned start coordinate
                // faults with "illegal instruction"): start at row0 rounded down to DW
                const int dc0 = row0 & ~(DW - 1);
                mbar_arrive_expect_tx(&bars[2], (uint32_t)(sizeof(T) * DW * 2 * B2));
                for (int q = 0; q < B2; q += BRd) {
                    tma_load_3d(dsm + q * DW, &dmap, dc0, B2 + q, 0, &bars[2]);
                    tma_load_3d(dsm + (B2 + q) * DW, &dmap, dc0, q, 0, &bars[2]);
                }
            }
        }
        mbar_wait(&bars[b], (it >> 1) & 1);
        const C2<T>* tl = tile + b * S * TB;
        C2<T>* grow = A.grid + r * A.GS;
        // complex128: outputs staged in tile[b] (consumed by the first stage) and stored by TMA
        // boxes -- MODE 1 as [k2][TB] (all N2 rows), MODE 0 as [2 B2][TB] (kept rows, d applied);
        // complex64 (16-byte-wide boxes) keeps plain stores (config 5: staging 0.87 ms vs 0.70)
        C2<T>* stg = tile + b * S * TB;
        C2<T>* frow = A.fhat + r * A.M;
        auto load = [&](int f, int n2, int, int) -> C2<T> { return tl[f * S + n2]; };
        // MODE 0 with B2 a multiple of the last stage's span L/kRB (e.g. sigma = 2): whether leg
        // m is kept, its output address and its d slot follow from m alone (warp-uniform tests,
        // one base per thread)
        constexpr int NsL = L / kRB;
        const bool fastband = (B2 % NsL) == 0;
        const int mlo = B2 / NsL;
        const int jl = threadIdx.x / TB, fl = threadIdx.x - (threadIdx.x / TB) * TB;
        const int doff = (row0 & (DW - 1)) + fl;
        auto store = [&](int f, int k2, C2<T> v, int m) {
            const int64_t k = (int64_t)(row0 + f) + (int64_t)N1 * k2;
            if (MODE == 0) {
                if (m == 0) mbar_wait(&bars[2], it & 1);
                int sr;
                if (fastband) {
                    if (m < mlo)
                        sr = jl + m * NsL;
                    else if (m >= kRB - mlo)
                        sr = jl + m * NsL - (L - 2 * B2);
                    else
                        return;
                } else if (k2 < B2) {
                    sr = k2;
                } else if (k2 >= L - B2) {
                    sr = k2 - (L - 2 * B2);
                } else {
                    return;
                }
                const T d = dsm[sr * DW + doff];
                if (kStageB) {
                    stg[sr * TB + f] = mk<T>(d * v.x, d * v.y);
                } else {
                    // fhat column c = k +- ... : staged row sr < B2 <-> fhat row sr + B2, else sr - B2
                    const int64_t c = (int64_t)(sr < B2 ? sr + B2 : sr - B2) * N1 + row0 + f;
                    frow[c] = mk<T>(d * v.x, d * v.y);
                }
            } else {
                if (kStageB)
                    stg[k2 * TB + f] = v;
                else
                    grow[k] = v;
                if (k < A.H) grow[A.N + k] = v;  // the gather's halo copy of the first cells
            }
        };
        cta_fft<T, SIGN, L>(tws, work, load, store);
        fence_proxy_async();  // staged outputs before the TMA store; tile[b] reads before reuse
        __syncthreads();
        if (kStageB && threadIdx.x == 0) {
            if (MODE == 0) {
                // staged rows [0, B2) -> fhat rows [B2, 2 B2); [B2, 2 B2) -> fhat rows [0, B2)
                for (int q = 0; q < B2; q += BRo) {
                    tma_store_3d(&omap, row0 * CE, B2 + q, (int)r, stg + q * TB);
                    tma_store_3d(&omap, row0 * CE, q, (int)r, stg + (B2 + q) * TB);
                }
            } else {
                for (int q = 0; q < L; q += BRo) tma_store_3d(&omap, row0 * CE, q, (int)r, stg + q * TB);
            }
            bulk_commit();
        }
    }
    if (kStageB && threadIdx.x == 0) bulk_wait<0>();
}

// Pass B in place (complex128): one buffer of max(ST TB, SW TB) elements plus the d side
// buffer (MODE 0), two CTAs per SM, plain stores from registers (the staged TMA stores of
// k_pass_b would hold the buffer the next tile lands in).
template <typename T, int SIGN, int MODE, int L, int TE = kTileIP, int RB = kRB>
__global__ void __launch_bounds__(Geo<T, L, TE, RB>::NT, TE == kTileIP ? (RB == 32 ? INFT_R32_MINB : 2) : (TE < kTileIP ? 4 : (RB == 32 ? 2 : 1)))
    k_pass_b_ip(const __grid_constant__ CUtensorMap dmap, const __grid_constant__ CUtensorMap omap, Args<T> A,
                int BRd, int BRo, int ntiles) {
    extern __shared__ __align__(128) unsigned char smraw[];
    using G = Geo<T, L, TE, RB>;
    constexpr int TB = G::TF, S = G::ST, SW = G::SW;
    constexpr int BUF = (S * TB > SW * TB ? S * TB : SW * TB);
    constexpr int DW = (int)(16 / sizeof(T)) > TB ? (int)(16 / sizeof(T)) : TB;
    const int N1 = A.N1;
    const int64_t half = A.M / 2;
    const int B2 = (int)(half / N1);
    C2<T>* buf = reinterpret_cast<C2<T>*>(smraw);
    C2<T>* tws = buf + BUF;
    T* dsm = reinterpret_cast<T*>(smraw + ((sizeof(C2<T>) * (size_t)(BUF + L / RB) + 127) / 128 * 128));
    uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + (MODE == 0 ? 2 * B2 * DW : 0));
    const int tiles_per_rhs = N1 / TB;
    const C2<T>* src = (MODE == 0) ? A.grid : A.ybuf;
    const int64_t src_stride = (MODE == 0) ? A.GS : A.N;
    if (threadIdx.x == 0) {
        if (MODE == 0) prefetch_tmap(&dmap);
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < L / RB; i += blockDim.x) tws[i] = A.tw2[i];
    const C2<T>* tws2 = stage_tab_fill<T, G>(smraw, A.tw2);
    __syncthreads();
    auto issue = [&](int id) {
        const int64_t r = id / tiles_per_rhs;
        const int row0 = (id % tiles_per_rhs) * TB;
        mbar_arrive_expect_tx(&bars[0], (uint32_t)(sizeof(C2<T>) * L * TB));
        for (int f = 0; f < TB; ++f)
            bulk_g2s(buf + f * S, src + r * src_stride + (int64_t)(row0 + f) * L, (uint32_t)(sizeof(C2<T>) * L),
                     &bars[0]);
    };
    auto prefetch = [&](int id) {
        const int64_t r = id / tiles_per_rhs;
        const int row0 = (id % tiles_per_rhs) * TB;
        for (int f = 0; f < TB; ++f)
            bulk_prefetch_l2(src + r * src_stride + (int64_t)(row0 + f) * L, (uint32_t)(sizeof(C2<T>) * L));
    };
    int it = 0;
    if (!kNoLoad && threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x);
    for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++it) {
        const int64_t r = id / tiles_per_rhs;
        const int row0 = (id % tiles_per_rhs) * TB;
        if (MODE == 0 && threadIdx.x == 0) {  // this tile's d factors (the previous tile is done)
            const int dc0 = row0 & ~(DW - 1);
            mbar_arrive_expect_tx(&bars[1], (uint32_t)(sizeof(T) * DW * 2 * B2));
            for (int q = 0; q < B2; q += BRd) {
                tma_load_3d(dsm + q * DW, &dmap, dc0, B2 + q, 0, &bars[1]);
                tma_load_3d(dsm + (B2 + q) * DW, &dmap, dc0, q, 0, &bars[1]);
            }
        }
        if (kPrefetch && threadIdx.x == 0 && id + (int)gridDim.x < ntiles) prefetch(id + (int)gridDim.x);
        if (!kNoLoad) mbar_wait(&bars[0], it & 1);
        C2<T>* grow = A.grid + r * A.GS;
        C2<T>* frow = A.fhat + r * A.M;
        auto load = [&](int f, int n2, int, int) -> C2<T> { return buf[f * S + n2]; };
        constexpr int NsL = L / RB;
        const bool fastband = (B2 % NsL) == 0;
        const int mlo = B2 / NsL;
        const int jl = threadIdx.x / TB, fl = threadIdx.x - (threadIdx.x / TB) * TB;
        const int doff = (row0 & (DW - 1)) + fl;
        auto store = [&](int f, int k2, C2<T> v, int m) {
            const int64_t k = (int64_t)(row0 + f) + (int64_t)N1 * k2;
            if (MODE == 0) {
                if (m == 0) mbar_wait(&bars[1], it & 1);
                int sr;
                if (fastband) {
                    if (m < mlo)
                        sr = jl + m * NsL;
                    else if (m >= RB - mlo)
                        sr = jl + m * NsL - (L - 2 * B2);
                    else
                        return;
                } else if (k2 < B2) {
                    sr = k2;
                } else if (k2 >= L - B2) {
                    sr = k2 - (L - 2 * B2);
                } else {
                    return;
                }
                const T d = dsm[sr * DW + doff];
                const int64_t c = (int64_t)(sr < B2 ? sr + B2 : sr - B2) * N1 + row0 + f;
                frow[c] = mk<T>(d * v.x, d * v.y);
            } else if (kPlainB1) {
                grow[k] = v;
                if (k < A.H) grow[A.N + k] = v;
            } else {
                // staged in the buffer the last stage has just read, [k2][TB], left by TMA store
                // boxes below; the halo copy of the first cells goes straight out
                buf[k2 * TB + f] = v;
                if (k < A.H) grow[A.N + k] = v;
            }
        };
        const int nxt = id + (int)gridDim.x;
        auto on_free = [&]() {
            if (!kNoLoad && (MODE == 0 || kPlainB1) && threadIdx.x == 0 && nxt < ntiles) issue(nxt);
        };
        fft_stages_ip<T, SIGN, G, 0, 1, false>(tws, tws2, buf, load, store, on_free);
        if (MODE == 0 || kPlainB1) {
            __syncthreads();  // every d read of this tile before the next tile's d copy
        } else {
            fence_proxy_async();  // staged outputs before the TMA store
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int q = 0; q < L; q += BRo) tma_store_3d(&omap, row0 * (int)(sizeof(C2<T>) / 8), q, (int)r,
                                                              buf + q * TB);
                bulk_commit();
                bulk_wait_read<0>();  // the store has read the buffer: the next tile may land
                if (nxt < ntiles) issue(nxt);
            }
        }
    }
    if (MODE == 1 && !kPlainB1 && threadIdx.x == 0) bulk_wait<0>();
}

}  // namespace fft

// =========================================================================== host
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

// Per-plan FFT tables; one plan per GPU may be driven from its own host thread, so the map is
// guarded (the state itself belongs to one plan, which the ABI does not share across threads).
static std::mutex g_fft_mu;
static std::map<const Plan*, FftState*>& fft_states() {
    static std::map<const Plan*, FftState*> m;
    return m;
}

template <typename T>
static size_t pass_b_smem(int L, int N1, int64_t M, int mode);

static int split_n1(int64_t N) {
    int lg = 0;
    while ((int64_t(1) << lg) < N) lg++;
    // INFT_FFT_N1_SHIFT=k: N1 = 2^(floor(lg/2) - k) (experiment: wider pass-A column tiles)
    static const int shift = [] {
        const char* e = getenv("INFT_FFT_N1_SHIFT");
        return e ? atoi(e) : 0;
    }();
    const int l1 = std::max(1, lg / 2 - shift);
    return 1 << l1;
}

bool fused_fft_available(const Plan& p) {
    if (p.d != 1) return false;
    const int64_t N = p.Ms[0];
    if (N < 256 || (N & (N - 1)) || N > (int64_t(1) << 24)) return false;
    if (p.GS < N || (p.GS & 1)) return false;
    // pass A of the adjoint fetches whole band rows of h: M/2 must be a multiple of N2
    const int64_t N2 = N / split_n1(N);
    const int64_t half = p.M[0] / 2;
    if (p.M[0] % 2 || half % N2) return false;
    const int64_t B = half / N2;
    if (B > 256 && B % 256) return false;
    // pass A of the adjoint stages d (2B rows x >= 16 bytes) in the tile's unused middle rows
    {
        const int N1 = split_n1(N);
        const int TE = p.prec == INFT_C128 ? fft::tile_elems<double>() : fft::tile_elems<float>();
        const int TF = N1 >= TE / 8 ? std::max(1, TE / N1) : 8;
        const size_t cs = p.prec == INFT_C128 ? 16 : 8, ds = cs / 2;
        const size_t dw = std::max<size_t>((size_t)TF, 16 / ds);
        if ((size_t)(N1 - 2 * B) * TF * cs < (size_t)2 * B * dw * ds) return false;
        // TMA destinations 128-byte aligned
        if (((size_t)B * TF * cs) % 128 || ((size_t)B * dw * ds) % 128) return false;
    }
    // pass B of the inverse stages the tile's d factors: shared memory must fit
    {
        const int64_t B2 = half / split_n1(N);
        const size_t ds = p.prec == INFT_C128 ? 8 : 4;
        const int TE = p.prec == INFT_C128 ? fft::tile_elems<double>() : fft::tile_elems<float>();
        const int TF = N2 >= TE / 8 ? std::max(1, (int)(TE / N2)) : 8;
        const size_t dw = std::max<size_t>((size_t)TF, 16 / ds);
        const size_t smem = p.prec == INFT_C128 ? pass_b_smem<double>((int)N2, split_n1(N), p.M[0], 0)
                                                : pass_b_smem<float>((int)N2, split_n1(N), p.M[0], 0);
        if (smem == 0 || smem > 227 * 1024) return false;
        if (B2 > 256 && B2 % 256) return false;
        if ((B2 * dw * ds) % 128) return false;
        if (((size_t)B2 * TF * 2 * ds) % 128) return false;  // staged output box offsets
    }
    // pass A's TMA box is TF columns wide and must span >= 16 bytes (TF = 1 only for N1 = 4096)
    if (p.prec == INFT_C64 && split_n1(N) >= 4096) return false;
    return true;
}

template <typename T>
static FftState& fft_state(Plan& p, cudaStream_t st) {
    FftState* sp;
    {
        std::lock_guard<std::mutex> g(g_fft_mu);
        FftState*& slot = fft_states()[&p];
        if (!slot) slot = new FftState();
        sp = slot;
    }
    FftState* s = sp;
    if (s->ready) return *s;
    const int64_t N = p.Ms[0];
    int lg = 0;
    while ((int64_t(1) << lg) < N) lg++;
    s->N1 = split_n1(N);         // strided pass (columns)
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
    std::lock_guard<std::mutex> g(g_fft_mu);
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
    A.tw1 = s.tw1.as<C2<T>>();
    A.tw2 = s.tw2.as<C2<T>>();
    A.tlo = s.tlo.as<C2<T>>();
    A.thi = s.thi.as<C2<T>>();
    return A;
}

template <typename T>
using PassAFn = void (*)(const CUtensorMap, const CUtensorMap, fft::Args<T>, int, int);
template <typename T>
using PassBFn = void (*)(const CUtensorMap, const CUtensorMap, fft::Args<T>, int, int, int);

template <typename T, int L>
static void pick_L(int mode, PassAFn<T>& a, PassBFn<T>& b) {
    // mode 0 = inverse NFFT (forward sign), mode 1 = inverse adjoint (inverse sign)
    a = mode == 0 ? fft::k_pass_a<T, -1, 0, L> : fft::k_pass_a<T, 1, 1, L>;
    b = mode == 0 ? fft::k_pass_b<T, -1, 0, L> : fft::k_pass_b<T, 1, 1, L>;
}

template <typename T>
static bool pick_kernels(int mode, int L, PassAFn<T>& a, PassBFn<T>& b, int& TF, int& ST, int& SW, int& NT) {
#define INFT_GEO(LL) TF = fft::Geo<T, LL>::TF, ST = fft::Geo<T, LL>::ST, SW = fft::Geo<T, LL>::SW, NT = fft::Geo<T, LL>::NT
    switch (L) {
        case 16: pick_L<T, 16>(mode, a, b); INFT_GEO(16); return true;
        case 32: pick_L<T, 32>(mode, a, b); INFT_GEO(32); return true;
        case 64: pick_L<T, 64>(mode, a, b); INFT_GEO(64); return true;
        case 128: pick_L<T, 128>(mode, a, b); INFT_GEO(128); return true;
        case 256: pick_L<T, 256>(mode, a, b); INFT_GEO(256); return true;
        case 512: pick_L<T, 512>(mode, a, b); INFT_GEO(512); return true;
        case 1024: pick_L<T, 1024>(mode, a, b); INFT_GEO(1024); return true;
        case 2048: pick_L<T, 2048>(mode, a, b); INFT_GEO(2048); return true;
        case 4096: pick_L<T, 4096>(mode, a, b); INFT_GEO(4096); return true;
    }
#undef INFT_GEO
    return false;
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// dynamic shared memory of pass B (0: unsupported length)
template <typename T>
static size_t pass_b_smem(int L, int N1, int64_t M, int mode) {
    PassAFn<T> ka = nullptr;
    PassBFn<T> kb = nullptr;
    int TB, ST, SW, threads;
    if (!pick_kernels<T>(mode, L, ka, kb, TB, ST, SW, threads)) return 0;
    const int B2 = (int)(M / 2 / N1);
    const int DW = std::max<int>(TB, (int)(16 / sizeof(T)));
    return fft::d_offset<T>(L, ST, SW, TB) + (mode == 0 ? sizeof(T) * (size_t)(2 * B2 * DW) : 0) + 32;
}

// pass B of the inverse in place with 8192-element tiles (INFT_FFT_TILE_B=8192): 4 rows of 2048,
// so each kept output column leaves as a 64-byte run instead of 32 (one CTA per SM)
template <typename T>
static bool pick_ip_b8(int L, PassBFn<T>& b, int& TF, int& ST, int& SW, int& NT, int mode = 0) {
#define INFT_IPG8(LL)                                                                                    \
    TF = fft::Geo<T, LL, 8192>::TF, ST = fft::Geo<T, LL, 8192>::ST, SW = fft::Geo<T, LL, 8192>::SW,      \
    NT = fft::Geo<T, LL, 8192>::NT;                                                                      \
    b = mode == 0 ? fft::k_pass_b_ip<T, -1, 0, LL, 8192> : fft::k_pass_b_ip<T, 1, 1, LL, 8192>;          \
    return true;
    switch (L) {
        case 1024: { INFT_IPG8(1024) }
        case 2048: { INFT_IPG8(2048) }
        default: return false;
    }
#undef INFT_IPG8
}

// complex64 pass B of the inverse in place on 16384-element tiles (128 KB: eight rows of 2048, the
// kept band leaves in 64-byte runs; one 1024-thread CTA per SM at 64 registers): config 5 c64
// 0.464 -> 0.437 ms against the double-buffered 8192-element kernel (INFT_FFT_C64_B0=0: that one).
// The adjoint's pass B measured slower on these tiles (0.460 against 0.431 ms) and keeps it.
template <typename T>
static bool pick_ip_b16f(int L, PassBFn<T>& b, int& TF, int& ST, int& SW, int& NT) {
    if constexpr (sizeof(T) == 4) {
        if (L == 2048) {
            using G = fft::Geo<T, 2048, 16384, 16>;
            TF = G::TF, ST = G::ST, SW = G::SW, NT = G::NT;
            b = fft::k_pass_b_ip<T, -1, 0, 2048, 16384, 16>;
            return true;
        }
    }
    return false;
}

// in-place kernels and their geometry (Geo<T, L, TE>) for the supported lengths; TE = 4096
// (two CTAs per SM) or 2048 (half-size tiles, four CTAs per SM)
template <typename T, int TE, int RB>
static bool pick_ip_te(int mode, int L, bool pass_a, PassAFn<T>& a, PassBFn<T>& b, int& TF, int& ST, int& SW,
                       int& NT, bool hz) {
#define INFT_IPG(LL)                                                                                          \
    TF = fft::Geo<T, LL, TE, RB>::TF, ST = fft::Geo<T, LL, TE, RB>::ST, SW = fft::Geo<T, LL, TE, RB>::SW,     \
    NT = fft::Geo<T, LL, TE, RB>::NT;                                                                         \
    if (pass_a) a = mode == 0 ? fft::k_pass_a_ip<T, -1, 0, LL, TE, RB>                                      \
                              : (hz ? fft::k_pass_a_ip<T, 1, 1, LL, TE, RB, true>                            \
                                    : fft::k_pass_a_ip<T, 1, 1, LL, TE, RB>);                                \
    else b = mode == 0 ? fft::k_pass_b_ip<T, -1, 0, LL, TE, RB> : fft::k_pass_b_ip<T, 1, 1, LL, TE, RB>;        \
    return true;
    switch (L) {
        case 128: { INFT_IPG(128) }
        case 256: { INFT_IPG(256) }
        case 512: { INFT_IPG(512) }
        case 1024: { INFT_IPG(1024) }
        case 2048: { INFT_IPG(2048) }
        case 4096: { INFT_IPG(4096) }
        default: return false;
    }
#undef INFT_IPG
}

// radix of the in-place kernels' bulk stages per pass and direction (INFT_FFT_RB_A0 / _A1 /
// _B0 / _B1 = 16 or 32; pass A / B, mode 0 = inverse, 1 = adjoint)
static int ip_rb(bool pass_a, int mode) {
    static int v[4] = {0, 0, 0, 0};
    static const bool init = [] {
        const char* names[4] = {"INFT_FFT_RB_A0", "INFT_FFT_RB_A1", "INFT_FFT_RB_B0", "INFT_FFT_RB_B1"};
        const int dflt[4] = {16, 32, 16, 16};  // adjoint pass A: radix 32 (config 5: 0.826 -> 0.740 ms)
        for (int i = 0; i < 4; ++i) {
            const char* e = getenv(names[i]);
            v[i] = e && atoi(e) == 32 ? 32 : (e && atoi(e) == 16 ? 16 : dflt[i]);
        }
        return true;
    }();
    (void)init;
    return v[(pass_a ? 0 : 2) + (mode ? 1 : 0)];
}

// complex64 in place: 8192-element tiles (64-byte column runs) with radix-32 stages (256 threads
// at two CTAs per SM).  Pass A by default (config 5 c64: inverse 0.451 -> 0.425 ms, adjoint
// 0.507 -> 0.428 ms; INFT_FFT_IP_C64A=0: double-buffered); pass B only with INFT_FFT_IP_C64=1
// (slower: 0.468 -> 0.512 ms, 0.434 -> 0.487 ms -- three stages for L = 2048)
static bool ip_c64(bool pass_a) {
    static const bool a = [] {
        const char* e = getenv("INFT_FFT_IP_C64A");
        return !(e && atoi(e) == 0);
    }();
    static const bool b = [] {
        const char* e = getenv("INFT_FFT_IP_C64");
        return e && atoi(e);
    }();
    return pass_a ? a : b;
}

template <typename T>
static bool pick_ip(int mode, int L, bool pass_a, PassAFn<T>& a, PassBFn<T>& b, int& TF, int& ST, int& SW, int& NT,
                    int& RB, bool hz = false) {
    if constexpr (sizeof(T) == 4) {
        RB = 32;
        if (L < 1024) return false;
        return pick_ip_te<T, 8192, 32>(mode, L, pass_a, a, b, TF, ST, SW, NT, hz);
    } else {
        RB = ip_rb(pass_a, mode);
        if (RB == 32 && L >= 1024) return pick_ip_te<T, fft::kTileIP, 32>(mode, L, pass_a, a, b, TF, ST, SW, NT, hz);
        RB = fft::kRB;
        return pick_ip_te<T, fft::kTileIP, fft::kRB>(mode, L, pass_a, a, b, TF, ST, SW, NT, hz);
    }
}

// pass A over `src` (MODE 0: the grid, rows GS; MODE 1: h, rows M)
template <typename T>
static void launch_pass_a(Plan& p, fft::Args<T>& A, int mode, const void* src, int64_t R, cudaStream_t st) {
    const size_t cs = sizeof(C2<T>);
    constexpr int CE = (int)(sizeof(C2<T>) / 8);
    const int L = A.N1;
    PassAFn<T> ka = nullptr;
    PassBFn<T> kb = nullptr;
    int TA, ST, SW, threads;
    if (!pick_kernels<T>(mode, L, ka, kb, TA, ST, SW, threads)) {
        set_error("fused FFT: unsupported factor length");
        throw Fail{INFT_ERR_UNSUPPORTED};
    }
    // in-place pass A (two CTAs per SM) unless INFT_FFT_IP=0: its own tile geometry
    static const bool ip = [] {
        const char* e = getenv("INFT_FFT_IP");
        return !(e && atoi(e) == 0);
    }();
    PassAFn<T> kip = nullptr;
    PassBFn<T> kunused = nullptr;
    // complex64: in place with 8192-element radix-32 tiles (ip_c64; the 4096-element in-place
    // tiles were slower than the double-buffered kernel: 3.21 vs 3.06 ms/step)
    int rb = fft::kRB;
    if (ip && (sizeof(T) == 8 || ip_c64(true))) {
        int tf, st_, sw, nt;
        // adjoint with a band of L/4 rows on each side (sigma = 2): first stage skips the zero rows
        // (INFT_FFT_HZ=0: off)
        static const bool hz_on = [] {
            const char* e = getenv("INFT_FFT_HZ");
            return !(e && atoi(e) == 0);
        }();
        const bool hz = hz_on && mode == 1 && A.M / 2 / A.N2 == L / 4;
        if (pick_ip<T>(mode, L, true, kip, kunused, tf, st_, sw, nt, rb, hz)) {
            TA = tf, ST = st_, SW = sw, threads = nt;
        } else {
            kip = nullptr;
        }
    }
    CUtensorMap map, dmap;
    int BR;
    bool ok;
    if (mode == 0) {
        BR = std::min(L, 256);
        ok = make_tmap_3d(&map, src, (uint64_t)A.N2 * CE, (uint64_t)A.N1, (uint64_t)R, cs * (uint64_t)A.N2,
                          cs * (uint64_t)A.GS, (uint32_t)(TA * CE), (uint32_t)BR);
    } else {
        const int B = (int)(A.M / 2 / A.N2);
        BR = std::min(B, 256);
        ok = make_tmap_3d(&map, src, (uint64_t)A.N2 * CE, (uint64_t)(A.M / A.N2), (uint64_t)R, cs * (uint64_t)A.N2,
                          cs * (uint64_t)A.M, (uint32_t)(TA * CE), (uint32_t)BR);
        // deconvolution table d as [M / N2][N2], boxes DW columns wide (>= 16 bytes)
        const int DW = std::max<int>(TA, (int)(16 / sizeof(T)));
        ok = ok && make_tmap_3d(&dmap, A.dk, (uint64_t)A.N2, (uint64_t)(A.M / A.N2), 1, sizeof(T) * (uint64_t)A.N2,
                                sizeof(T) * (uint64_t)A.M, (uint32_t)DW, (uint32_t)BR, (int)sizeof(T));
    }
    if (mode == 0) dmap = map;
    if (!ok) {
        set_error("cuTensorMapEncodeTiled failed (fused FFT pass A)");
        throw Fail{INFT_ERR_CUDA};
    }
    const int ntiles = (int)(R * (A.N2 / TA));
    if (kip) {
        const size_t smem_ip = ((cs * (size_t)(std::max(L * TA, SW * TA) + L / rb) + 16 + 15) & ~(size_t)15) +
                               cs * fft::kStageTabElems;  // + the stage twiddle table at the end
        ensure_smem_attr((const void*)kip, smem_ip);
        const int occ = occupancy_cached((const void*)kip, threads, smem_ip);
        kip<<<(unsigned)std::min(ntiles, num_sms() * std::max(1, occ)), threads, smem_ip, st>>>(map, dmap, A, BR,
                                                                                                 ntiles);
        INFT_CHECK_LAUNCH();
        p.launches++;
        return;
    }
    const size_t smem = cs * (size_t)(2 * L * TA + SW * TA + L / fft::kRB) + 16;
    ensure_smem_attr((const void*)ka, smem);
    const int occ = occupancy_cached((const void*)ka, threads, smem);
    ka<<<(unsigned)std::min(ntiles, num_sms() * std::max(1, occ)), threads, smem, st>>>(map, dmap, A, BR, ntiles);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

template <typename T>
static void launch_pass_b(Plan& p, fft::Args<T>& A, int mode, int64_t R, cudaStream_t st) {
    const size_t cs = sizeof(C2<T>);
    const int L = A.N2;
    PassAFn<T> ka = nullptr;
    PassBFn<T> kb = nullptr;
    int TB, ST, SW, threads;
    if (!pick_kernels<T>(mode, L, ka, kb, TB, ST, SW, threads)) {
        set_error("fused FFT: unsupported factor length");
        throw Fail{INFT_ERR_UNSUPPORTED};
    }
    // in-place pass B for the inverse (MODE 0: plain stores of the kept half; two CTAs per SM)
    // unless INFT_FFT_IP_B=0.  Config 5: 0.854 -> 0.766 ms (0.735 with the L2 prefetch of the
    // next tile).  MODE 1 writes the whole grid + halo, also in place with plain stores and the
    // prefetch (0.883 -> 0.84 ms; round 1 without the prefetch: 0.917, with staged TMA stores
    // -DINFT_FFT_PLAIN_B1=0: 1.0-1.3 ms).
    static const bool ipb = [] {
        const char* e = getenv("INFT_FFT_IP_B");
        return !(e && atoi(e) == 0);
    }();
    // adjoint (MODE 1) in place too: plain stores of the grid and an L2 prefetch of the next
    // tile (config 5: 0.883 -> 0.837 ms against the double-buffered k_pass_b); INFT_FFT_IP_B1=0:
    // the double-buffered kernel
    static const bool ipb1 = [] {
        const char* e = getenv("INFT_FFT_IP_B1");
        return !(e && atoi(e) == 0);
    }();
    PassBFn<T> kip = nullptr;
    int rb = fft::kRB;
    static const int c64_b0 = getenv("INFT_FFT_C64_B0") ? atoi(getenv("INFT_FFT_C64_B0")) : 16384;
    const bool c64big = sizeof(T) == 4 && mode == 0 && c64_b0 == 16384 && L == 2048 &&
                        R * (int64_t)(A.N1 / 8) >= 2 * (int64_t)num_sms();
    if (ipb && (sizeof(T) == 8 || ip_c64(false) || c64big) && (mode == 0 || ipb1)) {
        PassAFn<T> unused = nullptr;
        int tf, st_, sw, nt;
        static const int tile_b = [] {
            const char* e = getenv("INFT_FFT_TILE_B");
            return e ? atoi(e) : 4096;
        }();
        // adjoint (MODE 1), complex128: 8192-element tiles by default -- four rows per tile, so the
        // grid leaves in 64-byte runs instead of 32 (one 512-thread CTA per SM; config 5: 0.849 ->
        // 0.794 ms; the source view had 18 % of this pass's stall samples on its 32-byte-run stores
        // and 15 % in MIO throttle).  INFT_FFT_TILE_B1=4096: two CTAs per SM on 4096-element tiles.
        // The same tiles are slower for the inverse (0.709 -> 0.762 ms, INFT_FFT_TILE_B=8192) and
        // for pass A (0.82 -> 0.83 ms inverse, 0.64 -> 0.83-0.86 ms adjoint).
        static const int tile_b1 = [] {
            const char* e = getenv("INFT_FFT_TILE_B1");
            return e ? atoi(e) : 8192;
        }();
        // (big tiles only when they still give every SM two or more: small batches keep 4096)
        const bool many = L <= 8192 && R * (int64_t)(A.N1 / std::max(1, 8192 / L)) >= 2 * (int64_t)num_sms();
        if (c64big && pick_ip_b16f<T>(L, kip, tf, st_, sw, nt)) {
            TB = tf, ST = st_, SW = sw, threads = nt;
            rb = 16;
        } else if (sizeof(T) == 8 && ((mode == 0 && tile_b == 8192) || (mode == 1 && tile_b1 == 8192 && many)) &&
            pick_ip_b8<T>(L, kip, tf, st_, sw, nt, mode)) {
            TB = tf, ST = st_, SW = sw, threads = nt;
        } else if (pick_ip<T>(mode, L, false, unused, kip, tf, st_, sw, nt, rb)) {
            TB = tf, ST = st_, SW = sw, threads = nt;
        } else {
            kip = nullptr;
        }
    }
    const int B2 = (int)(A.M / 2 / A.N1);
    const int DW = std::max<int>(TB, (int)(16 / sizeof(T)));
    const size_t smem = pass_b_smem<T>(L, A.N1, A.M, mode);
    CUtensorMap dmap;
    const int BRd = std::min(B2, 256);
    if (mode == 0) {
        // deconvolution table d as [M / N1][N1]: row k2', column k1
        if (!make_tmap_3d(&dmap, A.dk, (uint64_t)A.N1, (uint64_t)(A.M / A.N1), 1, sizeof(T) * (uint64_t)A.N1,
                          sizeof(T) * (uint64_t)A.M, (uint32_t)DW, (uint32_t)BRd, (int)sizeof(T))) {
            set_error("cuTensorMapEncodeTiled failed (fused FFT pass B)");
            throw Fail{INFT_ERR_CUDA};
        }
    } else {
        memset(&dmap, 0, sizeof(dmap));
    }
    // output boxes: MODE 0 -> fhat viewed as [R][M / N1][N1] (kept rows), MODE 1 -> the grid
    // viewed as [R][N2][N1] (row k2, column k1 of k = k1 + N1 k2)
    constexpr int CE = (int)(sizeof(C2<T>) / 8);
    CUtensorMap omap;
    const int BRo = mode == 0 ? std::min(B2, 256) : std::min(L, 256);
    const bool ok = mode == 0
                        ? make_tmap_3d(&omap, A.fhat, (uint64_t)A.N1 * CE, (uint64_t)(A.M / A.N1), (uint64_t)R,
                                       cs * (uint64_t)A.N1, cs * (uint64_t)A.M, (uint32_t)(TB * CE), (uint32_t)BRo)
                        : make_tmap_3d(&omap, A.grid, (uint64_t)A.N1 * CE, (uint64_t)A.N2, (uint64_t)R,
                                       cs * (uint64_t)A.N1, cs * (uint64_t)A.GS, (uint32_t)(TB * CE), (uint32_t)BRo);
    if (!ok) {
        set_error("cuTensorMapEncodeTiled failed (fused FFT pass B output)");
        throw Fail{INFT_ERR_CUDA};
    }
    const int ntiles = (int)(R * (A.N1 / TB));
    if (kip) {
        const size_t head = (cs * (size_t)(std::max(ST * TB, SW * TB) + L / rb) + 127) / 128 * 128;
        const size_t smem_ip = ((head + (mode == 0 ? sizeof(T) * (size_t)(2 * B2 * DW) : 0) + 32 + 15) & ~(size_t)15) +
                               cs * fft::kStageTabElems;  // + the stage twiddle table at the end
        ensure_smem_attr((const void*)kip, smem_ip);  // <= ~150 KB for L <= 4096
        const int occ = occupancy_cached((const void*)kip, threads, smem_ip);
        kip<<<(unsigned)std::min(ntiles, num_sms() * std::max(1, occ)), threads, smem_ip, st>>>(dmap, omap, A, BRd,
                                                                                                 BRo, ntiles);
        INFT_CHECK_LAUNCH();
        p.launches++;
        return;
    }
    ensure_smem_attr((const void*)kb, smem);
    const int occ = occupancy_cached((const void*)kb, threads, smem);
    kb<<<(unsigned)std::min(ntiles, num_sms() * std::max(1, occ)), threads, smem, st>>>(dmap, omap, A, BRd, BRo,
                                                                                        ntiles);
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
static void fused_inverse_t(Plan& p, void* grid, void* fhat, int64_t R, cudaStream_t st, int part) {
    FftState& s = fft_state<T>(p, st);
    fft::Args<T> A = make_args<T>(p, s);
    A.grid = static_cast<C2<T>*>(grid);
    A.fhat = static_cast<C2<T>*>(fhat);
    A.dk = dtab_for<T>(p);
    if (part & 1) launch_pass_a<T>(p, A, 0, grid, R, st);
    if (part & 2) launch_pass_b<T>(p, A, 0, R, st);
}

// adjoint: h -> grid (D, zero pad, F), natural order with halo
template <typename T>
static void fused_adjoint_t(Plan& p, const void* h, void* grid, int64_t R, cudaStream_t st, int part) {
    FftState& s = fft_state<T>(p, st);
    if (s.y_rhs < R) {
        s.ybuf.alloc(sizeof(C2<T>) * (size_t)p.Ms[0] * R);
        s.y_rhs = R;
        p.state_version++;
    }
    fft::Args<T> A = make_args<T>(p, s);
    A.grid = static_cast<C2<T>*>(grid);
    A.ybuf = s.ybuf.as<C2<T>>();
    A.hin = static_cast<const C2<T>*>(h);
    A.dk = dtab_for<T>(p);
    if (part & 1) launch_pass_a<T>(p, A, 1, h, R, st);
    if (part & 2) launch_pass_b<T>(p, A, 1, R, st);
}

void fused_fft_inverse(Plan& p, void* grid, void* fhat, int64_t R, cudaStream_t st, int part) {
    if (p.prec == INFT_C128)
        fused_inverse_t<double>(p, grid, fhat, R, st, part);
    else
        fused_inverse_t<float>(p, grid, fhat, R, st, part);
}

void fused_fft_adjoint(Plan& p, const void* h, void* grid, int64_t R, cudaStream_t st, int part) {
    if (p.prec == INFT_C128)
        fused_adjoint_t<double>(p, h, grid, R, st, part);
    else
        fused_adjoint_t<float>(p, h, grid, R, st, part);
}

}  // namespace inft
