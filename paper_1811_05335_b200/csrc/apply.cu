// Apply stage on sm_100a.
//
//   inverse NFFT          fhat = s D^* F^* B_opt^* f
//       a2 spread  g = B_opt^* f        (register-window kernel, no atomics)
//       a3 FFT     ghat = F^* g         (cuFFT, forward sign)
//       a4 trunc   fhat_k = d_k ghat_{k mod M_sigma}
//   inverse adjoint NFFT  f = s B_opt F D h
//       a5 pad     ghat_{k mod M_sigma} = d_k h_k, 0 elsewhere
//       a6 FFT     g = F ghat           (cuFFT, inverse sign, unnormalised)
//       a7 gather  f_j = sum_t w_{j,t} g_{(l0_j + t) mod M_sigma}
//
// Grid vectors live in FFT order n = l mod M_sigma (reading A9); spectra are
// centered (c = k + M/2).  s is folded into d (reading A2).
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "inft_internal.cuh"

namespace inft {

template <typename T>
struct C2T;
template <>
struct C2T<double> {
    using type = double2;
};
template <>
struct C2T<float> {
    using type = float2;
};
template <typename T>
using C2 = typename C2T<T>::type;

template <typename T>
__device__ __forceinline__ C2<T> mk(T x, T y) {
    C2<T> v;
    v.x = x;
    v.y = y;
    return v;
}

__device__ __forceinline__ int64_t mod64(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

static inline unsigned blocks_for(int64_t n, int bs) { return (unsigned)std::max<int64_t>(1, ceil_div(n, bs)); }

// ---------------------------------------------------------------- uniform weight loads
// Load the P real weights of one sorted node record (16-byte aligned, padded to PP)
// with vector loads; every lane of the warp reads the same address (broadcast).
template <typename T, int P>
struct WeightLoader;

template <int P>
struct WeightLoader<double, P> {
    __device__ __forceinline__ static void load(const double* __restrict__ rec, double (&w)[P]) {
        const double2* v = reinterpret_cast<const double2*>(rec);
#pragma unroll
        for (int q = 0; q < (P + 1) / 2; ++q) {
            double2 a = __ldg(v + q);
            w[2 * q] = a.x;
            if (2 * q + 1 < P) w[2 * q + 1] = a.y;
        }
    }
};

template <int P>
struct WeightLoader<float, P> {
    __device__ __forceinline__ static void load(const float* __restrict__ rec, float (&w)[P]) {
        const float4* v = reinterpret_cast<const float4*>(rec);
#pragma unroll
        for (int q = 0; q < (P + 3) / 4; ++q) {
            float4 a = __ldg(v + q);
            w[4 * q] = a.x;
            if (4 * q + 1 < P) w[4 * q + 1] = a.y;
            if (4 * q + 2 < P) w[4 * q + 2] = a.z;
            if (4 * q + 3 < P) w[4 * q + 3] = a.w;
        }
    }
};

#define INFT_CASES_32(X) \
    X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
    X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31)

// ====================================================================== a2: spread
// Register-window spread, 1-D, real weights.
// A warp owns a chunk of Q consecutive grid segments (width SEG >= 2m) for 32
// right-hand sides (lane = RHS).  Nodes are bin-sorted, so the nodes of a
// segment are a contiguous range and their slot base n0 lies in the segment:
// a node adds w[t] f_j to window register delta+t, delta = n0 - seg*SEG (a
// warp-uniform switch makes every register index static).  After a segment,
// window[0, SEG) is complete (all nodes with n0 in [n - 2m, n] have been seen)
// and is stored once; window[SEG, SEG + 2m) is carried.  The chunk starts one
// segment early (prologue) to collect the carry from its left neighbour.
// No atomics, deterministic order, every grid point written exactly once.
template <typename T, int MC, int SEG>
__global__ void __launch_bounds__(128) k_spread_fast_1d(
    const int32_t* __restrict__ seg_start, const int32_t* __restrict__ delta, const int32_t* __restrict__ perm,
    int perm_identity, const T* __restrict__ w, int PP, const C2<T>* __restrict__ f, C2<T>* __restrict__ grid,
    int64_t N, int64_t Ms, int nseg, int Q, int nchunks, int R, int nrg) {
    constexpr int P = 2 * MC + 1;
    constexpr int K = SEG + 2 * MC;
    static_assert(SEG >= 2 * MC && SEG <= 32, "segment must cover the support");
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (gw >= (int64_t)nchunks * nrg) return;
    const int chunk = (int)(gw / nrg);
    const int rg = (int)(gw - (int64_t)chunk * nrg);
    const int r = rg * 32 + lane;
    const bool active = r < R;
    const C2<T>* __restrict__ fr = f + (int64_t)(active ? r : 0) * N;
    C2<T>* __restrict__ gr = grid + (int64_t)(active ? r : 0) * Ms;

    T ax[K], ay[K];
#pragma unroll
    for (int u = 0; u < K; ++u) ax[u] = ay[u] = T(0);

    const int s0 = chunk * Q;
    const int s1 = min(s0 + Q, nseg);
    for (int si = s0 - 1; si < s1; ++si) {
        const int s = si < 0 ? si + nseg : si;
        const int i0 = __ldg(seg_start + s), i1 = __ldg(seg_start + s + 1);
        for (int i = i0; i < i1; ++i) {
            const int dl = __ldg(delta + i);
            const int64_t j = perm_identity ? (int64_t)i : (int64_t)__ldg(perm + i);
            C2<T> fv = mk<T>(T(0), T(0));
            if (active) fv = __ldg(fr + j);
            T wv[P];
            WeightLoader<T, P>::load(w + (int64_t)i * PP, wv);
            switch (dl) {
#define INFT_SPREAD_CASE(D)                                       \
    case D:                                                       \
        if constexpr (D < SEG) {                                  \
            _Pragma("unroll") for (int t = 0; t < P; ++t) {       \
                ax[D + t] = fma(wv[t], fv.x, ax[D + t]);          \
                ay[D + t] = fma(wv[t], fv.y, ay[D + t]);          \
            }                                                     \
        }                                                         \
        break;
                INFT_CASES_32(INFT_SPREAD_CASE)
#undef INFT_SPREAD_CASE
                default:
                    break;
            }
        }
        if (si >= s0 && active) {
            C2<T>* out = gr + (int64_t)s * SEG;
#pragma unroll
            for (int u = 0; u < SEG; ++u) out[u] = mk<T>(ax[u], ay[u]);
        }
#pragma unroll
        for (int u = 0; u < K; ++u) {
            ax[u] = (u + SEG < K) ? ax[u + SEG] : T(0);
            ay[u] = (u + SEG < K) ? ay[u + SEG] : T(0);
        }
    }
}

// Generic spread (any m, any d = 1 layout, real or complex weights, aliasing
// 2m+1 > M_sigma): one thread per (grid point n, RHS r) sums
// conj(w_{j,t}) f_j over the nodes of the segments covering n-2m..n.
template <typename T, bool WC>
__global__ void k_spread_generic_1d(const int32_t* __restrict__ seg_start, const int32_t* __restrict__ n0s,
                                    const int32_t* __restrict__ perm, const T* __restrict__ w, int PP, int P,
                                    const C2<T>* __restrict__ f, C2<T>* __restrict__ grid, int64_t N, int64_t Ms,
                                    int S, int R) {
    const int64_t total = (int64_t)R * Ms;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / Ms;
        const int64_t n = idx - r * Ms;
        const C2<T>* fr = f + r * N;
        T sx = 0, sy = 0;
        int64_t span = std::min<int64_t>(P, Ms);
        int64_t pos = mod64(n - (span - 1), Ms);
        int64_t rem = span;
        while (rem > 0) {
            int64_t s = pos / S;
            int64_t send = std::min<int64_t>((s + 1) * S, Ms);
            int64_t len = std::min<int64_t>(send - pos, rem);
            for (int i = seg_start[s]; i < seg_start[s + 1]; ++i) {
                int64_t t = mod64(n - n0s[i], Ms);
                if (t >= P) continue;
                C2<T> fv = fr[perm[i]];
                for (; t < P; t += Ms) {
                    if (WC) {
                        T wr = w[((int64_t)i * PP + t) * 2], wi = w[((int64_t)i * PP + t) * 2 + 1];
                        sx += wr * fv.x + wi * fv.y;  // conj(w) f
                        sy += wr * fv.y - wi * fv.x;
                    } else {
                        T wr = w[(int64_t)i * PP + t];
                        sx += wr * fv.x;
                        sy += wr * fv.y;
                    }
                }
            }
            rem -= len;
            pos += len;
            if (pos == Ms) pos = 0;
        }
        grid[idx] = mk<T>(sx, sy);
    }
}

// Generic 2-D spread (tensor slots t = t1*P1 + t2, grid n = n1*Ms2 + n2).
template <typename T, bool WC>
__global__ void k_spread_generic_2d(const int32_t* __restrict__ seg_start, const int32_t* __restrict__ n0s,
                                    const int32_t* __restrict__ perm, const T* __restrict__ w, int PP, int P1,
                                    const C2<T>* __restrict__ f, C2<T>* __restrict__ grid, int64_t N, int64_t Ms1,
                                    int64_t Ms2, int S1, int S2, int64_t nseg2, int R) {
    const int64_t Mst = Ms1 * Ms2;
    const int64_t total = (int64_t)R * Mst;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / Mst;
        const int64_t n = idx - r * Mst;
        const int64_t n1 = n / Ms2, n2 = n - (n / Ms2) * Ms2;
        const C2<T>* fr = f + r * N;
        T sx = 0, sy = 0;
        int64_t span1 = std::min<int64_t>(P1, Ms1), span2 = std::min<int64_t>(P1, Ms2);
        int64_t pos1 = mod64(n1 - (span1 - 1), Ms1), rem1 = span1;
        while (rem1 > 0) {
            int64_t s1 = pos1 / S1;
            int64_t len1 = std::min<int64_t>(std::min<int64_t>((s1 + 1) * S1, Ms1) - pos1, rem1);
            int64_t pos2 = mod64(n2 - (span2 - 1), Ms2), rem2 = span2;
            while (rem2 > 0) {
                int64_t s2 = pos2 / S2;
                int64_t len2 = std::min<int64_t>(std::min<int64_t>((s2 + 1) * S2, Ms2) - pos2, rem2);
                int64_t tile = s1 * nseg2 + s2;
                for (int i = seg_start[tile]; i < seg_start[tile + 1]; ++i) {
                    int64_t t1 = mod64(n1 - n0s[2 * i], Ms1);
                    int64_t t2b = mod64(n2 - n0s[2 * i + 1], Ms2);
                    if (t1 >= P1 || t2b >= P1) continue;
                    C2<T> fv = fr[perm[i]];
                    for (; t1 < P1; t1 += Ms1)
                        for (int64_t t2 = t2b; t2 < P1; t2 += Ms2) {
                            int64_t t = t1 * P1 + t2;
                            if (WC) {
                                T wr = w[((int64_t)i * PP + t) * 2], wi = w[((int64_t)i * PP + t) * 2 + 1];
                                sx += wr * fv.x + wi * fv.y;
                                sy += wr * fv.y - wi * fv.x;
                            } else {
                                T wr = w[(int64_t)i * PP + t];
                                sx += wr * fv.x;
                                sy += wr * fv.y;
                            }
                        }
                }
                rem2 -= len2;
                pos2 += len2;
                if (pos2 == Ms2) pos2 = 0;
            }
            rem1 -= len1;
            pos1 += len1;
            if (pos1 == Ms1) pos1 = 0;
        }
        grid[idx] = mk<T>(sx, sy);
    }
}

// ====================================================================== a7: gather
// Register-window gather, 1-D, real weights: lane = RHS, the warp walks the
// segments of its chunk keeping grid window [seg*SEG, seg*SEG + SEG + 2m) in
// registers (2m carried, SEG loaded per segment); each node reads its P taps
// from the window with static indices (warp-uniform switch on delta).
template <typename T, int MC, int SEG>
__global__ void __launch_bounds__(128) k_gather_fast_1d(
    const int32_t* __restrict__ seg_start, const int32_t* __restrict__ delta, const int32_t* __restrict__ perm,
    int perm_identity, const T* __restrict__ w, int PP, const C2<T>* __restrict__ grid, C2<T>* __restrict__ f,
    int64_t N, int64_t Ms, int nseg, int Q, int nchunks, int R, int nrg) {
    constexpr int P = 2 * MC + 1;
    constexpr int K = SEG + 2 * MC;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (gw >= (int64_t)nchunks * nrg) return;
    const int chunk = (int)(gw / nrg);
    const int rg = (int)(gw - (int64_t)chunk * nrg);
    const int r = rg * 32 + lane;
    const bool active = r < R;
    const C2<T>* __restrict__ gr = grid + (int64_t)(active ? r : 0) * Ms;
    C2<T>* __restrict__ fr = f + (int64_t)(active ? r : 0) * N;

    T wx[K], wy[K];
    const int s0 = chunk * Q;
    const int s1 = min(s0 + Q, nseg);
    for (int s = s0; s < s1; ++s) {
        const int64_t base = (int64_t)s * SEG;
        if (s == s0) {
#pragma unroll
            for (int u = 0; u < K; ++u) {
                int64_t q = base + u;
                if (q >= Ms) q -= Ms;
                C2<T> v = active ? __ldg(gr + q) : mk<T>(T(0), T(0));
                wx[u] = v.x;
                wy[u] = v.y;
            }
        } else {
#pragma unroll
            for (int u = 0; u < K; ++u) {
                if (u + SEG < K) {
                    wx[u] = wx[u + SEG];
                    wy[u] = wy[u + SEG];
                } else {
                    int64_t q = base + u;
                    if (q >= Ms) q -= Ms;
                    C2<T> v = active ? __ldg(gr + q) : mk<T>(T(0), T(0));
                    wx[u] = v.x;
                    wy[u] = v.y;
                }
            }
        }
        const int i0 = __ldg(seg_start + s), i1 = __ldg(seg_start + s + 1);
        for (int i = i0; i < i1; ++i) {
            const int dl = __ldg(delta + i);
            const int64_t j = perm_identity ? (int64_t)i : (int64_t)__ldg(perm + i);
            T wv[P];
            WeightLoader<T, P>::load(w + (int64_t)i * PP, wv);
            T sx = 0, sy = 0;
            switch (dl) {
#define INFT_GATHER_CASE(D)                                   \
    case D:                                                   \
        if constexpr (D < SEG) {                              \
            _Pragma("unroll") for (int t = 0; t < P; ++t) {   \
                sx = fma(wv[t], wx[D + t], sx);               \
                sy = fma(wv[t], wy[D + t], sy);               \
            }                                                 \
        }                                                     \
        break;
                INFT_CASES_32(INFT_GATHER_CASE)
#undef INFT_GATHER_CASE
                default:
                    break;
            }
            if (active) fr[j] = mk<T>(sx, sy);
        }
    }
}

// Generic gather: one thread per (sorted node i, RHS r).
template <typename T, bool WC>
__global__ void k_gather_generic(const int32_t* __restrict__ n0s, const int32_t* __restrict__ perm,
                                 const T* __restrict__ w, int PP, int P1, int d, const C2<T>* __restrict__ grid,
                                 C2<T>* __restrict__ f, int64_t N, int64_t Ms1, int64_t Ms2, int R) {
    const int64_t Mst = Ms1 * (d == 2 ? Ms2 : 1);
    const int64_t total = (int64_t)R * N;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / N;
        const int64_t i = idx - r * N;
        const C2<T>* gr = grid + r * Mst;
        T sx = 0, sy = 0;
        const int P2 = d == 2 ? P1 : 1;
        const int64_t a1 = n0s[(int64_t)i * d];
        const int64_t a2 = d == 2 ? n0s[(int64_t)i * d + 1] : 0;
        for (int t1 = 0; t1 < P1; ++t1) {
            int64_t q1 = a1 + t1;
            while (q1 >= Ms1) q1 -= Ms1;
            for (int t2 = 0; t2 < P2; ++t2) {
                int64_t q = q1;
                if (d == 2) {
                    int64_t q2 = a2 + t2;
                    while (q2 >= Ms2) q2 -= Ms2;
                    q = q1 * Ms2 + q2;
                }
                const int64_t t = (int64_t)t1 * P2 + t2;
                C2<T> g = gr[q];
                if (WC) {
                    T wr = w[((int64_t)i * PP + t) * 2], wi = w[((int64_t)i * PP + t) * 2 + 1];
                    sx += wr * g.x - wi * g.y;
                    sy += wr * g.y + wi * g.x;
                } else {
                    T wr = w[(int64_t)i * PP + t];
                    sx += wr * g.x;
                    sy += wr * g.y;
                }
            }
        }
        f[r * N + perm[i]] = mk<T>(sx, sy);
    }
}

// ====================================================================== a4 / a5: deconvolution
// a4: fhat[r][c] = d1[c1] d2[c2] ghat[r][q], q_i = (c_i - M_i/2) mod Ms_i.
template <typename T>
__global__ void k_trunc_deconv(const C2<T>* __restrict__ grid, C2<T>* __restrict__ fhat, const T* __restrict__ dk,
                               int64_t M1, int64_t M2, int64_t Ms1, int64_t Ms2, int d, int R) {
    const int64_t Mt = M1 * M2, Mst = Ms1 * Ms2;
    const int64_t total = (int64_t)R * Mt;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / Mt;
        const int64_t c = idx - r * Mt;
        int64_t q;
        T dd;
        if (d == 1) {
            int64_t k = c - M1 / 2;
            q = k < 0 ? k + Ms1 : k;
            dd = dk[c];
        } else {
            int64_t c1 = c / M2, c2 = c - (c / M2) * M2;
            int64_t k1 = c1 - M1 / 2, k2 = c2 - M2 / 2;
            q = (k1 < 0 ? k1 + Ms1 : k1) * Ms2 + (k2 < 0 ? k2 + Ms2 : k2);
            dd = dk[c1] * dk[M1 + c2];
        }
        C2<T> g = grid[r * Mst + q];
        fhat[idx] = mk<T>(dd * g.x, dd * g.y);
    }
}

// a5: ghat[r][q] = d_k h[r][k + M/2] for |k| <= M/2 band, 0 elsewhere.
template <typename T>
__global__ void k_deconv_pad(const C2<T>* __restrict__ h, C2<T>* __restrict__ grid, const T* __restrict__ dk,
                             int64_t M1, int64_t M2, int64_t Ms1, int64_t Ms2, int d, int R) {
    const int64_t Mt = M1 * M2, Mst = Ms1 * Ms2;
    const int64_t total = (int64_t)R * Mst;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / Mst;
        const int64_t q = idx - r * Mst;
        C2<T> out = mk<T>(T(0), T(0));
        if (d == 1) {
            int64_t k = q < Ms1 / 2 ? q : q - Ms1;
            if (k >= -M1 / 2 && k < M1 / 2) {
                T dd = dk[k + M1 / 2];
                C2<T> v = h[r * Mt + k + M1 / 2];
                out = mk<T>(dd * v.x, dd * v.y);
            }
        } else {
            int64_t q1 = q / Ms2, q2 = q - (q / Ms2) * Ms2;
            int64_t k1 = q1 < Ms1 / 2 ? q1 : q1 - Ms1;
            int64_t k2 = q2 < Ms2 / 2 ? q2 : q2 - Ms2;
            if (k1 >= -M1 / 2 && k1 < M1 / 2 && k2 >= -M2 / 2 && k2 < M2 / 2) {
                T dd = dk[k1 + M1 / 2] * dk[M1 + k2 + M2 / 2];
                C2<T> v = h[r * Mt + (k1 + M1 / 2) * M2 + (k2 + M2 / 2)];
                out = mk<T>(dd * v.x, dd * v.y);
            }
        }
        grid[idx] = out;
    }
}

// ====================================================================== host orchestration
static constexpr int kQ = 32;  // segments per warp chunk

template <typename T>
using SpreadFastFn = void (*)(const int32_t*, const int32_t*, const int32_t*, int, const T*, int, const C2<T>*,
                              C2<T>*, int64_t, int64_t, int, int, int, int, int);
template <typename T>
using GatherFastFn = void (*)(const int32_t*, const int32_t*, const int32_t*, int, const T*, int, const C2<T>*,
                              C2<T>*, int64_t, int64_t, int, int, int, int, int);

template <typename T>
static SpreadFastFn<T> spread_fast_for(int m, int S) {
#define INFT_SF(MC, SG) \
    if (m == MC && S == SG) return k_spread_fast_1d<T, MC, SG>;
    INFT_SF(1, 16) INFT_SF(2, 16) INFT_SF(3, 16) INFT_SF(4, 16) INFT_SF(5, 16) INFT_SF(6, 16) INFT_SF(7, 16)
    INFT_SF(8, 16) INFT_SF(10, 32) INFT_SF(12, 32) INFT_SF(16, 32)
#undef INFT_SF
    return nullptr;
}

template <typename T>
static GatherFastFn<T> gather_fast_for(int m, int S) {
#define INFT_GF(MC, SG) \
    if (m == MC && S == SG) return k_gather_fast_1d<T, MC, SG>;
    INFT_GF(1, 16) INFT_GF(2, 16) INFT_GF(3, 16) INFT_GF(4, 16) INFT_GF(5, 16) INFT_GF(6, 16) INFT_GF(7, 16)
    INFT_GF(8, 16) INFT_GF(10, 32) INFT_GF(12, 32) INFT_GF(16, 32)
#undef INFT_GF
    return nullptr;
}

static unsigned sm_blocks(int per_sm = 8) {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (nsm <= 0) nsm = 148;
    }
    return (unsigned)(nsm * per_sm);
}

static unsigned gs_blocks(int64_t total, int bs) {
    return (unsigned)std::min<int64_t>(blocks_for(total, bs), (int64_t)sm_blocks(16));
}

static bool use_fast(const Plan& p) {
    if (!p.fast1d || p.wt != INFT_WEIGHTS_REAL) return false;
    return p.prec == INFT_C128 ? spread_fast_for<double>(p.m, p.S[0]) != nullptr
                               : spread_fast_for<float>(p.m, p.S[0]) != nullptr;
}

template <typename T>
static void spread(Plan& p, const C2<T>* f, C2<T>* grid, int64_t R, cudaStream_t st) {
    const T* w = p.w.as<T>();
    if (p.d == 1 && use_fast(p)) {
        int nseg = (int)p.nseg[0];
        int nchunks = (int)ceil_div(nseg, kQ);
        int nrg = (int)ceil_div(R, 32);
        int64_t warps = (int64_t)nchunks * nrg;
        spread_fast_for<T>(p.m, p.S[0])<<<blocks_for(warps * 32, 128), 128, 0, st>>>(
            p.seg_start.as<int32_t>(), p.delta.as<int32_t>(), p.perm.as<int32_t>(), p.perm_identity ? 1 : 0, w,
            p.PP, f, grid, p.N, p.Ms[0], nseg, kQ, nchunks, (int)R, nrg);
    } else if (p.d == 1) {
        int64_t total = R * p.Ms[0];
        if (p.wt == INFT_WEIGHTS_COMPLEX)
            k_spread_generic_1d<T, true><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P, f, grid, p.N,
                p.Ms[0], p.S[0], (int)R);
        else
            k_spread_generic_1d<T, false><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P, f, grid, p.N,
                p.Ms[0], p.S[0], (int)R);
    } else {
        int64_t total = R * p.Mstot;
        if (p.wt == INFT_WEIGHTS_COMPLEX)
            k_spread_generic_2d<T, true><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P1, f, grid, p.N,
                p.Ms[0], p.Ms[1], p.S[0], p.S[1], p.nseg[1], (int)R);
        else
            k_spread_generic_2d<T, false><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P1, f, grid, p.N,
                p.Ms[0], p.Ms[1], p.S[0], p.S[1], p.nseg[1], (int)R);
    }
    INFT_CHECK_LAUNCH();
    p.launches++;
}

template <typename T>
static void gather(Plan& p, const C2<T>* grid, C2<T>* f, int64_t R, cudaStream_t st) {
    if (p.N == 0) return;
    const T* w = p.w.as<T>();
    if (p.d == 1 && use_fast(p)) {
        int nseg = (int)p.nseg[0];
        int nchunks = (int)ceil_div(nseg, kQ);
        int nrg = (int)ceil_div(R, 32);
        int64_t warps = (int64_t)nchunks * nrg;
        gather_fast_for<T>(p.m, p.S[0])<<<blocks_for(warps * 32, 128), 128, 0, st>>>(
            p.seg_start.as<int32_t>(), p.delta.as<int32_t>(), p.perm.as<int32_t>(), p.perm_identity ? 1 : 0, w,
            p.PP, grid, f, p.N, p.Ms[0], nseg, kQ, nchunks, (int)R, nrg);
    } else {
        int64_t total = R * p.N;
        if (p.wt == INFT_WEIGHTS_COMPLEX)
            k_gather_generic<T, true><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P1, p.d, grid, f, p.N, p.Ms[0], p.Ms[1],
                (int)R);
        else
            k_gather_generic<T, false><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P1, p.d, grid, f, p.N, p.Ms[0], p.Ms[1],
                (int)R);
    }
    INFT_CHECK_LAUNCH();
    p.launches++;
}

static void ensure_grid(Plan& p, int64_t rhs) {
    if (p.grid_rhs >= rhs && p.grid.p) return;
    p.grid.alloc((size_t)rhs * p.Mstot * p.elem_bytes());
    p.grid_rhs = rhs;
}

static int64_t grid_capacity(Plan& p, int64_t want) {
    if (p.grid_rhs >= want) return want;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    size_t budget = std::min<size_t>(fr / 3, (size_t)8 << 30);
    int64_t cap = std::max<int64_t>(1, (int64_t)(budget / ((size_t)p.Mstot * p.elem_bytes())));
    cap = std::max<int64_t>(cap, p.grid_rhs);
    return std::min<int64_t>(want, cap);
}

static cufftHandle fft_plan(Plan& p, int batch) {
    auto it = p.fft.find(FftKey{batch});
    if (it != p.fft.end()) return it->second;
    cufftHandle h;
    int n[2] = {(int)p.Ms[0], (int)p.Ms[1]};
    cufftType ty = p.prec == INFT_C128 ? CUFFT_Z2Z : CUFFT_C2C;
    INFT_CUFFT(cufftPlanMany(&h, p.d, n, nullptr, 1, (int)p.Mstot, nullptr, 1, (int)p.Mstot, ty, batch));
    p.fft[FftKey{batch}] = h;
    return h;
}

static void fft_exec(Plan& p, void* grid, int batch, int dir, cudaStream_t st) {
    cufftHandle h = fft_plan(p, batch);
    INFT_CUFFT(cufftSetStream(h, st));
    if (p.prec == INFT_C128)
        INFT_CUFFT(cufftExecZ2Z(h, (cufftDoubleComplex*)grid, (cufftDoubleComplex*)grid, dir));
    else
        INFT_CUFFT(cufftExecC2C(h, (cufftComplex*)grid, (cufftComplex*)grid, dir));
}

template <typename T>
static const T* dtable(const Plan& p);
template <>
const double* dtable<double>(const Plan& p) {
    return p.dk.as<double>();
}
template <>
const float* dtable<float>(const Plan& p) {
    return p.dkf.as<float>();
}

// RAII stage timer: CUDA events on the launching stream around one stage.
struct StageTimer {
    Plan& p;
    int stage;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    StageTimer(Plan& pp, int sg, cudaStream_t s) : p(pp), stage(sg), st(s) {
        if (p.profiling) {
            a = p.take_event();
            INFT_CUDA(cudaEventRecord(a, st));
        }
    }
    ~StageTimer() {
        if (a) {
            cudaEvent_t b = p.take_event();
            cudaEventRecord(b, st);
            p.recs.push_back(Plan::Rec{stage, a, b});
            if (p.recs.size() > 4096) p.drain_profile();
        }
    }
};

// One device-resident chunk (Rc <= grid capacity) of the inverse: a2 -> a3 -> a4.
template <typename T>
static void inverse_chunk(Plan& p, const void* f, void* fhat, int64_t Rc, cudaStream_t st) {
    ensure_grid(p, Rc);
    C2<T>* g = p.grid.as<C2<T>>();
    {
        StageTimer t(p, 0, st);
        spread<T>(p, static_cast<const C2<T>*>(f), g, Rc, st);
    }
    {
        StageTimer t(p, 1, st);
        fft_exec(p, g, (int)Rc, CUFFT_FORWARD, st);
    }
    StageTimer t(p, 2, st);
    int64_t total = Rc * p.Mtot;
    k_trunc_deconv<T><<<gs_blocks(total, 256), 256, 0, st>>>(g, static_cast<C2<T>*>(fhat), dtable<T>(p), p.M[0],
                                                             p.d == 2 ? p.M[1] : 1, p.Ms[0],
                                                             p.d == 2 ? p.Ms[1] : 1, p.d, (int)Rc);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

// One chunk of the inverse adjoint: a5 -> a6 -> a7.
template <typename T>
static void adjoint_chunk(Plan& p, const void* h, void* f, int64_t Rc, cudaStream_t st) {
    ensure_grid(p, Rc);
    C2<T>* g = p.grid.as<C2<T>>();
    int64_t total = Rc * p.Mstot;
    {
        StageTimer t(p, 3, st);
        k_deconv_pad<T><<<gs_blocks(total, 256), 256, 0, st>>>(static_cast<const C2<T>*>(h), g, dtable<T>(p), p.M[0],
                                                               p.d == 2 ? p.M[1] : 1, p.Ms[0],
                                                               p.d == 2 ? p.Ms[1] : 1, p.d, (int)Rc);
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    {
        StageTimer t(p, 4, st);
        fft_exec(p, g, (int)Rc, CUFFT_INVERSE, st);
    }
    StageTimer t(p, 5, st);
    gather<T>(p, g, static_cast<C2<T>*>(f), Rc, st);
}

using ChunkFn = void (*)(Plan&, const void*, void*, int64_t, cudaStream_t);

static void ensure_streams(Plan& p) {
    if (p.s_h2d) return;
    INFT_CUDA(cudaStreamCreateWithFlags(&p.s_h2d, cudaStreamNonBlocking));
    INFT_CUDA(cudaStreamCreateWithFlags(&p.s_d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++) {
        INFT_CUDA(cudaEventCreateWithFlags(&p.ev_h2d[i], cudaEventDisableTiming));
        INFT_CUDA(cudaEventCreateWithFlags(&p.ev_comp[i], cudaEventDisableTiming));
        INFT_CUDA(cudaEventCreateWithFlags(&p.ev_d2h[i], cudaEventDisableTiming));
    }
    INFT_CUDA(cudaEventCreateWithFlags(&p.ev_entry, cudaEventDisableTiming));
    INFT_CUDA(cudaEventCreateWithFlags(&p.ev_exit, cudaEventDisableTiming));
}

// Device-resident path: chunks of the grid capacity.  Host path: double-buffered
// staging; H2D of chunk c+1 (stream s_h2d) and D2H of chunk c-1 (stream s_d2h)
// overlap the compute of chunk c on the caller's stream.
static void run(Plan& p, const void* in, size_t in_rhs_bytes, void* out, size_t out_rhs_bytes, int64_t R,
                cudaStream_t st, ChunkFn fn) {
    const bool in_dev = in_rhs_bytes == 0 || is_device_pointer(in);
    const bool out_dev = out_rhs_bytes == 0 || is_device_pointer(out);
    const char* ib = static_cast<const char*>(in);
    char* ob = static_cast<char*>(out);
    if (in_dev && out_dev) {
        int64_t cap = grid_capacity(p, R);
        for (int64_t r0 = 0; r0 < R; r0 += cap) {
            int64_t rc = std::min(cap, R - r0);
            fn(p, ib + r0 * in_rhs_bytes, ob + r0 * out_rhs_bytes, rc, st);
        }
        return;
    }
    ensure_streams(p);
    size_t per = std::max(in_dev ? 0 : in_rhs_bytes, out_dev ? 0 : out_rhs_bytes);
    int64_t Rh = std::max<int64_t>(1, std::min<int64_t>(R, (int64_t)(((size_t)256 << 20) / std::max<size_t>(per, 1))));
    Rh = grid_capacity(p, Rh);
    if (!in_dev && p.stage_in_bytes < in_rhs_bytes * Rh) {
        for (int i = 0; i < 2; i++) p.stage_in[i].alloc(in_rhs_bytes * Rh);
        p.stage_in_bytes = in_rhs_bytes * Rh;
    }
    if (!out_dev && p.stage_out_bytes < out_rhs_bytes * Rh) {
        for (int i = 0; i < 2; i++) p.stage_out[i].alloc(out_rhs_bytes * Rh);
        p.stage_out_bytes = out_rhs_bytes * Rh;
    }
    INFT_CUDA(cudaEventRecord(p.ev_entry, st));
    INFT_CUDA(cudaStreamWaitEvent(p.s_h2d, p.ev_entry, 0));
    INFT_CUDA(cudaStreamWaitEvent(p.s_d2h, p.ev_entry, 0));
    const int64_t nchunk = ceil_div(R, Rh);
    for (int64_t c = 0; c < nchunk; c++) {
        const int b = (int)(c & 1);
        const int64_t r0 = c * Rh, rc = std::min(Rh, R - r0);
        const void* src = in_dev ? (const void*)(ib + r0 * in_rhs_bytes) : p.stage_in[b].p;
        void* dst = out_dev ? (void*)(ob + r0 * out_rhs_bytes) : p.stage_out[b].p;
        if (!in_dev) {
            if (c >= 2) INFT_CUDA(cudaStreamWaitEvent(p.s_h2d, p.ev_comp[b], 0));
            INFT_CUDA(cudaMemcpyAsync(p.stage_in[b].p, ib + r0 * in_rhs_bytes, rc * in_rhs_bytes,
                                      cudaMemcpyHostToDevice, p.s_h2d));
            INFT_CUDA(cudaEventRecord(p.ev_h2d[b], p.s_h2d));
            INFT_CUDA(cudaStreamWaitEvent(st, p.ev_h2d[b], 0));
        }
        if (!out_dev && c >= 2) INFT_CUDA(cudaStreamWaitEvent(st, p.ev_d2h[b], 0));
        fn(p, src, dst, rc, st);
        INFT_CUDA(cudaEventRecord(p.ev_comp[b], st));
        if (!out_dev) {
            INFT_CUDA(cudaStreamWaitEvent(p.s_d2h, p.ev_comp[b], 0));
            INFT_CUDA(cudaMemcpyAsync(ob + r0 * out_rhs_bytes, p.stage_out[b].p, rc * out_rhs_bytes,
                                      cudaMemcpyDeviceToHost, p.s_d2h));
            INFT_CUDA(cudaEventRecord(p.ev_d2h[b], p.s_d2h));
        }
    }
    if (!out_dev) {
        INFT_CUDA(cudaEventRecord(p.ev_exit, p.s_d2h));
        INFT_CUDA(cudaStreamWaitEvent(st, p.ev_exit, 0));
    }
    // staging buffers are reused by the next call: make the caller's stream own the tail
    INFT_CUDA(cudaEventRecord(p.ev_exit, p.s_h2d));
    INFT_CUDA(cudaStreamWaitEvent(st, p.ev_exit, 0));
}

void apply_inverse(Plan& p, const void* f, void* fhat, int64_t R, cudaStream_t st) {
    const size_t e = p.elem_bytes();
    ChunkFn fn = p.prec == INFT_C128 ? (ChunkFn)inverse_chunk<double> : (ChunkFn)inverse_chunk<float>;
    run(p, f, (size_t)p.N * e, fhat, (size_t)p.Mtot * e, R, st, fn);
}

void apply_adjoint(Plan& p, const void* h, void* f, int64_t R, cudaStream_t st) {
    const size_t e = p.elem_bytes();
    ChunkFn fn = p.prec == INFT_C128 ? (ChunkFn)adjoint_chunk<double> : (ChunkFn)adjoint_chunk<float>;
    run(p, h, (size_t)p.Mtot * e, f, (size_t)p.N * e, R, st, fn);
}

}  // namespace inft
