// Apply stage on sm_100a: orchestration, generic kernels
// and the deconvolution passes.
//
//   inverse NFFT          fhat = s D^* F^* B_opt^* f
//       a2 spread  g = B_opt^* f        (stream1d.cu: staged register-window kernel)
//       a3 FFT     ghat = F^* g         (cuFFT, forward sign)
//       a4 trunc   fhat_k = d_k ghat_{k mod M_sigma}
//   inverse adjoint NFFT  f = s B_opt F D h
//       a5 pad     ghat_{k mod M_sigma} = d_k h_k, 0 elsewhere
//       a6 FFT     g = F ghat           (cuFFT, inverse sign, unnormalised)
//       a7 gather  f_j = sum_t w_{j,t} g_{(l0_j + t) mod M_sigma}
//
// Grid vectors live in FFT order n = l mod M_sigma (reading A9), one row per
// RHS with row stride GS >= M_sigma (1-D fast path: a 2m halo at the end);
// spectra are centered (c = k + M/2).  s is folded into d (reading A2).
#include <algorithm>
#include <cstring>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "inft_internal.cuh"
#include "tma.cuh"

namespace inft {

static inline unsigned blocks_for(int64_t n, int bs) { return (unsigned)std::max<int64_t>(1, ceil_div(n, bs)); }

// Generic spread (any m, any d = 1 layout, real or complex weights, aliasing
// 2m+1 > M_sigma): one thread per (grid point n, RHS r) sums
// conj(w_{j,t}) f_j over the nodes of the segments covering n-2m..n.
template <typename T, bool WC>
__global__ void k_spread_generic_1d(const int32_t* __restrict__ seg_start, const int32_t* __restrict__ n0s,
                                    const int32_t* __restrict__ perm, const T* __restrict__ w, int PP, int P,
                                    const C2<T>* __restrict__ f, C2<T>* __restrict__ grid, int64_t N, int64_t Ms,
                                    int64_t GS, int S, int R) {
    const int64_t total = (int64_t)R * Ms;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / Ms;
        const int64_t n = idx - r * Ms;
        const C2<T>* fr = f + r * N;
        T sx = 0, sy = 0;
        const int64_t nseg = (Ms + S - 1) / S;
        for_segments(n, std::min<int64_t>(P, Ms), Ms, S, nseg, [&](int64_t s) {
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
        });
        grid[r * GS + n] = mk<T>(sx, sy);
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
        const int64_t nseg1 = (Ms1 + S1 - 1) / S1;
        for_segments(n1, std::min<int64_t>(P1, Ms1), Ms1, S1, nseg1, [&](int64_t s1) {
            for_segments(n2, std::min<int64_t>(P1, Ms2), Ms2, S2, nseg2, [&](int64_t s2) {
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
            });
        });
        grid[idx] = mk<T>(sx, sy);
    }
}

// 2-D spread, output-stationary, one warp per (grid cell n, 32 RHS): the warp walks the
// candidate nodes of the (up to 2 x 2) tiles whose nodes can reach n -- a warp-uniform loop,
// so the slot test, the weight and the node record are shared by the 32 lanes -- and lane r
// accumulates w_{j,t} f_r(x_j) for its RHS from the node-major copy fT[i][r] (one coalesced
// 32-lane read per node).  Every grid value is written once: no atomics, deterministic.
template <typename T>
__global__ void k_transpose_f(const C2<T>* __restrict__ f, const int32_t* __restrict__ perm, C2<T>* __restrict__ fT,
                              int64_t N, int R, int RS) {
    const int64_t total = (int64_t)N * R;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx / R;
        const int r = (int)(idx - i * R);
        fT[i * RS + r] = f[(int64_t)r * N + perm[i]];
    }
}

template <typename T, bool WC>
__global__ void k_spread_2d_warp(const int32_t* __restrict__ seg_start, const int32_t* __restrict__ n0s,
                                 const T* __restrict__ w, int PP, int P1, const C2<T>* __restrict__ fT,
                                 C2<T>* __restrict__ grid, int64_t Ms1, int64_t Ms2, int S1, int S2, int64_t nseg2,
                                 int R, int64_t GS) {
    const int lane = threadIdx.x & 31;
    const int64_t wid0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nrc = (R + 31) >> 5;
    const int64_t Mst = Ms1 * Ms2;
    const int64_t nseg1 = (Ms1 + S1 - 1) / S1;
    for (int64_t wid = wid0; wid < Mst * nrc; wid += nwarps) {
        const int64_t n = wid / nrc;
        const int r = (int)(wid - n * nrc) * 32 + lane;
        const bool active = r < R;
        const int64_t n1 = n / Ms2, n2 = n - (n / Ms2) * Ms2;
        T sx = 0, sy = 0;
        for_segments(n1, std::min<int64_t>(P1, Ms1), Ms1, S1, nseg1, [&](int64_t s1) {
            for_segments(n2, std::min<int64_t>(P1, Ms2), Ms2, S2, nseg2, [&](int64_t s2) {
                const int64_t tile = s1 * nseg2 + s2;
                const int i1 = __ldg(seg_start + tile + 1);
                for (int i = __ldg(seg_start + tile); i < i1; ++i) {
                    int64_t t1 = mod64(n1 - __ldg(n0s + 2 * i), Ms1);
                    const int64_t t2b = mod64(n2 - __ldg(n0s + 2 * i + 1), Ms2);
                    if (t1 >= P1 || t2b >= P1) continue;
                    const C2<T> fv = active ? fT[(int64_t)i * R + r] : mk<T>(T(0), T(0));
                    for (; t1 < P1; t1 += Ms1)
                        for (int64_t t2 = t2b; t2 < P1; t2 += Ms2) {
                            const int64_t t = t1 * P1 + t2;
                            if (WC) {
                                const T wr = __ldg(w + ((int64_t)i * PP + t) * 2), wi = __ldg(w + ((int64_t)i * PP + t) * 2 + 1);
                                sx += wr * fv.x + wi * fv.y;
                                sy += wr * fv.y - wi * fv.x;
                            } else {
                                const T wr = __ldg(w + (int64_t)i * PP + t);
                                sx = fma(wr, fv.x, sx);
                                sy = fma(wr, fv.y, sy);
                            }
                        }
                }
            });
        });
        if (active) grid[(int64_t)r * GS + n] = mk<T>(sx, sy);
    }
}

// 2-D spread, tile-stationary (16 x 16 cells, P1 = 2m+1 <= 16): CTA = one output tile x 32
// RHS, 8 warps; warp w owns cell rows w and w + 8 of the tile, lane = RHS, and keeps those
// 2 x 16 accumulators in registers.  The warps walk the nodes of the 2 x 2 tiles whose nodes can reach
// the tile (warp-uniform loop: node record, row test and weights shared by the lanes); a node
// adds its row slice w[t1][0..P1) f_r to the row, the column offset dispatched by a
// warp-uniform switch so that every register index is static.  Each grid value is written
// once: no atomics, deterministic.  f is read from the node-major copy fT[i][r].
template <typename T, int P1, int C>
__device__ __forceinline__ void row_add(T (&ax)[16], T (&ay)[16], const T* wr, C2<T> fv) {
#pragma unroll
    for (int t2 = 0; t2 < P1; ++t2) {
        constexpr int lo = C < 0 ? -C : 0;  // first tap inside the tile
        if (t2 >= lo && C + t2 < 16) {
            const int col = (C + t2) < 0 ? 0 : ((C + t2) > 15 ? 15 : (C + t2));
            const T wv = wr[t2];
            ax[col] = fma(wv, fv.x, ax[col]);
            ay[col] = fma(wv, fv.y, ay[col]);
        }
    }
}

// warp-uniform column-offset dispatch c in [-(P1-1), 15] -> static register indices
template <typename T, int P1>
__device__ __forceinline__ void row_dispatch(int c, T (&ax)[16], T (&ay)[16], const T* wr, C2<T> fv) {
#define INFT_ROW_CASE(CC)                                   \
    case CC:                                                \
        if constexpr ((CC) > -P1) row_add<T, P1, CC>(ax, ay, wr, fv); \
        break;
    switch (c) {
        INFT_ROW_CASE(-15) INFT_ROW_CASE(-14) INFT_ROW_CASE(-13) INFT_ROW_CASE(-12) INFT_ROW_CASE(-11)
        INFT_ROW_CASE(-10) INFT_ROW_CASE(-9) INFT_ROW_CASE(-8) INFT_ROW_CASE(-7) INFT_ROW_CASE(-6)
        INFT_ROW_CASE(-5) INFT_ROW_CASE(-4) INFT_ROW_CASE(-3) INFT_ROW_CASE(-2) INFT_ROW_CASE(-1)
        INFT_ROW_CASE(0) INFT_ROW_CASE(1) INFT_ROW_CASE(2) INFT_ROW_CASE(3) INFT_ROW_CASE(4) INFT_ROW_CASE(5)
        INFT_ROW_CASE(6) INFT_ROW_CASE(7) INFT_ROW_CASE(8) INFT_ROW_CASE(9) INFT_ROW_CASE(10) INFT_ROW_CASE(11)
        INFT_ROW_CASE(12) INFT_ROW_CASE(13) INFT_ROW_CASE(14) INFT_ROW_CASE(15)
        default: break;
    }
#undef INFT_ROW_CASE
}

// Node batches of kB2 records are staged in shared memory, double-buffered: the batch's
// weights (one contiguous run of kB2 * PP values) by one 1-D bulk copy, its f values (kB2 x 32
// RHS) and slot bases by per-thread cp.async, all issued one batch ahead so that the warps
// only ever read shared memory in the node loop.
// nodes per batch and CTAs per SM: complex128 24 nodes, 2 CTAs/SM (config 4 spread 1.44 ->
// 1.34 ms against 48 nodes, 1 CTA/SM); complex64 48 nodes, 1 CTA/SM (0.93 vs 1.05 ms)
template <typename T>
constexpr int kB2T = sizeof(T) == 8 ? 24 : 48;
template <typename T>
constexpr int kMinB2d = sizeof(T) == 8 ? 2 : 1;

template <typename T>
__host__ __device__ constexpr size_t tile2d_stage_bytes(int PP) {
    constexpr int kB2 = kB2T<T>;
    return ((sizeof(C2<T>) * kB2 * 32 + sizeof(int2) * kB2 + sizeof(T) * (size_t)kB2 * PP) + 127) / 128 * 128;
}

template <typename T, int MC>
__global__ void __launch_bounds__(256, kMinB2d<T>) k_spread_2d_tile(const int4* __restrict__ work,
                                                        const int32_t* __restrict__ seg_start,
                                                        const int32_t* __restrict__ n0s, const T* __restrict__ w,
                                                        int PP, const C2<T>* __restrict__ fT, C2<T>* __restrict__ grid,
                                                        C2<T>* __restrict__ part, int Ms1, int Ms2, int nseg1,
                                                        int nseg2, int R, int64_t GS) {
    constexpr int P1 = 2 * MC + 1;
    constexpr int kB2 = kB2T<T>;
    extern __shared__ __align__(128) unsigned char sm2[];
    __shared__ uint64_t full[2];
    __shared__ int tlo[4], thi[4], tnb[5];  // candidate tile ranges, batch prefix counts
    const size_t stage_bytes = tile2d_stage_bytes<T>(PP);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // work item: (tile, first batch, end batch, partial-sum slot or -1): heavy tiles' batch lists
    // are split over several CTAs whose partial tiles k_spread_2d_combine adds up
    const int4 wk = work[blockIdx.x];
    const int s1 = wk.x / nseg2, s2 = wk.x - (wk.x / nseg2) * nseg2;
    const int row0 = s1 * 16, col0 = s2 * 16;
    const int rbase = blockIdx.y * 32;
    const int r = rbase + lane;
    const bool active = r < R;
    if (threadIdx.x == 0) {
        tnb[0] = 0;
        for (int tq = 0; tq < 4; ++tq) {
            const int d1 = (tq >> 1) - 1, d2 = (tq & 1) - 1;
            const int t1s = s1 + d1 < 0 ? s1 + d1 + nseg1 : s1 + d1;
            const int t2s = s2 + d2 < 0 ? s2 + d2 + nseg2 : s2 + d2;
            const int tile = t1s * nseg2 + t2s;
            tlo[tq] = __ldg(seg_start + tile);
            thi[tq] = __ldg(seg_start + tile + 1);
            tnb[tq + 1] = tnb[tq] + (thi[tq] - tlo[tq] + kB2 - 1) / kB2;
        }
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int bfirst = wk.y, bend = min(wk.z, tnb[4]);
    auto batch = [&](int b, int& base, int& nb) {
        int tq = 0;
        while (b >= tnb[tq + 1]) ++tq;
        base = tlo[tq] + (b - tnb[tq]) * kB2;
        nb = min(kB2, thi[tq] - base);
    };
    auto issue = [&](int b) {
        int base, nb;
        batch(b, base, nb);
        unsigned char* sb = sm2 + (size_t)(b & 1) * stage_bytes;
        C2<T>* fsm = reinterpret_cast<C2<T>*>(sb);
        int2* rec = reinterpret_cast<int2*>(fsm + kB2 * 32);
        T* wsm = reinterpret_cast<T*>(rec + kB2);
        if (threadIdx.x == 0) {
            const uint32_t wb = (uint32_t)(sizeof(T) * (size_t)nb * PP);
            mbar_arrive_expect_tx(&full[b & 1], wb);
            bulk_g2s(wsm, w + (int64_t)base * PP, wb, &full[b & 1]);
        }
        for (int e = threadIdx.x; e < nb * 32; e += blockDim.x) {
            const int j = e >> 5, l = e & 31;
            const bool ok = rbase + l < R;
            cp_async<(int)sizeof(C2<T>)>(fsm + e, fT + (int64_t)(base + j) * R + (ok ? rbase + l : 0),
                                         ok ? (int)sizeof(C2<T>) : 0);
        }
        for (int j = threadIdx.x; j < nb; j += blockDim.x) cp_async<8>(rec + j, n0s + 2 * (base + j), 8);
        cp_async_commit();
    };
    T ax[2][16], ay[2][16];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int c = 0; c < 16; ++c) ax[q][c] = ay[q][c] = T(0);
    // rows warp and warp + 8 of the tile: a node's 13-row footprint then spreads its work over
    // all warps (balanced batches between the barriers)
    const int myrow = row0 + warp;
    if (bfirst < bend) issue(bfirst);
#pragma unroll 1
    for (int b = bfirst; b < bend; ++b) {
        if (b + 1 < bend) {
            issue(b + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        mbar_wait(&full[b & 1], (b >> 1) & 1);
        __syncthreads();  // every thread's cp.async data of batch b visible
        int base, nb;
        batch(b, base, nb);
        const unsigned char* sb = sm2 + (size_t)(b & 1) * stage_bytes;
        const C2<T>* fsm = reinterpret_cast<const C2<T>*>(sb);
        const int2* rec = reinterpret_cast<const int2*>(fsm + kB2 * 32);
        const T* wsm = reinterpret_cast<const T*>(rec + kB2);
#pragma unroll 1
        for (int j = 0; j < nb; ++j) {
            const int2 a = rec[j];
            int dr = myrow - a.x;  // t1 of my first row (mod Ms1)
            if (dr < 0) dr += Ms1;
            if (dr >= Ms1) dr -= Ms1;
            int dr2 = dr + 8;
            if (dr2 >= Ms1) dr2 -= Ms1;
            if (dr >= P1 && dr2 >= P1) continue;
            int c = a.y - col0;  // column of tap 0 relative to the tile, in [-(P1-1), 15]
            if (c > 15) c -= Ms2;
            if (c < -(P1 - 1)) c += Ms2;
            const C2<T> fv = fsm[j * 32 + lane];
            const T* wj = wsm + j * PP;
            if (dr < P1) row_dispatch<T, P1>(c, ax[0], ay[0], wj + dr * P1, fv);
            if (dr2 < P1) row_dispatch<T, P1>(c, ax[1], ay[1], wj + dr2 * P1, fv);
        }
        fence_proxy_async();  // reads of this stage precede the bulk copy that reuses it
        __syncthreads();
    }
    if (active) {
        // whole tile: straight into the grid; partial tile: into its slot, [slot][R][16][16]
        C2<T>* g = wk.w < 0 ? grid + (int64_t)r * GS + (int64_t)myrow * Ms2 + col0
                            : part + (((int64_t)wk.w * R + r) * 16 + warp) * 16;
        const int64_t ld = wk.w < 0 ? Ms2 : 16;
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int c = 0; c < 16; ++c) g[(int64_t)q * 8 * ld + c] = mk<T>(ax[q][c], ay[q][c]);
    }
}

// Sum of the partial tiles of the heavy tiles: item (tile, first slot, slots).
template <typename T>
__global__ void k_spread_2d_combine(const int4* __restrict__ items, const C2<T>* __restrict__ part,
                                    C2<T>* __restrict__ grid, int Ms2, int nseg2, int R, int64_t GS) {
    const int4 it = items[blockIdx.x];
    const int s1 = it.x / nseg2, s2 = it.x - (it.x / nseg2) * nseg2;
    for (int e = threadIdx.x; e < R * 256; e += blockDim.x) {
        const int r = e >> 8, cell = e & 255;
        T sx = 0, sy = 0;
        for (int k = 0; k < it.z; ++k) {
            const C2<T> v = part[((int64_t)(it.y + k) * R + r) * 256 + cell];
            sx += v.x;
            sy += v.y;
        }
        grid[(int64_t)r * GS + (int64_t)(s1 * 16 + (cell >> 4)) * Ms2 + s2 * 16 + (cell & 15)] = mk<T>(sx, sy);
    }
}

template <typename T>
using Tile2dFn = void (*)(const int4*, const int32_t*, const int32_t*, const T*, int, const C2<T>*, C2<T>*, C2<T>*,
                          int, int, int, int, int, int64_t);

template <typename T>
static Tile2dFn<T> tile2d_fn(int m) {
    switch (m) {
        case 1: return k_spread_2d_tile<T, 1>;
        case 2: return k_spread_2d_tile<T, 2>;
        case 3: return k_spread_2d_tile<T, 3>;
        case 4: return k_spread_2d_tile<T, 4>;
        case 5: return k_spread_2d_tile<T, 5>;
        case 6: return k_spread_2d_tile<T, 6>;
        case 7: return k_spread_2d_tile<T, 7>;
    }
    return nullptr;
}

// Spread work list: one item per tile, or several for a tile whose 2 x 2 neighbourhood holds
// more than kSplitBatches node batches (partial tiles + combine items); built once per plan.
static int split_batches() {
    static const int v = [] {
        const char* e = getenv("INFT_SPLIT2D");
        const int x = e ? atoi(e) : 0;
        return x > 0 ? x : 24;  // config 4: 4 -> 1.95 ms, 8 -> 1.60, 12 -> 1.51, 24 -> 1.48
    }();
    return v;
}

static void ensure_spread2d_work(Plan& p, cudaStream_t st) {
    if (p.work2d_n >= 0) return;
    std::vector<int32_t> ss((size_t)p.nseg_tot + 1);
    INFT_CUDA(cudaMemcpyAsync(ss.data(), p.seg_start.p, sizeof(int32_t) * ss.size(), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    const int n1 = (int)p.nseg[0], n2 = (int)p.nseg[1];
    const int kB2 = p.prec == INFT_C128 ? kB2T<double> : kB2T<float>;
    std::vector<int4> work, comb;
    int slots = 0;
    for (int t = 0; t < n1 * n2; ++t) {
        const int s1 = t / n2, s2 = t % n2;
        int nb = 0;
        for (int tq = 0; tq < 4; ++tq) {
            const int a = (s1 + (tq >> 1) - 1 + n1) % n1, b = (s2 + (tq & 1) - 1 + n2) % n2;
            const int tt = a * n2 + b;
            nb += (ss[tt + 1] - ss[tt] + kB2 - 1) / kB2;
        }
        const int kSplitBatches = split_batches();
        const int parts = std::max(1, (nb + kSplitBatches - 1) / kSplitBatches);
        if (parts == 1) {
            work.push_back(make_int4(t, 0, 1 << 30, -1));
        } else {
            comb.push_back(make_int4(t, slots, parts, 0));
            for (int q = 0; q < parts; ++q) work.push_back(make_int4(t, q * kSplitBatches, (q + 1) * kSplitBatches, slots + q));
            slots += parts;
        }
    }
    p.work2d.alloc(sizeof(int4) * std::max<size_t>(1, work.size()));
    INFT_CUDA(cudaMemcpyAsync(p.work2d.p, work.data(), sizeof(int4) * work.size(), cudaMemcpyHostToDevice, st));
    p.comb2d.alloc(sizeof(int4) * std::max<size_t>(1, comb.size()));
    if (!comb.empty())
        INFT_CUDA(cudaMemcpyAsync(p.comb2d.p, comb.data(), sizeof(int4) * comb.size(), cudaMemcpyHostToDevice, st));
    p.work2d_n = (int64_t)work.size();
    p.comb2d_n = (int64_t)comb.size();
    p.slots2d = slots;
    INFT_CUDA(cudaStreamSynchronize(st));
}

static bool tile2d_available(const Plan& p) {
    return p.d == 2 && p.wt == INFT_WEIGHTS_REAL && p.m >= 1 && p.m <= 7 && p.S[0] == 16 && p.S[1] == 16 &&
           p.Ms[0] % 16 == 0 && p.Ms[1] % 16 == 0 && p.nseg[0] >= 2 && p.nseg[1] >= 2 &&
           !getenv_flag("INFT_SPREAD2D_WARP");
}

// Generic gather: one thread per (sorted node i, RHS r).
template <typename T, bool WC>
__global__ void k_gather_generic(const int32_t* __restrict__ n0s, const int32_t* __restrict__ perm,
                                 const T* __restrict__ w, int PP, int P1, int d, const C2<T>* __restrict__ grid,
                                 C2<T>* __restrict__ f, int64_t N, int64_t Ms1, int64_t Ms2, int64_t GS, int R) {
    const int64_t total = (int64_t)R * N;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / N;
        const int64_t i = idx - r * N;
        const C2<T>* gr = grid + r * GS;
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
                               int64_t M1, int64_t M2, int64_t Ms1, int64_t Ms2, int64_t GS, int d, int R) {
    const int64_t Mt = M1 * M2;
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
        C2<T> g = grid[r * GS + q];
        fhat[idx] = mk<T>(dd * g.x, dd * g.y);
    }
}

// a5: ghat[r][q] = d_k h[r][k + M/2] for |k| <= M/2 band, 0 elsewhere.
template <typename T>
__global__ void k_deconv_pad(const C2<T>* __restrict__ h, C2<T>* __restrict__ grid, const T* __restrict__ dk,
                             int64_t M1, int64_t M2, int64_t Ms1, int64_t Ms2, int64_t GS, int d, int R) {
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
        grid[r * GS + q] = out;
    }
}

// ====================================================================== host orchestration
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

template <typename T>
static void spread(Plan& p, const C2<T>* f, C2<T>* grid, int64_t R, cudaStream_t st) {
    if (ring_spread_available(p)) {
        spread_ring(p, f, grid, R, st);
        return;
    }
    if (stream1d_available(p)) {
        spread_stream1d(p, f, grid, R, st);
        return;
    }
    const T* w = p.w.as<T>();
    if (p.d == 1) {
        int64_t total = R * p.Ms[0];
        if (p.wt == INFT_WEIGHTS_COMPLEX)
            k_spread_generic_1d<T, true><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P, f, grid, p.N,
                p.Ms[0], p.GS, p.S[0], (int)R);
        else
            k_spread_generic_1d<T, false><<<gs_blocks(total, 256), 256, 0, st>>>(
                p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w, p.PP, p.P, f, grid, p.N,
                p.Ms[0], p.GS, p.S[0], (int)R);
    } else if (!getenv_flag("INFT_SPREAD2D_GENERIC")) {
        // node-major copy of f (sorted node order), then the line kernel (or the tile kernel, or one
        // warp per cell); the line kernel's bulk copies of f rows need 16-byte aligned row starts,
        // so its row stride is R rounded up to 16 bytes
        const bool line = line2d_available(p);
        const int64_t RS = line ? ceil_div(R * (int64_t)sizeof(C2<T>), 16) * 16 / (int64_t)sizeof(C2<T>) : R;
        if (p.fT_rhs < RS) {
            p.fT.alloc(sizeof(C2<T>) * (size_t)p.N * RS);
            p.fT_rhs = RS;
            p.state_version++;
        }
        C2<T>* fT = p.fT.as<C2<T>>();
        k_transpose_f<T><<<gs_blocks(R * p.N, 256), 256, 0, st>>>(f, p.perm.as<int32_t>(), fT, p.N, (int)R, (int)RS);
        INFT_CHECK_LAUNCH();
        p.launches++;
        if (line) {
            spread_line2d(p, fT, grid, R, (int)RS, st);
            return;
        }
        if (tile2d_available(p)) {
            ensure_spread2d_work(p, st);
            if (p.part2d_rhs < R && p.slots2d > 0) {
                p.part2d.alloc(sizeof(C2<T>) * (size_t)p.slots2d * R * 256);
                p.part2d_rhs = R;
                p.state_version++;
            }
            dim3 g((unsigned)p.work2d_n, (unsigned)ceil_div(R, 32));
            const size_t smem = 2 * tile2d_stage_bytes<T>(p.PP);
            ensure_smem_attr((const void*)tile2d_fn<T>(p.m), smem);
            tile2d_fn<T>(p.m)<<<g, 256, smem, st>>>(p.work2d.as<int4>(), p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(),
                                                 w, p.PP, fT, grid, p.part2d.as<C2<T>>(), (int)p.Ms[0],
                                                 (int)p.Ms[1], (int)p.nseg[0], (int)p.nseg[1], (int)R, p.GS);
            INFT_CHECK_LAUNCH();
            p.launches++;
            if (p.comb2d_n > 0) {
                k_spread_2d_combine<T><<<(unsigned)p.comb2d_n, 256, 0, st>>>(
                    p.comb2d.as<int4>(), p.part2d.as<C2<T>>(), grid, (int)p.Ms[1], (int)p.nseg[1], (int)R, p.GS);
                INFT_CHECK_LAUNCH();
                p.launches++;
            }
            return;
        }
        const int64_t warps = p.Mstot * ceil_div(R, 32);
        const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(warps * 32, 256), (int64_t)148 * 64);
        if (p.wt == INFT_WEIGHTS_COMPLEX)
            k_spread_2d_warp<T, true><<<blocks, 256, 0, st>>>(p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), w, p.PP,
                                                              p.P1, fT, grid, p.Ms[0], p.Ms[1], p.S[0], p.S[1],
                                                              p.nseg[1], (int)R, p.GS);
        else
            k_spread_2d_warp<T, false><<<blocks, 256, 0, st>>>(p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), w,
                                                               p.PP, p.P1, fT, grid, p.Ms[0], p.Ms[1], p.S[0],
                                                               p.S[1], p.nseg[1], (int)R, p.GS);
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

// 2-D gather, node-stationary: CTA = a chunk of <= kG2 nodes of one 16 x 16-cell tile x 32 RHS
// (lane = RHS).  The chunk's weights arrive by one bulk copy; the grid rows its footprints
// cover (16 + P1 - 1 of them, each 16 + P1 - 1 cells wide) stream through a double-buffered
// shared row (cp.async), and warp w accumulates, in registers, the nodes w, w + 8, ... of the
// chunk: node j adds sum_t2 w_j[t1][t2] g[row][c_j + t2] for the row's slot t1.  Heavy tiles
// are split into several chunks (balanced CTAs); one plain store per (node, RHS).
constexpr int kG2 = 64;

template <typename T, int MC>
__global__ void __launch_bounds__(256) k_gather_2d_tile(const int2* __restrict__ chunks, const int32_t* __restrict__ seg_start,
                                                        const int32_t* __restrict__ n0s, const int32_t* __restrict__ perm,
                                                        const T* __restrict__ w, int PP, const C2<T>* __restrict__ grid,
                                                        C2<T>* __restrict__ f, int64_t N, int Ms1, int Ms2, int nseg2,
                                                        int R, int64_t GS) {
    constexpr int P1 = 2 * MC + 1;
    constexpr int W = 16 + P1 - 1;  // rows and columns covered by the tile's footprints
    constexpr int NPW = kG2 / 8;    // nodes per warp
    extern __shared__ __align__(128) unsigned char sg[];
    C2<T>* gsm = reinterpret_cast<C2<T>*>(sg);                    // [2][W][32]
    T* wsm = reinterpret_cast<T*>(gsm + 2 * W * 32);              // [kG2][PP]
    __shared__ uint64_t wbar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2 ch = chunks[blockIdx.x];
    const int tile = ch.x, first = ch.y;
    const int nn = min(kG2, __ldg(seg_start + tile + 1) - first);
    const int s1 = tile / nseg2, s2 = tile - (tile / nseg2) * nseg2;
    const int row0 = s1 * 16, col0 = s2 * 16;
    const int rbase = blockIdx.y * 32;
    const int r = rbase + lane;
    if (threadIdx.x == 0) {
        mbar_init(&wbar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t wb = (uint32_t)(sizeof(T) * (size_t)nn * PP);
        mbar_arrive_expect_tx(&wbar, wb);
        bulk_g2s(wsm, w + (int64_t)first * PP, wb, &wbar);
    }
    auto stage_row = [&](int rho) {
        int grow = row0 + rho;
        if (grow >= Ms1) grow -= Ms1;
        C2<T>* dst = gsm + (rho & 1) * W * 32;
        for (int e = threadIdx.x; e < W * 32; e += blockDim.x) {
            const int c = e >> 5, l = e & 31;
            int gc = col0 + c;
            if (gc >= Ms2) gc -= Ms2;
            const bool ok = rbase + l < R;
            cp_async<(int)sizeof(C2<T>)>(dst + e, grid + (int64_t)(ok ? rbase + l : 0) * GS + (int64_t)grow * Ms2 + gc,
                                         ok ? (int)sizeof(C2<T>) : 0);
        }
        cp_async_commit();
    };
    // my nodes: slot base offsets inside the tile
    int d1[NPW], c2[NPW];
#pragma unroll
    for (int q = 0; q < NPW; ++q) {
        const int j = warp + 8 * q;
        d1[q] = 1 << 20;
        c2[q] = 0;
        if (j < nn) {
            d1[q] = __ldg(n0s + 2 * (first + j)) - row0;
            c2[q] = __ldg(n0s + 2 * (first + j) + 1) - col0;
        }
    }
    T ax[NPW], ay[NPW];
#pragma unroll
    for (int q = 0; q < NPW; ++q) ax[q] = ay[q] = T(0);
    stage_row(0);
    mbar_wait(&wbar, 0);
#pragma unroll 1
    for (int rho = 0; rho < W; ++rho) {
        if (rho + 1 < W) {
            stage_row(rho + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const C2<T>* g = gsm + (rho & 1) * W * 32 + lane;
#pragma unroll
        for (int q = 0; q < NPW; ++q) {
            const int t1 = rho - d1[q];
            if (t1 >= 0 && t1 < P1) {
                const T* wr = wsm + (warp + 8 * q) * PP + t1 * P1;
                const C2<T>* gq = g + c2[q] * 32;
                T sx = 0, sy = 0;
#pragma unroll
                for (int t2 = 0; t2 < P1; ++t2) {
                    const C2<T> gv = gq[t2 * 32];
                    sx = fma(wr[t2], gv.x, sx);
                    sy = fma(wr[t2], gv.y, sy);
                }
                ax[q] += sx;
                ay[q] += sy;
            }
        }
        __syncthreads();  // row buffer (rho & 1) free for row rho + 2
    }
    if (r < R) {
#pragma unroll
        for (int q = 0; q < NPW; ++q) {
            const int j = warp + 8 * q;
            if (j < nn) f[(int64_t)r * N + __ldg(perm + first + j)] = mk<T>(ax[q], ay[q]);
        }
    }
}

// 2-D gather with register row windows (default; INFT_GATHER2D_SMEM=1: k_gather_2d_tile).
// Same chunks (<= kG2 nodes of one tile x 32 RHS, lane = RHS) and the same streamed grid rows,
// but each warp loads the staged row ONCE into registers (W complex per lane) and every node of
// the warp whose footprint covers the row takes its P1 taps from registers (warp-uniform switch
// on the node's column offset: static register indices) -- k_gather_2d_tile read each tap from
// shared memory (4 wavefronts per tap and warp: shared-memory bound).  The node's weight row for
// the current grid row is staged with the grid row (cp.async, double-buffered), so the CTA keeps
// ~40 KB of shared memory instead of the chunk's whole weight block.  Deterministic: every
// node sums its rows in order, one store per (node, RHS).
template <typename T, int MC, int WPC, bool RWIN>
__global__ void __launch_bounds__(32 * WPC) k_gather_2d_rw(const int2* __restrict__ chunks,
                                                           const int32_t* __restrict__ seg_start,
                                                           const int32_t* __restrict__ n0s,
                                                           const int32_t* __restrict__ perm, const T* __restrict__ w,
                                                           int PP, const C2<T>* __restrict__ grid, C2<T>* __restrict__ f,
                                                           int64_t N, int Ms1, int Ms2, int nseg2, int R, int64_t GS) {
    constexpr int P1 = 2 * MC + 1;
    constexpr int W = 16 + P1 - 1;   // rows and columns covered by the tile's footprints
    constexpr int NPW = kG2 / WPC;   // nodes per warp
    constexpr int NT = 32 * WPC;
    constexpr int WRB = kG2 * P1;    // weight-row buffer (elements) per stage
    extern __shared__ __align__(128) unsigned char sg[];
    C2<T>* gsm = reinterpret_cast<C2<T>*>(sg);                        // [2][W][32]
    T* wrs = reinterpret_cast<T*>(gsm + 2 * W * 32);                  // [2][kG2][P1]
    int* meta = reinterpret_cast<int*>(wrs + 2 * WRB);                // [kG2]: d1 | c2 << 16
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2 ch = chunks[blockIdx.x];
    const int tile = ch.x, first = ch.y;
    const int nn = min(kG2, __ldg(seg_start + tile + 1) - first);
    const int s1 = tile / nseg2, s2 = tile - (tile / nseg2) * nseg2;
    const int row0 = s1 * 16, col0 = s2 * 16;
    const int rbase = blockIdx.y * 32;
    const int r = rbase + lane;
    for (int i = threadIdx.x; i < kG2; i += NT) {
        int v = 1 << 14;  // d1 out of range: never active
        if (i < nn) v = (__ldg(n0s + 2 * (first + i)) - row0) | ((__ldg(n0s + 2 * (first + i) + 1) - col0) << 16);
        meta[i] = v;
    }
    __syncthreads();
    auto stage_row = [&](int rho) {
        int grow = row0 + rho;
        if (grow >= Ms1) grow -= Ms1;
        C2<T>* dst = gsm + (rho & 1) * W * 32;
        for (int e = threadIdx.x; e < W * 32; e += NT) {
            const int c = e >> 5, l = e & 31;
            int gc = col0 + c;
            if (gc >= Ms2) gc -= Ms2;
            const bool ok = rbase + l < R;
            cp_async<(int)sizeof(C2<T>)>(dst + e, grid + (int64_t)(ok ? rbase + l : 0) * GS + (int64_t)grow * Ms2 + gc,
                                         ok ? (int)sizeof(C2<T>) : 0);
        }
        // weight rows t1 = rho - d1 of the nodes whose footprint covers grid row rho
        T* wd = wrs + (rho & 1) * WRB;
        for (int e = threadIdx.x; e < nn * P1; e += NT) {
            const int i = e / P1, t2 = e - (e / P1) * P1;
            const int t1 = rho - (meta[i] & 0xffff);
            if (t1 >= 0 && t1 < P1) cp_async<(int)sizeof(T)>(wd + e, w + (int64_t)(first + i) * PP + t1 * P1 + t2, (int)sizeof(T));
        }
        cp_async_commit();
    };
    T ax[NPW], ay[NPW];
#pragma unroll
    for (int q = 0; q < NPW; ++q) ax[q] = ay[q] = T(0);
    stage_row(0);
#pragma unroll 1
    for (int rho = 0; rho < W; ++rho) {
        if (rho + 1 < W) {
            stage_row(rho + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const C2<T>* g = gsm + (rho & 1) * W * 32 + lane;
        const T* wd = wrs + (rho & 1) * WRB;
        if constexpr (!RWIN) {
            // taps straight from the staged row (k_gather_2d_tile's inner loop)
#pragma unroll
            for (int q = 0; q < NPW; ++q) {
                const int mqq = meta[warp + WPC * q];
                const int t1 = rho - (mqq & 0xffff);
                if (t1 >= 0 && t1 < P1) {
                    const T* wr = wd + (warp + WPC * q) * P1;
                    const C2<T>* gq = g + (mqq >> 16) * 32;
                    T sx = 0, sy = 0;
#pragma unroll
                    for (int t2 = 0; t2 < P1; ++t2) {
                        const C2<T> gv = gq[t2 * 32];
                        sx = fma(wr[t2], gv.x, sx);
                        sy = fma(wr[t2], gv.y, sy);
                    }
                    ax[q] += sx;
                    ay[q] += sy;
                }
            }
            __syncthreads();
            continue;
        }
        T gx[W], gy[W];
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const C2<T> v = g[c * 32];
            gx[c] = v.x;
            gy[c] = v.y;
        }
#pragma unroll
        for (int q = 0; q < NPW; ++q) {
            const int mqq = meta[warp + WPC * q];  // broadcast
            const int t1 = rho - (mqq & 0xffff);
            if (t1 >= 0 && t1 < P1) {  // warp-uniform
                const T* wr = wd + (warp + WPC * q) * P1;
                T wv[P1];
#pragma unroll
                for (int t2 = 0; t2 < P1; ++t2) wv[t2] = wr[t2];
                T sx0 = 0, sy0 = 0, sx1 = 0, sy1 = 0;
                switch (mqq >> 16) {
#define INFT_G2RW_CASE(C)                                                \
    case C: {                                                            \
        _Pragma("unroll") for (int t2 = 0; t2 < P1; t2 += 2) {           \
            sx0 = fma(wv[t2], gx[C + t2], sx0);                          \
            sy0 = fma(wv[t2], gy[C + t2], sy0);                          \
            if (t2 + 1 < P1) {                                           \
                sx1 = fma(wv[t2 + 1], gx[C + t2 + 1], sx1);              \
                sy1 = fma(wv[t2 + 1], gy[C + t2 + 1], sy1);              \
            }                                                            \
        }                                                                \
    } break;
                    INFT_CASES_16(INFT_G2RW_CASE)
#undef INFT_G2RW_CASE
                    default:
                        break;
                }
                ax[q] += sx0 + sx1;
                ay[q] += sy0 + sy1;
            }
        }
        __syncthreads();  // row buffer (rho & 1) free for row rho + 2
    }
    if (r < R) {
#pragma unroll
        for (int q = 0; q < NPW; ++q) {
            const int j = warp + WPC * q;
            if (j < nn) f[(int64_t)r * N + __ldg(perm + first + j)] = mk<T>(ax[q], ay[q]);
        }
    }
}

template <typename T>
using Gather2dFn = void (*)(const int2*, const int32_t*, const int32_t*, const int32_t*, const T*, int, const C2<T>*,
                            C2<T>*, int64_t, int, int, int, int, int64_t);

// register windows (INFT_G2RW=1, 4 warps x 16 nodes) or taps from shared memory (default: 8
// warps x 8 nodes, the weight-row staging keeps two CTAs per SM where k_gather_2d_tile's
// whole-chunk weight block allowed one)
#ifndef INFT_G2RW
#define INFT_G2RW 0
#endif
constexpr bool kG2Rwin = INFT_G2RW != 0;
constexpr int kG2rwWpc = kG2Rwin ? 4 : 8;  // warps per chunk

template <typename T>
static Gather2dFn<T> gather2d_rw_fn(int m) {
    switch (m) {
        case 1: return k_gather_2d_rw<T, 1, kG2rwWpc, kG2Rwin>;
        case 2: return k_gather_2d_rw<T, 2, kG2rwWpc, kG2Rwin>;
        case 3: return k_gather_2d_rw<T, 3, kG2rwWpc, kG2Rwin>;
        case 4: return k_gather_2d_rw<T, 4, kG2rwWpc, kG2Rwin>;
        case 5: return k_gather_2d_rw<T, 5, kG2rwWpc, kG2Rwin>;
        case 6: return k_gather_2d_rw<T, 6, kG2rwWpc, kG2Rwin>;
        case 7: return k_gather_2d_rw<T, 7, kG2rwWpc, kG2Rwin>;
    }
    return nullptr;
}

template <typename T>
static size_t gather2d_rw_smem(int P1) {
    const int W = 16 + P1 - 1;
    return sizeof(C2<T>) * 2 * W * 32 + sizeof(T) * 2 * (size_t)kG2 * P1 + sizeof(int) * kG2;
}

template <typename T>
static Gather2dFn<T> gather2d_fn(int m) {
    switch (m) {
        case 1: return k_gather_2d_tile<T, 1>;
        case 2: return k_gather_2d_tile<T, 2>;
        case 3: return k_gather_2d_tile<T, 3>;
        case 4: return k_gather_2d_tile<T, 4>;
        case 5: return k_gather_2d_tile<T, 5>;
        case 6: return k_gather_2d_tile<T, 6>;
        case 7: return k_gather_2d_tile<T, 7>;
    }
    return nullptr;
}

// (tile, first node) of every chunk of <= kG2 nodes, built once per plan from seg_start
static void ensure_gather2d_chunks(Plan& p, cudaStream_t st) {
    if (p.chunks2d_n >= 0) return;
    std::vector<int32_t> ss((size_t)p.nseg_tot + 1);
    INFT_CUDA(cudaMemcpyAsync(ss.data(), p.seg_start.p, sizeof(int32_t) * ss.size(), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    std::vector<int2> ch;
    for (int64_t t = 0; t < p.nseg_tot; ++t)
        for (int32_t i = ss[t]; i < ss[t + 1]; i += kG2) ch.push_back(make_int2((int)t, i));
    p.chunks2d.alloc(sizeof(int2) * std::max<size_t>(1, ch.size()));
    if (!ch.empty())
        INFT_CUDA(cudaMemcpyAsync(p.chunks2d.p, ch.data(), sizeof(int2) * ch.size(), cudaMemcpyHostToDevice, st));
    p.chunks2d_n = (int64_t)ch.size();
}

template <typename T>
static void gather(Plan& p, const C2<T>* grid, C2<T>* f, int64_t R, cudaStream_t st) {
    if (p.N == 0) return;
    if (ring_available(p)) {
        gather_ring(p, grid, f, R, st);
        return;
    }
    if (stream1d_available(p)) {
        gather_stream1d(p, grid, f, R, st);
        return;
    }
    const T* w = p.w.as<T>();
    if (tile2d_available(p) && !getenv_flag("INFT_GATHER2D_GENERIC")) {
        ensure_gather2d_chunks(p, st);
        if (p.chunks2d_n > 0) {
            const int W = 16 + p.P1 - 1;
            const bool rw = !getenv_flag("INFT_GATHER2D_SMEM");
            const size_t smem = rw ? gather2d_rw_smem<T>(p.P1)
                                   : sizeof(C2<T>) * 2 * W * 32 + sizeof(T) * (size_t)kG2 * p.PP;
            Gather2dFn<T> fn = rw ? gather2d_rw_fn<T>(p.m) : gather2d_fn<T>(p.m);
            ensure_smem_attr((const void*)fn, smem);
            dim3 g((unsigned)p.chunks2d_n, (unsigned)ceil_div(R, 32));
            fn<<<g, rw ? 32 * kG2rwWpc : 256, smem, st>>>(p.chunks2d.as<int2>(), p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(),
                                     p.perm.as<int32_t>(), w, p.PP, grid, f, p.N, (int)p.Ms[0], (int)p.Ms[1],
                                     (int)p.nseg[1], (int)R, p.GS);
            INFT_CHECK_LAUNCH();
            p.launches++;
        }
        return;
    }
    int64_t total = R * p.N;
    if (p.wt == INFT_WEIGHTS_COMPLEX)
        k_gather_generic<T, true><<<gs_blocks(total, 256), 256, 0, st>>>(p.n0s.as<int32_t>(), p.perm.as<int32_t>(), w,
                                                                       p.PP, p.P1, p.d, grid, f, p.N, p.Ms[0],
                                                                       p.Ms[1], p.GS, (int)R);
    else
        k_gather_generic<T, false><<<gs_blocks(total, 256), 256, 0, st>>>(p.n0s.as<int32_t>(), p.perm.as<int32_t>(),
                                                                        w, p.PP, p.P1, p.d, grid, f, p.N, p.Ms[0],
                                                                        p.Ms[1], p.GS, (int)R);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

static void ensure_grid(Plan& p, int64_t rhs) {
    if (p.grid_rhs >= rhs && p.grid.p) return;
    p.grid.alloc((size_t)rhs * p.GS * p.elem_bytes());
    p.grid_rhs = rhs;
    p.state_version++;  // graphs captured on the old grid are stale
}

static int64_t grid_capacity(Plan& p, int64_t want) {
    if (p.grid_rhs >= want) return want;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    size_t budget = std::min<size_t>(fr / 3, (size_t)8 << 30);
    int64_t cap = std::max<int64_t>(1, (int64_t)(budget / ((size_t)p.GS * p.elem_bytes())));
    cap = std::max<int64_t>(cap, p.grid_rhs);
    return std::min<int64_t>(want, cap);
}

static cufftHandle fft_plan(Plan& p, int batch) {
    auto it = p.fft.find(FftKey{batch});
    if (it != p.fft.end()) return it->second;
    cufftHandle h;
    int n[2] = {(int)p.Ms[0], (int)p.Ms[1]};
    cufftType ty = p.prec == INFT_C128 ? CUFFT_Z2Z : CUFFT_C2C;
    // 1-D rows carry a halo: storage length GS >= M_sigma per batch entry
    int emb[2] = {(int)(p.d == 1 ? p.GS : p.Ms[0]), (int)p.Ms[1]};
    INFT_CUFFT(cufftPlanMany(&h, p.d, n, emb, 1, (int)p.GS, emb, 1, (int)p.GS, ty, batch));
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

// RAII stage timer: an NVTX range (header-only NVTX 3: a no-op unless a tool is attached)
// named after the SURVEY 8(a) row, and -- while profiling -- CUDA events on the launching
// stream around one stage.
static const char* const kStageNames[6] = {"inft:a2 spread",      "inft:a3 fft_forward", "inft:a4 trunc_deconv",
                                           "inft:a5 deconv_pad",  "inft:a6 fft_inverse", "inft:a7 gather"};
struct StageTimer {
    Plan& p;
    int stage;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    StageTimer(Plan& pp, int sg, cudaStream_t s) : p(pp), stage(sg), st(s) {
        nvtxRangePushA(kStageNames[sg]);
        if (p.profiling) {
            a = p.take_event();
            INFT_CUDA(cudaEventRecord(a, st));
        }
    }
    ~StageTimer() {
        nvtxRangePop();
        if (a) {
            cudaEvent_t b = p.take_event();
            cudaEventRecord(b, st);
            p.recs.push_back(Plan::Rec{stage, a, b});
            if (p.recs.size() > 4096) p.drain_profile();
        }
    }
};

// ====================================================================== small 1-D problems
// Configs 1-2 are launch-latency bound: for tiny batches (R M_sigma <= 8192, a
// power-of-two M_sigma, d = 1) one 1024-thread CTA per RHS runs the whole direction in shared
// memory in ONE launch (config 1: 0.028 -> 0.026 ms/step; config 2 with R = 16 stays on the
// multi-kernel pipeline: 0.034 there against 0.052 here) --
// inverse: spread (one thread per grid point, the nodes of its covering segments, written at
// the bit-reversed index) -> radix-2 FFT (twiddle table in shared memory) -> truncate and
// deconvolve; adjoint: deconvolve and zero-pad (bit-reversed) -> inverse FFT -> gather (one
// thread per node).  Same arithmetic as the generic kernels, deterministic.
#ifndef INFT_SMALL_THREADS
#define INFT_SMALL_THREADS 1024
#endif
constexpr int kSmallThreads = INFT_SMALL_THREADS;
__device__ __forceinline__ int bitrev_n(int v, int lg) { return (int)(__brev((unsigned)v) >> (32 - lg)); }

template <typename T, int SIGN>
__device__ void small_fft(C2<T>* g, const C2<T>* tw, int Ms, int lg) {
    // in-place radix-2 DIT on bit-reversed input; tw[k] = e^{-2 pi i k / Ms}, k < Ms/2
    for (int s = 1; s <= lg; ++s) {
        const int half = 1 << (s - 1), step = Ms >> s;
        for (int b = threadIdx.x; b < Ms / 2; b += blockDim.x) {
            const int grp = b >> (s - 1), j = b & (half - 1);
            const int i0 = (grp << s) + j, i1 = i0 + half;
            C2<T> w = tw[j * step];
            if (SIGN > 0) w.y = -w.y;
            const C2<T> u = g[i0], v = g[i1];
            const T vx = v.x * w.x - v.y * w.y, vy = v.x * w.y + v.y * w.x;
            g[i0] = mk<T>(u.x + vx, u.y + vy);
            g[i1] = mk<T>(u.x - vx, u.y - vy);
        }
        __syncthreads();
    }
}

// Stockham (self-sorting, out of place) radix-4 FFT of natural-order input, a radix-2 first stage
// when lg is odd: ceil(lg / 2) barriers instead of lg (config 1: 9 radix-2 stages took ~5000
// cycles of the single-CTA inverse's ~15600).  in -> out alternate between a and b; returns the
// buffer holding the result.  tw[k] = e^{-2 pi i k / Ms}, k < Ms/2.
template <typename T, int SIGN>
__device__ C2<T>* small_fft4(C2<T>* a, C2<T>* b, const C2<T>* tw, int Ms, int lg) {
    C2<T>* in = a;
    C2<T>* out = b;
    int ns = 1;
    auto twid = [&](int e) {  // e^{SIGN 2 pi i e / Ms}, 0 <= e < Ms
        C2<T> w = e < Ms / 2 ? tw[e] : mk<T>(-tw[e - Ms / 2].x, -tw[e - Ms / 2].y);
        if (SIGN > 0) w.y = -w.y;
        return w;
    };
    if (lg & 1) {  // radix 2, span 1: out[2 j + m] = in[j] +- in[j + Ms/2]
        for (int j = threadIdx.x; j < Ms / 2; j += blockDim.x) {
            const C2<T> u = in[j], v = in[j + Ms / 2];
            out[2 * j] = mk<T>(u.x + v.x, u.y + v.y);
            out[2 * j + 1] = mk<T>(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
        C2<T>* t = in;
        in = out;
        out = t;
        ns = 2;
    }
    for (; ns < Ms; ns *= 4) {
        for (int j = threadIdx.x; j < Ms / 4; j += blockDim.x) {
            const int k = j & (ns - 1);
            C2<T> x0 = in[j], x1 = in[j + Ms / 4], x2 = in[j + Ms / 2], x3 = in[j + 3 * (Ms / 4)];
            if (ns > 1) {
                const int e = k * (Ms / (4 * ns));
                const C2<T> w1 = twid(e), w2 = twid(2 * e), w3 = twid(3 * e);
                x1 = mk<T>(x1.x * w1.x - x1.y * w1.y, x1.x * w1.y + x1.y * w1.x);
                x2 = mk<T>(x2.x * w2.x - x2.y * w2.y, x2.x * w2.y + x2.y * w2.x);
                x3 = mk<T>(x3.x * w3.x - x3.y * w3.y, x3.x * w3.y + x3.y * w3.x);
            }
            // DFT4 with (SIGN i)^{nk}
            const C2<T> u0 = mk<T>(x0.x + x2.x, x0.y + x2.y), u1 = mk<T>(x0.x - x2.x, x0.y - x2.y);
            const C2<T> u2 = mk<T>(x1.x + x3.x, x1.y + x3.y);
            const C2<T> d = mk<T>(x1.x - x3.x, x1.y - x3.y);
            const C2<T> u3 = SIGN > 0 ? mk<T>(-d.y, d.x) : mk<T>(d.y, -d.x);
            const int base = (j - k) * 4 + k;
            out[base] = mk<T>(u0.x + u2.x, u0.y + u2.y);
            out[base + ns] = mk<T>(u1.x + u3.x, u1.y + u3.y);
            out[base + 2 * ns] = mk<T>(u0.x - u2.x, u0.y - u2.y);
            out[base + 3 * ns] = mk<T>(u1.x - u3.x, u1.y - u3.y);
        }
        __syncthreads();
        C2<T>* t = in;
        in = out;
        out = t;
    }
    return in;
}

template <typename T>
__device__ void small_twiddles(C2<T>* tw, int Ms) {
    for (int k = threadIdx.x; k < Ms / 2; k += blockDim.x) {
        double sn, cs;
        sincospi(-2.0 * (double)k / (double)Ms, &sn, &cs);
        tw[k] = mk<T>((T)cs, (T)sn);
    }
}

template <typename T, bool WC>
__global__ void __launch_bounds__(kSmallThreads) k_small_inverse(const int32_t* __restrict__ seg_start,
                                                       const int32_t* __restrict__ n0s,
                                                       const int32_t* __restrict__ perm, const T* __restrict__ w,
                                                       int PP, int P, const C2<T>* __restrict__ f,
                                                       C2<T>* __restrict__ fhat, const T* __restrict__ dk, int64_t N,
                                                       int Ms, int lg, int M, int S, int stage_bytes, int pshift) {
    extern __shared__ __align__(16) unsigned char smraw[];
    C2<T>* g = reinterpret_cast<C2<T>*>(smraw);
    C2<T>* gb = g + Ms;  // the Stockham FFT's second buffer
    C2<T>* tw = gb + Ms;
    const int r = blockIdx.x;
    const C2<T>* fr = f + (int64_t)r * N;
#ifdef INFT_SMALL_TIMING
    long long tcl[6];
    tcl[0] = clock64();
#define INFT_ST(i) if (threadIdx.x == 0) tcl[i] = clock64();
#else
#define INFT_ST(i)
#endif
    small_twiddles<T>(tw, Ms);
    const int64_t nseg = (Ms + S - 1) / S;
    // staged (when the plan's tables fit): f in sorted node order, slot bases, segment table and
    // weights copied to shared memory by coalesced loads first, so that the per-grid-point scan
    // below reads shared memory instead of chains of dependent global loads (config 1: 19 us)
    const bool staged = stage_bytes > 0;
    C2<T>* fs = tw + Ms / 2;
    int32_t* ns = reinterpret_cast<int32_t*>(fs + N);
    int32_t* ss = ns + N;
    T* ws = reinterpret_cast<T*>(smraw + ((((size_t)(2 * Ms + Ms / 2 + N) * sizeof(C2<T>) + 4 * (N + nseg + 1)) + 15) & ~(size_t)15));
    if (staged) {
        // the weight block (and the slot bases when their size is a 16-byte multiple) by one bulk
        // copy each, issued first so that they are in flight while the threads gather f through
        // perm: the per-thread copy loops waited for one global load after another (config 1:
        // ~4 us of the kernel's ~10)
        __shared__ uint64_t sbar;
        const uint32_t wbytes = (uint32_t)(sizeof(T) * (size_t)N * PP * (WC ? 2 : 1));
        const bool nbulk = (N * 4) % 16 == 0;
        if (threadIdx.x == 0) {
            mbar_init(&sbar, 1);
            fence_barrier_init();
            mbar_arrive_expect_tx(&sbar, wbytes + (nbulk ? (uint32_t)(4 * N) : 0u));
            bulk_g2s(ws, w, wbytes, &sbar);
            if (nbulk) bulk_g2s(ns, n0s, (uint32_t)(4 * N), &sbar);
        }
        // f in sorted order: a cyclic shift of the caller's order needs no perm load (one global
        // latency instead of two)
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            int j;
            if (pshift >= 0) {
                j = i + pshift;
                if (j >= N) j -= (int)N;
            } else {
                j = perm[i];
            }
            fs[i] = fr[j];
            if (!nbulk) ns[i] = n0s[i];
        }
        for (int i = threadIdx.x; i <= nseg; i += blockDim.x) ss[i] = seg_start[i];
        __syncthreads();  // also orders the barrier init before every thread's wait
        mbar_wait(&sbar, 0);
    }
    INFT_ST(1)
    // the deconvolution factors of this thread's outputs, loaded now (their latency overlaps the
    // spread and the FFT instead of following them)
    constexpr int kMaxOut = 4;
    T dv[kMaxOut];
#pragma unroll
    for (int q = 0; q < kMaxOut; ++q) {
        const int c = threadIdx.x + q * (int)blockDim.x;
        dv[q] = c < M ? dk[c] : T(0);
    }
    const int32_t* n0p = staged ? ns : n0s;
    const int32_t* ssp = staged ? ss : seg_start;
    const T* wp = staged ? ws : w;
    // covering segments of grid point n in int32 arithmetic (S is a power of two); the generic
    // int64 segment walk (for_segments) only when the span wraps onto itself
    const int lgS = __ffs(S) - 1;
    auto node_term = [&](int i, int t, T& sx, T& sy) {
        const C2<T> fv = staged ? fs[i] : fr[perm[i]];
        for (; t < P; t += Ms) {
            if (WC) {
                const T wr = wp[((int64_t)i * PP + t) * 2], wi = wp[((int64_t)i * PP + t) * 2 + 1];
                sx += wr * fv.x + wi * fv.y;
                sy += wr * fv.y - wi * fv.x;
            } else {
                const T wr = wp[(int64_t)i * PP + t];
                sx += wr * fv.x;
                sy += wr * fv.y;
            }
        }
    };
    for (int n = threadIdx.x; n < Ms; n += blockDim.x) {  // a2: conj(w) f over the covering segments
        T sx = 0, sy = 0;
        int lo = n - (P - 1);
        if (lo < 0) lo += Ms;
        const int s_lo = lo >> lgS, s_hi = n >> lgS;
        int cnt = s_hi - s_lo;
        if (cnt < 0) cnt += (int)nseg;
        if (P < Ms && (1 << lgS) == S && cnt + 1 <= nseg && !(cnt == 0 && lo > n)) {
            for (int k = 0; k <= cnt; ++k) {
                int sg = s_lo + k;
                if (sg >= nseg) sg -= (int)nseg;
                const int e = ssp[sg + 1];
                for (int i = ssp[sg]; i < e; ++i) {
                    int t = n - n0p[i];
                    if (t < 0) t += Ms;
                    if (t < P) node_term(i, t, sx, sy);
                }
            }
        } else {
            for_segments(n, P < Ms ? P : Ms, Ms, S, nseg, [&](int64_t sg) {
                for (int i = ssp[sg]; i < ssp[sg + 1]; ++i) {
                    int t = (int)mod64(n - n0p[i], Ms);
                    if (t >= P) continue;
                    node_term(i, t, sx, sy);
                }
            });
        }
        g[n] = mk<T>(sx, sy);
    }
    __syncthreads();
    INFT_ST(2)
    const C2<T>* gf = small_fft4<T, -1>(g, gb, tw, Ms, lg);  // a3: F^*
    INFT_ST(3)
    for (int c = threadIdx.x, q = 0; c < M; c += blockDim.x, ++q) {  // a4: truncate + s D^*
        const int k = c - M / 2;
        const C2<T> v = gf[k < 0 ? k + Ms : k];
        const T d = q < kMaxOut ? dv[q] : dk[c];
        fhat[(int64_t)r * M + c] = mk<T>(d * v.x, d * v.y);
    }
#ifdef INFT_SMALL_TIMING
    if (threadIdx.x == 0 && r == 0) {
        tcl[4] = clock64();
        printf("small_inverse cycles: stage %lld spread %lld fft %lld out %lld\n", tcl[1] - tcl[0], tcl[2] - tcl[1],
               tcl[3] - tcl[2], tcl[4] - tcl[3]);
    }
#endif
#undef INFT_ST
}

template <typename T, bool WC>
__global__ void __launch_bounds__(kSmallThreads) k_small_adjoint(const int32_t* __restrict__ n0s,
                                                       const int32_t* __restrict__ perm, const T* __restrict__ w,
                                                       int PP, int P, const C2<T>* __restrict__ h,
                                                       C2<T>* __restrict__ f, const T* __restrict__ dk, int64_t N,
                                                       int Ms, int lg, int M) {
    extern __shared__ __align__(16) unsigned char smraw[];
    C2<T>* g = reinterpret_cast<C2<T>*>(smraw);
    C2<T>* tw = g + Ms;
    const int r = blockIdx.x;
    small_twiddles<T>(tw, Ms);
    for (int q = threadIdx.x; q < Ms; q += blockDim.x) {  // a5: s D + zero pad
        const int k = q < Ms / 2 ? q : q - Ms;
        C2<T> v = mk<T>(T(0), T(0));
        if (k >= -M / 2 && k < M / 2) {
            const C2<T> hv = h[(int64_t)r * M + k + M / 2];
            const T d = dk[k + M / 2];
            v = mk<T>(d * hv.x, d * hv.y);
        }
        g[bitrev_n(q, lg)] = v;
    }
    __syncthreads();
    small_fft<T, 1>(g, tw, Ms, lg);  // a6: F
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {  // a7: B_opt
        T sx = 0, sy = 0;
        int q = n0s[i];
        for (int t = 0; t < P; ++t) {
            const C2<T> gv = g[q];
            if (WC) {
                const T wr = __ldg(w + ((int64_t)i * PP + t) * 2), wi = __ldg(w + ((int64_t)i * PP + t) * 2 + 1);
                sx += wr * gv.x - wi * gv.y;
                sy += wr * gv.y + wi * gv.x;
            } else {
                const T wr = __ldg(w + (int64_t)i * PP + t);
                sx += wr * gv.x;
                sy += wr * gv.y;
            }
            if (++q == Ms) q = 0;
        }
        f[(int64_t)r * N + perm[i]] = mk<T>(sx, sy);
    }
}

// (INFT_NO_SMALL=1 at plan creation turns it off; R * M_sigma bounds it to the latency-bound
// regime -- one CTA per RHS leaves the GPU idle for big batches)
static bool small_available(const Plan& p, int64_t R) {
    const int64_t Ms = p.Ms[0];
    return !p.no_small && p.d == 1 && Ms >= 16 && (Ms & (Ms - 1)) == 0 &&
           Ms * (int64_t)p.elem_bytes() <= 64 * 1024 && p.N <= (int64_t(1) << 16) && p.N > 0 &&
           R * Ms <= (int64_t(1) << 13);
}

template <typename T>
static void small_inverse(Plan& p, const void* f, void* fhat, int64_t R, cudaStream_t st) {
    const int Ms = (int)p.Ms[0];
    const int lg = __builtin_ctz((unsigned)Ms);
    const int64_t nseg = (Ms + p.S[0] - 1) / p.S[0];
    const size_t base = sizeof(C2<T>) * (size_t)(2 * Ms + Ms / 2);  // grid, FFT buffer, twiddles
    // staged tables: f (sorted order), slot bases, segment table, weights
    const size_t staged = ((base + sizeof(C2<T>) * p.N + 4 * (p.N + nseg + 1) + 15) & ~(size_t)15) +
                          sizeof(T) * (size_t)p.N * p.PP * (p.wt == INFT_WEIGHTS_COMPLEX ? 2 : 1);
    const bool stage = staged <= 160 * 1024 && !getenv_flag("INFT_SMALL_NOSTAGE");
    const size_t smem = stage ? staged : base;
    auto kfn = p.wt == INFT_WEIGHTS_COMPLEX ? k_small_inverse<T, true> : k_small_inverse<T, false>;
    ensure_smem_attr((const void*)kfn, smem);
    kfn<<<(unsigned)R, kSmallThreads, smem, st>>>(p.seg_start.as<int32_t>(), p.n0s.as<int32_t>(), p.perm.as<int32_t>(),
                                        p.w.as<T>(), p.PP, p.P, static_cast<const C2<T>*>(f),
                                        static_cast<C2<T>*>(fhat), dtable<T>(p), p.N, Ms, lg, (int)p.M[0],
                                        p.S[0], stage ? (int)staged : 0, p.perm_shift);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

template <typename T>
static void small_adjoint(Plan& p, const void* h, void* f, int64_t R, cudaStream_t st) {
    const int Ms = (int)p.Ms[0];
    const int lg = __builtin_ctz((unsigned)Ms);
    const size_t smem = sizeof(C2<T>) * (size_t)(Ms + Ms / 2);
    auto kfn = p.wt == INFT_WEIGHTS_COMPLEX ? k_small_adjoint<T, true> : k_small_adjoint<T, false>;
    ensure_smem_attr((const void*)kfn, smem);
    kfn<<<(unsigned)R, kSmallThreads, smem, st>>>(p.n0s.as<int32_t>(), p.perm.as<int32_t>(), p.w.as<T>(), p.PP, p.P,
                                        static_cast<const C2<T>*>(h), static_cast<C2<T>*>(f), dtable<T>(p), p.N, Ms,
                                        lg, (int)p.M[0]);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

static bool use_fused(const Plan& p) { return !p.no_fused_fft && fused_fft_available(p); }

// One device-resident chunk (Rc <= grid capacity) of the inverse: a2 -> a3 -> a4.
template <typename T>
static void inverse_chunk(Plan& p, const void* f, void* fhat, int64_t Rc, cudaStream_t st) {
    if (small_available(p, Rc)) {  // a2 -> a3 -> a4 in one launch
        StageTimer t(p, 0, st);
        small_inverse<T>(p, f, fhat, Rc, st);
        return;
    }
    ensure_grid(p, Rc);
    C2<T>* g = p.grid.as<C2<T>>();
    {
        StageTimer t(p, 0, st);
        spread<T>(p, static_cast<const C2<T>*>(f), g, Rc, st);
    }
    // a3 + a4 in two fused passes (fft.cu); pass B's TMA store boxes need a 16-byte aligned fhat
    if (use_fused(p) && (reinterpret_cast<uintptr_t>(fhat) & 15) == 0) {
        {
            StageTimer t(p, 1, st);  // pass A: column FFTs + four-step twiddles (in place)
            fused_fft_inverse(p, g, fhat, Rc, st, 1);
        }
        StageTimer t(p, 2, st);  // pass B: row FFTs + truncation + deconvolution
        fused_fft_inverse(p, g, fhat, Rc, st, 2);
        return;
    }
    {
        StageTimer t(p, 1, st);
        fft_exec(p, g, (int)Rc, CUFFT_FORWARD, st);
    }
    StageTimer t(p, 2, st);
    int64_t total = Rc * p.Mtot;
    k_trunc_deconv<T><<<gs_blocks(total, 256), 256, 0, st>>>(g, static_cast<C2<T>*>(fhat), dtable<T>(p), p.M[0],
                                                             p.d == 2 ? p.M[1] : 1, p.Ms[0],
                                                             p.d == 2 ? p.Ms[1] : 1, p.GS, p.d, (int)Rc);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

// One chunk of the inverse adjoint: a5 -> a6 -> a7.
template <typename T>
static void adjoint_chunk(Plan& p, const void* h, void* f, int64_t Rc, cudaStream_t st) {
    if (small_available(p, Rc)) {  // a5 -> a6 -> a7 in one launch
        StageTimer t(p, 5, st);
        small_adjoint<T>(p, h, f, Rc, st);
        return;
    }
    ensure_grid(p, Rc);
    C2<T>* g = p.grid.as<C2<T>>();
    int64_t total = Rc * p.Mstot;
    // a5 + a6 in two fused passes (fft.cu), grid written with its halo; the TMA boxes over h
    // need a 16-byte aligned base
    if (use_fused(p) && (reinterpret_cast<uintptr_t>(h) & 15) == 0) {
        {
            StageTimer t(p, 3, st);  // pass A: deconvolution + zero pad + column FFTs
            fused_fft_adjoint(p, h, g, Rc, st, 1);
        }
        {
            StageTimer t(p, 4, st);  // pass B: row FFTs, natural-order grid + halo
            fused_fft_adjoint(p, h, g, Rc, st, 2);
        }
        StageTimer t(p, 5, st);
        gather<T>(p, g, static_cast<C2<T>*>(f), Rc, st);
        return;
    }
    {
        StageTimer t(p, 3, st);
        k_deconv_pad<T><<<gs_blocks(total, 256), 256, 0, st>>>(static_cast<const C2<T>*>(h), g, dtable<T>(p), p.M[0],
                                                               p.d == 2 ? p.M[1] : 1, p.Ms[0],
                                                               p.d == 2 ? p.Ms[1] : 1, p.GS, p.d, (int)Rc);
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

// Device pointer on the plan's device -> true; host memory -> false; a device pointer on
// another GPU is an argument error (the kernels would fault with an illegal address).
static bool plan_device_ptr(const Plan& p, const void* ptr) {
    const int d = pointer_device(ptr);
    if (d >= 0 && d != p.device) {
        set_error("apply: buffer lives on cuda:" + std::to_string(d) + ", the plan on cuda:" +
                  std::to_string(p.device));
        throw Fail{INFT_ERR_INVALID_ARG};
    }
    return d >= 0;
}

// Device-resident path: chunks of the grid capacity.  Host path: double-buffered
// staging; H2D of chunk c+1 (stream s_h2d) and D2H of chunk c-1 (stream s_d2h)
// overlap the compute of chunk c on the caller's stream.
static void run(Plan& p, const void* in, size_t in_rhs_bytes, void* out, size_t out_rhs_bytes, int64_t R,
                cudaStream_t st, ChunkFn fn) {
    const bool in_dev = in_rhs_bytes == 0 || plan_device_ptr(p, in);
    const bool out_dev = out_rhs_bytes == 0 || plan_device_ptr(p, out);
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
    // chunks of ~stage_mb MB (INFT_STAGE_MB, default 256; e2e step on config 5: 256 MB 80.7 ms,
    // 64 MB 82.0 ms, 32 MB 87.6 ms -- per-chunk costs outweigh the shorter pipeline fill/drain)
    static const size_t stage_mb = [] {
        const char* e = getenv("INFT_STAGE_MB");
        const long v = e ? atol(e) : 256;
        return (size_t)(v > 0 ? v : 256);
    }();
    int64_t Rh = std::max<int64_t>(1, std::min<int64_t>(R, (int64_t)((stage_mb << 20) / std::max<size_t>(per, 1))));
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
    // chunk schedule: a quarter-size first and last chunk shorten the pipeline fill (first
    // H2D alone) and drain (last D2H alone); full chunks in between (INFT_STAGE_RAMP=0: uniform)
    static const bool ramp = [] {
        const char* e = getenv("INFT_STAGE_RAMP");
        return !(e && atoi(e) == 0);
    }();
    std::vector<int64_t> starts;
    {
        const int64_t q = std::max<int64_t>(1, Rh / 4);
        if (ramp && R >= 2 * q + Rh) {
            starts.push_back(0);
            int64_t r = q;
            while (R - q - r > 0) {
                starts.push_back(r);
                r += std::min(Rh, R - q - r);
            }
            starts.push_back(R - q);
        } else {
            for (int64_t r = 0; r < R; r += Rh) starts.push_back(r);
        }
        starts.push_back(R);
    }
    const int64_t nchunk = (int64_t)starts.size() - 1;
    for (int64_t c = 0; c < nchunk; c++) {
        const int b = (int)(c & 1);
        const int64_t r0 = starts[c], rc = starts[c + 1] - starts[c];
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

// Repeated applies on the same device buffers replay a CUDA graph: the second call captures
// the launch sequence on the plan's stream s_graph (forked from / joined back to the caller's
// stream by events, so the caller's stream may be the legacy default stream), later calls
// launch it -- one host call instead of one per kernel, and tighter kernel-to-kernel gaps
// (configs 1-2 are launch-latency bound).  Off while profiling, for host
// buffers, and with INFT_GRAPHS=0; the key includes the plan's state version.
static bool graphs_enabled() {
    static const bool on = [] {
        const char* e = getenv("INFT_GRAPHS");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

static void run_graphed(Plan& p, int dir, const void* in, size_t in_rhs_bytes, void* out, size_t out_rhs_bytes,
                        int64_t R, cudaStream_t st, ChunkFn fn) {
    const bool dev = (in_rhs_bytes == 0 || plan_device_ptr(p, in)) && (out_rhs_bytes == 0 || plan_device_ptr(p, out));
    if (!graphs_enabled() || p.profiling || !dev) {
        run(p, in, in_rhs_bytes, out, out_rhs_bytes, R, st, fn);
        return;
    }
    // drop graphs captured on an older plan state (stale buffers) and cap the cache: callers
    // whose buffer addresses rotate would otherwise accumulate one exec per address pair
    for (auto it = p.graphs.begin(); it != p.graphs.end();) {
        if (it->first.version < p.state_version) {
            if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
            it = p.graphs.erase(it);
        } else {
            ++it;
        }
    }
    const Plan::GraphKey key{dir, in, out, R, p.state_version};
    if (p.graphs.size() >= Plan::kMaxGraphs && !p.graphs.count(key)) {
        auto lru = p.graphs.begin();
        for (auto it = p.graphs.begin(); it != p.graphs.end(); ++it)
            if (it->second.last_use < lru->second.last_use) lru = it;
        if (lru->second.exec) cudaGraphExecDestroy(lru->second.exec);
        p.graphs.erase(lru);
    }
    Plan::GraphEntry& e = p.graphs[key];
    e.last_use = ++p.graph_clock;
    if (!e.exec && e.seen++ == 0) {  // first call: plain launches (allocations, one-time tables)
        run(p, in, in_rhs_bytes, out, out_rhs_bytes, R, st, fn);
        return;
    }
    if (!p.s_graph) {
        INFT_CUDA(cudaStreamCreateWithFlags(&p.s_graph, cudaStreamNonBlocking));
        INFT_CUDA(cudaEventCreateWithFlags(&p.ev_g0, cudaEventDisableTiming));
        INFT_CUDA(cudaEventCreateWithFlags(&p.ev_g1, cudaEventDisableTiming));
    }
    if (!e.exec) {
        const int64_t l0 = p.launches;
        INFT_CUDA(cudaStreamBeginCapture(p.s_graph, cudaStreamCaptureModeRelaxed));
        cudaGraph_t g = nullptr;
        try {
            run(p, in, in_rhs_bytes, out, out_rhs_bytes, R, p.s_graph, fn);
        } catch (...) {
            cudaStreamEndCapture(p.s_graph, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        INFT_CUDA(cudaStreamEndCapture(p.s_graph, &g));
        const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
        cudaGraphDestroy(g);
        INFT_CUDA(ie);
        e.launches = p.launches - l0;
        p.launches = l0;  // counted again below, when the graph actually runs
    }
    INFT_CUDA(cudaEventRecord(p.ev_g0, st));
    INFT_CUDA(cudaStreamWaitEvent(p.s_graph, p.ev_g0, 0));
    INFT_CUDA(cudaGraphLaunch(e.exec, p.s_graph));
    INFT_CUDA(cudaEventRecord(p.ev_g1, p.s_graph));
    INFT_CUDA(cudaStreamWaitEvent(st, p.ev_g1, 0));
    p.launches += e.launches;
}

void apply_inverse(Plan& p, const void* f, void* fhat, int64_t R, cudaStream_t st) {
    const size_t e = p.elem_bytes();
    ChunkFn fn = p.prec == INFT_C128 ? (ChunkFn)inverse_chunk<double> : (ChunkFn)inverse_chunk<float>;
    run_graphed(p, 0, f, (size_t)p.N * e, fhat, (size_t)p.Mtot * e, R, st, fn);
}

void apply_adjoint(Plan& p, const void* h, void* f, int64_t R, cudaStream_t st) {
    const size_t e = p.elem_bytes();
    ChunkFn fn = p.prec == INFT_C128 ? (ChunkFn)adjoint_chunk<double> : (ChunkFn)adjoint_chunk<float>;
    run_graphed(p, 1, h, (size_t)p.Mtot * e, f, (size_t)p.N * e, R, st, fn);
}

}  // namespace inft
