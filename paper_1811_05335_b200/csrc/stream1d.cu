// 1-D streaming spread (a2) and gather (a7) kernels for real B_opt weights.
//
// Both walk the bin-sorted node stream of a chunk of Q consecutive grid
// segments (width SEG >= 2m) with lane = right-hand side, keeping a window of
// SEG + 2m grid values per lane in registers.  A node's slot base n0 lies in
// its segment, so its P = 2m+1 taps hit window registers delta .. delta+2m,
// delta = n0 - seg*SEG; a warp-uniform switch on delta makes every register
// index static.  No atomics, deterministic summation order.
//
// k_spread_tma_1d / k_gather_tma_1d (caller node order == sorted order, the 1-D
// configs): every operand is staged through shared memory by the async copy
// engines in a kStages-deep mbarrier pipeline issued by one thread --
//   * node records (P weights + n0) by 1-D bulk copy (cp.async.bulk),
//   * spread: the f tile [rows = block RHS][16 nodes] by 2-D TMA
//     (cp.async.bulk.tensor, SWIZZLE_128B, OOB zero fill),
//   * gather: the next SEG grid points of every row by 2-D TMA over a grid
//     whose rows carry a 2m halo (filled after the FFT), so windows never wrap.
// The register-window kernels without staging remain for non-identity node
// permutations (per-lane gathers of f through perm).
#include <algorithm>
#include <cstdlib>

#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "inft_internal.cuh"
#include "tma.cuh"

namespace inft {

static constexpr int kQ = 32;       // segments per chunk
static constexpr int kNB = 16;      // nodes per staged batch
static constexpr int kStages = 4;   // pipeline depth

// ---------------------------------------------------------------------------------
// Spread, staged.  grid[r][n] (row stride GS) for n in the chunk's segments.
template <typename T, int MC, int SEG>
__global__ void __launch_bounds__(128) k_spread_tma_1d(const __grid_constant__ CUtensorMap fmap,
                                                       const int32_t* __restrict__ seg_start,
                                                       const T* __restrict__ w, int PP, C2<T>* __restrict__ grid,
                                                       int64_t GS, int nseg, int Q, int R, int N, int cshift,
                                                       int dbg) {
    constexpr int P = 2 * MC + 1;
    constexpr int K = SEG + 2 * MC;
    constexpr int EB = 128 / (int)sizeof(C2<T>);  // complex values per 128-byte box row
    constexpr int CE = (int)sizeof(C2<T>) / 8;     // 8-byte tensor-map elements per complex value
    constexpr int NB = sizeof(T) == 8 ? 16 : 32;  // nodes per staged batch: two 128-byte f boxes
    constexpr int NBOX = NB / EB;
    static_assert(SEG >= 2 * MC && SEG <= 32, "segment must cover the support");
    const int WPB = blockDim.x >> 5;
    const int rows = blockDim.x;
    const int lane = threadIdx.x & 31;
    const int row = threadIdx.x;
    const int r = blockIdx.y * rows + row;
    const bool active = r < R;

    // dynamic shared memory (no static smem in this kernel): base is 1024-aligned,
    // and indexing the __shared__ array keeps every access in the shared window (LDS)
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t box_bytes = (uint32_t)rows * 128u;
    const uint32_t fstage = NBOX * box_bytes;
    const uint32_t rstage = (uint32_t)((NB * PP * (int)sizeof(T) + 127) & ~127);
    unsigned char* fbuf = smem;
    unsigned char* rbuf = smem + kStages * fstage;
    uint64_t* full = reinterpret_cast<uint64_t*>(rbuf + kStages * rstage);
    uint64_t* empty = full + kStages;

    const int s0 = blockIdx.x * Q;
    const int s1 = min(s0 + Q, nseg);
    const int sp = s0 == 0 ? nseg - 1 : s0 - 1;
    const int a0 = __ldg(seg_start + sp), a1 = __ldg(seg_start + sp + 1);
    const int b0 = __ldg(seg_start + s0), b1 = __ldg(seg_start + s1);
    // Batches never straddle the sorted position where the caller column wraps
    // (node order = cyclic shift cshift of the sorted order), so every f tile is
    // one contiguous TMA box.  Sub-ranges (scalars, no local arrays):
    //   prologue [a0, aw) [aw, a1)  then  main [b0, bw) [bw, b1),
    // aw / bw = the wrap position if it lies strictly inside, else the range end.
    const int wrap = N - cshift;
    const int aw = (cshift > 0 && a0 < wrap && wrap < a1) ? wrap : a1;
    const int bw = (cshift > 0 && b0 < wrap && wrap < b1) ? wrap : b1;
    const int c1 = (aw - a0 + NB - 1) / NB;
    const int c2 = c1 + (a1 - aw + NB - 1) / NB;
    const int c3 = c2 + (bw - b0 + NB - 1) / NB;
    const int nb = c3 + (b1 - bw + NB - 1) / NB;

    auto batch_pos = [&](int b, int& pos, int& cnt, int& origin) {
        int s, e, base;
        if (b < c1) {
            s = a0; e = aw; base = 0; origin = 1;
        } else if (b < c2) {
            s = aw; e = a1; base = c1; origin = 1;
        } else if (b < c3) {
            s = b0; e = bw; base = c2; origin = 0;
        } else {
            s = bw; e = b1; base = c3; origin = 0;
        }
        pos = s + (b - base) * NB;
        cnt = min(NB, e - pos);
    };
    auto issue = [&](int b, int stage) {
        int pos, cnt, origin;
        batch_pos(b, pos, cnt, origin);
        const uint32_t rbytes = (uint32_t)(cnt * PP * (int)sizeof(T));
        int col = pos + cshift;
        if (col >= N) col -= N;
        mbar_arrive_expect_tx(&full[stage], ((dbg & 8) ? 0u : fstage) + rbytes);
        if (!(dbg & 8)) {
#pragma unroll
            for (int bx = 0; bx < NBOX; ++bx)
                tma_load_2d(fbuf + stage * fstage + bx * box_bytes, &fmap, (col + bx * EB) * CE, blockIdx.y * rows,
                            &full[stage]);
        }
        bulk_g2s(rbuf + stage * rstage, w + (int64_t)pos * PP, rbytes, &full[stage]);
    };

    if (threadIdx.x == 0) {
        prefetch_tmap(&fmap);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], WPB);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int b = 0; b < min(kStages, nb); ++b) issue(b, b);

    const uint32_t rowoff = (uint32_t)row * 128u;  // this lane's row in a 128-byte-swizzled box
    const int rx = row & 7;
    T ax[K], ay[K];
#pragma unroll
    for (int u = 0; u < K; ++u) ax[u] = ay[u] = T(0);
    int cur_k = 0;  // 0 = prologue segment sp, k >= 1 = main segment s0 + k - 1
    C2<T>* __restrict__ gr = grid + (int64_t)(active ? r : 0) * GS;
    auto flush = [&]() {
        if (cur_k >= 1 && active && !(dbg & 2)) {
            C2<T>* out = gr + (int64_t)(s0 + cur_k - 1) * SEG;
#pragma unroll
            for (int u = 0; u < SEG; ++u) __stcs(out + u, mk<T>(ax[u], ay[u]));
        }
#pragma unroll
        for (int u = 0; u < K; ++u) {
            ax[u] = (u + SEG < K) ? ax[u + SEG] : T(0);
            ay[u] = (u + SEG < K) ? ay[u + SEG] : T(0);
        }
        ++cur_k;
    };

    for (int b = 0; b < nb; ++b) {
        const int stage = b % kStages;
        const uint32_t parity = (uint32_t)((b / kStages) & 1);
        int pos, cnt, origin;
        batch_pos(b, pos, cnt, origin);
        mbar_wait(&full[stage], parity);
        const unsigned char* fb = fbuf + stage * fstage;
        const T* rbp = reinterpret_cast<const T*>(rbuf + stage * rstage);
        const bool pro = origin == 1;
        for (int q = 0; q < cnt; ++q) {
            const T* rec = rbp + q * PP;
            const unsigned n0 = (unsigned)rec_n0(rec, P);
            const int seg = (int)(n0 / SEG);
            const int dl = (int)(n0 % SEG);
            const int kq = pro ? 0 : seg - s0 + 1;
            while (cur_k < kq) flush();
            const int bx = q / EB, c = q % EB;
            C2<T> fv = mk<T>(T(0), T(0));
            if (!(dbg & 4)) {
                if (sizeof(C2<T>) == 16)
                    fv = *reinterpret_cast<const C2<T>*>(fb + bx * box_bytes + rowoff + ((c ^ rx) << 4));
                else
                    fv = *reinterpret_cast<const C2<T>*>(fb + bx * box_bytes + rowoff + (((c >> 1) ^ rx) << 4) +
                                                         (c & 1) * 8);
            }
            T wv[P];
            WeightLoader<T, P>::load_smem(rec, wv);
            switch ((dbg & 1) ? 99 : dl) {
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
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (threadIdx.x == 0 && b + kStages < nb) {
            mbar_wait(&empty[stage], parity);
            issue(b + kStages, stage);
        }
    }
    while (cur_k <= s1 - s0) flush();
}

// ---------------------------------------------------------------------------------
// Gather, staged.  f[r][j] = sum_t w[j][t] g[r][n0_j + t] (grid rows with a 2m halo).
template <typename T, int MC, int SEG>
__global__ void __launch_bounds__(128) k_gather_tma_1d(const __grid_constant__ CUtensorMap gmap,
                                                       const int32_t* __restrict__ seg_start,
                                                       const T* __restrict__ w, int PP, C2<T>* __restrict__ f,
                                                       int64_t N, int nseg, int Q, int R, int cshift, int dbg) {
    constexpr int P = 2 * MC + 1;
    constexpr int K = SEG + 2 * MC;
    constexpr int EB = 128 / (int)sizeof(C2<T>);
    constexpr int CE = (int)sizeof(C2<T>) / 8;
    constexpr int NWB = (SEG + EB - 1) / EB;  // boxes per window load
    const int WPB = blockDim.x >> 5;
    const int rows = blockDim.x;
    const int lane = threadIdx.x & 31;
    const int row = threadIdx.x;
    const int r = blockIdx.y * rows + row;
    const bool active = r < R;

    // dynamic shared memory (no static smem in this kernel): base is 1024-aligned,
    // and indexing the __shared__ array keeps every access in the shared window (LDS)
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t box_bytes = (uint32_t)rows * 128u;
    const uint32_t wstage = NWB * box_bytes;
    const uint32_t rstage = (uint32_t)((kNB * PP * (int)sizeof(T) + 127) & ~127);
    unsigned char* wbuf = smem;
    unsigned char* rbuf = smem + kStages * wstage;
    uint64_t* fullW = reinterpret_cast<uint64_t*>(rbuf + kStages * rstage);
    uint64_t* emptyW = fullW + kStages;
    uint64_t* fullR = emptyW + kStages;
    uint64_t* emptyR = fullR + kStages;

    const int s0 = blockIdx.x * Q;
    const int s1 = min(s0 + Q, nseg);
    const int nbox = s1 - s0 + 1;  // box L holds grid [(s0-1+L)*SEG + 2m, ... + SEG)
    const int b0 = __ldg(seg_start + s0), b1 = __ldg(seg_start + s1);
    const int nbat = (b1 - b0 + kNB - 1) / kNB;

    auto issueW = [&](int L, int stage) {
        mbar_arrive_expect_tx(&fullW[stage], wstage);
        const int col = (s0 - 1 + L) * SEG + 2 * MC;
#pragma unroll
        for (int bx = 0; bx < NWB; ++bx)
            tma_load_2d(wbuf + stage * wstage + bx * box_bytes, &gmap, (col + bx * EB) * CE, blockIdx.y * rows,
                        &fullW[stage]);
    };
    auto issueR = [&](int b, int stage) {
        const int pos = b0 + b * kNB;
        const int cnt = min(kNB, b1 - pos);
        const uint32_t rbytes = (uint32_t)(cnt * PP * (int)sizeof(T));
        mbar_arrive_expect_tx(&fullR[stage], rbytes);
        bulk_g2s(rbuf + stage * rstage, w + (int64_t)pos * PP, rbytes, &fullR[stage]);
    };

    if (threadIdx.x == 0) {
        prefetch_tmap(&gmap);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&fullW[i], 1);
            mbar_init(&emptyW[i], WPB);
            mbar_init(&fullR[i], 1);
            mbar_init(&emptyR[i], WPB);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int L = 0; L < min(kStages, nbox); ++L) issueW(L, L);
        for (int b = 0; b < min(kStages, nbat); ++b) issueR(b, b);
    }

    const uint32_t rowoff = (uint32_t)row * 128u;
    const int rx = row & 7;
    T wx[K], wy[K];
    int nextL = 0;
    // load box nextL into window registers [2m, K)
    auto consume_box = [&]() {
        const int L = nextL++;
        const int stage = L % kStages;
        const uint32_t parity = (uint32_t)((L / kStages) & 1);
        mbar_wait(&fullW[stage], parity);
        const unsigned char* wb = wbuf + stage * wstage;
#pragma unroll
        for (int v = 0; v < SEG; ++v) {
            const int bx = v / EB, c = v % EB;
            C2<T> g;
            if (sizeof(C2<T>) == 16)
                g = *reinterpret_cast<const C2<T>*>(wb + bx * box_bytes + rowoff + ((c ^ rx) << 4));
            else
                g = *reinterpret_cast<const C2<T>*>(wb + bx * box_bytes + rowoff + (((c >> 1) ^ rx) << 4) + (c & 1) * 8);
            wx[2 * MC + v] = g.x;
            wy[2 * MC + v] = g.y;
        }
        fence_proxy_async();  // generic-proxy reads done before the TMA may overwrite
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyW[stage]);
        if (threadIdx.x == 0 && L + kStages < nbox) {
            mbar_wait(&emptyW[stage], parity);
            issueW(L + kStages, stage);
        }
    };
    int cur_j = -1;
    auto advance = [&]() {
#pragma unroll
        for (int u = 0; u < 2 * MC; ++u) {
            wx[u] = wx[u + SEG];
            wy[u] = wy[u + SEG];
        }
        consume_box();
        ++cur_j;
    };
    consume_box();

    C2<T>* __restrict__ fr = f + (int64_t)(active ? r : 0) * N;
    for (int b = 0; b < nbat; ++b) {
        const int stage = b % kStages;
        const uint32_t parity = (uint32_t)((b / kStages) & 1);
        const int pos = b0 + b * kNB;
        const int cnt = min(kNB, b1 - pos);
        mbar_wait(&fullR[stage], parity);
        const T* rb = reinterpret_cast<const T*>(rbuf + stage * rstage);
        for (int q = 0; q < cnt; ++q) {
            const T* rec = rb + q * PP;
            const unsigned n0 = (unsigned)rec_n0(rec, P);
            const int seg = (int)(n0 / SEG);
            const int dl = (int)(n0 % SEG);
            while (cur_j < seg - s0) advance();
            T wv[P];
            WeightLoader<T, P>::load_smem(rec, wv);
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
            int64_t j = pos + q + cshift;
            if (j >= N) j -= N;
            if (active) __stcs(fr + j, mk<T>(sx, sy));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyR[stage]);
        if (threadIdx.x == 0 && b + kStages < nbat) {
            mbar_wait(&emptyR[stage], parity);
            issueR(b + kStages, stage);
        }
    }
    while (nextL < nbox) advance();  // drain: no bulk copy may be in flight at exit
}

// ---------------------------------------------------------------------------------
// Register-window kernels without staging (any node permutation).
template <typename T, int MC, int SEG>
__global__ void __launch_bounds__(128) k_spread_reg_1d(
    const int32_t* __restrict__ seg_start, const int32_t* __restrict__ delta, const int32_t* __restrict__ perm,
    const T* __restrict__ w, int PP, const C2<T>* __restrict__ f, C2<T>* __restrict__ grid, int64_t N, int64_t GS,
    int nseg, int Q, int nchunks, int R, int nrg) {
    constexpr int P = 2 * MC + 1;
    constexpr int K = SEG + 2 * MC;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (gw >= (int64_t)nchunks * nrg) return;
    const int chunk = (int)(gw / nrg);
    const int rg = (int)(gw - (int64_t)chunk * nrg);
    const int r = rg * 32 + lane;
    const bool active = r < R;
    const C2<T>* __restrict__ fr = f + (int64_t)(active ? r : 0) * N;
    C2<T>* __restrict__ gr = grid + (int64_t)(active ? r : 0) * GS;
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
            const int64_t j = __ldg(perm + i);
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

template <typename T, int MC, int SEG>
__global__ void __launch_bounds__(128) k_gather_reg_1d(
    const int32_t* __restrict__ seg_start, const int32_t* __restrict__ delta, const int32_t* __restrict__ perm,
    const T* __restrict__ w, int PP, const C2<T>* __restrict__ grid, C2<T>* __restrict__ f, int64_t N, int64_t GS,
    int64_t Ms, int nseg, int Q, int nchunks, int R, int nrg) {
    constexpr int P = 2 * MC + 1;
    constexpr int K = SEG + 2 * MC;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (gw >= (int64_t)nchunks * nrg) return;
    const int chunk = (int)(gw / nrg);
    const int rg = (int)(gw - (int64_t)chunk * nrg);
    const int r = rg * 32 + lane;
    const bool active = r < R;
    const C2<T>* __restrict__ gr = grid + (int64_t)(active ? r : 0) * GS;
    C2<T>* __restrict__ fr = f + (int64_t)(active ? r : 0) * N;
    T wx[K], wy[K];
    const int s0 = chunk * Q;
    const int s1 = min(s0 + Q, nseg);
    for (int s = s0; s < s1; ++s) {
        const int64_t base = (int64_t)s * SEG;
#pragma unroll
        for (int u = 0; u < K; ++u) {
            if (s != s0 && u + SEG < K) {
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
        const int i0 = __ldg(seg_start + s), i1 = __ldg(seg_start + s + 1);
        for (int i = i0; i < i1; ++i) {
            const int dl = __ldg(delta + i);
            const int64_t j = __ldg(perm + i);
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

// grid[r][Ms + u] = grid[r][u], u < H: the halo that lets gather windows run past M_sigma.
template <typename T>
__global__ void k_halo_fill(C2<T>* __restrict__ grid, int64_t GS, int64_t Ms, int H, int R) {
    const int64_t total = (int64_t)R * H;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / H;
        const int64_t u = idx - r * H;
        grid[r * GS + Ms + u] = grid[r * GS + (u % Ms)];
    }
}

// ===================================================================== host side
template <typename T>
struct Fns {
    using SpreadTma = void (*)(const CUtensorMap, const int32_t*, const T*, int, C2<T>*, int64_t, int, int, int, int,
                               int, int);
    using GatherTma = void (*)(const CUtensorMap, const int32_t*, const T*, int, C2<T>*, int64_t, int, int, int, int,
                               int);
    using SpreadReg = void (*)(const int32_t*, const int32_t*, const int32_t*, const T*, int, const C2<T>*, C2<T>*,
                               int64_t, int64_t, int, int, int, int, int);
    using GatherReg = void (*)(const int32_t*, const int32_t*, const int32_t*, const T*, int, const C2<T>*, C2<T>*,
                               int64_t, int64_t, int64_t, int, int, int, int, int);
    SpreadTma st = nullptr;
    GatherTma gt = nullptr;
    SpreadReg sr = nullptr;
    GatherReg gr = nullptr;
};

template <typename T>
static Fns<T> fns_for(int m, int S) {
    Fns<T> F;
#define INFT_FN(MC, SG)                                  \
    if (m == MC && S == SG) {                            \
        F.st = k_spread_tma_1d<T, MC, SG>;               \
        F.gt = k_gather_tma_1d<T, MC, SG>;               \
        F.sr = k_spread_reg_1d<T, MC, SG>;               \
        F.gr = k_gather_reg_1d<T, MC, SG>;               \
    }
    INFT_FN(1, 16) INFT_FN(2, 16) INFT_FN(3, 16) INFT_FN(4, 8) INFT_FN(5, 16) INFT_FN(6, 16) INFT_FN(7, 16)
    INFT_FN(8, 16) INFT_FN(10, 32) INFT_FN(12, 32) INFT_FN(16, 32)
#undef INFT_FN
    return F;
}

static bool force_reg() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("INFT_FORCE_REG");
        v = (e && atoi(e)) ? 1 : 0;
    }
    return v == 1;
}

static int debug_flags() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("INFT_DEBUG_SPREAD");
        v = e ? atoi(e) : 0;
    }
    return v;
}

bool stream1d_available(const Plan& p) {
    if (p.d != 1 || !p.fast1d || p.wt != INFT_WEIGHTS_REAL || p.N == 0) return false;

    return p.prec == INFT_C128 ? fns_for<double>(p.m, p.S[0]).st != nullptr
                               : fns_for<float>(p.m, p.S[0]).st != nullptr;
}

static int wpb_for(int64_t R) { return (int)std::min<int64_t>(4, std::max<int64_t>(1, ceil_div(R, 32))); }

template <typename T>
static size_t spread_smem(int rows, int PP) {
    const int EB = 128 / (int)sizeof(C2<T>);
    const int NB = sizeof(T) == 8 ? 16 : 32;
    size_t fst = (size_t)(NB / EB) * rows * 128;
    size_t rst = (size_t)((NB * PP * (int)sizeof(T) + 127) & ~127);
    return 1024 + kStages * (fst + rst) + 2 * kStages * sizeof(uint64_t);
}

template <typename T>
static size_t gather_smem(int rows, int PP, int S) {
    const int EB = 128 / (int)sizeof(C2<T>);
    size_t wst = (size_t)((S + EB - 1) / EB) * rows * 128;
    size_t rst = (size_t)((kNB * PP * (int)sizeof(T) + 127) & ~127);
    return 1024 + kStages * (wst + rst) + 4 * kStages * sizeof(uint64_t);
}

// segments per chunk: kQ, fewer when the problem is too small to give every SM ~8 warps
// (config 1: 64 segments, 1 RHS -> Q = 2)
static int stream_q(int nseg, int64_t rowgroups) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (int64_t)nsm * 8;
    const int64_t q = ((int64_t)nseg * rowgroups + want - 1) / want;
    return (int)std::max<int64_t>(2, std::min<int64_t>(kQ, q));
}

template <typename T>
static void spread_t(Plan& p, const void* f, void* grid, int64_t R, cudaStream_t st) {
    Fns<T> F = fns_for<T>(p.m, p.S[0]);
    const int nseg = (int)p.nseg[0];
    const int Q = stream_q(nseg, ceil_div(R, 32));
    const int nchunks = (int)ceil_div(nseg, Q);
    // complex64: the f-tile boxes start at arbitrary node offsets, i.e. 8-byte aligned,
    // and a tensor-map load whose innermost start is not 16-byte aligned raises
    // "illegal instruction" (measured: tools/tma_probe.cu, offset 1 faults, offset 2
    // runs), so complex64 spreads use the register-window kernel.
    if (p.perm_shift >= 0 && sizeof(T) == 8 && !force_reg()) {
        const int wpb = wpb_for(R);
        const int rows = 32 * wpb;
        CUtensorMap map;
        if (!make_tmap_2d(&map, f, (uint64_t)p.N * sizeof(C2<T>) / 8, (uint64_t)R, sizeof(C2<T>) * (uint64_t)p.N,
                          (uint32_t)rows)) {
            set_error("cuTensorMapEncodeTiled failed (spread f tile)");
            throw Fail{INFT_ERR_CUDA};
        }
        size_t smem = spread_smem<T>(rows, p.PP);
        ensure_smem_attr((const void*)F.st, smem);
        dim3 grid_dim((unsigned)nchunks, (unsigned)ceil_div(R, rows));
        F.st<<<grid_dim, rows, smem, st>>>(map, p.seg_start.as<int32_t>(), p.w.as<T>(), p.PP,
                                           static_cast<C2<T>*>(grid), p.GS, nseg, Q, (int)R, (int)p.N, p.perm_shift,
                                           debug_flags());
    } else {
        const int nrg = (int)ceil_div(R, 32);
        const int64_t warps = (int64_t)nchunks * nrg;
        F.sr<<<(unsigned)ceil_div(warps * 32, 128), 128, 0, st>>>(
            p.seg_start.as<int32_t>(), p.delta.as<int32_t>(), p.perm.as<int32_t>(), p.w.as<T>(), p.PP,
            static_cast<const C2<T>*>(f), static_cast<C2<T>*>(grid), p.N, p.GS, nseg, Q, nchunks, (int)R, nrg);
    }
    INFT_CHECK_LAUNCH();
    p.launches++;
}

template <typename T>
static void gather_t(Plan& p, const void* grid, void* f, int64_t R, cudaStream_t st) {
    Fns<T> F = fns_for<T>(p.m, p.S[0]);
    const int nseg = (int)p.nseg[0];
    const int Q = stream_q(nseg, ceil_div(R, 32));
    const int nchunks = (int)ceil_div(nseg, Q);
    if (p.perm_shift >= 0 && !force_reg()) {
        const int wpb = wpb_for(R);
        const int rows = 32 * wpb;
        // halo: grid[r][Ms + u] = grid[r][u]
        const int H = (int)(p.GS - p.Ms[0]);
        k_halo_fill<T><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(R * H, 256), 4096)), 256, 0, st>>>(
            static_cast<C2<T>*>(const_cast<void*>(grid)), p.GS, p.Ms[0], H, (int)R);
        INFT_CHECK_LAUNCH();
        p.launches++;
        CUtensorMap map;
        if (!make_tmap_2d(&map, grid, (uint64_t)p.GS * sizeof(C2<T>) / 8, (uint64_t)R, sizeof(C2<T>) * (uint64_t)p.GS,
                          (uint32_t)rows)) {
            set_error("cuTensorMapEncodeTiled failed (gather grid window)");
            throw Fail{INFT_ERR_CUDA};
        }
        size_t smem = gather_smem<T>(rows, p.PP, p.S[0]);
        ensure_smem_attr((const void*)F.gt, smem);
        dim3 grid_dim((unsigned)nchunks, (unsigned)ceil_div(R, rows));
        F.gt<<<grid_dim, rows, smem, st>>>(map, p.seg_start.as<int32_t>(), p.w.as<T>(), p.PP, static_cast<C2<T>*>(f),
                                           p.N, nseg, Q, (int)R, p.perm_shift, debug_flags());
    } else {
        const int nrg = (int)ceil_div(R, 32);
        const int64_t warps = (int64_t)nchunks * nrg;
        F.gr<<<(unsigned)ceil_div(warps * 32, 128), 128, 0, st>>>(
            p.seg_start.as<int32_t>(), p.delta.as<int32_t>(), p.perm.as<int32_t>(), p.w.as<T>(), p.PP,
            static_cast<const C2<T>*>(grid), static_cast<C2<T>*>(f), p.N, p.GS, p.Ms[0], nseg, Q, nchunks, (int)R,
            nrg);
    }
    INFT_CHECK_LAUNCH();
    p.launches++;
}

void spread_stream1d(Plan& p, const void* f, void* grid, int64_t R, cudaStream_t st) {
    if (p.prec == INFT_C128)
        spread_t<double>(p, f, grid, R, st);
    else
        spread_t<float>(p, f, grid, R, st);
}

void gather_stream1d(Plan& p, const void* grid, void* f, int64_t R, cudaStream_t st) {
    if (p.prec == INFT_C128)
        gather_t<double>(p, grid, f, R, st);
    else
        gather_t<float>(p, grid, f, R, st);
}

// ------------------------------------------------------------------ tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return nullptr;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    return encode;
}

// Encoded maps are cached by their arguments: an apply re-encodes the same few maps every call
// (the encode is a driver call of about a microsecond; configs 1-2 are launch-latency bound).
struct TmapKey {
    const void* base;
    uint64_t a[8];
    bool operator==(const TmapKey& o) const {
        return base == o.base && std::memcmp(a, o.a, sizeof(a)) == 0;
    }
};
struct TmapKeyHash {
    size_t operator()(const TmapKey& k) const {
        size_t h = std::hash<const void*>()(k.base);
        for (uint64_t v : k.a) h = h * 1000003u ^ std::hash<uint64_t>()(v);
        return h;
    }
};
static std::mutex g_tmap_mu;
static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash>& tmap_cache() {
    static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> m;
    return m;
}
static bool tmap_lookup(const TmapKey& k, CUtensorMap* out) {
    std::lock_guard<std::mutex> g(g_tmap_mu);
    auto it = tmap_cache().find(k);
    if (it == tmap_cache().end()) return false;
    *out = it->second;
    return true;
}
static void tmap_store(const TmapKey& k, const CUtensorMap& m) {
    std::lock_guard<std::mutex> g(g_tmap_mu);
    if (tmap_cache().size() > 1024) tmap_cache().clear();
    tmap_cache()[k] = m;
}

// L2 promotion of the tensor maps' requests (experiment knob INFT_TMAP_L2 = 0 | 64 | 128 | 256,
// default 256 bytes)
static CUtensorMapL2promotion tmap_l2() {
    static const CUtensorMapL2promotion v = [] {
        const char* e = getenv("INFT_TMAP_L2");
        const int x = e ? atoi(e) : 256;
        return x == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                      : (x == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                 : (x == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B));
    }();
    return v;
}

bool make_tmap_3d(CUtensorMap* out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                  uint64_t s2, uint32_t b0, uint32_t b1, int esize) {
    const TmapKey key{base, {d0, d1, d2, s1, s2, b0, b1, (uint64_t)esize}};
    if (tmap_lookup(key, out)) return true;
    PFN_cuTensorMapEncodeTiled_v12000 encode = tmap_encoder();
    if (!encode) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {s1, s2};
    cuuint32_t box[3] = {b0, b1, 1u};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(out, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                        const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, tmap_l2(),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    tmap_store(key, *out);
    return true;
}

bool make_tmap_2d(CUtensorMap* out, const void* base, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes,
                  uint32_t box_rows) {
    const TmapKey key{base, {inner, rows, row_stride_bytes, box_rows, ~0ull, 0, 0, 0}};
    if (tmap_lookup(key, out)) return true;
    PFN_cuTensorMapEncodeTiled_v12000 encode = tmap_encoder();
    if (!encode) return false;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {16u, box_rows};  // 16 x 8 bytes = one 128-byte swizzle row
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, tmap_l2(),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    tmap_store(key, *out);
    return true;
}

}  // namespace inft
