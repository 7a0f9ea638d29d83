// 2-D spread (SURVEY 8(a) a2 for d = 2, config 4) as a 1-D register-window spread along the
// row-major grid line.
//
// The grid [M_sigma1][M_sigma2] stored row-major IS a line of L = M_sigma1 M_sigma2 cells.  Node j
// with base cell (n0_1, n0_2) (reading A12: I(x_j) = I1 x I2, 2-D weights w[j][t1 P1 + t2]) adds,
// for each of its P1 = 2m+1 row slots t1, the 1-D row w[j][t1][0..P1) f_j at line positions
// y M_sigma2 + n0_2 + t2 with y = (n0_1 + t1) mod M_sigma1.  Each (j, t1) is a "virtual node" of a
// 1-D spread with P1 taps along the line; when the row slice wraps past the row end
// (n0_2 + P1 - 1 >= M_sigma2) it is split into two virtual nodes (taps before the wrap at
// y M_sigma2 + n0_2, taps after it at y M_sigma2 + n0_2 - M_sigma2 whose leading taps are zero), so
// every virtual node's taps run along the line and the line itself is periodic (row 0's wrap
// lands at the line end).  B_opt^* f is then exactly
//   g[p] = sum over virtual nodes v with p - pos_v in [0, P1) of  w_v[p - pos_v] f_{j(v)}.
//
// Kernel (k_spread_line): one warp per work item x 32 right-hand sides (lane = RHS), a window of
// SEG + P1 - 1 grid values per lane held in registers (accumulated in double for complex64 too:
// B_opt's large cancelling weights make float accumulation lose ~1e-5), virtual nodes
// in line order in batches of NB (records by one bulk copy, the f rows of the node-major copy
// fT[i][R] by one 512-byte bulk copy per node, double-buffered on mbarriers); a node adds its P1
// taps at its offset inside the current SEG-cell segment through a warp-uniform switch (static
// register indices).  A finished segment is stored once (no atomics); the first segment of an
// item and the spill past its last segment go to per-item slots that k_line_fix adds up in a
// fixed order (deterministic).  Heavy segments (polar centre) are split into node ranges.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"
#include "inft_internal.cuh"
#include "tma.cuh"

namespace inft {
namespace line2d {

#ifndef INFT_LINE_SEG
#define INFT_LINE_SEG 16
#endif
// segment width (cells): window SEG + P1 - 1 complex per lane; the fix-up assumes P1 - 1 <= SEG
// (the spill past an item lands in the next item's first segment only)
constexpr int SEG = INFT_LINE_SEG;
constexpr int LSEG = SEG == 16 ? 4 : (SEG == 8 ? 3 : 2);
constexpr int NB = 16;  // virtual nodes per staged batch

// record: int32 pos, int32 end of its equal-position run, 2 pad words, then P1 weights in double
// (also for complex64 plans: no conversions in the inner loop), record = 16-byte multiple
template <typename T>
__host__ __device__ constexpr int rec_bytes(int P1) {
    return (16 + P1 * 8 + 15) / 16 * 16;
}

// keys: line position of virtual node (i, t1, part) or INT_MAX (no virtual node)
template <typename T>
__global__ void k_line_keys(const int32_t* __restrict__ n0s, const T* __restrict__ w, int PP, int P1, int N,
                            int Ms1, int Ms2, int* __restrict__ keys, int* __restrict__ vals) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // e = i P1 + t1
    if (e >= (int64_t)N * P1) return;
    const int i = (int)(e / P1), t1 = (int)(e - (int64_t)i * P1);
    const T* wr = w + (int64_t)i * PP + t1 * P1;
    bool any = false;
    for (int t2 = 0; t2 < P1; ++t2) any |= wr[t2] != T(0);
    int k0 = INT_MAX, k1 = INT_MAX;
    if (any) {
        int y = n0s[2 * i] + t1;
        if (y >= Ms1) y -= Ms1;
        const int b = n0s[2 * i + 1];
        const int L = Ms1 * Ms2;
        k0 = y * Ms2 + b;
        if (b + P1 - 1 >= Ms2) {
            int q = y * Ms2 + b - Ms2;
            if (q < 0) q += L;
            k1 = q;
        }
    }
    keys[2 * e] = k0;
    keys[2 * e + 1] = k1;
    vals[2 * e] = (int)(2 * e);
    vals[2 * e + 1] = (int)(2 * e + 1);
}

template <typename T>
__global__ void k_line_records(const int* __restrict__ skeys, const int* __restrict__ svals, int nv,
                               const int32_t* __restrict__ n0s, const T* __restrict__ w, int PP, int P1, int Ms2,
                               unsigned char* __restrict__ rec, int* __restrict__ vidx) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const int e2 = svals[v];
    const int part = e2 & 1;
    const int e = e2 >> 1;
    const int i = e / P1, t1 = e - (e / P1) * P1;
    const int b = n0s[2 * i + 1];
    const bool wraps = b + P1 - 1 >= Ms2;
    const int k = Ms2 - b;  // taps t2 < k stay in the row, t2 >= k wrap to its start
    unsigned char* r = rec + (size_t)v * rec_bytes<T>(P1);
    // end of the run of virtual nodes at the same line position (the kernel dispatches on the
    // segment offset once per run)
    const int key = skeys[v];
    int lo = v + 1, hi = nv;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (skeys[mid] <= key)
            lo = mid + 1;
        else
            hi = mid;
    }
    reinterpret_cast<int*>(r)[0] = key;
    reinterpret_cast<int*>(r)[1] = lo;
    reinterpret_cast<int*>(r)[2] = 0;
    reinterpret_cast<int*>(r)[3] = 0;
    double* wv = reinterpret_cast<double*>(r + 16);
    const T* wr = w + (int64_t)i * PP + t1 * P1;
    for (int t2 = 0; t2 < P1; ++t2) {
        const bool keep = !wraps || (part == 0 ? t2 < k : t2 >= k);
        wv[t2] = keep ? (double)wr[t2] : 0.0;
    }
    for (int t2 = P1; (16 + t2 * 8) < rec_bytes<T>(P1); ++t2) wv[t2] = 0.0;
    vidx[v] = i;
}

// seg_start[s] = first virtual node with pos >= SEG s (s = 0..nseg); nseg = L / SEG
__global__ void k_line_segstart(const int* __restrict__ skeys, int n, int nseg, int* __restrict__ seg) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s > nseg) return;
    const int target = s == nseg ? INT_MAX : s * SEG;
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (skeys[mid] < target)
            lo = mid + 1;
        else
            hi = mid;
    }
    seg[s] = lo;
}

// add w[0..P1) v into the window at offset C (static register indices)
template <int P1, int C>
__device__ __forceinline__ void add_taps(double (&a)[SEG + P1 - 1], const double* wv, double v) {
#pragma unroll
    for (int t = 0; t < P1; ++t) a[C + t] = fma(wv[t], v, a[C + t]);
}

template <int P1>
__device__ __forceinline__ void load_w(double (&wv)[P1], const unsigned char* r) {
    const double* src = reinterpret_cast<const double*>(r + 16);
#pragma unroll
    for (int t = 0; t + 1 < P1; t += 2) {
        const double2 v = *reinterpret_cast<const double2*>(src + t);
        wv[t] = v.x;
        wv[t + 1] = v.y;
    }
    if constexpr (P1 & 1) wv[P1 - 1] = src[P1 - 1];
}

// nodes [q, qe) of a staged batch, all at segment offset C; lane = (RHS, component): the lane's
// component of f_j is fc[u * 32 + lane] (the staged rows hold 16 complex values = 32 reals)
template <typename T, int P1, int C>
__device__ __forceinline__ void run_taps(double (&a)[SEG + P1 - 1], const unsigned char* rs, const T* fc, int q,
                                         int qe, int lane) {
    constexpr int RB = rec_bytes<T>(P1);
#pragma unroll 1
    for (int u = q; u < qe; ++u) {
        double wv[P1];
        load_w<P1>(wv, rs + u * RB);
        add_taps<P1, C>(a, wv, (double)fc[u * 32 + lane]);
    }
}

// One warp = one work item x 16 right-hand sides; lane = (RHS r = lane / 2, component lane & 1)
// holds one real window of SEG + P1 - 1 values (half the registers of a complex window, so four
// warps fit each SM sub-partition's register file).
template <typename T, int P1>
__global__ void __maxnreg__(128) k_spread_line(const int4* __restrict__ items, const unsigned char* __restrict__ rec,
                                               const int* __restrict__ vidx, const C2<T>* __restrict__ fT,
                                               C2<T>* __restrict__ grid, int64_t GS, C2<double>* __restrict__ first,
                                               C2<double>* __restrict__ carry, int R, int RS) {
    constexpr int W = SEG + P1 - 1;
    constexpr int RB = rec_bytes<T>(P1);
    constexpr int RG = 16;  // right-hand sides per warp
    constexpr uint32_t FB = NB * RG * sizeof(C2<T>);
    constexpr uint32_t STAGE = FB + NB * RB;
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t full[2];
    const int item = blockIdx.x;
    const int lane = threadIdx.x;
    const int g = blockIdx.y;
    const int r = g * RG + (lane >> 1), comp = lane & 1;
    const int rows = min(RG, R - g * RG);
    const bool act = (lane >> 1) < rows;
    const int4 it = items[item];
    const int s0 = it.x, s1 = it.y, b0 = it.z, b1 = it.w;
    if (lane == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_barrier_init();
    }
    __syncwarp();
    // f rows of the node-major copy fT[i][RS] (RS: 16-byte multiple): 16-byte cp.async chunks
    // spread over the lanes (per-lane addresses; a bulk copy per node would be issued lane by
    // lane), node indices prefetched one batch ahead; records by one bulk copy on the mbarrier
    constexpr int CPN = RG * (int)sizeof(C2<T>) / 16;  // 16-byte chunks per node row
    constexpr int CPL = NB * CPN / 32;                 // chunks per lane per batch
    const int vbytes = rows * (int)sizeof(C2<T>);
    auto vload = [&](int b) { return (lane < NB && b + lane < b1) ? __ldg(vidx + b + lane) : 0; };
    auto issue = [&](int b, int st, int vi) {
        const int nb = min(NB, b1 - b);
        unsigned char* sb = sm + (size_t)st * STAGE;
        if (lane == 0) {
            mbar_arrive_expect_tx(&full[st], (uint32_t)nb * RB);
            bulk_g2s(sb + FB, rec + (size_t)b * RB, (uint32_t)nb * RB, &full[st]);
        }
#pragma unroll
        for (int k2 = 0; k2 < CPL; ++k2) {
            const int c = lane + 32 * k2;
            const int q = c / CPN, part = c - (c / CPN) * CPN;
            const int i = __shfl_sync(0xffffffffu, vi, q);
            const int nbytes = (q < nb && part * 16 < vbytes) ? 16 : 0;
            cp_async<16>(sb + (size_t)c * 16,
                         reinterpret_cast<const unsigned char*>(fT + (int64_t)i * RS + g * RG) + (nbytes ? part * 16 : 0),
                         nbytes);
        }
        cp_async_commit();
    };
    double a[W];
#pragma unroll
    for (int c = 0; c < W; ++c) a[c] = 0.0;
    int seg = s0;
    auto store_seg = [&](int s) {
        if (act) {
            if (s == s0) {
                double* d = reinterpret_cast<double*>(first + ((int64_t)item * R + r) * SEG) + comp;
#pragma unroll
                for (int c = 0; c < SEG; ++c) d[2 * c] = a[c];
            } else {
                T* d = reinterpret_cast<T*>(grid + (int64_t)r * GS + (int64_t)s * SEG) + comp;
#pragma unroll
                for (int c = 0; c < SEG; ++c) d[2 * c] = (T)a[c];
            }
        }
    };
    auto advance = [&]() {
        store_seg(seg);
#pragma unroll
        for (int c = 0; c < W; ++c) a[c] = c + SEG < W ? a[c + SEG] : 0.0;
        ++seg;
    };
    int k = 0;
    int vnext = vload(b0);
    if (b0 < b1) issue(b0, 0, vnext);
    vnext = vload(b0 + NB);
    if (b0 + NB < b1) issue(b0 + NB, 1, vnext);
    vnext = vload(b0 + 2 * NB);
#pragma unroll 1
    for (int b = b0; b < b1; b += NB, ++k) {
        const int st = k & 1;
        const int nb = min(NB, b1 - b);
        if (b + NB < b1)
            cp_async_wait<1>();
        else
            cp_async_wait<0>();
        mbar_wait(&full[st], (k >> 1) & 1);
        __syncwarp();  // every lane's f chunks of this batch landed
        const unsigned char* sb = sm + (size_t)st * STAGE;
        const T* fc = reinterpret_cast<const T*>(sb);
        const unsigned char* rs = sb + FB;
        // runs of equal line position (records sorted by position): one offset dispatch per run,
        // then a tight loop of P1-tap updates at a static offset
#pragma unroll 1
        for (int q = 0; q < nb;) {
            const int* hq = reinterpret_cast<const int*>(rs + q * RB);
            const int pos = hq[0];
            const int qe = min(hq[1] - b, nb);
            while ((pos >> LSEG) > seg) advance();
            switch (pos & (SEG - 1)) {
#define INFT_LINE_CASE(CC)                                  \
    case CC:                                                \
        run_taps<T, P1, CC>(a, rs, fc, q, qe, lane);        \
        break;
                INFT_LINE_CASE(0) INFT_LINE_CASE(1) INFT_LINE_CASE(2) INFT_LINE_CASE(3)
#if INFT_LINE_SEG > 4
                INFT_LINE_CASE(4) INFT_LINE_CASE(5) INFT_LINE_CASE(6) INFT_LINE_CASE(7)
#endif
#if INFT_LINE_SEG > 8
                INFT_LINE_CASE(8) INFT_LINE_CASE(9) INFT_LINE_CASE(10) INFT_LINE_CASE(11) INFT_LINE_CASE(12)
                INFT_LINE_CASE(13) INFT_LINE_CASE(14) INFT_LINE_CASE(15)
#endif
#undef INFT_LINE_CASE
            }
            q = qe;
        }
        fence_proxy_async();  // this stage's generic reads precede the bulk copies that reuse it
        __syncwarp();
        if (b + 2 * NB < b1) {
            issue(b + 2 * NB, st, vnext);
            vnext = vload(b + 3 * NB);
        }
    }
    while (seg < s1 - 1) advance();
    store_seg(seg);
    if (act) {
        double* d = reinterpret_cast<double*>(carry + ((int64_t)item * R + r) * (P1 - 1)) + comp;
#pragma unroll
        for (int c = 0; c < P1 - 1; ++c) d[2 * c] = a[SEG + c];
    }
}

// fix entry (s, first item k0, items k1, carry items [c0, c1) mod nitems): the first segment of
// the items starting at s = their first slots plus the spill of the items ending at s - 1
template <typename T>
__global__ void k_line_fix(const int4* __restrict__ fix, const C2<double>* __restrict__ first,
                           const C2<double>* __restrict__ carry, C2<T>* __restrict__ grid, int64_t GS, int R, int P1,
                           int nitems) {
    const int4 fe = fix[blockIdx.x];
    const int s = fe.x, kf0 = fe.y;
    const int nf = fe.z & 0xffff, nc = fe.z >> 16;
    const int c0 = fe.w;
    for (int e = threadIdx.x; e < R * SEG; e += blockDim.x) {
        const int rr = e / SEG, c = e - (e / SEG) * SEG;
        double sx = 0.0, sy = 0.0;
        for (int q = 0; q < nf; ++q) {
            const C2<double> v = first[((int64_t)(kf0 + q) * R + rr) * SEG + c];
            sx += v.x;
            sy += v.y;
        }
        if (c < P1 - 1)
            for (int q = 0; q < nc; ++q) {
                int kc = c0 + q;
                if (kc >= nitems) kc -= nitems;
                const C2<double> v = carry[((int64_t)kc * R + rr) * (P1 - 1) + c];
                sx += v.x;
                sy += v.y;
            }
        grid[(int64_t)rr * GS + (int64_t)s * SEG + c] = mk<T>((T)sx, (T)sy);
    }
}

template <typename T>
using LineFn = void (*)(const int4*, const unsigned char*, const int*, const C2<T>*, C2<T>*, int64_t, C2<double>*,
                        C2<double>*, int, int);

template <typename T>
static LineFn<T> line_fn(int P1) {
    switch (P1) {
        case 3: return k_spread_line<T, 3>;
        case 5: return k_spread_line<T, 5>;
        case 7: return k_spread_line<T, 7>;
        case 9: return k_spread_line<T, 9>;
        case 11: return k_spread_line<T, 11>;
        case 13: return k_spread_line<T, 13>;
        case 15: return k_spread_line<T, 15>;
    }
    return nullptr;
}

template <typename T>
static size_t stage_smem(int P1) {
    return 2 * ((size_t)NB * 16 * sizeof(C2<T>) + (size_t)NB * rec_bytes<T>(P1));
}

}  // namespace line2d

bool line2d_available(const Plan& p) {
    if (p.d != 2 || p.wt != INFT_WEIGHTS_REAL || p.m < 1 || p.m > 7) return false;
    if ((p.Ms[0] * p.Ms[1]) % line2d::SEG != 0 || p.Ms[1] < p.P1 || p.Ms[0] * p.Ms[1] >= INT_MAX / 2) return false;
    if ((int64_t)p.N * p.P1 * 2 >= INT_MAX) return false;
    return !getenv_flag("INFT_SPREAD2D_TILE");
}

// Virtual-node records, segment table, work items and fix entries: rebuilt when the weights change.
template <typename T>
static void ensure_line(Plan& p, cudaStream_t st) {
    using namespace line2d;
    if (p.line_version == p.w_version) return;
    const int P1 = p.P1;
    const int N = (int)p.N;
    const int Ms1 = (int)p.Ms[0], Ms2 = (int)p.Ms[1];
    const int L = Ms1 * Ms2;
    const int nseg = L / SEG;
    const int64_t ne = (int64_t)N * P1 * 2;
    DevBuf keys, vals, skeys, svals, tmp;
    keys.alloc(sizeof(int) * std::max<int64_t>(1, ne));
    vals.alloc(sizeof(int) * std::max<int64_t>(1, ne));
    skeys.alloc(sizeof(int) * std::max<int64_t>(1, ne));
    svals.alloc(sizeof(int) * std::max<int64_t>(1, ne));
    if (N > 0) {
        k_line_keys<T><<<(unsigned)ceil_div((int64_t)N * P1, 256), 256, 0, st>>>(
            p.n0s.as<int32_t>(), p.w.as<T>(), p.PP, P1, N, Ms1, Ms2, keys.as<int>(), vals.as<int>());
        INFT_CHECK_LAUNCH();
        size_t tb = 0;
        // keys < L or INT_MAX (no virtual node): all 31 bits (stable sort: ties keep (i, t1) order)
        INFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<int>(), skeys.as<int>(), vals.as<int>(),
                                                  svals.as<int>(), (int)ne, 0, 31, st));
        tmp.alloc(std::max<size_t>(tb, 1));
        INFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<int>(), skeys.as<int>(), vals.as<int>(),
                                                  svals.as<int>(), (int)ne, 0, 31, st));
    }
    p.line_seg.alloc(sizeof(int) * (nseg + 1));
    if (N > 0) {
        k_line_segstart<<<(unsigned)ceil_div(nseg + 1, 256), 256, 0, st>>>(skeys.as<int>(), (int)ne, nseg,
                                                                          p.line_seg.as<int>());
        INFT_CHECK_LAUNCH();
    } else {
        INFT_CUDA(cudaMemsetAsync(p.line_seg.p, 0, sizeof(int) * (nseg + 1), st));
    }
    std::vector<int> seg((size_t)nseg + 1);
    INFT_CUDA(cudaMemcpyAsync(seg.data(), p.line_seg.p, sizeof(int) * (nseg + 1), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    const int nv = seg[nseg];
    p.line_nv = nv;
    p.line_rec.alloc((size_t)rec_bytes<T>(P1) * std::max(1, nv));
    p.line_vidx.alloc(sizeof(int) * std::max(1, nv));
    if (nv > 0) {
        k_line_records<T><<<(unsigned)ceil_div(nv, 256), 256, 0, st>>>(skeys.as<int>(), svals.as<int>(), nv,
                                                                      p.n0s.as<int32_t>(), p.w.as<T>(), p.PP, P1, Ms2,
                                                                      p.line_rec.as<unsigned char>(),
                                                                      p.line_vidx.as<int>());
        INFT_CHECK_LAUNCH();
    }
    // work items: runs of whole segments up to T virtual nodes (<= 64 segments); a segment with
    // more than T nodes is split into node ranges of <= T (one item each)
    int nsm = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    static const int per_sm = [] {
        const char* e = getenv("INFT_LINE_ITEMS_PER_SM");
        const int v = e ? atoi(e) : 0;
        return v > 0 ? v : 8;
    }();
    const int T_nodes = std::max(64, (int)((int64_t)nv / ((int64_t)nsm * per_sm)) + 1);
    std::vector<int4> items;
    for (int s = 0; s < nseg;) {
        const int c = seg[s + 1] - seg[s];
        if (c > T_nodes) {
            const int parts = (c + T_nodes - 1) / T_nodes;
            const int per = (c + parts - 1) / parts;
            for (int b = seg[s]; b < seg[s + 1]; b += per) items.push_back(make_int4(s, s + 1, b, std::min(b + per, seg[s + 1])));
            ++s;
            continue;
        }
        int e = s + 1, cnt = c;
        while (e < nseg && e - s < 64) {
            const int ce = seg[e + 1] - seg[e];
            if (ce > T_nodes || cnt + ce > T_nodes) break;
            cnt += ce;
            ++e;
        }
        items.push_back(make_int4(s, e, seg[s], seg[e]));
        s = e;
    }
    const int nitems = (int)items.size();
    // fix entries: one per distinct item start segment; carries = the items ending just before
    std::vector<int4> fixes;
    for (int k = 0; k < nitems;) {
        int k1 = k + 1;
        while (k1 < nitems && items[k1].x == items[k].x) ++k1;
        const int s = items[k].x;
        // carries: the items ending at segment s - 1 (mod nseg), consecutive just before k (cyclic)
        const int want = s == 0 ? nseg : s;
        int nc = 0, c0 = k;
        while (nc < nitems) {
            const int prev = (c0 - 1 + nitems) % nitems;
            if (items[prev].y != want) break;
            c0 = prev;
            ++nc;
        }
        fixes.push_back(make_int4(s, k, (k1 - k) | (nc << 16), c0));
        k = k1;
    }
    p.line_items.alloc(sizeof(int4) * std::max(1, nitems));
    p.line_fix.alloc(sizeof(int4) * std::max<size_t>(1, fixes.size()));
    if (nitems)
        INFT_CUDA(cudaMemcpyAsync(p.line_items.p, items.data(), sizeof(int4) * nitems, cudaMemcpyHostToDevice, st));
    if (!fixes.empty())
        INFT_CUDA(cudaMemcpyAsync(p.line_fix.p, fixes.data(), sizeof(int4) * fixes.size(), cudaMemcpyHostToDevice, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    p.line_nitems = nitems;
    p.line_nfix = (int)fixes.size();
    p.line_slot_rhs = 0;
    p.line_version = p.w_version;
}

template <typename T>
void spread_line2d_t(Plan& p, const C2<T>* fT, C2<T>* grid, int64_t R, int RS, cudaStream_t st) {
    using namespace line2d;
    ensure_line<T>(p, st);
    if (p.line_slot_rhs < R) {
        p.line_first.alloc(sizeof(C2<double>) * (size_t)std::max(1, p.line_nitems) * R * SEG);
        p.line_carry.alloc(sizeof(C2<double>) * (size_t)std::max(1, p.line_nitems) * R * (p.P1 - 1));
        p.line_slot_rhs = R;
        p.state_version++;
    }
    if (p.line_nitems > 0) {
        const size_t smem = stage_smem<T>(p.P1);
        auto fn = line_fn<T>(p.P1);
        ensure_smem_attr((const void*)fn, smem);
        dim3 g((unsigned)p.line_nitems, (unsigned)ceil_div(R, 16));
        fn<<<g, 32, smem, st>>>(p.line_items.as<int4>(), p.line_rec.as<unsigned char>(), p.line_vidx.as<int>(), fT,
                                grid, p.GS, p.line_first.as<C2<double>>(), p.line_carry.as<C2<double>>(), (int)R, RS);
        INFT_CHECK_LAUNCH();
        p.launches++;
        k_line_fix<T><<<(unsigned)p.line_nfix, 256, 0, st>>>(p.line_fix.as<int4>(), p.line_first.as<C2<double>>(),
                                                            p.line_carry.as<C2<double>>(), grid, p.GS, (int)R, p.P1,
                                                            p.line_nitems);
        INFT_CHECK_LAUNCH();
        p.launches++;
    } else {
        for (int64_t r = 0; r < R; ++r)
            INFT_CUDA(cudaMemsetAsync(grid + r * p.GS, 0, sizeof(C2<T>) * p.Mstot, st));
    }
}

void spread_line2d(Plan& p, const void* fT, void* grid, int64_t R, int RS, cudaStream_t st) {
    if (p.prec == INFT_C128)
        spread_line2d_t<double>(p, static_cast<const C2<double>*>(fT), static_cast<C2<double>*>(grid), R, RS, st);
    else
        spread_line2d_t<float>(p, static_cast<const C2<float>*>(fT), static_cast<C2<float>*>(grid), R, RS, st);
}

}  // namespace inft
