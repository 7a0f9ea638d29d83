// 1-D streaming spread (a2) / gather (a7), "ring" variant for SEG = 2m.
//
// Same data flow as stream1d.cu (lane = right-hand side, bin-sorted node
// stream, warp-uniform switch on the node's slot offset), with three changes
// that remove most non-FMA instructions:
//  * Register ring.  With SEG = 2m the per-lane window of 2*SEG grid values
//    is two halves that swap roles every segment, so instead of shifting
//    registers the code is specialised on the segment parity (phase): grid
//    position pos of the window lives in register (pos + SEG*phase) mod 2*SEG.
//  * Stores through shared memory.  Spread: a finished segment (SEG values per
//    RHS row) is written to a per-warp SWIZZLE_128B staging tile and stored by
//    one 2-D TMA store; gather: the outputs of a 16-node batch likewise.
//  * Operands (node records, f tiles / grid windows) staged by TMA / bulk copy
//    in a 3-deep mbarrier pipeline as before; every stage release is preceded
//    by fence.proxy.async (generic reads vs. async-proxy overwrite).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include <vector>

#include "common.cuh"
#include "inft_internal.cuh"
#include "tma.cuh"

namespace inft {

namespace ring {

#ifndef INFT_RING_NB
#define INFT_RING_NB 16
#endif
#ifndef INFT_RING_STAGES
#define INFT_RING_STAGES 2
#endif
#ifndef INFT_RING_MINB
#define INFT_RING_MINB 1
#endif
constexpr int kQ = 32;                     // segments per chunk (one CTA)
// spread table modes (ring_spread_table)
constexpr int kSidePart = 1;   // node range of a heavy segment: own half and spill to side slots
constexpr int kSideNoPro = 2;  // previous segment heavy: no prologue (its parts' spills are added)
constexpr int kSideCarry = 4;  // next segment heavy: spill into s1 to a side slot
constexpr int kNB = INFT_RING_NB;          // nodes per staged batch
constexpr int kStages = INFT_RING_STAGES;  // spread load pipeline depth (2: more CTAs per SM beat a deeper pipe)
#ifndef INFT_RING_STAGES_G
#define INFT_RING_STAGES_G 2
#endif
// gather window pipeline depth: complex128 2 (config 5, aligned output ring: 2 -> 0.894 ms at 6
// CTAs/SM, 3 -> 0.938 at 5); complex64 3 (its 4-KB window boxes: 0.567 -> 0.534 ms, 8 CTAs/SM)
#ifndef INFT_RING_STAGES_GF
#define INFT_RING_STAGES_GF 3
#endif
template <typename T>
constexpr int stages_g() { return sizeof(T) == 8 ? INFT_RING_STAGES_G : INFT_RING_STAGES_GF; }
// gather window ring in 4-KB boxes (one mbarrier pair per box).  complex128 with m = 8 (two
// boxes per segment): 3 boxes = 1.5 segments ahead instead of 2 whole-segment stages (4 boxes):
// 33.3 -> 29.2 KB per CTA, and with the node-record ring in half batches 8 CTAs per SM instead of 6
#ifndef INFT_RING_WBOXES_G
#define INFT_RING_WBOXES_G 3
#endif
// complex64 spread: a full batch on an odd node reads its last f value from the next batch's
// tile instead of fetching a second box of its own (0: always the own box)
#ifndef INFT_SPREAD_BORROW
#define INFT_SPREAD_BORROW 1
#endif
constexpr bool kBorrowTail = INFT_SPREAD_BORROW != 0;
// gather: one-phase window (register moves per slide, one copy of the bodies) or the two-phase
// register ring (0)
#ifndef INFT_GATHER_1PH
#define INFT_GATHER_1PH 1
#endif
constexpr bool kOnePhase = INFT_GATHER_1PH != 0;
// dense gather body: explicit double buffer of the weight vectors (experiment)
#ifndef INFT_GATHER_WPRE
#define INFT_GATHER_WPRE 0
#endif
constexpr bool kGatherWPre = INFT_GATHER_WPRE != 0;
#ifndef INFT_GATHER_LATE_WAIT
#define INFT_GATHER_LATE_WAIT 1
#endif
constexpr bool kLateWait = INFT_GATHER_LATE_WAIT != 0;
template <typename T, int SBOX>
constexpr int win_boxes() {
    return (sizeof(T) == 8 && SBOX == 2) ? INFT_RING_WBOXES_G : stages_g<T>() * SBOX;
}
#ifndef INFT_RING_STAGES_GR
#define INFT_RING_STAGES_GR 2
#endif
// gather node-record pipeline depth: 2 keeps a CTA at <= 37 KB of shared memory (6 CTAs per SM
// instead of 5 with 3 record stages)
constexpr int kStagesGR = INFT_RING_STAGES_GR;

// experiment (timing only, wrong results): INFT_EXP_NOCOMPUTE=1 -- the dense gather body copies
// window values to the outputs (no weight loads, no FMAs): the kernel's data-movement skeleton
#ifndef INFT_EXP_NOCOMPUTE
#define INFT_EXP_NOCOMPUTE 0
#endif
constexpr bool kExpNoCompute = INFT_EXP_NOCOMPUTE != 0;
#define INFT_CASES_64(X)                                                                                      \
    X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) X(18)   \
    X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32) X(33) X(34) X(35)     \
    X(36) X(37) X(38) X(39) X(40) X(41) X(42) X(43) X(44) X(45) X(46) X(47) X(48) X(49) X(50) X(51) X(52)     \
    X(53) X(54) X(55) X(56) X(57) X(58) X(59) X(60) X(61) X(62) X(63)

// Tensor-map coordinate of complex column c (8-byte elements per complex = CE).
// Routed through an opaque mov: with CE == 1 (complex64) ptxas otherwise folds
// the coordinate into the uniform-register tuple of UTMALDG/UTMASTG in a way
// that faulted at run time (illegal instruction) on sm_100a.
template <int CE>
__device__ __forceinline__ int tcoord(int c) {
    int v = c * CE;
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}

// byte offset of complex value v (0..) of this lane's row inside a sequence of
// SWIZZLE_128B boxes of 32 rows (box = 32 x 128 bytes); sw = lane*128 | (lane&7)<<4
template <typename T>
__device__ __forceinline__ uint32_t cofs(int v, uint32_t sw) {
    constexpr int EB = 128 / (int)sizeof(C2<T>);
    const int bx = v / EB, c = v % EB;
    if (sizeof(C2<T>) == 16) return (uint32_t)bx * 4096u + (sw ^ ((uint32_t)c << 4));
    return (uint32_t)bx * 4096u + (sw ^ ((uint32_t)(c >> 1) << 4)) + (uint32_t)(c & 1) * 8u;
}

// Complex accumulator / window value: two doubles (two DFMA per tap), or a packed float pair for
// complex64, updated by ONE sm_100 paired FMA per tap (FFMA2: both lanes of the pair times the
// real weight as a scalar operand) -- the same two correctly rounded fused products as two FFMA.
template <typename T>
struct CA;
template <>
struct CA<double> {
    double x, y;
};
template <>
struct CA<float> {
    unsigned long long v;
};
__device__ __forceinline__ CA<double> ca_zero(double) { return CA<double>{0.0, 0.0}; }
__device__ __forceinline__ CA<float> ca_zero(float) { return CA<float>{0ull}; }
__device__ __forceinline__ CA<double> ca_from(C2<double> g) { return CA<double>{g.x, g.y}; }
__device__ __forceinline__ CA<float> ca_from(C2<float> g) {
    return CA<float>{((unsigned long long)__float_as_uint(g.y) << 32) | __float_as_uint(g.x)};
}
__device__ __forceinline__ C2<double> ca_to(CA<double> a) { return mk<double>(a.x, a.y); }
__device__ __forceinline__ C2<float> ca_to(CA<float> a) {
    return mk<float>(__uint_as_float((unsigned)(a.v & 0xffffffffull)), __uint_as_float((unsigned)(a.v >> 32)));
}
// a += w v
__device__ __forceinline__ void ca_fma(CA<double>& a, double w, CA<double> v) {
    a.x = fma(w, v.x, a.x);
    a.y = fma(w, v.y, a.y);
}
__device__ __forceinline__ void ca_fma(CA<float>& a, float w, CA<float> v) {
    const unsigned long long wp = ((unsigned long long)__float_as_uint(w) << 32) | __float_as_uint(w);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a.v) : "l"(v.v), "l"(wp));
}
// C2 load straight into the accumulator type (complex64: one 8-byte load)
template <typename T>
__device__ __forceinline__ CA<T> ca_load(const unsigned char* p) {
    return ca_from(*reinterpret_cast<const C2<T>*>(p));
}

// ------------------------------------------------------------------------- spread
template <typename T, int MC>
__global__ void __launch_bounds__(128, INFT_RING_MINB) k_spread_ring(const __grid_constant__ CUtensorMap fmap,
                                                     const __grid_constant__ CUtensorMap gmap,
                                                     const int32_t* __restrict__ seg_start,
                                                     const int32_t* __restrict__ chunks,
                                                     const T* __restrict__ w, int PPrt, int nseg, int Q, int N,
                                                     int cshift, C2<T>* __restrict__ side, int R) {
    constexpr int SEG = 2 * MC;
    constexpr int VEC = 16 / (int)sizeof(T);
    constexpr int PP = ((2 * MC + 2 + VEC - 1) / VEC) * VEC;  // record stride (host: Plan::PP)
    constexpr int K = 2 * SEG;
    constexpr int P = 2 * MC + 1;
    constexpr int EB = 128 / (int)sizeof(C2<T>);
    constexpr int CE = (int)sizeof(C2<T>) / 8;
    constexpr int NBOX = kNB / EB;   // f boxes per batch
    // complex64: a box may only start at an even node (16-byte aligned innermost start; an
    // 8-byte aligned start faults), so the batch's f tile is fetched from the even node at or
    // before it with one extra box and read at offset (col & 1)
    constexpr int NBF = NBOX + (CE == 1 ? 1 : 0);
    constexpr int SBOX = SEG / EB;   // store boxes per segment
    static_assert(SEG % EB == 0 && kNB % EB == 0, "tile shapes");
    const int WPB = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sw = ((uint32_t)lane << 7) | ((uint32_t)(lane & 7) << 4);

    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t fstage = (uint32_t)NBF * WPB * 4096u;  // [NBF][rows][128]
    const uint32_t rstage = (uint32_t)((kNB * PP * (int)sizeof(T) + 127) & ~127);
    unsigned char* fbuf = smem;
    unsigned char* stg = smem + kStages * fstage;                 // [WPB][SBOX][32][128]
    unsigned char* rbuf = stg + (size_t)WPB * SBOX * 4096u;
    uint64_t* full = reinterpret_cast<uint64_t*>(rbuf + kStages * rstage);
    uint64_t* empty = full + kStages;
    unsigned char* my_stg = stg + (size_t)warp * SBOX * 4096u;

    // chunk = Q segments, or an entry (s0, s1, first node, end node, mode, slot) of the spread
    // table (ring_spread_table): node-balanced runs of segments, and heavy segments split into
    // node ranges whose windows go to side slots (kSidePart); a run next to a heavy segment
    // skips the prologue (kSideNoPro) and/or parks its spill into segment s1 (kSideCarry);
    // k_spread_ring_fix adds the side slots in a fixed order
    // grid (row groups, chunks): the row groups of one chunk run side by side, so the second
    // reads the chunk's node records from L2
    const int cid = (int)blockIdx.y;
    const int* ce = chunks + 6 * cid;
    const int s0 = chunks ? __ldg(ce) : cid * Q;
    const int s1 = chunks ? __ldg(ce + 1) : min(s0 + Q, nseg);
    const int mode = chunks ? __ldg(ce + 4) : 0;
    const int slot = chunks ? __ldg(ce + 5) : 0;
    const int sp = s0 == 0 ? nseg - 1 : s0 - 1;
    const bool pro_on = !(mode & (kSideNoPro | kSidePart));
    const int a0 = pro_on ? __ldg(seg_start + sp) : 0, a1 = pro_on ? __ldg(seg_start + sp + 1) : 0;
    const int b0 = chunks ? __ldg(ce + 2) : __ldg(seg_start + s0);
    const int b1 = chunks ? __ldg(ce + 3) : __ldg(seg_start + s1);
    const int wrap = N - cshift;
    const int aw = (cshift > 0 && a0 < wrap && wrap < a1) ? wrap : a1;
    const int bw = (cshift > 0 && b0 < wrap && wrap < b1) ? wrap : b1;
    const int c1 = (aw - a0 + kNB - 1) / kNB;
    const int c2 = c1 + (a1 - aw + kNB - 1) / kNB;
    const int c3 = c2 + (bw - b0 + kNB - 1) / kNB;
    const int nb = c3 + (b1 - bw + kNB - 1) / kNB;
    auto batch_pos = [&](int b, int& pos, int& cnt, bool& pro) {
        int s, e, base;
        if (b < c1) { s = a0; e = aw; base = 0; pro = true; }
        else if (b < c2) { s = aw; e = a1; base = c1; pro = true; }
        else if (b < c3) { s = b0; e = bw; base = c2; pro = false; }
        else { s = bw; e = b1; base = c3; pro = false; }
        pos = s + (b - base) * kNB;
        cnt = min(kNB, e - pos);
    };
    const int row0 = (int)blockIdx.x * WPB * 32;
    // complex64: does batch b fetch its own extra box?  Only a full batch on an odd node reads
    // past its first NBOX boxes (its last node), and when the next batch's tile starts right
    // there (consecutive batches of one node range -- every batch of config 5) that node is read
    // from the next stage's tile instead: one box per batch, not two (the second box was an L2
    // hit, but the spread moves ~6 TB/s between L2 and the SMs with or without the FMAs).
    auto own_tail = [&](int b, int pos, int cnt) -> int {  // 0: no 17th value, 1: own box, 2: next stage
        if (CE != 1) return 0;
        int col = pos + cshift;
        if (col >= N) col -= N;
        if (!(col & 1) || cnt < kNB) return 0;
        if (!kBorrowTail || b + 1 >= nb) return 1;
        int p2, c2n;
        bool pr2;
        batch_pos(b + 1, p2, c2n, pr2);
        int col2 = p2 + cshift;
        if (col2 >= N) col2 -= N;
        return (col2 & ~1) == (col & ~1) + kNB ? 2 : 1;
    };
    auto issue = [&](int b, int stage) {
        int pos, cnt;
        bool pro;
        batch_pos(b, pos, cnt, pro);
        const uint32_t rbytes = (uint32_t)(cnt * PP * (int)sizeof(T));
        int col = pos + cshift;
        if (col >= N) col -= N;
        if (CE == 1) col &= ~1;
        const int nbx = CE == 1 ? NBOX + (own_tail(b, pos, cnt) == 1 ? 1 : 0) : NBF;
        mbar_arrive_expect_tx(&full[stage], (uint32_t)nbx * WPB * 4096u + rbytes);
        for (int wi = 0; wi < WPB; ++wi)
            for (int bx = 0; bx < nbx; ++bx)
                tma_load_2d(fbuf + stage * fstage + (wi * NBF + bx) * 4096u, &fmap, tcoord<CE>(col + bx * EB),
                            row0 + wi * 32, &full[stage]);
        bulk_g2s(rbuf + stage * rstage, w + (int64_t)pos * PP, rbytes, &full[stage]);
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], WPB);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int b = 0; b < min(kStages, nb); ++b) issue(b, b);

    CA<T> acc[K];
#pragma unroll
    for (int u = 0; u < K; ++u) acc[u] = ca_zero(T(0));
    int cur_k = 0;  // 0 = prologue segment sp, k >= 1 = main segment s0 + k - 1; phase = cur_k & 1
    const int rstore = row0 + warp * 32;

    // finish segment cur_k: store its own half (main segments only), zero it, advance.
    // The half is selected by a branch (never a runtime register index).
    // side slot q of this lane's row: [q][R][SEG] complex (plain stores: 16 consecutive values)
    auto side_store = [&](int q, int H0) {
        if (row0 + (int)threadIdx.x < R) {
            C2<T>* dst = side + ((int64_t)q * R + row0 + threadIdx.x) * SEG;
#pragma unroll
            for (int u = 0; u < SEG; ++u) dst[u] = ca_to(acc[H0 + u]);
        }
    };
    auto store_half = [&](auto HALF) {
        constexpr int H0 = decltype(HALF)::value * SEG;
        if (cur_k >= 1 && (mode & kSidePart)) {
            side_store(2 * slot, H0);  // a part of a heavy segment: its own half to the side
        } else if (cur_k >= 1) {
            if (lane == 0) bulk_wait_read<0>();  // staging tile free again
            __syncwarp();
#pragma unroll
            for (int u = 0; u < SEG; ++u)
                *reinterpret_cast<C2<T>*>(my_stg + cofs<T>(u, sw)) = ca_to(acc[H0 + u]);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                const int col = (s0 + cur_k - 1) * SEG;
#pragma unroll
                for (int bx = 0; bx < SBOX; ++bx) tma_store_2d(&gmap, tcoord<CE>(col + bx * EB), rstore, my_stg + bx * 4096u);
                bulk_commit();
            }
        }
#pragma unroll
        for (int u = 0; u < SEG; ++u) acc[H0 + u] = ca_zero(T(0));
    };
    // (the spread keeps a shifting window: a two-phase register ring costs more
    //  registers here than the SEG moves per segment it saves)
    auto flush = [&]() {
        store_half(std::integral_constant<int, 0>{});
#pragma unroll
        for (int u = 0; u < K; ++u) acc[u] = (u + SEG < K) ? acc[u + SEG] : ca_zero(T(0));
        ++cur_k;
    };

    const uint32_t frow = (uint32_t)warp * NBF * 4096u;  // this warp's boxes inside a stage
    for (int b = 0; b < nb; ++b) {
        const int stage = b % kStages;
        const uint32_t parity = (uint32_t)((b / kStages) & 1);
        int pos, cnt;
        bool pro;
        batch_pos(b, pos, cnt, pro);
        mbar_wait(&full[stage], parity);
        const unsigned char* fb = fbuf + stage * fstage + frow;
        const T* rec = reinterpret_cast<const T*>(rbuf + stage * rstage);
        int fo = 0;  // complex64: offset of the batch's first node inside the fetched tile
        const unsigned char* ft = fb + NBOX * 4096u;  // values kNB.. of the tile: the extra box
        if (CE == 1) {
            int col = pos + cshift;
            if (col >= N) col -= N;
            fo = col & 1;
            if (own_tail(b, pos, cnt) == 2) {  // ... or the next batch's tile (see own_tail)
                const int b2 = b + 1;
                mbar_wait(&full[b2 % kStages], (uint32_t)((b2 / kStages) & 1));
                ft = fbuf + (b2 % kStages) * fstage + frow;
            }
        }
        auto f_at = [&](int v) { return v < kNB ? fb + cofs<T>(v, sw) : ft + cofs<T>(v - kNB, sw); };
        // Dense batch: the kNB nodes are exactly one segment with slot offsets
        // 0..SEG-1 (jittered nodes with N = M_sigma).  Straight-line code, no
        // per-node dispatch: node q adds into window registers q .. q+2m.
        bool dense = false;
        if constexpr (SEG == kNB) {
            if (cnt == kNB) {
                // node q of the batch at offset q of one segment: every slot base checked (first
                // and last alone do not exclude a repeated offset beside a skipped one)
                const unsigned fa = (unsigned)rec_n0(rec, P);
                const unsigned nq = (unsigned)rec_n0(rec + (lane & (kNB - 1)) * PP, P);
                dense = __all_sync(0xffffffffu, (fa % SEG == 0) && nq == fa + (unsigned)(lane & (kNB - 1)));
            }
        }
        if (dense) {
            const int seg = (int)((unsigned)rec_n0(rec, P) / SEG);
            const int kq = pro ? 0 : seg - s0 + 1;
            while (cur_k < kq) flush();
#pragma unroll
            for (int q = 0; q < kNB; ++q) {
                const CA<T> fv = ca_load<T>(q + 1 < kNB ? fb + cofs<T>(q + fo, sw) : f_at(q + fo));
                if constexpr (kExpNoCompute) {  // timing experiment: the data-movement skeleton
                    acc[q] = fv;
                    continue;
                }
                T wv[P];
                WeightLoader<T, P>::load_smem(rec + q * PP, wv);
#pragma unroll
                for (int t = 0; t < P; ++t) {
                    if (q + t < K) ca_fma(acc[q + t], wv[t], fv);
                }
            }
            cnt = 0;  // skip the general loop
        }
        unsigned n0n = cnt ? (unsigned)rec_n0(rec, P) : 0u;
        for (int q = 0; q < cnt; ++q, rec += PP) {
            const unsigned n0 = n0n;
            if (q + 1 < cnt) n0n = (unsigned)rec_n0(rec + PP, P);
            const int seg = (int)(n0 / SEG);
            const int dl = (int)(n0 % SEG);
            const int kq = pro ? 0 : seg - s0 + 1;
            while (cur_k < kq) flush();
            const CA<T> fv = ca_load<T>(f_at(q + fo));
            T wv[P];
            WeightLoader<T, P>::load_smem(rec, wv);
            switch (dl) {
#define INFT_RS_CASE(D)                                                    \
    case D: {                                                              \
        if constexpr (D < SEG) {                                           \
            _Pragma("unroll") for (int t = 0; t < P; ++t) {                \
                ca_fma(acc[D + t], wv[t], fv);                             \
            }                                                              \
        }                                                                  \
    } break;
                INFT_CASES_32(INFT_RS_CASE)
#undef INFT_RS_CASE
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
    // the window's first half now holds the spill into segment s1
    if (mode & kSidePart) side_store(2 * slot + 1, 0);
    if (mode & kSideCarry) side_store(slot, 0);
    if (lane == 0) bulk_wait<0>();
}

// Side slots back into the grid (after k_spread_ring; one thread per (entry, row, u)):
// entry (t, kind, p0, p1, q0, q1, c, -) --
//   kind 0, heavy segment t: grid[t] = spill in + sum_{p0..p1} own(p), spill in = carry slot c
//           of the run ending at t, or (c < 0, t - 1 heavy too) sum_{q0..q1} spill(q);
//   kind 1, segment t after a heavy one: grid[t] += sum_{q0..q1} spill(q).
// Parts are slots 2p (own) / 2p + 1 (spill); carries are single slots; fixed summation order.
template <typename T, int SEG>
__global__ void k_spread_ring_fix(const int32_t* __restrict__ fix, int nfix, const C2<T>* __restrict__ side,
                                  C2<T>* __restrict__ grid, int64_t GS, int R) {
    const int64_t total = (int64_t)nfix * R * SEG;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int u = (int)(idx % SEG);
        const int64_t rr = idx / SEG;
        const int r = (int)(rr % R);
        const int e = (int)(rr / R);
        const int* f = fix + 8 * e;
        const int t = f[0], kind = f[1], p0 = f[2], p1 = f[3], q0 = f[4], q1 = f[5], c = f[6];
        auto at = [&](int q) { return side[((int64_t)q * R + r) * SEG + u]; };
        T x = 0, y = 0;
        if (kind == 0 && c >= 0) {
            const C2<T> v = at(c);
            x = v.x;
            y = v.y;
        } else {
            for (int q = q0; q < q1; ++q) {
                const C2<T> v = at(2 * q + 1);
                x += v.x;
                y += v.y;
            }
        }
        C2<T>* g = grid + (int64_t)r * GS + (int64_t)t * SEG + u;
        if (kind == 0) {
            for (int q = p0; q < p1; ++q) {
                const C2<T> v = at(2 * q);
                x += v.x;
                y += v.y;
            }
            *g = mk<T>(x, y);
        } else {
            const C2<T> v = *g;
            *g = mk<T>(v.x + x, v.y + y);
        }
    }
}

// ------------------------------------------------------------------------- gather
template <typename T, int MC>
__global__ void __launch_bounds__(128, INFT_RING_MINB) k_gather_ring(const __grid_constant__ CUtensorMap gmap,
                                                     const __grid_constant__ CUtensorMap omap,
                                                     const int32_t* __restrict__ seg_start,
                                                     const int32_t* __restrict__ chunks,
                                                     const T* __restrict__ w, int PPrt, C2<T>* __restrict__ f,
                                                     int64_t Nl, int nseg, int Q, int R, int cshift) {
    constexpr int SEG = 2 * MC;
    constexpr int VEC = 16 / (int)sizeof(T);
    constexpr int PP = ((2 * MC + 2 + VEC - 1) / VEC) * VEC;
    constexpr int K = 2 * SEG;
    constexpr int P = 2 * MC + 1;
    constexpr int EB = 128 / (int)sizeof(C2<T>);
    constexpr int CE = (int)sizeof(C2<T>) / 8;
    constexpr int SBOX = SEG / EB;  // window boxes per segment
    constexpr int OBOX = kNB / EB;  // output boxes per batch
    // output staging ring of NR boxes: output column c (caller node order) lives in ring slot
    // c mod RS, and only whole, 128-byte-aligned boxes of f leave by TMA store.  The sorted
    // node order is a cyclic shift of the caller's (perm_shift, odd for config 5), so batch-
    // aligned boxes started mid-sector: every 128-byte box row touched 5 sectors with two
    // partial ones (ncu: 1.25x the write sectors, L2 read-modify-writes).  The columns before a
    // run's first aligned box and after its last one are stored from the ring by plain stores.
    constexpr int NR = OBOX + 1;
    constexpr int RS = NR * EB;
    constexpr int NWB = win_boxes<T, SBOX>();  // window ring, in boxes
    static_assert(SEG % EB == 0 && kNB % EB == 0, "tile shapes");
    const int N = (int)Nl;
    const int WPB = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sw = ((uint32_t)lane << 7) | ((uint32_t)(lane & 7) << 4);
    const int row0 = (int)blockIdx.x * WPB * 32;
    const int r = row0 + threadIdx.x;
    const bool active = r < R;

    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t wbox = (uint32_t)WPB * 4096u;  // one ring slot: a box per warp
    const uint32_t rstage = (uint32_t)((kNB * PP * (int)sizeof(T) + 127) & ~127);
    unsigned char* wbuf = smem;
    unsigned char* stg = smem + NWB * wbox;  // [WPB][NR][32][128]
    unsigned char* rbuf = stg + (size_t)WPB * NR * 4096u;
    uint64_t* fullW = reinterpret_cast<uint64_t*>(rbuf + kStagesGR * rstage);
    uint64_t* emptyW = fullW + NWB;
    uint64_t* fullR = emptyW + NWB;
    uint64_t* emptyR = fullR + kStagesGR;
    unsigned char* my_stg = stg + (size_t)warp * NR * 4096u;

    // chunk = Q segments, or a node-balanced run of segments from the chunk table
    // chunk = Q segments, or an entry (s0, s1, first node, end node) of the gather's chunk
    // table: node-balanced runs of segments, and heavy segments split into node ranges
    const int cid = (int)blockIdx.y;  // grid (row groups, chunks), as the spread
    const int s0 = chunks ? __ldg(chunks + 4 * cid) : cid * Q;
    const int s1 = chunks ? __ldg(chunks + 4 * cid + 1) : min(s0 + Q, nseg);
    const int nbox = s1 - s0 + 1;  // window L = grid points of segment s0 + L (halo covers L = nseg)
    const int nwb = nbox * SBOX;   // ... = boxes L SBOX .. L SBOX + SBOX - 1
    const int b0 = chunks ? __ldg(chunks + 4 * cid + 2) : __ldg(seg_start + s0);
    const int b1 = chunks ? __ldg(chunks + 4 * cid + 3) : __ldg(seg_start + s1);
    const int wrap = N - cshift;
    const int bw = (cshift > 0 && b0 < wrap && wrap < b1) ? wrap : b1;
    const int c1 = (bw - b0 + kNB - 1) / kNB;
    const int nbat = c1 + (b1 - bw + kNB - 1) / kNB;
    auto batch_pos = [&](int b, int& pos, int& cnt) {
        if (b < c1) {
            pos = b0 + b * kNB;
            cnt = min(kNB, bw - pos);
        } else {
            pos = bw + (b - c1) * kNB;
            cnt = min(kNB, b1 - pos);
        }
    };
    auto issueW = [&](int bi, int stage) {
        mbar_arrive_expect_tx(&fullW[stage], wbox);
        const int col = s0 * SEG + bi * EB;
        for (int wi = 0; wi < WPB; ++wi)
            tma_load_2d(wbuf + stage * wbox + wi * 4096u, &gmap, tcoord<CE>(col), row0 + wi * 32, &fullW[stage]);
    };
    auto issueR = [&](int b, int stage) {
        int pos, cnt;
        batch_pos(b, pos, cnt);
        const uint32_t rbytes = (uint32_t)(cnt * PP * (int)sizeof(T));
        mbar_arrive_expect_tx(&fullR[stage], rbytes);
        bulk_g2s(rbuf + stage * rstage, w + (int64_t)pos * PP, rbytes, &fullR[stage]);
    };

    if (threadIdx.x == 0) {
        prefetch_tmap(&gmap);
        prefetch_tmap(&omap);
        for (int i = 0; i < NWB; ++i) {
            mbar_init(&fullW[i], 1);
            mbar_init(&emptyW[i], WPB);
        }
        for (int i = 0; i < kStagesGR; ++i) {
            mbar_init(&fullR[i], 1);
            mbar_init(&emptyR[i], WPB);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int bi = 0; bi < min(NWB, nwb); ++bi) issueW(bi, bi);
        for (int b = 0; b < min(kStagesGR, nbat); ++b) issueR(b, b);
    }

    CA<T> win[K];
    int nextL = 0;
    const uint32_t wrow = (uint32_t)warp * 4096u;
    // box L -> registers of half H = L & 1, H a compile-time constant (static register
    // indices: a run-time half made ptxas select every window register with FSEL, 2K extra
    // instructions per box)
    auto consume_box_h = [&](auto HC) {
        constexpr int H = decltype(HC)::value;
        const int L = nextL++;
#pragma unroll
        for (int bx = 0; bx < SBOX; ++bx) {
            const int bi = L * SBOX + bx;
            const int stage = bi % NWB;
            const uint32_t parity = (uint32_t)((bi / NWB) & 1);
            mbar_wait(&fullW[stage], parity);
            const unsigned char* wb = wbuf + stage * wbox + wrow;
#pragma unroll
            for (int v = 0; v < EB; ++v) win[H * SEG + bx * EB + v] = ca_load<T>(wb + cofs<T>(v, sw));
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&emptyW[stage]);
            if (threadIdx.x == 0 && bi + NWB < nwb) {
                mbar_wait(&emptyW[stage], parity);
                issueW(bi + NWB, stage);
            }
        }
    };
    // One phase (INFT_GATHER_1PH, default): the window always starts at register 0 -- a slide
    // moves the upper half down (SEG register moves) and loads the new box into the upper half,
    // so there is ONE copy of the node bodies.  The two-phase register ring (no moves, the
    // bodies specialised on the segment parity) made the dense path's hot code ~60 KB: past the
    // 32-KB instruction cache, 17 % of the warp stall samples were instruction fetches.
    auto consume_box = [&]() {
        if constexpr (kOnePhase) {
            if (nextL == 0) {
                consume_box_h(std::integral_constant<int, 0>{});
            } else {
                if (nextL >= 2) {
#pragma unroll
                    for (int v = 0; v < SEG; ++v) win[v] = win[v + SEG];
                }
                consume_box_h(std::integral_constant<int, 1>{});
            }
        } else if (nextL & 1) {
            consume_box_h(std::integral_constant<int, 1>{});
        } else {
            consume_box_h(std::integral_constant<int, 0>{});
        }
    };
    consume_box();
    consume_box();
    int cur_i = 0;  // window for segment s0 + cur_i: phase cur_i & 1

    C2<T>* __restrict__ fr = f + (int64_t)(active ? r : 0) * N;
    const int rstore = row0 + warp * 32;
    // output run state (warp-uniform): a run is a stretch of consecutive output columns
    // [run_start, run_next); boxes below box_next are stored, columns [run_start, plain_lo) too
    int run_next = -1, run_start = 0, lead_end = 0, plain_lo = 0, box_next = 0;
    auto ring_ofs = [&](int c) { return cofs<T>(c % RS, sw); };
    auto store_plain = [&](int c0, int c1) {  // this lane's row, its own ring slots
        if (active)
            for (int c = c0; c < c1; ++c) fr[c] = *reinterpret_cast<const C2<T>*>(my_stg + ring_ofs(c));
    };
    auto end_run = [&]() {
        const int c0 = max(plain_lo, box_next * EB);
        if (run_next >= 0 && c0 < run_next) store_plain(c0, run_next);
    };
    for (int b = 0; b < nbat; ++b) {
        const int stage = b % kStagesGR;
        const uint32_t parity = (uint32_t)((b / kStagesGR) & 1);
        int pos, cnt;
        batch_pos(b, pos, cnt);
        mbar_wait(&fullR[stage], parity);
        const T* rec = reinterpret_cast<const T*>(rbuf + stage * rstage);
        const bool full_tile = cnt == kNB;
        int col = pos + cshift;
        if (col >= N) col -= N;
        if (col != run_next) {  // a new run (chunk start, the wrap of the node order)
            end_run();
            run_start = col;
            plain_lo = col;
            box_next = (col + EB - 1) / EB;
            lead_end = box_next * EB;
        }
        const int cm = col % RS;  // ring slot of the batch's first output
        // ring slots free: every earlier TMA store has read its box -- waited for just before
        // the batch's first write into the ring (INFT_GATHER_LATE_WAIT=0: at the batch start), so
        // the store's shared-memory read overlaps the window slide and the first node group
        bool ring_ok = false;
        auto ring_wait = [&]() {
            if (!ring_ok) {
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
                ring_ok = true;
            }
        };
        if (!kLateWait) ring_wait();
        bool dense = false;
        if constexpr (SEG == kNB) {
            if (full_tile) {
                // as the spread: every node's slot base checked
                const unsigned fa = (unsigned)rec_n0(rec, P);
                const unsigned nq = (unsigned)rec_n0(rec + (lane & (kNB - 1)) * PP, P);
                dense = __all_sync(0xffffffffu, (fa % SEG == 0) && nq == fa + (unsigned)(lane & (kNB - 1)));
            }
        }
        int ncnt = cnt;
        if (dense) {
            const int seg = (int)((unsigned)rec_n0(rec, P) / SEG);
            const bool step1 = seg - s0 == cur_i + 1;
            if (!step1) {
                while (cur_i < seg - s0) {
                    consume_box();
                    ++cur_i;
                }
            }
            // Tap-major: the QG nodes of a group advance together one tap (vector of VEC
            // weights) at a time, so 2 QG accumulation chains are independent (one chain per
            // output in tap order, as the general path: bit-identical results).  Node-major
            // order left 4 short chains per node and stalled on the FP64 latency at ~6 warps
            // per SM (ncu: 'wait' 37 % of the stalls, FP64 pipe 29 %).
            auto dense_body = [&](auto PHC) {
                constexpr int PH = decltype(PHC)::value;
#ifndef INFT_GATHER_QG
#define INFT_GATHER_QG 8
#endif
                constexpr int QG = INFT_GATHER_QG;  // nodes per group
                static_assert(kNB % QG == 0, "node groups");
#pragma unroll
                for (int g0 = 0; g0 < kNB; g0 += QG) {
                    CA<T> sacc[QG];
#pragma unroll
                    for (int qq = 0; qq < QG; ++qq) sacc[qq] = ca_zero(T(0));
                    if constexpr (kExpNoCompute) {  // timing experiment: the data-movement skeleton
#pragma unroll
                        for (int qq = 0; qq < QG; ++qq) sacc[qq] = win[(g0 + qq + SEG * PH) % K];
                    }
                    // weights t0 .. t0 + VEC - 1 of the group's nodes: one broadcast vector load per
                    // node (slots past P - 1 are the record's tail, never used)
                    auto load_w = [&](T (&wv)[QG][VEC], int t0) {
#pragma unroll
                        for (int qq = 0; qq < QG; ++qq) {
                            if constexpr (VEC == 2) {
                                const double2 a = *reinterpret_cast<const double2*>(rec + (g0 + qq) * PP + t0);
                                wv[qq][0] = a.x;
                                wv[qq][1] = a.y;
                            } else {
                                const float4 a = *reinterpret_cast<const float4*>(rec + (g0 + qq) * PP + t0);
                                wv[qq][0] = a.x;
                                wv[qq][1] = a.y;
                                wv[qq][2] = a.z;
                                wv[qq][3] = a.w;
                            }
                        }
                    };
                    T wvn[QG][VEC];
                    if constexpr (kGatherWPre && !kExpNoCompute) load_w(wvn, 0);
#pragma unroll
                    for (int t0 = 0; t0 < (kExpNoCompute ? 0 : P); t0 += VEC) {
                        T wv[QG][VEC];
                        if constexpr (kGatherWPre) {
                            // explicit double buffer: the next tap vector's loads are issued before
                            // this one's FMAs
#pragma unroll
                            for (int qq = 0; qq < QG; ++qq)
#pragma unroll
                                for (int u = 0; u < VEC; ++u) wv[qq][u] = wvn[qq][u];
                            if (t0 + VEC < P) load_w(wvn, t0 + VEC);
                        } else {
                            load_w(wv, t0);
                        }
#pragma unroll
                        for (int u = 0; u < VEC; ++u) {
                            if (t0 + u < P) {
#pragma unroll
                                for (int qq = 0; qq < QG; ++qq) {
                                    const int rg = (g0 + qq + t0 + u + SEG * PH) % K;
                                    ca_fma(sacc[qq], wv[qq][u], win[rg]);
                                }
                            }
                        }
                    }
                    if (g0 == 0) ring_wait();
#pragma unroll
                    for (int qq = 0; qq < QG; ++qq) {
                        const int sl = cm + g0 + qq;
                        *reinterpret_cast<C2<T>*>(my_stg + cofs<T>(sl >= RS ? sl - RS : sl, sw)) = ca_to(sacc[qq]);
                    }
                }
            };
            // the common case, the batch one segment past the window's first one: slide the
            // window by one box into the half of the current phase (static indices), then run
            // the body in the other phase
            auto slide_body = [&](auto PHC) {
                constexpr int PH = decltype(PHC)::value;
                consume_box_h(std::integral_constant<int, PH>{});
                ++cur_i;
                dense_body(std::integral_constant<int, 1 - PH>{});
            };
            if constexpr (kOnePhase) {
                if (step1) {
                    consume_box();
                    ++cur_i;
                }
                dense_body(std::integral_constant<int, 0>{});
            } else if (step1) {
                if (cur_i & 1)
                    slide_body(std::integral_constant<int, 1>{});
                else
                    slide_body(std::integral_constant<int, 0>{});
            } else if (cur_i & 1) {
                dense_body(std::integral_constant<int, 1>{});
            } else {
                dense_body(std::integral_constant<int, 0>{});
            }
            ncnt = 0;
        }
        unsigned n0n = ncnt ? (unsigned)rec_n0(rec, P) : 0u;
        for (int q = 0; q < ncnt; ++q, rec += PP) {
            const unsigned n0 = n0n;
            if (q + 1 < ncnt) n0n = (unsigned)rec_n0(rec + PP, P);
            const int seg = (int)(n0 / SEG);
            const int dl = (int)(n0 % SEG);
            while (cur_i < seg - s0) {
                consume_box();
                ++cur_i;
            }
            T wv[P];
            WeightLoader<T, P>::load_smem(rec, wv);
            CA<T> sa = ca_zero(T(0));
            switch ((kOnePhase ? 0 : (cur_i & 1)) * 32 + dl) {
#define INFT_RG_CASE(CID)                                                  \
    case CID: {                                                            \
        constexpr int PH = (CID) / 32, D = (CID) % 32;                     \
        if constexpr (D < SEG) {                                           \
            _Pragma("unroll") for (int t = 0; t < P; ++t) {                \
                const int rg = (D + t + SEG * PH) % K;                     \
                ca_fma(sa, wv[t], win[rg]);                                \
            }                                                              \
        }                                                                  \
    } break;
                INFT_CASES_64(INFT_RG_CASE)
#undef INFT_RG_CASE
                default:
                    break;
            }
            const int sl = cm + q;
            ring_wait();
            *reinterpret_cast<C2<T>*>(my_stg + cofs<T>(sl >= RS ? sl - RS : sl, sw)) = ca_to(sa);
        }
        run_next = col + cnt;
        if (plain_lo < lead_end) {  // the run's columns before its first aligned box
            const int c1 = min(lead_end, run_next);
            store_plain(plain_lo, c1);
            plain_lo = c1;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && (box_next + 1) * EB <= run_next) {
            do {
                tma_store_2d(&omap, tcoord<CE>(box_next * EB), rstore, my_stg + (box_next % NR) * 4096u);
                ++box_next;
            } while ((box_next + 1) * EB <= run_next);
            bulk_commit();
        }
        box_next = __shfl_sync(0xffffffffu, box_next, 0);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyR[stage]);
        if (threadIdx.x == 0 && b + kStagesGR < nbat) {
            mbar_wait(&emptyR[stage], parity);
            issueR(b + kStagesGR, stage);
        }
    }
    end_run();
    while (nextL < nbox) consume_box();  // no copy may be in flight at exit
    if (lane == 0) bulk_wait<0>();
}

}  // namespace ring

// =========================================================================== host
template <typename T>
struct RingFns {
    void (*spread)(const CUtensorMap, const CUtensorMap, const int32_t*, const int32_t*, const T*, int, int, int, int,
                   int, C2<T>*, int) = nullptr;
    void (*fix)(const int32_t*, int, const C2<T>*, C2<T>*, int64_t, int) = nullptr;
    void (*gather)(const CUtensorMap, const CUtensorMap, const int32_t*, const int32_t*, const T*, int, C2<T>*, int64_t,
                   int, int, int, int) = nullptr;
};

template <typename T>
static RingFns<T> ring_fns(int m) {
    RingFns<T> F;
    constexpr int EB = 128 / (int)sizeof(C2<T>);
    if constexpr (8 % EB == 0) {
        if (m == 4) {
            F.spread = ring::k_spread_ring<T, 4>;
            F.gather = ring::k_gather_ring<T, 4>;
            F.fix = ring::k_spread_ring_fix<T, 8>;
        }
    }
    if (m == 8) {
        F.spread = ring::k_spread_ring<T, 8>;
        F.gather = ring::k_gather_ring<T, 8>;
        F.fix = ring::k_spread_ring_fix<T, 16>;
    } else if (m == 16) {
        F.spread = ring::k_spread_ring<T, 16>;
        F.gather = ring::k_gather_ring<T, 16>;
        F.fix = ring::k_spread_ring_fix<T, 32>;
    }
    return F;
}

static bool ring_env_disabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("INFT_NO_RING");
        v = (e && atoi(e)) ? 1 : 0;
    }
    return v == 1;
}

// complex64: a tensor-map copy whose innermost start is not 16-byte aligned raises "illegal
// instruction" (measured with tools/tma_probe.cu: start offset 1 x 8 B faults, 2 x 8 B runs),
// and node-side boxes start at arbitrary nodes; k_spread_ring therefore fetches each batch's
// f tile from the even node at or before it (one extra box) and k_gather_ring stores a batch
// that starts on an odd node with plain stores.  INFT_RING_C64=0 routes complex64 to the
// register-window / stream1d kernels instead.
static bool ring_c64_spread_enabled() {
    const char* e = getenv("INFT_RING_C64");
    return !(e && atoi(e) == 0);
}

bool ring_spread_available(const Plan& p) { return ring_available(p); }

bool ring_available(const Plan& p) {
    if (ring_env_disabled() || p.d != 1 || !p.fast1d || p.wt != INFT_WEIGHTS_REAL || p.N == 0 || p.perm_shift < 0)
        return false;
    if (p.S[0] != 2 * p.m) return false;
    if (p.prec == INFT_C64 && !ring_c64_spread_enabled()) return false;
    // chunks are gridDim.y (<= 65535): at most nseg / kQ + the node-balanced / split ones
    if (p.nseg[0] / ring::kQ + 2 * 148 * 64 > 65535) return false;
    // the f / output tensor maps need a row stride (N elements) that is a multiple of 16 bytes
    if ((p.N * (int64_t)p.elem_bytes()) % 16) return false;
    return p.prec == INFT_C128 ? ring_fns<double>(p.m).spread != nullptr : ring_fns<float>(p.m).spread != nullptr;
}

template <typename T>
static int ring_wpb(int64_t R) {
    static const int cap = [] {
        const char* e = getenv("INFT_RING_WPB");
        const int v = e ? atoi(e) : 0;
        return v >= 1 && v <= 4 ? v : 1;  // config 5: 1 warp 5.455 ms/step, 2 warps 5.55
    }();
    return (int)std::min<int64_t>(cap, std::max<int64_t>(1, ceil_div(R, 32)));
}

template <typename T>
static size_t ring_spread_smem(int wpb, int PP, int SEG) {
    const int EB = 128 / (int)sizeof(C2<T>);
    const int nbf = ring::kNB / EB + (sizeof(C2<T>) == 8 ? 1 : 0);  // k_spread_ring's NBF
    size_t f = (size_t)ring::kStages * nbf * wpb * 4096;
    size_t st = (size_t)wpb * (SEG / EB) * 4096;
    size_t r = (size_t)ring::kStages * ((ring::kNB * PP * (int)sizeof(T) + 127) & ~127);
    return f + st + r + 2 * ring::kStages * sizeof(uint64_t);
}

template <typename T>
static size_t ring_gather_smem(int wpb, int PP, int SEG) {
    const int EB = 128 / (int)sizeof(C2<T>);
    const int sbox = SEG / EB;
    const int nwb = (sizeof(T) == 8 && sbox == 2) ? ring::win_boxes<T, 2>() : ring::stages_g<T>() * sbox;
    size_t wsz = (size_t)nwb * wpb * 4096;
    size_t st = (size_t)wpb * (ring::kNB / EB + 1) * 4096;  // output ring (NR boxes per warp)
    size_t r = (size_t)ring::kStagesGR * ((ring::kNB * PP * (int)sizeof(T) + 127) & ~127);
    return wsz + st + r + 2 * (nwb + ring::kStagesGR) * sizeof(uint64_t);
}

static void tmap_or_throw(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t stride,
                          uint32_t box_rows, const char* what) {
    if (!make_tmap_2d(m, base, inner, rows, stride, box_rows)) {
        set_error(std::string("cuTensorMapEncodeTiled failed: ") + what);
        throw Fail{INFT_ERR_CUDA};
    }
}

// target chunk-CTAs per SM over all row groups (INFT_RING_CPS, default 16; config 3 c128:
// 8 -> 0.516 ms/step, 16 -> 0.477, 32 -> 0.469; config 5 unchanged within noise)
static int ring_cps() {
    static const int v = [] {
        const char* e = getenv("INFT_RING_CPS");
        const int x = e ? atoi(e) : 0;
        return x >= 1 && x <= 64 ? x : 16;  // <= 64: chunk counts stay below gridDim.y's limit
    }();
    return v;
}

// Spread table: as ring_gather_chunks (defined below), entries (s0, s1, first node, end node, mode, slot), but
// a heavy segment's node ranges cannot write the grid directly (they share its cells and its
// spill into the next segment): each writes its window halves to side slots, and the runs
// around it skip the prologue / park their spill (kSide*); the fix entries (8 ints, see
// k_spread_ring_fix) sum the side slots into the grid in a fixed order.  Without heavy
// segments this is ring_chunks' table with no side slots.
struct SpreadTable {
    const int32_t* chunks = nullptr;
    const int32_t* fix = nullptr;
    int nchunks = 0, nfix = 0, nslots = 0;
};

// Node target T per chunk.  Chunks close at T nodes or kQ segments; the launch has
// rowgroups x chunks CTAs of about equal work, so the chunk count is rounded to whole waves of
// resident CTAs (INFT_RING_WAVES=0: off) -- a last wave a fifth full cost the config-5 gather ~8 %
// (9.2 waves of 888 CTAs).  T = ceil(N / C) makes the greedy closing produce at most C chunks.
static int64_t ring_target_T(const Plan& p, int64_t rowgroups, const void* fn, int threads, size_t smem) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    rowgroups = std::max<int64_t>(1, rowgroups);
    const int64_t want = std::max<int64_t>(1, (int64_t)nsm * ring_cps() / rowgroups);
    static const bool waves = [] {
        const char* e = getenv("INFT_RING_WAVES");
        return !(e && atoi(e) == 0);
    }();
    if (!waves || !fn) return std::max<int64_t>(1, (p.N + want - 1) / want);
    const int64_t wave = (int64_t)nsm * std::max(1, occupancy_cached(fn, threads, smem));
    int64_t C = std::max<int64_t>(want, ceil_div(p.nseg[0], (int64_t)ring::kQ));
    const int64_t k = ceil_div(C * rowgroups, wave);
    C = std::max<int64_t>(1, k * wave / rowgroups);
    return std::max<int64_t>(1, (p.N + C - 1) / C);
}

static SpreadTable ring_spread_table(Plan& p, int64_t rowgroups, cudaStream_t st, int64_t T) {
    const int64_t key = (int64_t(1) << 40) + T;  // spread tables
    auto it = p.ring_chunk_cache.find(key);
    if (it == p.ring_chunk_cache.end()) {
        const int nseg = (int)p.nseg[0];
        if (p.seg_host.empty()) {
            p.seg_host.resize((size_t)nseg + 1);
            INFT_CUDA(cudaMemcpyAsync(p.seg_host.data(), p.seg_start.p, sizeof(int32_t) * (nseg + 1),
                                      cudaMemcpyDeviceToHost, st));
            INFT_CUDA(cudaStreamSynchronize(st));
        }
        const std::vector<int32_t>& ss = p.seg_host;
        auto heavy = [&](int sg) {
            sg = ((sg % nseg) + nseg) % nseg;
            return ss[sg + 1] - ss[sg] > T;
        };
        // pass 1: runs and parts; part indices per heavy segment
        std::vector<int32_t> c;          // 6 ints per chunk
        std::vector<int> part0(nseg + 1, 0);  // first part index of heavy segment s (prefix)
        int nparts = 0;
        int open = 0;
        int64_t acc = 0;
        auto close = [&](int s1) {
            if (s1 > open) {
                int mode = 0;
                if (heavy(open - 1)) mode |= ring::kSideNoPro;
                if (heavy(s1)) mode |= ring::kSideCarry;
                c.insert(c.end(), {open, s1, ss[open], ss[s1], mode, -1});
            }
            open = s1;
            acc = 0;
        };
        for (int sgi = 0; sgi < nseg; ++sgi) {
            const int64_t n = ss[sgi + 1] - ss[sgi];
            part0[sgi] = nparts;
            if (n > T) {
                close(sgi);
                const int parts = (int)((n + T - 1) / T);
                for (int q = 0; q < parts; ++q)
                    c.insert(c.end(), {sgi, sgi + 1, (int)(ss[sgi] + n * q / parts),
                                       (int)(ss[sgi] + n * (q + 1) / parts), ring::kSidePart, nparts++});
                open = sgi + 1;
                continue;
            }
            acc += n;
            if (acc >= T || sgi + 1 - open >= ring::kQ) close(sgi + 1);
        }
        close(nseg);
        part0[nseg] = nparts;
        // carry slots after the part slots; carry_of[t] = slot of the run ending at t
        int nslots = 2 * nparts;
        std::vector<int> carry_of(nseg, -1);
        for (size_t i = 0; i < c.size(); i += 6)
            if (c[i + 4] & ring::kSideCarry) {
                c[i + 5] = nslots;
                carry_of[c[i + 1] % nseg] = nslots++;
            }
        // fix entries
        std::vector<int32_t> fx;
        for (int t = 0; t < nseg && nparts > 0; ++t) {
            const int tp = (t + nseg - 1) % nseg;
            const bool hp = heavy(tp);
            const int q0 = part0[tp], q1 = part0[tp + 1];
            if (heavy(t)) {
                fx.insert(fx.end(), {t, 0, part0[t], part0[t + 1], hp ? q0 : 0, hp ? q1 : 0, hp ? -1 : carry_of[t], 0});
            } else if (hp) {
                fx.insert(fx.end(), {t, 1, 0, 0, q0, q1, -1, 0});
            }
        }
        Plan::ChunkTable ct;
        ct.n = (int)(c.size() / 6);
        ct.nfix = (int)(fx.size() / 8);
        ct.nslots = nslots;
        std::vector<int32_t> all(c);
        all.insert(all.end(), fx.begin(), fx.end());
        ct.buf.alloc(sizeof(int32_t) * std::max<size_t>(8, all.size()));
        if (!all.empty())
            INFT_CUDA(cudaMemcpyAsync(ct.buf.p, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice, st));
        INFT_CUDA(cudaStreamSynchronize(st));
        it = p.ring_chunk_cache.emplace(key, std::move(ct)).first;
    }
    SpreadTable t;
    t.nchunks = it->second.n;
    t.nfix = it->second.nfix;
    t.nslots = it->second.nslots;
    t.chunks = it->second.buf.as<int32_t>();
    t.fix = t.chunks + 6 * t.nchunks;
    return t;
}

// Chunks of consecutive segments, one CTA each (per row group): balanced by node count, not
// by segment count, so that dense regions (Chebyshev edges) do not set the tail.  A chunk
// closes at >= T nodes or kQ segments, T = N / (~8 CTAs per SM / row groups).  Cached per T.
// Gather chunks (s0, s1, first node, end node): a segment holding more
// than T nodes is split into node ranges of about T (each output is independent in the
// gather; Chebyshev nodes put 651 of 32768 nodes in one segment of config 3).
static const int32_t* ring_gather_chunks(Plan& p, int& nchunks, cudaStream_t st, int64_t T) {
    const int64_t key = -1 - T;  // negative keys: gather tables
    auto it = p.ring_chunk_cache.find(key);
    if (it == p.ring_chunk_cache.end()) {
        const int nseg = (int)p.nseg[0];
        if (p.seg_host.empty()) {
            p.seg_host.resize((size_t)nseg + 1);
            INFT_CUDA(cudaMemcpyAsync(p.seg_host.data(), p.seg_start.p, sizeof(int32_t) * (nseg + 1),
                                      cudaMemcpyDeviceToHost, st));
            INFT_CUDA(cudaStreamSynchronize(st));
        }
        const std::vector<int32_t>& ss = p.seg_host;
        std::vector<int32_t> c;
        int open = 0;  // first segment of the open chunk
        int64_t acc = 0;
        auto close = [&](int s1) {
            if (s1 > open) c.insert(c.end(), {open, s1, ss[open], ss[s1]});
            open = s1;
            acc = 0;
        };
        for (int sgi = 0; sgi < nseg; ++sgi) {
            const int64_t n = ss[sgi + 1] - ss[sgi];
            if (n > T) {  // heavy segment: its own chunks, node ranges of ~T
                close(sgi);
                const int parts = (int)((n + T - 1) / T);
                for (int q = 0; q < parts; ++q)
                    c.insert(c.end(), {sgi, sgi + 1, (int)(ss[sgi] + n * q / parts), (int)(ss[sgi] + n * (q + 1) / parts)});
                open = sgi + 1;
                continue;
            }
            acc += n;
            if (acc >= T || sgi + 1 - open >= ring::kQ) close(sgi + 1);
        }
        close(nseg);
        Plan::ChunkTable ct;
        ct.n = (int)(c.size() / 4);
        ct.buf.alloc(sizeof(int32_t) * std::max<size_t>(4, c.size()));
        if (!c.empty())
            INFT_CUDA(cudaMemcpyAsync(ct.buf.p, c.data(), sizeof(int32_t) * c.size(), cudaMemcpyHostToDevice, st));
        INFT_CUDA(cudaStreamSynchronize(st));
        it = p.ring_chunk_cache.emplace(key, std::move(ct)).first;
    }
    nchunks = it->second.n;
    return it->second.buf.as<int32_t>();
}

template <typename T>
static void ring_spread_t(Plan& p, const void* f, void* grid, int64_t R, cudaStream_t st) {
    RingFns<T> F = ring_fns<T>(p.m);
    const int wpb = ring_wpb<T>(R);
    const int nseg = (int)p.nseg[0];
    const size_t smem = ring_spread_smem<T>(wpb, p.PP, p.S[0]);
    ensure_smem_attr((const void*)F.spread, smem);
    const SpreadTable tb = ring_spread_table(
        p, ceil_div(R, 32 * wpb), st, ring_target_T(p, ceil_div(R, 32 * wpb), (const void*)F.spread, 32 * wpb, smem));
    const int nchunks = tb.nchunks;
    const int32_t* chunks = tb.chunks;
    const size_t side_bytes = sizeof(C2<T>) * (size_t)tb.nslots * (size_t)R * p.S[0];
    if (side_bytes > p.ring_side.bytes) {
        p.ring_side.alloc(side_bytes);
        p.state_version++;
    }
    const uint64_t ce = sizeof(C2<T>) / 8;
    CUtensorMap fm, gm;
    tmap_or_throw(&fm, f, (uint64_t)p.N * ce, (uint64_t)R, sizeof(C2<T>) * (uint64_t)p.N, 32u, "spread f");
    tmap_or_throw(&gm, grid, (uint64_t)p.GS * ce, (uint64_t)R, sizeof(C2<T>) * (uint64_t)p.GS, 32u, "spread grid");
    dim3 g((unsigned)ceil_div(R, 32 * wpb), (unsigned)nchunks);
    F.spread<<<g, 32 * wpb, smem, st>>>(fm, gm, p.seg_start.as<int32_t>(), chunks, p.w.as<T>(), p.PP, nseg, 0,
                                        (int)p.N, p.perm_shift, p.ring_side.as<C2<T>>(), (int)R);
    INFT_CHECK_LAUNCH();
    p.launches++;
    if (tb.nfix > 0) {
        const int64_t total = (int64_t)tb.nfix * R * p.S[0];
        F.fix<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 4096), 256, 0, st>>>(
            tb.fix, tb.nfix, p.ring_side.as<C2<T>>(), static_cast<C2<T>*>(grid), p.GS, (int)R);
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
}

template <typename T>
__global__ void k_ring_halo(C2<T>* __restrict__ grid, int64_t GS, int64_t Ms, int H, int R) {
    const int64_t total = (int64_t)R * H;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / H;
        const int64_t u = idx - r * H;
        grid[r * GS + Ms + u] = grid[r * GS + (u % Ms)];
    }
}

template <typename T>
static void ring_gather_t(Plan& p, const void* grid, void* f, int64_t R, cudaStream_t st) {
    RingFns<T> F = ring_fns<T>(p.m);
    const int wpb = ring_wpb<T>(R);
    const int nseg = (int)p.nseg[0];
    int nchunks = 0;
    const size_t smem = ring_gather_smem<T>(wpb, p.PP, p.S[0]);
    ensure_smem_attr((const void*)F.gather, smem);
    const int32_t* chunks = ring_gather_chunks(
        p, nchunks, st, ring_target_T(p, ceil_div(R, 32 * wpb), (const void*)F.gather, 32 * wpb, smem));
    const uint64_t ce = sizeof(C2<T>) / 8;
    const int H = (int)(p.GS - p.Ms[0]);
    k_ring_halo<T><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(R * H, 256), 4096)), 256, 0, st>>>(
        static_cast<C2<T>*>(const_cast<void*>(grid)), p.GS, p.Ms[0], H, (int)R);
    INFT_CHECK_LAUNCH();
    p.launches++;
    CUtensorMap gm, om;
    tmap_or_throw(&gm, grid, (uint64_t)p.GS * ce, (uint64_t)R, sizeof(C2<T>) * (uint64_t)p.GS, 32u, "gather grid");
    // experiment (timing only, the output is NOT the caller's): INFT_EXP_OSTRIDE=k stores the
    // full batches into a scratch [R][N + k] array (row stride off the power of two)
    static const int ostride = [] {
        const char* e = getenv("INFT_EXP_OSTRIDE");
        return e ? atoi(e) : 0;
    }();
    if (ostride > 0) {
        static DevBuf scratch;
        const size_t need = sizeof(C2<T>) * (size_t)R * (size_t)(p.N + ostride);
        if (scratch.bytes < need) scratch.alloc(need);
        tmap_or_throw(&om, scratch.p, (uint64_t)p.N * ce, (uint64_t)R, sizeof(C2<T>) * (uint64_t)(p.N + ostride), 32u,
                      "gather f (experiment)");
    } else {
        tmap_or_throw(&om, f, (uint64_t)p.N * ce, (uint64_t)R, sizeof(C2<T>) * (uint64_t)p.N, 32u, "gather f");
    }
    dim3 g((unsigned)ceil_div(R, 32 * wpb), (unsigned)nchunks);
    F.gather<<<g, 32 * wpb, smem, st>>>(gm, om, p.seg_start.as<int32_t>(), chunks, p.w.as<T>(), p.PP,
                                        static_cast<C2<T>*>(f), p.N, nseg, 0, (int)R, p.perm_shift);
    INFT_CHECK_LAUNCH();
    p.launches++;
}

void spread_ring(Plan& p, const void* f, void* grid, int64_t R, cudaStream_t st) {
    if (p.prec == INFT_C128)
        ring_spread_t<double>(p, f, grid, R, st);
    else
        ring_spread_t<float>(p, f, grid, R, st);
}

void gather_ring(Plan& p, const void* grid, void* f, int64_t R, cudaStream_t st) {
    if (p.prec == INFT_C128)
        ring_gather_t<double>(p, grid, f, R, st);
    else
        ring_gather_t<float>(p, grid, f, R, st);
}

}  // namespace inft
