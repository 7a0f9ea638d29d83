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

#include "common.cuh"
#include "inft_internal.cuh"

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
    if (ring_available(p)) {
        gather_ring(p, grid, f, R, st);
        return;
    }
    if (stream1d_available(p)) {
        gather_stream1d(p, grid, f, R, st);
        return;
    }
    const T* w = p.w.as<T>();
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

static bool use_fused(const Plan& p) { return !p.no_fused_fft && fused_fft_available(p); }

// One device-resident chunk (Rc <= grid capacity) of the inverse: a2 -> a3 -> a4.
template <typename T>
static void inverse_chunk(Plan& p, const void* f, void* fhat, int64_t Rc, cudaStream_t st) {
    ensure_grid(p, Rc);
    C2<T>* g = p.grid.as<C2<T>>();
    {
        StageTimer t(p, 0, st);
        spread<T>(p, static_cast<const C2<T>*>(f), g, Rc, st);
    }
    if (use_fused(p)) {  // a3 + a4 in two fused passes (fft.cu)
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
