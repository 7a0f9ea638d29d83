// Plan construction, B_opt import/export and the C ABI entry points.
//
// a0: validate nodes (P:37 x_j in [-1/2, 1/2)), l0_j = ceil(M_sigma x_j) - m per
// dimension (index set P:768-774; the product is one correctly rounded
// __dmul_rn, reading A20), tile bins and the stable permutation by bin
// (reading A19), and the deconvolution table d_k = s / (M_sigma what(k))
// (eq. matrix_D; KB pair reading A7).
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include <mutex>
#include <map>
#include <tuple>
#include <unordered_map>
#include "inft_internal.cuh"

namespace inft {

static thread_local std::string g_last_error;
// Dynamic shared-memory attribute set once per (kernel, largest size so far) and occupancy
// queried once per (kernel, threads, smem): both are driver calls on every apply otherwise.
// Keyed by (device, kernel): the attribute is per device context, so a second plan on another
// GPU in the same process must set it again.
static std::mutex g_attr_mu;
static int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    return dev;
}
void ensure_smem_attr(const void* fn, size_t smem) {
    static std::map<std::pair<int, const void*>, size_t> done;
    const auto key = std::make_pair(current_device(), fn);
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= smem) return;
    INFT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done[key] = smem;
}

int occupancy_cached(const void* fn, int threads, size_t smem) {
    static std::map<std::tuple<int, const void*, int, size_t>, int> done;
    auto key = std::make_tuple(current_device(), fn, threads, smem);
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto it = done.find(key);
    if (it != done.end()) return it->second;
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess) occ = 1;
    occ = occ < 1 ? 1 : occ;
    done[key] = occ;
    return occ;
}

bool getenv_flag(const char* name) {
    const char* e = getenv(name);
    return e && atoi(e) != 0;
}

bool sync_check_enabled() {
    static const bool on = [] {
        const char* e = getenv("INFT_SYNC_CHECK");
        return e && atoi(e) != 0;
    }();
    return on;
}

void set_error(const std::string& msg) { g_last_error = msg; }

void DevBuf::alloc(size_t b) {
    free_();
    if (b == 0) return;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
        p = nullptr;
        set_error(std::string("cudaMalloc(") + std::to_string(b) + "): " + cudaGetErrorString(e));
        cudaGetLastError();
        throw Fail{INFT_ERR_OOM};
    }
    bytes = b;
}

void DevBuf::free_() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

size_t Plan::workspace_bytes() const {
    size_t t = nodes.bytes + l0.bytes + bin.bytes + perm.bytes + seg_start.bytes + n0s.bytes +
               delta.bytes + dk.bytes + dkf.bytes + w.bytes + w64.bytes + grid.bytes + fT.bytes + ring_side.bytes;
    for (int i = 0; i < 2; i++) t += stage_in[i].bytes + stage_out[i].bytes;
    for (auto& kv : fft) {
        size_t ws = 0;
        if (cufftGetSize(kv.second, &ws) == CUFFT_SUCCESS) t += ws;
    }
    return t;
}

cudaEvent_t Plan::take_event() {
    if (!ev_pool.empty()) {
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    INFT_CUDA(cudaEventCreate(&e));
    return e;
}

void Plan::drain_profile() {
    for (auto& r : recs) {
        float ms = 0.f;
        INFT_CUDA(cudaEventSynchronize(r.b));
        INFT_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        prof_ms[r.stage] += ms;
        prof_cnt[r.stage] += 1;
        ev_pool.push_back(r.a);
        ev_pool.push_back(r.b);
    }
    recs.clear();
}

Plan::~Plan() {
    DeviceGuard g(device);
    release_fft_state(this);
    for (auto& r : recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto& kv : fft) cufftDestroy(kv.second);
    fft.clear();
    for (auto& kv : graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
    if (s_graph) cudaStreamDestroy(s_graph);
    if (ev_g0) cudaEventDestroy(ev_g0);
    if (ev_g1) cudaEventDestroy(ev_g1);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    for (int i = 0; i < 2; i++) {
        if (ev_h2d[i]) cudaEventDestroy(ev_h2d[i]);
        if (ev_comp[i]) cudaEventDestroy(ev_comp[i]);
        if (ev_d2h[i]) cudaEventDestroy(ev_d2h[i]);
    }
    if (ev_entry) cudaEventDestroy(ev_entry);
    if (ev_exit) cudaEventDestroy(ev_exit);
}

bool is_device_pointer(const void* ptr) {
    return pointer_device(ptr) >= 0;
}

// Device ordinal of a device (or managed) pointer, -1 for host memory (pageable or pinned).
int pointer_device(const void* ptr) {
    if (!ptr) return -1;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (a.type == cudaMemoryTypeDevice) return a.device;
    if (a.type == cudaMemoryTypeManaged) return a.device < 0 ? 0 : a.device;
    return -1;
}

// ------------------------------------------------------------------ kernels

// One thread per node: range check, l0 (caller order), tile bin.
__global__ void k_bins(const double* __restrict__ x, int64_t N, int d, int64_t Ms0, int64_t Ms1,
                       int m, int S0, int S1, int64_t nseg1, int32_t* __restrict__ l0,
                       int32_t* __restrict__ bin, int* __restrict__ bad) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= N) return;
    int64_t b = 0;
    for (int i = 0; i < d; i++) {
        double xi = x[j * d + i];
        int64_t Ms = i == 0 ? Ms0 : Ms1;
        int S = i == 0 ? S0 : S1;
        if (!(xi >= -0.5 && xi < 0.5)) {  // also catches NaN
            atomicOr(bad, 1);
            xi = 0.0;
        }
        // reading A20: one correctly rounded product, then ceil (no FMA contraction)
        double t = __dmul_rn((double)Ms, xi);
        int64_t l = (int64_t)ceil(t) - m;
        l0[j * d + i] = (int32_t)l;
        int64_t n0 = mod64(l, Ms);
        int64_t s = n0 / S;
        b = (i == 0) ? s : b * nseg1 + s;
    }
    bin[j] = (int32_t)b;
}

__global__ void k_n0_key(const int32_t* __restrict__ l0, int64_t N, int64_t Ms, int32_t* __restrict__ key) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < N) key[j] = (int32_t)mod64(l0[j], Ms);
}

__global__ void k_iota(int32_t* a, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

__global__ void k_hist(const int32_t* __restrict__ bin, int64_t N, int32_t* __restrict__ cnt) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < N) atomicAdd(&cnt[bin[j]], 1);
}

// Sorted per-node integers: n0 per dim, segment-local delta (1-D), identity check.
__global__ void k_sorted_ints(const int32_t* __restrict__ perm, const int32_t* __restrict__ l0, int64_t N,
                              int d, int64_t Ms0, int64_t Ms1, int S0, int32_t* __restrict__ n0s,
                              int32_t* __restrict__ delta, int* __restrict__ not_identity) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int32_t j = perm[i];
    if (j != i) atomicOr(not_identity, 1);
    int64_t c = perm[0];
    int64_t js = i + c;
    if (js >= N) js -= N;
    if (j != js) atomicOr(not_identity + 1, 1);  // not a cyclic shift
    for (int k = 0; k < d; k++) {
        int64_t Ms = k == 0 ? Ms0 : Ms1;
        n0s[i * d + k] = (int32_t)mod64(l0[(int64_t)j * d + k], Ms);
    }
    int32_t n00 = n0s[i * d];
    delta[i] = n00 - (n00 / S0) * S0;
}

// d_k = s / (M_sigma what(k)) = s / I0(m sqrt(b^2 - (2 pi k/M_sigma)^2)), k = -M/2..M/2-1.
__global__ void k_deconv(double* __restrict__ dk, int64_t M, int64_t Ms, int m, double sigma, double s,
                         int window, int* __restrict__ bad) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= M) return;
    if (window == INFT_DIRICHLET) {  // what = 1, the unpaired k = -M/2 (c = 0) zeroed (reading A21)
        dk[c] = c == 0 ? 0.0 : s / (double)Ms;
        return;
    }
    if (window == INFT_BSPLINE) {  // M_sigma what(k) = sinc(pi k/M_sigma)^{2m} (reading A24)
        const int64_t k = c - M / 2;
        const double t = (double)k / (double)Ms;  // |t| <= 1/(2 sigma) <= 1/2
        const double sc = k == 0 ? 1.0 : sinpi(t) / (3.141592653589793238462643383279502884 * t);
        const double v = pow(sc, 2.0 * m);
        if (!(v > 0.0)) atomicOr(bad, 1);
        dk[c] = s / v;
        return;
    }
    double k = (double)(c - M / 2);
    const double pi = 3.141592653589793238462643383279502884;
    double b = pi * (2.0 - 1.0 / sigma);
    double u = 2.0 * pi * k / (double)Ms;
    double arg = __dsub_rn(__dmul_rn(b, b), __dmul_rn(u, u));
    if (arg < 0.0 && arg > -1e-12 * b * b) arg = 0.0;  // |k| = M/2 at sigma = 1: b = 2 pi k/Ms exactly
    if (arg < 0.0) {
        atomicOr(bad, 1);
        dk[c] = 0.0;
        return;
    }
    double what_times_Ms = cyl_bessel_i0((double)m * sqrt(arg));
    if (!(what_times_Ms > 0.0)) atomicOr(bad, 1);
    dk[c] = s / what_times_Ms;
}

__global__ void k_d2f(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}

// Sort caller-order weights into the padded sorted records of the plan precision.
template <typename T>
__global__ void k_sort_weights(const double* __restrict__ wcaller, const int32_t* __restrict__ perm, int64_t N,
                               int P, int PP, int cplx, T* __restrict__ wsorted, double* __restrict__ w64sorted,
                               const int32_t* __restrict__ n0s, int d) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= N * PP) return;
    int64_t i = idx / PP;
    int t = (int)(idx - i * PP);
    int64_t j = perm[i];
    if (cplx) {
        double re = t < P ? wcaller[(j * P + t) * 2] : 0.0;
        double im = t < P ? wcaller[(j * P + t) * 2 + 1] : 0.0;
        wsorted[idx * 2] = (T)re;
        wsorted[idx * 2 + 1] = (T)im;
        if (t < P) {
            w64sorted[(i * P + t) * 2] = re;
            w64sorted[(i * P + t) * 2 + 1] = im;
        }
    } else {
        double v = t < P ? wcaller[j * P + t] : 0.0;
        // record = P weights, then n0 (int32 bits) in the first padding slot
        wsorted[idx] = (t == P) ? n0_as(T(0), n0s[i * d]) : (T)v;
        if (t < P) w64sorted[i * P + t] = v;
    }
}

// From sorted double weights (setup output) into padded plan-precision records.
template <typename T>
__global__ void k_pack_sorted(const double* __restrict__ w64sorted, int64_t N, int P, int PP, int cplx,
                              T* __restrict__ wsorted, const int32_t* __restrict__ n0s, int d) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= N * PP) return;
    int64_t i = idx / PP;
    int t = (int)(idx - i * PP);
    if (cplx) {
        wsorted[idx * 2] = (T)(t < P ? w64sorted[(i * P + t) * 2] : 0.0);
        wsorted[idx * 2 + 1] = (T)(t < P ? w64sorted[(i * P + t) * 2 + 1] : 0.0);
    } else {
        wsorted[idx] = (t == P) ? n0_as(T(0), n0s[i * d]) : (T)(t < P ? w64sorted[i * P + t] : 0.0);
    }
}

__global__ void k_absmax(const double* __restrict__ a, int64_t n, unsigned long long* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double v = 0.0;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) v = fmax(v, fabs(a[i]));
    // non-negative doubles order like their bit patterns
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(v));
}

static inline unsigned grid1d(int64_t n, int bs = 256) { return (unsigned)ceil_div(n > 0 ? n : 1, bs); }

// ------------------------------------------------------------------ host logic
static int choose_segment(int m) {
    if (m == 4) return 8;  // SEG = 2m: register-ring kernels (stream1d_ring.cu)
    if (2 * m <= 16) return 16;
    if (2 * m <= 32) return 32;
    return (int)ceil_div(2 * m, 8) * 8;
}

void plan_build(Plan& p, const double* nodes_any, cudaStream_t st) {
    const int d = p.d;
    p.nodes.alloc(sizeof(double) * std::max<int64_t>(1, p.N * d));
    if (p.N > 0) {
        // cudaMemcpyDefault (UVA): host, this device or a peer device's buffer
        INFT_CUDA(cudaMemcpyAsync(p.nodes.p, nodes_any, sizeof(double) * p.N * d, cudaMemcpyDefault, st));
    }
    // tiles
    if (d == 1) {
        p.S[0] = choose_segment(p.m);
        p.S[1] = 1;
        p.nseg[0] = ceil_div(p.Ms[0], p.S[0]);
        p.nseg[1] = 1;
    } else {
        // 2-D tiles: 16 x 16 cells for m <= 7 (the tile spread k_spread_2d_tile needs P1 <= 16)
        p.S[0] = p.S[1] = (2 * p.m + 1 <= 16) ? 16 : choose_segment(p.m);
        p.nseg[0] = ceil_div(p.Ms[0], p.S[0]);
        p.nseg[1] = ceil_div(p.Ms[1], p.S[1]);
    }
    p.nseg_tot = p.nseg[0] * p.nseg[1];
    const int64_t Nn = std::max<int64_t>(1, p.N);
    p.l0.alloc(sizeof(int32_t) * Nn * d);
    p.bin.alloc(sizeof(int32_t) * Nn);
    p.perm.alloc(sizeof(int32_t) * Nn);
    p.n0s.alloc(sizeof(int32_t) * Nn * d);
    p.delta.alloc(sizeof(int32_t) * Nn);
    p.seg_start.alloc(sizeof(int32_t) * (p.nseg_tot + 1));

    DevBuf flags;
    flags.alloc(sizeof(int) * 4);
    INFT_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 4, st));
    int* dflags = flags.as<int>();
    if (p.N > 0) {
        k_bins<<<grid1d(p.N), 256, 0, st>>>(p.nodes.as<double>(), p.N, d, p.Ms[0], p.Ms[1], p.m, p.S[0], p.S[1],
                                            p.nseg[1], p.l0.as<int32_t>(), p.bin.as<int32_t>(), dflags);
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    int hflags[4];
    INFT_CUDA(cudaMemcpyAsync(hflags, dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    if (hflags[0]) {
        set_error("node outside [-1/2, 1/2) or not finite");
        throw Fail{INFT_ERR_NODE_RANGE};
    }
    // stable sort of node indices by bin (LSD radix sort is stable): reading A19
    INFT_CUDA(cudaMemsetAsync(p.seg_start.p, 0, sizeof(int32_t) * (p.nseg_tot + 1), st));
    if (p.N > 0) {
        DevBuf keys_out, idx_in, tmp;
        keys_out.alloc(sizeof(int32_t) * p.N);
        idx_in.alloc(sizeof(int32_t) * p.N);
        k_iota<<<grid1d(p.N), 256, 0, st>>>(idx_in.as<int32_t>(), p.N);
        INFT_CHECK_LAUNCH();
        p.launches++;
        // 1-D key: n0 (sorting by n0 also sorts by bin; increasing node sets stay a
        // cyclic shift of the caller order).  2-D key: the tile bin.
        DevBuf keys_in;
        const int32_t* kin = p.bin.as<int32_t>();
        int64_t kmax = p.nseg_tot;
        if (d == 1) {
            keys_in.alloc(sizeof(int32_t) * p.N);
            k_n0_key<<<grid1d(p.N), 256, 0, st>>>(p.l0.as<int32_t>(), p.N, p.Ms[0], keys_in.as<int32_t>());
            INFT_CHECK_LAUNCH();
            p.launches++;
            kin = keys_in.as<int32_t>();
            kmax = p.Ms[0];
        }
        int end_bit = 1;
        while ((int64_t(1) << end_bit) < kmax + 1) end_bit++;
        size_t tmp_bytes = 0;
        INFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, keys_out.as<int32_t>(),
                                                  idx_in.as<int32_t>(), p.perm.as<int32_t>(), (int)p.N, 0,
                                                  end_bit, st));
        tmp.alloc(tmp_bytes);
        INFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kin, keys_out.as<int32_t>(),
                                                  idx_in.as<int32_t>(), p.perm.as<int32_t>(), (int)p.N, 0,
                                                  end_bit, st));
        // segment starts = exclusive scan of the bin histogram
        DevBuf cnt;
        cnt.alloc(sizeof(int32_t) * (p.nseg_tot + 1));
        INFT_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (p.nseg_tot + 1), st));
        k_hist<<<grid1d(p.N), 256, 0, st>>>(p.bin.as<int32_t>(), p.N, cnt.as<int32_t>());
        INFT_CHECK_LAUNCH();
        p.launches++;
        size_t scan_bytes = 0;
        INFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt.as<int32_t>(), p.seg_start.as<int32_t>(),
                                                (int)(p.nseg_tot + 1), st));
        DevBuf stmp;
        stmp.alloc(scan_bytes);
        INFT_CUDA(cub::DeviceScan::ExclusiveSum(stmp.p, scan_bytes, cnt.as<int32_t>(), p.seg_start.as<int32_t>(),
                                                (int)(p.nseg_tot + 1), st));
        k_sorted_ints<<<grid1d(p.N), 256, 0, st>>>(p.perm.as<int32_t>(), p.l0.as<int32_t>(), p.N, d, p.Ms[0],
                                                   p.Ms[1], p.S[0], p.n0s.as<int32_t>(), p.delta.as<int32_t>(),
                                                   dflags + 1);
        INFT_CHECK_LAUNCH();
        p.launches++;
        INFT_CUDA(cudaMemcpyAsync(hflags, dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
        INFT_CUDA(cudaStreamSynchronize(st));
        p.perm_identity = hflags[1] == 0;
        int32_t c0 = 0;
        INFT_CUDA(cudaMemcpy(&c0, p.perm.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
        p.perm_shift = hflags[2] == 0 ? c0 : -1;
    }
    p.fast1d = (d == 1) && (p.m <= 16) && (p.Ms[0] % p.S[0] == 0) && (p.nseg[0] >= 2) && (p.P1 <= p.Ms[0]);
    // padded record stride: 16-byte aligned rows
    int vec = p.prec == INFT_C128 ? 2 : 4;
    p.PP = (int)ceil_div(p.P + 1, vec) * vec;  // >= 1 padding slot (holds n0 for the streaming kernels)
    p.GS = p.fast1d ? p.Ms[0] + ceil_div(2 * p.m, 8) * 8 : p.Mstot;
    {
        const char* e = getenv("INFT_NO_FUSED_FFT");
        p.no_fused_fft = e && atoi(e);
    }
    {
        const char* e = getenv("INFT_NO_SMALL");
        p.no_small = e && atoi(e);
    }
    compute_deconv(p, 1.0, st);
}

void compute_deconv(Plan& p, double s, cudaStream_t st) {
    int64_t tot = p.M[0] + (p.d == 2 ? p.M[1] : 0);
    if (p.dk.bytes != sizeof(double) * tot) p.dk.alloc(sizeof(double) * tot);
    DevBuf flag;
    flag.alloc(sizeof(int));
    INFT_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    for (int i = 0; i < p.d; i++) {
        double* dst = p.dk.as<double>() + (i == 0 ? 0 : p.M[0]);
        k_deconv<<<grid1d(p.M[i]), 256, 0, st>>>(dst, p.M[i], p.Ms[i], p.m, p.sigma, i == 0 ? s : 1.0,
                                                 (int)p.window, flag.as<int>());
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    if (p.prec == INFT_C64) {
        if (p.dkf.bytes != sizeof(float) * tot) p.dkf.alloc(sizeof(float) * tot);
        k_d2f<<<grid1d(tot), 256, 0, st>>>(p.dk.as<double>(), p.dkf.as<float>(), tot);
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    int h = 0;
    INFT_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    if (h) {
        set_error("window Fourier coefficient what(k) <= 0 for some |k| <= M/2");
        throw Fail{INFT_ERR_ZERO_WINDOW_HAT};
    }
    p.scale = s;
}

static void finish_weights(Plan& p, inft_method method, inft_weights wt, cudaStream_t st) {
    p.state_version++;  // captured apply graphs refer to the old weight buffers
    p.w_version++;      // tables derived from the weights (2-D line records) are stale
    // max |w| over the double copy
    DevBuf mx;
    mx.alloc(sizeof(unsigned long long));
    INFT_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
    int64_t n = p.N * p.P * (wt == INFT_WEIGHTS_COMPLEX ? 2 : 1);
    if (n > 0) {
        k_absmax<<<(unsigned)std::min<int64_t>(grid1d(n), 1184), 256, 0, st>>>(p.w64.as<double>(), n,
                                                                               mx.as<unsigned long long>());
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    unsigned long long bits = 0;
    INFT_CUDA(cudaMemcpyAsync(&bits, mx.p, sizeof(bits), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    double v;
    std::memcpy(&v, &bits, sizeof(v));
    p.max_abs_w = v;
    p.method = method;
    p.wt = wt;
    double s = (method == INFT_ALG1_NODEWISE) ? 1.0 / (double)p.Mtot : 1.0;
    compute_deconv(p, s, st);
}

void upload_weights(Plan& p, const double* w_host, inft_method method, inft_weights wt, cudaStream_t st) {
    int cp = wt == INFT_WEIGHTS_COMPLEX ? 2 : 1;
    int64_t n = p.N * p.P * cp;
    DevBuf tmp;
    tmp.alloc(sizeof(double) * std::max<int64_t>(1, n));
    if (n > 0) {
        INFT_CUDA(cudaMemcpyAsync(tmp.p, w_host, sizeof(double) * n, cudaMemcpyDefault, st));
    }
    size_t es = p.prec == INFT_C128 ? sizeof(double) : sizeof(float);
    p.w.alloc(es * std::max<int64_t>(1, p.N * p.PP * cp));
    p.w64.alloc(sizeof(double) * std::max<int64_t>(1, n));
    if (p.N > 0) {
        if (p.prec == INFT_C128)
            k_sort_weights<double><<<grid1d(p.N * p.PP), 256, 0, st>>>(tmp.as<double>(), p.perm.as<int32_t>(), p.N,
                                                                      p.P, p.PP, cp == 2, p.w.as<double>(),
                                                                      p.w64.as<double>(), p.n0s.as<int32_t>(), p.d);
        else
            k_sort_weights<float><<<grid1d(p.N * p.PP), 256, 0, st>>>(tmp.as<double>(), p.perm.as<int32_t>(), p.N,
                                                                     p.P, p.PP, cp == 2, p.w.as<float>(),
                                                                     p.w64.as<double>(), p.n0s.as<int32_t>(), p.d);
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    finish_weights(p, method, wt, st);
}

void install_weights_from_device(Plan& p, const double* w64_sorted_dev, inft_method method, inft_weights wt,
                                 cudaStream_t st) {
    int cp = wt == INFT_WEIGHTS_COMPLEX ? 2 : 1;
    int64_t n = p.N * p.P * cp;
    size_t es = p.prec == INFT_C128 ? sizeof(double) : sizeof(float);
    p.w.alloc(es * std::max<int64_t>(1, p.N * p.PP * cp));
    p.w64.alloc(sizeof(double) * std::max<int64_t>(1, n));
    if (n > 0) {
        INFT_CUDA(cudaMemcpyAsync(p.w64.p, w64_sorted_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        if (p.prec == INFT_C128)
            k_pack_sorted<double><<<grid1d(p.N * p.PP), 256, 0, st>>>(p.w64.as<double>(), p.N, p.P, p.PP, cp == 2,
                                                                     p.w.as<double>(), p.n0s.as<int32_t>(), p.d);
        else
            k_pack_sorted<float><<<grid1d(p.N * p.PP), 256, 0, st>>>(p.w64.as<double>(), p.N, p.P, p.PP, cp == 2,
                                                                    p.w.as<float>(), p.n0s.as<int32_t>(), p.d);
        INFT_CHECK_LAUNCH();
        p.launches++;
    }
    finish_weights(p, method, wt, st);
}

}  // namespace inft

// =========================================================================== C ABI
using inft::Fail;
using inft::Plan;

#define INFT_API_BEGIN try {
#define INFT_API_END                                      \
    }                                                     \
    catch (const Fail& f_) {                              \
        return f_.st;                                     \
    }                                                     \
    catch (const std::bad_alloc&) {                       \
        inft::set_error("host allocation failed");        \
        return INFT_ERR_OOM;                              \
    }                                                     \
    catch (...) {                                         \
        inft::set_error("unexpected C++ exception");      \
        return INFT_ERR_CUDA;                             \
    }                                                     \
    return INFT_OK;

// NVTX range over one C-ABI call (a0 plan, a1 setup, the two apply directions); the per-stage
// ranges a2-a7 nest inside (apply.cu StageTimer).  Header-only NVTX 3: no cost without a tool.
struct ApiRange {
    explicit ApiRange(const char* name) { nvtxRangePushA(name); }
    ~ApiRange() { nvtxRangePop(); }
};

extern "C" {

const char* inft_status_string(inft_status s) {
    switch (s) {
        case INFT_OK: return "INFT_OK";
        case INFT_ERR_INVALID_ARG: return "INFT_ERR_INVALID_ARG";
        case INFT_ERR_NODE_RANGE: return "INFT_ERR_NODE_RANGE";
        case INFT_ERR_ZERO_WINDOW_HAT: return "INFT_ERR_ZERO_WINDOW_HAT";
        case INFT_ERR_NOT_PRECOMPUTED: return "INFT_ERR_NOT_PRECOMPUTED";
        case INFT_ERR_CUDA: return "INFT_ERR_CUDA";
        case INFT_ERR_CUFFT: return "INFT_ERR_CUFFT";
        case INFT_ERR_OOM: return "INFT_ERR_OOM";
        case INFT_ERR_UNSUPPORTED: return "INFT_ERR_UNSUPPORTED";
    }
    return "INFT_ERR_UNKNOWN";
}

const char* inft_last_error(void) { return inft::g_last_error.c_str(); }

inft_status inft_plan(inft_plan_t* out, int d, const int64_t* M, int64_t N, const double* nodes, double sigma,
                      int m, inft_window window, inft_precision prec, int device, inft_stream_t stream) {
    if (!out) return INFT_ERR_INVALID_ARG;
    *out = nullptr;
    if (d < 1 || d > 2 || !M || N < 0 || (N > 0 && !nodes) ||
        (window != INFT_KAISER_BESSEL && window != INFT_DIRICHLET && window != INFT_BSPLINE) ||
        (prec != INFT_C128 && prec != INFT_C64) || !(sigma >= 1.0) || m < 1 || N > INT32_MAX ||
        (window == INFT_BSPLINE && m > 16)) {  // B-spline evaluation buffer: order 2m <= 32
        inft::set_error("inft_plan: invalid argument");
        return INFT_ERR_INVALID_ARG;
    }
    Plan* p = nullptr;
    ApiRange nvtx_("inft_plan (a0)");
    INFT_API_BEGIN
    int ndev = 0;
    INFT_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) {
        inft::set_error("inft_plan: bad device ordinal");
        return INFT_ERR_INVALID_ARG;
    }
    inft::DeviceGuard g(device);
    p = new Plan();
    p->device = device;
    p->window = window;
    p->d = d;
    p->N = N;
    p->m = m;
    p->sigma = sigma;
    p->prec = prec;
    for (int i = 0; i < d; i++) {
        if (M[i] <= 0 || (M[i] & 1)) throw Fail{INFT_ERR_INVALID_ARG};
        double ms = sigma * (double)M[i];
        int64_t ims = (int64_t)std::llround(ms);
        if (std::fabs(ms - (double)ims) > 1e-9 || (ims & 1) || ims < M[i]) throw Fail{INFT_ERR_INVALID_ARG};
        if (2 * (int64_t)m > ims) throw Fail{INFT_ERR_INVALID_ARG};  // m <= M_sigma/2
        if (ims > INT32_MAX / 2) throw Fail{INFT_ERR_INVALID_ARG};
        p->M[i] = M[i];
        p->Ms[i] = ims;
    }
    p->Mtot = p->M[0] * (d == 2 ? p->M[1] : 1);
    p->Mstot = p->Ms[0] * (d == 2 ? p->Ms[1] : 1);
    p->P1 = 2 * m + 1;
    p->P = d == 2 ? p->P1 * p->P1 : p->P1;
    inft::plan_build(*p, nodes, (cudaStream_t)stream);
    *out = reinterpret_cast<inft_plan_t>(p);
    p = nullptr;
    }
    catch (const Fail& f_) {
        if (f_.st == INFT_ERR_INVALID_ARG && inft::g_last_error.empty()) inft::set_error("inft_plan: invalid argument");
        delete p;
        return f_.st;
    }
    catch (...) {
        delete p;
        inft::set_error("inft_plan: unexpected exception");
        return INFT_ERR_CUDA;
    }
    return INFT_OK;
}

inft_status inft_destroy(inft_plan_t plan) {
    delete reinterpret_cast<Plan*>(plan);
    return INFT_OK;
}

inft_status inft_precompute(inft_plan_t plan, inft_method method, inft_weights wt, double tau,
                            inft_stream_t stream) {
    if (!plan) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (method < INFT_AUTO || method > INFT_PLAIN_NFFT || (wt != INFT_WEIGHTS_REAL && wt != INFT_WEIGHTS_COMPLEX))
        return INFT_ERR_INVALID_ARG;
    ApiRange nvtx_("inft_precompute (a1)");
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    inft::precompute(*p, method, wt, tau > 0 ? tau : 1e-6, (cudaStream_t)stream);
    INFT_API_END
}

inft_status inft_apply(inft_plan_t plan, const void* f, void* fhat, int64_t R, inft_stream_t stream) {
    if (!plan || R < 0) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (p->method < 0) return INFT_ERR_NOT_PRECOMPUTED;
    if (R == 0) return INFT_OK;
    if ((!f && p->N > 0) || !fhat) return INFT_ERR_INVALID_ARG;
    ApiRange nvtx_("inft_apply (a2-a4)");
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    inft::apply_inverse(*p, f, fhat, R, (cudaStream_t)stream);
    INFT_API_END
}

inft_status inft_adjoint_apply(inft_plan_t plan, const void* h, void* f, int64_t R, inft_stream_t stream) {
    if (!plan || R < 0) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (p->method < 0) return INFT_ERR_NOT_PRECOMPUTED;
    if (R == 0) return INFT_OK;
    if (!h || (!f && p->N > 0)) return INFT_ERR_INVALID_ARG;
    ApiRange nvtx_("inft_adjoint_apply (a5-a7)");
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    inft::apply_adjoint(*p, h, f, R, (cudaStream_t)stream);
    INFT_API_END
}

inft_status inft_get_bins(inft_plan_t plan, int32_t* l0, int32_t* bin, int32_t* perm) {
    if (!plan) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    INFT_CUDA(cudaDeviceSynchronize());
    if (p->N > 0) {
        if (l0) INFT_CUDA(cudaMemcpy(l0, p->l0.p, sizeof(int32_t) * p->N * p->d, cudaMemcpyDeviceToHost));
        if (bin) INFT_CUDA(cudaMemcpy(bin, p->bin.p, sizeof(int32_t) * p->N, cudaMemcpyDeviceToHost));
        if (perm) INFT_CUDA(cudaMemcpy(perm, p->perm.p, sizeof(int32_t) * p->N, cudaMemcpyDeviceToHost));
    }
    INFT_API_END
}

inft_status inft_get_bopt(inft_plan_t plan, void* w) {
    if (!plan || !w) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (p->method < 0) return INFT_ERR_NOT_PRECOMPUTED;
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    INFT_CUDA(cudaDeviceSynchronize());
    int cp = p->wt == INFT_WEIGHTS_COMPLEX ? 2 : 1;
    int64_t rec = (int64_t)p->P * cp;
    std::vector<double> sorted((size_t)std::max<int64_t>(1, p->N * rec));
    std::vector<int32_t> perm((size_t)std::max<int64_t>(1, p->N));
    if (p->N > 0) {
        INFT_CUDA(cudaMemcpy(sorted.data(), p->w64.p, sizeof(double) * p->N * rec, cudaMemcpyDeviceToHost));
        INFT_CUDA(cudaMemcpy(perm.data(), p->perm.p, sizeof(int32_t) * p->N, cudaMemcpyDeviceToHost));
    }
    double* out = static_cast<double*>(w);
    for (int64_t i = 0; i < p->N; i++)
        std::memcpy(out + (int64_t)perm[i] * rec, sorted.data() + i * rec, sizeof(double) * rec);
    INFT_API_END
}

inft_status inft_set_bopt(inft_plan_t plan, inft_method method, inft_weights wt, const void* w) {
    if (!plan || (!w && reinterpret_cast<Plan*>(plan)->N > 0)) return INFT_ERR_INVALID_ARG;
    if (method < INFT_ALG1_NODEWISE || method > INFT_PLAIN_NFFT) return INFT_ERR_INVALID_ARG;
    if (wt != INFT_WEIGHTS_REAL && wt != INFT_WEIGHTS_COMPLEX) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    inft::upload_weights(*p, static_cast<const double*>(w), method, wt, nullptr);
    INFT_CUDA(cudaDeviceSynchronize());
    INFT_API_END
}

inft_status inft_get_deconv(inft_plan_t plan, double* d) {
    if (!plan || !d) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    INFT_CUDA(cudaDeviceSynchronize());
    INFT_CUDA(cudaMemcpy(d, p->dk.p, p->dk.bytes, cudaMemcpyDeviceToHost));
    INFT_API_END
}

inft_status inft_get_info(inft_plan_t plan, inft_info* info) {
    if (!plan || !info) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    std::memset(info, 0, sizeof(*info));
    info->d = p->d;
    info->M[0] = p->M[0];
    info->M[1] = p->d == 2 ? p->M[1] : 1;
    info->Msigma[0] = p->Ms[0];
    info->Msigma[1] = p->d == 2 ? p->Ms[1] : 1;
    info->N = p->N;
    info->m = p->m;
    info->P = p->P;
    info->tile[0] = p->S[0];
    info->tile[1] = p->S[1];
    info->precision = p->prec;
    info->method = p->method;
    info->weights = p->wt;
    info->scale = p->scale;
    info->tau = p->tau;
    info->n_rank_deficient = p->n_rank_deficient;
    info->n_empty_cols = p->n_empty_cols;
    info->max_col_size = p->max_col_size;
    info->max_abs_w = p->max_abs_w;
    info->perm_identity = p->perm_identity ? 1 : 0;
    info->fast_path = p->fast1d ? (inft::ring_available(*p) ? 2 : 1) : 0;
    info->fused_fft = (inft::fused_fft_available(*p) && !p->no_fused_fft) ? 1 : 0;
    info->max_lowrank_rank = (int32_t)p->max_lowrank_rank;
    info->workspace_bytes = p->workspace_bytes();
    return INFT_OK;
}

inft_status inft_set_profiling(inft_plan_t plan, int enable) {
    if (!plan) return INFT_ERR_INVALID_ARG;
    reinterpret_cast<Plan*>(plan)->profiling = enable != 0;
    return INFT_OK;
}

inft_status inft_get_profile(inft_plan_t plan, inft_profile* out, int reset) {
    if (!plan) return INFT_ERR_INVALID_ARG;
    Plan* p = reinterpret_cast<Plan*>(plan);
    INFT_API_BEGIN
    inft::DeviceGuard g(p->device);
    p->drain_profile();
    if (out)
        for (int i = 0; i < 6; i++) {
            out->ms[i] = p->prof_ms[i];
            out->count[i] = p->prof_cnt[i];
        }
    if (reset)
        for (int i = 0; i < 6; i++) {
            p->prof_ms[i] = 0;
            p->prof_cnt[i] = 0;
        }
    INFT_API_END
}

int64_t inft_kernel_launches(inft_plan_t plan) {
    return plan ? reinterpret_cast<Plan*>(plan)->launches : 0;
}

}  // extern "C"
