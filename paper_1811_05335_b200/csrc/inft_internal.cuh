// Internal declarations of the sm_100a iNFFT library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <map>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/inft.h"

namespace inft {

// ------------------------------------------------------------ errors
void set_error(const std::string& msg);

struct Fail {
    inft_status st;
};

#define INFT_CUDA(call)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            ::inft::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));       \
            throw ::inft::Fail{e_ == cudaErrorMemoryAllocation ? INFT_ERR_OOM : INFT_ERR_CUDA}; \
        }                                                                                \
    } while (0)

#define INFT_CUFFT(call)                                                                 \
    do {                                                                                 \
        cufftResult r_ = (call);                                                         \
        if (r_ != CUFFT_SUCCESS) {                                                       \
            ::inft::set_error(std::string(#call) + ": cufftResult " + std::to_string((int)r_)); \
            throw ::inft::Fail{r_ == CUFFT_ALLOC_FAILED ? INFT_ERR_OOM : INFT_ERR_CUFFT}; \
        }                                                                                \
    } while (0)

#define INFT_STR2_(x) #x
#define INFT_STR_(x) INFT_STR2_(x)
// INFT_SYNC_CHECK=1: synchronize after every launch so a fault names its kernel's call site
bool sync_check_enabled();
bool getenv_flag(const char* name);  // name set to a nonzero integer
void ensure_smem_attr(const void* fn, size_t smem);     // cached cudaFuncSetAttribute
int occupancy_cached(const void* fn, int threads, size_t smem);
#define INFT_CHECK_LAUNCH()                                                              \
    do {                                                                                 \
        cudaError_t e_ = cudaGetLastError();                                             \
        if (e_ == cudaSuccess && ::inft::sync_check_enabled()) e_ = cudaDeviceSynchronize(); \
        if (e_ != cudaSuccess) {                                                         \
            ::inft::set_error(std::string("kernel launch at " __FILE__ ":" INFT_STR_(__LINE__) ": ") + \
                              cudaGetErrorString(e_));                                   \
            throw ::inft::Fail{INFT_ERR_CUDA};                                           \
        }                                                                                \
    } while (0)

// ------------------------------------------------------------ device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            free_();
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    void alloc(size_t b);
    void free_();
    ~DevBuf() { free_(); }
    template <typename T>
    T* as() const { return reinterpret_cast<T*>(p); }
};

// ------------------------------------------------------------ plan
struct FftKey {
    int batch;
    bool operator<(const FftKey& o) const { return batch < o.batch; }
};

struct Plan {
    int device = 0;
    int d = 1;
    int64_t M[2] = {1, 1};
    int64_t Ms[2] = {1, 1};
    int64_t Mtot = 1, Mstot = 1;
    int64_t N = 0;
    int m = 1;
    int P1 = 3;          // 2m+1
    int P = 3;           // P1^d
    int PP = 4;          // padded slot stride of the sorted weight records (elements)
    double sigma = 2.0;
    inft_precision prec = INFT_C128;
    int S[2] = {16, 1};  // tile (segment) width per dim
    int64_t nseg[2] = {1, 1};
    int64_t nseg_tot = 1;
    bool perm_identity = true;
    int perm_shift = 0;  // c >= 0 if perm[i] = (i + c) mod N (caller order = cyclic shift of sorted), else -1
    bool fast1d = false;
    bool no_fused_fft = false;  // INFT_NO_FUSED_FFT=1: cuFFT + separate deconvolution passes
    bool no_small = false;      // INFT_NO_SMALL=1: no single-launch path for small 1-D problems
    int64_t GS = 1;  // grid row stride in complex elements (1-D fast path: M_sigma + halo)

    // method state
    int method = -1;
    inft_window window = INFT_KAISER_BESSEL;
    inft_weights wt = INFT_WEIGHTS_REAL;
    double scale = 1.0;
    double tau = 1e-6;
    int64_t n_rank_deficient = 0, n_empty_cols = 0, max_col_size = 0, max_lowrank_rank = 0;
    double max_abs_w = 0.0;

    // device arrays (plan-owned)
    DevBuf nodes;      // double [N*d] caller order
    DevBuf l0;         // int32 [N*d] caller order
    DevBuf bin;        // int32 [N] caller order
    DevBuf perm;       // int32 [N] sorted -> caller
    DevBuf seg_start;  // int32 [nseg_tot+1]
    DevBuf n0s;        // int32 [N*d] sorted: n0 = l0 mod Ms per dim
    DevBuf delta;      // int32 [N] sorted: segment-local offset (1-D: n0 - seg*S)
    DevBuf dk;         // double [M1 (+M2)] deconvolution tables (s folded into dim 0)
    DevBuf dkf;        // float copy for C64
    DevBuf w;          // sorted weights: [N][PP] (real) or [N][PP] complex, in plan precision
    DevBuf w64;        // sorted weights in double (real: [N][P]; complex: [N][P] pairs) -- checkpoint copy

    // workspace
    DevBuf grid;          // [Rt][Mstot] complex (plan precision)
    DevBuf fT;            // 2-D spread: node-major copy of f, [N][R] (sorted node order)
    DevBuf chunks2d;      // 2-D gather: (tile, first node) per chunk of <= 64 nodes
    DevBuf work2d, comb2d, part2d;  // 2-D spread: work items, combine items, partial tiles
    int64_t work2d_n = -1, comb2d_n = 0, part2d_rhs = 0;
    int slots2d = 0;
    int64_t chunks2d_n = -1;
    int64_t fT_rhs = 0;
    int64_t grid_rhs = 0; // capacity in RHS
    DevBuf stage_in[2], stage_out[2];
    size_t stage_in_bytes = 0, stage_out_bytes = 0;
    std::map<FftKey, cufftHandle> fft;  // batch -> plan
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    // CUDA graphs of repeated device-pointer applies (apply.cu): keyed by direction, buffers,
    // batch and plan state; captured on the plan's own stream s_graph at the second call
    struct GraphKey {
        int dir;
        const void* in;
        const void* out;
        int64_t R;
        int64_t version;
        bool operator<(const GraphKey& o) const {
            return std::tie(dir, in, out, R, version) < std::tie(o.dir, o.in, o.out, o.R, o.version);
        }
    };
    struct GraphEntry {
        int seen = 0;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        int64_t last_use = 0;
    };
    static constexpr size_t kMaxGraphs = 16;  // LRU cap on captured graphs per plan
    std::map<GraphKey, GraphEntry> graphs;
    int64_t graph_clock = 0;
    // ring kernels: node-balanced chunk tables (segment boundaries), per target node count
    struct ChunkTable {
        DevBuf buf;
        int n = 0;
        int nfix = 0, nslots = 0;  // spread tables: fix entries after the chunks, side slots
    };
    std::map<int64_t, ChunkTable> ring_chunk_cache;
    std::vector<int32_t> seg_host;  // host copy of seg_start (1-D)
    DevBuf ring_side;               // ring spread: side slots of split heavy segments [slot][R][2m]
    int64_t state_version = 0;  // bumped whenever weights / tables change
    int64_t w_version = 0;      // bumped whenever the weights change (tables derived from them)
    // 2-D line spread (spread2d_line.cu): virtual-node records, segment table, items, fix entries
    DevBuf line_rec, line_vidx, line_seg, line_items, line_fix, line_first, line_carry;
    int64_t line_version = -1, line_slot_rhs = 0;
    int line_nv = 0, line_nitems = 0, line_nfix = 0;
    cudaStream_t s_graph = nullptr;
    cudaEvent_t ev_g0 = nullptr, ev_g1 = nullptr;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr},
                ev_d2h[2] = {nullptr, nullptr}, ev_entry = nullptr, ev_exit = nullptr;

    int64_t launches = 0;

    // per-stage profiling (inft_set_profiling)
    bool profiling = false;
    struct Rec {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[6] = {0, 0, 0, 0, 0, 0};
    int64_t prof_cnt[6] = {0, 0, 0, 0, 0, 0};
    cudaEvent_t take_event();
    void drain_profile();

    size_t elem_bytes() const { return prec == INFT_C128 ? 16 : 8; }
    size_t workspace_bytes() const;
    ~Plan();
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------ entry points implemented per file
// plan.cu
void plan_build(Plan& p, const double* nodes_any, cudaStream_t st);
void upload_weights(Plan& p, const double* w_host_caller_order, inft_method method, inft_weights wt,
                    cudaStream_t st);
void install_weights_from_device(Plan& p, const double* w64_sorted_dev, inft_method method,
                                 inft_weights wt, cudaStream_t st);
void compute_deconv(Plan& p, double s, cudaStream_t st);
// apply.cu
void apply_inverse(Plan& p, const void* f, void* fhat, int64_t R, cudaStream_t st);
void apply_adjoint(Plan& p, const void* h, void* f, int64_t R, cudaStream_t st);
// stream1d.cu
bool stream1d_available(const Plan& p);
void spread_stream1d(Plan& p, const void* f, void* grid, int64_t R, cudaStream_t st);
void gather_stream1d(Plan& p, const void* grid, void* f, int64_t R, cudaStream_t st);
// stream1d_ring.cu
bool ring_available(const Plan& p);
bool ring_spread_available(const Plan& p);
void spread_ring(Plan& p, const void* f, void* grid, int64_t R, cudaStream_t st);
void gather_ring(Plan& p, const void* grid, void* f, int64_t R, cudaStream_t st);
// spread2d_line.cu
bool line2d_available(const Plan& p);
void spread_line2d(Plan& p, const void* fT, void* grid, int64_t R, int RS, cudaStream_t st);
// fft.cu
bool fused_fft_available(const Plan& p);
// part: 1 = pass A (columns), 2 = pass B (rows), 3 = both
void fused_fft_inverse(Plan& p, void* grid, void* fhat, int64_t R, cudaStream_t st, int part = 3);
void fused_fft_adjoint(Plan& p, const void* h, void* grid, int64_t R, cudaStream_t st, int part = 3);
void release_fft_state(const Plan* p);
// setup.cu
void precompute(Plan& p, inft_method method, inft_weights wt, double tau, cudaStream_t st);

bool is_device_pointer(const void* ptr);
int pointer_device(const void* ptr);  // device ordinal, -1 for host memory

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#ifdef __CUDACC__
__device__ __forceinline__ int64_t dmod(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

// Call fn(s) once for every distinct segment (width S, nseg = ceil(Ms/S)) that
// touches the periodic grid range [n - span + 1, n] (mod Ms).  A range may
// re-enter its first segment after wrapping (Ms <= 2S, or span >= Ms); each
// segment is still visited once, so no node is counted twice.
template <typename Fn>
__device__ __forceinline__ void for_segments(int64_t n, int64_t span, int64_t Ms, int S, int64_t nseg, Fn&& fn) {
    if (span >= Ms) {
        for (int64_t s = 0; s < nseg; ++s) fn(s);
        return;
    }
    int64_t seen[4];
    int ns = 0;
    int64_t pos = dmod(n - (span - 1), Ms), rem = span;
    while (rem > 0) {
        int64_t s = pos / S;
        bool dup = false;
        for (int k = 0; k < ns; ++k) dup |= (seen[k] == s);
        if (!dup) {
            if (ns < 4) seen[ns++] = s;
            fn(s);
        }
        int64_t send = ((s + 1) * S < Ms) ? (s + 1) * S : Ms;
        int64_t len = (send - pos < rem) ? send - pos : rem;
        rem -= len;
        pos += len;
        if (pos == Ms) pos = 0;
    }
}
#endif

}  // namespace inft
