// Quadratic case M = N (paper Section "The quadratic case", P:344-489,
// adjoint Remark P:576-584): the inverse NFFT by the Lagrange relation
//   g_l = a_l sum_j f_j b_j (cot(pi (x_l - y_j)) - i)                     (eq. lagrange_formula)
// at equispaced targets x_l = -1/2 + l/N + delta, then fcheck = (1/N) E^* g by one FFT
// (Alg. "Fast inverse NFFT - quadratic case" step 6), and its adjoint
//   f_j = b_j sum_l a_l v_l (cot(pi (x_l - y_j)) + i),  v = (1/N) E h   (eq. lagrange_formula_adjoint).
// a_l = prod_n sin(pi (x_l - y_n)) and b_j = prod_{n != j} 1/sin(pi (y_j - y_n)) (eq. coeff_ab)
// are formed in the log domain with counted signs and the balancing shift s
// (Remark P:431-449, reading A22).
//
// B200 design: the three O(N^2) sums (ln|sin| for a and b, the cotangent sum per RHS) are
// evaluated directly, exactly, by tiled kernels -- one thread per target, sources streamed
// through shared memory, one sin/cos per (target, source) pair reused for a group of 16
// right-hand sides held in registers; fixed summation order (deterministic).  The paper's
// fast summation (O(N log N) with near-field corrections) accelerates exactly
// these sums; at the sizes measured here (N <= 2^17) the direct GPU sums take milliseconds.
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "inft_internal.cuh"

namespace inft {
namespace quad {

constexpr int kTile = 256;  // sources per shared-memory tile
constexpr int kRG = 16;     // right-hand sides per cotangent-sum block

static int64_t nb(int64_t n, int t = 256) { return (n + t - 1) / t; }

// logsum[t] = sgn * sum_{n (!= t if self)} ln|sin(pi (tgt_t - src_n))|, neg[t] = #{n: factor < 0};
// *bad set if a factor is exactly zero (coincident nodes).
__global__ void k_logsum(const double* __restrict__ tgt, int64_t nt, const double* __restrict__ src, int64_t ns,
                         int self, double sgn, double* __restrict__ logsum, int* __restrict__ negs,
                         int* __restrict__ bad) {
    __shared__ double ys[kTile];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const double xt = t < nt ? tgt[t] : 0.0;
    double acc = 0.0;
    int neg = 0, zero = 0;
    for (int64_t n0 = 0; n0 < ns; n0 += kTile) {
        const int cnt = (int)(ns - n0 < kTile ? ns - n0 : kTile);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) ys[i] = src[n0 + i];
        __syncthreads();
        if (t >= nt) continue;
        for (int i = 0; i < cnt; ++i) {
            if (self && n0 + i == t) continue;
            const double d = xt - ys[i];  // in (-1, 1): sin(pi d) < 0 iff d < 0
            const double sv = sinpi(d);
            zero |= sv == 0.0;
            neg += d < 0.0;
            acc += log(fabs(sv));
        }
    }
    if (t < nt) {
        logsum[t] = sgn * acc;
        negs[t] = neg;
        if (zero) atomicOr(bad, 1);
    }
}

// s = (max btilde - max atilde) / 2 (reading A22), one block, fixed reduction order
__global__ void k_shift(const double* __restrict__ at, const double* __restrict__ bt, int64_t N,
                        double* __restrict__ s) {
    __shared__ double ma[256], mb[256];
    double a = -INFINITY, b = -INFINITY;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        a = fmax(a, at[i]);
        b = fmax(b, bt[i]);
    }
    ma[threadIdx.x] = a;
    mb[threadIdx.x] = b;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            ma[threadIdx.x] = fmax(ma[threadIdx.x], ma[threadIdx.x + o]);
            mb[threadIdx.x] = fmax(mb[threadIdx.x], mb[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *s = 0.5 * (mb[0] - ma[0]);
}

// a_l = (-1)^neg e^{atilde + s},  b_j = (-1)^neg e^{btilde - s}   (Alg. steps 2-3)
__global__ void k_signed(const double* __restrict__ lg, const int* __restrict__ negs, int64_t N,
                         const double* __restrict__ s, double ssgn, double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double v = exp(lg[i] + ssgn * *s);
    out[i] = (negs[i] & 1) ? -v : v;
}

// out[r][t] = sum_s cf[r][s] cot(pi (tgt_t - src_s)), r in this block's group of kRG
__global__ void __launch_bounds__(128) k_cotsum(const double* __restrict__ tgt, int64_t nt,
                                                const double* __restrict__ src, int64_t ns,
                                                const double2* __restrict__ cf, int64_t R,
                                                double2* __restrict__ out) {
    __shared__ double ys[128];
    __shared__ double2 cs[kRG][128];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.y * kRG;
    const int nr = (int)(R - r0 < kRG ? R - r0 : kRG);
    const double xt = t < nt ? tgt[t] : 0.0;
    double ax[kRG], ay[kRG];
#pragma unroll
    for (int q = 0; q < kRG; ++q) ax[q] = ay[q] = 0.0;
    for (int64_t n0 = 0; n0 < ns; n0 += 128) {
        const int cnt = (int)(ns - n0 < 128 ? ns - n0 : 128);
        __syncthreads();
        if ((int)threadIdx.x < cnt) ys[threadIdx.x] = src[n0 + threadIdx.x];
        for (int q = 0; q < kRG; ++q)
            cs[q][threadIdx.x] = (q < nr && (int)threadIdx.x < cnt) ? cf[(r0 + q) * ns + n0 + threadIdx.x]
                                                                    : make_double2(0.0, 0.0);
        __syncthreads();
        for (int i = 0; i < cnt; ++i) {
            double sn, cn;
            sincospi(xt - ys[i], &sn, &cn);
            const double ct = cn / sn;
#pragma unroll
            for (int q = 0; q < kRG; ++q) {
                ax[q] = fma(cs[q][i].x, ct, ax[q]);
                ay[q] = fma(cs[q][i].y, ct, ay[q]);
            }
        }
    }
    if (t < nt)
        for (int q = 0; q < nr; ++q) out[(r0 + q) * nt + t] = make_double2(ax[q], ay[q]);
}

// sums[r] = sum_i v[r][i] (one block per row, fixed order)
__global__ void k_rowsum(const double2* __restrict__ v, int64_t n, double2* __restrict__ sums) {
    __shared__ double sx[256], sy[256];
    double x = 0.0, y = 0.0;
    const double2* row = v + (int64_t)blockIdx.x * n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        x += row[i].x;
        y += row[i].y;
    }
    sx[threadIdx.x] = x;
    sy[threadIdx.x] = y;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sx[threadIdx.x] += sx[threadIdx.x + o];
            sy[threadIdx.x] += sy[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[blockIdx.x] = make_double2(sx[0], sy[0]);
}

// c[r][j] = f[r][j] * w[j]  (real weights)
__global__ void k_scale(const double2* __restrict__ f, const double* __restrict__ w, int64_t n, int64_t total,
                        double2* __restrict__ c) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const double s = w[i % n];
    c[i] = make_double2(f[i].x * s, f[i].y * s);
}

// g[r][l] = a_l (gt[r][l] - i S_r)   (eq. coeff_g)
__global__ void k_glue_inv(const double2* __restrict__ gt, const double* __restrict__ a, const double2* __restrict__ S,
                           int64_t N, int64_t total, double2* __restrict__ g) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, l = i - r * N;
    const double2 v = gt[i], s = S[r];
    // (v - i s) = (v.x + s.y, v.y - s.x)
    g[i] = make_double2(a[l] * (v.x + s.y), a[l] * (v.y - s.x));
}

// fcheck[r][k + N/2] = (1/N) (-1)^k e^{-2 pi i k delta} G[r][k mod N]   (Alg. step 6 with
// x_l = -1/2 + l/N + delta: e^{-2 pi i k x_l} = (-1)^k e^{-2 pi i k delta} e^{-2 pi i k l/N})
__global__ void k_post_inv(const double2* __restrict__ G, int64_t N, int64_t total, double delta,
                           double2* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, c = i - r * N;
    const int64_t k = c - N / 2;
    const double2 v = G[r * N + (k < 0 ? k + N : k)];
    double sn, cs;
    sincospi(-2.0 * ((double)k * delta), &sn, &cs);
    const double sg = (k & 1) ? -1.0 / (double)N : 1.0 / (double)N;
    out[i] = make_double2(sg * (v.x * cs - v.y * sn), sg * (v.x * sn + v.y * cs));
}

// u[r][k mod N] = (1/N) (-1)^k e^{2 pi i k delta} h[r][k + N/2]; the inverse FFT then gives
// v_l = (1/N) sum_k h_k e^{2 pi i k x_l}
__global__ void k_pre_adj(const double2* __restrict__ h, int64_t N, int64_t total, double delta,
                          double2* __restrict__ u) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, c = i - r * N;
    const int64_t k = c - N / 2;
    const double2 v = h[i];
    double sn, cs;
    sincospi(2.0 * ((double)k * delta), &sn, &cs);
    const double sg = (k & 1) ? -1.0 / (double)N : 1.0 / (double)N;
    u[r * N + (k < 0 ? k + N : k)] = make_double2(sg * (v.x * cs - v.y * sn), sg * (v.x * sn + v.y * cs));
}

// f[r][j] = b_j (-ct[r][j] + i W_r), ct = sum_l w_l cot(pi (y_j - x_l)) = -sum_l w_l cot(pi (x_l - y_j))
__global__ void k_glue_adj(const double2* __restrict__ ct, const double* __restrict__ b, const double2* __restrict__ W,
                           int64_t N, int64_t total, double2* __restrict__ f) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t r = i / N, j = i - r * N;
    const double2 v = ct[i], w = W[r];
    // -v + i w = (-v.x - w.y, -v.y + w.x)
    f[i] = make_double2(b[j] * (-v.x - w.y), b[j] * (-v.y + w.x));
}

struct QPlan {
    int64_t N = 0;
    int device = 0;
    double delta = 0.0;
    DevBuf x, y, a, b, s;
    DevBuf w1, w2, w3, sums;  // per-apply workspaces ([R][N] complex x 3, [R] complex)
    int64_t wsR = 0;
    std::map<int64_t, cufftHandle> fft;  // batch -> plan
    int64_t launches = 0;
    ~QPlan() {
        for (auto& kv : fft) cufftDestroy(kv.second);
    }
    cufftHandle plan_for(int64_t R, cudaStream_t st) {
        auto it = fft.find(R);
        cufftHandle h;
        if (it == fft.end()) {
            int n[1] = {(int)N};
            INFT_CUFFT(cufftPlanMany(&h, 1, n, nullptr, 1, (int)N, nullptr, 1, (int)N, CUFFT_Z2Z, (int)R));
            fft[R] = h;
        } else {
            h = it->second;
        }
        cufftSetStream(h, st);
        return h;
    }
    void ensure_ws(int64_t R) {
        if (R <= wsR) return;
        const size_t bytes = sizeof(double2) * (size_t)R * (size_t)N;
        w1.alloc(bytes);
        w2.alloc(bytes);
        w3.alloc(bytes);
        sums.alloc(sizeof(double2) * (size_t)R);
        wsR = R;
    }
};

static void build(QPlan& q, const double* nodes_host_or_dev, cudaStream_t st) {
    const int64_t N = q.N;
    std::vector<double> yh(N), xh(N);
    if (is_device_pointer(nodes_host_or_dev)) {
        INFT_CUDA(cudaMemcpyAsync(yh.data(), nodes_host_or_dev, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        INFT_CUDA(cudaStreamSynchronize(st));
    } else {
        std::memcpy(yh.data(), nodes_host_or_dev, sizeof(double) * N);
    }
    for (int64_t j = 0; j < N; ++j)
        if (!std::isfinite(yh[j]) || yh[j] < -0.5 || yh[j] >= 0.5) {
            set_error("quadratic case: node outside [-1/2, 1/2)");
            throw Fail{INFT_ERR_NODE_RANGE};
        }
    for (int64_t l = 0; l < N; ++l) xh[l] = -0.5 + (double)l / (double)N + q.delta;
    q.x.alloc(sizeof(double) * N);
    q.y.alloc(sizeof(double) * N);
    q.a.alloc(sizeof(double) * N);
    q.b.alloc(sizeof(double) * N);
    q.s.alloc(sizeof(double));
    INFT_CUDA(cudaMemcpyAsync(q.x.p, xh.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    INFT_CUDA(cudaMemcpyAsync(q.y.p, yh.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    DevBuf la, lb, na, nbn, bad;
    la.alloc(sizeof(double) * N);
    lb.alloc(sizeof(double) * N);
    na.alloc(sizeof(int) * N);
    nbn.alloc(sizeof(int) * N);
    bad.alloc(sizeof(int));
    INFT_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    // step 1: atilde_l = sum_n ln|sin(pi(x_l - y_n))|, btilde_j = -sum_{n != j} ln|sin(pi(y_j - y_n))|
    k_logsum<<<(unsigned)nb(N), 256, 0, st>>>(q.x.as<double>(), N, q.y.as<double>(), N, 0, 1.0, la.as<double>(),
                                              na.as<int>(), bad.as<int>());
    INFT_CHECK_LAUNCH();
    k_logsum<<<(unsigned)nb(N), 256, 0, st>>>(q.y.as<double>(), N, q.y.as<double>(), N, 1, -1.0, lb.as<double>(),
                                              nbn.as<int>(), bad.as<int>());
    INFT_CHECK_LAUNCH();
    // steps 2-3: shift, exponentials, signs
    k_shift<<<1, 256, 0, st>>>(la.as<double>(), lb.as<double>(), N, q.s.as<double>());
    INFT_CHECK_LAUNCH();
    k_signed<<<(unsigned)nb(N), 256, 0, st>>>(la.as<double>(), na.as<int>(), N, q.s.as<double>(), 1.0, q.a.as<double>());
    INFT_CHECK_LAUNCH();
    k_signed<<<(unsigned)nb(N), 256, 0, st>>>(lb.as<double>(), nbn.as<int>(), N, q.s.as<double>(), -1.0,
                                              q.b.as<double>());
    INFT_CHECK_LAUNCH();
    q.launches += 5;
    int hb = 0;
    INFT_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    INFT_CUDA(cudaStreamSynchronize(st));
    if (hb) {
        set_error("quadratic case: coincident nodes (a node equals a target x_l or another node)");
        throw Fail{INFT_ERR_NODE_RANGE};
    }
}

// in/out: device or host [R][N] complex128 (host data staged synchronously)
template <typename Body>
static void with_device_io(QPlan& q, const void* in, void* out, int64_t R, cudaStream_t st, Body&& body) {
    const size_t bytes = sizeof(double2) * (size_t)R * (size_t)q.N;
    const bool din = is_device_pointer(in), dout = is_device_pointer(out);
    DevBuf ti, to;
    const double2* di = static_cast<const double2*>(in);
    double2* dov = static_cast<double2*>(out);
    if (!din) {
        ti.alloc(bytes);
        INFT_CUDA(cudaMemcpyAsync(ti.p, in, bytes, cudaMemcpyHostToDevice, st));
        di = ti.as<double2>();
    }
    if (!dout) {
        to.alloc(bytes);
        dov = to.as<double2>();
    }
    body(di, dov);
    if (!dout) {
        INFT_CUDA(cudaMemcpyAsync(out, dov, bytes, cudaMemcpyDeviceToHost, st));
    }
    if (!din || !dout) INFT_CUDA(cudaStreamSynchronize(st));
}

static void apply_inverse(QPlan& q, const double2* f, double2* fhat, int64_t R, cudaStream_t st) {
    const int64_t N = q.N, tot = R * N;
    q.ensure_ws(R);
    double2 *c = q.w1.as<double2>(), *gt = q.w2.as<double2>(), *g = q.w3.as<double2>();
    k_scale<<<(unsigned)nb(tot), 256, 0, st>>>(f, q.b.as<double>(), N, tot, c);  // f_j b_j
    k_rowsum<<<(unsigned)R, 256, 0, st>>>(c, N, q.sums.as<double2>());          // sum_j f_j b_j
    dim3 grid((unsigned)nb(N, 128), (unsigned)nb(R, kRG));
    k_cotsum<<<grid, 128, 0, st>>>(q.x.as<double>(), N, q.y.as<double>(), N, c, R, gt);  // eq. coeff_g_tilde
    k_glue_inv<<<(unsigned)nb(tot), 256, 0, st>>>(gt, q.a.as<double>(), q.sums.as<double2>(), N, tot, g);
    INFT_CHECK_LAUNCH();
    cufftHandle h = q.plan_for(R, st);
    if (cufftExecZ2Z(h, (cufftDoubleComplex*)g, (cufftDoubleComplex*)gt, CUFFT_FORWARD) != CUFFT_SUCCESS) {
        set_error("cufftExecZ2Z (quadratic case, step 6) failed");
        throw Fail{INFT_ERR_CUFFT};
    }
    k_post_inv<<<(unsigned)nb(tot), 256, 0, st>>>(gt, N, tot, q.delta, fhat);
    INFT_CHECK_LAUNCH();
    q.launches += 5;
}

static void apply_adjoint(QPlan& q, const double2* h, double2* f, int64_t R, cudaStream_t st) {
    const int64_t N = q.N, tot = R * N;
    q.ensure_ws(R);
    double2 *u = q.w1.as<double2>(), *v = q.w2.as<double2>(), *ct = q.w3.as<double2>();
    k_pre_adj<<<(unsigned)nb(tot), 256, 0, st>>>(h, N, tot, q.delta, u);
    INFT_CHECK_LAUNCH();
    cufftHandle hp = q.plan_for(R, st);
    if (cufftExecZ2Z(hp, (cufftDoubleComplex*)u, (cufftDoubleComplex*)v, CUFFT_INVERSE) != CUFFT_SUCCESS) {
        set_error("cufftExecZ2Z (quadratic case, adjoint) failed");
        throw Fail{INFT_ERR_CUFFT};
    }
    k_scale<<<(unsigned)nb(tot), 256, 0, st>>>(v, q.a.as<double>(), N, tot, u);  // w_l = a_l v_l
    k_rowsum<<<(unsigned)R, 256, 0, st>>>(u, N, q.sums.as<double2>());          // sum_l w_l
    dim3 grid((unsigned)nb(N, 128), (unsigned)nb(R, kRG));
    k_cotsum<<<grid, 128, 0, st>>>(q.y.as<double>(), N, q.x.as<double>(), N, u, R, ct);
    k_glue_adj<<<(unsigned)nb(tot), 256, 0, st>>>(ct, q.b.as<double>(), q.sums.as<double2>(), N, tot, f);
    INFT_CHECK_LAUNCH();
    q.launches += 5;
}

}  // namespace quad
}  // namespace inft

using inft::Fail;

#define INFT_Q_TRY try {
#define INFT_Q_CATCH                                          \
    }                                                         \
    catch (const Fail& f_) {                                  \
        return f_.st;                                         \
    }                                                         \
    catch (const std::bad_alloc&) {                           \
        inft::set_error("host allocation failed");            \
        return INFT_ERR_OOM;                                  \
    }                                                         \
    catch (...) {                                             \
        inft::set_error("unexpected C++ exception");          \
        return INFT_ERR_CUDA;                                 \
    }                                                         \
    return INFT_OK;

extern "C" {

inft_status inft_quad_plan(inft_quad_t* out, int64_t N, const double* nodes, double delta, int device,
                           inft_stream_t stream) {
    if (!out) return INFT_ERR_INVALID_ARG;
    *out = nullptr;
    if (N < 2 || (N & 1) || !nodes || N > (int64_t(1) << 30)) return INFT_ERR_INVALID_ARG;
    if (delta == 0.0) delta = 0.5 / (double)N;  // reading A23
    if (!(delta > 0.0 && delta < 1.0 / (double)N)) return INFT_ERR_INVALID_ARG;
    INFT_Q_TRY
    inft::DeviceGuard g(device);
    auto* q = new inft::quad::QPlan();
    q->N = N;
    q->device = device;
    q->delta = delta;
    try {
        inft::quad::build(*q, nodes, (cudaStream_t)stream);
    } catch (...) {
        delete q;
        throw;
    }
    *out = reinterpret_cast<inft_quad_t>(q);
    INFT_Q_CATCH
}

inft_status inft_quad_apply(inft_quad_t plan, const void* f, void* fhat, int64_t R, inft_stream_t stream) {
    if (!plan || R < 0) return INFT_ERR_INVALID_ARG;
    if (R == 0) return INFT_OK;
    if (!f || !fhat) return INFT_ERR_INVALID_ARG;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    const cudaStream_t st = (cudaStream_t)stream;
    inft::quad::with_device_io(*q, f, fhat, R, st, [&](const double2* di, double2* dout) {
        inft::quad::apply_inverse(*q, di, dout, R, st);
    });
    INFT_Q_CATCH
}

inft_status inft_quad_adjoint_apply(inft_quad_t plan, const void* h, void* f, int64_t R, inft_stream_t stream) {
    if (!plan || R < 0) return INFT_ERR_INVALID_ARG;
    if (R == 0) return INFT_OK;
    if (!h || !f) return INFT_ERR_INVALID_ARG;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    const cudaStream_t st = (cudaStream_t)stream;
    inft::quad::with_device_io(*q, h, f, R, st, [&](const double2* di, double2* dout) {
        inft::quad::apply_adjoint(*q, di, dout, R, st);
    });
    INFT_Q_CATCH
}

inft_status inft_quad_get_coeffs(inft_quad_t plan, double* x, double* a, double* b, double* s) {
    if (!plan) return INFT_ERR_INVALID_ARG;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    INFT_CUDA(cudaDeviceSynchronize());
    const size_t bytes = sizeof(double) * (size_t)q->N;
    if (x) INFT_CUDA(cudaMemcpy(x, q->x.p, bytes, cudaMemcpyDeviceToHost));
    if (a) INFT_CUDA(cudaMemcpy(a, q->a.p, bytes, cudaMemcpyDeviceToHost));
    if (b) INFT_CUDA(cudaMemcpy(b, q->b.p, bytes, cudaMemcpyDeviceToHost));
    if (s) INFT_CUDA(cudaMemcpy(s, q->s.p, sizeof(double), cudaMemcpyDeviceToHost));
    INFT_Q_CATCH
}

inft_status inft_quad_kernel_launches(inft_quad_t plan, int64_t* count) {
    if (!plan || !count) return INFT_ERR_INVALID_ARG;
    *count = reinterpret_cast<inft::quad::QPlan*>(plan)->launches;
    return INFT_OK;
}

inft_status inft_quad_destroy(inft_quad_t plan) {
    if (!plan) return INFT_OK;
    auto* q = reinterpret_cast<inft::quad::QPlan*>(plan);
    INFT_Q_TRY
    inft::DeviceGuard g(q->device);
    delete q;
    INFT_Q_CATCH
}

}  // extern "C"
