/*
 * inft.h -- C ABI of the B200-native (sm_100a) direct inverse NFFT.
 *
 * Method: M. Kircheis, D. Potts, "Direct inversion of the nonequispaced fast
 * Fourier transform", arXiv:1811.05335.  Citations "P:<n>" refer to lines of
 * the paper's source; readings "A<n>" to DESIGN.md.
 *
 * The library solves, for FIXED nodes x_j ("fixed nodes for several
 * problems") and many right-hand sides,
 *   problem (1) inverse NFFT          A fhat = f
 *   problem (2) inverse adjoint NFFT  A^* f  = h
 * with A = (e^{2 pi i k x_j})_{j, k} (eq. matrix_A), by the paper's
 * modified (adjoint) NFFT with an optimised (2m+1)-sparse matrix B_opt:
 *   inverse:          fhat ~= s D^* F^* B_opt^* f
 *   inverse adjoint:  f    ~= s B_opt F D h
 * D = diag(1/(M_sigma what(k))) (eq. matrix_D), F the truncated M_sigma-point
 * Fourier matrix (eq. matrix_F), s = 1/M for the node-wise Alg. "Fast
 * optimization of the matrix B*" and s = 1 for the grid-wise Alg. "Fast
 * optimization of the matrix B" (reading A2).
 *
 * Conventions (all calls):
 *  - Every call returns inft_status; nothing throws or aborts across the ABI.
 *  - Complex data are interleaved (re, im): double pairs for INFT_C128 plans,
 *    float pairs for INFT_C64 plans (= torch.complex128 / complex64 memory).
 *  - Batches are RHS-major: f[r*N + j], fhat[r*Mtot + c] with the centered
 *    spectral index c = k + M/2 (2-D: c = (k1 + M1/2)*M2 + (k2 + M2/2)),
 *    Mtot = prod(M).
 *  - "host or device" pointers are detected with cudaPointerGetAttributes;
 *    host data are staged through plan-owned device buffers with pipelined
 *    copies (pinned host memory overlaps copies with compute).
 *  - Calls are stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *    default stream) and asynchronous unless stated.  A plan owns scratch
 *    memory: do not run two applies of one plan concurrently on two streams.
 *  - The caller owns every buffer it passes; the plan owns copies of nodes,
 *    bins, B_opt, the deconvolution table, cuFFT plans and workspaces, and
 *    frees them in inft_destroy.
 */
#ifndef INFT_H
#define INFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct inft_plan_s* inft_plan_t; /* opaque plan handle */
typedef void* inft_stream_t;             /* a cudaStream_t */

typedef enum {
    INFT_OK = 0,
    INFT_ERR_INVALID_ARG = 1,     /* bad size/enum/pointer, M odd, sigma*M not an even integer, ... */
    INFT_ERR_NODE_RANGE = 2,      /* a node coordinate not finite or outside [-1/2, 1/2) */
    INFT_ERR_ZERO_WINDOW_HAT = 3, /* what(k) <= 0 for some |k| <= M/2 (D would not exist) */
    INFT_ERR_NOT_PRECOMPUTED = 4, /* apply before inft_precompute / inft_set_bopt */
    INFT_ERR_CUDA = 5,            /* a CUDA runtime call failed (message: inft_last_error) */
    INFT_ERR_CUFFT = 6,           /* a cuFFT call failed */
    INFT_ERR_OOM = 7,             /* device allocation failed */
    INFT_ERR_UNSUPPORTED = 8      /* valid request this build does not implement */
} inft_status;

typedef enum {
    INFT_KAISER_BESSEL = 0, /* reading A7: what(k) = I0(m sqrt(b^2-(2 pi k/M_sigma)^2))/M_sigma, b = pi(2-1/sigma) */
    INFT_DIRICHLET = 1,     /* Dirichlet-kernel variant, Remarks P:934-957 / P:1343-1358 (reading A21):
                             * what(k) = 1 for |k| < M/2, the k = -M/2 entry of D zeroed, so
                             * d_k = s/M_sigma (k != -M/2); only with the optimised B_opt
                             * (ALG1/ALG2 or inft_set_bopt): there is no window function in space,
                             * INFT_PLAIN_NFFT returns INFT_ERR_INVALID_ARG */
    INFT_BSPLINE = 2        /* B-spline window of the paper's experiments (reading A24):
                             * w(x) = M_2m(M_sigma x), the centred cardinal B-spline of order 2m
                             * (support [-m, m]/M_sigma, exact), what(k) = sinc(pi k/M_sigma)^2m / M_sigma */
} inft_window;

typedef enum {
    INFT_AUTO = 0,           /* Alg. 1 if prod(M) >= N, else Alg. 2 */
    INFT_ALG1_NODEWISE = 1,  /* Alg. "Fast optimization of the matrix B*", s = 1/M */
    INFT_ALG2_GRIDWISE = 2,  /* Alg. "Fast optimization of the matrix B",  P:1298-1333, s = 1 */
    INFT_PLAIN_NFFT = 3      /* B = window matrix (eq. matrix_B), s = 1: the ordinary adjoint NFFT / NFFT */
} inft_method;

typedef enum { INFT_C128 = 0, INFT_C64 = 1 } inft_precision;
typedef enum { INFT_WEIGHTS_REAL = 0, INFT_WEIGHTS_COMPLEX = 1 } inft_weights;

typedef struct {
    int32_t d;                 /* 1 or 2 */
    int64_t M[2];              /* coefficients per dimension (M[1] = 1 for d = 1) */
    int64_t Msigma[2];         /* oversampled grid per dimension */
    int64_t N;                 /* nodes */
    int32_t m;                 /* cut-off */
    int32_t P;                 /* slots per node: 2m+1 (1-D), (2m+1)^2 (2-D) */
    int32_t tile[2];           /* bin / segment width per dimension (reading A19) */
    int32_t precision;         /* inft_precision */
    int32_t method;            /* inft_method in effect, -1 before precompute */
    int32_t weights;           /* inft_weights in effect */
    double scale;              /* s folded into D (reading A2) */
    double tau;                /* min-norm cutoff used by inft_precompute (reading A6) */
    int64_t n_rank_deficient;  /* columns whose system dropped singular directions */
    int64_t n_empty_cols;      /* grid columns with I(l) empty (Alg. 2) */
    int64_t max_col_size;      /* max |I(l)| (Alg. 2) or max |I(x_j)| (Alg. 1) */
    double max_abs_w;          /* max |B_opt entry| */
    int32_t perm_identity;     /* 1 if the bin sort left the caller's node order unchanged */
    int32_t fast_path;         /* 1: register-window spread/gather kernels, 2: their TMA-staged ring variant */
    int32_t fused_fft;         /* 1 if the fused two-pass FFT (with deconvolution) replaces cuFFT */
    int32_t max_lowrank_rank;  /* Alg. 2: largest pivoted-Cholesky rank among columns with |I(l)| > 64 */
    size_t workspace_bytes;    /* device bytes currently owned by the plan */
} inft_info;

/* Build a plan for fixed nodes.
 *   out     : receives the handle (NULL on failure).
 *   d       : 1 or 2 (2-D is the tensor-product reading A12).
 *   M       : [d] even coefficient counts (P:37 M in 2N).
 *   N       : number of nodes, >= 0.
 *   nodes   : host or device pointer, N x d row-major doubles, each coordinate
 *             finite and in [-1/2, 1/2) (else INFT_ERR_NODE_RANGE; no wrapping).
 *   sigma   : oversampling; sigma*M[i] must be an even integer.
 *   m       : cut-off, 1 <= m <= M_sigma_i / 2.
 *   device  : CUDA device ordinal the plan lives on.
 * Computes l0_j = ceil(M_sigma x_j) - m per dimension with a correctly
 * rounded product (reading A20), the tile bins and the stable node
 * permutation (A19), and d_k = s/(M_sigma what(k)) (eq. matrix_D).  Synchronous. */
inft_status inft_plan(inft_plan_t* out, int d, const int64_t* M, int64_t N, const double* nodes,
                      double sigma, int m, inft_window window, inft_precision prec, int device,
                      inft_stream_t stream);

/* Compute B_opt on the GPU (setup stage):
 *   INFT_ALG2_GRIDWISE: per grid point l minimise ||L_l b - e_l||
 *     through the normal equations in Gram form.
 *   INFT_ALG1_NODEWISE: per node j minimise ||K_j b - M e_j||.
 *   INFT_PLAIN_NFFT: B = window matrix (eq. matrix_B).
 *   INFT_AUTO: Alg. 1 if prod(M) >= N else Alg. 2.
 *   wt  : real-constrained ("B in R^{N x M_sigma}", default) or complex.
 *   tau : relative singular-value cutoff of the min-norm solution (A6);
 *         <= 0 selects the default 1e-6.
 * Synchronous.  Errors: INFT_ERR_UNSUPPORTED for combinations this build lacks. */
inft_status inft_precompute(inft_plan_t plan, inft_method method, inft_weights wt, double tau,
                            inft_stream_t stream);

/* Inverse NFFT, problem (1): fhat[r] = s D^* F^* B_opt^* f[r], r < R.
 *   f    : host or device, [R][N] complex (caller node order).
 *   fhat : host or device, [R][Mtot] complex, centered.
 * Steps: spread (B_opt^*), M_sigma-point FFT (F^*), truncate + deconvolve (D^*).
 * R = 0 is a no-op.  Errors: INFT_ERR_NOT_PRECOMPUTED, INFT_ERR_INVALID_ARG. */
inft_status inft_apply(inft_plan_t plan, const void* f, void* fhat, int64_t R, inft_stream_t stream);

/* Inverse adjoint NFFT, problem (2): f[r] = s B_opt F D h[r].
 *   h : host or device, [R][Mtot] complex centered;  f : host or device, [R][N].
 * Steps: deconvolve + zero-pad (D), FFT (F), gather (B_opt). */
inft_status inft_adjoint_apply(inft_plan_t plan, const void* h, void* f, int64_t R,
                               inft_stream_t stream);

/* Release every allocation of the plan (NULL is accepted). */
inft_status inft_destroy(inft_plan_t plan);

/* Introspection / checkpoint of the expensive setup.  All output pointers are
 * HOST pointers; calls are synchronous.
 *   inft_get_bins : l0 [N*d] (caller order, row-major), bin [N] (caller order),
 *                   perm [N] (sorted position -> caller index).  Any may be NULL.
 *   inft_get_bopt : w [N][P] doubles (real weights) or [N][P] complex doubles
 *                   (complex weights), caller order, slot t <-> grid l0_j + t
 *                   (2-D: t = t1*(2m+1) + t2).
 *   inft_set_bopt : import such a w (host pointer) as B_opt for `method`
 *                   (sets s: 1/prod(M) for INFT_ALG1_NODEWISE, else 1).
 *   inft_get_deconv: d [sum M_i] doubles, the per-dimension tables with s
 *                   folded into the first dimension (D = diag(d1 (x) d2)). */
inft_status inft_get_bins(inft_plan_t plan, int32_t* l0, int32_t* bin, int32_t* perm);
inft_status inft_get_bopt(inft_plan_t plan, void* w);
inft_status inft_set_bopt(inft_plan_t plan, inft_method method, inft_weights wt, const void* w);
inft_status inft_get_deconv(inft_plan_t plan, double* d);
inft_status inft_get_info(inft_plan_t plan, inft_info* info);

/* Per-stage device time of the apply, measured with CUDA events recorded on
 * the launching stream around every stage of every apply while profiling is
 * enabled.  Stages (one kernel each on the fused 1-D path, info.fused_fft = 1):
 *   0 spread a2;
 *   1 FFT a3 (unfused: cuFFT; fused: pass A, column FFTs + four-step twiddles);
 *   2 truncate+deconvolve a4 (fused: pass B, row FFTs + a4);
 *   3 deconvolve+pad a5 (fused: pass A, a5 + column FFTs);
 *   4 FFT a6 (unfused: cuFFT; fused: pass B, row FFTs + grid halo);
 *   5 gather a7.
 * inft_get_profile synchronises with the recorded events; reset != 0 clears
 * the accumulators. */
typedef struct {
    double ms[6];
    int64_t count[6];
} inft_profile;
inft_status inft_set_profiling(inft_plan_t plan, int enable);
inft_status inft_get_profile(inft_plan_t plan, inft_profile* out, int reset);

/* Number of kernel launches this plan issued since creation (evidence for
 * benchmarks; cuFFT's internal kernels are not counted). */
int64_t inft_kernel_launches(inft_plan_t plan);

/* ---------------------------------------------------------------------------
 * Quadratic case M = N (paper Section "The quadratic case",
 * P:344-489, adjoint Remark P:576-584).  For N distinct nodes y_j and the
 * equispaced targets x_l = -1/2 + l/N + delta (delta in (0, 1/N),
 * 0 selects 1/(2N), reading A23), the inverse NFFT A fhat = f with
 * A = (e^{2 pi i k y_j})_{j, k=-N/2..N/2-1} is solved by the Lagrange relation
 *   g_l = a_l sum_j f_j b_j (cot(pi (x_l - y_j)) - i)        (eq. lagrange_formula)
 *   fcheck_k = (1/N) sum_l g_l e^{-2 pi i k x_l}              (Alg. step 6, one FFT)
 * a_l = prod_n sin(pi (x_l - y_n)), b_j = prod_{n != j} 1/sin(pi (y_j - y_n))
 * (eq. coeff_ab) in the log domain with counted signs and the
 * balancing shift s = (max ln|b| - max ln|a|)/2 (Remark P:431-449, reading A22).
 * The sums run by the paper's NFFT-based fast summation (O(N log N),
 * error ~1e-15 N relative) for N >= 512, by exact direct O(N^2) GPU sums below
 * that or with INFT_QUAD_DIRECT=1 set at plan time.  Complex128 only; RHS-major
 * [R][N] data, host or device pointers (host data staged synchronously).
 * ------------------------------------------------------------------------- */
typedef struct inft_quad_s* inft_quad_t; /* opaque quadratic-case plan */

/* Build: copies the nodes (host or device, N doubles in [-1/2, 1/2)), computes
 * x, a, b, s on `device`.  N even, >= 2.  Synchronous.  Errors:
 * INFT_ERR_INVALID_ARG (N odd / < 2, delta outside (0, 1/N)), INFT_ERR_NODE_RANGE
 * (a node outside [-1/2, 1/2), or coincident nodes: y_j = y_n or y_j = x_l). */
inft_status inft_quad_plan(inft_quad_t* out, int64_t N, const double* nodes, double delta, int device,
                           inft_stream_t stream);
/* Inverse NFFT, quadratic case: f [R][N] (samples at the nodes, caller order)
 * -> fhat [R][N], centered index c = k + N/2.  Stream-ordered (device data). */
inft_status inft_quad_apply(inft_quad_t plan, const void* f, void* fhat, int64_t R, inft_stream_t stream);
/* Inverse adjoint NFFT, quadratic case (eq. lagrange_formula_adjoint):
 * h [R][N] centered -> f [R][N] with f = (A^*)^{-1} h, v = (1/N) sum_k h_k e^{2 pi i k x_l}. */
inft_status inft_quad_adjoint_apply(inft_quad_t plan, const void* h, void* f, int64_t R, inft_stream_t stream);
/* Host copies of the targets x [N], signed stabilised a [N], b [N] and the shift s
 * (any pointer may be NULL).  Synchronous. */
inft_status inft_quad_get_coeffs(inft_quad_t plan, double* x, double* a, double* b, double* s);
/* Kernel launches issued by this plan (cuFFT's not counted). */
inft_status inft_quad_kernel_launches(inft_quad_t plan, int64_t* count);
inft_status inft_quad_destroy(inft_quad_t plan);

const char* inft_status_string(inft_status status);
/* Thread-local text of the last error (CUDA / cuFFT message), "" if none. */
const char* inft_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* INFT_H */
