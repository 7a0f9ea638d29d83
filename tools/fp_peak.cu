// FP64 / FP32 FMA throughput microbenchmark (MEASURED_PEAKS.json has no FP64 entry).
// Each thread runs 8 independent FMA chains for ITER iterations; grid = 148 SMs x 8 CTAs x 256
// threads.  Reports TFLOP/s (2 flops per FMA).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp_peak tools/fp_peak.cu && tools/fp_peak
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void k_fma(T* out, int iters, T a, T b) {
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == (T)1.2345) out[0] = x0;  // keep the chains live
}

template <typename T>
static double run(const char* name) {
    int dev = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    T* out;
    cudaMalloc(&out, sizeof(T));
    const int iters = 4096, blocks = nsm * 8, threads = 256;
    k_fma<T><<<blocks, threads>>>(out, 16, (T)0.999, (T)0.001);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_fma<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    const double tf = flops / (ms * 1e-3) / 1e12;
    printf("%s FMA: %.2f TFLOP/s (%.3f ms, %d SMs)\n", name, tf, ms, nsm);
    cudaFree(out);
    return tf;
}

int main() {
    run<double>("FP64");
    run<float>("FP32");
    run<double>("FP64");
    run<float>("FP32");
    return 0;
}
