// Standalone probe: 2-D TMA load of [rows][16 x 8-byte] boxes (SWIZZLE_128B) from a
// [R][N] array of complex values, plus a 1-D bulk copy completing on the same barrier.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <typename C>
__global__ void probe(const __grid_constant__ CUtensorMap map, const C* src, C* out, int N, int R, int with_bulk,
                      const double* bulk_src, int off) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bar;
    const int col = blockIdx.x * 16 / (int)(sizeof(C) / 8);  // complex index of this tile
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t bytes = 4096 + (with_bulk ? 1280 : 0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(sa(smem)),
            "l"((uint64_t)&map), "r"(col * (int)(sizeof(C) / 8) + off), "r"(0), "r"(sa(&bar)));
        if (with_bulk)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa(smem + 8192)),
                         "l"(bulk_src), "r"(1280), "r"(sa(&bar)));
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                     : "=r"(ok)
                     : "r"(sa(&bar)));
    const int lane = threadIdx.x;
    const int EB = 128 / (int)sizeof(C);
    for (int v = 0; v < EB; ++v) {
        int c = sizeof(C) == 16 ? v : v >> 1;
        uint32_t off = lane * 128 + ((c ^ (lane & 7)) << 4) + (sizeof(C) == 16 ? 0 : (v & 1) * 8);
        C val = *reinterpret_cast<const C*>(smem + off);
        if (col + v < N && lane < R) out[(size_t)lane * N + col + v] = val;
    }
}

template <typename C>
int run(int N, int R, int with_bulk, int off, int swz) {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    size_t n = (size_t)N * R;
    std::vector<C> h(n);
    for (size_t i = 0; i < n; i++) {
        ((double*)&h[i])[0] = (double)i;
    }
    if (sizeof(C) == 8)
        for (size_t i = 0; i < n; i++) {
            ((float*)&h[i])[0] = (float)(i % 100000);
            ((float*)&h[i])[1] = -1.f;
        }
    C *d, *o;
    double* b;
    cudaMalloc(&d, n * sizeof(C));
    cudaMalloc(&o, n * sizeof(C));
    cudaMalloc(&b, 4096);
    cudaMemcpy(d, h.data(), n * sizeof(C), cudaMemcpyHostToDevice);
    cudaMemset(o, 0, n * sizeof(C));
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)N * sizeof(C) / 8, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)N * sizeof(C)};
    cuuint32_t box[2] = {swz ? 16u : 2u, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int tiles = (int)((N + 128 / sizeof(C) - 1) / (128 / sizeof(C)));
    cudaFuncSetAttribute(probe<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    if (!swz) {
        // expect_tx below counts a 4096-byte box; a {2, 32} box is 512 bytes: launch the
        // alignment check through the swizzle-free variant with matching byte count
    }
    probe<C><<<tiles, 32, 16384>>>(map, d, o, N, R, with_bulk, b, off);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<C> g(n);
    cudaMemcpy(g.data(), o, n * sizeof(C), cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < n; i++)
        if (memcmp(&g[i], &h[i], sizeof(C))) bad++;
    printf("sizeof(C)=%zu N=%d R=%d bulk=%d off=%d swz=%d encode=%d sync=%s bad=%zu\n", sizeof(C), N, R, with_bulk,
           off, swz, (int)r, cudaGetErrorString(e), bad);
    cudaFree(d);
    cudaFree(o);
    cudaFree(b);
    return e != cudaSuccess;
}

int main(int argc, char** argv) {
    int N = atoi(argv[2]), R = atoi(argv[3]), bulk = atoi(argv[4]);
    int off = argc > 5 ? atoi(argv[5]) : 0;  // extra inner start offset in 8-byte elements
    if (argv[1][0] == 'f') return run<float2>(N, R, bulk, off, 1);
    return run<double2>(N, R, bulk, off, 1);
}
