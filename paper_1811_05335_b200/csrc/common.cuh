// Device helpers shared by the apply kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace inft {

template <typename T>
struct C2T;
template <>
struct C2T<double> {
    using type = double2;
};
template <>
struct C2T<float> {
    using type = float2;
};
template <typename T>
using C2 = typename C2T<T>::type;

template <typename T>
__device__ __forceinline__ C2<T> mk(T x, T y) {
    C2<T> v;
    v.x = x;
    v.y = y;
    return v;
}

__device__ __forceinline__ int64_t mod64(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

// The P real weights of one sorted node record (16-byte aligned, padded to PP).
// Global version: every lane of the warp reads the same address (broadcast).
template <typename T, int P>
struct WeightLoader;

template <int P>
struct WeightLoader<double, P> {
    __device__ __forceinline__ static void load(const double* __restrict__ rec, double (&w)[P]) {
        const double2* v = reinterpret_cast<const double2*>(rec);
#pragma unroll
        for (int q = 0; q < (P + 1) / 2; ++q) {
            double2 a = __ldg(v + q);
            w[2 * q] = a.x;
            if (2 * q + 1 < P) w[2 * q + 1] = a.y;
        }
    }
    // shared-memory record (broadcast LDS.128)
    __device__ __forceinline__ static void load_smem(const double* rec, double (&w)[P]) {
        const double2* v = reinterpret_cast<const double2*>(rec);
#pragma unroll
        for (int q = 0; q < (P + 1) / 2; ++q) {
            double2 a = v[q];
            w[2 * q] = a.x;
            if (2 * q + 1 < P) w[2 * q + 1] = a.y;
        }
    }
};

template <int P>
struct WeightLoader<float, P> {
    __device__ __forceinline__ static void load(const float* __restrict__ rec, float (&w)[P]) {
        const float4* v = reinterpret_cast<const float4*>(rec);
#pragma unroll
        for (int q = 0; q < (P + 3) / 4; ++q) {
            float4 a = __ldg(v + q);
            w[4 * q] = a.x;
            if (4 * q + 1 < P) w[4 * q + 1] = a.y;
            if (4 * q + 2 < P) w[4 * q + 2] = a.z;
            if (4 * q + 3 < P) w[4 * q + 3] = a.w;
        }
    }
    __device__ __forceinline__ static void load_smem(const float* rec, float (&w)[P]) {
        const float4* v = reinterpret_cast<const float4*>(rec);
#pragma unroll
        for (int q = 0; q < (P + 3) / 4; ++q) {
            float4 a = v[q];
            w[4 * q] = a.x;
            if (4 * q + 1 < P) w[4 * q + 1] = a.y;
            if (4 * q + 2 < P) w[4 * q + 2] = a.z;
            if (4 * q + 3 < P) w[4 * q + 3] = a.w;
        }
    }
};

// The node's slot base n0 = l0 mod M_sigma is stored as int32 bits in the first
// padding element (index P) of its weight record.
__device__ __forceinline__ int rec_n0(const double* rec, int P) { return (int)__double_as_longlong(rec[P]); }
__device__ __forceinline__ int rec_n0(const float* rec, int P) { return __float_as_int(rec[P]); }
__device__ __forceinline__ double n0_as(double, int n0) { return __longlong_as_double((long long)n0); }
__device__ __forceinline__ float n0_as(float, int n0) { return __int_as_float(n0); }

#define INFT_CASES_16(X) \
    X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)

#define INFT_CASES_32(X) \
    X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
    X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31)

}  // namespace inft
