// Shared helpers for the mdkk_b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/mdkk_b200.h"

struct mdkk_ctx {
    int device = 0;
    int sm_count = 148;
    void* scratch = nullptr;     // reduction partials, CUB temp storage
    size_t scratch_bytes = 0;
};

namespace mdkk {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
// Grow-only scratch arena (synchronises the device only when it grows).
void* scratch(mdkk_ctx* ctx, size_t bytes);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(long long n, int block, int max_blocks = 1 << 30) {
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return static_cast<int>(g);
}

// AoS-padded double4 row access as two 16-byte vector loads.
__device__ __forceinline__ double4 ld4(const double* p, long long i) {
    const double2* q = reinterpret_cast<const double2*>(p + 4 * i);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ double4 ld4_nc(const double* p, long long i) {  // mutable data
    const double2* q = reinterpret_cast<const double2*>(p + 4 * i);
    double2 a = q[0], b = q[1];
    return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4(double* p, long long i, double4 v) {
    double2* q = reinterpret_cast<double2*>(p + 4 * i);
    q[0] = make_double2(v.x, v.y);
    q[1] = make_double2(v.z, v.w);
}

// r^2 with explicit rounding and no FMA contraction.  The reference evaluates
// np.einsum("ij,ij->i", dr, dr) (mdkk/neighbor.py:126); the product/sum order
// below is the one SURVEY §7 measured as bit-identical to that einsum.
__device__ __forceinline__ double r2_exact(double dx, double dy, double dz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum of K doubles per thread into out[K] (thread 0 holds result).
template <int K, int BLOCK>
__device__ __forceinline__ void block_sum(double (&v)[K], double* out) {
    __shared__ double sm[BLOCK / 32][K];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) sm[wid][k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int w = 0; w < BLOCK / 32; ++w) s += sm[w][k];
            out[k] = s;
        }
    }
}

// Deterministic second stage: out[k] = sum_b partials[b*K + k], fixed order.
void reduce_partials(const double* partials, int nblocks, int K, double* out, cudaStream_t s);

// Non-negative doubles order like their int64 bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace mdkk

namespace mdkk {
void count_launch();
}

// Every kernel launch site checks the launch and bumps the process-wide
// launch counter (mdkk_launch_count) that bench.py reports as gpu_launches.
#define MDKK_CHECK_LAUNCH(what)                                      \
    do {                                                             \
        cudaError_t e_ = cudaGetLastError();                         \
        if (e_ != cudaSuccess) return mdkk::cuda_fail(e_, what);     \
        mdkk::count_launch();                                        \
    } while (0)
