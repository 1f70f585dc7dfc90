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
    void* scratch = nullptr;     // reduction partials, sort / binning buffers
    size_t scratch_bytes = 0;
    void* scratch_tail = nullptr;  // the prefix-sum tile totals (used while `scratch` is held)
    size_t scratch_tail_bytes = 0;
};

namespace mdkk {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
// Grow-only scratch arena (synchronises the device only when it grows; a pointer
// from an earlier call is invalid after a call that grows it).
void* scratch(mdkk_ctx* ctx, size_t bytes);
// A second, independent arena for the prefix sums' tile totals.
void* scratch_tail(mdkk_ctx* ctx, size_t bytes);
// Exclusive prefix sums (csrc/sort.cu), out[k] = in[0] + ... + in[k-1]; in != out.
int exclusive_scan_i32(mdkk_ctx* ctx, const int* in, int* out, long long n, cudaStream_t s);
int exclusive_scan_i64(mdkk_ctx* ctx, const long long* in, long long* out, long long n, cudaStream_t s);
// mdkk_bucket_sort (many buckets) from counts the caller already took: cnt[nbuckets + 1]
// (zeroed, then one increment per key; cnt[nbuckets] = 0), reused as the scatter cursors.
int bucket_sort_counted(mdkk_ctx* ctx, const int* keys, int n, int nbuckets, int* cnt, int* bucket_start,
                        int* order, cudaStream_t s);
constexpr int kSortSmallBuckets = 64;   // mdkk_bucket_sort's few-bucket path (per-block tables) up to here

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(long long n, int block, int max_blocks = 1 << 30) {
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return static_cast<int>(g);
}

// AoS-padded double4 row access: one 256-bit load per row (sm_100
// LDG.E.ENL2.256), i.e. one 32-byte sector per neighbour gather.
__device__ __forceinline__ double4 ld4(const double* p, long long i) {  // read-only in this kernel
    double4 v;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + 4 * i));
    return v;
}
__device__ __forceinline__ double4 ld4_nc(const double* p, long long i) {  // data this kernel may write
    double4 v;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p + 4 * i)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st4(double* p, long long i, double4 v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 4 * i), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}

// r^2 with explicit rounding and no FMA contraction.  The reference evaluates
// np.einsum("ij,ij->i", dr, dr) (mdkk/neighbor.py:126); the product/sum order
// below is the one SURVEY §7 measured as bit-identical to that einsum.
__device__ __forceinline__ double r2_exact(double dx, double dy, double dz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
}

// 1/x to ~1 ulp: the MUFU.RCP64H seed refined by two Newton steps (5 FP64 ops instead of
// the IEEE division sequence; the pair kernels' tolerances are 1e-10 relative).
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
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
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum of K doubles per thread into out[K] (thread 0 holds result).
// acc: add to out[k] (a second pass over the same blocks) instead of storing.
template <int K, int BLOCK>
__device__ __forceinline__ void block_sum(double (&v)[K], double* out, bool acc = false) {
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
            out[k] = acc ? out[k] + s : s;
        }
    }
}

// Deterministic second stage: out[k] = sum_b partials[b*K + k], fixed order;
// out[K .. zero_to) are cleared in the same launch.
void reduce_partials(const double* partials, int nblocks, int K, double* out, cudaStream_t s, int zero_to = 0);
// The same, with a halo pack (x_ghost[k] = x[idx[k]] + shifts[code[k]], k < n_pack) in the same
// launch; *zero_slot (optional) is cleared too.
void reduce_partials_pack(const double* partials, int nblocks, int K, double* out, int zero_to, const double* x,
                          const int* idx, const int8_t* code, const double* shifts, int n_pack, double* x_ghost,
                          double* zero_slot, cudaStream_t s);

// A drift maximum that cannot hide a blow-up: NaN / inf become +inf before the
// (NaN-dropping) fmax reductions, so the host's per-step read-back sees it
// (the every-step non-finite abort, mdkk/driver/simulation.py:459-478).
__device__ __forceinline__ double finite_or_inf(double v) { return v <= 1.7976931348623157e308 ? v : __longlong_as_double(0x7ff0000000000000LL); }

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
