// Scatter deconfliction strategies (mdkk/memspace.py:165-257, ScatterAccumulator).
//
// The reference accumulates indexed contributions with one of three
// strategies that agree up to floating-point reassociation:
//   Serial    -- ordered sequential np.add.at            -> mdkk_scatter_ordered
//   Atomic    -- concurrent adds on shared storage       -> mdkk_scatter_atomic (FP64 RED)
//   Duplicate -- per-worker staging copies + a combine   -> mdkk_scatter_combine
// Targets are row-major [n_rows][ld] doubles; a contribution updates the
// first `width` entries of a row.  All kernels are grid-stride, HBM-bound.
#include "common.cuh"

namespace {

constexpr int kBlock = 256;

__global__ void k_scatter_atomic(double* __restrict__ target, int ld, int width, const long long* __restrict__ idx,
                                 const double* __restrict__ vals, long long n) {
    const long long total = n * width;
    for (long long t = blockIdx.x * (long long)kBlock + threadIdx.x; t < total; t += (long long)gridDim.x * kBlock) {
        const long long e = t / width;
        const int c = (int)(t - e * width);
        atomicAdd(target + idx[e] * ld + c, vals[t]);
    }
}

// Segmented ordered sum: `sorted_idx` is the stable sort of the contribution
// indices and `perm` the matching positions, so each segment lists one row's
// contributions in their original order.  The segment head adds them one by
// one onto the row's current value: bit-identical to sequential np.add.at.
__global__ void k_scatter_ordered(double* __restrict__ target, int ld, int width,
                                  const long long* __restrict__ sorted_idx, const long long* __restrict__ perm,
                                  const double* __restrict__ vals, long long n) {
    for (long long k = blockIdx.x * (long long)kBlock + threadIdx.x; k < n; k += (long long)gridDim.x * kBlock) {
        const long long row = sorted_idx[k];
        if (k > 0 && sorted_idx[k - 1] == row) continue;
        double* dst = target + row * ld;
        for (int c = 0; c < width; ++c) {
            double acc = dst[c];
            for (long long q = k; q < n && sorted_idx[q] == row; ++q) acc += vals[perm[q] * width + c];
            dst[c] = acc;
        }
    }
}

// out[e] += ((s_0[e] + s_1[e]) + s_2[e]) + ... (np.add.reduce over the copies).
__global__ void k_scatter_combine(const double* __restrict__ stage, int copies, long long stride,
                                  double* __restrict__ out, long long n) {
    for (long long e = blockIdx.x * (long long)kBlock + threadIdx.x; e < n; e += (long long)gridDim.x * kBlock) {
        double acc = stage[e];
        for (int c = 1; c < copies; ++c) acc += stage[c * stride + e];
        out[e] += acc;
    }
}

__global__ void k_index_range(const long long* __restrict__ idx, long long n, long long n_rows,
                              unsigned long long* __restrict__ bad) {
    for (long long e = blockIdx.x * (long long)kBlock + threadIdx.x; e < n; e += (long long)gridDim.x * kBlock) {
        const long long v = idx[e];
        if (v < 0 || v >= n_rows) atomicMin(bad, (unsigned long long)e);
    }
}

int blocks_for(long long n) { return mdkk::grid_for(n, kBlock, 148 * 16); }

}  // namespace

extern "C" int mdkk_scatter_atomic(double* target, int ld, int width, const long long* idx, const double* vals,
                                   long long n, void* stream) {
    if (!target || ld < width || width < 1 || n < 0 || (n && (!idx || !vals))) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_scatter_atomic<<<blocks_for(n * width), kBlock, 0, mdkk::as_stream(stream)>>>(target, ld, width, idx, vals, n);
    MDKK_CHECK_LAUNCH("k_scatter_atomic");
    return MDKK_OK;
}

extern "C" int mdkk_scatter_ordered(double* target, int ld, int width, const long long* sorted_idx,
                                    const long long* perm, const double* vals, long long n, void* stream) {
    if (!target || ld < width || width < 1 || n < 0 || (n && (!sorted_idx || !perm || !vals))) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_scatter_ordered<<<blocks_for(n), kBlock, 0, mdkk::as_stream(stream)>>>(target, ld, width, sorted_idx, perm,
                                                                             vals, n);
    MDKK_CHECK_LAUNCH("k_scatter_ordered");
    return MDKK_OK;
}

extern "C" int mdkk_scatter_combine(const double* stage, int copies, long long stride, double* out, long long n,
                                    void* stream) {
    if (!stage || !out || copies < 1 || n < 0 || stride < n) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_scatter_combine<<<blocks_for(n), kBlock, 0, mdkk::as_stream(stream)>>>(stage, copies, stride, out, n);
    MDKK_CHECK_LAUNCH("k_scatter_combine");
    return MDKK_OK;
}

extern "C" int mdkk_index_range(const long long* idx, long long n, long long n_rows, unsigned long long* bad,
                                void* stream) {
    if (n < 0 || !bad || (n && !idx)) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_index_range<<<blocks_for(n), kBlock, 0, mdkk::as_stream(stream)>>>(idx, n, n_rows, bad);
    MDKK_CHECK_LAUNCH("k_index_range");
    return MDKK_OK;
}
