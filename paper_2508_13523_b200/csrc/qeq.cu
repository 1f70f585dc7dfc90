// Charge equilibration on the GPU (mdkk/qeq.py): over-allocated CSR assembly
// with 64-bit row offsets, SpMV / fused dual SpMV, Gershgorin guard, and the
// conjugate-gradient vector stages.  Every reduction is a fixed-order
// two-stage sum, so a fused two-system solve reproduces two sequential solves
// bit for bit (mdkk/qeq.py:233-274): the per-row SpMV sums and the dot
// partials do not depend on how many systems share the traversal.

#include "common.cuh"

namespace {

constexpr int kBlock = 256;
constexpr int kRowLanes = 8;   // lanes per matrix row in the SpMV

__global__ void k_qeq_caps(const int* __restrict__ counts, int n, int cap, long long* __restrict__ caps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) caps[i] = (long long)min(counts[i], cap) + 1;   // list row + diagonal (mdkk/qeq.py:104-106)
    if (i == n) caps[i] = 0;
}

// Row i: diagonal eta first, then the list partners within the QEq cutoff in
// table order, value (r^3 + gamma^-3)^(-1/3), column = owner's local index
// (ghosts fold onto their owner, mdkk/qeq.py:90-133).
__global__ void k_qeq_build(const double* __restrict__ x, int n_local, const int* __restrict__ table,
                            const int* __restrict__ counts, int cap, const int* __restrict__ oidx,
                            const long long* __restrict__ off, double eta, double g3, double rc2,
                            double* __restrict__ values, int* __restrict__ columns, int* __restrict__ row_nnz) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    const double4 xi = mdkk::ld4(x, i);
    const int n = min(counts[i], cap);
    long long s = off[i];
    values[s] = eta;
    columns[s] = i;
    int k1 = 1;
    for (int k = 0; k < n; ++k) {
        const int j = table[((long long)(i >> 5) * cap + k) * 32 + (i & 31)];
        const double4 xj = mdkk::ld4(x, j);
        const double r2 = mdkk::r2_exact(xj.x - xi.x, xj.y - xi.y, xj.z - xi.z);
        if (!(r2 < rc2)) continue;
        const double r = sqrt(r2);
        values[s + k1] = pow(r * r * r + g3, -1.0 / 3.0);
        columns[s + k1] = oidx[j];
        ++k1;
    }
    row_nnz[i] = k1;
}

// y_s = H x_s for s < NS systems sharing one traversal; optional per-block
// partials of x_s . y_s.  kRowLanes lanes per row, fixed shuffle tree.
template <int NS>
__global__ void __launch_bounds__(kBlock) k_qeq_spmv(const long long* __restrict__ off,
                                                     const double* __restrict__ values,
                                                     const int* __restrict__ columns, const int* __restrict__ nnz,
                                                     int n, const double* __restrict__ x1,
                                                     const double* __restrict__ x2, double* __restrict__ y1,
                                                     double* __restrict__ y2, double* __restrict__ partials) {
    const int t = blockIdx.x * kBlock + threadIdx.x;
    const int row = t / kRowLanes, l = t % kRowLanes;
    double acc[2] = {0.0, 0.0};
    if (row < n) {
        const long long s0 = off[row];
        const int m = nnz[row];
        for (int k = l; k < m; k += kRowLanes) {
            const double v = values[s0 + k];
            const int c = columns[s0 + k];
            acc[0] += v * x1[c];
            if (NS == 2) acc[1] += v * x2[c];
        }
    }
#pragma unroll
    for (int o = kRowLanes / 2; o > 0; o >>= 1) {
        acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
        if (NS == 2) acc[1] += __shfl_xor_sync(0xffffffffu, acc[1], o);
    }
    double d[2] = {0.0, 0.0};
    if (row < n && l == 0) {
        y1[row] = acc[0];
        d[0] = x1[row] * acc[0];
        if (NS == 2) {
            y2[row] = acc[1];
            d[1] = x2[row] * acc[1];
        }
    }
    if (partials) mdkk::block_sum<2, kBlock>(d, partials + 2LL * blockIdx.x);
}

// Gershgorin guard (mdkk/qeq.py:180-194): first row with diag <= sum |offdiag|.
__global__ void k_qeq_gershgorin(const long long* __restrict__ off, const double* __restrict__ values,
                                 const int* __restrict__ columns, const int* __restrict__ nnz, int n,
                                 int* __restrict__ bad, double* __restrict__ diag, double* __restrict__ offsum) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double dg = 0.0, os = 0.0;
    for (int k = 0; k < nnz[i]; ++k) {
        const double v = values[off[i] + k];
        if (columns[off[i] + k] == i)
            dg += v;
        else
            os += fabs(v);
    }
    diag[i] = dg;
    offsum[i] = os;
    if (dg <= os) atomicMin(bad, i);
}

// Deterministic a . b (block partials + fixed-order second stage).
__global__ void __launch_bounds__(kBlock) k_dot(const double* __restrict__ a, const double* __restrict__ b, int n,
                                                double* __restrict__ partials) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    double v[1] = {i < n ? a[i] * b[i] : 0.0};
    mdkk::block_sum<1, kBlock>(v, partials + blockIdx.x);
}

// CG update (mdkk/qeq.py:197-207): alpha = rr / pAp; x += alpha p; r -= alpha Ap;
// partials of r . r.
__global__ void __launch_bounds__(kBlock) k_cg_update(int n, double* __restrict__ x, double* __restrict__ r,
                                                      const double* __restrict__ p, const double* __restrict__ ap,
                                                      const double* __restrict__ rr, const double* __restrict__ pap,
                                                      double* __restrict__ partials) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    const double alpha = rr[0] / pap[0];
    double v[1] = {0.0};
    if (i < n) {
        x[i] = x[i] + alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        v[0] = ri * ri;
    }
    mdkk::block_sum<1, kBlock>(v, partials + blockIdx.x);
}

// p = r + (rr_new / rr) p
__global__ void k_cg_direction(int n, const double* __restrict__ r, double* __restrict__ p,
                               const double* __restrict__ rr, const double* __restrict__ rr_new) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = r[i] + (rr_new[0] / rr[0]) * p[i];
}

}  // namespace

extern "C" {

int mdkk_qeq_offsets(mdkk_ctx* ctx, const int* counts, int n, int cap, long long* caps, long long* offsets,
                     void* stream) {
    if (!ctx || n < 0) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    k_qeq_caps<<<mdkk::grid_for(n + 1, kBlock), kBlock, 0, s>>>(counts, n, cap, caps);
    MDKK_CHECK_LAUNCH("k_qeq_caps");
    return mdkk::exclusive_scan_i64(ctx, caps, offsets, (long long)n + 1, s);
}

int mdkk_qeq_build(const double* x, int n_local, const int* table, const int* counts, int cap, const int* oidx,
                   const long long* offsets, double eta, double gamma, double cutoff, double* values, int* columns,
                   int* row_nnz, void* stream) {
    if (n_local < 0 || cap < 1 || gamma <= 0.0) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    k_qeq_build<<<mdkk::grid_for(n_local, 128), 128, 0, mdkk::as_stream(stream)>>>(
        x, n_local, table, counts, cap, oidx, offsets, eta, pow(gamma, -3.0), cutoff * cutoff, values, columns,
        row_nnz);
    MDKK_CHECK_LAUNCH("k_qeq_build");
    return MDKK_OK;
}

int mdkk_qeq_spmv(mdkk_ctx* ctx, const long long* offsets, const double* values, const int* columns,
                  const int* row_nnz, int n, const double* x1, const double* x2, double* y1, double* y2,
                  double* dots, void* stream) {
    if (!ctx || n < 0 || !x1 || !y1 || (x2 && !y2)) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    if (n == 0) {
        if (dots) cudaMemsetAsync(dots, 0, 2 * sizeof(double), s);
        return MDKK_OK;
    }
    const int nb = mdkk::grid_for((long long)n * kRowLanes, kBlock);
    double* partials = nullptr;
    if (dots) {
        partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * 2 * (size_t)nb));
        if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    }
    if (x2)
        k_qeq_spmv<2><<<nb, kBlock, 0, s>>>(offsets, values, columns, row_nnz, n, x1, x2, y1, y2, partials);
    else
        k_qeq_spmv<1><<<nb, kBlock, 0, s>>>(offsets, values, columns, row_nnz, n, x1, nullptr, y1, nullptr, partials);
    MDKK_CHECK_LAUNCH("k_qeq_spmv");
    if (dots) {
        mdkk::reduce_partials(partials, nb, 2, dots, s);
        MDKK_CHECK_LAUNCH("k_reduce_partials");
    }
    return MDKK_OK;
}

int mdkk_qeq_gershgorin(const long long* offsets, const double* values, const int* columns, const int* row_nnz, int n,
                        int* bad_row, double* diag, double* offsum, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_qeq_gershgorin<<<mdkk::grid_for(n, kBlock), kBlock, 0, mdkk::as_stream(stream)>>>(offsets, values, columns,
                                                                                       row_nnz, n, bad_row, diag,
                                                                                       offsum);
    MDKK_CHECK_LAUNCH("k_qeq_gershgorin");
    return MDKK_OK;
}

int mdkk_dot(mdkk_ctx* ctx, const double* a, const double* b, int n, double* out, void* stream) {
    if (!ctx || n < 0) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    const int nb = mdkk::grid_for(n, kBlock);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    k_dot<<<nb, kBlock, 0, s>>>(a, b, n, partials);
    MDKK_CHECK_LAUNCH("k_dot");
    mdkk::reduce_partials(partials, nb, 1, out, s);
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}

int mdkk_cg_update(mdkk_ctx* ctx, int n, double* x, double* r, const double* p, const double* ap, const double* rr,
                   const double* pap, double* rr_new, void* stream) {
    if (!ctx || n < 0) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    const int nb = mdkk::grid_for(n, kBlock);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    k_cg_update<<<nb, kBlock, 0, s>>>(n, x, r, p, ap, rr, pap, partials);
    MDKK_CHECK_LAUNCH("k_cg_update");
    mdkk::reduce_partials(partials, nb, 1, rr_new, s);
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}

int mdkk_cg_direction(int n, const double* r, double* p, const double* rr, const double* rr_new, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_cg_direction<<<mdkk::grid_for(n, kBlock), kBlock, 0, mdkk::as_stream(stream)>>>(n, r, p, rr, rr_new);
    MDKK_CHECK_LAUNCH("k_cg_direction");
    return MDKK_OK;
}

}  // extern "C"
