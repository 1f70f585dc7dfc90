// Velocity-Verlet half-kick + drift fused with the skin displacement test,
// and the closing half-kick fused with the kinetic-energy sum.
// Reference: mdkk/driver/simulation.py:407-450, mdkk/neighbor.py:66-74.
#include "common.cuh"

namespace {

constexpr int kBlock = 256;

// PENDING: the previous step's closing half-kick was deferred into this pass
// (same force, applied first with its own rounding: bit-identical to running
// k_verlet_second then this kernel).
template <bool PENDING>
__global__ void __launch_bounds__(kBlock) k_verlet_first(double* __restrict__ x, double* __restrict__ v,
                                                         const double* __restrict__ f,
                                                         const double* __restrict__ xr, int n, double dt,
                                                         double h, double* __restrict__ maxd2) {
    int i = blockIdx.x * kBlock + threadIdx.x;
    double d2 = 0.0;
    if (i < n) {
        double4 vi = mdkk::ld4_nc(v, i), fi = mdkk::ld4_nc(f, i), xi = mdkk::ld4_nc(x, i);
        if (PENDING) {
            vi.x += h * fi.x;
            vi.y += h * fi.y;
            vi.z += h * fi.z;
        }
        vi.x += h * fi.x;
        vi.y += h * fi.y;
        vi.z += h * fi.z;
        xi.x += dt * vi.x;
        xi.y += dt * vi.y;
        xi.z += dt * vi.z;
        mdkk::st4(v, i, vi);
        mdkk::st4(x, i, xi);
        double4 r = mdkk::ld4(xr, i);
        d2 = mdkk::finite_or_inf(mdkk::r2_exact(xi.x - r.x, xi.y - r.y, xi.z - r.z));
    }
    d2 = mdkk::warp_max(d2);
    if ((threadIdx.x & 31) == 0) mdkk::atomic_max_nonneg(maxd2, d2);
}

template <bool KE>
__global__ void __launch_bounds__(kBlock) k_verlet_second(double* __restrict__ v, const double* __restrict__ f,
                                                          int n, double h, double* __restrict__ partials) {
    int i = blockIdx.x * kBlock + threadIdx.x;
    double acc[1] = {0.0};
    if (i < n) {
        double4 vi = mdkk::ld4_nc(v, i), fi = mdkk::ld4_nc(f, i);
        vi.x += h * fi.x;
        vi.y += h * fi.y;
        vi.z += h * fi.z;
        mdkk::st4(v, i, vi);
        if (KE) acc[0] = vi.x * vi.x + vi.y * vi.y + vi.z * vi.z;
    }
    if (KE) mdkk::block_sum<1, kBlock>(acc, partials + blockIdx.x);
}

__global__ void __launch_bounds__(kBlock) k_v2(const double* __restrict__ v, int n, double* __restrict__ partials) {
    int i = blockIdx.x * kBlock + threadIdx.x;
    double acc[1] = {0.0};
    if (i < n) {
        double4 vi = mdkk::ld4_nc(v, i);
        acc[0] = vi.x * vi.x + vi.y * vi.y + vi.z * vi.z;
    }
    mdkk::block_sum<1, kBlock>(acc, partials + blockIdx.x);
}

__global__ void k_scale(double* p, double s) { *p *= s; }

}  // namespace

extern "C" {

int mdkk_verlet_first(mdkk_ctx*, double* x, double* v, const double* f, const double* x_ref, int n, double dt,
                      double h, double* maxdisp2, int pending_kick, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    cudaMemsetAsync(maxdisp2, 0, sizeof(double), s);
    if (n == 0) return MDKK_OK;
    if (pending_kick)
        k_verlet_first<true><<<mdkk::grid_for(n, kBlock), kBlock, 0, s>>>(x, v, f, x_ref, n, dt, h, maxdisp2);
    else
        k_verlet_first<false><<<mdkk::grid_for(n, kBlock), kBlock, 0, s>>>(x, v, f, x_ref, n, dt, h, maxdisp2);
    MDKK_CHECK_LAUNCH("k_verlet_first");
    return MDKK_OK;
}

int mdkk_verlet_second(mdkk_ctx* ctx, double* v, const double* f, int n, double h, double mass, double* ke,
                       void* stream) {
    if (n < 0 || !ctx) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    if (n == 0) {
        if (ke) cudaMemsetAsync(ke, 0, sizeof(double), s);
        return MDKK_OK;
    }
    int nb = mdkk::grid_for(n, kBlock);
    if (!ke) {
        k_verlet_second<false><<<nb, kBlock, 0, s>>>(v, f, n, h, nullptr);
        MDKK_CHECK_LAUNCH("k_verlet_second");
        return MDKK_OK;
    }
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    k_verlet_second<true><<<nb, kBlock, 0, s>>>(v, f, n, h, partials);
    MDKK_CHECK_LAUNCH("k_verlet_second");
    mdkk::reduce_partials(partials, nb, 1, ke, s);
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    k_scale<<<1, 1, 0, s>>>(ke, 0.5 * mass);
    MDKK_CHECK_LAUNCH("k_scale");
    return MDKK_OK;
}

int mdkk_kinetic(mdkk_ctx* ctx, const double* v, int n, double mass, double* ke, void* stream) {
    if (n < 0 || !ctx) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    if (n == 0) {
        cudaMemsetAsync(ke, 0, sizeof(double), s);
        return MDKK_OK;
    }
    int nb = mdkk::grid_for(n, kBlock);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    k_v2<<<nb, kBlock, 0, s>>>(v, n, partials);
    MDKK_CHECK_LAUNCH("k_v2");
    mdkk::reduce_partials(partials, nb, 1, ke, s);
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    k_scale<<<1, 1, 0, s>>>(ke, 0.5 * mass);
    MDKK_CHECK_LAUNCH("k_scale");
    return MDKK_OK;
}

}  // extern "C"
