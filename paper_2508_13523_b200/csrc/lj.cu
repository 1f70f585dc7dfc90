// Truncated 12-6 Lennard-Jones force / energy / virial over a cluster
// neighbour list.  Reference: mdkk/pair_lj.py:81-91 (kernel) and :114-179
// (engine: weights, partner writes, 6-virial).
//
// One warp per 32-atom cluster.  The cluster's union of candidate partners is
// staged once in shared memory (SoA doubles, coalesced row gathers) and every
// listed pair then reads x_j from shared memory instead of L1/L2; the table is
// uint16 local indices, 8 per 16-byte lane load.
//
// full          : owner writes f_i (no atomics); energy/virial weight 1/2 per entry
// half, newton  : f_i in registers, f_j via FP64 RED atomics; ghosts folded by reverse comm
// half, !newton : f_j written only for local j; ghost entries weight 1/2
#include "cluster.cuh"

namespace {

constexpr int kWarps = 4;

template <int STYLE, bool NEWTON, bool VIR>
__global__ void __launch_bounds__(kWarps * 32) k_lj(
    const double* __restrict__ x, int n_local, const int* __restrict__ uni, int ucap,
    const int* __restrict__ ucount, const uint16_t* __restrict__ table, const int* __restrict__ counts, int cap,
    int S, double eps4, double eps24, double sig2, double rc2, double* __restrict__ f,
    double* __restrict__ partials, int* __restrict__ flags) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x * kWarps + w;
    const int ncl = (n_local + 31) >> 5;
    double* sx = smem + (size_t)w * S * 3;
    double* sy = sx + S;
    double* sz = sy + S;
    int* su = reinterpret_cast<int*>(smem + (size_t)kWarps * S * 3) + (size_t)w * S;
    const int* ug = uni + (long long)c * ucap;

    const int m = c < ncl ? ucount[c] : 0;
    const int ms = min(m, S);
    for (int u = lane; u < ms; u += 32) {
        const int j = ug[u];
        const double4 p = mdkk::ld4(x, j);
        sx[u] = p.x;
        sy[u] = p.y;
        sz[u] = p.z;
        if (STYLE == 1) su[u] = j;
    }
    __syncwarp();

    double acc[7] = {0, 0, 0, 0, 0, 0, 0};  // E, Wxx, Wyy, Wzz, Wxy, Wxz, Wyz
    const int i = c * 32 + lane;
    if (c < ncl && i < n_local) {
        const double4 xi = mdkk::ld4(x, i);
        const int n = min(counts[i], cap);
        const int capb = cap >> 3;
        double fx = 0.0, fy = 0.0, fz = 0.0;
        bool bad = false;
        const uint4* tp = reinterpret_cast<const uint4*>(table) + ((long long)c * capb) * 32 + lane;
        uint4 nxt = n > 0 ? __ldg(tp) : make_uint4(0, 0, 0, 0);
        for (int kb = 0; kb * 8 < n; ++kb) {
            const uint4 pk = nxt;
            if ((kb + 1) * 8 < n) nxt = __ldg(tp + (long long)(kb + 1) * 32);
            const unsigned words[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (kb * 8 + e < n) {
                    const int u = (words[e >> 1] >> ((e & 1) * 16)) & 0xffff;
                    double px, py, pz;
                    int j = 0;
                    if (u < S) {
                        px = sx[u];
                        py = sy[u];
                        pz = sz[u];
                        if (STYLE == 1) j = su[u];
                    } else {
                        j = ug[u];
                        const double4 p = mdkk::ld4(x, j);
                        px = p.x;
                        py = p.y;
                        pz = p.z;
                    }
                    const double dx = px - xi.x, dy = py - xi.y, dz = pz - xi.z;
                    const double r2 = mdkk::r2_exact(dx, dy, dz);
                    if (r2 < rc2) {
                        bad |= !(r2 > 0.0);
                        const double inv = 1.0 / r2;
                        const double s2 = sig2 * inv;
                        const double s6 = s2 * s2 * s2;
                        const double s12 = s6 * s6;
                        const double fp = eps24 * (2.0 * s12 - s6) * inv;
                        const bool wj = (STYLE == 1) && (NEWTON || j < n_local);
                        const double wgt = (STYLE == 0) ? 0.5 : ((NEWTON || j < n_local) ? 1.0 : 0.5);
                        const double gx = fp * dx, gy = fp * dy, gz = fp * dz;
                        fx -= gx;
                        fy -= gy;
                        fz -= gz;
                        if (wj) {
                            double* fj = f + 4LL * j;
                            atomicAdd(fj + 0, gx);
                            atomicAdd(fj + 1, gy);
                            atomicAdd(fj + 2, gz);
                        }
                        acc[0] += wgt * (eps4 * (s12 - s6));
                        if (VIR) {
                            const double wf = wgt * fp;
                            acc[1] += wf * (dx * dx);
                            acc[2] += wf * (dy * dy);
                            acc[3] += wf * (dz * dz);
                            acc[4] += wf * (dx * dy);
                            acc[5] += wf * (dx * dz);
                            acc[6] += wf * (dy * dz);
                        }
                    }
                }
            }
        }
        if (STYLE == 0) {
            mdkk::st4(f, i, make_double4(fx, fy, fz, 0.0));
        } else {
            double* fi = f + 4LL * i;
            atomicAdd(fi + 0, fx);
            atomicAdd(fi + 1, fy);
            atomicAdd(fi + 2, fz);
        }
        if (bad) atomicOr(flags, MDKK_FLAG_COINCIDENT);
    }
    if (VIR) {
        mdkk::block_sum<7, kWarps * 32>(acc, partials + 7LL * blockIdx.x);
    } else {
        double e1[1] = {acc[0]};
        mdkk::block_sum<1, kWarps * 32>(e1, partials + blockIdx.x);
    }
}

}  // namespace

extern "C" int mdkk_lj_force(mdkk_ctx* ctx, const double* x, int n_local, const int* uni, int ucap,
                             const int* ucount, const uint16_t* table, const int* counts, int cap, int stage,
                             int style, int newton, int virial, double epsilon, double sigma, double rc, double* f,
                             double* ev, int* flags, void* stream) {
    if (!ctx || n_local < 0 || cap < 8 || (cap & 7) || stage < 32 || (style != 0 && style != 1)) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    if (n_local == 0) {
        cudaMemsetAsync(ev, 0, 7 * sizeof(double), s);
        return MDKK_OK;
    }
    const int ncl = (n_local + 31) / 32;
    const int nb = (ncl + kWarps - 1) / kWarps;
    const int K = virial ? 7 : 1;
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * 7 * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    const double e4 = 4.0 * epsilon, e24 = 24.0 * epsilon, s2 = sigma * sigma, rc2 = rc * rc;
    const size_t sm = (size_t)kWarps * stage * (3 * sizeof(double) + (style == 1 ? sizeof(int) : 0)) +
                      (style == 1 ? 0 : (size_t)kWarps * stage * sizeof(int));
#define MDKK_LJ(ST, NW, VR)                                                                                   \
    do {                                                                                                      \
        auto kern = k_lj<ST, NW, VR>;                                                                         \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                     \
        kern<<<nb, kWarps * 32, sm, s>>>(x, n_local, uni, ucap, ucount, table, counts, cap, stage, e4, e24, s2, \
                                         rc2, f, partials, flags);                                            \
    } while (0)
    if (style == 0) {
        if (virial) MDKK_LJ(0, false, true); else MDKK_LJ(0, false, false);
    } else if (newton) {
        if (virial) MDKK_LJ(1, true, true); else MDKK_LJ(1, true, false);
    } else {
        if (virial) MDKK_LJ(1, false, true); else MDKK_LJ(1, false, false);
    }
#undef MDKK_LJ
    MDKK_CHECK_LAUNCH("k_lj");
    if (!virial) cudaMemsetAsync(ev, 0, 7 * sizeof(double), s);
    mdkk::reduce_partials(partials, nb, K, ev, s);
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}
