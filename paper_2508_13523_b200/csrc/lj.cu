// Truncated 12-6 Lennard-Jones force / energy / virial over a transposed
// neighbour table.  Reference: mdkk/pair_lj.py:81-91 (kernel) and :114-179
// (engine: weights, partner writes, 6-virial).
//
// One thread per owned atom (rows cell-sorted, so a warp's partners overlap
// and the 256-bit double4 gathers hit L1); the cluster-blocked table
// [ncl][cap][32] makes every per-k read one coalesced 128-byte line.
// full          : owner writes f_i (no atomics); energy/virial weight 1/2 per entry
// half, newton  : f_i in registers, f_j via FP64 RED atomics; ghosts folded by reverse comm
// half, !newton : f_j written only for local j; ghost entries weight 1/2
// VIR=false skips the six virial accumulators (the integrator never reads them).
#include "common.cuh"

namespace {

constexpr int kBlock = 128;

// Speculative launch gate: the step's skin test (mdkk/neighbor.py:73-74, the host's
// sqrt(maxdisp2) > skin/2 in the same FP64 operations) read on the device, so the
// force launch can be queued before the host has seen the rebuild decision.
// The count gate is the build's capacity check (max_count > cap: the table overflowed
// and the list is rebuilt with a grown cap before the relaunch).
struct Gate {
    const double* d2;
    double half_skin;
    const int* count;
    int count_limit;
};
__device__ __forceinline__ bool gated_off(const Gate& g) {
    return (g.d2 != nullptr && sqrt(*g.d2) > g.half_skin) || (g.count != nullptr && *g.count > g.count_limit);
}

// Velocity-Verlet fused into the full-list force epilogue (mdkk_lj_force_integrate):
// MODE 1 closes the step (v += h f); MODE 2 also opens the next one and drifts
// (v += h f; x_next = x + dt v) and takes the next skin-test maximum
// max |x_next - x_ref|^2 -- the same operations, in the same order, as
// k_verlet_second + k_verlet_first<false> (or k_verlet_first<true>), so the
// trajectory is bit-identical.  Positions are double-buffered: the kernel reads x
// (owned + ghost rows) and writes the owned rows of x_next.
// Pair coefficients in the r^-6 form: F/r = r^-6 (c1 r^-6 - c2) r^-2, E = r^-6 (c3 r^-6 - c4)
// with c1 = 48 eps sig^12, c2 = 24 eps sig^6, c3 = 4 eps sig^12, c4 = 4 eps sig^6 (the
// reference's 4 eps ((sig/r)^12 - (sig/r)^6), mdkk/pair_lj.py:81-91, in 26 instead of 35
// FP64 operations per pair); h3 / h4 = c3 / 2, c4 / 2 (the full list's pair weight).
struct LJc {
    double c1, c2, c3, c4, h3, h4;
};
__device__ __forceinline__ LJc lj_coeffs(double eps4, double eps24, double sig2) {
    const double s6 = sig2 * sig2 * sig2, s12 = s6 * s6;
    LJc c;
    c.c1 = 2.0 * eps24 * s12;
    c.c2 = eps24 * s6;
    c.c3 = eps4 * s12;
    c.c4 = eps4 * s6;
    c.h3 = 0.5 * c.c3;
    c.h4 = 0.5 * c.c4;
    return c;
}

//
// Halo overlap (one rank per GPU): `part` 1 runs only the clusters whose flag is 0
// (no partner can be a ghost from another rank: launched while the halo exchange is
// in flight), `part` 2 the flagged ones once it has landed (its block partials add to
// part 1's); part 0 = every cluster.  Each atom is computed in exactly one part.
struct Integ {
    double* v;
    const double* x_ref;
    double* x_next;
    double* d2_next;
    double dt;
    double h;
    const unsigned char* part_flags;   // per 32-row cluster (mdkk_cluster_flags), parts 1 / 2
    int part;
};

// Half-list partner-write deconfliction (compute_pair's `strategy`, the
// reference's ScatterAccumulator strategies, mdkk/memspace.py:165-254):
// SCAT 0 Atomic    -- FP64 RED straight into f (the default engine path);
// SCAT 1 Duplicate -- RED into staging copy (blockIdx % copies), combined afterwards
//                     in a fixed order by mdkk_scatter_combine;
// SCAT 2 Serial    -- no atomics: own rows stored, each partner contribution staged
//                     per table entry (double4 (g, 1) in the table's blocked layout)
//                     and applied in entry order by mdkk_scatter_ordered -- run-to-run
//                     deterministic.
struct Scat {
    double* stage;
    long long stride;
    int copies;
};

template <int STYLE, bool NEWTON, bool VIR, int MODE = 0, int SCAT = 0>
__global__ void __launch_bounds__(kBlock) k_lj(const double* __restrict__ x, int n_local,
                                               const int* __restrict__ table, const int* __restrict__ counts,
                                               int cap, double eps4, double eps24, double sig2, double rc2,
                                               double* __restrict__ f, double* __restrict__ partials,
                                               int* __restrict__ flags, Gate gate, Integ integ = Integ{},
                                               Scat scat = Scat{}) {
    static_assert(MODE == 0 || STYLE == 0, "integration needs the complete f_i: full lists only");
    static_assert(SCAT == 0 || STYLE == 1, "strategies apply to half lists (full lists write owner rows only)");
    if (gated_off(gate)) return;   // block-uniform: the step rebuilds and relaunches
    const LJc lj = lj_coeffs(eps4, eps24, sig2);
    const int i = blockIdx.x * kBlock + threadIdx.x;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};  // E, Wxx, Wyy, Wzz, Wxy, Wxz, Wyz
    double d2n = 0.0;
    bool mine = true;   // warp-uniform: this warp's cluster belongs to the launched part
    if (MODE > 0 && integ.part != 0 && i < n_local) mine = (integ.part_flags[i >> 5] != 0) == (integ.part == 2);
    if (i < n_local && mine) {
        const double4 xi = mdkk::ld4(x, i);
        const int n = min(counts[i], cap);
        double fx = 0.0, fy = 0.0, fz = 0.0;
        bool bad = false;
        const int* col = table + ((long long)(i >> 5) * cap) * 32 + (i & 31);
        double* fw = f;   // partner / own-row RED target
        if (SCAT == 1) fw = scat.stage + (long long)(blockIdx.x % scat.copies) * scat.stride;
        auto pair = [&](int j, const double4& xj, int kk) {
            const double dx = xj.x - xi.x, dy = xj.y - xi.y, dz = xj.z - xi.z;
            const double r2 = mdkk::r2_exact(dx, dy, dz);
            if (r2 < rc2) {
                bad |= !(r2 > 0.0);
                const double inv = mdkk::rcp_nr(r2);
                const double r6 = inv * inv * inv;
                const double fp = r6 * fma(lj.c1, r6, -lj.c2) * inv;
                const bool wj = (STYLE == 1) && (NEWTON || j < n_local);
                const double wgt = (STYLE == 0) ? 0.5 : ((NEWTON || j < n_local) ? 1.0 : 0.5);
                if (STYLE == 0) {
                    fx = fma(-fp, dx, fx);
                    fy = fma(-fp, dy, fy);
                    fz = fma(-fp, dz, fz);
                    acc[0] += r6 * fma(lj.h3, r6, -lj.h4);   // 0.5 * E_pair (the weight is exact)
                } else {
                    const double gx = fp * dx, gy = fp * dy, gz = fp * dz;
                    fx -= gx;
                    fy -= gy;
                    fz -= gz;
                    if (wj) {
                        if (SCAT == 2) {
                            mdkk::st4(scat.stage, ((long long)(i >> 5) * cap + kk) * 32 + (i & 31),
                                      make_double4(gx, gy, gz, 1.0));
                        } else {
                            double* fj = fw + 4LL * j;
                            atomicAdd(fj + 0, gx);
                            atomicAdd(fj + 1, gy);
                            atomicAdd(fj + 2, gz);
                        }
                    }
                    acc[0] += wgt * (r6 * fma(lj.c3, r6, -lj.c4));
                }
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
        };
        // Gathers in batches of kB with the next batch's indices already in
        // flight: kB independent x_j loads per wait (the loop is L2-latency
        // bound otherwise).  Pair order (k ascending) is unchanged.
        constexpr int kB = 4;
        int jn[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) jn[b] = b < n ? __ldg(col + (long long)b * 32) : i;
        int k = 0;
        for (; k + kB <= n; k += kB) {
            int jc[kB];
            double4 xc[kB];
#pragma unroll
            for (int b = 0; b < kB; ++b) jc[b] = jn[b];
#pragma unroll
            for (int b = 0; b < kB; ++b) xc[b] = mdkk::ld4(x, jc[b]);
#pragma unroll
            for (int b = 0; b < kB; ++b) jn[b] = (k + kB + b < n) ? __ldg(col + (long long)(k + kB + b) * 32) : i;
#pragma unroll
            for (int b = 0; b < kB; ++b) pair(jc[b], xc[b], k + b);
        }
#pragma unroll
        for (int b = 0; b < kB; ++b)
            if (k + b < n) pair(jn[b], mdkk::ld4(x, jn[b]), k + b);
        if (STYLE == 0) {
            mdkk::st4(f, i, make_double4(fx, fy, fz, 0.0));
            if (MODE > 0) {
                const double h = integ.h, dt = integ.dt;
                double4 vi = mdkk::ld4_nc(integ.v, i);
                vi.x += h * fx;   // closing half-kick of this step
                vi.y += h * fy;
                vi.z += h * fz;
                if (MODE == 2) {
                    vi.x += h * fx;   // opening half-kick of the next step
                    vi.y += h * fy;
                    vi.z += h * fz;
                    double4 xn = xi;
                    xn.x += dt * vi.x;
                    xn.y += dt * vi.y;
                    xn.z += dt * vi.z;
                    xn.w = 0.0;
                    mdkk::st4(integ.x_next, i, xn);
                    const double4 r = mdkk::ld4_nc(integ.x_ref, i);
                    d2n = mdkk::finite_or_inf(mdkk::r2_exact(xn.x - r.x, xn.y - r.y, xn.z - r.z));
                }
                mdkk::st4(integ.v, i, vi);
            }
        } else if (SCAT == 2) {
            mdkk::st4(f, i, make_double4(fx, fy, fz, 0.0));   // partners are applied afterwards
        } else {
            double* fi = fw + 4LL * i;
            atomicAdd(fi + 0, fx);
            atomicAdd(fi + 1, fy);
            atomicAdd(fi + 2, fz);
        }
        if (bad) atomicOr(flags, MDKK_FLAG_COINCIDENT);
    }
    if (MODE == 2) {
        d2n = mdkk::warp_max(d2n);
        if ((threadIdx.x & 31) == 0) mdkk::atomic_max_nonneg(integ.d2_next, d2n);
    }
    const bool add = MODE > 0 && integ.part == 2;
    if (VIR) {
        mdkk::block_sum<7, kBlock>(acc, partials + 7LL * blockIdx.x, add);
    } else {
        double e1[1] = {acc[0]};
        mdkk::block_sum<1, kBlock>(e1, partials + blockIdx.x, add);
    }
}

// Boundary flags of the 32-row clusters for the halo overlap: 1 when the cluster's
// bounding box comes within `halo` of a brick face in a dimension whose neighbour
// bricks are other ranks (dims_mask bit d) -- only such clusters can list ghosts that
// arrive by the exchange (mdkk/domain.py:246-293 selects ghosts within the halo of
// the faces).  With halo = list cutoff + skin/2 the flags hold from any positions
// between the build and the next rebuild (no atom has moved more than skin/2).
__global__ void k_cluster_flags(const double* __restrict__ x, int n_local, double lox, double loy, double loz,
                                double hix, double hiy, double hiz, double halo, int dims_mask,
                                unsigned char* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = i >> 5;
    if (c * 32 >= n_local) return;
    const double4 p = mdkk::ld4(x, i < n_local ? i : c * 32);
    const double bnx = mdkk::warp_min_d(p.x), bxx = mdkk::warp_max(p.x);
    const double bny = mdkk::warp_min_d(p.y), bxy = mdkk::warp_max(p.y);
    const double bnz = mdkk::warp_min_d(p.z), bxz = mdkk::warp_max(p.z);
    bool f = false;
    if (dims_mask & 1) f |= bnx - halo < lox || bxx + halo >= hix;
    if (dims_mask & 2) f |= bny - halo < loy || bxy + halo >= hiy;
    if (dims_mask & 4) f |= bnz - halo < loz || bxz + halo >= hiz;
    if ((threadIdx.x & 31) == 0) flags[c] = f ? 1 : 0;
}

// Neighbour-parallel variant (mode "neighbor", the lj/cut/opt default,
// mdkk/pair_lj.py:118-143 and mdkk/driver/simulation.py:148-149): a team of T
// lanes per atom splits the atom's list (lane l takes entries l, l+T, ...)
// and the partial force / energy / virial are reduced with shuffles.  T times
// more threads for the same pairs: the small-N / low-occupancy regime.
template <int STYLE, bool NEWTON, bool VIR, int T>
__global__ void __launch_bounds__(kBlock) k_lj_team(const double* __restrict__ x, int n_local,
                                                    const int* __restrict__ table, const int* __restrict__ counts,
                                                    int cap, double eps4, double eps24, double sig2, double rc2,
                                                    double* __restrict__ f, double* __restrict__ partials,
                                                    int* __restrict__ flags, Gate gate) {
    if (gated_off(gate)) return;
    const LJc lj = lj_coeffs(eps4, eps24, sig2);
    const int t = blockIdx.x * kBlock + threadIdx.x;
    const int i = t / T, l = t % T;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    double fx = 0.0, fy = 0.0, fz = 0.0;
    const bool valid = i < n_local;
    bool bad = false;
    if (valid) {
        const double4 xi = mdkk::ld4(x, i);
        const int n = min(counts[i], cap);
        const int* col = table + ((long long)(i >> 5) * cap) * 32 + (i & 31);
        for (int k = l; k < n; k += T) {
            const int j = __ldg(col + (long long)k * 32);
            const double4 xj = mdkk::ld4(x, j);
            const double dx = xj.x - xi.x, dy = xj.y - xi.y, dz = xj.z - xi.z;
            const double r2 = mdkk::r2_exact(dx, dy, dz);
            if (r2 < rc2) {
                bad |= !(r2 > 0.0);
                const double inv = mdkk::rcp_nr(r2);
                const double r6 = inv * inv * inv;
                const double fp = r6 * fma(lj.c1, r6, -lj.c2) * inv;
                const bool wj = (STYLE == 1) && (NEWTON || j < n_local);
                const double wgt = (STYLE == 0) ? 0.5 : ((NEWTON || j < n_local) ? 1.0 : 0.5);
                if (STYLE == 0) {
                    fx = fma(-fp, dx, fx);
                    fy = fma(-fp, dy, fy);
                    fz = fma(-fp, dz, fz);
                    acc[0] += r6 * fma(lj.h3, r6, -lj.h4);
                } else {
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
                    acc[0] += wgt * (r6 * fma(lj.c3, r6, -lj.c4));
                }
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
#pragma unroll
    for (int o = T / 2; o > 0; o >>= 1) {   // team reduction of the partial force
        fx += __shfl_xor_sync(0xffffffffu, fx, o);
        fy += __shfl_xor_sync(0xffffffffu, fy, o);
        fz += __shfl_xor_sync(0xffffffffu, fz, o);
    }
    if (valid && l == 0) {
        if (STYLE == 0) {
            mdkk::st4(f, i, make_double4(fx, fy, fz, 0.0));
        } else {
            double* fi = f + 4LL * i;
            atomicAdd(fi + 0, fx);
            atomicAdd(fi + 1, fy);
            atomicAdd(fi + 2, fz);
        }
    }
    if (bad) atomicOr(flags, MDKK_FLAG_COINCIDENT);
    if (VIR) {
        mdkk::block_sum<7, kBlock>(acc, partials + 7LL * blockIdx.x);
    } else {
        double e1[1] = {acc[0]};
        mdkk::block_sum<1, kBlock>(e1, partials + blockIdx.x);
    }
}

}  // namespace

namespace {

int lj_team_launch(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts, int cap,
                   int style, int newton, int virial, double epsilon, double sigma, double rc, double* f, double* ev,
                   int* flags, const Gate& gate, cudaStream_t s) {
    if (!ctx || n_local < 0 || cap < 1 || (style != 0 && style != 1)) return MDKK_E_ARG;
    if (n_local == 0) {
        cudaMemsetAsync(ev, 0, 7 * sizeof(double), s);
        return MDKK_OK;
    }
    constexpr int T = 8;
    const int nb = mdkk::grid_for((long long)n_local * T, kBlock);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * 7 * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    const double e4 = 4.0 * epsilon, e24 = 24.0 * epsilon, s2 = sigma * sigma, rc2 = rc * rc;
#define MDKK_LJT(ST, NW, VR)                                                                                   \
    k_lj_team<ST, NW, VR, T><<<nb, kBlock, 0, s>>>(x, n_local, table, counts, cap, e4, e24, s2, rc2, f, partials, \
                                                    flags, gate)
    if (style == 0) {
        if (virial) MDKK_LJT(0, false, true); else MDKK_LJT(0, false, false);
    } else if (newton) {
        if (virial) MDKK_LJT(1, true, true); else MDKK_LJT(1, true, false);
    } else {
        if (virial) MDKK_LJT(1, false, true); else MDKK_LJT(1, false, false);
    }
#undef MDKK_LJT
    MDKK_CHECK_LAUNCH("k_lj_team");
    mdkk::reduce_partials(partials, nb, virial ? 7 : 1, ev, s, 7);   // clears the unused virial slots
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}

int lj_launch(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts, int cap, int style,
              int newton, int virial, double epsilon, double sigma, double rc, double* f, double* ev, int* flags,
              const Gate& gate, cudaStream_t s) {
    if (!ctx || n_local < 0 || cap < 1 || (style != 0 && style != 1)) return MDKK_E_ARG;
    if (n_local == 0) {
        cudaMemsetAsync(ev, 0, 7 * sizeof(double), s);
        return MDKK_OK;
    }
    const int nb = mdkk::grid_for(n_local, kBlock);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * 7 * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    const double e4 = 4.0 * epsilon, e24 = 24.0 * epsilon, s2 = sigma * sigma, rc2 = rc * rc;
#define MDKK_LJ(ST, NW, VR)                                                                                    \
    k_lj<ST, NW, VR><<<nb, kBlock, 0, s>>>(x, n_local, table, counts, cap, e4, e24, s2, rc2, f, partials, flags, \
                                           gate)
    if (style == 0) {
        if (virial) MDKK_LJ(0, false, true); else MDKK_LJ(0, false, false);
    } else if (newton) {
        if (virial) MDKK_LJ(1, true, true); else MDKK_LJ(1, true, false);
    } else {
        if (virial) MDKK_LJ(1, false, true); else MDKK_LJ(1, false, false);
    }
#undef MDKK_LJ
    MDKK_CHECK_LAUNCH("k_lj");
    mdkk::reduce_partials(partials, nb, virial ? 7 : 1, ev, s, 7);   // clears the unused virial slots
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}

}  // namespace

extern "C" int mdkk_lj_force_neighbor(mdkk_ctx* ctx, const double* x, int n_local, const int* table,
                                      const int* counts, int cap, int style, int newton, int virial, double epsilon,
                                      double sigma, double rc, double* f, double* ev, int* flags, void* stream) {
    return lj_team_launch(ctx, x, n_local, table, counts, cap, style, newton, virial, epsilon, sigma, rc, f, ev,
                          flags, Gate{nullptr, 0.0, nullptr, 0}, mdkk::as_stream(stream));
}

extern "C" int mdkk_lj_force(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts,
                             int cap, int style, int newton, int virial, double epsilon, double sigma, double rc,
                             double* f, double* ev, int* flags, void* stream) {
    return lj_launch(ctx, x, n_local, table, counts, cap, style, newton, virial, epsilon, sigma, rc, f, ev, flags,
                     Gate{nullptr, 0.0, nullptr, 0}, mdkk::as_stream(stream));
}

static int lj_integrate(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts, int cap,
                        int virial, double epsilon, double sigma, double rc, double* f, double* ev, int* flags,
                        const double* maxdisp2, double half_skin, const int* max_count, int count_limit, int mode,
                        double* v, const double* x_ref, double* x_next, double* d2_next, double dt, double h,
                        const unsigned char* part_flags, int part, const int* pack_idx, const int8_t* pack_code,
                        const double* pack_shifts, int pack_n, double* d2_zero, void* stream) {
    if (!ctx || n_local < 0 || cap < 1 || mode < 1 || mode > 2 || !v) return MDKK_E_ARG;
    if (part < 0 || part > 2 || (part && !part_flags)) return MDKK_E_ARG;
    if (mode == 2 && (!x_ref || !x_next || !d2_next || x_next == x)) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    if (n_local == 0) {
        if (part != 1) cudaMemsetAsync(ev, 0, 7 * sizeof(double), s);
        return MDKK_OK;
    }
    const int nb = mdkk::grid_for(n_local, kBlock);
    // part 1 leaves its block partials in the scratch arena for part 2 (same launch shape, same
    // stream, nothing in between uses the arena)
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * 7 * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    const double e4 = 4.0 * epsilon, e24 = 24.0 * epsilon, s2 = sigma * sigma, rc2 = rc * rc;
    const Gate gate{maxdisp2, half_skin, max_count, count_limit};
    const Integ integ{v, x_ref, x_next, d2_next, dt, h, part_flags, part};
#define MDKK_LJI(VR, MD)                                                                                        \
    k_lj<0, false, VR, MD><<<nb, kBlock, 0, s>>>(x, n_local, table, counts, cap, e4, e24, s2, rc2, f, partials,  \
                                                 flags, gate, integ)
    if (mode == 1) {
        if (virial) MDKK_LJI(true, 1); else MDKK_LJI(false, 1);
    } else {
        if (virial) MDKK_LJI(true, 2); else MDKK_LJI(false, 2);
    }
#undef MDKK_LJI
    MDKK_CHECK_LAUNCH("k_lj (integrate)");
    if (part == 1) return MDKK_OK;   // the reduction follows part 2
    if (pack_n > 0 && mode == 2) {   // + the next step's halo pack from x_next, same launch
        mdkk::reduce_partials_pack(partials, nb, virial ? 7 : 1, ev, 7, x_next, pack_idx, pack_code, pack_shifts,
                                   pack_n, x_next + 4LL * n_local, d2_zero, s);
        MDKK_CHECK_LAUNCH("k_reduce_pack");
        return MDKK_OK;
    }
    mdkk::reduce_partials(partials, nb, virial ? 7 : 1, ev, s, 7);   // clears the unused virial slots
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}

extern "C" int mdkk_lj_force_integrate(mdkk_ctx* ctx, const double* x, int n_local, const int* table,
                                       const int* counts, int cap, int virial, double epsilon, double sigma, double rc,
                                       double* f, double* ev, int* flags, const double* maxdisp2, double half_skin,
                                       const int* max_count, int count_limit, int mode, double* v,
                                       const double* x_ref, double* x_next, double* d2_next, double dt, double h,
                                       const unsigned char* part_flags, int part, void* stream) {
    return lj_integrate(ctx, x, n_local, table, counts, cap, virial, epsilon, sigma, rc, f, ev, flags, maxdisp2,
                        half_skin, max_count, count_limit, mode, v, x_ref, x_next, d2_next, dt, h, part_flags, part,
                        nullptr, nullptr, nullptr, 0, nullptr, stream);
}

extern "C" int mdkk_lj_force_integrate_pack(mdkk_ctx* ctx, const double* x, int n_local, const int* table,
                                            const int* counts, int cap, int virial, double epsilon, double sigma,
                                            double rc, double* f, double* ev, int* flags, const double* maxdisp2,
                                            double half_skin, const int* max_count, int count_limit, double* v,
                                            const double* x_ref, double* x_next, double* d2_next, double dt, double h,
                                            const int* pack_idx, const int8_t* pack_code, const double* pack_shifts,
                                            int pack_n, double* d2_zero, void* stream) {
    if (pack_n < 0 || (pack_n > 0 && (!pack_idx || !pack_code || !pack_shifts))) return MDKK_E_ARG;
    return lj_integrate(ctx, x, n_local, table, counts, cap, virial, epsilon, sigma, rc, f, ev, flags, maxdisp2,
                        half_skin, max_count, count_limit, 2, v, x_ref, x_next, d2_next, dt, h, nullptr, 0, pack_idx,
                        pack_code, pack_shifts, pack_n, d2_zero, stream);
}

extern "C" int mdkk_cluster_flags(const double* x, int n_local, const double* lo_host, const double* hi_host,
                                  double halo, int dims_mask, unsigned char* flags, void* stream) {
    if (n_local < 0 || !lo_host || !hi_host || !(halo >= 0.0)) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    const long long nthreads = ((long long)n_local + 31) / 32 * 32;
    k_cluster_flags<<<mdkk::grid_for(nthreads, 128), 128, 0, mdkk::as_stream(stream)>>>(
        x, n_local, lo_host[0], lo_host[1], lo_host[2], hi_host[0], hi_host[1], hi_host[2], halo, dims_mask, flags);
    MDKK_CHECK_LAUNCH("k_cluster_flags");
    return MDKK_OK;
}

extern "C" int mdkk_lj_force_gated(mdkk_ctx* ctx, const double* x, int n_local, const int* table,
                                   const int* counts, int cap, int style, int newton, int virial, int mode,
                                   double epsilon, double sigma, double rc, double* f, double* ev, int* flags,
                                   const double* maxdisp2, double half_skin, const int* max_count, int count_limit,
                                   void* stream) {
    if (mode != 0 && mode != 1) return MDKK_E_ARG;
    return (mode == 0 ? lj_launch : lj_team_launch)(ctx, x, n_local, table, counts, cap, style, newton, virial,
                                                    epsilon, sigma, rc, f, ev, flags,
                                                    Gate{maxdisp2, half_skin, max_count, count_limit},
                                                    mdkk::as_stream(stream));
}

// Half-list force with an explicit partner-write strategy (compute_pair's
// `strategy`; see Scat above).  strategy 1 = Duplicate (`stage` holds `copies`
// zeroed f-shaped copies `stride` doubles apart; the caller combines them),
// 2 = Serial (`stage` is a zeroed double4 per table entry, [ncl][cap][32]).
extern "C" int mdkk_lj_force_strategy(mdkk_ctx* ctx, const double* x, int n_local, const int* table,
                                      const int* counts, int cap, int newton, int virial, double epsilon,
                                      double sigma, double rc, double* f, double* ev, int* flags, int strategy,
                                      double* stage, long long stride, int copies, void* stream) {
    if (!ctx || n_local < 0 || cap < 1 || !stage || (strategy != 1 && strategy != 2)) return MDKK_E_ARG;
    if (strategy == 1 && (copies < 1 || stride < 4LL * n_local)) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    if (n_local == 0) {
        cudaMemsetAsync(ev, 0, 7 * sizeof(double), s);
        return MDKK_OK;
    }
    const int nb = mdkk::grid_for(n_local, kBlock);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * 7 * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    const double e4 = 4.0 * epsilon, e24 = 24.0 * epsilon, s2 = sigma * sigma, rc2 = rc * rc;
    const Gate gate{nullptr, 0.0, nullptr, 0};
    const Scat scat{stage, stride, copies};
#define MDKK_LJS(NW, VR, SC)                                                                                  \
    k_lj<1, NW, VR, 0, SC><<<nb, kBlock, 0, s>>>(x, n_local, table, counts, cap, e4, e24, s2, rc2, f, partials, \
                                                 flags, gate, Integ{}, scat)
    if (strategy == 1) {
        if (newton) {
            if (virial) MDKK_LJS(true, true, 1); else MDKK_LJS(true, false, 1);
        } else {
            if (virial) MDKK_LJS(false, true, 1); else MDKK_LJS(false, false, 1);
        }
    } else {
        if (newton) {
            if (virial) MDKK_LJS(true, true, 2); else MDKK_LJS(true, false, 2);
        } else {
            if (virial) MDKK_LJS(false, true, 2); else MDKK_LJS(false, false, 2);
        }
    }
#undef MDKK_LJS
    MDKK_CHECK_LAUNCH("k_lj (strategy)");
    mdkk::reduce_partials(partials, nb, virial ? 7 : 1, ev, s, 7);   // clears the unused virial slots
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}
