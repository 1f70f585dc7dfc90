// SNAP descriptor pipeline in FP64 on sm_100a.
// Reference: mdkk/snap/compute.py (map :27-63, recursion :125-235,
// compute_ui :279-292, compute_yi :303-340, energy :354-387,
// compute_fused_deidrj :390-409) with mdkk's conventions: rfac0 = 0.99,
// rmin0 = 0, plain cosine switch, no self term, full (tj+1)^2 blocks and the
// full three-slot adjoint Y.
//
// Data: U, Y are complex128 [n_flat][n_atoms] (atom fastest — the reference's
// transposed layout "b"), double2 = (re, im).
//
// compute_ui / fused deidrj: one warp per atom, its neighbours processed one
// at a time; the warp computes each level of the Wigner-U recursion with the
// level's elements spread over lanes (element idx -> lane idx%32, slot idx/32)
// and the previous level in shared memory.  Each lane keeps its 14 slots of
// U_i (ui) or Y_i (deidrj) in registers, so the per-atom sums need no atomics.
// compute_yi: one thread per atom walking an output-sorted contribution list
// (uniform across the warp -> broadcast table reads, coalesced U reads).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

struct mdkk_snap {
    int twojmax = 0;
    int n_flat = 0;
    int n_contrib = 0;
    int* f_start = nullptr;     // [n_flat + 1]
    int4* contrib = nullptr;    // {g, h, conj, 0}
    double* coef = nullptr;     // [n_contrib]
};

namespace {

constexpr int kMaxTwoJ = 8;
constexpr int kLevelMax = (kMaxTwoJ + 1) * (kMaxTwoJ + 1);  // 81
constexpr int kSlots = 14;                                   // sum_tj ceil((tj+1)^2 / 32) for 2J = 8
constexpr int kWarps = 4;
constexpr double kPi = 3.141592653589793;

__host__ __device__ constexpr int level_size(int tj) { return (tj + 1) * (tj + 1); }
__host__ __device__ constexpr int level_slots(int tj) { return (level_size(tj) + 31) / 32; }
__host__ __device__ constexpr int block_offset(int tj) { return tj * (tj + 1) * (2 * tj + 1) / 6; }
__host__ __device__ constexpr int slot_base(int tj) {
    int s = 0;
    for (int t = 0; t < tj; ++t) s += level_slots(t);
    return s;
}

struct cplx {
    double re, im;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ cplx cconj(cplx a) { return {a.re, -a.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx cscale(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx cneg(cplx a) { return {-a.re, -a.im}; }

// Recursion weights of element (P, Q) of level tj (mdkk/snap/compute.py:130-147):
// w[0] = sqrt(PQ)/tj (a * prev[P-1][Q-1]), w[1] = sqrt(P(tj-Q))/tj (b * prev[P-1][Q]),
// w[2] = sqrt((tj-P)Q)/tj (-conj(b) * prev[P][Q-1]), w[3] = sqrt((tj-P)(tj-Q))/tj (conj(a) * prev[P][Q]).
__constant__ double c_w[block_offset(kMaxTwoJ + 1)][4];

struct PairGeo {
    cplx a, b;
    double fc, dfc, r;
    cplx da[3], db[3];
};

// a, b, f_c, f_c' (mdkk/snap/compute.py:27-45) and optionally d a / d dr, d b / d dr (:48-63).
template <bool GRAD>
__device__ __forceinline__ void pair_geometry(double dx, double dy, double dz, double r2, double rc, PairGeo& g) {
    const double r = sqrt(r2);
    const double ct = 0.99 * kPi / rc;
    const double z0 = r / tan(ct * r);
    const double r0 = sqrt(r * r + z0 * z0);
    g.r = r;
    g.a = {z0 / r0, -dz / r0};
    g.b = {dy / r0, -dx / r0};
    g.fc = 0.5 * (1.0 + cos(kPi * r / rc));
    g.dfc = -kPi / (2.0 * rc) * sin(kPi * r / rc);
    if (GRAD) {
        const double dz0_dr = z0 / r - ct * (r * r + z0 * z0) / r;
        const double d[3] = {dx, dy, dz};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double dz0 = dz0_dr * (d[k] / r);
            const double dr0 = (d[k] + z0 * dz0) / r0;
            // da = (dz0 + unit_z*(-i)) / r0 - a dr0 / r0
            g.da[k] = {dz0 / r0 - g.a.re * dr0 / r0, (k == 2 ? -1.0 / r0 : 0.0) - g.a.im * dr0 / r0};
            // db = unit_b / r0 - b dr0 / r0,  unit_b = (-i, 1, 0)
            g.db[k] = {(k == 1 ? 1.0 / r0 : 0.0) - g.b.re * dr0 / r0, (k == 0 ? -1.0 / r0 : 0.0) - g.b.im * dr0 / r0};
        }
    }
}

// One element of level tj from the previous level stored row-major (tj x tj) in `prev`.
__device__ __forceinline__ cplx level_elem(const cplx* prev, int tj, int P, int Q, const double* w, cplx a, cplx b) {
    cplx v = {0.0, 0.0};
    if (P >= 1 && Q >= 1) v = cadd(v, cscale(w[0], cmul(prev[(P - 1) * tj + (Q - 1)], a)));
    if (P >= 1 && Q <= tj - 1) v = cadd(v, cscale(w[1], cmul(prev[(P - 1) * tj + Q], b)));
    if (P <= tj - 1 && Q >= 1) v = cadd(v, cscale(w[2], cmul(prev[P * tj + (Q - 1)], cneg(cconj(b)))));
    if (P <= tj - 1 && Q <= tj - 1) v = cadd(v, cscale(w[3], cmul(prev[P * tj + Q], cconj(a))));
    return v;
}

// Product-rule companion (mdkk/snap/compute.py:150-162).
__device__ __forceinline__ cplx level_elem_d(const cplx* prev, const cplx* dprev, int tj, int P, int Q,
                                             const double* w, cplx a, cplx b, cplx da, cplx db) {
    cplx v = {0.0, 0.0};
    if (P >= 1 && Q >= 1) {
        const int k = (P - 1) * tj + (Q - 1);
        v = cadd(v, cscale(w[0], cadd(cmul(dprev[k], a), cmul(prev[k], da))));
    }
    if (P >= 1 && Q <= tj - 1) {
        const int k = (P - 1) * tj + Q;
        v = cadd(v, cscale(w[1], cadd(cmul(dprev[k], b), cmul(prev[k], db))));
    }
    if (P <= tj - 1 && Q >= 1) {
        const int k = P * tj + (Q - 1);
        v = cadd(v, cscale(w[2], cadd(cmul(dprev[k], cneg(cconj(b))), cmul(prev[k], cneg(cconj(db))))));
    }
    if (P <= tj - 1 && Q <= tj - 1) {
        const int k = P * tj + Q;
        v = cadd(v, cscale(w[3], cadd(cmul(dprev[k], cconj(a)), cmul(prev[k], cconj(da)))));
    }
    return v;
}

__device__ __forceinline__ bool neighbour(const double* x, const int* table, int cap, int i, int k, double4 xi,
                                          double rc2, int& j, double& dx, double& dy, double& dz, double& r2) {
    j = table[((long long)(i >> 5) * cap + k) * 32 + (i & 31)];
    const double4 xj = mdkk::ld4(x, j);
    dx = xj.x - xi.x;
    dy = xj.y - xi.y;
    dz = xj.z - xi.z;
    r2 = mdkk::r2_exact(dx, dy, dz);
    return r2 < rc2;  // mdkk/snap/compute.py:114-115 (strict)
}

// ---------------------------------------------------------------- compute_ui
template <int TWOJ>
__global__ void __launch_bounds__(kWarps * 32) k_snap_ui(const double* __restrict__ x, int n_local,
                                                         const int* __restrict__ table,
                                                         const int* __restrict__ counts, int cap, double rc,
                                                         double2* __restrict__ U, int* __restrict__ flags) {
    __shared__ cplx s_lvl[kWarps][2][kLevelMax];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i = blockIdx.x * kWarps + w;
    if (i >= n_local) return;
    cplx acc[kSlots];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) acc[s] = {0.0, 0.0};
    const double4 xi = mdkk::ld4(x, i);
    const int n = min(counts[i], cap);
    const double rc2 = rc * rc;
    bool bad = false;
    for (int k = 0; k < n; ++k) {
        int j;
        double dx, dy, dz, r2;
        if (!neighbour(x, table, cap, i, k, xi, rc2, j, dx, dy, dz, r2)) continue;
        bad |= !(r2 > 0.0);
        PairGeo g;
        pair_geometry<false>(dx, dy, dz, r2, rc, g);
        if (lane == 0) {
            s_lvl[w][0][0] = {1.0, 0.0};
            acc[0].re += g.fc;
        }
        __syncwarp();
#pragma unroll
        for (int tj = 1; tj <= TWOJ; ++tj) {
            const cplx* prev = s_lvl[w][(tj - 1) & 1];
            cplx* cur = s_lvl[w][tj & 1];
#pragma unroll
            for (int s = 0; s < level_slots(tj); ++s) {
                const int idx = lane + 32 * s;
                if (idx < level_size(tj)) {
                    const int P = idx / (tj + 1), Q = idx % (tj + 1);
                    const cplx v = level_elem(prev, tj, P, Q, c_w[block_offset(tj) + idx], g.a, g.b);
                    cur[idx] = v;
                    acc[slot_base(tj) + s] = cadd(acc[slot_base(tj) + s], cscale(g.fc, v));
                }
            }
            __syncwarp();
        }
    }
    if (bad && lane == 0) atomicOr(flags, MDKK_FLAG_COINCIDENT);
#pragma unroll
    for (int tj = 0; tj <= TWOJ; ++tj)
#pragma unroll
        for (int s = 0; s < level_slots(tj); ++s) {
            const int idx = lane + 32 * s;
            if (idx < level_size(tj))
                U[(long long)(block_offset(tj) + idx) * n_local + i] =
                    make_double2(acc[slot_base(tj) + s].re, acc[slot_base(tj) + s].im);
        }
}

// ---------------------------------------------------------------- compute_yi
// Y[f] = sum_k coef_k * op(U[g_k]) * U[h_k]  (op = conj for slot-1/2 terms);
// e_atom = Re sum_f Y[f] conj(U[f]) / 3 (energy_from_y, mdkk/snap/compute.py:376-387).
__global__ void __launch_bounds__(128) k_snap_yi(const double2* __restrict__ U, int n, int n_flat,
                                                 const int* __restrict__ f_start, const int4* __restrict__ contrib,
                                                 const double* __restrict__ coef, double2* __restrict__ Y,
                                                 double* __restrict__ partials) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double e[1] = {0.0};
    if (i < n) {
        for (int f = 0; f < n_flat; ++f) {
            double are = 0.0, aim = 0.0;
            const int k1 = __ldg(f_start + f + 1);
            for (int k = __ldg(f_start + f); k < k1; ++k) {
                const int4 t = __ldg(contrib + k);
                const double c = __ldg(coef + k);
                const double2 ug = U[(long long)t.x * n + i];
                const double2 uh = U[(long long)t.y * n + i];
                const double gi = t.z ? -ug.y : ug.y;
                // c * (g * h)
                are += c * (ug.x * uh.x - gi * uh.y);
                aim += c * (ug.x * uh.y + gi * uh.x);
            }
            Y[(long long)f * n + i] = make_double2(are, aim);
            const double2 uf = U[(long long)f * n + i];
            e[0] += are * uf.x + aim * uf.y;  // Re(Y conj(U))
        }
        e[0] /= 3.0;
    }
    mdkk::block_sum<1, 128>(e, partials + blockIdx.x);
}

// ------------------------------------------------------- compute_fused_deidrj
template <int TWOJ>
__global__ void __launch_bounds__(kWarps * 32) k_snap_deidrj(const double* __restrict__ x, int n_local,
                                                             const int* __restrict__ table,
                                                             const int* __restrict__ counts, int cap, double rc,
                                                             const double2* __restrict__ Y,
                                                             double* __restrict__ f) {
    __shared__ cplx s_u[kWarps][2][kLevelMax];
    __shared__ cplx s_du[kWarps][2][3][kLevelMax];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i = blockIdx.x * kWarps + w;
    if (i >= n_local) return;
    cplx y[kSlots];
#pragma unroll
    for (int tj = 0; tj <= TWOJ; ++tj)
#pragma unroll
        for (int s = 0; s < level_slots(tj); ++s) {
            const int idx = lane + 32 * s;
            y[slot_base(tj) + s] = {0.0, 0.0};
            if (idx < level_size(tj)) {
                const double2 v = Y[(long long)(block_offset(tj) + idx) * n_local + i];
                y[slot_base(tj) + s] = {v.x, v.y};
            }
        }
    const double4 xi = mdkk::ld4(x, i);
    const int n = min(counts[i], cap);
    const double rc2 = rc * rc;
    double fi[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < n; ++k) {
        int j;
        double dx, dy, dz, r2;
        if (!neighbour(x, table, cap, i, k, xi, rc2, j, dx, dy, dz, r2)) continue;
        PairGeo g;
        pair_geometry<true>(dx, dy, dz, r2, rc, g);
        const double rh[3] = {dx / g.r, dy / g.r, dz / g.r};
        double t[3] = {0.0, 0.0, 0.0};
        if (lane == 0) {
            s_u[w][0][0] = {1.0, 0.0};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                s_du[w][0][d][0] = {0.0, 0.0};
                // level 0: wdu = dfc * rhat * 1 -> Re(Y0 * conj(.))
                t[d] += y[0].re * g.dfc * rh[d];
            }
        }
        __syncwarp();
#pragma unroll
        for (int tj = 1; tj <= TWOJ; ++tj) {
            const int pb = (tj - 1) & 1, cb = tj & 1;
#pragma unroll
            for (int s = 0; s < level_slots(tj); ++s) {
                const int idx = lane + 32 * s;
                if (idx < level_size(tj)) {
                    const int P = idx / (tj + 1), Q = idx % (tj + 1);
                    const double* wt = c_w[block_offset(tj) + idx];
                    const cplx u = level_elem(s_u[w][pb], tj, P, Q, wt, g.a, g.b);
                    s_u[w][cb][idx] = u;
                    const cplx yv = y[slot_base(tj) + s];
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const cplx du =
                            level_elem_d(s_u[w][pb], s_du[w][pb][d], tj, P, Q, wt, g.a, g.b, g.da[d], g.db[d]);
                        s_du[w][cb][d][idx] = du;
                        // wdu = fc du + dfc rhat u ; t += Re(Y conj(wdu))
                        const double wre = g.fc * du.re + g.dfc * rh[d] * u.re;
                        const double wim = g.fc * du.im + g.dfc * rh[d] * u.im;
                        t[d] += yv.re * wre + yv.im * wim;
                    }
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) t[d] = mdkk::warp_sum(t[d]);
        if (lane == 0) {
            fi[0] += t[0];
            fi[1] += t[1];
            fi[2] += t[2];
            double* fj = f + 4LL * j;
            atomicAdd(fj + 0, -t[0]);
            atomicAdd(fj + 1, -t[1]);
            atomicAdd(fj + 2, -t[2]);
        }
    }
    if (lane == 0) {
        double* p = f + 4LL * i;
        atomicAdd(p + 0, fi[0]);
        atomicAdd(p + 1, fi[1]);
        atomicAdd(p + 2, fi[2]);
    }
}

void upload_weights() {
    static bool done = false;
    if (done) return;
    double h[block_offset(kMaxTwoJ + 1)][4] = {};
    for (int tj = 1; tj <= kMaxTwoJ; ++tj)
        for (int P = 0; P <= tj; ++P)
            for (int Q = 0; Q <= tj; ++Q) {
                double* wv = h[block_offset(tj) + P * (tj + 1) + Q];
                wv[0] = std::sqrt((double)(P * Q)) / tj;
                wv[1] = std::sqrt((double)(P * (tj - Q))) / tj;
                wv[2] = std::sqrt((double)((tj - P) * Q)) / tj;
                wv[3] = std::sqrt((double)((tj - P) * (tj - Q))) / tj;
            }
    cudaMemcpyToSymbol(c_w, h, sizeof(h));
    done = true;
}

// Launch a kernel template for the runtime 2J (0..8).
#define MDKK_SNAP_DISPATCH(TWOJ_RT, KERNEL, GRID, BLOCK, STREAM, ...)                     \
    switch (TWOJ_RT) {                                                                  \
        case 0: KERNEL<0><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        case 1: KERNEL<1><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        case 2: KERNEL<2><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        case 3: KERNEL<3><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        case 4: KERNEL<4><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        case 5: KERNEL<5><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        case 6: KERNEL<6><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        case 7: KERNEL<7><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
        default: KERNEL<8><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;             \
    }

}  // namespace

extern "C" {

int mdkk_snap_create(mdkk_ctx* ctx, int twojmax, int n_contrib, const int* f_start_host, const int* g_host,
                     const int* h_host, const int* conj_host, const double* coef_host, mdkk_snap** out_host) {
    if (!ctx || !out_host || twojmax < 0 || twojmax > kMaxTwoJ || n_contrib < 0) {
        mdkk::set_error("mdkk_snap_create: 2J must be in [0, 8]");
        return MDKK_E_ARG;
    }
    auto* s = new mdkk_snap();
    s->twojmax = twojmax;
    s->n_flat = block_offset(twojmax + 1);
    s->n_contrib = n_contrib;
    std::vector<int4> c(std::max(n_contrib, 1));
    for (int k = 0; k < n_contrib; ++k) c[k] = make_int4(g_host[k], h_host[k], conj_host[k], 0);
    cudaError_t e = cudaMalloc(&s->f_start, sizeof(int) * (s->n_flat + 1));
    if (e == cudaSuccess) e = cudaMalloc(&s->contrib, sizeof(int4) * c.size());
    if (e == cudaSuccess) e = cudaMalloc(&s->coef, sizeof(double) * c.size());
    if (e == cudaSuccess) e = cudaMemcpy(s->f_start, f_start_host, sizeof(int) * (s->n_flat + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && n_contrib)
        e = cudaMemcpy(s->contrib, c.data(), sizeof(int4) * n_contrib, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && n_contrib) e = cudaMemcpy(s->coef, coef_host, sizeof(double) * n_contrib, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(s->f_start);
        cudaFree(s->contrib);
        cudaFree(s->coef);
        delete s;
        return mdkk::cuda_fail(e, "mdkk_snap_create");
    }
    upload_weights();
    *out_host = s;
    return MDKK_OK;
}

int mdkk_snap_destroy(mdkk_snap* s) {
    if (!s) return MDKK_OK;
    cudaFree(s->f_start);
    cudaFree(s->contrib);
    cudaFree(s->coef);
    delete s;
    return MDKK_OK;
}

int mdkk_snap_ui(mdkk_snap* s, const double* x, int n_local, const int* table, const int* counts, int cap, double rc,
                 double* U, int* flags, void* stream) {
    if (!s || n_local < 0 || cap < 1) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    upload_weights();
    const int nb = (n_local + kWarps - 1) / kWarps;
    MDKK_SNAP_DISPATCH(s->twojmax, k_snap_ui, nb, kWarps * 32, mdkk::as_stream(stream), x, n_local, table, counts,
                       cap, rc, reinterpret_cast<double2*>(U), flags);
    MDKK_CHECK_LAUNCH("k_snap_ui");
    return MDKK_OK;
}

int mdkk_snap_yi(mdkk_ctx* ctx, mdkk_snap* s, const double* U, int n_local, double* Y, double* energy, void* stream) {
    if (!ctx || !s || n_local < 0) return MDKK_E_ARG;
    cudaStream_t st = mdkk::as_stream(stream);
    if (n_local == 0) {
        cudaMemsetAsync(energy, 0, sizeof(double), st);
        return MDKK_OK;
    }
    const int nb = mdkk::grid_for(n_local, 128);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    k_snap_yi<<<nb, 128, 0, st>>>(reinterpret_cast<const double2*>(U), n_local, s->n_flat, s->f_start, s->contrib,
                                  s->coef, reinterpret_cast<double2*>(Y), partials);
    MDKK_CHECK_LAUNCH("k_snap_yi");
    mdkk::reduce_partials(partials, nb, 1, energy, st);
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}

int mdkk_snap_deidrj(mdkk_snap* s, const double* x, int n_local, const int* table, const int* counts, int cap,
                     double rc, const double* Y, double* f, void* stream) {
    if (!s || n_local < 0 || cap < 1) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    upload_weights();
    const int nb = (n_local + kWarps - 1) / kWarps;
    MDKK_SNAP_DISPATCH(s->twojmax, k_snap_deidrj, nb, kWarps * 32, mdkk::as_stream(stream), x, n_local, table,
                       counts, cap, rc, reinterpret_cast<const double2*>(Y), f);
    MDKK_CHECK_LAUNCH("k_snap_deidrj");
    return MDKK_OK;
}

}  // extern "C"
