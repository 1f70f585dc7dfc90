// SNAP API-parity stages around the fused engine path (FP64, sm_100a):
//   * the neighbour map (mdkk/snap/compute.py:66-119): in-range pairs of a
//     full list in (row, dz, dy, dx) order with a, b, f_c, f_c';
//   * the staged force path (compute_duidrj + compute_deidrj,
//     mdkk/snap/compute.py:412-436): d(f_c u)/d dr materialised per pair,
//     then contracted with Y;
//   * the descriptors (compute_bi_complex, mdkk/snap/compute.py:354-373):
//     B_t = sum_terms c U[iu1] U[iu2] conj(U[iz]) per atom and triple.
// The engine never calls these (its forces come from the fused reverse-mode
// kernel in snap.cu); they serve the reference's staged API and its tests.

#include "snap_common.cuh"

namespace {

// ------------------------------------------------------------ neighbour map
__global__ void k_snap_pair_count(const double* __restrict__ x, int n_local, const int* __restrict__ table,
                                  const int* __restrict__ counts, int cap, double rc2, int* __restrict__ npair,
                                  int* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    const double4 xi = mdkk::ld4(x, i);
    const int n = min(counts[i], cap);
    int c = 0;
    bool bad = false;
    for (int k = 0; k < n; ++k) {
        int j;
        double dx, dy, dz, r2;
        if (neighbour(x, table, cap, i, k, xi, rc2, j, dx, dy, dz, r2)) {
            ++c;
            bad |= !(r2 > 0.0);
        }
    }
    npair[i] = c;
    if (bad) atomicOr(flags, MDKK_FLAG_COINCIDENT);
}

__device__ __forceinline__ bool zyx_less(const double* a, const double* b) {
    if (a[2] != b[2]) return a[2] < b[2];
    if (a[1] != b[1]) return a[1] < b[1];
    return a[0] < b[0];
}

// One thread per row: its in-range pairs, insertion-sorted by (dz, dy, dx)
// (np.lexsort((dx, dy, dz, rows)), mdkk/snap/compute.py:78-80), then the
// hypersphere parameters (mdkk/snap/compute.py:27-45).
__global__ void k_snap_pair_fill(const double* __restrict__ x, int n_local, const int* __restrict__ table,
                                 const int* __restrict__ counts, int cap, double rc, const int* __restrict__ off,
                                 int* __restrict__ rows, int* __restrict__ cols, double* __restrict__ dr,
                                 double* __restrict__ rr, double2* __restrict__ a, double2* __restrict__ b,
                                 double* __restrict__ fc, double* __restrict__ dfc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    const double4 xi = mdkk::ld4(x, i);
    const int n = min(counts[i], cap);
    const int o = off[i];
    int c = 0;
    for (int k = 0; k < n; ++k) {
        int j;
        double d[3], r2;
        if (!neighbour(x, table, cap, i, k, xi, rc * rc, j, d[0], d[1], d[2], r2)) continue;
        // insertion into the sorted prefix [o, o + c)
        int m = c - 1;
        while (m >= 0 && zyx_less(d, dr + 3LL * (o + m))) {
            const long long s = o + m;
            cols[s + 1] = cols[s];
            dr[3 * (s + 1) + 0] = dr[3 * s + 0];
            dr[3 * (s + 1) + 1] = dr[3 * s + 1];
            dr[3 * (s + 1) + 2] = dr[3 * s + 2];
            --m;
        }
        const long long s = o + m + 1;
        cols[s] = j;
        dr[3 * s + 0] = d[0];
        dr[3 * s + 1] = d[1];
        dr[3 * s + 2] = d[2];
        ++c;
    }
    for (int q = 0; q < c; ++q) {
        const long long s = o + q;
        const double dx = dr[3 * s + 0], dy = dr[3 * s + 1], dz = dr[3 * s + 2];
        PairGeo g;
        double z0, r0;
        pair_geometry(dx, dy, dz, mdkk::r2_exact(dx, dy, dz), rc, g, z0, r0);
        rows[s] = i;
        rr[s] = g.r;
        a[s] = make_double2(g.a.re, g.a.im);
        b[s] = make_double2(g.b.re, g.b.im);
        fc[s] = g.fc;
        dfc[s] = g.dfc;
    }
}

// ------------------------------------------------------ staged derivatives
// wdu[p][d][f] = f_c du[f]/d dr_d + f_c' (dr_d / r) u[f] (mdkk/snap/compute.py:187-235,
// 412-422): forward-mode product rule on the two-term column recursion
// (snap_common.cuh rec2) over the column halves, mirrored with
// X[tj-P][tj-Q] = (-1)^(P+Q) conj(X[P][Q]) (real coordinates keep the relation).
// One warp per pair, levels ping-ponged in shared memory (column-major).
constexpr int kDW = 4;   // warps per CTA

template <int TWOJ>
__global__ void __launch_bounds__(kDW * 32) k_snap_duidrj(int n_pairs, const double* __restrict__ dr,
                                                          double rc, double2* __restrict__ wdu) {
    constexpr int NF = block_offset(TWOJ + 1);
    __shared__ RS rs;
    __shared__ cplx s_l[kDW][2][4][kLevelMax];   // [buffer][u, du_x, du_y, du_z][element]
    stage_rs(rs);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long p = (long long)blockIdx.x * kDW + w;
    if (p >= n_pairs) return;
    const double d[3] = {dr[3 * p + 0], dr[3 * p + 1], dr[3 * p + 2]};
    PairGeo g;
    double z0, r0;
    pair_geometry(d[0], d[1], d[2], mdkk::r2_exact(d[0], d[1], d[2]), rc, g, z0, r0);
    cplx da[3], db[3];
    pair_grads(d, g, rc, z0, r0, da, db);
    const cplx ab = cconj(g.a);
    double2* out = wdu + p * 3 * NF;
    if (lane == 0) {
        s_l[w][0][0][0] = {1.0, 0.0};
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            s_l[w][0][q + 1][0] = {0.0, 0.0};
            out[q * NF] = make_double2(g.dfc * (d[q] / g.r), 0.0);
        }
    }
    __syncwarp();
#pragma unroll
    for (int tj = 1; tj <= TWOJ; ++tj) {
        const int pb = (tj - 1) & 1, cb = tj & 1;
        for (int c = lane; c < half_size(tj); c += 32) {
            int P, Q;
            col_elem(tj, c, P, Q);
            const cplx* v = s_l[w][pb][0];
            cplx u = {0.0, 0.0}, du[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
            if (P < tj) {
                const double wa = rs.v[tj - P][tj - Q];
                const cplx v0 = v[Q * tj + P];
                u = cadd(u, cscale(wa, cmul(ab, v0)));
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    du[q] = cadd(du[q], cscale(wa, cadd(cmul(cconj(da[q]), v0), cmul(ab, s_l[w][pb][q + 1][Q * tj + P]))));
            }
            if (P >= 1) {
                const double wb = rs.v[P][tj - Q];
                const cplx v1 = v[Q * tj + P - 1];
                u = cadd(u, cscale(wb, cmul(g.b, v1)));
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    du[q] = cadd(du[q], cscale(wb, cadd(cmul(db[q], v1), cmul(g.b, s_l[w][pb][q + 1][Q * tj + P - 1]))));
            }
            store_mirrored(s_l[w][cb][0], tj, P, Q, u);
            const int e = block_offset(tj) + P * (tj + 1) + Q;
            const int em = block_offset(tj) + (tj - P) * (tj + 1) + (tj - Q);
            const double sg = ((P + Q) & 1) ? -1.0 : 1.0;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                store_mirrored(s_l[w][cb][q + 1], tj, P, Q, du[q]);
                const double rad = g.dfc * (d[q] / g.r);
                const cplx wv = {g.fc * du[q].re + rad * u.re, g.fc * du[q].im + rad * u.im};
                out[q * NF + e] = make_double2(wv.re, wv.im);
                if (em != e) out[q * NF + em] = make_double2(sg * wv.re, -sg * wv.im);
            }
        }
        __syncwarp();
    }
}

// t_d = Re sum_f Y[row][f] conj(wdu[p][d][f]); F[row] += t, F[col] -= t
// (mdkk/snap/compute.py:425-436).  One warp per pair, FP64 atomics.
__global__ void k_snap_deidrj_staged(int n_pairs, int nf, const int* __restrict__ rows, const int* __restrict__ cols,
                                     const double2* __restrict__ Y, const double2* __restrict__ wdu,
                                     double* __restrict__ f) {
    const int lane = threadIdx.x & 31;
    const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (p >= n_pairs) return;
    const int i = rows[p];
    const double2* y = Y + (long long)i * nf;
    const double2* w = wdu + p * 3 * nf;
    double t[3] = {0.0, 0.0, 0.0};
    for (int e = lane; e < nf; e += 32) {
        const double2 yv = y[e];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double2 wv = w[q * nf + e];
            t[q] += yv.x * wv.x + yv.y * wv.y;
        }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) t[q] = mdkk::warp_sum(t[q]);
    if (lane == 0) {
        const int j = cols[p];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            atomicAdd(f + 4LL * i + q, t[q]);
            atomicAdd(f + 4LL * j + q, -t[q]);
        }
    }
}

// Per-pair contraction only (no scatter): t[p][d] = Re sum_f Y[row][f] conj(wdu[p][d][f]).
// The caller applies F[row] += t, F[col] -= t with the ordered scatter
// (np.add.at / np.subtract.at order, mdkk/snap/compute.py:405-408): deterministic.
__global__ void k_snap_pair_dedr(int n_pairs, int nf, const int* __restrict__ rows, const double2* __restrict__ Y,
                                 const double2* __restrict__ wdu, double* __restrict__ t_out) {
    const int lane = threadIdx.x & 31;
    const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (p >= n_pairs) return;
    const double2* y = Y + (long long)rows[p] * nf;
    const double2* w = wdu + p * 3 * nf;
    double t[3] = {0.0, 0.0, 0.0};
    for (int e = lane; e < nf; e += 32) {
        const double2 yv = y[e];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double2 wv = w[q * nf + e];
            t[q] += yv.x * wv.x + yv.y * wv.y;
        }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) t[q] = mdkk::warp_sum(t[q]);
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) t_out[3 * p + q] = t[q];
    }
}

// ------------------------------------------------------------- descriptors
// B[i][t] = sum over the triple's terms of c * op(U[g]) * op(U[h]) * op(U[z]),
// U from the half set (mirrored operands conj'ed, signs in c; op_z is conj
// for an unmirrored z).  Atoms across lanes over a shared-memory U tile (the
// yi layout); each warp owns whole triples.
constexpr int kBW = 8;

template <int NF, int NH>
__global__ void __launch_bounds__(kBW * 32) k_snap_bi(const double2* __restrict__ U, int n,
                                                      const double* __restrict__ coef, const int* __restrict__ code,
                                                      const int* __restrict__ tri, const int* __restrict__ chunk,
                                                      int n_tri, double2* __restrict__ B, long long su, long long sf) {
    extern __shared__ double2 s_bu[];   // [NH][33]
    constexpr int S = 33;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a0 = blockIdx.x * 32;
    for (int t = threadIdx.x; t < 32 * NH; t += blockDim.x) {
        const int a = t / NH, e = t - a * NH;
        s_bu[e * S + a] = (a0 + a < n) ? U[(long long)(a0 + a) * su + c_hflat[e] * sf] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const bool valid = a0 + lane < n;
    double re = 0.0, im = 0.0;
    for (int k = chunk[w]; k < chunk[w + 1]; ++k) {
        const int cd = __ldg(code + k);
        const double c = __ldg(coef + k);
        double2 ug = s_bu[(cd & 255) * S + lane], uh = s_bu[((cd >> 8) & 255) * S + lane];
        double2 uz = s_bu[((cd >> 16) & 255) * S + lane];
        if (cd & (1 << 24)) ug.y = -ug.y;
        if (cd & (1 << 25)) uh.y = -uh.y;
        if (cd & (1 << 26)) uz.y = -uz.y;
        const double pr = ug.x * uh.x - ug.y * uh.y, pi = ug.x * uh.y + ug.y * uh.x;
        re += c * (pr * uz.x - pi * uz.y);
        im += c * (pr * uz.y + pi * uz.x);
        if (cd & (1 << 27)) {
            if (valid) B[(long long)(a0 + lane) * n_tri + __ldg(tri + k)] = make_double2(re, im);
            re = im = 0.0;
        }
    }
}


// ------------------------------------------------------------ pair levels
// pair_u_flat (mdkk/snap/compute.py:165-184): unweighted levels u_0..u_2J of
// arbitrary (a, b) by the reference's four-term recursion (:138-147), every
// (tj+1)^2 block in full (no mirror: (a, b) need not be unitary here).  One warp
// per pair, levels ping-ponged in shared memory; the terms are added in the
// reference's order with explicit roundings.
constexpr int kUW = 4;

__device__ __forceinline__ cplx cmul_rn(cplx x, cplx y) {
    return {__dsub_rn(__dmul_rn(x.re, y.re), __dmul_rn(x.im, y.im)),
            __dadd_rn(__dmul_rn(x.re, y.im), __dmul_rn(x.im, y.re))};
}
__device__ __forceinline__ cplx cacc_rn(cplx acc, double c, cplx v) {
    return {__dadd_rn(acc.re, __dmul_rn(c, v.re)), __dadd_rn(acc.im, __dmul_rn(c, v.im))};
}

__global__ void __launch_bounds__(kUW * 32) k_snap_pair_u(int n_pairs, int twojmax, const double2* __restrict__ a_in,
                                                          const double2* __restrict__ b_in, double2* __restrict__ out) {
    __shared__ cplx s_l[kUW][2][kLevelMax];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long p = (long long)blockIdx.x * kUW + w;
    if (p >= n_pairs) return;
    const int nf = block_offset(twojmax + 1);
    const cplx a = {a_in[p].x, a_in[p].y}, b = {b_in[p].x, b_in[p].y};
    const cplx ac = {a.re, -a.im}, nbc = {-b.re, b.im};
    double2* o = out + p * nf;
    if (lane == 0) {
        s_l[w][0][0] = {1.0, 0.0};
        o[0] = make_double2(1.0, 0.0);
    }
    __syncwarp();
    for (int tj = 1; tj <= twojmax; ++tj) {
        const cplx* v = s_l[w][(tj - 1) & 1];   // previous level, row-major tj x tj
        cplx* nw = s_l[w][tj & 1];
        const double itj = (double)tj;
        for (int e = lane; e < (tj + 1) * (tj + 1); e += 32) {
            const int P = e / (tj + 1), Q = e % (tj + 1);
            cplx acc = {0.0, 0.0};
            if (P >= 1 && Q >= 1) acc = cacc_rn(acc, sqrt((double)(P * Q)) / itj, cmul_rn(v[(P - 1) * tj + Q - 1], a));
            if (P >= 1 && Q < tj) acc = cacc_rn(acc, sqrt((double)(P * (tj - Q))) / itj, cmul_rn(v[(P - 1) * tj + Q], b));
            if (P < tj && Q >= 1) acc = cacc_rn(acc, sqrt((double)((tj - P) * Q)) / itj, cmul_rn(v[P * tj + Q - 1], nbc));
            if (P < tj && Q < tj) acc = cacc_rn(acc, sqrt((double)((tj - P) * (tj - Q))) / itj, cmul_rn(v[P * tj + Q], ac));
            nw[e] = acc;
            o[block_offset(tj) + e] = make_double2(acc.re, acc.im);
        }
        __syncwarp();
    }
}

// NeighborMap.deriv_params (mdkk/snap/compute.py:48-63,98-102): (da, db) per pair,
// [n][3] complex each, from the same device geometry the force kernels use.
__global__ void k_snap_pair_grads(int n_pairs, const double* __restrict__ dr, double rc, double2* __restrict__ da_out,
                                  double2* __restrict__ db_out) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_pairs) return;
    const double d[3] = {dr[3 * p + 0], dr[3 * p + 1], dr[3 * p + 2]};
    PairGeo g;
    double z0, r0;
    pair_geometry(d[0], d[1], d[2], mdkk::r2_exact(d[0], d[1], d[2]), rc, g, z0, r0);
    cplx da[3], db[3];
    pair_grads(d, g, rc, z0, r0, da, db);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        da_out[3 * p + q] = make_double2(da[q].re, da[q].im);
        db_out[3 * p + q] = make_double2(db[q].re, db[q].im);
    }
}

}  // namespace

extern "C" {

int mdkk_snap_pair_u(int n_pairs, int twojmax, const double* a, const double* b, double* out, void* stream) {
    if (n_pairs < 0 || twojmax < 0 || twojmax > kMaxTwoJ || (n_pairs && (!a || !b || !out))) return MDKK_E_ARG;
    if (n_pairs == 0) return MDKK_OK;
    k_snap_pair_u<<<(n_pairs + kUW - 1) / kUW, kUW * 32, 0, mdkk::as_stream(stream)>>>(
        n_pairs, twojmax, reinterpret_cast<const double2*>(a), reinterpret_cast<const double2*>(b),
        reinterpret_cast<double2*>(out));
    MDKK_CHECK_LAUNCH("k_snap_pair_u");
    return MDKK_OK;
}

int mdkk_snap_pair_grads(int n_pairs, const double* dr, double rc, double* da, double* db, void* stream) {
    if (n_pairs < 0 || (n_pairs && (!dr || !da || !db))) return MDKK_E_ARG;
    if (n_pairs == 0) return MDKK_OK;
    upload_weights();
    k_snap_pair_grads<<<mdkk::grid_for(n_pairs, 128), 128, 0, mdkk::as_stream(stream)>>>(
        n_pairs, dr, rc, reinterpret_cast<double2*>(da), reinterpret_cast<double2*>(db));
    MDKK_CHECK_LAUNCH("k_snap_pair_grads");
    return MDKK_OK;
}

int mdkk_snap_pair_count(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts, int cap,
                         double rc, int* npair, int* offsets, int* flags, void* stream) {
    if (!ctx || n_local < 0 || cap < 1) return MDKK_E_ARG;
    cudaStream_t st = mdkk::as_stream(stream);
    if (n_local > 0) {
        k_snap_pair_count<<<mdkk::grid_for(n_local, 128), 128, 0, st>>>(x, n_local, table, counts, cap, rc * rc,
                                                                         npair, flags);
        MDKK_CHECK_LAUNCH("k_snap_pair_count");
    }
    cudaMemsetAsync(npair + n_local, 0, sizeof(int), st);
    return mdkk::exclusive_scan_i32(ctx, npair, offsets, (long long)n_local + 1, st);
}

int mdkk_snap_pair_fill(const double* x, int n_local, const int* table, const int* counts, int cap, double rc,
                        const int* offsets, int* rows, int* cols, double* dr, double* r, double* a, double* b,
                        double* fc, double* dfc, void* stream) {
    if (n_local < 0 || cap < 1) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    upload_weights();
    k_snap_pair_fill<<<mdkk::grid_for(n_local, 128), 128, 0, mdkk::as_stream(stream)>>>(
        x, n_local, table, counts, cap, rc, offsets, rows, cols, dr, r, reinterpret_cast<double2*>(a),
        reinterpret_cast<double2*>(b), fc, dfc);
    MDKK_CHECK_LAUNCH("k_snap_pair_fill");
    return MDKK_OK;
}

int mdkk_snap_duidrj(mdkk_snap* s, int n_pairs, const double* dr, double rc, double* wdu, void* stream) {
    if (!s || n_pairs < 0) return MDKK_E_ARG;
    if (n_pairs == 0) return MDKK_OK;
    upload_weights();
    const int nb = (n_pairs + kDW - 1) / kDW;
    MDKK_SNAP_DISPATCH(s->twojmax, k_snap_duidrj, nb, kDW * 32, mdkk::as_stream(stream), n_pairs, dr, rc,
                       reinterpret_cast<double2*>(wdu));
    MDKK_CHECK_LAUNCH("k_snap_duidrj");
    return MDKK_OK;
}

int mdkk_snap_deidrj_staged(mdkk_snap* s, int n_pairs, const int* rows, const int* cols, const double* Y,
                            const double* wdu, double* f, void* stream) {
    if (!s || n_pairs < 0) return MDKK_E_ARG;
    if (n_pairs == 0) return MDKK_OK;
    const long long threads = (long long)n_pairs * 32;
    k_snap_deidrj_staged<<<(unsigned)((threads + 127) / 128), 128, 0, mdkk::as_stream(stream)>>>(
        n_pairs, s->n_flat, rows, cols, reinterpret_cast<const double2*>(Y), reinterpret_cast<const double2*>(wdu),
        f);
    MDKK_CHECK_LAUNCH("k_snap_deidrj_staged");
    return MDKK_OK;
}

int mdkk_snap_pair_dedr(mdkk_snap* s, int n_pairs, const int* rows, const double* Y, const double* wdu,
                        double* t_out, void* stream) {
    if (!s || n_pairs < 0 || (n_pairs && (!rows || !Y || !wdu || !t_out))) return MDKK_E_ARG;
    if (n_pairs == 0) return MDKK_OK;
    const long long threads = (long long)n_pairs * 32;
    k_snap_pair_dedr<<<(unsigned)((threads + 127) / 128), 128, 0, mdkk::as_stream(stream)>>>(
        n_pairs, s->n_flat, rows, reinterpret_cast<const double2*>(Y), reinterpret_cast<const double2*>(wdu),
        t_out);
    MDKK_CHECK_LAUNCH("k_snap_pair_dedr");
    return MDKK_OK;
}

int mdkk_snap_bi(mdkk_snap* s, const double* U, int n_local, const double* coef, const int* code, const int* tri,
                 const int* chunk, int n_tri, double* B, int layout, int ldu, void* stream) {
    if (!s || n_local < 0 || n_tri < 1 || (layout == 1 && ldu < n_local)) return MDKK_E_ARG;
    const long long su = layout ? 1 : s->n_flat, sf = layout ? ldu : 1;
    if (n_local == 0) return MDKK_OK;
    upload_weights();
    cudaStream_t st = mdkk::as_stream(stream);
    const int nb = (n_local + 31) / 32;
    const double2* u = reinterpret_cast<const double2*>(U);
    double2* out = reinterpret_cast<double2*>(B);
    switch (s->twojmax) {
#define MDKK_BI(TJ)                                                                                        \
    case TJ: {                                                                                             \
        constexpr int NF = block_offset(TJ + 1), NH = half_offset(TJ + 1);                                 \
        const size_t sm = NH * 33 * sizeof(double2);                                                       \
        cudaFuncSetAttribute(k_snap_bi<NF, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);    \
        k_snap_bi<NF, NH><<<nb, kBW * 32, sm, st>>>(u, n_local, coef, code, tri, chunk, n_tri, out, su, sf); \
        break;                                                                                             \
    }
        MDKK_BI(0) MDKK_BI(1) MDKK_BI(2) MDKK_BI(3) MDKK_BI(4) MDKK_BI(5) MDKK_BI(6) MDKK_BI(7) MDKK_BI(8)
#undef MDKK_BI
        default: return MDKK_E_ARG;
    }
    MDKK_CHECK_LAUNCH("k_snap_bi");
    return MDKK_OK;
}

int mdkk_snap_bi_warps(void) { return kBW; }

}  // extern "C"
