// Shared SNAP device helpers (included by snap.cu and snap_aux.cu; everything
// lives in an anonymous namespace, so each translation unit owns its copy of
// the __device__/__constant__ tables and uploads it with upload_weights()).
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

struct ZEntry {      // one U*U product of the Z-list adjoint (16 B, one broadcast LDS.128)
    double coef;
    int goff;        // byte offset of U[g] in the shared tile (g * row stride)
    int hcode;       // byte offset of U[h] | conj_g << 20 | conj_h << 21 | last-of-output << 22 | center << 23
};

struct mdkk_snap {
    int twojmax = 0;
    int n_flat = 0;
    int n_half = 0;
    int n_entries = 0;
    ZEntry* ent = nullptr;   // [n_entries], sorted by output
    int* chunk = nullptr;    // [kYW + 1] per-warp entry ranges (output-aligned, balanced)
    int* chunkf = nullptr;   // [kYW] first output (half index) of each warp's range
    int* fmap = nullptr;     // [n_flat] half index | mirrored << 16 | odd sign << 17
    double* work = nullptr;  // mdkk_snap_compute workspace: U [n][n_flat] then Yh [n_half][n] (complex)
    size_t work_bytes = 0;
    // schedule knobs (SnapState.batch_u / batch_y, mdkk/snap/compute.py:238-276; scheduling only):
    int ui_ppw = 2;    // compute_ui: pairs expanded concurrently per warp (1, 2, 4 -> 32-, 16-, 8-lane teams)
                       // = batch_u / 2 (batch_u pairs in flight per two warps), clamped to [1, 4]
    int yi_batch = 1;  // compute_yi: atoms per lane (1 or 2: each Z-list broadcast serves 2 atoms)
};

namespace {

constexpr int kMaxTwoJ = 8;
constexpr int kLevelMax = (kMaxTwoJ + 1) * (kMaxTwoJ + 1);  // 81
constexpr int kWarps = 4;
constexpr double kPi = 3.141592653589793;

__host__ __device__ constexpr int block_offset(int tj) { return tj * (tj + 1) * (2 * tj + 1) / 6; }

struct cplx {
    double re, im;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ cplx cconj(cplx a) { return {a.re, -a.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx cscale(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx cneg(cplx a) { return {-a.re, -a.im}; }

// Weights of the two-term column recursion, rs[k][l] = sqrt(k / l) (0 <= k, l <= 8).
// Staged per CTA in shared memory (lanes read different entries: constant
// memory would serialise).
__device__ double g_rs[kMaxTwoJ + 1][kMaxTwoJ + 1];

struct RS {
    double v[kMaxTwoJ + 1][kMaxTwoJ + 1];
};

__device__ __forceinline__ void stage_rs(RS& rs) {
    for (int t = threadIdx.x; t < (kMaxTwoJ + 1) * (kMaxTwoJ + 1); t += blockDim.x)
        rs.v[t / (kMaxTwoJ + 1)][t % (kMaxTwoJ + 1)] = g_rs[t / (kMaxTwoJ + 1)][t % (kMaxTwoJ + 1)];
    __syncthreads();
}

struct PairGeo {
    cplx a, b;
    double fc, dfc, r;
};

// a, b, f_c, f_c' (mdkk/snap/compute.py:27-45).  One sincospi per angle and one
// reciprocal of r0 instead of tan / cos / sin and four divisions (equal to the
// reference's expressions to a few ulp).
__device__ __forceinline__ void pair_geometry(double dx, double dy, double dz, double r2, double rc, PairGeo& g,
                                              double& z0, double& r0) {
    const double r = sqrt(r2);
    double s1, c1, s2, c2;
    sincospi(0.99 * r / rc, &s1, &c1);   // z0 = r / tan(0.99 pi r / rc)
    sincospi(r / rc, &s2, &c2);
    z0 = r * c1 / s1;
    r0 = sqrt(r * r + z0 * z0);
    const double ir0 = 1.0 / r0;
    g.r = r;
    g.a = {z0 * ir0, -dz * ir0};
    g.b = {dy * ir0, -dx * ir0};
    g.fc = 0.5 * (1.0 + c2);
    g.dfc = -kPi / (2.0 * rc) * s2;
}

// d a / d dr_k, d b / d dr_k (mdkk/snap/compute.py:48-63), with reciprocals of r and r0.
__device__ __forceinline__ void pair_grads(const double d[3], const PairGeo& g, double rc, double z0, double r0,
                                           cplx da[3], cplx db[3]) {
    const double r = g.r, ct = 0.99 * kPi / rc;
    const double ir = 1.0 / r, ir0 = 1.0 / r0;
    const double dz0_dr = (z0 - ct * (r * r + z0 * z0)) * ir;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double dz0 = dz0_dr * (d[k] * ir);
        const double t = (d[k] + z0 * dz0) * ir0 * ir0;   // dr0 / r0
        da[k] = {dz0 * ir0 - g.a.re * t, (k == 2 ? -ir0 : 0.0) - g.a.im * t};
        db[k] = {(k == 1 ? ir0 : 0.0) - g.b.re * t, (k == 0 ? -ir0 : 0.0) - g.b.im * t};
    }
}

// Two-term column recursion for the Wigner-U levels (levels column-major: v[Q*tj + P]).  With level 1 =
// [[conj(a), -conj(b)], [b, a]] (mdkk/snap/compute.py:125-147), every column
// Q < tj of level tj follows from column Q of level tj-1:
//   u[P][Q] = sqrt((tj-P)/(tj-Q)) conj(a) v[P][Q] + sqrt(P/(tj-Q)) b v[P-1][Q]
// (the same matrices as the reference's four-term recursion, half the
// products; checked against it to ~1e-16 in the parity tests).  The right
// half of each level follows from the mirror X[tj-P][tj-Q] = (-1)^(P+Q)
// conj(X[P][Q]), so only the column half C_tj = {2Q < tj, or 2Q == tj and
// 2P <= tj} is computed; it has half_size(tj) elements, enumerated column-major.
// Branch-free at the column ends: the weights vanish there (sqrt(0) for P == tj
// resp. P == 0) and the out-of-column operand is a finite neighbour (clamped
// index, buffers zero-initialised), so both terms are always evaluated.
// `vmax` (compact level storage): the last readable slot of the level, so the
// zero-weight read below the last column (P == tj) stays inside it instead of
// touching the next level's first slot, which the same pass writes.
__device__ __forceinline__ cplx rec2(const cplx* v, int tj, int P, int Q, const RS& rs, cplx ab, cplx b,
                                     int vmax = 0x7fffffff) {
    const cplx v0 = v[min(Q * tj + P, vmax)], v1 = v[max(Q * tj + P - 1, 0)];
    const cplx t0 = cmul(ab, v0), t1 = cmul(b, v1);
    const double w0 = rs.v[tj - P][tj - Q], w1 = rs.v[P][tj - Q];
    return {fma(w0, t0.re, w1 * t1.re), fma(w0, t0.im, w1 * t1.im)};
}

__device__ __forceinline__ bool in_col_half(int tj, int P, int Q) {
    return 2 * Q < tj || (2 * Q == tj && 2 * P <= tj);
}

// c-th element (column-major) of C_tj.
__device__ __forceinline__ void col_elem(int tj, int c, int& P, int& Q) {
    const int nfull = ((tj + 1) >> 1) * (tj + 1);
    if (c < nfull) {
        Q = c / (tj + 1);
        P = c - Q * (tj + 1);
    } else {
        Q = tj >> 1;
        P = c - nfull;
    }
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

// ---------------------------------------------- half-block helpers (both kernels)
// Every level obeys X[tj-P][tj-Q] = (-1)^(P+Q) conj(X[P][Q]) (u, U, Y and the
// adjoint lambda), so only the half set H_tj = {2P < tj, or 2P == tj
// and 2Q <= tj} is computed: it is the row-major prefix P*(tj+1)+Q < half_size.
__host__ __device__ constexpr int half_size(int tj) {
    return (tj & 1) ? (tj + 1) * (tj + 1) / 2 : (tj / 2) * (tj + 1) + tj / 2 + 1;
}
__host__ __device__ constexpr int half_offset(int tj) {
    int s = 0;
    for (int t = 0; t < tj; ++t) s += half_size(t);
    return s;
}
// Compact column-major level storage for the recursion: level t keeps columns
// 0..(t+1)>>1 (all the next level reads: C_t plus the mirror of its last column).
__host__ __device__ constexpr int lvl_size(int t) { return (t + 1) * (((t + 1) >> 1) + 1); }
__host__ __device__ constexpr int lvl_offset(int t) {
    int s = 0;
    for (int k = 0; k < t; ++k) s += lvl_size(k);
    return s;
}

// slots of a TEAM-lane team over the column halves (level tj) and their prefix
template <int TEAM>
__host__ __device__ constexpr int tslots(int tj) { return (half_size(tj) + TEAM - 1) / TEAM; }
template <int TEAM>
__host__ __device__ constexpr int tslot_base(int tj) {
    int s = 0;
    for (int t = 0; t < tj; ++t) s += tslots<TEAM>(t);
    return s;
}
constexpr int kHalfAll = half_offset(kMaxTwoJ + 1);      // 145

// Store element (P, Q) of a full level held COLUMN-major in shared memory
// (L[Q*(tj+1) + P]: lanes walk C_tj down a column, so reads and writes of a
// half-warp hit consecutive 16-byte words) and its mirror.
// Store (P, Q) of C_tj for the next level's recursion: the next level reads
// columns 0..(tj+1)>>1 only, i.e. C_tj plus the mirror image of C_tj's last
// column (Q == tj>>1), so only that column writes its mirror.
__device__ __forceinline__ void store_for_next(cplx* L, int tj, int P, int Q, cplx v) {
    L[Q * (tj + 1) + P] = v;
    if (Q == (tj >> 1)) {
        const double sg = ((P + Q) & 1) ? -1.0 : 1.0;
        L[(tj - Q) * (tj + 1) + (tj - P)] = {sg * v.re, -sg * v.im};
    }
}

__device__ __forceinline__ void store_mirrored(cplx* L, int tj, int P, int Q, cplx v) {
    L[Q * (tj + 1) + P] = v;
    const int hm = (tj - Q) * (tj + 1) + (tj - P);
    const double sg = ((P + Q) & 1) ? -1.0 : 1.0;
    L[hm] = {sg * v.re, -sg * v.im};  // the center element writes itself twice (same value)
}

// One in-range partner with its hypersphere geometry, computed once by the
// compaction lane (not by every lane of the half-warp that expands it).
struct NbPair {
    double dx, dy, dz, r;
    double ar, ai, br, bi;   // a, b
    double fc, dfc, z0, r0;
    int j, pad;
};
constexpr int kNbChunk = 16;   // table entries compacted per pass (s_nb holds kNbChunk pairs)

// Compact the in-range partners (r^2 < rc^2, mdkk/snap/compute.py:114-115) of
// table entries [k0, k0+16) of row i into s_nb with their geometry; returns their count.
__device__ __forceinline__ int compact_pairs(const double* x, const int* table, int cap, int i, int k0, int n,
                                             double4 xi, double rc2, double rc, NbPair* s_nb, bool& bad) {
    const int lane = threadIdx.x & 31, k = k0 + lane;
    int j = 0;
    double dx = 0, dy = 0, dz = 0, r2 = 0;
    const bool ok = lane < kNbChunk && k < n && neighbour(x, table, cap, i, k, xi, rc2, j, dx, dy, dz, r2);
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (ok) {
        bad |= !(r2 > 0.0);
        PairGeo g;
        double z0, r0;
        pair_geometry(dx, dy, dz, r2, rc, g, z0, r0);
        s_nb[__popc(m & ((1u << lane) - 1u))] = {dx, dy, dz, g.r, g.a.re, g.a.im, g.b.re, g.b.im,
                                                 g.fc, g.dfc, z0, r0, j, 0};
    }
    __syncwarp();
    return __popc(m);
}

__device__ __forceinline__ void geo_of(const NbPair& nb, PairGeo& g, double& z0, double& r0) {
    g.r = nb.r;
    g.a = {nb.ar, nb.ai};
    g.b = {nb.br, nb.bi};
    g.fc = nb.fc;
    g.dfc = nb.dfc;
    z0 = nb.z0;
    r0 = nb.r0;
}

__constant__ short c_hflat[kHalfAll];       // half index -> flat index

void upload_weights() {
    static bool done = false;
    if (done) return;
    static double h[kMaxTwoJ + 1][kMaxTwoJ + 1] = {};
    for (int k = 0; k <= kMaxTwoJ; ++k)
        for (int l = 1; l <= kMaxTwoJ; ++l) h[k][l] = std::sqrt((double)k / (double)l);
    cudaMemcpyToSymbol(g_rs, h, sizeof(h));
    static short hf[kHalfAll];
    for (int tj = 0; tj <= kMaxTwoJ; ++tj)
        for (int k = 0; k < half_size(tj); ++k) hf[half_offset(tj) + k] = (short)(block_offset(tj) + k);
    cudaMemcpyToSymbol(c_hflat, hf, sizeof(hf));
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
