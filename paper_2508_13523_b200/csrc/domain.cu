// Domain kernels: wrap, halo selection (stable multi-way compaction),
// forward-comm pack with periodic shift, reverse-comm fold, row permutes.
// Reference: mdkk/domain.py:56-63, :246-334.

#include "common.cuh"

namespace {

constexpr int kHaloBlock = 256;
constexpr int kMaxCombos = 27 * 64;

__global__ void k_wrap(double* __restrict__ x, int n, double Lx, double Ly, double Lz) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double4 p = mdkk::ld4_nc(x, i);
    // pos - L * floor(pos / L) exactly as mdkk/domain.py:62
    // (explicit roundings: no FMA contraction, bit-identical to numpy)
    p.x = __dsub_rn(p.x, __dmul_rn(Lx, floor(p.x / Lx)));
    p.y = __dsub_rn(p.y, __dmul_rn(Ly, floor(p.y / Ly)));
    p.z = __dsub_rn(p.z, __dmul_rn(Lz, floor(p.z / Lz)));
    mdkk::st4(x, i, p);
}

__device__ __forceinline__ bool in_combo(const double4& p, const double* c) {
    // shifted = x + shift ; lo <= shifted < hi on every axis (mdkk/domain.py:273-274)
    double sx = p.x + c[6], sy = p.y + c[7], sz = p.z + c[8];
    return sx >= c[0] && sx < c[3] && sy >= c[1] && sy < c[4] && sz >= c[2] && sz < c[5];
}

// Per-thread bit mask of the combos (<= 64 per call) the atom falls in, and the
// block-wide OR: blocks of cell-sorted rows are compact, so most of them touch no
// halo at all and skip every per-combo block reduction.  (Pre-testing the combos
// against each warp's bounding box measured slower: the kernels are latency bound.)
__device__ __forceinline__ unsigned long long combo_mask(const double4& p, const double* sc, int c0, int C,
                                                         bool valid) {
    unsigned long long m = 0ull;
    if (valid)
        for (int c = c0; c < min(C, c0 + 64); ++c)
            if (in_combo(p, sc + 9 * c)) m |= 1ull << (c - c0);
    return m;
}

__device__ __forceinline__ unsigned long long block_or(unsigned long long m, unsigned long long* s_or) {
    if (threadIdx.x == 0) *s_or = 0ull;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
    if ((threadIdx.x & 31) == 0 && m) atomicOr(s_or, m);
    __syncthreads();
    return *s_or;
}

// rows / n_dev (optional): scan only rows[k] for k < *n_dev (ascending: the boundary-layer
// rows of a cell-sorted brick, the only ones a halo no wider than a cell can select);
// blocks past the device count contribute empty counts.
__device__ __forceinline__ int halo_row(int k, int n, const int* rows, const int* n_dev, bool& ok) {
    ok = k < n && (n_dev == nullptr || k < *n_dev);
    return ok ? (rows ? rows[k] : k) : 0;
}

__global__ void k_halo_count(const double* __restrict__ x, int n, const double* __restrict__ combos,
                             int C, int* __restrict__ block_counts, const int* __restrict__ rows,
                             const int* __restrict__ n_dev) {
    extern __shared__ double sc[];
    __shared__ unsigned long long s_or;
    if (n_dev && (long long)blockIdx.x * blockDim.x >= *n_dev) {   // block-uniform: nothing to select
        for (int c = threadIdx.x; c < C; c += blockDim.x) block_counts[(long long)c * gridDim.x + blockIdx.x] = 0;
        return;
    }
    for (int t = threadIdx.x; t < 9 * C; t += blockDim.x) sc[t] = combos[t];
    __syncthreads();
    bool ok;
    const int i = halo_row(blockIdx.x * blockDim.x + threadIdx.x, n, rows, n_dev, ok);
    double4 p = make_double4(0, 0, 0, 0);
    if (ok) p = mdkk::ld4(x, i);
    __shared__ int s_wc[kHaloBlock / 32][64];   // per-warp counts of the group's combos
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int c0 = 0; c0 < C; c0 += 64) {   // combos in groups of 64 (one mask word)
        const unsigned long long mine = combo_mask(p, sc, c0, C, ok);
        const unsigned long long any = block_or(mine, &s_or);
        // one ballot per present combo per warp, one barrier for the group (not one per combo)
        for (unsigned long long a = any; a; a &= a - 1ull) {   // block-uniform
            const int cb = __ffsll((long long)a) - 1;
            const int cnt = __popc(__ballot_sync(0xffffffffu, (mine >> cb) & 1ull));
            if (lane == 0) s_wc[wid][cb] = cnt;
        }
        __syncthreads();
        for (int cb = threadIdx.x; cb < min(64, C - c0); cb += blockDim.x) {
            int t = 0;
            if ((any >> cb) & 1ull)
                for (int q = 0; q < kHaloBlock / 32; ++q) t += s_wc[q][cb];
            block_counts[(long long)(c0 + cb) * gridDim.x + blockIdx.x] = t;   // combo-major
        }
        __syncthreads();
    }
}

// One block per combo: exclusive scan of that combo's per-block counts in place
// (combo-major [C][nb]: contiguous, four consecutive entries per thread per pass);
// totals[c].
__global__ void __launch_bounds__(1024) k_halo_scan(int* __restrict__ block_counts, int nb, int C,
                                                    int* __restrict__ totals) {
    __shared__ int warp_tot[32];
    __shared__ int carry;
    const int c = blockIdx.x;
    int* col = block_counts + (long long)c * nb;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = 0; base < nb; base += 4 * blockDim.x) {
        const int b = base + 4 * threadIdx.x;
        int v[4], s = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[q] = b + q < nb ? col[b + q] : 0;
            s += v[q];
        }
        int incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int w = lane < nw ? warp_tot[lane] : 0;
            int wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            if (lane < nw) warp_tot[lane] = wi - w;   // exclusive warp offsets
        }
        __syncthreads();
        int run = carry + warp_tot[wid] + incl - s;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (b + q < nb) col[b + q] = run;
            run += v[q];
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = run;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[c] = carry;
}

__global__ void k_halo_fill(const double* __restrict__ x, int n, const double* __restrict__ combos, int C,
                            const int* __restrict__ block_off, const int* __restrict__ totals,
                            int* __restrict__ out, const int8_t* __restrict__ combo_code,
                            int8_t* __restrict__ out_code, const int* __restrict__ rows,
                            const int* __restrict__ n_dev) {
    extern __shared__ double sc[];
    int* base = reinterpret_cast<int*>(sc + 9 * C);
    __shared__ unsigned s_bal[kHaloBlock / 32][64];   // per-warp ballots of the group's combos
    __shared__ unsigned long long s_or;
    if (n_dev && (long long)blockIdx.x * blockDim.x >= *n_dev) return;
    for (int t = threadIdx.x; t < 9 * C; t += blockDim.x) sc[t] = combos[t];
    if (threadIdx.x == 0) {
        int s = 0;
        for (int c = 0; c < C; ++c) {
            base[c] = s;
            s += totals[c];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    bool ok;
    const int i = halo_row(blockIdx.x * blockDim.x + threadIdx.x, n, rows, n_dev, ok);
    double4 p = make_double4(0, 0, 0, 0);
    if (ok) p = mdkk::ld4(x, i);
    for (int c0 = 0; c0 < C; c0 += 64) {   // combos in groups of 64 (one mask word)
        const unsigned long long mine = combo_mask(p, sc, c0, C, ok);
        const unsigned long long any = block_or(mine, &s_or);
        // the ballots of every present combo, then one barrier: each row's rank in its combo
        // = rows of earlier warps + earlier lanes (rows ascending, as the one-barrier-per-combo
        // form had it)
        for (unsigned long long a = any; a; a &= a - 1ull) {   // block-uniform
            const int cb = __ffsll((long long)a) - 1;
            const unsigned m = __ballot_sync(0xffffffffu, (mine >> cb) & 1ull);
            if (lane == 0) s_bal[wid][cb] = m;
        }
        __syncthreads();
        for (unsigned long long a = mine; a; a &= a - 1ull) {
            const int cb = __ffsll((long long)a) - 1;
            const int c = c0 + cb;
            int r = __popc(s_bal[wid][cb] & ((1u << lane) - 1u));
            for (int q = 0; q < wid; ++q) r += __popc(s_bal[q][cb]);
            const int o = base[c] + block_off[(long long)c * gridDim.x + blockIdx.x] + r;
            out[o] = i;
            if (out_code) out_code[o] = combo_code[c];
        }
        __syncthreads();
    }
}


// Rows of the cells within `layer` cells of the grid's faces, ascending (cells in key
// order, each a contiguous ascending row range of a cell-sorted brick).  Keys follow
// the serpentine order of csrc/cluster.cuh.
__global__ void k_boundary_counts(const int* __restrict__ cell_start, int nx, int ny, int nz, int layer,
                                  int* __restrict__ cnt) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int ncell = nx * ny * nz;
    if (c > ncell) return;
    if (c == ncell) {
        cnt[c] = 0;
        return;
    }
    const int col = c / nz, czs = c - col * nz;
    const int cz = (col & 1) ? nz - 1 - czs : czs;
    const int cx = col / ny, cys = col - cx * ny;
    const int cy = (cx & 1) ? ny - 1 - cys : cys;
    const bool edge = cx <= layer || cx >= nx - 1 - layer || cy <= layer || cy >= ny - 1 - layer ||
                      cz <= layer || cz >= nz - 1 - layer;
    cnt[c] = edge ? cell_start[c + 1] - cell_start[c] : 0;
}

__global__ void k_boundary_fill(const int* __restrict__ cell_start, int ncell, const int* __restrict__ cnt,
                                const int* __restrict__ off, int* __restrict__ rows, int* __restrict__ count) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c == 0) *count = off[ncell];
    if (c >= ncell || cnt[c] == 0) return;
    const int r0 = cell_start[c], o = off[c];
    for (int t = 0; t < cnt[c]; ++t) rows[o + t] = r0 + t;
}

__global__ void k_pack_shift(const double* __restrict__ x, const int* __restrict__ idx,
                             const int8_t* __restrict__ code, const double* __restrict__ shifts, int n,
                             double* __restrict__ out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double4 p = mdkk::ld4_nc(x, idx[k]);
    const double* s = shifts + 3 * code[k];
    // ghost x = owner x + shift: one rounding, as mdkk/domain.py:281,300
    mdkk::st4(out, k, make_double4(p.x + s[0], p.y + s[1], p.z + s[2], 0.0));
}

// New ghost rows in one pass: position (= pack), global id and owner index.
__global__ void k_ghost_rows(const double* __restrict__ x, const int64_t* __restrict__ gid,
                             const int* __restrict__ idx, const int8_t* __restrict__ code,
                             const double* __restrict__ shifts, int n, double* __restrict__ out_x,
                             int64_t* __restrict__ out_gid, int* __restrict__ out_oidx) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = idx[k];
    double4 p = mdkk::ld4_nc(x, i);
    const double* s = shifts + 3 * code[k];
    mdkk::st4(out_x, k, make_double4(p.x + s[0], p.y + s[1], p.z + s[2], 0.0));
    out_gid[k] = gid[i];
    out_oidx[k] = i;
}

__global__ void k_fold_add(double* __restrict__ f, const int* __restrict__ idx,
                           const double* __restrict__ buf, int n) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double4 b = mdkk::ld4_nc(buf, k);
    double* t = f + 4LL * idx[k];
    atomicAdd(t + 0, b.x);
    atomicAdd(t + 1, b.y);
    atomicAdd(t + 2, b.z);
}

__global__ void k_gather4(const double* __restrict__ src, const int* __restrict__ perm, int n,
                          double* __restrict__ dst) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mdkk::st4(dst, i, mdkk::ld4_nc(src, perm[i]));
}
__global__ void k_scatter4(const double* __restrict__ src, const int* __restrict__ perm, int n,
                           double* __restrict__ dst) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mdkk::st4(dst, perm[i], mdkk::ld4_nc(src, i));
}
template <typename T>
__global__ void k_gather(const T* __restrict__ src, const int* __restrict__ perm, int n, T* __restrict__ dst) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

}  // namespace

extern "C" {

int mdkk_wrap(double* x, int n, const double* L, void* stream) {
    if (n < 0 || !L) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_wrap<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(x, n, L[0], L[1], L[2]);
    MDKK_CHECK_LAUNCH("k_wrap");
    return MDKK_OK;
}

int mdkk_halo_count(mdkk_ctx*, const double* x, int n, const double* combos, int C, int* block_scratch,
                    int* totals, const int* rows, const int* n_dev, void* stream) {
    if (n < 0 || C < 0 || C > kMaxCombos) return MDKK_E_ARG;
    if (C == 0) return MDKK_OK;
    cudaStream_t s = mdkk::as_stream(stream);
    int nb = mdkk::grid_for(n, kHaloBlock);
    size_t sm = sizeof(double) * 9 * C;
    k_halo_count<<<nb, kHaloBlock, sm, s>>>(x, n, combos, C, block_scratch, rows, n_dev);
    MDKK_CHECK_LAUNCH("k_halo_count");
    k_halo_scan<<<C, 1024, 0, s>>>(block_scratch, nb, C, totals);
    MDKK_CHECK_LAUNCH("k_halo_scan");
    return MDKK_OK;
}

int mdkk_halo_fill(mdkk_ctx*, const double* x, int n, const double* combos, int C, const int* block_scratch,
                   const int* totals, int* out_idx, const int8_t* combo_code, int8_t* out_code, const int* rows,
                   const int* n_dev, void* stream) {
    if (n < 0 || C < 0 || C > kMaxCombos || (out_code && !combo_code)) return MDKK_E_ARG;
    if (C == 0 || n == 0) return MDKK_OK;
    int nb = mdkk::grid_for(n, kHaloBlock);
    size_t sm = sizeof(double) * 9 * C + sizeof(int) * C;
    k_halo_fill<<<nb, kHaloBlock, sm, mdkk::as_stream(stream)>>>(x, n, combos, C, block_scratch, totals,
                                                                  out_idx, combo_code, out_code, rows, n_dev);
    MDKK_CHECK_LAUNCH("k_halo_fill");
    return MDKK_OK;
}

int mdkk_boundary_rows(mdkk_ctx* ctx, const int* cell_start, const int* ncell_host, int layer, int* rows,
                       int* count, void* stream) {
    if (!ctx || !cell_start || !ncell_host || !rows || !count || layer < 0) return MDKK_E_ARG;
    const long long ncl = (long long)ncell_host[0] * ncell_host[1] * ncell_host[2];
    if (ncl < 1 || ncl >= (1LL << 30)) return MDKK_E_ARG;
    const int ncell = (int)ncl;
    cudaStream_t s = mdkk::as_stream(stream);
    int* cnt = static_cast<int*>(mdkk::scratch(ctx, sizeof(int) * ((size_t)ncell + 2) * 2));
    if (!cnt) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    int* off = cnt + ncell + 2;
    const int nx = ncell_host[0], ny = ncell_host[1], nz = ncell_host[2];
    k_boundary_counts<<<mdkk::grid_for(ncell + 1, 256), 256, 0, s>>>(cell_start, nx, ny, nz, layer, cnt);
    MDKK_CHECK_LAUNCH("k_boundary_counts");
    const int st = mdkk::exclusive_scan_i32(ctx, cnt, off, (long long)ncell + 1, s);
    if (st != MDKK_OK) return st;
    k_boundary_fill<<<mdkk::grid_for(ncell, 256), 256, 0, s>>>(cell_start, ncell, cnt, off, rows, count);
    MDKK_CHECK_LAUNCH("k_boundary_fill");
    return MDKK_OK;
}

int mdkk_pack_shift(const double* x, const int* idx, const int8_t* code, const double* shifts, int n,
                    double* out, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_pack_shift<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(x, idx, code, shifts, n, out);
    MDKK_CHECK_LAUNCH("k_pack_shift");
    return MDKK_OK;
}

int mdkk_ghost_rows(const double* x, const int64_t* gid, const int* idx, const int8_t* code, const double* shifts,
                    int n, double* out_x, int64_t* out_gid, int* out_oidx, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_ghost_rows<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(x, gid, idx, code, shifts, n, out_x,
                                                                              out_gid, out_oidx);
    MDKK_CHECK_LAUNCH("k_ghost_rows");
    return MDKK_OK;
}

int mdkk_fold_add(double* f, const int* idx, const double* buf, int n, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_fold_add<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(f, idx, buf, n);
    MDKK_CHECK_LAUNCH("k_fold_add");
    return MDKK_OK;
}

int mdkk_gather_rows4(const double* src, const int* perm, int n, double* dst, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_gather4<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(src, perm, n, dst);
    MDKK_CHECK_LAUNCH("k_gather4");
    return MDKK_OK;
}

int mdkk_scatter_rows4(const double* src, const int* perm, int n, double* dst, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_scatter4<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(src, perm, n, dst);
    MDKK_CHECK_LAUNCH("k_scatter4");
    return MDKK_OK;
}

int mdkk_gather_i64(const int64_t* src, const int* perm, int n, int64_t* dst, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_gather<int64_t><<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(src, perm, n, dst);
    MDKK_CHECK_LAUNCH("k_gather_i64");
    return MDKK_OK;
}

int mdkk_gather_i32(const int32_t* src, const int* perm, int n, int32_t* dst, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_gather<int32_t><<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(src, perm, n, dst);
    MDKK_CHECK_LAUNCH("k_gather_i32");
    return MDKK_OK;
}

}  // extern "C"
