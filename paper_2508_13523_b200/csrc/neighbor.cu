// Cell binning (counting sort) and the per-atom stencil neighbour build.
// Reference: mdkk/neighbor.py:83-219 (candidate pairs, style rules, table).
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace {

struct Grid {
    double ox, oy, oz;
    double ix, iy, iz;
    int nx, ny, nz;
};

__device__ __forceinline__ int clampi(int v, int hi) { return v < 0 ? 0 : (v >= hi ? hi - 1 : v); }

__device__ __forceinline__ int3 cell_of(const Grid& g, double x, double y, double z) {
    return make_int3(clampi((int)floor((x - g.ox) * g.ix), g.nx), clampi((int)floor((y - g.oy) * g.iy), g.ny),
                     clampi((int)floor((z - g.oz) * g.iz), g.nz));
}

__global__ void k_cell_keys(const double* __restrict__ x, int n, Grid g, int* __restrict__ key) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double4 p = mdkk::ld4(x, i);
    int3 c = cell_of(g, p.x, p.y, p.z);
    key[i] = (c.x * g.ny + c.y) * g.nz + c.z;
}

// Owning brick: floor(pos / L * grid) clipped (mdkk/domain.py:89-95).
__global__ void k_rank_keys(const double* __restrict__ x, int n, double Lx, double Ly, double Lz, int gx,
                            int gy, int gz, int* __restrict__ key) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double4 p = mdkk::ld4(x, i);
    int cx = clampi((int)floor(p.x / Lx * (double)gx), gx);
    int cy = clampi((int)floor(p.y / Ly * (double)gy), gy);
    int cz = clampi((int)floor(p.z / Lz * (double)gz), gz);
    key[i] = (cx * gy + cy) * gz + cz;
}

__global__ void k_key_count(int n, const int* __restrict__ key, int* __restrict__ counts) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(counts + key[i], 1);
}

__global__ void k_cell_scatter(int n, const int* __restrict__ cid, const int* __restrict__ start,
                               int* __restrict__ cursor, int* __restrict__ atoms) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int c = cid[i];
    atoms[start[c] + atomicAdd(cursor + c, 1)] = i;
}

// Deterministic order inside a cell: ascending row index (insertion sort).
__global__ void k_cell_sort(int ncell, const int* __restrict__ start, int* __restrict__ atoms) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    int b = start[c], e = start[c + 1];
    for (int k = b + 1; k < e; ++k) {
        int v = atoms[k], m = k - 1;
        while (m >= b && atoms[m] > v) {
            atoms[m + 1] = atoms[m];
            --m;
        }
        atoms[m + 1] = v;
    }
}

__device__ __forceinline__ bool lex_zyx_less(const double4& a, const double4& b) {
    // mdkk/neighbor.py:163-166: z, then y, then x
    return (a.z < b.z) || (a.z == b.z && (a.y < b.y || (a.y == b.y && a.x < b.x)));
}

template <int STYLE, bool NEWTON>
__global__ void __launch_bounds__(128) k_nbr_build(const double* __restrict__ x, int n_local, Grid g,
                                                   const int* __restrict__ cell_start,
                                                   const int* __restrict__ cell_atoms,
                                                   const int64_t* __restrict__ gid,
                                                   const int32_t* __restrict__ owner_rank, int my_rank,
                                                   double bc2, int cap, int* __restrict__ table,
                                                   int* __restrict__ counts, int* __restrict__ max_count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int cnt = 0;
    if (i < n_local) {
        const double4 xi = mdkk::ld4(x, i);
        const int3 c = cell_of(g, xi.x, xi.y, xi.z);
        int64_t gi = 0;
        if (STYLE == 1) gi = gid[i];
        for (int ax = c.x - 1; ax <= c.x + 1; ++ax) {
            if (ax < 0 || ax >= g.nx) continue;
            for (int ay = c.y - 1; ay <= c.y + 1; ++ay) {
                if (ay < 0 || ay >= g.ny) continue;
                // cells (ax, ay, c.z-1 .. c.z+1) are contiguous in cell order
                int z0 = max(c.z - 1, 0), z1 = min(c.z + 1, g.nz - 1);
                int base = (ax * g.ny + ay) * g.nz;
                int s0 = cell_start[base + z0], s1 = cell_start[base + z1 + 1];
                for (int s = s0; s < s1; ++s) {
                    int j = cell_atoms[s];
                    if (j == i) continue;
                    double4 xj = mdkk::ld4(x, j);
                    double r2 = mdkk::r2_exact(xj.x - xi.x, xj.y - xi.y, xj.z - xi.z);
                    if (!(r2 < bc2)) continue;
                    if (STYLE == 1) {
                        bool keep;
                        if (j < n_local) {
                            keep = gi < gid[j];
                        } else if (NEWTON) {
                            int orank = owner_rank[j];
                            keep = orank > my_rank || (orank == my_rank && lex_zyx_less(xi, xj));
                        } else {
                            keep = true;
                        }
                        if (!keep) continue;
                    }
                    if (cnt < cap) table[(long long)cnt * n_local + i] = j;
                    ++cnt;
                }
            }
        }
        counts[i] = cnt;
    }
    // warp max then one atomic per warp
    int m = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(max_count, m);
}

// Canonical per-row order: (gid[j], z_j, y_j, x_j) ascending (mdkk/neighbor.py:192-197).
__device__ __forceinline__ bool canon_less(int a, int b, const double* x, const int64_t* gid) {
    int64_t ga = gid[a], gb = gid[b];
    if (ga != gb) return ga < gb;
    double4 pa = mdkk::ld4(x, a), pb = mdkk::ld4(x, b);
    if (pa.z != pb.z) return pa.z < pb.z;
    if (pa.y != pb.y) return pa.y < pb.y;
    return pa.x < pb.x;
}

__global__ void k_canonicalize(const double* __restrict__ x, const int64_t* __restrict__ gid, int n_local,
                               int cap, int* __restrict__ table, const int* __restrict__ counts) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    int n = min(counts[i], cap);
    for (int k = 1; k < n; ++k) {
        int v = table[(long long)k * n_local + i];
        int m = k - 1;
        while (m >= 0 && canon_less(v, table[(long long)m * n_local + i], x, gid)) {
            table[(long long)(m + 1) * n_local + i] = table[(long long)m * n_local + i];
            --m;
        }
        table[(long long)(m + 1) * n_local + i] = v;
    }
}

__global__ void k_max_disp2(const double* __restrict__ x, const double* __restrict__ xr, int n,
                            double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double d2 = 0.0;
    if (i < n) {
        double4 a = mdkk::ld4_nc(x, i), b = mdkk::ld4_nc(xr, i);
        d2 = mdkk::r2_exact(a.x - b.x, a.y - b.y, a.z - b.z);
    }
    d2 = mdkk::warp_max(d2);
    if ((threadIdx.x & 31) == 0) mdkk::atomic_max_nonneg(out, d2);
}

Grid make_grid(const double* gh, const int* nc) {
    Grid g;
    g.ox = gh[0];
    g.oy = gh[1];
    g.oz = gh[2];
    g.ix = gh[3];
    g.iy = gh[4];
    g.iz = gh[5];
    g.nx = nc[0];
    g.ny = nc[1];
    g.nz = nc[2];
    return g;
}

}  // namespace

extern "C" {

int mdkk_bucket_sort(mdkk_ctx* ctx, const int* keys, int n, int nbuckets, int* bucket_start, int* order,
                     void* stream) {
    if (!ctx || n < 0 || nbuckets < 1 || nbuckets > (1 << 30)) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int*)nullptr, (int*)nullptr, nbuckets + 1, s);
    size_t off_cnt = 0;
    size_t off_cur = off_cnt + sizeof(int) * ((size_t)nbuckets + 64);
    size_t off_cub = off_cur + sizeof(int) * ((size_t)nbuckets + 64);
    off_cub = (off_cub + 255) & ~size_t(255);
    char* base = static_cast<char*>(mdkk::scratch(ctx, off_cub + cub_bytes + 256));
    if (!base) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    int* cnt = reinterpret_cast<int*>(base + off_cnt);
    int* cur = reinterpret_cast<int*>(base + off_cur);
    void* tmp = base + off_cub;
    cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)nbuckets + 1), s);
    cudaMemsetAsync(cur, 0, sizeof(int) * (size_t)nbuckets, s);
    if (n > 0) {
        k_key_count<<<mdkk::grid_for(n, 256), 256, 0, s>>>(n, keys, cnt);
        MDKK_CHECK_LAUNCH("k_key_count");
    }
    cub::DeviceScan::ExclusiveSum(tmp, cub_bytes, cnt, bucket_start, nbuckets + 1, s);
    if (n > 0) {
        k_cell_scatter<<<mdkk::grid_for(n, 256), 256, 0, s>>>(n, keys, bucket_start, cur, order);
        MDKK_CHECK_LAUNCH("k_cell_scatter");
        k_cell_sort<<<mdkk::grid_for(nbuckets, 128), 128, 0, s>>>(nbuckets, bucket_start, order);
        MDKK_CHECK_LAUNCH("k_cell_sort");
    }
    return MDKK_OK;
}

int mdkk_cell_keys(const double* x, int n, const double* grid_host, const int* ncell_host, int* keys,
                   void* stream) {
    if (n < 0 || !grid_host || !ncell_host) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    Grid g = make_grid(grid_host, ncell_host);
    if (g.nx < 1 || g.ny < 1 || g.nz < 1) return MDKK_E_ARG;
    k_cell_keys<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(x, n, g, keys);
    MDKK_CHECK_LAUNCH("k_cell_keys");
    return MDKK_OK;
}

int mdkk_rank_keys(const double* x, int n, const double* lengths_host, const int* grid_host, int* keys,
                   void* stream) {
    if (n < 0 || !lengths_host || !grid_host) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    k_rank_keys<<<mdkk::grid_for(n, 256), 256, 0, mdkk::as_stream(stream)>>>(
        x, n, lengths_host[0], lengths_host[1], lengths_host[2], grid_host[0], grid_host[1], grid_host[2], keys);
    MDKK_CHECK_LAUNCH("k_rank_keys");
    return MDKK_OK;
}

int mdkk_bin_atoms(mdkk_ctx* ctx, const double* x, int n, const double* grid_host, const int* ncell_host,
                   int* keys, int* cell_start, int* cell_atoms, void* stream) {
    if (!ctx || n < 0 || !grid_host || !ncell_host) return MDKK_E_ARG;
    long long ncell = (long long)ncell_host[0] * ncell_host[1] * ncell_host[2];
    if (ncell < 1 || ncell > (1LL << 30)) return MDKK_E_ARG;
    int st = mdkk_cell_keys(x, n, grid_host, ncell_host, keys, stream);
    if (st != MDKK_OK) return st;
    return mdkk_bucket_sort(ctx, keys, n, (int)ncell, cell_start, cell_atoms, stream);
}

int mdkk_nbr_build(mdkk_ctx*, const double* x, int n_local, int n_total, const double* grid_host,
                   const int* ncell_host, const int* cell_start, const int* cell_atoms, const int64_t* gid,
                   const int32_t* owner_rank, int my_rank, double bc2, int style, int newton, int cap,
                   int* table, int* counts, int* max_count, void* stream) {
    if (n_local < 0 || n_total < n_local || cap < 1 || (style != 0 && style != 1)) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    Grid g = make_grid(grid_host, ncell_host);
    cudaStream_t s = mdkk::as_stream(stream);
    int nb = mdkk::grid_for(n_local, 128);
    if (style == 0)
        k_nbr_build<0, false><<<nb, 128, 0, s>>>(x, n_local, g, cell_start, cell_atoms, gid, owner_rank,
                                                 my_rank, bc2, cap, table, counts, max_count);
    else if (newton)
        k_nbr_build<1, true><<<nb, 128, 0, s>>>(x, n_local, g, cell_start, cell_atoms, gid, owner_rank,
                                                my_rank, bc2, cap, table, counts, max_count);
    else
        k_nbr_build<1, false><<<nb, 128, 0, s>>>(x, n_local, g, cell_start, cell_atoms, gid, owner_rank,
                                                 my_rank, bc2, cap, table, counts, max_count);
    MDKK_CHECK_LAUNCH("k_nbr_build");
    return MDKK_OK;
}

int mdkk_nbr_canonicalize(const double* x, const int64_t* gid, int n_local, int cap, int* table,
                          const int* counts, void* stream) {
    if (n_local < 0 || cap < 1) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    k_canonicalize<<<mdkk::grid_for(n_local, 128), 128, 0, mdkk::as_stream(stream)>>>(x, gid, n_local, cap,
                                                                                       table, counts);
    MDKK_CHECK_LAUNCH("k_canonicalize");
    return MDKK_OK;
}

int mdkk_max_disp2(const double* x, const double* x_ref, int n, double* out, void* stream) {
    if (n < 0) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    cudaMemsetAsync(out, 0, sizeof(double), s);
    if (n == 0) return MDKK_OK;
    k_max_disp2<<<mdkk::grid_for(n, 256), 256, 0, s>>>(x, x_ref, n, out);
    MDKK_CHECK_LAUNCH("k_max_disp2");
    return MDKK_OK;
}

}  // extern "C"
