// Cell grid (serpentine order) shared by the binning, the spatial sort and the
// neighbour build.
//
// Neighbour table layout ("cluster-blocked"): owned rows are cell-sorted and
// cluster c = rows [32c, 32c+32) (one warp in the build and force kernels);
// table[c][k][lane] (int32, row index of the k-th partner of row 32c+lane) so
// every per-k read of a warp is one coalesced 128-byte line; counts[i] entries
// are valid for row i, the rest undefined.
#pragma once

#include "common.cuh"

namespace mdkk {

struct Grid {
    double ox, oy, oz;
    double ix, iy, iz;
    int nx, ny, nz;
};

__host__ __device__ inline Grid make_grid(const double* gh, const int* nc) {
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

__device__ __forceinline__ int clampi(int v, int hi) { return v < 0 ? 0 : (v >= hi ? hi - 1 : v); }

__device__ __forceinline__ int3 cell_of(const Grid& g, double x, double y, double z) {
    return make_int3(clampi((int)floor((x - g.ox) * g.ix), g.nx), clampi((int)floor((y - g.oy) * g.iy), g.ny),
                     clampi((int)floor((z - g.oz) * g.iz), g.nz));
}

// Serpentine (boustrophedon) cell order: consecutive keys are face-adjacent
// cells, so 32 consecutive cell-sorted atoms form a compact cluster.  A z-run
// of one (x, y) column is still a contiguous key range.
__device__ __forceinline__ int column_of(const Grid& g, int cx, int cy) {
    return cx * g.ny + ((cx & 1) ? g.ny - 1 - cy : cy);
}
__device__ __forceinline__ int cell_key(const Grid& g, int cx, int cy, int cz) {
    int col = column_of(g, cx, cy);
    return col * g.nz + ((col & 1) ? g.nz - 1 - cz : cz);
}
// Key range [k0, k1] covering cz in [z0, z1] of column (cx, cy).
__device__ __forceinline__ int2 zrun_keys(const Grid& g, int cx, int cy, int z0, int z1) {
    int col = column_of(g, cx, cy);
    return (col & 1) ? make_int2(col * g.nz + g.nz - 1 - z1, col * g.nz + g.nz - 1 - z0)
                     : make_int2(col * g.nz + z0, col * g.nz + z1);
}


}  // namespace mdkk
