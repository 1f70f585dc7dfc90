// Cell grid (serpentine order) and the cluster neighbour-table layout shared by
// the build, force and SNAP kernels.
//
// Cluster list format ("mdkk cluster list"):
//   * owned atoms are cell-sorted; cluster c = owned rows [32c, 32c+32) (one warp)
//   * union[c][0..ucount[c]) (int32, row stride ucap): every row within the build
//     cutoff of the cluster's bounding box (the only rows its atoms can list)
//   * table: uint16 local index u into union[c], blocked so one lane loads 8
//     entries with one 16-byte load:  ((c*capb + k/8)*32 + lane)*8 + k%8,
//     capb = cap/8.  counts[i] entries are valid for row i.
// Positions of union[c] are staged in shared memory by the force kernels.
#pragma once

#include "common.cuh"

namespace mdkk {

constexpr int kClusterSize = 32;

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

__device__ __forceinline__ long long tbl_index(int c, int capb, int k, int lane) {
    return ((((long long)c * capb + (k >> 3)) * kClusterSize + lane) << 3) + (k & 7);
}

}  // namespace mdkk
