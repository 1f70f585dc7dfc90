// Cell binning (counting sort) and the cluster neighbour build.
// Reference: mdkk/neighbor.py:83-219 (candidate pairs, style rules, table).
//
// Build = one warp per 32-atom cluster of cell-sorted owned rows:
//   1. bounding box of the cluster (warp min/max)
//   2. union: every row (owned or ghost) in the cells overlapping bbox +/- bc
//      whose distance to the bbox is < bc, ballot-compacted in shared memory
//   3. each lane scans the union (broadcast loads: one wavefront per candidate
//      per warp) and keeps j != i with r^2 < bc^2 (strict, same rounding as
//      the reference) passing the style predicate (mdkk/neighbor.py:134-179).
// Full lists use the streaming variant k_nbr_build_full (union members in a
// 128-entry ring, tested block by block while the cell rows stream); half lists
// use k_nbr_build (whole union staged, gids / owner ranks in shared memory).
// Output: int32 cluster-blocked table [ncl][cap][32] of row indices + counts.
#include <type_traits>

#include "cluster.cuh"

namespace {

using mdkk::Grid;

__global__ void k_cell_keys(const double* __restrict__ x, int n, Grid g, int* __restrict__ key) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double4 p = mdkk::ld4(x, i);
    int3 c = mdkk::cell_of(g, p.x, p.y, p.z);
    key[i] = mdkk::cell_key(g, c.x, c.y, c.z);
}

// k_cell_keys + the counting sort's count pass (one atomic per distinct key per warp).
__global__ void k_cell_keys_count(const double* __restrict__ x, int n, Grid g, int* __restrict__ key,
                                  int* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const double4 p = mdkk::ld4(x, i);
    const int3 c = mdkk::cell_of(g, p.x, p.y, p.z);
    const int k = mdkk::cell_key(g, c.x, c.y, c.z);
    key[i] = k;
    const unsigned same = __match_any_sync(act, k);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(cnt + k, __popc(same));
}

// Binning = cell keys + stable counting sort; with many cells the key pass also counts.
int bin_rows(mdkk_ctx* ctx, const double* x, int n, const double* grid_host, const int* ncell_host, int ncell,
             int* keys, int* cell_start, int* cell_atoms, cudaStream_t s) {
    if (n == 0 || ncell <= mdkk::kSortSmallBuckets) {
        int st = mdkk_cell_keys(x, n, grid_host, ncell_host, keys, s);
        if (st != MDKK_OK) return st;
        return mdkk_bucket_sort(ctx, keys, n, ncell, cell_start, cell_atoms, s);
    }
    int* cnt = static_cast<int*>(mdkk::scratch(ctx, sizeof(int) * ((size_t)ncell + 1)));
    if (!cnt) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "sort scratch");
    cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)ncell + 1), s);
    k_cell_keys_count<<<mdkk::grid_for(n, 256), 256, 0, s>>>(x, n, mdkk::make_grid(grid_host, ncell_host), keys,
                                                             cnt);
    MDKK_CHECK_LAUNCH("k_cell_keys_count");
    return mdkk::bucket_sort_counted(ctx, keys, n, ncell, cnt, cell_start, cell_atoms, s);
}

// Owning brick: floor(pos / L * grid) clipped (mdkk/domain.py:89-95).
__global__ void k_rank_keys(const double* __restrict__ x, int n, double Lx, double Ly, double Lz, int gx,
                            int gy, int gz, int* __restrict__ key) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double4 p = mdkk::ld4(x, i);
    int cx = mdkk::clampi((int)floor(p.x / Lx * (double)gx), gx);
    int cy = mdkk::clampi((int)floor(p.y / Ly * (double)gy), gy);
    int cz = mdkk::clampi((int)floor(p.z / Lz * (double)gz), gz);
    key[i] = (cx * gy + cy) * gz + cz;
}

__global__ void k_cell_positions(const double* __restrict__ x, const int* __restrict__ cell_atoms, int n,
                                 float4* __restrict__ xs) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int j = cell_atoms[s];
    const double4 p = mdkk::ld4(x, j);
    xs[s] = make_float4((float)p.x, (float)p.y, (float)p.z, __int_as_float(j));   // .w = the row
}

// Merged cell lists (mdkk_bin_merge), eight lanes per cell: cell_start[c] = owned_start[c] +
// ghost_start[c]; the cell's owned rows (rows owned_start[c] .. owned_start[c+1] of the
// cell-sorted brick) then its ghost rows (n_local + ghost_order[...]) -- exactly the
// bin_atoms order over all rows (owned then ghost rows per cell, each ascending).
__global__ void k_merge_cells(const int* __restrict__ owned_start, const int* __restrict__ ghost_start,
                              const int* __restrict__ ghost_order, int ncell, int n_local, int n_total,
                              int* __restrict__ cell_start, int* __restrict__ cell_atoms) {
    // eight lanes per cell (cells hold ~20 rows: a warp per cell left most lanes idle and
    // the kernel latency bound on one cell's loads per warp)
    constexpr int G = 8;
    const int c = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) / G);
    const int sl = threadIdx.x & (G - 1);
    if (c >= ncell) return;
    const int os = owned_start[c], no = owned_start[c + 1] - os;
    const int gs = ghost_start[c], ng = ghost_start[c + 1] - gs;
    const int b = os + gs;
    if (sl == 0) {
        cell_start[c] = b;
        if (c == ncell - 1) cell_start[ncell] = n_total;
    }
    for (int t = sl; t < no; t += G) cell_atoms[b + t] = os + t;
    for (int t = sl; t < ng; t += G) cell_atoms[b + no + t] = n_local + ghost_order[gs + t];
}

__device__ __forceinline__ bool lex_zyx_less(double ax, double ay, double az, double bx, double by, double bz) {
    // mdkk/neighbor.py:163-166: z, then y, then x
    return (az < bz) || (az == bz && (ay < by || (ay == by && ax < bx)));
}

// Packed FP32 pair arithmetic (sm_100 FADD2 / FMUL2 / FFMA2): r^2 of two
// staged candidates against one atom in 6 instructions.
__device__ __forceinline__ unsigned long long f32x2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void r2_pair(const float* px, const float* py, const float* pz, unsigned long long xi2,
                                        unsigned long long yi2, unsigned long long zi2, float& r0, float& r1) {
    const unsigned long long x = *reinterpret_cast<const unsigned long long*>(px);
    const unsigned long long y = *reinterpret_cast<const unsigned long long*>(py);
    const unsigned long long z = *reinterpret_cast<const unsigned long long*>(pz);
    unsigned long long dx, dy, dz, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(x), "l"(xi2));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(y), "l"(yi2));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(z), "l"(zi2));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(dx), "l"(dx));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(dy), "l"(dy), "l"(r));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(dz), "l"(dz), "l"(r));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r0), "=f"(r1) : "l"(r));
}

// the same on register operands (an LDS.128 of a pair-interleaved union entry
// already holds (x0, x1) and (y0, y1) as register pairs)
__device__ __forceinline__ void r2_pair_v(float x0, float x1, float y0, float y1, float z0, float z1,
                                          unsigned long long xi2, unsigned long long yi2, unsigned long long zi2,
                                          float& r0, float& r1) {
    const unsigned long long x = f32x2(x0, x1), y = f32x2(y0, y1), z = f32x2(z0, z1);
    unsigned long long dx, dy, dz, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(x), "l"(xi2));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(y), "l"(yi2));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(z), "l"(zi2));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(dx), "l"(dx));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(dy), "l"(dy), "l"(r));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(dz), "l"(dz), "l"(r));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r0), "=f"(r1) : "l"(r));
}

constexpr int kWarps = 4;
constexpr int kUnion = 1024;  // candidate indices per cluster in shared memory (4 KB per warp)
constexpr int kChunk = 64;    // candidate positions staged per pass (1.5 KB per warp)

// One warp per 32-atom cluster of cell-sorted owned rows.  The union pass
// collects every row within bc of the cluster's bounding box (a superset of
// each lane's partners); the scan stages union positions in shared memory 64
// at a time (4 independent loads in flight per lane) and every lane tests
// each staged candidate against its own atom (broadcast reads).
template <int STYLE, bool NEWTON>
__global__ void __launch_bounds__(kWarps * 32) k_nbr_build(
    const double* __restrict__ x, int n_local, Grid g, const int* __restrict__ cell_start,
    const int* __restrict__ cell_atoms, const int64_t* __restrict__ gid, const int32_t* __restrict__ owner_rank,
    int my_rank, double bc, double bc2, int cap, int* __restrict__ table, int* __restrict__ counts,
    int* __restrict__ max_count, const float4* __restrict__ xs) {
    __shared__ int s_union[kWarps][kUnion];
    __shared__ double s_pos[kWarps][3][kChunk];
    // cluster-relative FP32 coordinates, SoA: an aligned float2 = two candidates for the packed
    // FFMA2/FADD2 prefilter (one broadcast LDS.64 per coordinate and candidate pair)
    __shared__ __align__(16) float s_rel[kWarps][3][kChunk];
    __shared__ int64_t s_gid[STYLE == 1 ? kWarps : 1][kChunk];      // half lists: the style predicate's
    __shared__ int s_rank[(STYLE == 1 && NEWTON) ? kWarps : 1][kChunk];  // gids / owner ranks, staged
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x * kWarps + w;
    const int ncl = (n_local + 31) >> 5;
    if (c >= ncl) return;
    int* su = s_union[w];
    double* spx = s_pos[w][0];
    double* spy = s_pos[w][1];
    double* spz = s_pos[w][2];
    float* sfx = s_rel[w][0];
    float* sfy = s_rel[w][1];
    float* sfz = s_rel[w][2];
    int64_t* sgid = s_gid[STYLE == 1 ? w : 0];
    int* srk = s_rank[(STYLE == 1 && NEWTON) ? w : 0];
    const int i = c * 32 + lane;
    const bool valid = i < n_local;
    const double4 xi = mdkk::ld4(x, valid ? i : c * 32);
    // 1. cluster bounding box and the cells it can reach
    const double bmin_x = mdkk::warp_min_d(xi.x), bmax_x = mdkk::warp_max(xi.x);
    const double bmin_y = mdkk::warp_min_d(xi.y), bmax_y = mdkk::warp_max(xi.y);
    const double bmin_z = mdkk::warp_min_d(xi.z), bmax_z = mdkk::warp_max(xi.z);
    const int3 clo = mdkk::cell_of(g, bmin_x - bc, bmin_y - bc, bmin_z - bc);
    const int3 chi = mdkk::cell_of(g, bmax_x + bc, bmax_y + bc, bmax_z + bc);
    const double ccx = 0.5 * (bmin_x + bmax_x), ccy = 0.5 * (bmin_y + bmax_y), ccz = 0.5 * (bmin_z + bmax_z);
    const double hwx = 0.5 * (bmax_x - bmin_x), hwy = 0.5 * (bmax_y - bmin_y), hwz = 0.5 * (bmax_z - bmin_z);
    // FP32 union test: coordinates carry <= 1 ulp of the largest |coordinate| each (the
    // copy, the center); the radius is widened by 16 such ulps (+ 1e-5 bc) so the union
    // stays a superset of every member's partners
    const float ccxf = (float)ccx, ccyf = (float)ccy, cczf = (float)ccz;
    const float hwxf = (float)hwx, hwyf = (float)hwy, hwzf = (float)hwz;
    const double ext = fmax(fmax(fmax(fabs(bmin_x), fabs(bmax_x)), fmax(fabs(bmin_y), fabs(bmax_y))),
                            fmax(fabs(bmin_z), fabs(bmax_z))) + bc;
    const double ru = bc * (1.0 + 1e-5) + 16.0 * 1.2e-7 * ext;
    const float ru2f = (float)(ru * ru);
    // 2. union of candidate rows
    int m = 0;
    // the z-run bounds of the first 32 (cx, cy) columns are loaded up front, one per
    // lane, so the runs' row loads do not wait on a cell_start round trip each
    const int ny = chi.y - clo.y + 1, nrun = (chi.x - clo.x + 1) * ny;
    int run_s0 = 0, run_s1 = 0;
    if (lane < nrun) {
        const int2 kr = mdkk::zrun_keys(g, clo.x + lane / ny, clo.y + lane % ny, clo.z, chi.z);
        run_s0 = cell_start[kr.x];
        run_s1 = cell_start[kr.y + 1];
    }
    for (int cx = clo.x; cx <= chi.x; ++cx) {
        for (int cy = clo.y; cy <= chi.y; ++cy) {
            const int r = (cx - clo.x) * ny + (cy - clo.y);
            int s0 = __shfl_sync(0xffffffffu, run_s0, r & 31), s1 = __shfl_sync(0xffffffffu, run_s1, r & 31);
            if (r >= 32) {
                const int2 kr = mdkk::zrun_keys(g, cx, cy, clo.z, chi.z);
                s0 = cell_start[kr.x];
                s1 = cell_start[kr.y + 1];
            }
            // two 32-row batches per pass: both batches' index and position loads are in
            // flight together (the pass is latency bound); union order is unchanged
            for (int base = s0; base < s1; base += 64) {
                const int sa = base + lane, sb = base + 32 + lane;
                const int ja = sa < s1 ? cell_atoms[sa] : -1;
                const int jb = sb < s1 ? cell_atoms[sb] : -1;
                // cell-ordered FP32 copies: coalesced, and independent of the index loads
                const float4 pa = xs[sa < s1 ? sa : s0], pb = xs[sb < s1 ? sb : s0];
                // distance to the bbox in FP32 against a widened radius (a superset
                // filter: every member is re-tested exactly below)
                auto near = [&](const float4& p) {
                    float dx = fabsf(p.x - ccxf) - hwxf, dy = fabsf(p.y - ccyf) - hwyf, dz = fabsf(p.z - cczf) - hwzf;
                    dx = dx > 0.f ? dx : 0.f;
                    dy = dy > 0.f ? dy : 0.f;
                    dz = dz > 0.f ? dz : 0.f;
                    return dx * dx + dy * dy + dz * dz < ru2f;
                };
                const bool ka = ja >= 0 && near(pa), kb = jb >= 0 && near(pb);
                const unsigned ma = __ballot_sync(0xffffffffu, ka);
                const int posa = m + __popc(ma & ((1u << lane) - 1u));
                if (ka && posa < kUnion) su[posa] = ja;
                m += __popc(ma);
                const unsigned mb = __ballot_sync(0xffffffffu, kb);
                const int posb = m + __popc(mb & ((1u << lane) - 1u));
                if (kb && posb < kUnion) su[posb] = jb;
                m += __popc(mb);
            }
        }
    }
    __syncwarp();
    // 3. per-lane test: FP32 prefilter on cluster-relative coordinates (rejects
    //    ~85% of candidates at twice the FP64 rate), then the exact FP64 test
    //    (strict r^2 < bc^2, reference rounding) + style predicate.
    // invalid lanes sit at -1e18 and padded candidates at +1e18: no FP32 hit, no checks
    const float fxi = valid ? (float)(xi.x - ccx) : -1e18f, fyi = valid ? (float)(xi.y - ccy) : -1e18f;
    const float fzi = valid ? (float)(xi.z - ccz) : -1e18f;
    const unsigned long long fxi2 = f32x2(fxi, fxi), fyi2 = f32x2(fyi, fyi), fzi2 = f32x2(fzi, fzi);
    // margin >> FP32 rounding: |r2_f - r2| <~ 6 eps_f D^2 with D the farthest cluster-relative coordinate
    const double hx = 0.5 * (bmax_x - bmin_x) + bc, hy = 0.5 * (bmax_y - bmin_y) + bc, hz = 0.5 * (bmax_z - bmin_z) + bc;
    const float bc2f = (float)(bc2 * (1.0 + 1e-4) + 4e-6 * (hx * hx + hy * hy + hz * hz));
    const float lo2f = (float)(bc2 * (1.0 - 1e-4) - 4e-6 * (hx * hx + hy * hy + hz * hz));  // certainly inside
    int cnt = 0;
    const int64_t gi = (STYLE == 1 && valid) ? gid[i] : 0;
    int* trow = table + ((long long)c * cap) * 32 + lane;
    // jgid / jrank: the candidate's global id and owner rank (staged in shared memory
    // for the union scan; read from global memory on the overflow path)
    auto visit = [&](int j, double px, double py, double pz, int64_t jgid, int jrank) {
        if (!valid || j == i) return;
        const double r2 = mdkk::r2_exact(px - xi.x, py - xi.y, pz - xi.z);
        if (!(r2 < bc2)) return;
        if (STYLE == 1) {
            bool keep;
            if (j < n_local) {
                keep = gi < jgid;
            } else if (NEWTON) {
                const int orank = jrank;
                keep = orank > my_rank || (orank == my_rank && lex_zyx_less(xi.x, xi.y, xi.z, px, py, pz));
            } else {
                keep = true;
            }
            if (!keep) return;
        }
        if (cnt < cap) trow[(long long)cnt * 32] = j;
        ++cnt;
    };
    if (m <= kUnion) {
        for (int u0 = 0; u0 < m; u0 += kChunk) {
            const int cn = min(kChunk, m - u0);
            for (int t = lane; t < cn; t += 32) {
                const double4 p = mdkk::ld4(x, su[u0 + t]);
                spx[t] = p.x;
                spy[t] = p.y;
                spz[t] = p.z;
                sfx[t] = (float)(p.x - ccx);
                sfy[t] = (float)(p.y - ccy);
                sfz[t] = (float)(p.z - ccz);
                if (STYLE == 1) {
                    const int j = su[u0 + t];
                    sgid[t] = gid[j];
                    if (NEWTON) srk[t] = owner_rank[j];
                }
            }
            for (int t = cn + lane; t < ((cn + 31) & ~31); t += 32) {   // pad to whole groups of 32
                sfx[t] = 1e18f;
                sfy[t] = 1e18f;
                sfz[t] = 1e18f;
            }
            __syncwarp();
            // branch-free prefilter into a per-lane bit mask, then each lane visits only
            // its own survivors (in candidate order): the warp runs max-popcount exact
            // tests per chunk instead of one divergent test per candidate
            for (int h0 = 0; h0 < cn; h0 += 32) {   // 32 candidates per mask: compile-time bit positions
                unsigned bits = 0u;
                const int lim = cn - h0;
                if (STYLE == 0) {
                    // full list: two-sided FP32 test.  Certain members are stored right here,
                    // branch-free (predicated stores in candidate order: no per-lane bit loops,
                    // whose trip count is the warp's max popcount); only the thin shell around
                    // bc goes to the exact FP64 test below.  Overflowing lanes keep counting
                    // and overwrite their last row (the table is rebuilt with the grown cap).
#pragma unroll
                    for (int t = 0; t < 32; t += 2) {   // pads sit at +1e18: never hits
                        float r0, r1;
                        r2_pair(sfx + h0 + t, sfy + h0 + t, sfz + h0 + t, fxi2, fyi2, fzi2, r0, r1);
                        const int2 jj = *reinterpret_cast<const int2*>(su + u0 + h0 + t);
                        const bool in0 = r0 < lo2f, in1 = r1 < lo2f;
                        if (in0 && jj.x != i) {
                            trow[(long long)min(cnt, cap - 1) * 32] = jj.x;
                            ++cnt;
                        }
                        if (in1 && jj.y != i) {
                            trow[(long long)min(cnt, cap - 1) * 32] = jj.y;
                            ++cnt;
                        }
                        bits |= ((!in0 && r0 < bc2f) ? (1u << t) : 0u) | ((!in1 && r1 < bc2f) ? (2u << t) : 0u);
                    }
                } else {
                    // half lists: certain members that are owned rows only need the gid
                    // rule (mdkk/neighbor.py:146-150; gi < gj also excludes i itself) and
                    // are stored here, branch-free; ghosts (owner-rank / zyx rules) and the
                    // shell take the exact path below
#pragma unroll
                    for (int t = 0; t < 32; t += 2) {   // pads sit at +1e18: never hits
                        float r0, r1;
                        r2_pair(sfx + h0 + t, sfy + h0 + t, sfz + h0 + t, fxi2, fyi2, fzi2, r0, r1);
                        const int2 jj = *reinterpret_cast<const int2*>(su + u0 + h0 + t);
                        const bool c0 = r0 < lo2f && jj.x < n_local, c1 = r1 < lo2f && jj.y < n_local;
                        if (c0 && gi < sgid[h0 + t]) {
                            trow[(long long)min(cnt, cap - 1) * 32] = jj.x;
                            ++cnt;
                        }
                        if (c1 && gi < sgid[h0 + t + 1]) {
                            trow[(long long)min(cnt, cap - 1) * 32] = jj.y;
                            ++cnt;
                        }
                        bits |= ((!c0 && r0 < bc2f) ? (1u << t) : 0u) | ((!c1 && r1 < bc2f) ? (2u << t) : 0u);
                    }
                }
                if (lim < 32) bits &= (1u << lim) - 1u;
                while (bits) {
                    const int t = h0 + __ffs(bits) - 1;
                    bits &= bits - 1u;
                    visit(su[u0 + t], spx[t], spy[t], spz[t], STYLE == 1 ? sgid[t] : 0,
                          (STYLE == 1 && NEWTON) ? srk[t] : 0);
                }
            }
            __syncwarp();
        }
    } else {  // union overflow (pathological density): scan the raw cell range instead
        for (int cx = clo.x; cx <= chi.x; ++cx)
            for (int cy = clo.y; cy <= chi.y; ++cy) {
                const int2 kr = mdkk::zrun_keys(g, cx, cy, clo.z, chi.z);
                const int s1 = cell_start[kr.y + 1];
                for (int s = cell_start[kr.x]; s < s1; ++s) {
                    const int j = cell_atoms[s];
                    const double4 p = mdkk::ld4(x, j);
                    visit(j, p.x, p.y, p.z, STYLE == 1 ? gid[j] : 0,
                          (STYLE == 1 && NEWTON && j >= n_local) ? owner_rank[j] : 0);
                }
            }
    }
    if (valid) counts[i] = cnt;
    int mc = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    if (lane == 0 && mc > 0) atomicMax(max_count, mc);
}

// ---------------------------------------------------------------------------
// Full-list build (streaming): the cluster / union scheme of k_nbr_build with its
// two stalls removed (half lists keep k_nbr_build: their ghost-partner rules need
// the staged gids / owner ranks).
//  * The cell rows stream through a two-deep software pipeline of 64-row
//    batches (the next batch's loads are in flight while the current one is
//    filtered and tested), reading only the cell-ordered FP32 copy xs (.w = the
//    row), so no load waits on another.
//  * Union members go to a 128-member ring in shared memory with their FP32
//    cluster-relative coordinates and row (16 B, pair-interleaved: one LDS.128
//    per coordinate pair); every full 32-member block is tested as soon as it
//    exists, so the per-lane test overlaps the union scan and shared memory per
//    warp stays at 2 KB (occupancy is set by registers).  FP64 positions are
//    read only for the thin shell |r^2 - bc^2| < M that FP32 cannot decide.
//  * The cluster's own rows are not union members: a 32-step shuffle pass tests
//    them first, so the union test needs no j != i check.
// Table rows: own-cluster partners first, then union members in union (cell)
// order, each 32-member block's certain partners before its exactly-tested shell.
constexpr int kW2 = 4;       // clusters (warps) per CTA
constexpr int kRing = 128;   // union ring per warp (a block of 32 + two batches of 32 pending)

struct __align__(16) UxY {   // union members 2p, 2p+1: x0, x1, y0, y1
    float x0, x1, y0, y1;
};
struct __align__(16) UzJ {   // z0, z1, row0, row1
    float z0, z1;
    int j0, j1;
};

__global__ void __launch_bounds__(kW2 * 32, 1) k_nbr_build_full(
    const double* __restrict__ x, int n_local, Grid g, const int* __restrict__ cell_start, double bc, double bc2,
    int cap, int* __restrict__ table, int* __restrict__ counts, int* __restrict__ max_count,
    const float4* __restrict__ xs) {
    __shared__ UxY s_ra[kW2][kRing / 2];
    __shared__ UzJ s_rb[kW2][kRing / 2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    UxY* sa = s_ra[w];
    UzJ* sb = s_rb[w];
    float* fa = reinterpret_cast<float*>(sa);
    float* fb = reinterpret_cast<float*>(sb);
    int* jb = reinterpret_cast<int*>(sb);
    const int c = blockIdx.x * kW2 + w;
    const int ncl = (n_local + 31) >> 5;
    if (c >= ncl) return;
    const int c0 = c * 32;
    const int nown = min(32, n_local - c0);   // the cluster's owned rows [c0, c0 + nown)
    const int i = c0 + lane;
    const bool valid = lane < nown;
    const double4 xi = mdkk::ld4(x, valid ? i : c0);
    // 1. cluster bounding box, the cells it can reach, FP32 frame at its center
    const double bmin_x = mdkk::warp_min_d(xi.x), bmax_x = mdkk::warp_max(xi.x);
    const double bmin_y = mdkk::warp_min_d(xi.y), bmax_y = mdkk::warp_max(xi.y);
    const double bmin_z = mdkk::warp_min_d(xi.z), bmax_z = mdkk::warp_max(xi.z);
    const int3 clo = mdkk::cell_of(g, bmin_x - bc, bmin_y - bc, bmin_z - bc);
    const int3 chi = mdkk::cell_of(g, bmax_x + bc, bmax_y + bc, bmax_z + bc);
    const double ccx = 0.5 * (bmin_x + bmax_x), ccy = 0.5 * (bmin_y + bmax_y), ccz = 0.5 * (bmin_z + bmax_z);
    const double hwx = 0.5 * (bmax_x - bmin_x), hwy = 0.5 * (bmax_y - bmin_y), hwz = 0.5 * (bmax_z - bmin_z);
    const float ccxf = (float)ccx, ccyf = (float)ccy, cczf = (float)ccz;
    const float hwxf = (float)hwx, hwyf = (float)hwy, hwzf = (float)hwz;
    const double ext = fmax(fmax(fmax(fabs(bmin_x), fabs(bmax_x)), fmax(fabs(bmin_y), fabs(bmax_y))),
                            fmax(fabs(bmin_z), fabs(bmax_z))) + bc;
    const double ru = bc * (1.0 + 1e-5) + 16.0 * 1.2e-7 * ext;
    const float ru2f = (float)(ru * ru);
    // FP32 decision margins.  A relative coordinate u = fl(fl(x) - fl(cc)) is within
    // 2^-24 (2 ext + D) of x - cc (D >= |u|); a packed difference within
    // e_d = 2^-23 (2 ext + D) + 2^-23 D; r^2 (FMA chain) within
    // 2 sqrt(3) |d| e_d + 3 e_d^2 + 2e-7 r^2.  M doubles that bound.
    const double dmax = fmax(fmax(hwx, hwy), hwz) * 2.0 + ru;
    const double e_d = 1.2e-7 * (2.0 * ext + 2.0 * dmax);
    const double rmax = sqrt(bc2) * 1.01;
    const double M = 2.0 * (3.4642 * rmax * e_d + 3.0 * e_d * e_d + 2e-7 * bc2) + 1e-5 * bc2;
    const float lo2f = (float)(bc2 - M), bc2f = (float)(bc2 + M);
    const float fxi = valid ? (float)xi.x - ccxf : -1e18f, fyi = valid ? (float)xi.y - ccyf : -1e18f;
    const float fzi = valid ? (float)xi.z - cczf : -1e18f;
    const unsigned long long fxi2 = f32x2(fxi, fxi), fyi2 = f32x2(fyi, fyi), fzi2 = f32x2(fzi, fzi);
    // exact FP64 test (strict r^2 < bc^2 in the reference's rounding, mdkk/neighbor.py:121-126)
    // for the candidates FP32 cannot decide
    int cnt = 0;
    int* const trow = table + ((long long)c * cap) * 32 + lane;
    auto visit = [&](int j) {
        if (!valid || j == i) return;
        const double4 p = mdkk::ld4(x, j);
        const double r2 = mdkk::r2_exact(p.x - xi.x, p.y - xi.y, p.z - xi.z);
        if (!(r2 < bc2)) return;
        trow[(long long)min(cnt, cap - 1) * 32] = j;
        ++cnt;
    };
    // 2. the cluster's own rows, broadcast by shuffles
    for (int k = 0; k < 32; ++k) {
        const float dx = __shfl_sync(0xffffffffu, fxi, k) - fxi, dy = __shfl_sync(0xffffffffu, fyi, k) - fyi;
        const float dz = __shfl_sync(0xffffffffu, fzi, k) - fzi;
        const float r2f = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        const bool own = valid && k < nown && k != lane;
        const bool cert = own && r2f < lo2f;
        if (cert) {
            trow[(long long)min(cnt, cap - 1) * 32] = c0 + k;
            ++cnt;
        }
        if (own && !cert && r2f < bc2f) visit(c0 + k);
    }
    // 3. stream the cell rows within bc of the bbox through the ring, testing every full block
    int m = 0, done = 0;   // members put / tested
    auto put = [&](const float4& p, bool keep) {
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int pos = (m + __popc(mk & ((1u << lane) - 1u))) & (kRing - 1);
            const int o = (pos >> 1) * 4 + (pos & 1);
            fa[o] = p.x - ccxf;
            fa[o + 2] = p.y - ccyf;
            fb[o] = p.z - cczf;
            jb[o + 2] = __float_as_int(p.w);
        }
        m += __popc(mk);
    };
    auto near = [&](const float4& p) {
        float dx = fabsf(p.x - ccxf) - hwxf, dy = fabsf(p.y - ccyf) - hwyf, dz = fabsf(p.z - cczf) - hwzf;
        dx = dx > 0.f ? dx : 0.f;
        dy = dy > 0.f ? dy : 0.f;
        dz = dz > 0.f ? dz : 0.f;
        return dx * dx + dy * dy + dz * dz < ru2f;
    };
    auto test = [&](const float4& p, bool in_range) {
        return in_range && (unsigned)(__float_as_int(p.w) - c0) >= (unsigned)nown && near(p);
    };
    // one 32-member block at ring offset h (certain partners: branch-free predicated
    // stores in member order; the shell is flagged and tested exactly after the block)
    auto run_block = [&](int h) {
        __syncwarp();
        unsigned bits = 0u;
        const UxY* ra = sa + (h >> 1);   // a block never wraps the ring (h is a multiple of 32)
        const UzJ* rb = sb + (h >> 1);
        auto body = [&](auto roomy_tag) {
            constexpr bool kRoomy = decltype(roomy_tag)::value;
            int off = cnt * 32;   // roomy: cnt + 32 <= cap
#pragma unroll
            for (int t = 0; t < 32; t += 2) {
                const UxY a = ra[t >> 1];
                const UzJ b = rb[t >> 1];
                float r0, r1;
                r2_pair_v(a.x0, a.x1, a.y0, a.y1, b.z0, b.z1, fxi2, fyi2, fzi2, r0, r1);
                const bool k0 = r0 < lo2f, k1 = r1 < lo2f;
                const bool e0 = r0 < bc2f && !k0, e1 = r1 < bc2f && !k1;
                if (kRoomy) {
                    if (k0) {
                        trow[off] = b.j0;
                        off += 32;
                    }
                    if (k1) {
                        trow[off] = b.j1;
                        off += 32;
                    }
                } else {
                    if (k0) {
                        trow[(long long)min(cnt, cap - 1) * 32] = b.j0;
                        ++cnt;
                    }
                    if (k1) {
                        trow[(long long)min(cnt, cap - 1) * 32] = b.j1;
                        ++cnt;
                    }
                }
                bits |= (e0 ? (1u << t) : 0u) | (e1 ? (2u << t) : 0u);
            }
            if (kRoomy) cnt = off >> 5;
        };
        if (__all_sync(0xffffffffu, cnt + 32 <= cap))
            body(std::true_type{});
        else
            body(std::false_type{});
        while (bits) {
            const int t = h + __ffs(bits) - 1;
            bits &= bits - 1u;
            visit(jb[(t >> 1) * 4 + 2 + (t & 1)]);
        }
        __syncwarp();   // the ring slots are refilled next
    };
    const int ny = chi.y - clo.y + 1, nrun = (chi.x - clo.x + 1) * ny;
    int run_s0 = 0, run_s1 = 0;
    if (lane < nrun) {
        const int2 kr = mdkk::zrun_keys(g, clo.x + lane / ny, clo.y + lane % ny, clo.z, chi.z);
        run_s0 = cell_start[kr.x];
        run_s1 = cell_start[kr.y + 1];
    }
    int r = -1, bs = 0, be = 0;
    auto advance = [&]() -> bool {   // to the next 64-row batch (warp-uniform state)
        bs += 64;
        while (bs >= be) {
            if (++r >= nrun) return false;
            if (r < 32) {
                bs = __shfl_sync(0xffffffffu, run_s0, r);
                be = __shfl_sync(0xffffffffu, run_s1, r);
            } else {
                const int2 kr = mdkk::zrun_keys(g, clo.x + r / ny, clo.y + r % ny, clo.z, chi.z);
                bs = cell_start[kr.x];
                be = cell_start[kr.y + 1];
            }
        }
        return true;
    };
    {
        float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pb = pa;
        int n_cur = 0;
        if (advance()) {
            pa = xs[min(bs + lane, be - 1)];
            pb = xs[min(bs + 32 + lane, be - 1)];
            n_cur = be - bs;
        }
        bool more = n_cur > 0 && advance();
        while (n_cur > 0) {
            float4 qa = pa, qb = pb;
            int n_next = 0;
            if (more) {   // the next batch's loads go out before this batch is filtered and tested
                qa = xs[min(bs + lane, be - 1)];
                qb = xs[min(bs + 32 + lane, be - 1)];
                n_next = be - bs;
                more = advance();
            }
            put(pa, test(pa, lane < n_cur));
            put(pb, test(pb, lane + 32 < n_cur));
            while (m - done >= 32) {
                run_block(done & (kRing - 1));
                done += 32;
            }
            pa = qa;
            pb = qb;
            n_cur = n_next;
        }
    }
    if (m > done) {   // the last partial block, padded (pads sit at +1e18: never a hit)
        const int pos = (m + lane) & (kRing - 1);
        if (m + lane < done + 32) {
            const int o = (pos >> 1) * 4 + (pos & 1);
            fa[o] = 1e18f;
            fa[o + 2] = 1e18f;
            fb[o] = 1e18f;
            jb[o + 2] = -1;
        }
        run_block(done & (kRing - 1));
    }
    if (valid) counts[i] = cnt;
    int mc = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    if (lane == 0 && mc > 0) atomicMax(max_count, mc);
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

// Geometric row order for the cluster-blocked table: each row's entries sorted by the
// partner's displacement (dz, dy, dx) = x_j - x_i, the reference's NeighborMap order
// (mdkk/snap/compute.py:66-104: lexsort (row, dz, dy, dx)), so order-dependent sums
// over a row (compute_ui's U accumulation) do not depend on atom labels.
__global__ void k_geo_order(const double* __restrict__ x, int n_local, int cap, int* __restrict__ table,
                            const int* __restrict__ counts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    const int n = min(counts[i], cap);
    int* row = table + ((long long)(i >> 5) * cap) * 32 + (i & 31);
    const double4 xi = mdkk::ld4(x, i);
    auto less = [&](int a, int b) {
        const double4 pa = mdkk::ld4(x, a), pb = mdkk::ld4(x, b);
        const double az = pa.z - xi.z, bz = pb.z - xi.z;
        if (az != bz) return az < bz;
        const double ay = pa.y - xi.y, by = pb.y - xi.y;
        if (ay != by) return ay < by;
        return (pa.x - xi.x) < (pb.x - xi.x);
    };
    for (int k = 1; k < n; ++k) {
        const int v = row[(long long)k * 32];
        int m = k - 1;
        while (m >= 0 && less(v, row[(long long)m * 32])) {
            row[(long long)(m + 1) * 32] = row[(long long)m * 32];
            --m;
        }
        row[(long long)(m + 1) * 32] = v;
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

}  // namespace

extern "C" {

int mdkk_cell_keys(const double* x, int n, const double* grid_host, const int* ncell_host, int* keys,
                   void* stream) {
    if (n < 0 || !grid_host || !ncell_host) return MDKK_E_ARG;
    if (n == 0) return MDKK_OK;
    Grid g = mdkk::make_grid(grid_host, ncell_host);
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
    return bin_rows(ctx, x, n, grid_host, ncell_host, (int)ncell, keys, cell_start, cell_atoms,
                    mdkk::as_stream(stream));
}

int mdkk_nbr_build(mdkk_ctx* ctx, const double* x, int n_local, int n_total, const double* grid_host,
                   const int* ncell_host, const int* cell_start, const int* cell_atoms, const int64_t* gid,
                   const int32_t* owner_rank, int my_rank, double bc, int style, int newton, int cap, int* table,
                   int* counts, int* max_count, void* stream) {
    if (!ctx || n_local < 0 || n_total < n_local || cap < 1 || (style != 0 && style != 1)) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    Grid g = mdkk::make_grid(grid_host, ncell_host);
    cudaStream_t s = mdkk::as_stream(stream);
    // FP32 positions in cell order for the union pass (coalesced instead of gathered)
    float4* xs = static_cast<float4*>(mdkk::scratch(ctx, sizeof(float4) * (size_t)std::max(n_total, 1)));
    if (!xs) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    k_cell_positions<<<mdkk::grid_for(n_total, 256), 256, 0, s>>>(x, cell_atoms, n_total, xs);
    MDKK_CHECK_LAUNCH("k_cell_positions");
    const int ncl = (n_local + 31) / 32;
    const int nb = (ncl + kWarps - 1) / kWarps;
    const double bc2 = bc * bc;
    static const bool v1 = getenv("MDKK_NB_V1") && getenv("MDKK_NB_V1")[0] == '1';   // A/B switch
    if (style == 0 && !v1) {
        k_nbr_build_full<<<(ncl + kW2 - 1) / kW2, kW2 * 32, 0, s>>>(x, n_local, g, cell_start, bc, bc2, cap, table,
                                                                    counts, max_count, xs);
        MDKK_CHECK_LAUNCH("k_nbr_build_full");
        return MDKK_OK;
    }
    if (style == 0)
        k_nbr_build<0, false><<<nb, kWarps * 32, 0, s>>>(x, n_local, g, cell_start, cell_atoms, gid, owner_rank,
                                                         my_rank, bc, bc2, cap, table, counts, max_count, xs);
    else if (newton)
        k_nbr_build<1, true><<<nb, kWarps * 32, 0, s>>>(x, n_local, g, cell_start, cell_atoms, gid, owner_rank,
                                                        my_rank, bc, bc2, cap, table, counts, max_count, xs);
    else
        k_nbr_build<1, false><<<nb, kWarps * 32, 0, s>>>(x, n_local, g, cell_start, cell_atoms, gid, owner_rank,
                                                         my_rank, bc, bc2, cap, table, counts, max_count, xs);
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

int mdkk_bin_merge(mdkk_ctx* ctx, const double* x, int n_local, int n_total, const double* grid_host,
                   const int* ncell_host, const int* owned_start, int* keys, int* cell_start, int* cell_atoms,
                   void* stream) {
    if (!ctx || n_local < 0 || n_total < n_local || !grid_host || !ncell_host || !owned_start) return MDKK_E_ARG;
    const long long ncl = (long long)ncell_host[0] * ncell_host[1] * ncell_host[2];
    if (ncl < 1 || ncl >= (1LL << 30)) return MDKK_E_ARG;
    const int ncell = (int)ncl, n_ghost = n_total - n_local;
    Grid g = mdkk::make_grid(grid_host, ncell_host);
    cudaStream_t s = mdkk::as_stream(stream);
    // ghost bins in ctx scratch, after the bucket sort's own counters: [cnt | ghost_start | ghost_order]
    // (the whole arena is requested first, so the sort's smaller request does not move it)
    // (the bucket sort's footprint: ncell + 1 counters, or the few-bucket path's block table)
    const size_t nbk = ((size_t)n_ghost + 255) / 256;
    const size_t sort_words = ncell > 64 ? (size_t)ncell + 1 : 2 * ((size_t)ncell * nbk + 1);
    const size_t cnt_words = (sort_words + 63) & ~(size_t)63;
    int* base = static_cast<int*>(
        mdkk::scratch(ctx, sizeof(int) * (cnt_words + (size_t)ncell + 64 + (size_t)n_ghost + 64)));
    if (!base) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    int* gstart = base + cnt_words;
    int* gord = gstart + ncell + 64;
    // (the sort's counters are the arena's first ncell + 1 words: `base`)
    int st = bin_rows(ctx, x + 4LL * n_local, n_ghost, grid_host, ncell_host, ncell, keys, gstart, gord, s);
    if (st != MDKK_OK) return st;
    // per cell: its owned rows (a contiguous range of the sorted brick) then its ghost rows
    k_merge_cells<<<mdkk::grid_for((long long)ncell * 8, 256), 256, 0, s>>>(owned_start, gstart, gord, ncell,
                                                                              n_local, n_total, cell_start,
                                                                              cell_atoms);
    MDKK_CHECK_LAUNCH("k_merge_cells");
    return MDKK_OK;
}

int mdkk_nbr_geo_order(const double* x, int n_local, int cap, int* table, const int* counts, void* stream) {
    if (n_local < 0 || cap < 1) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    k_geo_order<<<mdkk::grid_for(n_local, 128), 128, 0, mdkk::as_stream(stream)>>>(x, n_local, cap, table, counts);
    MDKK_CHECK_LAUNCH("k_geo_order");
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
