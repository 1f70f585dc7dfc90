// One-rank engine rebuild, selection phase: the device sequence of
// RankedSystem.migrate's single-rank path (mdkk/domain.py:324-334: wrap, then the
// ghost selection of exchange_ghosts, :246-293) issued from one host call.
//
// The rebuild is a chain of ~25 short kernels ahead of one host read-back (the
// ghost totals); issued one ctypes call at a time, the host was slower than the
// device and the GPU idled between launches.  Here the whole chain up to the
// read-back is queued back to back, the velocity / gid gathers go behind the
// totals' copy (device work while the host waits), and the host waits on an
// event for that copy only.
#include "cluster.cuh"

namespace {
cudaEvent_t g_totals_ev[64];   // per device, created lazily

__device__ __forceinline__ double4 wrapped(double4 p, double Lx, double Ly, double Lz) {
    p.x = __dsub_rn(p.x, __dmul_rn(Lx, floor(p.x / Lx)));
    p.y = __dsub_rn(p.y, __dmul_rn(Ly, floor(p.y / Ly)));
    p.z = __dsub_rn(p.z, __dmul_rn(Lz, floor(p.z / Lz)));
    return p;
}


// Wrap (pos - L floor(pos / L) with explicit roundings, as k_wrap / mdkk/domain.py:62)
// and the cell key of the wrapped row (as k_cell_keys), one pass over x (few cells).
__global__ void k_wrap_keys(double* __restrict__ x, int n, double Lx, double Ly, double Lz, mdkk::Grid g,
                            int* __restrict__ key) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 p = wrapped(mdkk::ld4_nc(x, i), Lx, Ly, Lz);
    mdkk::st4(x, i, p);
    const int3 c = mdkk::cell_of(g, p.x, p.y, p.z);
    key[i] = mdkk::cell_key(g, c.x, c.y, c.z);
}

// The many-cell form: the wrapped row's cell key plus the sort's count pass (one atomic per
// distinct key per warp), without writing x back -- the gather below wraps the rows it
// moves, with the same operations, so the sorted positions are bit-identical.
__global__ void k_wrap_keys_count(const double* __restrict__ x, int n, double Lx, double Ly, double Lz,
                                  mdkk::Grid g, int* __restrict__ key, int* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const double4 p = wrapped(mdkk::ld4(x, i), Lx, Ly, Lz);
    const int3 c = mdkk::cell_of(g, p.x, p.y, p.z);
    const int k = mdkk::cell_key(g, c.x, c.y, c.z);
    key[i] = k;
    const unsigned same = __match_any_sync(act, k);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(cnt + k, __popc(same));
}

// The sort's position gather of unwrapped rows, wrapping each; with `ref` it also writes
// the rows into the new lists' skin-test reference (the build-time positions) -- one
// pass over x instead of a later copy.
__global__ void k_gather4_wrap(const double* __restrict__ src, const int* __restrict__ perm, int n, double Lx,
                               double Ly, double Lz, double* __restrict__ dst, double* __restrict__ ref) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 p = wrapped(mdkk::ld4(src, perm[i]), Lx, Ly, Lz);
    mdkk::st4(dst, i, p);
    if (ref) mdkk::st4(ref, i, p);
}

// As k_gather4_wrap for rows x already wrapped in place (the few-cell path).
__global__ void k_gather4_ref(const double* __restrict__ src, const int* __restrict__ perm, int n,
                              double* __restrict__ dst, double* __restrict__ ref) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 p = mdkk::ld4(src, perm[i]);
    mdkk::st4(dst, i, p);
    mdkk::st4(ref, i, p);
}
}

extern "C" {

int mdkk_bucket_sort(mdkk_ctx* ctx, const int* keys, int n, int nbuckets, int* bucket_start, int* order,
                     void* stream);
int mdkk_gather_rows4(const double* src, const int* perm, int n, double* dst, void* stream);
int mdkk_gather_i64(const int64_t* src, const int* perm, int n, int64_t* dst, void* stream);
int mdkk_boundary_rows(mdkk_ctx* ctx, const int* cell_start, const int* ncell_host, int layer, int* rows,
                       int* count, void* stream);
int mdkk_halo_count(mdkk_ctx* ctx, const double* x, int n, const double* combos, int C, int* block_scratch,
                    int* totals, const int* rows, const int* n_dev, void* stream);

int mdkk_rebuild1_select(mdkk_ctx* ctx, double* x, int n, const double* lengths_host, const double* grid_host,
                         const int* ncell_host, int* keys, int* cell_start, int* order, double* x_sorted,
                         const double* v, double* v_sorted, const int64_t* gid, int64_t* gid_sorted, int* brows,
                         int* bcount, const double* combos_dev, int C, int* block_scratch, int* totals,
                         int* totals_host, int* n_ghost_host, double* x_ref, void* stream) {
    if (!ctx || n < 2 || C < 1 || !totals_host || !n_ghost_host || x_sorted == x || v_sorted == v ||
        gid_sorted == gid)
        return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    const long long ncl = (long long)ncell_host[0] * ncell_host[1] * ncell_host[2];
    if (ncl < 1 || ncl > (1LL << 30)) return MDKK_E_ARG;
    const mdkk::Grid g = mdkk::make_grid(grid_host, ncell_host);
    const double Lx = lengths_host[0], Ly = lengths_host[1], Lz = lengths_host[2];
    int st = MDKK_OK;
    if (ncl > mdkk::kSortSmallBuckets) {
        // wrap folded into the key / count pass and the gather (x itself is not rewritten:
        // after the sort it is the spare buffer)
        int* cnt = static_cast<int*>(mdkk::scratch(ctx, sizeof(int) * ((size_t)ncl + 1)));
        if (!cnt) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "sort scratch");
        cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)ncl + 1), s);
        k_wrap_keys_count<<<mdkk::grid_for(n, 256), 256, 0, s>>>(x, n, Lx, Ly, Lz, g, keys, cnt);
        MDKK_CHECK_LAUNCH("k_wrap_keys_count");
        st = mdkk::bucket_sort_counted(ctx, keys, n, (int)ncl, cnt, cell_start, order, s);
        if (st == MDKK_OK) {
            k_gather4_wrap<<<mdkk::grid_for(n, 256), 256, 0, s>>>(x, order, n, Lx, Ly, Lz, x_sorted, x_ref);
            MDKK_CHECK_LAUNCH("k_gather4_wrap");
        }
    } else {
        k_wrap_keys<<<mdkk::grid_for(n, 256), 256, 0, s>>>(x, n, Lx, Ly, Lz, g, keys);
        MDKK_CHECK_LAUNCH("k_wrap_keys");
        st = mdkk_bucket_sort(ctx, keys, n, (int)ncl, cell_start, order, stream);
        if (st == MDKK_OK) {
            if (x_ref) {
                k_gather4_ref<<<mdkk::grid_for(n, 256), 256, 0, s>>>(x, order, n, x_sorted, x_ref);
                MDKK_CHECK_LAUNCH("k_gather4_ref");
            } else {
                st = mdkk_gather_rows4(x, order, n, x_sorted, stream);
            }
        }
    }
    // owned rows are now cell-sorted on the shell grid (cells >= halo wide): only rows within
    // two cell layers of the faces can be selected
    if (st == MDKK_OK) st = mdkk_boundary_rows(ctx, cell_start, ncell_host, 2, brows, bcount, stream);
    if (st == MDKK_OK)
        st = mdkk_halo_count(ctx, x_sorted, n, combos_dev, C, block_scratch, totals, brows, bcount, stream);
    if (st != MDKK_OK) return st;
    cudaEvent_t& ev = g_totals_ev[ctx->device & 63];
    cudaError_t e = cudaSuccess;
    if (!ev) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMemcpyAsync(totals_host, totals, sizeof(int) * (size_t)C, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaEventRecord(ev, s);
    if (e != cudaSuccess) return mdkk::cuda_fail(e, "mdkk_rebuild1_select");
    st = mdkk_gather_rows4(v, order, n, v_sorted, stream);
    if (st == MDKK_OK) st = mdkk_gather_i64(gid, order, n, gid_sorted, stream);
    if (st != MDKK_OK) return st;
    e = cudaEventSynchronize(ev);
    if (e != cudaSuccess) return mdkk::cuda_fail(e, "mdkk_rebuild1_select (totals)");
    long long ng = 0;
    for (int c = 0; c < C; ++c) ng += totals_host[c];
    if (ng > 0x7fffffffLL) {
        mdkk::set_error("mdkk_rebuild1_select: ghost count overflows int");
        return MDKK_E_ARG;
    }
    *n_ghost_host = (int)ng;
    return MDKK_OK;
}

}  // extern "C"
