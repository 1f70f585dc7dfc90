// Hand-written prefix sums and the counting-sort bucket sort (no CUB).
//
// Replaces the reference's stable argsort + bincount + cumsum binning
// (mdkk/neighbor.py:88-96) and the owner partition of migrate
// (mdkk/domain.py:324-334): rows are grouped by an int key, ascending row index
// inside every bucket (the stable order), bucket starts from an exclusive scan.
//
//   many buckets (cells, ~16 rows each): histogram (atomics) -> scan -> scatter
//     through per-bucket atomic cursors -> every bucket re-ordered by row index in
//     registers (one warp per bucket, rank = number of smaller rows): 4 launches;
//   few buckets (rank partitions, <= 64): per-256-row block counts [bucket][block]
//     -> scan -> in-block stable ranks from __match_any_sync + warp prefixes.
//
// exclusive_scan: tile sums -> single-block scan of the tile sums -> tile scans
// with their offsets (three launches, int32 and int64).
#include "common.cuh"

namespace {

constexpr int kScanThreads = 512;
constexpr int kScanPer = 8;
constexpr int kTile = kScanThreads * kScanPer;

// Block-wide exclusive scan of one value per thread; *total gets the block sum.
template <typename T>
__device__ __forceinline__ T block_exclusive(T v, T* total) {
    __shared__ T s_warp[kScanThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
        T t = lane < kScanThreads / 32 ? s_warp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        if (lane < kScanThreads / 32) s_warp[lane] = t;   // inclusive warp prefixes
    }
    __syncthreads();
    const T before = w ? s_warp[w - 1] : T(0);
    *total = s_warp[kScanThreads / 32 - 1];
    __syncthreads();
    return before + incl - v;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const T* __restrict__ in, long long n, T* __restrict__ sums) {
    const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kScanPer;
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k)
        if (base + k < n) s += in[base + k];
    T tot;
    block_exclusive<T>(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// One block: exclusive scan of the tile sums in place, any count.
template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(T* __restrict__ sums, int ntiles) {
    T carry = 0;
    for (int b0 = 0; b0 < ntiles; b0 += kScanThreads) {
        const int k = b0 + threadIdx.x;
        const T v = k < ntiles ? sums[k] : T(0);
        T tot;
        const T ex = block_exclusive<T>(v, &tot);
        if (k < ntiles) sums[k] = carry + ex;
        carry += tot;
    }
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const T* __restrict__ in, T* __restrict__ out,
                                                              long long n, const T* __restrict__ offs) {
    const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kScanPer;
    T v[kScanPer];
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        v[k] = base + k < n ? in[base + k] : T(0);
        s += v[k];
    }
    T tot;
    T run = offs[blockIdx.x] + block_exclusive<T>(s, &tot);
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

template <typename T>
int scan_impl(mdkk_ctx* ctx, const T* in, T* out, long long n, cudaStream_t s) {
    if (n <= 0) return MDKK_OK;
    const long long ntiles = (n + kTile - 1) / kTile;
    if (ntiles > (1LL << 30)) return MDKK_E_ARG;
    T* sums = static_cast<T*>(mdkk::scratch_tail(ctx, sizeof(T) * (size_t)ntiles));
    if (!sums) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scan scratch");
    k_tile_sums<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, sums);
    MDKK_CHECK_LAUNCH("k_tile_sums");
    k_scan_sums<T><<<1, kScanThreads, 0, s>>>(sums, (int)ntiles);
    MDKK_CHECK_LAUNCH("k_scan_sums");
    k_scan_tiles<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, out, n, sums);
    MDKK_CHECK_LAUNCH("k_scan_tiles");
    return MDKK_OK;
}

// ------------------------------------------------------------ many buckets
// Warp-aggregated: the engine's keys are nearly sorted (rows keep the previous cell
// order), so a warp's 32 rows fall in ~2 cells and per-row atomics would serialise on
// the same counters; one atomic per distinct key per warp instead.
__global__ void k_key_count(int n, const int* __restrict__ key, int* __restrict__ counts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const int c = key[i];
    const unsigned same = __match_any_sync(act, c);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(counts + c, __popc(same));
}

__global__ void k_key_scatter(int n, const int* __restrict__ key, const int* __restrict__ start,
                              int* __restrict__ cursor, int* __restrict__ order) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const int c = key[i];
    const int lane = threadIdx.x & 31;
    const unsigned same = __match_any_sync(act, c);
    const int leader = __ffs(same) - 1;
    // the counts count down as the cursors (each warp's run of a bucket lands ascending;
    // the row sort orders the runs)
    const int m = __popc(same);
    int base = 0;
    if (lane == leader) base = atomicSub(cursor + c, m) - m;
    base = __shfl_sync(same, base, leader);
    order[start[c] + base + __popc(same & ((1u << lane) - 1u))] = i;
}

// kRsG lanes per bucket (32 / kRsG buckets per warp): the rows the scatter placed in
// arrival order, re-ordered ascending (rank = how many rows of the bucket are
// smaller; rows are distinct).  A lane holds rows sl, sl + kRsG, ... of its bucket
// (up to 32 rows per bucket); the group walks the bucket once by shuffles.  The
// kernel is latency bound (start -> rows -> stores per bucket): several buckets per
// warp keep that many more loads in flight than a warp per bucket.  Buckets over 32
// rows (rare: cells hold ~18) are insertion-sorted by the group's first lane.
constexpr int kRsG = 8;              // lanes per bucket (8: 24.6 + 11.1 us per rebuild at 2M; 4: 20.2 + 14.2)
constexpr int kRsV = 32 / kRsG;      // rows per lane
__global__ void k_bucket_rowsort(int nbuckets, const int* __restrict__ start, int* __restrict__ order) {
    const int lane = threadIdx.x & 31, sl = lane & (kRsG - 1);
    const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / kRsG;
    int s = 0, len = 0;
    if (b < nbuckets) {
        s = start[b];
        len = start[b + 1] - s;
    }
    const bool grp = len > 1 && len <= 32;
    int v[kRsV], r[kRsV];
#pragma unroll
    for (int q = 0; q < kRsV; ++q) {
        v[q] = (grp && sl + kRsG * q < len) ? order[s + sl + kRsG * q] : 0x7fffffff;
        r[q] = 0;
    }
    int lmax = grp ? len : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    for (int k0 = 0; k0 < lmax; k0 += kRsG) {   // warp-uniform: kRsG rows per register slot
        int src = v[0];
#pragma unroll
        for (int q = 1; q < kRsV; ++q)
            if (k0 / kRsG == q) src = v[q];
#pragma unroll
        for (int t = 0; t < kRsG; ++t) {
            const int u = __shfl_sync(0xffffffffu, src, t, kRsG);
            if (k0 + t < len) {
#pragma unroll
                for (int q = 0; q < kRsV; ++q) r[q] += u < v[q];
            }
        }
    }
    if (grp) {
#pragma unroll
        for (int q = 0; q < kRsV; ++q)
            if (sl + kRsG * q < len) order[s + r[q]] = v[q];
    }
    if (len > 32 && sl == 0) {   // oversized bucket: insertion sort
        for (int k = s + 1; k < s + len; ++k) {
            const int x = order[k];
            int m = k - 1;
            while (m >= s && order[m] > x) {
                order[m + 1] = order[m];
                --m;
            }
            order[m + 1] = x;
        }
    }
}

// ------------------------------------------------------------- few buckets
constexpr int kSmallBuckets = 64;
constexpr int kSmallBlock = 256;

__global__ void __launch_bounds__(kSmallBlock) k_small_count(int n, const int* __restrict__ key, int nbuckets,
                                                              int nblocks, int* __restrict__ table) {
    __shared__ int cnt[kSmallBuckets];
    if (threadIdx.x < kSmallBuckets) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int i = blockIdx.x * kSmallBlock + threadIdx.x;
    if (i < n) atomicAdd(cnt + key[i], 1);
    __syncthreads();
    if (threadIdx.x < nbuckets) table[(long long)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kSmallBlock) k_small_scatter(int n, const int* __restrict__ key, int nbuckets,
                                                                int nblocks, const int* __restrict__ offs,
                                                                int* __restrict__ order, int* __restrict__ start) {
    __shared__ int wcnt[kSmallBlock / 32][kSmallBuckets];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < (kSmallBlock / 32) * kSmallBuckets; t += kSmallBlock) (&wcnt[0][0])[t] = 0;
    __syncthreads();
    const int i = blockIdx.x * kSmallBlock + threadIdx.x;
    const bool valid = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    int k = 0, rank = 0;
    if (valid) {
        k = key[i];
        const unsigned same = __match_any_sync(act, k);
        rank = __popc(same & ((1u << lane) - 1u));
        if (rank == 0) wcnt[w][k] = __popc(same);
    }
    __syncthreads();
    if (threadIdx.x < nbuckets) {   // per-bucket exclusive prefix over the block's warps
        int run = 0;
        for (int q = 0; q < kSmallBlock / 32; ++q) {
            const int c = wcnt[q][threadIdx.x];
            wcnt[q][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
    if (valid) order[offs[(long long)k * nblocks + blockIdx.x] + wcnt[w][k] + rank] = i;
    if (blockIdx.x == 0 && threadIdx.x <= nbuckets)
        start[threadIdx.x] = offs[(long long)threadIdx.x * nblocks];   // offs[nbuckets * nblocks] = n
}

}  // namespace

namespace mdkk {

int exclusive_scan_i32(mdkk_ctx* ctx, const int* in, int* out, long long n, cudaStream_t s) {
    return scan_impl<int>(ctx, in, out, n, s);
}
int exclusive_scan_i64(mdkk_ctx* ctx, const long long* in, long long* out, long long n, cudaStream_t s) {
    return scan_impl<long long>(ctx, in, out, n, s);
}

}  // namespace mdkk

extern "C" int mdkk_bucket_sort(mdkk_ctx* ctx, const int* keys, int n, int nbuckets, int* bucket_start, int* order,
                                void* stream) {
    if (!ctx || n < 0 || nbuckets < 1 || nbuckets > (1 << 30)) return MDKK_E_ARG;
    cudaStream_t s = mdkk::as_stream(stream);
    if (n == 0) {
        cudaMemsetAsync(bucket_start, 0, sizeof(int) * ((size_t)nbuckets + 1), s);
        return MDKK_OK;
    }
    if (nbuckets <= kSmallBuckets) {
        const int nb = (n + kSmallBlock - 1) / kSmallBlock;
        const size_t cells = (size_t)nbuckets * nb + 1;
        int* table = static_cast<int*>(mdkk::scratch(ctx, sizeof(int) * 2 * cells));
        if (!table) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "sort scratch");
        int* offs = table + cells;
        cudaMemsetAsync(table + cells - 1, 0, sizeof(int), s);
        k_small_count<<<nb, kSmallBlock, 0, s>>>(n, keys, nbuckets, nb, table);
        MDKK_CHECK_LAUNCH("k_small_count");
        int st = mdkk::exclusive_scan_i32(ctx, table, offs, (long long)cells, s);
        if (st != MDKK_OK) return st;
        k_small_scatter<<<nb, kSmallBlock, 0, s>>>(n, keys, nbuckets, nb, offs, order, bucket_start);
        MDKK_CHECK_LAUNCH("k_small_scatter");
        return MDKK_OK;
    }
    int* cnt = static_cast<int*>(mdkk::scratch(ctx, sizeof(int) * ((size_t)nbuckets + 1)));
    if (!cnt) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "sort scratch");
    cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)nbuckets + 1), s);
    k_key_count<<<mdkk::grid_for(n, 256), 256, 0, s>>>(n, keys, cnt);
    MDKK_CHECK_LAUNCH("k_key_count");
    return mdkk::bucket_sort_counted(ctx, keys, n, nbuckets, cnt, bucket_start, order, s);
}

namespace mdkk {

// The many-bucket sort after its count pass: cnt[nbuckets + 1] holds the per-bucket
// counts (cnt[nbuckets] = 0), e.g. taken by the producer of the keys.
int bucket_sort_counted(mdkk_ctx* ctx, const int* keys, int n, int nbuckets, int* cnt, int* bucket_start,
                        int* order, cudaStream_t s) {
    int st = mdkk::exclusive_scan_i32(ctx, cnt, bucket_start, (long long)nbuckets + 1, s);
    if (st != MDKK_OK) return st;
    // the counts themselves are the per-bucket cursors (counted down by the scatter)
    k_key_scatter<<<mdkk::grid_for(n, 256), 256, 0, s>>>(n, keys, bucket_start, cnt, order);
    MDKK_CHECK_LAUNCH("k_key_scatter");
    const long long threads = (long long)nbuckets * kRsG;
    k_bucket_rowsort<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(nbuckets, bucket_start, order);
    MDKK_CHECK_LAUNCH("k_bucket_rowsort");
    return MDKK_OK;
}

}  // namespace mdkk
