/*
 * mdkk_b200.h — C ABI of the B200-native force-and-neighbor hot path.
 *
 * This is the drop-in boundary for the reference `mdkk` engine
 * (/root/reference/pkg/src/mdkk).  Every entry point replaces one reference
 * function (cited per declaration); the Python host layer
 * (paper_2508_13523_b200/) keeps the reference's Python signatures and binds
 * these through ctypes.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers owned by the caller unless the
 *    name ends in `_host`.  No torch types cross this boundary.
 *  - Positions / forces / velocities are AoS-padded double4 rows
 *    (x, y, z, pad): one 32-byte sector per neighbour gather.
 *  - Neighbour tables are int32, cluster-blocked [ceil(n_local/32)][cap][32]:
 *    entry k of row i lives at ((i/32)*cap + k)*32 + i%32 — the reference's
 *    transposed `layout_b` (atom index fastest, mdkk/memspace.py:99-100)
 *    tiled by 32 rows so one warp's k-th entries are one 128-byte line.
 *  - `stream` is a cudaStream_t (may be NULL = legacy default stream).
 *  - Every function returns an mdkk_status; calls are asynchronous on
 *    `stream` unless documented otherwise.  No C++ exception crosses the ABI.
 *  - One host thread and one stream per device at a time (the reference
 *    driver is single-threaded): a context's scratch arena and the
 *    energy/virial reductions' device-side stage are shared by the calls
 *    issued on a device.
 */
#ifndef MDKK_B200_H
#define MDKK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MDKK_OK = 0,
    MDKK_E_CAPACITY = 1,   /* neighbour row overflow: grow cap x1.5 and rebuild (mdkk/neighbor.py:199-205) */
    MDKK_E_COINCIDENT = 2, /* r^2 <= 0 (mdkk/pair_lj.py:83-84, mdkk/snap/compute.py:117-118) */
    MDKK_E_NONFINITE = 3,  /* non-finite energy / force (mdkk/driver/simulation.py:459-464) */
    MDKK_E_ARG = 4,        /* invalid argument */
    MDKK_E_CUDA = 5        /* CUDA runtime error (see mdkk_last_error) */
} mdkk_status;

/* Device error-word bits written by kernels (read lazily by the host). */
#define MDKK_FLAG_COINCIDENT 1
#define MDKK_FLAG_NONFINITE 2

typedef struct mdkk_ctx mdkk_ctx;   /* per-device scratch arena (opaque) */
typedef struct mdkk_snap mdkk_snap; /* SNAP coupling tables on device (opaque) */

/* ------------------------------------------------------------------ misc */
int mdkk_version(void);
/* Number of kernels this library has launched in the process (all devices). */
unsigned long long mdkk_launch_count(void);
const char* mdkk_last_error(void);
int mdkk_device_sm_count(int device, int* out_host);
int mdkk_ctx_create(int device, mdkk_ctx** out_host);
int mdkk_ctx_destroy(mdkk_ctx* ctx);
/* FP64 FMA throughput probe: blocks x 256 threads x iters x 8 DFMA (2 flops
 * each); timed by the caller to measure the FP64 roofline denominator. */
int mdkk_fp64_probe(int blocks, int iters, double* out, void* stream);

/* ------------------------------------------------------ domain / halo comm
 * Replaces mdkk/domain.py:56-63 (wrap), :246-293 (exchange_ghosts selection),
 * :295-305 (forward_comm pack), :307-322 (reverse_comm fold), :324-334
 * (migrate: wrap + reorder).
 */
/* x[i] wrapped into [0, L) per axis. */
int mdkk_wrap(double* x, int n, const double* lengths_host, void* stream);

/* Halo selection over `n` owned rows of x against C combos.  combos_dev is
 * double[C][9] = {lo[3], hi[3], shift[3]}; an atom is selected for combo c iff
 * x + shift lies in [lo, hi) on every axis (half-open, mdkk/domain.py:274).
 * Two phases: count writes totals[C] (device) and per-block offsets into
 * block_scratch (int[ceil(n/256) * C]); fill writes out_idx combo-major, atoms
 * ascending within a combo — the reference's src/shift/index order; with
 * out_code (optional, int8[total]) each selected row also gets its combo's
 * shift code combo_code[c] (device int8[C]). */
int mdkk_halo_count(mdkk_ctx* ctx, const double* x, int n, const double* combos_dev, int C,
                    int* block_scratch, int* totals, const int* rows, const int* n_dev, void* stream);
int mdkk_halo_fill(mdkk_ctx* ctx, const double* x, int n, const double* combos_dev, int C,
                   const int* block_scratch, const int* totals, int* out_idx, const int8_t* combo_code,
                   int8_t* out_code, const int* rows, const int* n_dev, void* stream);
/* rows / n_dev (both optional, for count and fill alike): scan only rows[k], k < *n_dev
 * (ascending; n then bounds k) instead of every row -- mdkk_boundary_rows' output for a
 * cell-sorted brick whose cells are at least the halo wide. */
/* Rows of the cells within `layer` cells of the faces of a (serpentine-keyed) grid,
 * ascending, for owned rows sorted by cell with bucket starts cell_start[ncell + 1];
 * *count (device) = their number. */
int mdkk_boundary_rows(mdkk_ctx* ctx, const int* cell_start, const int* ncell_host, int layer, int* rows,
                       int* count, void* stream);

/* Forward-comm pack: out[k] = x[idx[k]] + shift_table[code[k]] (shift_table is
 * double[27][3] device, code int8 in 0..26).  `out` may alias ghost rows of x. */
int mdkk_pack_shift(const double* x, const int* idx, const int8_t* code, const double* shift_table,
                    int n, double* out, void* stream);
/* Reverse-comm unpack: f[idx[k]] += buf[k] (FP64 atomics; idx may repeat). */
int mdkk_fold_add(double* f, const int* idx, const double* buf, int n, void* stream);
/* A lane's new ghost rows in one pass (exchange_ghosts, mdkk/domain.py:276-293):
 * out_x[k] = x[idx[k]] + shift_table[code[k]] (as mdkk_pack_shift), out_gid[k] =
 * gid[idx[k]], out_oidx[k] = idx[k]. */
int mdkk_ghost_rows(const double* x, const int64_t* gid, const int* idx, const int8_t* code, const double* shifts,
                    int n, double* out_x, int64_t* out_gid, int* out_oidx, void* stream);
/* Gather rows by permutation: dst[i] = src[perm[i]] for double4 rows / int64 / int32. */
int mdkk_gather_rows4(const double* src, const int* perm, int n, double* dst, void* stream);
int mdkk_gather_i64(const int64_t* src, const int* perm, int n, int64_t* dst, void* stream);
int mdkk_gather_i32(const int32_t* src, const int* perm, int n, int32_t* dst, void* stream);
/* Scatter rows by permutation: dst[perm[i]] = src[i] (gid-ordered gather for host views). */
int mdkk_scatter_rows4(const double* src, const int* perm, int n, double* dst, void* stream);

/* ----------------------------------------------------------------- binning
 * Counting-sort cell binning (replaces the bbox/argsort/bincount of
 * mdkk/neighbor.py:88-96).  grid_host = {origin[3], inv_width[3]} and
 * ncell_host = {nx, ny, nz}; cell id = (cx*ny + cy)*nz + cz (x slowest, as
 * mdkk/neighbor.py:93).  Out-of-grid atoms clamp to edge cells, which keeps
 * the 27-cell stencil complete when every width >= the build cutoff. */
int mdkk_cell_keys(const double* x, int n, const double* grid_host, const int* ncell_host, int* keys,
                   void* stream);
/* Owning brick of each row: floor(pos / L * grid) clipped (mdkk/domain.py:89-95). */
int mdkk_rank_keys(const double* x, int n, const double* lengths_host, const int* grid_host, int* keys,
                   void* stream);
/* Stable bucket sort by int key in [0, nbuckets): bucket_start[nbuckets+1],
 * order[n] (rows of a bucket contiguous, ascending row index). */
int mdkk_bucket_sort(mdkk_ctx* ctx, const int* keys, int n, int nbuckets, int* bucket_start, int* order,
                     void* stream);
/* cell_keys + bucket_sort.  keys is caller scratch int[n]. */
int mdkk_bin_atoms(mdkk_ctx* ctx, const double* x, int n, const double* grid_host, const int* ncell_host,
                   int* keys, int* cell_start, int* cell_atoms, void* stream);

/* One-rank engine rebuild, selection phase (RankedSystem.migrate's single-rank path,
 * mdkk/domain.py:324-334, with the halo selection of exchange_ghosts :246-293) in one
 * call: wrap x[0, n), counting-sort the rows by cell of the shell grid (keys / cell_start
 * / order as mdkk_bin_atoms), gather x into x_sorted, list the boundary-layer rows
 * (mdkk_boundary_rows, 2 layers) and count the halo entries per combo (mdkk_halo_count
 * over x_sorted); the totals are copied into totals_host (pinned, int[C]) and the
 * velocity / gid gathers are queued behind that copy; returns once the totals have
 * arrived, with their sum in *n_ghost_host.  x_ref (optional, double4[n]): also receives
 * the sorted rows (the next lists' skin-test reference, mdkk/neighbor.py:66-80).  The
 * caller then fills the ghost rows (mdkk_halo_fill with the same block_scratch / totals /
 * brows / bcount). */
int mdkk_rebuild1_select(mdkk_ctx* ctx, double* x, int n, const double* lengths_host, const double* grid_host,
                         const int* ncell_host, int* keys, int* cell_start, int* order, double* x_sorted,
                         const double* v, double* v_sorted, const int64_t* gid, int64_t* gid_sorted, int* brows,
                         int* bcount, const double* combos_dev, int C, int* block_scratch, int* totals,
                         int* totals_host, int* n_ghost_host, double* x_ref, void* stream);

/* Cell lists for a build whose owned rows [0, n_local) are already sorted by cell on
 * this grid with bucket starts owned_start[ncell + 1] (the engine's spatial sort):
 * bins only the ghost rows [n_local, n_total) and merges, giving exactly
 * mdkk_bin_atoms over all rows (owned then ghost rows per cell, each ascending).
 * keys: int[n_total - n_local] scratch; cell_start int[ncell + 1]; cell_atoms
 * int[n_total]. */
int mdkk_bin_merge(mdkk_ctx* ctx, const double* x, int n_local, int n_total, const double* grid_host,
                   const int* ncell_host, const int* owned_start, int* keys, int* cell_start, int* cell_atoms,
                   void* stream);
/* -------------------------------------------------------------- neighbour
 * Cluster-scan neighbour build (replaces mdkk/neighbor.py:83-219 +
 * _apply_style :134-179).  Owned rows should be cell-sorted (any order is
 * correct, sorted is fast): one warp takes 32 consecutive rows, gathers the
 * union of rows within bc of their bounding box, and each lane keeps every
 * j != i with r^2 < bc^2 (strict; r^2 rounded as the reference's einsum,
 * mdkk/neighbor.py:126) passing the style predicate: style 0 = full; 1 =
 * half with the gid / owner-rank / z-y-x rules (newton on) or ghost pairs on
 * both sides (newton off).  table is the cluster-blocked int32 layout above
 * (ceil(n_local/32)*cap*32 ints), entries beyond counts[i] undefined; counts[i] is the true count even when
 * > cap and *max_count (device int, caller-zeroed) the max, so the caller
 * grows cap x1.5 and relaunches — never truncates (mdkk/neighbor.py:199-205);
 * after an overflow the table's contents are undefined.  ctx's scratch holds a
 * cell-ordered FP32 copy of the positions for the (superset) union test. */
int mdkk_nbr_build(mdkk_ctx* ctx, const double* x, int n_local, int n_total,
                   const double* grid_host, const int* ncell_host, const int* cell_start,
                   const int* cell_atoms, const int64_t* gid, const int32_t* owner_rank, int my_rank,
                   double bc, int style, int newton, int cap, int* table, int* counts, int* max_count,
                   void* stream);
/* Canonical per-row order (partner gid, z, y, x) — mdkk/neighbor.py:192-197.
 * In-place sort of each row of a plain [cap][n_local] table (the host API
 * transposes the cluster-blocked table into this form first). */
int mdkk_nbr_canonicalize(const double* x, const int64_t* gid, int n_local, int cap,
                          int* table, const int* counts, void* stream);
/* max_i |x_i - x_ref_i|^2 into *out (device double) — mdkk/neighbor.py:66-74. */
/* Sort every row of a cluster-blocked table by the partner displacement (dz, dy, dx)
 * = x_j - x_i (the reference's NeighborMap order, mdkk/snap/compute.py:66-104), making
 * per-row accumulation orders label-independent.  In place. */
int mdkk_nbr_geo_order(const double* x, int n_local, int cap, int* table, const int* counts, void* stream);
int mdkk_max_disp2(const double* x, const double* x_ref, int n, double* out, void* stream);

/* --------------------------------------------------------------------- LJ
 * Truncated 12-6 LJ (mdkk/pair_lj.py:81-91) over a cluster-blocked table
 * (compute_pair, mdkk/pair_lj.py:114-179).  style/newton select the entry
 * semantics of mdkk/neighbor.py:134-179:
 *   full          : f_i only, weight 1/2, no atomics (owner writes)
 *   half, newton  : f_i and f_j (FP64 atomics; ghosts folded by reverse comm)
 *   half, !newton : f_j written only for local j; ghost entries weight 1/2
 * f must be zeroed by the caller for half lists (atomics accumulate).
 * ev (device double[7]) receives {E, Wxx, Wyy, Wzz, Wxy, Wxz, Wyz}; with
 * virial == 0 only E is accumulated (W* = 0).  Deterministic two-stage
 * reduction.  flags (device int) gets MDKK_FLAG_COINCIDENT if any in-range
 * r^2 <= 0. */
int mdkk_lj_force(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts,
                  int cap, int style, int newton, int virial, double epsilon, double sigma, double rc,
                  double* f, double* ev, int* flags, void* stream);
/* Neighbour-parallel LJ (mode "neighbor", lj/cut/opt; mdkk/pair_lj.py:118-143): a
 * team of 8 lanes per atom splits its list and reduces the partials; same
 * arguments and results (to rounding) as mdkk_lj_force. */
int mdkk_lj_force_neighbor(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts,
                           int cap, int style, int newton, int virial, double epsilon, double sigma, double rc,
                           double* f, double* ev, int* flags, void* stream);
/* Full-list force with the velocity-Verlet update fused into its epilogue (the engine's
 * advance loop; mdkk/driver/simulation.py:431-450): mode 1 = closing half-kick
 * v += h f; mode 2 = closing + next opening half-kick and drift x_next = x + dt v
 * for the owned rows (x_next must not alias x: positions are double-buffered; its
 * ghost rows are refreshed by the next pack) and *d2_next = max |x_next - x_ref|^2
 * (atomic max; caller-zeroed).  Bit-identical to mdkk_lj_force + mdkk_verlet_second
 * + mdkk_verlet_first.  Gates as mdkk_lj_force_gated (a gated-off launch changes
 * nothing).  Halo overlap (one rank per GPU): part 1 computes only the clusters with
 * part_flags[c] == 0 (launched while the ghost exchange is in flight; no reduction),
 * part 2 the others and the energy reduction (same gate / arguments); part 0 = all. */
int mdkk_lj_force_integrate(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts,
                            int cap, int virial, double epsilon, double sigma, double rc, double* f, double* ev,
                            int* flags, const double* maxdisp2, double half_skin, const int* max_count,
                            int count_limit, int mode, double* v, const double* x_ref, double* x_next,
                            double* d2_next, double dt, double h, const unsigned char* part_flags, int part,
                            void* stream);
/* mdkk_lj_force_integrate in mode 2 (close step s, open and drift step s+1) that also
 * writes step s+1's periodic ghost rows (forward_comm, mdkk/domain.py:295-305):
 * x_next[n_local + k] = x_next[pack_idx[k]] + pack_shifts[pack_code[k]] for k < pack_n, in
 * the reduction's launch -- one rank with its own periodic images (the engine's fused
 * loop, which then skips the separate pack).  d2_zero (optional): a drift-maximum slot
 * cleared in the same launch (the engine's three-slot ring: the slot two steps ahead). */
int mdkk_lj_force_integrate_pack(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts,
                                 int cap, int virial, double epsilon, double sigma, double rc, double* f, double* ev,
                                 int* flags, const double* maxdisp2, double half_skin, const int* max_count,
                                 int count_limit, double* v, const double* x_ref, double* x_next, double* d2_next,
                                 double dt, double h, const int* pack_idx, const int8_t* pack_code,
                                 const double* pack_shifts, int pack_n, double* d2_zero, void* stream);
/* Boundary flags per 32-row cluster for the halo overlap (engine-internal; no reference
 * counterpart): flags[c] = 1 when the cluster's bounding box lies within `halo` of a
 * brick face [lo, hi) in a dimension of dims_mask (bit d: the neighbour bricks along d
 * are other ranks).  halo = list cutoff + skin/2 keeps the flags valid until the next
 * rebuild. */
int mdkk_cluster_flags(const double* x, int n_local, const double* lo_host, const double* hi_host, double halo,
                       int dims_mask, unsigned char* flags, void* stream);
/* Speculative step launch (engine-internal pipelining): as mdkk_lj_force (mode 0) or
 * mdkk_lj_force_neighbor (mode 1), but the kernel does nothing when
 * sqrt(*maxdisp2) > half_skin -- the step's skin test, evaluated on the device in the
 * host's FP64 operations -- or when *max_count > count_limit (the build's capacity
 * check), so the launch can be queued before the host has read either decision; a
 * rebuilding / regrowing step relaunches afterwards.  Either gate may be NULL.  ev
 * is undefined after a skipped launch. */
int mdkk_lj_force_gated(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts,
                        int cap, int style, int newton, int virial, int mode, double epsilon, double sigma,
                        double rc, double* f, double* ev, int* flags, const double* maxdisp2, double half_skin,
                        const int* max_count, int count_limit, void* stream);
/* Half-list force with an explicit partner-write strategy: compute_pair's
 * `strategy` (mdkk/pair_lj.py:114-139 -> ScatterAccumulator, mdkk/memspace.py:165-254).
 * strategy 1 = Duplicate: own and partner REDs go into staging copy
 * (block % copies) of `copies` zeroed f-shaped ([n][4]) copies `stride` doubles apart;
 * the caller combines them with mdkk_scatter_combine.  strategy 2 = Serial: own rows
 * are stored into f, each partner contribution is written as double4 (g, 1) per table
 * entry into `stage` (zeroed, the table's [ncl][cap][32] layout) and applied in entry
 * order by mdkk_scatter_ordered (no atomics: deterministic).  Atomic is mdkk_lj_force. */
int mdkk_lj_force_strategy(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts,
                           int cap, int newton, int virial, double epsilon, double sigma, double rc, double* f,
                           double* ev, int* flags, int strategy, double* stage, long long stride, int copies,
                           void* stream);

/* ---------------------------------------------------------------- scatter
 * ScatterAccumulator strategies (mdkk/memspace.py:198-257) on row-major
 * [n_rows][ld] f64 targets; a contribution updates `width` leading entries.
 * atomic : target[idx[e]][c] += vals[e][c] with FP64 RED (Atomic).
 * ordered: `sorted_idx`/`perm` are the stable sort of the contribution indices;
 *          each row's contributions are added one by one in their original order
 *          onto its current value -- bit-identical to sequential np.add.at (Serial).
 * combine: out[e] += ((stage[0][e] + stage[1][e]) + ...) over `copies` staging copies
 *          `stride` doubles apart (Duplicate's finalize, np.add.reduce order).
 * index_range: *bad = min(*bad, e) for every idx[e] outside [0, n_rows) (caller
 *          initialises *bad to ~0): the reference's IndexError check. */
int mdkk_scatter_atomic(double* target, int ld, int width, const long long* idx, const double* vals, long long n,
                        void* stream);
int mdkk_scatter_ordered(double* target, int ld, int width, const long long* sorted_idx, const long long* perm,
                         const double* vals, long long n, void* stream);
int mdkk_scatter_combine(const double* stage, int copies, long long stride, double* out, long long n, void* stream);
int mdkk_index_range(const long long* idx, long long n, long long n_rows, unsigned long long* bad, void* stream);

/* ------------------------------------------------------------- integrator
 * Velocity Verlet (mdkk/driver/simulation.py:431-450) fused with the skin
 * test (mdkk/neighbor.py:66-74).  first: v += h f; x += dt v;
 * *maxdisp2 = max |x - x_ref|^2; pending_kick != 0 first applies the previous
 * step's deferred closing v += h f (same f; bit-identical to calling second
 * then first).  second: v += h f; ke (optional, device double) = sum 1/2 m v^2
 * (mdkk/driver/simulation.py:407-415). */
int mdkk_verlet_first(mdkk_ctx* ctx, double* x, double* v, const double* f, const double* x_ref,
                      int n, double dt, double half_dt_over_m, double* maxdisp2, int pending_kick, void* stream);
int mdkk_verlet_second(mdkk_ctx* ctx, double* v, const double* f, int n, double half_dt_over_m,
                       double mass, double* ke, void* stream);
/* Sum of 1/2 m |v|^2 over n rows into *ke (device double). */
int mdkk_kinetic(mdkk_ctx* ctx, const double* v, int n, double mass, double* ke, void* stream);

/* ------------------------------------------------------------------- SNAP
 * FP64 descriptor pipeline with mdkk's conventions (mdkk/snap/compute.py:
 * rfac0 0.99, rmin0 0, cosine switch, no self term, full (2j+1)^2 blocks,
 * full three-slot adjoint).  U is complex128 row-major [n_local][n_flat]
 * (the reference's layout "a"), n_flat = sum_{tj<=2J} (tj+1)^2.  The engine
 * keeps Y as its half set (2p < tj, or 2p == tj and 2q <= tj; n_half entries,
 * the rest follows from Y[tj-p][tj-q] = (-1)^(p+q) conj(Y[p][q])) transposed,
 * Yh[e][i] with leading dimension ld >= n_local; mdkk_snap_y_expand /
 * _compress convert to / from the reference layout.  U and the reference-layout
 * Y take the SnapState `layout` knob (mdkk/snap/compute.py:238-276): layout 0
 * ("a") = row-major [n][n_flat], layout 1 ("b") = transposed [n_flat][ldu],
 * atoms fastest.
 * Pairs are the entries of a FULL cluster-blocked table with r^2 < rc^2.
 *
 * mdkk_snap_create copies the product list built on the host from the exact
 * Clebsch-Gordan terms and beta (mdkk/snap/coupling.py:106-133; the Z-list form
 * of mdkk/snap/compute.py:303-340, see snap/coupling.py zlist_entries):
 *   Yh[f] = sum_k coef[k] * op_g(U[g_k]) * op_h(U[h_k])      (half indices)
 * code[k] = g | h << 8 | f << 16 | conj_g << 24 | conj_h << 25 | last << 26 |
 * center << 27, sorted by output f, `last` on the final product of each output,
 * `center` when f is its own mirror; fmap[flat] = half index | mirrored << 16 |
 * odd sign << 17.  0 <= 2J <= 8. */
int mdkk_snap_create(mdkk_ctx* ctx, int twojmax, int n_entries, const double* coef_host, const int* code_host,
                     int n_half, const int* fmap_host, mdkk_snap** out_host);
int mdkk_snap_destroy(mdkk_snap* snap);
/* Schedule knobs of SnapState (mdkk/snap/compute.py:238-276: batch_u scales the
 * expansion pass's pair batch, batch_y groups the contraction; scheduling only).
 * batch_u -> neighbour pairs expanded concurrently per two warps in compute_ui
 * (<=3, 4..7, >=8 -> 32-, 16-, 8-lane teams per pair; the reference default 4 is the
 * fastest on B200); batch_y -> atoms per lane in compute_yi (1, >=2 -> 2). */
int mdkk_snap_set_schedule(mdkk_snap* snap, int batch_u, int batch_y);
/* U_i = sum_k f_c(r_ik) u(a_ik, b_ik) (compute_ui, mdkk/snap/compute.py:279-292); flags gets
 * MDKK_FLAG_COINCIDENT for r = 0 pairs (mdkk/snap/compute.py:117-118). */
int mdkk_snap_ui(mdkk_snap* snap, const double* x, int n_local, const int* table, const int* counts, int cap,
                 double rc, double* U, int layout, int ldu, int* flags, void* stream);
/* Yh from U (compute_yi, mdkk/snap/compute.py:303-340) and *energy (device double)
 * = sum_i Re(Y_i . conj(U_i)) / 3 (energy_from_y, mdkk/snap/compute.py:376-387). */
int mdkk_snap_yi(mdkk_ctx* ctx, mdkk_snap* snap, const double* U, int n_local, double* Yh, int ld, double* energy,
                 int layout, int ldu, void* stream);
/* Reference layout: Y[i][flat] (complex128 row-major) from Yh, and back. */
int mdkk_snap_y_expand(mdkk_snap* snap, const double* Yh, int ld, int n_local, double* Y, int layout, int ldy,
                       void* stream);
int mdkk_snap_y_compress(mdkk_snap* snap, const double* Y, int n_local, double* Yh, int ld, int layout, int ldy,
                         void* stream);
/* Fused 3-direction forces (compute_fused_deidrj, mdkk/snap/compute.py:390-409):
 * t = Re sum_f Y_i[f] conj(d(f_c u)/d r_ik [f]) evaluated in reverse mode (u
 * forward, adjoint backward, 4 complex partials per pair); f_i += t, f_k -= t (FP64
 * atomics, f double4 rows incl. ghosts, caller-zeroed; ghosts -> reverse comm). */
int mdkk_snap_deidrj(mdkk_snap* snap, const double* x, int n_local, const int* table, const int* counts, int cap,
                     double rc, const double* Yh, int ld, double* f, void* stream);
/* The whole per-step pipeline in one call (SnapStyle.compute, mdkk/driver/simulation.py:123-142):
 * ui -> yi -> fused deidrj on one stream.  U ([n_local][n_flat] complex, layout a) and Yh
 * ([n_half][n_local] complex) are optional dumps: pass both NULL to use a workspace owned by
 * the handle (grown on demand, freed by mdkk_snap_destroy).  f as mdkk_snap_deidrj (caller
 * zeroed, ghost rows -> reverse comm); *energy (device) and *flags as mdkk_snap_yi / _ui. */
int mdkk_snap_compute(mdkk_ctx* ctx, mdkk_snap* snap, const double* x, int n_local, const int* table,
                      const int* counts, int cap, double rc, double* U, double* Yh, double* f, double* energy,
                      int* flags, void* stream);

/* --- SNAP API-parity stages (not on the engine path; csrc/snap_aux.cu) ---
 * Neighbour map (build_neighbor_map / NeighborMap, mdkk/snap/compute.py:66-119):
 * per-row in-range pair counts npair[n_local+1] and their exclusive scan
 * offsets[n_local+1] (offsets[n_local] = total pairs P), then the pairs in
 * (row, dz, dy, dx) order: rows/cols int32 [P], dr f64 [P][3], r [P],
 * a/b complex128 [P], fc/dfc [P]. */
int mdkk_snap_pair_count(mdkk_ctx* ctx, const double* x, int n_local, const int* table, const int* counts, int cap,
                         double rc, int* npair, int* offsets, int* flags, void* stream);
int mdkk_snap_pair_fill(const double* x, int n_local, const int* table, const int* counts, int cap, double rc,
                        const int* offsets, int* rows, int* cols, double* dr, double* r, double* a, double* b,
                        double* fc, double* dfc, void* stream);
/* Staged force path (compute_duidrj / compute_deidrj, mdkk/snap/compute.py:412-436):
 * wdu complex128 [P][3][n_flat] = f_c du/d dr_d + f_c' (dr_d / r) u; then
 * f[row] += t, f[col] -= t with t_d = Re sum_f Y[row][f] conj(wdu[p][d][f]) (Y in the
 * reference layout, f double4 rows, caller-zeroed). */
int mdkk_snap_duidrj(mdkk_snap* snap, int n_pairs, const double* dr, double rc, double* wdu, void* stream);
int mdkk_snap_deidrj_staged(mdkk_snap* snap, int n_pairs, const int* rows, const int* cols, const double* Y,
                            const double* wdu, double* f, void* stream);
/* Descriptors (compute_bi_complex, mdkk/snap/compute.py:354-373): B complex128
 * [n_local][n_tri], B_t = sum c * op(U[g]) op(U[h]) op(U[z]) over the triple's
 * terms (half indices; code = g | h << 8 | z << 16 | conj_g << 24 | conj_h << 25 |
 * conj_z << 26 | last-of-triple << 27; tri[k] = triple of term k; chunk[w] =
 * first term of warp w, output-aligned, mdkk_snap_bi_warps() + 1 entries). */
/* pair_u_flat (mdkk/snap/compute.py:165-184): u_0..u_2J of arbitrary (a, b) (complex128
 * [n]) by the reference's four-term recursion, out complex128 [n][n_flat]. */
int mdkk_snap_pair_u(int n_pairs, int twojmax, const double* a, const double* b, double* out, void* stream);
/* NeighborMap.deriv_params (mdkk/snap/compute.py:48-63,98-102): da, db complex128 [n][3]
 * from dr f64 [n][3]. */
int mdkk_snap_pair_grads(int n_pairs, const double* dr, double rc, double* da, double* db, void* stream);
/* Per-pair force contraction of staged derivatives, no scatter (the drop-in's
 * compute_fused_deidrj / compute_deidrj over the reference's pair arrays,
 * mdkk/snap/compute.py:390-436): t_out[p][d] = Re sum_f Y[rows[p]][f] conj(wdu[p][d][f]),
 * Y complex128 [n][n_flat] (layout "a"), wdu complex128 [n_pairs][3][n_flat]. */
int mdkk_snap_pair_dedr(mdkk_snap* snap, int n_pairs, const int* rows, const double* Y, const double* wdu,
                        double* t_out, void* stream);
int mdkk_snap_bi(mdkk_snap* snap, const double* U, int n_local, const double* coef, const int* code, const int* tri,
                 const int* chunk, int n_tri, double* B, int layout, int ldu, void* stream);
int mdkk_snap_bi_warps(void);

/* ------------------------------------------------------------------- QEq
 * Charge equilibration (mdkk/qeq.py): over-allocated CSR with int64 row
 * offsets = exclusive scan of capacities min(counts, cap) + 1 (caps scratch
 * [n+1], offsets [n+1]); values f64 / columns int32 / row_nnz int32; diagonal
 * eta first, then list partners within the cutoff, value (r^3 + gamma^-3)^(-1/3),
 * column = owner index (mdkk/qeq.py:41-133).  SpMV: y1 = H x1 and, when x2 is
 * non-NULL, y2 = H x2 in the same traversal; dots (optional, device [2]) gets
 * x1.y1 and x2.y2.  All reductions fixed-order: a fused two-system CG is
 * bit-identical to two sequential solves (mdkk/qeq.py:233-274). */
int mdkk_qeq_offsets(mdkk_ctx* ctx, const int* counts, int n, int cap, long long* caps, long long* offsets,
                     void* stream);
int mdkk_qeq_build(const double* x, int n_local, const int* table, const int* counts, int cap, const int* oidx,
                   const long long* offsets, double eta, double gamma, double cutoff, double* values, int* columns,
                   int* row_nnz, void* stream);
int mdkk_qeq_spmv(mdkk_ctx* ctx, const long long* offsets, const double* values, const int* columns,
                  const int* row_nnz, int n, const double* x1, const double* x2, double* y1, double* y2,
                  double* dots, void* stream);
/* Gershgorin guard (mdkk/qeq.py:180-194): *bad_row (device, caller-set to INT_MAX)
 * gets the first row with diag <= sum |offdiag|; diag / offsum per row. */
int mdkk_qeq_gershgorin(const long long* offsets, const double* values, const int* columns, const int* row_nnz, int n,
                        int* bad_row, double* diag, double* offsum, void* stream);
/* *out = a . b (device), fixed order. */
int mdkk_dot(mdkk_ctx* ctx, const double* a, const double* b, int n, double* out, void* stream);
/* CG stages (mdkk/qeq.py:197-207): alpha = *rr / *pap; x += alpha p; r -= alpha Ap;
 * *rr_new = r . r; then p = r + (*rr_new / *rr) p. */
int mdkk_cg_update(mdkk_ctx* ctx, int n, double* x, double* r, const double* p, const double* ap, const double* rr,
                   const double* pap, double* rr_new, void* stream);
int mdkk_cg_direction(int n, const double* r, double* p, const double* rr, const double* rr_new, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MDKK_B200_H */
