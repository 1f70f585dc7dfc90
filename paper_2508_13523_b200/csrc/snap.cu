// SNAP descriptor pipeline in FP64 on sm_100a.
// Reference: mdkk/snap/compute.py (map :27-63, recursion :125-235,
// compute_ui :279-292, compute_yi :303-340, energy :354-387,
// compute_fused_deidrj :390-409) with mdkk's conventions: rfac0 = 0.99,
// rmin0 = 0, plain cosine switch, no self term, full (tj+1)^2 blocks and the
// full three-slot adjoint Y.
//
// Data: U complex128 in the state's layout (a: [n][n_flat], b: [n_flat][ld]);
// the engine's Y is the half set, transposed (Yh[e][i]); double2 = (re, im).
//
// compute_ui: one warp per atom; each team of lanes expands one neighbour at a
// time with the two-term column recursion over the column halves C_tj (the
// previous level mirrored into shared memory), keeping its slots of U_i in
// registers (no atomics).  compute_yi: atoms across lanes over a shared U tile,
// the Z-list product stream as warp broadcasts.  compute_fused_deidrj: reverse
// mode over the same recursion (u forward, adjoint backward), 8-lane teams.
#include "snap_common.cuh"

namespace {

// ---------------------------------------------------------------- compute_ui
// U_i = sum_k f_c u(a_k, b_k) (mdkk/snap/compute.py:279-292), row-major U.
// One warp per atom, two neighbours at a time (half-warp each); each half
// computes the column half C_tj of every level with the two-term recursion
// (16 lanes, previous level in shared memory as a full mirrored level),
// accumulates f_c u in registers, and the full U_i row is written from C and
// its mirror.
template <int TWOJ, int TEAM, int DW>
__global__ void __launch_bounds__(DW * 32, (TEAM == 16 ? 4 : 8 / DW)) k_snap_ui(const double* __restrict__ x, int n_local,
                                                         const int* __restrict__ table,
                                                         const int* __restrict__ counts, int cap, double rc,
                                                         double2* __restrict__ U, long long su, long long sf,
                                                         int* __restrict__ flags) {
    constexpr int NF = block_offset(TWOJ + 1);
    constexpr int PPW = 32 / TEAM;                       // pairs in flight per warp
    constexpr int NS = tslot_base<TEAM>(kMaxTwoJ + 1);   // accumulator slots per lane
    __shared__ RS rs;
    __shared__ NbPair s_nb[DW][kNbChunk];
    __shared__ cplx s_lvl[DW][PPW][2][kLevelMax];
    for (int t = threadIdx.x; t < DW * PPW * 2 * kLevelMax; t += blockDim.x)
        (&s_lvl[0][0][0][0])[t] = {0.0, 0.0};   // rec2 reads finite neighbours at the column ends
    stage_rs(rs);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, hl = lane & (TEAM - 1), hh = lane / TEAM;
    const int i = blockIdx.x * DW + w;
    if (i >= n_local) return;
    cplx acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = {0.0, 0.0};
    const double4 xi = mdkk::ld4(x, i);
    const int n = min(counts[i], cap);
    const double rc2 = rc * rc;
    bool bad = false;
    for (int k0 = 0; k0 < n; k0 += kNbChunk) {
        const int m = compact_pairs(x, table, cap, i, k0, n, xi, rc2, rc, s_nb[w], bad);
        for (int t = 0; t < m; t += PPW) {
            const int pi = t + hh;
            const NbPair nb = s_nb[w][pi < m ? pi : t];
            PairGeo g;
            double z0, r0;
            geo_of(nb, g, z0, r0);
            const double fc = pi < m ? g.fc : 0.0;
            const cplx ab = cconj(g.a);
            cplx(*L)[kLevelMax] = s_lvl[w][hh];
            if (hl == 0) {
                L[0][0] = {1.0, 0.0};
                acc[0].re += fc;
            }
            __syncwarp();
#pragma unroll
            for (int tj = 1; tj <= TWOJ; ++tj) {
                const cplx* prev = L[(tj - 1) & 1];
                cplx* cur = L[tj & 1];
#pragma unroll
                for (int s = 0; s < tslots<TEAM>(tj); ++s) {
                    const int c = hl + TEAM * s;
                    if (c < half_size(tj)) {
                        int P, Q;
                        col_elem(tj, c, P, Q);
                        const cplx v = rec2(prev, tj, P, Q, rs, ab, g.b);
                        if (tj < TWOJ) store_for_next(cur, tj, P, Q, v);   // the top level is never re-read
                        acc[tslot_base<TEAM>(tj) + s] = cadd(acc[tslot_base<TEAM>(tj) + s], cscale(fc, v));
                    }
                }
                __syncwarp();
            }
        }
    }
    if (bad && lane == 0) atomicOr(flags, MDKK_FLAG_COINCIDENT);
    // every team owns the same elements: fold the teams onto team 0
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int o = 16; o >= TEAM; o >>= 1) {
            acc[s].re += __shfl_xor_sync(0xffffffffu, acc[s].re, o);
            acc[s].im += __shfl_xor_sync(0xffffffffu, acc[s].im, o);
        }
    if (hh) return;
    double2* Ui = U + (long long)i * su;   // layout a: su = NF, sf = 1; layout b: su = 1, sf = ld
#pragma unroll
    for (int tj = 0; tj <= TWOJ; ++tj)
#pragma unroll
        for (int s = 0; s < tslots<TEAM>(tj); ++s) {
            const int c = hl + TEAM * s;
            if (c < half_size(tj)) {
                int P, Q;
                col_elem(tj, c, P, Q);
                const cplx v = acc[tslot_base<TEAM>(tj) + s];
                const int e = P * (tj + 1) + Q, em = (tj - P) * (tj + 1) + (tj - Q);
                Ui[(block_offset(tj) + e) * sf] = make_double2(v.re, v.im);
                if (em != e) {
                    const double sg = ((P + Q) & 1) ? -1.0 : 1.0;
                    Ui[(block_offset(tj) + em) * sf] = make_double2(sg * v.re, -sg * v.im);
                }
            }
        }
}


// ---------------------------------------------------------------- compute_yi
// Half-block Y (outputs 2p < tj, or 2p == tj and 2q <= tj) as a list of U*U
// products, the Z-list form of the reference's three-slot adjoint
// (mdkk/snap/compute.py:303-340; equivalence: snap/coupling.py zlist_entries):
//   Y[f] = sum_k coef_k * op_g(U[g_k]) * op_h(U[h_k]),  op = identity or conj.
// Atoms run across lanes (32 per CTA, one per lane) and the product list is
// uniform across the warp: every lane reads U of its own atom from a
// shared-memory tile [half index][atom] (row stride 33: conflict-free stores
// and reads), the entry itself is one broadcast.  Each warp owns a contiguous,
// output-aligned slice of the list, so every output is one register sum
// (no atomics, deterministic) written coalesced to Yh[f][atom] (the engine's
// half/transposed layout; the reference layout comes from mdkk_snap_y_expand).
// Also e_i = Re sum_f Y_i[f] conj(U_i[f]) / 3 (energy_from_y, :376-387) from
// the half set with mirror weight 2.
constexpr int kYW = 16;                      // warps per CTA (2 CTAs per SM: 32 warps)
constexpr int kUS = 33;                      // tile row stride (double2)


__device__ __forceinline__ double flip_sign(double v, unsigned mask) {   // mask: 0 or 0x80000000
    return __hiloint2double(__double2hiint(v) ^ (int)mask, __double2loint(v));
}

// B atoms per lane (the batch_y knob): B tiles of 32 atoms, each Z-list entry broadcast serves
// B atoms (work batching, paper Table 2); B = 1 keeps two CTAs per SM, B = 2 one.
template <int NF, int NH, int B>
__global__ void __launch_bounds__(kYW * 32, B == 1 ? 2 : 1) k_snap_yi(const double2* __restrict__ U, int n,
                                                                      const ZEntry* __restrict__ ent,
                                                                      const int* __restrict__ chunk,
                                                                      const int* __restrict__ chunkf,
                                                                      double2* __restrict__ Yh, int ld,
                                                                      double* __restrict__ partials, long long su,
                                                                      long long sf) {
    extern __shared__ double2 s_dyn2[];
    double2* s_u = s_dyn2;                                                   // B x [NH][kUS]
    ZEntry* s_e = reinterpret_cast<ZEntry*>(s_u + B * NH * kUS);              // [kYW][32]
    constexpr int kTile = NH * kUS * (int)sizeof(double2);                    // bytes between atom tiles
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a0 = blockIdx.x * 32 * B;
    for (int t = threadIdx.x; t < 32 * B * NH; t += blockDim.x) {
        const int a = t / NH, e = t - a * NH;
        s_u[(a >> 5) * NH * kUS + e * kUS + (a & 31)] =
            (a0 + a < n) ? U[(long long)(a0 + a) * su + c_hflat[e] * sf] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int beg = chunk[w], end = chunk[w + 1];
    int f = chunkf[w];   // outputs are consecutive inside a warp's range
    const char* su_l = reinterpret_cast<const char*>(s_u + lane);
    ZEntry* se = s_e + w * 32;
    double are[B], aim[B], en[B];
    double2 ug[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
        are[b] = aim[b] = en[b] = 0.0;
        ug[b] = make_double2(0.0, 0.0);
    }
    int last_g = -1;      // products are sorted by g inside an output: half reuse the previous U[g]
    for (int base = beg; base < end; base += 32) {
        if (base + lane < end) se[lane] = ent[base + lane];
        __syncwarp();
        const int cnt = min(32, end - base);
        for (int j = 0; j < cnt; ++j) {
            const ZEntry e = se[j];
            if (e.goff != last_g) {   // warp-uniform
#pragma unroll
                for (int b = 0; b < B; ++b) ug[b] = *reinterpret_cast<const double2*>(su_l + b * kTile + e.goff);
                last_g = e.goff;
            }
            const unsigned cg = ((unsigned)e.hcode << 11) & 0x80000000u, ch = ((unsigned)e.hcode << 10) & 0x80000000u;
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const double2 uh = *reinterpret_cast<const double2*>(su_l + b * kTile + (e.hcode & 0xfffff));
                const double gy = flip_sign(ug[b].y, cg);   // conj_g
                const double hy = flip_sign(uh.y, ch);      // conj_h
                const double tre = ug[b].x * uh.x - gy * hy;
                const double tim = ug[b].x * hy + gy * uh.x;
                are[b] = fma(e.coef, tre, are[b]);
                aim[b] = fma(e.coef, tim, aim[b]);
            }
            if (e.hcode & (1 << 22)) {   // warp-uniform: output f complete
                const double wgt = (e.hcode & (1 << 23)) ? 1.0 : 2.0;
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int a = a0 + 32 * b + lane;
                    if (a < n) Yh[(long long)f * ld + a] = make_double2(are[b], aim[b]);
                    const double2 u = s_u[b * NH * kUS + f * kUS + lane];
                    en[b] += wgt * (are[b] * u.x + aim[b] * u.y);
                    are[b] = aim[b] = 0.0;
                }
                ++f;
            }
        }
        __syncwarp();
    }
    double v[1] = {0.0};
#pragma unroll
    for (int b = 0; b < B; ++b) v[0] += (a0 + 32 * b + lane < n) ? en[b] / 3.0 : 0.0;
    mdkk::block_sum<1, kYW * 32>(v, partials + blockIdx.x);
}

// Reference layout "a": full Y rows [n][NF] from the half/transposed Yh, using
// Y[tj-p][tj-q] = (-1)^(p+q) conj(Y[p][q]).
__global__ void k_snap_y_expand(const double2* __restrict__ Yh, int ld, int n, int nf,
                                const int* __restrict__ fmap, double2* __restrict__ Y, long long su, long long sf) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n * nf) return;
    const int i = (int)(t / nf), f = (int)(t - (long long)i * nf);
    const int m = __ldg(fmap + f);
    double2 v = Yh[(long long)(m & 0xffff) * ld + i];
    if ((m >> 16) & 1) v.y = -v.y;
    if ((m >> 17) & 1) v = make_double2(-v.x, -v.y);
    Y[i * su + f * sf] = v;
}

// Inverse of the expansion (a host-written reference-layout Y -> engine layout).
__global__ void k_snap_y_compress(const double2* __restrict__ Y, int n, int nf, int nh, double2* __restrict__ Yh,
                                  int ld, long long su, long long sf) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n * nh) return;
    const int e = (int)(t / n), i = (int)(t - (long long)e * n);
    Yh[(long long)e * ld + i] = Y[i * su + c_hflat[e] * sf];
}

// ------------------------------------------------------- compute_fused_deidrj
// Reverse-mode form of compute_fused_deidrj (mdkk/snap/compute.py:390-409).
// The reference evaluates t_d = Re sum_f Y[f] conj(d(f_c u[f])/d dr_d) with a
// forward derivative recursion per direction.  Here u runs forward over the
// column halves C_tj (two-term recursion, full mirrored levels kept in shared
// memory) and the adjoint runs backward over the same computational graph:
// with S = Re sum_f conj(Y[f]) u[f], the total adjoint on C_tj is
//   lambda[x] = Y[x] + g(x) + s_x conj(Y[m] + g(m)),   m = mirror(x),
//             = 2 Y[x] + g(x) + s_x conj(g(m))         (x != m; Y is mirror-symmetric)
// where g(y) = sum over the level-(tj+1) elements z in C_{tj+1} that read y of
// conj(coef_z) lambda[z].  The recursion coefficients are conj(a) and b only,
// so dS = Re(G_abar conj(da) + G_b db) with G_abar = sum conj(lambda) w v[P][Q],
// G_b = sum conj(lambda) w v[P-1][Q], and
//   t_d = f_c' rhat_d S + f_c Re(G_abar conj(da_d) + G_b db_d).
// Same quantity (equal to rounding) for ~1/6 of the reference's complex MACs.
// One warp per atom, two neighbours at a time (one per half-warp).
constexpr int kLamMax = 41;   // half_size(8): lambda levels keep only their column-major C prefix
#ifndef MDKK_DE_TEAM
#define MDKK_DE_TEAM 8
#endif
#ifndef MDKK_DE_WARPS
#define MDKK_DE_WARPS 2
#endif
constexpr int kDeTeam = MDKK_DE_TEAM;     // lanes per pair in k_snap_deidrj (4 pairs per warp at 8)
constexpr int kDeWarps = MDKK_DE_WARPS;   // atoms (warps) per CTA

// TEAM lanes expand one pair (32 / TEAM pairs per warp), DW warps (atoms) per CTA.
template <int TWOJ, int TEAM, int DW>
__global__ void __launch_bounds__(DW * 32, (TEAM == 16 ? 4 : 10 / DW)) k_snap_deidrj(const double* __restrict__ x, int n_local,
                                                             const int* __restrict__ table,
                                                             const int* __restrict__ counts, int cap, double rc,
                                                             const double2* __restrict__ Yh, int ld,
                                                             double* __restrict__ f) {
    // levels 0..TWOJ-1 in compact storage (the top is never re-read), +pad for the clamped edge reads
    constexpr int NU = lvl_offset(TWOJ) + TWOJ + 1;
    constexpr int NH = half_offset(TWOJ + 1);
    constexpr int PPW = 32 / TEAM;   // pairs in flight per warp
    extern __shared__ double s_dyn_d[];  // rs | pairs | Y_i (C order) | u levels | lambda C prefixes
    RS& rs = *reinterpret_cast<RS*>(s_dyn_d);
    auto s_nb = reinterpret_cast<NbPair(*)[kNbChunk]>(reinterpret_cast<char*>(s_dyn_d) + sizeof(RS));
    auto s_y = reinterpret_cast<cplx(*)[NH]>(s_nb + DW);
    auto s_u = reinterpret_cast<cplx(*)[PPW][NU]>(s_y + DW);
    auto s_l = reinterpret_cast<cplx(*)[PPW][2][kLamMax]>(s_u + DW);
    // zero the level buffers once: the branch-free edges read finite neighbours
    for (int t = threadIdx.x; t < DW * PPW * (NU + 2 * kLamMax); t += blockDim.x)
        reinterpret_cast<cplx*>(s_u)[t] = {0.0, 0.0};
    stage_rs(rs);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, hl = lane & (TEAM - 1), hh = lane / TEAM;
    const int i = blockIdx.x * DW + w;
    if (i >= n_local) return;
    // Y_i at the column-half elements, in the lanes' (column-major) order, from the row-half Yh
#pragma unroll
    for (int tj = 0; tj <= TWOJ; ++tj)
        for (int c = lane; c < half_size(tj); c += 32) {
            int P, Q;
            col_elem(tj, c, P, Q);
            const int h = P * (tj + 1) + Q;
            const bool mir = h >= half_size(tj);
            const double2 v = Yh[(long long)(half_offset(tj) + (mir ? (tj - P) * (tj + 1) + (tj - Q) : h)) * ld + i];
            const double sg = (mir && ((P + Q) & 1)) ? -1.0 : 1.0;
            s_y[w][half_offset(tj) + c] = {sg * v.x, mir ? -sg * v.y : v.y};
        }
    __syncwarp();
    const cplx* sy = s_y[w];
    cplx* ul = s_u[w][hh];
    cplx(*lam)[kLamMax] = s_l[w][hh];
    const double4 xi = mdkk::ld4(x, i);
    const int n = min(counts[i], cap);
    const double rc2 = rc * rc;
    double fi[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    for (int k0 = 0; k0 < n; k0 += kNbChunk) {
        const int m = compact_pairs(x, table, cap, i, k0, n, xi, rc2, rc, s_nb[w], bad);
        for (int t = 0; t < m; t += PPW) {
            const int pi = t + hh;
            const bool active = pi < m;
            const NbPair nb = s_nb[w][active ? pi : t];
            PairGeo g;
            double z0, r0;
            geo_of(nb, g, z0, r0);
            const cplx ab = cconj(g.a), bb = cconj(g.b);
            // forward: C_tj of every level, S = Re sum_f conj(Y) u (mirror pairs counted twice)
            double S = 0.0;
            if (hl == 0) {
                ul[0] = {1.0, 0.0};
                S = sy[0].re;
            }
            __syncwarp();
#pragma unroll
            for (int tj = 1; tj <= TWOJ; ++tj) {
#pragma unroll
                for (int s = 0; s < tslots<TEAM>(tj); ++s) {
                    const int c = hl + TEAM * s;
                    if (c < half_size(tj)) {
                        int P, Q;
                        col_elem(tj, c, P, Q);
                        const cplx v = rec2(ul + lvl_offset(tj - 1), tj, P, Q, rs, ab, g.b, lvl_size(tj - 1) - 1);
                        if (tj < TWOJ) store_for_next(ul + lvl_offset(tj), tj, P, Q, v);
                        const cplx yv = sy[half_offset(tj) + c];
                        const double wgt = (2 * P == tj && 2 * Q == tj) ? 1.0 : 2.0;
                        S += wgt * (yv.re * v.re + yv.im * v.im);
                    }
                }
                __syncwarp();
            }
            // backward: total adjoint on C_tj from level tj+1, accumulate G_abar, G_b
            cplx Ga = {0, 0}, Gb = {0, 0};
#pragma unroll
            for (int tj = TWOJ; tj >= 1; --tj) {
                cplx* lc = lam[tj & 1];
                const cplx* ln = lam[(tj + 1) & 1];   // level tj+1, column-major (stride tj+2), valid on C_{tj+1}
                const cplx* v = ul + lvl_offset(tj - 1);
#pragma unroll
                for (int s = 0; s < tslots<TEAM>(tj); ++s) {
                    const int c = hl + TEAM * s;
                    if (c < half_size(tj)) {
                        int P, Q;
                        col_elem(tj, c, P, Q);
                        const bool center = 2 * P == tj && 2 * Q == tj;
                        const cplx yv = sy[half_offset(tj) + c];
                        cplx l = center ? yv : cscale(2.0, yv);
                        if (tj < TWOJ) {
                            const int T = tj + 1;
                            // g(x): readers of v[P][Q] at level T are (P, Q) and (P+1, Q), both in C_T
                            const cplx* lq = ln + Q * (T + 1);
                            l = cadd(l, cscale(rs.v[T - P][T - Q], cmul(g.a, lq[P])));
                            l = cadd(l, cscale(rs.v[P + 1][T - Q], cmul(bb, lq[P + 1])));
                            if (!center && Q == (tj >> 1)) {   // g(mirror) is non-zero only in the last column
                                const int mP = tj - P, mQ = tj - Q;
                                const cplx* lm = ln + mQ * (T + 1);
                                cplx gm = {0.0, 0.0};
                                if (in_col_half(T, mP, mQ)) gm = cscale(rs.v[T - mP][T - mQ], cmul(g.a, lm[mP]));
                                if (in_col_half(T, mP + 1, mQ))
                                    gm = cadd(gm, cscale(rs.v[mP + 1][T - mQ], cmul(bb, lm[mP + 1])));
                                l = ((P + Q) & 1) ? cadd(l, cneg(cconj(gm))) : cadd(l, cconj(gm));
                            }
                        }
                        lc[Q * (tj + 1) + P] = l;
                        // zero weights at the column ends (see rec2): no branches
                        const cplx lcj = cconj(l);
                        const cplx t0 = cmul(lcj, v[Q * tj + P]), t1 = cmul(lcj, v[max(Q * tj + P - 1, 0)]);
                        const double w0 = rs.v[tj - P][tj - Q], w1 = rs.v[P][tj - Q];
                        Ga = {fma(w0, t0.re, Ga.re), fma(w0, t0.im, Ga.im)};
                        Gb = {fma(w1, t1.re, Gb.re), fma(w1, t1.im, Gb.im)};
                    }
                }
                __syncwarp();
            }
            cplx da[3], db[3];
            const double d[3] = {nb.dx, nb.dy, nb.dz};
            pair_grads(d, g, rc, z0, r0, da, db);
            double tt[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double v = g.dfc * (d[q] / g.r) * S +
                           g.fc * ((Ga.re * da[q].re + Ga.im * da[q].im) + (Gb.re * db[q].re - Gb.im * db[q].im));
#pragma unroll
                for (int o = TEAM / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                tt[q] = v;
            }
            if (hl == 0 && active) {
                fi[0] += tt[0];
                fi[1] += tt[1];
                fi[2] += tt[2];
                double* fj = f + 4LL * nb.j;
                atomicAdd(fj + 0, -tt[0]);
                atomicAdd(fj + 1, -tt[1]);
                atomicAdd(fj + 2, -tt[2]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int o = 16; o >= TEAM; o >>= 1) fi[q] += __shfl_xor_sync(0xffffffffu, fi[q], o);
    if (lane == 0) {
        double* p = f + 4LL * i;
        atomicAdd(p + 0, fi[0]);
        atomicAdd(p + 1, fi[1]);
        atomicAdd(p + 2, fi[2]);
    }
}

}  // namespace

extern "C" {

int mdkk_snap_create(mdkk_ctx* ctx, int twojmax, int n_entries, const double* coef_host, const int* code_host,
                     int n_half, const int* fmap_host, mdkk_snap** out_host) {
    if (!ctx || !out_host || twojmax < 0 || twojmax > kMaxTwoJ || n_entries < 1 || !coef_host || !code_host ||
        n_half != half_offset(twojmax + 1)) {
        mdkk::set_error("mdkk_snap_create: 2J must be in [0, 8] with a non-empty product list");
        return MDKK_E_ARG;
    }
    // host copy of the list + output-aligned per-warp chunks balanced on entry counts
    std::vector<ZEntry> h(n_entries);
    std::vector<int> ends;  // entry index one past each output
    std::vector<int> fout(n_entries);
    for (int k = 0; k < n_entries; ++k) {
        const int c = code_host[k];
        const int g = c & 255, hh = (c >> 8) & 255;
        fout[k] = (c >> 16) & 255;
        h[k].coef = coef_host[k];
        h[k].goff = g * kUS * (int)sizeof(double2);
        h[k].hcode = hh * kUS * (int)sizeof(double2) | ((c >> 24) & 1) << 20 | ((c >> 25) & 1) << 21 |
                     ((c >> 26) & 1) << 22 | ((c >> 27) & 1) << 23;
        if (c & (1 << 26)) ends.push_back(k + 1);
    }
    if (ends.empty() || ends.back() != n_entries) {
        mdkk::set_error("mdkk_snap_create: product list must end on an output boundary");
        return MDKK_E_ARG;
    }
    std::vector<int> chunk(kYW + 1, n_entries);
    chunk[0] = 0;
    {
        size_t o = 0;
        for (int w = 1; w < kYW; ++w) {
            const double target = (double)n_entries * w / kYW;
            while (o < ends.size() && ends[o] < target) ++o;
            chunk[w] = o < ends.size() ? std::max(chunk[w - 1], ends[o]) : n_entries;
            if (o < ends.size() && o > 0 && (ends[o] - target) > (target - ends[o - 1]))
                chunk[w] = std::max(chunk[w - 1], ends[o - 1]);
        }
    }
    std::vector<int> chunkf(kYW);
    for (int w = 0; w < kYW; ++w) chunkf[w] = chunk[w] < n_entries ? fout[chunk[w]] : 0;
    auto* s = new mdkk_snap();
    s->twojmax = twojmax;
    s->n_flat = block_offset(twojmax + 1);
    s->n_half = n_half;
    s->n_entries = n_entries;
    cudaError_t e = cudaMalloc(&s->ent, sizeof(ZEntry) * n_entries);
    if (e == cudaSuccess) e = cudaMalloc(&s->chunk, sizeof(int) * (kYW + 1));
    if (e == cudaSuccess) e = cudaMalloc(&s->chunkf, sizeof(int) * kYW);
    if (e == cudaSuccess) e = cudaMalloc(&s->fmap, sizeof(int) * s->n_flat);
    if (e == cudaSuccess) e = cudaMemcpy(s->ent, h.data(), sizeof(ZEntry) * n_entries, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->chunk, chunk.data(), sizeof(int) * (kYW + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->chunkf, chunkf.data(), sizeof(int) * kYW, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->fmap, fmap_host, sizeof(int) * s->n_flat, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(s->ent);
        cudaFree(s->chunk);
        cudaFree(s->chunkf);
        cudaFree(s->fmap);
        delete s;
        return mdkk::cuda_fail(e, "mdkk_snap_create");
    }
    upload_weights();
    *out_host = s;
    return MDKK_OK;
}

int mdkk_snap_set_schedule(mdkk_snap* s, int batch_u, int batch_y) {
    if (!s || batch_u < 1 || batch_y < 1) return MDKK_E_ARG;
    s->ui_ppw = batch_u >= 8 ? 4 : (batch_u >= 4 ? 2 : 1);   // batch_u pairs per 64 lanes
    s->yi_batch = batch_y >= 2 ? 2 : 1;
    return MDKK_OK;
}

int mdkk_snap_destroy(mdkk_snap* s) {
    if (!s) return MDKK_OK;
    cudaFree(s->ent);
    cudaFree(s->chunk);
    cudaFree(s->chunkf);
    cudaFree(s->fmap);
    cudaFree(s->work);
    delete s;
    return MDKK_OK;
}

int mdkk_snap_ui(mdkk_snap* s, const double* x, int n_local, const int* table, const int* counts, int cap, double rc,
                 double* U, int layout, int ldu, int* flags, void* stream) {
    if (!s || n_local < 0 || cap < 1 || (layout == 1 && ldu < n_local)) return MDKK_E_ARG;
    const long long su = layout ? 1 : s->n_flat, sf = layout ? ldu : 1;
    if (n_local == 0) return MDKK_OK;
    upload_weights();
    cudaStream_t st = mdkk::as_stream(stream);
    double2* u = reinterpret_cast<double2*>(U);
    // batch_u: pairs expanded concurrently per warp -> team width (DW atoms per CTA)
    const int team = s->ui_ppw >= 4 ? 8 : (s->ui_ppw >= 2 ? 16 : 32);
#define MDKK_UI_T(TJ, TM)                                                                                     \
    {                                                                                                         \
        constexpr int DW = TM == 16 ? 4 : 2;                                                                  \
        k_snap_ui<TJ, TM, DW><<<(n_local + DW - 1) / DW, DW * 32, 0, st>>>(x, n_local, table, counts, cap, rc, \
                                                                          u, su, sf, flags);                  \
    }
#define MDKK_UI(TJ)                                                                                           \
    case TJ:                                                                                                  \
        if (team == 8) MDKK_UI_T(TJ, 8) else if (team == 16) MDKK_UI_T(TJ, 16) else MDKK_UI_T(TJ, 32)         \
        break;
    switch (s->twojmax) {
        MDKK_UI(0) MDKK_UI(1) MDKK_UI(2) MDKK_UI(3) MDKK_UI(4) MDKK_UI(5) MDKK_UI(6) MDKK_UI(7) MDKK_UI(8)
#undef MDKK_UI
#undef MDKK_UI_T
        default: return MDKK_E_ARG;
    }
    MDKK_CHECK_LAUNCH("k_snap_ui");
    return MDKK_OK;
}

int mdkk_snap_yi(mdkk_ctx* ctx, mdkk_snap* s, const double* U, int n_local, double* Yh, int ld, double* energy,
                 int layout, int ldu, void* stream) {
    if (!ctx || !s || n_local < 0 || ld < n_local || (layout == 1 && ldu < n_local)) return MDKK_E_ARG;
    const long long su = layout ? 1 : s->n_flat, sf = layout ? ldu : 1;
    cudaStream_t st = mdkk::as_stream(stream);
    if (n_local == 0) {
        cudaMemsetAsync(energy, 0, sizeof(double), st);
        return MDKK_OK;
    }
    upload_weights();
    const int B = s->yi_batch == 2 ? 2 : 1;
    const int nb = (n_local + 32 * B - 1) / (32 * B);
    double* partials = static_cast<double*>(mdkk::scratch(ctx, sizeof(double) * (size_t)nb));
    if (!partials) return mdkk::cuda_fail(cudaErrorMemoryAllocation, "scratch");
    const double2* u = reinterpret_cast<const double2*>(U);
    double2* y = reinterpret_cast<double2*>(Yh);
    switch (s->twojmax) {
#define MDKK_YI_B(TJ, BB)                                                                                       \
    {                                                                                                           \
        constexpr int NF = block_offset(TJ + 1), NH = half_offset(TJ + 1);                                      \
        const size_t sm = BB * NH * kUS * sizeof(double2) + kYW * 32 * sizeof(ZEntry);                          \
        cudaFuncSetAttribute(k_snap_yi<NF, NH, BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
        k_snap_yi<NF, NH, BB><<<nb, kYW * 32, sm, st>>>(u, n_local, s->ent, s->chunk, s->chunkf, y, ld,        \
                                                        partials, su, sf);                                      \
    }
#define MDKK_YI(TJ)                                                                                             \
    case TJ:                                                                                                    \
        if (B == 2) MDKK_YI_B(TJ, 2) else MDKK_YI_B(TJ, 1)                                                      \
        break;
        MDKK_YI(0) MDKK_YI(1) MDKK_YI(2) MDKK_YI(3) MDKK_YI(4) MDKK_YI(5) MDKK_YI(6) MDKK_YI(7) MDKK_YI(8)
#undef MDKK_YI
#undef MDKK_YI_B
        default: return MDKK_E_ARG;
    }
    MDKK_CHECK_LAUNCH("k_snap_yi");
    mdkk::reduce_partials(partials, nb, 1, energy, st);
    MDKK_CHECK_LAUNCH("k_reduce_partials");
    return MDKK_OK;
}

int mdkk_snap_y_expand(mdkk_snap* s, const double* Yh, int ld, int n_local, double* Y, int layout, int ldy,
                       void* stream) {
    if (!s || n_local < 0 || ld < n_local || (layout == 1 && ldy < n_local)) return MDKK_E_ARG;
    const long long su = layout ? 1 : s->n_flat, sf = layout ? ldy : 1;
    if (n_local == 0) return MDKK_OK;
    const long long tot = (long long)n_local * s->n_flat;
    k_snap_y_expand<<<(unsigned)((tot + 255) / 256), 256, 0, mdkk::as_stream(stream)>>>(
        reinterpret_cast<const double2*>(Yh), ld, n_local, s->n_flat, s->fmap, reinterpret_cast<double2*>(Y), su, sf);
    MDKK_CHECK_LAUNCH("k_snap_y_expand");
    return MDKK_OK;
}

int mdkk_snap_y_compress(mdkk_snap* s, const double* Y, int n_local, double* Yh, int ld, int layout, int ldy,
                         void* stream) {
    if (!s || n_local < 0 || ld < n_local || (layout == 1 && ldy < n_local)) return MDKK_E_ARG;
    const long long su = layout ? 1 : s->n_flat, sf = layout ? ldy : 1;
    if (n_local == 0) return MDKK_OK;
    upload_weights();
    const long long tot = (long long)n_local * s->n_half;
    k_snap_y_compress<<<(unsigned)((tot + 255) / 256), 256, 0, mdkk::as_stream(stream)>>>(
        reinterpret_cast<const double2*>(Y), n_local, s->n_flat, s->n_half, reinterpret_cast<double2*>(Yh), ld, su, sf);
    MDKK_CHECK_LAUNCH("k_snap_y_compress");
    return MDKK_OK;
}

int mdkk_snap_deidrj(mdkk_snap* s, const double* x, int n_local, const int* table, const int* counts, int cap,
                     double rc, const double* Yh, int ld, double* f, void* stream) {
    if (!s || n_local < 0 || cap < 1 || ld < n_local) return MDKK_E_ARG;
    if (n_local == 0) return MDKK_OK;
    upload_weights();
    switch (s->twojmax) {
#define MDKK_DE(TJ)                                                                                          \
    case TJ: {                                                                                               \
        constexpr int TEAM = kDeTeam, DW = kDeWarps, PPW = 32 / TEAM;                                        \
        const size_t sm = sizeof(RS) + DW * (kNbChunk * sizeof(NbPair) +                                     \
            (half_offset(TJ + 1) + PPW * (lvl_offset(TJ) + TJ + 1 + 2 * kLamMax)) *                           \
            sizeof(cplx));                                                                                   \
        cudaFuncSetAttribute(k_snap_deidrj<TJ, TEAM, DW>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                             (int)sm);                                                                       \
        k_snap_deidrj<TJ, TEAM, DW><<<(n_local + DW - 1) / DW, DW * 32, sm, mdkk::as_stream(stream)>>>(      \
            x, n_local, table, counts, cap, rc, reinterpret_cast<const double2*>(Yh), ld, f);                \
        break;                                                                                               \
    }
        MDKK_DE(0) MDKK_DE(1) MDKK_DE(2) MDKK_DE(3) MDKK_DE(4) MDKK_DE(5) MDKK_DE(6) MDKK_DE(7) MDKK_DE(8)
#undef MDKK_DE
        default: return MDKK_E_ARG;
    }
    MDKK_CHECK_LAUNCH("k_snap_deidrj");
    return MDKK_OK;
}

int mdkk_snap_compute(mdkk_ctx* ctx, mdkk_snap* s, const double* x, int n_local, const int* table, const int* counts,
                      int cap, double rc, double* U, double* Yh, double* f, double* energy, int* flags,
                      void* stream) {
    if (!ctx || !s || n_local < 0 || cap < 1 || !f || !energy || !flags) return MDKK_E_ARG;
    if ((U == nullptr) != (Yh == nullptr)) return MDKK_E_ARG;
    if (!U) {   // handle-owned workspace, grown on demand and kept for the next step
        const size_t need = (size_t)n_local * (s->n_flat + s->n_half) * sizeof(double2);
        if (need > s->work_bytes) {
            cudaFree(s->work);
            s->work = nullptr;
            s->work_bytes = 0;
            cudaError_t e = cudaMalloc(&s->work, need + need / 4);
            if (e != cudaSuccess) return mdkk::cuda_fail(e, "mdkk_snap_compute workspace");
            s->work_bytes = need + need / 4;
        }
        U = s->work;
        Yh = s->work + (size_t)n_local * s->n_flat * 2;
    }
    int rc_ = mdkk_snap_ui(s, x, n_local, table, counts, cap, rc, U, 0, 0, flags, stream);
    if (rc_ != MDKK_OK) return rc_;
    rc_ = mdkk_snap_yi(ctx, s, U, n_local, Yh, n_local, energy, 0, 0, stream);
    if (rc_ != MDKK_OK) return rc_;
    return mdkk_snap_deidrj(s, x, n_local, table, counts, cap, rc, Yh, n_local, f, stream);
}

}  // extern "C"
