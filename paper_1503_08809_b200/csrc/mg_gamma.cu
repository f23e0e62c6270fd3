// mg_gamma.cu — separable Γ on the tetrahedral domain, row-factorised onto DMMA GEMMs.
//
// Reference: engine3d.py:86-136 (_block_accumulate / _sweep_chunk): per triple t,
//   P[n,t]  = Σ_6perms q q q,  X[n',t] = zm_t Σ_x wr2_x Σ_6perms q̃ q̃ q̃,  Γ += P Xᵀ.
// The reference spends 96-98% of its time building X (engine3d.py:115-116).
//
// B200 formulation.  Single out l1 (the smallest multipole) and group the
// ordered triples into (l2,l3)-rows; l1 runs over a parity class window of the row.  With
// pair sums Sq_ab = q_a(l2)q_b(l3) + q_b(l2)q_a(l3), S_ab(x) = q̃_a(x,l2)q̃_b(x,l3) + (a<->b):
//   P[(ijk),t]     = q_k(l1) Sq_ij + q_j(l1) Sq_ik + q_i(l1) Sq_jk
//   f[(i'j'k'),x,t] = q̃_k'(x,l1) S_i'j'(x) + q̃_j'(x,l1) S_i'k'(x) + q̃_i'(x,l1) S_j'k'(x)
// so, contracting the l1-run first and x second,
//   H_row[c,c',x]   = Σ_{l1} zm(l1,l2,l3) q_c(l1) wr2_x q̃_c'(x,l1)        (K1, GEMM over l1)
//   G_row[ab',c,c'] = Σ_x S_ab'(x) H_row[c,c',x]                           (K2, GEMM over x)
//   Z[ab,c,n']     += Σ_rows Sq_ab(row) Σ_{(a'b',c'') ∈ dec(n')} G_row[a'b',c,c'']  (K3, GEMM over rows)
//   Γ[(ijk),n']     = Z[ij,k,n'] + Z[ik,j,n'] + Z[jk,i,n']                   (final gather)
// All three contractions are FP64 DMMA block GEMMs (mg_dmma.cuh) whose operand loaders
// generate the pair products / weights / gathers on the fly.  No atomics: every output tile
// is owned by exactly one CTA per launch and rows are reduced in a fixed order, so a run is
// bitwise reproducible.
#include <algorithm>
#include <memory>
#include <mutex>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "mg_dmma.cuh"
#include "mg_gamma.cuh"

namespace mg {

#ifndef MG_RUN_WARPS
#define MG_RUN_WARPS 12  // consumer warps of the 128 x 96 run/pair tile: 12 (32x32 per warp) or 16
#endif
// Checked build (MG_CHECKED=1: tools/build_variant.sh checked -DMG_CHECKED=1).  compute-
// sanitizer is closed on this pool, so the pipeline kernels carry their own bounds checks:
// every global-memory write and every bulk-copy (TMA) source range is checked against the
// extent of its buffer, and violations are COUNTED per check site (no trap, no fault),
// read back through mg_debug_checks().  In the normal build the checks compile to nothing.
#ifndef MG_CHECKED
#define MG_CHECKED 0
#endif
struct MgBounds {  // buffer extents in doubles (0 = unchecked)
    int64_t panel, wqb, h, s, g, r, sq, z, qts, q1w;
};
enum MgCheck {
    CK_PANEL_W, CK_K1_PANEL, CK_K1_WQB, CK_K1_H_W, CK_S_W, CK_K2_S, CK_K2_H, CK_K2_G_W,
    CK_GATHER_W, CK_K3_SQ, CK_K3_R, CK_K3_Z_W, CK_NS_QTS, CK_NS_Q1W, CK_NS_L, CK_COUNT
};
#if MG_CHECKED
static __device__ unsigned int g_chk[16];
#define MG_DCHECK(cond, site)                                  \
    do {                                                       \
        if (!(cond)) atomicAdd(&g_chk[(int)(site)], 1u);       \
    } while (0)
#else
#define MG_DCHECK(cond, site) \
    do {                      \
    } while (0)
#endif
// [lo, lo + n) inside [0, extent)
__device__ __forceinline__ bool in_range(int64_t lo, int64_t n, int64_t extent) {
    return lo >= 0 && n >= 0 && lo + n <= extent;
}

constexpr int RUN_TN = 96;              // run-contraction N tile ((c', x) columns)
constexpr int RUN_TM_ = 128;            // (row, c) slots per tile
constexpr int RUN_LDB = RUN_TN + 4;     // smem-identical row stride of WQB rows
constexpr int RUN_LDA = RUN_TM_ + 4;    // smem-identical row stride of the A panels

// ------------------------------------------------------------------------------------------
// setup kernels
// ------------------------------------------------------------------------------------------

// QT[l][c][x] = q̃[c][x][l]  (x zero-padded to NxP), and the run contraction's B operand
// WQB: for parity class par, column block nb of RUN_TN columns n = c*Nxw + x,
//   WQB[base[par] + (nb*Rpar + j)*RUN_LDB + n%RUN_TN] = wr2[x] q̃[c][x][l],  l = l0(par) + 2j
// (Rpar = class size + RUN_BK zero rows; smem-identical rows, so a stage is one bulk copy)
__global__ void k_transpose_qt(const double* __restrict__ qt, const double* __restrict__ wr2,
                               int p, int Nx, int NxP, int Nxw, int L, int l_min,
                               longlong2 wbase, int2 wrows, double* __restrict__ QT,
                               double* __restrict__ WQT) {
    int64_t total = (int64_t)L * p * NxP;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int x = (int)(i % NxP);
        int64_t r = i / NxP;
        int c = (int)(r % p);
        int li = (int)(r / p);
        double val = x < Nx ? qt[((int64_t)c * Nx + x) * L + li] : 0.0;
        QT[i] = val;
        const int l = l_min + li, par = l & 1;
        const int j = (l - (l_min + ((l_min ^ par) & 1))) / 2;
        if (x < Nxw) {
            const int n = c * Nxw + x, nb = n / RUN_TN;
            const int64_t o = (par ? wbase.y : wbase.x) +
                              ((int64_t)nb * (par ? wrows.y : wrows.x) + j) * RUN_LDB + n % RUN_TN;
            WQT[o] = x < Nx ? wr2[x] * val : 0.0;
        }
    }
}

// ------------------------------------------------------------------------------------------
// K0: explicit-triple weights (only for arbitrary domains): ZT pre-zeroed, zm scattered
// ------------------------------------------------------------------------------------------
__global__ void k_scatter_weights(const int32_t* __restrict__ t1, const int32_t* __restrict__ t2,
                                  const int32_t* __restrict__ t3, const int64_t* __restrict__ pos,
                                  const double* __restrict__ dup, int64_t n, int64_t zbase,
                                  int l_min, const double* __restrict__ C,
                                  const double* __restrict__ v, const double* __restrict__ lf,
                                  int mode, double* __restrict__ ZT) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        ZT[pos[i] - zbase] = dup[i] * zm_weight(mode, t1[i], t2[i], t3[i], C, v, l_min, lf);
}

// ------------------------------------------------------------------------------------------
// K1a: A panels of the run contraction, one per M-tile, k-major [jl][slot]:
//   panel[jl][slot=(r,c)] = zm(l1(j), l2_r, l3_r) q_c(l1(j))  (0 outside row r's window)
// ------------------------------------------------------------------------------------------
#ifndef MG_SIDE  // operand kernels on the side stream: 0 none, 1 pair products, 2 + panels
#define MG_SIDE 1
#endif
#ifndef MG_NB1
#define MG_NB1 8288  // rows per run/x-contraction batch (upper bound; 148 x 56)
#endif
#ifndef MG_NB3
#define MG_NB3 16576  // rows per pair-contraction group (upper bound)
#endif
#ifndef MG_HBUDGET
#define MG_HBUDGET 24.0e9  // bytes of H per batch (S gets half, G as much); HBM is 180 GB
#endif
#ifndef MG_NO_EPI
#define MG_NO_EPI 0  // diagnostics only: 1 skips the run/x contraction output stores
#endif
#ifndef MG_RUN_BK
#define MG_RUN_BK 32
#define MG_RUN_ST 3
#endif
constexpr int RUN_BK = MG_RUN_BK, RUN_ST = MG_RUN_ST;
constexpr int X_BK = 32;
constexpr int X_LDK = X_BK + 4;  // x-blocked S/H row stride: [row][x/32][m][36], smem-identical
using CfgX120 = TileCfg<5, 3, 3, 5>;  // 120 x 120, 15 warps, 30 accumulators per lane
// run contraction: 128 packed (row,c) slots x 96 columns; the consumer warps are a multiple
// of 4 so every SM sub-partition's DMMA unit serves the same number of warps
#if MG_RUN_WARPS == 12
// 12 consumer warps (3 per SM sub-partition, 4x4 fragments each) + 1 producer: 13 warps
// allocate 128 registers per thread, so the accumulators and double-buffered fragments fit
// without spills (16 consumer warps + producer cap at 96 and spill)
using CfgRun = TileCfg<4, 3, 4, 4>;
#else
using CfgRun = TileCfg<4, 4, 4, 3>;
#endif
constexpr int RUN_TM = CfgRun::BM;     // (row, c) slots per run tile = A panel width
static_assert(RUN_TN == CfgRun::BN && RUN_TM == RUN_TM_ && RUN_LDA == ld_kmajor(RUN_TM) &&
                  RUN_LDB == ld_kmajor(RUN_TN),
              "bulk-copied run tiles must match the shared-memory layout");
constexpr int PANEL_THREADS = 256;
constexpr int PANEL_JC = 32;  // j values per shared-memory weight chunk

// Slot s (0 <= s < 128) of tile tl is (row, c) = (row0 + (c0 + s) / p, (c0 + s) % p).
__global__ void __launch_bounds__(PANEL_THREADS)
k_run_panels(const MgTile* __restrict__ tiles, const MgRow* __restrict__ rows,
             const int64_t* __restrict__ poff, const int64_t* __restrict__ zoff, int64_t zbase,
             const double* __restrict__ ZT, const int* __restrict__ l0,
             const double* __restrict__ q, int L, int l_min, int p,
             const double* __restrict__ C, const double* __restrict__ v,
             const double* __restrict__ lf, const double* __restrict__ fl, int mode,
             double* __restrict__ panel, unsigned magic_p, MgBounds bd) {
    extern __shared__ double zs[];  // [nrows][PANEL_JC]: zm of (row, j) for this chunk
    const MgTile tl = tiles[blockIdx.x];
    const int kt = (tl.jhi - tl.jlo + RUN_BK) / RUN_BK * RUN_BK;
    double* out = panel + poff[blockIdx.x];
    const int par = rows[tl.row0].par;
    {  // one block per (tile, chunk of PANEL_JC j values)
        const int jc = blockIdx.y * PANEL_JC;
        if (jc >= kt) return;
        // 1) each (row, j) weight once
        for (int e = threadIdx.x; e < tl.nrows * PANEL_JC; e += PANEL_THREADS) {
            const int rr = e / PANEL_JC, jl = e % PANEL_JC;
            const int j = tl.jlo + jc + jl;
            const MgRow rw = rows[tl.row0 + rr];
            double z = 0.0;
            if (jc + jl < kt && j >= rw.jlo && j <= rw.jhi) {
                if (ZT) {
                    z = ZT[zoff[tl.row0 + rr] - zbase + (j - rw.jlo)];
                } else {
                    const int l1 = l0[rw.par] + 2 * j;
                    z = mode == 0 ? zm_gosper_fast(l1, rw.l2, rw.l3, fl, l_min)
                                  : zm_weight(mode, l1, rw.l2, rw.l3, C, v, l_min, lf);
                }
            }
            zs[rr * PANEL_JC + jl] = z;
        }
        __syncthreads();
        // 2) panel[j][slot] = zm(row(slot), j) * q_c(slot)(l1(j)), slot-contiguous stores
        for (int e = threadIdx.x; e < PANEL_JC * RUN_TM; e += PANEL_THREADS) {
            const int jl = e / RUN_TM, slot = e % RUN_TM;
            if (jc + jl >= kt) break;
            double val = 0.0;
            if (slot < tl.nslots) {
                const int cm = tl.c0 + slot, rr = (int)(((unsigned)cm * magic_p) >> 16),
                          c = cm - rr * p;  // (c0 + slot) / p, % p (exact: cm < p + 128)
                const double z = zs[rr * PANEL_JC + jl];
                if (z != 0.0) {
                    const int l1 = l0[par] + 2 * (tl.jlo + jc + jl);
                    val = z * q[(int64_t)c * L + (l1 - l_min)];
                }
            }
            MG_DCHECK(in_range(poff[blockIdx.x] + (int64_t)(jc + jl) * RUN_LDA + slot, 1, bd.panel),
                      CK_PANEL_W);
            out[(int64_t)(jc + jl) * RUN_LDA + slot] = val;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// K1: run contraction  H[slot][(c',x)] = Σ_j panel[j][slot] WQT[cls+j][(c',x)]
//   slot = (row, c) flattened over the batch; WQT rows are p*Nxw wide (x unpadded when Nx is
//   even); H rows are [c'][NxP] (x padded to the x-contraction's BK, pads stay zero).
// ------------------------------------------------------------------------------------------
// Persistent run contraction: item it = tile * NB + column block; items are strided over the
// CTAs (one per SM).  The producer warp streams the next item while consumers write H.
struct RunItems {
    static constexpr bool kComputeA = false;
    MgBounds bd;
    const MgTile* tiles;
    const int64_t* poff;
    const double* panel;
    const MgRow* rows;
    const double* WQB;
    longlong2 wbase;
    int2 wrows;
    int NB;
    int ldb;  // p * Nxw columns
    __device__ int ktiles(int it) const {
        const MgTile& t = tiles[it / NB];
        return (t.jhi - t.jlo + RUN_BK) / RUN_BK;
    }
    __device__ int2 valid_mn(int it) const {
        const int ti = it / NB;
        return make_int2(tiles[ti].nslots, min(RUN_TN, ldb - (it - ti * NB) * RUN_TN));
    }
    __device__ int kvalid_last(int it) const {
        const MgTile& t = tiles[it / NB];
        const int nk = t.jhi - t.jlo + 1;
        return nk - (nk - 1) / RUN_BK * RUN_BK;
    }
    __device__ uint32_t stage_bytes(int, int) const {
        return RUN_BK * (RUN_LDA + RUN_LDB) * (uint32_t)sizeof(double);
    }
    __device__ void bulk_rows(int it, int kt, double* As, double* Bs, int lane,
                              uint64_t* bar) const {
        if (lane > 1) return;
        const int ti = it / NB, nb = it - ti * NB;
        const MgTile& t = tiles[ti];
        if (lane == 0) {
            MG_DCHECK(in_range(poff[ti] + (int64_t)kt * RUN_BK * RUN_LDA, RUN_BK * RUN_LDA, bd.panel),
                      CK_K1_PANEL);
            bulk_g2s(As, panel + poff[ti] + (int64_t)kt * RUN_BK * RUN_LDA,
                     RUN_BK * RUN_LDA * sizeof(double), bar);
        } else {
            const int par = rows[t.row0].par;
            const int64_t wo = (par ? wbase.y : wbase.x) +
                               ((int64_t)nb * (par ? wrows.y : wrows.x) + t.jlo + kt * RUN_BK) *
                                   RUN_LDB;
            MG_DCHECK(in_range(wo, RUN_BK * RUN_LDB, bd.wqb), CK_K1_WQB);
            bulk_g2s(Bs, WQB + wo, RUN_BK * RUN_LDB * sizeof(double), bar);
        }
    }
};
using RunPipeP = PipeTMAPersistent<CfgRun, RUN_BK, RUN_ST, true, true, true>;

__global__ void __launch_bounds__(RunPipeP::THREADS, 1)
k_run_contract(const MgTile* __restrict__ tiles, int ntiles, const int64_t* __restrict__ poff,
               const double* __restrict__ panel, int row_base, const MgRow* __restrict__ rows,
               const double* __restrict__ WQB, int p, int Nx, int Nxw, int NxP,
               longlong2 wbase, int2 wrows, double* __restrict__ H, unsigned magic_p,
               unsigned magic_nx, MgBounds bd) {
    extern __shared__ __align__(16) double smem[];
    const int64_t ldb = (int64_t)p * Nxw;
    RunItems items{bd, tiles, poff, panel, rows, WQB, wbase, wrows,
                   (int)((ldb + RUN_TN - 1) / RUN_TN), (int)ldb};
    const int nitems = ntiles * items.NB;
    const int64_t pp = (int64_t)p * p;
    const int XB = NxP / X_BK;
    RunPipeP::run(blockIdx.x, gridDim.x, nitems, items, [&](int it, const Acc<CfgRun>& acc) {
        const int ti = it / items.NB, nb = it - ti * items.NB;
        const MgTile tl = tiles[ti];
        const int n0 = nb * RUN_TN;
        // Per-thread offsets, computed once per item (no divisions at all):
        // slot (rr, c) -> (rr*XB*pp + c*p)*X_LDK ; column gn = c'*Nxw + x ->
        // ((x/32)*pp + c')*X_LDK + x%32   (Nxw even: columns gn, gn+1 share c' and x-block)
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int wm = (warp / CfgRun::WARPS_N) * (8 * CfgRun::FM) + (lane >> 2);
        const int wn = (warp % CfgRun::WARPS_N) * (8 * CfgRun::FN) + 2 * (lane & 3);
        int64_t roff[CfgRun::FM];
        bool rok[CfgRun::FM];
#pragma unroll
        for (int fm = 0; fm < CfgRun::FM; ++fm) {
            const int m = wm + fm * 8;
            // (c0 + m) / p by multiply-shift (c0 + m < p + 128: exact with a 16-bit magic)
            const int cm = tl.c0 + m, dq = (int)(((unsigned)cm * magic_p) >> 16);
            const int rr = tl.row0 - row_base + dq, c = cm - dq * p;
            rok[fm] = m < tl.nslots;
            roff[fm] = ((int64_t)rr * XB * pp + (int64_t)c * p) * X_LDK;
        }
#pragma unroll
        for (int fn = 0; fn < CfgRun::FN; ++fn) {
            const int gn = n0 + wn + fn * 8;
            const int cp = (int)__umulhi((unsigned)gn, magic_nx), x = gn - cp * Nxw;  // gn / Nxw
            const bool both = gn < ldb && x + 1 < Nx, one = gn < ldb && x < Nx;
            const int64_t coff = ((int64_t)(x / X_BK) * pp + cp) * X_LDK + (x & (X_BK - 1));
#pragma unroll
            for (int fm = 0; fm < CfgRun::FM; ++fm) {
                if (!rok[fm] || MG_NO_EPI) continue;
                double* h = H + roff[fm] + coff;
                MG_DCHECK(!one || in_range(roff[fm] + coff, both ? 2 : 1, bd.h), CK_K1_H_W);
                if (both) {
                    *reinterpret_cast<double2*>(h) =
                        make_double2(acc.c[fm][fn][0], acc.c[fm][fn][1]);
                } else if (one) {
                    h[0] = acc.c[fm][fn][0];
                }
            }
        }
    }, smem);
}

// ------------------------------------------------------------------------------------------
// K2: x contraction  G[r][(c,c')][ab] = Σ_x S_ab(x) H[r][(c,c')][x]
//   K2a writes the pair products S[r][ab][x] = q̃_a(x,l2)q̃_b(x,l3) + q̃_b(x,l2)q̃_a(x,l3) of the
//   batch (elementwise, <2 % of K2's time in bytes), so K2 is a pure cp.async GEMM with both
//   operands m-major (x contiguous).  The CTA tile is chosen per config to minimise padding
//   of M = p(p+1)/2 and N = p^2 (120x120 for p = 15, 30; 128x128 for p = 22).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void pair_of(int pr, int& a, int& b) {
    int bb = (int)((sqrt(8.0 * pr + 1.0) - 1.0) * 0.5);
    while ((bb + 1) * (bb + 2) / 2 <= pr) ++bb;
    while (bb * (bb + 1) / 2 > pr) --bb;
    b = bb;
    a = pr - bb * (bb + 1) / 2;
}
__host__ __device__ __forceinline__ int pair_idx(int a, int b) {  // a <= b
    return b * (b + 1) / 2 + a;
}

constexpr int PP_CHUNK = 16;  // pairs per block of the pair-product kernel

// K2a: S[r][ab][x] = q̃_a(x,l2)q̃_b(x,l3) + q̃_b(x,l2)q̃_a(x,l3) in the x-blocked layout of the
// x contraction.  One block per (row, chunk of 16 pairs); a thread owns an x pair (double2) and
// walks the chunk b-major: q̃_b(l2), q̃_b(l3) stay in registers while four a's are loaded at once.
#ifndef MG_PP_THREADS
#define MG_PP_THREADS 128
#endif
#ifndef MG_PP_MAXREG
#define MG_PP_MAXREG 32
#endif
#ifndef MG_PP_UNROLL
#define MG_PP_UNROLL 2
#endif
// 128 threads x <= 32 registers: one warp per SM sub-partition, 1024 registers each.  Beside
// the 13-warp x 128-register run contraction no side CTA of any size is placed (registers are
// allocated per CTA in units of 4 warps, so 13 warps take the whole file: tools/coresidency.cu,
// profiles/r02_coresidency.txt), so the side stream fills the contractions' tails — capping
// the run contraction at 120 registers to make room was measured slower.
__global__ void __maxnreg__(MG_PP_MAXREG)
k_pair_products(const MgRow* __restrict__ rows, int row_b1, const double* __restrict__ QT,
                int p, int P2, int NxP, int l_min, double* __restrict__ S, MgBounds bd) {
    const int r = blockIdx.y;
    const MgRow rw = rows[row_b1 + r];
    const double2* q2 = reinterpret_cast<const double2*>(QT + (int64_t)(rw.l2 - l_min) * p * NxP);
    const double2* q3 = reinterpret_cast<const double2*>(QT + (int64_t)(rw.l3 - l_min) * p * NxP);
    double* out = S + (int64_t)r * P2 * (NxP / X_BK) * X_LDK;
    const int nx2 = NxP / 2;
    const int pr0 = blockIdx.x * PP_CHUNK, pr1 = min(pr0 + PP_CHUNK, P2);
    int a0, b0;
    pair_of(pr0, a0, b0);
    for (int x = threadIdx.x; x < nx2; x += blockDim.x) {
        const int xx = 2 * x;
        double* o = out + (int64_t)(xx / X_BK) * P2 * X_LDK + (xx & (X_BK - 1));
        int a = a0, b = b0, pr = pr0;
        while (pr < pr1) {
            const double2 ub = __ldg(q2 + b * nx2 + x), wb = __ldg(q3 + b * nx2 + x);
            const int na = min(b + 1 - a, pr1 - pr);  // pairs (a .. a+na-1, b)
            int i = 0;
            for (; i + MG_PP_UNROLL <= na; i += MG_PP_UNROLL) {
                double2 u[MG_PP_UNROLL], w[MG_PP_UNROLL];
#pragma unroll
                for (int k = 0; k < MG_PP_UNROLL; ++k) {
                    u[k] = __ldg(q2 + (a + i + k) * nx2 + x);
                    w[k] = __ldg(q3 + (a + i + k) * nx2 + x);
                }
#pragma unroll
                for (int k = 0; k < MG_PP_UNROLL; ++k) {
                    MG_DCHECK(in_range(o + (int64_t)(pr + i + k) * X_LDK - S, 2, bd.s), CK_S_W);
                }
#pragma unroll
                for (int k = 0; k < MG_PP_UNROLL; ++k)
                    *reinterpret_cast<double2*>(o + (int64_t)(pr + i + k) * X_LDK) =
                        make_double2(u[k].x * wb.x + ub.x * w[k].x, u[k].y * wb.y + ub.y * w[k].y);
            }
            for (; i < na; ++i) {
                const double2 u = __ldg(q2 + (a + i) * nx2 + x), w = __ldg(q3 + (a + i) * nx2 + x);
                MG_DCHECK(in_range(o + (int64_t)(pr + i) * X_LDK - S, 2, bd.s), CK_S_W);
                *reinterpret_cast<double2*>(o + (int64_t)(pr + i) * X_LDK) =
                    make_double2(u.x * wb.x + ub.x * w.x, u.y * wb.y + ub.y * w.y);
            }
            pr += na;
            a = 0;
            ++b;
        }
    }
}

// Persistent x contraction: item it = (row r, M tile, N tile); tile shape per config.
template <class Cfg>
struct XItems {
    static constexpr bool kComputeA = false;
    MgBounds bd;
    const double* S;
    const double* H;
    int P2, pp, XB, MT, NT, kv_last;
    int flip = 0;  // N-split tiles: rotate nt every `flip` items (a multiple of NT) so a CTA
                   // striding by the grid size alternates between full and partial N tiles
    __device__ void decode(int it, int& r, int& mt, int& nt) const {
        nt = it % NT;
        if (flip) nt = (nt + it / flip) % NT;
        mt = (it / NT) % MT;
        r = it / (NT * MT);
    }
    __device__ int ktiles(int) const { return XB; }
    __device__ int kvalid_last(int) const { return kv_last; }
    __device__ int2 valid_mn(int it) const {
        int r, mt, nt;
        decode(it, r, mt, nt);
        return make_int2(min(Cfg::BM, P2 - mt * Cfg::BM), min(Cfg::BN, pp - nt * Cfg::BN));
    }
    __device__ int nfrags(int it) const {  // valid n-fragments of the item's N tile
        int r, mt, nt;
        decode(it, r, mt, nt);
        return (min(Cfg::BN, pp - nt * Cfg::BN) + 7) / 8;
    }
    __device__ uint32_t stage_bytes(int it, int) const {
        int r, mt, nt;
        decode(it, r, mt, nt);
        const int mv = min(Cfg::BM, P2 - mt * Cfg::BM);
        const int nv = min(Cfg::BN, pp - nt * Cfg::BN);
        return (mv + nv) * X_LDK * (uint32_t)sizeof(double);
    }
    __device__ void bulk_rows(int it, int kt, double* As, double* Bs, int lane,
                              uint64_t* bar) const {
        if (lane > 1) return;
        int r, mt, nt;
        decode(it, r, mt, nt);
        if (lane == 0) {
            const int mv = min(Cfg::BM, P2 - mt * Cfg::BM);
            const int64_t so = (((int64_t)r * XB + kt) * P2 + mt * Cfg::BM) * X_LDK;
            MG_DCHECK(in_range(so, (int64_t)mv * X_LDK, bd.s), CK_K2_S);
            bulk_g2s(As, S + so, mv * X_LDK * sizeof(double), bar);
        } else {
            const int nv = min(Cfg::BN, pp - nt * Cfg::BN);
            const int64_t ho = (((int64_t)r * XB + kt) * pp + nt * Cfg::BN) * X_LDK;
            MG_DCHECK(in_range(ho, (int64_t)nv * X_LDK, bd.h), CK_K2_H);
            bulk_g2s(Bs, H + ho, nv * X_LDK * sizeof(double), bar);
        }
    }
};
template <class Cfg>
using XPipeP = PipeTMAPersistent<Cfg, X_BK, 3, false, false>;

template <class Cfg>
__global__ void __launch_bounds__(XPipeP<Cfg>::THREADS, 1)
k_x_contract_p(const double* __restrict__ S, const double* __restrict__ H, int nrows,
               int row_b1, int row_b3, int p, int P2, int Nx, int NxP, double* __restrict__ G,
               MgBounds bd) {
    extern __shared__ __align__(16) double smem[];
    const int pp = p * p;
    XItems<Cfg> items{bd, S, H, P2, pp, NxP / X_BK, (P2 + Cfg::BM - 1) / Cfg::BM,
                      (pp + Cfg::BN - 1) / Cfg::BN, 0};
    items.kv_last = Nx - (items.XB - 1) * X_BK;
    const int nitems = nrows * items.MT * items.NT;
    XPipeP<Cfg>::run(blockIdx.x, gridDim.x, nitems, items, [&](int it, const Acc<Cfg>& acc) {
        int r, mt, nt;
        items.decode(it, r, mt, nt);
        const int m0 = mt * Cfg::BM, n0 = nt * Cfg::BN;
        double* Gr = G + (int64_t)(row_b1 + r - row_b3) * pp * P2;
        acc_foreach_pair<Cfg>(acc, [&](int m, int n, double v0, double v1) {
            const int prr = m0 + m, cc = n0 + n;
            if (prr < P2 && !MG_NO_EPI) {
                MG_DCHECK(cc >= pp || in_range(Gr + (int64_t)cc * P2 + prr - G, 1, bd.g), CK_K2_G_W);
                MG_DCHECK(cc + 1 >= pp || in_range(Gr + (int64_t)(cc + 1) * P2 + prr - G, 1, bd.g),
                          CK_K2_G_W);
                if (cc < pp) Gr[(int64_t)cc * P2 + prr] = v0;
                if (cc + 1 < pp) Gr[(int64_t)(cc + 1) * P2 + prr] = v1;
            }
        });
    }, smem);
}

// N-split x contraction (PipeTMAPersistentNS): 120 x 128 tile on 12 consumer warps of 5 x 4
// fragments; the partial last N tile deals its valid n-fragments over the four warp columns
// (p = 15: 225 columns = 16 + 13 n-fragments -> warps run 4 or 3 n-fragments).
template <class Cfg>
using XPipeNS = PipeTMAPersistentNS<Cfg, X_BK, 3, false, false>;

template <class Cfg>
__global__ void __launch_bounds__(XPipeNS<Cfg>::THREADS, 1)
k_x_contract_ns(const double* __restrict__ S, const double* __restrict__ H, int nrows,
                int row_b1, int row_b3, int p, int P2, int Nx, int NxP, double* __restrict__ G,
                MgBounds bd) {
    extern __shared__ __align__(16) double smem[];
    const int pp = p * p;
    XItems<Cfg> items{bd, S, H, P2, pp, NxP / X_BK, (P2 + Cfg::BM - 1) / Cfg::BM,
                      (pp + Cfg::BN - 1) / Cfg::BN, 0};
    items.kv_last = Nx - (items.XB - 1) * X_BK;
    items.flip = (int)gridDim.x % items.NT == 0 ? (int)gridDim.x : 0;
    const int nitems = nrows * items.MT * items.NT;
    XPipeNS<Cfg>::run(blockIdx.x, gridDim.x, nitems, items,
                      [&](int it, const Acc<Cfg>& acc, int wm, int wn, int nf) {
        int r, mt, nt;
        items.decode(it, r, mt, nt);
        const int lane = threadIdx.x & 31;
        const int m0 = mt * Cfg::BM + wm + (lane >> 2), n0 = nt * Cfg::BN + wn + 2 * (lane & 3);
        double* Gr = G + (int64_t)(row_b1 + r - row_b3) * pp * P2;
#pragma unroll
        for (int mi = 0; mi < Cfg::FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < Cfg::FN; ++ni) {
                const int prr = m0 + mi * 8, cc = n0 + ni * 8;
                if (ni < nf && prr < P2 && !MG_NO_EPI) {
                    MG_DCHECK(cc >= pp || in_range(Gr + (int64_t)cc * P2 + prr - G, 1, bd.g), CK_K2_G_W);
                    MG_DCHECK(cc + 1 >= pp || in_range(Gr + (int64_t)(cc + 1) * P2 + prr - G, 1, bd.g),
                              CK_K2_G_W);
                    if (cc < pp) Gr[(int64_t)cc * P2 + prr] = acc.c[mi][ni][0];
                    if (cc + 1 < pp) Gr[(int64_t)(cc + 1) * P2 + prr] = acc.c[mi][ni][1];
                }
            }
    }, smem);
}

// x-contraction tiles.  The CTA tile is chosen per basis size from M = p(p+1)/2 pairs and
// N = p^2 (c,c') columns (choose_xtile).  Consumer warps are 12 (3 per SM sub-partition: every
// DMMA unit serves the same number of warps; 13 warps allocate up to 128 registers) or 15
// (120 x 120, p = 15, where no 12-warp tiling of M = 120 fits N = 225 better):
//   T120     120 x 120, 15 warps, 3x5 fragments              p = 15: M exact, N 225 -> 240
//   T120x96  120 x 96,  12 warps, 5x3 fragments              (round 1's p = 30 tile)
//   T128x72  128 x 72,  12 warps, 4x3 fragments              p = 22: 253 x 484 -> 256 x 504
//   T160x72  160 x 72,  12 warps, 5x3 fragments              p = 30: 465 x 900 -> 480 x 936
//   T128     128 x 128,  8 warps, 8x4 fragments (spills)     kept for A/B measurements
// Measured in round 1 (ncu): the 8-warp 128 x 128 tile at p = 22 ran the DMMA pipe at 78 %
// (168 registers with local-memory spills); the 12-warp 120 x 96 tile at p = 30 at 96 %.
using CfgX120x96 = TileCfg<3, 4, 5, 3>;
using CfgX128x72 = TileCfg<4, 3, 4, 3>;
using CfgX160x72 = TileCfg<4, 3, 5, 3>;
using CfgX128 = TileCfg<2, 4, 8, 4>;
//   T120x128NS 120 x 128, 12 warps, 5x4 fragments, N-split (k_x_contract_ns)
//                                                            p = 15: 225 = 16 + 13 n-fragments
using CfgX120x128 = TileCfg<3, 4, 5, 4>;

enum class XTile { T120 = 0, T120x96, T128x72, T160x72, T128, T120x128NS, T128x72NS, T160x72NS,
                   COUNT };

// DMMA-pipe model of an N-split tile: fragment-steps of the busiest SM sub-partition per row
// (sub-partition = warp % 4; warp w sits in warp row w / WARPS_N and warp column
// (w + w / WARPS_N) % WARPS_N) against the useful ones; 0 when a warp column of the partial N
// tile would get fewer than max(1, FN - 2) fragments.
template <class C>
static double nsplit_efficiency(int P2, int pp) {
    const int MT = ceil_div(P2, C::BM), NT = ceil_div(pp, C::BN);
    double cost = 0.0;
    for (int nt = 0; nt < NT; ++nt) {
        const int nfr = (std::min(C::BN, pp - nt * C::BN) + 7) / 8;
        const int base = nfr / C::WARPS_N, rem = nfr % C::WARPS_N;
        if (base < std::max(1, C::FN - 2)) return 0.0;
        int load[4] = {0, 0, 0, 0};
        for (int w = 0; w < C::WARPS_M * C::WARPS_N; ++w) {
            const int wni = (w + w / C::WARPS_N) % C::WARPS_N;
            load[w % 4] += C::FM * (base + (wni < rem ? 1 : 0));
        }
        cost += *std::max_element(load, load + 4);
    }
    return ((double)P2 * pp / 64.0 / 4.0) / (cost * MT);
}

// Padded-area efficiency of M = P2, N = pp on a bm x bn tile, times a per-tile pipe factor
// (sub-partition balance / measured DMMA-pipe utilisation).  MG_XTILE=<index> forces a tile
// (A/B measurements).
static XTile choose_xtile(int P2, int pp) {
    const double ens[3] = {nsplit_efficiency<CfgX120x128>(P2, pp),
                           nsplit_efficiency<CfgX128x72>(P2, pp),
                           nsplit_efficiency<CfgX160x72>(P2, pp)};
    if (const char* f = std::getenv("MG_XTILE")) {
        const int i = std::atoi(f);
        if (i >= 0 && i < (int)XTile::COUNT &&
            (i < (int)XTile::T120x128NS || ens[i - (int)XTile::T120x128NS] > 0.0))
            return (XTile)i;
    }
    struct Cand { XTile t; int bm, bn; double pipe; };
    const Cand cands[] = {{XTile::T120, 120, 120, 15.0 / 16.0},
                          {XTile::T120x96, CfgX120x96::BM, CfgX120x96::BN, 1.0},
                          {XTile::T128x72, CfgX128x72::BM, CfgX128x72::BN, 1.0},
                          {XTile::T160x72, CfgX160x72::BM, CfgX160x72::BN, 1.0},
                          {XTile::T128, 128, 128, 0.8}};
    XTile best = XTile::T120;
    double be = -1.0;
    for (const Cand& c : cands) {
        const double e = c.pipe * (double)P2 * pp /
                         ((double)ceil_div(P2, c.bm) * c.bm * ceil_div(pp, c.bn) * c.bn);
        if (e > be + 1e-9) { be = e; best = c.t; }
    }
    // N-split forms (same tiles, partial last N tile dealt over the warp columns)
    for (int i = 0; i < 3; ++i)
        if (ens[i] > be + 1e-9) { be = ens[i]; best = (XTile)((int)XTile::T120x128NS + i); }
    return best;
}

template <class Cfg>
static void launch_x(int num_sms, cudaStream_t st, const double* S, const double* H, int nrows,
                     int row_b1, int row_b3, int p, int P2, int Nx, int NxP, double* G,
                     const MgBounds& bd) {
    k_x_contract_p<Cfg><<<num_sms, XPipeP<Cfg>::THREADS, XPipeP<Cfg>::smem_bytes, st>>>(
        S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd);
}
template <class Cfg>
static void attr_x() {
    MG_CUDA(cudaFuncSetAttribute(k_x_contract_p<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)XPipeP<Cfg>::smem_bytes));
}
template <class Cfg>
static void launch_x_ns(int num_sms, cudaStream_t st, const double* S, const double* H, int nrows,
                        int row_b1, int row_b3, int p, int P2, int Nx, int NxP, double* G,
                        const MgBounds& bd) {
    MG_REQUIRE(nsplit_efficiency<Cfg>(P2, p * p) > 0.0,
               "N-split x tile does not fit this basis size (a warp column would get fewer "
               "than FN - 2 n-fragments)");
    k_x_contract_ns<Cfg><<<num_sms, XPipeNS<Cfg>::THREADS, XPipeNS<Cfg>::smem_bytes, st>>>(
        S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd);
}
template <class Cfg>
static void attr_x_ns() {
    MG_CUDA(cudaFuncSetAttribute(k_x_contract_ns<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)XPipeNS<Cfg>::smem_bytes));
}
static void launch_xtile(XTile xt, int num_sms, cudaStream_t st, const double* S, const double* H,
                         int nrows, int row_b1, int row_b3, int p, int P2, int Nx, int NxP,
                         double* G, const MgBounds& bd) {
    switch (xt) {
        case XTile::T120: launch_x<CfgX120>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
        case XTile::T120x96: launch_x<CfgX120x96>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
        case XTile::T128x72: launch_x<CfgX128x72>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
        case XTile::T160x72: launch_x<CfgX160x72>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
        case XTile::T120x128NS: launch_x_ns<CfgX120x128>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
        case XTile::T128x72NS: launch_x_ns<CfgX128x72>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
        case XTile::T160x72NS: launch_x_ns<CfgX160x72>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
        default: launch_x<CfgX128>(num_sms, st, S, H, nrows, row_b1, row_b3, p, P2, Nx, NxP, G, bd); break;
    }
}

// ------------------------------------------------------------------------------------------
// K2b: gather  R[r][c*nm + n'] = G[r][c,k'][i'j'] + G[r][c,j'][i'k'] + G[r][c,i'][j'k']
//      and pair sums Sq[r][ab] = q_a(l2) q_b(l3) + q_b(l2) q_a(l3)
// ------------------------------------------------------------------------------------------
__global__ void k_gather(const MgRow* __restrict__ rows, const double* __restrict__ G,
                         const int* __restrict__ modes, const double* __restrict__ q, int L,
                         int l_min, int p, int P2, int nm, int n3, int64_t kp,
                         double* __restrict__ RB, double* __restrict__ SqB, MgBounds bd) {
    // Blocked, smem-identical layouts of the pair contraction's operands (one bulk copy per
    // stage): RB[nt][r][RUN_LDB] (column c = nt*RUN_TN + cn), SqB[mt][r][RUN_LDA] (pair
    // pr = mt*RUN_TM + m).  Rows r in [n3, gridDim.y) are the zero K-padding of the last tile.
    const int r = blockIdx.y;
    const bool live = r < n3;
    const int pp = p * p;
    const double* Gr = G + (int64_t)r * pp * P2;
    const int ncols = p * nm;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < ncols;
         idx += gridDim.x * blockDim.x) {
        double val = 0.0;
        if (live) {
            int c = idx / nm, np = idx - c * nm;
            int a = modes[3 * np], b = modes[3 * np + 1], d = modes[3 * np + 2];
            int cp = c * p;
            val = Gr[(int64_t)(cp + d) * P2 + pair_idx(a, b)] +
                  Gr[(int64_t)(cp + b) * P2 + pair_idx(a, d)] +
                  Gr[(int64_t)(cp + a) * P2 + pair_idx(b, d)];
        }
        const int nt = idx / RUN_TN, cn = idx - nt * RUN_TN;
        MG_DCHECK(in_range(((int64_t)nt * kp + r) * RUN_LDB + cn, 1, bd.r), CK_GATHER_W);
        RB[((int64_t)nt * kp + r) * RUN_LDB + cn] = val;
    }
    if (blockIdx.x == 0) {
        const MgRow w = rows[live ? r : 0];
        for (int pr = threadIdx.x; pr < P2; pr += blockDim.x) {
            double s = 0.0;
            if (live) {
                int a, b;
                pair_of(pr, a, b);
                const double* qa = q + (int64_t)a * L - l_min;
                const double* qb = q + (int64_t)b * L - l_min;
                s = qa[w.l2] * qb[w.l3] + qb[w.l2] * qa[w.l3];
            }
            const int mt = pr / RUN_TM, m = pr - mt * RUN_TM;
            MG_DCHECK(in_range(((int64_t)mt * kp + r) * RUN_LDA + m, 1, bd.sq), CK_GATHER_W);
            SqB[((int64_t)mt * kp + r) * RUN_LDA + m] = s;
        }
    }
}

// ------------------------------------------------------------------------------------------
// K3: pair contraction over rows  Z_s[ab][(c,n')] += Σ_{r in split s} Sq[r][ab] R[r][(c,n')]
// ------------------------------------------------------------------------------------------
// Persistent pair contraction: item it = (split s, M tile, N tile) over the 128 x 96 run
// tile and pipeline; stages are one bulk copy of SqB and one of RB.
struct PairItems {
    static constexpr bool kComputeA = false;
    MgBounds bd;
    const double* SqB;
    const double* RB;
    int64_t kp;
    int n3, per, MT, NT;
    __device__ void decode(int it, int& s, int& mt, int& nt) const {
        nt = it % NT;
        mt = (it / NT) % MT;
        s = it / (NT * MT);
    }
    int P2, ncols;
    __device__ int rows_of(int s) const { return min(per, n3 - s * per); }
    __device__ int2 valid_mn(int it) const {
        int s, mt, nt;
        decode(it, s, mt, nt);
        return make_int2(min(RUN_TM, P2 - mt * RUN_TM), min(RUN_TN, ncols - nt * RUN_TN));
    }
    __device__ int ktiles(int it) const {
        int s, mt, nt;
        decode(it, s, mt, nt);
        return (rows_of(s) + RUN_BK - 1) / RUN_BK;
    }
    __device__ int kvalid_last(int it) const {
        int s, mt, nt;
        decode(it, s, mt, nt);
        const int nr = rows_of(s);
        return nr - (nr - 1) / RUN_BK * RUN_BK;
    }
    __device__ uint32_t stage_bytes(int, int) const {
        return RUN_BK * (RUN_LDA + RUN_LDB) * (uint32_t)sizeof(double);
    }
    __device__ void bulk_rows(int it, int kt, double* As, double* Bs, int lane,
                              uint64_t* bar) const {
        if (lane > 1) return;
        int s, mt, nt;
        decode(it, s, mt, nt);
        const int64_t r = (int64_t)s * per + kt * RUN_BK;
        if (lane == 0) {
            MG_DCHECK(in_range(((int64_t)mt * kp + r) * RUN_LDA, RUN_BK * RUN_LDA, bd.sq), CK_K3_SQ);
            bulk_g2s(As, SqB + ((int64_t)mt * kp + r) * RUN_LDA,
                     RUN_BK * RUN_LDA * sizeof(double), bar);
        } else {
            MG_DCHECK(in_range(((int64_t)nt * kp + r) * RUN_LDB, RUN_BK * RUN_LDB, bd.r), CK_K3_R);
            bulk_g2s(Bs, RB + ((int64_t)nt * kp + r) * RUN_LDB,
                     RUN_BK * RUN_LDB * sizeof(double), bar);
        }
    }
};

__global__ void __launch_bounds__(RunPipeP::THREADS, 1)
k_pair_contract(const double* __restrict__ SqB, const double* __restrict__ RB, int64_t kp,
                int n3, int per, int nsplit, int P2, int ncols, int64_t zsplit,
                double* __restrict__ Z, MgBounds bd) {
    extern __shared__ __align__(16) double smem[];
    PairItems items{bd, SqB, RB, kp, n3, per, (P2 + RUN_TM - 1) / RUN_TM,
                    (ncols + RUN_TN - 1) / RUN_TN, P2, ncols};
    const int nitems = nsplit * items.MT * items.NT;
    RunPipeP::run(blockIdx.x, gridDim.x, nitems, items, [&](int it, const Acc<CfgRun>& acc) {
        int s, mt, nt;
        items.decode(it, s, mt, nt);
        double* Zs = Z + s * zsplit;
        const int m0 = mt * RUN_TM, n0 = nt * RUN_TN;
        acc_foreach_pair<CfgRun>(acc, [&](int m, int n, double v0, double v1) {
            const int prr = m0 + m, c = n0 + n;
            if (prr < P2) {
                double* z = Zs + (int64_t)prr * ncols;
                MG_DCHECK(c >= ncols || in_range(z + c - Z, c + 1 < ncols ? 2 : 1, bd.z), CK_K3_Z_W);
                if (c < ncols) z[c] += v0;
                if (c + 1 < ncols) z[c + 1] += v1;
            }
        });
    }, smem);
}

// Γ[(ijk)][n'] = Σ_s Z_s[ij][k][n'] + Z_s[ik][j][n'] + Z_s[jk][i][n']   (splits in order)
__global__ void k_final(const double* __restrict__ Z, int nsplit, int64_t zsplit,
                        const int* __restrict__ modes, int p, int nm, double* __restrict__ gamma) {
    int64_t total = (int64_t)nm * nm;
    const int64_t ncols = (int64_t)p * nm;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int n = (int)(i / nm), np = (int)(i % nm);
        int a = modes[3 * n], b = modes[3 * n + 1], d = modes[3 * n + 2];
        double acc = 0.0;
        for (int s = 0; s < nsplit; ++s) {
            const double* Zs = Z + s * zsplit;
            acc += Zs[pair_idx(a, b) * ncols + (int64_t)d * nm + np] +
                   Zs[pair_idx(a, d) * ncols + (int64_t)b * nm + np] +
                   Zs[pair_idx(b, d) * ncols + (int64_t)a * nm + np];
        }
        gamma[i] = acc;
    }
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------

// Counters of the checked build's bounds checks, per site (MgCheck); zeros in a normal build.
int debug_checks(uint32_t* out, int n, bool reset) {
    for (int i = 0; i < n; ++i) out[i] = 0;
#if MG_CHECKED
    unsigned int h[16] = {0};
    MG_CUDA(cudaDeviceSynchronize());
    MG_CUDA(cudaMemcpyFromSymbol(h, g_chk, sizeof(h)));
    for (int i = 0; i < n && i < 16; ++i) out[i] = h[i];
    if (reset) {
        const unsigned int z[16] = {0};
        MG_CUDA(cudaMemcpyToSymbol(g_chk, z, sizeof(z)));
    }
    return 1;
#else
    (void)reset;
    return 0;
#endif
}

std::vector<double> log_factorials(int n) {
    // t[k] = log(k!) accumulated left to right like np.cumsum(np.log(arange(1, size)))
    std::vector<double> t(n + 1, 0.0);
    for (int k = 1; k <= n; ++k) t[k] = t[k - 1] + std::log((double)k);
    return t;
}

void plan_init(mg_plan* P, const double* q, const double* qt_host, const double* qt_dev,
               const double* C, const double* v, const double* wr2, const int64_t* modes,
               int p, int Nx, int n, int l_min, int l_max, int h2_mode) {
    MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
    MG_REQUIRE(p >= 1 && Nx >= 1 && n >= 1, "p, Nx, n must be >= 1");
    MG_REQUIRE(h2_mode == MG_H2_GOSPER || h2_mode == MG_H2_EXACT, "unknown h2_mode");
    // (row, c) slot division by multiply-shift is exact for p < 197 (slot + c0 < p + 128);
    // beyond that the per-row operands (G: p^4/2 doubles, Z: p^3 n) outgrow HBM anyway
    MG_REQUIRE(p <= 196, "p_max > 196 not supported");
    const int L = l_max - l_min + 1;
    for (int i = 0; i < L; ++i) {
        MG_REQUIRE(C[i] > 0, "power spectrum C_l must be strictly positive");
        MG_REQUIRE(std::isfinite(C[i]) && std::isfinite(v[i]), "table contains non-finite values");
    }
    std::vector<int> md(3 * (size_t)n);
    for (int i = 0; i < n; ++i) {
        int64_t a = modes[3 * i], b = modes[3 * i + 1], c = modes[3 * i + 2];
        MG_REQUIRE(0 <= a && a <= b && b <= c && c < p, "mapping triples must satisfy i<=j<=k<p");
        md[3 * i] = (int)a; md[3 * i + 1] = (int)b; md[3 * i + 2] = (int)c;
    }
    P->sc = scratch_pool(P->device);
    P->p = p; P->Nx = Nx; P->nm = n; P->l_min = l_min; P->l_max = l_max; P->L = L;
    P->h2_mode = h2_mode;
    P->NxP = (int)round_up(Nx, X_BK);
    P->P2 = p * (p + 1) / 2;
    P->Nxw = (Nx % 2 == 0) ? Nx : P->NxP;
    P->l0[l_min & 1] = l_min;
    P->l0[(l_min + 1) & 1] = l_min + 1;
    P->nclass[l_min & 1] = (L + 1) / 2;
    P->nclass[(l_min + 1) & 1] = L / 2;
    P->hC.assign(C, C + L);
    P->hv.assign(v, v + L);

    P->q.upload(q, (size_t)p * L);
    P->l0d.upload(P->l0, 2);
    {
        std::vector<double> fl(L);
        for (int i = 0; i < L; ++i)
            fl[i] = (2.0 * (l_min + i) + 1.0) / (v[i] * std::sqrt(C[i]));
        P->fl.upload(fl.data(), L);
    }
    P->C.upload(C, L);
    P->v.upload(v, L);
    P->wr2.upload(wr2, Nx);
    P->modes.upload(md.data(), md.size());
    P->hmodes = md;
    std::vector<double> lf = log_factorials(3 * l_max + 2);
    P->lf.upload(lf.data(), lf.size());

    const size_t nq = (size_t)p * Nx * L;
    DBuf<double> staged;
    const double* qt_src = qt_dev;
    if (!qt_src) {
        staged.upload(qt_host, nq);
        qt_src = staged.p;
    }
    P->QT.alloc((size_t)L * p * P->NxP);
    const int nb = ceil_div((int64_t)p * P->Nxw, RUN_TN);
    for (int par = 0; par < 2; ++par) P->wrows[par] = P->nclass[par] + RUN_BK;
    P->wbase[0] = 0;
    P->wbase[1] = (int64_t)nb * P->wrows[0] * RUN_LDB;
    const size_t wsize = (size_t)nb * (P->wrows[0] + P->wrows[1]) * RUN_LDB;
    P->WQT.alloc(wsize);
    MG_CUDA(cudaMemset(P->WQT.p, 0, wsize * sizeof(double)));
    k_transpose_qt<<<1184, 256>>>(qt_src, P->wr2.p, p, Nx, P->NxP, P->Nxw, L, l_min,
                                  make_longlong2(P->wbase[0], P->wbase[1]),
                                  make_int2(P->wrows[0], P->wrows[1]), P->QT.p, P->WQT.p);
    MG_LAUNCHED();
    // A device-resident q̃ belongs to the caller, who may release it once this returns; a
    // host q̃ was staged into the plan's own buffer (freed stream-ordered), so the transposes
    // may still run while the caller prepares the rows of its first execute.
    if (qt_dev) MG_CUDA(cudaDeviceSynchronize());
}


static inline bool lex_ge(int a2, int a3, int b2, int b3) {
    return a2 > b2 || (a2 == b2 && a3 >= b3);
}

void build_rows(const mg_plan* P, int l2a, int l2b, const int* s, const int* e,
                std::vector<MgRow>& rows) {
    build_rows_range(P->l_min, P->l_max, l2a, l2b, s, e, rows);
}

void build_rows_range(int lmin, int lmax, int l2a, int l2b, const int* s, const int* e,
                      std::vector<MgRow>& rows) {
    rows.clear();
    const int l0[2] = {(lmin & 1) ? lmin + 1 : lmin, (lmin & 1) ? lmin : lmin + 1};
    l2a = std::max(l2a, lmin);
    l2b = std::min(l2b, lmax + 1);
    for (int l2 = l2a; l2 < l2b; ++l2) {
        if (l2 < s[0]) continue;  // no l1 <= l2 can reach the range start
        for (int par = 0; par < 2; ++par) {
            // l1 parity par  <=>  l3 = l2 + par (mod 2)
            int l3top = std::min(2 * l2, lmax);
            for (int l3 = l2 + par; l3 <= l3top; l3 += 2) {
                int lo = std::max(lmin, l3 - l2);
                int hi = l2;
                int clo = lex_ge(l2, l3, s[1], s[2]) ? s[0] : s[0] + 1;
                int chi = lex_ge(l2, l3, e[1], e[2]) ? e[0] - 1 : e[0];
                lo = std::max(lo, clo);
                hi = std::min(hi, chi);
                if ((lo & 1) != par) ++lo;
                if ((hi & 1) != par) --hi;
                if (lo > hi) continue;
                MgRow r;
                r.l2 = l2; r.l3 = l3; r.par = par;
                r.jlo = (lo - l0[par]) / 2;
                r.jhi = (hi - l0[par]) / 2;
                r.pad = 0;
                rows.push_back(r);
            }
        }
    }
}

MgScratch* scratch_pool(int device) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<MgScratch>> pools;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)pools.size() <= device) pools.resize(device + 1);
    if (!pools[device]) pools[device].reset(new MgScratch());
    return pools[device].get();
}

// Every plan on a device shares that device's scratch (MgScratch).  Executes are serialised
// per device by holding this lock across the host-side enqueue: each pipeline starts by
// waiting on the legacy stream 0 and ends by making stream 0 wait for it, so on the GPU the
// next execute's use of the scratch (and any reallocation by ensure(), stream-ordered on
// stream 0) starts only after the previous one finished.  Recursive: execute_triples may
// delegate to execute_rows.
std::recursive_mutex& device_mutex(int device) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<std::recursive_mutex>> locks;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)locks.size() <= device) locks.resize(device + 1);
    if (!locks[device]) locks[device].reset(new std::recursive_mutex());
    return *locks[device];
}

// Batch geometry: K1/K2 work on nb1 rows at a time (H buffer), K3 on nb3 (G buffer).
static void choose_batches(mg_plan* P) {
    // Scratch per row: H (run contraction out), S (pair products), G (x contraction out),
    // R (gathered G).  Budgets are tens of GB of the 180 GB HBM: large batches keep every
    // launch many waves deep and the launch count low (config 1: 8288-row batches, 607
    // launches per Γ; measured 0.9 % faster than 2048-row batches, 2207 launches).
    const double hrow = (double)P->p * P->p * P->NxP * 8.0;
    const double srow = (double)P->P2 * P->NxP * 8.0;
    const double grow = (double)P->P2 * P->p * P->p * 8.0 + (double)P->p * P->nm * 8.0;
    int nb1 = (int)std::min({(double)MG_NB1, MG_HBUDGET / hrow, MG_HBUDGET / 2 / srow});
    nb1 = std::max(16, nb1 / 16 * 16);
    int nb3 = (int)std::min((double)MG_NB3, std::max((double)nb1, MG_HBUDGET / grow));
    nb3 = std::max(nb1, nb3 / nb1 * nb1);
    P->nb1 = nb1;
    P->nb3 = nb3;
}

// Optional per-family kernel timing (mg_plan_set_profile): one event before every launch,
// duration of launch i = event[i+1] - event[i] on the launching stream.
static void prof_mark(mg_plan* P, int tag, cudaStream_t st) {
    if (!P->profile) return;
    if (P->prof_used == P->prof_events.size()) {
        cudaEvent_t e;
        MG_CUDA(cudaEventCreate(&e));
        P->prof_events.push_back(e);
    }
    MG_CUDA(cudaEventRecord(P->prof_events[P->prof_used], st));
    P->prof_tags.push_back(tag);
    ++P->prof_used;
}

// Side-stream operand kernels: (start, end) event pairs, summed into prof_ms[6].
static void prof_side(mg_plan* P, cudaStream_t ss, bool start) {
    if (!P->profile) return;
    if (P->side_used == P->side_events.size()) {
        cudaEvent_t e;
        MG_CUDA(cudaEventCreate(&e));
        P->side_events.push_back(e);
    }
    MG_CUDA(cudaEventRecord(P->side_events[P->side_used++], ss));
    (void)start;
}

// Pipeline streams and dependency events, created once per plan on its device.
static void plan_streams(mg_plan* P) {
    if (P->ms) return;
    int least = 0, greatest = 0;
    MG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    MG_CUDA(cudaStreamCreateWithPriority(&P->ms, cudaStreamNonBlocking, greatest));
    MG_CUDA(cudaStreamCreateWithPriority(&P->ss, cudaStreamNonBlocking, least));
    for (cudaEvent_t* e : {&P->ev_start[0], &P->ev_start[1], &P->ev_end[0], &P->ev_end[1],
                           &P->ev_panel[0], &P->ev_panel[1], &P->ev_s, &P->ev_x})
        MG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

void prof_collect(mg_plan* P) {
    if (P->side_used) MG_CUDA(cudaEventSynchronize(P->side_events[P->side_used - 1]));
    if (P->prof_used) MG_CUDA(cudaEventSynchronize(P->prof_events[P->prof_used - 1]));
    for (size_t i = 0; i + 1 < P->side_used; i += 2) {
        float ms = 0.f;
        MG_CUDA(cudaEventElapsedTime(&ms, P->side_events[i], P->side_events[i + 1]));
        P->prof_ms[6] += ms;
    }
    P->side_used = 0;
    for (size_t i = 0; i + 1 < P->prof_used; ++i) {
        float ms = 0.f;
        MG_CUDA(cudaEventElapsedTime(&ms, P->prof_events[i], P->prof_events[i + 1]));
        int tag = P->prof_tags[i];
        if (tag >= 0 && tag < MG_NPROF) P->prof_ms[tag] += ms;
    }
    P->prof_used = 0;
    P->prof_tags.clear();
}

// Host-side batch preparation (tiles, panel offsets, uploads of the row/tile tables).  The
// result is cached in the plan (P->prep) and reused while the same slab is executed again.
static void prepare_batches(mg_plan* P, const std::vector<MgRow>& hrows,
                            const std::vector<int64_t>& hzoff, cudaStream_t st) {
    const int p = P->p;
    const int64_t nrows = (int64_t)hrows.size();
    const int nb1 = P->nb1;
    MgPrepared& pre = P->prep;
    // tiles: 128 consecutive (row, c) slots of one (l2, par) group (rows may straddle two
    // tiles), per nb1-batch; each tile owns a k-major A panel of round_up(window, BK) x 128.
    std::vector<MgTile>& tiles = pre.tiles;
    std::vector<int64_t> poff;      // panel offset of each tile, relative to its batch
    std::vector<int>& tile_first = pre.tile_first;
    std::vector<int64_t> panel_len; // per nb1 batch
    tiles.clear();
    tile_first.clear();
    int max_tile_rows = 1;
    for (int64_t b1 = 0; b1 < nrows; b1 += nb1) {
        int64_t e1 = std::min<int64_t>(b1 + nb1, nrows);
        tile_first.push_back((int)tiles.size());
        int64_t off = 0;
        int64_t g0 = b1;
        while (g0 < e1) {  // one (l2, par) group [g0, g1)
            int64_t g1 = g0;
            while (g1 < e1 && hrows[g1].l2 == hrows[g0].l2 && hrows[g1].par == hrows[g0].par) ++g1;
            const int64_t nsl = (g1 - g0) * p;
            for (int64_t s0 = 0; s0 < nsl; s0 += RUN_TM) {
                MgTile t;
                const int64_t s1 = std::min<int64_t>(s0 + RUN_TM, nsl);
                t.row0 = (int)(g0 + s0 / p);
                t.c0 = (int)(s0 % p);
                t.nslots = (int)(s1 - s0);
                const int rlast = (int)(g0 + (s1 - 1) / p);
                t.nrows = rlast - t.row0 + 1;
                t.jlo = hrows[t.row0].jlo;
                t.jhi = hrows[t.row0].jhi;
                for (int r = t.row0; r <= rlast; ++r) {
                    t.jlo = std::min(t.jlo, hrows[r].jlo);
                    t.jhi = std::max(t.jhi, hrows[r].jhi);
                }
                t.pad0 = t.pad1 = 0;
                max_tile_rows = std::max(max_tile_rows, t.nrows);
                tiles.push_back(t);
                poff.push_back(off);
                off += round_up(t.jhi - t.jlo + 1, RUN_BK) * RUN_LDA;
            }
            g0 = g1;
        }
        panel_len.push_back(off);
    }
    tile_first.push_back((int)tiles.size());

    pre.rows.upload(hrows.data(), hrows.size(), st);
    pre.zoff.upload(hzoff.data(), hzoff.size(), st);
    pre.tiles_d.upload(tiles.data(), tiles.size(), st);
    pre.poff.upload(poff.data(), poff.size(), st);
    int64_t maxzt = 1, maxpanel = 1;
    for (size_t bi = 0; bi + 1 < tile_first.size(); ++bi) {
        int64_t b1 = bi * (int64_t)nb1, e1 = std::min<int64_t>(b1 + nb1, nrows);
        maxzt = std::max(maxzt, hzoff[e1] - hzoff[b1]);
        maxpanel = std::max(maxpanel, panel_len[bi]);
    }
    pre.max_tile_rows = max_tile_rows;
    pre.maxzt = maxzt;
    pre.maxpanel = maxpanel;
    pre.nrows = nrows;
    pre.valid = true;
}

static void run_pipeline(mg_plan* P, const std::vector<MgRow>& hrows,
                         const std::vector<int64_t>& hzoff, cudaStream_t st,
                         const int32_t* dt1, const int32_t* dt2, const int32_t* dt3,
                         const int64_t* dpos, const double* ddup,
                         const std::vector<int64_t>* tri_of_row) {
    const int p = P->p, NxP = P->NxP, P2 = P->P2, nm = P->nm;
    const int64_t nrows = (int64_t)hrows.size();
    if (!P->nb1) choose_batches(P);
    const int nb1 = P->nb1, nb3 = P->nb3;
    const int pp = p * p;
    const int ncols = p * nm;

    MG_NVTX("mg:run_pipeline");
    MgPrepared& pre = P->prep;
    if (!pre.valid) {
        MG_NVTX("mg:prepare_batches");
        prepare_batches(P, hrows, hzoff, st);
    }
    const std::vector<MgTile>& tiles = pre.tiles;
    const std::vector<int>& tile_first = pre.tile_first;
    const int max_tile_rows = pre.max_tile_rows;
    const int64_t maxzt = pre.maxzt, maxpanel = pre.maxpanel;
    if (dt1) P->sc->ZT.ensure(2 * maxzt);
    P->sc->panel.ensure(2 * maxpanel);
    const size_t hsize = (size_t)nb1 * pp * (NxP / X_BK) * X_LDK;
    const bool zero_h = P->sc->H.n < hsize;  // x pads of H are never written: zero them once
    if (zero_h) P->sc->H.ensure(hsize);
    P->sc->G.ensure((size_t)nb3 * pp * P2);
    // pair contraction operands in tile-blocked layouts, kp rows per block (K padded to BK)
    const int64_t kp = round_up(nb3, RUN_BK);
    const int mt3 = ceil_div(P2, RUN_TM), nt3 = ceil_div(ncols, RUN_TN);
    P->sc->R.ensure((size_t)nt3 * kp * RUN_LDB);
    P->sc->S.ensure((size_t)nb1 * P2 * (NxP / X_BK) * X_LDK);
    P->sc->Sq.ensure((size_t)mt3 * kp * RUN_LDA);
    int num_sms = 148;
    MG_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, P->device));
    // K-split of the pair contraction (Z copies, summed in order by k_final) so that its
    // persistent items fill the SMs evenly
    int nsplit = 1;
    {
        double best = 0;
        const int tiles3 = mt3 * nt3;
        for (int s = 1; s <= 8; ++s) {
            const int items = tiles3 * s;
            const double eff = (double)items / (ceil_div(items, num_sms) * (double)num_sms);
            if (s > 1 && nb3 / s < 4 * RUN_BK) break;
            if (eff > best + 0.02) { best = eff; nsplit = s; }
        }
    }
    const int64_t zsplit = (int64_t)P2 * ncols;
    P->sc->Z.ensure((size_t)nsplit * zsplit);
    P->gamma.ensure((size_t)nm * nm);
    // buffer extents for the checked build's bounds checks (MG_CHECKED; free otherwise)
    const MgBounds bd{maxpanel, (int64_t)P->WQT.n, (int64_t)P->sc->H.n, (int64_t)P->sc->S.n,
                      (int64_t)P->sc->G.n, (int64_t)P->sc->R.n, (int64_t)P->sc->Sq.n,
                      (int64_t)P->sc->Z.n, 0, 0};

    static bool attr_done_dev[64] = {false};  // function attributes are per device context
    bool& attr_done = attr_done_dev[P->device & 63];
    const size_t smem_run = RunPipeP::smem_bytes;
    const XTile xt = choose_xtile(P2, pp);
    if (!attr_done) {
        MG_CUDA(cudaFuncSetAttribute(k_run_contract, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_run));
        attr_x<CfgX120>();
        attr_x<CfgX120x96>();
        attr_x<CfgX128x72>();
        attr_x<CfgX160x72>();
        attr_x<CfgX128>();
        attr_x_ns<CfgX120x128>();
        attr_x_ns<CfgX128x72>();
        attr_x_ns<CfgX160x72>();
        MG_CUDA(cudaFuncSetAttribute(k_pair_contract, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_run));
        attr_done = true;
    }

    // Streams: the contractions run on the plan's high-priority stream `ms`; the operand
    // kernels (A panels of the run contraction, pair products of the x contraction) run on
    // the low-priority side stream `ss`, one batch ahead, in the registers/threads the
    // persistent contraction CTA leaves free on each SM.  Panels (and explicit-triple weights)
    // are double-buffered; S is single-buffered (pair products of batch i start once the x
    // contraction of batch i-1 has consumed S, i.e. while the run contraction of batch i runs).
    plan_streams(P);
    cudaStream_t ms = P->ms, ss = P->ss;
    MG_CUDA(cudaEventRecord(P->ev_start[0], st));
    MG_CUDA(cudaEventRecord(P->ev_start[1], 0));  // scratch allocations are ordered on stream 0
    for (cudaStream_t x : {ms, ss})
        for (int k = 0; k < 2; ++k) MG_CUDA(cudaStreamWaitEvent(x, P->ev_start[k], 0));
    if (zero_h) MG_CUDA(cudaMemsetAsync(P->sc->H.p, 0, P->sc->H.n * sizeof(double), ms));
    MG_CUDA(cudaMemsetAsync(P->sc->Z.p, 0, (size_t)nsplit * zsplit * sizeof(double), ms));
    prof_mark(P, 0, ms);

    struct Batch { int64_t b1, e1, b3, e3; int bidx; };
    std::vector<Batch> batches;
    {
        int bidx = 0;
        for (int64_t b3 = 0; b3 < nrows; b3 += nb3) {
            const int64_t e3 = std::min<int64_t>(b3 + nb3, nrows);
            for (int64_t b1 = b3; b1 < e3; b1 += nb1, ++bidx)
                batches.push_back({b1, std::min<int64_t>(b1 + nb1, e3), b3, e3, bidx});
        }
    }
    double* panel_buf[2] = {P->sc->panel.p, P->sc->panel.p + maxpanel};
    double* zt_buf[2] = {dt1 ? P->sc->ZT.p : nullptr, dt1 ? P->sc->ZT.p + maxzt : nullptr};
    // operands of batch k: explicit-triple weights + A panels (buffer k % 2), on stream `os`
    auto issue_panels = [&](int k, cudaStream_t os) {
        const Batch& B = batches[k];
        const int64_t zbase = hzoff[B.b1];
        const double* zt = nullptr;
        if (dt1) {
            double* ztb = zt_buf[k & 1];
            const int64_t t0 = (*tri_of_row)[B.b1], t1 = (*tri_of_row)[B.e1];
            MG_CUDA(cudaMemsetAsync(ztb, 0, (hzoff[B.e1] - zbase) * sizeof(double), os));
            if (t1 > t0)
                k_scatter_weights<<<std::min<int64_t>((t1 - t0 + 255) / 256, 4096), 256, 0, os>>>(
                    dt1 + t0, dt2 + t0, dt3 + t0, dpos + t0, ddup + t0, t1 - t0, zbase, P->l_min,
                    P->C.p, P->v.p, P->lf.p, P->h2_mode, ztb);
            MG_LAUNCHED();
            zt = ztb;
        }
        const int tf = tile_first[B.bidx], tl = tile_first[B.bidx + 1];
        int nch = 1;
        for (int t = tf; t < tl; ++t)
            nch = std::max(nch, ceil_div(round_up(tiles[t].jhi - tiles[t].jlo + 1, RUN_BK), PANEL_JC));
        k_run_panels<<<dim3(tl - tf, nch), PANEL_THREADS, max_tile_rows * PANEL_JC * sizeof(double),
                       os>>>(
            P->prep.tiles_d.p + tf, P->prep.rows.p, P->prep.poff.p + tf, P->prep.zoff.p, zbase,
            zt, P->l0d.p, P->q.p, P->L, P->l_min, p, P->C.p, P->v.p, P->lf.p, P->fl.p,
            P->h2_mode, panel_buf[k & 1], (65536u + p - 1) / p, bd);
        MG_LAUNCHED();
    };

    auto issue_pairs = [&](int k, cudaStream_t os) {
        const Batch& B = batches[k];
        dim3 gs(ceil_div(P2, PP_CHUNK), (int)(B.e1 - B.b1));
        k_pair_products<<<gs, MG_PP_THREADS, 0, os>>>(P->prep.rows.p, (int)B.b1, P->QT.p, p, P2, NxP,
                                             P->l_min, P->sc->S.p, bd);
        MG_LAUNCHED();
    };

    double f_run = 0, f_x = 0, f_pair = 0;
    int64_t launches = 0;
    const int nbat = (int)batches.size();
    for (int k = 0; k < nbat; ++k) {
        const Batch& B = batches[k];
        const int nb = (int)(B.e1 - B.b1);
        const int tf = tile_first[B.bidx], tl = tile_first[B.bidx + 1];
        MG_NVTX("mg:batch_enqueue");
#if MG_SIDE == 3
        // panels of batch k alone on the main stream, then the pair products of batch k on the
        // side stream (it waits for the panels, which follow x(k-1) on the main stream, so S
        // has been consumed): they become runnable together with the run contraction, whose
        // higher-priority CTAs are placed first
        prof_mark(P, 0, ms);
        issue_panels(k, ms);
        MG_CUDA(cudaEventRecord(P->ev_panel[0], ms));
        MG_CUDA(cudaStreamWaitEvent(ss, P->ev_panel[0], 0));
        prof_side(P, ss, true);
        issue_pairs(k, ss);
        prof_side(P, ss, false);
        MG_CUDA(cudaEventRecord(P->ev_s, ss));
#elif MG_SIDE
        // side stream, once x(k-1) has consumed S: pair products of batch k (and, MG_SIDE 2,
        // the panels of batch k), beside the run contraction of batch k
        if (k > 0) MG_CUDA(cudaStreamWaitEvent(ss, P->ev_x, 0));
        prof_side(P, ss, true);
        issue_pairs(k, ss);
        prof_side(P, ss, false);
        MG_CUDA(cudaEventRecord(P->ev_s, ss));
#if MG_SIDE == 2
        if (k == 0) {
            issue_panels(0, ss);
            MG_CUDA(cudaEventRecord(P->ev_panel[0], ss));
        }
        if (k + 1 < nbat) {  // into the buffer run(k-1) read (run(k-1) precedes x(k-1))
            prof_side(P, ss, true);
            issue_panels(k + 1, ss);
            prof_side(P, ss, false);
            MG_CUDA(cudaEventRecord(P->ev_panel[(k + 1) & 1], ss));
        }
        prof_mark(P, 0, ms);
        MG_CUDA(cudaStreamWaitEvent(ms, P->ev_panel[k & 1], 0));
#else
        prof_mark(P, 0, ms);
        issue_panels(k, ms);
#endif
#else
        prof_mark(P, 0, ms);
        issue_pairs(k, ms);
        issue_panels(k, ms);
#endif
        prof_mark(P, 1, ms);
        k_run_contract<<<num_sms, RunPipeP::THREADS, smem_run, ms>>>(
            P->prep.tiles_d.p + tf, tl - tf, P->prep.poff.p + tf, panel_buf[k & 1], (int)B.b1,
            P->prep.rows.p, P->WQT.p, p, P->Nx, P->Nxw, NxP,
            make_longlong2(P->wbase[0], P->wbase[1]), make_int2(P->wrows[0], P->wrows[1]),
            P->sc->H.p, (65536u + p - 1) / p,
            (unsigned)(((1ull << 32) + P->Nxw - 1) / P->Nxw), bd);
        MG_LAUNCHED();
#if MG_SIDE
        prof_mark(P, 0, ms);
        MG_CUDA(cudaStreamWaitEvent(ms, P->ev_s, 0));
#endif
        prof_mark(P, 2, ms);
        launch_xtile(xt, num_sms, ms, P->sc->S.p, P->sc->H.p, nb, (int)B.b1, (int)B.b3, p, P2,
                     P->Nx, NxP, P->sc->G.p, bd);
        MG_LAUNCHED();
        MG_CUDA(cudaEventRecord(P->ev_x, ms));
        launches += 4 + (dt1 ? 1 : 0);
        for (int64_t r = B.b1; r < B.e1; ++r) {
            double m = (double)(hrows[r].jhi - hrows[r].jlo + 1);
            f_run += 2.0 * p * p * P->Nx * m;
        }
        f_x += 2.0 * P2 * pp * P->Nx * (double)nb;
        if (B.e1 != B.e3) continue;
        // end of a pair-contraction group: gather + pair contraction over its rows
        const int n3 = (int)(B.e3 - B.b3);
        prof_mark(P, 3, ms);
        dim3 gg(std::min(ceil_div(ncols, 256), 64), (int)round_up(n3, RUN_BK));
        k_gather<<<gg, 256, 0, ms>>>(P->prep.rows.p + B.b3, P->sc->G.p, P->modes.p, P->q.p, P->L,
                                     P->l_min, p, P2, nm, n3, kp, P->sc->R.p, P->sc->Sq.p, bd);
        MG_LAUNCHED();
        const int per = (int)round_up(ceil_div(n3, nsplit), RUN_BK);
        prof_mark(P, 4, ms);
        k_pair_contract<<<num_sms, RunPipeP::THREADS, smem_run, ms>>>(
            P->sc->Sq.p, P->sc->R.p, kp, n3, per, ceil_div(n3, per), P2, ncols, zsplit,
            P->sc->Z.p, bd);
        MG_LAUNCHED();
        launches += 2;
        f_pair += 2.0 * P2 * ncols * (double)n3;
    }
    prof_mark(P, 5, ms);
    k_final<<<std::min<int64_t>(((int64_t)nm * nm + 255) / 256, 4096), 256, 0, ms>>>(
        P->sc->Z.p, nsplit, zsplit, P->modes.p, p, nm, P->gamma.p);
    MG_LAUNCHED();
    prof_mark(P, -1, ms);
    launches += 1;
    P->flops_run = f_run;
    P->flops_x = f_x;
    P->flops_pair = f_pair;
    P->launches = launches;
    // the caller's stream (and stream 0, which frees/reallocates scratch) resume after both
    MG_CUDA(cudaEventRecord(P->ev_end[0], ms));
    MG_CUDA(cudaEventRecord(P->ev_end[1], ss));
    // No host synchronisation: the execute is asynchronous (include/modal_b200.h); kernel
    // timings are resolved when they are read (prof_collect).
    for (cudaStream_t x : {st, (cudaStream_t)0})
        for (int k = 0; k < 2; ++k) MG_CUDA(cudaStreamWaitEvent(x, P->ev_end[k], 0));
}

static void zero_result(mg_plan* P, cudaStream_t st) {
    P->gamma.ensure((size_t)P->nm * P->nm);
    MG_CUDA(cudaMemsetAsync(P->gamma.p, 0, (size_t)P->nm * P->nm * sizeof(double), st));
    P->flops_run = P->flops_x = P->flops_pair = 0;
    P->launches = 0;
}

static void set_rows(mg_plan* P, std::vector<MgRow>&& rows) {
    MgPrepared& pre = P->prep;
    pre.valid = false;
    pre.key_a = pre.key_b = -1;
    pre.hrows = std::move(rows);
    pre.hzoff.assign(pre.hrows.size() + 1, 0);
    for (size_t i = 0; i < pre.hrows.size(); ++i)
        pre.hzoff[i + 1] = pre.hzoff[i] + (pre.hrows[i].jhi - pre.hrows[i].jlo + 1);
}

void execute_rows(mg_plan* P, std::vector<MgRow>&& rows, cudaStream_t st) {
    std::lock_guard<std::recursive_mutex> lock(device_mutex(P->device));
    set_rows(P, std::move(rows));
    if (P->prep.hrows.empty()) return zero_result(P, st);
    run_pipeline(P, P->prep.hrows, P->prep.hzoff, st, nullptr, nullptr, nullptr, nullptr,
                 nullptr, nullptr);
}

// l2 slab [l2a, l2b) of the full domain; the batch tables are reused when the same slab is
// executed again on this plan (bench steps, multi-GPU ranks).
void execute_slab(mg_plan* P, int l2a, int l2b, cudaStream_t st) {
    std::lock_guard<std::recursive_mutex> lock(device_mutex(P->device));
    MgPrepared& pre = P->prep;
    if (!(pre.valid && pre.key_a == l2a && pre.key_b == l2b)) {
        int s[3] = {P->l_min, 0, 0}, e[3] = {P->l_max + 1, 0, 0};
        std::vector<MgRow> rows;
        build_rows(P, l2a, l2b, s, e, rows);
        set_rows(P, std::move(rows));
    }
    if (pre.hrows.empty()) return zero_result(P, st);
    run_pipeline(P, pre.hrows, pre.hzoff, st, nullptr, nullptr, nullptr, nullptr, nullptr,
                 nullptr);
    pre.key_a = l2a;
    pre.key_b = l2b;
}

void execute_triples(mg_plan* P, const int32_t* l1, const int32_t* l2, const int32_t* l3,
                     int64_t count, cudaStream_t st) {
    std::lock_guard<std::recursive_mutex> lock(device_mutex(P->device));
    const int lmin = P->l_min, lmax = P->l_max;
    struct T { int l2, l3, par, l1; };
    std::vector<T> ts;
    ts.reserve(count);
    for (int64_t i = 0; i < count; ++i) {
        int a = l1[i], b = l2[i], c = l3[i];
        MG_REQUIRE(a <= b && b <= c, "permutation_multiplicity requires l1 <= l2 <= l3");
        MG_REQUIRE(a >= lmin && c <= lmax, "triple outside [l_min, l_max]");
        ts.push_back({b, c, a & 1, a});
    }
    std::sort(ts.begin(), ts.end(), [](const T& x, const T& y) {
        if (x.l2 != y.l2) return x.l2 < y.l2;
        if (x.par != y.par) return x.par < y.par;
        if (x.l3 != y.l3) return x.l3 < y.l3;
        return x.l1 < y.l1;
    });
    std::vector<MgRow> rows;
    std::vector<int64_t> zoff(1, 0), tri_of_row(1, 0);
    std::vector<int32_t> h1, h2, h3;
    std::vector<int64_t> pos;
    std::vector<double> dup;
    size_t i = 0;
    while (i < ts.size()) {
        size_t j = i;
        while (j < ts.size() && ts[j].l2 == ts[i].l2 && ts[j].l3 == ts[i].l3 &&
               ts[j].par == ts[i].par)
            ++j;
        MgRow r;
        r.l2 = ts[i].l2; r.l3 = ts[i].l3; r.par = ts[i].par; r.pad = 0;
        r.jlo = (ts[i].l1 - P->l0[r.par]) / 2;
        r.jhi = (ts[j - 1].l1 - P->l0[r.par]) / 2;
        for (size_t k = i; k < j;) {
            size_t k2 = k;
            while (k2 < j && ts[k2].l1 == ts[k].l1) ++k2;  // duplicates add up
            h1.push_back(ts[k].l1); h2.push_back(r.l2); h3.push_back(r.l3);
            pos.push_back(zoff.back() + (ts[k].l1 - P->l0[r.par]) / 2 - r.jlo);
            dup.push_back((double)(k2 - k));
            k = k2;
        }
        rows.push_back(r);
        zoff.push_back(zoff.back() + (r.jhi - r.jlo + 1));
        tri_of_row.push_back((int64_t)h1.size());
        i = j;
    }
    if (rows.empty()) {
        execute_rows(P, std::move(rows), st);
        return;
    }
    P->prep.valid = false;
    P->prep.key_a = P->prep.key_b = -1;
    DBuf<int32_t> d1, d2, d3;
    DBuf<int64_t> dp;
    DBuf<double> dd;
    d1.upload(h1.data(), h1.size(), st);
    d2.upload(h2.data(), h2.size(), st);
    d3.upload(h3.data(), h3.size(), st);
    dp.upload(pos.data(), pos.size(), st);
    dd.upload(dup.data(), dup.size(), st);
    run_pipeline(P, rows, zoff, st, d1.p, d2.p, d3.p, dp.p, dd.p, &tri_of_row);
    P->prep.valid = false;  // tables belong to this explicit triple list
}

// ------------------------------------------------------------------------------------------
// weights / enumeration on the device (mg_weights, mg_domain_triples)
// ------------------------------------------------------------------------------------------
__global__ void k_weights(const int64_t* __restrict__ l1_base, const int64_t* __restrict__ row_base,
                          const int64_t* __restrict__ pair_off, int l_min, int l_max,
                          int64_t begin, int64_t end, const double* __restrict__ C,
                          const double* __restrict__ v, const double* __restrict__ lf, int mode,
                          double* __restrict__ zm, int32_t* __restrict__ o1,
                          int32_t* __restrict__ o2, int32_t* __restrict__ o3) {
    const int L = l_max - l_min + 1;
    for (int64_t idx = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < end;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = L;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (l1_base[mid] <= idx) lo = mid; else hi = mid;
        }
        int64_t a = pair_off[lo], b = pair_off[lo + 1];
        while (b - a > 1) {
            int64_t mid = (a + b) >> 1;
            if (row_base[mid] <= idx) a = mid; else b = mid;
        }
        int l1 = l_min + lo;
        int l2 = l1 + (int)(a - pair_off[lo]);
        int l3 = row_start(l1, l2) + 2 * (int)(idx - row_base[a]);
        int64_t o = idx - begin;
        if (o1) { o1[o] = l1; o2[o] = l2; o3[o] = l3; }
        if (zm) zm[o] = zm_weight(mode, l1, l2, l3, C, v, l_min, lf);
    }
}

void weights(int l_min, int l_max, const double* C, const double* v, int h2_mode,
             int64_t begin, int64_t end, double* zm, int32_t* o1, int32_t* o2, int32_t* o3) {
    DomainIndex D;
    D.build(l_min, l_max);
    if (end < 0 || end > D.count) end = D.count;
    MG_REQUIRE(0 <= begin && begin <= end, "invalid flat range");
    const int64_t n = end - begin;
    if (n == 0) return;
    const int L = l_max - l_min + 1;
    DBuf<int64_t> b1, rb, po;
    b1.upload(D.l1_base.data(), D.l1_base.size());
    rb.upload(D.row_base.data(), D.row_base.size());
    po.upload(D.pair_off.data(), D.pair_off.size());
    DBuf<double> dC, dv, dlf, dz;
    DBuf<int32_t> d1, d2, d3;
    if (zm) {
        if (h2_mode != MG_H2_GOSPER && h2_mode != MG_H2_EXACT) fail(MG_EINVAL, "unknown h2_mode");
        for (int i = 0; i < L; ++i)
            MG_REQUIRE(C[i] > 0, "power spectrum C_l must be strictly positive");
        dC.upload(C, L);
        dv.upload(v, L);
        std::vector<double> lf = log_factorials(3 * l_max + 2);
        dlf.upload(lf.data(), lf.size());
        dz.alloc(n);
    }
    if (o1) { d1.alloc(n); d2.alloc(n); d3.alloc(n); }
    int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 32);
    k_weights<<<grid, 256>>>(b1.p, rb.p, po.p, l_min, l_max, begin, end, dC.p, dv.p, dlf.p,
                             h2_mode, dz.p, d1.p, d2.p, d3.p);
    MG_LAUNCHED();
    if (zm) MG_CUDA(cudaMemcpy(zm, dz.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    if (o1) {
        MG_CUDA(cudaMemcpy(o1, d1.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        MG_CUDA(cudaMemcpy(o2, d2.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        MG_CUDA(cudaMemcpy(o3, d3.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    }
}

// ------------------------------------------------------------------------------------------
// Non-separable pointwise path (config 3).  k_nonsep is the generic (any p, slow) kernel
// used for p > 16; k_nonsep_warp below is the compile-time-P kernel.
//   B(t,x) = Σ_n' α_n' Σ_6perms q̃q̃q̃  evaluated per (triple, x) — no factoring through Γ
//   b[m]  += W_t zm_t P[m,t] Σ_x wr2_x B(t,x)
// One CTA walks a strided subset of triples; per-CTA partial b's are summed in CTA order.
// ------------------------------------------------------------------------------------------
constexpr int NS_THREADS = 256;

__global__ void __launch_bounds__(NS_THREADS)
k_nonsep(const int4* __restrict__ trip, const double* __restrict__ W, int64_t count,
         const double* __restrict__ QT, const double* __restrict__ wr2,
         const double* __restrict__ q, const double* __restrict__ C, const double* __restrict__ v,
         const double* __restrict__ lf, int mode, const double* __restrict__ alpha,
         const int* __restrict__ modes, int p, int nm, int Nx, int NxP, int L, int l_min,
         double* __restrict__ partial) {
    extern __shared__ double sh[];
    double* b_acc = sh;             // [nm]
    double* red = sh + nm;          // [NS_THREADS/32]
    int* md = reinterpret_cast<int*>(red + NS_THREADS / 32);  // [3*nm]
    double* al = reinterpret_cast<double*>(md + 3 * nm + (3 * nm & 1));  // [nm]
    for (int i = threadIdx.x; i < nm; i += blockDim.x) {
        b_acc[i] = 0.0;
        al[i] = alpha[i];
        md[3 * i] = modes[3 * i];
        md[3 * i + 1] = modes[3 * i + 1];
        md[3 * i + 2] = modes[3 * i + 2];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t t = blockIdx.x; t < count; t += gridDim.x) {
        const int4 tr = trip[t];
        const int a1 = tr.x, a2 = tr.y, a3 = tr.z;
        const double* g1 = QT + (int64_t)(a1 - l_min) * p * NxP;
        const double* g2 = QT + (int64_t)(a2 - l_min) * p * NxP;
        const double* g3 = QT + (int64_t)(a3 - l_min) * p * NxP;
        double xs = 0.0;
        for (int x = threadIdx.x; x < Nx; x += blockDim.x) {
            double Bx = 0.0;
            for (int m = 0; m < nm; ++m) {
                int i = md[3 * m], j = md[3 * m + 1], k = md[3 * m + 2];
                double i1 = g1[i * NxP + x], j1 = g1[j * NxP + x], k1 = g1[k * NxP + x];
                double i2 = g2[i * NxP + x], j2 = g2[j * NxP + x], k2 = g2[k * NxP + x];
                double i3 = g3[i * NxP + x], j3 = g3[j * NxP + x], k3 = g3[k * NxP + x];
                double f = i1 * (j2 * k3 + k2 * j3) + j1 * (i2 * k3 + k2 * i3) +
                           k1 * (i2 * j3 + j2 * i3);
                Bx += al[m] * f;
            }
            xs += wr2[x] * Bx;
        }
        for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
        if (lane == 0) red[warp] = xs;
        __syncthreads();
        double X = 0.0;
        for (int w = 0; w < NS_THREADS / 32; ++w) X += red[w];
        double wz = W[t] * zm_weight(mode, a1, a2, a3, C, v, l_min, lf) * X;
        for (int m = threadIdx.x; m < nm; m += blockDim.x) {
            int i = md[3 * m], j = md[3 * m + 1], k = md[3 * m + 2];
            const double* qi = q + (int64_t)i * L - l_min;
            const double* qj = q + (int64_t)j * L - l_min;
            const double* qk = q + (int64_t)k * L - l_min;
            double P = qi[a1] * (qj[a2] * qk[a3] + qk[a2] * qj[a3]) +
                       qj[a1] * (qi[a2] * qk[a3] + qk[a2] * qi[a3]) +
                       qk[a1] * (qi[a2] * qj[a3] + qj[a2] * qi[a3]);
            b_acc[m] += wz * P;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < nm; i += blockDim.x) partial[(int64_t)blockIdx.x * nm + i] = b_acc[i];
}

// Warp-per-triple pointwise kernel for a compile-time basis size P (<= MG_NS_PMAX).
// Per (triple, x) — one lane per x — q̃ at l1, l2, l3 is loaded into registers and the
// primordial bispectrum is summed pointwise over the mode set through the symmetric
// coefficient table Ã (kernel parameter, i.e. constant-bank operands of the DFMAs):
//   B(t,x) = Σ_c q̃_c(x,l1) Σ_{a<=b} Ã[c][ab] S_ab(x),   S_ab = q̃_a(l2)q̃_b(l3) + q̃_b(l2)q̃_a(l3)
// with Ã[k][ij] += α_n, Ã[j][ik] += α_n, Ã[i][jk] += α_n for every mode n = (i<=j<=k) — the
// same 3-term split of the 6-permutation product as f in engine3d.py:115-116, so the sum is
// identical term by term (only its order changes).  The x integral is a warp butterfly; the
// projection b[m] += W_t zm_t X_t P[m,t] is done by the same warp (lane m mod 32 owns mode m,
// q at l1/l2/l3 exchanged by shuffles) into a per-warp shared-memory partial, reduced in warp
// order at the end: one deterministic partial per CTA, no atomics.
// Projection of one triple onto the late-time modes by one warp: my[m] += wz P[m,t], lane =
// mode (mod 32), q_c at l1/l2/l3 held by lane c (P <= 32) and exchanged by shuffles.
__device__ __forceinline__ void ns_project(const int4 tr, double wz, const double* __restrict__ q,
                                           const int* md, int P, int nm, int L, int l_min,
                                           int lane, double* my) {
    double qa = 0.0, qb = 0.0, qc = 0.0;
    if (lane < P) {
        const double* ql = q + (int64_t)lane * L - l_min;
        qa = ql[tr.x];
        qb = ql[tr.y];
        qc = ql[tr.z];
    }
    for (int m0 = 0; m0 < nm; m0 += 32) {
        const int m = m0 + lane;
        const int i = m < nm ? md[3 * m] : 0, j = m < nm ? md[3 * m + 1] : 0,
                  k = m < nm ? md[3 * m + 2] : 0;
        const double i1 = __shfl_sync(0xffffffffu, qa, i), j1 = __shfl_sync(0xffffffffu, qa, j),
                     k1 = __shfl_sync(0xffffffffu, qa, k);
        const double i2 = __shfl_sync(0xffffffffu, qb, i), j2 = __shfl_sync(0xffffffffu, qb, j),
                     k2 = __shfl_sync(0xffffffffu, qb, k);
        const double i3 = __shfl_sync(0xffffffffu, qc, i), j3 = __shfl_sync(0xffffffffu, qc, j),
                     k3 = __shfl_sync(0xffffffffu, qc, k);
        const double Pm = i1 * (j2 * k3 + k2 * j3) + j1 * (i2 * k3 + k2 * i3) +
                          k1 * (i2 * j3 + j2 * i3);
        if (m < nm) my[m] += wz * Pm;
    }
}

template <int P>
struct NsAlpha {
    double a[P][P * (P + 1) / 2];
};

#ifndef NSW_THREADS_
#define NSW_THREADS_ 128  // 168 registers: 3 CTAs (12 warps) per SM
#endif
constexpr int NSW_THREADS = NSW_THREADS_;
#ifndef NS_XV
#define NS_XV 1  // x columns per lane in k_nonsep_warp (2 and 3 measured slower)
#endif

template <int P>
__global__ void __launch_bounds__(NSW_THREADS, 1)
k_nonsep_warp(const int4* __restrict__ trip, const double* __restrict__ W, int64_t count,
              const double* __restrict__ QT, const double* __restrict__ wr2,
              const double* __restrict__ q, const double* __restrict__ C,
              const double* __restrict__ v, const double* __restrict__ lf, int mode,
              const NsAlpha<P> al, const int* __restrict__ modes, int nm, int Nx, int NxP, int L,
              int l_min, double* __restrict__ partial) {
    constexpr int NW = NSW_THREADS / 32;
    extern __shared__ double sh[];
    double* bacc = sh;                                       // [NW][nm]
    int* md = reinterpret_cast<int*>(bacc + (size_t)NW * nm);  // [nm][3]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < NW * nm; i += NSW_THREADS) bacc[i] = 0.0;
    for (int i = tid; i < 3 * nm; i += NSW_THREADS) md[i] = modes[i];
    __syncthreads();
    double* my = bacc + (size_t)warp * nm;
    const int64_t nwarps = (int64_t)gridDim.x * NW;
    for (int64_t t = (int64_t)blockIdx.x * NW + warp; t < count; t += nwarps) {
        const int4 tr = trip[t];
        const double* g1 = QT + (int64_t)(tr.x - l_min) * P * NxP;
        const double* g2 = QT + (int64_t)(tr.y - l_min) * P * NxP;
        const double* g3 = QT + (int64_t)(tr.z - l_min) * P * NxP;
        double xs = 0.0;
        // XV x columns per lane: every coefficient Ã[c][ab] (a uniform-register load) feeds
        // XV DFMAs, and the XV independent accumulator sets double the ILP
#pragma unroll 1
        for (int x0 = lane; x0 < Nx; x0 += 32 * NS_XV) {
            double q1[NS_XV][P], q2[NS_XV][P], q3[NS_XV][P], T[NS_XV][P];
#pragma unroll
            for (int u = 0; u < NS_XV; ++u) {
                const int x = x0 + 32 * u;
                const bool ok = x < Nx;
#pragma unroll
                for (int c = 0; c < P; ++c) {
                    q1[u][c] = ok ? g1[c * NxP + x] : 0.0;
                    q2[u][c] = ok ? g2[c * NxP + x] : 0.0;
                    q3[u][c] = ok ? g3[c * NxP + x] : 0.0;
                    T[u][c] = 0.0;
                }
            }
#pragma unroll
            for (int b = 0; b < P; ++b) {
#pragma unroll
                for (int a = 0; a <= b; ++a) {
                    double sv[NS_XV];
#pragma unroll
                    for (int u = 0; u < NS_XV; ++u) sv[u] = q2[u][a] * q3[u][b] + q2[u][b] * q3[u][a];
#pragma unroll
                    for (int c = 0; c < P; ++c) {
                        const double coef = al.a[c][b * (b + 1) / 2 + a];
#pragma unroll
                        for (int u = 0; u < NS_XV; ++u) T[u][c] = fma(coef, sv[u], T[u][c]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < NS_XV; ++u) {
                const int x = x0 + 32 * u;
                double B = 0.0;
#pragma unroll
                for (int c = 0; c < P; ++c) B = fma(q1[u][c], T[u][c], B);
                if (x < Nx) xs = fma(wr2[x], B, xs);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
        const double wz = W[t] * zm_weight(mode, tr.x, tr.y, tr.z, C, v, l_min, lf) * xs;
        ns_project(tr, wz, q, md, P, nm, L, l_min, lane, my);
    }
    __syncthreads();
    for (int m = tid; m < nm; m += NSW_THREADS) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += bacc[(size_t)w * nm + m];
        partial[(int64_t)blockIdx.x * nm + m] = s;
    }
}

__global__ void k_sum_partials(const double* __restrict__ partial, int nblocks, int nm,
                               double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nm) return;
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partial[(int64_t)b * nm + i];
    out[i] = s;
}

// ------------------------------------------------------------------------------------------
// DMMA form of the pointwise kernel (p <= 8; config 3 has p = 8).  The dominant term of the
// pointwise bispectrum, T[c][(t,x)] = Σ_{a<=b} Ã[c][ab] S_ab(t,x) (576 of the 702 FLOPs per
// (triple, x) at p = 8), is an [8 x 36] x [36 x (t,x)] GEMM with M = p: the m8n8k4 DMMA
// shape, with Ã as the (constant) A operand held in registers for the whole kernel.
//
// The B operand is built in registers, no shared memory: for a chunk of 8 x columns, lane
// (g, t4) owns column x0 + g and k-slot t4 of every k-step, i.e. it must produce S_ab for a
// pair (a, b) that depends on t4.  The K order makes those register indices compile-time:
// the 36 unordered pairs of Z_PP are grouped by cyclic difference d = b - a (mod PP) into
// groups of 4 consecutive rotations {(r, r+d) : r = i0..i0+3}, and lane t4 holds its q̃
// components ROTATED by t4 (register i = component (i + t4) mod PP: per-lane offsets).  Pair (i0 + t4, i0 + d + t4)
// is then registers (i0, (i0 + d) mod PP) in every lane: 9 k-steps at PP = 8, no padding.
//   rotations r < PP/2 only for d = PP/2 (r and r + PP/2 are the same pair);
//   p < PP: components >= p are zero in the tables and the Ã fragments.
// C fragment: lane holds T[c = g][x0 + 2 t4 + {0,1}]; B(x) = Σ_c q̃_c(x,l1) wr2_x T[c][x] is
// accumulated per lane against the wr2-weighted l1 table and reduced across the warp once
// per triple.  Per 8 columns: 9 DMMA + 18 DMUL/DFMA (S) + 2 DFMA + 17 shared-memory loads.
// ------------------------------------------------------------------------------------------
template <int PP>
__host__ __device__ constexpr int ns_groups() { return (PP / 2) * (PP / 4) + (PP / 2 + 3) / 4; }
template <int PP>
__host__ __device__ constexpr int ns_gd(int k) {
    return k < (PP / 2) * (PP / 4) ? k / (PP / 4) : PP / 2;
}
template <int PP>
__host__ __device__ constexpr int ns_gi0(int k) {
    return k < (PP / 2) * (PP / 4) ? (k % (PP / 4)) * 4 : (k - (PP / 2) * (PP / 4)) * 4;
}
// The K order as a "design": R registers per lane and table, k-step k multiplies registers
// (I(k), J(k)) — the same in every lane — and lane t4's register i holds component
// comp(t4, i), so k-slot t4 of k-step k is the pair (comp(t4, I), comp(t4, J)).  A design is
// valid when the 4 x NK (lane, k-step) pairs cover every unordered pair once (padding slots
// get Ã = 0).  In a chunk block, component c lives in row row(c), its 8 columns rotated by 4 h(c)
// (the swizzle that keeps the per-lane-component LDS.64 bank-conflict free: the components a
// register takes across the four lanes of a quad must fall in different 32-byte quarters of
// the 128-byte bank window, quarter = 2 (row & 1) + (h ^ (column >= 4))).
//   NsRot<PP>   the rotation design above: R = PP registers.
//   NsSix       PP = 8 on R = 6 registers (found by exhaustive search, tools/ns_design.py):
//               shared-memory read traffic is 4 lanes x R x 2 tables per column, so 6
//               registers read 3 KB per 8-column chunk instead of 4 KB.  The kernel was
//               co-limited by the shared-memory pipe (44 wavefronts per chunk-warp against
//               180 FP64-datapath cycles on four sub-partitions).
template <int PP>
struct NsRot {
    static constexpr int R = PP, NK = ns_groups<PP>();
    __host__ __device__ static constexpr int I(int k) { return ns_gi0<PP>(k); }
    __host__ __device__ static constexpr int J(int k) { return (ns_gi0<PP>(k) + ns_gd<PP>(k)) % PP; }
    __host__ __device__ static constexpr int comp(int t4, int i) { return (i + t4) % PP; }
    __host__ __device__ static constexpr bool live(int k, int t4) {
        return 2 * ns_gd<PP>(k) < PP || ns_gi0<PP>(k) + t4 < PP / 2;
    }
    __host__ __device__ static constexpr int row(int c) { return c; }
    __host__ __device__ static constexpr int h(int c) { return (c >> 1) & 1; }
};
struct NsSix {
    static constexpr int R = 6, NK = 9;
    __host__ __device__ static constexpr int I(int k) {
        constexpr int t[9] = {0, 1, 0, 0, 0, 0, 0, 1, 1};
        return t[k];
    }
    __host__ __device__ static constexpr int J(int k) {
        constexpr int t[9] = {0, 1, 1, 2, 3, 4, 5, 2, 3};
        return t[k];
    }
    __host__ __device__ static constexpr int comp(int t4, int i) {
        constexpr int t[4][6] = {{0, 1, 2, 3, 4, 5}, {6, 2, 4, 7, 0, 1}, {7, 4, 1, 3, 0, 5},
                                 {5, 3, 2, 6, 1, 4}};
        return t[t4][i];
    }
    __host__ __device__ static constexpr bool live(int, int) { return true; }
    // quarter labels (0,1,0,2,3,2,1,3): even rows <- components 0,1,2,6; odd rows <- 3,4,5,7
    __host__ __device__ static constexpr int row(int c) {
        constexpr int t[8] = {0, 2, 4, 1, 3, 5, 6, 7};
        return t[c];
    }
    __host__ __device__ static constexpr int h(int c) {
        constexpr int t[8] = {0, 1, 0, 0, 1, 0, 1, 1};
        return t[c];
    }
};
#ifndef NS_ROT8
#define NS_ROT8 0  // 1: rotation design at PP = 8 too (A/B measurements)
#endif
template <int PP> struct NsDesignOf { using type = NsRot<PP>; };
#if !NS_ROT8
template <> struct NsDesignOf<8> { using type = NsSix; };
#endif
template <int PP> using NsDesign = typename NsDesignOf<PP>::type;
// slot (doubles) of (component c, column xi) inside a PP x 8 chunk block
template <int PP>
__host__ __device__ inline int ns_slot(int c, int xi) {
    return NsDesign<PP>::row(c) * 8 + ((xi + 4 * NsDesign<PP>::h(c)) & 7);
}

template <int PP>
struct NsAfrag {
    double a[NsDesign<PP>::NK][32];  // [k-step][lane]: lane (g, t4) holds Ã[g][pair(k, t4)]
};

// Tables of the DMMA kernel, x in blocks of 8 columns ("chunks"), one 8-column row per
// component, PP*64 bytes per (l, chunk):
//   QTS[l][xb][c][8]: q̃[c][8 xb + i][l] at column position (i + 4 ((c >> 1) & 1)) & 7 —
//                     the swizzle makes the rotated B-operand reads bank-conflict free (a half
//                     warp reads 4 consecutive components x 4 columns: the two component pairs
//                     land on opposite column halves of the 128-byte bank window);
//   Q1W[l][xb][c][8]: wr2[x] q̃[c][x][l] (no swizzle: read as double2 per lane).
// Components >= p and columns >= Nx are zero.  Built from the plan's QT[l][c][NxP].
template <int PP>
__global__ void k_ns_tables(const double* __restrict__ QT, const double* __restrict__ wr2, int p,
                            int Nx, int NxP, int L, int XB8, double* __restrict__ QTS,
                            double* __restrict__ Q1W) {
    const int64_t total = (int64_t)L * XB8 * PP * 8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int xi = (int)(i & 7);
        int64_t r = i >> 3;
        const int c = (int)(r % PP);
        r /= PP;
        const int xb = (int)(r % XB8);
        const int l = (int)(r / XB8);
        const int x = xb * 8 + xi;
        const double val = (c < p && x < Nx) ? QT[((int64_t)l * p + c) * NxP + x] : 0.0;
        Q1W[i] = x < Nx ? wr2[x] * val : 0.0;
        QTS[(i / (PP * 8)) * (PP * 8) + ns_slot<PP>(c, xi)] = val;
    }
}

// WZ[t] = W_t zm_t of the resident sparse domain (once per domain).
__global__ void k_ns_weights(const int4* __restrict__ trip, const double* __restrict__ W,
                             int64_t count, const double* __restrict__ C,
                             const double* __restrict__ v, const double* __restrict__ lf,
                             int mode, int l_min, double* __restrict__ WZ) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int4 tr = trip[t];
        WZ[t] = W[t] * zm_weight(mode, tr.x, tr.y, tr.z, C, v, l_min, lf);
    }
}

// Staging of the B-operand inputs.  Read straight from global memory, the rotated layout
// costs 16 LDG.64 per lane per chunk (every component is read by all four lanes of a quad)
// and round 2's first version was bound by L1 wavefronts (one 256-byte LDG.64 occupies the
// L1 data pipe for ~4 cycles; profiles/r02_ncu_nonsep_dmma_v1.txt).  Here each warp streams
// its triples' data into shared memory with cp.async.bulk (TMA engine, no LSU wavefronts),
// NS_ST stages of NS_CH chunks: [l2 chunks][l3 chunks], completing on a per-warp, per-stage
// mbarrier; the rotated reads are then LDS.64 (2 wavefronts each).  The wr2-weighted l1 row
// (one double2 per lane per chunk, no redundancy) is read from global memory.
// Lane 0 of the warp is the producer: after the warp has consumed a stage it refills the slot
// with the stage NS_ST ahead (crossing into the warp's next triple), so copies run under the
// DMMAs of the stages in between.
// Warps and chains (measured, profiles/r02_nonsep_dmma_variants.txt): a warp that has issued
// a DMMA cannot issue anything for ~14 cycles, so its ~300 non-tensor instructions per stage
// (LDS, pair products, refill, loop) never overlap its own tensor work — only other warps'.
// With w warps per SM sub-partition each on the FP64 datapath a fraction d ~ 1/3 of its time,
// the datapath is busy ~1 - (1 - d)^w: 12 warps per CTA (w = 3) reach 69 %, 16 warps 75 %,
// where it levels off (20 and 24 warps: same).  16 warps leave 128 registers per lane, so the
// pair products of only NS_G = 2 chunks are live at once (2 accumulator chains per warp; the
// other warps of the sub-partition cover the DMMA D -> C latency), in NS_CH / NS_G groups per
// stage, and 2 stages of 4 KB per warp keep the CTA at 128 KB of shared memory.
#ifndef NSD_THREADS_
#define NSD_THREADS_ 512
#endif
constexpr int NSD_THREADS = NSD_THREADS_;
#ifndef NS_CH
#define NS_CH 4  // chunks of 8 x columns per stage
#endif
#ifndef NS_ST
#define NS_ST 2  // stages per warp
#endif
#ifndef NS_FENCE
#define NS_FENCE 0  // 1: generic->async proxy fence before a slot's refill (A/B measurements)
#endif
#ifndef NS_ASMEM
#define NS_ASMEM 0  // 1: Ã fragments read from shared memory per k-step (more warps per CTA)
#endif
#ifndef NS_FOLD
#define NS_FOLD 0  // 1: a = b pairs as one product, factor 2 folded into the Ã fragment
                   // (2 of 18 FP64 operand instructions fewer, yet measured slower: 5.69 vs 5.58 ms)
#endif
#ifndef NS_G
#define NS_G 2  // chunks whose pair products are live at once (accumulator chains in flight)
#endif

template <int PP>
struct NsStage {
    static constexpr int CHUNK = PP * 8;                 // doubles per (l, chunk)
    static constexpr int DOUBLES = 2 * NS_CH * CHUNK;     // l2, l3 blocks
    static constexpr size_t WARP_BYTES = (size_t)NS_ST * DOUBLES * 8 + NS_ST * 8;
};

template <int PP>
__global__ void __launch_bounds__(NSD_THREADS, 1)
k_nonsep_dmma(const int4* __restrict__ trip, const double* __restrict__ WZ, int64_t count,
              const double* __restrict__ QTS, const double* __restrict__ Q1W, int XB8,
              const NsAfrag<PP> af, const double* __restrict__ q, const int* __restrict__ modes,
              int P, int nm, int L, int l_min, double* __restrict__ partial, MgBounds bd) {
    using SG = NsStage<PP>;
    using DS = NsDesign<PP>;
    constexpr int NK = DS::NK, NR = DS::R, CH = NS_CH, NST = NS_ST, CHUNK = SG::CHUNK;
    constexpr int NW = NSD_THREADS / 32;
    extern __shared__ __align__(16) double sh[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    // [NW warps x NST stages x DOUBLES][NW x NST mbarriers][NW][nm] partial b [3 nm] modes
    double* stg = sh + (size_t)warp * NST * SG::DOUBLES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sh + (size_t)NW * NST * SG::DOUBLES) + warp * NST;
    double* bacc = reinterpret_cast<double*>(reinterpret_cast<uint64_t*>(
                       sh + (size_t)NW * NST * SG::DOUBLES) + NW * NST);
    int* md = reinterpret_cast<int*>(bacc + (size_t)NW * nm);
    for (int i = tid; i < NW * nm; i += NSD_THREADS) bacc[i] = 0.0;
    for (int i = tid; i < 3 * nm; i += NSD_THREADS) md[i] = modes[i];
    if (lane == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(full + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    // Ã fragments: registers for the whole kernel.  The empty asm makes each value opaque, so
    // under register pressure ptxas spills it instead of re-reading the kernel parameter with a
    // per-lane index (LDC with 32 different addresses serialises: measured 6.7 -> 17.5 ms).
#if NS_ASMEM
    // Ã fragments in shared memory instead (one conflict-free LDS.64 per k-step and group):
    // frees 2 NK registers per lane for CTAs of more than 16 warps (96-register cap)
    double* a_s = reinterpret_cast<double*>(md + 3 * nm + (nm & 1));
    for (int i = tid; i < NK * 32; i += NSD_THREADS) a_s[i] = af.a[i >> 5][i & 31];
    a_s += lane;
#else
    double a[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        a[k] = af.a[k][lane];
        asm volatile("" : "+d"(a[k]));
    }
#endif
    // lane's rotated component offsets (doubles) within a chunk block: register i holds
    // component (i + t4) mod PP of column g, stored at swizzled column position
    int off[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) off[i] = ns_slot<PP>(DS::comp(t4, i), g);
    __syncthreads();
    double* my = bacc + (size_t)warp * nm;
    const int64_t nwarps = (int64_t)gridDim.x * NW;
    const int nstg = (XB8 + CH - 1) / CH;  // stages per triple
    const int64_t lstride = (int64_t)XB8 * CHUNK;

    // producer cursor (lane 0): the (triple, stage) to issue next and its source rows
    int64_t pt = (int64_t)blockIdx.x * NW + warp;
    int ps = 0;
    const double *src2 = QTS, *src3 = QTS;
    auto load_cursor = [&]() {
        const int4 ptr = trip[pt];
        MG_DCHECK(ptr.x >= l_min && ptr.y >= ptr.x && ptr.z >= ptr.y && ptr.z - l_min < L, CK_NS_L);
        src2 = QTS + (ptr.y - l_min) * lstride;
        src3 = QTS + (ptr.z - l_min) * lstride;
    };
    if (pt < count) load_cursor();
    auto issue = [&](int slot) {
        if (pt >= count) return;
        const int nch = min(CH, XB8 - ps * CH);
        const uint32_t bytes = (uint32_t)nch * CHUNK * 8;
        double* st = stg + (size_t)slot * SG::DOUBLES;
        MG_DCHECK(in_range(src2 - QTS, (int64_t)nch * CHUNK, bd.qts) &&
                      in_range(src3 - QTS, (int64_t)nch * CHUNK, bd.qts),
                  CK_NS_QTS);
        mbar_arrive_expect_tx(full + slot, 2 * bytes);
        bulk_g2s(st, src2, bytes, full + slot);
        bulk_g2s(st + CH * CHUNK, src3, bytes, full + slot);
        src2 += CH * CHUNK;
        src3 += CH * CHUNK;
        if (++ps == nstg) {
            ps = 0;
            pt += nwarps;
            if (pt < count) load_cursor();
        }
    };
    if (lane == 0)
        for (int s = 0; s < NST; ++s) issue(s);
    __syncwarp();

    // One stage = NS_CH chunks: their pair products S first (each chunk's rotated q̃ rows are
    // dead once its NK S values exist), then the DMMAs of the NS_CH independent accumulator
    // chains (a warp keeps several DMMAs in flight; the DMMA D -> C latency is ~4 issue slots
    // of the sub-partition's DMMA pipe), then the l1 contraction.  FULL: all NS_CH chunks hold
    // data (straight-line code, no zero fill); otherwise chunks >= nch are skipped, DMMAs
    // included (the last stage of a triple: 38 chunks = 9 x 4 + 2 at Nx = 300).
    // One group of NS_G chunks: pair products, DMMA chains, l1 contraction.  FULL: every chunk
    // of the group holds data (straight-line code); otherwise chunks >= nv are skipped.
    auto group_body = [&](auto full_c, const double* st, const double* b1, int u0, int nv,
                          double& xs0, double& xs1) {
        constexpr bool FULL = decltype(full_c)::value;
        constexpr int G = NS_G;
        double S[G][NK];
#pragma unroll
        for (int v = 0; v < G; ++v) {
            if (FULL || v < nv) {
                const double* b2 = st + (u0 + v) * CHUNK;
                const double* b3 = st + (CH + u0 + v) * CHUNK;
                double r2[NR], r3[NR];
#pragma unroll
                for (int i = 0; i < NR; ++i) {
                    r2[i] = b2[off[i]];
                    r3[i] = b3[off[i]];
                }
#pragma unroll
                for (int k = 0; k < NK; ++k) {
                    const int i0 = DS::I(k), j = DS::J(k);
                    S[v][k] = (NS_FOLD && i0 == j) ? r2[i0] * r3[i0]
                                                   : r2[i0] * r3[j] + r2[j] * r3[i0];
                }
            }
        }
        // accumulator row c = g exists only for g < PP (PP = 4: lanes g >= 4 hold zero rows of
        // T and must not read past their chunk's PP component rows)
        double2 w[G];
#pragma unroll
        for (int v = 0; v < G; ++v) {
            MG_DCHECK(!((FULL || v < nv) && g < PP) ||
                          in_range(b1 + (u0 + v) * CHUNK - Q1W, 2, bd.q1w), CK_NS_Q1W);
            w[v] = ((FULL || v < nv) && g < PP)
                       ? __ldg(reinterpret_cast<const double2*>(b1 + (u0 + v) * CHUNK))
                       : make_double2(0.0, 0.0);
        }
        double acc[G][2];
#pragma unroll
        for (int v = 0; v < G; ++v) acc[v][0] = acc[v][1] = 0.0;
#pragma unroll
        for (int k = 0; k < NK; ++k)
#if NS_ASMEM
            {
                const double ak = a_s[k * 32];
#pragma unroll
                for (int v = 0; v < G; ++v)
                    if (FULL || v < nv) dmma884(acc[v], ak, S[v][k]);
            }
#else
#pragma unroll
            for (int v = 0; v < G; ++v)
                if (FULL || v < nv) dmma884(acc[v], a[k], S[v][k]);
#endif
#pragma unroll
        for (int v = 0; v < G; ++v) {
            xs0 = fma(w[v].x, acc[v][0], xs0);
            xs1 = fma(w[v].y, acc[v][1], xs1);
        }
    };
    // One stage = NS_CH chunks in groups of NS_G (NS_G chains in flight, NS_G x NK pair products
    // live).  A stage whose chunks all hold data is one straight-line block; the last stage of
    // a triple (38 chunks = 9 x 4 + 2 at Nx = 300) runs its full groups, then the remainder.
    auto stage_body = [&](const double* st, const double* b1, int nch, double& xs0, double& xs1) {
        constexpr int G = NS_G;
        static_assert(CH % G == 0, "chunk groups must divide the stage");
        if (nch == CH) {
#pragma unroll
            for (int u0 = 0; u0 < CH; u0 += G)
                group_body(std::true_type{}, st, b1, u0, G, xs0, xs1);
        } else {
#pragma unroll
            for (int u0 = 0; u0 < CH; u0 += G) {
                if (u0 + G <= nch)
                    group_body(std::true_type{}, st, b1, u0, G, xs0, xs1);
                else if (u0 < nch)
                    group_body(std::false_type{}, st, b1, u0, nch - u0, xs0, xs1);
            }
        }
    };

    uint32_t gst = 0;  // stages consumed by this warp (slot = gst % NST, phase = gst / NST)
    for (int64_t t = (int64_t)blockIdx.x * NW + warp; t < count; t += nwarps) {
        const int4 tr = trip[t];
        const double* p1 = Q1W + (tr.x - l_min) * lstride + g * 8 + 2 * t4;
        double xs0 = 0.0, xs1 = 0.0;
        for (int s = 0; s < nstg; ++s, ++gst) {
            const int slot = (int)(gst % NST);
            mbar_wait(full + slot, (int)((gst / NST) & 1));
            const double* st = stg + (size_t)slot * SG::DOUBLES;
            const int nch = min(CH, XB8 - s * CH);
            const double* b1 = p1 + (int64_t)s * CH * CHUNK;
            stage_body(st, b1, nch, xs0, xs1);
            // Slot consumed by every lane (its LDS results have been used by the FP64 ops
            // above, so the reads are complete before the warp converges here): refill it
            // with the stage NST ahead.
            __syncwarp();
            if (lane == 0) {
#if NS_FENCE
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#endif
                issue(slot);
            }
            __syncwarp();
        }
        double xs = xs0 + xs1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
        ns_project(tr, WZ[t] * xs, q, md, P, nm, L, l_min, lane, my);
    }
    __syncthreads();
    for (int m = tid; m < nm; m += NSD_THREADS) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += bacc[(size_t)w * nm + m];
        partial[(int64_t)blockIdx.x * nm + m] = s;
    }
}

// Ã fragments of the DMMA kernel from the symmetric table at[c][pair] (see above).
template <int PP>
static NsAfrag<PP> ns_afrag(const std::vector<double>& at, int p, int P2) {
    NsAfrag<PP> f;
    using DS = NsDesign<PP>;
    for (int k = 0; k < DS::NK; ++k)
        for (int lane = 0; lane < 32; ++lane) {
            const int g = lane >> 2, t4 = lane & 3;
            const int a = DS::comp(t4, DS::I(k)), b = DS::comp(t4, DS::J(k));
            const bool ok = DS::live(k, t4) && a < p && b < p && g < p;
            f.a[k][lane] = ok ? (NS_FOLD && a == b ? 2.0 : 1.0) *
                                    at[(size_t)g * P2 + pair_idx(std::min(a, b), std::max(a, b))]
                              : 0.0;
        }
    return f;
}

template <int PP>
static void launch_nonsep_dmma(mg_plan* Pl, const std::vector<double>& at, cudaStream_t st) {
    const int XB8 = ceil_div(Pl->Nx, 8);
    if (!Pl->ns_qt2.p) {  // x-chunked, swizzled q̃ tables (once per plan)
        Pl->ns_qt2.alloc((size_t)Pl->L * XB8 * PP * 8);
        Pl->ns_q1w.alloc((size_t)Pl->L * XB8 * PP * 8);
        k_ns_tables<PP><<<1184, 256, 0, st>>>(Pl->QT.p, Pl->wr2.p, Pl->p, Pl->Nx, Pl->NxP, Pl->L,
                                              XB8, Pl->ns_qt2.p, Pl->ns_q1w.p);
        MG_LAUNCHED();
    }
    const NsAfrag<PP> af = ns_afrag<PP>(at, Pl->p, Pl->P2);
    constexpr int NW = NSD_THREADS / 32;
    const size_t shm = NW * NsStage<PP>::WARP_BYTES + (size_t)NW * Pl->nm * 8 +
                       (size_t)(3 * Pl->nm + (Pl->nm & 1)) * 4 +
                       (NS_ASMEM ? sizeof(NsAfrag<PP>) : 0);
    MG_REQUIRE(shm <= 227 * 1024, "too many modes for the non-separable DMMA kernel");
    static bool attr[64] = {false};
    if (!attr[Pl->device & 63]) {
        MG_CUDA(cudaFuncSetAttribute(k_nonsep_dmma<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024));
        attr[Pl->device & 63] = true;
    }
    int sms = 148;
    MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, Pl->device));
    Pl->ns_blocks = sms;  // one CTA of NW warps per SM (shared memory holds every warp's stages)
    Pl->ns_part.ensure((size_t)Pl->ns_blocks * Pl->nm);
    k_nonsep_dmma<PP><<<Pl->ns_blocks, NSD_THREADS, shm, st>>>(
        reinterpret_cast<const int4*>(Pl->ns_trip.p), Pl->ns_wz.p, Pl->ns_count, Pl->ns_qt2.p,
        Pl->ns_q1w.p, XB8, af, Pl->q.p, Pl->modes.p, Pl->p, Pl->nm, Pl->L, Pl->l_min,
        Pl->ns_part.p,
        MgBounds{0, 0, 0, 0, 0, 0, 0, 0, (int64_t)Pl->ns_qt2.n, (int64_t)Pl->ns_q1w.n});
}

template <int P>
static void launch_nonsep_warp(mg_plan* Pl, const std::vector<double>& at, cudaStream_t st) {
    NsAlpha<P> al;
    constexpr int P2 = P * (P + 1) / 2;
    for (int c = 0; c < P; ++c)
        for (int ab = 0; ab < P2; ++ab) al.a[c][ab] = at[(size_t)c * P2 + ab];
    const size_t shm = (size_t)(NSW_THREADS / 32) * Pl->nm * 8 + (size_t)3 * Pl->nm * 4;
    static int resident[64] = {0};  // CTAs per SM of this instance (per device)
    int& res = resident[Pl->device & 63];
    if (!res) {
        MG_CUDA(cudaFuncSetAttribute(k_nonsep_warp<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     100 * 1024));
        MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, k_nonsep_warp<P>, NSW_THREADS,
                                                              shm));
        res = std::max(res, 1);
    }
    int sms = 148;
    MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, Pl->device));
    Pl->ns_blocks = sms * res;
    Pl->ns_part.ensure((size_t)Pl->ns_blocks * Pl->nm);
    k_nonsep_warp<P><<<Pl->ns_blocks, NSW_THREADS, shm, st>>>(
        reinterpret_cast<const int4*>(Pl->ns_trip.p), Pl->ns_W.p, Pl->ns_count, Pl->QT.p,
        Pl->wr2.p, Pl->q.p, Pl->C.p, Pl->v.p, Pl->lf.p, Pl->h2_mode, al, Pl->modes.p, Pl->nm,
        Pl->Nx, Pl->NxP, Pl->L, Pl->l_min, Pl->ns_part.p);
}

// Kernel timing of the non-separable path without a host synchronisation per call: event
// pairs accumulate and are resolved when the timings are read (mg_plan_kernel_ms).
static void ns_mark(mg_plan* P, cudaStream_t st) {
    if (!P->profile) return;
    if (P->ns_used == P->ns_events.size()) {
        cudaEvent_t e;
        MG_CUDA(cudaEventCreate(&e));
        P->ns_events.push_back(e);
    }
    MG_CUDA(cudaEventRecord(P->ns_events[P->ns_used++], st));
}

void nonsep_collect(mg_plan* P) {
    for (size_t i = 0; i + 1 < P->ns_used; i += 2) {
        MG_CUDA(cudaEventSynchronize(P->ns_events[i + 1]));
        float ms = 0.f;
        MG_CUDA(cudaEventElapsedTime(&ms, P->ns_events[i], P->ns_events[i + 1]));
        P->prof_ms[7] += ms;
    }
    P->ns_used = 0;
}

// Resident sparse domain of the non-separable path: validated, packed (l1,l2,l3,0) int4 + W.
void nonsep_set_domain(mg_plan* P, const int32_t* l1, const int32_t* l2, const int32_t* l3,
                       const double* W, int64_t count) {
    MG_NVTX("mg:nonsep_set_domain");
    std::vector<int32_t> packed(4 * (size_t)count);
    for (int64_t i = 0; i < count; ++i) {
        MG_REQUIRE(l1[i] <= l2[i] && l2[i] <= l3[i], "triples must satisfy l1 <= l2 <= l3");
        MG_REQUIRE(l1[i] >= P->l_min && l3[i] <= P->l_max, "triple outside [l_min, l_max]");
        MG_REQUIRE(std::isfinite(W[i]), "sparse-domain weights must be finite");
        packed[4 * i] = l1[i];
        packed[4 * i + 1] = l2[i];
        packed[4 * i + 2] = l3[i];
        packed[4 * i + 3] = 0;
    }
    P->ns_count = count;
    if (!count) return;
    P->ns_trip.upload(packed.data(), packed.size());
    P->ns_W.upload(W, count);
    P->ns_wz.ensure(count);
    k_ns_weights<<<std::min<int64_t>((count + 255) / 256, 4096), 256>>>(
        reinterpret_cast<const int4*>(P->ns_trip.p), P->ns_W.p, count, P->C.p, P->v.p, P->lf.p,
        P->h2_mode, P->l_min, P->ns_wz.p);
    MG_LAUNCHED();
    MG_CUDA(cudaStreamSynchronize(0));  // packed is pageable host memory
}

// b = Σ_t W_t zm_t P[:,t] Σ_x wr2_x B(t,x) over the resident sparse domain; b_dev (device,
// optional) and b_host (optional) receive the nm coefficients.
void nonsep_execute(mg_plan* P, const double* alpha, double* b_dev, double* b_host,
                    cudaStream_t st) {
    MG_NVTX("mg:nonsep_execute");
    const int nm = P->nm, p = P->p, P2 = P->P2;
    P->ns_b.ensure(nm);
    if (P->ns_count == 0) {
        MG_CUDA(cudaMemsetAsync(P->ns_b.p, 0, nm * sizeof(double), st));
    } else {
        // symmetric coefficient table Ã[c][ab] (see k_nonsep_warp), host-built per call
        std::vector<double> at((size_t)p * P2, 0.0);
        for (int m = 0; m < nm; ++m) {
            const int i = P->hmodes[3 * m], j = P->hmodes[3 * m + 1], k = P->hmodes[3 * m + 2];
            at[(size_t)k * P2 + pair_idx(i, j)] += alpha[m];
            at[(size_t)j * P2 + pair_idx(i, k)] += alpha[m];
            at[(size_t)i * P2 + pair_idx(j, k)] += alpha[m];
        }
        if (!P->ns_blocks || p > 16) {  // generic kernel (p > 16): 2 CTAs per SM
            int sms = 148;
            MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device));
            P->ns_blocks = 2 * sms;
        }
        P->ns_part.ensure((size_t)P->ns_blocks * nm);
        MG_REQUIRE((size_t)(NSW_THREADS / 32) * nm * 8 + (size_t)3 * nm * 4 <= 100 * 1024,
                   "too many modes for the non-separable kernel");
        ns_mark(P, st);  // (start, end) event pair, resolved lazily by nonsep_collect
        static const bool no_dmma = std::getenv("MG_NS_DFMA") != nullptr;  // A/B switch
        switch ((no_dmma || p > 8) ? 100 + p : p) {
            case 1: case 2: case 3: case 4: launch_nonsep_dmma<4>(P, at, st); break;
            case 5: case 6: case 7: case 8: launch_nonsep_dmma<8>(P, at, st); break;
#define MG_NS_CASE(N) \
    case 100 + N: launch_nonsep_warp<N>(P, at, st); break;
            MG_NS_CASE(1) MG_NS_CASE(2) MG_NS_CASE(3) MG_NS_CASE(4) MG_NS_CASE(5) MG_NS_CASE(6)
            MG_NS_CASE(7) MG_NS_CASE(8) MG_NS_CASE(9) MG_NS_CASE(10) MG_NS_CASE(11)
            MG_NS_CASE(12) MG_NS_CASE(13) MG_NS_CASE(14) MG_NS_CASE(15) MG_NS_CASE(16)
#undef MG_NS_CASE
            default: {
                P->ns_alpha.upload(alpha, nm, st);
                const size_t shm = (size_t)nm * 8 + NS_THREADS / 32 * 8 + (3 * nm + 1) * 4 + 8 +
                                   (size_t)nm * 8;
                MG_REQUIRE(shm <= 227 * 1024, "too many modes for the non-separable path");
                MG_CUDA(cudaFuncSetAttribute(k_nonsep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)std::max<size_t>(shm, 48 * 1024)));
                k_nonsep<<<P->ns_blocks, NS_THREADS, shm, st>>>(
                    reinterpret_cast<const int4*>(P->ns_trip.p), P->ns_W.p, P->ns_count, P->QT.p,
                    P->wr2.p, P->q.p, P->C.p, P->v.p, P->lf.p, P->h2_mode, P->ns_alpha.p, P->modes.p, p,
                    nm, P->Nx, P->NxP, P->L, P->l_min, P->ns_part.p);
                break;
            }
        }
        MG_LAUNCHED();
        k_sum_partials<<<(nm + 127) / 128, 128, 0, st>>>(P->ns_part.p, P->ns_blocks, nm, P->ns_b.p);
        MG_LAUNCHED();
        ns_mark(P, st);
        P->launches = 2;
    }
    if (b_dev)
        MG_CUDA(cudaMemcpyAsync(b_dev, P->ns_b.p, nm * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (b_host) {
        MG_CUDA(cudaMemcpyAsync(b_host, P->ns_b.p, nm * sizeof(double), cudaMemcpyDeviceToHost, st));
        MG_CUDA(cudaStreamSynchronize(st));
    }
}

void nonsep(mg_plan* P, const double* alpha, const int32_t* l1, const int32_t* l2,
            const int32_t* l3, const double* W, int64_t count, double* b, cudaStream_t st) {
    nonsep_set_domain(P, l1, l2, l3, W, count);
    nonsep_execute(P, alpha, nullptr, b, st);
}

}  // namespace mg
