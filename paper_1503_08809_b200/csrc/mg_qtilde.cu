// mg_qtilde.cu — stage 1: Δ_l(k), C_l and the projected modes q̃_p(x,l) on the device.
//
// Equation (BASELINE.json config 0):
//   q̃_p(x,l) = Σ_k wk k^2 q_p(k) Δ_l(k) j_l(k x),  Δ_l(k) = j_l(X k) e^{-(k/kd)^2}(1 + a ε_lk)
// The reference has no stage 1; its stand-in q̃ = q(l) w(r) is
// synthesize_basis (basis.py:279-297).  Oracle: oracle/qtilde_ref.py (scipy).
//
// The L x Nk x Nx Bessel values (3e10 at config 4, 240 GB) are never stored: a CTA owns
// XT x-values, marches l in chunks of LT, and for each k-tile of KT advances the per-(k,x)
// recurrence states (kept in global memory between chunks), writes u = Δ_l(k) j_l(kx) to
// shared memory and contracts it with b_p(k) = wk k^2 q_p(k).  Two sweeps cover the two
// recurrence regimes (mg_bessel.cuh): ascending l for l <= l_sw(kx), descending l (Miller,
// normalised by a pre-pass) for l > l_sw.  Accumulation order is fixed -> deterministic.
#include <algorithm>
#include <climits>
#include <vector>

#include "mg_bessel.cuh"
#include "mg_common.cuh"
#include "mg_dmma.cuh"

namespace mg {

#ifndef MG_QB_XT
#define MG_QB_XT 2  // measured: 2 beats 4 at c1 (0.042 vs 0.056 s), ties at c4; 1 is slower
#endif
constexpr int QB_XT = MG_QB_XT;       // x values per CTA
#ifndef MG_QB_KT
#define MG_QB_KT 256
#endif
constexpr int QB_KT = MG_QB_KT;       // k per tile (= threads)
constexpr int QB_LT = 32 / QB_XT;     // l per chunk (XT * LT = 32 output columns)
#ifndef MG_QB_RECIP
#define MG_QB_RECIP 1  // sweep recurrences multiply by 1/z (one DMUL + one DFMA per step)
                       // instead of scipy's operation order with an IEEE division per step
                       // (mg_bessel.cuh bessel_step, kept for the Bessel table and Δ): the
                       // division was ~3/4 of the sweep's instructions
#endif
#ifndef MG_QB_PREFETCH
#define MG_QB_PREFETCH 1  // load a chunk's Δ_l(k) values before its recurrence steps
#endif
// resident CTAs per SM the register allocation must allow: the shared-memory tiles of MF
// m-fragments ((32 + 8 MF) rows of QB_KT + 4 doubles) decide how many actually fit
#ifndef MG_QB_MINB
#define MG_QB_MINB(MF) ((MF) <= 2 ? 2 : 1)
#endif
#ifndef MG_QB_SKIP
#define MG_QB_SKIP 1  // skip (k tile, l chunk) pairs outside the sweep's regime (k_qb_tile_range)
#endif
#ifndef MG_QB_DMMA
#define MG_QB_DMMA 1  // contraction over k on DMMA (1) or as per-thread DFMA dot products (0)
#endif
// row strides of the shared-memory u and b tiles: +4 keeps the m8n8k4 fragment reads (lane
// (g,t) reads row 8f+g, column 4s+t) bank-conflict free; +1 the scalar dot products'
constexpr int QB_LDU = MG_QB_DMMA ? QB_KT + 4 : QB_KT + 1;
constexpr int QB_LDB = MG_QB_DMMA ? QB_KT + 4 : QB_KT;
constexpr int QB_NC = QB_LT * QB_XT;  // (l, x) output columns per chunk = 32 = 4 n-fragments

// Recurrence step of the q̃ sweeps: j_{l±1} = (2l+1)/z j_l - j_{l∓1}.
__device__ __forceinline__ double qb_step(int l, double jl, double jother, double z, double rz) {
#if MG_QB_RECIP
    return fma((double)(2 * l + 1) * rz, jl, -jother);
#else
    return bessel_step(l, jl, jother, z);
#endif
}

// Δ[l-l_min][k] for one thread per k (z = X k), plus b[c][k] = wk k^2 qk[c][k].
__global__ void k_delta(const double* __restrict__ k, const double* __restrict__ wk, int Nk,
                        const double* __restrict__ eps, const double* __restrict__ qk, int p,
                        int l_min, int l_max, double X, double kd, double amp,
                        double* __restrict__ delta, double* __restrict__ b) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nk) return;
    const double kk = k[i];
    const double damp = exp(-((kk / kd) * (kk / kd)));
    bessel_sequence(X * kk, l_max, [&](int l, double j) {
        if (l >= l_min) {
            int64_t o = (int64_t)(l - l_min) * Nk + i;
            delta[o] = (j * damp) * (1.0 + amp * eps[o]);
        }
    });
    const double w = (wk[i] * kk) * kk;
    for (int c = 0; c < p; ++c) b[(int64_t)c * Nk + i] = qk[(int64_t)c * Nk + i] * w;
}

// C[l] = Σ_k Δ^2 (wk/k), one block per l, fixed-order tree reduction.
__global__ void k_cell(const double* __restrict__ delta, const double* __restrict__ k,
                       const double* __restrict__ wk, int Nk, double* __restrict__ C) {
    __shared__ double red[256];
    const double* d = delta + (int64_t)blockIdx.x * Nk;
    double s = 0.0;
    for (int i = threadIdx.x; i < Nk; i += blockDim.x) s += (d[i] * d[i]) * (wk[i] / k[i]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) C[blockIdx.x] = red[0];
}

// Per (x,k) pair: normalisation + initial states of both sweeps.  Layout [x][k].
struct QState {
    double* ua;  // upward j_{l-1}
    double* ub;  // upward j_l
    double* da;  // downward jhat_{l+1}
    double* db;  // downward jhat_l
    int* ds;     // downward rescale count
    double* nrm;
    int* lsw;
    int* stot;
    int* tmin;  // [x block][k tile]: smallest / largest switch point l_sw in the tile; a sweep
    int* tmax;  // skips the (k tile, l chunk) pairs that lie wholly outside its regime
};

__global__ void k_qb_prepare(const double* __restrict__ k, int Nk, const double* __restrict__ x,
                             int Nx, int l_min, int l_max, QState st) {
    int64_t total = (int64_t)Nk * Nx;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int xi = (int)(i / Nk), ki = (int)(i % Nk);
        double z = k[ki] * x[xi];
        if (!(z > 0.0)) {  // j_l(0) = 0 for l >= 1: both sweeps emit nothing
            st.nrm[i] = 0.0; st.lsw[i] = l_max; st.stot[i] = 0;
            st.ua[i] = st.ub[i] = st.da[i] = st.db[i] = 0.0; st.ds[i] = 0;
            continue;
        }
        const double rz = 1.0 / z;
        auto step = [z, rz](int l, double jl, double jo) { return qb_step(l, jl, jo, z, rz); };
        BesselNorm bn = bessel_prepare_with(z, l_max, step);
        st.nrm[i] = bn.norm;
        st.lsw[i] = bn.lsw;
        st.stot[i] = bn.stot;
        // upward state at l = l_min - 1: (j_{l_min-2}, j_{l_min-1})
        double j0 = MGB_DIV(sin(z), z);
        double jm = j0, jc = MGB_DIV(MGB_SUB(j0, cos(z)), z);  // (j0, j1)
        for (int l = 1; l < l_min - 1; ++l) {
            double jn = step(l, jc, jm);
            jm = jc;
            jc = jn;
        }
        st.ua[i] = jm;
        st.ub[i] = jc;
        // downward state at l = l_max: (jhat_{l_max+1}, jhat_{l_max}, s)
        double jp = 0.0, jd = MGB_SEED;
        int s = 0;
        if (bn.lsw < l_max) {
            for (int l = bn.ls; l > l_max; --l) {
                double jn = step(l, jd, jp);
                jp = jd;
                jd = jn;
                if (fabs(jd) > MGB_BIG) {
                    jd = ldexp(jd, -MGB_SHIFT);
                    jp = ldexp(jp, -MGB_SHIFT);
                    ++s;
                }
            }
        }
        st.da[i] = jp;
        st.db[i] = jd;
        st.ds[i] = s;
    }
}

// Range of the switch points of one (x block, k tile): block (k tile, x block), QB_KT threads.
// Upward recurrences are live for l <= l_sw, downward ones for l > l_sw, so a chunk starting
// at l = lc0 has no live recurrence in the tile when lc0 > max l_sw (ascending sweep: every
// recurrence of the tile has finished) or lc0 <= min l_sw (descending sweep: likewise).  About
// half of all (k tile, chunk) visits of the two sweeps are such dead pairs.
__global__ void __launch_bounds__(QB_KT)
k_qb_tile_range(int Nk, int Nx, QState st) {
    __shared__ int smin[QB_KT / 32], smax[QB_KT / 32];
    const int ki = blockIdx.x * QB_KT + threadIdx.x;
    int lo = INT_MAX, hi = -1;
    for (int xi = 0; xi < QB_XT; ++xi) {
        const int xg = blockIdx.y * QB_XT + xi;
        if (ki < Nk && xg < Nx) {
            const int v = st.lsw[(int64_t)xg * Nk + ki];
            lo = min(lo, v);
            hi = max(hi, v);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        smin[threadIdx.x >> 5] = lo;
        smax[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < QB_KT / 32; ++w) {
            lo = min(lo, smin[w]);
            hi = max(hi, smax[w]);
        }
        st.tmin[blockIdx.y * gridDim.x + blockIdx.x] = lo;
        st.tmax[blockIdx.y * gridDim.x + blockIdx.x] = hi;
    }
}

// One sweep (dir = +1 ascending/upward, -1 descending/Miller) over all l for XT x-values.
// DMMA contraction (MG_QB_DMMA): per chunk, C[c][(l,x)] = Σ_k b[c][k] u[(l,x)][k] with
// M = p (MF m-fragments), N = 32 (l,x) columns, K = Nk; warp w owns the k-slice
// [32w, 32w+32) of every k-tile and all MF x 4 output fragments; the 8 warp partials are
// summed in warp order at the end of the chunk (deterministic).
template <int MF>
__global__ void __launch_bounds__(QB_KT, MG_QB_MINB(MF))
k_qb_sweep(int dir, const double* __restrict__ k, int Nk, const double* __restrict__ x, int Nx,
           const double* __restrict__ delta, const double* __restrict__ b, int p, int l_min,
           int l_max, QState st, double* __restrict__ qt) {
    extern __shared__ double sh[];
    double* us = sh;                                   // [LT][XT][LDU]
    double* bs = sh + QB_LT * QB_XT * QB_LDU;          // [MF*8][LDB] (rows >= p stay zero)
    const int x0 = blockIdx.x * QB_XT;
#if MG_QB_DMMA
    for (int i = threadIdx.x; i < (MF * 8 - p) * QB_LDB; i += QB_KT) bs[p * QB_LDB + i] = 0.0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
#endif
    const int L = l_max - l_min + 1;
#if !MG_QB_DMMA
    const int nout = p * QB_XT * QB_LT;
#endif
    const int nchunk = (L + QB_LT - 1) / QB_LT;
    for (int ch = 0; ch < nchunk; ++ch) {
        // chunk covers l = lc0 + dir*li, li < nl
        const int lc0 = dir > 0 ? l_min + ch * QB_LT : l_max - ch * QB_LT;
        const int nl = min(QB_LT, L - ch * QB_LT);
#if MG_QB_DMMA
        double cf[MF][4][2];
#pragma unroll
        for (int mf = 0; mf < MF; ++mf)
#pragma unroll
            for (int nf = 0; nf < 4; ++nf) cf[mf][nf][0] = cf[mf][nf][1] = 0.0;
#else
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#endif
        for (int kt = 0; kt < Nk; kt += QB_KT) {
#if MG_QB_SKIP
            {  // CTA-uniform: no recurrence of this k tile is live anywhere in the chunk
                const int ti = blockIdx.x * ((Nk + QB_KT - 1) / QB_KT) + kt / QB_KT;
                if (dir > 0 ? st.tmax[ti] < lc0 : lc0 <= st.tmin[ti]) continue;
            }
#endif
            const int ki = kt + threadIdx.x;
            bool any = false;
            // the XT recurrences of this k advance together (l outer, x inner): XT independent
            // dependency chains per step instead of one long chain per x
            bool okp[QB_XT], live_u[QB_XT];
            double z[QB_XT], rz[QB_XT];
            int lsw[QB_XT];
            int64_t si[QB_XT];
#pragma unroll
            for (int xi = 0; xi < QB_XT; ++xi) {
                const int xg = x0 + xi;
                okp[xi] = ki < Nk && xg < Nx;
                si[xi] = (int64_t)xg * Nk + ki;
                z[xi] = okp[xi] ? k[ki] * x[xg] : 1.0;
                rz[xi] = 1.0 / z[xi];
                lsw[xi] = okp[xi] ? st.lsw[si[xi]] : l_max;
                live_u[xi] = okp[xi] && z[xi] > 0.0;  // z = 0 contributes nothing
            }
            // the chunk's Δ_l(k) values up front: QB_LT independent loads in flight at once
            // (inside the recurrence loop they were issued a few at a time and each group
            // paid an L2 round trip with only 2-4 warps per sub-partition to hide it)
#if MG_QB_PREFETCH
            double dlv[QB_LT];
#pragma unroll
            for (int li = 0; li < QB_LT; ++li)
                dlv[li] = li < nl ? __ldg(delta + (int64_t)(lc0 + dir * li - l_min) * Nk +
                                          min(ki, Nk - 1))
                                  : 0.0;
#define QB_DL(li, l) dlv[li]
#define QB_UNROLL _Pragma("unroll")
#else
#define QB_DL(li, l) ((li) < nl ? delta[(int64_t)((l) - l_min) * Nk + min(ki, Nk - 1)] : 0.0)
#define QB_UNROLL
#endif
            if (dir > 0) {
                double jm[QB_XT], jc[QB_XT];
#pragma unroll
                for (int xi = 0; xi < QB_XT; ++xi) {
                    jm[xi] = okp[xi] ? st.ua[si[xi]] : 0.0;
                    jc[xi] = okp[xi] ? st.ub[si[xi]] : 0.0;
                }
QB_UNROLL
                for (int li = 0; li < QB_LT; ++li) {
                    const int l = lc0 + li;
                    const double dl = QB_DL(li, l);
#pragma unroll
                    for (int xi = 0; xi < QB_XT; ++xi) {
                        double u = 0.0;
                        if (live_u[xi] && li < nl && l <= lsw[xi]) {
                            const double jn = qb_step(l - 1, jc[xi], jm[xi], z[xi], rz[xi]);
                            jm[xi] = jc[xi];
                            jc[xi] = jn;
                            u = dl * jn;
                            any = true;
                        }
                        us[(li * QB_XT + xi) * QB_LDU + threadIdx.x] = u;
                    }
                }
#pragma unroll
                for (int xi = 0; xi < QB_XT; ++xi)
                    if (okp[xi]) { st.ua[si[xi]] = jm[xi]; st.ub[si[xi]] = jc[xi]; }
            } else {
                double jp[QB_XT], jd[QB_XT];
                int sc[QB_XT];
                BesselNorm bn[QB_XT];
#pragma unroll
                for (int xi = 0; xi < QB_XT; ++xi) {
                    jp[xi] = okp[xi] ? st.da[si[xi]] : 0.0;
                    jd[xi] = okp[xi] ? st.db[si[xi]] : 0.0;
                    sc[xi] = okp[xi] ? st.ds[si[xi]] : 0;
                    bn[xi].norm = okp[xi] ? st.nrm[si[xi]] : 0.0;
                    bn[xi].stot = okp[xi] ? st.stot[si[xi]] : 0;
                }
QB_UNROLL
                for (int li = 0; li < QB_LT; ++li) {
                    const int l = lc0 - li;
                    const double dl = QB_DL(li, l);
#pragma unroll
                    for (int xi = 0; xi < QB_XT; ++xi) {
                        double u = 0.0;
                        if (live_u[xi] && li < nl && l > lsw[xi]) {
                            u = dl * bessel_denorm(jd[xi], sc[xi], bn[xi]);
                            any = true;
                            const double jn = qb_step(l, jd[xi], jp[xi], z[xi], rz[xi]);  // jhat_{l-1}
                            jp[xi] = jd[xi];
                            jd[xi] = jn;
                            if (fabs(jd[xi]) > MGB_BIG) {
                                jd[xi] = ldexp(jd[xi], -MGB_SHIFT);
                                jp[xi] = ldexp(jp[xi], -MGB_SHIFT);
                                ++sc[xi];
                            }
                        }
                        us[(li * QB_XT + xi) * QB_LDU + threadIdx.x] = u;
                    }
                }
#pragma unroll
                for (int xi = 0; xi < QB_XT; ++xi)
                    if (okp[xi]) { st.da[si[xi]] = jp[xi]; st.db[si[xi]] = jd[xi]; st.ds[si[xi]] = sc[xi]; }
            }
            for (int c = 0; c < p; ++c)
                bs[c * QB_LDB + threadIdx.x] = ki < Nk ? b[(int64_t)c * Nk + ki] : 0.0;
            const int live = __syncthreads_or(any);
#if MG_QB_DMMA
            if (live) {  // u, b past Nk are zero, so the full k-slice is summed
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const int kk = warp * 32 + ks * 4 + t4;
                    double af[MF], bf[4];
#pragma unroll
                    for (int mf = 0; mf < MF; ++mf) af[mf] = bs[(mf * 8 + g) * QB_LDB + kk];
#pragma unroll
                    for (int nf = 0; nf < 4; ++nf) bf[nf] = us[(nf * 8 + g) * QB_LDU + kk];
#pragma unroll
                    for (int mf = 0; mf < MF; ++mf)
#pragma unroll
                        for (int nf = 0; nf < 4; ++nf) dmma884(cf[mf][nf], af[mf], bf[nf]);
                }
            }
#else
            if (live) {
                const int kn = min(QB_KT, Nk - kt);
                for (int r = 0; r < 4; ++r) {
                    int o = threadIdx.x + r * QB_KT;
                    if (o < nout) {
                        int li = o % QB_LT, xi = (o / QB_LT) % QB_XT, c = o / (QB_LT * QB_XT);
                        const double* ur = us + (li * QB_XT + xi) * QB_LDU;
                        const double* br = bs + c * QB_KT;
                        double s = 0.0;
                        for (int kk = 0; kk < kn; ++kk) s += br[kk] * ur[kk];
                        acc[r] += s;
                    }
                }
            }
#endif
            __syncthreads();
        }
#if MG_QB_DMMA
        // warp partials -> us (free after the last k-tile), then summed in warp order
        double* red = us;  // [8 warps][MF*8][32]
#pragma unroll
        for (int mf = 0; mf < MF; ++mf)
#pragma unroll
            for (int nf = 0; nf < 4; ++nf) {
                const int m = mf * 8 + g, n = nf * 8 + 2 * t4;
                red[(warp * MF * 8 + m) * QB_NC + n] = cf[mf][nf][0];
                red[(warp * MF * 8 + m) * QB_NC + n + 1] = cf[mf][nf][1];
            }
        __syncthreads();
        for (int o = threadIdx.x; o < p * QB_NC; o += QB_KT) {
            const int c = o / QB_NC, n = o % QB_NC, li = n / QB_XT, xi = n % QB_XT;
            double v = 0.0;
            for (int w = 0; w < QB_KT / 32; ++w) v += red[(w * MF * 8 + c) * QB_NC + n];
            const int l = lc0 + dir * li, xg = x0 + xi;
            if (li < nl && xg < Nx) {
                const int64_t oi = ((int64_t)c * Nx + xg) * L + (l - l_min);
                qt[oi] = dir > 0 ? v : qt[oi] + v;
            }
        }
        __syncthreads();  // red aliases us
#else
        for (int r = 0; r < 4; ++r) {
            int o = threadIdx.x + r * QB_KT;
            if (o < nout) {
                int li = o % QB_LT, xi = (o / QB_LT) % QB_XT, c = o / (QB_LT * QB_XT);
                int l = lc0 + dir * li, xg = x0 + xi;
                if (li < nl && xg < Nx) {
                    int64_t oi = ((int64_t)c * Nx + xg) * L + (l - l_min);
                    qt[oi] = dir > 0 ? acc[r] : qt[oi] + acc[r];
                }
            }
        }
#endif
    }
}

template <int MF>
static void launch_qb_sweep(int grid, size_t shm, cudaStream_t s, int dir, const double* k, int Nk,
                            const double* x, int Nx, const double* delta, const double* b, int p,
                            int l_min, int l_max, QState st, double* qt) {
    MG_CUDA(cudaFuncSetAttribute(k_qb_sweep<MF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)shm));
    k_qb_sweep<MF><<<grid, QB_KT, shm, s>>>(dir, k, Nk, x, Nx, delta, b, p, l_min, l_max, st, qt);
    MG_LAUNCHED();
}

// Build Δ, C and q̃ on the device.  Inputs are host arrays; outputs device buffers
// (C_dev [L], qt_dev [p][Nx][L], optional delta_dev [L][Nk]).
void build_qtilde_dev(const double* k, const double* wk, int Nk, const double* x, int Nx,
                      const double* eps, const double* qk, int p, int l_min, int l_max,
                      double X, double kd, double amp, double* C_dev, double* qt_dev,
                      double* delta_out_dev, cudaStream_t s) {
    MG_NVTX("mg:build_qtilde");
    MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
    MG_REQUIRE(Nk >= 1 && Nx >= 1 && p >= 1, "Nk, Nx, p must be >= 1");
    // the sweep kernel holds up to QB_PMAX components (4 DMMA m-fragments); larger bases are
    // built in component blocks (each block re-runs the Bessel recurrences)
    constexpr int QB_PMAX = MG_QB_DMMA ? 32 : 4 * QB_KT / (QB_XT * QB_LT);
    for (int i = 0; i < Nk; ++i) MG_REQUIRE(k[i] > 0, "k grid must be > 0");
    const int L = l_max - l_min + 1;
    DBuf<double> dk, dwk, dx, deps, dqk, ddelta, db;
    dk.upload(k, Nk, s);
    dwk.upload(wk, Nk, s);
    dx.upload(x, Nx, s);
    deps.upload(eps, (size_t)L * Nk, s);
    dqk.upload(qk, (size_t)p * Nk, s);
    double* delta = delta_out_dev;
    if (!delta) {
        ddelta.alloc((size_t)L * Nk);
        delta = ddelta.p;
    }
    db.alloc((size_t)p * Nk);
    k_delta<<<(Nk + 127) / 128, 128, 0, s>>>(dk.p, dwk.p, Nk, deps.p, dqk.p, p, l_min, l_max, X,
                                            kd, amp, delta, db.p);
    MG_LAUNCHED();
    if (C_dev) {
        k_cell<<<L, 256, 0, s>>>(delta, dk.p, dwk.p, Nk, C_dev);
        MG_LAUNCHED();
    }
    if (qt_dev) {
        const size_t np = (size_t)Nk * Nx;
        DBuf<double> ua(np), ub(np), da(np), dbb(np), nrm(np);
        DBuf<int> ds(np), lsw(np), stot(np);
        const int grid = (Nx + QB_XT - 1) / QB_XT;
        const int nkt = (Nk + QB_KT - 1) / QB_KT;
        DBuf<int> tmin((size_t)grid * nkt), tmax((size_t)grid * nkt);
        QState st{ua.p, ub.p, da.p, dbb.p, ds.p, nrm.p, lsw.p, stot.p, tmin.p, tmax.p};
        for (int c0 = 0; c0 < p; c0 += QB_PMAX) {  // component blocks: qt is [p][Nx][L]
            const int pb = std::min(QB_PMAX, p - c0);
            const double* bb = db.p + (size_t)c0 * Nk;
            double* qo = qt_dev + (size_t)c0 * Nx * L;
            k_qb_prepare<<<(int)std::min<size_t>((np + 255) / 256, 148 * 64), 256, 0, s>>>(
                dk.p, Nk, dx.p, Nx, l_min, l_max, st);
            MG_LAUNCHED();
            k_qb_tile_range<<<dim3(nkt, grid), QB_KT, 0, s>>>(Nk, Nx, st);
            MG_LAUNCHED();
            const int mf = (pb + 7) / 8;
            const size_t shm = (size_t)(QB_LT * QB_XT * QB_LDU + (MG_QB_DMMA ? mf * 8 : pb) * QB_LDB) *
                               sizeof(double);
            for (int dir : {+1, -1}) {
                switch (MG_QB_DMMA ? mf : 1) {
                    case 1: launch_qb_sweep<1>(grid, shm, s, dir, dk.p, Nk, dx.p, Nx, delta, bb, pb, l_min, l_max, st, qo); break;
                    case 2: launch_qb_sweep<2>(grid, shm, s, dir, dk.p, Nk, dx.p, Nx, delta, bb, pb, l_min, l_max, st, qo); break;
                    case 3: launch_qb_sweep<3>(grid, shm, s, dir, dk.p, Nk, dx.p, Nx, delta, bb, pb, l_min, l_max, st, qo); break;
                    default: launch_qb_sweep<4>(grid, shm, s, dir, dk.p, Nk, dx.p, Nx, delta, bb, pb, l_min, l_max, st, qo); break;
                }
            }
        }
        MG_CUDA(cudaStreamSynchronize(s));  // temporaries die with this scope
    } else {
        MG_CUDA(cudaStreamSynchronize(s));
    }
}

__global__ void k_bessel_table(const double* __restrict__ z, int nz, int l_max,
                               double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nz) return;
    double* o = out + (int64_t)i * (l_max + 1);
    bessel_sequence(z[i], l_max, [&](int l, double v) { o[l] = v; });
}

void bessel_table(const double* z, int nz, int l_max, double* out) {
    MG_REQUIRE(nz >= 0 && l_max >= 0, "invalid bessel table size");
    if (nz == 0) return;
    DBuf<double> dz, dout;
    dz.upload(z, nz);
    dout.alloc((size_t)nz * (l_max + 1));
    k_bessel_table<<<(nz + 127) / 128, 128>>>(dz.p, nz, l_max, dout.p);
    MG_LAUNCHED();
    MG_CUDA(cudaMemcpy(out, dout.p, (size_t)nz * (l_max + 1) * sizeof(double),
                       cudaMemcpyDeviceToHost));
}

}  // namespace mg
