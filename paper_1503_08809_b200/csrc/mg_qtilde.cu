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
#include <vector>

#include "mg_bessel.cuh"
#include "mg_common.cuh"

namespace mg {

constexpr int QB_XT = 4;     // x values per CTA
constexpr int QB_KT = 256;   // k per tile (= threads)
constexpr int QB_LT = 8;     // l per chunk
constexpr int QB_LDU = QB_KT + 1;

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
        BesselNorm bn = bessel_prepare(z, l_max);
        st.nrm[i] = bn.norm;
        st.lsw[i] = bn.lsw;
        st.stot[i] = bn.stot;
        // upward state at l = l_min - 1: (j_{l_min-2}, j_{l_min-1})
        double j0 = MGB_DIV(sin(z), z);
        double jm = j0, jc = MGB_DIV(MGB_SUB(j0, cos(z)), z);  // (j0, j1)
        for (int l = 1; l < l_min - 1; ++l) {
            double jn = bessel_step(l, jc, jm, z);
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
                double jn = bessel_step(l, jd, jp, z);
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

// One sweep (dir = +1 ascending/upward, -1 descending/Miller) over all l for XT x-values.
__global__ void __launch_bounds__(QB_KT)
k_qb_sweep(int dir, const double* __restrict__ k, int Nk, const double* __restrict__ x, int Nx,
           const double* __restrict__ delta, const double* __restrict__ b, int p, int l_min,
           int l_max, QState st, double* __restrict__ qt) {
    extern __shared__ double sh[];
    double* us = sh;                                   // [LT][XT][LDU]
    double* bs = sh + QB_LT * QB_XT * QB_LDU;          // [p][KT]
    const int x0 = blockIdx.x * QB_XT;
    const int L = l_max - l_min + 1;
    const int nout = p * QB_XT * QB_LT;
    const int nchunk = (L + QB_LT - 1) / QB_LT;
    for (int ch = 0; ch < nchunk; ++ch) {
        // chunk covers l = lc0 + dir*li, li < nl
        const int lc0 = dir > 0 ? l_min + ch * QB_LT : l_max - ch * QB_LT;
        const int nl = min(QB_LT, L - ch * QB_LT);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int kt = 0; kt < Nk; kt += QB_KT) {
            const int ki = kt + threadIdx.x;
            bool any = false;
            for (int xi = 0; xi < QB_XT; ++xi) {
                const int xg = x0 + xi;
                const bool okp = ki < Nk && xg < Nx;
                const int64_t si = (int64_t)xg * Nk + ki;
                double z = okp ? k[ki] * x[xg] : 1.0;
                int lsw = okp ? st.lsw[si] : l_max;
                const bool live_u = okp && z > 0.0;  // z = 0 contributes nothing
                if (dir > 0) {
                    double jm = okp ? st.ua[si] : 0.0, jc = okp ? st.ub[si] : 0.0;
                    for (int li = 0; li < QB_LT; ++li) {
                        int l = lc0 + li;
                        double u = 0.0;
                        if (live_u && li < nl && l <= lsw) {
                            double jn = bessel_step(l - 1, jc, jm, z);
                            jm = jc;
                            jc = jn;
                            u = delta[(int64_t)(l - l_min) * Nk + ki] * jn;
                            any = true;
                        }
                        us[(li * QB_XT + xi) * QB_LDU + threadIdx.x] = u;
                    }
                    if (okp) { st.ua[si] = jm; st.ub[si] = jc; }
                } else {
                    double jp = okp ? st.da[si] : 0.0, jd = okp ? st.db[si] : 0.0;
                    int s = okp ? st.ds[si] : 0;
                    BesselNorm bn;
                    bn.norm = okp ? st.nrm[si] : 0.0;
                    bn.stot = okp ? st.stot[si] : 0;
                    for (int li = 0; li < QB_LT; ++li) {
                        int l = lc0 - li;
                        double u = 0.0;
                        if (live_u && li < nl && l > lsw) {
                            u = delta[(int64_t)(l - l_min) * Nk + ki] * bessel_denorm(jd, s, bn);
                            any = true;
                            double jn = bessel_step(l, jd, jp, z);  // jhat_{l-1}
                            jp = jd;
                            jd = jn;
                            if (fabs(jd) > MGB_BIG) {
                                jd = ldexp(jd, -MGB_SHIFT);
                                jp = ldexp(jp, -MGB_SHIFT);
                                ++s;
                            }
                        }
                        us[(li * QB_XT + xi) * QB_LDU + threadIdx.x] = u;
                    }
                    if (okp) { st.da[si] = jp; st.db[si] = jd; st.ds[si] = s; }
                }
            }
            for (int c = 0; c < p; ++c)
                bs[c * QB_KT + threadIdx.x] = ki < Nk ? b[(int64_t)c * Nk + ki] : 0.0;
            const int live = __syncthreads_or(any);
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
            __syncthreads();
        }
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
    }
}

// Build Δ, C and q̃ on the device.  Inputs are host arrays; outputs device buffers
// (C_dev [L], qt_dev [p][Nx][L], optional delta_dev [L][Nk]).
void build_qtilde_dev(const double* k, const double* wk, int Nk, const double* x, int Nx,
                      const double* eps, const double* qk, int p, int l_min, int l_max,
                      double X, double kd, double amp, double* C_dev, double* qt_dev,
                      double* delta_out_dev, cudaStream_t s) {
    MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
    MG_REQUIRE(Nk >= 1 && Nx >= 1 && p >= 1, "Nk, Nx, p must be >= 1");
    MG_REQUIRE(p * QB_XT * QB_LT <= 4 * QB_KT, "p_max too large for the q-tilde kernel (<= 32)");
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
        QState st{ua.p, ub.p, da.p, dbb.p, ds.p, nrm.p, lsw.p, stot.p};
        k_qb_prepare<<<(int)std::min<size_t>((np + 255) / 256, 148 * 64), 256, 0, s>>>(
            dk.p, Nk, dx.p, Nx, l_min, l_max, st);
        MG_LAUNCHED();
        const size_t shm = (size_t)(QB_LT * QB_XT * QB_LDU + p * QB_KT) * sizeof(double);
        MG_CUDA(cudaFuncSetAttribute(k_qb_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)shm));
        const int grid = (Nx + QB_XT - 1) / QB_XT;
        k_qb_sweep<<<grid, QB_KT, shm, s>>>(+1, dk.p, Nk, dx.p, Nx, delta, db.p, p, l_min, l_max,
                                            st, qt_dev);
        MG_LAUNCHED();
        k_qb_sweep<<<grid, QB_KT, shm, s>>>(-1, dk.p, Nk, dx.p, Nx, delta, db.p, p, l_min, l_max,
                                            st, qt_dev);
        MG_LAUNCHED();
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
