// mg_gamma2d.cu — the μ-quadrature ("separable", Modal2D) Γ engine on the device.
//
// Reference: engine2d.py:62-211.
//   P[a,b,x,m] = Σ_l lw_l q_a(l) q̃_b(x,l) P_l(μ_m),   lw_l = (2l+1)/(v_l sqrt C_l)
//     (build_ptable, :62-95: ascending l, Kahan-compensated)
//   Γ2d[n,n'] = Σ_x w_x r_x^2 Σ_m w_m perm3(P[rows(n), cols(n')](x,m)) / (48π)
//     (gamma2d_entry, :112-129: μ first, then the radial rule)
// The P table is built with the reference's exact operation order (term = ((lw q_a) q̃_b) P_l,
// Kahan update y = term - comp; t = acc + y; comp = (t - acc) - y), each FP64 op an explicit
// round-to-nearest intrinsic, so it reproduces the reference table bit for bit.  The cell
// kernel stages P[:, :, x, μ-chunk] in shared memory and gives every thread one Γ cell.
#include <algorithm>
#include <vector>

#include "mg_common.cuh"

namespace mg {

// P[((a*p + b)*Nx + x)*nmu + m], one thread per element, sequential Kahan over l.
__global__ void k_ptable(const double* __restrict__ q, const double* __restrict__ qt,
                         const double* __restrict__ lw, const double* __restrict__ leg, int p,
                         int Nx, int L, int nmu, double* __restrict__ P) {
    const int64_t total = (int64_t)p * p * Nx * nmu;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(i % nmu);
        int64_t r = i / nmu;
        const int x = (int)(r % Nx);
        r /= Nx;
        const int b = (int)(r % p), a = (int)(r / p);
        const double* qa = q + (int64_t)a * L;
        const double* qb = qt + ((int64_t)b * Nx + x) * L;
        double acc = 0.0, comp = 0.0;
        for (int l = 0; l < L; ++l) {
            const double lwq = __dmul_rn(lw[l], qa[l]);
            const double term = __dmul_rn(__dmul_rn(lwq, qb[l]), leg[(int64_t)l * nmu + m]);
            const double y = __dsub_rn(term, comp);
            const double t = __dadd_rn(acc, y);
            comp = __dsub_rn(__dsub_rn(t, acc), y);
            acc = t;
        }
        P[i] = acc;
    }
}

constexpr int G2_TILE = 16;  // 16 x 16 cells per CTA

__global__ void __launch_bounds__(G2_TILE* G2_TILE)
k_gamma2d_cells(const double* __restrict__ P, const int* __restrict__ modes, int n, int p,
                int Nx, int nmu, int mc, const double* __restrict__ mu_w,
                const double* __restrict__ wr2, double* __restrict__ gamma) {
    extern __shared__ double sp[];  // [p*p][mc]
    const int tn = threadIdx.x / G2_TILE, tq = threadIdx.x % G2_TILE;
    const int nrow = blockIdx.y * G2_TILE + tn, ncol = blockIdx.x * G2_TILE + tq;
    const bool ok = nrow < n && ncol < n;
    int r0 = 0, r1 = 0, r2 = 0, c0 = 0, c1 = 0, c2 = 0;
    if (ok) {
        r0 = modes[3 * nrow]; r1 = modes[3 * nrow + 1]; r2 = modes[3 * nrow + 2];
        c0 = modes[3 * ncol]; c1 = modes[3 * ncol + 1]; c2 = modes[3 * ncol + 2];
    }
    const int pp = p * p;
    double acc = 0.0;
    for (int x = 0; x < Nx; ++x) {
        double inner = 0.0;
        for (int m0 = 0; m0 < nmu; m0 += mc) {
            const int mn = min(mc, nmu - m0);
            __syncthreads();
            for (int e = threadIdx.x; e < pp * mc; e += blockDim.x) {
                const int ab = e / mc, mm = e % mc;
                sp[e] = mm < mn ? P[((int64_t)ab * Nx + x) * nmu + m0 + mm] : 0.0;
            }
            __syncthreads();
            if (ok) {
                const double* s00 = sp + (r0 * p + c0) * mc;
                const double* s01 = sp + (r0 * p + c1) * mc;
                const double* s02 = sp + (r0 * p + c2) * mc;
                const double* s10 = sp + (r1 * p + c0) * mc;
                const double* s11 = sp + (r1 * p + c1) * mc;
                const double* s12 = sp + (r1 * p + c2) * mc;
                const double* s20 = sp + (r2 * p + c0) * mc;
                const double* s21 = sp + (r2 * p + c1) * mc;
                const double* s22 = sp + (r2 * p + c2) * mc;
                for (int mm = 0; mm < mn; ++mm) {
                    const double m00 = s00[mm], m01 = s01[mm], m02 = s02[mm];
                    const double m10 = s10[mm], m11 = s11[mm], m12 = s12[mm];
                    const double m20 = s20[mm], m21 = s21[mm], m22 = s22[mm];
                    // engine2d.py:101-109 term order
                    const double per = m00 * m11 * m22 + m00 * m12 * m21 + m01 * m10 * m22 +
                                       m01 * m12 * m20 + m02 * m10 * m21 + m02 * m11 * m20;
                    inner += per * mu_w[m0 + mm];
                }
            }
        }
        acc += wr2[x] * inner;
    }
    if (ok) gamma[(int64_t)nrow * n + ncol] = acc / (48.0 * 3.141592653589793);
}

void ptable_dev(const double* q, const double* qt, const double* lw, const double* leg, int p,
                int Nx, int L, int nmu, double* P_dev) {
    DBuf<double> dq, dqt, dlw, dleg;
    dq.upload(q, (size_t)p * L);
    dqt.upload(qt, (size_t)p * Nx * L);
    dlw.upload(lw, L);
    dleg.upload(leg, (size_t)L * nmu);
    const int64_t total = (int64_t)p * p * Nx * nmu;
    k_ptable<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 64), 256>>>(
        dq.p, dqt.p, dlw.p, dleg.p, p, Nx, L, nmu, P_dev);
    MG_LAUNCHED();
    MG_CUDA(cudaDeviceSynchronize());
}

void gamma2d_dev(const double* P_dev, const int* modes_host, int n, int p, int Nx, int nmu,
                 const double* mu_w, const double* wr2, double* gamma_host) {
    DBuf<int> dm;
    DBuf<double> dw, dr, dg;
    dm.upload(modes_host, 3 * (size_t)n);
    dw.upload(mu_w, nmu);
    dr.upload(wr2, Nx);
    dg.alloc((size_t)n * n);
    const int mc = std::max(1, std::min(32, 12288 / (p * p)));
    const size_t shm = (size_t)p * p * mc * sizeof(double);
    if (shm > 48 * 1024)
        MG_CUDA(cudaFuncSetAttribute(k_gamma2d_cells, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)shm));
    dim3 grid(ceil_div(n, G2_TILE), ceil_div(n, G2_TILE));
    k_gamma2d_cells<<<grid, G2_TILE * G2_TILE, shm>>>(P_dev, dm.p, n, p, Nx, nmu, mc, dw.p,
                                                        dr.p, dg.p);
    MG_LAUNCHED();
    MG_CUDA(cudaMemcpy(gamma_host, dg.p, (size_t)n * n * sizeof(double),
                       cudaMemcpyDeviceToHost));
}

}  // namespace mg
