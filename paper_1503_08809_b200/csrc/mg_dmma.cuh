// mg_dmma.cuh — FP64 tensor-core (DMMA) block GEMM with pluggable operand generators.
//
// Blackwell has no FP64 tcgen05 kind; FP64 tensor math is the legacy `mma.sync ... .f64`
// path, which ptxas lowers to DMMA.8x8x4 on sm_100a (every f64 mma shape becomes a sequence
// of 8x8x4 DMMAs, see profiles/r01_fp64_peak.txt).  Measured on this pool's B200: DMMA
// 37.0 TFLOP/s vs DFMA 36.4 TFLOP/s, so the Γ contractions are written as DMMA GEMMs.
//
// Tile: BM=128 x BN=128 x BK=16, 256 threads (8 warps as 2 x 4), warp tile 64 x 32 made of
// 8 x 4 m8n8k4 fragments (64 FP64 accumulators per lane).  Operands are staged in shared
// memory k-major (As[k][m], Bs[k][n]) with a +4 double row pad so the m8n8k4 fragment loads
// (lane (g,t) reads [k0+t][m0+g]) are bank-conflict free.  Two smem stages; the next
// k-tile's operands are produced into registers (by the loader functors, which may compute
// them: pair products, weights, gathers) while the DMMAs of the current tile run.
#pragma once

#include <cuda_runtime.h>

namespace mg {

constexpr int GB_M = 128;
constexpr int GB_N = 128;
constexpr int GB_K = 16;
constexpr int GB_THREADS = 256;
constexpr int GB_PAD = 4;
constexpr int GB_LDA = GB_M + GB_PAD;  // row stride of As[k][*] in doubles
constexpr int GB_LDB = GB_N + GB_PAD;
constexpr int GB_STAGE = GB_K * (GB_LDA + GB_LDB);  // doubles per stage
constexpr size_t GB_SMEM = 2 * GB_STAGE * sizeof(double);

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

// Per-thread operand registers for one k-tile: 2048 elements / 256 threads = 8 each.
struct Frag8 {
    double v[8];
};

// Loader contract (A side; B identical with n in place of m):
//   __device__ void load(int kt, Frag8& r) const;      // produce this thread's 8 elements
//   __device__ void store(double* As, const Frag8& r) const;  // write them to As[k][m]
// Two canonical thread->element maps are provided:
//   "k-run":  m = tid % 128, k = (tid / 128) * 8 + i      (8 consecutive k of one m)
//   "m-run":  k = tid / 16,  m = (tid % 16) * 8 + i       (8 consecutive m of one k)
__device__ __forceinline__ void store_krun(double* S, int ld, const Frag8& r) {
    int m = threadIdx.x & 127, k0 = (threadIdx.x >> 7) * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) S[(k0 + i) * ld + m] = r.v[i];
}
__device__ __forceinline__ void store_mrun(double* S, int ld, const Frag8& r) {
    int k = threadIdx.x >> 4, m0 = (threadIdx.x & 15) * 8;
    double2* d = reinterpret_cast<double2*>(S + k * ld + m0);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = make_double2(r.v[2 * i], r.v[2 * i + 1]);
}

// Accumulator ownership: lane (g = lane/4, t = lane%4) of warp (wm, wn) holds, for
// fragment (mi, ni), C[wm*64 + mi*8 + g][wn*32 + ni*8 + 2t + {0,1}].
struct Acc {
    double c[8][4][2];
};

// Core loop.  `ktiles` k-tiles of 16; A/B loaders as above; returns accumulators.
template <class LA, class LB>
__device__ __forceinline__ void gemm_mainloop(int ktiles, const LA& la, const LB& lb,
                                              double* smem, Acc& acc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc.c[mi][ni][0] = acc.c[mi][ni][1] = 0.0;
    if (ktiles <= 0) return;

    Frag8 ra, rb;
    la.load(0, ra);
    lb.load(0, rb);
    la.store(smem, ra);
    lb.store(smem + GB_K * GB_LDA, rb);
    __syncthreads();

    for (int kt = 0; kt < ktiles; ++kt) {
        const double* As = smem + (kt & 1) * GB_STAGE;
        const double* Bs = As + GB_K * GB_LDA;
        const bool more = kt + 1 < ktiles;
        if (more) {
            la.load(kt + 1, ra);
            lb.load(kt + 1, rb);
        }
#pragma unroll
        for (int ks = 0; ks < GB_K / 4; ++ks) {
            double a[8], b[4];
            const double* Ak = As + (ks * 4 + t) * GB_LDA + wm + g;
            const double* Bk = Bs + (ks * 4 + t) * GB_LDB + wn + g;
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) a[mi] = Ak[mi * 8];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Bk[ni * 8];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma884(acc.c[mi][ni], a[mi], b[ni]);
        }
        if (more) {
            double* An = smem + ((kt + 1) & 1) * GB_STAGE;
            la.store(An, ra);
            lb.store(An + GB_K * GB_LDA, rb);
        }
        __syncthreads();
    }
}

// Visit every accumulator element: f(m_local, n_local, value) with n in pairs (n, n+1).
template <class F>
__device__ __forceinline__ void acc_foreach_pair(const Acc& acc, F&& f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
            f(wm + mi * 8 + g, wn + ni * 8 + 2 * t, acc.c[mi][ni][0], acc.c[mi][ni][1]);
}

}  // namespace mg
