// mg_gamma2d.cu — the μ-quadrature ("separable", Modal2D) Γ engine on the device.
//
// Reference: engine2d.py:62-211.
//   P[a,b,x,m] = Σ_l lw_l q_a(l) q̃_b(x,l) P_l(μ_m),   lw_l = (2l+1)/(v_l sqrt C_l)
//     (build_ptable, :62-95: ascending l, Kahan-compensated)
//   Γ2d[n,n'] = Σ_x w_x r_x^2 Σ_m w_m perm3(P[rows(n), cols(n')](x,m)) / (48π)
//     (gamma2d_entry, :112-129: μ first, then the radial rule)
// The P table is built with the reference's exact operation order (term = ((lw q_a) q̃_b) P_l,
// Kahan update y = term - comp; t = acc + y; comp = (t - acc) - y), each FP64 op an explicit
// round-to-nearest intrinsic, so it reproduces the reference table bit for bit.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "mg_common.cuh"
#include "mg_dmma.cuh"

namespace mg {

// kernel times of the calling thread's last P-table / cell-sum launch (mg_gamma2d_timings)
thread_local double g2d_ms[2] = {0.0, 0.0};

struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair() {
        MG_CUDA(cudaEventCreate(&a));
        MG_CUDA(cudaEventCreate(&b));
        MG_CUDA(cudaEventRecord(a, 0));
    }
    double stop() {  // records the end event, waits for it, returns the elapsed ms
        float ms = 0.f;
        MG_CUDA(cudaEventRecord(b, 0));
        MG_CUDA(cudaEventSynchronize(b));
        MG_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
    ~EventPair() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

// ---- P table -----------------------------------------------------------------------------
// P[((a*p + b)*Nx + x)*nmu + m] as a register-tiled product over l: rows r = (a, b, x), columns
// m, a CTA owns a 64 x 64 tile and walks l in ascending chunks of PT_BK staged through shared
// memory (A[r][l] = (lw_l q_a(l)) q̃_b(x,l) formed once per element with the reference's two
// roundings, B[l][m] = P_l(μ_m)); a thread keeps a 4 x 4 block of (sum, compensation) pairs,
// so one staged A/B value feeds four Kahan updates.  Each output still sees exactly the
// reference's sequence of rounded operations in ascending l: the table is bit-identical.
constexpr int PT_BM = 64, PT_BN = 64, PT_BK = 32;

__global__ void __launch_bounds__(256, 2)
k_ptable_tiled(const double* __restrict__ q, const double* __restrict__ qt,
               const double* __restrict__ lw, const double* __restrict__ leg, int p, int Nx,
               int L, int nmu, double* __restrict__ P) {
    __shared__ double As[PT_BK][PT_BM + 1];  // odd stride: the transposing store is conflict-free
    __shared__ double Bs[PT_BK][PT_BN];
    const int64_t R = (int64_t)p * p * Nx;
    const int64_t r0 = (int64_t)blockIdx.y * PT_BM;
    const int m0 = blockIdx.x * PT_BN;
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    double acc[4][4], comp[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = comp[i][j] = 0.0;

    // this thread's staging slots: A rows (t/32 + 8 i) at l-offset t%32; B row t/64 + 4 i at
    // column t%64.  Row offsets into q̃ and q are decoded once per CTA (−1: row past the end).
    __shared__ int64_t row_qt[PT_BM];
    __shared__ int row_q[PT_BM];
    if (t < PT_BM) {
        const int64_t r = r0 + t;
        if (r < R) {
            const int x = (int)(r % Nx);
            const int ab = (int)(r / Nx);
            row_qt[t] = ((int64_t)(ab % p) * Nx + x) * L;
            row_q[t] = (ab / p) * L;
        } else {
            row_qt[t] = -1;
            row_q[t] = 0;
        }
    }
    const int al = t & 31, ar = t >> 5;
    const int bc = t & 63, bl = t >> 6;
    const bool bok = m0 + bc < nmu;

    for (int l0 = 0; l0 < L; l0 += PT_BK) {
        const int kn = min(PT_BK, L - l0);
        __syncthreads();
        {
            const int l = l0 + al;
            const double w = l < L ? lw[l] : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t oq = row_qt[ar + 8 * i];
                double v = 0.0;
                if (l < L && oq >= 0)
                    v = __dmul_rn(__dmul_rn(w, q[row_q[ar + 8 * i] + l]), qt[oq + l]);
                As[al][ar + 8 * i] = v;
            }
#pragma unroll
            for (int i = 0; i < PT_BK / 4; ++i) {
                const int l2 = l0 + bl + 4 * i;
                Bs[bl + 4 * i][bc] = (bok && l2 < L) ? leg[(int64_t)l2 * nmu + m0 + bc] : 0.0;
            }
        }
        __syncthreads();
        for (int kk = 0; kk < kn; ++kk) {  // never past L: a padded step would still apply comp
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double term = __dmul_rn(a[i], b[j]);
                    const double y = __dsub_rn(term, comp[i][j]);
                    const double s = __dadd_rn(acc[i][j], y);
                    comp[i][j] = __dsub_rn(__dsub_rn(s, acc[i][j]), y);
                    acc[i][j] = s;
                }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = r0 + ty * 4 + i;
        if (r >= R) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = m0 + tx + 16 * j;
            if (m < nmu) P[r * nmu + m] = acc[i][j];
        }
    }
}

// ---- Γ cells --------------------------------------------------------------------------------
// A CTA owns a 16 x 16 tile of (n, n') cells and one contiguous chunk of the radial points
// (grid.z): for each x it stages P[:, :, x, μ-chunk] as [a*p+b][MC + 1] (odd row stride: lanes
// that differ in (a, b) hit different banks, lanes that agree are a broadcast), so the nine
// operands of a cell's 3 x 3 matrix sit at nine fixed per-thread row bases and the μ index is
// an immediate offset in the unrolled loop.  The permanent is expanded along its first row
// (3 mul + 5 fma instead of the reference's 12 mul + 5 add; Γ2d agrees to rounding, which is
// all the reference claims for this engine), summed against the μ rule, and w_x r_x² times
// that is added to the chunk's partial.  Shared-memory bandwidth bounds the kernel: ten 8-byte
// reads per (cell, x, μ) against nine FP64 instructions.  k_gamma2d_reduce adds the chunk
// partials in ascending x order (deterministic for a given split) and applies 1/(48π).
constexpr int G2_TILE = 16;  // 16 x 16 cells per CTA

template <int MC>
__global__ void __launch_bounds__(G2_TILE* G2_TILE)
k_gamma2d_cells(const double* __restrict__ P, const int* __restrict__ modes, int n, int p,
                int Nx, int nmu, int xsplit, const double* __restrict__ mu_w,
                const double* __restrict__ wr2, double* __restrict__ partial) {
    constexpr int MCP = MC + 1;
    extern __shared__ double sp[];  // [p*p][MCP], then the μ weights of the chunk [MC]
    const int pp = p * p;
    double* sw = sp + (size_t)pp * MCP;
    const int tn = threadIdx.x / G2_TILE, tq = threadIdx.x % G2_TILE;
    const int nrow = blockIdx.y * G2_TILE + tn, ncol = blockIdx.x * G2_TILE + tq;
    const bool ok = nrow < n && ncol < n;
    const double* s[9];
    {
        int r[3] = {0, 0, 0}, c[3] = {0, 0, 0};
        if (ok) {
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                r[i] = modes[3 * nrow + i];
                c[i] = modes[3 * ncol + i];
            }
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) s[3 * i + j] = sp + (r[i] * p + c[j]) * MCP;
    }
    const int xa = (int)((int64_t)Nx * blockIdx.z / xsplit);
    const int xb = (int)((int64_t)Nx * (blockIdx.z + 1) / xsplit);
    double acc = 0.0;
    for (int x = xa; x < xb; ++x) {
        double inner = 0.0;
        for (int m0 = 0; m0 < nmu; m0 += MC) {
            const int mn = min(MC, nmu - m0);
            __syncthreads();
            // a short last chunk is zero-filled (its permanents vanish): the loop below runs
            // in unrolled groups of 8
            for (int e = threadIdx.x; e < pp * MC; e += blockDim.x) {
                const int ab = e / MC, mm = e % MC;
                sp[ab * MCP + mm] = mm < mn ? P[((int64_t)ab * Nx + x) * nmu + m0 + mm] : 0.0;
            }
            for (int e = threadIdx.x; e < MC; e += blockDim.x)
                sw[e] = e < mn ? mu_w[m0 + e] : 0.0;
            __syncthreads();
            constexpr int U = MC < 8 ? MC : 8;  // zero-filled up to the next multiple of U
            for (int mb = 0; mb < mn; mb += U) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int mm = mb + u;
                    const double m00 = s[0][mm], m01 = s[1][mm], m02 = s[2][mm];
                    const double m10 = s[3][mm], m11 = s[4][mm], m12 = s[5][mm];
                    const double m20 = s[6][mm], m21 = s[7][mm], m22 = s[8][mm];
                    const double per = m00 * (m11 * m22 + m12 * m21) +
                                       m01 * (m10 * m22 + m12 * m20) +
                                       m02 * (m10 * m21 + m11 * m20);
                    inner += per * sw[mm];
                }
            }
        }
        acc += wr2[x] * inner;
    }
    if (ok) partial[((int64_t)blockIdx.z * n + nrow) * n + ncol] = acc;
}

__global__ void k_gamma2d_reduce(const double* __restrict__ partial, int64_t cells, int xsplit,
                                 double* __restrict__ gamma) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cells) return;
    double acc = 0.0;
    for (int z = 0; z < xsplit; ++z) acc += partial[z * cells + i];
    gamma[i] = acc / (48.0 * 3.141592653589793);
}

// ---- Γ cells on the FP64 tensor pipe (p ≤ 24) ------------------------------------------------
// The permanent splits along its last row:  perm = Σ_k P[r2,c_k] · V[(r0,r1)][(c_i,c_j)]  with
// V[(a,b)][(c,d)] = P[a,c]P[b,d] + P[a,d]P[b,c]  ((i,j) the two columns other than k), so with
// the sample index s = (x, μ) and W_s = w_x r_x² w_μ
//     D[(a,c)][(a'≤b'),(c'≤d')] = Σ_s P_s[a,c] · W_s V_s[(a',b')][(c',d')]
// is one GEMM — M = p² rows, N = (p(p+1)/2)² columns, K = Nx·n_μ — and every cell is three
// entries of D.  It costs about as many FLOPs as the per-cell form (p⁶/2 against 10·p⁶/36 FP64
// instructions per sample) but runs them as DMMA.8x8x4 with ~0.9 shared-memory reads per DMMA
// instead of ten per cell-sample, which is what bounded k_gamma2d_cells.  A CTA owns 24-32
// n-fragments, one M tile of up to 64 rows (p > 8: several M tiles, grid.z) and a contiguous
// range of samples (split-K, partials reduced in order by k_gamma2d_gather); chunks of all p²
// rows of P_s are double-buffered through shared memory with 8-byte cp.async (128 samples per
// chunk at p <= 8, 64 / 32 / 16 as p² grows); the B operand is never stored: a lane forms its
// element from four P reads.
// Tile: WARPS warps of FN n-fragments each, KC samples per stage, row stride KC + 4 (fragment
// reads of (row g, sample t) are then bank-conflict free).  Measured (profiles/r02_2d_engine.txt):
// 12 warps x 2 fragments x 128 samples is fastest at p = 7, 8 (7-8 m-fragments feed 14-16 DMMAs
// per operand pair), 16 warps x 2 x 128 below that, where a warp has less tensor work per
// operand and more warps hide its loads.
__host__ __device__ inline int g2d_pair(int a, int b) { return b * (b + 1) / 2 + a; }  // a <= b

__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes));
}

template <int MF, int G2D_WARPS, int G2D_FN, int G2D_KC>
__global__ void __launch_bounds__(G2D_WARPS * 32, 1)
k_gamma2d_dmma(const double* __restrict__ P, const double* __restrict__ wr2,
               const double* __restrict__ mu_w, int p, int nmu, int64_t S, int nchunks,
               int N, int Npad, int srows, double* __restrict__ Dpart) {
    // srows = p² rounded up to whole M tiles of MF*8 rows: every CTA stages all p² rows of P
    // (the B operand pairs any two of them); its A rows are M tile blockIdx.z of those
    extern __shared__ double sm[];
    constexpr int G2D_LD = G2D_KC + 4;
    double* Ps = sm;                               // [2][srows][G2D_LD]
    double* Ws = sm + 2 * srows * G2D_LD;          // [2][G2D_KC]
    const int arow0 = blockIdx.z * MF * 8;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int pp = p * p, P2 = p * (p + 1) / 2;
    // this lane's B columns: n = (a'<=b', c'<=d') -> four row offsets into the staged P block
    const int nf0 = (blockIdx.x * G2D_WARPS + warp) * G2D_FN;
    int o[G2D_FN][4];
    double vm[G2D_FN];
#pragma unroll
    for (int f = 0; f < G2D_FN; ++f) {
        const int n = (nf0 + f) * 8 + g;
        vm[f] = n < N ? 1.0 : 0.0;
        int ab = n < N ? n / P2 : 0, cd = n < N ? n % P2 : 0;
        int b = 0, d = 0;
        while (g2d_pair(0, b + 1) <= ab) ++b;
        while (g2d_pair(0, d + 1) <= cd) ++d;
        const int a = ab - g2d_pair(0, b), c = cd - g2d_pair(0, d);
        o[f][0] = (a * p + c) * G2D_LD;
        o[f][1] = (b * p + d) * G2D_LD;
        o[f][2] = (a * p + d) * G2D_LD;
        o[f][3] = (b * p + c) * G2D_LD;
    }
    const bool warp_live = nf0 * 8 < N;
    // sample chunks of this CTA
    const int c0 = (int)((int64_t)nchunks * blockIdx.y / gridDim.y);
    const int c1 = (int)((int64_t)nchunks * (blockIdx.y + 1) / gridDim.y);
    // padding rows (pp <= row < srows) stay zero in both buffers
    for (int e = tid; e < 2 * srows * G2D_LD; e += blockDim.x)
        if ((e / G2D_LD) % srows >= pp) Ps[e] = 0.0;

    // staging: a thread copies one sample column k of rows kr, kr + RSTEP, ... (8-byte cp.async,
    // zero-filled past the last sample), so a chunk costs it one copy and two adds per element
    constexpr int RSTEP = G2D_WARPS * 32 / G2D_KC;
    static_assert(G2D_WARPS * 32 % G2D_KC == 0, "threads must tile the sample columns");
    const int kcol = tid % G2D_KC, kr = tid / G2D_KC;
    auto stage = [&](int ch, int buf) {
        const int64_t sidx = (int64_t)ch * G2D_KC + kcol;
        const bool ok = sidx < S;
        const double* src = ok ? P + (int64_t)kr * S + sidx : P;
        double* dst = Ps + buf * srows * G2D_LD + kr * G2D_LD + kcol;
        const int64_t sstep = ok ? (int64_t)RSTEP * S : 0;
        const int bytes = ok ? 8 : 0;
        for (int row = kr; row < pp; row += RSTEP) {
            cp_async8(dst, src, bytes);
            src += sstep;
            dst += RSTEP * G2D_LD;
        }
        if (kr == 0) Ws[buf * G2D_KC + kcol] = ok ? wr2[sidx / nmu] * mu_w[sidx % nmu] : 0.0;
        cp_async_commit();
    };

    double acc[MF][G2D_FN][2];
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int f = 0; f < G2D_FN; ++f) acc[m][f][0] = acc[m][f][1] = 0.0;

    if (c0 < c1) stage(c0, 0);
    for (int ch = c0; ch < c1; ++ch) {
        const int buf = (ch - c0) & 1;
        if (ch + 1 < c1) {
            stage(ch + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (warp_live) {
            const double* ps = Ps + buf * srows * G2D_LD;
            const double* pa = ps + (arow0 + g) * G2D_LD;
            const double* ws = Ws + buf * G2D_KC;
#pragma unroll 4
            for (int k = t; k < G2D_KC; k += 4) {
                const double w = ws[k];
                double b[G2D_FN];
#pragma unroll
                for (int f = 0; f < G2D_FN; ++f)
                    b[f] = (w * vm[f]) * (ps[o[f][0] + k] * ps[o[f][1] + k] +
                                          ps[o[f][2] + k] * ps[o[f][3] + k]);
#pragma unroll
                for (int m = 0; m < MF; ++m) {
                    const double a = pa[m * 8 * G2D_LD + k];
#pragma unroll
                    for (int f = 0; f < G2D_FN; ++f) dmma884(acc[m][f], a, b[f]);
                }
            }
        }
        __syncthreads();  // the next iteration's stage() overwrites the other buffer
    }
    if (!warp_live) return;
    double* out = Dpart + ((int64_t)blockIdx.y * srows + arow0) * Npad;
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int f = 0; f < G2D_FN; ++f) {
            const int col = (nf0 + f) * 8 + 2 * t;
            if (col < Npad) {
                out[(int64_t)(m * 8 + g) * Npad + col] = acc[m][f][0];
                out[(int64_t)(m * 8 + g) * Npad + col + 1] = acc[m][f][1];
            }
        }
}

// Γ2d[n,n'] = Σ_k D[(r2,c_k)][(r0,r1),(c_i,c_j)] / 48π, D summed over the split-K partials in
// ascending order (deterministic).
__global__ void k_gamma2d_gather(const double* __restrict__ Dpart, int ksplit, int rows, int Npad,
                                 const int* __restrict__ modes, int n, int p,
                                 double* __restrict__ gamma) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * n) return;
    const int nr = (int)(i / n), nc = (int)(i % n);
    const int r0 = modes[3 * nr], r1 = modes[3 * nr + 1], r2 = modes[3 * nr + 2];
    const int c[3] = {modes[3 * nc], modes[3 * nc + 1], modes[3 * nc + 2]};
    const int P2 = p * (p + 1) / 2;
    const int ab = g2d_pair(r0, r1);
    // columns other than k, in ascending order (the mapping keeps i <= j <= k)
    const int64_t e0 = (int64_t)(r2 * p + c[0]) * Npad + ab * P2 + g2d_pair(c[1], c[2]);
    const int64_t e1 = (int64_t)(r2 * p + c[1]) * Npad + ab * P2 + g2d_pair(c[0], c[2]);
    const int64_t e2 = (int64_t)(r2 * p + c[2]) * Npad + ab * P2 + g2d_pair(c[0], c[1]);
    double acc = 0.0;
    for (int z = 0; z < ksplit; ++z) {
        const double* D = Dpart + (int64_t)z * rows * Npad;
        acc += (D[e0] + D[e1]) + D[e2];
    }
    gamma[i] = acc / (48.0 * 3.141592653589793);
}

void ptable_dev(const double* q, const double* qt, const double* lw, const double* leg, int p,
                int Nx, int L, int nmu, double* P_dev) {
    MG_NVTX("mg:ptable");
    DBuf<double> dq, dqt, dlw, dleg;
    dq.upload(q, (size_t)p * L);
    dqt.upload(qt, (size_t)p * Nx * L);
    dlw.upload(lw, L);
    dleg.upload(leg, (size_t)L * nmu);
    const int64_t R = (int64_t)p * p * Nx;
    MG_REQUIRE(ceil_div(R, PT_BM) <= 65535, "P table has too many (a, b, x) rows");
    dim3 grid(ceil_div(nmu, PT_BN), ceil_div(R, PT_BM));
    EventPair ev;
    k_ptable_tiled<<<grid, 256>>>(dq.p, dqt.p, dlw.p, dleg.p, p, Nx, L, nmu, P_dev);
    MG_LAUNCHED();
    g2d_ms[0] = ev.stop();
    MG_CUDA(cudaDeviceSynchronize());
}

// x chunks per cell tile: about 16 CTAs per SM in total (4 resident at a time, so the last
// wave's idle tail stays small), at most one chunk per radial point and 1 GiB of partials.
int gamma2d_xsplit(int n, int Nx) {
    const int64_t tiles = (int64_t)ceil_div(n, G2_TILE) * ceil_div(n, G2_TILE);
    int64_t xs = (148 * 16 + tiles - 1) / tiles;
    xs = std::min<int64_t>(xs, Nx);
    xs = std::min<int64_t>(xs, std::max<int64_t>(1, (int64_t(1) << 27) / ((int64_t)n * n)));
    return (int)std::max<int64_t>(1, xs);
}

// Shared memory of one CTA: two staged blocks of srows x (KC + 4) doubles plus the weights.
static size_t g2d_smem(int srows, int kc) {
    return ((size_t)2 * srows * (kc + 4) + 2 * kc) * sizeof(double);
}
constexpr size_t G2D_SMEM_CAP = 200 * 1024;
constexpr size_t G2D_PART_CAP = size_t(1) << 30;  // split-K partials of D

template <int MF, int WARPS, int FN, int KC>
static void launch_gamma2d_dmma(const double* P_dev, const int* modes_dev, int n, int p, int Nx,
                                int nmu, const double* mu_w_dev, const double* wr2_dev,
                                double* gamma_dev) {
    const int P2 = p * (p + 1) / 2, N = P2 * P2, Npad = (int)round_up(N, 8);
    const int mtiles = ceil_div(p * p, MF * 8), srows = mtiles * MF * 8;
    const int64_t S = (int64_t)Nx * nmu;
    const int nchunks = ceil_div(S, KC);
    const int gx = ceil_div(Npad / 8, FN * WARPS);
    // split-K: one CTA per SM in total when the (N tile, M tile) grid divides the machine well
    // (at least 85 % of the SMs busy); otherwise about six waves of CTAs (one resident per SM), so the last, partly
    // filled wave costs little; at least 4 chunks per CTA, partials within their cap
    const int tiles = gx * mtiles;
    int ksplit = tiles <= 148 ? 148 / tiles : 0;
    if (ksplit * tiles * 100 < 85 * 148) ksplit = ceil_div(6 * 148, tiles);  // < 85 % of one wave
    ksplit = std::max(1, std::min(ksplit, std::max(nchunks / 4, 1)));
    ksplit = (int)std::max<size_t>(
        1, std::min<size_t>(ksplit, G2D_PART_CAP / ((size_t)srows * Npad * sizeof(double))));
    DBuf<double> dpart((size_t)ksplit * srows * Npad);
    const size_t shm = g2d_smem(srows, KC);
    MG_CUDA(cudaFuncSetAttribute(k_gamma2d_dmma<MF, WARPS, FN, KC>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    k_gamma2d_dmma<MF, WARPS, FN, KC><<<dim3(gx, ksplit, mtiles), WARPS * 32, shm>>>(
        P_dev, wr2_dev, mu_w_dev, p, nmu, S, nchunks, N, Npad, srows, dpart.p);
    MG_LAUNCHED();
    const int64_t cells = (int64_t)n * n;
    k_gamma2d_gather<<<ceil_div(cells, 256), 256>>>(dpart.p, ksplit, srows, Npad, modes_dev, n, p,
                                                      gamma_dev);
    MG_LAUNCHED();
}

// The DMMA form serves a basis if its staged P block fits shared memory with at least 16
// samples per chunk and one set of D partials fits the cap (p <= 24 with these caps); larger
// bases use the per-cell kernel.
static bool gamma2d_dmma_fits(int p) {
    if (p <= 8) return true;
    const int srows = (int)round_up(p * p, 64), P2 = p * (p + 1) / 2;
    return g2d_smem(srows, 16) <= G2D_SMEM_CAP &&
           (size_t)srows * round_up((int64_t)P2 * P2, 8) * sizeof(double) <= G2D_PART_CAP;
}

static void gamma2d_dmma(const double* P_dev, const int* modes_dev, int n, int p, int Nx, int nmu,
                         const double* mu_w_dev, const double* wr2_dev, double* gamma_dev) {
#define MG_G2D_GO(MF, W, KC)                                                                   \
    launch_gamma2d_dmma<MF, W, 2, KC>(P_dev, modes_dev, n, p, Nx, nmu, mu_w_dev, wr2_dev,      \
                                      gamma_dev)
    if (p > 8) {  // several M tiles of 64 rows; the chunk length is what shared memory allows
        const int srows = (int)round_up(p * p, 64);
        if (g2d_smem(srows, 64) <= G2D_SMEM_CAP) MG_G2D_GO(8, 12, 64);
        else if (g2d_smem(srows, 32) <= G2D_SMEM_CAP) MG_G2D_GO(8, 12, 32);
        else MG_G2D_GO(8, 12, 16);
        return;
    }
    switch (ceil_div(p * p, 8)) {  // m-fragments: p = 1..8 -> 1, 1, 2, 2, 4, 5, 7, 8
        case 1: MG_G2D_GO(1, 16, 128); break;
        case 2: MG_G2D_GO(2, 16, 128); break;
        case 4: MG_G2D_GO(4, 16, 128); break;
        case 5: MG_G2D_GO(5, 16, 128); break;
        case 7: MG_G2D_GO(7, 12, 128); break;
        default: MG_G2D_GO(8, 12, 128); break;
    }
#undef MG_G2D_GO
}

void gamma2d_dev(const double* P_dev, const int* modes_host, int n, int p, int Nx, int nmu,
                 const double* mu_w, const double* wr2, double* gamma_host) {
    MG_NVTX("mg:gamma2d_cells");
    DBuf<int> dm;
    DBuf<double> dw, dr, dg, dpart;
    dm.upload(modes_host, 3 * (size_t)n);
    dw.upload(mu_w, nmu);
    dr.upload(wr2, Nx);
    dg.alloc((size_t)n * n);
    EventPair ev;
    const bool force_lds = std::getenv("MG_G2D_LDS") != nullptr;  // A/B switch (read per call)
    if (!force_lds && gamma2d_dmma_fits(p)) {
        gamma2d_dmma(P_dev, dm.p, n, p, Nx, nmu, dw.p, dr.p, dg.p);
    } else {
        const int xsplit = gamma2d_xsplit(n, Nx);
        dpart.alloc((size_t)xsplit * n * n);
        MG_REQUIRE(ceil_div(n, G2_TILE) <= 65535, "too many modes for the cell grid");
        dim3 grid(ceil_div(n, G2_TILE), ceil_div(n, G2_TILE), xsplit);
        // μ chunk: the largest of 64 / 16 / 4 / 1 whose staged [p²][MC + 1] block fits 200 KB
        auto launch = [&](auto mc_tag) {
            constexpr int MC = decltype(mc_tag)::value;
            const size_t shm = ((size_t)p * p * (MC + 1) + MC) * sizeof(double);
            if (shm > 48 * 1024)
                MG_CUDA(cudaFuncSetAttribute(k_gamma2d_cells<MC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
            k_gamma2d_cells<MC><<<grid, G2_TILE * G2_TILE, shm>>>(P_dev, dm.p, n, p, Nx, nmu, xsplit,
                                                                    dw.p, dr.p, dpart.p);
        };
        const size_t cap = 200 * 1024 / sizeof(double), pp = (size_t)p * p;
        if (pp * 65 + 64 <= cap) launch(std::integral_constant<int, 64>{});
        else if (pp * 17 + 16 <= cap) launch(std::integral_constant<int, 16>{});
        else if (pp * 5 + 4 <= cap) launch(std::integral_constant<int, 4>{});
        else {
            MG_REQUIRE(pp * 2 + 1 <= cap, "p_max too large for the 2D cell kernel");
            launch(std::integral_constant<int, 1>{});
        }
        MG_LAUNCHED();
        const int64_t cells = (int64_t)n * n;
        k_gamma2d_reduce<<<ceil_div(cells, 256), 256>>>(dpart.p, cells, xsplit, dg.p);
        MG_LAUNCHED();
    }
    g2d_ms[1] = ev.stop();
    MG_CUDA(cudaMemcpy(gamma_host, dg.p, (size_t)n * n * sizeof(double),
                       cudaMemcpyDeviceToHost));
}

void gamma2d_timings(double* ptable_ms, double* cells_ms) {
    if (ptable_ms) *ptable_ms = g2d_ms[0];
    if (cells_ms) *cells_ms = g2d_ms[1];
}

void gamma2d_reset_timings() { g2d_ms[0] = g2d_ms[1] = 0.0; }

}  // namespace mg
