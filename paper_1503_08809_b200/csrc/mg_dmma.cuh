// mg_dmma.cuh — FP64 tensor-core (DMMA) block GEMM pipelines for the Γ contractions.
//
// Blackwell has no FP64 tcgen05 kind; FP64 tensor math is the legacy `mma.sync ... .f64`
// path, which ptxas lowers to DMMA.8x8x4 on sm_100a (every f64 mma shape becomes a sequence
// of 8x8x4 DMMAs; the NOP between consecutive DMMAs is ISA padding — the microbenchmark in
// tools/fp64_peak.cu has the same pattern and reaches 37.0 of 37.2 nominal TFLOP/s).
//
// Tile geometry is a template (Cfg): WARPS_M x WARPS_N warps, each owning FM x FN m8n8k4
// fragments, so BM = 8*FM*WARPS_M, BN = 8*FN*WARPS_N.  Operand tiles live in shared memory
// either k-major (X[k][m], row stride W+4) or m-major (X[m][k], row stride BK+4); both pads
// keep the fragment reads (lane (g,t) reads element (m0+g, k0+t)) bank-conflict free and
// rows 16-byte aligned.  Fragments are double-buffered in registers across the k4 steps and
// all-zero k4 steps of the last k-tile are skipped.  Two pipelines:
//   Pipe               all threads stream tiles with 16-byte cp.async (zero-fill at edges)
//                      through a STAGES-deep ring, one CTA barrier per k-tile (pair
//                      contraction, p = 22 x contraction);
//   PipeTMA(Persistent) one producer warp moves whole tiles with cp.async.bulk (TMA engine)
//                      completing on per-stage mbarriers; 15 consumer warps wait on "full",
//                      release through "empty"; no CTA barrier in the loop; the persistent
//                      form walks work items so the next item streams in during an epilogue
//                      (run and x contractions).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mg {

template <int WM_, int WN_, int FM_, int FN_>
struct TileCfg {
    static constexpr int WARPS_M = WM_, WARPS_N = WN_, FM = FM_, FN = FN_;
    static constexpr int BM = 8 * FM_ * WM_, BN = 8 * FN_ * WN_;
    static constexpr int THREADS = 32 * WM_ * WN_;
};

__host__ __device__ constexpr int ld_kmajor(int w) { return w + 4; }   // X[k][m]
__host__ __device__ constexpr int ld_mmajor(int bk) { return bk + 4; }  // X[m][k]
__host__ __device__ constexpr int tile_doubles(bool kmajor, int w, int bk) {
    return kmajor ? bk * ld_kmajor(w) : w * ld_mmajor(bk);
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy global->shared; src_bytes < 16 zero-fills the remainder.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// k-major tile: rows k in [0,BK), each W doubles from src_row(k) (nullptr -> zeros);
// columns [w_valid, W) zero-filled.
template <int BK, int W, int THREADS, class RowPtr>
__device__ __forceinline__ void copy_kmajor(double* dst, RowPtr&& src_row, int w_valid) {
    constexpr int CPR = W / 2, CH = BK * CPR;
    static_assert(CH % THREADS == 0, "tile chunks must divide the thread count");
#pragma unroll
    for (int i = 0; i < CH / THREADS; ++i) {
        int c = threadIdx.x + i * THREADS;
        int k = c / CPR, m = (c % CPR) * 2;
        const double* s = src_row(k);
        double* d = dst + k * ld_kmajor(W) + m;
        int bytes = (s && m < w_valid) ? ((w_valid - m) >= 2 ? 16 : 8) : 0;
        cp_async16(d, bytes ? s + m : d, bytes);
    }
}
// m-major tile: rows m in [0,W), each BK doubles from src_row(m) (nullptr -> zeros);
// k in [k_valid, BK) zero-filled.
template <int BK, int W, int THREADS, class RowPtr>
__device__ __forceinline__ void copy_mmajor(double* dst, RowPtr&& src_row, int k_valid) {
    constexpr int CPR = BK / 2, CH = W * CPR;
    static_assert(CH % THREADS == 0, "tile chunks must divide the thread count");
#pragma unroll
    for (int i = 0; i < CH / THREADS; ++i) {
        int c = threadIdx.x + i * THREADS;
        int m = c / CPR, k = (c % CPR) * 2;
        const double* s = src_row(m);
        double* d = dst + m * ld_mmajor(BK) + k;
        int bytes = (s && k < k_valid) ? ((k_valid - k) >= 2 ? 16 : 8) : 0;
        cp_async16(d, bytes ? s + k : d, bytes);
    }
}

template <class Cfg>
struct Acc {
    double c[Cfg::FM][Cfg::FN][2];
};

template <bool KMAJ, int W, int BK>
__device__ __forceinline__ double frag_ld(const double* X, int k, int m) {
    return KMAJ ? X[k * ld_kmajor(W) + m] : X[m * ld_mmajor(BK) + k];
}

// A-operand source of the pipeline.
enum class ASrc { KMajor, MMajor, Raw };

// Producer contract:
//   __device__ void issue(int kt, double* As, double* Bs, double* raw) const;   // cp.async
//   __device__ int kvalid_last() const;   // k values with data in the last k-tile (1..BK)
//   (ASrc::Raw only) __device__ double a_frag(const double* raw, int k, int fm) const;
//     — value of A at (m = this lane's row of fragment fm, k) built from staged raw data.
// Stage layout: [A tile (absent for Raw)][B tile][raw (kRaw doubles)].
template <class Cfg, int BK, int STAGES, ASrc AS, bool BKM, int kRaw>
struct Pipe {
    static constexpr int THREADS = Cfg::THREADS;
    static constexpr int SA = AS == ASrc::Raw ? 0 : tile_doubles(AS == ASrc::KMajor, Cfg::BM, BK);
    static constexpr int SB = tile_doubles(BKM, Cfg::BN, BK);
    static constexpr int SS = SA + SB + kRaw;
    static constexpr size_t smem_bytes = (size_t)STAGES * SS * sizeof(double);

    template <class Prod>
    __device__ static void run(int ktiles, const Prod& prod, double* smem, Acc<Cfg>& acc) {
        constexpr int FM = Cfg::FM, FN = Cfg::FN;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int g = lane >> 2, t = lane & 3;
        const int wm = (warp / Cfg::WARPS_N) * (8 * FM), wn = (warp % Cfg::WARPS_N) * (8 * FN);
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) acc.c[mi][ni][0] = acc.c[mi][ni][1] = 0.0;
        if (ktiles <= 0) return;

#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < ktiles) {
                double* st = smem + s * SS;
                prod.issue(s, st, st + SA, st + SA + SB);
            }
            cp_async_commit();
        }

        for (int kt = 0; kt < ktiles; ++kt) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            const double* st = smem + (kt % STAGES) * SS;
            const double* As = st;
            const double* Bs = st + SA;
            const double* raw = st + SA + SB;
            // refill of the stage consumed in iteration kt-1 (safe after the barrier above);
            // issued after the first k4 step's DMMAs so the address/issue work of cp.async
            // overlaps tensor work instead of delaying it
            auto refill = [&]() {
                int nk = kt + STAGES - 1;
                if (nk < ktiles) {
                    double* ns = smem + (nk % STAGES) * SS;
                    prod.issue(nk, ns, ns + SA, ns + SA + SB);
                }
                cp_async_commit();
            };
            double a[2][FM], b[2][FN];
            auto load_frags = [&](int buf, int k) {
#pragma unroll
                for (int mi = 0; mi < FM; ++mi) {
                    if constexpr (AS == ASrc::Raw)
                        a[buf][mi] = prod.a_frag(raw, k, mi);
                    else
                        a[buf][mi] = frag_ld<AS == ASrc::KMajor, Cfg::BM, BK>(As, k, wm + mi * 8 + g);
                }
#pragma unroll
                for (int ni = 0; ni < FN; ++ni)
                    b[buf][ni] = frag_ld<BKM, Cfg::BN, BK>(Bs, k, wn + ni * 8 + g);
            };
            // k4 steps that hold data (the tail of the last tile is all zeros: skip it)
            const int nks = kt + 1 < ktiles ? BK / 4 : (prod.kvalid_last() + 3) / 4;
            load_frags(0, t);
#pragma unroll
            for (int ks = 0; ks < BK / 4; ++ks) {
                if (ks < nks) {
                    const int cur = ks & 1;
                    if (ks + 1 < BK / 4) load_frags(cur ^ 1, (ks + 1) * 4 + t);
#pragma unroll
                    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                        for (int ni = 0; ni < FN; ++ni)
                            dmma884(acc.c[mi][ni], a[cur][mi], b[cur][ni]);
                }
                if (ks == 0) refill();
            }
        }
        cp_async_wait<0>();
    }
};


// ------------------------------------------------------------------------------------------
// mbarrier helpers for the warp-specialised pipelines below
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(
        smem_u32(bar)) : "memory");
}
// Blocking wait for the phase with the given parity.  The "memory" clobber keeps the compiler
// from hoisting shared-memory reads of the stage above the wait.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, int parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        " WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity) : "memory");
}
// Non-blocking probe of the same phase (1 = complete).  Issued well before the data is
// needed, its result is consumed only at the stage boundary, so the probe's latency overlaps
// the DMMAs of the current stage instead of stalling every consumer warp at once.
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, int parity) {
    uint32_t r;
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n"
        "}\n" : "=r"(r) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return r;
}

// ------------------------------------------------------------------------------------------
// Bulk-copy (TMA engine) variant of the warp-specialised pipeline.  The producer warp moves
// whole contiguous rows with cp.async.bulk (one instruction per row, SASS UBLKCP) completing
// on the stage's "full" mbarrier by transaction bytes (expect_tx), so a stage costs ~64-240
// copy instructions instead of thousands of 16-byte cp.async chunks.  No zero fill: the
// producers arrange that rows/columns outside the matrix are either real zeros (padded
// panels) or only feed accumulator rows/columns the epilogue discards.
// Producer contract: __device__ void bulk_rows(int kt, double* As, double* Bs, int lane,
//                        uint64_t* bar) const;   // issues the copies, all 32 lanes
//                    __device__ uint32_t stage_bytes(int kt) const;  // total bytes of stage kt
//                    __device__ int kvalid_last() const;
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(bytes));
}
// Raise the transaction count of the current phase without arriving (the arrivals come
// later, from the lanes that also write part of the stage with ordinary shared stores).
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <class Cfg, int BK, int STAGES, bool AK, bool BKM>
struct PipeTMA {
    static constexpr int WARPS = Cfg::WARPS_M * Cfg::WARPS_N;
    static constexpr int THREADS = Cfg::THREADS + 32;
    static constexpr int SA = tile_doubles(AK, Cfg::BM, BK);
    static constexpr int SB = tile_doubles(BKM, Cfg::BN, BK);
    static constexpr int SS = SA + SB;
    static constexpr size_t smem_bytes = (size_t)STAGES * SS * sizeof(double) + 2 * STAGES * 8;

    template <class Prod>
    __device__ static bool run(int ktiles, const Prod& prod, double* smem, Acc<Cfg>& acc) {
        constexpr int FM = Cfg::FM, FN = Cfg::FN;
        uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SS);
        uint64_t* empty = full + STAGES;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, WARPS);
            }
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        }
        __syncthreads();
        if (warp == WARPS) {  // ---------------- producer warp
            for (int kt = 0; kt < ktiles; ++kt) {
                const int s = kt % STAGES;
                if (kt >= STAGES) mbar_wait(empty + s, ((kt / STAGES) - 1) & 1);
                if (lane == 0) mbar_arrive_expect_tx(full + s, prod.stage_bytes(kt));
                __syncwarp();
                double* st = smem + s * SS;
                prod.bulk_rows(kt, st, st + SA, lane, full + s);
            }
            return false;
        }
        // ------------------------------------------------------------- consumer warps
        const int g = lane >> 2, t = lane & 3;
        const int wm = (warp / Cfg::WARPS_N) * (8 * FM), wn = (warp % Cfg::WARPS_N) * (8 * FN);
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) acc.c[mi][ni][0] = acc.c[mi][ni][1] = 0.0;
        for (int kt = 0; kt < ktiles; ++kt) {
            const int s = kt % STAGES;
            mbar_wait(full + s, (kt / STAGES) & 1);
            const double* As = smem + s * SS;
            const double* Bs = As + SA;
            double a[2][FM], b[2][FN];
            auto load_frags = [&](int buf, int k) {
#pragma unroll
                for (int mi = 0; mi < FM; ++mi) a[buf][mi] = frag_ld<AK, Cfg::BM, BK>(As, k, wm + mi * 8 + g);
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) b[buf][ni] = frag_ld<BKM, Cfg::BN, BK>(Bs, k, wn + ni * 8 + g);
            };
            const int nks = kt + 1 < ktiles ? BK / 4 : (prod.kvalid_last() + 3) / 4;
            load_frags(0, t);
#pragma unroll
            for (int ks = 0; ks < BK / 4; ++ks) {
                if (ks < nks) {
                    const int cur = ks & 1;
                    if (ks + 1 < BK / 4) load_frags(cur ^ 1, (ks + 1) * 4 + t);
#pragma unroll
                    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                        for (int ni = 0; ni < FN; ++ni)
                            dmma884(acc.c[mi][ni], a[cur][mi], b[cur][ni]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        return true;
    }
};


// Persistent form of PipeTMA: the CTA walks work items it = first, first + stride, ... and
// the producer keeps streaming the next item's stages while the consumers finish the current
// item and run its epilogue, so per-item pipeline fill is hidden.
// Item producer contract: int ktiles(int it); uint32_t stage_bytes(int it, int kt);
//   void bulk_rows(int it, int kt, double* As, double* Bs, int lane, uint64_t* bar);
//   int kvalid_last(int it);  int2 valid_mn(int it) (valid rows/columns of the item's tile);
//   and the consumer epilogue epi(it, acc).
template <class Cfg, int BK, int STAGES, bool AK, bool BKM, bool IDLE_SKIP = false>
struct PipeTMAPersistent {
    using Base = PipeTMA<Cfg, BK, STAGES, AK, BKM>;
    static constexpr int WARPS = Base::WARPS, THREADS = Base::THREADS;
    static constexpr int SA = Base::SA, SB = Base::SB, SS = Base::SS;
    static constexpr size_t smem_bytes = Base::smem_bytes;

    template <class Prod, class Epi>
    __device__ static void run(int first, int stride, int nitems, const Prod& prod, Epi&& epi,
                               double* smem) {
        constexpr int FM = Cfg::FM, FN = Cfg::FN;
        uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SS);
        uint64_t* empty = full + STAGES;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(full + s, Prod::kComputeA ? 32 : 1);
                mbar_init(empty + s, WARPS);
            }
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        }
        __syncthreads();
        if (warp == WARPS) {  // ---------------- producer warp
            int g = 0;
            for (int it = first; it < nitems; it += stride) {
                const int kts = prod.ktiles(it);
                for (int kt = 0; kt < kts; ++kt, ++g) {
                    const int s = g % STAGES;
                    if (g >= STAGES) mbar_wait(empty + s, ((g / STAGES) - 1) & 1);
                    double* st = smem + s * SS;
                    if constexpr (Prod::kComputeA) {
                        // B by bulk copy; A computed by the 32 lanes with shared stores, each
                        // lane's arrive releasing its own stores to the consumers
                        if (lane == 0) {
                            mbar_expect_tx(full + s, prod.stage_bytes(it, kt));
                            prod.bulk_b(it, kt, st + SA, full + s);
                        }
                        prod.compute_a(it, kt, st, lane);
                        mbar_arrive(full + s);
                    } else {
                        if (lane == 0) mbar_arrive_expect_tx(full + s, prod.stage_bytes(it, kt));
                        __syncwarp();
                        prod.bulk_rows(it, kt, st, st + SA, lane, full + s);
                    }
                }
            }
            return;
        }
        // ------------------------------------------------------------- consumer warps
        // The fragments of a stage's first k4 step are loaded while the previous stage's last
        // k4 step is still in the DMMA pipe, and the stage's barrier is probed one stage
        // early, so crossing a stage boundary costs no exposed barrier or LDS latency.
        static_assert((BK / 4) % 2 == 0, "cross-stage fragment prefetch needs an even k4 count");
        const int g4 = lane >> 2, t = lane & 3;
        const int wm = (warp / Cfg::WARPS_N) * (8 * FM), wn = (warp % Cfg::WARPS_N) * (8 * FN);
        Acc<Cfg> acc;
        double a[2][FM], b[2][FN];
        auto load_frags = [&](int buf, const double* As, const double* Bs, int k) {
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
                a[buf][mi] = frag_ld<AK, Cfg::BM, BK>(As, k, wm + mi * 8 + g4);
#pragma unroll
            for (int ni = 0; ni < FN; ++ni)
                b[buf][ni] = frag_ld<BKM, Cfg::BN, BK>(Bs, k, wn + ni * 8 + g4);
        };
        int g = 0;
        // item metadata (k-tile count, valid k of the last tile) is read one item ahead, so
        // its global-load latency hides under the current item's DMMAs
        // IDLE_SKIP: a warp whose whole sub-tile lies in the item's padding (rows >= valid M or
        // columns >= valid N: partial tiles at group ends, the last column block) skips its
        // fragment loads and DMMAs for that item but still walks the barriers (one
        // warp-uniform flag; measured -0.5 % on the run contraction, +1.4 % on the p=30 x
        // contraction through register pressure, so it is enabled per pipeline).
        auto warp_idle = [&](int it) {
            if constexpr (IDLE_SKIP) {
                const int2 v = prod.valid_mn(it);
                return wm >= v.x || wn >= v.y;
            } else {
                return false;
            }
        };
        int kts_n = first < nitems ? prod.ktiles(first) : 0;
        int kvl_n = first < nitems ? prod.kvalid_last(first) : 0;
        bool idle_n = first < nitems ? warp_idle(first) : false;
        for (int it = first; it < nitems; it += stride) {
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) acc.c[mi][ni][0] = acc.c[mi][ni][1] = 0.0;
            const int kts = kts_n;
            const int kvl = kvl_n;
            const bool idle = idle_n;
            if (it + stride < nitems) {
                kts_n = prod.ktiles(it + stride);
                kvl_n = prod.kvalid_last(it + stride);
                idle_n = warp_idle(it + stride);
            }
            {
                const int s = g % STAGES;
                mbar_wait(full + s, (g / STAGES) & 1);
                load_frags(0, smem + s * SS, smem + s * SS + SA, t);
            }
            for (int kt = 0; kt < kts; ++kt, ++g) {
                const int s = g % STAGES, s2 = (g + 1) % STAGES;
                const int ph2 = ((g + 1) / STAGES) & 1;
                const double* As = smem + s * SS;
                const double* Bs = As + SA;
                const double* As2 = smem + s2 * SS;
                const double* Bs2 = As2 + SA;
                const bool more = kt + 1 < kts;
                const int nks = idle ? 0 : more ? BK / 4 : (kvl + 3) / 4;
                uint32_t ready = more ? mbar_test(full + s2, ph2) : 1u;
                if (idle && more && !ready) mbar_wait(full + s2, ph2);  // stay in phase
#pragma unroll
                for (int ks = 0; ks < BK / 4; ++ks) {
                    if (ks < nks) {
                        const int cur = ks & 1;
                        if (ks + 1 < BK / 4) {
                            load_frags(cur ^ 1, As, Bs, (ks + 1) * 4 + t);
                        } else if (more) {
                            if (!ready) mbar_wait(full + s2, ph2);
                            load_frags(cur ^ 1, As2, Bs2, t);
                        }
#pragma unroll
                        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                            for (int ni = 0; ni < FN; ++ni)
                                dmma884(acc.c[mi][ni], a[cur][mi], b[cur][ni]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
            }
            epi(it, acc);
        }
    }
};

// N-split form of the persistent pipeline, for tiles whose last N tile is mostly padding
// (p = 15 x contraction: N = 225 = 128 + 97).  The item's valid n-fragments nfr (of
// FN * WARPS_N) are dealt to the WARPS_N warp columns as evenly as possible, so a warp owns
// FN, FN - 1 or FN - 2 n-fragments (one warp-uniform dispatch per item into separately
// compiled loop bodies: no per-DMMA predicates) starting at a per-item column offset.  Warp columns are rotated by
// the warp row (wn = (warp + warp / WARPS_N) % WARPS_N), so the warps with the extra fragment
// fall on different SM sub-partitions (warp % 4) and the four DMMA units stay balanced:
// 13 n-fragments run as 4,3,3,3 -> 50 fragment-steps per sub-partition instead of 60.
// Extra producer contract: int nfrags(int it) (valid n-fragments of the item, each warp
// column must get FN - 2 .. FN and at least 1); the epilogue is epi(it, acc, wm, wn, nf).
template <class Cfg, int BK, int STAGES, bool AK, bool BKM>
struct PipeTMAPersistentNS {
    using Base = PipeTMA<Cfg, BK, STAGES, AK, BKM>;
    static constexpr int WARPS = Base::WARPS, THREADS = Base::THREADS;
    static constexpr int SA = Base::SA, SB = Base::SB, SS = Base::SS;
    static constexpr size_t smem_bytes = Base::smem_bytes;

    template <int NF, class Prod>
    __device__ __forceinline__ static void item_loop(const Prod& prod, double* smem,
                                                     uint64_t* full, uint64_t* empty, int kts,
                                                     int kvl, int wm, int wn, int& g,
                                                     Acc<Cfg>& acc) {
        constexpr int FM = Cfg::FM;
        const int lane = threadIdx.x & 31;
        const int g4 = lane >> 2, t = lane & 3;
        // B fragments are double-buffered in registers; each A fragment is reloaded for the next
        // k4 step right after its own row of DMMAs has been issued (a warp's k4 steps are
        // hundreds of pipe cycles apart with three warps per DMMA unit, so the reload latency
        // is covered) — 13 fragment doubles instead of 18, which keeps the 5 x 4 tile's 40
        // accumulators inside the 128 registers a 13-warp CTA can allocate.
        double a[FM], b[2][NF];
        auto load_b = [&](int buf, const double* Bs, int k) {
#pragma unroll
            for (int ni = 0; ni < NF; ++ni)
                b[buf][ni] = frag_ld<BKM, Cfg::BN, BK>(Bs, k, wn + ni * 8 + g4);
        };
        {
            const int s = g % STAGES;
            mbar_wait(full + s, (g / STAGES) & 1);
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
                a[mi] = frag_ld<AK, Cfg::BM, BK>(smem + s * SS, t, wm + mi * 8 + g4);
            load_b(0, smem + s * SS + SA, t);
        }
        for (int kt = 0; kt < kts; ++kt, ++g) {
            const int s = g % STAGES, s2 = (g + 1) % STAGES;
            const int ph2 = ((g + 1) / STAGES) & 1;
            const double* As = smem + s * SS;
            const double* Bs = As + SA;
            const double* As2 = smem + s2 * SS;
            const double* Bs2 = As2 + SA;
            const bool more = kt + 1 < kts;
            const int nks = more ? BK / 4 : (kvl + 3) / 4;
            uint32_t ready = more ? mbar_test(full + s2, ph2) : 1u;
#pragma unroll
            for (int ks = 0; ks < BK / 4; ++ks) {
                if (ks < nks) {
                    const int cur = ks & 1;
                    // source of the next k4 step's fragments: this stage, the next stage, none
                    const bool in_stage = ks + 1 < BK / 4;
                    const bool next = in_stage || more;
                    if (!in_stage && more && !ready) mbar_wait(full + s2, ph2);
                    const double* An = in_stage ? As : As2;
                    const double* Bn = in_stage ? Bs : Bs2;
                    const int kn = in_stage ? (ks + 1) * 4 + t : t;
                    if (next) load_b(cur ^ 1, Bn, kn);
#pragma unroll
                    for (int mi = 0; mi < FM; ++mi) {
#pragma unroll
                        for (int ni = 0; ni < NF; ++ni) dmma884(acc.c[mi][ni], a[mi], b[cur][ni]);
                        if (next) a[mi] = frag_ld<AK, Cfg::BM, BK>(An, kn, wm + mi * 8 + g4);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
    }

    template <class Prod, class Epi>
    __device__ static void run(int first, int stride, int nitems, const Prod& prod, Epi&& epi,
                               double* smem) {
        constexpr int FM = Cfg::FM, FN = Cfg::FN, WN = Cfg::WARPS_N;
        static_assert((BK / 4) % 2 == 0, "cross-stage fragment prefetch needs an even k4 count");
        static_assert(FN >= 2, "a warp column owns FN or FN - 1 fragments");
        uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SS);
        uint64_t* empty = full + STAGES;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, WARPS);
            }
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        }
        __syncthreads();
        if (warp == WARPS) {  // ---------------- producer warp
            int g = 0;
            for (int it = first; it < nitems; it += stride) {
                const int kts = prod.ktiles(it);
                for (int kt = 0; kt < kts; ++kt, ++g) {
                    const int s = g % STAGES;
                    if (g >= STAGES) mbar_wait(empty + s, ((g / STAGES) - 1) & 1);
                    double* st = smem + s * SS;
                    if (lane == 0) mbar_arrive_expect_tx(full + s, prod.stage_bytes(it, kt));
                    __syncwarp();
                    prod.bulk_rows(it, kt, st, st + SA, lane, full + s);
                }
            }
            return;
        }
        // ------------------------------------------------------------- consumer warps
        const int wmi = warp / WN, wni = (warp + wmi) % WN;
        const int wm = wmi * (8 * FM);
        Acc<Cfg> acc;
        int g = 0;
        for (int it = first; it < nitems; it += stride) {
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) acc.c[mi][ni][0] = acc.c[mi][ni][1] = 0.0;
            const int kts = prod.ktiles(it), kvl = prod.kvalid_last(it);
            const int nfr = prod.nfrags(it);
            const int base = nfr / WN, rem = nfr - base * WN;
            const int nf = base + (wni < rem ? 1 : 0);
            const int wn = 8 * (wni * base + min(wni, rem));
            if (nf == FN)
                item_loop<FN>(prod, smem, full, empty, kts, kvl, wm, wn, g, acc);
            else if (FN < 3 || nf == FN - 1)
                item_loop<FN - 1>(prod, smem, full, empty, kts, kvl, wm, wn, g, acc);
            else
                item_loop<(FN >= 3 ? FN - 2 : 1)>(prod, smem, full, empty, kts, kvl, wm, wn, g,
                                                  acc);
            epi(it, acc, wm, wn, nf);
        }
    }
};

// Visit every accumulator element: f(m_local, n_local, v(n), v(n+1)).
template <class Cfg, class F>
__device__ __forceinline__ void acc_foreach_pair(const Acc<Cfg>& acc, F&& f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp / Cfg::WARPS_N) * (8 * Cfg::FM), wn = (warp % Cfg::WARPS_N) * (8 * Cfg::FN);
#pragma unroll
    for (int mi = 0; mi < Cfg::FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::FN; ++ni)
            f(wm + mi * 8 + g, wn + ni * 8 + 2 * t, acc.c[mi][ni][0], acc.c[mi][ni][1]);
}

// Lane's row (within the CTA tile) of fragment fm: wm + 8 fm + g.
template <class Cfg>
__device__ __forceinline__ int frag_row(int fm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    return (warp / Cfg::WARPS_N) * (8 * Cfg::FM) + fm * 8 + (lane >> 2);
}

}  // namespace mg
