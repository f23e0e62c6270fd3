// mg_gamma.cuh — the resident Γ plan (shared by mg_gamma.cu and mg_api.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

#include "mg_common.cuh"
#include "mg_domain.cuh"

// One (l2,l3)-row of the factorised sum: l1 runs over l0[par] + 2 j, j in [jlo, jhi].
// (par = l1 parity; for the reference domain par = (l2 + l3) & 1.)
struct MgRow {
    int l2, l3, par, jlo, jhi, pad;
};
// One M-tile of the run-contraction GEMM: `nslots` (<= 128) consecutive (row, c) slots of one
// (l2, parity) group, starting at slot c0 of row row0 (global row index); rows touched: nrows.
struct MgTile {
    int row0, c0, nslots, nrows, jlo, jhi, pad0, pad1;
};

constexpr int MG_NPROF = 8;

// Batch scratch, pooled per device so that one-shot calls (the drop-in API) do not pay for
// allocating and zeroing gigabytes every time.  Buffers only grow; they are zeroed when
// (re)allocated (H's x pads must never hold NaN) and never shrink.  Executes on one device
// are serialised by device_mutex(), so concurrent callers (threads, shards) share it safely.
struct MgScratch {
    mg::DBuf<double> ZT, panel, H, S, G, R, Sq, Z;
};

// Prepared (host-built, device-uploaded) batch tables of one slab; cached in the plan so a
// repeated execute of the same slab skips the host preparation.
struct MgPrepared {
    bool valid = false;
    int key_a = -1, key_b = -1;
    int64_t nrows = 0;
    std::vector<MgRow> hrows;
    std::vector<int64_t> hzoff;
    std::vector<MgTile> tiles;
    std::vector<int> tile_first;
    int max_tile_rows = 1;
    int64_t maxzt = 1, maxpanel = 1;
    mg::DBuf<MgRow> rows;
    mg::DBuf<int64_t> zoff;
    mg::DBuf<MgTile> tiles_d;
    mg::DBuf<int64_t> poff;
};

struct mg_plan {
    int device = 0;
    int p = 0, Nx = 0, NxP = 0, nm = 0, l_min = 2, l_max = 2, L = 0, h2_mode = 0;
    int P2 = 0;        // p(p+1)/2 unordered basis pairs
    int Nxw = 0;       // x stride of WQT rows (Nx when even, else NxP)
    int l0[2] = {0, 0};      // first l of each parity class
    int64_t wbase[2] = {0, 0};  // WQB offset of each parity class
    int wrows[2] = {0, 0};      // WQB rows per column block of each class (+ zero rows)
    int nclass[2] = {0, 0};  // number of l in each parity class
    mg::DBuf<double> q, QT, WQT, C, v, lf, wr2, fl;
    mg::DBuf<int> modes;  // [nm][3]
    // scratch
    mg::DBuf<double> gamma;     // Γ of the last execute (owned by the plan)
    MgScratch* sc = nullptr;    // per-device scratch pool (shared by plans on the device)
    MgPrepared prep;            // cached batch tables of the last executed slab
    int nb1 = 0, nb3 = 0;  // rows per run/x-contraction batch, rows per pair-contraction batch
    // stats of the last execute
    double flops_run = 0, flops_x = 0, flops_pair = 0;
    int64_t launches = 0;
    // optional kernel timing: ms per family {exposed operand wait, run, x, gather, pair,
    // final, side-stream operand kernels (overlapped)}
    bool profile = false;
    double prof_ms[MG_NPROF] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::vector<cudaEvent_t> prof_events;
    std::vector<int> prof_tags;
    size_t prof_used = 0;
    std::vector<cudaEvent_t> side_events;  // (start, end) pairs on the side stream
    size_t side_used = 0;
    // streams/events of the batch pipeline (created on first execute, on the plan's device)
    cudaStream_t ms = nullptr, ss = nullptr;
    cudaEvent_t ev_start[2] = {}, ev_end[2] = {}, ev_panel[2] = {};
    cudaEvent_t ev_s = nullptr, ev_x = nullptr;
    mg::DBuf<int> l0d;
    ~mg_plan() {
        for (auto e : prof_events) cudaEventDestroy(e);
        for (auto e : side_events) cudaEventDestroy(e);
        for (auto e : ns_events) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_start[0], ev_start[1], ev_end[0], ev_end[1], ev_panel[0],
                              ev_panel[1], ev_s, ev_x})
            if (e) cudaEventDestroy(e);
        if (ms) cudaStreamDestroy(ms);
        if (ss) cudaStreamDestroy(ss);
    }
    // host copies (for the direct/nonsep paths)
    std::vector<double> hC, hv;
    std::vector<int> hmodes;  // [nm][3]
    // resident sparse domain + buffers of the non-separable path
    mg::DBuf<int32_t> ns_trip;  // [count][4] = l1, l2, l3, 0
    mg::DBuf<double> ns_W, ns_part, ns_b, ns_alpha;
    mg::DBuf<double> ns_wz;          // [count] W_t * zm_t (h2_mode of the plan), DMMA kernel
    mg::DBuf<double> ns_qt2, ns_q1w; // x-blocked q̃ tables of the DMMA kernel (built lazily)
    int64_t ns_count = 0;
    int ns_blocks = 0;
    int ns_dmma_blocks = 0;
    std::vector<cudaEvent_t> ns_events;  // (start, end) pairs of profiled nonsep calls
    size_t ns_used = 0;
};

namespace mg {
MgScratch* scratch_pool(int device);
std::recursive_mutex& device_mutex(int device);
void plan_init(mg_plan* P, const double* q, const double* qt_host, const double* qt_dev,
               const double* C, const double* v, const double* wr2, const int64_t* modes,
               int p, int Nx, int n, int l_min, int l_max, int h2_mode);
// Rows of the l2-slab [l2a, l2b) clipped to the flat range (s1,s2,s3) <= t < (e1,e2,e3).
void build_rows(const mg_plan* P, int l2a, int l2b, const int* s, const int* e,
                std::vector<MgRow>& rows);
// Same without a plan (host only; safe to run on another thread while the plan is built).
void build_rows_range(int l_min, int l_max, int l2a, int l2b, const int* s, const int* e,
                      std::vector<MgRow>& rows);
void execute_rows(mg_plan* P, std::vector<MgRow>&& rows, cudaStream_t st);
void execute_slab(mg_plan* P, int l2a, int l2b, cudaStream_t st);
void execute_triples(mg_plan* P, const int32_t* l1, const int32_t* l2, const int32_t* l3,
                     int64_t count, cudaStream_t st);
void nonsep_set_domain(mg_plan* P, const int32_t* l1, const int32_t* l2, const int32_t* l3,
                       const double* W, int64_t count);
void nonsep_execute(mg_plan* P, const double* alpha, double* b_dev, double* b_host,
                    cudaStream_t st);
void nonsep_collect(mg_plan* P);
// Resolve the recorded per-launch timing events of profiled executes into prof_ms.
void prof_collect(mg_plan* P);
void nonsep(mg_plan* P, const double* alpha, const int32_t* l1, const int32_t* l2,
            const int32_t* l3, const double* W, int64_t count, double* b, cudaStream_t st);
void weights(int l_min, int l_max, const double* C, const double* v, int h2_mode,
             int64_t begin, int64_t end, double* zm, int32_t* o1, int32_t* o2, int32_t* o3);
std::vector<double> log_factorials(int n);
int debug_checks(uint32_t* out, int n, bool reset);
}  // namespace mg
