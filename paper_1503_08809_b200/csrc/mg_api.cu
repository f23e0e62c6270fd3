// mg_api.cu — the extern "C" boundary declared in include/modal_b200.h.
//
// Every entry point: validate arguments, select the device, run, and translate failures
// into MG_E* codes with a thread-local message (mg_last_error).  No CPU fallback exists:
// without an sm_100 device the compute entry points return MG_ECUDA.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <functional>
#include <future>
#include <string>
#include <thread>
#include <vector>

#include "mg_common.cuh"
#include "mg_domain.cuh"
#include "mg_gamma.cuh"

namespace mg {
void build_qtilde_dev(const double* k, const double* wk, int Nk, const double* x, int Nx,
                      const double* eps, const double* qk, int p, int l_min, int l_max,
                      double X, double kd, double amp, double* C_dev, double* qt_dev,
                      double* delta_out_dev, cudaStream_t s);
void bessel_table(const double* z, int nz, int l_max, double* out);
void ptable_dev(const double* q, const double* qt, const double* lw, const double* leg, int p,
                int Nx, int L, int nmu, double* P_dev);
void gamma2d_timings(double* ptable_ms, double* cells_ms);
void gamma2d_reset_timings();
void gamma2d_dev(const double* P_dev, const int* modes_host, int n, int p, int Nx, int nmu,
                 const double* mu_w, const double* wr2, double* gamma_host);

static thread_local std::string g_last_error;

void ensure_pool_configured() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    static bool done[64] = {false};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t threshold = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    done[dev] = true;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }

DeviceGuard::DeviceGuard(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(MG_ECUDA, "no CUDA device available (the Γ library has no CPU fallback)");
    }
    MG_REQUIRE(device >= 0 && device < n, "device index out of range");
    MG_CUDA(cudaGetDevice(&prev));
    MG_CUDA(cudaSetDevice(device));
    // architecture check once per device (cudaGetDeviceProperties costs ~ms per call)
    static std::atomic<int> checked[64];
    if (device >= 64 || checked[device].load() == 0) {
        int major = 0;
        MG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        if (major != 10) fail(MG_ECUDA, "library is built for sm_100a (B200) only");
        if (device < 64) checked[device].store(1);
    }
}
}  // namespace mg

using namespace mg;

template <class F>
static int guarded_named(const char* name, F&& f) {
    NvtxRange range(name);
    try {
        f();
        g_last_error.clear();
        return MG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host out of memory";
        return MG_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return MG_ECUDA;
    }
}

// every entry point: an NVTX range named after the C-ABI function around the guarded body
#define guarded(...) guarded_named(__func__, __VA_ARGS__)

static void full_range_bounds(const DomainIndex& D, int64_t begin, int64_t end, int* s, int* e) {
    MG_REQUIRE(0 <= begin && begin <= end && end <= D.count, "invalid flat range");
    D.triple(begin, s[0], s[1], s[2]);
    D.triple(end, e[0], e[1], e[2]);
}

// Cost model of one (l2,l3)-row with an l1 window of m triples (scheduler.py slab_costs,
// calibrated on a B200: the run contraction pays ~20 padded l1 per row, per-row work outside
// the run contraction is ~1.35x the x contraction).
static inline double row_cost(double m, int p, int Nx) {
    const double pairs = p * (p + 1) / 2.0;
    return (double)p * p * Nx * (m + 20.0) + 1.35 * pairs * p * p * Nx;
}

// Balanced contiguous l2 slabs of the full domain: bounds[0] = l_min .. bounds[n] = l_max+1
// (mg_slab_plan; the shard plan of both the torchrun ranks and the multi-device call).
static std::vector<int> slab_bounds(int l_min, int l_max, int p, int Nx, int nshards) {
    std::vector<double> cum(l_max - l_min + 2, 0.0);
    for (int l2 = l_min; l2 <= l_max; ++l2) {
        double c = 0;
        for (int l3 = l2; l3 <= std::min(2 * l2, l_max); ++l3) {
            int par = (l2 + l3) & 1;
            int lo = std::max(l_min, l3 - l2);
            if ((lo & 1) != par) ++lo;
            int hi = (l2 & 1) == par ? l2 : l2 - 1;
            if (lo > hi) continue;
            c += row_cost((hi - lo) / 2 + 1, p, Nx);
        }
        cum[l2 - l_min + 1] = cum[l2 - l_min] + c;
    }
    std::vector<int> bounds(nshards + 1);
    bounds[0] = l_min;
    for (int s = 1; s < nshards; ++s) {
        double target = cum.back() * s / nshards;
        int idx = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        bounds[s] = std::max(bounds[s - 1], std::min(l_min + idx, l_max + 1));
    }
    bounds[nshards] = l_max + 1;
    return bounds;
}

// Balanced l2 cut points for an arbitrary row list (flat sub-range or explicit triples):
// per-l2 modelled cost of the rows actually present, cut at the first l2 whose preceding
// cost reaches each target.  Returns bounds as above.
static std::vector<int> row_bounds(const std::vector<MgRow>& rows, int l_min, int l_max, int p,
                                   int Nx, int nshards) {
    std::vector<double> cum(l_max - l_min + 2, 0.0);
    for (const MgRow& r : rows) cum[r.l2 - l_min + 1] += row_cost(r.jhi - r.jlo + 1, p, Nx);
    for (size_t i = 1; i < cum.size(); ++i) cum[i] += cum[i - 1];
    std::vector<int> bounds(nshards + 1);
    bounds[0] = l_min;
    for (int s = 1; s < nshards; ++s) {
        double target = cum.back() * s / nshards;
        int idx = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        bounds[s] = std::max(bounds[s - 1], std::min(l_min + idx, l_max + 1));
    }
    bounds[nshards] = l_max + 1;
    return bounds;
}

static std::vector<int> device_list(int ndev, const int* devs) {
    MG_REQUIRE(ndev >= 1 && ndev <= 64, "ndev must be in [1, 64]");
    std::vector<int> d(ndev);
    for (int i = 0; i < ndev; ++i) d[i] = devs ? devs[i] : i;
    return d;
}


extern "C" {

int mg_version(void) { return 100; }

const char* mg_last_error(void) { return g_last_error.c_str(); }

int mg_debug_checks(uint32_t* counts, int n, int reset, int* checked, int device) {
    return guarded([&] {
        MG_REQUIRE(counts && n >= 0, "invalid argument");
        DeviceGuard g(device);
        const int c = debug_checks(counts, n, reset != 0);
        if (checked) *checked = c;
    });
}

int mg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int mg_domain_count(int l_min, int l_max, int64_t* count, int64_t* rows) {
    return guarded([&] {
        MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
        int64_t c = 0, r = 0;
        for (int l1 = l_min; l1 <= l_max; ++l1)
            for (int l2 = l1; l2 <= l_max; ++l2) {
                int n = row_len(l1, l2, l_max);
                c += n;
                r += n > 0;
            }
        if (count) *count = c;
        if (rows) *rows = r;
    });
}

int mg_domain_triples(int l_min, int l_max, int64_t begin, int64_t end, int32_t* l1,
                      int32_t* l2, int32_t* l3, int device) {
    return guarded([&] {
        MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
        MG_REQUIRE(l1 && l2 && l3, "null output");
        DeviceGuard g(device);
        weights(l_min, l_max, nullptr, nullptr, 0, begin, end, nullptr, l1, l2, l3);
    });
}

int mg_domain_match_range(int l_min, int l_max, const int32_t* l1, const int32_t* l2,
                          const int32_t* l3, int64_t count, int64_t* begin) {
    return guarded([&] {
        MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
        MG_REQUIRE(begin && count >= 0, "invalid argument");
        MG_REQUIRE(count == 0 || (l1 && l2 && l3), "null triple arrays");
        *begin = -1;
        if (count == 0) {
            *begin = 0;
            return;
        }
        int a = l1[0], b = l2[0], c = l3[0];
        if (a < l_min || a > l_max || b < a || b > l_max) return;
        const int st = row_start(a, b), n = row_len(a, b, l_max);
        if (n <= 0 || c < st || ((c - st) & 1) || (c - st) / 2 >= n) return;
        DomainIndex D;
        D.build(l_min, l_max);
        const int64_t flat0 = D.row_base[D.pair_off[a - l_min] + (b - a)] + (c - st) / 2;
        if (flat0 + count > D.count) return;
        // walk the enumeration order (geometry.py:161-171) alongside the list
        for (int64_t i = 1; i < count; ++i) {
            c += 2;
            if (c > std::min(a + b, l_max)) {
                for (++b;; ++b) {
                    if (b > l_max) {
                        ++a;
                        b = a;
                        if (a > l_max) return;  // unreachable: flat0 + count <= D.count
                    }
                    if (row_len(a, b, l_max) > 0) break;
                }
                c = row_start(a, b);
            }
            if (l1[i] != a || l2[i] != b || l3[i] != c) return;
        }
        *begin = flat0;
    });
}

int mg_weights(int l_min, int l_max, const double* C, const double* v, int h2_mode,
               int64_t begin, int64_t end, double* zm, int device) {
    return guarded([&] {
        MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
        MG_REQUIRE(C && v && zm, "null argument");
        MG_REQUIRE(h2_mode == MG_H2_GOSPER || h2_mode == MG_H2_EXACT, "unknown h2_mode");
        DeviceGuard g(device);
        weights(l_min, l_max, C, v, h2_mode, begin, end, zm, nullptr, nullptr, nullptr);
    });
}

int mg_plan_create(const double* q, const double* qt, const double* C, const double* v,
                   const double* wr2, const int64_t* modes, int p, int Nx, int n, int l_min,
                   int l_max, int h2_mode, int device, mg_plan** plan) {
    return guarded([&] {
        MG_REQUIRE(q && qt && C && v && wr2 && modes && plan, "null argument");
        DeviceGuard g(device);
        auto* P = new mg_plan();
        try {
            P->device = device;
            plan_init(P, q, qt, nullptr, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode);
        } catch (...) {
            delete P;
            throw;
        }
        *plan = P;
    });
}

int mg_plan_create_dev(const double* q, const double* qt_dev, const double* C,
                       const double* v, const double* wr2, const int64_t* modes, int p,
                       int Nx, int n, int l_min, int l_max, int h2_mode, int device,
                       mg_plan** plan) {
    return guarded([&] {
        MG_REQUIRE(q && qt_dev && C && v && wr2 && modes && plan, "null argument");
        DeviceGuard g(device);
        auto* P = new mg_plan();
        try {
            P->device = device;
            plan_init(P, q, nullptr, qt_dev, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode);
        } catch (...) {
            delete P;
            throw;
        }
        *plan = P;
    });
}

int mg_plan_execute(mg_plan* P, int l2_begin, int l2_end, double* gamma_dev, void* stream) {
    return guarded([&] {
        MG_REQUIRE(P, "null plan");
        DeviceGuard g(P->device);
        if (l2_end < 0) l2_end = P->l_max + 1;
        cudaStream_t st = (cudaStream_t)stream;
        execute_slab(P, l2_begin, l2_end, st);
        if (gamma_dev)
            MG_CUDA(cudaMemcpyAsync(gamma_dev, P->gamma.p, (size_t)P->nm * P->nm * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st));
    });
}

int mg_plan_fetch(mg_plan* P, double* gamma, void* stream) {
    return guarded([&] {
        MG_REQUIRE(P && gamma, "null argument");
        DeviceGuard g(P->device);
        cudaStream_t st = (cudaStream_t)stream;
        MG_CUDA(cudaMemcpyAsync(gamma, P->gamma.p, (size_t)P->nm * P->nm * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
        MG_CUDA(cudaStreamSynchronize(st));
    });
}

int mg_plan_stats(mg_plan* P, double* f_run, double* f_x, double* f_pair, int64_t* launches) {
    return guarded([&] {
        MG_REQUIRE(P, "null plan");
        if (f_run) *f_run = P->flops_run;
        if (f_x) *f_x = P->flops_x;
        if (f_pair) *f_pair = P->flops_pair;
        if (launches) *launches = P->launches;
    });
}

int mg_plan_set_profile(mg_plan* P, int on) {
    return guarded([&] {
        MG_REQUIRE(P, "null plan");
        DeviceGuard g(P->device);
        if (P->prof_used) MG_CUDA(cudaEventSynchronize(P->prof_events[P->prof_used - 1]));
        if (P->side_used) MG_CUDA(cudaEventSynchronize(P->side_events[P->side_used - 1]));
        P->profile = on != 0;
        for (double& m : P->prof_ms) m = 0.0;
        P->ns_used = 0;
        P->prof_used = 0;
        P->side_used = 0;
        P->prof_tags.clear();
    });
}

int mg_plan_kernel_ms(mg_plan* P, double* ms) {
    return guarded([&] {
        MG_REQUIRE(P && ms, "null argument");
        DeviceGuard g(P->device);
        prof_collect(P);
        nonsep_collect(P);
        for (int i = 0; i < MG_NPROF; ++i) ms[i] = P->prof_ms[i];
    });
}

int mg_plan_set_sparse_domain(mg_plan* P, const int32_t* l1, const int32_t* l2,
                              const int32_t* l3, const double* W, int64_t count) {
    return guarded([&] {
        MG_REQUIRE(P, "null plan");
        MG_REQUIRE(count >= 0, "count must be >= 0");
        MG_REQUIRE(count == 0 || (l1 && l2 && l3 && W), "null triple arrays");
        DeviceGuard g(P->device);
        nonsep_set_domain(P, l1, l2, l3, W, count);
    });
}

int mg_plan_nonsep(mg_plan* P, const double* alpha, double* b_dev, double* b_host,
                   void* stream) {
    return guarded([&] {
        MG_REQUIRE(P && alpha, "null argument");
        for (int i = 0; i < P->nm; ++i)
            MG_REQUIRE(std::isfinite(alpha[i]), "alpha contains non-finite values");
        DeviceGuard g(P->device);
        nonsep_execute(P, alpha, b_dev, b_host, (cudaStream_t)stream);
    });
}

void mg_plan_destroy(mg_plan* P) {
    if (!P) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(P->device);
    delete P;
    if (prev >= 0) cudaSetDevice(prev);
}

static void gamma_common(const double* q, const double* qt, const double* C, const double* v,
                         const double* wr2, const int64_t* modes, int p, int Nx, int n,
                         int l_min, int l_max, int h2_mode, int device, double* gamma,
                         const std::function<void(mg_plan*)>& run) {
    MG_REQUIRE(q && qt && C && v && wr2 && modes && gamma, "null argument");
    DeviceGuard g(device);
    mg_plan P;
    P.device = device;
    plan_init(&P, q, qt, nullptr, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode);
    run(&P);
    MG_CUDA(cudaMemcpy(gamma, P.gamma.p, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToHost));
}

// Run one shard per entry of `devs`, each on its own host thread with its own plan on its
// device (q̃ uploaded to every device, like the reference's per-worker copies), then merge the
// partial Γ's in shard order — merge_partials (scheduler.py:48-66) — so the result is bitwise
// reproducible for a given device list.  Shards on the same device serialise through the
// device's execute lock (device_mutex).  `run(P, s)` executes shard s on plan P.
static void gamma_shards(const double* q, const double* qt, const double* C, const double* v,
                         const double* wr2, const int64_t* modes, int p, int Nx, int n,
                         int l_min, int l_max, int h2_mode, const std::vector<int>& devs,
                         double* gamma, const std::function<void(mg_plan*, int)>& run) {
    const int ns = (int)devs.size();
    if (ns == 1) {
        gamma_common(q, qt, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode, devs[0], gamma,
                     [&](mg_plan* P) { run(P, 0); });
        return;
    }
    MG_REQUIRE(gamma, "null argument");
    const size_t nn = (size_t)n * n;
    std::vector<std::vector<double>> parts(ns);
    std::vector<std::exception_ptr> errs(ns);
    std::vector<std::thread> th;
    for (int s = 0; s < ns; ++s)
        th.emplace_back([&, s] {
            try {
                parts[s].assign(nn, 0.0);
                gamma_common(q, qt, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode, devs[s],
                             parts[s].data(), [&](mg_plan* P) { run(P, s); });
            } catch (...) {
                errs[s] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    std::memcpy(gamma, parts[0].data(), nn * sizeof(double));
    for (int s = 1; s < ns; ++s)
        for (size_t i = 0; i < nn; ++i) gamma[i] += parts[s][i];
}

int mg_gamma_sep(const double* q, const double* qt, const double* C, const double* v,
                 const double* wr2, const int64_t* modes, int p, int Nx, int n, int l_min,
                 int l_max, int h2_mode, int64_t begin, int64_t end, int ndev, const int* devs,
                 double* gamma) {
    return guarded([&] {
        MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
        const std::vector<int> dv = device_list(ndev, devs);
        // The rows of the flat range are enumerated on a host thread while the plans upload
        // and transpose q̃ (the one-shot drop-in call pays both every time), then cut into
        // one l2-slab shard per device: the full domain with the mg_slab_plan bounds (so the
        // shards are exactly the torchrun ranks' slabs), a sub-range with the same cost model
        // over its rows.
        std::vector<std::vector<MgRow>> shard(dv.size());
        std::shared_future<void> host_rows = std::async(std::launch::async, [&] {
            DomainIndex D;
            D.build(l_min, l_max);
            const int64_t e_ = end < 0 ? D.count : end;
            int s[3], e[3];
            full_range_bounds(D, begin, e_, s, e);
            std::vector<MgRow> rows;
            if (begin < e_) build_rows_range(l_min, l_max, l_min, l_max + 1, s, e, rows);
            const int nsh = (int)dv.size();
            if (nsh == 1) {
                shard[0] = std::move(rows);
                return;
            }
            const std::vector<int> b = (begin == 0 && e_ == D.count)
                                           ? slab_bounds(l_min, l_max, p, Nx, nsh)
                                           : row_bounds(rows, l_min, l_max, p, Nx, nsh);
            for (const MgRow& r : rows) {
                int k = (int)(std::upper_bound(b.begin(), b.end(), r.l2) - b.begin()) - 1;
                shard[std::min(std::max(k, 0), nsh - 1)].push_back(r);
            }
        });
        gamma_shards(q, qt, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode, dv, gamma,
                     [&](mg_plan* P, int s) {
                         host_rows.wait();
                         execute_rows(P, std::move(shard[s]), 0);
                     });
        host_rows.get();  // rethrows a range error from the host thread
    });
}

int mg_gamma_sep_slab(const double* q, const double* qt, const double* C, const double* v,
                      const double* wr2, const int64_t* modes, int p, int Nx, int n,
                      int l_min, int l_max, int h2_mode, int l2_begin, int l2_end,
                      int device, double* gamma) {
    return guarded([&] {
        gamma_common(q, qt, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode, device, gamma,
                     [&](mg_plan* P) {
                         execute_slab(P, l2_begin, l2_end < 0 ? l_max + 1 : l2_end, 0);
                     });
    });
}

int mg_gamma_sep_triples(const double* q, const double* qt, const double* C,
                         const double* v, const double* wr2, const int64_t* modes, int p,
                         int Nx, int n, int l_min, int l_max, int h2_mode,
                         const int32_t* l1, const int32_t* l2, const int32_t* l3,
                         int64_t count, int ndev, const int* devs, double* gamma) {
    return guarded([&] {
        MG_REQUIRE(count == 0 || (l1 && l2 && l3), "null triple arrays");
        MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
        const std::vector<int> dv = device_list(ndev, devs);
        const int ns = (int)dv.size();
        if (ns == 1) {
            gamma_common(q, qt, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode, dv[0], gamma,
                         [&](mg_plan* P) { execute_triples(P, l1, l2, l3, count, 0); });
            return;
        }
        // l2-slab shards of the explicit list, balanced by the per-l2 row cost model
        std::vector<MgRow> rows;
        {
            std::vector<std::pair<int, int>> keys((size_t)count);
            for (int64_t i = 0; i < count; ++i) {
                MG_REQUIRE(l2[i] >= l_min && l2[i] <= l_max, "triple outside [l_min, l_max]");
                keys[i] = {l2[i], l3[i] * 2 + (l1[i] & 1)};
            }
            std::sort(keys.begin(), keys.end());
            for (size_t i = 0; i < keys.size();) {
                size_t j = i;
                while (j < keys.size() && keys[j] == keys[i]) ++j;
                MgRow r{keys[i].first, 0, 0, 0, (int)(j - i) - 1, 0};
                rows.push_back(r);
                i = j;
            }
        }
        const std::vector<int> b = row_bounds(rows, l_min, l_max, p, Nx, ns);
        std::vector<std::vector<int32_t>> s1(ns), s2(ns), s3(ns);
        for (int64_t i = 0; i < count; ++i) {
            int k = (int)(std::upper_bound(b.begin(), b.end(), l2[i]) - b.begin()) - 1;
            k = std::min(std::max(k, 0), ns - 1);
            s1[k].push_back(l1[i]);
            s2[k].push_back(l2[i]);
            s3[k].push_back(l3[i]);
        }
        gamma_shards(q, qt, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode, dv, gamma,
                     [&](mg_plan* P, int s) {
                         execute_triples(P, s1[s].data(), s2[s].data(), s3[s].data(),
                                         (int64_t)s1[s].size(), 0);
                     });
    });
}

int mg_slab_plan(int l_min, int l_max, int p, int Nx, int nshards, int* bounds) {
    return guarded([&] {
        MG_REQUIRE(2 <= l_min && l_min <= l_max, "require 2 <= l_min <= l_max");
        MG_REQUIRE(nshards >= 1 && bounds, "invalid shard count");
        std::vector<int> b = slab_bounds(l_min, l_max, p, Nx, nshards);
        std::copy(b.begin(), b.end(), bounds);
    });
}

int mg_build_qtilde(const double* k, const double* wk, int Nk, const double* x, int Nx,
                    const double* eps, const double* qk, int p, int l_min, int l_max,
                    double x_delta, double k_damp, double eps_amp, int device, double* C,
                    double* qt, double* delta) {
    return guarded([&] {
        MG_REQUIRE(k && wk && x && eps && qk, "null argument");
        DeviceGuard g(device);
        const int L = l_max - l_min + 1;
        DBuf<double> dC, dqt, dd;
        if (C) dC.alloc(L);
        if (qt) dqt.alloc((size_t)p * Nx * L);
        if (delta) dd.alloc((size_t)L * Nk);
        build_qtilde_dev(k, wk, Nk, x, Nx, eps, qk, p, l_min, l_max, x_delta, k_damp, eps_amp,
                         dC.p, dqt.p, dd.p, 0);
        if (C) MG_CUDA(cudaMemcpy(C, dC.p, L * sizeof(double), cudaMemcpyDeviceToHost));
        if (qt)
            MG_CUDA(cudaMemcpy(qt, dqt.p, (size_t)p * Nx * L * sizeof(double),
                               cudaMemcpyDeviceToHost));
        if (delta)
            MG_CUDA(cudaMemcpy(delta, dd.p, (size_t)L * Nk * sizeof(double),
                               cudaMemcpyDeviceToHost));
    });
}

int mg_build_qtilde_dev(const double* k, const double* wk, int Nk, const double* x, int Nx,
                        const double* eps, const double* qk, int p, int l_min, int l_max,
                        double x_delta, double k_damp, double eps_amp, int device,
                        double* C_dev, double* qt_dev, void* stream) {
    return guarded([&] {
        MG_REQUIRE(k && wk && x && eps && qk, "null argument");
        DeviceGuard g(device);
        build_qtilde_dev(k, wk, Nk, x, Nx, eps, qk, p, l_min, l_max, x_delta, k_damp, eps_amp,
                         C_dev, qt_dev, nullptr, (cudaStream_t)stream);
    });
}

int mg_bessel_table(const double* z, int nz, int l_max, int device, double* out) {
    return guarded([&] {
        MG_REQUIRE(z && out, "null argument");
        DeviceGuard g(device);
        bessel_table(z, nz, l_max, out);
    });
}

int mg_ptable(const double* q, const double* qt, const double* lw, const double* legendre,
              int p, int Nx, int L, int nmu, int device, double* ptable) {
    return guarded([&] {
        MG_REQUIRE(q && qt && lw && legendre && ptable, "null argument");
        MG_REQUIRE(p >= 1 && Nx >= 1 && L >= 1 && nmu >= 1, "invalid sizes");
        DeviceGuard g(device);
        gamma2d_reset_timings();
        const size_t np = (size_t)p * p * Nx * nmu;
        DBuf<double> dP(np);
        ptable_dev(q, qt, lw, legendre, p, Nx, L, nmu, dP.p);
        MG_CUDA(cudaMemcpy(ptable, dP.p, np * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int mg_gamma2d(const double* q, const double* qt, const double* lw, const double* legendre,
               const double* ptable, const double* mu_w, const double* wr2,
               const int64_t* modes, int p, int Nx, int L, int nmu, int n, int device,
               double* gamma) {
    return guarded([&] {
        MG_REQUIRE(mu_w && wr2 && modes && gamma, "null argument");
        MG_REQUIRE(ptable || (q && qt && lw && legendre), "need the P table or its inputs");
        MG_REQUIRE(p >= 1 && Nx >= 1 && nmu >= 1 && n >= 1, "invalid sizes");
        std::vector<int> md(3 * (size_t)n);
        for (int i = 0; i < n; ++i) {
            int64_t a = modes[3 * i], b = modes[3 * i + 1], c = modes[3 * i + 2];
            MG_REQUIRE(0 <= a && a <= b && b <= c && c < p, "mapping triples must satisfy i<=j<=k<p");
            md[3 * i] = (int)a; md[3 * i + 1] = (int)b; md[3 * i + 2] = (int)c;
        }
        DeviceGuard g(device);
        gamma2d_reset_timings();
        const size_t np = (size_t)p * p * Nx * nmu;
        DBuf<double> dP(np);
        if (ptable)
            dP.upload(ptable, np);
        else
            ptable_dev(q, qt, lw, legendre, p, Nx, L, nmu, dP.p);
        gamma2d_dev(dP.p, md.data(), n, p, Nx, nmu, mu_w, wr2, gamma);
    });
}

int mg_gamma2d_timings(double* ptable_ms, double* cells_ms) {
    return guarded([&] { gamma2d_timings(ptable_ms, cells_ms); });
}

int mg_gamma_nonsep(const double* q, const double* qt, const double* C, const double* v,
                    const double* wr2, const int64_t* modes, int p, int Nx, int n, int l_min,
                    int l_max, int h2_mode, const double* alpha, const int32_t* l1,
                    const int32_t* l2, const int32_t* l3, const double* W, int64_t count,
                    int device, double* b) {
    return guarded([&] {
        MG_REQUIRE(q && qt && C && v && wr2 && modes && alpha && b, "null argument");
        MG_REQUIRE(count == 0 || (l1 && l2 && l3 && W), "null triple arrays");
        DeviceGuard g(device);
        mg_plan P;
        P.device = device;
        plan_init(&P, q, qt, nullptr, C, v, wr2, modes, p, Nx, n, l_min, l_max, h2_mode);
        if (count == 0) {
            std::memset(b, 0, sizeof(double) * n);
            return;
        }
        nonsep(&P, alpha, l1, l2, l3, W, count, b, 0);
    });
}

}  // extern "C"
