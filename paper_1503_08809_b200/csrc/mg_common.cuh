// mg_common.cuh — error plumbing and device-memory RAII for the C-ABI library.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/modal_b200.h"

namespace mg {

// A failed library call carries one of the MG_E* codes up to the C boundary.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

// Device memory comes from the device's stream-ordered pool with an unbounded release
// threshold: freeing a plan's tables returns them to the pool instead of the driver, so the
// one-shot drop-in call does not pay cudaMalloc/cudaFree (which synchronise) every time.
void ensure_pool_configured();

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line,
                  cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) fail(MG_ENOMEM, buf);
    fail(MG_ECUDA, buf);
}

#define MG_CUDA(x) ::mg::check_cuda((x), #x, __FILE__, __LINE__)
#define MG_LAUNCHED() ::mg::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)
#define MG_REQUIRE(cond, msg) \
    do {                      \
        if (!(cond)) ::mg::fail(MG_EINVAL, (msg)); \
    } while (0)

// NVTX range for the enclosing scope (header-only nvtx3: a no-op unless a tool such as nsys or
// ncu --nvtx is attached).  Every C-ABI entry point opens one named after itself; the Γ
// pipeline adds ranges for row preparation, each batch's enqueue and the final gather.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define MG_NVTX_CAT2(a, b) a##b
#define MG_NVTX_CAT(a, b) MG_NVTX_CAT2(a, b)
#define MG_NVTX(name) ::mg::NvtxRange MG_NVTX_CAT(mg_nvtx_, __LINE__)(name)

// Selects `device` for the lifetime of the guard and verifies it is an sm_100 part.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int device);
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Owning device buffer (typed, zero-copy moves).
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count == 0) return;
        ensure_pool_configured();
        MG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), 0));
        n = count;
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p) cudaFreeAsync(p, 0);
        p = nullptr;
        n = 0;
    }
    void upload(const T* h, size_t count, cudaStream_t s = 0) {
        ensure(count);
        if (count) MG_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void zero(cudaStream_t s = 0) {
        if (n) MG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace mg
