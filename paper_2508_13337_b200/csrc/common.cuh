// Shared helpers for the xmoe sm_100a kernels and the C-ABI host layer.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "xmoe/xmoe.h"

namespace xmoe {

// Typed failures, 1:1 with the reference's exception family
// (/root/reference/proj/include/moesim/error.hpp:10-38) plus CUDA/NCCL.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }
inline void require(bool ok, int code, const char* m) {
    if (!ok) fail(code, m);
}

// C-ABI wrapper: runs f, maps typed failures to status codes and keeps the
// message for xmoe_last_error() (thread-local).
extern thread_local std::string g_last_error;
template <class F>
int guarded(F&& f) {
    try {
        f();
        return XMOE_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return XMOE_ERR_INTERNAL;
    }
}

#define XMOE_CUDA(expr)                                                               \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess)                                                        \
            ::xmoe::fail(XMOE_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

// Every kernel launch of the library passes through this check, which also
// counts it (xmoe_kernel_launches()).
// XMOE_SYNC_CHECK=1 (debugging): synchronise after every launch and name
// the failing launch site.
extern std::atomic<unsigned long long> g_kernel_launches;
bool sync_check_enabled();
void sync_check(const char* file, int line);
#define XMOE_LAUNCH_CHECK()                                              \
    do {                                                                 \
        ::xmoe::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
        XMOE_CUDA(cudaGetLastError());                                   \
        if (::xmoe::sync_check_enabled()) ::xmoe::sync_check(__FILE__, __LINE__); \
    } while (0)

constexpr int kNumSMs = 148;

// NVTX range over a C-ABI call (host-side; free when no profiler is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ---------------------------------------------------------------- device utils
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_na_v4(void* p, const int4& v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w));
}

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

}  // namespace xmoe
