#include <torch/extension.h>
#include <cuda_runtime.h>
#include <c10/cuda/CUDAStream.h>
#include <cstdint>

__global__ void sm_copy(const int4* __restrict__ src, int4* __restrict__ dst, long long n) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        int4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
        dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
    }
    for (; i < n; i += stride) dst[i] = src[i];
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA bulk: 4 buffers of 16 KB per CTA; load (global->smem, mbarrier), store (smem->global, bulk group)
__global__ void tma_copy(const char* __restrict__ src, char* __restrict__ dst, long long nbytes) {
    constexpr int kBuf = 4, kChunk = 16384;
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[kBuf];
    if (threadIdx.x != 0) return;
    for (int b = 0; b < kBuf; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long nchunks = nbytes / kChunk;
    uint32_t phase[kBuf] = {0, 0, 0, 0};
    int it = 0;
    for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int b = it % kBuf;
        char* buf = sm + b * kChunk;
        // buffer reuse: the store that read it must be done
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBuf - 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(kChunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(buf)), "l"(src + c * kChunk), "r"(kChunk), "r"(su32(&bar[b])) : "memory");
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}\n"
                         : "=r"(done) : "r"(su32(&bar[b])), "r"(phase[b]) : "memory");
        }
        phase[b] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * kChunk), "r"(su32(buf)), "r"(kChunk) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

void run_sm(torch::Tensor src, int64_t dst_ptr, int64_t nbytes, int64_t grid) {
    auto st = c10::cuda::getCurrentCUDAStream();
    sm_copy<<<grid, 256, 0, st>>>((const int4*)src.data_ptr(), (int4*)dst_ptr, nbytes / 16);
}
void run_tma(torch::Tensor src, int64_t dst_ptr, int64_t nbytes, int64_t grid) {
    auto st = c10::cuda::getCurrentCUDAStream();
    static bool set = false;
    if (!set) { cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384); set = true; }
    tma_copy<<<grid, 32, 4 * 16384, st>>>((const char*)src.data_ptr(), (char*)dst_ptr, nbytes);
}
// pull variants: src pointer given raw (peer), dst local tensor
void run_sm_pull(int64_t src_ptr, torch::Tensor dst, int64_t nbytes, int64_t grid) {
    auto st = c10::cuda::getCurrentCUDAStream();
    sm_copy<<<grid, 256, 0, st>>>((const int4*)src_ptr, (int4*)dst.data_ptr(), nbytes / 16);
}
__global__ void __launch_bounds__(1024) sm_copy8(const int4* __restrict__ src, int4* __restrict__ dst, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < 8; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n; i += stride) dst[i] = src[i];
}
// one fat block per SM (1024 threads, 32 KB smem reserved so no 2-CTA GEMM CTA shares the SM)
void run_fat(int64_t src_ptr, int64_t dst_ptr, int64_t nbytes, int64_t grid, int64_t smem) {
    auto st = c10::cuda::getCurrentCUDAStream();
    static bool set = false;
    if (!set) { cudaFuncSetAttribute(sm_copy8, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); set = true; }
    sm_copy8<<<grid, 1024, smem, st>>>((const int4*)src_ptr, (int4*)dst_ptr, nbytes / 16);
}
void run_tma_pull(int64_t src_ptr, torch::Tensor dst, int64_t nbytes, int64_t grid) {
    auto st = c10::cuda::getCurrentCUDAStream();
    static bool set = false;
    if (!set) { cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384); set = true; }
    tma_copy<<<grid, 32, 4 * 16384, st>>>((const char*)src_ptr, (char*)dst.data_ptr(), nbytes);
}

// fat pull staged through shared memory with cp.async (LDGSTS): each of the
// 1024 threads keeps a ring of R 16-byte slots in flight (R * 16 KB of smem
// per block), no registers held by the loads in flight
template <int R>
__global__ void __launch_bounds__(1024) lds_pull(const int4* __restrict__ src, int4* __restrict__ dst, long long n) {
    extern __shared__ int4 sm4[];
    const int tid = threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long i0 = blockIdx.x * (long long)blockDim.x + tid;
    long long k = 0;  // element index of this thread: i0 + k * stride
    const long long cnt = i0 < n ? (n - i0 + stride - 1) / stride : 0;
    for (; k < cnt + R - 1; ++k) {
        if (k < cnt) {
            uint32_t d = (uint32_t)__cvta_generic_to_shared(&sm4[(k % R) * blockDim.x + tid]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src + i0 + k * stride) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        const long long w = k - (R - 1);
        if (w >= 0) {
            asm volatile("cp.async.wait_group %0;" :: "n"(R - 1) : "memory");
            dst[i0 + w * stride] = sm4[(w % R) * blockDim.x + tid];
        }
    }
}
void run_lds_pull(int64_t src_ptr, torch::Tensor dst, int64_t nbytes, int64_t grid, int64_t ring) {
    auto st = c10::cuda::getCurrentCUDAStream();
    if (ring == 8) {
        cudaFuncSetAttribute(lds_pull<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
        lds_pull<8><<<grid, 1024, 8 * 16384, st>>>((const int4*)src_ptr, (int4*)dst.data_ptr(), nbytes / 16);
    } else {
        cudaFuncSetAttribute(lds_pull<13>, cudaFuncAttributeMaxDynamicSharedMemorySize, 13 * 16384);
        lds_pull<13><<<grid, 1024, 13 * 16384, st>>>((const int4*)src_ptr, (int4*)dst.data_ptr(), nbytes / 16);
    }
}

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
    m.def("run_sm", &run_sm); m.def("run_tma", &run_tma);
    m.def("run_sm_pull", &run_sm_pull); m.def("run_fat", &run_fat); m.def("run_lds_pull", &run_lds_pull); m.def("run_tma_pull", &run_tma_pull);
}
