// FP64 parity (and F32) instantiations of the grouped expert FFN — reproduces
// moesim::grouped_expert_mlp (/root/reference/proj/src/pf_pipeline.cpp:83-105)
// bit for bit: each output is sum_p a[i,p]*b[p,j] accumulated in ascending p
// with separately rounded multiply and add (kernels_scalar.cpp:11-23,
// -ffp-contract=off), then ReLU (kernels_scalar.cpp:25-27).
//
// This is the drop-in parity mode, not the performance path (that is the
// tcgen05 bf16 kernel in gemm_tc.cu).  One thread per output element; the
// warp spans output columns so B rows are coalesced and A is a broadcast.
#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

template <typename T>
__global__ void grouped_gemm_simt_kernel(const T* __restrict__ A, int K, const int32_t* __restrict__ rows_per_group,
                                         int G, const T* __restrict__ B, int N, T* __restrict__ D, int relu) {
    extern __shared__ int32_t pre[];  // [G+1] row prefix
    if (threadIdx.x == 0) {
        int a = 0;
        for (int g = 0; g < G; ++g) {
            pre[g] = a;
            a += rows_per_group[g];
        }
        pre[G] = a;
    }
    __syncthreads();
    const int row = blockIdx.x;
    const int col = blockIdx.y * blockDim.x + threadIdx.x;
    if (row >= pre[G] || col >= N) return;
    int lo = 0, hi = G - 1;  // last g with pre[g] <= row (skips empty groups)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= row) lo = mid;
        else hi = mid - 1;
    }
    const T* a = A + static_cast<size_t>(row) * K;
    const T* b = B + static_cast<size_t>(lo) * K * N + col;
    // F64: the reference's order and rounding; F32: the same order with the
    // exact fp32 products accumulated in fp64, rounded once to fp32
    double acc = 0.0;
    for (int p = 0; p < K; ++p)
        acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(a[p]), static_cast<double>(b[static_cast<size_t>(p) * N])));
    if (relu) acc = acc > 0.0 ? acc : 0.0;
    D[static_cast<size_t>(row) * N + col] = static_cast<T>(acc);
}

void launch_grouped_gemm_f64(const double* A, long long rows_bound, int K,
                             const int32_t* rows_per_group, int G, const double* B, int N,
                             double* D, int relu, cudaStream_t st) {
    if (rows_bound == 0 || N == 0) return;
    require(rows_bound < (1ll << 31), XMOE_ERR_VALIDATION, "too many rows");
    dim3 grid(static_cast<unsigned>(rows_bound), ceil_div(N, 128));
    grouped_gemm_simt_kernel<double><<<grid, 128, sizeof(int32_t) * (G + 1), st>>>(A, K, rows_per_group, G, B, N,
                                                                                  D, relu);
    XMOE_LAUNCH_CHECK();
}

// F32 instantiation: fp32 operands, the reference's order (ascending p,
// separate multiply and add) with fp64 accumulation, one rounding to fp32.
void launch_grouped_gemm_f32(const float* A, long long rows_bound, int K, const int32_t* rows_per_group, int G,
                             const float* B, int N, float* D, int relu, cudaStream_t st) {
    if (rows_bound == 0 || N == 0) return;
    require(rows_bound < (1ll << 31), XMOE_ERR_VALIDATION, "too many rows");
    dim3 grid(static_cast<unsigned>(rows_bound), ceil_div(N, 128));
    grouped_gemm_simt_kernel<float><<<grid, 128, sizeof(int32_t) * (G + 1), st>>>(A, K, rows_per_group, G, B, N, D,
                                                                                 relu);
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
