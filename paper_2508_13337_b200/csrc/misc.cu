// Small helper kernels of the layer pipeline.
#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

// rows landing on each local expert of rank dst: sum over sources of the
// all-gathered per-expert counts (pf_pipeline.cpp:50-55).
__global__ void recv_counts_kernel(const int32_t* __restrict__ tpe_all, int W, int E, int dst,
                                   int32_t* __restrict__ rpe) {
    const int El = E / W;
    const int le = blockIdx.x * blockDim.x + threadIdx.x;
    if (le >= El) return;
    int a = 0;
    for (int s = 0; s < W; ++s) a += tpe_all[s * E + dst * El + le];
    rpe[le] = a;
}

// CountMismatch check of a grouped FFN on the device (pf_pipeline.cpp:102-103):
// the groups must cover exactly `rows` rows.  Writes the counts clamped so
// that their running sum never passes `rows` (the GEMMs run on these: no
// access past the buffers whatever the caller passed) and, on a mismatch,
// records XMOE_ERR_COUNT_MISMATCH in the context's host-mapped error word
// (xmoe_ctx_status reports it) — no host synchronisation.
__global__ void count_check_kernel(const int32_t* __restrict__ rpe, int G, long long rows,
                                   int32_t* __restrict__ clamped, int* err) {
    if (threadIdx.x != 0) return;
    long long run = 0;
    bool bad = false;
    for (int g = 0; g < G; ++g) {
        const long long v = rpe[g];
        bad |= v < 0;
        const long long c = v < 0 ? 0 : (run + v > rows ? rows - run : v);
        clamped[g] = static_cast<int32_t>(c);
        run += v < 0 ? 0 : v;
    }
    if (bad || run != rows) atomicCAS(err, 0, XMOE_ERR_COUNT_MISMATCH);
}

void launch_count_check(const int32_t* rpe, int G, long long rows, int32_t* clamped, int* err, cudaStream_t st) {
    count_check_kernel<<<1, 32, 0, st>>>(rpe, G, rows, clamped, err);
    XMOE_LAUNCH_CHECK();
}

__global__ void fill_i32_kernel(int32_t* p, int n, int32_t v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// out[b, c, r] = in[b, r, c] with optional f64 -> bf16 conversion (weights
// into the K-major B200 layout at layer creation).
template <typename Tin, typename Tout>
__global__ void transpose_kernel(const Tin* __restrict__ in, int rows, int cols,
                                 Tout* __restrict__ out) {
    __shared__ float tile[32][33];
    const int b = blockIdx.z;
    const Tin* src = in + static_cast<size_t>(b) * rows * cols;
    Tout* dst = out + static_cast<size_t>(b) * rows * cols;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = static_cast<float>(src[static_cast<size_t>(r) * cols + c]);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[static_cast<size_t>(c) * rows + r] = static_cast<Tout>(tile[threadIdx.x][i]);
    }
}

void launch_recv_counts(const int32_t* tpe_all, int W, int E, int dst, int32_t* rpe,
                        cudaStream_t st) {
    const int El = E / W;
    recv_counts_kernel<<<ceil_div(El, 128), 128, 0, st>>>(tpe_all, W, E, dst, rpe);
    XMOE_LAUNCH_CHECK();
}

void launch_fill_i32(int32_t* p, int n, int32_t v, cudaStream_t st) {
    if (n == 0) return;
    fill_i32_kernel<<<ceil_div(n, 256), 256, 0, st>>>(p, n, v);
    XMOE_LAUNCH_CHECK();
}

__global__ void f32_to_f64_kernel(const float* __restrict__ in, long long n, double* __restrict__ out) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<double>(in[i]);
}

void launch_f32_to_f64(const float* in, long long n, double* out, cudaStream_t st) {
    if (n == 0) return;
    f32_to_f64_kernel<<<ceil_div(n, 256), 256, 0, st>>>(in, n, out);
    XMOE_LAUNCH_CHECK();
}

__global__ void adjacent_diff_kernel(const int32_t* __restrict__ ptr, int n, int32_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ptr[i + 1] - ptr[i];
}

void launch_adjacent_diff(const int32_t* ptr, int n, int32_t* out, cudaStream_t st) {
    if (n == 0) return;
    adjacent_diff_kernel<<<ceil_div(n, 256), 256, 0, st>>>(ptr, n, out);
    XMOE_LAUNCH_CHECK();
}

void launch_transpose(int dtype_in, const void* in, int batch, int rows, int cols, int dtype_out,
                      void* out, cudaStream_t st) {
    if (batch == 0 || rows == 0 || cols == 0) return;
    dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32), batch);
    dim3 block(32, 8);
    if (dtype_in == XMOE_BF16 && dtype_out == XMOE_BF16)
        transpose_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, block, 0, st>>>(
            static_cast<const __nv_bfloat16*>(in), rows, cols, static_cast<__nv_bfloat16*>(out));
    else if (dtype_in == XMOE_F64 && dtype_out == XMOE_BF16)
        transpose_kernel<double, __nv_bfloat16><<<grid, block, 0, st>>>(
            static_cast<const double*>(in), rows, cols, static_cast<__nv_bfloat16*>(out));
    else
        fail(XMOE_ERR_VALIDATION, "transpose: unsupported dtype pair");
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
