// Weighted combine — B200 restatement of moesim::scatter_combine
// (/root/reference/proj/src/pft.cpp:79-91) as a deterministic gather-reduce.
//
// The reference zero-initialises out and applies out[t_i] += w_i * rows[i]
// (axpy, kernels_scalar.cpp:29-31) for i ascending, so a token sums its
// copies in ascending packed row, i.e. ascending expert id.  Here one warp
// owns one token, walks that token's copies in the same ascending order and
// writes the row once: no atomics, no zero-fill pass, run-to-run identical.
//   F64 : acc = __dadd_rn(acc, __dmul_rn(w, y))  -> bit-exact to the reference
//   BF16: fp32 accumulation of bf16 rows, 16-byte vectors, bf16 out.
// An optional dense addend (the shared-expert output, weight 1.0) is added
// after the routed copies.  HBM-bound: bytes per token = (copies+1)*H*2 + H*2.
#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

constexpr int kCombWarps = 8;

// Copy list of token t: CSR (ptr/idx) or fixed-stride slots (-1 padded).
struct CopyList {
    const int32_t* ptr;   // [S+1] or null
    const int32_t* idx;   // CSR indices, or slot_pos [S,k]
    int k;                // slot stride when ptr == null
    // optional indirection: copy c lives at tab[drank[c]] row drow[c] (the
    // owners' grouped expert-output buffers) instead of rows[c]
    const char* const* tab;
    const int32_t* drank;
    const int32_t* drow;
    template <typename T>
    __device__ __forceinline__ const T* row(const T* rows, int c, int H) const {
        if (tab) return reinterpret_cast<const T*>(tab[drank[c]]) + static_cast<size_t>(drow[c]) * H;
        return rows + static_cast<size_t>(c) * H;
    }
    __device__ __forceinline__ int count(int t) const {
        if (ptr) return ptr[t + 1] - ptr[t];
        int c = 0;
        while (c < k && idx[static_cast<size_t>(t) * k + c] >= 0) ++c;
        return c;
    }
    __device__ __forceinline__ int at(int t, int j) const {
        return ptr ? idx[ptr[t] + j] : idx[static_cast<size_t>(t) * k + j];
    }
};

__global__ void __launch_bounds__(32 * kCombWarps) combine_f64_kernel(
    const double* __restrict__ rows, int H, CopyList cl, const double* __restrict__ w, int S,
    const double* __restrict__ addend, double* __restrict__ out) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= S) return;
    const int n = cl.count(t);
    for (int h = lane; h < H; h += 32) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) {
            const int c = cl.at(t, j);
            acc = __dadd_rn(acc, __dmul_rn(w[c], cl.row(rows, c, H)[h]));
        }
        if (addend) acc = __dadd_rn(acc, addend[static_cast<size_t>(t) * H + h]);
        out[static_cast<size_t>(t) * H + h] = acc;
    }
}

// BF16: each lane owns kV 16-byte chunks (8 bf16 each) of the row per pass.
template <int kV>
__global__ void __launch_bounds__(32 * kCombWarps) combine_bf16_kernel(
    const __nv_bfloat16* __restrict__ rows, int H, CopyList cl, const double* __restrict__ w,
    int S, const __nv_bfloat16* __restrict__ addend, __nv_bfloat16* __restrict__ out) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= S) return;
    const int nn = cl.count(t);
    const int nchunk = H >> 3;
    for (int c0 = 0; c0 < nchunk; c0 += 32 * kV) {
        float acc[kV][8];
#pragma unroll
        for (int v = 0; v < kV; ++v)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[v][q] = 0.f;
        for (int j = 0; j < nn; ++j) {
            const int cj = cl.at(t, j);  // warp-uniform
            const float wj = static_cast<float>(w[cj]);
            const int4* src = reinterpret_cast<const int4*>(cl.row(rows, cj, H));
            int4 r[kV];
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                const int c = c0 + lane + 32 * v;
                r[v] = c < nchunk ? ld_nc_v4(src + c) : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                const uint32_t u[4] = {static_cast<uint32_t>(r[v].x), static_cast<uint32_t>(r[v].y),
                                       static_cast<uint32_t>(r[v].z), static_cast<uint32_t>(r[v].w)};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[v][2 * q] = fmaf(wj, bf16_lo(u[q]), acc[v][2 * q]);
                    acc[v][2 * q + 1] = fmaf(wj, bf16_hi(u[q]), acc[v][2 * q + 1]);
                }
            }
        }
        if (addend) {
            const int4* src = reinterpret_cast<const int4*>(addend + static_cast<size_t>(t) * H);
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                const int c = c0 + lane + 32 * v;
                if (c >= nchunk) continue;
                const int4 r = ld_nc_v4(src + c);
                const uint32_t u[4] = {static_cast<uint32_t>(r.x), static_cast<uint32_t>(r.y),
                                       static_cast<uint32_t>(r.z), static_cast<uint32_t>(r.w)};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[v][2 * q] += bf16_lo(u[q]);
                    acc[v][2 * q + 1] += bf16_hi(u[q]);
                }
            }
        }
        int4* dst = reinterpret_cast<int4*>(out + static_cast<size_t>(t) * H);
#pragma unroll
        for (int v = 0; v < kV; ++v) {
            const int c = c0 + lane + 32 * v;
            if (c >= nchunk) continue;
            int4 o;
            o.x = static_cast<int>(pack_bf16(acc[v][0], acc[v][1]));
            o.y = static_cast<int>(pack_bf16(acc[v][2], acc[v][3]));
            o.z = static_cast<int>(pack_bf16(acc[v][4], acc[v][5]));
            o.w = static_cast<int>(pack_bf16(acc[v][6], acc[v][7]));
            st_na_v4(dst + c, o);
        }
    }
}

void launch_combine(int dtype, const void* rows, int H, const int32_t* ptr, const int32_t* idx,
                    int k, const double* w, int S, const void* addend, void* out,
                    cudaStream_t st, const char* const* tab, const int32_t* drank,
                    const int32_t* drow) {
    if (S == 0) return;
    CopyList cl{ptr, idx, k, tab, drank, drow};
    const int blocks = ceil_div(S, kCombWarps);
    if (dtype == XMOE_F64) {
        combine_f64_kernel<<<blocks, 32 * kCombWarps, 0, st>>>(
            static_cast<const double*>(rows), H, cl, w, S, static_cast<const double*>(addend),
            static_cast<double*>(out));
    } else {
        require(H % 8 == 0, XMOE_ERR_VALIDATION, "bf16 path requires model_dim % 8 == 0");
        combine_bf16_kernel<8><<<blocks, 32 * kCombWarps, 0, st>>>(
            static_cast<const __nv_bfloat16*>(rows), H, cl, w, S,
            static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out));
    }
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
