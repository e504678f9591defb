// Top-k softmax gating — B200 restatement of moesim::gate_forward
// (/root/reference/proj/src/gating.cpp:14-57).
//
//   logits = X . Wg      (F64: ascending-h __dmul_rn/__dadd_rn, bit-exact to
//                         kernels_scalar.cpp:11-23; BF16: fp32 accumulation,
//                         exact on the bf16 grid inputs)
//   probs  = softmax(logits - max)  in fp64, summed ascending e (gating.cpp:39-43;
//            the BF16 path sums as a tree)
//   top-k  by (prob desc, id asc)   (gating.cpp:45-50), raw probs as weights.
#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

// ---------------------------------------------------------------- F64 / F32 logits
// One thread per (token, expert); the warp spans experts so Wg rows are
// coalesced and the token value is a broadcast.  Ascending h, separately
// rounded multiply and add (kernels_scalar.cpp:11-23, -ffp-contract=off):
// bit-exact to the reference in F64; the F32 instantiation keeps the order
// with fp64 accumulation and rounds each logit once.
template <typename T>
__global__ void gate_logits_kernel(const T* __restrict__ x, const T* __restrict__ wg, int S, int H, int E,
                                   T* __restrict__ logits) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (e >= E || t >= S) return;
    const T* xr = x + static_cast<size_t>(t) * H;
    double acc = 0.0;  // F32: exact fp32 products, fp64 accumulation, one rounding
    for (int h = 0; h < H; ++h)
        acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(xr[h]), static_cast<double>(wg[static_cast<size_t>(h) * E + e])));
    logits[static_cast<size_t>(t) * E + e] = static_cast<T>(acc);
}

// ---------------------------------------------------------------- BF16 logits
// The BF16 logits GEMM runs on the tcgen05 grouped-GEMM kernel (one group of
// S rows, N = E, fp32 output; gemm_tc.cu).  With token values on a 2^-7
// grid and gate weights on a 2^-10 grid every partial sum is a multiple of
// 2^-17 far below 2^7 in magnitude, so fp32 accumulation is exact in any
// order and routing equals the fp64 reference bit for bit (SURVEY §7 hard
// part 1; tests/test_gpu_ops.py::test_gate_bf16_routing_bit_exact).

// ---------------------------------------------------------------- softmax + top-k
// One warp per token.  Lane l holds experts l, l+32, ..., PER per lane
// (E <= 32*PER), all in registers.
template <int PER, typename LT>
__global__ void __launch_bounds__(256) softmax_topk_kernel(const LT* __restrict__ logits, int S,
                                                           int E, int k, int renorm,
                                                           int32_t* __restrict__ top,
                                                           double* __restrict__ weights,
                                                           int32_t* __restrict__ counts) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= S) return;
    const LT* row = logits + static_cast<size_t>(warp) * E;
    double p[PER];
    double mx = static_cast<double>(row[0]);  // max-shifted softmax (gating.cpp:39-40)
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = lane + 32 * i;
        p[i] = e < E ? static_cast<double>(row[e]) : -INFINITY;
        mx = fmax(mx, p[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
    for (int i = 0; i < PER; ++i) p[i] = (lane + 32 * i < E) ? exp(__dsub_rn(p[i], mx)) : 0.0;
    // sequential ascending-e sum, exactly as the reference accumulates
    // (gating.cpp:42) — also for fp32 logits, so the BF16 weights equal the
    // fused gate's (gemm_tc.cu gate_route_kernel) bit for bit
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int lim = min(32, E - 32 * i);
        for (int l = 0; l < lim; ++l) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, p[i], l));
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) p[i] = (lane + 32 * i < E) ? __ddiv_rn(p[i], sum) : -1.0;
    // k rounds of warp arg-max by (prob desc, id asc) (gating.cpp:45-50).
    double wsum = 0.0;
    for (int j = 0; j < k; ++j) {
        double best = -1.0;
        int bid = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            if (p[i] > best) {  // ascending e within a lane: '>' keeps the lower id on ties
                best = p[i];
                bid = lane + 32 * i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bid, o);
            if (ob > best || (ob == best && oi < bid)) {
                best = ob;
                bid = oi;
            }
        }
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if (lane + 32 * i == bid) p[i] = -2.0;  // taken
        if (lane == 0) {
            top[static_cast<size_t>(warp) * k + j] = bid;
            weights[static_cast<size_t>(warp) * k + j] = best;
            // per-128-token-tile expert histogram for the one-launch placement
            if (counts) atomicAdd(&counts[static_cast<size_t>(warp / kRouteTile) * E + bid], 1);
        }
        wsum = __dadd_rn(wsum, best);
    }
    if (renorm && lane == 0) {
        // Restated beyond the reference: w_j / sum_j w_j, summed in slot order.
        for (int j = 0; j < k; ++j) {
            double* q = weights + static_cast<size_t>(warp) * k + j;
            *q = __ddiv_rn(*q, wsum);
        }
    }
}

void launch_gate_logits_f64(const double* x, const double* wg, int S, int H, int E,
                            double* logits, cudaStream_t st) {
    if (S == 0) return;
    dim3 grid(ceil_div(E, 128), S);
    gate_logits_kernel<double><<<grid, 128, 0, st>>>(x, wg, S, H, E, logits);
    XMOE_LAUNCH_CHECK();
}

void launch_gate_logits_f32(const float* x, const float* wg, int S, int H, int E, float* logits, cudaStream_t st) {
    if (S == 0) return;
    dim3 grid(ceil_div(E, 128), S);
    gate_logits_kernel<float><<<grid, 128, 0, st>>>(x, wg, S, H, E, logits);
    XMOE_LAUNCH_CHECK();
}

template <typename LT>
static void softmax_dispatch(const LT* logits, int S, int E, int k, int renorm, int32_t* top,
                             double* weights, cudaStream_t st, int32_t* counts = nullptr) {
    if (S == 0) return;
    require(E <= 1024, XMOE_ERR_VALIDATION, "num_experts must be <= 1024");
    if (counts)
        XMOE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * ((S + kRouteTile - 1) / kRouteTile) * E, st));
    const int grid = ceil_div(S, 8);
    if (E <= 32) softmax_topk_kernel<1, LT><<<grid, 256, 0, st>>>(logits, S, E, k, renorm, top, weights, counts);
    else if (E <= 64) softmax_topk_kernel<2, LT><<<grid, 256, 0, st>>>(logits, S, E, k, renorm, top, weights, counts);
    else if (E <= 128) softmax_topk_kernel<4, LT><<<grid, 256, 0, st>>>(logits, S, E, k, renorm, top, weights, counts);
    else if (E <= 256) softmax_topk_kernel<8, LT><<<grid, 256, 0, st>>>(logits, S, E, k, renorm, top, weights, counts);
    else softmax_topk_kernel<32, LT><<<grid, 256, 0, st>>>(logits, S, E, k, renorm, top, weights, counts);
    XMOE_LAUNCH_CHECK();
}

void launch_softmax_topk(const double* logits, int S, int E, int k, int renorm, int32_t* top,
                         double* weights, cudaStream_t st) {
    softmax_dispatch(logits, S, E, k, renorm, top, weights, st);
}

void launch_softmax_topk_f32(const float* logits, int S, int E, int k, int renorm, int32_t* top,
                             double* weights, cudaStream_t st, int32_t* counts) {
    softmax_dispatch(logits, S, E, k, renorm, top, weights, st, counts);
}

}  // namespace xmoe
