// Top-k softmax gating — B200 restatement of moesim::gate_forward
// (/root/reference/proj/src/gating.cpp:14-57).
//
//   logits = X . Wg      (F64: ascending-h __dmul_rn/__dadd_rn, bit-exact to
//                         kernels_scalar.cpp:11-23; BF16: fp32 accumulation,
//                         exact on the bf16 grid inputs)
//   probs  = softmax(logits - max)  in fp64, summed ascending e (gating.cpp:39-43)
//   top-k  by (prob desc, id asc)   (gating.cpp:45-50), raw probs as weights.
#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

// ---------------------------------------------------------------- F64 logits
// One thread per (token, expert); the warp spans experts so Wg rows are
// coalesced and the token value is a broadcast.
__global__ void gate_logits_f64_kernel(const double* __restrict__ x,
                                       const double* __restrict__ wg, int S, int H, int E,
                                       double* __restrict__ logits) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (e >= E || t >= S) return;
    const double* xr = x + static_cast<size_t>(t) * H;
    double acc = 0.0;
    for (int h = 0; h < H; ++h) acc = __dadd_rn(acc, __dmul_rn(xr[h], wg[static_cast<size_t>(h) * E + e]));
    logits[static_cast<size_t>(t) * E + e] = acc;
}

// ---------------------------------------------------------------- BF16 logits
// Register-tiled fp32 GEMM on CUDA cores: each CTA computes 64 tokens x 64
// experts, each thread 4x4, K staged through shared memory 32 at a time.
// With token values on a 2^-7 grid and gate weights on a 2^-10 grid every
// partial sum is a multiple of 2^-17 below 2^7 in magnitude, so fp32
// accumulation is exact in any order (SURVEY §7 hard part 1).
constexpr int kGT = 64, kGE = 64, kGK = 32;

__global__ void __launch_bounds__(256) gate_logits_bf16_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wgt, int S, int H,
    int E, double* __restrict__ logits) {
    __shared__ float xs[kGK][kGT + 4];
    __shared__ float ws[kGK][kGE + 4];
    const int t0 = blockIdx.x * kGT;
    const int e0 = blockIdx.y * kGE;
    const int tx = threadIdx.x % 16;  // expert group
    const int ty = threadIdx.x / 16;  // token group
    float acc[4][4] = {};
    for (int k0 = 0; k0 < H; k0 += kGK) {
        // 64 rows x 32 k for both operands: 2048 elements, 8 per thread
        for (int i = threadIdx.x; i < kGT * kGK; i += 256) {
            const int r = i / kGK, c = i % kGK;
            const int t = t0 + r, e = e0 + r, kk = k0 + c;
            xs[c][r] = (t < S && kk < H) ? __bfloat162float(x[static_cast<size_t>(t) * H + kk]) : 0.f;
            ws[c][r] = (e < E && kk < H) ? __bfloat162float(wgt[static_cast<size_t>(e) * H + kk]) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int c = 0; c < kGK; ++c) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = xs[c][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = ws[c][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int t = t0 + ty * 4 + i, e = e0 + tx * 4 + j;
            if (t < S && e < E) logits[static_cast<size_t>(t) * E + e] = static_cast<double>(acc[i][j]);
        }
}

// ---------------------------------------------------------------- softmax + top-k
// One warp per token.  Lane l holds experts l, l+32, ... (E <= 32*kMaxPerLane).
constexpr int kMaxPerLane = 32;  // E <= 1024

__global__ void softmax_topk_kernel(const double* __restrict__ logits, int S, int E, int k,
                                    int renorm, int32_t* __restrict__ top,
                                    double* __restrict__ weights) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= S) return;
    const double* row = logits + static_cast<size_t>(warp) * E;
    const int per = (E + 31) / 32;
    double p[kMaxPerLane];
    double mx = row[0];  // max-shifted softmax (gating.cpp:39-40); max is order-free
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
        const int e = lane + 32 * i;
        if (i < per && e < E) {
            p[i] = row[e];
            mx = fmax(mx, p[i]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
        const int e = lane + 32 * i;
        if (i < per && e < E) p[i] = exp(__dsub_rn(p[i], mx));
    }
    // Sequential ascending-e sum, as the reference accumulates (gating.cpp:42).
    double sum = 0.0;
    for (int i = 0; i < per; ++i) {
        for (int l = 0; l < 32; ++l) {
            const double v = __shfl_sync(0xffffffffu, p[i < kMaxPerLane ? i : 0], l);
            if (l + 32 * i < E) sum = __dadd_rn(sum, v);
        }
    }
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
        const int e = lane + 32 * i;
        if (i < per && e < E) p[i] = __ddiv_rn(p[i], sum);
    }
    // k rounds of warp arg-max by (prob desc, id asc), ties -> lower id.
    unsigned taken[(kMaxPerLane + 31) / 32] = {};
    double wsum = 0.0;
    double wsel[16];
    for (int j = 0; j < k; ++j) {
        double best = -1.0;
        int bid = 0x7fffffff;
        for (int i = 0; i < per; ++i) {
            const int e = lane + 32 * i;
            if (e < E && !((taken[i / 32] >> (i % 32)) & 1u)) {
                if (p[i] > best || (p[i] == best && e < bid)) {
                    best = p[i];
                    bid = e;
                }
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
        if ((bid & 31) == lane) {
            const int i = bid / 32;
            taken[i / 32] |= 1u << (i % 32);
        }
        if (lane == 0) {
            top[static_cast<size_t>(warp) * k + j] = bid;
            weights[static_cast<size_t>(warp) * k + j] = best;
        }
        if (j < 16) wsel[j] = best;
        wsum = __dadd_rn(wsum, best);
    }
    if (renorm && lane == 0) {
        // Restated beyond the reference: w_j / sum_j w_j, summed in slot order.
        for (int j = 0; j < k; ++j) {
            const double v = j < 16 ? wsel[j] : weights[static_cast<size_t>(warp) * k + j];
            weights[static_cast<size_t>(warp) * k + j] = __ddiv_rn(v, wsum);
        }
    }
}

void launch_gate_logits_f64(const double* x, const double* wg, int S, int H, int E,
                            double* logits, cudaStream_t st) {
    if (S == 0) return;
    dim3 grid(ceil_div(E, 128), S);
    gate_logits_f64_kernel<<<grid, 128, 0, st>>>(x, wg, S, H, E, logits);
    XMOE_LAUNCH_CHECK();
}

void launch_gate_logits_bf16(const __nv_bfloat16* x, const __nv_bfloat16* wgt, int S, int H,
                             int E, double* logits, cudaStream_t st) {
    if (S == 0) return;
    dim3 grid(ceil_div(S, kGT), ceil_div(E, kGE));
    gate_logits_bf16_kernel<<<grid, 256, 0, st>>>(x, wgt, S, H, E, logits);
    XMOE_LAUNCH_CHECK();
}

void launch_softmax_topk(const double* logits, int S, int E, int k, int renorm, int32_t* top,
                         double* weights, cudaStream_t st) {
    if (S == 0) return;
    require(E <= 32 * kMaxPerLane, XMOE_ERR_VALIDATION, "num_experts must be <= 1024");
    const int warps_per_block = 8;
    softmax_topk_kernel<<<ceil_div(S, warps_per_block), 32 * warps_per_block, 0, st>>>(
        logits, S, E, k, renorm, top, weights);
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
