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
#include <algorithm>
#include <cstdlib>
#include <string>

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

template <typename T>
__global__ void __launch_bounds__(32 * kCombWarps) combine_simt_kernel(
    const T* __restrict__ rows, int H, CopyList cl, const double* __restrict__ w, int S,
    const T* __restrict__ addend, T* __restrict__ out) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= S) return;
    const int n = cl.count(t);
    for (int h = lane; h < H; h += 32) {  // F32: same order, fp64 accumulation, one rounding
        double acc = 0.0;
        for (int j = 0; j < n; ++j) {
            const int c = cl.at(t, j);
            acc = __dadd_rn(acc, __dmul_rn(w[c], static_cast<double>(cl.row(rows, c, H)[h])));
        }
        if (addend) acc = __dadd_rn(acc, static_cast<double>(addend[static_cast<size_t>(t) * H + h]));
        out[static_cast<size_t>(t) * H + h] = static_cast<T>(acc);
    }
}

// BF16: a warp owns one 512-column segment of one token (2 x 16-byte chunks
// per lane).  The copy list is fetched in one step (lane j loads copy j's
// index, weight and row address) and broadcast with shuffles, so each token
// pays two dependent memory latencies, and every copy's row loads are issued
// before any math (up to 2*kBatch 16-byte loads in flight per lane).
constexpr int kSegCols = 512;
constexpr int kBatch = 8;

__global__ void __launch_bounds__(32 * kCombWarps) combine_bf16_kernel(
    const __nv_bfloat16* __restrict__ rows, int H, CopyList cl, const double* __restrict__ w,
    int S, const __nv_bfloat16* __restrict__ addend, __nv_bfloat16* __restrict__ out) {
    const int nseg = (H + kSegCols - 1) / kSegCols;
    const int lane = threadIdx.x & 31;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
         gw < static_cast<long long>(S) * nseg; gw += nw) {
    const int t = static_cast<int>(gw / nseg);
    const int seg = static_cast<int>(gw % nseg);
    const int nchunk = H >> 3;
    const int seg_end = min(nchunk, (seg + 1) * (kSegCols / 8));
    const int c0 = seg * (kSegCols / 8) + lane;
    const int c1 = c0 + 32;
    const bool v0 = c0 < seg_end;
    const bool v1 = c1 < seg_end;
    float acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.f;
    // copy list, one entry per lane
    int n;
    int base = 0;
    if (cl.ptr) {
        base = cl.ptr[t];
        n = cl.ptr[t + 1] - base;
    } else {
        const int v = lane < cl.k ? cl.idx[static_cast<size_t>(t) * cl.k + lane] : -1;
        n = __popc(__ballot_sync(0xffffffffu, v >= 0));  // kept copies are a -1 padded prefix
    }
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        int cj = -1;
        float wv = 0.f;
        const int4* rp = nullptr;
        if (j < n) {
            cj = cl.ptr ? cl.idx[base + j] : cl.idx[static_cast<size_t>(t) * cl.k + j];
            wv = static_cast<float>(w[cj]);
            rp = reinterpret_cast<const int4*>(cl.row(rows, cj, H));
        }
        const int m = min(32, n - j0);
        for (int b0 = 0; b0 < m; b0 += kBatch) {
            int4 r[kBatch][2];
            float wj[kBatch];
#pragma unroll
            for (int b = 0; b < kBatch; ++b) {
                const int src_lane = b0 + b;
                const int4* p = reinterpret_cast<const int4*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rp), src_lane & 31));
                wj[b] = __shfl_sync(0xffffffffu, wv, src_lane & 31);
                if (src_lane < m) {
                    r[b][0] = v0 ? ld_nc_v4(p + c0) : make_int4(0, 0, 0, 0);
                    r[b][1] = v1 ? ld_nc_v4(p + c1) : make_int4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int b = 0; b < kBatch; ++b) {
                if (b0 + b < m) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t u[4] = {static_cast<uint32_t>(r[b][h].x), static_cast<uint32_t>(r[b][h].y),
                                               static_cast<uint32_t>(r[b][h].z), static_cast<uint32_t>(r[b][h].w)};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            acc[8 * h + 2 * q] = fmaf(wj[b], bf16_lo(u[q]), acc[8 * h + 2 * q]);
                            acc[8 * h + 2 * q + 1] = fmaf(wj[b], bf16_hi(u[q]), acc[8 * h + 2 * q + 1]);
                        }
                    }
                }
            }
        }
    }
    const int4* add = addend ? reinterpret_cast<const int4*>(addend + static_cast<size_t>(t) * H) : nullptr;
    int4* dst = reinterpret_cast<int4*>(out + static_cast<size_t>(t) * H);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = h ? c1 : c0;
        if (!(h ? v1 : v0)) continue;
        if (add) {
            const int4 a4 = ld_nc_v4(add + c);
            const uint32_t u[4] = {static_cast<uint32_t>(a4.x), static_cast<uint32_t>(a4.y),
                                   static_cast<uint32_t>(a4.z), static_cast<uint32_t>(a4.w)};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                acc[8 * h + 2 * q] += bf16_lo(u[q]);
                acc[8 * h + 2 * q + 1] += bf16_hi(u[q]);
            }
        }
        int4 o;
        o.x = static_cast<int>(pack_bf16(acc[8 * h + 0], acc[8 * h + 1]));
        o.y = static_cast<int>(pack_bf16(acc[8 * h + 2], acc[8 * h + 3]));
        o.z = static_cast<int>(pack_bf16(acc[8 * h + 4], acc[8 * h + 5]));
        o.w = static_cast<int>(pack_bf16(acc[8 * h + 6], acc[8 * h + 7]));
        st_na_v4(dst + c, o);
    }
    }
}

// BF16 combine over per-slot source addresses (written by the token-major
// scatter): lane j loads copy j's expert-output address and weight — the only
// dependent load before the rows stream.  One warp per (token, 512-column
// segment); rows may live in a peer GPU's memory (NVLink loads).
// partial mode (partial != null): the fp32 sums of the routed copies go to
// partial [S, H] and every (token, segment) item adds 1 to its 128-token
// block's counter ready[(t_base + t) / 128] (release) — the shared-expert
// GEMM2 epilogue finishes the rows (layer.cu, chunked forward).
template <int kWarps>
__global__ void __launch_bounds__(32 * kWarps) combine_slots_bf16_kernel(
    const unsigned long long* __restrict__ slot_src, const float* __restrict__ slot_w, int k, int H, int S,
    const __nv_bfloat16* __restrict__ addend, __nv_bfloat16* __restrict__ out, long long src_delta,
    const __nv_bfloat16* __restrict__ addend2, float* __restrict__ partial, unsigned* __restrict__ ready,
    int t_base) {
    const int nseg = (H + kSegCols - 1) / kSegCols;
    const int lane = threadIdx.x & 31;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
         gw < static_cast<long long>(S) * nseg; gw += nw) {
    const int t = static_cast<int>(gw / nseg);
    const int seg = static_cast<int>(gw % nseg);
    const int nchunk = H >> 3;
    const int seg_end = min(nchunk, (seg + 1) * (kSegCols / 8));
    const int c0 = seg * (kSegCols / 8) + lane;
    const int c1 = c0 + 32;
    const bool v0 = c0 < seg_end, v1 = c1 < seg_end;
    unsigned long long rp = 0;
    float wv = 0.f;
    if (lane < k) {
        rp = slot_src[static_cast<size_t>(t) * k + lane];
        wv = slot_w ? slot_w[static_cast<size_t>(t) * k + lane] : 1.f;
    }
    const int n = __popc(__ballot_sync(0xffffffffu, lane < k && rp != 0));  // kept copies: a prefix
    if (rp) rp += static_cast<unsigned long long>(src_delta);
    // addend issued early: independent of the slot chain
    int4 a4[2] = {make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0)};
    if (addend) {
        const int4* add = reinterpret_cast<const int4*>(addend + static_cast<size_t>(t) * H);
        if (v0) a4[0] = ld_nc_v4(add + c0);
        if (v1) a4[1] = ld_nc_v4(add + c1);
    }
    int4 b4[2] = {make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0)};
    if (addend2) {  // issued early too (the backward's dx adds two addends)
        const int4* add = reinterpret_cast<const int4*>(addend2 + static_cast<size_t>(t) * H);
        if (v0) b4[0] = ld_nc_v4(add + c0);
        if (v1) b4[1] = ld_nc_v4(add + c1);
    }
    float acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.f;
    for (int b0 = 0; b0 < n; b0 += kBatch) {
        int4 r[kBatch][2];
        float wj[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int4* p = reinterpret_cast<const int4*>(__shfl_sync(0xffffffffu, rp, (b0 + b) & 31));
            wj[b] = __shfl_sync(0xffffffffu, wv, (b0 + b) & 31);
            if (b0 + b < n) {
                r[b][0] = v0 ? ld_nc_v4(p + c0) : make_int4(0, 0, 0, 0);
                r[b][1] = v1 ? ld_nc_v4(p + c1) : make_int4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            if (b0 + b < n) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t u[4] = {static_cast<uint32_t>(r[b][h].x), static_cast<uint32_t>(r[b][h].y),
                                           static_cast<uint32_t>(r[b][h].z), static_cast<uint32_t>(r[b][h].w)};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        acc[8 * h + 2 * q] = fmaf(wj[b], bf16_lo(u[q]), acc[8 * h + 2 * q]);
                        acc[8 * h + 2 * q + 1] = fmaf(wj[b], bf16_hi(u[q]), acc[8 * h + 2 * q + 1]);
                    }
                }
            }
        }
    }
    if (partial) {
        float4* pd = reinterpret_cast<float4*>(partial + static_cast<size_t>(t) * H);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = h ? c1 : c0;
            if (!(h ? v1 : v0)) continue;
            pd[2 * c] = make_float4(acc[8 * h + 0], acc[8 * h + 1], acc[8 * h + 2], acc[8 * h + 3]);
            pd[2 * c + 1] = make_float4(acc[8 * h + 4], acc[8 * h + 5], acc[8 * h + 6], acc[8 * h + 7]);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(ready + ((t_base + t) >> 7), 1u);
        }
        continue;
    }
    int4* dst = reinterpret_cast<int4*>(out + static_cast<size_t>(t) * H);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = h ? c1 : c0;
        if (!(h ? v1 : v0)) continue;
        if (addend) {
            const uint32_t u[4] = {static_cast<uint32_t>(a4[h].x), static_cast<uint32_t>(a4[h].y),
                                   static_cast<uint32_t>(a4[h].z), static_cast<uint32_t>(a4[h].w)};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                acc[8 * h + 2 * q] += bf16_lo(u[q]);
                acc[8 * h + 2 * q + 1] += bf16_hi(u[q]);
            }
        }
        if (addend2) {
            const uint32_t u[4] = {static_cast<uint32_t>(b4[h].x), static_cast<uint32_t>(b4[h].y),
                                   static_cast<uint32_t>(b4[h].z), static_cast<uint32_t>(b4[h].w)};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                acc[8 * h + 2 * q] += bf16_lo(u[q]);
                acc[8 * h + 2 * q + 1] += bf16_hi(u[q]);
            }
        }
        int4 o;
        o.x = static_cast<int>(pack_bf16(acc[8 * h + 0], acc[8 * h + 1]));
        o.y = static_cast<int>(pack_bf16(acc[8 * h + 2], acc[8 * h + 3]));
        o.z = static_cast<int>(pack_bf16(acc[8 * h + 4], acc[8 * h + 5]));
        o.w = static_cast<int>(pack_bf16(acc[8 * h + 6], acc[8 * h + 7]));
        st_na_v4(dst + c, o);
    }
    }
}

// One CTA per token (default on a full grid): every copy's whole row is
// read contiguously by the CTA (thread i owns 16-byte chunk i), the k loads
// of a thread issued together, the slot list fetched once per token into
// shared memory.  Same fp32 accumulation order per element as the warp
// kernel (copies ascending, then the addends), so the output is identical.
constexpr int kCtaThreads = 256;
__global__ void __launch_bounds__(kCtaThreads, 4) combine_rows_cta_kernel(
    const unsigned long long* __restrict__ slot_src, const float* __restrict__ slot_w, int k, int H, int S,
    const __nv_bfloat16* __restrict__ addend, __nv_bfloat16* __restrict__ out, long long src_delta,
    const __nv_bfloat16* __restrict__ addend2, float* __restrict__ partial, unsigned* __restrict__ ready) {
    __shared__ unsigned long long sp[2][32];
    __shared__ float sw[2][32];
    __shared__ int sn[2];
    __shared__ int st_next[2];
    const int nchunk = H >> 3;
    int buf = 0;
    // partial mode: tokens are taken from a device counter (ready[ceil(S/128)])
    // so any resident CTA advances every 128-token block — the consuming GEMM
    // may hold the SMs some CTAs of this grid would need
    unsigned* next = partial ? ready + ((S + 127) >> 7) : nullptr;
    int t = blockIdx.x;
    if (next) {
        if (threadIdx.x == 0) st_next[0] = static_cast<int>(atomicAdd(next, 1u));
        __syncthreads();
        t = st_next[0];
    }
    for (; t < S; buf ^= 1) {
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            unsigned long long rp = 0;
            float wv = 0.f;
            if (lane < k) {
                rp = slot_src[static_cast<size_t>(t) * k + lane];
                wv = slot_w ? slot_w[static_cast<size_t>(t) * k + lane] : 1.f;
            }
            const int n = __popc(__ballot_sync(0xffffffffu, lane < k && rp != 0));
            sp[buf][lane] = rp ? rp + static_cast<unsigned long long>(src_delta) : 0ull;
            sw[buf][lane] = wv;
            if (lane == 0) sn[buf] = n;
        }
        __syncthreads();  // double-buffered: token t+1's list goes to the other half
        const int n = sn[buf];
        for (int c = threadIdx.x; c < nchunk; c += blockDim.x) {
            int4 a4 = make_int4(0, 0, 0, 0), b4 = make_int4(0, 0, 0, 0);
            if (addend) a4 = ld_nc_v4(reinterpret_cast<const int4*>(addend + static_cast<size_t>(t) * H) + c);
            if (addend2) b4 = ld_nc_v4(reinterpret_cast<const int4*>(addend2 + static_cast<size_t>(t) * H) + c);
            float acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = 0.f;
            for (int j0 = 0; j0 < n; j0 += kBatch) {
                int4 r[kBatch];
#pragma unroll
                for (int b = 0; b < kBatch; ++b)
                    if (j0 + b < n) r[b] = ld_nc_v4(reinterpret_cast<const int4*>(sp[buf][j0 + b]) + c);
#pragma unroll
                for (int b = 0; b < kBatch; ++b) {
                    if (j0 + b >= n) break;
                    const float wj = sw[buf][j0 + b];
                    const uint32_t u[4] = {static_cast<uint32_t>(r[b].x), static_cast<uint32_t>(r[b].y),
                                           static_cast<uint32_t>(r[b].z), static_cast<uint32_t>(r[b].w)};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        acc[2 * q] = fmaf(wj, bf16_lo(u[q]), acc[2 * q]);
                        acc[2 * q + 1] = fmaf(wj, bf16_hi(u[q]), acc[2 * q + 1]);
                    }
                }
            }
            if (addend) {
                const uint32_t u[4] = {static_cast<uint32_t>(a4.x), static_cast<uint32_t>(a4.y),
                                       static_cast<uint32_t>(a4.z), static_cast<uint32_t>(a4.w)};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[2 * q] += bf16_lo(u[q]);
                    acc[2 * q + 1] += bf16_hi(u[q]);
                }
            }
            if (addend2) {
                const uint32_t u[4] = {static_cast<uint32_t>(b4.x), static_cast<uint32_t>(b4.y),
                                       static_cast<uint32_t>(b4.z), static_cast<uint32_t>(b4.w)};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[2 * q] += bf16_lo(u[q]);
                    acc[2 * q + 1] += bf16_hi(u[q]);
                }
            }
            if (partial) {  // fp32 sums of the routed copies; the shared GEMM2 epilogue finishes the row
                float4* pd = reinterpret_cast<float4*>(partial + static_cast<size_t>(t) * H) + 2 * c;
                pd[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                pd[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
                continue;
            }
            int4 o;
            o.x = static_cast<int>(pack_bf16(acc[0], acc[1]));
            o.y = static_cast<int>(pack_bf16(acc[2], acc[3]));
            o.z = static_cast<int>(pack_bf16(acc[4], acc[5]));
            o.w = static_cast<int>(pack_bf16(acc[6], acc[7]));
            st_na_v4(reinterpret_cast<int4*>(out + static_cast<size_t>(t) * H) + c, o);
        }
        if (partial) {  // publish token t: its 128-row block's counter (release), take the next token
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(ready + (t >> 7), 1u);
                st_next[buf ^ 1] = static_cast<int>(atomicAdd(next, 1u));
            }
            __syncthreads();
            t = st_next[buf ^ 1];
        } else {
            t += gridDim.x;
        }
    }
}

// CTA-per-token variant on a full grid (measured on B200, C2 N=1: combine
// 0.104-0.118 -> 0.097 ms, 0.70-0.79 -> 0.85 of HBM); the warp kernel when the
// grid is capped to run beside GEMMs (chunked forward: its per-warp items keep
// more rows in flight per block there; the CTA variant measured 40 -> 32 M
// tokens/s at N=4).  XMOE_COMBINE=warp|cta forces one (A/B).
static int combine_variant() {
    static const int v = [] {
        const char* e = std::getenv("XMOE_COMBINE");
        if (e && std::string(e) == "cta") return 1;
        if (e && std::string(e) == "warp") return 2;
        return 0;
    }();
    return v == 0 ? (g_copy_blocks == 0 ? 1 : 0) : (v == 1 ? 1 : 0);
}

void launch_combine_slots(const unsigned long long* slot_src, const float* slot_w, int k, int H, int S,
                          const void* addend, void* out, cudaStream_t st, long long src_delta, const void* addend2) {
    if (S == 0) return;
    require(H % 8 == 0 && k <= 32, XMOE_ERR_VALIDATION, "slot combine needs model_dim % 8 == 0, k <= 32");
    if (combine_variant() == 1) {
        int blocks = S < 8 * kNumSMs ? S : 8 * kNumSMs;
        if (g_copy_blocks > 0 && blocks > g_copy_blocks) blocks = g_copy_blocks;
        combine_rows_cta_kernel<<<blocks, kCtaThreads, g_copy_smem, st>>>(
            slot_src, slot_w, k, H, S, static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out),
            src_delta, static_cast<const __nv_bfloat16*>(addend2), nullptr, nullptr);
        XMOE_LAUNCH_CHECK();
        return;
    }
    const long long warps = static_cast<long long>(S) * ((H + kSegCols - 1) / kSegCols);
    if (g_copy_fat > 0) {  // whole-SM blocks: 16 warps x 128 registers fill an SM's register file
        combine_slots_bf16_kernel<16><<<g_copy_fat, 32 * 16, 0, st>>>(
            slot_src, slot_w, k, H, S, static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out),
            src_delta, static_cast<const __nv_bfloat16*>(addend2), nullptr, nullptr, 0);
        XMOE_LAUNCH_CHECK();
        return;
    }
    long long blocks = ceil_div(warps, kCombWarps);
    if (g_copy_blocks > 0 && blocks > g_copy_blocks) blocks = g_copy_blocks;
    combine_slots_bf16_kernel<kCombWarps><<<static_cast<int>(blocks), 32 * kCombWarps, g_copy_smem, st>>>(
        slot_src, slot_w, k, H, S, static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out),
        src_delta, static_cast<const __nv_bfloat16*>(addend2), nullptr, nullptr, 0);
    XMOE_LAUNCH_CHECK();
}

int combine_segments(int H) { return (H + kSegCols - 1) / kSegCols; }

void launch_combine_slots_seg_partial(const unsigned long long* slot_src, const float* slot_w, int k, int H, int S,
                                      float* partial, unsigned* ready, int t_base, cudaStream_t st) {
    if (S == 0) return;
    require(H % 8 == 0 && k <= 32, XMOE_ERR_VALIDATION, "slot combine needs model_dim % 8 == 0, k <= 32");
    if (g_copy_fat > 0) {
        combine_slots_bf16_kernel<16><<<g_copy_fat, 32 * 16, 0, st>>>(slot_src, slot_w, k, H, S, nullptr, nullptr, 0,
                                                                      nullptr, partial, ready, t_base);
        XMOE_LAUNCH_CHECK();
        return;
    }
    const long long warps = static_cast<long long>(S) * combine_segments(H);
    long long blocks = ceil_div(warps, kCombWarps);
    if (g_copy_blocks > 0 && blocks > g_copy_blocks) blocks = g_copy_blocks;
    combine_slots_bf16_kernel<kCombWarps><<<static_cast<int>(blocks), 32 * kCombWarps, 0, st>>>(
        slot_src, slot_w, k, H, S, nullptr, nullptr, 0, nullptr, partial, ready, t_base);
    XMOE_LAUNCH_CHECK();
}

void launch_combine_slots_partial(const unsigned long long* slot_src, const float* slot_w, int k, int H, int S,
                                  float* partial, unsigned* ready, cudaStream_t st) {
    if (S == 0) return;
    require(H % 8 == 0 && k <= 32, XMOE_ERR_VALIDATION, "slot combine needs model_dim % 8 == 0, k <= 32");
    // Launched BEFORE the GEMM that consumes it (that GEMM waits on the ready
    // counters, so it must never hold SMs the combine cannot share): one CTA
    // per SM by default (XMOE_LATE_GRID), preferring the maximum shared-memory
    // carveout so a 2-CTA GEMM CTA (223 KB) still fits beside it.
    static const int grid_cap = [] {
        const char* e = std::getenv("XMOE_LATE_GRID");
        return e ? std::max(1, std::atoi(e)) : kNumSMs;
    }();
    static bool attr = false;
    if (!attr) {
        XMOE_CUDA(cudaFuncSetAttribute(combine_rows_cta_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       static_cast<int>(cudaSharedmemCarveoutMaxShared)));
        attr = true;
    }
    const int blocks = S < grid_cap ? S : grid_cap;
    combine_rows_cta_kernel<<<blocks, kCtaThreads, 0, st>>>(slot_src, slot_w, k, H, S, nullptr, nullptr, 0, nullptr,
                                                           partial, ready);
    XMOE_LAUNCH_CHECK();
}

void launch_combine(int dtype, const void* rows, int H, const int32_t* ptr, const int32_t* idx,
                    int k, const double* w, int S, const void* addend, void* out,
                    cudaStream_t st, const char* const* tab, const int32_t* drank,
                    const int32_t* drow) {
    if (S == 0) return;
    CopyList cl{ptr, idx, k, tab, drank, drow};
    const int blocks = ceil_div(S, kCombWarps);
    if (dtype == XMOE_F64) {
        combine_simt_kernel<double><<<blocks, 32 * kCombWarps, 0, st>>>(
            static_cast<const double*>(rows), H, cl, w, S, static_cast<const double*>(addend),
            static_cast<double*>(out));
    } else if (dtype == XMOE_F32) {
        combine_simt_kernel<float><<<blocks, 32 * kCombWarps, 0, st>>>(
            static_cast<const float*>(rows), H, cl, w, S, static_cast<const float*>(addend),
            static_cast<float*>(out));
    } else {
        require(H % 8 == 0, XMOE_ERR_VALIDATION, "bf16 path requires model_dim % 8 == 0");
        const long long warps = static_cast<long long>(S) * ((H + kSegCols - 1) / kSegCols);
        combine_bf16_kernel<<<ceil_div(warps, kCombWarps), 32 * kCombWarps, 0, st>>>(
            static_cast<const __nv_bfloat16*>(rows), H, cl, w, S,
            static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out));
    }
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
