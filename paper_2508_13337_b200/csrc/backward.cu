// Backward of the MoE block (the reference is
// forward-only, SPEC.md:15 — gradients are restated):
//
//   y_t = sum_c w_c E_e(x_t) + shared(x_t),   E_e(x) = relu(x W1_e) W2_e,
//   w = softmax(x Wg)[selected]  (raw probabilities, gating.cpp:39-54)
//
// Kernels here are the memory-bound pieces; the contractions run on the
// tcgen05 grouped GEMM (dgrad: grouped-M with a ReLU-mask epilogue; wgrad:
// grouped-K over zero-padded, transposed activations).
#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

// Owner side, one warp per grouped row r (all local experts):
//   dw_c = <dy_t, y_c>          -> the copy's home slot (peer store)
//   dz_r = w_c * dy_t  (bf16)   -> input of the expert dgrad GEMMs
__global__ void __launch_bounds__(256) bwd_owner_prep_kernel(
    const __nv_bfloat16* __restrict__ dyg, const __nv_bfloat16* __restrict__ eout, const float* __restrict__ gw,
    const unsigned long long* __restrict__ gsrc, const int32_t* __restrict__ rpe, int El, int H,
    float* const* __restrict__ slotdw_tab, __nv_bfloat16* __restrict__ dz, int me) {
    int rows = 0;
    for (int i = 0; i < El; ++i) rows += rpe[i];
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const int nvec = H >> 3;
    for (long long r = warp; r < rows; r += nwarps) {
        const unsigned long long s = gsrc[r];
        if (static_cast<int>(s >> 32) == me) continue;  // finished by bwd_scatter_dy_kernel at the source
        const int4* a = reinterpret_cast<const int4*>(dyg + static_cast<size_t>(r) * H);
        const int4* b = reinterpret_cast<const int4*>(eout + static_cast<size_t>(r) * H);
        int4* o = reinterpret_cast<int4*>(dz + static_cast<size_t>(r) * H);
        const float w = gw[r];
        float dot = 0.f;
        for (int v = lane; v < nvec; v += 32) {
            const int4 av = ld_nc_v4(a + v), bv = ld_nc_v4(b + v);
            const uint32_t ua[4] = {static_cast<uint32_t>(av.x), static_cast<uint32_t>(av.y),
                                    static_cast<uint32_t>(av.z), static_cast<uint32_t>(av.w)};
            const uint32_t ub[4] = {static_cast<uint32_t>(bv.x), static_cast<uint32_t>(bv.y),
                                    static_cast<uint32_t>(bv.z), static_cast<uint32_t>(bv.w)};
            int4 ov;
            uint32_t uo[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                dot = fmaf(bf16_lo(ua[q]), bf16_lo(ub[q]), dot);
                dot = fmaf(bf16_hi(ua[q]), bf16_hi(ub[q]), dot);
                uo[q] = pack_bf16(w * bf16_lo(ua[q]), w * bf16_hi(ua[q]));
            }
            ov.x = static_cast<int>(uo[0]);
            ov.y = static_cast<int>(uo[1]);
            ov.z = static_cast<int>(uo[2]);
            ov.w = static_cast<int>(uo[3]);
            st_na_v4(o + v, ov);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        if (lane == 0) slotdw_tab[s >> 32][static_cast<uint32_t>(s)] = dot;
    }
    __threadfence_system();
}

// B1 + B2 fused, token side, one warp per token (bf16 rows, H % 8 == 0):
// dy_t is read once; for every kept copy c of t
//   * owned by this rank: dw_c = <dy_t, y_c> (y_c read from the local expert
//     output) goes straight to the home slot, and dz = w_c * dy_t is written
//     into the grouped dz buffer — the owner-side pass never sees the row;
//   * owned by a peer: dy_t goes to the peer's grouped dy buffer with the
//     copy's weight and home slot, for bwd_owner_prep_kernel over there.
// The dot product uses the owner-side pass's per-lane order (ascending 16 B
// chunks, lo/hi halves, then the xor-shuffle tree), so both give the same
// bits.  Algorithmic bytes at W = 1: dy once, y and dz once per copy.
constexpr int kBsVec = 8;  // int4 per lane per pass (4 KB rows in one pass)

__global__ void __launch_bounds__(512) bwd_scatter_dy_kernel(
    const char* __restrict__ dy, int H, int S, int k, const int32_t* __restrict__ slot_pos,
    const int32_t* __restrict__ dest_rank, const int32_t* __restrict__ dest_row, const double* __restrict__ cw,
    int me, char* __restrict__ dz, char* const* __restrict__ eout_tab, char* const* __restrict__ dyg_tab,
    char* const* __restrict__ dxc_tab, float* const* __restrict__ gw_tab,
    unsigned long long* const* __restrict__ gsrc_tab, float* __restrict__ slot_dw,
    unsigned long long* __restrict__ bslot_src) {
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const size_t rb = static_cast<size_t>(H) * 2;
    const int nvec = H >> 3;
    const bool one_pass = nvec <= 32 * kBsVec;
    for (long long t = warp; t < S; t += nwarps) {
        const int4* src = reinterpret_cast<const int4*>(dy + static_cast<size_t>(t) * rb);
        int4 v[kBsVec];
#pragma unroll
        for (int u = 0; u < kBsVec; ++u) {
            const int c = lane + 32 * u;
            v[u] = c < nvec ? ld_nc_v4(src + c) : make_int4(0, 0, 0, 0);
        }
        int p = -1, r = -1, row = 0;
        float wv = 0.f;
        if (lane < k) {
            p = slot_pos[static_cast<size_t>(t) * k + lane];
            if (p >= 0) {
                r = dest_rank[p];
                row = dest_row[p];
                wv = static_cast<float>(cw[p]);
                // home slot at the owner (rank == me tells its pass to skip the row)
                gsrc_tab[r][row] = (static_cast<unsigned long long>(me) << 32) | static_cast<unsigned>(t * k + lane);
                if (r != me) gw_tab[r][row] = wv;  // the owner finishes this copy (bwd_owner_prep_kernel)
            }
            bslot_src[static_cast<size_t>(t) * k + lane] =
                p >= 0 ? reinterpret_cast<unsigned long long>(dxc_tab[r] + static_cast<size_t>(row) * rb) : 0ull;
        }
        const int n = __popc(__ballot_sync(0xffffffffu, lane < k && p >= 0));  // kept copies: a prefix
        for (int j = 0; j < n; ++j) {
            const int rj = __shfl_sync(0xffffffffu, r, j);
            const size_t off = static_cast<size_t>(__shfl_sync(0xffffffffu, row, j)) * rb;
            if (rj == me) {
                const float w = __shfl_sync(0xffffffffu, wv, j);
                const int4* y = reinterpret_cast<const int4*>(eout_tab[me] + off);
                int4* o = reinterpret_cast<int4*>(dz + off);
                float dot = 0.f;
                for (int base = 0; base < nvec; base += 32 * kBsVec) {
                    int4 e[kBsVec];
#pragma unroll
                    for (int u = 0; u < kBsVec; ++u) {
                        const int c = base + lane + 32 * u;
                        if (!one_pass) v[u] = c < nvec ? ld_nc_v4(src + c) : make_int4(0, 0, 0, 0);
                        e[u] = c < nvec ? ld_nc_v4(y + c) : make_int4(0, 0, 0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < kBsVec; ++u) {
                        const int c = base + lane + 32 * u;
                        if (c >= nvec) continue;
                        const uint32_t ua[4] = {static_cast<uint32_t>(v[u].x), static_cast<uint32_t>(v[u].y),
                                                static_cast<uint32_t>(v[u].z), static_cast<uint32_t>(v[u].w)};
                        const uint32_t ub[4] = {static_cast<uint32_t>(e[u].x), static_cast<uint32_t>(e[u].y),
                                                static_cast<uint32_t>(e[u].z), static_cast<uint32_t>(e[u].w)};
                        uint32_t uo[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            dot = fmaf(bf16_lo(ua[q]), bf16_lo(ub[q]), dot);
                            dot = fmaf(bf16_hi(ua[q]), bf16_hi(ub[q]), dot);
                            uo[q] = pack_bf16(w * bf16_lo(ua[q]), w * bf16_hi(ua[q]));
                        }
                        st_na_v4(o + c, make_int4(static_cast<int>(uo[0]), static_cast<int>(uo[1]),
                                                  static_cast<int>(uo[2]), static_cast<int>(uo[3])));
                    }
                }
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, s);
                if (lane == 0) slot_dw[static_cast<size_t>(t) * k + j] = dot;
            } else {
                int4* d = reinterpret_cast<int4*>(dyg_tab[rj] + off);
                for (int base = 0; base < nvec; base += 32 * kBsVec) {
#pragma unroll
                    for (int u = 0; u < kBsVec; ++u) {
                        const int c = base + lane + 32 * u;
                        if (!one_pass) v[u] = c < nvec ? ld_nc_v4(src + c) : make_int4(0, 0, 0, 0);
                        if (c < nvec) st_na_v4(d + c, v[u]);
                    }
                }
            }
        }
    }
    __threadfence_system();  // peer (NVLink) stores complete before the rank barrier
}

// Per-group K padding for the wgrad GEMMs: kpg[g] = roundup(rows_g, 64),
// koff = exclusive prefix of kpg, roff = exclusive prefix of rows.
__global__ void pad_offsets_kernel(const int32_t* __restrict__ rows, int G, int32_t* __restrict__ kpg,
                                   int32_t* __restrict__ koff, int32_t* __restrict__ roff) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int k = 0, r = 0;
    for (int g = 0; g < G; ++g) {
        const int n = rows[g];
        koff[g] = k;
        roff[g] = r;
        kpg[g] = (n + 63) & ~63;
        k += kpg[g];
        r += n;
    }
    koff[G] = k;
    roff[G] = r;
}

// out[c, j] for j in group g's padded column range: in[roff[g] + j - koff[g], c]
// when inside the group, else 0.  in [rows, C] bf16 -> out [C, ld] bf16.
__global__ void __launch_bounds__(256) transpose_pad_kernel(const __nv_bfloat16* __restrict__ in, int C,
                                                            const int32_t* __restrict__ rows,
                                                            const int32_t* __restrict__ koff,
                                                            const int32_t* __restrict__ roff, int G, long long ld,
                                                            __nv_bfloat16* __restrict__ out) {
    __shared__ __nv_bfloat16 tile[32][34];
    __shared__ long long srcrow[32];
    const long long j0 = static_cast<long long>(blockIdx.x) * 32;
    const int c0 = blockIdx.y * 32;
    const long long kend = koff[G];
    if (j0 >= kend) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    if (threadIdx.x < 32) {  // source row of padded column j0 + tx (-1: padding)
        const long long j = j0 + tx;
        long long src = -1;
        if (j < kend) {
            int lo = 0, hi = G - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (koff[mid] <= j) lo = mid;
                else hi = mid - 1;
            }
            const long long local = j - koff[lo];
            if (local < rows[lo]) src = roff[lo] + local;
        }
        srcrow[tx] = src;
    }
    __syncthreads();
    for (int jj = ty; jj < 32; jj += 8) {  // coalesced along C
        const int c = c0 + tx;
        const long long r = srcrow[jj];
        tile[jj][tx] = (r >= 0 && c < C) ? in[static_cast<size_t>(r) * C + c] : __float2bfloat16_rn(0.f);
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {  // coalesced along the padded K
        const int c = c0 + i;
        const long long jj = j0 + tx;
        if (c < C && jj < kend) out[static_cast<size_t>(c) * ld + jj] = tile[tx][i];
    }
}

// Gate backward, one warp per token: recompute the softmax from the fp32
// logits (as the forward did, in fp64), gather dL/dw of the kept copies and
// apply the softmax Jacobian:  dl_e = p_e (dp_e - sum_j p_j dp_j).
template <int PER>
__global__ void __launch_bounds__(256) gate_bwd_kernel(const float* __restrict__ logits, const int32_t* __restrict__ slot_pos,
                                                       const int32_t* __restrict__ expert_ids,
                                                       const float* __restrict__ slot_dw, int S, int E, int k,
                                                       __nv_bfloat16* __restrict__ dl) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= S) return;
    const float* row = logits + static_cast<size_t>(t) * E;
    double p[PER], dp[PER];
    double mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = lane + 32 * i;
        p[i] = e < E ? static_cast<double>(row[e]) : -INFINITY;
        dp[i] = 0.0;
        mx = fmax(mx, p[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        p[i] = (lane + 32 * i < E) ? exp(p[i] - mx) : 0.0;
        sum += p[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    // dL/dw for kept copies (dropped copies contribute nothing)
    int ej = -1;
    float dwj = 0.f;
    if (lane < k) {
        const int pp = slot_pos[static_cast<size_t>(t) * k + lane];
        if (pp >= 0) {
            ej = expert_ids[pp];
            dwj = slot_dw[static_cast<size_t>(t) * k + lane];
        }
    }
    for (int j = 0; j < k && j < 32; ++j) {
        const int e = __shfl_sync(0xffffffffu, ej, j);
        const float d = __shfl_sync(0xffffffffu, dwj, j);
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if (e == lane + 32 * i) dp[i] += d;
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        p[i] /= sum;
        s += p[i] * dp[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = lane + 32 * i;
        if (e < E) dl[static_cast<size_t>(t) * E + e] = __float2bfloat16_rn(static_cast<float>(p[i] * (dp[i] - s)));
    }
}

static int warp_grid(long long items) {
    const long long b = (items + 7) / 8;
    return static_cast<int>(b < 1 ? 1 : (b < 8 * kNumSMs ? b : 8 * kNumSMs));
}

void launch_bwd_owner_prep(const void* dyg, const void* eout, const float* gw, const unsigned long long* gsrc,
                           const int32_t* rpe, int El, int H, long long max_rows, float* const* slotdw_tab,
                           void* dz, int me, cudaStream_t st) {
    require(H % 8 == 0, XMOE_ERR_VALIDATION, "backward requires model_dim % 8 == 0");
    int grid = warp_grid(max_rows);
    if (g_copy_blocks > 0 && grid > g_copy_blocks) grid = g_copy_blocks;
    bwd_owner_prep_kernel<<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dyg), static_cast<const __nv_bfloat16*>(eout), gw, gsrc, rpe, El, H,
        slotdw_tab, static_cast<__nv_bfloat16*>(dz), me);
    XMOE_LAUNCH_CHECK();
}

void launch_bwd_scatter_dy(const void* dy, int H, int S, int k, const int32_t* slot_pos, const int32_t* dest_rank,
                           const int32_t* dest_row, const double* cw, int me, void* dz, char* const* eout_tab,
                           char* const* dyg_tab, char* const* dxc_tab, float* const* gw_tab,
                           unsigned long long* const* gsrc_tab, float* slot_dw, unsigned long long* bslot_src,
                           cudaStream_t st) {
    require(H % 8 == 0 && k <= 32, XMOE_ERR_VALIDATION, "backward requires model_dim % 8 == 0, top_k <= 32");
    if (S == 0) return;
    long long blocks = (static_cast<long long>(S) + 7) / 8;
    if (blocks > 8LL * kNumSMs) blocks = 8LL * kNumSMs;
    if (g_copy_blocks > 0 && blocks > g_copy_blocks) blocks = g_copy_blocks;
    int threads = 256;
    size_t smem = 0;
    if (g_copy_fat > 0) {  // whole-SM blocks of the SM partition (kernels.cuh g_copy_fat)
        static bool attr = false;
        if (!attr) {
            XMOE_CUDA(cudaFuncSetAttribute(bwd_scatter_dy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kFatSmemBytes));
            attr = true;
        }
        blocks = g_copy_fat;
        threads = 512;
        smem = kFatSmemBytes;
    }
    bwd_scatter_dy_kernel<<<static_cast<int>(blocks), threads, smem, st>>>(
        static_cast<const char*>(dy), H, S, k, slot_pos, dest_rank, dest_row, cw, me, static_cast<char*>(dz),
        eout_tab, dyg_tab, dxc_tab, gw_tab, gsrc_tab, slot_dw, bslot_src);
    XMOE_LAUNCH_CHECK();
}

void launch_pad_offsets(const int32_t* rows, int G, int32_t* kpg, int32_t* koff, int32_t* roff, cudaStream_t st) {
    pad_offsets_kernel<<<1, 32, 0, st>>>(rows, G, kpg, koff, roff);
    XMOE_LAUNCH_CHECK();
}

void launch_transpose_pad(const void* in, int C, const int32_t* rows, const int32_t* koff, const int32_t* roff,
                          int G, long long ld, void* out, cudaStream_t st) {
    if (ld == 0 || C == 0) return;
    dim3 grid(static_cast<unsigned>((ld + 31) / 32), static_cast<unsigned>((C + 31) / 32));
    transpose_pad_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(in), C, rows, koff, roff, G, ld,
                                               static_cast<__nv_bfloat16*>(out));
    XMOE_LAUNCH_CHECK();
}

void launch_gate_bwd(const float* logits, const int32_t* slot_pos, const int32_t* expert_ids, const float* slot_dw,
                     int S, int E, int k, void* dl, cudaStream_t st) {
    if (S == 0) return;
    require(E <= 256 && k <= 32, XMOE_ERR_VALIDATION, "gate backward supports num_experts <= 256, top_k <= 32");
    auto* o = static_cast<__nv_bfloat16*>(dl);
    const int grid = ceil_div(S, 8);
    if (E <= 64) gate_bwd_kernel<2><<<grid, 256, 0, st>>>(logits, slot_pos, expert_ids, slot_dw, S, E, k, o);
    else if (E <= 128) gate_bwd_kernel<4><<<grid, 256, 0, st>>>(logits, slot_pos, expert_ids, slot_dw, S, E, k, o);
    else gate_bwd_kernel<8><<<grid, 256, 0, st>>>(logits, slot_pos, expert_ids, slot_dw, S, E, k, o);
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
