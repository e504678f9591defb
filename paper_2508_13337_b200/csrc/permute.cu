// Row movement kernels: the padding-free permute (moesim::gather_rows,
// /root/reference/proj/src/pft.cpp:68-77) and the expert-parallel placement
// of packed rows into the receiver's grouped layout (pf_dispatch regroup,
// src/pf_pipeline.cpp:47-79, done at the sender instead of after arrival).
//
// One warp per row, 16-byte vectors, several vectors in flight per lane,
// L1::no_allocate on the streaming side.  HBM-bound: algorithmic bytes per
// row are 2 * row_bytes (+4 B index).
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

thread_local int g_copy_blocks = 0;
thread_local int g_copy_smem = 0;
thread_local int g_copy_fat = 0;

constexpr int kRowWarps = 8;
constexpr int kUnroll = 8;

// Copy one row with the whole warp.  Rows whose size is a multiple of 16 B
// (every bf16 row with H % 8 == 0) move as int4 vectors, kUnroll in flight per
// lane; other sizes (odd-width parity rows) fall back to 8- or 2-byte words.
__device__ __forceinline__ void warp_copy_row(const char* __restrict__ src, char* __restrict__ dst,
                                              int row_bytes, int lane) {
    if ((row_bytes & 15) == 0) {
        const int nvec = row_bytes >> 4;
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        int v = lane;
        for (; v + 32 * (kUnroll - 1) < nvec; v += 32 * kUnroll) {
            int4 r[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) r[u] = ld_nc_v4(s4 + v + 32 * u);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) st_na_v4(d4 + v + 32 * u, r[u]);
        }
        for (; v < nvec; v += 32) st_na_v4(d4 + v, ld_nc_v4(s4 + v));
    } else if ((row_bytes & 7) == 0) {
        const long long* s8 = reinterpret_cast<const long long*>(src);
        long long* d8 = reinterpret_cast<long long*>(dst);
        for (int v = lane; v < (row_bytes >> 3); v += 32) d8[v] = s8[v];
    } else {
        const short* s2 = reinterpret_cast<const short*>(src);
        short* d2 = reinterpret_cast<short*>(dst);
        for (int v = lane; v < (row_bytes >> 1); v += 32) d2[v] = s2[v];
    }
}

// out[i] = src[ids[i]] for i < n (n read from n_dev when given).
__global__ void __launch_bounds__(32 * kRowWarps) gather_rows_kernel(
    const char* __restrict__ src, long long rows, int row_bytes, const int32_t* __restrict__ ids,
    long long n, const int32_t* __restrict__ n_dev, char* __restrict__ out,
    int* __restrict__ err) {
    const long long total = n_dev ? *n_dev : n;
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long i = warp; i < total; i += nwarps) {
        const int id = ids[i];
        if (id < 0 || id >= rows) {
            if (lane == 0 && err) atomicExch(err, 1);
            continue;
        }
        warp_copy_row(src + static_cast<size_t>(id) * row_bytes,
                      out + static_cast<size_t>(i) * row_bytes, row_bytes, lane);
    }
}

// Placement map for expert-parallel dispatch.  Source rank `src` holds its
// packed rows expert-major (tokens_per_expert tpe_src[E]); packed row r of
// expert e lands on rank j = e / El at grouped row
//     expert_base_j[le] + sum_{s < src} tpe_s[e] + (r - blk_src[e])
// which is the (local expert, source, position) order of pf_dispatch
// (pf_pipeline.cpp:47-73).  tpe_all is the all-gathered [W, E] matrix.
// exclusive scan of v[0..n) by one warp (n <= 32 * 32), out may alias v
__device__ __forceinline__ void warp_exscan(const int32_t* v, int32_t* out, int n, int lane) {
    int carry = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
        const int x = b0 + lane < n ? v[b0 + lane] : 0;
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (b0 + lane < n) out[b0 + lane] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

__global__ void dispatch_dest_kernel(const int32_t* __restrict__ tpe_all, int W, int E, int src,
                                     const int32_t* __restrict__ expert_ids,
                                     const int32_t* __restrict__ B_dev,
                                     int32_t* __restrict__ dest_rank,
                                     int32_t* __restrict__ dest_row) {
    extern __shared__ int32_t sh[];
    int32_t* blk = sh;              // [E] packed block start of each expert at src
    int32_t* before = sh + E;       // [E] rows of expert e from sources < src
    int32_t* ebase = before + E;    // [E] grouped base of expert e on its owner
    const int El = E / W;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {  // column sums and the sources before src
        int b = 0, all = 0;
        for (int s = 0; s < W; ++s) {
            const int c = tpe_all[s * E + e];
            all += c;
            if (s < src) b += c;
        }
        before[e] = b;
        ebase[e] = all;
        blk[e] = tpe_all[src * E + e];
    }
    __syncthreads();
    if (wid == 0) warp_exscan(blk, blk, E, lane);
    else if (wid == 1) warp_exscan(ebase, ebase, E, lane);
    __syncthreads();
    const int B = *B_dev;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < B; r += gridDim.x * blockDim.x) {
        const int e = expert_ids[r];
        dest_rank[r] = e / El;
        // grouped base of e on its owner: column sums of the owner's experts before e
        dest_row[r] = ebase[e] - ebase[(e / El) * El] + before[e] + (r - blk[e]);
    }
}

// Fused permute + placement for ranks that share one device (rank == -1
// contexts, the reference's all-workers-in-one-call shape): packed row r of
// source `src` is read straight from the token matrix (token_ids[r]) and
// written into the owner's grouped buffer.
__global__ void __launch_bounds__(32 * kRowWarps) scatter_rows_kernel(
    const char* __restrict__ x, int row_bytes, const int32_t* __restrict__ token_ids,
    const int32_t* __restrict__ B_dev, const int32_t* __restrict__ dest_rank,
    const int32_t* __restrict__ dest_row, char* const* __restrict__ dest_bufs) {
    const int B = *B_dev;
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long r = warp; r < B; r += nwarps) {
        const long long t = token_ids ? token_ids[r] : r;  // null: x is already packed
        char* dst = dest_bufs[dest_rank[r]] + static_cast<size_t>(dest_row[r]) * row_bytes;
        warp_copy_row(x + static_cast<size_t>(t) * row_bytes, dst, row_bytes, lane);
    }
    __threadfence_system();  // peer (NVLink) stores complete before the rank barrier
}

// TMA-staged variant of the fused permute + placement (XMOE_PERMUTE=tma;
// measured on par with the warp kernel, which is the default because it
// needs no shared memory and co-resides with the persistent GEMM CTAs): every warp owns a
// ring of kTmaSlots row buffers in shared memory; lane 0 moves each row with
// two bulk-async copies (global -> shared, completion on an mbarrier; then
// shared -> global, which may be a peer GPU's memory over NVLink), keeping up
// to kTmaSlots rows in flight per warp without touching registers.
constexpr int kTmaSlots = 4;
constexpr int kTmaWarps = 4;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32 * kTmaWarps) scatter_rows_tma_kernel(
    const char* __restrict__ x, int row_bytes, const int32_t* __restrict__ token_ids,
    const int32_t* __restrict__ B_dev, const int32_t* __restrict__ dest_rank,
    const int32_t* __restrict__ dest_row, char* const* __restrict__ dest_bufs) {
    extern __shared__ __align__(128) char ring[];  // [kTmaWarps][kTmaSlots][row_bytes]
    __shared__ __align__(8) uint64_t bars[kTmaWarps][kTmaSlots];
    const int B = *B_dev;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    if (lane != 0) return;
    char* my = ring + static_cast<size_t>(wl) * kTmaSlots * row_bytes;
    for (int q = 0; q < kTmaSlots; ++q)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[wl][q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase_bits = 0;
    int i = 0;
    for (long long r = warp; r < B; r += nwarps, ++i) {
        const int q = i % kTmaSlots;
        char* slot = my + static_cast<size_t>(q) * row_bytes;
        if (i >= kTmaSlots)  // the store that last read this slot must be done reading
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaSlots - 1) : "memory");
        const char* src = x + static_cast<size_t>(token_ids ? token_ids[r] : r) * row_bytes;
        char* dst = dest_bufs[dest_rank[r]] + static_cast<size_t>(dest_row[r]) * row_bytes;
        const uint32_t bar = smem_addr(&bars[wl][q]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(row_bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_addr(slot)),
                     "l"(src), "r"(row_bytes), "r"(bar)
                     : "memory");
        const uint32_t par = (phase_bits >> q) & 1u;
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, P;\n}\n"
                : "=r"(done)
                : "r"(bar), "r"(par)
                : "memory");
        }
        phase_bits ^= 1u << q;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(slot)),
                     "r"(row_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __threadfence_system();
}

// Reverse of the placement: expert outputs come back from the owners'
// grouped buffers into the source's packed order (pf_combine un-regroup +
// reverse exchange, pf_pipeline.cpp:118-128).
__global__ void __launch_bounds__(32 * kRowWarps) unscatter_rows_kernel(
    int row_bytes, const int32_t* __restrict__ B_dev, const int32_t* __restrict__ dest_rank,
    const int32_t* __restrict__ dest_row, const char* const* __restrict__ src_bufs,
    char* __restrict__ out) {
    const int B = *B_dev;
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long r = warp; r < B; r += nwarps) {
        const char* s = src_bufs[dest_rank[r]] + static_cast<size_t>(dest_row[r]) * row_bytes;
        warp_copy_row(s, out + static_cast<size_t>(r) * row_bytes, row_bytes, lane);
    }
}

// Token-major fused permute + placement (bf16 rows, row_bytes % 16 == 0):
// one warp per token reads the token row ONCE (up to 8 x 16 B per lane in
// flight) and stores it to every kept copy's slot in the owners' grouped
// buffers (peer addresses over NVLink when the owner is another GPU).  It
// also records, per (token, slot), the address the combine will read the
// copy's expert output from and the copy's weight, so the combine needs a
// single dependent load before streaming rows.  Algorithmic bytes: one read
// of x, k writes.
constexpr int kTokWarps = 8;
constexpr int kTokVec = 8;  // int4 per lane per pass (4 KB rows in one pass)

__global__ void __launch_bounds__(32 * kTokWarps) scatter_tokens_kernel(
    const char* __restrict__ x, int row_bytes, int S, int k, const int32_t* __restrict__ slot_pos,
    const int32_t* __restrict__ dest_rank, const int32_t* __restrict__ dest_row, const double* __restrict__ cw,
    char* const* __restrict__ dest_bufs, char* const* __restrict__ src_bufs,
    unsigned long long* __restrict__ slot_src, float* __restrict__ slot_w) {
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const int nvec = row_bytes >> 4;
    for (long long t = warp; t < S; t += nwarps) {
        // issue the row loads first; the index chain overlaps them
        const int4* src = reinterpret_cast<const int4*>(x + static_cast<size_t>(t) * row_bytes);
        int4 v[kTokVec];
#pragma unroll
        for (int u = 0; u < kTokVec; ++u) {
            const int c = lane + 32 * u;
            v[u] = c < nvec ? ld_nc_v4(src + c) : make_int4(0, 0, 0, 0);
        }
        int p = -1;
        unsigned long long dst = 0, rd = 0;
        float wv = 0.f;
        if (lane < k) {
            p = slot_pos[static_cast<size_t>(t) * k + lane];
            if (p >= 0) {
                const int r = dest_rank[p];
                const size_t off = static_cast<size_t>(dest_row[p]) * row_bytes;
                dst = reinterpret_cast<unsigned long long>(dest_bufs[r] + off);
                if (src_bufs) rd = reinterpret_cast<unsigned long long>(src_bufs[r] + off);
                wv = static_cast<float>(cw[p]);
            }
            if (slot_src) slot_src[static_cast<size_t>(t) * k + lane] = rd;
            if (slot_w) slot_w[static_cast<size_t>(t) * k + lane] = wv;
        }
        const int n = __popc(__ballot_sync(0xffffffffu, lane < k && p >= 0));
        for (int base = 0; base < nvec; base += 32 * kTokVec) {
            if (base > 0) {
#pragma unroll
                for (int u = 0; u < kTokVec; ++u) {
                    const int c = base + lane + 32 * u;
                    v[u] = c < nvec ? ld_nc_v4(src + c) : make_int4(0, 0, 0, 0);
                }
            }
            for (int j = 0; j < n; ++j) {
                int4* d = reinterpret_cast<int4*>(__shfl_sync(0xffffffffu, dst, j));
#pragma unroll
                for (int u = 0; u < kTokVec; ++u) {
                    const int c = base + lane + 32 * u;
                    if (c < nvec) st_na_v4(d + c, v[u]);
                }
            }
        }
    }
    __threadfence_system();  // peer (NVLink) stores complete before the rank barrier
}

static int row_grid(long long n) {
    const long long warps = n > 0 ? n : 1;
    const long long blocks = (warps + kRowWarps - 1) / kRowWarps;
    return static_cast<int>(blocks < 4 * kNumSMs ? blocks : 4 * kNumSMs);
}

void launch_gather_rows(const void* src, long long rows, int row_bytes, const int32_t* ids,
                        long long n, const int32_t* n_dev, void* out, int* err,
                        cudaStream_t st) {
    if (!n_dev && n == 0) return;
    gather_rows_kernel<<<row_grid(n), 32 * kRowWarps, 0, st>>>(
        static_cast<const char*>(src), rows, row_bytes, ids, n, n_dev, static_cast<char*>(out),
        err);
    XMOE_LAUNCH_CHECK();
}

void launch_dispatch_dest(const int32_t* tpe_all, int W, int E, int src,
                          const int32_t* expert_ids, const int32_t* B_dev, long long max_rows,
                          int32_t* dest_rank, int32_t* dest_row, cudaStream_t st) {
    const int blocks = ceil_div(max_rows > 0 ? max_rows : 1, 256);
    require(blocks >= 1 && E <= 1024, XMOE_ERR_VALIDATION, "dispatch destinations: num_experts <= 1024");
    dispatch_dest_kernel<<<blocks < 4 * kNumSMs ? blocks : 4 * kNumSMs, 256,
                           sizeof(int32_t) * (3 * E + 1), st>>>(tpe_all, W, E, src, expert_ids,
                                                               B_dev, dest_rank, dest_row);
    XMOE_LAUNCH_CHECK();
}

static bool permute_tma(int row_bytes) {
    static const int mode = [] {
        const char* e = std::getenv("XMOE_PERMUTE");
        return (e && std::string(e) == "tma") ? 1 : 0;
    }();
    return mode == 1 && (row_bytes & 15) == 0 && row_bytes <= 16384;
}

void launch_scatter_rows(const void* x, int row_bytes, const int32_t* token_ids,
                         const int32_t* B_dev, long long max_rows, const int32_t* dest_rank,
                         const int32_t* dest_row, char* const* dest_bufs, cudaStream_t st) {
    if (permute_tma(row_bytes)) {
        const size_t smem = static_cast<size_t>(kTmaWarps) * kTmaSlots * row_bytes;
        static size_t smem_set = 0;
        if (smem > smem_set) {
            XMOE_CUDA(cudaFuncSetAttribute(scatter_rows_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
            smem_set = smem;
        }
        const long long warps = max_rows > 0 ? max_rows : 1;
        long long blocks = (warps + kTmaWarps - 1) / kTmaWarps;
        if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
        scatter_rows_tma_kernel<<<static_cast<int>(blocks), 32 * kTmaWarps, smem, st>>>(
            static_cast<const char*>(x), row_bytes, token_ids, B_dev, dest_rank, dest_row, dest_bufs);
        XMOE_LAUNCH_CHECK();
        return;
    }
    scatter_rows_kernel<<<row_grid(max_rows), 32 * kRowWarps, 0, st>>>(
        static_cast<const char*>(x), row_bytes, token_ids, B_dev, dest_rank, dest_row, dest_bufs);
    XMOE_LAUNCH_CHECK();
}

void launch_scatter_tokens(const void* x, int row_bytes, int S, int k, const int32_t* slot_pos,
                           const int32_t* dest_rank, const int32_t* dest_row, const double* cw,
                           char* const* dest_bufs, char* const* src_bufs, unsigned long long* slot_src,
                           float* slot_w, cudaStream_t st) {
    require((row_bytes & 15) == 0 && k <= 32, XMOE_ERR_VALIDATION, "token scatter needs 16-byte rows, k <= 32");
    if (S == 0) return;
    long long blocks = (static_cast<long long>(S) + kTokWarps - 1) / kTokWarps;
    const long long cap = g_copy_blocks > 0 ? g_copy_blocks : 8LL * kNumSMs;
    if (blocks > cap) blocks = cap;
    scatter_tokens_kernel<<<static_cast<int>(blocks), 32 * kTokWarps, g_copy_smem, st>>>(
        static_cast<const char*>(x), row_bytes, S, k, slot_pos, dest_rank, dest_row, cw, dest_bufs, src_bufs,
        slot_src, slot_w);
    XMOE_LAUNCH_CHECK();
}

void launch_unscatter_rows(int row_bytes, const int32_t* B_dev, long long max_rows,
                           const int32_t* dest_rank, const int32_t* dest_row,
                           const char* const* src_bufs, void* out, cudaStream_t st) {
    unscatter_rows_kernel<<<row_grid(max_rows), 32 * kRowWarps, 0, st>>>(
        row_bytes, B_dev, dest_rank, dest_row, src_bufs, static_cast<char*>(out));
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
