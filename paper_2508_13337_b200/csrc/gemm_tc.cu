// Variable-length grouped GEMM on the 5th-generation tensor cores (sm_100a):
// the fine-grained expert FFN of moesim::grouped_expert_mlp
// (/root/reference/proj/src/pf_pipeline.cpp:83-105) as a bf16 tcgen05 kernel.
//
//   D[r, n] = act( sum_k A[r, k] * B_g[n, k] )   for rows r of group g
//
// A [rows, K] is the grouped expert input (K-major), B [G*N, K] the stacked
// per-expert weights in K-major layout (W1^T / W2^T), D [rows, N].  Groups are
// contiguous row segments whose sizes live in device memory, so the kernel
// needs no host synchronisation and empty or oversized groups cost nothing
// special.
//
// Structure (persistent, one CTA per SM, 6 warps):
//   warp 0      TMA producer: 128x64 A box + 256x64 B box per stage,
//               128B swizzle, 4-stage mbarrier ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N<=256, K=16 per instruction, fp32 accumulate)
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> ReLU -> bf16/fp32 -> global,
//               rows past the group end masked
// Accumulators are double-buffered in TMEM (2 x 256 columns), so the epilogue
// of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

// SM budget of the next 2-CTA GEMM launches (0 = all SMs); the layer lowers it
// for GEMMs that run on a side stream next to bandwidth-bound kernels.
thread_local int g_gemm_sm_limit = 0;
thread_local const float* g_gemm_addf = nullptr;
thread_local const unsigned* g_gemm_ready = nullptr;
thread_local int g_gemm_ready_mult = 1;

namespace tc {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int UK = 16;
constexpr int kStages = 4;
constexpr int kAccBufs = 2;
constexpr int kTmemCols = 512;
constexpr int kThreads = 192;
constexpr int kMaxGroups = 1024;
constexpr uint32_t kABytes = BM * BK * 2;
constexpr uint32_t kBBytes = BN * BK * 2;
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr size_t kSmemBytes = 1024 /*align*/ + kStages * kStageBytes + 1024 /*barriers*/ +
                              sizeof(int32_t) * 2 * (kMaxGroups + 1);

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Waits for the phase with the given parity.  A watchdog traps after ~2^31
// polls (tens of seconds) so a protocol bug surfaces as a launch error
// instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    for (uint32_t it = 0;; ++it) {
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) return;
        if (it == 0x7fffffffu) asm volatile("trap;");
    }
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, 128B swizzle, 8-row core groups
// 1024 B apart (SBO), LBO unused (1), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major.
__device__ __forceinline__ uint32_t make_idesc(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}

// one thread of a converged warp (elect.sync): keeps the issue code on the
// uniform datapath (see tc2::mma2_kblock)
__device__ __forceinline__ bool elect_one_sync() {
    uint32_t e;
    asm volatile(
        "{\n"
        ".reg .b32 rx;\n"
        ".reg .pred px;\n"
        "elect.sync rx|px, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, px;\n"
        "}\n"
        : "=r"(e));
    return e != 0;
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- scheduler
struct TileInfo {
    int g, row0, rows_left, n0;
};

__device__ __forceinline__ TileInfo tile_of(int t, const int32_t* tile_start,
                                            const int32_t* row_off, int G, int ntn) {
    int lo = 0, hi = G - 1;  // last g with tile_start[g] <= t (skips empty groups)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_start[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    const int local = t - tile_start[lo];
    const int mb = local / ntn, nb = local % ntn;
    TileInfo ti;
    ti.g = lo;
    ti.row0 = row_off[lo] + mb * BM;
    ti.rows_left = (row_off[lo + 1] - row_off[lo]) - mb * BM;
    ti.n0 = nb * BN;
    return ti;
}

// ---------------------------------------------------------------- kernel
template <typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_a,
                           const __grid_constant__ CUtensorMap tmap_b,
                           const int32_t* __restrict__ rows_per_group, int G, int N, int K,
                           OutT* __restrict__ D, int relu) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + kStages * kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + kStages;
    uint64_t* tfull_bar = bars + 2 * kStages;
    uint64_t* tempty_bar = bars + 2 * kStages + kAccBufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kAccBufs);
    int32_t* tile_start = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 1024);
    int32_t* row_off = tile_start + kMaxGroups + 1;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ntn = (N + BN - 1) / BN;
    const int nkb = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        int t = 0, r = 0;
        for (int g = 0; g < G; ++g) {
            tile_start[g] = t;
            row_off[g] = r;
            const int m = rows_per_group[g];
            t += ((m + BM - 1) / BM) * ntn;
            r += m;
        }
        tile_start[G] = t;
        row_off[G] = r;
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int num_tiles = tile_start[G];

    if (warp == 0) {
        // ===================== TMA producer (whole warp, one elected issuer) =====================
        {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                const TileInfo ti = tile_of(t, tile_start, row_off, G, ntn);
                const int brow = ti.g * N + ti.n0;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    if (elect_one_sync()) {
                        mbar_expect_tx(&full_bar[stage], kStageBytes);
                        tma_load_2d(&tmap_a, &full_bar[stage], smem_a + stage * kABytes, kb * BK, ti.row0);
                        tma_load_2d(&tmap_b, &full_bar[stage], smem_b + stage * kBBytes, kb * BK, brow);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const TileInfo ti = tile_of(t, tile_start, row_off, G, ntn);
            const int nw = min(BN, N - ti.n0);
            const int n_mma = (nw + 15) & ~15;
            const uint32_t idesc = make_idesc(n_mma);
            const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
            mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
            tc_fence_after();
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (elect_one_sync()) {
                    const uint64_t da = make_desc(smem_u32(smem_a + stage * kABytes));
                    const uint64_t db = make_desc(smem_u32(smem_b + stage * kBBytes));
#pragma unroll
                    for (int kk = 0; kk < BK / UK; ++kk) {
                        // +32 bytes along K inside the 128B swizzle atom
                        mma_bf16(tmem_d, da + static_cast<uint64_t>(kk * 2),
                                 db + static_cast<uint64_t>(kk * 2), idesc,
                                 (kb > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(&empty_bar[stage]);
                    if (kb == nkb - 1) mma_commit(&tfull_bar[acc]);
                }
                __syncwarp();
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++acc == kAccBufs) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const TileInfo ti = tile_of(t, tile_start, row_off, G, ntn);
            const int nw = min(BN, N - ti.n0);
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            const int r = quarter * 32 + lane;
            const bool row_ok = r < ti.rows_left;
            OutT* drow = D + static_cast<size_t>(ti.row0 + r) * N + ti.n0;
            for (int c0 = 0; c0 < nw; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                              static_cast<uint32_t>(acc * BN + c0),
                          v);
                if (!row_ok) continue;
                float f[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    f[i] = __uint_as_float(v[i]);
                    if (relu) f[i] = fmaxf(f[i], 0.f);
                }
                const int cn = min(32, nw - c0);
                if constexpr (sizeof(OutT) == 2) {
                    if (cn == 32 && (N & 7) == 0) {
                        int4* dst = reinterpret_cast<int4*>(drow + c0);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            int4 o;
                            o.x = static_cast<int>(pack_bf16(f[8 * q + 0], f[8 * q + 1]));
                            o.y = static_cast<int>(pack_bf16(f[8 * q + 2], f[8 * q + 3]));
                            o.z = static_cast<int>(pack_bf16(f[8 * q + 4], f[8 * q + 5]));
                            o.w = static_cast<int>(pack_bf16(f[8 * q + 6], f[8 * q + 7]));
                            dst[q] = o;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < cn) drow[c0 + i] = __float2bfloat16_rn(f[i]);
                    }
                } else {
                    if (cn == 32 && (N & 3) == 0) {
                        float4* dst = reinterpret_cast<float4*>(drow + c0);
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            dst[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < cn) drow[c0 + i] = f[i];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[acc]);
            if (++acc == kAccBufs) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(kTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------- fused gate
// moesim::gate_forward (gating.cpp:14-57) in ONE kernel: the logits GEMM
// x [S,H] . Wg^T [E,H] (E <= 256: one N tile) on the tensor cores, then the
// epilogue thread that owns a token row reads its E fp32 logits straight from
// TMEM and does the softmax and top-k in registers — no logits round trip
// through HBM, no second launch.  Per row:
//   pass 1  max and the top-k by (logit desc, id asc) — exp is monotone and
//           on the grid inputs distinct logits differ by >= 2^-17, so this is
//           the reference's (prob desc, id asc) order;
//   pass 2  sum_e exp(l_e - max) in fp64, ascending e (gating.cpp:39-43);
//           weights exp(l_j - max) / sum (raw probabilities, gating.cpp:51-54).
// It also writes each tile's expert histogram (counts [tile, E]) for the
// fused dropless placement (pft.cu route_place_kernel) and, for training
// layers, the fp32 logits (the gate backward's input).
template <int KMAX>
__global__ void __launch_bounds__(kThreads, 1)
    gate_route_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b, int S,
                      int E, int K, int k, int renorm, int32_t* __restrict__ top, double* __restrict__ weights,
                      float* __restrict__ logits, int32_t* __restrict__ counts) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + kStages * kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + kStages;
    uint64_t* tfull_bar = bars + 2 * kStages;
    uint64_t* tempty_bar = bars + 2 * kStages + kAccBufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kAccBufs);
    int32_t* hist = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 1024);  // [256]

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nkb = (K + BK - 1) / BK;
    const int num_tiles = (S + BM - 1) / BM;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&empty_bar[stage], phase ^ 1);
                if (elect_one_sync()) {
                    mbar_expect_tx(&full_bar[stage], kStageBytes);
                    tma_load_2d(&tmap_a, &full_bar[stage], smem_a + stage * kABytes, kb * BK, t * BM);
                    tma_load_2d(&tmap_b, &full_bar[stage], smem_b + stage * kBBytes, kb * BK, 0);
                }
                __syncwarp();
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        const uint32_t idesc = make_idesc((E + 15) & ~15);
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
            mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
            tc_fence_after();
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (elect_one_sync()) {
                    const uint64_t da = make_desc(smem_u32(smem_a + stage * kABytes));
                    const uint64_t db = make_desc(smem_u32(smem_b + stage * kBBytes));
#pragma unroll
                    for (int kk = 0; kk < BK / UK; ++kk)
                        mma_bf16(tmem_d, da + static_cast<uint64_t>(kk * 2), db + static_cast<uint64_t>(kk * 2), idesc,
                                 (kb > 0 || kk > 0) ? 1u : 0u);
                    mma_commit(&empty_bar[stage]);
                    if (kb == nkb - 1) mma_commit(&tfull_bar[acc]);
                }
                __syncwarp();
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++acc == kAccBufs) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        const int quarter = warp & 3;
        const int et = threadIdx.x - 64;  // 0..127 over the epilogue warps
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            if (counts)
                for (int e = et; e < E; e += 128) hist[e] = 0;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int row = t * BM + quarter * 32 + lane;
            const bool row_ok = row < S;
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN);
            float tv[KMAX];
            int ti[KMAX];
#pragma unroll
            for (int j = 0; j < KMAX; ++j) {
                tv[j] = -INFINITY;
                ti[j] = 0x7fffffff;
            }
            float mx = -INFINITY;
            for (int c0 = 0; c0 < E; c0 += 32) {  // pass 1: max, top-k, logits out
                uint32_t v[32];
                tmem_ld32(taddr + static_cast<uint32_t>(c0), v);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int e = c0 + i;
                    if (e >= E) break;
                    float nv = __uint_as_float(v[i]);
                    mx = fmaxf(mx, nv);
                    int ni = e;
#pragma unroll
                    for (int j = 0; j < KMAX; ++j) {  // bubble insert by (logit desc, id asc): an
                        // element pushed down must still pass equal logits of higher ids
                        if (j < k && (nv > tv[j] || (nv == tv[j] && ni < ti[j]))) {
                            const float fv = tv[j];
                            const int fi = ti[j];
                            tv[j] = nv;
                            ti[j] = ni;
                            nv = fv;
                            ni = fi;
                        }
                    }
                }
                if (logits && row_ok) {
                    float4* dst = reinterpret_cast<float4*>(logits + static_cast<size_t>(row) * E + c0);
                    if (c0 + 32 <= E && (E & 3) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                                 __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
                    } else {
                        for (int i = 0; i < 32 && c0 + i < E; ++i) logits[static_cast<size_t>(row) * E + c0 + i] = __uint_as_float(v[i]);
                    }
                }
            }
            const double m = static_cast<double>(mx);
            double sum = 0.0;
            for (int c0 = 0; c0 < E; c0 += 32) {  // pass 2: sum in ascending expert order
                uint32_t v[32];
                tmem_ld32(taddr + static_cast<uint32_t>(c0), v);
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (c0 + i < E) sum = __dadd_rn(sum, exp(__dsub_rn(static_cast<double>(__uint_as_float(v[i])), m)));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[acc]);  // accumulator free for tile t + grid
            if (++acc == kAccBufs) {
                acc = 0;
                acc_phase ^= 1;
            }
            if (row_ok) {
                double w[KMAX], wsum = 0.0;
#pragma unroll
                for (int j = 0; j < KMAX; ++j) {
                    w[j] = j < k ? __ddiv_rn(exp(__dsub_rn(static_cast<double>(tv[j]), m)), sum) : 0.0;
                    if (j < k) wsum = __dadd_rn(wsum, w[j]);
                }
#pragma unroll
                for (int j = 0; j < KMAX; ++j) {
                    if (j >= k) break;
                    top[static_cast<size_t>(row) * k + j] = ti[j];
                    weights[static_cast<size_t>(row) * k + j] = renorm ? __ddiv_rn(w[j], wsum) : w[j];
                    if (counts) atomicAdd(&hist[ti[j]], 1);
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (counts)
                for (int e = et; e < E; e += 128) counts[static_cast<size_t>(t) * E + e] = hist[e];
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
    }
}

}  // namespace tc

// ============================================================================
// 2-CTA variant (cta_group::2): a cluster of two CTAs on a TPC computes one
// 256 x 256 tile.  Each CTA stages its own 128 rows of A and its half of the
// 256-wide B slice (128 rows) per 64-deep K block, so per-SM shared-memory
// and L2->SM traffic drop by a third against the 1-CTA 128x256 tile.  The
// leader CTA issues tcgen05.mma.cta_group::2 (M=256); each CTA's TMEM holds
// its 128 accumulator rows.  Barrier protocol:
//   full[s]   leader only, 2 arrivals (each CTA's expect_tx) + TMA bytes
//   empty[s]  per CTA, arrived by the leader's multicast commit
//   tfull[b]  per CTA, arrived by the leader's multicast commit
//   tempty[b] leader only, 8 arrivals (4 epilogue warps x 2 CTAs)
// ============================================================================
namespace tc2 {

constexpr int BM = 256;   // rows per CTA pair
constexpr int BMC = 128;  // rows per CTA
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int UK = 16;
constexpr int kStages = 6;
constexpr int kAccBufs = 2;
constexpr int kTmemCols = 512;
constexpr int kThreads = 192;
constexpr int kMaxGroups = 1024;
constexpr uint32_t kABytes = BMC * BK * 2;
constexpr uint32_t kBBytes = (BN / 2) * BK * 2;
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr size_t kGroupTabBytes = sizeof(int32_t) * 2 * (kMaxGroups + 1);
constexpr size_t kEpiWarpWords = 32 * 33;  // per epilogue warp: a 32 x 32 transpose tile (+1 pad)
constexpr size_t kEpiWarpBytes = 5120;     // per-warp staging slot (1024-aligned, >= 32*33*4)
// epilogue staging area: 1024-aligned (the TMA-store tile uses the 128B swizzle)
constexpr size_t kEpiOff = (kStages * kStageBytes + 1024 + kGroupTabBytes + 1023) / 1024 * 1024;
constexpr size_t kSmemBytes = 1024 + kEpiOff + 4 * kEpiWarpBytes;

using tc::make_desc;
using tc::mbar_init;
using tc::mbar_wait;
using tc::prefetch_tmap;
using tc::smem_u32;
using tc::tc_fence_after;
using tc::tc_fence_before;
using tc::tmem_ld32;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_cluster(uint32_t cl_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ void expect_tx_cluster(uint32_t cl_addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(cl_addr), "r"(bytes)
                 : "memory");
}
// TMA load into this CTA's smem, completion counted on the leader's barrier.
__device__ __forceinline__ void tma_load_2sm(const CUtensorMap* map, uint32_t bar_cl, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cl)
        : "memory");
}
// TMA gather of 4 arbitrary rows (box {BK, 1}) into 4 consecutive 128-byte
// smem rows, completion counted on the leader's barrier.
__device__ __forceinline__ void tma_gather4_2sm(const CUtensorMap* map, uint32_t bar_cl, void* dst, int c0,
                                                int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar_cl)
        : "memory");
}
// TMA store of a staged smem box to global (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint32_t make_idesc2(int n, int m = BM) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
// One K block (BK = 64 = four K=16 MMAs) issued from ONE thread in one asm
// block, followed by the commit that frees the smem stage in both CTAs.
// Descriptor start addresses advance by INC (16-byte units) per MMA: 2 for
// K-major operands (32 B per 16 K-columns), 128 for MN-major (2 KB per 16
// K-rows).  Keeping the four MMAs and the commit in one block lets the
// compiler move the operands to uniform registers once per K block instead
// of electing and broadcasting per instruction (the issue loop, not the
// tensor pipe, was the limit: ncu showed the MMA warp never waiting on data).
__device__ __forceinline__ bool elect_one() {
    uint32_t e;
    asm volatile(
        "{\n"
        ".reg .b32 rx;\n"
        ".reg .pred px;\n"
        "elect.sync rx|px, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, px;\n"
        "}\n"
        : "=r"(e));
    return e != 0;
}
static_assert(BK / UK == 4, "mma2_kblock issues four K=16 MMAs per K block");
template <int INC>
__device__ __forceinline__ void mma2_kblock(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc,
                                            uint32_t empty_bar) {
    asm volatile(
        "{\n"
        ".reg .pred p, q;\n"
        ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 q, 0, 0;\n"
        "add.s64 a1, %1, %6;\n"
        "add.s64 b1, %2, %6;\n"
        "add.s64 a2, %1, %7;\n"
        "add.s64 b2, %2, %7;\n"
        "add.s64 a3, %1, %8;\n"
        "add.s64 b3, %2, %8;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, q;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, q;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, q;\n"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %9;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(empty_bar), "n"(INC), "n"(2 * INC), "n"(3 * INC),
        "h"(static_cast<uint16_t>(0x3))
        : "memory");
}
__device__ __forceinline__ void commit_both(uint64_t* bar) {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

struct TileInfo {
    int g, row0, rows_left, n0, kofs, nkb;
};

// kVarK == false: groups are row segments of A/D sharing K (forward, dgrad).
// kVarK == true : groups are K segments (wgrad): group g reduces over its
//                 gk[g] columns of A [M, Ktot] and B [N, Ktot] into D_g [M, N].
template <bool kVarK>
__device__ __forceinline__ TileInfo tile_of(int t, const int32_t* tile_start, const int32_t* off, int G, int ntn,
                                            int M, int K) {
    int lo = 0, hi = G - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_start[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    const int local = t - tile_start[lo];
    const int mb = local / ntn, nb = local % ntn;
    TileInfo ti;
    ti.g = lo;
    ti.n0 = nb * BN;
    if constexpr (kVarK) {
        ti.row0 = mb * BM;
        ti.rows_left = M - mb * BM;
        ti.kofs = off[lo];
        ti.nkb = (off[lo + 1] - off[lo]) / BK;
    } else {
        ti.row0 = off[lo] + mb * BM;
        ti.rows_left = (off[lo + 1] - off[lo]) - mb * BM;
        ti.kofs = 0;
        ti.nkb = (K + BK - 1) / BK;
    }
    return ti;
}

// D (+)= epilogue(A . B^T) on 256x256 pair tiles.  Epilogue options: ReLU,
// and mask (multiply by mask[r,n] > 0 — the ReLU derivative in dgrad).
// Epilogue store of one 32-column chunk: lane l holds row l's 32 fp32
// values; they go through a per-warp [32][33] shared tile so that each
// store instruction writes whole 128-byte row segments (fp32: one row per
// instruction; bf16: two 64-byte row segments) instead of 32 scattered
// 16-byte pieces.  rows_valid: rows of this warp inside the output.
template <typename OutT>
__device__ __forceinline__ void store_chunk_coalesced(uint32_t* tile, const float* f, OutT* D, size_t ldd,
                                                      size_t row_base, int rows_valid, int col0, int cn,
                                                      int lane) {
    if constexpr (sizeof(OutT) == 4) {
#pragma unroll
        for (int i = 0; i < 32; ++i) tile[lane * 33 + i] = __float_as_uint(f[i]);
        __syncwarp();
        const int rmax = min(32, rows_valid);
        for (int rr = 0; rr < rmax; ++rr)
            if (lane < cn) D[(row_base + rr) * ldd + col0 + lane] = __uint_as_float(tile[rr * 33 + lane]);
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) tile[lane * 33 + i] = pack_bf16(f[2 * i], f[2 * i + 1]);
        __syncwarp();
        const int rmax = min(32, rows_valid);
        const int ci = lane & 15;
        uint32_t* D32 = reinterpret_cast<uint32_t*>(D);
        for (int rr = 0; rr < rmax; rr += 2) {
            const int r = rr + (lane >> 4);
            if (r < rmax && 2 * ci < cn) D32[((row_base + r) * ldd + col0) / 2 + ci] = tile[r * 33 + ci];
        }
    }
    __syncwarp();
}

template <typename OutT, bool kVarK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    grouped_gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                            const int32_t* __restrict__ group_sizes, int G, int M, int N, int K,
                            OutT* __restrict__ D, int relu, const uint32_t* __restrict__ mbits_in,
                            uint32_t* __restrict__ mbits_out, int coalesced, const int32_t* __restrict__ a_idx,
                            int a_rows, const __grid_constant__ CUtensorMap tmap_d, int tma_d, int half_ok,
                            const float* addf, const unsigned* ready, int ready_mult) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + kStages * kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + kStages;
    uint64_t* tfull_bar = bars + 2 * kStages;
    uint64_t* tempty_bar = bars + 2 * kStages + kAccBufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kAccBufs);
    int32_t* tile_start = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 1024);
    int32_t* off = tile_start + kMaxGroups + 1;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1;
    const int npairs = gridDim.x >> 1;
    const int ntn = (N + BN - 1) / BN;

    if (threadIdx.x == 0) {
        int t = 0, r = 0;
        for (int g = 0; g < G; ++g) {
            tile_start[g] = t;
            off[g] = r;
            const int m = group_sizes[g];
            t += (kVarK ? (M + BM - 1) / BM : (m + BM - 1) / BM) * ntn;
            r += m;
        }
        tile_start[G] = t;
        off[G] = r;
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 2);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // barrier inits and TMEM allocation visible to the peer
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int num_tiles = tile_start[G];
    // Half tiles: a group's last row tile with <= 128 rows runs as an M = 128
    // pair MMA (64 rows per CTA; accumulator columns [0, n/2) in TMEM lanes
    // 0-63 and [n/2, n) in lanes 64-127 of each CTA), half the tensor work
    // of padding it to 256 rows.  Every role derives it from the tile alone.
    auto is_half = [&](const TileInfo& ti, int nw) {
        return !kVarK && half_ok && ti.rows_left <= BMC && (nw & 63) == 0;
    };

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (a_idx) {
            // row-gathered A (a_idx: physical row of every logical row): lane l
            // brings rows 4l..4l+3 of this CTA's 128 with one gather4 per k-block
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair; t < num_tiles; t += npairs) {
                const TileInfo ti = tile_of<kVarK>(t, tile_start, off, G, ntn, M, K);
                const int nw = min(BN, N - ti.n0);
                const int n_mma = (nw + 15) & ~15;
                const int arow = ti.row0 + (is_half(ti, nw) ? BMC / 2 : BMC) * static_cast<int>(rank);
                const int brow = (kVarK ? 0 : ti.g * N) + ti.n0 + (n_mma / 2) * static_cast<int>(rank);
                int r4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) r4[q] = a_idx[min(arow + 4 * lane + q, a_rows - 1)];
                for (int kb = 0; kb < ti.nkb; ++kb) {
                    const uint32_t fb = mapa(&full_bar[stage], 0);
                    if (lane == 0) {
                        mbar_wait(&empty_bar[stage], phase ^ 1);
                        expect_tx_cluster(fb, kStageBytes);
                    }
                    __syncwarp();
                    const int kc = ti.kofs + kb * BK;
                    tma_gather4_2sm(&tmap_a, fb, smem_a + stage * kABytes + lane * 512, kc, r4[0], r4[1], r4[2],
                                    r4[3]);
                    if (lane == 0) tma_load_2sm(&tmap_b, fb, smem_b + stage * kBBytes, kc, brow);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        } else {  // whole warp in the loop, one elected thread issues (see the wgrad producer)
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair; t < num_tiles; t += npairs) {
                const TileInfo ti = tile_of<kVarK>(t, tile_start, off, G, ntn, M, K);
                const int nw = min(BN, N - ti.n0);
                const int n_mma = (nw + 15) & ~15;
                const int arow = ti.row0 + (is_half(ti, nw) ? BMC / 2 : BMC) * static_cast<int>(rank);
                const int brow = (kVarK ? 0 : ti.g * N) + ti.n0 + (n_mma / 2) * static_cast<int>(rank);
                for (int kb = 0; kb < ti.nkb; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    const int kc = ti.kofs + kb * BK;
                    if (elect_one()) {
                        const uint32_t fb = mapa(&full_bar[stage], 0);
                        expect_tx_cluster(fb, kStageBytes);
                        tma_load_2sm(&tmap_a, fb, smem_a + stage * kABytes, kc, arow);
                        tma_load_2sm(&tmap_b, fb, smem_b + stage * kBBytes, kc, brow);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA; one elected thread issues) =====================
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = pair; t < num_tiles; t += npairs) {
                const TileInfo ti = tile_of<kVarK>(t, tile_start, off, G, ntn, M, K);
                if (ti.nkb == 0) continue;  // empty reduction: the epilogue writes zeros
                const int nw = min(BN, N - ti.n0);
                const int n_mma = (nw + 15) & ~15;
                const uint32_t idesc = make_idesc2(n_mma, is_half(ti, nw) ? BM / 2 : BM);
                const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
                mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < ti.nkb; ++kb) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    if (elect_one()) {
                        mma2_kblock<2>(tmem_d, make_desc(smem_u32(smem_a + stage * kABytes)),
                                       make_desc(smem_u32(smem_b + stage * kBBytes)), idesc, kb > 0 ? 1u : 0u,
                                       smem_u32(&empty_bar[stage]));
                        if (kb == ti.nkb - 1) commit_both(&tfull_bar[acc]);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (++acc == kAccBufs) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // ===================== epilogue (warps 2..5, both CTAs) =====================
        const int quarter = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = pair; t < num_tiles; t += npairs) {
            const TileInfo ti = tile_of<kVarK>(t, tile_start, off, G, ntn, M, K);
            const int nw_tile = min(BN, N - ti.n0);
            // this warp's rows and columns of the tile: full tiles — 32 rows of
            // the CTA's 128, every column; half tiles — 32 rows of the CTA's 64,
            // one half of the columns (TMEM lanes 64-127 hold the second half)
            const bool hf = is_half(ti, nw_tile);
            const int wrow = hf ? (BMC / 2) * static_cast<int>(rank) + (quarter & 1) * 32
                                : BMC * static_cast<int>(rank) + quarter * 32;  // first row of this warp
            const int cbase = hf ? (quarter >> 1) * (nw_tile / 2) : 0;           // first column of this warp
            const int nw = hf ? nw_tile / 2 : nw_tile;                          // columns of this warp
            const int r = wrow + lane;
            const bool row_ok = r < ti.rows_left;
            OutT* drow = D + (kVarK ? static_cast<size_t>(ti.g) * M * N : 0) +
                         static_cast<size_t>(ti.row0 + r) * N + ti.n0 + cbase;
            if (ti.nkb == 0) {  // nothing to reduce: zeros, no accumulator used
                if (row_ok)
                    for (int c = 0; c < nw; ++c) drow[c] = static_cast<OutT>(0.f);
                continue;
            }
            // ReLU masks as bits: one word per (row, 32 columns), ceil(N/32) words per row;
            // the tile's words are loaded before the accumulator wait (off the critical path)
            const int mwords = (N + 31) >> 5;
            const uint32_t* mrow = mbits_in ? mbits_in + static_cast<size_t>(ti.row0 + r) * mwords +
                                                  ((ti.n0 + cbase) >> 5)
                                            : nullptr;
            uint32_t mpre[BN / 32];
#pragma unroll
            for (int q = 0; q < BN / 32; ++q) mpre[q] = (mrow && row_ok && 32 * q < nw) ? __ldg(mrow + q) : 0u;
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            // fused addend (shared experts after the routed combine, layer.cu):
            // D = bf16(addf + float(bf16(acc))) once the combine has published
            // this warp's 128-row block (ready[block] == rows in the block)
            const float* arow_f = nullptr;
            if (addf && ti.row0 + wrow < off[G]) {
                const int blk = (ti.row0 + wrow) >> 7;
                const unsigned want = static_cast<unsigned>(min(128, off[G] - (blk << 7)) * ready_mult);
                if (lane == 0) {
                    for (uint32_t it = 0;; ++it) {
                        unsigned v;
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + blk) : "memory");
                        if (v >= want) break;
                        __nanosleep(200);
                        if (it == (1u << 27)) asm volatile("trap;");  // a producer never published: fail loudly
                    }
                }
                __syncwarp();
                if (row_ok) arow_f = addf + static_cast<size_t>(ti.row0 + r) * N + ti.n0 + cbase;
            }
            uint32_t* orow = mbits_out ? mbits_out + static_cast<size_t>(ti.row0 + r) * mwords +
                                             ((ti.n0 + cbase) >> 5)
                                       : nullptr;
            uint32_t* etile = reinterpret_cast<uint32_t*>(smem + kEpiOff + (warp - 2) * kEpiWarpBytes);
            // bf16 output boxes of 32 rows x 64 columns leave through TMA stores when
            // the warp's 32 rows all belong to the group (a box must not touch the
            // next group's rows)
            const bool use_tma = sizeof(OutT) == 2 && !kVarK && tma_d && ti.rows_left - wrow >= 32 && (nw & 63) == 0;
            for (int c0 = 0; c0 < nw; c0 += 32) {
                // this chunk's mask word; the prefetched words shift down one
                // per chunk (constant indices keep them in registers)
                const uint32_t mask_w = mpre[0];
#pragma unroll
                for (int q = 0; q + 1 < BN / 32; ++q) mpre[q] = mpre[q + 1];
                uint32_t v[32];
                tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                              static_cast<uint32_t>(acc * BN + c0),
                          v);
                if (coalesced) {
                    float f[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        f[i] = __uint_as_float(v[i]);
                        if (relu) f[i] = fmaxf(f[i], 0.f);
                    }
                    const int cn = min(32, nw - c0);
                    if (mrow && row_ok) {
                        const uint32_t mw = mask_w;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!((mw >> i) & 1u)) f[i] = 0.f;
                    }
                    store_chunk_coalesced<OutT>(etile, f, D + (kVarK ? static_cast<size_t>(ti.g) * M * N : 0),
                                                static_cast<size_t>(N), static_cast<size_t>(ti.row0 + wrow),
                                                ti.rows_left - wrow, ti.n0 + cbase + c0, cn, lane);
                    continue;
                }
                if (!row_ok) continue;
                float f[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    f[i] = __uint_as_float(v[i]);
                    if (relu) f[i] = fmaxf(f[i], 0.f);
                }
                const int cn = min(32, nw - c0);
                if (mrow) {
                    const uint32_t mw = mask_w;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!((mw >> i) & 1u)) f[i] = 0.f;
                }
                if (arow_f) {  // same arithmetic as the combine's addend: fp32 sum + bf16(shared)
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 pv;
                        asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                                     : "=f"(pv.x), "=f"(pv.y), "=f"(pv.z), "=f"(pv.w)
                                     : "l"(arow_f + c0 + 4 * q));
                        f[4 * q + 0] = pv.x + __bfloat162float(__float2bfloat16_rn(f[4 * q + 0]));
                        f[4 * q + 1] = pv.y + __bfloat162float(__float2bfloat16_rn(f[4 * q + 1]));
                        f[4 * q + 2] = pv.z + __bfloat162float(__float2bfloat16_rn(f[4 * q + 2]));
                        f[4 * q + 3] = pv.w + __bfloat162float(__float2bfloat16_rn(f[4 * q + 3]));
                    }
                }
                if constexpr (sizeof(OutT) == 2) {
                    if (cn == 32 && (N & 7) == 0) {
                        int4* dst = reinterpret_cast<int4*>(drow + c0);
                        uint8_t* srow = reinterpret_cast<uint8_t*>(etile) + lane * 128;  // staging row (128B swizzle)
                        if (use_tma && (c0 & 63) == 0) {
                            if (lane == 0) tma_store_wait_read();  // the previous box left the buffer
                            __syncwarp();
                        }
                        uint32_t mw = 0;  // ReLU mask of the stored bf16 values (bit i: y_i != 0)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint32_t u[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                u[e] = pack_bf16(f[8 * q + 2 * e], f[8 * q + 2 * e + 1]);
                                if (orow) {
                                    mw |= ((u[e] & 0x7FFFu) ? 1u : 0u) << (8 * q + 2 * e);
                                    mw |= ((u[e] & 0x7FFF0000u) ? 1u : 0u) << (8 * q + 2 * e + 1);
                                }
                            }
                            const int4 o = make_int4(static_cast<int>(u[0]), static_cast<int>(u[1]),
                                                     static_cast<int>(u[2]), static_cast<int>(u[3]));
                            if (use_tma) {
                                const int chunk = ((c0 & 32) >> 3) + q;  // 16-byte chunk in the 128-byte row
                                *reinterpret_cast<int4*>(srow + ((chunk ^ (lane & 7)) << 4)) = o;
                            } else {
                                dst[q] = o;
                            }
                        }
                        if (orow) orow[c0 >> 5] = mw;
                        if (use_tma && (c0 & 63) == 32) {
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            __syncwarp();
                            if (lane == 0) tma_store_2d(&tmap_d, etile, ti.n0 + cbase + c0 - 32, ti.row0 + wrow);
                        }
                    } else {
                        uint32_t mw = 0;
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            if (i >= cn) continue;
                            const __nv_bfloat16 b = __float2bfloat16_rn(f[i]);
                            drow[c0 + i] = b;
                            mw |= (__bfloat162float(b) != 0.f ? 1u : 0u) << i;
                        }
                        if (orow) orow[c0 >> 5] = mw;
                    }
                } else {
                    if (cn == 32 && (N & 3) == 0) {
                        float4* dst = reinterpret_cast<float4*>(drow + c0);
#pragma unroll
                        for (int q = 0; q < 8; ++q) dst[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < cn) drow[c0 + i] = f[i];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_cluster(mapa(&tempty_bar[acc], 0));
            if (++acc == kAccBufs) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    if (tma_d && warp >= 2 && lane == 0) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the peer is done with the pair's TMEM and barriers
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// Weight-gradient GEMM with MN-major operands, straight on the grouped
// activations (no transposes):  D_g[M, N] = sum_{r in group g} A[r, :]^T B[r, :]
// A [rows, M], B [rows, N] row-major bf16 (M, N contiguous).  Each K block is
// 64 rows; a group's last partial block comes from zero-padded tail copies
// (at_tail/bt_tail: [G*64, M|N]) so other groups' rows never leak in.
// smem per CTA and stage: two 64(MN) x 64(K) boxes of A and of B, 128B
// swizzle; UMMA descriptors: LBO = 8 KB (next 64-wide MN atom), SBO = 1 KB
// (next 8 K-rows), K advances 2 KB per 16-row MMA; a_major = b_major = MN.
__device__ __forceinline__ uint64_t make_desc_mn(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(8192 >> 4) << 16;  // LBO: MN atom stride
    d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO: 8-row K group stride
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
__device__ __forceinline__ uint32_t make_idesc2_mn(int n) { return make_idesc2(n) | (1u << 15) | (1u << 16); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    grouped_wgrad_mn_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                            const __grid_constant__ CUtensorMap tmap_at, const __grid_constant__ CUtensorMap tmap_bt,
                            const int32_t* __restrict__ group_rows, int G, int M, int N, float* __restrict__ D,
                            int coalesced, const __grid_constant__ CUtensorMap tmap_d, int tma_store,
                            int transpose_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + kStages * kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + kStages;
    uint64_t* tfull_bar = bars + 2 * kStages;
    uint64_t* tempty_bar = bars + 2 * kStages + kAccBufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kAccBufs);
    int32_t* tile_start = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 1024);
    int32_t* roff = tile_start + kMaxGroups + 1;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1;
    const int npairs = gridDim.x >> 1;
    const int ntn = (N + BN - 1) / BN;
    const int ntm = (M + BM - 1) / BM;

    if (threadIdx.x == 0) {
        int r = 0;
        for (int g = 0; g < G; ++g) {
            tile_start[g] = g * ntm * ntn;
            roff[g] = r;
            r += group_rows[g];
        }
        tile_start[G] = G * ntm * ntn;
        roff[G] = r;
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 2);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
        prefetch_tmap(&tmap_at);
        prefetch_tmap(&tmap_bt);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int num_tiles = tile_start[G];
    auto info = [&](int t, int& g, int& row0, int& n0, int& nkb, int& rows_g) {
        g = t / (ntm * ntn);
        const int local = t - g * ntm * ntn;
        row0 = (local / ntn) * BM;
        n0 = (local % ntn) * BN;
        rows_g = roff[g + 1] - roff[g];
        nkb = (rows_g + BK - 1) / BK;
    };

    if (warp == 0) {
        // TMA producer: the whole warp runs the loop (uniform control flow)
        // and one elected thread issues; a `lane == 0` branch made ptxas wrap
        // every TMA in an elect/broadcast loop, and with four loads per stage
        // the producer fell behind the MMAs (ncu: the MMA warp waited on full
        // stages while the producer never waited on empty ones)
        int stage = 0;
        uint32_t phase = 0;
        for (int t = pair; t < num_tiles; t += npairs) {
            int g, row0, n0, nkb, rows_g;
            info(t, g, row0, n0, nkb, rows_g);
            const int nw = min(BN, N - n0);
            const int n_mma = (nw + 15) & ~15;
            const int am = row0 + BMC * static_cast<int>(rank);
            const int bn = n0 + (n_mma / 2) * static_cast<int>(rank);
            const int r0 = roff[g];
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&empty_bar[stage], phase ^ 1);
                const bool tail = (kb + 1) * BK > rows_g;
                const int kr = tail ? g * BK : r0 + kb * BK;
                if (elect_one()) {
                    const uint32_t fb = mapa(&full_bar[stage], 0);
                    expect_tx_cluster(fb, kStageBytes);
                    const CUtensorMap* ma = tail ? &tmap_at : &tmap_a;
                    const CUtensorMap* mb = tail ? &tmap_bt : &tmap_b;
                    uint8_t* sa = smem_a + stage * kABytes;
                    uint8_t* sb = smem_b + stage * kBBytes;
                    tma_load_2sm(ma, fb, sa, am, kr);
                    tma_load_2sm(ma, fb, sa + 8192, am + 64, kr);
                    tma_load_2sm(mb, fb, sb, bn, kr);
                    tma_load_2sm(mb, fb, sb + 8192, bn + 64, kr);
                }
                __syncwarp();
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = pair; t < num_tiles; t += npairs) {
                int g, row0, n0, nkb, rows_g;
                info(t, g, row0, n0, nkb, rows_g);
                if (nkb == 0) continue;
                const int nw = min(BN, N - n0);
                const int n_mma = (nw + 15) & ~15;
                const uint32_t idesc = make_idesc2_mn(n_mma);
                const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
                mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    // 16 K-rows = 2 KB per MMA
                    if (elect_one()) {
                        mma2_kblock<128>(tmem_d, make_desc_mn(smem_u32(smem_a + stage * kABytes)),
                                         make_desc_mn(smem_u32(smem_b + stage * kBBytes)), idesc, kb > 0 ? 1u : 0u,
                                         smem_u32(&empty_bar[stage]));
                        if (kb == nkb - 1) commit_both(&tfull_bar[acc]);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (++acc == kAccBufs) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        const int quarter = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = pair; t < num_tiles; t += npairs) {
            int g, row0, n0, nkb, rows_g;
            info(t, g, row0, n0, nkb, rows_g);
            const int nw = min(BN, N - n0);
            const int r = BMC * static_cast<int>(rank) + quarter * 32 + lane;
            const bool row_ok = row0 + r < M;
            float* drow = D + static_cast<size_t>(g) * M * N + static_cast<size_t>(row0 + r) * N + n0;
            if (nkb == 0) {
                if (row_ok)
                    for (int c = 0; c < nw; ++c) drow[c] = 0.f;
                continue;
            }
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            uint32_t* etile = reinterpret_cast<uint32_t*>(smem + kEpiOff + (warp - 2) * kEpiWarpBytes);
            const int wrow = BMC * static_cast<int>(rank) + quarter * 32;
            for (int c0 = 0; c0 < nw; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN + c0),
                          v);
                if (transpose_out) {
                    // D_g^T: output row n holds the M values of column n ([G, N, M]);
                    // lane l (row m = l of the warp) writes element (n = i, m = l)
                    if (tma_store) {
                        // 32 (n) x 32 (m) box, 128B-swizzled, stored by TMA (map [G*N, M])
                        if (lane == 0) tma_store_wait_read();
                        __syncwarp();
                        uint8_t* tb = reinterpret_cast<uint8_t*>(etile);
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            *reinterpret_cast<uint32_t*>(tb + i * 128 + ((((lane >> 2) ^ (i & 7))) << 4) +
                                                         (lane & 3) * 4) = v[i];
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) tma_store_2d(&tmap_d, etile, row0 + wrow, g * N + n0 + c0);
                    } else if (row_ok) {
                        const int cn = min(32, nw - c0);
                        float* dt = D + static_cast<size_t>(g) * M * N + static_cast<size_t>(n0 + c0) * M + row0 + r;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < cn) dt[static_cast<size_t>(i) * M] = __uint_as_float(v[i]);
                    }
                    continue;
                }
                if (tma_store) {
                    // 32 x 32 fp32 box through 128B-swizzled smem, stored by TMA
                    // (the D map is [G*M, N]; M % 256 == 0, so a box never
                    // crosses into the next group)
                    if (lane == 0) tma_store_wait_read();  // the previous box left the buffer
                    __syncwarp();
                    uint8_t* row = reinterpret_cast<uint8_t*>(etile) + lane * 128;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<uint4*>(row + ((q ^ (lane & 7)) << 4)) =
                            make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) tma_store_2d(&tmap_d, etile, n0 + c0, g * M + row0 + wrow);
                    continue;
                }
                if (coalesced) {
                    float f[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
                    store_chunk_coalesced<float>(etile, f, D + static_cast<size_t>(g) * M * N, static_cast<size_t>(N),
                                                 static_cast<size_t>(row0 + wrow), M - (row0 + wrow), n0 + c0,
                                                 min(32, nw - c0), lane);
                    continue;
                }
                if (!row_ok) continue;
                const int cn = min(32, nw - c0);
                if (cn == 32 && (N & 3) == 0) {
                    float4* dst = reinterpret_cast<float4*>(drow + c0);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < cn) drow[c0 + i] = __uint_as_float(v[i]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_cluster(mapa(&tempty_bar[acc], 0));
            if (++acc == kAccBufs) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    if (tma_store && warp >= 2 && lane == 0) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
    }
}

// Tail staging: the last (rows_g mod 64) rows of every group, zero-padded to
// 64 rows, for A [rows, C] -> tail [G*64, C].  One block per (group, row),
// 16-byte vectors (C % 8 == 0).
__global__ void wgrad_tail_kernel(const __nv_bfloat16* __restrict__ X, int C, const int32_t* __restrict__ group_rows,
                                  int G, __nv_bfloat16* __restrict__ tail) {
    const int g = blockIdx.x, rr = blockIdx.y;
    __shared__ int s_r0, s_rows;
    if (threadIdx.x == 0) {
        int r0 = 0;
        for (int q = 0; q < g; ++q) r0 += group_rows[q];
        s_r0 = r0;
        s_rows = group_rows[g];
    }
    __syncthreads();
    const int rem = s_rows & 63;
    int4* dst = reinterpret_cast<int4*>(tail + (static_cast<size_t>(g) * 64 + rr) * C);
    const int nv = C >> 3;
    if (rr < rem) {
        const int4* src = reinterpret_cast<const int4*>(X + static_cast<size_t>(s_r0 + s_rows - rem + rr) * C);
        for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = src[v];
    } else {
        for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = make_int4(0, 0, 0, 0);
    }
}

// Split-K of one long reduction into `splits` row groups (each a multiple of
// 64 rows but the last), so a single-group weight gradient with few output
// tiles (shared experts, gate) fills every SM pair.
__global__ void split_rows_kernel(int rows, int splits, int32_t* __restrict__ out) {
    const int g = threadIdx.x;
    if (g >= splits) return;
    const int per = ((rows + splits - 1) / splits + 63) & ~63;
    const int r0 = min(rows, g * per);
    out[g] = min(rows, r0 + per) - r0;
}

// D[m, n] = sum over s ascending of P[s, m, n] for n < Nv (P row stride N);
// four columns per thread (Nv % 4 == 0, N % 4 == 0).
__global__ void __launch_bounds__(256) sum_partials_kernel(const float* __restrict__ P, int splits, int M, int N,
                                                           int Nv, float* __restrict__ D) {
    const int nq = Nv >> 2;
    const long long total = static_cast<long long>(M) * nq;
    const size_t plane = static_cast<size_t>(M) * N;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(i / nq), c = static_cast<int>(i % nq) * 4;
        const float* p = P + static_cast<size_t>(m) * N + c;
        float4 acc = __ldg(reinterpret_cast<const float4*>(p));
        for (int sp = 1; sp < splits; ++sp) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(p + sp * plane));
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        *reinterpret_cast<float4*>(D + static_cast<size_t>(m) * Nv + c) = acc;
    }
}

}  // namespace tc2

// ---------------------------------------------------------------- host side
// fp32 outputs (weight gradients) leave the epilogue through a per-warp
// shared-memory transpose as whole-row segments (measured: wgrad 1.59 ->
// 1.23 ms); bf16 outputs keep the direct per-row 16-byte stores, which
// measured faster.  XMOE_EPI=0 selects the direct stores everywhere.
// weight gradients leave through TMA stores (XMOE_WGRAD_TMA=0: the
// shared-memory transpose + coalesced stores)
// bf16 GEMM outputs leave through TMA stores where a warp's rows are whole
// (XMOE_FWD_TMA=0: direct per-row stores)
static bool fwd_tma_store() {
    static const bool v = [] {
        const char* e = std::getenv("XMOE_FWD_TMA");
        return !(e && std::atoi(e) == 0);
    }();
    return v;
}
// a group's last row tile with <= 128 rows runs as an M = 128 pair MMA
// (XMOE_HALF_TILES=0: padded to 256 rows like every other tile)
static bool half_tiles() {
    static const bool v = [] {
        const char* e = std::getenv("XMOE_HALF_TILES");
        return !(e && std::atoi(e) == 0);
    }();
    return v;
}
static bool wgrad_tma_store() {
    static const bool v = [] {
        const char* e = std::getenv("XMOE_WGRAD_TMA");
        return !(e && std::atoi(e) == 0);
    }();
    return v;
}
static int epi_coalesced() {
    static const int v = [] {
        const char* e = std::getenv("XMOE_EPI");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        XMOE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        require(p != nullptr && q == cudaDriverEntryPointSuccess, XMOE_ERR_CUDA,
                "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// 2D bf16 K-major tensor [rows, K] with a (box_rows x 64) 128B-swizzled box.
static CUtensorMap make_tmap(const void* base, long long rows, long long K, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(tc::BK), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                    const_cast<void*>(base), dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(XMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

template <typename OutT>
static void launch_tc(const void* A, long long rows, int K, const int32_t* rows_per_group, int G,
                      const void* B, int N, OutT* D, int relu, cudaStream_t st) {
    require(G >= 1 && G <= tc::kMaxGroups, XMOE_ERR_VALIDATION, "grouped gemm: 1 <= groups <= 1024");
    require(K % 8 == 0 && K > 0, XMOE_ERR_VALIDATION, "bf16 path requires K % 8 == 0");
    require(N % 16 == 0 && N > 0, XMOE_ERR_VALIDATION, "bf16 path requires N % 16 == 0");
    require((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
            XMOE_ERR_VALIDATION, "bf16 operands must be 16-byte aligned");
    if (rows == 0) return;
    const CUtensorMap ta = make_tmap(A, rows, K, tc::BM);
    const CUtensorMap tb = make_tmap(B, static_cast<long long>(G) * N, K, tc::BN);
    static bool attr_set = false;
    if (!attr_set) {
        XMOE_CUDA(cudaFuncSetAttribute(tc::grouped_gemm_tc_kernel<OutT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(tc::kSmemBytes)));
        attr_set = true;
    }
    // Upper bound on tiles from the row bound: every group could be one row
    // short of a tile boundary.
    const long long max_tiles =
        ((rows + tc::BM - 1) / tc::BM + G) * static_cast<long long>((N + tc::BN - 1) / tc::BN);
    int sms = 0;
    XMOE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = static_cast<int>(max_tiles < sms ? max_tiles : sms);
    tc::grouped_gemm_tc_kernel<OutT><<<grid, tc::kThreads, tc::kSmemBytes, st>>>(
        ta, tb, rows_per_group, G, N, K, D, relu);
    XMOE_LAUNCH_CHECK();
}

template <typename OutT, bool kVarK>
static void launch_tc2(const void* A, long long a_rows, long long a_cols, const int32_t* group_sizes, int G,
                       const void* B, long long b_rows, int M, int N, int K, OutT* D, int relu,
                       const uint32_t* mbits_in, uint32_t* mbits_out, long long tile_bound, cudaStream_t st,
                       const int32_t* a_idx = nullptr, long long idx_rows = 0) {
    require(G >= 1 && G <= tc2::kMaxGroups, XMOE_ERR_VALIDATION, "grouped gemm: 1 <= groups <= 1024");
    require(a_cols % 8 == 0 && a_cols > 0, XMOE_ERR_VALIDATION, "bf16 path requires K % 8 == 0");
    require(N % 32 == 0 && N > 0, XMOE_ERR_VALIDATION, "bf16 2-CTA path requires N % 32 == 0");
    require((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
            XMOE_ERR_VALIDATION, "bf16 operands must be 16-byte aligned");
    if (a_rows == 0 || tile_bound == 0) return;
    const CUtensorMap ta = make_tmap(A, a_rows, a_cols, a_idx ? 1 : tc2::BMC);  // gather4: {BK, 1} boxes
    const CUtensorMap tb = make_tmap(B, b_rows, a_cols, tc2::BN / 2);
    // bf16 D [rows, N] for the TMA-store epilogue (boxes of 64 columns x 32 rows, 128B swizzle)
    const long long d_rows = a_idx ? idx_rows : a_rows;
    const bool tma_d = sizeof(OutT) == 2 && !kVarK && fwd_tma_store() && N % 64 == 0 && d_rows > 0;
    CUtensorMap td{};
    if (tma_d) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(d_rows)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(N) * 2};
        const cuuint32_t box[2] = {64, 32};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = get_encode()(&td, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(XMOE_ERR_CUDA, "cuTensorMapEncodeTiled (D) failed: " + std::to_string(r));
    }
    static bool attr_set = false;
    if (!attr_set) {
        XMOE_CUDA(cudaFuncSetAttribute(tc2::grouped_gemm_tc2_kernel<OutT, kVarK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(tc2::kSmemBytes)));
        attr_set = true;
    }
    int sms = 0;
    XMOE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    long long cap_pairs = sms / 2;
    if (g_gemm_sm_limit > 0 && g_gemm_sm_limit / 2 < cap_pairs) cap_pairs = g_gemm_sm_limit / 2;
    static const int env_sms = [] {  // XMOE_GEMM_SMS: cap on every 2-CTA GEMM grid (A/B, SM partitions)
        const char* e = std::getenv("XMOE_GEMM_SMS");
        return e ? std::atoi(e) : 0;
    }();
    if (env_sms > 0 && env_sms / 2 < cap_pairs) cap_pairs = env_sms / 2;
    const long long pairs = tile_bound < cap_pairs ? tile_bound : cap_pairs;
    tc2::grouped_gemm_tc2_kernel<OutT, kVarK><<<static_cast<int>(2 * pairs), tc2::kThreads, tc2::kSmemBytes, st>>>(
        ta, tb, group_sizes, G, M, N, K, D, relu, mbits_in, mbits_out,
        sizeof(OutT) == 4 && !mbits_out ? epi_coalesced() : 0, a_idx, static_cast<int>(idx_rows), td, tma_d ? 1 : 0,
        half_tiles() ? 1 : 0, kVarK ? nullptr : g_gemm_addf, kVarK ? nullptr : g_gemm_ready, g_gemm_ready_mult);
    XMOE_LAUNCH_CHECK();
}

// Grouped-M: D[rows, N] over row segments (forward and dgrad).
template <typename OutT>
static void launch_tc2_rows(const void* A, long long rows, int K, const int32_t* rows_per_group, int G,
                            const void* B, int N, OutT* D, int relu, const uint32_t* mbits_in, uint32_t* mbits_out,
                            cudaStream_t st, const int32_t* a_idx = nullptr, long long phys_rows = 0) {
    const long long bound = ((rows + tc2::BM - 1) / tc2::BM + G) * static_cast<long long>((N + tc2::BN - 1) / tc2::BN);
    launch_tc2<OutT, false>(A, a_idx ? phys_rows : rows, K, rows_per_group, G, B, static_cast<long long>(G) * N, 0, N,
                            K, D, relu, mbits_in, mbits_out, bound, st, a_idx, rows);
}

// The expert FFN GEMMs run on the 2-CTA kernel; XMOE_GEMM=1cta selects the
// single-CTA kernel (kept for A/B measurement and for N % 32 != 0).
static bool use_2cta(int N) {
    static const int mode = [] {
        const char* e = std::getenv("XMOE_GEMM");
        return (e && std::string(e) == "1cta") ? 1 : 2;
    }();
    return mode == 2 && N % 32 == 0;
}

bool gemm_2cta_enabled(int N) { return use_2cta(N); }

void launch_grouped_gemm_bf16(const void* A, long long rows, int K, const int32_t* rows_per_group,
                              int G, const void* B, int N, void* D, int relu, cudaStream_t st, uint32_t* mbits_out) {
    require(!mbits_out || (relu && use_2cta(N)), XMOE_ERR_VALIDATION, "ReLU mask output needs the 2-CTA ReLU GEMM");
    require(!g_gemm_addf || (use_2cta(N) && !relu && !mbits_out), XMOE_ERR_VALIDATION,
            "fused addend needs the 2-CTA GEMM without ReLU");
    if (use_2cta(N))
        launch_tc2_rows<__nv_bfloat16>(A, rows, K, rows_per_group, G, B, N, static_cast<__nv_bfloat16*>(D), relu,
                                       nullptr, mbits_out, st);
    else
        launch_tc<__nv_bfloat16>(A, rows, K, rows_per_group, G, B, N, static_cast<__nv_bfloat16*>(D), relu, st);
}

void launch_grouped_gemm_bf16_gather(const void* A, long long phys_rows, long long rows, int K,
                                     const int32_t* rows_per_group, int G, const void* B, int N, void* D, int relu,
                                     const int32_t* a_idx, cudaStream_t st) {
    require(use_2cta(N), XMOE_ERR_VALIDATION, "row-gathered GEMM needs the 2-CTA kernel (N % 32 == 0)");
    require(phys_rows < (1LL << 31) && rows >= 1, XMOE_ERR_VALIDATION, "row-gathered GEMM: 1 <= rows, phys rows < 2^31");
    launch_tc2_rows<__nv_bfloat16>(A, rows, K, rows_per_group, G, B, N, static_cast<__nv_bfloat16*>(D), relu,
                                   nullptr, nullptr, st, a_idx, phys_rows);
}

void launch_grouped_gemm_bf16_mask(const void* A, long long rows, int K, const int32_t* rows_per_group, int G,
                                   const void* B, int N, void* D, const uint32_t* mbits, cudaStream_t st) {
    launch_tc2_rows<__nv_bfloat16>(A, rows, K, rows_per_group, G, B, N, static_cast<__nv_bfloat16*>(D), 0, mbits,
                                   nullptr, st);
}

// Grouped-K (weight gradients): D_g[M, N] (fp32) = A[:, Kg] . B[:, Kg]^T where
// A [M, Ktot] and B [N, Ktot] are K-major and group g owns the next
// k_per_group[g] columns (multiples of 64, zero-padded).
void launch_grouped_wgrad_bf16(const void* A, int M, long long Ktot, const int32_t* k_per_group, int G,
                               const void* B, int N, float* D, cudaStream_t st) {
    require(Ktot % 64 == 0, XMOE_ERR_VALIDATION, "wgrad: K segments must be padded to 64");
    const long long bound = static_cast<long long>(G) * ((M + tc2::BM - 1) / tc2::BM) * ((N + tc2::BN - 1) / tc2::BN);
    launch_tc2<float, true>(A, M, Ktot, k_per_group, G, B, N, M, N, 0, D, 0, nullptr, nullptr, bound, st);
}

// MN-major grouped weight gradient straight on the grouped activations.
// B has b_cols physical columns (b_cols <= N); columns past them read as
// zeros (TMA out-of-bounds fill), so N may be padded up to a multiple of 128.
static void wgrad_mn_impl(const void* A, int M, const void* B, int N, int b_cols, long long rows,
                          const int32_t* group_rows, int G, void* tail_a, void* tail_b, float* D, cudaStream_t st,
                          bool transpose_out = false) {
    require(G >= 1 && G <= tc2::kMaxGroups, XMOE_ERR_VALIDATION, "wgrad: 1 <= groups <= 1024");
    require(M % 64 == 0 && N % 128 == 0, XMOE_ERR_VALIDATION, "wgrad (MN-major) needs M % 64 == 0, N % 128 == 0");
    require(b_cols % 8 == 0 && b_cols <= N, XMOE_ERR_VALIDATION, "wgrad (MN-major): B columns % 8 == 0, <= N");
    tc2::wgrad_tail_kernel<<<dim3(G, 64), 128, 0, st>>>(static_cast<const __nv_bfloat16*>(A), M, group_rows, G,
                                                        static_cast<__nv_bfloat16*>(tail_a));
    XMOE_LAUNCH_CHECK();
    tc2::wgrad_tail_kernel<<<dim3(G, 64), 128, 0, st>>>(static_cast<const __nv_bfloat16*>(B), b_cols, group_rows, G,
                                                        static_cast<__nv_bfloat16*>(tail_b));
    XMOE_LAUNCH_CHECK();
    const long long r = rows > 0 ? rows : 1;
    const CUtensorMap ta = make_tmap(A, r, M, 64);
    const CUtensorMap tb = make_tmap(B, r, b_cols, 64);
    const CUtensorMap tat = make_tmap(tail_a, 64LL * G, M, 64);
    const CUtensorMap tbt = make_tmap(tail_b, 64LL * G, b_cols, 64);
    // fp32 D [G*M, N] for the TMA-store epilogue: boxes of 32 x 32, 128B swizzle
    // (transposed: D_g^T, map [G*N, M])
    const bool tma_store = wgrad_tma_store() && M % tc2::BM == 0 && N % 32 == 0;
    CUtensorMap td{};
    if (tma_store) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(transpose_out ? M : N),
                                    static_cast<cuuint64_t>(G) * (transpose_out ? N : M)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(transpose_out ? M : N) * 4};
        const cuuint32_t box[2] = {32, 32};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = get_encode()(&td, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(XMOE_ERR_CUDA, "cuTensorMapEncodeTiled (wgrad D) failed: " + std::to_string(r));
    }
    static bool attr_set = false;
    if (!attr_set) {
        XMOE_CUDA(cudaFuncSetAttribute(tc2::grouped_wgrad_mn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(tc2::kSmemBytes)));
        attr_set = true;
    }
    int sms = 0;
    XMOE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long tiles = static_cast<long long>(G) * ((M + tc2::BM - 1) / tc2::BM) * ((N + tc2::BN - 1) / tc2::BN);
    long long cap_pairs = sms / 2;
    if (g_gemm_sm_limit > 0 && g_gemm_sm_limit / 2 < cap_pairs) cap_pairs = g_gemm_sm_limit / 2;
    const long long pairs = tiles < cap_pairs ? tiles : cap_pairs;
    tc2::grouped_wgrad_mn_kernel<<<static_cast<int>(2 * pairs), tc2::kThreads, tc2::kSmemBytes, st>>>(
        ta, tb, tat, tbt, group_rows, G, M, N, D, epi_coalesced(), td, tma_store ? 1 : 0, transpose_out ? 1 : 0);
    XMOE_LAUNCH_CHECK();
}

// D_g^T [N, M] = (A_g^T B_g)^T: the same product written transposed, so that
// an output with few rows (M) and many columns runs as M = the long side
// (whole 256-row tiles) — the routed W2 gradient, M = H, N = F.
void launch_grouped_wgrad_mn_t(const void* A, int M, const void* B, int N, long long rows,
                               const int32_t* group_rows, int G, void* tail_a, void* tail_b, float* D,
                               cudaStream_t st) {
    wgrad_mn_impl(A, M, B, N, N, rows, group_rows, G, tail_a, tail_b, D, st, true);
}

void launch_grouped_wgrad_mn(const void* A, int M, const void* B, int N, long long rows,
                             const int32_t* group_rows, int G, void* tail_a, void* tail_b, float* D,
                             cudaStream_t st) {
    wgrad_mn_impl(A, M, B, N, N, rows, group_rows, G, tail_a, tail_b, D, st);
}

// One weight gradient D[M, Nb] = A^T B over all `rows` (A [rows, M], B
// [rows, Nb], bf16, MN-major), split into `splits` K segments whose fp32
// partials ([splits, M, roundup(Nb, 128)] in `partial`) are summed in order
// (deterministic).  tails: 64 * splits rows of M and of Nb columns;
// split_rows: `splits` ints of device scratch.
void launch_wgrad_mn_split(const void* A, int M, const void* B, int Nb, long long rows, int splits,
                           int32_t* split_rows, void* tail_a, void* tail_b, float* partial, float* D,
                           cudaStream_t st) {
    require(splits >= 1 && splits <= 32 && rows < (1LL << 31), XMOE_ERR_VALIDATION,
            "split wgrad: 1 <= splits <= 32, rows < 2^31");
    require(Nb % 8 == 0, XMOE_ERR_VALIDATION, "split wgrad: columns % 8 == 0");
    const int N = (Nb + 127) / 128 * 128;
    tc2::split_rows_kernel<<<1, 32, 0, st>>>(static_cast<int>(rows), splits, split_rows);
    XMOE_LAUNCH_CHECK();
    wgrad_mn_impl(A, M, B, N, Nb, rows, split_rows, splits, tail_a, tail_b, partial, st);
    const long long quads = static_cast<long long>(M) * (Nb / 4);
    long long blocks = (quads + 255) / 256;
    if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
    tc2::sum_partials_kernel<<<static_cast<int>(blocks < 1 ? 1 : blocks), 256, 0, st>>>(partial, splits, M, N, Nb, D);
    XMOE_LAUNCH_CHECK();
}

bool gate_route_supported(int E, int k, int H) { return E >= 16 && E <= 256 && E % 16 == 0 && k >= 1 && k <= 8 && H % 8 == 0; }

void launch_gate_route(const void* x, int S, int H, const void* gate_kmajor, int E, int k, int renorm, int32_t* top,
                       double* weights, float* logits, int32_t* counts, cudaStream_t st) {
    require(gate_route_supported(E, k, H), XMOE_ERR_VALIDATION,
            "fused gate: 16 <= num_experts <= 256 (multiple of 16), top_k <= 8, model_dim % 8 == 0");
    if (S == 0) return;
    const CUtensorMap ta = make_tmap(x, S, H, tc::BM);
    const CUtensorMap tb = make_tmap(gate_kmajor, E, H, tc::BN);
    static bool attr_set = false;
    if (!attr_set) {
        XMOE_CUDA(cudaFuncSetAttribute(tc::gate_route_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(tc::kSmemBytes)));
        attr_set = true;
    }
    const int tiles = (S + tc::BM - 1) / tc::BM;
    const int grid = tiles < kNumSMs ? tiles : kNumSMs;
    tc::gate_route_kernel<8><<<grid, tc::kThreads, tc::kSmemBytes, st>>>(ta, tb, S, E, H, k, renorm, top, weights,
                                                                         logits, counts);
    XMOE_LAUNCH_CHECK();
}

void launch_grouped_gemm_bf16_f32out(const void* A, long long rows, int K,
                                     const int32_t* rows_per_group, int G, const void* B, int N,
                                     float* D, int relu, cudaStream_t st) {
    launch_tc<float>(A, rows, K, rows_per_group, G, B, N, D, relu, st);
}

}  // namespace xmoe
