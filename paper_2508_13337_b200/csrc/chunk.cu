// Token-chunked forward pipeline (layer.cu: layer_forward_chunked).
//
// The S tokens of every source are cut into C contiguous chunks
// [floor(cS/C), floor((c+1)S/C)).  Each owner keeps one fixed region of Rc
// rows per chunk, laid out inside it exactly like the unchunked grouped
// buffer — (local expert, source, position), pf_pipeline.cpp:47-73 — so
// chunk c's rows can be dispatched, run through the grouped GEMMs and
// combined while the neighbouring chunks are in a different phase.  Every
// row's arithmetic is unchanged (a GEMM row does not depend on its
// neighbours, the combine sums a token's copies in slot order), so the
// chunked forward is bit-identical to the unchunked one.
//
// Cross-GPU phase ordering uses epoch flags in the symmetric (IPC-mapped)
// region instead of NCCL all-reduces: flag[phase][c][src] on every owner,
// written with st.release.sys by the source after its phase-c work, polled
// with ld.acquire.sys by the consumer.
//
// Row movement (default): owners PULL.  Every source stages its tokens in
// its symmetric region and writes, for each kept copy, (source, token) into
// the owner's row table; one flag later each owner copies its chunk-c rows
// over NVLink (pull_rows_kernel), and the combine reads the owners' expert
// outputs the same way.  Beside the expert GEMMs these kernels run as
// whole-SM blocks on XMOE_COMM_SMS SMs the GEMMs leave free (layer.cu):
// SM-driven NVLink traffic on the GEMMs' own SMs slows them up to 1.6x
// (profiles/interference/).  XMOE_DISPATCH=push keeps the source-side
// scatter (scatter_tokens_kernel with peer stores, a flag per chunk).
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace xmoe {

// chunk_t0 / chunk_of: kernels.cuh

// per (chunk c, expert e): kept copies of e whose token lies in chunk c, and
// their offset inside e's packed segment (tokens ascend within a segment,
// pft.cpp:35-57, so a chunk is a contiguous sub-range found by binary search)
__global__ void chunk_counts_kernel(const int32_t* __restrict__ token_ids, const int32_t* __restrict__ tpe,
                                    int E, int S, int C, int32_t* __restrict__ tpe_c,
                                    int32_t* __restrict__ pfx_c, int32_t* __restrict__ seg) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= C * E) return;
    const int c = idx / E, e = idx % E;
    int s0 = 0;
    for (int j = 0; j < e; ++j) s0 += tpe[j];
    const int n = tpe[e];
    auto lb = [&](int t) {
        int lo = 0, hi = n;
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (token_ids[s0 + m] < t) lo = m + 1;
            else hi = m;
        }
        return lo;
    };
    const int a = lb(chunk_t0(c, S, C));
    const int b = c == C - 1 ? n : lb(chunk_t0(c + 1, S, C));
    tpe_c[idx] = b - a;
    pfx_c[idx] = a;
    if (c == 0) seg[e] = s0;
}

// base[c][e]: first row of (expert e, source me) in e's owner's chunk-c
// region; rpe_c[c][le]: rows of my local expert le in my chunk-c region.
// T = [W][C][E] per-source chunk counts.
__global__ void chunk_bases_kernel(const int32_t* __restrict__ T, int W, int C, int E, int me, int Rc,
                                   int32_t* __restrict__ base, int32_t* __restrict__ rpe_c) {
    const int El = E / W;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    auto t = [&](int s, int c, int e) { return T[(static_cast<size_t>(s) * C + c) * E + e]; };
    if (idx < C * E) {
        const int c = idx / E, e = idx % E;
        const int o = e / El, le = e % El;
        int a = c * Rc;
        for (int l2 = 0; l2 < le; ++l2)
            for (int s = 0; s < W; ++s) a += t(s, c, o * El + l2);
        for (int s = 0; s < me; ++s) a += t(s, c, e);
        base[idx] = a;
    } else if (idx < C * E + C * El) {
        const int j = idx - C * E;
        const int c = j / El, le = j % El;
        int a = 0;
        for (int s = 0; s < W; ++s) a += t(s, c, me * El + le);
        rpe_c[j] = a;
    }
}

__global__ void dispatch_dest_chunked_kernel(const int32_t* __restrict__ expert_ids,
                                             const int32_t* __restrict__ token_ids,
                                             const int32_t* __restrict__ B_dev, int S, int C, int E, int El,
                                             const int32_t* __restrict__ seg, const int32_t* __restrict__ pfx_c,
                                             const int32_t* __restrict__ base, int32_t* __restrict__ dest_rank,
                                             int32_t* __restrict__ dest_row, int32_t* const* __restrict__ rsrc_tab,
                                             int me) {
    const int B = *B_dev;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < B; r += gridDim.x * blockDim.x) {
        const int e = expert_ids[r];
        const int t = token_ids[r];
        const int c = chunk_of(t, S, C);
        const int d = e / El;
        const int row = base[c * E + e] + (r - seg[e]) - pfx_c[c * E + e];
        dest_rank[r] = d;
        dest_row[r] = row;
        // pull dispatch: tell the owner which (source, token) fills that row
        if (rsrc_tab) rsrc_tab[d][row] = (me << 24) | t;
    }
    if (rsrc_tab) __threadfence_system();  // peer stores visible before the flag that follows
}

// Pull dispatch, per token: where the combine reads each kept copy's expert
// output (the owner's eout row) and the copy's weight.
__global__ void slot_addrs_kernel(const int32_t* __restrict__ slot_pos, int n, const int32_t* __restrict__ dest_rank,
                                  const int32_t* __restrict__ dest_row, const double* __restrict__ cw,
                                  char* const* __restrict__ eout_tab, int row_bytes,
                                  unsigned long long* __restrict__ slot_src, float* __restrict__ slot_w) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int p = slot_pos[i];
        unsigned long long a = 0;
        float wv = 0.f;
        if (p >= 0) {
            a = reinterpret_cast<unsigned long long>(eout_tab[dest_rank[p]] +
                                                     static_cast<size_t>(dest_row[p]) * row_bytes);
            wv = static_cast<float>(cw[p]);
        }
        slot_src[i] = a;
        slot_w[i] = wv;
    }
}

// Pull dispatch, owner side: one warp per grouped row of chunk region c
// copies the token row from its source's staged input (xs_tab[source], a
// peer address over NVLink for other ranks) into the owner's grouped buffer.
// Reading peers instead of storing to them keeps the NVLink traffic from
// stalling the expert GEMMs that share the SMs (B200, 2 GPUs: a GEMM beside
// an SM-driven peer store stream runs 1.2-1.8x slower, beside peer loads
// 1.07x).  rows = sum of the region's per-expert counts.
constexpr int kPullWarps = 8;
constexpr int kPullVec = 8;  // int4 per lane in flight (4 KB rows in one pass)
__global__ void __launch_bounds__(1024) pull_rows_kernel(const int32_t* __restrict__ rsrc,
                                                                    const int32_t* __restrict__ rpe, int El,
                                                                    char* const* __restrict__ xs_tab, int row_bytes,
                                                                    char* __restrict__ recv) {
    __shared__ int s_rows;
    if (threadIdx.x < 32) {
        int v = 0;
        for (int i = threadIdx.x; i < El; i += 32) v += rpe[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) s_rows = v;
    }
    __syncthreads();
    const int rows = s_rows;
    const int lane = threadIdx.x & 31;
    const int nvec = row_bytes >> 4;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarps) {
        const unsigned e = static_cast<unsigned>(__ldg(rsrc + r));
        const int4* src = reinterpret_cast<const int4*>(xs_tab[e >> 24] + static_cast<size_t>(e & 0xFFFFFFu) * row_bytes);
        int4* dst = reinterpret_cast<int4*>(recv + static_cast<size_t>(r) * row_bytes);
        for (int base = 0; base < nvec; base += 32 * kPullVec) {
            int4 v[kPullVec];
#pragma unroll
            for (int u = 0; u < kPullVec; ++u) {
                const int c = base + lane + 32 * u;
                v[u] = c < nvec ? ld_nc_v4(src + c) : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kPullVec; ++u) {
                const int c = base + lane + 32 * u;
                if (c < nvec) st_na_v4(dst + c, v[u]);
            }
        }
    }
}

void launch_slot_addrs(const int32_t* slot_pos, long long n, const int32_t* dest_rank, const int32_t* dest_row,
                       const double* cw, char* const* eout_tab, int row_bytes, unsigned long long* slot_src,
                       float* slot_w, cudaStream_t st) {
    if (n <= 0) return;
    const long long blocks = (n + 255) / 256;
    slot_addrs_kernel<<<static_cast<int>(blocks < 4 * kNumSMs ? blocks : 4 * kNumSMs), 256, 0, st>>>(
        slot_pos, static_cast<int>(n), dest_rank, dest_row, cw, eout_tab, row_bytes, slot_src, slot_w);
    XMOE_LAUNCH_CHECK();
}

void launch_pull_rows(const int32_t* rsrc, const int32_t* rpe, int El, char* const* xs_tab, int row_bytes,
                      long long max_rows, void* recv, cudaStream_t st) {
    require(row_bytes % 16 == 0, XMOE_ERR_VALIDATION, "pull dispatch needs 16-byte rows");
    if (max_rows <= 0) return;
    if (g_copy_fat > 0) {  // one 1024-thread block per SM (the shared reservation keeps others off it)
        static bool attr = false;
        if (!attr) {
            XMOE_CUDA(cudaFuncSetAttribute(pull_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kFatSmemBytes));
            attr = true;
        }
        pull_rows_kernel<<<g_copy_fat, 1024, kFatSmemBytes, st>>>(rsrc, rpe, El, xs_tab, row_bytes,
                                                            static_cast<char*>(recv));
        XMOE_LAUNCH_CHECK();
        return;
    }
    long long blocks = (max_rows + kPullWarps - 1) / kPullWarps;
    const long long cap = g_copy_blocks > 0 ? g_copy_blocks : 4 * kNumSMs;
    if (blocks > cap) blocks = cap;
    pull_rows_kernel<<<static_cast<int>(blocks), 32 * kPullWarps, 0, st>>>(rsrc, rpe, El, xs_tab, row_bytes,
                                                                          static_cast<char*>(recv));
    XMOE_LAUNCH_CHECK();
}

// Peer-flag wait with a bounded spin.  A peer that never arrives (rank
// skew beyond the timeout, a dead process) must not kill the CUDA context:
// the waiter records the failed slot in the layer's host-mapped error word
// and returns; the host turns it into XMOE_ERR_PEER_TIMEOUT on the next call
// (xmoe_layer_status).  Once the word is set every later wait returns at once.
// The timeout is XMOE_PEER_TIMEOUT_S (default 300 s), read once per process.
__device__ __forceinline__ void wait_flag(const unsigned* f, unsigned e, unsigned long long timeout_ns, int slot,
                                          int* err, unsigned ns) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (static_cast<int>(v - e) >= 0) return;
        if (*reinterpret_cast<volatile int*>(err) != 0) return;
        __nanosleep(ns);
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > timeout_ns) {
            atomicCAS(err, 0, 0x100 | slot);
            __threadfence_system();
            return;
        }
    }
}

unsigned long long peer_timeout_ns() {
    static const unsigned long long ns = [] {
        const char* e = std::getenv("XMOE_PEER_TIMEOUT_S");
        const double s = e ? std::atof(e) : 300.0;
        return static_cast<unsigned long long>((s > 0 ? s : 300.0) * 1e9);
    }();
    return ns;
}

__global__ void forward_begin_kernel(int32_t* s_rows, int S, unsigned* epoch) {
    if (threadIdx.x == 0) {
        *s_rows = S;
        if (epoch) *epoch += 1u;
    }
}

__global__ void flag_signal_kernel(unsigned* const* __restrict__ flag_tab, int W, int me, int slot,
                                   const unsigned* __restrict__ epoch) {
    const int p = threadIdx.x;
    if (p >= W) return;
    const unsigned e = *epoch;
    unsigned* f = flag_tab[p] + static_cast<size_t>(slot) * W + me;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(e) : "memory");
}

__global__ void flag_wait_kernel(const unsigned* __restrict__ flags, int W, int slot,
                                 const unsigned* __restrict__ epoch, unsigned long long tmo, int* err) {
    const int s = threadIdx.x;
    if (s < W) wait_flag(flags + static_cast<size_t>(slot) * W + s, *epoch, tmo, slot, err, 100);
    __syncthreads();
}

// Count all-gather over the symmetric regions (replaces ncclAllGather of
// the routing counts): every rank stores its rows into every peer's count
// area (double-buffered by forward parity: a peer at most one forward
// behind is still reading the other half), raises its flag, waits for all
// flags, and copies the gathered area into the layer's local arrays.
// Passing it also proves every peer finished its previous forward.
__global__ void counts_exchange_kernel(CountSegs segs, int32_t* const* __restrict__ area_tab, int area_ints,
                                       int me, int W, unsigned* const* __restrict__ flag_tab,
                                       const unsigned* __restrict__ my_flags, int slot,
                                       const unsigned* __restrict__ epoch, unsigned long long tmo, int* err) {
    const unsigned e = *epoch;
    const int par = static_cast<int>(e & 1u);
    for (int p = 0; p < W; ++p) {
        int32_t* area = area_tab[p] + static_cast<size_t>(par) * area_ints;
        for (int q = 0; q < segs.n; ++q) {
            const CountSeg& sg = segs.s[q];
            for (int i = threadIdx.x; i < sg.row; i += blockDim.x) area[sg.off + me * sg.row + i] = sg.src[i];
        }
    }
    __threadfence_system();
    __syncthreads();
    const int t = threadIdx.x;
    if (t < W) {
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag_tab[t] + static_cast<size_t>(slot) * W + me),
                     "r"(e)
                     : "memory");
        wait_flag(my_flags + static_cast<size_t>(slot) * W + t, e, tmo, slot, err, 64);
    }
    __syncthreads();
    const int32_t* mine = area_tab[me] + static_cast<size_t>(par) * area_ints;
    for (int q = 0; q < segs.n; ++q) {
        const CountSeg& sg = segs.s[q];
        for (int i = threadIdx.x; i < W * sg.row; i += blockDim.x) sg.local[i] = mine[sg.off + i];
    }
}

// Cross-GPU barrier on one flag slot (every rank's previous kernels on this
// stream are complete and their peer stores visible when it passes).
__global__ void flag_barrier_kernel(unsigned* const* __restrict__ flag_tab, const unsigned* __restrict__ my_flags,
                                    int W, int me, int slot, const unsigned* __restrict__ epoch,
                                    unsigned long long tmo, int* err) {
    const unsigned e = *epoch;
    const int t = threadIdx.x;
    __threadfence_system();
    __syncthreads();
    if (t < W) {
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag_tab[t] + static_cast<size_t>(slot) * W + me),
                     "r"(e)
                     : "memory");
        wait_flag(my_flags + static_cast<size_t>(slot) * W + t, e, tmo, slot, err, 64);
    }
    __syncthreads();
}

void launch_counts_exchange(const CountSegs& segs, int32_t* const* area_tab, int area_ints, int me, int W,
                            unsigned* const* flag_tab, const unsigned* my_flags, int slot, const unsigned* epoch,
                            int* err, cudaStream_t st) {
    counts_exchange_kernel<<<1, 256, 0, st>>>(segs, area_tab, area_ints, me, W, flag_tab, my_flags, slot, epoch,
                                              peer_timeout_ns(), err);
    XMOE_LAUNCH_CHECK();
}

void launch_flag_barrier(unsigned* const* flag_tab, const unsigned* my_flags, int W, int me, int slot,
                         const unsigned* epoch, int* err, cudaStream_t st) {
    flag_barrier_kernel<<<1, 32 * ((W + 31) / 32), 0, st>>>(flag_tab, my_flags, W, me, slot, epoch,
                                                            peer_timeout_ns(), err);
    XMOE_LAUNCH_CHECK();
}

void launch_chunk_counts(const int32_t* token_ids, const int32_t* tpe, int E, int S, int C, int32_t* tpe_c,
                         int32_t* pfx_c, int32_t* seg, cudaStream_t st) {
    const int n = C * E;
    chunk_counts_kernel<<<(n + 127) / 128, 128, 0, st>>>(token_ids, tpe, E, S, C, tpe_c, pfx_c, seg);
    XMOE_LAUNCH_CHECK();
}

void launch_chunk_bases(const int32_t* T, int W, int C, int E, int me, int Rc, int32_t* base, int32_t* rpe_c,
                        cudaStream_t st) {
    const int n = C * E + C * (E / W);
    chunk_bases_kernel<<<(n + 127) / 128, 128, 0, st>>>(T, W, C, E, me, Rc, base, rpe_c);
    XMOE_LAUNCH_CHECK();
}

void launch_dispatch_dest_chunked(const int32_t* expert_ids, const int32_t* token_ids, const int32_t* B_dev,
                                  long long max_rows, int S, int C, int E, int El, const int32_t* seg,
                                  const int32_t* pfx_c, const int32_t* base, int32_t* dest_rank,
                                  int32_t* dest_row, cudaStream_t st, int32_t* const* rsrc_tab, int me) {
    const long long blocks = (max_rows + 255) / 256;
    dispatch_dest_chunked_kernel<<<static_cast<int>(blocks < 4 * kNumSMs ? (blocks > 0 ? blocks : 1) : 4 * kNumSMs),
                                   256, 0, st>>>(expert_ids, token_ids, B_dev, S, C, E, El, seg, pfx_c, base,
                                                 dest_rank, dest_row, rsrc_tab, me);
    XMOE_LAUNCH_CHECK();
}

void launch_forward_begin(int32_t* s_rows, int S, unsigned* epoch, cudaStream_t st) {
    forward_begin_kernel<<<1, 32, 0, st>>>(s_rows, S, epoch);
    XMOE_LAUNCH_CHECK();
}

void launch_flag_signal(unsigned* const* flag_tab, int W, int me, int slot, const unsigned* epoch,
                        cudaStream_t st) {
    flag_signal_kernel<<<1, 32 * ((W + 31) / 32), 0, st>>>(flag_tab, W, me, slot, epoch);
    XMOE_LAUNCH_CHECK();
}

void launch_flag_wait(const unsigned* flags, int W, int slot, const unsigned* epoch, int* err, cudaStream_t st) {
    flag_wait_kernel<<<1, 32 * ((W + 31) / 32), 0, st>>>(flags, W, slot, epoch, peer_timeout_ns(), err);
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
