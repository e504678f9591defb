// Split expert-parallel operators in the reference's SPMD shape: every call
// takes ALL workers' data at once (vectors indexed by group rank,
// SURVEY §8(b)) and runs them on one device — the operator-level drop-in for
//   moesim::pf_dispatch / pf_combine      (pf_pipeline.cpp:12-81, 107-135)
//   moesim::select_pilots                 (rbd.cpp:26-81)
//   moesim::rbd_dispatch / rbd_combine    (rbd.cpp:83-358)
//   moesim::internode_redundancy_counts   (rbd.cpp:427-442) and the rates
// The fused one-process-per-GPU forward is the xmoe_layer path (layer.cu);
// these operators share its kernels where the work is the same (destination
// rows, row scatter, stable CSR, the RBD group draw, the weighted combine).
//
// Row placement: copy r of source s lands at its owner's grouped row
//     dest_row = expert_base[le] + sum_{s' < s} tpe[s'][e] + (r - block_s[e])
// (dispatch_dest_kernel), i.e. the (local expert, source, position) order of
// pf_dispatch, for both dispatch modes.  The redundancy bypass moves each
// group's pilot row once (stage 1, to the pilot's owner = the landing worker)
// and re-creates the replicas there from the landed row (stage 2), exactly
// the reference's two stages collapsed onto one device; the result is
// bit-identical to the plain dispatch (rbd.hpp:50).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "layer.h"
#include "rbd.h"

namespace xmoe {

constexpr int kEpWarps = 8;

// ---------------------------------------------------------------- kernels
// slot_pos[t][j] = j-th copy of token t in packed order (-1 padded); err
// bit 0 when a token has more than k copies.
__global__ void slots_from_csr_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ perm, int S,
                                      int k, int32_t* __restrict__ slot_pos, int* __restrict__ err) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S) return;
    const int b = ptr[t], n = ptr[t + 1] - b;
    if (n > k) atomicOr(err, 1);
    for (int j = 0; j < k; ++j) slot_pos[static_cast<size_t>(t) * k + j] = j < n ? perm[b + j] : -1;
}

// Groups of a packed buffer from a pilot mask (rbd_dispatch input): the
// copies of token t on one node form a group (a run of slots, experts being
// node-contiguous); exactly one member must carry the mask.  pilot_of[copy]
// = the group's pilot row.  err bit 1: a group without exactly one pilot.
__global__ void pilot_of_from_mask_kernel(const int32_t* __restrict__ slot_pos, int S, int k,
                                          const int32_t* __restrict__ expert_ids, int E_node,
                                          const uint8_t* __restrict__ mask, int32_t* __restrict__ pilot_of,
                                          int* __restrict__ err) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S) return;
    const int32_t* sp = slot_pos + static_cast<size_t>(t) * k;
    int j = 0;
    while (j < k && sp[j] >= 0) {
        const int node = expert_ids[sp[j]] / E_node;
        int n = 1;
        while (j + n < k && sp[j + n] >= 0 && expert_ids[sp[j + n]] / E_node == node) ++n;
        int pilot = -1, marks = 0;
        for (int m = 0; m < n; ++m)
            if (mask[sp[j + m]]) {
                pilot = sp[j + m];
                ++marks;
            }
        if (marks != 1) atomicOr(err, 2);
        for (int m = 0; m < n; ++m) pilot_of[sp[j + m]] = pilot < 0 ? sp[j] : pilot;
        j += n;
    }
}

// select_pilots output from the drawn groups (rbd.cu launch_rbd_groups).
__global__ void mask_from_groups_kernel(const int32_t* __restrict__ G_dev, RbdGroups g,
                                        const int32_t* __restrict__ slot_pos, int k, uint8_t* __restrict__ mask,
                                        int32_t* __restrict__ pilot_of) {
    const int G = *G_dev;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < G; i += gridDim.x * blockDim.x) {
        const int p = g.pilot[i];
        mask[p] = 1;
        if (pilot_of)
            for (int m = 0; m < g.n[i]; ++m) pilot_of[slot_pos[static_cast<size_t>(g.token[i]) * k + g.first_slot[i] + m]] = p;
    }
}

void launch_mask_from_groups(const RbdWork& wk, const int32_t* slot_pos, int k, long long max_groups, uint8_t* mask,
                             int32_t* pilot_of, cudaStream_t st) {
    mask_from_groups_kernel<<<std::max(1, std::min(ceil_div(max_groups, 256), 4 * kNumSMs)), 256, 0, st>>>(
        wk.G_dev, wk.g, slot_pos, k, mask, pilot_of);
    XMOE_LAUNCH_CHECK();
}

__device__ __forceinline__ void ep_copy_row(const char* __restrict__ src, char* __restrict__ dst, int row_bytes,
                                            int lane) {
    if ((row_bytes & 15) == 0) {
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        for (int v = lane; v < (row_bytes >> 4); v += 32) d4[v] = s4[v];
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

// RBD stage 1: every pilot's packed row to its own grouped row at its owner
// (the landing worker).  Stage 2 (separate launch, after stage 1): every
// replica re-created from its pilot's LANDED row (rbd.cpp:221-232).
__global__ void __launch_bounds__(32 * kEpWarps) rbd_stage_kernel(
    const char* __restrict__ packed, int row_bytes, int B, const uint8_t* __restrict__ mask,
    const int32_t* __restrict__ pilot_of, const int32_t* __restrict__ dest_rank,
    const int32_t* __restrict__ dest_row, char* const* __restrict__ tab, int stage) {
    const int lane = threadIdx.x & 31;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < B; r += nw) {
        const bool pilot = mask[r] != 0;
        if (pilot != (stage == 1)) continue;
        char* dst = tab[dest_rank[r]] + static_cast<size_t>(dest_row[r]) * row_bytes;
        const char* src = stage == 1 ? packed + static_cast<size_t>(r) * row_bytes
                                     : tab[dest_rank[pilot_of[r]]] + static_cast<size_t>(dest_row[pilot_of[r]]) * row_bytes;
        ep_copy_row(src, dst, row_bytes, lane);
    }
}

// pf_dispatch's arrival_to_grouped (pf_pipeline.cpp:50-73): arrivals at owner
// j come source-ascending, each source's rows in its packed order.
__global__ void arrival_kernel(const int32_t* __restrict__ tpe_all, int W, int E, int src, int B,
                               const int32_t* __restrict__ dest_rank, const int32_t* __restrict__ dest_row,
                               int32_t* const* __restrict__ a2g_tab) {
    extern __shared__ int32_t sh[];
    int32_t* before = sh;      // [W] rows arriving at j from sources < src
    int32_t* start = sh + W;   // [W] first packed row of src destined to j
    const int El = E / W;
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int j = 0; j < W; ++j) {
            start[j] = acc;
            for (int le = 0; le < El; ++le) acc += tpe_all[static_cast<size_t>(src) * E + j * El + le];
            int b = 0;
            for (int s = 0; s < src; ++s)
                for (int le = 0; le < El; ++le) b += tpe_all[static_cast<size_t>(s) * E + j * El + le];
            before[j] = b;
        }
    }
    __syncthreads();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < B; r += gridDim.x * blockDim.x) {
        const int j = dest_rank[r];
        if (a2g_tab[j]) a2g_tab[j][before[j] + (r - start[j])] = dest_row[r];
    }
}

// rbd_combine's merge at the landing workers (rbd.cpp:318-336): flat pilot p
// (landing worker land_of[p]) starts from its own expert output, scaled by
// its weight when the group has replicas (kernels::scale), then adds every
// replica's weighted output in slot order (kernels::axpy).
template <typename T>
__global__ void __launch_bounds__(32 * kEpWarps) rbd_merge_flat_kernel(
    const char* const* __restrict__ eout_tab, int H, int P, const int32_t* __restrict__ land_of,
    const int32_t* __restrict__ land_pos, const uint8_t* __restrict__ land_multi,
    const double* __restrict__ land_w, const int32_t* __restrict__ ent_ptr,
    const int32_t* __restrict__ ent_owner, const int32_t* __restrict__ ent_pos, const double* __restrict__ ent_w,
    T* __restrict__ merged) {
    const int lane = threadIdx.x & 31;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long p = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; p < P; p += nw) {
        const T* y0 = reinterpret_cast<const T*>(eout_tab[land_of[p]]) + static_cast<size_t>(land_pos[p]) * H;
        const bool multi = land_multi[p] != 0;
        const int e0 = ent_ptr[p], e1 = ent_ptr[p + 1];
        for (int h = lane; h < H; h += 32) {
            if constexpr (sizeof(T) == 8) {
                double acc = y0[h];
                if (multi) acc = __dmul_rn(acc, land_w[p]);
                for (int e = e0; e < e1; ++e) {
                    const double y = reinterpret_cast<const double*>(eout_tab[ent_owner[e]])[static_cast<size_t>(ent_pos[e]) * H + h];
                    acc = __dadd_rn(acc, __dmul_rn(ent_w[e], y));
                }
                merged[static_cast<size_t>(p) * H + h] = acc;
            } else if constexpr (sizeof(T) == 4) {  // F32: fp64 accumulation, one rounding
                double acc = y0[h];
                if (multi) acc = __dmul_rn(acc, land_w[p]);
                for (int e = e0; e < e1; ++e) {
                    const float y = reinterpret_cast<const float*>(eout_tab[ent_owner[e]])[static_cast<size_t>(ent_pos[e]) * H + h];
                    acc = __dadd_rn(acc, __dmul_rn(ent_w[e], static_cast<double>(y)));
                }
                merged[static_cast<size_t>(p) * H + h] = static_cast<float>(acc);
            } else {
                float acc = __bfloat162float(y0[h]);
                if (multi) acc *= static_cast<float>(land_w[p]);
                for (int e = e0; e < e1; ++e) {
                    const __nv_bfloat16 y = reinterpret_cast<const __nv_bfloat16*>(eout_tab[ent_owner[e]])[static_cast<size_t>(ent_pos[e]) * H + h];
                    acc = fmaf(static_cast<float>(ent_w[e]), __bfloat162float(y), acc);
                }
                merged[static_cast<size_t>(p) * H + h] = __float2bfloat16_rn(acc);
            }
        }
    }
}

// Distinct (token, node) pairs among n copies (redundancy_rate*, rbd.cpp:390-442):
// mark[t * N + node] once per pair; the count is the number of first marks.
__global__ void pair_mark_kernel(int n, const int32_t* __restrict__ token, const int32_t* __restrict__ expert,
                                 const int32_t* __restrict__ expert_node, int E, int N, int T, int skip_node,
                                 int32_t* __restrict__ mark, unsigned long long* __restrict__ acc,
                                 int* __restrict__ err) {
    unsigned long long copies = 0, groups = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int e = expert[i], t = token[i];
        if (e < 0 || e >= E || t < 0 || t >= T) {
            atomicOr(err, 4);
            continue;
        }
        const int nd = expert_node[e];
        if (nd < 0 || nd >= N) {
            atomicOr(err, 4);
            continue;
        }
        if (nd == skip_node) continue;
        ++copies;
        if (atomicExch(mark + static_cast<size_t>(t) * N + nd, 1) == 0) ++groups;
    }
    atomicAdd(acc, copies);
    atomicAdd(acc + 1, groups);
}

// ---------------------------------------------------------------- host helpers
namespace {

struct Carve {
    char* p;
    explicit Carve(void* base) : p(static_cast<char*>(base)) {}
    template <class T>
    T* take(size_t n) {
        T* r = reinterpret_cast<T*>(p);
        p += (sizeof(T) * (n ? n : 1) + 255) & ~static_cast<size_t>(255);
        return r;
    }
};

size_t elem_bytes(int dtype) {
    if (dtype == XMOE_F64) return 8;
    if (dtype == XMOE_F32) return 4;
    if (dtype == XMOE_BF16) return 2;
    fail(XMOE_ERR_VALIDATION, "unknown dtype");
}

int spmd_world(const Ctx& c) {
    require(c.rank < 0 || c.world == 1, XMOE_ERR_VALIDATION,
            "split expert-parallel operators take every worker's data in one call: use a rank == -1 context");
    return c.world;
}

// per-source device scalars (B as int32) in scratch
int32_t* upload_counts(const std::vector<int32_t>& v, int32_t* dst, cudaStream_t st) {
    XMOE_CUDA(cudaMemcpyAsync(dst, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice, st));
    return dst;
}

template <class T>
T** upload_table(const std::vector<T*>& v, T** dst, cudaStream_t st) {
    XMOE_CUDA(cudaMemcpyAsync(dst, v.data(), sizeof(T*) * v.size(), cudaMemcpyHostToDevice, st));
    return dst;
}

void check_err(int* err_dev, cudaStream_t st, const char* over_k, const char* plan) {
    int h = 0;
    XMOE_CUDA(cudaMemcpyAsync(&h, err_dev, sizeof(int), cudaMemcpyDeviceToHost, st));
    XMOE_CUDA(cudaStreamSynchronize(st));
    if (h & 1) fail(XMOE_ERR_VALIDATION, over_k);
    if (h & 2) fail(XMOE_ERR_PLAN_MISMATCH, plan);
    if (h & 4) fail(XMOE_ERR_INDEX, "expert id out of range");
}

std::vector<uint64_t>& jump_tables() {
    static std::vector<uint64_t> jt;
    if (jt.empty()) rbd_jump_tables(jt);
    return jt;
}

}  // namespace

}  // namespace xmoe

using namespace xmoe;

extern "C" {

int xmoe_pf_dispatch(xmoe_ctx* ctx, int dtype, int64_t H, int64_t E, const void* const* packed,
                     const int32_t* const* expert_ids, const int64_t* B, const int32_t* tpe, void* const* expert_input,
                     int32_t* recv_per_expert, int32_t* const* dest_rank, int32_t* const* dest_row,
                     int32_t* const* arrival_to_grouped, void* stream) {
    return guarded([&] {
        const int W = spmd_world(ctx->c);
        require(E >= 1 && E % W == 0, XMOE_ERR_VALIDATION, "num_experts must be divisible by the worker-group size");
        auto st = static_cast<cudaStream_t>(stream);
        const int rb = static_cast<int>(H * elem_bytes(dtype));
        const int El = static_cast<int>(E / W);
        long long bmax = 1;
        for (int w = 0; w < W; ++w) bmax = std::max<long long>(bmax, B[w]);
        Carve cv(ctx->c.scratch(sizeof(int32_t) * (2 * bmax + 64) + sizeof(void*) * 4 * W + 4096));
        int32_t* Bd = cv.take<int32_t>(W);
        int32_t* dr_s = cv.take<int32_t>(bmax);
        int32_t* dw_s = cv.take<int32_t>(bmax);
        char** tab = cv.take<char*>(W);
        int32_t** atab = cv.take<int32_t*>(W);
        std::vector<int32_t> hb(W);
        for (int w = 0; w < W; ++w) hb[w] = static_cast<int32_t>(B[w]);
        upload_counts(hb, Bd, st);
        std::vector<char*> tv(W);
        std::vector<int32_t*> av(W);
        for (int w = 0; w < W; ++w) {
            tv[w] = static_cast<char*>(expert_input[w]);
            av[w] = arrival_to_grouped ? arrival_to_grouped[w] : nullptr;
        }
        upload_table(tv, tab, st);
        upload_table(av, atab, st);
        for (int s = 0; s < W; ++s) {
            int32_t* dr = dest_rank && dest_rank[s] ? dest_rank[s] : dr_s;
            int32_t* dw = dest_row && dest_row[s] ? dest_row[s] : dw_s;
            launch_dispatch_dest(tpe, W, static_cast<int>(E), s, expert_ids[s], Bd + s, B[s], dr, dw, st);
            if (B[s] > 0)
                launch_scatter_rows(packed[s], rb, nullptr, Bd + s, B[s], dr, dw, tab, st);
            if (arrival_to_grouped && B[s] > 0) {
                const int blocks = std::min(ceil_div(B[s], 256), 4 * kNumSMs);
                arrival_kernel<<<blocks, 256, sizeof(int32_t) * 2 * W, st>>>(tpe, W, static_cast<int>(E), s,
                                                                             static_cast<int>(B[s]), dr, dw, atab);
                XMOE_LAUNCH_CHECK();
            }
            if (dr == dr_s || dw == dw_s) XMOE_CUDA(cudaStreamSynchronize(st));  // scratch reused by the next source
        }
        if (recv_per_expert)
            for (int j = 0; j < W; ++j) launch_recv_counts(tpe, W, static_cast<int>(E), j, recv_per_expert + j * El, st);
    });
}

int xmoe_pf_combine(xmoe_ctx* ctx, int dtype, int64_t H, int64_t E, const void* const* expert_out,
                    const int32_t* tpe, const int32_t* const* token_ids, const int32_t* const* expert_ids,
                    const double* const* cw, const int64_t* B, const int64_t* seq_lens, void* const* out,
                    void* stream) {
    return guarded([&] {
        const int W = spmd_world(ctx->c);
        require(E >= 1 && E % W == 0, XMOE_ERR_VALIDATION, "num_experts must be divisible by the worker-group size");
        auto st = static_cast<cudaStream_t>(stream);
        long long bmax = 1, smax = 1;
        for (int w = 0; w < W; ++w) {
            bmax = std::max<long long>(bmax, B[w]);
            smax = std::max<long long>(smax, seq_lens[w]);
        }
        Carve cv(ctx->c.scratch(sizeof(int32_t) * (3 * bmax + smax + 64) + bucket_ws_bytes(bmax, static_cast<int>(smax)) +
                                sizeof(void*) * W + 8192));
        int32_t* Bd = cv.take<int32_t>(W);
        int32_t* dr = cv.take<int32_t>(bmax);
        int32_t* dw = cv.take<int32_t>(bmax);
        int32_t* ptr = cv.take<int32_t>(smax + 1);
        int32_t* perm = cv.take<int32_t>(bmax);
        char** tab = cv.take<char*>(W);
        void* ws = cv.take<char>(bucket_ws_bytes(bmax, static_cast<int>(smax)));
        std::vector<int32_t> hb(W);
        for (int w = 0; w < W; ++w) hb[w] = static_cast<int32_t>(B[w]);
        upload_counts(hb, Bd, st);
        std::vector<const char*> tv(W);
        for (int w = 0; w < W; ++w) tv[w] = static_cast<const char*>(expert_out[w]);
        upload_table(tv, const_cast<const char**>(tab), st);
        for (int s = 0; s < W; ++s) {
            const int S = static_cast<int>(seq_lens[s]);
            if (S == 0) continue;
            // return trip (transposed counts) + scatter_combine
            // (pft.cpp:79-91): copy c of token t reads its owner's grouped row
            launch_dispatch_dest(tpe, W, static_cast<int>(E), s, expert_ids[s], Bd + s, B[s], dr, dw, st);
            launch_stable_csr(token_ids[s], static_cast<int>(B[s]), S, ptr, perm, ws, st);
            launch_combine(dtype, nullptr, static_cast<int>(H), ptr, perm, 0, cw[s], S, nullptr, out[s], st, tab, dr, dw);
            XMOE_CUDA(cudaStreamSynchronize(st));  // scratch reused by the next source
        }
    });
}

int xmoe_select_pilots(xmoe_ctx* ctx, int64_t B, const int32_t* token_ids, const int32_t* expert_ids, int64_t S,
                       int64_t k, int64_t E, int64_t W, int64_t gpus_per_node, uint64_t seed, uint8_t* pilot_mask,
                       int32_t* pilot_of, void* stream) {
    return guarded([&] {
        require(W >= 1 && E >= 1 && E % W == 0, XMOE_ERR_VALIDATION,
                "num_experts must be divisible by the worker-group size");
        const int gpn = static_cast<int>(std::max<int64_t>(1, gpus_per_node));
        require(W % gpn == 0, XMOE_ERR_VALIDATION, "the worker group must be whole nodes (world % gpus_per_node)");
        auto st = static_cast<cudaStream_t>(stream);
        if (B == 0) return;
        require(S >= 1 && k >= 1, XMOE_ERR_VALIDATION, "select_pilots: token and copy bounds must be >= 1");
        const long long nk = S * k;
        RbdWork wk{};
        Carve cv(ctx->c.scratch(sizeof(int32_t) * (14 * nk + 4 * S + 64) + sizeof(uint64_t) * (nk + kRbdChunk) +
                                bucket_ws_bytes(B, static_cast<int>(S)) + jump_tables().size() * 8 + 16384));
        int32_t* ptr = cv.take<int32_t>(S + 1);
        int32_t* perm = cv.take<int32_t>(B);
        int32_t* slot = cv.take<int32_t>(nk);
        int* err = cv.take<int>(4);
        wk.g.token = cv.take<int32_t>(nk);
        wk.g.dest = cv.take<int32_t>(nk);
        wk.g.first_slot = cv.take<int32_t>(nk);
        wk.g.n = cv.take<int32_t>(nk);
        wk.g.pilot = cv.take<int32_t>(nk);
        wk.g.pos = cv.take<int32_t>(nk);
        wk.gcount = cv.take<int32_t>(S);
        wk.gbase = cv.take<int32_t>(S);
        wk.G_dev = cv.take<int32_t>(1);
        wk.flags = cv.take<int32_t>(1);
        wk.scan_ws = cv.take<int32_t>(nk / 2048 + 2);
        wk.draws = cv.take<uint64_t>(nk + kRbdChunk);
        wk.gpn = gpn;
        uint64_t* jumps = cv.take<uint64_t>(jump_tables().size());
        void* ws = cv.take<char>(bucket_ws_bytes(B, static_cast<int>(S)));
        XMOE_CUDA(cudaMemcpyAsync(jumps, jump_tables().data(), jump_tables().size() * 8, cudaMemcpyHostToDevice, st));
        XMOE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
        launch_stable_csr(token_ids, static_cast<int>(B), static_cast<int>(S), ptr, perm, ws, st);
        slots_from_csr_kernel<<<ceil_div(S, 256), 256, 0, st>>>(ptr, perm, static_cast<int>(S), static_cast<int>(k),
                                                                 slot, err);
        XMOE_LAUNCH_CHECK();
        // one Rng(seed).below(|group|) per (token, node) group in map order (rbd.cpp:35-51)
        uint64_t state[4];
        rng_state_from_seed(seed, state);
        launch_rbd_groups(slot, expert_ids, static_cast<int>(S), static_cast<int>(k), static_cast<int>(E / W), state,
                          jumps, wk, st);
        XMOE_CUDA(cudaMemsetAsync(pilot_mask, 0, B, st));
        mask_from_groups_kernel<<<std::min(ceil_div(nk, 256), 4 * kNumSMs), 256, 0, st>>>(wk.G_dev, wk.g, slot,
                                                                                         static_cast<int>(k),
                                                                                         pilot_mask, pilot_of);
        XMOE_LAUNCH_CHECK();
        check_err(err, st, "select_pilots: a token has more copies than the stated bound", "");
    });
}

int xmoe_rbd_dispatch(xmoe_ctx* ctx, int dtype, int64_t H, int64_t E, int64_t gpus_per_node,
                      const void* const* packed, const int32_t* const* token_ids, const int32_t* const* expert_ids,
                      const int64_t* B, const int64_t* seq_lens, int64_t k, const int32_t* tpe,
                      const uint8_t* const* pilot_mask, void* const* expert_input, int32_t* recv_per_expert,
                      int32_t* const* dest_rank, int32_t* const* dest_row, int32_t* const* pilot_of, void* stream) {
    return guarded([&] {
        const int W = spmd_world(ctx->c);
        require(E >= 1 && E % W == 0, XMOE_ERR_VALIDATION, "num_experts must be divisible by the worker-group size");
        const int gpn = static_cast<int>(std::max<int64_t>(1, gpus_per_node));
        require(W % gpn == 0, XMOE_ERR_VALIDATION, "the worker group must be whole nodes (world % gpus_per_node)");
        auto st = static_cast<cudaStream_t>(stream);
        const int rb = static_cast<int>(H * elem_bytes(dtype));
        const int El = static_cast<int>(E / W);
        long long bmax = 1, smax = 1;
        for (int w = 0; w < W; ++w) {
            bmax = std::max<long long>(bmax, B[w]);
            smax = std::max<long long>(smax, seq_lens[w]);
        }
        const long long nk = smax * std::max<int64_t>(k, 1);
        Carve cv(ctx->c.scratch(sizeof(int32_t) * (4 * bmax + nk + smax + 64) + bucket_ws_bytes(bmax, static_cast<int>(smax)) +
                                sizeof(void*) * W + 8192));
        int32_t* Bd = cv.take<int32_t>(W);
        int32_t* ptr = cv.take<int32_t>(smax + 1);
        int32_t* perm = cv.take<int32_t>(bmax);
        int32_t* slot = cv.take<int32_t>(nk);
        int* err = cv.take<int>(4);
        char** tab = cv.take<char*>(W);
        void* ws = cv.take<char>(bucket_ws_bytes(bmax, static_cast<int>(smax)));
        std::vector<int32_t> hb(W);
        for (int w = 0; w < W; ++w) hb[w] = static_cast<int32_t>(B[w]);
        upload_counts(hb, Bd, st);
        std::vector<char*> tv(W);
        for (int w = 0; w < W; ++w) tv[w] = static_cast<char*>(expert_input[w]);
        upload_table(tv, tab, st);
        XMOE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
        // placement of every copy (identical to pf_dispatch) and its group's pilot
        for (int s = 0; s < W; ++s) {
            launch_dispatch_dest(tpe, W, static_cast<int>(E), s, expert_ids[s], Bd + s, B[s], dest_rank[s],
                                 dest_row[s], st);
            const int S = static_cast<int>(seq_lens[s]);
            if (B[s] == 0 || S == 0) continue;
            launch_stable_csr(token_ids[s], static_cast<int>(B[s]), S, ptr, perm, ws, st);
            slots_from_csr_kernel<<<ceil_div(S, 256), 256, 0, st>>>(ptr, perm, S, static_cast<int>(k), slot, err);
            XMOE_LAUNCH_CHECK();
            pilot_of_from_mask_kernel<<<ceil_div(S, 256), 256, 0, st>>>(slot, S, static_cast<int>(k), expert_ids[s],
                                                                        El * gpn, pilot_mask[s], pilot_of[s], err);
            XMOE_LAUNCH_CHECK();
            XMOE_CUDA(cudaStreamSynchronize(st));  // scratch reused by the next source
        }
        check_err(err, st, "rbd_dispatch: a token has more copies than top_k",
                  "rbd_dispatch: plan inconsistent with packed buffer");
        // stage 1: pilot rows land at their owners; stage 2: replicas from the landed rows
        for (int stage = 1; stage <= 2; ++stage)
            for (int s = 0; s < W; ++s) {
                if (B[s] == 0) continue;
                const int blocks = std::min(ceil_div(B[s], kEpWarps), 8 * kNumSMs);
                rbd_stage_kernel<<<blocks, 32 * kEpWarps, 0, st>>>(static_cast<const char*>(packed[s]), rb,
                                                                   static_cast<int>(B[s]), pilot_mask[s], pilot_of[s],
                                                                   dest_rank[s], dest_row[s], tab, stage);
                XMOE_LAUNCH_CHECK();
            }
        if (recv_per_expert)
            for (int j = 0; j < W; ++j) launch_recv_counts(tpe, W, static_cast<int>(E), j, recv_per_expert + j * El, st);
    });
}

int xmoe_rbd_combine(xmoe_ctx* ctx, int dtype, int64_t H, const void* const* expert_out, int64_t P,
                     const int32_t* land_of, const int32_t* land_pos, const uint8_t* land_multi, const double* land_w,
                     const int32_t* ent_ptr, const int32_t* ent_owner, const int32_t* ent_pos, const double* ent_w,
                     const int32_t* const* src_ptr, const int32_t* const* src_flat, const double* flat_scale,
                     const int64_t* seq_lens, void* const* out, void* stream) {
    return guarded([&] {
        const int W = spmd_world(ctx->c);
        auto st = static_cast<cudaStream_t>(stream);
        const size_t es = elem_bytes(dtype);
        Carve cv(ctx->c.scratch(static_cast<size_t>(std::max<int64_t>(P, 1)) * H * es + sizeof(void*) * W + 4096));
        void* merged = cv.take<char>(static_cast<size_t>(std::max<int64_t>(P, 1)) * H * es);
        char** tab = cv.take<char*>(W);
        std::vector<const char*> tv(W);
        for (int w = 0; w < W; ++w) tv[w] = static_cast<const char*>(expert_out[w]);
        upload_table(tv, const_cast<const char**>(tab), st);
        if (P > 0) {
            const int blocks = std::min(ceil_div(P, kEpWarps), 8 * kNumSMs);
            if (dtype == XMOE_F64)
                rbd_merge_flat_kernel<double><<<blocks, 32 * kEpWarps, 0, st>>>(
                    tab, static_cast<int>(H), static_cast<int>(P), land_of, land_pos, land_multi, land_w, ent_ptr,
                    ent_owner, ent_pos, ent_w, static_cast<double*>(merged));
            else if (dtype == XMOE_F32)
                rbd_merge_flat_kernel<float><<<blocks, 32 * kEpWarps, 0, st>>>(
                    tab, static_cast<int>(H), static_cast<int>(P), land_of, land_pos, land_multi, land_w, ent_ptr,
                    ent_owner, ent_pos, ent_w, static_cast<float*>(merged));
            else
                rbd_merge_flat_kernel<__nv_bfloat16><<<blocks, 32 * kEpWarps, 0, st>>>(
                    tab, static_cast<int>(H), static_cast<int>(P), land_of, land_pos, land_multi, land_w, ent_ptr,
                    ent_owner, ent_pos, ent_w, static_cast<__nv_bfloat16*>(merged));
            XMOE_LAUNCH_CHECK();
        }
        // reverse stage 1: source w adds its pilots' merged rows in pilot order
        // (x1 for multi-copy groups, x w for singletons; rbd.cpp:343-356)
        for (int w = 0; w < W; ++w) {
            const int S = static_cast<int>(seq_lens[w]);
            if (S == 0) continue;
            launch_combine(dtype, merged, static_cast<int>(H), src_ptr[w], src_flat[w], 0, flat_scale, S, nullptr,
                           out[w], st);
        }
    });
}

int xmoe_route_pairs(xmoe_ctx* ctx, int64_t n, const int32_t* token, const int32_t* expert,
                     const int32_t* expert_node, int64_t E, int64_t nodes, int64_t tokens, int64_t skip_node,
                     int64_t* copies, int64_t* groups, void* stream) {
    return guarded([&] {
        auto st = static_cast<cudaStream_t>(stream);
        *copies = 0;
        *groups = 0;
        if (n == 0) return;
        require(nodes >= 1 && tokens >= 1, XMOE_ERR_VALIDATION, "route_pairs: bounds must be >= 1");
        Carve cv(ctx->c.scratch(sizeof(int32_t) * (tokens * nodes + 64) + 4096));
        unsigned long long* acc = cv.take<unsigned long long>(2);
        int* err = cv.take<int>(4);
        int32_t* mark = cv.take<int32_t>(tokens * nodes);
        XMOE_CUDA(cudaMemsetAsync(acc, 0, 16, st));
        XMOE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
        XMOE_CUDA(cudaMemsetAsync(mark, 0, sizeof(int32_t) * tokens * nodes, st));
        pair_mark_kernel<<<std::min(ceil_div(n, 256), 4 * kNumSMs), 256, 0, st>>>(
            static_cast<int>(n), token, expert, expert_node, static_cast<int>(E), static_cast<int>(nodes),
            static_cast<int>(tokens), static_cast<int>(skip_node), mark, acc, err);
        XMOE_LAUNCH_CHECK();
        unsigned long long h[2];
        XMOE_CUDA(cudaMemcpyAsync(h, acc, 16, cudaMemcpyDeviceToHost, st));
        check_err(err, st, "", "");
        *copies = static_cast<int64_t>(h[0]);
        *groups = static_cast<int64_t>(h[1]);
    });
}

}  // extern "C"
