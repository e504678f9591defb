// MoE layer: weights in the B200 layout, per-rank workspace, and the forward
// pipeline that restates moesim::pf_moe_forward (pf_pipeline.cpp:137-169),
// rbd_moe_forward (rbd.cpp:360-386) and ssmb_forward (ssmb.cpp:12-46):
//
//   gate -> PFT -> [RBD groups] -> count all-gather -> dispatch
//        -> grouped expert FFN (+ shared experts) -> [RBD merge]
//        -> combine
//
// Row movement between ranks.  Ranks that share a device (rank == -1
// contexts, or world 1) and ranks in separate processes with NVLink peer
// access ("p2p") use the SAME kernels over device pointer tables: the
// unchunked dispatch kernel gathers token rows and stores them straight into
// the owner's grouped expert input (a peer address when the owner is another
// GPU); the token-chunked pipeline (default at N > 1) has the owners pull
// their rows instead, on SMs the expert GEMMs leave free (chunk.cu); the
// combine kernel reads expert outputs straight out of the owners' buffers
// while it reduces.  No host synchronisation: the count all-gather and epoch
// flags in the symmetric regions order the ranks.  The NCCL send/recv
// transport (XMOE_TRANSPORT=nccl, plain dispatch only) is kept as the
// library-collective baseline it is measured against.
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "layer.h"
#include "rbd.h"

namespace xmoe {

#define XMOE_NCCL(expr)                                                                \
    do {                                                                               \
        ncclResult_t _r = (expr);                                                      \
        if (_r != ncclSuccess)                                                         \
            ::xmoe::fail(XMOE_ERR_NCCL, std::string(#expr ": ") + ncclGetErrorString(_r)); \
    } while (0)

// Split-K factor of a single-group weight gradient D[M, N] over `rows`
// tokens: the fewest splits whose tiles fill >= 85 % of the last round of
// the 74 SM pairs (at most 16, and at least 512 rows per split).
static int wgrad_splits(long long M, long long N, long long rows) {
    const long long pairs = kNumSMs / 2;
    const long long tiles = ((M + 255) / 256) * (((N + 127) / 128 * 128 + 255) / 256);
    int s = 1;
    for (; s < 16; ++s) {
        const long long t = tiles * s;
        if (static_cast<double>(t) / (static_cast<double>((t + pairs - 1) / pairs) * pairs) >= 0.85) break;
    }
    while (s > 1 && rows / s < 512) --s;
    return s;
}

static size_t elem_size_of(int dtype) { return dtype == XMOE_F64 ? 8 : dtype == XMOE_F32 ? 4 : 2; }

Layer::~Layer() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (side) cudaStreamDestroy(side);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (comm) cudaStreamDestroy(comm);
    for (cudaEvent_t e : {ev_fork, ev_join, ev_side0, ev_side1, ev_done, ev_routed})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : evA) cudaEventDestroy(e);
    for (cudaEvent_t e : evB) cudaEventDestroy(e);
    for (cudaEvent_t e : tl) cudaEventDestroy(e);
    for (cudaEvent_t e : bev) cudaEventDestroy(e);
    for (void* p : peer_maps) cudaIpcCloseMemHandle(p);
    for (void* p : allocs) cudaFree(p);
    for (auto& e : events) cudaEventDestroy(e);
    if (peer_err_h) cudaFreeHost(peer_err_h);
}

// Cross-rank quiesce before the symmetric region is unmapped and freed: a
// peer's last combine may still be reading this rank's expert outputs over
// NVLink.  One flag barrier on a dedicated slot (same epoch on every rank:
// every rank ran the same forwards), then a local synchronise.
void Layer::quiesce() {
    if (!(distributed && p2p) || !flag_tab || !epoch) return;
    XMOE_CUDA(cudaDeviceSynchronize());  // this rank's own passes are done
    launch_flag_barrier(flag_tab, workers[0].flags, W, workers[0].rank, kSlotQuiesce, epoch, peer_err_d, cap_stream);
    XMOE_CUDA(cudaStreamSynchronize(cap_stream));
}

// XMOE_ERR_PEER_TIMEOUT when a peer-flag wait of an earlier pass gave up
void Layer::check_peers() const {
    if (peer_err_h && *reinterpret_cast<volatile int*>(peer_err_h) != 0)
        fail(XMOE_ERR_PEER_TIMEOUT, "a peer rank did not reach flag slot " +
                                        std::to_string(*peer_err_h & 0xff) +
                                        " within XMOE_PEER_TIMEOUT_S; the layer's exchange state is invalid");
}

void* Layer::alloc(size_t bytes) {
    void* p = nullptr;
    XMOE_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    allocs.push_back(p);
    return p;
}

// Stage boundary: a CUDA event in timing mode, and always an NVTX range per
// stage (gate, pft, dispatch, experts, shared, combine) for nsys/ncu timelines.
void Layer::mark(int ev, cudaStream_t st) {
    if (timing) XMOE_CUDA(cudaEventRecord(events[ev], st));
    static const char* const kNames[kNumEvents] = {"xmoe.gate", "xmoe.pft", "xmoe.dispatch", "xmoe.experts",
                                                   "xmoe.shared", "xmoe.combine", nullptr, nullptr,
                                                   nullptr, nullptr};
    if (ev == kEvCounts || ev == kEvMoved || ev == kEvReturn) return;  // sub-stage markers
    if (nvtx_open) nvtxRangePop();
    nvtx_open = ev != kEvCombine && kNames[ev] != nullptr;
    if (nvtx_open) nvtxRangePushA(kNames[ev]);
}

void Layer::barrier(cudaStream_t st) {
    XMOE_NCCL(ncclAllReduce(bar, bar, 1, ncclInt32, ncclSum, static_cast<ncclComm_t>(ctx->nccl), st));
}

long long Layer::C(int s, int d) const {
    long long a = 0;
    for (int le = 0; le < El; ++le) a += h_tpe[static_cast<size_t>(s) * E + d * El + le];
    return a;
}

// Weights in, from the reference layouts (moe_instance.hpp:17-21): F64 keeps
// them; BF16 goes K-major (gate [E,H], w1 [El,F,H], w2 [El,H,F], merged
// shared [ns*Fs,H] / [H,ns*Fs]); training layers also refresh their
// reference-layout copies (the dgrad B operands).  Stream-ordered on st.
void layer_load_weights(Layer& L, const void* gate, const void* w1, const void* w2, const void* sw1, const void* sw2,
                        cudaStream_t st) {
    const int H = L.H, F = L.F, E = L.E;
    const size_t es = L.es;
    const bool bf = L.d.dtype == XMOE_BF16;
    const size_t ew = static_cast<size_t>(L.E_held) * H * F;
    const auto cp = [&](void* d, const void* s, size_t b) {
        XMOE_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToDevice, st));
    };
    if (!bf) {
        cp(L.gate, gate, static_cast<size_t>(H) * E * es);
        cp(L.w1, w1, ew * es);
        cp(L.w2, w2, ew * es);
    } else {
        launch_transpose(XMOE_BF16, gate, 1, H, E, XMOE_BF16, L.gate, st);       // [E,H]
        launch_transpose(XMOE_BF16, w1, L.E_held, H, F, XMOE_BF16, L.w1, st);    // [El,F,H]
        launch_transpose(XMOE_BF16, w2, L.E_held, F, H, XMOE_BF16, L.w2, st);    // [El,H,F]
    }
    const int ns = static_cast<int>(L.d.n_shared), Fs1 = static_cast<int>(L.d.shared_ffn_dim);
    // merged shared FFN (moe_oracle.shared_expert_forward): W1cat [H, ns*Fs], W2cat [ns*Fs, H]
    const auto cat_w1 = [&](void* dst) {
        for (int s = 0; s < ns; ++s)
            XMOE_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + static_cast<size_t>(s) * Fs1 * es,
                                        static_cast<size_t>(L.Fs) * es,
                                        static_cast<const char*>(sw1) + static_cast<size_t>(s) * H * Fs1 * es,
                                        static_cast<size_t>(Fs1) * es, static_cast<size_t>(Fs1) * es, H,
                                        cudaMemcpyDeviceToDevice, st));
    };
    if (L.Fs > 0) {
        if (!bf) {
            cat_w1(L.sw1);
            cp(L.sw2, sw2, static_cast<size_t>(H) * L.Fs * es);
        } else {
            launch_transpose(XMOE_BF16, sw1, ns, H, Fs1, XMOE_BF16, L.sw1, st);  // [ns*Fs, H]
            launch_transpose(XMOE_BF16, sw2, 1, L.Fs, H, XMOE_BF16, L.sw2, st);  // [H, ns*Fs]
        }
    }
    if (L.train) {
        cp(L.w1r, w1, ew * es);
        cp(L.w2r, w2, ew * es);
        cp(L.gater, gate, static_cast<size_t>(H) * E * es);
        if (L.Fs > 0) {
            cat_w1(L.sw1r);
            cp(L.sw2r, sw2, static_cast<size_t>(H) * L.Fs * es);
        }
    }
}

// ---------------------------------------------------------------- creation
void layer_create(Ctx& ctx, const xmoe_layer_desc& d, const void* gate, const void* w1,
                  const void* w2, const void* sw1, const void* sw2, Layer& L) {
    const bool ssmb = d.flags & XMOE_LAYER_SSMB;
    const int W = ssmb ? 1 : ctx.world;
    require(d.num_experts >= 1, XMOE_ERR_VALIDATION, "num_experts must be >= 1");
    require(d.top_k >= 1, XMOE_ERR_VALIDATION, "top_k must be >= 1");
    require(d.top_k <= d.num_experts, XMOE_ERR_VALIDATION, "top_k must be <= num_experts");
    require(d.max_token_count >= 1, XMOE_ERR_VALIDATION, "max_token_count must be >= 1");
    require(d.num_experts % W == 0, XMOE_ERR_VALIDATION,
            "num_experts must be divisible by the worker-group size");
    require(d.model_dim >= 1 && d.ffn_dim >= 1, XMOE_ERR_VALIDATION, "dims must be >= 1");
    // kernel limits checked up front, so a layer never fails half-way through a pass
    require(d.num_experts <= 1024, XMOE_ERR_VALIDATION, "num_experts must be <= 1024");
    require(!(d.flags & XMOE_LAYER_TRAIN) || (d.num_experts <= 256 && d.top_k <= 32), XMOE_ERR_VALIDATION,
            "training layers support num_experts <= 256 and top_k <= 32");
    require(d.dispatch_mode == XMOE_DISPATCH_NAIVE || d.dispatch_mode == XMOE_DISPATCH_RBD,
            XMOE_ERR_VALIDATION, "unknown dispatch mode");
    const bool bf = d.dtype == XMOE_BF16;
    require(bf || d.dtype == XMOE_F64 || d.dtype == XMOE_F32, XMOE_ERR_VALIDATION, "unknown dtype");
    if (bf) {
        require(d.num_experts % 16 == 0, XMOE_ERR_VALIDATION,
                "bf16 path requires num_experts to be a multiple of 16");
        require(d.top_k <= 32, XMOE_ERR_VALIDATION, "bf16 path requires top_k <= 32");
        require(d.model_dim % 16 == 0 && d.ffn_dim % 16 == 0, XMOE_ERR_VALIDATION,
                "bf16 path requires model_dim and ffn_dim to be multiples of 16");
        require(d.n_shared == 0 || (d.n_shared * d.shared_ffn_dim) % 16 == 0, XMOE_ERR_VALIDATION,
                "bf16 path requires n_shared*shared_ffn_dim to be a multiple of 16");
    }
    L.ctx = &ctx;
    L.d = d;
    L.ssmb = ssmb;
    L.W = W;
    L.nl = ssmb ? 1 : ctx.n_local();
    L.distributed = !ssmb && ctx.rank >= 0 && W > 1;
    L.E = static_cast<int>(d.num_experts);
    L.H = static_cast<int>(d.model_dim);
    L.F = static_cast<int>(d.ffn_dim);
    L.k = static_cast<int>(d.top_k);
    L.El = L.E / W;
    L.E_held = L.distributed ? L.El : L.E;
    L.Fs = static_cast<int>(d.n_shared * d.shared_ffn_dim);
    L.es = elem_size_of(d.dtype);
    const bool rbd = d.dispatch_mode == XMOE_DISPATCH_RBD;
    if (L.distributed) {
        const char* tr = std::getenv("XMOE_TRANSPORT");
        L.p2p = !(tr && std::string(tr) == "nccl");
        require(L.p2p || !rbd, XMOE_ERR_VALIDATION,
                "the redundancy-bypassing dispatch runs on the NVLink peer transport");
    }
    L.gpn = std::max(1, XMOE_LAYER_GPUS_PER_NODE_OF(d.flags));
    {
        // XMOE_RBD_GATHER=1: RBD replicas read their pilot's row through a TMA
        // gather4 A-load in GEMM1 instead of the expand copy (training layers
        // keep the copies: the wgrad reads them).  Bit-identical, but measured
        // slower (GEMM1 0.97 -> 1.83 ms at N=2 for 0.05 ms of expand saved:
        // 4-row gathers move A at a fraction of a 128-row box), so opt-in.
        const char* e = std::getenv("XMOE_RBD_GATHER");
        L.rbd_gather = d.dispatch_mode == XMOE_DISPATCH_RBD && d.dtype == XMOE_BF16 && L.gpn == 1 &&
                       !(d.flags & XMOE_LAYER_TRAIN) && d.ffn_dim % 32 == 0 && e && std::atoi(e) == 1;
    }
    require(W % L.gpn == 0, XMOE_ERR_VALIDATION, "the worker group must be whole nodes (world % gpus_per_node)");
    require(L.gpn == 1 || rbd, XMOE_ERR_VALIDATION, "gpus_per_node applies to the redundancy-bypassing dispatch");
    const int H = L.H, F = L.F, E = L.E;
    const size_t es = L.es;
    cudaStream_t st = nullptr;

    // ---- weights: F64 keeps the reference layouts; BF16 goes K-major
    L.gate = L.alloc(static_cast<size_t>(H) * E * es);
    L.w1 = L.alloc(static_cast<size_t>(L.E_held) * H * F * es);
    L.w2 = L.alloc(static_cast<size_t>(L.E_held) * H * F * es);
    if (L.Fs > 0) {
        require(sw1 && sw2, XMOE_ERR_VALIDATION, "shared expert weights missing");
        L.sw1 = L.alloc(static_cast<size_t>(H) * L.Fs * es);
        L.sw2 = L.alloc(static_cast<size_t>(H) * L.Fs * es);
    }
    (void)st;
    // ---- per-rank workspace
    const long long S = d.max_tokens;
    require(S >= 1, XMOE_ERR_VALIDATION, "max_tokens must be >= 1");
    const long long nk = S * L.k;
    const long long per_src = S * std::min<long long>(L.k, L.El);
    const long long cap_bound = static_cast<long long>(W) * L.El * d.max_token_count;
    L.R_max = std::max<long long>(1, std::min<long long>(static_cast<long long>(W) * per_src, cap_bound));
    L.S_max = S;
    // token-chunked pipeline (chunk.cu): BF16 plain dispatch over pointer tables
    L.train = (d.flags & XMOE_LAYER_TRAIN) != 0;
    {
        const int req = XMOE_LAYER_CHUNKS_OF(d.flags);
        require(req <= kMaxChunks, XMOE_ERR_VALIDATION, "at most 8 token chunks");
        const bool can = bf && !L.train && (!L.distributed || L.p2p) && L.k <= 32 && L.gpn == 1 && L.H % 8 == 0;
        // default: up to min(4, W) chunks, keeping >= 512 rows per local
        // expert per chunk on average (W*S*k/E per expert and forward): below
        // that the chunk GEMMs pay padding tiles for the overlap (B200, N=4:
        // C3 / C4 are fastest at 2 chunks, C2 / C5 at 4)
        const long long rows_pe = static_cast<long long>(W) * S * L.k / std::max(1, L.E);
        const int C_auto = static_cast<int>(std::max<long long>(1, std::min<long long>(std::min(4, W), rows_pe / 512)));
        int C = req > 0 ? req : (S >= 4096 && L.distributed && !rbd ? C_auto : 1);
        if (const char* e = std::getenv("XMOE_CHUNKS")) C = std::max(1, std::min(kMaxChunks, std::atoi(e)));
        L.nchunks = can ? static_cast<int>(std::max<long long>(1, std::min<long long>(C, S))) : 1;
        if (L.nchunks > 1) {
            const long long cs = chunk_max_tokens(S, L.nchunks);
            const long long rc = std::min<long long>(static_cast<long long>(W) * cs * std::min<long long>(L.k, L.El),
                                                     static_cast<long long>(W) * L.El *
                                                         std::min<long long>(d.max_token_count, cs));
            require(rc * L.nchunks < (1LL << 31), XMOE_ERR_VALIDATION, "chunk regions exceed 2^31 rows");
            L.Rc = static_cast<int>(std::max<long long>(1, rc));
            L.R_max = std::max<long long>(L.R_max, static_cast<long long>(L.Rc) * L.nchunks);
        }
    }
    // pull dispatch (default on the chunked plain path; XMOE_DISPATCH=push
    // keeps the source-side stores, A/B)
    {
        const char* e = std::getenv("XMOE_DISPATCH");
        L.pull = L.nchunks > 1 && !rbd && H % 8 == 0 && !(e && std::string(e) == "push");
        require(!L.pull || (S < (1LL << 24) && W <= 255), XMOE_ERR_VALIDATION,
                "pull dispatch: max_tokens < 2^24 and world <= 255");
    }
    L.route_cnt_ok = bf && gate_route_supported(L.E, L.k, L.H);
    if (bf && !L.distributed && L.nl == 1 && L.Fs > 0 && !L.ssmb) {  // late shared GEMM2 (layer_forward_v)
        L.partial = static_cast<float*>(L.alloc(sizeof(float) * S * L.H));
        L.ready = static_cast<unsigned*>(L.alloc(sizeof(unsigned) * ((S + 127) / 128 + 1)));
    }
    const long long gmax = S * std::min<long long>(L.k, W);  // RBD groups per source
    const long long rmax = static_cast<long long>(W) * S;   // RBD groups received
    L.tpe_all = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * W * E));
    L.G_all = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * W * W));
    L.bar = static_cast<int32_t*>(L.alloc(64));
    if (L.nchunks > 1) L.tpe_c_all = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * W * L.nchunks * E));
    if (rbd) L.gd_all = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * 2 * W * W * L.nchunks));
    // symmetric region (same offsets on every rank; exported over IPC in p2p mode)
    auto up = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    const size_t off_recv = 0;
    const size_t off_eout = off_recv + up(static_cast<size_t>(L.R_max) * H * es);
    const size_t off_recv_u = off_eout + up(static_cast<size_t>(L.R_max) * H * es);
    const size_t off_desc = off_recv_u;  // RBD rows land in place (pilot slot): no unique-row buffer
    const size_t off_back = off_desc + (rbd ? up(sizeof(RbdDesc) * L.R_max) : 0);
    const size_t off_train = off_back + (rbd ? up(static_cast<size_t>(rmax) * H * es) : 0);
    require(!L.train || (bf && !d.renorm && (!L.distributed || L.p2p) && L.nl == 1), XMOE_ERR_VALIDATION,
            "training layers need bf16, no renorm, one rank per process (or world 1) and the NVLink peer transport");
    require(!L.train || (H % 128 == 0 && F % 128 == 0 && E % 32 == 0 && L.Fs % 128 == 0), XMOE_ERR_VALIDATION,
            "training layers need model_dim, ffn_dim and shared width multiples of 128, num_experts of 32");
    const size_t off_dyg = off_train;
    const size_t off_dxc = off_dyg + (L.train ? up(static_cast<size_t>(L.R_max) * H * es) : 0);
    const size_t off_gw = off_dxc + (L.train ? up(static_cast<size_t>(L.R_max) * H * es) : 0);
    const size_t off_gsrc = off_gw + (L.train ? up(sizeof(float) * L.R_max) : 0);
    const size_t off_sdw = off_gsrc + (L.train ? up(sizeof(unsigned long long) * L.R_max) : 0);
    const size_t off_xs = off_sdw + (L.train ? up(sizeof(float) * nk) : 0);
    const size_t off_rsrc = off_xs + (L.pull ? up(static_cast<size_t>(S) * H * es) : 0);
    const size_t off_flags = off_rsrc + (L.pull ? up(sizeof(int32_t) * L.R_max) : 0);
    const size_t flag_bytes = sizeof(unsigned) * kFlagSlots * W;
    // count all-gather area (double-buffered): tpe [W,E] | tpe_c [W,C,E] | G [W,W] | gd [W,2,W,C]
    L.area_ints = W * E + W * L.nchunks * E + W * W + 2 * W * W * L.nchunks;
    const size_t off_counts = off_flags + up(flag_bytes);
    const size_t sym_bytes = off_counts + up(sizeof(int32_t) * 2 * L.area_ints);
    L.off_eout = static_cast<long long>(off_eout);
    L.off_dxc = static_cast<long long>(off_dxc);
    L.workers.resize(L.nl);
    std::vector<char*> t_recv(W), t_eout(W), t_recv_u(W), t_desc(W), t_back(W);
    std::vector<char*> t_dyg(W), t_dxc(W), t_gw(W), t_gsrc(W), t_sdw(W), t_flags(W), t_counts(W), t_xs(W), t_rsrc(W);
    for (int i = 0; i < L.nl; ++i) {
        Worker& w = L.workers[i];
        w.rank = ssmb ? 0 : ctx.rank_of(i);
        w.logits = static_cast<double*>(L.alloc(sizeof(double) * S * E));
        w.top = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.wts = static_cast<double*>(L.alloc(sizeof(double) * nk));
        w.token_ids = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.expert_ids = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.cw = static_cast<double*>(L.alloc(sizeof(double) * nk));
        w.slot_pos = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.B_dev = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * 4));
        w.tpe = L.distributed ? static_cast<int32_t*>(L.alloc(sizeof(int32_t) * E))
                              : L.tpe_all + static_cast<size_t>(w.rank) * E;
        w.pft_ws = L.alloc(bucket_ws_bytes(nk, E));
        if (L.route_cnt_ok)
            w.route_cnt = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * ((S + kRouteTile - 1) / kRouteTile) * E));
        w.dest_rank = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.dest_row = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.slot_src = static_cast<unsigned long long*>(L.alloc(sizeof(unsigned long long) * nk));
        w.slot_w = static_cast<float*>(L.alloc(sizeof(float) * nk));
        w.rpe = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * L.El));
        w.sym = static_cast<char*>(L.alloc(sym_bytes));
        w.flags = reinterpret_cast<unsigned*>(w.sym + off_flags);
        XMOE_CUDA(cudaMemset(w.flags, 0, flag_bytes));
        t_counts[w.rank] = w.sym + off_counts;
        if (L.nchunks > 1) {
            const int CE = L.nchunks * E;
            w.tpe_c = L.distributed ? static_cast<int32_t*>(L.alloc(sizeof(int32_t) * CE)) : nullptr;
            w.pfx_c = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * CE));
            w.seg = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * E));
            w.cbase = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * CE));
            w.rpe_c = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * L.nchunks * L.El));
        }
        w.recv = w.sym + off_recv;
        w.eout = w.sym + off_eout;
        if (L.pull) {
            w.xs = w.sym + off_xs;
            w.rsrc = reinterpret_cast<int32_t*>(w.sym + off_rsrc);
            const char* le = std::getenv("XMOE_CHUNK_LATE");
            if (L.Fs > 0 && le && std::atoi(le) == 1) {  // late shared GEMM2 of the chunked forward (A/B)
                w.lpartial = static_cast<float*>(L.alloc(sizeof(float) * S * H));
                w.lready = static_cast<unsigned*>(L.alloc(sizeof(unsigned) * ((S + 127) / 128 + 1)));
            }
        }
        w.mid = L.alloc(static_cast<size_t>(L.R_max) * F * es);
        if (L.distributed && !L.p2p) {
            w.send = L.alloc(static_cast<size_t>(nk) * H * es);
            w.back = L.alloc(static_cast<size_t>(nk) * H * es);
        }
        w.s_rows = static_cast<int32_t*>(L.alloc(sizeof(int32_t)));
        if (L.Fs > 0) {
            w.smid = L.alloc(static_cast<size_t>(S) * L.Fs * es);
            w.sout = L.alloc(static_cast<size_t>(S) * H * es);
        }
        if (rbd) {
            RbdWork& r = w.rbd;
            auto i32 = [&](long long n) { return static_cast<int32_t*>(L.alloc(sizeof(int32_t) * (n + 1))); };
            r.g.token = i32(nk);
            r.g.dest = i32(nk);
            r.g.first_slot = i32(nk);
            r.g.n = i32(nk);
            r.g.pilot = i32(nk);
            r.g.pos = i32(nk);
            r.gcount = i32(S);
            r.gbase = i32(S);
            r.G_dev = i32(1);
            r.flags = i32(1);
            r.draws = static_cast<uint64_t*>(L.alloc(sizeof(uint64_t) * (nk + kRbdChunk)));
            r.dptr = i32(W + 1);
            r.perm = i32(nk);
            r.nsorted = i32(nk);
            r.scan_ws = i32(nk / 2048 + 2);
            r.coff = i32(nk);
            r.csr_ws = L.alloc(bucket_ws_bytes(nk, W));
            r.C = L.nchunks;
            r.gpn = L.gpn;
            if (L.rbd_gather) {  // identity until the first expand rewrites the received rows
                std::vector<int32_t> iota(static_cast<size_t>(L.R_max));
                for (size_t q = 0; q < iota.size(); ++q) iota[q] = static_cast<int32_t>(q);
                w.a_idx = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * iota.size()));
                XMOE_CUDA(cudaMemcpy(w.a_idx, iota.data(), sizeof(int32_t) * iota.size(), cudaMemcpyHostToDevice));
            }
            r.gpos = i32(static_cast<long long>(W) * (r.C + 1));
            r.gd_own = L.distributed ? i32(2LL * W * r.C)
                                     : L.gd_all + static_cast<size_t>(w.rank) * 2 * W * r.C;
            r.ru = i32(static_cast<long long>(W) * r.C);
            r.rd = i32(static_cast<long long>(W) * r.C);
            r.cs = i32(static_cast<long long>(W) * r.C);
            r.rx = i32(4LL * r.C);
            rng_state_from_seed(salt_seed_host(d.seed, static_cast<uint64_t>(w.rank), 0), r.state);
            w.recv_u = w.sym + off_recv_u;
            w.desc_recv = reinterpret_cast<RbdDesc*>(w.sym + off_desc);
            w.back_u = w.sym + off_back;
            w.gstart = i32(rmax);
        }
        if (L.train) {
            const long long Fs = L.Fs;
            w.dyg = w.sym + off_dyg;
            w.dxc = w.sym + off_dxc;
            w.gw = reinterpret_cast<float*>(w.sym + off_gw);
            w.gsrc = reinterpret_cast<unsigned long long*>(w.sym + off_gsrc);
            w.slot_dw = reinterpret_cast<float*>(w.sym + off_sdw);
            w.dz = L.alloc(static_cast<size_t>(L.R_max) * H * es);
            w.dH = L.alloc(static_cast<size_t>(L.R_max) * F * es);
            const size_t wide = std::max<size_t>({static_cast<size_t>(H), static_cast<size_t>(F),
                                                  static_cast<size_t>(Fs)});
            w.tail_a = L.alloc(64 * static_cast<size_t>(L.El + 1) * wide * es);
            w.tail_b = L.alloc(64 * static_cast<size_t>(L.El + 1) * wide * es);
            // ReLU masks of the forward's first GEMMs (bits), the dgrad's masks
            w.mbits = static_cast<uint32_t*>(L.alloc(sizeof(uint32_t) * L.R_max * ((F + 31) / 32)));
            if (Fs > 0) w.smbits = static_cast<uint32_t*>(L.alloc(sizeof(uint32_t) * S * ((Fs + 31) / 32)));
            // single-group weight gradients, split along the tokens (K) so
            // that their few output tiles fill the SM pairs
            L.splits_s1 = wgrad_splits(H, static_cast<int>(Fs), S);
            L.splits_s2 = wgrad_splits(static_cast<int>(Fs), H, S);
            L.splits_g = wgrad_splits(H, E, S);
            const int ss = std::max(L.splits_s1, L.splits_s2);
            w.tail_sa = L.alloc(64 * static_cast<size_t>(std::max(ss, 2)) * wide * es);  // side-stream copies
            w.tail_sb = L.alloc(64 * static_cast<size_t>(std::max(ss, 2)) * wide * es);
            w.split_s = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * 32));
            w.split_g = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * 32));
            const auto r128 = [](long long n) { return (n + 127) / 128 * 128; };
            if (Fs > 0)
                w.part_s = static_cast<float*>(L.alloc(sizeof(float) * ss *
                                                       std::max(H * r128(Fs), Fs * r128(H))));
            w.part_g = static_cast<float*>(L.alloc(sizeof(float) * L.splits_g * H * r128(E)));
            w.tail_ga = L.alloc(64 * static_cast<size_t>(L.splits_g) * H * es);
            w.tail_gb = L.alloc(64 * static_cast<size_t>(L.splits_g) * E * es);
            w.dl = L.alloc(static_cast<size_t>(S) * E * es);
            w.dxg = L.alloc(static_cast<size_t>(S) * H * es);
            if (Fs > 0) {
                w.dHs = L.alloc(static_cast<size_t>(S) * Fs * es);
                w.dxs = L.alloc(static_cast<size_t>(S) * H * es);
            }
            w.bslot_src = static_cast<unsigned long long*>(L.alloc(sizeof(unsigned long long) * nk));
        }
        if (L.nchunks > 1 && !L.distributed) w.tpe_c = L.tpe_c_all + static_cast<size_t>(w.rank) * L.nchunks * E;
        t_flags[w.rank] = reinterpret_cast<char*>(w.flags);
        t_recv[w.rank] = static_cast<char*>(w.recv);
        t_eout[w.rank] = static_cast<char*>(w.eout);
        t_dyg[w.rank] = static_cast<char*>(w.dyg);
        t_dxc[w.rank] = static_cast<char*>(w.dxc);
        t_gw[w.rank] = reinterpret_cast<char*>(w.gw);
        t_gsrc[w.rank] = reinterpret_cast<char*>(w.gsrc);
        t_sdw[w.rank] = reinterpret_cast<char*>(w.slot_dw);
        t_recv_u[w.rank] = static_cast<char*>(w.recv_u);
        t_desc[w.rank] = reinterpret_cast<char*>(w.desc_recv);
        t_back[w.rank] = static_cast<char*>(w.back_u);
        t_xs[w.rank] = w.xs;
        t_rsrc[w.rank] = reinterpret_cast<char*>(w.rsrc);
    }
    if (L.distributed && L.p2p) {
        // export my symmetric region, import every peer's (CUDA IPC over NVLink)
        Worker& w = L.workers[0];
        cudaIpcMemHandle_t mine;
        XMOE_CUDA(cudaIpcGetMemHandle(&mine, w.sym));
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
        char* hb = static_cast<char*>(L.alloc(64 * W));
        XMOE_CUDA(cudaMemcpy(hb + 64 * w.rank, &mine, 64, cudaMemcpyHostToDevice));
        XMOE_NCCL(ncclAllGather(hb + 64 * w.rank, hb, 64, ncclUint8, static_cast<ncclComm_t>(ctx.nccl), st));
        std::vector<cudaIpcMemHandle_t> hs(W);
        XMOE_CUDA(cudaMemcpy(hs.data(), hb, 64 * W, cudaMemcpyDeviceToHost));
        for (int r = 0; r < W; ++r) {
            if (r == w.rank) continue;
            void* p = nullptr;
            XMOE_CUDA(cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess));
            L.peer_maps.push_back(p);
            char* b = static_cast<char*>(p);
            t_recv[r] = b + off_recv;
            t_eout[r] = b + off_eout;
            t_dyg[r] = b + off_dyg;
            t_dxc[r] = b + off_dxc;
            t_gw[r] = b + off_gw;
            t_gsrc[r] = b + off_gsrc;
            t_sdw[r] = b + off_sdw;
            t_recv_u[r] = b + off_recv_u;
            t_desc[r] = b + off_desc;
            t_back[r] = b + off_back;
            t_flags[r] = b + off_flags;
            t_counts[r] = b + off_counts;
            t_xs[r] = b + off_xs;
            t_rsrc[r] = b + off_rsrc;
        }
    }
    auto table = [&](const std::vector<char*>& v) {
        char** t = static_cast<char**>(L.alloc(sizeof(char*) * W));
        XMOE_CUDA(cudaMemcpy(t, v.data(), sizeof(char*) * W, cudaMemcpyHostToDevice));
        return t;
    };
    L.recv_tab = table(t_recv);
    L.flag_tab = reinterpret_cast<unsigned**>(table(t_flags));
    L.cnt_tab = reinterpret_cast<int32_t**>(table(t_counts));
    XMOE_CUDA(cudaHostAlloc(&L.peer_err_h, sizeof(int), cudaHostAllocMapped));
    *L.peer_err_h = 0;
    XMOE_CUDA(cudaHostGetDevicePointer(&L.peer_err_d, L.peer_err_h, 0));
    L.epoch = static_cast<unsigned*>(L.alloc(sizeof(unsigned)));
    XMOE_CUDA(cudaMemset(L.epoch, 0, sizeof(unsigned)));
    L.eout_tab = table(t_eout);
    if (L.pull) {
        L.xs_tab = table(t_xs);
        L.rsrc_tab = reinterpret_cast<int32_t**>(table(t_rsrc));
    }
    if (L.train) {
        L.dyg_tab = table(t_dyg);
        L.dxc_tab = table(t_dxc);
        L.gw_tab = reinterpret_cast<float**>(table(t_gw));
        L.gsrc_tab = reinterpret_cast<unsigned long long**>(table(t_gsrc));
        L.slotdw_tab = reinterpret_cast<float**>(table(t_sdw));
        // reference-layout copies of the weights (dgrad B operands) + fp32 grads
        const size_t ew = static_cast<size_t>(L.E_held) * H * F;
        L.w1r = L.alloc(ew * es);
        L.w2r = L.alloc(ew * es);
        L.gater = L.alloc(static_cast<size_t>(H) * E * es);
        L.dgate = static_cast<float*>(L.alloc(sizeof(float) * H * E));
        L.dw1 = static_cast<float*>(L.alloc(sizeof(float) * ew));
        L.dw2 = static_cast<float*>(L.alloc(sizeof(float) * ew));
        if (L.Fs > 0) {
            L.sw1r = L.alloc(static_cast<size_t>(H) * L.Fs * es);
            L.sw2r = L.alloc(static_cast<size_t>(H) * L.Fs * es);
            L.dsw1 = static_cast<float*>(L.alloc(sizeof(float) * H * L.Fs));
            L.dsw2 = static_cast<float*>(L.alloc(sizeof(float) * H * L.Fs));
        }
    }
    if (rbd) {
        L.recv_u_tab = table(t_recv_u);
        L.desc_tab = reinterpret_cast<RbdDesc**>(table(t_desc));
        L.back_tab = table(t_back);
        std::vector<uint64_t> jt;
        rbd_jump_tables(jt);
        L.jumps = static_cast<uint64_t*>(L.alloc(sizeof(uint64_t) * jt.size()));
        XMOE_CUDA(cudaMemcpy(L.jumps, jt.data(), sizeof(uint64_t) * jt.size(), cudaMemcpyHostToDevice));
    }
    layer_load_weights(L, gate, w1, w2, sw1, sw2, nullptr);
    L.events.resize(kNumEvents);
    for (auto& e : L.events) XMOE_CUDA(cudaEventCreate(&e));
    if (L.train) {
        L.bev.resize(kBwdEvents);
        for (auto& e : L.bev) XMOE_CUDA(cudaEventCreate(&e));
    }
    XMOE_CUDA(cudaStreamCreateWithFlags(&L.side, cudaStreamNonBlocking));
    XMOE_CUDA(cudaStreamCreateWithFlags(&L.cap_stream, cudaStreamNonBlocking));
    XMOE_CUDA(cudaEventCreateWithFlags(&L.ev_fork, cudaEventDisableTiming));
    XMOE_CUDA(cudaEventCreateWithFlags(&L.ev_join, cudaEventDisableTiming));
    XMOE_CUDA(cudaEventCreateWithFlags(&L.ev_routed, cudaEventDisableTiming));
    XMOE_CUDA(cudaEventCreate(&L.ev_side0));
    XMOE_CUDA(cudaEventCreate(&L.ev_side1));
    if (L.nchunks > 1) {
        XMOE_CUDA(cudaStreamCreateWithFlags(&L.comm, cudaStreamNonBlocking));
        L.evA.resize(L.nchunks);
        L.evB.resize(L.nchunks);
        for (auto* v : {&L.evA, &L.evB})
            for (auto& e : *v) XMOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        XMOE_CUDA(cudaEventCreateWithFlags(&L.ev_done, cudaEventDisableTiming));
        L.tl.resize(4 * L.nchunks);
        for (auto& e : L.tl) XMOE_CUDA(cudaEventCreate(&e));
    }
    XMOE_CUDA(cudaDeviceSynchronize());
}

// expert weights of the worker owning rank r, inside this layer's allocation
static const void* w1_of(const Layer& L, int r) {
    const size_t off = L.distributed ? 0 : static_cast<size_t>(r) * L.El * L.H * L.F * L.es;
    return static_cast<const char*>(L.w1) + off;
}
static const void* w2_of(const Layer& L, int r) {
    const size_t off = L.distributed ? 0 : static_cast<size_t>(r) * L.El * L.H * L.F * L.es;
    return static_cast<const char*>(L.w2) + off;
}

static void run_gemm(int dtype, const void* A, long long rows_bound, int K, const int32_t* rpg, int G,
                     const void* B, int N, void* D, int relu, cudaStream_t st, uint32_t* mbits_out = nullptr) {
    if (dtype == XMOE_F64)
        launch_grouped_gemm_f64(static_cast<const double*>(A), rows_bound, K, rpg, G,
                                static_cast<const double*>(B), N, static_cast<double*>(D), relu, st);
    else if (dtype == XMOE_F32)
        launch_grouped_gemm_f32(static_cast<const float*>(A), rows_bound, K, rpg, G, static_cast<const float*>(B), N,
                                static_cast<float*>(D), relu, st);
    else
        launch_grouped_gemm_bf16(A, rows_bound, K, rpg, G, B, N, D, relu, st, mbits_out);
}

// Count all-gather of the routing counts over the peer tables (one process
// per GPU): this rank's tpe row [+ chunk counts] [+ RBD group counts].
static void exchange_counts(Layer& L, cudaStream_t st) {
    Worker& w = L.workers[0];
    const int W = L.W, E = L.E, C = L.nchunks;
    const bool rbd = L.d.dispatch_mode == XMOE_DISPATCH_RBD;
    CountSegs sg{};
    sg.s[sg.n++] = CountSeg{w.tpe, E, 0, L.tpe_all};
    if (C > 1) sg.s[sg.n++] = CountSeg{w.tpe_c, C * E, W * E, L.tpe_c_all};
    if (rbd) {
        sg.s[sg.n++] = CountSeg{L.G_all + static_cast<size_t>(w.rank) * W, W, W * E + W * C * E, L.G_all};
        sg.s[sg.n++] = CountSeg{w.rbd.gd_own, 2 * W * C, W * E + W * C * E + W * W, L.gd_all};
    }
    launch_counts_exchange(sg, L.cnt_tab, L.area_ints, w.rank, W, L.flag_tab, w.flags, kSlotCounts, L.epoch, L.peer_err_d, st);
}

// XMOE_LATE_SHARED=1 (A/B, off by default): one GPU, shared GEMM2 after the
// routed GEMMs beside a combine into fp32 sums (below).  Bit-identical, but
// measured slower on B200 (C2 N=1: 1.40-1.54 ms vs 1.23-1.25 ms): the combine
// must take tokens dynamically and run beside a persistent GEMM that holds
// most of each SM, so it loses more than the overlap gains.
static bool late_shared_on() {
    static const bool on = [] {
        const char* e = std::getenv("XMOE_LATE_SHARED");
        return e && std::atoi(e) == 1;
    }();
    return on;
}

// Fused routing (BF16): the gate GEMM's epilogue does softmax + top-k from
// TMEM and writes per-tile expert histograms; the dropless placement is then
// one launch (gemm_tc.cu gate_route_kernel, pft.cu route_place_kernel) instead
// of gate GEMM + softmax + six PFT kernels.  Applies when no bucket can
// overflow (cap >= S); XMOE_FUSED_ROUTE=0 keeps the general path (A/B).
static bool fused_route(const Layer& L, long long S) {
    static const bool on = [] {
        const char* e = std::getenv("XMOE_FUSED_ROUTE");
        return !(e && std::atoi(e) == 0);
    }();
    return on && L.d.dtype == XMOE_BF16 && L.route_cnt_ok && L.d.max_token_count >= S;
}

static void route_gate(Layer& L, Worker& w, const void* x, long long S, cudaStream_t st) {
    float* lg = reinterpret_cast<float*>(w.logits);
    // XMOE_FUSED_GATE=1: softmax + top-k in the gate GEMM's epilogue (one
    // thread per token row reading TMEM).  Default: gate GEMM + warp-per-token
    // softmax/top-k writing the tile histograms — measured faster (ncu, C2:
    // 65 us for the fused kernel, whose serial per-row epilogue runs at one
    // warp per SM sub-partition, vs ~35 us for the two kernels).
    static const bool epilogue_gate = [] {
        const char* e = std::getenv("XMOE_FUSED_GATE");
        return e && std::atoi(e) == 1;
    }();
    if (fused_route(L, S) && epilogue_gate) {
        launch_gate_route(x, static_cast<int>(S), L.H, L.gate, L.E, L.k, L.d.renorm, w.top, w.wts,
                          L.train ? lg : nullptr, w.route_cnt, st);
        return;
    }
    if (fused_route(L, S)) {
        launch_grouped_gemm_bf16_f32out(x, S, L.H, w.s_rows, 1, L.gate, L.E, lg, 0, st);
        launch_softmax_topk_f32(lg, S, L.E, L.k, L.d.renorm, w.top, w.wts, st, w.route_cnt);
        return;
    }
    launch_grouped_gemm_bf16_f32out(x, S, L.H, w.s_rows, 1, L.gate, L.E, lg, 0, st);
    launch_softmax_topk_f32(lg, S, L.E, L.k, L.d.renorm, w.top, w.wts, st);
}

static void route_pft(Layer& L, Worker& w, long long S, cudaStream_t st) {
    if (fused_route(L, S)) {
        launch_route_place(w.top, w.wts, w.route_cnt, static_cast<int>(S), L.E, L.k, w.token_ids, w.expert_ids, w.cw,
                           w.tpe, w.slot_pos, w.B_dev, st);
        return;
    }
    launch_pft(w.top, w.wts, S, L.k, L.E, static_cast<int>(std::min<long long>(L.d.max_token_count, 0x7fffffff)),
               w.token_ids, w.expert_ids, w.cw, w.tpe, w.slot_pos, w.B_dev, w.pft_ws, st);
}

// ---------------------------------------------------------------- chunked forward
// BF16 forward (plain or RBD dispatch), cut into L.nchunks token chunks
// (chunk.cu).  Streams:
//   st   gate | shared-expert GEMMs | per chunk: [wait A_c] (RBD expand) GEMM1, GEMM2 (RBD merge) [signal B_c]
//   comm       PFT (+RBD groups), count exchange, destinations | per chunk: scatter / pack [signal A_c]
//              | per chunk: [wait B_c] combine
// so chunk c's expert GEMMs run while chunk c+1's rows are still moving and
// chunk c-1's outputs are being combined; the row-movement kernels need no
// shared memory and co-reside with the persistent GEMM CTAs on a bounded
// grid.  A_c / B_c are local events plus, across GPUs, epoch flags in the
// peers' symmetric regions.  Every row's arithmetic equals the unchunked
// forward's.
static void layer_forward_chunked(Layer& L, const void* x, long long S, void* out, cudaStream_t st) {
    const int W = L.W, E = L.E, H = L.H, F = L.F, k = L.k, El = L.El, C = L.nchunks;
    const size_t rb = static_cast<size_t>(H) * L.es;
    const int nl = L.nl;
    const bool dist = L.distributed;
    const long long nk = S * k;
    cudaStream_t cm = L.comm;
    const char* xb = static_cast<const char*>(x);
    char* ob = static_cast<char*>(out);
    auto x_of = [&](int i) { return xb + static_cast<size_t>(i) * S * rb; };
    auto o_of = [&](int i) { return ob + static_cast<size_t>(i) * S * rb; };
    auto t0_of = [&](int c) { return chunk_t0(c, S, C); };
    const int me = L.workers[0].rank;
    const bool rbd = L.d.dispatch_mode == XMOE_DISPATCH_RBD;
    // row-movement kernels run on a bounded grid beside the GEMMs
    static const int blk_scatter = [] {
        const char* e = std::getenv("XMOE_COPY_BLOCKS");
        return e ? std::max(1, std::atoi(e)) : 64;
    }();
    static const int blk_combine = [] {
        const char* e = std::getenv("XMOE_COPY_BLOCKS");
        const char* c = e ? std::strchr(e, ',') : nullptr;
        return c ? std::max(1, std::atoi(c + 1)) : 64;
    }();
    // optional SM partition (XMOE_PART_SMS=n): the chunk GEMMs use n SMs and
    // the row movement reserves enough shared memory to stay off them
    static const int part_sms = [] {
        const char* e = std::getenv("XMOE_PART_SMS");
        return e ? std::atoi(e) : 0;
    }();
    const int copy_smem = part_sms > 0 ? 32 * 1024 : 0;
    // SM partition (pull dispatch): XMOE_COMM_SMS whole SMs move rows, the
    // GEMMs take the rest (measured on B200: a chunk GEMM beside SM-driven
    // row copies on shared SMs runs 1.5x slower; on 124 SMs beside 24 copy
    // SMs, 1.07-1.17x, the copies at 460-660 GB/s)
    static const int comm_sms_env = [] {
        const char* e = std::getenv("XMOE_COMM_SMS");
        return e ? std::max(0, std::min(kNumSMs / 2, std::atoi(e))) : 28;
    }();
    // (C2, N=4, same box: 24 / 26 / 28 / 32 SMs -> 42.2 / 43.4 / 42.9-43.0 /
    // 42.1-42.4 M tokens/s; N=2: 21.9 / - / 21.9 / 21.5; 20 and 16 starve the
    // combines.  28 leaves headroom for N=8's larger off-rank share.)
    // RBD on the partition (XMOE_RBD_PARTITION=1, A/B): pack and combine as
    // whole-SM blocks.  Measured slower (C2 N=4, 2 chunks: 36.6 -> 33.5 M
    // tokens/s): the RBD combine's per-token group ordering needs more than
    // 24 SMs' issue rate.
    static const bool rbd_part = [] {
        const char* e = std::getenv("XMOE_RBD_PARTITION");
        return e && std::atoi(e) == 1;
    }();
    const int comm_sms = (L.pull || (rbd && rbd_part)) ? comm_sms_env : 0;
    const int gemm_sms = comm_sms > 0 ? kNumSMs - comm_sms : part_sms;
    // Late shared GEMM2 (XMOE_CHUNK_LATE=1, A/B; SM partition only): the head
    // runs shared GEMM1 alone, so the first routed chunk starts as soon as its
    // rows land; every chunk's combine writes fp32 routed sums and publishes
    // 128-token blocks; shared GEMM2 runs last, beside the final combine, its
    // epilogue adding the published sums (the combine's own arithmetic:
    // bit-identical output).  The combines keep their own SMs, so the
    // epilogue's wait cannot starve them.  Measured slower on B200 (C2, N=4:
    // 42.3 -> 40.7 M tok/s; N=2: 21.9 -> 17.9): the fp32 sums double the
    // combine's writes and the last combine runs on the partition's SMs.
    static const bool late_env = [] {
        const char* e = std::getenv("XMOE_CHUNK_LATE");
        return e && std::atoi(e) == 1;
    }();
    const bool late = late_env && comm_sms > 0 && L.Fs > 0 && L.workers[0].lpartial != nullptr;
    auto slot_A = [](int c) { return c; };
    auto slot_B = [](int c) { return kMaxChunks + c; };

    L.mark(kEvStart, st);
    for (int i = 0; i < nl; ++i)
        launch_forward_begin(L.workers[i].s_rows, static_cast<int>(S), i == 0 ? L.epoch : nullptr, st);
    for (int i = 0; i < nl; ++i) route_gate(L, L.workers[i], x_of(i), S, st);  // 1. gate (gating.cpp:14-57)
    L.mark(kEvGate, st);
    XMOE_CUDA(cudaEventRecord(L.ev_fork, st));
    XMOE_CUDA(cudaStreamWaitEvent(cm, L.ev_fork, 0));
    if (L.pull)  // stage the input where the owners can read it (peers finished reading the last one)
        for (int i = 0; i < nl; ++i)
            XMOE_CUDA(cudaMemcpyAsync(L.workers[i].xs, x_of(i), static_cast<size_t>(S) * rb, cudaMemcpyDeviceToDevice,
                                      cm));
    if (late)  // the previous forward's GEMM2 (earlier on st) has read them
        for (int i = 0; i < nl; ++i)
            XMOE_CUDA(cudaMemsetAsync(L.workers[i].lready, 0, sizeof(unsigned) * ((S + 127) / 128 + 1), cm));
    // 2. comm stream: PFT (pft.cpp:12-60), chunk counts, count all-gather,
    //    destinations, then every chunk's rows
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        route_pft(L, w, S, cm);
        launch_chunk_counts(w.token_ids, w.tpe, E, static_cast<int>(S), C, w.tpe_c, w.pfx_c, w.seg, cm);
        if (rbd) {  // groups, pilots (rbd.cpp:26-81), per (dest, chunk) counts
            launch_rbd_groups(w.slot_pos, w.expert_ids, static_cast<int>(S), k, El, w.rbd.state, L.jumps, w.rbd,
                              cm);
            launch_rbd_sort(W, nk, w.rbd, cm);
            launch_adjacent_diff(w.rbd.dptr, W, L.G_all + static_cast<size_t>(w.rank) * W, cm);
            launch_rbd_chunk_counts(W, static_cast<int>(S), w.rbd, cm);
        }
    }
    L.mark(kEvPft, cm);
    if (dist) exchange_counts(L, cm);
    L.mark(kEvCounts, cm);
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        launch_chunk_bases(L.tpe_c_all, W, C, E, w.rank, L.Rc, w.cbase, w.rpe_c, cm);
        launch_dispatch_dest_chunked(w.expert_ids, w.token_ids, w.B_dev, nk, static_cast<int>(S), C, E, El, w.seg,
                                     w.pfx_c, w.cbase, w.dest_rank, w.dest_row, cm, L.pull ? L.rsrc_tab : nullptr,
                                     w.rank);
        if (L.pull)
            launch_slot_addrs(w.slot_pos, nk, w.dest_rank, w.dest_row, w.cw, L.eout_tab, static_cast<int>(rb),
                              w.slot_src, w.slot_w, cm);
        if (rbd) launch_rbd_offsets(L.gd_all, W, w.rank, w.rbd, cm);
    }
    g_copy_smem = copy_smem;
    if (L.pull) {
        // every source's row table and staged input complete, then each
        // chunk region is pulled (chunk 0 on the full grid, later chunks on
        // XMOE_PULL_BLOCKS blocks beside the GEMMs)
        static const int blk_pull = [] {
            const char* e = std::getenv("XMOE_PULL_BLOCKS");
            return e ? std::max(1, std::atoi(e)) : kNumSMs;
        }();
        if (dist) {
            launch_flag_signal(L.flag_tab, W, me, slot_A(0), L.epoch, cm);
            launch_flag_wait(L.workers[0].flags, W, slot_A(0), L.epoch, L.peer_err_d, cm);
        }
        g_copy_fat = comm_sms;
        for (int c = 0; c < C; ++c) {
            g_copy_blocks = c == 0 ? 0 : blk_pull;
            for (int i = 0; i < nl; ++i) {
                Worker& w = L.workers[i];
                const size_t r0 = static_cast<size_t>(c) * L.Rc;
                launch_pull_rows(w.rsrc + r0, w.rpe_c + c * El, El, L.xs_tab, static_cast<int>(rb), L.Rc,
                                 static_cast<char*>(w.recv) + r0 * rb, cm);
            }
            if (L.timing) XMOE_CUDA(cudaEventRecord(L.tl[4 * c], cm));
            XMOE_CUDA(cudaEventRecord(L.evA[c], cm));
        }
        g_copy_fat = 0;
    }
    for (int c = 0; c < C && !L.pull; ++c) {
        // chunk 0 gates the first expert GEMM: full grid; later chunks run
        // beside the GEMMs on a bounded grid
        g_copy_blocks = c == 0 ? 0 : blk_scatter;
        const int t0 = t0_of(c), n = t0_of(c + 1) - t0;
        if (rbd) {  // each (token, dest) group's row once + a descriptor per copy
            g_copy_fat = comm_sms;
            for (int i = 0; i < nl; ++i) {
                Worker& w = L.workers[i];
                launch_rbd_pack(x_of(i), static_cast<int>(rb), w.rbd, W, c, nk, w.slot_pos, k, w.dest_row, w.cw,
                                L.recv_tab, L.desc_tab, cm, static_cast<int>(S), w.expert_ids, El);
            }
            g_copy_fat = 0;
        }
        else if (n > 0)
            for (int i = 0; i < nl; ++i) {
                Worker& w = L.workers[i];
                launch_scatter_tokens(x_of(i) + static_cast<size_t>(t0) * rb, static_cast<int>(rb), n, k,
                                      w.slot_pos + static_cast<size_t>(t0) * k, w.dest_rank, w.dest_row, w.cw,
                                      L.recv_tab, L.eout_tab, w.slot_src + static_cast<size_t>(t0) * k,
                                      w.slot_w + static_cast<size_t>(t0) * k, cm);
            }
        if (dist) launch_flag_signal(L.flag_tab, W, me, slot_A(c), L.epoch, cm);
        if (L.timing) XMOE_CUDA(cudaEventRecord(L.tl[4 * c], cm));
        XMOE_CUDA(cudaEventRecord(L.evA[c], cm));
    }
    g_copy_blocks = 0;
    L.mark(kEvMoved, cm);
    L.mark(kEvDispatch, cm);
    // 3. st: shared experts (x only), then the routed experts chunk by chunk
    //    (pf_pipeline.cpp:83-105)
    if (L.Fs > 0) {
        if (L.timing) XMOE_CUDA(cudaEventRecord(L.ev_side0, st));
        g_gemm_sm_limit = gemm_sms;
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_grouped_gemm_bf16(x_of(i), S, H, w.s_rows, 1, L.sw1, L.Fs, w.smid, 1, st);
            if (!late) launch_grouped_gemm_bf16(w.smid, S, L.Fs, w.s_rows, 1, L.sw2, H, w.sout, 0, st);
        }
        g_gemm_sm_limit = 0;
        if (L.timing) XMOE_CUDA(cudaEventRecord(L.ev_side1, st));
    }
    for (int c = 0; c < C; ++c) {
        XMOE_CUDA(cudaStreamWaitEvent(st, L.evA[c], 0));
        if (dist && !L.pull) launch_flag_wait(L.workers[0].flags, W, slot_A(c), L.epoch, L.peer_err_d, st);
        if (L.timing) XMOE_CUDA(cudaEventRecord(L.tl[4 * c + 1], st));
        const size_t r0 = static_cast<size_t>(c) * L.Rc;
        g_copy_blocks = 0;
        g_gemm_sm_limit = gemm_sms;
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            if (rbd)  // replicas read (gather) or copy the row from their pilot's slot
                launch_rbd_expand(static_cast<int>(rb), w.desc_recv, w.rbd, c, L.R_max, w.recv, L.recv_tab, w.gstart,
                                  st, L.rbd_gather ? w.a_idx : nullptr);
            if (rbd && L.rbd_gather)
                launch_grouped_gemm_bf16_gather(w.recv, L.R_max, L.Rc, H, w.rpe_c + c * El, El, w1_of(L, w.rank), F,
                                                static_cast<char*>(w.mid) + r0 * F * L.es, 1, w.a_idx + r0, st);
            else
                launch_grouped_gemm_bf16(static_cast<char*>(w.recv) + r0 * rb, L.Rc, H, w.rpe_c + c * El, El,
                                         w1_of(L, w.rank), F, static_cast<char*>(w.mid) + r0 * F * L.es, 1, st);
            launch_grouped_gemm_bf16(static_cast<char*>(w.mid) + r0 * F * L.es, L.Rc, F, w.rpe_c + c * El, El,
                                     w2_of(L, w.rank), H, static_cast<char*>(w.eout) + r0 * rb, 0, st);
            if (rbd)  // weighted sum of each group's outputs, pilot first (rbd.cpp:318-336)
                launch_rbd_merge(XMOE_BF16, L.eout_tab, H, w.desc_recv, w.gstart, w.rbd, c,
                                 static_cast<long long>(W) * S, w.back_u, st);
        }
        g_gemm_sm_limit = 0;
        if (L.timing) XMOE_CUDA(cudaEventRecord(L.tl[4 * c + 2], st));
        if (dist) launch_flag_signal(L.flag_tab, W, me, slot_B(c), L.epoch, st);
        XMOE_CUDA(cudaEventRecord(L.evB[c], st));
    }
    L.mark(kEvGemm, st);
    L.mark(kEvShared, st);
    // 4. comm: each chunk's weighted combine as soon as every owner finished
    //    it (pf_pipeline.cpp:107-135)
    for (int c = 0; c < C; ++c) {
        g_copy_blocks = c == C - 1 ? 0 : blk_combine;  // the last combine runs alone
        g_copy_fat = c == C - 1 && !late ? 0 : comm_sms;  // (late: beside shared GEMM2)
        XMOE_CUDA(cudaStreamWaitEvent(cm, L.evB[c], 0));
        if (dist) launch_flag_wait(L.workers[0].flags, W, slot_B(c), L.epoch, L.peer_err_d, cm);
        if (c == C - 1) L.mark(kEvReturn, cm);
        const int t0 = t0_of(c), n = t0_of(c + 1) - t0;
        if (n == 0) continue;
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            if (rbd) {  // one merged row per group, in pilot order (rbd.cpp:343-356)
                launch_rbd_combine(XMOE_BF16, L.back_tab, H, static_cast<int>(S), w.rbd, c, w.cw,
                                   L.Fs > 0 ? w.sout : nullptr, o_of(i), cm);
                continue;
            }
            if (late) {
                launch_combine_slots_seg_partial(w.slot_src + static_cast<size_t>(t0) * k,
                                                 w.slot_w + static_cast<size_t>(t0) * k, k, H, n,
                                                 w.lpartial + static_cast<size_t>(t0) * H, w.lready, t0, cm);
                continue;
            }
            launch_combine_slots(w.slot_src + static_cast<size_t>(t0) * k, w.slot_w + static_cast<size_t>(t0) * k,
                                 k, H, n, L.Fs > 0 ? static_cast<const char*>(w.sout) + t0 * rb : nullptr,
                                 o_of(i) + static_cast<size_t>(t0) * rb, cm);
        }
        if (L.timing) XMOE_CUDA(cudaEventRecord(L.tl[4 * c + 3], cm));
    }
    g_copy_blocks = 0;
    g_copy_smem = 0;
    g_copy_fat = 0;
    if (late) {
        // shared GEMM2 finishing every row from the published routed sums.
        // Enqueued after the combines it waits on: streams may share a
        // hardware queue, and a spinning GEMM ahead of them in it would
        // never let them start.
        g_gemm_sm_limit = gemm_sms;
        g_gemm_ready_mult = combine_segments(H);
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            g_gemm_addf = w.lpartial;
            g_gemm_ready = w.lready;
            launch_grouped_gemm_bf16(w.smid, S, L.Fs, w.s_rows, 1, L.sw2, H, o_of(i), 0, st);
        }
        g_gemm_addf = nullptr;
        g_gemm_ready = nullptr;
        g_gemm_ready_mult = 1;
        g_gemm_sm_limit = 0;
    }
    XMOE_CUDA(cudaEventRecord(L.ev_done, cm));
    XMOE_CUDA(cudaStreamWaitEvent(st, L.ev_done, 0));
    L.mark(kEvCombine, st);
    L.last_S = S;
    L.bwd_pending = true;
}

// ---------------------------------------------------------------- forward
// x/out: [nl, S, H] (nl = ranks this process drives).
void layer_forward(Layer& L, const void* x, long long S, void* out, cudaStream_t st) {
    L.check_peers();
    require(S >= 0 && S <= L.S_max, XMOE_ERR_VALIDATION, "sequence longer than the layer's max_tokens");
    L.last_ssmb = false;
    g_copy_blocks = 0;  // launch-shaping globals start clean even after an aborted forward
    g_copy_smem = 0;
    g_copy_fat = 0;
    g_gemm_sm_limit = 0;
    // A distributed layer takes the same path on every rank whatever its own
    // S: the chunked and unchunked forwards use different peer-flag slots, so
    // a rank with no tokens (S == 0) must still run the chunked protocol.
    if (L.nchunks > 1 && (S > 0 || L.distributed)) {
        L.last_Sw.assign(L.nl, S);
        layer_forward_chunked(L, x, S, out, st);
        return;
    }
    std::vector<long long> Sw(L.nl, S);
    layer_forward_v(L, x, Sw.data(), out, st);
}

// Per-worker token counts (rank == -1 contexts: the reference's MoeInstance
// allows a different S_w per worker, moe_instance.hpp:27): x/out are the
// workers' [S_w, H] blocks back to back.  Always the unchunked pipeline.
void layer_forward_v(Layer& L, const void* x, const long long* Sw, void* out, cudaStream_t st) {
    Ctx& ctx = *L.ctx;
    L.check_peers();
    long long Smax = 0;
    std::vector<long long> xoff(L.nl + 1, 0);
    for (int i = 0; i < L.nl; ++i) {
        require(Sw[i] >= 0 && Sw[i] <= L.S_max, XMOE_ERR_VALIDATION, "sequence longer than the layer's max_tokens");
        Smax = std::max(Smax, Sw[i]);
        xoff[i + 1] = xoff[i] + Sw[i];
    }
    L.last_ssmb = false;
    L.last_Sw.assign(Sw, Sw + L.nl);
    g_copy_blocks = 0;
    g_copy_smem = 0;
    g_gemm_sm_limit = 0;
    const int W = L.W, E = L.E, H = L.H, F = L.F, k = L.k;
    const int dt = L.d.dtype;
    const size_t row_bytes = static_cast<size_t>(H) * L.es;
    const int nl = L.nl;
    const bool dist = L.distributed;
    const bool tables = !dist || L.p2p;  // row movement by kernels over pointer tables
    const bool rbd = L.d.dispatch_mode == XMOE_DISPATCH_RBD;
    // bf16 rows: token-major permute (x read once) + slot-address combine
    const bool token_major = dt == XMOE_BF16 && (row_bytes & 15) == 0 && k <= 32;
    // One GPU, plain dispatch, shared experts: shared GEMM1 runs beside the
    // routing and the permute, shared GEMM2 beside the combine.  The combine
    // writes fp32 sums of the routed copies and publishes 128-token blocks;
    // GEMM2's epilogue adds them (out = bf16(sum + bf16(shared))) — the same
    // arithmetic as the combine's addend, so the output is unchanged bit for
    // bit — and the combine's HBM traffic hides under GEMM2's tensor work.
    const bool late_shared = late_shared_on() && L.partial && token_major && !rbd && !dist && nl == 1 &&
                             L.Fs > 0 && !L.timing && Sw[0] > 0 && H % 64 == 0 && gemm_2cta_enabled(H);
    const char* xb = static_cast<const char*>(x);
    char* ob = static_cast<char*>(out);
    auto x_of = [&](int i) { return xb + static_cast<size_t>(xoff[i]) * row_bytes; };
    auto o_of = [&](int i) { return ob + static_cast<size_t>(xoff[i]) * row_bytes; };

    L.mark(kEvStart, st);
    for (int i = 0; i < nl; ++i)  // one dense group of S rows; the forward's epoch
        launch_forward_begin(L.workers[i].s_rows, static_cast<int>(Sw[i]), i == 0 ? L.epoch : nullptr, st);
    const int me = L.workers[0].rank;
    auto fbar = [&](int j) {  // cross-rank barrier of the peer transport
        if (L.p2p) launch_flag_barrier(L.flag_tab, L.workers[0].flags, W, me, kSlotBar + j, L.epoch, L.peer_err_d, st);
        else L.barrier(st);
    };
    // 1. gate (gating.cpp:14-57)
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        const long long S = Sw[i];
        if (dt == XMOE_F64) {
            launch_gate_logits_f64(reinterpret_cast<const double*>(x_of(i)), static_cast<const double*>(L.gate),
                                   S, H, E, w.logits, st);
            launch_softmax_topk(w.logits, S, E, k, L.d.renorm, w.top, w.wts, st);
        } else if (dt == XMOE_F32) {
            float* lg = reinterpret_cast<float*>(w.logits);
            launch_gate_logits_f32(reinterpret_cast<const float*>(x_of(i)), static_cast<const float*>(L.gate), S, H, E,
                                   lg, st);
            launch_softmax_topk_f32(lg, S, E, k, L.d.renorm, w.top, w.wts, st);
        } else {
            route_gate(L, w, x_of(i), S, st);
        }
    }
    L.mark(kEvGate, st);
    // 1b. shared experts depend on x only: they run on a side stream, concurrent
    //     with PFT and the exchange, and join before the combine.  Forked after
    //     the gate so the two persistent GEMMs do not contend for SMs.  Timing
    //     mode issues them in line at the join instead, so that every stage
    //     (and "shared") is an isolated kernel time.
    auto issue_shared = [&](cudaStream_t ss) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            const long long S = Sw[i];
            run_gemm(dt, x_of(i), S, H, w.s_rows, 1, L.sw1, L.Fs, w.smid, 1, ss, w.smbits);
            run_gemm(dt, w.smid, S, L.Fs, w.s_rows, 1, L.sw2, H, w.sout, 0, ss);
        }
    };
    if (L.Fs > 0 && !L.timing) {
        XMOE_CUDA(cudaEventRecord(L.ev_fork, st));
        XMOE_CUDA(cudaStreamWaitEvent(L.side, L.ev_fork, 0));
        // leave SMs to the routing / exchange kernels running beside it
        // (multi-GPU by default: at N=1 there is no exchange to overlap;
        // XMOE_SHARED_SMS_N1 applies a limit at N=1 too, for A/B runs)
        static const int shared_sms = [] {
            const char* e = std::getenv("XMOE_SHARED_SMS");
            return e ? std::atoi(e) : 104;
        }();
        static const int shared_sms_n1 = [] {
            const char* e = std::getenv("XMOE_SHARED_SMS_N1");
            return e ? std::atoi(e) : 0;
        }();
        g_gemm_sm_limit = dist ? shared_sms : shared_sms_n1;
        if (late_shared) {  // GEMM1 now, GEMM2 after the routed GEMMs (below)
            Worker& w = L.workers[0];
            run_gemm(dt, x_of(0), Sw[0], H, w.s_rows, 1, L.sw1, L.Fs, w.smid, 1, L.side, w.smbits);
        } else {
            issue_shared(L.side);
            XMOE_CUDA(cudaEventRecord(L.ev_join, L.side));
        }
        g_gemm_sm_limit = 0;
    }
    // 2. padding-free token buffer (pft.cpp:12-60) [+ RBD groups and pilots, rbd.cpp:26-81]
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        const long long S = Sw[i], nk = S * k;
        if (dt == XMOE_BF16) route_pft(L, w, S, st);
        else launch_pft(w.top, w.wts, S, k, E, static_cast<int>(std::min<long long>(L.d.max_token_count, 0x7fffffff)),
                        w.token_ids, w.expert_ids, w.cw, w.tpe, w.slot_pos, w.B_dev, w.pft_ws, st);
        if (rbd) {
            launch_rbd_groups(w.slot_pos, w.expert_ids, static_cast<int>(S), k, L.El, w.rbd.state, L.jumps,
                              w.rbd, st);
            launch_rbd_sort(W, nk, w.rbd, st);
            launch_adjacent_diff(w.rbd.dptr, W, L.G_all + static_cast<size_t>(w.rank) * W, st);
            launch_rbd_chunk_counts(W, static_cast<int>(S), w.rbd, st);
        }
    }
    L.mark(kEvPft, st);
    // 3. per-expert (and per-destination group) counts to every rank
    //    (pf_pipeline.cpp:30-36).  Completing it also proves every peer is
    //    past its previous forward, so their buffers may be overwritten.
    if (dist && L.p2p) {
        exchange_counts(L, st);
    } else if (dist) {  // NCCL transport baseline
        Worker& w = L.workers[0];
        auto comm = static_cast<ncclComm_t>(ctx.nccl);
        XMOE_NCCL(ncclGroupStart());
        XMOE_NCCL(ncclAllGather(w.tpe, L.tpe_all, E, ncclInt32, comm, st));
        XMOE_NCCL(ncclGroupEnd());
    }
    // 4. dispatch: destination rows in the owner's (local expert, source,
    //    position) layout (pf_pipeline.cpp:47-73), then the rows themselves
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        launch_dispatch_dest(L.tpe_all, W, E, w.rank, w.expert_ids, w.B_dev, Sw[i] * k, w.dest_rank, w.dest_row, st);
        if (rbd) launch_rbd_offsets(L.gd_all, W, w.rank, w.rbd, st);
    }
    L.mark(kEvCounts, st);  // counts + destinations; rows_moved is the row kernel alone
    if (rbd) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_rbd_pack(x_of(i), static_cast<int>(row_bytes), w.rbd, W, 0, Sw[i] * k, w.slot_pos, k, w.dest_row,
                            w.cw, L.recv_tab, L.desc_tab, st, static_cast<int>(Sw[i]), w.expert_ids, L.El);
        }
        L.mark(kEvMoved, st);
        if (dist) fbar(0);
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_rbd_expand(static_cast<int>(row_bytes), w.desc_recv, w.rbd, 0, L.R_max, w.recv, L.recv_tab,
                              w.gstart, st, L.rbd_gather ? w.a_idx : nullptr);
        }
        if (dist && L.gpn > 1) fbar(1);  // stage-2 rows landed in peers' inputs
    } else if (tables) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            if (token_major)
                launch_scatter_tokens(x_of(i), static_cast<int>(row_bytes), static_cast<int>(Sw[i]), k, w.slot_pos,
                                      w.dest_rank, w.dest_row, w.cw, L.recv_tab, L.eout_tab, w.slot_src, w.slot_w, st);
            else
                launch_scatter_rows(x_of(i), static_cast<int>(row_bytes), w.token_ids, w.B_dev, Sw[i] * k, w.dest_rank,
                                    w.dest_row, L.recv_tab, st);
        }
        L.mark(kEvMoved, st);
        if (dist) fbar(0);
    } else {
        Worker& w = L.workers[0];
        launch_gather_rows(xb, Sw[0], static_cast<int>(row_bytes), w.token_ids, Sw[0] * k, w.B_dev, w.send, nullptr, st);
        L.h_tpe.resize(static_cast<size_t>(W) * E);
        XMOE_CUDA(cudaMemcpyAsync(L.h_tpe.data(), L.tpe_all, sizeof(int32_t) * W * E, cudaMemcpyDeviceToHost, st));
        XMOE_CUDA(cudaStreamSynchronize(st));
        L.exchange_nccl(/*forward=*/true, st);
        L.mark(kEvMoved, st);
    }
    L.mark(kEvDispatch, st);
    // 5. expert FFNs over each owner's contiguous segments (pf_pipeline.cpp:83-105)
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        launch_recv_counts(L.tpe_all, W, E, w.rank, w.rpe, st);
        if (rbd && L.rbd_gather)  // replica rows come straight from their pilot's row (TMA gather4)
            launch_grouped_gemm_bf16_gather(w.recv, L.R_max, L.R_max, H, w.rpe, L.El, w1_of(L, w.rank), F, w.mid, 1,
                                            w.a_idx, st);
        else
            run_gemm(dt, w.recv, L.R_max, H, w.rpe, L.El, w1_of(L, w.rank), F, w.mid, 1, st, w.mbits);
        run_gemm(dt, w.mid, L.R_max, F, w.rpe, L.El, w2_of(L, w.rank), H, w.eout, 0, st);
    }
    L.mark(kEvGemm, st);
    if (late_shared) {
        Worker& w = L.workers[0];
        // side: shared GEMM2 once the routed GEMMs are done (it must not hold
        // SMs while they still need them), its epilogue waiting per 128-row
        // block for the combine below; st: the combine into fp32 sums
        // the combine goes first: GEMM2's epilogue waits on its ready
        // counters, so GEMM2 must never occupy SMs the combine cannot share
        // (launched the other way round it deadlocked on B200: the combine's
        // CTAs were not co-scheduled beside the persistent GEMM CTAs)
        XMOE_CUDA(cudaMemsetAsync(L.ready, 0, sizeof(unsigned) * ((Sw[0] + 127) / 128 + 1), st));
        XMOE_CUDA(cudaEventRecord(L.ev_routed, st));  // routed GEMMs done, counters cleared
        L.mark(kEvShared, st);
        L.mark(kEvReturn, st);
        static const bool gemm_first = [] {  // A/B: enqueue GEMM2 before the combine
            const char* e = std::getenv("XMOE_LATE_ORDER");
            return e && std::atoi(e) == 2;
        }();
        if (!gemm_first)
            launch_combine_slots_partial(w.slot_src, w.slot_w, k, H, static_cast<int>(Sw[0]), L.partial, L.ready,
                                         st);
        XMOE_CUDA(cudaStreamWaitEvent(L.side, L.ev_routed, 0));
        // GEMM2 leaves SMs free (XMOE_LATE_GEMM_SMS, default 128 of 148) so
        // that combine CTAs always run; the combine takes tokens dynamically
        static const int late_sms = [] {
            const char* e = std::getenv("XMOE_LATE_GEMM_SMS");
            return e ? std::max(2, std::atoi(e)) : 128;
        }();
        g_gemm_addf = L.partial;
        g_gemm_ready = L.ready;
        g_gemm_sm_limit = late_sms;
        run_gemm(dt, w.smid, Sw[0], L.Fs, w.s_rows, 1, L.sw2, H, o_of(0), 0, L.side);
        g_gemm_sm_limit = 0;
        g_gemm_addf = nullptr;
        g_gemm_ready = nullptr;
        XMOE_CUDA(cudaEventRecord(L.ev_join, L.side));
        if (gemm_first)
            launch_combine_slots_partial(w.slot_src, w.slot_w, k, H, static_cast<int>(Sw[0]), L.partial, L.ready,
                                         st);
        XMOE_CUDA(cudaStreamWaitEvent(st, L.ev_join, 0));
        L.mark(kEvCombine, st);
        L.last_S = Sw[0];
        L.bwd_pending = true;
        return;
    }
    if (L.Fs > 0) {
        if (L.timing) {
            XMOE_CUDA(cudaEventRecord(L.ev_side0, st));
            issue_shared(st);
            XMOE_CUDA(cudaEventRecord(L.ev_side1, st));
        } else {
            XMOE_CUDA(cudaStreamWaitEvent(st, L.ev_join, 0));
        }
    }
    L.mark(kEvShared, st);
    // 6. return path + weighted combine (pf_pipeline.cpp:107-135, rbd.cpp:287-358)
    if (rbd) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            if (i == 0 && dist && L.gpn > 1) fbar(2);  // replicas' outputs are read from their owners
            launch_rbd_merge(dt, L.eout_tab, H, w.desc_recv, w.gstart, w.rbd, 0, static_cast<long long>(W) * Smax,
                             w.back_u, st);
        }
        if (dist) fbar(3);
        L.mark(kEvReturn, st);
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_rbd_combine(dt, L.back_tab, H, static_cast<int>(Sw[i]), w.rbd, 0, w.cw,
                               L.Fs > 0 ? w.sout : nullptr, o_of(i), st);
        }
    } else if (tables) {
        if (dist) fbar(3);
        L.mark(kEvReturn, st);
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            if (token_major)
                launch_combine_slots(w.slot_src, w.slot_w, k, H, static_cast<int>(Sw[i]), L.Fs > 0 ? w.sout : nullptr,
                                     o_of(i), st);
            else
                launch_combine(dt, nullptr, H, nullptr, w.slot_pos, k, w.cw, static_cast<int>(Sw[i]),
                               L.Fs > 0 ? w.sout : nullptr, o_of(i), st, L.eout_tab, w.dest_rank, w.dest_row);
        }
    } else {
        L.exchange_nccl(/*forward=*/false, st);
        L.mark(kEvReturn, st);
        Worker& w = L.workers[0];
        launch_combine(dt, w.back, H, nullptr, w.slot_pos, k, w.cw, static_cast<int>(Sw[0]),
                       L.Fs > 0 ? w.sout : nullptr, ob, st);
    }
    L.mark(kEvCombine, st);
    L.last_S = Sw[0];
    L.bwd_pending = true;
}

// NCCL alltoallv of rows (the library-collective baseline), chunked per
// (peer, local expert) so arrivals land directly in the (local expert,
// source, position) layout.  Forward: send -> recv; reverse (transposed
// counts): eout -> back.
void Layer::exchange_nccl(bool forward, cudaStream_t st) {
    Worker& w = workers[0];
    const int me = w.rank;
    const size_t rb = static_cast<size_t>(H) * es;
    auto comm = static_cast<ncclComm_t>(ctx->nccl);
    const ncclDataType_t ty = d.dtype == XMOE_F64 ? ncclFloat64 : d.dtype == XMOE_F32 ? ncclFloat32 : ncclBfloat16;
    std::vector<int64_t> send_off(E + 1), recv_off(static_cast<size_t>(W) * El);
    if (xmoe_plan_dispatch(W, E, h_tpe.data(), me, send_off.data(), recv_off.data(), nullptr) != XMOE_OK)
        fail(XMOE_ERR_VALIDATION, "num_experts must be divisible by the worker-group size");
    auto tpe = [&](int s, int e) { return static_cast<long long>(h_tpe[static_cast<size_t>(s) * E + e]); };
    XMOE_NCCL(ncclGroupStart());
    for (int peer = 0; peer < W; ++peer) {
        for (int le = 0; le < El; ++le) {  // my rows for the experts peer owns
            const int e = peer * El + le;
            const long long n = tpe(me, e);
            if (n == 0) continue;
            if (forward) XMOE_NCCL(ncclSend(static_cast<char*>(w.send) + send_off[e] * rb, n * H, ty, peer, comm, st));
            else XMOE_NCCL(ncclRecv(static_cast<char*>(w.back) + send_off[e] * rb, n * H, ty, peer, comm, st));
        }
        for (int le = 0; le < El; ++le) {  // peer's rows for my experts
            const long long n = tpe(peer, me * El + le);
            if (n == 0) continue;
            char* p = static_cast<char*>(forward ? w.recv : w.eout) + recv_off[static_cast<size_t>(peer) * El + le] * rb;
            if (forward) XMOE_NCCL(ncclRecv(p, n * H, ty, peer, comm, st));
            else XMOE_NCCL(ncclSend(p, n * H, ty, peer, comm, st));
        }
    }
    XMOE_NCCL(ncclGroupEnd());
}

// ---------------------------------------------------------------- backward
// Gradient of the last forward (bf16, pointer-table transports).  Per rank:
//   B1 dy rows to the owners (token-major, read once), each copy's weight and
//      home slot recorded at the owner
//   B2 dL/dw_c = <dy_t, y_c> to the home slot; dz = w_c dy_t — at the source
//      for copies this rank owns (fused into B1), at the owner for the rest
//   B3 dgrad: dH = (dz W2^T) * [mid > 0];  dxc = dH W1^T      (grouped-M)
//   B4 wgrad: dW1_e = x_e^T dH_e, dW2_e = a_e^T dz_e   (grouped-K, MN-major
//      operands read straight from the grouped buffers)
//   B5 shared experts (dense) and the gate: dl = softmax Jacobian of dL/dw,
//      dx_gate = dl Wg^T, dWg = x^T dl
//   B6 dx_t = sum of its copies' dxc rows (read from the owners) + shared
//      + gate parts
void layer_backward(Layer& L, const void* x, const void* dy, long long S, void* dx, cudaStream_t st) {
    require(L.train, XMOE_ERR_VALIDATION, "layer was not created with XMOE_LAYER_TRAIN");
    L.check_peers();
    require(S == L.last_S, XMOE_ERR_VALIDATION, "backward must follow a forward of the same sequence");
    // one backward per forward: the cross-rank barriers are keyed by the forward's epoch
    require(L.bwd_pending, XMOE_ERR_VALIDATION, "backward must follow a forward (one backward per forward)");
    L.bwd_pending = false;
    g_copy_blocks = 0;  // launch-shaping globals start clean even after an aborted call
    g_copy_fat = 0;
    g_gemm_sm_limit = 0;
    Ctx& ctx = *L.ctx;
    const int W = L.W, E = L.E, H = L.H, F = L.F, k = L.k, El = L.El;
    const size_t rb = static_cast<size_t>(H) * L.es;
    const bool dist = L.distributed;
    auto xo = [&](const void* b, int i) { return static_cast<const char*>(b) + static_cast<size_t>(i) * S * rb; };
    auto bmark = [&](int e) {
        if (L.timing) XMOE_CUDA(cudaEventRecord(L.bev[e], st));
    };
    bmark(kBwStart);
    // B5a token-level work that needs only x, dy and the forward's shared
    // activations (x transpose for the gate, shared-expert dgrad + wgrad):
    // on the side stream, overlapping the routed backward (own tail
    // scratch).  Timing mode runs it in line as the "token_level" stage.
    auto token_level = [&](cudaStream_t ss) {
        for (int i = 0; i < L.nl; ++i) {
            Worker& w = L.workers[i];
            if (L.Fs > 0) {
                launch_grouped_gemm_bf16_mask(xo(dy, i), S, H, w.s_rows, 1, L.sw2r, L.Fs, w.dHs, w.smbits, ss);
                launch_grouped_gemm_bf16(w.dHs, S, L.Fs, w.s_rows, 1, L.sw1r, H, w.dxs, 0, ss);
                launch_wgrad_mn_split(xo(x, i), H, w.dHs, L.Fs, S, L.splits_s1, w.split_s, w.tail_sa, w.tail_sb,
                                      w.part_s, L.dsw1, ss);
                launch_wgrad_mn_split(w.smid, L.Fs, xo(dy, i), H, S, L.splits_s2, w.split_s, w.tail_sa, w.tail_sb,
                                      w.part_s, L.dsw2, ss);
            }
        }
    };
    // NVLink row movement beside GEMMs on the other stream runs on a bounded
    // grid (as in the chunked forward): with every SM's worth of blocks its
    // remote traffic stalls the GEMM CTAs.  XMOE_BWD_COPY_BLOCKS (default
    // 128; 0 = full grid) applies when distributed, outside timing mode
    // (N=4 fwd+bwd, M tok/s: 32 blocks 9.9, 64 11.6, 128 11.9, full 11.8).
    static const int bwd_copy_blocks = [] {
        const char* e = std::getenv("XMOE_BWD_COPY_BLOCKS");
        return e ? std::max(0, std::atoi(e)) : 128;
    }();
    const int copy_cap = dist && !L.timing ? bwd_copy_blocks : 0;
    // SM partition (as the chunked forward's; XMOE_BWD_COMM_SMS=n, A/B, off
    // by default): the dy scatter and the dx combine run as whole-SM blocks
    // on n SMs, the GEMMs beside them on the rest.  Measured neutral to
    // slightly slower on B200 (C2 fwd+bwd, N=4: 12.93 M tokens/s off, 12.64
    // at 24 SMs, 12.99 at 32; N=2: 7.32 off, 7.07 at 24)
    static const int bwd_comm_env = [] {
        const char* e = std::getenv("XMOE_BWD_COMM_SMS");
        return e ? std::max(0, std::min(kNumSMs / 2, std::atoi(e))) : 0;
    }();
    const int bwd_comm = dist && !L.timing ? bwd_comm_env : 0;
    const int bwd_gemm_sms = bwd_comm > 0 ? kNumSMs - bwd_comm : 0;
    if (!L.timing) {
        XMOE_CUDA(cudaEventRecord(L.ev_fork, st));
        XMOE_CUDA(cudaStreamWaitEvent(L.side, L.ev_fork, 0));
        static const int side_sms = [] {
            const char* e = std::getenv("XMOE_BWD_SIDE_SMS");
            return e ? std::atoi(e) : 0;
        }();
        g_gemm_sm_limit = bwd_gemm_sms > 0 ? bwd_gemm_sms : side_sms;
        token_level(L.side);
        g_gemm_sm_limit = 0;
    }
    g_copy_blocks = copy_cap;
    g_copy_fat = bwd_comm;
    for (int i = 0; i < L.nl; ++i) {  // B1
        Worker& w = L.workers[i];
        launch_bwd_scatter_dy(xo(dy, i), H, static_cast<int>(S), k, w.slot_pos, w.dest_rank, w.dest_row, w.cw,
                              w.rank, w.dz, L.eout_tab, L.dyg_tab, L.dxc_tab, L.gw_tab, L.gsrc_tab, w.slot_dw,
                              w.bslot_src, st);
    }
    // cross-rank barriers: peer flags (a one-block kernel; an NCCL kernel
    // could not start while the side stream's persistent GEMMs hold every
    // SM's shared memory — it waited for them, 0.1 ms at N=4)
    const int me_rank = L.workers[0].rank;
    auto bbar = [&](int j) {
        launch_flag_barrier(L.flag_tab, L.workers[0].flags, W, me_rank, kSlotBwdBar + j, L.epoch, L.peer_err_d, st);
    };
    g_copy_fat = 0;
    if (dist) bbar(0);
    bmark(kBwScatter);
    for (int i = 0; i < L.nl; ++i) {  // B2-B3 at the owner
        Worker& w = L.workers[i];
        const size_t eo = dist ? 0 : static_cast<size_t>(w.rank) * El * H * F * L.es;
        g_copy_blocks = 0;  // local HBM work: full grid
        if (W > 1)  // copies from peers (this rank's own were finished at the source)
            launch_bwd_owner_prep(w.dyg, w.eout, w.gw, w.gsrc, w.rpe, El, H, L.R_max, L.slotdw_tab, w.dz, w.rank,
                                  st);
        bmark(kBwPrep);
        launch_grouped_gemm_bf16_mask(w.dz, L.R_max, H, w.rpe, El, static_cast<const char*>(L.w2r) + eo, F, w.dH,
                                      w.mbits, st);
        launch_grouped_gemm_bf16(w.dH, L.R_max, F, w.rpe, El, static_cast<const char*>(L.w1r) + eo, H, w.dxc, 0, st);
    }
    bmark(kBwDgrad);
    // B5 gate, B6 dx: need every owner's dxc rows and dL/dw home-slot writes
    // (barrier), not the weight gradients.  Outside timing mode the gate's
    // two small GEMMs run on the layer stream first (persistent GEMMs cannot
    // share SMs with the wgrad GEMMs, so on the side stream they would wait
    // for the wgrads to finish), then the dx combine — NVLink reads of every
    // copy's dxc row — runs on the side stream beside the wgrad GEMMs.
    auto gate_part = [&](cudaStream_t gs, bool with_wgrad) {
        for (int i = 0; i < L.nl; ++i) {
            Worker& w = L.workers[i];
            launch_gate_bwd(reinterpret_cast<const float*>(w.logits), w.slot_pos, w.expert_ids, w.slot_dw,
                            static_cast<int>(S), E, k, w.dl, gs);
            launch_grouped_gemm_bf16(w.dl, S, E, w.s_rows, 1, L.gater, H, w.dxg, 0, gs);
            if (with_wgrad)
                launch_wgrad_mn_split(xo(x, i), H, w.dl, E, S, L.splits_g, w.split_g, w.tail_ga, w.tail_gb,
                                      w.part_g, L.dgate, gs);
        }
    };
    auto gate_wgrad = [&](cudaStream_t gs) {
        for (int i = 0; i < L.nl; ++i) {
            Worker& w = L.workers[i];
            launch_wgrad_mn_split(xo(x, i), H, w.dl, E, S, L.splits_g, w.split_g, w.tail_ga, w.tail_gb, w.part_g,
                                  L.dgate, gs);
        }
    };
    auto dx_combine = [&](cudaStream_t gs) {
        for (int i = 0; i < L.nl; ++i) {
            Worker& w = L.workers[i];
            g_copy_blocks = copy_cap;
            g_copy_fat = bwd_comm;
            launch_combine_slots(w.bslot_src, nullptr, k, H, static_cast<int>(S), L.Fs > 0 ? w.dxs : nullptr,
                                 static_cast<char*>(dx) + static_cast<size_t>(i) * S * rb, gs, 0, w.dxg);
            g_copy_fat = 0;
            g_copy_blocks = 0;
        }
    };
    if (dist) bbar(1);  // every owner wrote dL/dw and dxc
    if (!L.timing) {
        gate_part(st, false);
        XMOE_CUDA(cudaEventRecord(L.ev_fork, st));
        XMOE_CUDA(cudaStreamWaitEvent(L.side, L.ev_fork, 0));  // side: token level, then the dx combine
        dx_combine(L.side);
        XMOE_CUDA(cudaEventRecord(L.ev_join, L.side));
        g_gemm_sm_limit = bwd_gemm_sms;  // beside the dx combine's SMs
        gate_wgrad(st);
    }
    g_gemm_sm_limit = bwd_gemm_sms;
    for (int i = 0; i < L.nl; ++i) {  // B4 wgrad straight on the grouped activations (MN-major operands)
        Worker& w = L.workers[i];
        const size_t go = dist ? 0 : static_cast<size_t>(w.rank) * El * H * F;
        launch_grouped_wgrad_mn(w.recv, H, w.dH, F, L.R_max, w.rpe, El, w.tail_a, w.tail_b, L.dw1 + go, st);
        // dW2_e [F, H] as (dz_e^T mid_e)^T: M = H fills whole 256-row tiles
        launch_grouped_wgrad_mn_t(w.dz, H, w.mid, F, L.R_max, w.rpe, El, w.tail_a, w.tail_b, L.dw2 + go, st);
    }
    g_gemm_sm_limit = 0;
    bmark(kBwWgrad);
    if (L.timing) {
        token_level(st);
        bmark(kBwToken);
        gate_part(st, true);
        dx_combine(st);
    } else {
        XMOE_CUDA(cudaStreamWaitEvent(st, L.ev_join, 0));  // dx, gate and shared-expert gradients
        bmark(kBwToken);
    }
    bmark(kBwEnd);
    (void)ctx;
    (void)W;
}

// ---------------------------------------------------------------- SSMB
// moesim::ssmb_forward (ssmb.cpp:12-46): contiguous shards, the last one
// takes the remainder; every rank routes its shard over the full (replicated)
// expert set; then the shards are all-gathered.  With one process per GPU
// the all-gather is a group of NCCL broadcasts (shards may differ in size).
void ssmb_forward(Ctx& ctx, Layer& L, const void* x_full, long long S, void* out_full, cudaStream_t st) {
    const int G = ctx.world;
    require(G >= 1, XMOE_ERR_VALIDATION, "ssmb_forward: shard count must be >= 1");
    require(G <= S, XMOE_ERR_VALIDATION, "ssmb_forward: more shards than sequence rows");
    const long long base = S / G;
    const size_t rb = static_cast<size_t>(L.H) * L.es;
    auto rows_of = [&](int g) { return g == G - 1 ? S - static_cast<long long>(g) * base : base; };
    const char* xb = static_cast<const char*>(x_full);
    char* ob = static_cast<char*>(out_full);
    if (!L.ssmb) {
        // Sequence shards over an EXPERT-PARALLEL layer (SSMB composed with
        // EP): shard g's tokens are rank g's tokens, experts
        // stay partitioned, and the exchange replaces the replicated weights.
        // Capacity applies per source rank as in pft_construct, so the drop
        // sets equal the reference's local-per-shard ones (§8(e)); every row's
        // arithmetic is row-independent, so the output equals the replicated
        // SSMB layer's bit for bit.
        require(L.W == G, XMOE_ERR_VALIDATION, "ssmb_forward: shard count must match the worker-group size");
        if (ctx.rank < 0 || G == 1) {  // shards are the workers' blocks, back to back
            std::vector<long long> Sw(G);
            for (int g = 0; g < G; ++g) Sw[g] = rows_of(g);
            layer_forward_v(L, x_full, Sw.data(), out_full, st);
            return;
        }
        const int me = ctx.rank;
        layer_forward(L, xb + me * base * rb, rows_of(me), ob + me * base * rb, st);
        auto comm = static_cast<ncclComm_t>(ctx.nccl);
        XMOE_NCCL(ncclGroupStart());
        for (int g = 0; g < G; ++g) {
            char* p = ob + g * base * rb;
            XMOE_NCCL(ncclBroadcast(p, p, rows_of(g) * rb, ncclUint8, g, comm, st));
        }
        XMOE_NCCL(ncclGroupEnd());
        return;
    }
    if (L.ssmb_cap < G) {  // kept copies per shard, for the ledger
        L.ssmb_B = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * G));
        L.ssmb_cap = G;
    }
    XMOE_CUDA(cudaMemsetAsync(L.ssmb_B, 0, sizeof(int32_t) * G, st));
    L.ssmb_rows.assign(G, 0);
    for (int g = 0; g < G; ++g) L.ssmb_rows[g] = rows_of(g);
    auto keep_count = [&](int g) {
        XMOE_CUDA(cudaMemcpyAsync(L.ssmb_B + g, L.workers[0].B_dev, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    };
    if (ctx.rank < 0 || G == 1) {
        for (int g = 0; g < G; ++g) {
            layer_forward(L, xb + g * base * rb, rows_of(g), ob + g * base * rb, st);
            keep_count(g);
        }
        L.last_ssmb = true;
        return;
    }
    const int me = ctx.rank;
    layer_forward(L, xb + me * base * rb, rows_of(me), ob + me * base * rb, st);
    keep_count(me);
    L.last_ssmb = true;
    auto comm = static_cast<ncclComm_t>(ctx.nccl);
    XMOE_NCCL(ncclGroupStart());
    for (int g = 0; g < G; ++g) {
        char* p = ob + g * base * rb;
        XMOE_NCCL(ncclBroadcast(p, p, rows_of(g) * rb, ncclUint8, g, comm, st));
    }
    XMOE_NCCL(ncclGroupEnd());
}

}  // namespace xmoe
