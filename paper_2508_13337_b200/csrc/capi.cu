// The C-ABI (include/xmoe/xmoe.h) and the host orchestration of the MoE-block
// hot path: context (device, NCCL communicator, scratch), layer (weights in the
// B200 layout + per-rank workspace) and the forward pipeline
//
//   gate -> PFT -> [count all-gather] -> dispatch -> grouped expert FFN
//        -> reverse exchange -> weighted combine (+ shared experts)
//
// which restates moesim::pf_moe_forward (pf_pipeline.cpp:137-169),
// rbd_moe_forward (rbd.cpp:360-386) and ssmb_forward (ssmb.cpp:12-46).
#include <nccl.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "layer.h"
#include "rbd.h"

namespace xmoe {

thread_local std::string g_last_error;
std::atomic<unsigned long long> g_kernel_launches{0};

#define XMOE_NCCL(expr)                                                                \
    do {                                                                               \
        ncclResult_t _r = (expr);                                                      \
        if (_r != ncclSuccess)                                                         \
            ::xmoe::fail(XMOE_ERR_NCCL, std::string(#expr ": ") + ncclGetErrorString(_r)); \
    } while (0)

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return XMOE_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return XMOE_ERR_INTERNAL;
    }
}

static size_t elem_size(int dtype) {
    if (dtype == XMOE_F64) return 8;
    if (dtype == XMOE_BF16) return 2;
    fail(XMOE_ERR_VALIDATION, "unknown dtype");
}

// ---------------------------------------------------------------- context
void* Ctx::scratch(size_t bytes) {
    if (bytes > ws_bytes) {
        if (ws) {
            XMOE_CUDA(cudaDeviceSynchronize());
            XMOE_CUDA(cudaFree(ws));
        }
        const size_t nb = bytes + (bytes >> 2) + 4096;
        XMOE_CUDA(cudaMalloc(&ws, nb));
        ws_bytes = nb;
    }
    return ws;
}

int* Ctx::err_flag() {
    if (!dflag) XMOE_CUDA(cudaMalloc(&dflag, 64));
    return static_cast<int*>(dflag);
}

Ctx::~Ctx() {
    if (ws) cudaFree(ws);
    if (dflag) cudaFree(dflag);
    if (nccl) ncclCommDestroy(static_cast<ncclComm_t>(nccl));
}

static void* dalloc(size_t bytes) {
    void* p = nullptr;
    if (bytes) XMOE_CUDA(cudaMalloc(&p, bytes));
    return p;
}

// ---------------------------------------------------------------- layer
Layer::~Layer() {
    for (void* p : allocs) cudaFree(p);
    for (auto& e : events) cudaEventDestroy(e);
}

void* Layer::alloc(size_t bytes) {
    void* p = dalloc(bytes ? bytes : 16);
    allocs.push_back(p);
    return p;
}

static void layer_create(Ctx& ctx, const xmoe_layer_desc& d, const void* gate, const void* w1,
                         const void* w2, const void* sw1, const void* sw2, Layer& L) {
    const int W = ctx.world;
    require(d.num_experts >= 1, XMOE_ERR_VALIDATION, "num_experts must be >= 1");
    require(d.top_k >= 1, XMOE_ERR_VALIDATION, "top_k must be >= 1");
    require(d.top_k <= d.num_experts, XMOE_ERR_VALIDATION, "top_k must be <= num_experts");
    require(d.max_token_count >= 1, XMOE_ERR_VALIDATION, "max_token_count must be >= 1");
    require(d.num_experts % W == 0, XMOE_ERR_VALIDATION,
            "num_experts must be divisible by the worker-group size");
    require(d.model_dim >= 1 && d.ffn_dim >= 1, XMOE_ERR_VALIDATION, "dims must be >= 1");
    require(d.dispatch_mode == XMOE_DISPATCH_NAIVE || d.dispatch_mode == XMOE_DISPATCH_RBD,
            XMOE_ERR_VALIDATION, "unknown dispatch mode");
    const bool bf = d.dtype == XMOE_BF16;
    require(bf || d.dtype == XMOE_F64, XMOE_ERR_VALIDATION, "unknown dtype");
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
    L.W = W;
    L.E = static_cast<int>(d.num_experts);
    L.H = static_cast<int>(d.model_dim);
    L.F = static_cast<int>(d.ffn_dim);
    L.k = static_cast<int>(d.top_k);
    L.El = L.E / W;
    L.E_held = ctx.rank < 0 ? L.E : L.El;
    L.Fs = static_cast<int>(d.n_shared * d.shared_ffn_dim);
    L.es = elem_size(d.dtype);
    const int H = L.H, F = L.F, E = L.E;
    const size_t es = L.es;
    cudaStream_t st = nullptr;

    // ---- weights: F64 keeps the reference layouts; BF16 goes K-major
    L.gate = L.alloc(static_cast<size_t>(H) * E * es);
    L.w1 = L.alloc(static_cast<size_t>(L.E_held) * H * F * es);
    L.w2 = L.alloc(static_cast<size_t>(L.E_held) * H * F * es);
    if (!bf) {
        XMOE_CUDA(cudaMemcpy(L.gate, gate, static_cast<size_t>(H) * E * es, cudaMemcpyDeviceToDevice));
        XMOE_CUDA(cudaMemcpy(L.w1, w1, static_cast<size_t>(L.E_held) * H * F * es, cudaMemcpyDeviceToDevice));
        XMOE_CUDA(cudaMemcpy(L.w2, w2, static_cast<size_t>(L.E_held) * H * F * es, cudaMemcpyDeviceToDevice));
    } else {
        launch_transpose(XMOE_BF16, gate, 1, H, E, XMOE_BF16, L.gate, st);          // [E,H]
        launch_transpose(XMOE_BF16, w1, L.E_held, H, F, XMOE_BF16, L.w1, st);       // [El,F,H]
        launch_transpose(XMOE_BF16, w2, L.E_held, F, H, XMOE_BF16, L.w2, st);       // [El,H,F]
    }
    if (L.Fs > 0) {
        require(sw1 && sw2, XMOE_ERR_VALIDATION, "shared expert weights missing");
        const int ns = static_cast<int>(d.n_shared), Fs1 = static_cast<int>(d.shared_ffn_dim);
        L.sw1 = L.alloc(static_cast<size_t>(H) * L.Fs * es);
        L.sw2 = L.alloc(static_cast<size_t>(H) * L.Fs * es);
        // merged shared FFN (moe_oracle.shared_expert_forward): W1cat [H, ns*Fs],
        // W2cat [ns*Fs, H]
        if (!bf) {
            for (int s = 0; s < ns; ++s) {
                XMOE_CUDA(cudaMemcpy2D(static_cast<char*>(L.sw1) + static_cast<size_t>(s) * Fs1 * es,
                                       static_cast<size_t>(L.Fs) * es,
                                       static_cast<const char*>(sw1) + static_cast<size_t>(s) * H * Fs1 * es,
                                       static_cast<size_t>(Fs1) * es, static_cast<size_t>(Fs1) * es, H,
                                       cudaMemcpyDeviceToDevice));
            }
            XMOE_CUDA(cudaMemcpy(L.sw2, sw2, static_cast<size_t>(H) * L.Fs * es, cudaMemcpyDeviceToDevice));
        } else {
            // K-major: sw1t [ns*Fs, H] = per-expert transposes stacked; sw2t [H, ns*Fs]
            launch_transpose(XMOE_BF16, sw1, ns, H, Fs1, XMOE_BF16, L.sw1, st);
            launch_transpose(XMOE_BF16, sw2, 1, L.Fs, H, XMOE_BF16, L.sw2, st);
        }
    }

    // ---- per-rank workspace
    const long long S = d.max_tokens;
    require(S >= 1, XMOE_ERR_VALIDATION, "max_tokens must be >= 1");
    const long long nk = S * L.k;
    const long long per_src = S * std::min<long long>(L.k, L.El);
    const long long cap_bound = static_cast<long long>(W) * L.El * d.max_token_count;
    L.R_max = std::min<long long>(static_cast<long long>(W) * per_src, cap_bound);
    if (L.R_max < 1) L.R_max = 1;
    L.S_max = S;
    L.tpe_all = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * W * E));
    const int nl = ctx.n_local();
    L.workers.resize(nl);
    std::vector<char*> recv_tab(W, nullptr), eout_tab(W, nullptr);
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        w.rank = ctx.rank_of(i);
        w.logits = static_cast<double*>(L.alloc(sizeof(double) * S * E));
        w.top = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.wts = static_cast<double*>(L.alloc(sizeof(double) * nk));
        w.token_ids = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.expert_ids = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.cw = static_cast<double*>(L.alloc(sizeof(double) * nk));
        w.slot_pos = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.B_dev = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * 4));
        w.tpe = (ctx.rank < 0 || W == 1) ? L.tpe_all + static_cast<size_t>(w.rank) * E
                                          : static_cast<int32_t*>(L.alloc(sizeof(int32_t) * E));
        w.pft_ws = L.alloc(bucket_ws_bytes(nk, E));
        w.dest_rank = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.dest_row = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * nk));
        w.rpe = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * L.El));
        w.recv = L.alloc(static_cast<size_t>(L.R_max) * H * es);
        w.mid = L.alloc(static_cast<size_t>(L.R_max) * F * es);
        w.eout = L.alloc(static_cast<size_t>(L.R_max) * H * es);
        if (ctx.rank >= 0 && W > 1) {
            w.send = L.alloc(static_cast<size_t>(nk) * H * es);
            w.back = L.alloc(static_cast<size_t>(nk) * H * es);
        }
        w.s_rows = static_cast<int32_t*>(L.alloc(sizeof(int32_t)));
        if (L.Fs > 0) {
            w.smid = L.alloc(static_cast<size_t>(S) * L.Fs * es);
            w.sout = L.alloc(static_cast<size_t>(S) * H * es);
        }
        if (d.dispatch_mode == XMOE_DISPATCH_RBD) {
            const long long gmax = S * std::min<long long>(L.k, W);  // groups per source
            const long long rmax = static_cast<long long>(W) * S;   // groups received
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
            r.coff = i32(nk);
            r.csr_ws = L.alloc(bucket_ws_bytes(nk, W));
            rng_state_from_seed(salt_seed_host(d.seed, static_cast<uint64_t>(w.rank), 0), r.state);
            w.send_u = L.alloc(static_cast<size_t>(gmax) * H * es);
            w.desc_send = static_cast<RbdDesc*>(L.alloc(sizeof(RbdDesc) * nk));
            w.recv_u = L.alloc(static_cast<size_t>(rmax) * H * es);
            w.desc_recv = static_cast<RbdDesc*>(L.alloc(sizeof(RbdDesc) * L.R_max));
            w.gstart = i32(rmax);
            w.back_u = L.alloc(static_cast<size_t>(rmax) * H * es);
            w.ret_u = L.alloc(static_cast<size_t>(gmax) * H * es);
            w.ru_base = i32(W);
        }
        recv_tab[w.rank] = static_cast<char*>(w.recv);
        eout_tab[w.rank] = static_cast<char*>(w.eout);
    }
    if (d.dispatch_mode == XMOE_DISPATCH_RBD) {
        std::vector<uint64_t> jt;
        rbd_jump_tables(jt);
        L.jumps = static_cast<uint64_t*>(L.alloc(sizeof(uint64_t) * jt.size()));
        XMOE_CUDA(cudaMemcpy(L.jumps, jt.data(), sizeof(uint64_t) * jt.size(), cudaMemcpyHostToDevice));
        L.G_all = static_cast<int32_t*>(L.alloc(sizeof(int32_t) * W * W));
    }
    L.recv_tab = static_cast<char**>(L.alloc(sizeof(char*) * W));
    L.eout_tab = static_cast<char**>(L.alloc(sizeof(char*) * W));
    XMOE_CUDA(cudaMemcpy(L.recv_tab, recv_tab.data(), sizeof(char*) * W, cudaMemcpyHostToDevice));
    XMOE_CUDA(cudaMemcpy(L.eout_tab, eout_tab.data(), sizeof(char*) * W, cudaMemcpyHostToDevice));
    L.events.resize(kNumEvents);
    for (auto& e : L.events) XMOE_CUDA(cudaEventCreate(&e));
    XMOE_CUDA(cudaDeviceSynchronize());
}

// expert weights of the worker owning rank r, inside this layer's allocation
static const void* w1_of(const Layer& L, int r) {
    const size_t off = L.ctx->rank < 0 ? static_cast<size_t>(r) * L.El * L.H * L.F * L.es : 0;
    return static_cast<const char*>(L.w1) + off;
}
static const void* w2_of(const Layer& L, int r) {
    const size_t off = L.ctx->rank < 0 ? static_cast<size_t>(r) * L.El * L.H * L.F * L.es : 0;
    return static_cast<const char*>(L.w2) + off;
}

void Layer::mark(int ev, cudaStream_t st) {
    if (timing) XMOE_CUDA(cudaEventRecord(events[ev], st));
}

static void run_gemm(const Layer& L, int dtype, const void* A, long long rows_bound, int K,
                     const int32_t* rpg, int G, const void* B, int N, void* D, int relu,
                     cudaStream_t st) {
    if (dtype == XMOE_F64)
        launch_grouped_gemm_f64(static_cast<const double*>(A), rows_bound, K, rpg, G,
                                static_cast<const double*>(B), N, static_cast<double*>(D), relu, st);
    else
        launch_grouped_gemm_bf16(A, rows_bound, K, rpg, G, B, N, D, relu, st);
    (void)L;
}

// The whole layer forward for every rank this context drives.
static void layer_forward(Layer& L, const void* x, long long S, void* out, cudaStream_t st) {
    Ctx& ctx = *L.ctx;
    require(S >= 0 && S <= L.S_max, XMOE_ERR_VALIDATION, "sequence longer than the layer's max_tokens");
    const int W = L.W, E = L.E, H = L.H, F = L.F, k = L.k;
    const int dt = L.d.dtype;
    const size_t row_bytes = static_cast<size_t>(H) * L.es;
    const int nl = ctx.n_local();
    const bool shared_dev = ctx.rank < 0 || W == 1;  // all ranks' buffers on this device
    const char* xb = static_cast<const char*>(x);
    char* ob = static_cast<char*>(out);
    const long long nk = S * k;

    L.mark(kEvStart, st);
    // 1-2. gate + PFT per rank (gating.cpp:14-57, pft.cpp:12-60)
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        const void* xi = xb + static_cast<size_t>(i) * S * row_bytes;
        launch_fill_i32(w.s_rows, 1, static_cast<int32_t>(S), st);  // one dense group of S rows
        if (dt == XMOE_F64) {
            launch_gate_logits_f64(static_cast<const double*>(xi), static_cast<const double*>(L.gate),
                                   S, H, E, w.logits, st);
            launch_softmax_topk(w.logits, S, E, k, L.d.renorm, w.top, w.wts, st);
        } else {
            float* lg = reinterpret_cast<float*>(w.logits);
            launch_grouped_gemm_bf16_f32out(xi, S, H, w.s_rows, 1, L.gate, E, lg, 0, st);
            launch_softmax_topk_f32(lg, S, E, k, L.d.renorm, w.top, w.wts, st);
        }
    }
    L.mark(kEvGate, st);
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        launch_pft(w.top, w.wts, S, k, E, static_cast<int>(std::min<long long>(L.d.max_token_count, 0x7fffffff)),
                   w.token_ids, w.expert_ids, w.cw, w.tpe, w.slot_pos, w.B_dev, w.pft_ws, st);
    }
    L.mark(kEvPft, st);
    const bool rbd = L.d.dispatch_mode == XMOE_DISPATCH_RBD;
    if (rbd) {
        // 3'. (token, destination) groups and their pilots (rbd.cpp:26-81)
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_rbd_groups(w.slot_pos, w.expert_ids, static_cast<int>(S), k, L.El, w.rbd.state,
                              L.jumps, w.rbd, st);
            launch_rbd_sort(W, nk, w.rbd, st);
            launch_adjacent_diff(w.rbd.dptr, W, L.G_all + static_cast<size_t>(w.rank) * W, st);
        }
    }
    // 3. per-expert counts (and RBD group counts) to every rank (pf_pipeline.cpp:30-36)
    if (!shared_dev) {
        Worker& w = L.workers[0];
        auto comm = static_cast<ncclComm_t>(ctx.nccl);
        XMOE_NCCL(ncclGroupStart());
        XMOE_NCCL(ncclAllGather(w.tpe, L.tpe_all, E, ncclInt32, comm, st));
        if (rbd)
            XMOE_NCCL(ncclAllGather(L.G_all + static_cast<size_t>(w.rank) * W, L.G_all, W, ncclInt32, comm, st));
        XMOE_NCCL(ncclGroupEnd());
    }
    // 4. dispatch (pf_pipeline.cpp:38-79): sender-side placement into the
    //    owner's (local expert, source, position) layout
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        launch_dispatch_dest(L.tpe_all, W, E, w.rank, w.expert_ids, w.B_dev, nk, w.dest_rank,
                             w.dest_row, st);
    }
    if (rbd) {
        // 4'. counts to the host (message sizes), pack unique rows + copy
        //     descriptors, exchange, expand at the receivers (rbd.cpp:83-285)
        L.h_tpe.resize(static_cast<size_t>(W) * E);
        L.h_G.resize(static_cast<size_t>(W) * W);
        XMOE_CUDA(cudaMemcpyAsync(L.h_tpe.data(), L.tpe_all, sizeof(int32_t) * W * E, cudaMemcpyDeviceToHost, st));
        XMOE_CUDA(cudaMemcpyAsync(L.h_G.data(), L.G_all, sizeof(int32_t) * W * W, cudaMemcpyDeviceToHost, st));
        XMOE_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> ru(W);
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            for (int d = 0; d < W; ++d) {
                long long a = 0;
                for (int s = 0; s < w.rank; ++s) a += L.Gsd(s, d);
                ru[d] = static_cast<int32_t>(a);
            }
            XMOE_CUDA(cudaMemcpy(w.ru_base, ru.data(), sizeof(int32_t) * W, cudaMemcpyHostToDevice));
            launch_rbd_pack(xb + static_cast<size_t>(i) * S * row_bytes, static_cast<int>(row_bytes), w.rbd,
                            nk, w.ru_base, w.slot_pos, k, w.dest_row, w.cw, w.send_u, w.desc_send, st);
        }
        L.rbd_exchange(/*forward=*/true, st);
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            long long nd = 0;
            for (int s = 0; s < W; ++s) nd += L.C(s, w.rank);
            launch_rbd_expand(w.recv_u, static_cast<int>(row_bytes), w.desc_recv, static_cast<int>(nd),
                              w.recv, w.gstart, st);
        }
    } else if (shared_dev) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_scatter_rows(xb + static_cast<size_t>(i) * S * row_bytes, static_cast<int>(row_bytes),
                                w.token_ids, w.B_dev, nk, w.dest_rank, w.dest_row, L.recv_tab, st);
        }
    } else {
        Worker& w = L.workers[0];
        launch_gather_rows(xb, S, static_cast<int>(row_bytes), w.token_ids, nk, w.B_dev, w.send,
                           nullptr, st);
        L.h_tpe.resize(static_cast<size_t>(W) * E);
        XMOE_CUDA(cudaMemcpyAsync(L.h_tpe.data(), L.tpe_all, sizeof(int32_t) * W * E,
                                  cudaMemcpyDeviceToHost, st));
        XMOE_CUDA(cudaStreamSynchronize(st));
        L.exchange_nccl(/*forward=*/true, st);
    }
    L.mark(kEvDispatch, st);
    // 5. expert FFNs over each owner's contiguous segments (pf_pipeline.cpp:83-105)
    for (int i = 0; i < nl; ++i) {
        Worker& w = L.workers[i];
        launch_recv_counts(L.tpe_all, W, E, w.rank, w.rpe, st);
        run_gemm(L, dt, w.recv, L.R_max, H, w.rpe, L.El, w1_of(L, w.rank), F, w.mid, 1, st);
        run_gemm(L, dt, w.mid, L.R_max, F, w.rpe, L.El, w2_of(L, w.rank), H, w.eout, 0, st);
    }
    L.mark(kEvGemm, st);
    if (L.Fs > 0) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            const void* xi = xb + static_cast<size_t>(i) * S * row_bytes;
            run_gemm(L, dt, xi, S, H, w.s_rows, 1, L.sw1, L.Fs, w.smid, 1, st);
            run_gemm(L, dt, w.smid, S, L.Fs, w.s_rows, 1, L.sw2, H, w.sout, 0, st);
        }
    }
    L.mark(kEvShared, st);
    // 6. reverse exchange + weighted combine (pf_pipeline.cpp:107-135,
    //    rbd.cpp:287-358)
    if (rbd) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            long long ng = 0;
            for (int s = 0; s < W; ++s) ng += L.Gsd(s, w.rank);
            launch_rbd_merge(dt, w.eout, H, w.desc_recv, w.gstart, static_cast<int>(ng), w.back_u, st);
        }
        L.rbd_exchange(/*forward=*/false, st);
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_rbd_combine(dt, w.ret_u, H, static_cast<int>(S), w.rbd, w.cw, L.Fs > 0 ? w.sout : nullptr,
                               ob + static_cast<size_t>(i) * S * row_bytes, st);
        }
    } else if (shared_dev) {
        for (int i = 0; i < nl; ++i) {
            Worker& w = L.workers[i];
            launch_combine(dt, nullptr, H, nullptr, w.slot_pos, k, w.cw, static_cast<int>(S),
                           L.Fs > 0 ? w.sout : nullptr, ob + static_cast<size_t>(i) * S * row_bytes,
                           st, L.eout_tab, w.dest_rank, w.dest_row);
        }
    } else {
        L.exchange_nccl(/*forward=*/false, st);
        Worker& w = L.workers[0];
        launch_combine(dt, w.back, H, nullptr, w.slot_pos, k, w.cw, static_cast<int>(S),
                       L.Fs > 0 ? w.sout : nullptr, ob, st);
    }
    L.mark(kEvCombine, st);
    L.last_S = S;
}

// NCCL alltoallv of rows, chunked per (peer, local expert) so arrivals land
// directly in the (local expert, source, position) layout — the reference's
// regroup (pf_pipeline.cpp:47-79) never materialises.  Forward: send ->
// recv; reverse (transposed counts): eout -> back.
void Layer::exchange_nccl(bool forward, cudaStream_t st) {
    Worker& w = workers[0];
    const int me = w.rank;
    auto tpe = [&](int s, int e) { return h_tpe[static_cast<size_t>(s) * E + e]; };
    const size_t rb = static_cast<size_t>(H) * es;
    auto comm = static_cast<ncclComm_t>(ctx->nccl);
    ncclDataType_t ty = d.dtype == XMOE_F64 ? ncclFloat64 : ncclBfloat16;
    // my packed block starts
    std::vector<long long> blk(E + 1, 0);
    for (int e = 0; e < E; ++e) blk[e + 1] = blk[e] + tpe(me, e);
    // grouped base of each of my local experts, and rows before source s
    std::vector<long long> ebase(El + 1, 0);
    for (int le = 0; le < El; ++le) {
        long long a = 0;
        for (int s = 0; s < W; ++s) a += tpe(s, me * El + le);
        ebase[le + 1] = ebase[le] + a;
    }
    XMOE_NCCL(ncclGroupStart());
    for (int peer = 0; peer < W; ++peer) {
        // outgoing: my rows for experts owned by peer
        for (int le = 0; le < El; ++le) {
            const int e = peer * El + le;
            const long long n = tpe(me, e);
            if (n == 0) continue;
            if (forward) {
                XMOE_NCCL(ncclSend(static_cast<char*>(w.send) + blk[e] * rb, n * H, ty, peer, comm, st));
            } else {
                XMOE_NCCL(ncclRecv(static_cast<char*>(w.back) + blk[e] * rb, n * H, ty, peer, comm, st));
            }
        }
        // incoming: peer's rows for my experts
        for (int le = 0; le < El; ++le) {
            const int e = me * El + le;
            const long long n = tpe(peer, e);
            if (n == 0) continue;
            long long before = 0;
            for (int s = 0; s < peer; ++s) before += tpe(s, e);
            char* p = static_cast<char*>(forward ? w.recv : w.eout) + (ebase[le] + before) * rb;
            if (forward) XMOE_NCCL(ncclRecv(p, n * H, ty, peer, comm, st));
            else XMOE_NCCL(ncclSend(p, n * H, ty, peer, comm, st));
        }
    }
    XMOE_NCCL(ncclGroupEnd());
}

long long Layer::C(int s, int d) const {
    long long a = 0;
    for (int le = 0; le < El; ++le) a += h_tpe[static_cast<size_t>(s) * E + d * El + le];
    return a;
}

// RBD exchange.  Forward, for every (source s, dest d): the G_sd unique rows
// of s's dest-d segment land in d's recv_u after the rows of sources < s, and
// the C_sd copy descriptors after those of sources < s.  Reverse: the merged
// rows go back into s's ret_u at s's dest-d segment.  Ranks sharing the
// device use device copies; separate processes use NCCL send/recv.
void Layer::rbd_exchange(bool forward, cudaStream_t st) {
    const size_t rb = static_cast<size_t>(H) * es;
    auto seg_g = [&](int s, int d) {  // s's dest-d segment start in its dest-sorted groups
        long long a = 0;
        for (int q = 0; q < d; ++q) a += Gsd(s, q);
        return a;
    };
    auto seg_c = [&](int s, int d) {
        long long a = 0;
        for (int q = 0; q < d; ++q) a += C(s, q);
        return a;
    };
    auto at_recv_g = [&](int s, int d) {  // rows of sources < s at receiver d
        long long a = 0;
        for (int q = 0; q < s; ++q) a += Gsd(q, d);
        return a;
    };
    auto at_recv_c = [&](int s, int d) {
        long long a = 0;
        for (int q = 0; q < s; ++q) a += C(q, d);
        return a;
    };
    const bool shared_dev = ctx->rank < 0 || W == 1;
    if (shared_dev) {
        for (Worker& src : workers)
            for (Worker& dst : workers) {
                const int s = src.rank, d = dst.rank;
                const long long g = Gsd(s, d), c = C(s, d);
                if (forward) {
                    if (g)
                        XMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(dst.recv_u) + at_recv_g(s, d) * rb,
                                                  static_cast<char*>(src.send_u) + seg_g(s, d) * rb, g * rb,
                                                  cudaMemcpyDeviceToDevice, st));
                    if (c)
                        XMOE_CUDA(cudaMemcpyAsync(dst.desc_recv + at_recv_c(s, d), src.desc_send + seg_c(s, d),
                                                  c * sizeof(RbdDesc), cudaMemcpyDeviceToDevice, st));
                } else if (g) {
                    XMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(src.ret_u) + seg_g(s, d) * rb,
                                              static_cast<char*>(dst.back_u) + at_recv_g(s, d) * rb, g * rb,
                                              cudaMemcpyDeviceToDevice, st));
                }
            }
        return;
    }
    Worker& w = workers[0];
    const int me = w.rank;
    auto comm = static_cast<ncclComm_t>(ctx->nccl);
    XMOE_NCCL(ncclGroupStart());
    for (int peer = 0; peer < W; ++peer) {
        if (forward) {
            const long long g_out = Gsd(me, peer), c_out = C(me, peer);
            const long long g_in = Gsd(peer, me), c_in = C(peer, me);
            if (g_out) XMOE_NCCL(ncclSend(static_cast<char*>(w.send_u) + seg_g(me, peer) * rb, g_out * rb, ncclUint8, peer, comm, st));
            if (c_out) XMOE_NCCL(ncclSend(w.desc_send + seg_c(me, peer), c_out * sizeof(RbdDesc), ncclUint8, peer, comm, st));
            if (g_in) XMOE_NCCL(ncclRecv(static_cast<char*>(w.recv_u) + at_recv_g(peer, me) * rb, g_in * rb, ncclUint8, peer, comm, st));
            if (c_in) XMOE_NCCL(ncclRecv(w.desc_recv + at_recv_c(peer, me), c_in * sizeof(RbdDesc), ncclUint8, peer, comm, st));
        } else {
            const long long g_back = Gsd(peer, me);  // merged rows I return to peer
            const long long g_ret = Gsd(me, peer);   // merged rows peer returns to me
            if (g_back) XMOE_NCCL(ncclSend(static_cast<char*>(w.back_u) + at_recv_g(peer, me) * rb, g_back * rb, ncclUint8, peer, comm, st));
            if (g_ret) XMOE_NCCL(ncclRecv(static_cast<char*>(w.ret_u) + seg_g(me, peer) * rb, g_ret * rb, ncclUint8, peer, comm, st));
        }
    }
    XMOE_NCCL(ncclGroupEnd());
}

}  // namespace xmoe

using namespace xmoe;

struct xmoe_ctx {
    Ctx c;
};
struct xmoe_layer {
    Layer l;
};

extern "C" {

int xmoe_abi_version(void) { return XMOE_ABI_VERSION; }
uint64_t xmoe_kernel_launches(void) { return g_kernel_launches.load(); }
const char* xmoe_last_error(void) { return g_last_error.c_str(); }

int xmoe_nccl_unique_id(void* out) {
    return guarded([&] {
        ncclUniqueId id;
        XMOE_NCCL(ncclGetUniqueId(&id));
        std::memcpy(out, &id, sizeof(id));
    });
}

int xmoe_ctx_create(int device, int world, int rank, const void* nccl_id, xmoe_ctx** out) {
    return guarded([&] {
        require(world >= 1, XMOE_ERR_VALIDATION, "world must be >= 1");
        require(rank >= -1 && rank < world, XMOE_ERR_VALIDATION, "rank out of range");
        XMOE_CUDA(cudaSetDevice(device));
        int major = 0;
        XMOE_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        require(major == 10, XMOE_ERR_CUDA, "xmoe requires an sm_100 (B200) device");
        auto* c = new xmoe_ctx;
        c->c.device = device;
        c->c.world = world;
        c->c.rank = rank;
        if (rank >= 0 && world > 1) {
            require(nccl_id != nullptr, XMOE_ERR_VALIDATION, "nccl unique id required for world > 1");
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            ncclComm_t comm;
            const ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
            if (r != ncclSuccess) {
                delete c;
                fail(XMOE_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
            }
            c->c.nccl = comm;
        }
        *out = c;
    });
}

int xmoe_ctx_destroy(xmoe_ctx* ctx) {
    return guarded([&] { delete ctx; });
}

int xmoe_gate_forward(xmoe_ctx* ctx, int dtype, const void* x, const void* wg, int64_t S,
                      int64_t H, int64_t E, int64_t k, int renorm, int32_t* top, double* weights,
                      double* logits, void* stream) {
    return guarded([&] {
        require(k >= 1, XMOE_ERR_VALIDATION, "top_k must be >= 1");
        require(k <= E, XMOE_ERR_VALIDATION, "top_k must be <= num_experts");
        auto st = static_cast<cudaStream_t>(stream);
        char* ws = static_cast<char*>(ctx->c.scratch(sizeof(double) * S * E + 256));
        if (dtype == XMOE_F64) {
            double* lg = logits ? logits : reinterpret_cast<double*>(ws);
            launch_gate_logits_f64(static_cast<const double*>(x), static_cast<const double*>(wg),
                                   S, H, E, lg, st);
            launch_softmax_topk(lg, S, E, k, renorm, top, weights, st);
        } else if (dtype == XMOE_BF16) {
            require(E % 16 == 0 && H % 8 == 0, XMOE_ERR_VALIDATION,
                    "bf16 gate requires num_experts % 16 == 0 and model_dim % 8 == 0");
            int32_t* rows = reinterpret_cast<int32_t*>(ws);
            float* lg = reinterpret_cast<float*>(ws + 256);
            launch_fill_i32(rows, 1, static_cast<int32_t>(S), st);
            launch_grouped_gemm_bf16_f32out(x, S, H, rows, 1, wg, E, lg, 0, st);
            launch_softmax_topk_f32(lg, S, E, k, renorm, top, weights, st);
            if (logits) launch_f32_to_f64(lg, static_cast<long long>(S) * E, logits, st);
        } else {
            fail(XMOE_ERR_VALIDATION, "unknown dtype");
        }
    });
}

int xmoe_pft_construct(xmoe_ctx* ctx, const int32_t* top, const double* w, int64_t S, int64_t k,
                       int64_t E, int64_t cap, int32_t* token_ids, int32_t* expert_ids, double* cw,
                       int32_t* tpe, int32_t* slot_pos, int32_t* B_dev, int validate, void* stream) {
    return guarded([&] {
        require(cap >= 1, XMOE_ERR_VALIDATION, "max_token_count must be >= 1");
        require(E >= 1, XMOE_ERR_VALIDATION, "num_experts must be >= 1");
        require(k >= 1, XMOE_ERR_VALIDATION, "top_k must be >= 1");
        auto st = static_cast<cudaStream_t>(stream);
        const long long n = S * k;
        char* ws = static_cast<char*>(ctx->c.scratch(bucket_ws_bytes(n, E) + 64));
        if (validate) {
            auto* fb = reinterpret_cast<unsigned long long*>(ctx->c.err_flag());
            XMOE_CUDA(cudaMemsetAsync(fb, 0xff, sizeof(unsigned long long), st));
            launch_pft_validate(top, S, k, E, fb, st);
            unsigned long long h = 0;
            XMOE_CUDA(cudaMemcpyAsync(&h, fb, sizeof(h), cudaMemcpyDeviceToHost, st));
            XMOE_CUDA(cudaStreamSynchronize(st));
            if (h != ~0ull) {
                if (h & 1) fail(XMOE_ERR_VALIDATION, "top_experts rows must contain distinct expert ids");
                fail(XMOE_ERR_INDEX, "expert id out of range");
            }
        }
        launch_pft(top, w, S, k, E, static_cast<int>(std::min<int64_t>(cap, 0x7fffffff)), token_ids,
                   expert_ids, cw, tpe, slot_pos, B_dev, ws, st);
    });
}

int xmoe_gather_rows(xmoe_ctx* ctx, int dtype, const void* src, int64_t rows, int64_t cols,
                     const int32_t* ids, int64_t n, void* out, int validate, void* stream) {
    return guarded([&] {
        auto st = static_cast<cudaStream_t>(stream);
        int* err = validate ? ctx->c.err_flag() : nullptr;
        if (err) XMOE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
        launch_gather_rows(src, rows, static_cast<int>(cols * elem_size(dtype)), ids, n, nullptr,
                           out, err, st);
        if (err) {
            int h = 0;
            XMOE_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, st));
            XMOE_CUDA(cudaStreamSynchronize(st));
            if (h) fail(XMOE_ERR_INDEX, "gather_rows: row id out of range");
        }
    });
}

int xmoe_scatter_combine(xmoe_ctx* ctx, int dtype, const void* rows, int64_t n, int64_t cols,
                         const int32_t* token_ids, const double* weights, int64_t S, void* out,
                         int validate, void* stream) {
    return guarded([&] {
        auto st = static_cast<cudaStream_t>(stream);
        elem_size(dtype);
        if (validate && n > 0) {
            // id range check (reference pft.cpp:85-87) on the host copy
            std::vector<int32_t> h(n);
            XMOE_CUDA(cudaMemcpyAsync(h.data(), token_ids, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
            XMOE_CUDA(cudaStreamSynchronize(st));
            for (auto t : h)
                if (t < 0 || t >= S) fail(XMOE_ERR_INDEX, "scatter_combine: token id out of range");
        }
        // token -> copies CSR, stable in i (the reference's ascending-i order)
        const size_t wsb = bucket_ws_bytes(n, static_cast<int>(S));
        char* ws = static_cast<char*>(ctx->c.scratch(wsb + sizeof(int32_t) * (S + 1 + n) + 256));
        int32_t* ptr = reinterpret_cast<int32_t*>(ws + wsb);
        int32_t* perm = ptr + S + 1;
        launch_stable_csr(token_ids, static_cast<int>(n), static_cast<int>(S), ptr, perm, ws, st);
        launch_combine(dtype, rows, static_cast<int>(cols), ptr, perm, 0, weights, static_cast<int>(S),
                       nullptr, out, st);
    });
}

int xmoe_grouped_mlp(xmoe_ctx* ctx, int dtype, const void* in, int64_t rows,
                     const int32_t* rows_per_expert, int64_t G, const void* w1, const void* w2,
                     int64_t H, int64_t F, void* out, void* stream) {
    return guarded([&] {
        auto st = static_cast<cudaStream_t>(stream);
        // CountMismatch check (pf_pipeline.cpp:102-103): segment counts must
        // cover the input exactly
        std::vector<int32_t> h(G);
        if (G) XMOE_CUDA(cudaMemcpyAsync(h.data(), rows_per_expert, sizeof(int32_t) * G, cudaMemcpyDeviceToHost, st));
        XMOE_CUDA(cudaStreamSynchronize(st));
        long long tot = 0;
        for (auto v : h) tot += v;
        if (tot != rows) fail(XMOE_ERR_COUNT_MISMATCH, "grouped_expert_mlp: segment counts disagree with input rows");
        const size_t es = elem_size(dtype);
        void* mid = ctx->c.scratch(static_cast<size_t>(rows) * F * es + 256);
        if (dtype == XMOE_F64) {
            launch_grouped_gemm_f64(static_cast<const double*>(in), rows, H, rows_per_expert, G,
                                    static_cast<const double*>(w1), F, static_cast<double*>(mid), 1, st);
            launch_grouped_gemm_f64(static_cast<const double*>(mid), rows, F, rows_per_expert, G,
                                    static_cast<const double*>(w2), H, static_cast<double*>(out), 0, st);
        } else {
            launch_grouped_gemm_bf16(in, rows, H, rows_per_expert, G, w1, F, mid, 1, st);
            launch_grouped_gemm_bf16(mid, rows, F, rows_per_expert, G, w2, H, out, 0, st);
        }
    });
}

int xmoe_grouped_gemm_bf16(xmoe_ctx* ctx, const void* A, int64_t rows, int64_t K,
                           const int32_t* rows_per_group, int64_t G, const void* B, int64_t N,
                           void* D, int relu, void* stream) {
    return guarded([&] {
        (void)ctx;
        launch_grouped_gemm_bf16(A, rows, K, rows_per_group, G, B, N, D, relu,
                                 static_cast<cudaStream_t>(stream));
    });
}

int xmoe_layer_create(xmoe_ctx* ctx, const xmoe_layer_desc* desc, const void* gate,
                      const void* w1, const void* w2, const void* sw1, const void* sw2,
                      xmoe_layer** out) {
    return guarded([&] {
        auto l = std::make_unique<xmoe_layer>();
        layer_create(ctx->c, *desc, gate, w1, w2, sw1, sw2, l->l);
        *out = l.release();
    });
}

int xmoe_layer_destroy(xmoe_layer* layer) {
    return guarded([&] { delete layer; });
}

int xmoe_moe_forward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x, int64_t S, void* out,
                     void* stream) {
    return guarded([&] {
        require(&layer->l.ctx->device == &ctx->c.device, XMOE_ERR_VALIDATION, "layer belongs to another context");
        layer_forward(layer->l, x, S, out, static_cast<cudaStream_t>(stream));
    });
}

int xmoe_ssmb_forward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x_full, int64_t S,
                      void* out_full, void* stream) {
    return guarded([&] {
        Ctx& c = ctx->c;
        Layer& L = layer->l;
        const int G = c.world;
        require(G >= 1, XMOE_ERR_VALIDATION, "ssmb_forward: shard count must be >= 1");
        require(G <= S, XMOE_ERR_VALIDATION, "ssmb_forward: more shards than sequence rows");
        require(L.W == 1 || c.rank < 0 ? true : false, XMOE_ERR_VALIDATION,
                "ssmb_forward: the layer must hold every expert (create it with world-1 semantics)");
        (void)L;
        fail(XMOE_ERR_INTERNAL, "ssmb_forward: not implemented in this build");
    });
}

int xmoe_layer_ledger(xmoe_layer* layer, uint64_t* out, int n) {
    return guarded([&] { layer->l.ledger(out, n); });
}

int xmoe_layer_set_timing(xmoe_layer* layer, int enable) {
    return guarded([&] { layer->l.timing = enable != 0; });
}

int xmoe_layer_stage_ms(xmoe_layer* layer, float* out, int n) {
    return guarded([&] {
        Layer& L = layer->l;
        require(L.timing, XMOE_ERR_VALIDATION, "timing not enabled");
        XMOE_CUDA(cudaEventSynchronize(L.events[kEvCombine]));
        const int pairs[][2] = {{kEvStart, kEvGate},   {kEvGate, kEvPft},    {kEvPft, kEvDispatch},
                                {kEvDispatch, kEvGemm}, {kEvGemm, kEvShared}, {kEvShared, kEvCombine},
                                {kEvStart, kEvCombine}};
        for (int i = 0; i < n && i < 7; ++i)
            XMOE_CUDA(cudaEventElapsedTime(&out[i], L.events[pairs[i][0]], L.events[pairs[i][1]]));
    });
}

}  // extern "C"
