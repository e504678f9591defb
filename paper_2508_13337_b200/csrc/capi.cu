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

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.cuh"
#include "layer.h"
#include "rbd.h"

namespace xmoe {

thread_local std::string g_last_error;
std::atomic<unsigned long long> g_kernel_launches{0};

bool sync_check_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("XMOE_SYNC_CHECK");
        return e && std::atoi(e) == 1;
    }();
    return on;
}

void sync_check(const char* file, int line) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(cudaStreamLegacy, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return;
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess)
        fail(XMOE_ERR_CUDA, std::string("kernel launched at ") + file + ":" + std::to_string(line) + ": " +
                                cudaGetErrorString(e));
}

#define XMOE_NCCL(expr)                                                                \
    do {                                                                               \
        ncclResult_t _r = (expr);                                                      \
        if (_r != ncclSuccess)                                                         \
            ::xmoe::fail(XMOE_ERR_NCCL, std::string(#expr ": ") + ncclGetErrorString(_r)); \
    } while (0)


static size_t elem_size(int dtype) {
    if (dtype == XMOE_F64) return 8;
    if (dtype == XMOE_F32) return 4;
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
    if (async_err_h) cudaFreeHost(async_err_h);
    if (nccl) ncclCommDestroy(static_cast<ncclComm_t>(nccl));
}

}  // namespace xmoe

using namespace xmoe;


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
        XMOE_CUDA(cudaHostAlloc(&c->c.async_err_h, sizeof(int), cudaHostAllocMapped));
        *c->c.async_err_h = 0;
        XMOE_CUDA(cudaHostGetDevicePointer(&c->c.async_err_d, c->c.async_err_h, 0));
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
        } else if (dtype == XMOE_F32) {  // single-precision instantiation of the reference order
            float* lg = reinterpret_cast<float*>(ws);
            launch_gate_logits_f32(static_cast<const float*>(x), static_cast<const float*>(wg), S, H, E, lg, st);
            launch_softmax_topk_f32(lg, S, E, k, renorm, top, weights, st);
            if (logits) launch_f32_to_f64(lg, static_cast<long long>(S) * E, logits, st);
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
        require(G >= 1, XMOE_ERR_VALIDATION, "grouped_expert_mlp: at least one expert");
        // CountMismatch check (pf_pipeline.cpp:102-103) on the device, no host
        // sync: the GEMMs run on counts clamped to the buffer and a mismatch
        // is reported by xmoe_ctx_status
        const size_t es = elem_size(dtype);
        const size_t mid_bytes = (static_cast<size_t>(rows) * F * es + 255) & ~static_cast<size_t>(255);
        char* scr = static_cast<char*>(ctx->c.scratch(mid_bytes + sizeof(int32_t) * G + 256));
        void* mid = scr;
        auto* counts = reinterpret_cast<int32_t*>(scr + mid_bytes);
        launch_count_check(rows_per_expert, static_cast<int>(G), rows, counts, ctx->c.async_err_d, st);
        rows_per_expert = counts;
        if (dtype == XMOE_F64) {
            launch_grouped_gemm_f64(static_cast<const double*>(in), rows, H, rows_per_expert, G,
                                    static_cast<const double*>(w1), F, static_cast<double*>(mid), 1, st);
            launch_grouped_gemm_f64(static_cast<const double*>(mid), rows, F, rows_per_expert, G,
                                    static_cast<const double*>(w2), H, static_cast<double*>(out), 0, st);
        } else if (dtype == XMOE_F32) {
            launch_grouped_gemm_f32(static_cast<const float*>(in), rows, H, rows_per_expert, G,
                                    static_cast<const float*>(w1), F, static_cast<float*>(mid), 1, st);
            launch_grouped_gemm_f32(static_cast<const float*>(mid), rows, F, rows_per_expert, G,
                                    static_cast<const float*>(w2), H, static_cast<float*>(out), 0, st);
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

int xmoe_grouped_wgrad_bf16(xmoe_ctx* ctx, const void* X, const void* Y, int64_t rows,
                             const int32_t* rows_per_group, int64_t G, int64_t M, int64_t N, float* D,
                             void* stream) {
    return guarded([&] {
        auto st = static_cast<cudaStream_t>(stream);
        if (M % 64 == 0 && N % 128 == 0) {  // MN-major kernel on the row-major operands
            char* ws = static_cast<char*>(ctx->c.scratch(2 * 64 * G * (M + N) + 1024));
            launch_grouped_wgrad_mn(X, static_cast<int>(M), Y, static_cast<int>(N), rows, rows_per_group,
                                    static_cast<int>(G), ws, ws + 2 * 64 * G * M, D, st);
            return;
        }
        const long long Kp = (rows + 64 * G + 63) / 64 * 64;
        char* ws = static_cast<char*>(ctx->c.scratch(2 * (M + N) * Kp + 4096 + 12 * (G + 2)));
        int32_t* kpg = reinterpret_cast<int32_t*>(ws);
        int32_t* koff = kpg + (G + 1);
        int32_t* roff = koff + (G + 1);
        char* xT = ws + 4096;
        char* yT = xT + 2 * M * Kp;
        launch_pad_offsets(rows_per_group, static_cast<int>(G), kpg, koff, roff, st);
        launch_transpose_pad(X, static_cast<int>(M), rows_per_group, koff, roff, static_cast<int>(G), Kp, xT, st);
        launch_transpose_pad(Y, static_cast<int>(N), rows_per_group, koff, roff, static_cast<int>(G), Kp, yT, st);
        launch_grouped_wgrad_bf16(xT, static_cast<int>(M), Kp, kpg, static_cast<int>(G), yT, static_cast<int>(N), D, st);
    });
}

int xmoe_wgrad_split_bf16(xmoe_ctx* ctx, const void* X, const void* Y, int64_t rows, int64_t M, int64_t N,
                          int64_t splits, float* D, void* stream) {
    return guarded([&] {
        require(rows >= 0 && M > 0 && N > 0, XMOE_ERR_VALIDATION, "split wgrad: rows >= 0, M > 0, N > 0");
        require(M % 64 == 0, XMOE_ERR_VALIDATION, "split wgrad: M % 64 == 0");
        const long long Np = (N + 127) / 128 * 128;
        const size_t tails = 2 * 64 * static_cast<size_t>(splits) * (M + N);
        const size_t part = sizeof(float) * static_cast<size_t>(splits) * M * Np;
        char* ws = static_cast<char*>(ctx->c.scratch(256 + tails + part + 1024));
        char* ta = ws + 256;
        char* tb = ta + 2 * 64 * splits * M;
        float* pp = reinterpret_cast<float*>(ws + 256 + (tails + 255) / 256 * 256);
        launch_wgrad_mn_split(X, static_cast<int>(M), Y, static_cast<int>(N), rows, static_cast<int>(splits),
                              reinterpret_cast<int32_t*>(ws), ta, tb, pp, D, static_cast<cudaStream_t>(stream));
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
    return guarded([&] {
        if (!layer) return;
        std::unique_ptr<xmoe_layer> own(layer);
        own->l.quiesce();  // peers may still read this rank's symmetric region
    });
}

int xmoe_layer_set_weights(xmoe_layer* layer, const void* gate, const void* w1, const void* w2, const void* sw1,
                           const void* sw2, void* stream) {
    return guarded([&] {
        Layer& L = layer->l;
        require(gate && w1 && w2, XMOE_ERR_VALIDATION, "gate, w1 and w2 are required");
        require(L.Fs == 0 || (sw1 && sw2), XMOE_ERR_VALIDATION, "shared expert weights missing");
        layer_load_weights(L, gate, w1, w2, sw1, sw2, static_cast<cudaStream_t>(stream));
        // captured forwards read the weight buffers in place: still valid
    });
}

int xmoe_layer_inspect(xmoe_layer* layer, int worker, int what, const void** ptr, int64_t* count) {
    return guarded([&] {
        Layer& L = layer->l;
        require(ptr && count, XMOE_ERR_VALIDATION, "null output");
        require(worker >= 0 && worker < L.nl, XMOE_ERR_VALIDATION, "worker out of range");
        Worker& w = L.workers[worker];
        XMOE_CUDA(cudaDeviceSynchronize());
        int32_t B = 0;
        XMOE_CUDA(cudaMemcpy(&B, w.B_dev, sizeof(int32_t), cudaMemcpyDeviceToHost));
        const long long S = L.last_S, Sk = S * L.k;
        const void* p = nullptr;
        long long n = 0;
        switch (what) {
            case XMOE_INSPECT_TOP_EXPERTS: p = w.top; n = Sk; break;
            case XMOE_INSPECT_WEIGHTS: p = w.wts; n = Sk; break;
            case XMOE_INSPECT_TOKEN_IDS: p = w.token_ids; n = B; break;
            case XMOE_INSPECT_EXPERT_IDS: p = w.expert_ids; n = B; break;
            case XMOE_INSPECT_COMBINE_WEIGHTS: p = w.cw; n = B; break;
            case XMOE_INSPECT_TOKENS_PER_EXPERT: p = w.tpe; n = L.E; break;
            case XMOE_INSPECT_TPE_ALL: p = L.tpe_all; n = static_cast<long long>(L.W) * L.E; break;
            case XMOE_INSPECT_EXPERT_INPUT: p = w.recv; n = L.R_max * L.H; break;
            case XMOE_INSPECT_EXPERT_OUTPUT: p = w.eout; n = L.R_max * L.H; break;
            case XMOE_INSPECT_RECV_PER_EXPERT:
                require(L.nchunks == 1, XMOE_ERR_VALIDATION, "chunked layers keep per-chunk regions (XMOE_INSPECT_TPE_CHUNKS)");
                p = w.rpe; n = L.El; break;
            case XMOE_INSPECT_TPE_CHUNKS:
                require(L.nchunks > 1, XMOE_ERR_VALIDATION, "layer is not chunked");
                p = L.tpe_c_all; n = static_cast<long long>(L.W) * L.nchunks * L.E; break;
            case XMOE_INSPECT_DEST_RANK: p = w.dest_rank; n = B; break;
            case XMOE_INSPECT_DEST_ROW: p = w.dest_row; n = B; break;
            case XMOE_INSPECT_SLOT_POS: p = w.slot_pos; n = Sk; break;
            case XMOE_INSPECT_SSMB_KEPT:
                require(L.last_ssmb, XMOE_ERR_VALIDATION, "last forward was not ssmb_forward");
                p = L.ssmb_B; n = static_cast<long long>(L.ssmb_rows.size()); break;
            case XMOE_INSPECT_PILOT_MASK: {
                require(L.d.dispatch_mode == XMOE_DISPATCH_RBD, XMOE_ERR_VALIDATION, "not a redundancy-bypassing layer");
                if (!L.dbg_mask) L.dbg_mask = static_cast<uint8_t*>(L.alloc(static_cast<size_t>(L.S_max) * L.k + 16));
                XMOE_CUDA(cudaMemset(L.dbg_mask, 0, static_cast<size_t>(L.S_max) * L.k + 16));
                launch_mask_from_groups(w.rbd, w.slot_pos, L.k, Sk, L.dbg_mask, nullptr, nullptr);
                XMOE_CUDA(cudaDeviceSynchronize());
                p = L.dbg_mask; n = B; break;
            }
            default: fail(XMOE_ERR_VALIDATION, "unknown inspect item");
        }
        *ptr = p;
        *count = n;
    });
}

int xmoe_rng_uniform(xmoe_ctx* ctx, uint64_t seed, uint64_t offset, int64_t n, double lo, double hi, double grid,
                     int dtype, void* out, void* stream) {
    return guarded([&] {
        (void)ctx;
        require(dtype == XMOE_F64 || dtype == XMOE_F32 || dtype == XMOE_BF16, XMOE_ERR_VALIDATION, "unknown dtype");
        launch_rng_uniform(seed, offset, n, lo, hi, grid, dtype, out, static_cast<cudaStream_t>(stream));
    });
}

uint64_t xmoe_salt_seed(uint64_t seed, uint64_t a, uint64_t b) { return salt_seed_host(seed, a, b); }

int xmoe_rng_uniform_state(xmoe_ctx* ctx, const uint64_t* state, uint64_t offset, int64_t n, double lo, double hi,
                           double grid, int dtype, void* out, void* stream) {
    return guarded([&] {
        (void)ctx;
        require(state != nullptr, XMOE_ERR_VALIDATION, "null generator state");
        require(dtype == XMOE_F64 || dtype == XMOE_F32 || dtype == XMOE_BF16, XMOE_ERR_VALIDATION, "unknown dtype");
        launch_rng_uniform_state(state, offset, n, lo, hi, grid, dtype, out, static_cast<cudaStream_t>(stream));
    });
}

int xmoe_rng_advance(uint64_t* state, uint64_t n) {
    return guarded([&] {
        require(state != nullptr, XMOE_ERR_VALIDATION, "null generator state");
        rng_advance(state, n);
    });
}

int xmoe_make_layer_weights(xmoe_ctx* ctx, uint64_t seed, uint64_t offset, int64_t E, int64_t H, int64_t F,
                            int64_t first_expert, int64_t n_experts, double gate_grid, int dtype, void* gate,
                            void* w1, void* w2, void* stream) {
    return guarded([&] {
        require(E >= 1 && H >= 1 && F >= 1, XMOE_ERR_VALIDATION, "dims must be >= 1");
        require(first_expert >= 0 && n_experts >= 0 && first_expert + n_experts <= E, XMOE_ERR_VALIDATION,
                "expert slice out of range");
        require(dtype == XMOE_F64 || dtype == XMOE_F32 || dtype == XMOE_BF16, XMOE_ERR_VALIDATION, "unknown dtype");
        (void)ctx;
        auto st = static_cast<cudaStream_t>(stream);
        const size_t es = dtype == XMOE_F64 ? 8 : dtype == XMOE_F32 ? 4 : 2;
        const unsigned long long hf = static_cast<unsigned long long>(H) * F;
        // make_layer_weights draw order (padded_pipeline.cpp:13-27, gating.cpp:59-63):
        // gate [H,E], then per expert w1 [H,F] and w2 [F,H], all uniform(-0.1, 0.1)
        if (gate) launch_rng_uniform(seed, offset, H * E, -0.1, 0.1, gate_grid, dtype, gate, st);
        for (int64_t i = 0; i < n_experts; ++i) {
            const unsigned long long o = offset + static_cast<unsigned long long>(H) * E + 2 * hf * (first_expert + i);
            if (w1) launch_rng_uniform(seed, o, static_cast<long long>(hf), -0.1, 0.1, 0.0, dtype,
                                       static_cast<char*>(w1) + i * hf * es, st);
            if (w2) launch_rng_uniform(seed, o + hf, static_cast<long long>(hf), -0.1, 0.1, 0.0, dtype,
                                       static_cast<char*>(w2) + i * hf * es, st);
        }
    });
}

// asynchronous NCCL failures of the context's communicator (ncclCommGetAsyncError)
static void check_nccl_async(const Ctx& c) {
    if (!c.nccl) return;
    ncclResult_t async = ncclSuccess;
    XMOE_NCCL(ncclCommGetAsyncError(static_cast<ncclComm_t>(c.nccl), &async));
    if (async != ncclSuccess && async != ncclInProgress)
        fail(XMOE_ERR_NCCL, std::string("asynchronous NCCL error: ") + ncclGetErrorString(async));
}

int xmoe_ctx_status(xmoe_ctx* ctx) {
    return guarded([&] {
        check_nccl_async(ctx->c);
        if (ctx->c.async_err_h) {
            const int e = *reinterpret_cast<volatile int*>(ctx->c.async_err_h);
            if (e != 0) {
                *ctx->c.async_err_h = 0;  // reported once
                if (e == XMOE_ERR_COUNT_MISMATCH)
                    fail(e, "grouped_expert_mlp: segment counts disagree with input rows");
                fail(e, "asynchronous check failed");
            }
        }
    });
}

int xmoe_layer_status(xmoe_layer* layer) {
    return guarded([&] {
        layer->l.check_peers();
        check_nccl_async(*layer->l.ctx);
    });
}

int xmoe_moe_forward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x, int64_t S, void* out,
                     void* stream) {
    return guarded([&] {
        NvtxRange nvtx("xmoe_moe_forward");
        require(layer->l.ctx == &ctx->c, XMOE_ERR_VALIDATION, "layer belongs to another context");
        Layer& L = layer->l;
        auto st = static_cast<cudaStream_t>(stream);
        // CUDA-graph replay of the whole (host-sync-free) forward: one launch
        // instead of ~25, keyed by the buffers and length it was captured with
        const bool graphable = L.use_graph && !L.timing && (!L.distributed || L.p2p);
        if (!graphable) {
            layer_forward(L, x, S, out, st);
            return;
        }
        for (auto& g : L.graphs)
            if (g.x == x && g.out == out && g.S == S) {
                XMOE_CUDA(cudaGraphLaunch(g.exec, st));
                g_kernel_launches.fetch_add(g.kernels, std::memory_order_relaxed);  // our kernel nodes
                L.last_S = S;
                L.bwd_pending = true;
                return;
            }
        // capture on the layer's own stream (the caller's may be the legacy
        // default stream, which cannot be captured); replay on the caller's
        cudaGraph_t graph = nullptr;
        cudaStream_t cs = L.cap_stream;
        const unsigned long long before = g_kernel_launches.load();
        XMOE_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        try {
            layer_forward(L, x, S, out, cs);
        } catch (...) {
            cudaStreamEndCapture(cs, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        XMOE_CUDA(cudaStreamEndCapture(cs, &graph));
        // captured launches did not run: count them when the graph does
        const unsigned long long kernels = g_kernel_launches.load() - before;
        g_kernel_launches.fetch_sub(kernels, std::memory_order_relaxed);
        cudaGraphExec_t exec = nullptr;
        XMOE_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        XMOE_CUDA(cudaGraphDestroy(graph));
        if (L.graphs.size() >= 4) {
            cudaGraphExecDestroy(L.graphs.front().exec);
            L.graphs.erase(L.graphs.begin());
        }
        L.graphs.push_back({x, out, S, exec, kernels});
        XMOE_CUDA(cudaGraphLaunch(exec, st));
        g_kernel_launches.fetch_add(kernels, std::memory_order_relaxed);
    });
}

int xmoe_moe_forward_v(xmoe_ctx* ctx, xmoe_layer* layer, const void* x, const int64_t* S_per_worker, void* out,
                       void* stream) {
    return guarded([&] {
        require(layer->l.ctx == &ctx->c, XMOE_ERR_VALIDATION, "layer belongs to another context");
        require(S_per_worker != nullptr, XMOE_ERR_VALIDATION, "null token counts");
        Layer& L = layer->l;
        std::vector<long long> Sw(S_per_worker, S_per_worker + L.nl);
        layer_forward_v(L, x, Sw.data(), out, static_cast<cudaStream_t>(stream));
    });
}

int xmoe_layer_bwd_stage_ms(xmoe_layer* layer, float* out, int n) {
    return guarded([&] {
        Layer& L = layer->l;
        require(L.timing && L.train, XMOE_ERR_VALIDATION, "timing not enabled on a training layer");
        XMOE_CUDA(cudaEventSynchronize(L.bev[kBwEnd]));
        for (int i = 0; i < n && i < kBwdEvents - 1; ++i)
            XMOE_CUDA(cudaEventElapsedTime(&out[i], L.bev[i], L.bev[i + 1]));
    });
}

int xmoe_layer_chunks(const xmoe_layer* layer, int32_t* out) {
    return guarded([&] {
        require(out != nullptr, XMOE_ERR_VALIDATION, "null output");
        *out = layer->l.nchunks;
    });
}

int xmoe_layer_set_graph(xmoe_layer* layer, int enable) {
    return guarded([&] { layer->l.use_graph = enable != 0; });
}

int xmoe_moe_backward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x, const void* dy, int64_t S,
                      void* dx, void* stream) {
    return guarded([&] {
        NvtxRange nvtx("xmoe_moe_backward");
        require(layer->l.ctx == &ctx->c, XMOE_ERR_VALIDATION, "layer belongs to another context");
        layer_backward(layer->l, x, dy, S, dx, static_cast<cudaStream_t>(stream));
    });
}

int xmoe_layer_grads(xmoe_layer* layer, float** dgate, float** dw1, float** dw2, float** dsw1, float** dsw2) {
    return guarded([&] {
        Layer& L = layer->l;
        require(L.train, XMOE_ERR_VALIDATION, "layer was not created with XMOE_LAYER_TRAIN");
        if (dgate) *dgate = L.dgate;
        if (dw1) *dw1 = L.dw1;
        if (dw2) *dw2 = L.dw2;
        if (dsw1) *dsw1 = L.dsw1;
        if (dsw2) *dsw2 = L.dsw2;
    });
}

int xmoe_ssmb_forward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x_full, int64_t S,
                      void* out_full, void* stream) {
    return guarded([&] {
        NvtxRange nvtx("xmoe_ssmb_forward");
        ssmb_forward(ctx->c, layer->l, x_full, S, out_full, static_cast<cudaStream_t>(stream));
    });
}

static xmoe_topology topo_or_default(const xmoe_topology* t) {
    if (t) return *t;
    xmoe_topology d{};  // moesim::Topology defaults (config.hpp:30-37)
    d.gpus_per_node = 8;
    d.bw_intra = 200e9;
    d.bw_inter = 25e9;
    return d;
}

int xmoe_layer_ledger_entries(xmoe_layer* layer, const xmoe_topology* topo, xmoe_ledger_entry* out, int cap,
                              int* n) {
    return guarded([&] {
        require(n != nullptr, XMOE_ERR_VALIDATION, "null output");
        std::vector<xmoe_ledger_entry> v;
        layer->l.ledger_entries(topo_or_default(topo), v);
        *n = static_cast<int>(v.size());
        for (int i = 0; i < cap && i < *n; ++i) out[i] = v[i];
    });
}

static int ledger_csv(xmoe_layer* layer, const xmoe_topology* topo, char* buf, int64_t cap, int64_t* len,
                      bool padded) {
    return guarded([&] {
        require(len != nullptr, XMOE_ERR_VALIDATION, "null output");
        std::vector<xmoe_ledger_entry> v;
        if (padded) layer->l.padded_ledger_entries(topo_or_default(topo), v);
        else layer->l.ledger_entries(topo_or_default(topo), v);
        std::string csv = "collective_id,kind,intra_bytes,inter_bytes,modeled_time_s\n";
        char tb[64];
        for (const auto& e : v) {
            std::snprintf(tb, sizeof tb, "%.12g", e.time_s);
            csv += std::to_string(e.id) + ',' + e.kind + ',' + std::to_string(e.intra_bytes) + ',' +
                   std::to_string(e.inter_bytes) + ',' + tb + '\n';
        }
        *len = static_cast<int64_t>(csv.size());
        if (buf && cap > 0) {
            const size_t m = std::min<size_t>(csv.size(), static_cast<size_t>(cap - 1));
            std::memcpy(buf, csv.data(), m);
            buf[m] = '\0';
        }
    });
}

int xmoe_layer_ledger_csv(xmoe_layer* layer, const xmoe_topology* topo, char* buf, int64_t cap, int64_t* len) {
    return ledger_csv(layer, topo, buf, cap, len, false);
}

int xmoe_layer_padded_ledger_csv(xmoe_layer* layer, const xmoe_topology* topo, char* buf, int64_t cap,
                                 int64_t* len) {
    return ledger_csv(layer, topo, buf, cap, len, true);
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
        const int pairs[][2] = {{kEvStart, kEvGate},    {kEvGate, kEvPft},     {kEvPft, kEvDispatch},
                                {kEvDispatch, kEvGemm},  {kEvGemm, kEvShared},  {kEvShared, kEvCombine},
                                {kEvStart, kEvCombine},  {kEvPft, kEvCounts},   {kEvCounts, kEvMoved},
                                {kEvMoved, kEvDispatch}, {kEvShared, kEvReturn}, {kEvReturn, kEvCombine}};
        for (int i = 0; i < n && i < 12; ++i)
            XMOE_CUDA(cudaEventElapsedTime(&out[i], L.events[pairs[i][0]], L.events[pairs[i][1]]));
        if (n > 12) {  // shared-expert GEMMs on the side stream (0 when absent)
            out[12] = 0.f;
            if (L.Fs > 0) XMOE_CUDA(cudaEventElapsedTime(&out[12], L.ev_side0, L.ev_side1));
        }
        // chunked forward: per chunk, ms from the start to its scatter end,
        // GEMM start, GEMM end and combine end
        for (int i = 13; i < n && i - 13 < static_cast<int>(L.tl.size()); ++i)
            XMOE_CUDA(cudaEventElapsedTime(&out[i], L.events[kEvStart], L.tl[i - 13]));
    });
}

}  // extern "C"
