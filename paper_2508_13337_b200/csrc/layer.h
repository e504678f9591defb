// Host-side state behind the C-ABI handles: context and MoE layer.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "rbd.h"
#include "xmoe/xmoe.h"

namespace xmoe {

// moesim::Comm analogue (collectives.hpp:71-76): the expert-parallel group.
struct Ctx {
    int device = 0;
    int world = 1;
    int rank = -1;          // -1: this process drives every rank on `device`
    void* nccl = nullptr;   // ncclComm_t when rank >= 0 && world > 1
    void* ws = nullptr;     // grow-only scratch for the stateless operators
    size_t ws_bytes = 0;
    void* dflag = nullptr;  // device error flag
    int* async_err_h = nullptr;  // sticky error of asynchronous checks (host-mapped; xmoe_ctx_status)
    int* async_err_d = nullptr;

    int n_local() const { return rank < 0 ? world : 1; }
    int rank_of(int i) const { return rank < 0 ? i : rank; }
    void* scratch(size_t bytes);
    int* err_flag();
    ~Ctx();
};

// Per-rank buffers of one layer forward.
struct Worker {
    int rank = 0;
    double* logits = nullptr;     // [S, E]
    int32_t* top = nullptr;       // [S, k]
    double* wts = nullptr;        // [S, k]
    int32_t* token_ids = nullptr; // [S*k] packed ERI arrays (pft.hpp:17-25)
    int32_t* expert_ids = nullptr;
    double* cw = nullptr;
    int32_t* slot_pos = nullptr;  // [S, k] kept packed rows per token, ascending
    int32_t* B_dev = nullptr;     // packed row count
    int32_t* tpe = nullptr;       // [E] tokens per expert (row of tpe_all when shared)
    void* pft_ws = nullptr;
    int32_t* route_cnt = nullptr; // [ceil(S/128), E] per-tile expert histograms of the fused gate
    int32_t* dest_rank = nullptr; // [S*k] owner of each packed row
    int32_t* dest_row = nullptr;  // [S*k] its row in the owner's grouped buffer
    int32_t* rpe = nullptr;       // [El] rows per local expert (recv_per_expert)
    void* recv = nullptr;         // [R_max, H] grouped expert input (PfDispatch::expert_input)
    void* mid = nullptr;          // [R_max, F]
    void* eout = nullptr;         // [R_max, H]
    void* send = nullptr;         // [S*k, H] NCCL path: packed rows
    void* back = nullptr;         // [S*k, H] NCCL path: returned rows, packed order
    void* smid = nullptr;         // shared experts [S, Fs]
    void* sout = nullptr;         // [S, H]
    int32_t* s_rows = nullptr;
    unsigned long long* slot_src = nullptr;  // [S*k] address of each copy's expert output
    float* slot_w = nullptr;                 // [S*k] its combine weight
    char* sym = nullptr;          // symmetric region: recv | eout | recv_u | desc_recv | back_u
    char* xs = nullptr;           // pull dispatch: staged input [S_max, H] (symmetric region)
    float* lpartial = nullptr;    // chunked late shared: fp32 routed sums [S_max, H]
    unsigned* lready = nullptr;   // chunked late shared: per 128-token block publication counts
    int32_t* rsrc = nullptr;      // pull dispatch: (source << 24 | token) of every grouped row
    // redundancy-bypassing dispatch (rbd.cu)
    RbdWork rbd{};
    void* recv_u = nullptr;       // [W*S, H] unique rows received from every source
    RbdDesc* desc_recv = nullptr; // [R_max]
    int32_t* gstart = nullptr;    // [W*S] first descriptor of each received group
    void* back_u = nullptr;       // [W*S, H] merged group outputs, read by the sources
    // training (XMOE_LAYER_TRAIN): symmetric-region pieces
    void* dyg = nullptr;          // [R_max, H] dy of each received copy (grouped order)
    void* dxc = nullptr;          // [R_max, H] dx of each received copy
    float* gw = nullptr;          // [R_max] combine weight of each received copy
    unsigned long long* gsrc = nullptr;  // [R_max] home (rank << 32 | token*k + slot)
    float* slot_dw = nullptr;     // [S*k] dL/dw of my copies (written by the owners)
    // training: local
    void* dz = nullptr;           // [R_max, H]
    void* dH = nullptr;           // [R_max, F]
    void* tail_a = nullptr;       // wgrad tail blocks [64*(El+1), max(H,F,Fs)]
    void* tail_b = nullptr;
    int32_t* a_idx = nullptr;     // [R_max] RBD gather: physical recv row of every grouped row
    uint32_t* mbits = nullptr;    // [R_max, ceil(F/32)] ReLU mask bits of mid (training)
    uint32_t* smbits = nullptr;   // [S, ceil(Fs/32)] of the shared experts' mid
    void* tail_sa = nullptr;      // the same for the side-stream (shared-expert) wgrad
    void* tail_sb = nullptr;
    // split-K weight gradients of the single-group (token-level) products:
    // shared experts on the side stream (_s), the gate on the layer stream (_g)
    int32_t* split_s = nullptr;   // [32] rows per split
    int32_t* split_g = nullptr;
    float* part_s = nullptr;      // [splits, M, roundup(N, 128)] fp32 partials
    float* part_g = nullptr;
    void* tail_ga = nullptr;      // [64*splits_g, H], [64*splits_g, E]
    void* tail_gb = nullptr;
    void* dl = nullptr;           // [S, E]
    void* dxg = nullptr;          // [S, H] gate part of dx
    void* dHs = nullptr;          // [S, Fs]
    void* dxs = nullptr;          // [S, H] shared part of dx
    unsigned long long* bslot_src = nullptr;  // [S*k] dxc row of each kept copy
    // token-chunked pipeline (chunk.cu)
    int32_t* tpe_c = nullptr;     // [C, E] my kept copies per (chunk, expert)
    int32_t* pfx_c = nullptr;     // [C, E] their offset inside the expert's packed segment
    int32_t* seg = nullptr;       // [E] packed segment start of each expert
    int32_t* cbase = nullptr;     // [C, E] first destination row of (chunk, expert) at its owner
    int32_t* rpe_c = nullptr;     // [C, El] rows per local expert in my chunk regions
    unsigned* flags = nullptr;    // [2, kMaxChunks, W] epoch flags (symmetric region)
};

// stage boundaries; kEvCounts/kEvMoved/kEvReturn split the exchange phases
// backward stage boundaries: start, dy scattered, owner prep, dgrad GEMMs,
// wgrad GEMMs, token-level (transpose + shared experts), gate + dx combine
enum { kBwStart = 0, kBwScatter, kBwPrep, kBwDgrad, kBwWgrad, kBwToken, kBwEnd, kBwdEvents };
enum { kEvStart = 0, kEvGate, kEvPft, kEvDispatch, kEvGemm, kEvShared, kEvCombine, kEvCounts, kEvMoved, kEvReturn, kNumEvents };

struct Layer {
    Ctx* ctx = nullptr;
    xmoe_layer_desc d{};
    int W = 1, E = 0, H = 0, F = 0, k = 0, El = 0, E_held = 0, Fs = 0;
    int nl = 1;                // ranks driven by this process
    int gpn = 1;               // RBD GPUs per node (node_of = rank / gpn)
    bool rbd_gather = false;   // RBD GEMM1 gathers replica rows (no expand copy)
    bool ssmb = false;         // sequence-sharded block: experts replicated, MoE local
    bool route_cnt_ok = false; // fused gate + dropless placement available (BF16, E <= 256, k <= 8)
    float* partial = nullptr;  // [S, H] fp32 routed sums (one GPU, late shared GEMM2)
    unsigned* ready = nullptr; // [ceil(S/128)] tokens of each block the combine has published
    bool distributed = false;  // one process per GPU, world > 1
    bool p2p = false;          // NVLink peer tables (else NCCL send/recv baseline)
    int32_t* bar = nullptr;    // 4-byte all-reduce used as a cross-rank barrier
    std::vector<void*> peer_maps;
    size_t es = 2;
    long long R_max = 0, S_max = 0, last_S = 0;
    std::vector<long long> last_Sw;  // per-worker token counts of the last forward
    bool bwd_pending = false;  // a forward ran since the last backward (one backward per forward)
    void* gate = nullptr;  // F64 [H,E]; BF16 [E,H]
    void* w1 = nullptr;    // F64 [E_held,H,F]; BF16 [E_held,F,H]
    void* w2 = nullptr;    // F64 [E_held,F,H]; BF16 [E_held,H,F]
    void* sw1 = nullptr;   // merged shared: F64 [H,Fs]; BF16 [Fs,H]
    void* sw2 = nullptr;   // F64 [Fs,H]; BF16 [H,Fs]
    int32_t* tpe_all = nullptr;  // [W, E]
    char** recv_tab = nullptr;   // device table: rank -> recv buffer (shared-device ranks)
    // pull dispatch (chunked plain dispatch): owners copy their rows from the
    // sources' staged inputs instead of the sources storing into the owners
    bool pull = false;
    char** xs_tab = nullptr;      // rank -> staged input [S_max, H] (symmetric region)
    int32_t** rsrc_tab = nullptr; // rank -> [R_max] (source << 24 | token) of every grouped row
    char** eout_tab = nullptr;
    // training tables and weights in the reference layouts (dgrad B operands)
    bool train = false;
    long long off_eout = 0, off_dxc = 0;
    char** dyg_tab = nullptr;
    char** dxc_tab = nullptr;
    float** gw_tab = nullptr;
    unsigned long long** gsrc_tab = nullptr;
    float** slotdw_tab = nullptr;
    void* w1r = nullptr;   // [E_held, H, F]
    void* w2r = nullptr;   // [E_held, F, H]
    void* gater = nullptr; // [H, E]
    void* sw1r = nullptr;  // [H, Fs] merged
    void* sw2r = nullptr;  // [Fs, H]
    float* dgate = nullptr;
    int splits_s1 = 1, splits_s2 = 1, splits_g = 1;  // split-K factors (wgrad_splits)
    float* dw1 = nullptr;
    float* dw2 = nullptr;
    float* dsw1 = nullptr;
    float* dsw2 = nullptr;
    char** recv_u_tab = nullptr;  // RBD tables (local or NVLink peer addresses)
    RbdDesc** desc_tab = nullptr;
    char** back_tab = nullptr;
    std::vector<int32_t> h_tpe;
    uint64_t* jumps = nullptr;   // RBD jump-ahead matrices (device)
    int32_t* G_all = nullptr;    // [W, W] groups source -> dest (device)
    std::vector<int32_t> h_G;
    std::vector<Worker> workers;
    std::vector<void*> allocs;
    std::vector<cudaEvent_t> events;
    bool timing = false;
    bool nvtx_open = false;  // an NVTX stage range is pushed (Layer::mark)
    bool use_graph = false;
    struct GraphEntry {
        const void* x;
        void* out;
        long long S;
        cudaGraphExec_t exec;
        unsigned long long kernels;  // our kernel nodes in it (xmoe_kernel_launches)
    };
    std::vector<GraphEntry> graphs;  // captured forwards (xmoe_layer_set_graph)
    cudaStream_t cap_stream = nullptr;
    cudaStream_t side = nullptr;  // shared-expert GEMMs overlap routing + exchange
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_side0 = nullptr, ev_side1 = nullptr;
    cudaEvent_t ev_routed = nullptr;  // late shared GEMM2: routed GEMMs done, ready counters cleared
    // token-chunked pipeline: C chunks of Rc rows per owner, comm stream for
    // the row movement, per-chunk events and cross-GPU epoch flags
    int nchunks = 1;
    int Rc = 0;
    int32_t* tpe_c_all = nullptr;  // [W, C, E]
    int32_t* gd_all = nullptr;     // RBD [W_src, 2, W, C] groups / copies per (dest, chunk)
    unsigned** flag_tab = nullptr; // rank -> its flags (peer addresses)
    int32_t** cnt_tab = nullptr;   // rank -> its count all-gather area (peer addresses)
    int area_ints = 0;             // ints per half of the count area
    unsigned* epoch = nullptr;     // forwards issued (device)
    cudaStream_t comm = nullptr;
    std::vector<cudaEvent_t> evA, evB;
    std::vector<cudaEvent_t> tl;   // timing: per chunk scatter end, GEMM start, GEMM end, combine end
    std::vector<cudaEvent_t> bev;  // timing: backward stage boundaries (kBwdEvents)
    cudaEvent_t ev_done = nullptr;
    // peer-wait failures (chunk.cu wait_flag): host-mapped word, 0 = healthy,
    // 0x100 | slot = a peer never raised that flag within XMOE_PEER_TIMEOUT_S
    uint8_t* dbg_mask = nullptr;  // xmoe_layer_inspect: RBD pilot mask of the last forward
    int* peer_err_h = nullptr;
    int* peer_err_d = nullptr;

    void* alloc(size_t bytes);
    void mark(int ev, cudaStream_t st);
    void exchange_nccl(bool forward, cudaStream_t st);
    void barrier(cudaStream_t st);
    long long C(int s, int d) const;  // copies source s -> dest d (needs h_tpe)
    void ledger(uint64_t* out, int n);
    unsigned long long* led_cnt = nullptr;  // device ledger counters (rbd.cu ledger_counts_kernel)
    std::vector<uint64_t> device_counts(const Worker& w, long long S, bool groups);
    void quiesce();            // cross-rank barrier before teardown (p2p layers)
    void check_peers() const;  // throws XMOE_ERR_PEER_TIMEOUT after a failed peer wait
    // reference-schema ledger (ledger.cpp)
    bool last_ssmb = false;             // last forward was ssmb_forward
    std::vector<long long> ssmb_rows;   // its shard lengths
    int32_t* ssmb_B = nullptr;          // [G] kept copies per shard (device)
    int ssmb_cap = 0;
    void ledger_entries(const xmoe_topology& topo, std::vector<xmoe_ledger_entry>& out);
    void padded_ledger_entries(const xmoe_topology& topo, std::vector<xmoe_ledger_entry>& out);
    ~Layer();
};

void layer_create(Ctx& ctx, const xmoe_layer_desc& d, const void* gate, const void* w1,
                  const void* w2, const void* sw1, const void* sw2, Layer& L);
void layer_load_weights(Layer& L, const void* gate, const void* w1, const void* w2, const void* sw1, const void* sw2,
                        cudaStream_t st);
void layer_forward(Layer& L, const void* x, long long S, void* out, cudaStream_t st);
void layer_forward_v(Layer& L, const void* x, const long long* Sw, void* out, cudaStream_t st);
void layer_backward(Layer& L, const void* x, const void* dy, long long S, void* dx, cudaStream_t st);
void ssmb_forward(Ctx& ctx, Layer& L, const void* x_full, long long S, void* out_full, cudaStream_t st);

}  // namespace xmoe

// C-ABI handles (xmoe.h)
struct xmoe_ctx {
    xmoe::Ctx c;
};
struct xmoe_layer {
    xmoe::Layer l;
};
