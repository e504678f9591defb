// Reference-shaped C++ API (include/xmoe/moesim_compat.hpp) over the C-ABI.
// Each function mirrors one moesim operator: same argument meaning, same
// validation order and message text, same exception types; the work runs on
// the B200 in the F64 parity instantiation.
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>

#include "xmoe/moesim_compat.hpp"
#include "xmoe/xmoe.h"

namespace xmoe {
namespace {

[[noreturn]] void rethrow(int rc) {
    const std::string m = xmoe_last_error();
    switch (rc) {
        case XMOE_ERR_PARSE: throw ParseError(m);
        case XMOE_ERR_VALIDATION: throw ValidationError(m);
        case XMOE_ERR_DIMENSION: throw DimensionError(m);
        case XMOE_ERR_INDEX: throw IndexError(m);
        case XMOE_ERR_COUNT_MISMATCH: throw CountMismatch(m);
        case XMOE_ERR_PLAN_MISMATCH: throw PlanMismatch(m);
        default: throw std::runtime_error("xmoe: " + m);
    }
}
void ck(int rc) {
    if (rc != XMOE_OK) rethrow(rc);
}
void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("xmoe: ") + cudaGetErrorString(e));
}

// Device buffer with upload/download helpers.
struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    explicit DBuf(size_t bytes) : n(bytes) { cuda(cudaMalloc(&p, bytes ? bytes : 8)); }
    ~DBuf() { cudaFree(p); }
    DBuf(const DBuf&) = delete;
    template <class T>
    T* as() { return static_cast<T*>(p); }
    void up(const void* h, size_t bytes) { if (bytes) cuda(cudaMemcpy(p, h, bytes, cudaMemcpyHostToDevice)); }
    void down(void* h, size_t bytes) const { if (bytes) cuda(cudaMemcpy(h, p, bytes, cudaMemcpyDeviceToHost)); }
};

std::unique_ptr<DBuf> upload(const std::vector<double>& v) {
    auto b = std::make_unique<DBuf>(v.size() * sizeof(double));
    b->up(v.data(), v.size() * sizeof(double));
    return b;
}
// int64 ids -> int32 (out-of-range values become -1 so the device range check fires)
std::unique_ptr<DBuf> upload_ids(const std::vector<std::int64_t>& v) {
    std::vector<std::int32_t> h(v.size());
    for (size_t i = 0; i < v.size(); ++i)
        h[i] = (v[i] < 0 || v[i] > 0x7fffffff) ? -1 : static_cast<std::int32_t>(v[i]);
    auto b = std::make_unique<DBuf>(h.size() * 4);
    b->up(h.data(), h.size() * 4);
    return b;
}

// One rank == -1 context per group size, on the current device.
xmoe_ctx* ctx_for(int world) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, xmoe_ctx*> cache;
    int dev = 0;
    cuda(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    auto& c = cache[{dev, world}];
    if (!c) ck(xmoe_ctx_create(dev, world, -1, nullptr, &c));
    return c;
}

struct LayerHandle {
    xmoe_layer* l = nullptr;
    ~LayerHandle() { if (l) xmoe_layer_destroy(l); }
};

// Packs per-expert matrices [first, first+n) of the reference layout.
std::vector<double> pack(const std::vector<Matrix>& ms, std::int64_t first, std::int64_t n) {
    std::vector<double> out;
    for (std::int64_t e = first; e < first + n; ++e) out.insert(out.end(), ms[e].data.begin(), ms[e].data.end());
    return out;
}

void make_layer(xmoe_ctx* ctx, const MoeLayerWeights& w, std::int64_t E, std::int64_t k, std::int64_t cap,
                std::int64_t max_tokens, int mode, std::uint64_t seed, int flags, LayerHandle& lh) {
    if (w.w1.size() < static_cast<size_t>(E) || w.w2.size() < static_cast<size_t>(E))
        throw DimensionError("xmoe: weights hold fewer experts than num_experts");
    const std::int64_t H = static_cast<std::int64_t>(w.gate.rows);
    const std::int64_t F = E > 0 ? static_cast<std::int64_t>(w.w1[0].cols) : 0;
    xmoe_layer_desc d{};
    d.num_experts = E;
    d.model_dim = H;
    d.ffn_dim = F;
    d.top_k = k;
    d.max_token_count = cap;
    d.max_tokens = max_tokens > 0 ? max_tokens : 1;
    d.dtype = XMOE_F64;
    d.dispatch_mode = mode;
    d.flags = flags;
    d.seed = seed;
    auto g = upload(w.gate.data);
    auto w1 = upload(pack(w.w1, 0, E));
    auto w2 = upload(pack(w.w2, 0, E));
    ck(xmoe_layer_create(ctx, &d, g->p, w1->p, w2->p, nullptr, nullptr, &lh.l));
}

std::vector<Matrix> run_layer(const MoeInstance& inst, Comm& comm, int mode, std::uint64_t seed,
                              const char* who, int flags = 0) {
    const size_t W = comm.group.size();
    if (inst.tokens.size() != W) throw DimensionError(std::string(who) + ": need one token matrix per worker");
    const std::int64_t E = inst.num_experts;
    if (W == 0 || E % static_cast<std::int64_t>(W) != 0)
        throw ValidationError("num_experts must be divisible by the worker-group size");
    const size_t S = inst.tokens[0].rows, H = inst.weights.gate.rows;
    for (const auto& t : inst.tokens)
        if (t.rows != S) throw DimensionError("xmoe: every worker must hold the same number of tokens");
    std::vector<double> x;
    for (const auto& t : inst.tokens) x.insert(x.end(), t.data.begin(), t.data.end());
    xmoe_ctx* ctx = ctx_for(static_cast<int>(W));
    LayerHandle lh;
    make_layer(ctx, inst.weights, E, inst.top_k, inst.max_token_count, static_cast<std::int64_t>(S), mode, seed, flags,
               lh);
    auto dx = upload(x);
    DBuf dout(x.size() * sizeof(double));
    ck(xmoe_moe_forward(ctx, lh.l, dx->p, static_cast<std::int64_t>(S), dout.p, nullptr));
    cuda(cudaDeviceSynchronize());
    std::vector<Matrix> out(W, Matrix(S, H));
    for (size_t w = 0; w < W; ++w) cuda(cudaMemcpy(out[w].data.data(), dout.as<char>() + w * S * H * sizeof(double),
                                                   S * H * sizeof(double), cudaMemcpyDeviceToHost));
    return out;
}

}  // namespace

GateOutput gate_forward(const Matrix& tokens, const Matrix& gate_weights, std::int64_t top_k) {
    if (tokens.cols != gate_weights.rows) throw DimensionError("gate_forward: tokens.cols != gate_weights.rows");
    const std::int64_t S = static_cast<std::int64_t>(tokens.rows), E = static_cast<std::int64_t>(gate_weights.cols);
    if (top_k < 1) throw ValidationError("top_k must be >= 1");
    if (top_k > E) throw ValidationError("top_k must be <= num_experts");
    GateOutput g;
    g.top_k = top_k;
    g.gate_out = tokens;
    g.top_experts.resize(S * top_k);
    g.combine_weights.resize(S * top_k);
    if (S == 0) return g;
    auto dx = upload(tokens.data);
    auto dw = upload(gate_weights.data);
    DBuf top(S * top_k * 4), wt(S * top_k * 8);
    ck(xmoe_gate_forward(ctx_for(1), XMOE_F64, dx->p, dw->p, S, static_cast<std::int64_t>(tokens.cols), E, top_k,
                         0, top.as<std::int32_t>(), wt.as<double>(), nullptr, nullptr));
    std::vector<std::int32_t> t32(S * top_k);
    top.down(t32.data(), t32.size() * 4);
    wt.down(g.combine_weights.data(), g.combine_weights.size() * 8);
    for (size_t i = 0; i < t32.size(); ++i) g.top_experts[i] = t32[i];
    return g;
}

Pft pft_construct(std::int64_t cap, std::int64_t E, std::size_t S, std::int64_t k,
                  const std::vector<std::int64_t>& top, const std::vector<double>& w) {
    if (cap < 1) throw ValidationError("max_token_count must be >= 1");
    if (E < 1) throw ValidationError("num_experts must be >= 1");
    if (k < 1) throw ValidationError("top_k must be >= 1");
    const size_t flat = S * static_cast<size_t>(k);
    if (top.size() != flat || w.size() != flat)
        throw DimensionError("pft_construct: routing arrays must be seq_len * top_k");
    Pft p;
    p.tokens_per_expert.assign(E, 0);
    if (flat == 0) return p;
    auto dt = upload_ids(top);
    auto dw = upload(w);
    DBuf tid(flat * 4), eid(flat * 4), cw(flat * 8), tpe(E * 4), B(16);
    ck(xmoe_pft_construct(ctx_for(1), dt->as<std::int32_t>(), dw->as<double>(), static_cast<std::int64_t>(S), k, E,
                          cap, tid.as<std::int32_t>(), eid.as<std::int32_t>(), cw.as<double>(),
                          tpe.as<std::int32_t>(), nullptr, B.as<std::int32_t>(), 1, nullptr));
    std::int32_t b = 0;
    B.down(&b, 4);
    std::vector<std::int32_t> a(b), c(b), t(E);
    tid.down(a.data(), b * 4);
    eid.down(c.data(), b * 4);
    tpe.down(t.data(), E * 4);
    p.combine_weights.resize(b);
    cw.down(p.combine_weights.data(), b * 8);
    p.token_ids.assign(a.begin(), a.end());
    p.expert_ids.assign(c.begin(), c.end());
    for (std::int64_t e = 0; e < E; ++e) p.tokens_per_expert[e] = t[e];
    return p;
}

Pft pft_construct(std::int64_t cap, std::int64_t E, const GateOutput& gate) {
    return pft_construct(cap, E, gate.gate_out.rows, gate.top_k, gate.top_experts, gate.combine_weights);
}

Matrix gather_rows(const Matrix& src, const std::vector<std::int64_t>& ids) {
    Matrix out(ids.size(), src.cols);
    if (ids.empty()) return out;
    auto ds = upload(src.data);
    auto di = upload_ids(ids);
    DBuf dout(out.data.size() * 8);
    ck(xmoe_gather_rows(ctx_for(1), XMOE_F64, ds->p, static_cast<std::int64_t>(src.rows),
                        static_cast<std::int64_t>(src.cols), di->as<std::int32_t>(),
                        static_cast<std::int64_t>(ids.size()), dout.p, 1, nullptr));
    dout.down(out.data.data(), out.data.size() * 8);
    return out;
}

Matrix scatter_combine(const Matrix& rows, const std::vector<std::int64_t>& token_ids,
                       const std::vector<double>& weights, std::size_t seq_len) {
    if (rows.rows != token_ids.size() || rows.rows != weights.size())
        throw DimensionError("scatter_combine: rows and ERI arrays disagree");
    Matrix out(seq_len, rows.cols);
    for (auto t : token_ids)
        if (t < 0 || static_cast<std::size_t>(t) >= seq_len) throw IndexError("scatter_combine: token id out of range");
    if (seq_len == 0 || rows.cols == 0) return out;
    auto dr = upload(rows.data);
    auto di = upload_ids(token_ids);
    auto dw = upload(weights);
    DBuf dout(out.data.size() * 8);
    ck(xmoe_scatter_combine(ctx_for(1), XMOE_F64, dr->p, static_cast<std::int64_t>(rows.rows),
                            static_cast<std::int64_t>(rows.cols), di->as<std::int32_t>(), dw->as<double>(),
                            static_cast<std::int64_t>(seq_len), dout.p, 0, nullptr));
    dout.down(out.data.data(), out.data.size() * 8);
    return out;
}

Matrix grouped_expert_mlp(const Matrix& input, const std::vector<std::int64_t>& rpe,
                          const MoeLayerWeights& weights, std::int64_t first_expert) {
    const std::int64_t G = static_cast<std::int64_t>(rpe.size());
    Matrix out(input.rows, input.cols);
    std::int64_t F = 0;
    for (std::int64_t i = 0; i < G; ++i) {
        if (rpe[i] == 0) continue;
        const auto& w1 = weights.w1[first_expert + i];
        if (input.cols != w1.rows) throw DimensionError("grouped_expert_mlp: activation width mismatch");
        F = static_cast<std::int64_t>(w1.cols);
    }
    std::int64_t tot = 0;
    for (auto v : rpe) tot += v;
    if (tot != static_cast<std::int64_t>(input.rows))
        throw CountMismatch("grouped_expert_mlp: segment counts disagree with input rows");
    if (input.rows == 0) return out;
    std::vector<std::int64_t> counts(rpe);
    auto dc = upload_ids(counts);
    auto dx = upload(input.data);
    auto w1 = upload(pack(weights.w1, first_expert, G));
    auto w2 = upload(pack(weights.w2, first_expert, G));
    DBuf dout(out.data.size() * 8);
    ck(xmoe_grouped_mlp(ctx_for(1), XMOE_F64, dx->p, static_cast<std::int64_t>(input.rows), dc->as<std::int32_t>(),
                        G, w1->p, w2->p, static_cast<std::int64_t>(input.cols), F, dout.p, nullptr));
    dout.down(out.data.data(), out.data.size() * 8);
    return out;
}

std::vector<Matrix> pf_moe_forward(const MoeInstance& inst, Comm& comm, ActivationCounters*) {
    return run_layer(inst, comm, XMOE_DISPATCH_NAIVE, 0, "pf_moe_forward");
}

// node_of must be contiguous blocks of equal size (node n = ranks
// [n*g, (n+1)*g)); g > 1 is the two-tier bypass (rbd.cpp:83-358)
std::vector<Matrix> rbd_moe_forward(const MoeInstance& inst, Comm& comm, std::uint64_t seed) {
    const auto& no = comm.group.node_of;
    const size_t W = no.size();
    size_t g = 1;
    while (g < W && no[g] == no[0]) ++g;
    bool blocks = W % g == 0;
    for (size_t i = 0; blocks && i < W; ++i) {
        if (no[i] != no[(i / g) * g]) blocks = false;
        if (i % g == 0)
            for (size_t j = 0; j < i; j += g)
                if (no[j] == no[i]) blocks = false;
    }
    if (!blocks)
        throw ValidationError("xmoe: node_of must be contiguous blocks of equal size (rank / gpus_per_node)");
    return run_layer(inst, comm, XMOE_DISPATCH_RBD, seed, "rbd_moe_forward",
                     XMOE_LAYER_GPUS_PER_NODE(static_cast<int>(g)));
}

Matrix ssmb_forward(const Matrix& tokens, std::int64_t G, const MoeLayerWeights& weights, std::int64_t E,
                    std::int64_t k, std::int64_t cap, Comm& comm, ActivationCounters*) {
    const std::int64_t S = static_cast<std::int64_t>(tokens.rows);
    if (G < 1) throw ValidationError("ssmb_forward: shard count must be >= 1");
    if (G > S) throw ValidationError("ssmb_forward: more shards than sequence rows");
    if (static_cast<size_t>(G) != comm.group.size())
        throw ValidationError("ssmb_forward: shard count must match the worker-group size");
    xmoe_ctx* ctx = ctx_for(static_cast<int>(G));
    LayerHandle lh;
    make_layer(ctx, weights, E, k, cap, S - (G - 1) * (S / G), XMOE_DISPATCH_NAIVE, 0, XMOE_LAYER_SSMB, lh);
    auto dx = upload(tokens.data);
    DBuf dout(tokens.data.size() * 8);
    ck(xmoe_ssmb_forward(ctx, lh.l, dx->p, S, dout.p, nullptr));
    Matrix out(tokens.rows, tokens.cols);
    cuda(cudaDeviceSynchronize());
    dout.down(out.data.data(), out.data.size() * 8);
    return out;
}

}  // namespace xmoe
