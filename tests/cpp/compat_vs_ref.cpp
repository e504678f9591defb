// Drop-in check: the reference's own operator API (moesim::, the UNMODIFIED
// reference compiled into oracle/_ref/libmoesim_ref.so) and the xmoe
// reference-shaped API (include/xmoe/moesim_compat.hpp, running on the B200)
// on the same inputs, plus the reference unit tests' known answers replayed
// through xmoe::.  TEST INFRASTRUCTURE: links the reference only as the
// checker.  Exit 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>

#include "moesim/gating.hpp"
#include "moesim/pf_pipeline.hpp"
#include "moesim/pft.hpp"
#include "moesim/rbd.hpp"
#include "moesim/ssmb.hpp"
#include "xmoe/moesim_compat.hpp"

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (c) ++g_pass;                                                      \
        else {                                                                \
            ++g_fail;                                                         \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);          \
        }                                                                     \
    } while (0)

template <class Ex, class F>
static bool throws(F&& f, const char* msg = nullptr) {
    try {
        f();
    } catch (const Ex& e) {
        return msg == nullptr || std::string(e.what()) == msg;
    } catch (...) {
        return false;
    }
    return false;
}

static xmoe::Matrix X(const moesim::Matrix& m) {
    xmoe::Matrix o(m.rows, m.cols);
    o.data = m.data;
    return o;
}
static xmoe::MoeLayerWeights X(const moesim::MoeLayerWeights& w) {
    xmoe::MoeLayerWeights o;
    o.gate = X(w.gate);
    for (const auto& m : w.w1) o.w1.push_back(X(m));
    for (const auto& m : w.w2) o.w2.push_back(X(m));
    return o;
}
static double rel(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return 1e300;
    double m = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double s = std::max({std::fabs(a[i]), std::fabs(b[i]), 1.0});
        m = std::max(m, std::fabs(a[i] - b[i]) / s);
    }
    return m;
}

int main() {
    using moesim::Rng;
    // ---------------- known answers (test_gating.cpp, test_pft.cpp)
    {
        xmoe::Matrix t(1, 2);
        t.at(0, 0) = 1.0;
        t.at(0, 1) = -2.0;
        const auto g = xmoe::gate_forward(t, xmoe::Matrix(2, 2), 1);
        CHECK(g.expert_at(0, 0) == 0 && std::fabs(g.weight_at(0, 0) - 0.5) < 1e-12);
        CHECK(throws<xmoe::DimensionError>([] { xmoe::gate_forward(xmoe::Matrix(2, 4), xmoe::Matrix(3, 4), 1); }));
        CHECK(throws<xmoe::ValidationError>([] { xmoe::gate_forward(xmoe::Matrix(2, 4), xmoe::Matrix(4, 4), 0); },
                                           "top_k must be >= 1"));
        CHECK(throws<xmoe::ValidationError>([] { xmoe::gate_forward(xmoe::Matrix(2, 4), xmoe::Matrix(4, 4), 5); },
                                           "top_k must be <= num_experts"));
        const auto p = xmoe::pft_construct(2, 2, 4, 1, {0, 1, 0, 0}, {0.9, 0.8, 0.5, 0.7});
        CHECK((p.token_ids == std::vector<std::int64_t>{0, 3, 1}));
        CHECK((p.expert_ids == std::vector<std::int64_t>{0, 0, 1}));
        CHECK((p.tokens_per_expert == std::vector<std::int64_t>{2, 1}));
        CHECK((p.combine_weights == std::vector<double>{0.9, 0.7, 0.8}));
        CHECK((xmoe::pft_construct(2, 1, 3, 1, {0, 0, 0}, {0.4, 0.4, 0.4}).token_ids == std::vector<std::int64_t>{0, 1}));
        CHECK(throws<xmoe::ValidationError>([] { xmoe::pft_construct(0, 1, 2, 1, {0, 0}, {0.5, 0.5}); },
                                           "max_token_count must be >= 1"));
        CHECK(throws<xmoe::ValidationError>([] { xmoe::pft_construct(1, 1, 1, 2, {0, 0}, {0.5, 0.5}); }));
        CHECK(throws<xmoe::IndexError>([] { xmoe::pft_construct(1, 1, 2, 1, {0, 3}, {0.5, 0.5}); }));
        CHECK(throws<xmoe::DimensionError>([] { xmoe::pft_construct(1, 1, 1, 1, {0, 0}, {0.5, 0.5}); }));
        xmoe::Matrix src(3, 2);
        for (int i = 0; i < 6; ++i) src.data[i] = i + 1;
        const auto gr = xmoe::gather_rows(src, {2, 0, 2});
        CHECK(gr.at(0, 0) == 5.0 && gr.at(1, 0) == 1.0);
        const auto sc = xmoe::scatter_combine(gr, {2, 0, 2}, {0.5, 1.0, 0.25}, 3);
        CHECK(sc.at(0, 0) == 1.0 && sc.at(0, 1) == 2.0 && sc.at(1, 0) == 0.0 && std::fabs(sc.at(2, 0) - 3.75) < 1e-12);
        CHECK(throws<xmoe::IndexError>([&] { xmoe::gather_rows(src, {3}); }));
        CHECK(throws<xmoe::IndexError>([&] { xmoe::scatter_combine(gr, {0, 1, 5}, {1, 1, 1}, 3); }));
        CHECK(throws<xmoe::DimensionError>([&] { xmoe::scatter_combine(gr, {0, 1}, {1, 1}, 3); }));
    }
    // ---------------- operator-by-operator against the reference (random)
    {
        Rng rng(11);
        for (int trial = 0; trial < 20; ++trial) {
            const std::size_t S = 1 + rng.below(64);
            const std::int64_t E = 2 + rng.below(30), k = 1 + rng.below(std::min<std::int64_t>(E, 6));
            const std::int64_t H = 1 + rng.below(40), F = 1 + rng.below(24);
            moesim::Matrix x(S, H);
            for (auto& v : x.data) v = rng.uniform(-1.0, 1.0);
            const auto w = moesim::make_layer_weights(rng, E, H, F);
            const auto gr = moesim::gate_forward(x, w.gate, k);
            const auto gx = xmoe::gate_forward(X(x), X(w.gate), k);
            CHECK(gr.top_experts == gx.top_experts);
            CHECK(rel(gr.combine_weights, gx.combine_weights) < 1e-15);
            const std::int64_t cap = 1 + rng.below(S * k + 2);
            const auto pr = moesim::pft_construct(cap, E, gr);
            // the reference's own weights into the device PFT: bit-exact integer outputs
            const auto px = xmoe::pft_construct(cap, E, S, k, gr.top_experts, gr.combine_weights);
            CHECK(pr.token_ids == px.token_ids && pr.expert_ids == px.expert_ids &&
                  pr.tokens_per_expert == px.tokens_per_expert && pr.combine_weights == px.combine_weights);
            const auto xr = moesim::gather_rows(x, pr.token_ids);
            const auto xx = xmoe::gather_rows(X(x), px.token_ids);
            CHECK(xr.data == xx.data);
            const auto yr = moesim::grouped_expert_mlp(xr, pr.tokens_per_expert, w, 0);
            const auto yx = xmoe::grouped_expert_mlp(xx, px.tokens_per_expert, X(w), 0);
            CHECK(yr.data == yx.data);  // ascending-k fp64, no FMA: bit-exact
            const auto cr = moesim::scatter_combine(yr, pr.token_ids, pr.combine_weights, S);
            const auto cx = xmoe::scatter_combine(yx, px.token_ids, px.combine_weights, S);
            CHECK(cr.data == cx.data);
        }
    }
    // ---------------- whole layers: pf / rbd (one GPU per node) / ssmb
    {
        Rng rng(1717);
        for (int trial = 0; trial < 12; ++trial) {
            const std::size_t W = 1u << rng.below(4);  // 1, 2, 4, 8
            moesim::MoeInstance inst;
            inst.num_experts = static_cast<std::int64_t>(W) * (1 + rng.below(4));
            inst.top_k = 1 + rng.below(std::min<std::int64_t>(inst.num_experts, 4));
            const std::int64_t H = 2 + rng.below(12), F = 2 + rng.below(12);
            inst.weights = moesim::make_layer_weights(rng, inst.num_experts, H, F);
            const std::size_t S = 2 + rng.below(40);
            inst.max_token_count = (trial % 2) ? 1 + rng.below(4) : static_cast<std::int64_t>(S) * inst.top_k;
            for (std::size_t w = 0; w < W; ++w) {
                moesim::Matrix x(S, H);
                for (auto& v : x.data) v = rng.uniform(-1.0, 1.0);
                inst.tokens.push_back(std::move(x));
            }
            xmoe::MoeInstance xi;
            for (const auto& t : inst.tokens) xi.tokens.push_back(X(t));
            xi.weights = X(inst.weights);
            xi.num_experts = inst.num_experts;
            xi.top_k = inst.top_k;
            xi.max_token_count = inst.max_token_count;
            moesim::Comm rc;
            xmoe::Comm xc;
            for (std::size_t w = 0; w < W; ++w) {
                rc.group.node_of.push_back(static_cast<std::int64_t>(w));
                xc.group.node_of.push_back(static_cast<std::int64_t>(w));
            }
            const auto a = moesim::pf_moe_forward(inst, rc);
            const auto b = xmoe::pf_moe_forward(xi, xc);
            for (std::size_t w = 0; w < W; ++w) CHECK(rel(a[w].data, b[w].data) < 1e-14);
            const std::uint64_t seed = rng.next_u64();
            const auto c = moesim::rbd_moe_forward(inst, rc, seed);
            const auto d = xmoe::rbd_moe_forward(xi, xc, seed);
            for (std::size_t w = 0; w < W; ++w) CHECK(rel(c[w].data, d[w].data) < 1e-14);
            if (W % 2 == 0) {  // two-tier bypass: nodes of 2 GPUs
                moesim::Comm r2;
                xmoe::Comm x2;
                for (std::size_t w = 0; w < W; ++w) {
                    r2.group.node_of.push_back(static_cast<std::int64_t>(w / 2));
                    x2.group.node_of.push_back(static_cast<std::int64_t>(w / 2));
                }
                const auto c2 = moesim::rbd_moe_forward(inst, r2, seed);
                const auto d2 = xmoe::rbd_moe_forward(xi, x2, seed);
                for (std::size_t w = 0; w < W; ++w) CHECK(rel(c2[w].data, d2[w].data) < 1e-14);
            }
            if (W >= 2 && static_cast<std::size_t>(W) <= S) {
                moesim::Comm sc;
                xmoe::Comm sx;
                for (std::size_t g = 0; g < W; ++g) {
                    sc.group.node_of.push_back(g / 2);
                    sx.group.node_of.push_back(g);
                }
                const auto e = moesim::ssmb_forward(inst.tokens[0], W, inst.weights, inst.num_experts,
                                                    inst.top_k, inst.max_token_count, sc);
                const auto f = xmoe::ssmb_forward(xi.tokens[0], W, xi.weights, xi.num_experts, xi.top_k,
                                                  xi.max_token_count, sx);
                CHECK(rel(e.data, f.data) < 1e-14);
            }
        }
    }
    std::printf("compat_vs_ref: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
