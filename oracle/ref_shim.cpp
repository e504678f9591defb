// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Flat extern "C" entry points over the UNMODIFIED reference simulator
// (`/root/reference/proj/src/*.cpp`, compiled where it lies by
// oracle/Makefile into oracle/_ref/libmoesim_ref.so).  Only tests/, the
// smoke check and bench.py's cpu_baseline / --impl reference arm load it.
//
// Every function copies flat arrays into the reference's value types, calls the
// reference operator and copies the result back out; exceptions become status
// codes with the same numbering the product C-ABI uses (include/xmoe/xmoe.h):
//   1 ParseError 2 ValidationError 3 DimensionError 4 IndexError
//   5 CountMismatch 6 PlanMismatch 99 other.
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "moesim/collectives.hpp"
#include "moesim/error.hpp"
#include "moesim/gating.hpp"
#include "moesim/kernels.hpp"
#include "moesim/moe_instance.hpp"
#include "moesim/padded_pipeline.hpp"
#include "moesim/pf_pipeline.hpp"
#include "moesim/pft.hpp"
#include "moesim/rbd.hpp"
#include "moesim/rng.hpp"
#include "moesim/ssmb.hpp"

using namespace moesim;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 2;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 3;
    } catch (const IndexError& e) {
        g_err = e.what();
        return 4;
    } catch (const CountMismatch& e) {
        g_err = e.what();
        return 5;
    } catch (const PlanMismatch& e) {
        g_err = e.what();
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

Matrix to_matrix(const double* p, std::int64_t r, std::int64_t c) {
    Matrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));
    if (r * c > 0) std::memcpy(m.data.data(), p, sizeof(double) * r * c);
    return m;
}

void from_matrix(const Matrix& m, double* out) {
    if (!m.data.empty()) std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
}

struct Layer {
    MoeLayerWeights w;
    std::int64_t E = 0, H = 0, F = 0;
};

Comm make_comm(std::int64_t W, const std::int64_t* node_of, CostLedger* ledger) {
    Comm c;
    c.group.node_of.assign(node_of, node_of + W);
    c.topo = Topology{};
    c.dtype_bytes = 2;
    c.ledger = ledger;
    return c;
}

MoeInstance make_inst(const Layer& L, std::int64_t W, const double* tokens, std::int64_t S,
                      std::int64_t k, std::int64_t cap) {
    MoeInstance inst;
    inst.weights = L.w;
    inst.num_experts = L.E;
    inst.top_k = k;
    inst.max_token_count = cap;
    for (std::int64_t w = 0; w < W; ++w) inst.tokens.push_back(to_matrix(tokens + w * S * L.H, S, L.H));
    return inst;
}

// Ledger kinds reported by ref_*_forward, in this order, 3 words each
// (self, intra, inter bytes).
const char* const kKinds[] = {"dispatch_counts",    "dispatch_rows",      "combine_rows",
                              "rbd_dispatch_counts", "rbd_dispatch_meta",  "rbd_dispatch_rows1",
                              "rbd_dispatch_meta2", "rbd_dispatch_rows2", "rbd_combine_rows2",
                              "rbd_combine_rows1",  "ssmb_gather_rows"};
constexpr int kNumKinds = sizeof(kKinds) / sizeof(kKinds[0]);

// The last forward's ledger in CostLedger::write_csv's format
// (collectives.cpp:26-34), formatted here from led.entries() with the same
// "%.12g": the reference's ostream writer is not called across the
// libstdc++ the host process loads.
std::string g_last_csv;

void dump_ledger(const CostLedger& led, std::uint64_t* out) {
    g_last_csv = "collective_id,kind,intra_bytes,inter_bytes,modeled_time_s\n";
    char buf[64];
    for (const auto& e : led.entries()) {
        std::snprintf(buf, sizeof buf, "%.12g", e.time_s);
        g_last_csv += std::to_string(e.id) + ',' + e.kind + ',' + std::to_string(e.intra_bytes) + ',' +
                      std::to_string(e.inter_bytes) + ',' + buf + '\n';
    }
    if (!out) return;
    for (int i = 0; i < kNumKinds; ++i) {
        std::uint64_t s = 0, a = 0, r = 0;
        for (const auto& e : led.entries())
            if (e.kind == kKinds[i]) {
                s += e.self_bytes;
                a += e.intra_bytes;
                r += e.inter_bytes;
            }
        out[3 * i + 0] = s;
        out[3 * i + 1] = a;
        out[3 * i + 2] = r;
    }
}

std::vector<Pft> build_pfts(const MoeInstance& inst) {
    std::vector<Pft> pfts;
    for (const auto& tk : inst.tokens) {
        const auto g = gate_forward(tk, inst.weights.gate, inst.top_k);
        auto p = pft_construct(inst.max_token_count, inst.num_experts, g);
        p.x = gather_rows(tk, p.token_ids);
        pfts.push_back(std::move(p));
    }
    return pfts;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
const char* ref_last_ledger_csv(void) { return g_last_csv.c_str(); }
int ref_num_ledger_kinds(void) { return kNumKinds; }
const char* ref_ledger_kind(int i) { return (i >= 0 && i < kNumKinds) ? kKinds[i] : ""; }
const char* ref_kernel_backend(void) { return kernels::active().name; }

std::uint64_t ref_salt_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b) {
    return salt_seed(seed, a, b);
}

void ref_rng_u64(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

void ref_rng_uniform(std::uint64_t seed, std::int64_t n, double lo, double hi, double* out) {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}

std::int64_t ref_rng_below_seq(std::uint64_t seed, std::int64_t n, const std::uint64_t* bounds,
                               std::uint64_t* out) {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.below(bounds[i]);
    return n;
}

// gate [H,E], w1 [E,H,F], w2 [E,F,H] in make_layer_weights draw order.
void ref_make_layer_weights(std::uint64_t seed, std::int64_t E, std::int64_t H, std::int64_t F,
                            double* gate, double* w1, double* w2) {
    Rng r(seed);
    const auto w = make_layer_weights(r, E, H, F);
    from_matrix(w.gate, gate);
    for (std::int64_t e = 0; e < E; ++e) {
        from_matrix(w.w1[e], w1 + e * H * F);
        from_matrix(w.w2[e], w2 + e * F * H);
    }
}

int ref_gate_forward(const double* x, const double* wg, std::int64_t S, std::int64_t H,
                     std::int64_t Hg, std::int64_t E, std::int64_t k, std::int64_t* top,
                     double* w) {
    return guarded([&] {
        const auto g = gate_forward(to_matrix(x, S, H), to_matrix(wg, Hg, E), k);
        std::memcpy(top, g.top_experts.data(), sizeof(std::int64_t) * g.top_experts.size());
        std::memcpy(w, g.combine_weights.data(), sizeof(double) * g.combine_weights.size());
    });
}

int ref_pft_construct(std::int64_t cap, std::int64_t E, std::int64_t S, std::int64_t k,
                      std::int64_t flat_len, const std::int64_t* top, const double* w,
                      std::int64_t* token_ids, std::int64_t* expert_ids, double* cw,
                      std::int64_t* tpe, std::int64_t* B) {
    return guarded([&] {
        std::vector<std::int64_t> t(top, top + flat_len);
        std::vector<double> ww(w, w + flat_len);
        const auto p = pft_construct(cap, E, static_cast<std::size_t>(S), k, t, ww);
        *B = static_cast<std::int64_t>(p.size());
        std::memcpy(token_ids, p.token_ids.data(), sizeof(std::int64_t) * p.size());
        std::memcpy(expert_ids, p.expert_ids.data(), sizeof(std::int64_t) * p.size());
        std::memcpy(cw, p.combine_weights.data(), sizeof(double) * p.size());
        std::memcpy(tpe, p.tokens_per_expert.data(), sizeof(std::int64_t) * E);
    });
}

int ref_gather_rows(const double* src, std::int64_t rows, std::int64_t cols,
                    const std::int64_t* ids, std::int64_t n, double* out) {
    return guarded([&] {
        std::vector<std::int64_t> v(ids, ids + n);
        from_matrix(gather_rows(to_matrix(src, rows, cols), v), out);
    });
}

int ref_scatter_combine(const double* rows, std::int64_t n, std::int64_t cols,
                        const std::int64_t* token_ids, std::int64_t n_ids, const double* w,
                        std::int64_t n_w, std::int64_t S, double* out) {
    return guarded([&] {
        std::vector<std::int64_t> t(token_ids, token_ids + n_ids);
        std::vector<double> ww(w, w + n_w);
        from_matrix(scatter_combine(to_matrix(rows, n, cols), t, ww, static_cast<std::size_t>(S)),
                    out);
    });
}

void* ref_layer_create(std::int64_t E, std::int64_t H, std::int64_t F, const double* gate,
                       const double* w1, const double* w2) {
    auto* L = new Layer;
    L->E = E;
    L->H = H;
    L->F = F;
    L->w.gate = to_matrix(gate, H, E);
    for (std::int64_t e = 0; e < E; ++e) {
        L->w.w1.push_back(to_matrix(w1 + e * H * F, H, F));
        L->w.w2.push_back(to_matrix(w2 + e * F * H, F, H));
    }
    return L;
}

void ref_layer_destroy(void* p) { delete static_cast<Layer*>(p); }

int ref_grouped_expert_mlp(void* layer, const double* in, std::int64_t rows,
                           const std::int64_t* rpe, std::int64_t n_groups,
                           std::int64_t first_expert, double* out) {
    return guarded([&] {
        const auto& L = *static_cast<Layer*>(layer);
        std::vector<std::int64_t> r(rpe, rpe + n_groups);
        from_matrix(grouped_expert_mlp(to_matrix(in, rows, L.H), r, L.w, first_expert), out);
    });
}

// tokens/out: [W, S, H].  ledger: 3 * ref_num_ledger_kinds() words or null.
int ref_pf_moe_forward(void* layer, std::int64_t W, const std::int64_t* node_of,
                       const double* tokens, std::int64_t S, std::int64_t k, std::int64_t cap,
                       double* out, std::uint64_t* ledger) {
    return guarded([&] {
        const auto& L = *static_cast<Layer*>(layer);
        CostLedger led;
        auto comm = make_comm(W, node_of, &led);
        const auto inst = make_inst(L, W, tokens, S, k, cap);
        const auto res = pf_moe_forward(inst, comm);
        for (std::int64_t w = 0; w < W; ++w) from_matrix(res[w], out + w * S * L.H);
        dump_ledger(led, ledger);
    });
}

// The same composition as moesim::pf_moe_forward (pf_pipeline.cpp:137-169),
// step for step through the reference's own gate_forward / pft_construct /
// gather_rows / pf_dispatch / grouped_expert_mlp / pf_combine, but with the
// layer's weights by const reference: the MoeInstance above holds its
// MoeLayerWeights by value, so every call through it first copies all of
// them (2.9 GB of fp64 at C2) — shim overhead, not reference work, which
// dominated small per-thread samples of the CPU baseline.  Identical output
// (tests/test_oracle.py).
int ref_pf_moe_forward_noncopy(void* layer, std::int64_t W, const std::int64_t* node_of,
                               const double* tokens, std::int64_t S, std::int64_t k, std::int64_t cap,
                               double* out) {
    return guarded([&] {
        const auto& L = *static_cast<Layer*>(layer);
        auto comm = make_comm(W, node_of, nullptr);
        const std::int64_t E = L.E;
        if (E % W != 0) throw ValidationError("num_experts must be divisible by the worker-group size");
        const std::int64_t e_local = E / W;
        std::vector<Matrix> toks;
        for (std::int64_t w = 0; w < W; ++w) toks.push_back(to_matrix(tokens + w * S * L.H, S, L.H));
        std::vector<Pft> pfts(static_cast<std::size_t>(W));
        for (std::int64_t w = 0; w < W; ++w) {
            const auto gate = gate_forward(toks[w], L.w.gate, k);
            pfts[w] = pft_construct(cap, E, gate);
            pfts[w].x = gather_rows(toks[w], pfts[w].token_ids);
        }
        auto disp = pf_dispatch(comm, pfts, E);
        std::vector<Matrix> expert_out(static_cast<std::size_t>(W));
        std::vector<std::size_t> seq_lens(static_cast<std::size_t>(W));
        for (std::int64_t w = 0; w < W; ++w) {
            expert_out[w] = grouped_expert_mlp(disp.expert_input[w], disp.recv_per_expert[w], L.w, w * e_local);
            seq_lens[w] = toks[w].rows;
        }
        const auto res = pf_combine(comm, disp, expert_out, pfts, seq_lens);
        for (std::int64_t w = 0; w < W; ++w) from_matrix(res[w], out + w * S * L.H);
    });
}

int ref_rbd_moe_forward(void* layer, std::int64_t W, const std::int64_t* node_of,
                        const double* tokens, std::int64_t S, std::int64_t k, std::int64_t cap,
                        std::uint64_t seed, double* out, std::uint64_t* ledger) {
    return guarded([&] {
        const auto& L = *static_cast<Layer*>(layer);
        CostLedger led;
        auto comm = make_comm(W, node_of, &led);
        const auto inst = make_inst(L, W, tokens, S, k, cap);
        const auto res = rbd_moe_forward(inst, comm, seed);
        for (std::int64_t w = 0; w < W; ++w) from_matrix(res[w], out + w * S * L.H);
        dump_ledger(led, ledger);
    });
}

int ref_padded_moe_forward(void* layer, std::int64_t W, const std::int64_t* node_of,
                           const double* tokens, std::int64_t S, std::int64_t k,
                           std::int64_t cap, double* out) {
    return guarded([&] {
        const auto& L = *static_cast<Layer*>(layer);
        CostLedger led;
        auto comm = make_comm(W, node_of, &led);
        const auto inst = make_inst(L, W, tokens, S, k, cap);
        const auto res = padded_moe_forward(inst, comm);
        for (std::int64_t w = 0; w < W; ++w) from_matrix(res[w], out + w * S * L.H);
        dump_ledger(led, nullptr);
    });
}

// Dispatch-level view: gate + PFT + gather per worker, then pf_dispatch (or
// rbd_dispatch with per-worker salt_seed(seed, w, 0) when rbd != 0).
// expert_input: per worker n_w rows concatenated (caller sizes it W*S*k*H);
// rows_out[w] = n_w; recv_per_expert [W, E/W]; row_counts [W, W] (s1 counts
// for rbd); pilot_mask: per worker B_w bytes concatenated (rbd only).
int ref_dispatch(void* layer, std::int64_t W, const std::int64_t* node_of, const double* tokens,
                 std::int64_t S, std::int64_t k, std::int64_t cap, int rbd, std::uint64_t seed,
                 double* expert_input, std::int64_t* rows_out, std::int64_t* recv_per_expert,
                 std::int64_t* row_counts, std::uint8_t* pilot_mask, std::uint64_t* ledger) {
    return guarded([&] {
        const auto& L = *static_cast<Layer*>(layer);
        CostLedger led;
        auto comm = make_comm(W, node_of, &led);
        const auto inst = make_inst(L, W, tokens, S, k, cap);
        const auto pfts = build_pfts(inst);
        std::vector<Matrix> ei;
        std::vector<std::vector<std::int64_t>> rpe;
        CountMatrix counts;
        if (rbd) {
            std::vector<RbdPlan> plans;
            for (std::int64_t w = 0; w < W; ++w)
                plans.push_back(select_pilots(pfts[w], comm.group, L.E, salt_seed(seed, w, 0)));
            auto d = rbd_dispatch(comm, pfts, plans, L.E);
            ei = std::move(d.expert_input);
            rpe = std::move(d.recv_per_expert);
            counts = std::move(d.s1_counts);
            std::size_t off = 0;
            for (const auto& pl : plans) {
                if (pilot_mask) std::memcpy(pilot_mask + off, pl.pilot_mask.data(), pl.pilot_mask.size());
                off += pl.pilot_mask.size();
            }
        } else {
            auto d = pf_dispatch(comm, pfts, L.E);
            ei = std::move(d.expert_input);
            rpe = std::move(d.recv_per_expert);
            counts = std::move(d.row_counts);
        }
        const std::int64_t el = L.E / W;
        std::size_t off = 0;
        for (std::int64_t w = 0; w < W; ++w) {
            from_matrix(ei[w], expert_input + off);
            off += ei[w].data.size();
            rows_out[w] = static_cast<std::int64_t>(ei[w].rows);
            for (std::int64_t le = 0; le < el; ++le) recv_per_expert[w * el + le] = rpe[w][le];
            for (std::int64_t j = 0; j < W; ++j) row_counts[w * W + j] = counts[w][j];
        }
        dump_ledger(led, ledger);
    });
}

// select_pilots over a caller-provided packed buffer's ERI arrays.
int ref_select_pilots(std::int64_t B, const std::int64_t* token_ids, const std::int64_t* expert_ids,
                      const double* cw, const std::int64_t* tpe, std::int64_t E, std::int64_t W,
                      const std::int64_t* node_of, std::uint64_t seed, std::uint8_t* pilot_mask) {
    return guarded([&] {
        Pft p;
        p.token_ids.assign(token_ids, token_ids + B);
        p.expert_ids.assign(expert_ids, expert_ids + B);
        p.combine_weights.assign(cw, cw + B);
        p.tokens_per_expert.assign(tpe, tpe + E);
        WorkerGroup g;
        g.node_of.assign(node_of, node_of + W);
        const auto plan = select_pilots(p, g, E, seed);
        std::memcpy(pilot_mask, plan.pilot_mask.data(), plan.pilot_mask.size());
    });
}

int ref_ssmb_forward(void* layer, std::int64_t G, const std::int64_t* node_of,
                     const double* tokens, std::int64_t S, std::int64_t k, std::int64_t cap,
                     double* out, std::uint64_t* ledger) {
    return guarded([&] {
        const auto& L = *static_cast<Layer*>(layer);
        CostLedger led;
        auto comm = make_comm(G, node_of, &led);
        const auto res =
            ssmb_forward(to_matrix(tokens, S, L.H), G, L.w, L.E, k, cap, comm, nullptr);
        from_matrix(res, out);
        dump_ledger(led, ledger);
    });
}

double ref_sample_redundancy(std::uint64_t seed, std::int64_t tokens, std::int64_t k,
                             std::int64_t E, const std::int64_t* expert_node) {
    Rng r(seed);
    std::vector<std::int64_t> nodes(expert_node, expert_node + E);
    return sample_redundancy(r, static_cast<std::size_t>(tokens), k, nodes);
}

}  // extern "C"
