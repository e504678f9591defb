// Reference-shaped C++ API (include/xmoe/moesim_compat.hpp) over the C-ABI.
// The operators come from compat_impl.inc (shared with the drop-in build of
// the reference's own acceptance suite, tests/cpp/dropin.cpp); this file adds
// what the reference keeps outside the hot path and the drop-in build takes
// from the reference itself: the generator, the cost ledger and its charge,
// the weight initialiser and the matrix metrics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>

#include "xmoe/moesim_compat.hpp"
#include "xmoe/xmoe.h"

namespace xmoe {

#include "compat_impl.inc"

// ---------------------------------------------------------------- matrix.hpp:33-62
double max_abs_diff(const Matrix& a, const Matrix& b) {
    if (!a.same_shape(b)) throw DimensionError("max_abs_diff: shape mismatch");
    double m = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::abs(a.data[i] - b.data[i]));
    return m;
}

double max_rel_diff(const Matrix& a, const Matrix& b) {
    if (!a.same_shape(b)) throw DimensionError("max_rel_diff: shape mismatch");
    double m = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i) {
        const double den = std::max({std::abs(a.data[i]), std::abs(b.data[i]), 1.0});
        m = std::max(m, std::abs(a.data[i] - b.data[i]) / den);
    }
    return m;
}

// ---------------------------------------------------------------- rng.hpp:8-61
std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

std::uint64_t salt_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b) { return xmoe_salt_seed(seed, a, b); }

Rng::Rng(std::uint64_t seed) {
    std::uint64_t x = seed;
    for (auto& w : s) w = x = splitmix64(x);
}

std::uint64_t Rng::next_u64() {
    const auto rotl = [](std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); };
    const std::uint64_t out = rotl(s[1] * 5, 7) * 9;
    const std::uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

std::uint64_t Rng::below(std::uint64_t n) {
    const std::uint64_t limit = ~0ULL - (~0ULL % n + 1) % n;  // reject the top partial bucket
    std::uint64_t x;
    do x = next_u64();
    while (x > limit);
    return x % n;
}

void Rng::advance(std::uint64_t n) {
    if (xmoe_rng_advance(s, n) != XMOE_OK) throw std::runtime_error(std::string("xmoe: ") + xmoe_last_error());
}

// make_layer_weights (padded_pipeline.cpp:13-27) drawn on the device from the
// caller's generator state, which then advances past every draw.
MoeLayerWeights make_layer_weights(Rng& rng, std::int64_t E, std::int64_t H, std::int64_t F) {
    using namespace compat_detail;
    MoeLayerWeights w;
    const std::uint64_t he = static_cast<std::uint64_t>(H) * E, hf = static_cast<std::uint64_t>(H) * F;
    const std::uint64_t total = he + 2 * hf * static_cast<std::uint64_t>(E);
    DBuf d(total * sizeof(double) + 8);
    ck(xmoe_rng_uniform_state(ctx_for(1), rng.s, 0, static_cast<std::int64_t>(total), -0.1, 0.1, 0.0, XMOE_F64, d.p,
                              nullptr));
    std::vector<double> h(total);
    d.down(h.data(), total * sizeof(double));
    w.gate = Matrix(H, E);
    std::copy_n(h.begin(), he, w.gate.data.begin());
    for (std::int64_t e = 0; e < E; ++e) {
        Matrix a(H, F), b(F, H);
        std::copy_n(h.begin() + he + 2 * hf * e, hf, a.data.begin());
        std::copy_n(h.begin() + he + 2 * hf * e + hf, hf, b.data.begin());
        w.w1.push_back(std::move(a));
        w.w2.push_back(std::move(b));
    }
    rng.advance(total);
    return w;
}

// ---------------------------------------------------------------- collectives.cpp:12-202
LedgerTotals CostLedger::totals(std::string_view prefix) const {
    LedgerTotals t;
    for (const auto& e : entries_) {
        if (e.kind.compare(0, prefix.size(), prefix) != 0) continue;
        t.self_bytes += e.self_bytes;
        t.intra_bytes += e.intra_bytes;
        t.inter_bytes += e.inter_bytes;
        t.intra_msgs += e.intra_msgs;
        t.inter_msgs += e.inter_msgs;
        t.time_s += e.time_s;
    }
    return t;
}

void CostLedger::write_csv(std::ostream& out) const {
    out << "collective_id,kind,intra_bytes,inter_bytes,modeled_time_s\n";
    for (const auto& e : entries_) {
        char tb[64];
        std::snprintf(tb, sizeof tb, "%.12g", e.time_s);
        out << e.id << ',' << e.kind << ',' << e.intra_bytes << ',' << e.inter_bytes << ',' << tb << '\n';
    }
}

namespace {
void check_square(const CountMatrix& m, size_t w, const char* who) {
    if (m.size() != w) throw DimensionError(std::string(who) + ": counts must be W x W");
    for (const auto& r : m) {
        if (r.size() != w) throw DimensionError(std::string(who) + ": counts must be W x W");
        for (auto v : r)
            if (v < 0) throw ValidationError(std::string(who) + ": counts must be >= 0");
    }
}
}  // namespace

CountMatrix alltoall_counts(const CountMatrix& counts) {
    const size_t w = counts.size();
    check_square(counts, w, "alltoall_counts");
    CountMatrix t(w, std::vector<std::int64_t>(w, 0));
    for (size_t i = 0; i < w; ++i)
        for (size_t j = 0; j < w; ++j) t[j][i] = counts[i][j];
    return t;
}

// self / intra-node / inter-node classes by node_of; each sender pays
// latency + bytes / bandwidth per message; the collective takes the slowest
void charge_bytes(Comm& comm, const CountMatrix& bytes, std::string kind) {
    const size_t w = comm.group.size();
    check_square(bytes, w, "charge_bytes");
    if (!comm.ledger) return;
    LedgerEntry& e = comm.ledger->add(std::move(kind));
    std::vector<double> busy(w, 0.0);
    for (size_t i = 0; i < w; ++i)
        for (size_t j = 0; j < w; ++j) {
            const std::int64_t b = bytes[i][j];
            if (b <= 0) continue;
            const auto ub = static_cast<std::uint64_t>(b);
            if (i == j) {
                e.self_bytes += ub;
            } else if (comm.group.node_of[i] == comm.group.node_of[j]) {
                e.intra_bytes += ub;
                e.intra_msgs += 1;
                busy[i] += comm.topo.latency_intra + static_cast<double>(ub) / comm.topo.bw_intra;
            } else {
                e.inter_bytes += ub;
                e.inter_msgs += 1;
                busy[i] += comm.topo.latency_inter + static_cast<double>(ub) / comm.topo.bw_inter;
            }
        }
    e.time_s = busy.empty() ? 0.0 : *std::max_element(busy.begin(), busy.end());
}

}  // namespace xmoe
