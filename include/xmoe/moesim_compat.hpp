// Reference-shaped C++ host API over the xmoe C-ABI.
//
// Same types, names, argument meaning, value semantics and exception types as
// the reference simulator's operator API (namespace moesim,
// /root/reference/proj/include/moesim/*.hpp), re-homed in namespace xmoe:
// a caller of the reference switches by changing the namespace (or with
// `namespace moesim = xmoe;`).  Every operator runs on the B200 in the F64
// parity instantiation (the reference's arithmetic order), inputs uploaded
// and outputs downloaded around the device calls; the BF16 performance path
// is the xmoe_layer C-ABI (include/xmoe/xmoe.h).
//
// The implementations live in csrc/compat_impl.inc, which is compiled twice:
// here (namespace xmoe, these types) and, for the drop-in check, inside
// namespace moesim against the reference's own headers (tests/cpp/dropin.cpp),
// so the reference's acceptance suite runs unchanged on the GPU path.
#pragma once

#include <cstddef>
#include <cstdint>
#include <ostream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace xmoe {

// ---- error.hpp:10-38
struct ParseError : std::runtime_error {
    explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};
struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct DimensionError : std::runtime_error {
    explicit DimensionError(const std::string& m) : std::runtime_error(m) {}
};
struct IndexError : std::runtime_error {
    explicit IndexError(const std::string& m) : std::runtime_error(m) {}
};
struct CountMismatch : std::runtime_error {
    explicit CountMismatch(const std::string& m) : std::runtime_error(m) {}
};
struct PlanMismatch : std::runtime_error {
    explicit PlanMismatch(const std::string& m) : std::runtime_error(m) {}
};

// ---- matrix.hpp:15-62
struct Matrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<double> data;
    Matrix() = default;
    Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
    double* row(std::size_t i) { return data.data() + i * cols; }
    const double* row(std::size_t i) const { return data.data() + i * cols; }
    double& at(std::size_t i, std::size_t j) { return data[i * cols + j]; }
    double at(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
    bool same_shape(const Matrix& o) const { return rows == o.rows && cols == o.cols; }
};
double max_abs_diff(const Matrix& a, const Matrix& b);
// |a - b| / max(|a|, |b|, 1) elementwise, maximum over the matrix
double max_rel_diff(const Matrix& a, const Matrix& b);

// ---- rng.hpp:8-61 (state public: the device generator continues it)
std::uint64_t splitmix64(std::uint64_t x);
std::uint64_t salt_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b = 0);
class Rng {
  public:
    explicit Rng(std::uint64_t seed);
    std::uint64_t next_u64();
    double uniform();
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    std::uint64_t below(std::uint64_t n);
    // jump the stream forward by n outputs (GF(2) powers of one step)
    void advance(std::uint64_t n);
    std::uint64_t s[4];
};

// ---- config.hpp:30-40 (the fields the collectives read)
struct Topology {
    std::int64_t num_nodes = 1;
    std::int64_t gpus_per_node = 8;
    double bw_intra = 200e9;
    double bw_inter = 25e9;
    double latency_intra = 0.0;
    double latency_inter = 0.0;
    std::int64_t workers() const { return num_nodes * gpus_per_node; }
    std::int64_t node_of(std::int64_t w) const { return w / gpus_per_node; }
};

// ---- gating.hpp:15-32
struct GateOutput {
    std::vector<std::int64_t> top_experts;
    std::vector<double> combine_weights;
    Matrix gate_out;
    std::int64_t top_k = 0;
    std::int64_t expert_at(std::size_t t, std::int64_t s) const { return top_experts[t * top_k + s]; }
    double weight_at(std::size_t t, std::int64_t s) const { return combine_weights[t * top_k + s]; }
};

// ---- pft.hpp:17-25
struct Pft {
    Matrix x;
    std::vector<std::int64_t> token_ids;
    std::vector<std::int64_t> expert_ids;
    std::vector<std::int64_t> tokens_per_expert;
    std::vector<double> combine_weights;
    std::size_t size() const { return token_ids.size(); }
};

// ---- moe_instance.hpp:17-46
struct MoeLayerWeights {
    Matrix gate;             // [H, E]
    std::vector<Matrix> w1;  // per expert [H, F]
    std::vector<Matrix> w2;  // per expert [F, H]
};
struct MoeInstance {
    std::vector<Matrix> tokens;  // per group-rank [S_w, H]
    MoeLayerWeights weights;
    std::int64_t num_experts = 0;
    std::int64_t top_k = 1;
    std::int64_t max_token_count = 1;
};
struct ActivationCounters {
    std::vector<std::uint64_t> dispatch_in_elements;
    std::vector<std::uint64_t> dispatch_out_elements;
    std::uint64_t total() const {
        std::uint64_t t = 0;
        for (auto v : dispatch_in_elements) t += v;
        for (auto v : dispatch_out_elements) t += v;
        return t;
    }
};

// ---- placement.hpp:51-54, collectives.hpp:29-77
struct WorkerGroup {
    std::vector<std::int64_t> node_of;
    std::size_t size() const { return node_of.size(); }
};
using CountMatrix = std::vector<std::vector<std::int64_t>>;
struct LedgerEntry {
    std::int64_t id = 0;
    std::string kind;
    std::uint64_t self_bytes = 0;
    std::uint64_t intra_bytes = 0;
    std::uint64_t inter_bytes = 0;
    std::uint64_t intra_msgs = 0;
    std::uint64_t inter_msgs = 0;
    double time_s = 0.0;
};
struct LedgerTotals {
    std::uint64_t self_bytes = 0;
    std::uint64_t intra_bytes = 0;
    std::uint64_t inter_bytes = 0;
    std::uint64_t intra_msgs = 0;
    std::uint64_t inter_msgs = 0;
    double time_s = 0.0;
};
class CostLedger {
  public:
    LedgerEntry& add(std::string kind) {
        entries_.push_back(LedgerEntry{next_id_++, std::move(kind), 0, 0, 0, 0, 0, 0.0});
        return entries_.back();
    }
    const std::vector<LedgerEntry>& entries() const { return entries_; }
    LedgerTotals totals(std::string_view kind_prefix = {}) const;
    // collective_id,kind,intra_bytes,inter_bytes,modeled_time_s
    void write_csv(std::ostream& out) const;

  private:
    std::vector<LedgerEntry> entries_;
    std::int64_t next_id_ = 0;
};
struct Comm {
    WorkerGroup group;
    Topology topo;
    std::int64_t dtype_bytes = 2;
    CostLedger* ledger = nullptr;  // non-owning; null = no accounting
};
CountMatrix alltoall_counts(const CountMatrix& counts);
// prices an explicit [W, W] byte matrix under `kind` (no payload moves)
void charge_bytes(Comm& comm, const CountMatrix& bytes, std::string kind);
inline double serialized_time(const LedgerTotals& t, const Topology& topo) {
    return static_cast<double>(t.intra_bytes) / topo.bw_intra + static_cast<double>(t.inter_bytes) / topo.bw_inter;
}

// ---- pf_pipeline.hpp:18-29
struct PfDispatch {
    std::vector<Matrix> expert_input;  // per worker, (local expert, source, position) order
    std::vector<std::vector<std::int64_t>> recv_per_expert;
    CountMatrix row_counts;
    std::vector<std::vector<std::int64_t>> arrival_to_grouped;
};

// ---- rbd.hpp:28-71
struct RbdPlan {
    std::vector<std::uint8_t> pilot_mask;
    Pft pilots;
    Pft replicas;
    std::vector<std::int64_t> replica_pilot_seq;
    std::vector<std::int64_t> s1_mapping;
};
struct RbdDispatch {
    std::vector<Matrix> expert_input;
    std::vector<std::vector<std::int64_t>> recv_per_expert;
    CountMatrix s1_counts;
    CountMatrix s2_counts;
    std::vector<std::vector<std::int64_t>> landed_pos;
    std::vector<std::vector<double>> landed_weight;
    std::vector<std::vector<std::uint8_t>> landed_multi;
    std::vector<std::vector<std::vector<std::int64_t>>> s2_slot_pilot;
    std::vector<std::vector<std::vector<double>>> s2_slot_weight;
    std::vector<std::vector<std::vector<std::int64_t>>> s2_recv_pos;
    std::vector<std::vector<std::uint8_t>> source_pilot_multi;
};
struct RedundancyCounts {
    std::int64_t copies = 0;
    std::int64_t groups = 0;
};

// ---- operators (device-backed; csrc/compat_impl.inc)
GateOutput gate_forward(const Matrix& tokens, const Matrix& gate_weights, std::int64_t top_k);
Matrix make_gate_weights(Rng& rng, std::int64_t model_dim, std::int64_t num_experts);
MoeLayerWeights make_layer_weights(Rng& rng, std::int64_t num_experts, std::int64_t model_dim,
                                   std::int64_t ffn_dim);
Pft pft_construct(std::int64_t max_token_count, std::int64_t num_experts, std::size_t seq_len,
                  std::int64_t top_k, const std::vector<std::int64_t>& top_experts,
                  const std::vector<double>& combine_weights);
Pft pft_construct(std::int64_t max_token_count, std::int64_t num_experts, const GateOutput& gate);
Matrix gather_rows(const Matrix& src, const std::vector<std::int64_t>& ids);
Matrix scatter_combine(const Matrix& rows, const std::vector<std::int64_t>& token_ids,
                       const std::vector<double>& weights, std::size_t seq_len);
PfDispatch pf_dispatch(Comm& comm, const std::vector<Pft>& pfts, std::int64_t num_experts);
Matrix grouped_expert_mlp(const Matrix& input, const std::vector<std::int64_t>& rows_per_expert,
                          const MoeLayerWeights& weights, std::int64_t first_expert);
std::vector<Matrix> pf_combine(Comm& comm, const PfDispatch& dispatch, const std::vector<Matrix>& expert_out,
                               const std::vector<Pft>& pfts, const std::vector<std::size_t>& seq_lens);
std::vector<Matrix> pf_moe_forward(const MoeInstance& inst, Comm& comm,
                                   ActivationCounters* counters = nullptr);
std::vector<std::int64_t> expert_nodes(const WorkerGroup& group, std::int64_t num_experts);
RbdPlan select_pilots(const Pft& pft, const WorkerGroup& group, std::int64_t num_experts, std::uint64_t seed);
RbdDispatch rbd_dispatch(Comm& comm, const std::vector<Pft>& pfts, const std::vector<RbdPlan>& plans,
                         std::int64_t num_experts);
std::vector<Matrix> rbd_combine(Comm& comm, const RbdDispatch& dispatch, const std::vector<Matrix>& expert_out,
                                const std::vector<RbdPlan>& plans, const std::vector<std::size_t>& seq_lens);
std::vector<Matrix> rbd_moe_forward(const MoeInstance& inst, Comm& comm, std::uint64_t seed);
double redundancy_rate(const std::vector<std::int64_t>& top_experts, std::int64_t top_k,
                       const std::vector<std::int64_t>& expert_node);
double redundancy_rate(const Pft& pft, const std::vector<std::int64_t>& expert_node);
double redundancy_rate_internode(const Pft& pft, std::int64_t source_node,
                                 const std::vector<std::int64_t>& expert_node);
RedundancyCounts internode_redundancy_counts(const Pft& pft, std::int64_t source_node,
                                             const std::vector<std::int64_t>& expert_node);
double sample_redundancy(Rng& rng, std::size_t tokens, std::int64_t top_k,
                         const std::vector<std::int64_t>& expert_node);
Matrix ssmb_forward(const Matrix& tokens, std::int64_t G, const MoeLayerWeights& weights,
                    std::int64_t num_experts, std::int64_t top_k, std::int64_t max_token_count,
                    Comm& comm, ActivationCounters* counters = nullptr);

}  // namespace xmoe
