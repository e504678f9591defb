// Reference-shaped C++ host API over the xmoe C-ABI.
//
// Same types, names, argument meaning, value semantics and exception types as
// the reference simulator's operator API (namespace moesim,
// /root/reference/proj/include/moesim/*.hpp), re-homed in namespace xmoe:
// a caller of the reference switches by changing the namespace (or with
// `namespace moesim = xmoe;`).  Every call runs on the B200 in the F64
// parity instantiation (the reference's arithmetic order), with inputs
// uploaded and outputs downloaded around the device operators; the BF16
// performance path is the xmoe_layer C-ABI (include/xmoe/xmoe.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
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

// ---- matrix.hpp:15-30
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
};

// ---- placement.hpp:51-54 / collectives.hpp:71-76 (node_of: contiguous
// blocks of equal size; rbd_moe_forward runs the two-tier bypass when a block
// holds several GPUs)
struct WorkerGroup {
    std::vector<std::int64_t> node_of;
    std::size_t size() const { return node_of.size(); }
};
struct Comm {
    WorkerGroup group;
    std::int64_t dtype_bytes = 2;
};

// ---- operators (device-backed)
GateOutput gate_forward(const Matrix& tokens, const Matrix& gate_weights, std::int64_t top_k);
Pft pft_construct(std::int64_t max_token_count, std::int64_t num_experts, std::size_t seq_len,
                  std::int64_t top_k, const std::vector<std::int64_t>& top_experts,
                  const std::vector<double>& combine_weights);
Pft pft_construct(std::int64_t max_token_count, std::int64_t num_experts, const GateOutput& gate);
Matrix gather_rows(const Matrix& src, const std::vector<std::int64_t>& ids);
Matrix scatter_combine(const Matrix& rows, const std::vector<std::int64_t>& token_ids,
                       const std::vector<double>& weights, std::size_t seq_len);
Matrix grouped_expert_mlp(const Matrix& input, const std::vector<std::int64_t>& rows_per_expert,
                          const MoeLayerWeights& weights, std::int64_t first_expert);
std::vector<Matrix> pf_moe_forward(const MoeInstance& inst, Comm& comm,
                                   ActivationCounters* counters = nullptr);
std::vector<Matrix> rbd_moe_forward(const MoeInstance& inst, Comm& comm, std::uint64_t seed);
Matrix ssmb_forward(const Matrix& tokens, std::int64_t G, const MoeLayerWeights& weights,
                    std::int64_t num_experts, std::int64_t top_k, std::int64_t max_token_count,
                    Comm& comm, ActivationCounters* counters = nullptr);

}  // namespace xmoe
