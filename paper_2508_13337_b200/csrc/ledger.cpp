// Byte ledger of the last layer forward — the measured counterpart of the
// reference's CostLedger (collectives.hpp:31-69, charge_message in
// collectives.cpp:45-76).  Self traffic stays on the GPU; off-rank traffic
// crosses NVLink.  Row bytes use the layer's real element size.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "layer.h"

namespace xmoe {

// the device ledger counters of worker w's last forward (rbd.cu layout)
std::vector<uint64_t> Layer::device_counts(const Worker& w, long long S, bool groups) {
    const int ncnt = 1 + 3 * W + W * W;
    if (!led_cnt) led_cnt = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * ncnt));
    launch_ledger_counts(w.slot_pos, static_cast<int>(S), k, w.expert_ids, El, w.rank, groups ? &w.rbd : nullptr, W,
                         led_cnt, nullptr);
    std::vector<uint64_t> h(ncnt, 0);
    XMOE_CUDA(cudaMemcpy(h.data(), led_cnt, sizeof(uint64_t) * ncnt, cudaMemcpyDeviceToHost));
    return h;
}

void Layer::ledger(uint64_t* out, int n) {
    std::vector<int32_t> tpe(static_cast<size_t>(W) * E);
    XMOE_CUDA(cudaDeviceSynchronize());
    XMOE_CUDA(cudaMemcpy(tpe.data(), tpe_all, sizeof(int32_t) * tpe.size(), cudaMemcpyDeviceToHost));
    const uint64_t rb = static_cast<uint64_t>(H) * es;
    uint64_t v[8] = {};
    for (const Worker& w : workers) {
        for (int e = 0; e < E; ++e) {
            const uint64_t c = static_cast<uint64_t>(tpe[static_cast<size_t>(w.rank) * E + e]);
            const bool self = (e / El) == w.rank;
            v[self ? 0 : 1] += c * rb;  // dispatch rows
            v[self ? 3 : 4] += c * rb;  // combine rows (transposed counts)
            v[5] += c;
            if (!self) v[7] += c;
        }
        if (W > 1) v[2] += static_cast<uint64_t>(W - 1) * E * sizeof(int32_t);  // count all-gather
        // distinct (token, destination rank) groups leaving the rank: the rows
        // the redundancy bypass sends (rbd.cpp:427-442 with node_of = rank),
        // counted on the device
        const long long S = last_Sw.empty() ? last_S : last_Sw[static_cast<size_t>(&w - workers.data())];
        v[6] += device_counts(w, S, false)[0];
    }
    if (d.dispatch_mode == XMOE_DISPATCH_RBD) {
        h_G.resize(static_cast<size_t>(W) * W);
        XMOE_CUDA(cudaMemcpy(h_G.data(), G_all, sizeof(int32_t) * h_G.size(), cudaMemcpyDeviceToHost));
        // bypass: one row per (token, destination) group each way, plus the
        // 24-byte copy descriptors (rbd.h RbdDesc)
        v[0] = v[1] = v[2] = v[3] = v[4] = 0;
        for (const Worker& w : workers) {
            for (int dd = 0; dd < W; ++dd) {
                const uint64_t g = static_cast<uint64_t>(h_G[static_cast<size_t>(w.rank) * W + dd]);
                uint64_t c = 0;
                for (int le = 0; le < El; ++le) c += tpe[static_cast<size_t>(w.rank) * E + dd * El + le];
                if (dd == w.rank) {
                    v[0] += g * rb;
                    v[3] += g * rb;
                } else {
                    v[1] += g * rb;
                    v[4] += g * rb;
                    v[2] += c * 24;
                }
            }
            if (W > 1) v[2] += static_cast<uint64_t>(W - 1) * (E + W) * sizeof(int32_t);
        }
    }
    for (int i = 0; i < n && i < 8; ++i) out[i] = v[i];
}

// ---------------------------------------------------------------- reference-schema ledger
// Byte matrices M[i][j] (sender i -> receiver j) per collective kind, from
// the routing of the last forward, then moesim's classification and
// alpha-beta model (collectives.cpp:36-76, 143-202).  Each process adds the
// contributions of the sources it drives; with one process per GPU the
// matrices are summed over the group, so every rank gets the global ledger.
namespace {

struct Kind {
    const char* name;
    std::vector<uint64_t> M;  // W * W
    bool ring = false;        // ssmb_gather_rows: synchronous ring all-gather
};

int node_of(const xmoe_topology& t, int w) { return t.gpus_per_node > 0 ? static_cast<int>(w / t.gpus_per_node) : w; }

xmoe_ledger_entry finish(const Kind& k, int W, const xmoe_topology& t, const std::vector<long long>& ring_rows,
                         uint64_t ring_row_bytes) {
    xmoe_ledger_entry e{};
    std::strncpy(e.kind, k.name, sizeof(e.kind) - 1);
    auto charge = [&](int i, int j, uint64_t bytes, std::vector<double>& sender) {
        if (i == j) {
            e.self_bytes += bytes;
        } else if (node_of(t, i) == node_of(t, j)) {
            e.intra_bytes += bytes;
            e.intra_msgs += 1;
            sender[i] += t.latency_intra + static_cast<double>(bytes) / t.bw_intra;
        } else {
            e.inter_bytes += bytes;
            e.inter_msgs += 1;
            sender[i] += t.latency_inter + static_cast<double>(bytes) / t.bw_inter;
        }
    };
    if (k.ring) {
        if (W > 1) {
            double total = 0.0;
            std::vector<double> one(W, 0.0);
            for (int step = 0; step < W - 1; ++step) {
                double step_time = 0.0;
                for (int i = 0; i < W; ++i) {
                    const int j = (i + 1) % W, chunk = (i + W - step) % W;
                    const uint64_t bytes = static_cast<uint64_t>(ring_rows[chunk]) * ring_row_bytes;
                    if (bytes == 0) continue;
                    one[i] = 0.0;
                    charge(i, j, bytes, one);
                    step_time = std::max(step_time, one[i]);
                }
                total += step_time;
            }
            e.time_s = total;
        }
        return e;
    }
    std::vector<double> sender(W, 0.0);
    for (int i = 0; i < W; ++i)
        for (int j = 0; j < W; ++j)
            if (k.M[static_cast<size_t>(i) * W + j] > 0) charge(i, j, k.M[static_cast<size_t>(i) * W + j], sender);
    e.time_s = W ? *std::max_element(sender.begin(), sender.end()) : 0.0;
    return e;
}

}  // namespace

void Layer::ledger_entries(const xmoe_topology& topo, std::vector<xmoe_ledger_entry>& out) {
    out.clear();
    XMOE_CUDA(cudaDeviceSynchronize());
    const uint64_t db = topo.dtype_bytes > 0 ? static_cast<uint64_t>(topo.dtype_bytes) : es;
    const uint64_t rbytes = static_cast<uint64_t>(H) * db;
    auto comm_sum = [&](std::vector<uint64_t>& v) {  // one process per GPU: sum over the group
        if (!distributed || v.empty()) return;
        uint64_t* d = nullptr;
        XMOE_CUDA(cudaMalloc(&d, sizeof(uint64_t) * v.size()));
        XMOE_CUDA(cudaMemcpy(d, v.data(), sizeof(uint64_t) * v.size(), cudaMemcpyHostToDevice));
        ncclResult_t r = ncclAllReduce(d, d, v.size(), ncclUint64, ncclSum, static_cast<ncclComm_t>(ctx->nccl), nullptr);
        if (r != ncclSuccess) {
            cudaFree(d);
            fail(XMOE_ERR_NCCL, std::string("ledger all-reduce: ") + ncclGetErrorString(r));
        }
        XMOE_CUDA(cudaMemcpy(v.data(), d, sizeof(uint64_t) * v.size(), cudaMemcpyDeviceToHost));
        XMOE_CUDA(cudaFree(d));
    };
    if (last_ssmb) {  // ssmb.cpp:12-46: G local pf forwards (W = 1 each), then the ring all-gather
        const int G = static_cast<int>(ssmb_rows.size());
        std::vector<int32_t> Bh(G, 0);
        XMOE_CUDA(cudaMemcpy(Bh.data(), ssmb_B, sizeof(int32_t) * G, cudaMemcpyDeviceToHost));
        std::vector<uint64_t> B(Bh.begin(), Bh.end());
        comm_sum(B);
        for (int g = 0; g < G; ++g) {
            const char* names[3] = {"dispatch_counts", "dispatch_rows", "combine_rows"};
            for (int q = 0; q < 3; ++q) {
                Kind k{names[q], std::vector<uint64_t>(1, q == 0 ? 0 : B[g] * rbytes)};
                out.push_back(finish(k, 1, topo, {}, 0));
            }
        }
        Kind ring{"ssmb_gather_rows", {}, true};
        if (G > 1) out.push_back(finish(ring, G, topo, ssmb_rows, rbytes));
        for (size_t i = 0; i < out.size(); ++i) out[i].id = static_cast<int64_t>(i);
        return;
    }
    std::vector<int32_t> tpe(static_cast<size_t>(W) * E);
    XMOE_CUDA(cudaMemcpy(tpe.data(), tpe_all, sizeof(int32_t) * tpe.size(), cudaMemcpyDeviceToHost));
    const size_t WW = static_cast<size_t>(W) * W;
    const bool rbd = d.dispatch_mode == XMOE_DISPATCH_RBD;
    std::vector<Kind> kinds;
    if (!rbd) {
        kinds = {{"dispatch_counts", std::vector<uint64_t>(WW, 0)},
                 {"dispatch_rows", std::vector<uint64_t>(WW, 0)},
                 {"combine_rows", std::vector<uint64_t>(WW, 0)}};
    } else {
        for (const char* n : {"rbd_dispatch_counts", "rbd_dispatch_meta", "rbd_dispatch_rows1", "rbd_dispatch_meta2",
                              "rbd_dispatch_rows2", "rbd_combine_rows2", "rbd_combine_rows1"})
            kinds.push_back({n, std::vector<uint64_t>(WW, 0)});
    }
    auto at = [&](int kind, int i, int j) -> uint64_t& { return kinds[kind].M[static_cast<size_t>(i) * W + j]; };
    for (const Worker& w : workers) {
        const int s = w.rank;
        for (int j = 0; j < W; ++j)
            if (j != s) at(0, s, j) = static_cast<uint64_t>(El) * 8;  // per-expert counts of j's block
        if (!rbd) {  // pf_pipeline.cpp:30-40, 128
            for (int e = 0; e < E; ++e) {
                const uint64_t c = static_cast<uint64_t>(tpe[static_cast<size_t>(s) * E + e]) * rbytes;
                at(1, s, e / El) += c;
                at(2, e / El, s) += c;
            }
            continue;
        }
        // rbd.cpp:130-233, 300-345: per (token, node) group of source s, from
        // the device counters (rbd.cu ledger_counts_kernel)
        const long long S = last_Sw.empty() ? last_S : last_Sw[static_cast<size_t>(&w - workers.data())];
        const std::vector<uint64_t> c = device_counts(w, S, true);
        for (int L = 0; L < W; ++L) {
            const uint64_t pil = c[1 + L], multi = c[1 + W + L], reps = c[1 + 2 * W + L];
            at(2, s, L) += pil * rbytes;                   // rows1: the pilot rows
            at(6, L, s) += pil * rbytes;                   // combine rows1: one merged row home
            at(1, s, L) += multi * db + reps * (3 * 8 + db);  // weights + replica descriptors
            for (int o = 0; o < W; ++o) {
                const uint64_t r2 = c[1 + 3 * W + static_cast<size_t>(L) * W + o];
                at(3, L, o) += r2 * 3 * 8;  // stage-2 descriptors
                at(4, L, o) += r2 * rbytes;  // stage-2 rows
                at(5, o, L) += r2 * rbytes;  // reverse stage 2
            }
        }
    }
    for (auto& kd : kinds) {
        comm_sum(kd.M);
        out.push_back(finish(kd, W, topo, {}, 0));
    }
    for (size_t i = 0; i < out.size(); ++i) out[i].id = static_cast<int64_t>(i);
}

// padded_pipeline.cpp:106-143: an even all-to-all of e_local * C slots per
// pair each way (self included), independent of the routing.
void Layer::padded_ledger_entries(const xmoe_topology& topo, std::vector<xmoe_ledger_entry>& out) {
    out.clear();
    const uint64_t db = topo.dtype_bytes > 0 ? static_cast<uint64_t>(topo.dtype_bytes) : es;
    const uint64_t slot_bytes = static_cast<uint64_t>(El) * static_cast<uint64_t>(d.max_token_count) * H * db;
    for (const char* n : {"padded_dispatch_rows", "padded_combine_rows"}) {
        Kind kd{n, std::vector<uint64_t>(static_cast<size_t>(W) * W, slot_bytes)};
        out.push_back(finish(kd, W, topo, {}, 0));
    }
    for (size_t i = 0; i < out.size(); ++i) out[i].id = static_cast<int64_t>(i);
}

}  // namespace xmoe
