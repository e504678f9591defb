// Byte ledger of the last layer forward — the measured counterpart of the
// reference's CostLedger (collectives.hpp:31-69, charge_message in
// collectives.cpp:45-76).  Self traffic stays on the GPU; off-rank traffic
// crosses NVLink.  Row bytes use the layer's real element size.
#include <cuda_runtime.h>

#include <set>
#include <utility>
#include <vector>

#include "common.cuh"
#include "layer.h"

namespace xmoe {

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
        // the redundancy bypass sends (rbd.cpp:427-442 with node_of = rank)
        const long long S = last_S;
        if (S > 0) {
            std::vector<int32_t> slot(static_cast<size_t>(S) * k), eid(static_cast<size_t>(S) * k);
            XMOE_CUDA(cudaMemcpy(slot.data(), w.slot_pos, sizeof(int32_t) * slot.size(), cudaMemcpyDeviceToHost));
            int32_t B = 0;
            XMOE_CUDA(cudaMemcpy(&B, w.B_dev, sizeof(int32_t), cudaMemcpyDeviceToHost));
            std::vector<int32_t> ex(B > 0 ? B : 1);
            if (B > 0) XMOE_CUDA(cudaMemcpy(ex.data(), w.expert_ids, sizeof(int32_t) * B, cudaMemcpyDeviceToHost));
            for (long long t = 0; t < S; ++t) {
                std::set<int> dests;
                for (int j = 0; j < k; ++j) {
                    const int p = slot[static_cast<size_t>(t) * k + j];
                    if (p < 0) break;
                    const int d = ex[p] / El;
                    if (d != w.rank) dests.insert(d);
                }
                v[6] += dests.size();
            }
        }
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

}  // namespace xmoe
