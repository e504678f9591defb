// Host-side exchange plan of the plain expert-parallel dispatch, shared by
// the NCCL send/recv transport and exposed through the C-ABI so the
// multi-rank arithmetic can be exercised on CPU-only hosts.  It restates the
// reference's placement: receiver j lays rows out as (local expert, source,
// position) (pf_pipeline.cpp:47-73); a source's packed buffer is expert-major
// (pft.cpp:35-57), so its rows for expert e are one contiguous block.
#include <cstdint>
#include <string>

#include "xmoe/xmoe.h"

namespace xmoe {
extern thread_local std::string g_last_error;
}

extern "C" int xmoe_plan_dispatch(int W, int E, const int32_t* tpe_all, int me, int64_t* send_off,
                                  int64_t* recv_off, int64_t* recv_per_expert) {
    if (W < 1 || E < 1 || E % W != 0 || me < 0 || me >= W || !tpe_all) {
        xmoe::g_last_error = "num_experts must be divisible by the worker-group size";
        return XMOE_ERR_VALIDATION;
    }
    const int El = E / W;
    auto tpe = [&](int s, int e) { return static_cast<int64_t>(tpe_all[static_cast<int64_t>(s) * E + e]); };
    if (send_off) {
        int64_t a = 0;
        for (int e = 0; e < E; ++e) {
            send_off[e] = a;
            a += tpe(me, e);
        }
        send_off[E] = a;
    }
    int64_t base = 0;
    for (int le = 0; le < El; ++le) {
        const int e = me * El + le;
        int64_t before = 0;
        for (int s = 0; s < W; ++s) {
            if (recv_off) recv_off[static_cast<int64_t>(s) * El + le] = base + before;
            before += tpe(s, e);
        }
        if (recv_per_expert) recv_per_expert[le] = before;
        base += before;
    }
    return XMOE_OK;
}
