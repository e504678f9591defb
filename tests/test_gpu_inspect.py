"""The fused layer's own internal arrays against the reference, bit for bit
(xmoe_layer_inspect): routing (top_experts), the packed order (token_ids,
expert_ids, tokens_per_expert), the grouped expert input of every owner and
its recv_per_expert, the exchange counts, and the RBD pilot masks — compared
with the compiled reference's gate_forward / pft_construct / pf_dispatch /
rbd_dispatch / select_pilots (ref_shim.cpp ref_dispatch) on the same inputs,
for F64 and BF16 layers, plain and redundancy-bypassing, W in {1, 2, 4, 8}
workers (rank == -1: all workers on one GPU), unchunked and token-chunked."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu


def _layer(ctx, dtype, E, H, F, k, cap, S, gate, w1, w2, mode=0, seed=0, chunks=1, gpn=1):
    from paper_2508_13337_b200 import capi
    t = torch.float64 if dtype == capi.F64 else torch.bfloat16
    return capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap, max_tokens=S,
                      dtype=dtype, gate=dev(gate, t), w1=dev(w1, t), w2=dev(w2, t), dispatch_mode=mode, seed=seed,
                      chunks=chunks, gpus_per_node=gpn)


def grouped_from_chunks(L, W, E, H, me, dtype_np=np.float64):
    """Reassemble a chunked owner's regions into the reference's
    (local expert, source, position) order: region c holds chunk c's rows,
    laid out inside like the unchunked buffer (chunk.cu)."""
    C = L.chunks()
    T = host(L.inspect("tpe_chunks")).reshape(W, C, E)
    buf = host(L.inspect("expert_input", me)).reshape(-1, H)
    Rc = buf.shape[0] // C
    El = E // W
    rows = []
    for le in range(El):
        e = me * El + le
        for s in range(W):
            for c in range(C):
                base = c * Rc + sum(int(T[s2, c, me * El + l2]) for l2 in range(le) for s2 in range(W)) + \
                    sum(int(T[s2, c, e]) for s2 in range(s))
                rows.append(buf[base:base + int(T[s, c, e])])
    return np.concatenate(rows) if rows else np.zeros((0, H))


def check_layer(ref, L, toks, gate, w1, w2, E, k, cap, W, rbd=False, seed=0, gpn=1, chunked=False):
    S = toks.shape[1]
    node_of = [w // gpn for w in range(W)]
    want_ei, want_rpe, want_rc, want_pm, _ = ref.Layer(gate, w1, w2).dispatch(toks, k, cap, node_of=node_of,
                                                                             rbd=rbd, seed=seed)
    tpe_all = host(L.inspect("tpe_all")).reshape(W, E)
    El = E // W
    off = 0
    for w in range(W):
        top, wt = ref.gate_forward(toks[w], gate, k)
        assert np.array_equal(host(L.inspect("top_experts", w)).reshape(S, k), top), w
        tid, eid, cw, tpe = ref.pft_construct(cap, E, S, k, top, wt)
        assert np.array_equal(host(L.inspect("token_ids", w)), tid), w
        assert np.array_equal(host(L.inspect("expert_ids", w)), eid), w
        assert np.array_equal(host(L.inspect("tokens_per_expert", w)), tpe), w
        assert np.array_equal(tpe_all[w], tpe)
        n = int(want_rpe[w].sum())
        got = grouped_from_chunks(L, W, E, toks.shape[2], w) if chunked else \
            host(L.inspect("expert_input", w)).reshape(-1, toks.shape[2])[:n]
        assert np.array_equal(got, want_ei[w]), w          # grouped layout bit-exact
        if not chunked:
            assert np.array_equal(host(L.inspect("recv_per_expert", w)), want_rpe[w])
        if rbd:
            B = len(tid)
            assert np.array_equal(host(L.inspect("pilot_mask", w)), want_pm[off:off + B]), w
            off += B
    if not rbd:  # row_counts [W, W] from the all-gathered counts
        rc = np.stack([[tpe_all[i, j * El:(j + 1) * El].sum() for j in range(W)] for i in range(W)])
        assert np.array_equal(rc, want_rc)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("rbd", [False, True])
def test_f64_layer_internals(ref, W, rbd):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = O.Rng(500 + W + 7 * rbd)
    for trial in range(4):
        E = W * (1 + rng.below(4))
        k = 1 + rng.below(min(E, 4))
        H, F = 2 + rng.below(9), 2 + rng.below(9)
        S = 2 + rng.below(40)
        cap = S * k if trial % 2 == 0 else 1 + rng.below(3)
        w = O.make_layer_weights(rng, E, H, F)
        toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
        L = _layer(ctx, capi.F64, E, H, F, k, cap, S, w.gate, w.w1, w.w2, mode=int(rbd), seed=11 + trial)
        L.forward(dev(toks))
        check_layer(ref, L, toks, w.gate, w.w1, w.w2, E, k, cap, W, rbd=rbd, seed=11 + trial)


@pytest.mark.parametrize("W,gpn", [(4, 2), (8, 2), (8, 4)])
def test_f64_two_tier_pilots(ref, W, gpn):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = O.Rng(900 + W + gpn)
    E, k, H, F, S = 2 * W, 4, 6, 5, 33
    w = O.make_layer_weights(rng, E, H, F)
    toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
    L = _layer(ctx, capi.F64, E, H, F, k, S * k, S, w.gate, w.w1, w.w2, mode=1, seed=5, gpn=gpn)
    L.forward(dev(toks))
    check_layer(ref, L, toks, w.gate, w.w1, w.w2, E, k, S * k, W, rbd=True, seed=5, gpn=gpn)


@pytest.mark.parametrize("W,rbd,chunks", [(1, False, 1), (2, False, 1), (2, True, 1), (4, False, 4), (4, True, 1),
                                          (8, False, 2), (8, True, 1)])
def test_bf16_layer_internals(ref, W, rbd, chunks):
    """BF16 on the bf16-exact grid: logits exact in fp32, so routing, packed
    order and the (copied) grouped rows equal the reference's bit for bit."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(60 + W + rbd)
    E, k, H, F, S = 16 * W, 6, 128, 64, 512
    gate = np.round(rng.uniform(-0.1, 0.1, (H, E)) * 1024) / 1024
    w1 = rng.uniform(-0.1, 0.1, (E, H, F))
    w2 = rng.uniform(-0.1, 0.1, (E, F, H))
    toks = np.round(rng.uniform(-1, 1, (W, S, H)) * 128) / 128
    L = _layer(ctx, capi.BF16, E, H, F, k, S * k, S, gate, w1, w2, mode=int(rbd), seed=3, chunks=chunks)
    assert L.chunks() == chunks
    L.forward(dev(toks, torch.bfloat16))
    check_layer(ref, L, toks, gate, w1, w2, E, k, S * k, W, rbd=rbd, seed=3, chunked=chunks > 1)


@pytest.mark.parametrize("W,E,k,S,rbd", [(1, 64, 6, 4096, False), (2, 32, 8, 1000, False), (4, 64, 6, 777, True),
                                         (1, 256, 8, 300, False), (1, 16, 1, 129, False)])
def test_fused_routing_matches_general_path(ref, W, E, k, S, rbd):
    """The fused gate (softmax + top-k in the GEMM epilogue) and the one-launch
    dropless placement (taken when cap >= S) against the general gate + PFT
    path (cap = S - 1: the general kernels, no bucket reaches it here): every
    routing array, the grouped layout and the output bit-identical, and the
    routing equal to the reference's."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(E + k + S)
    H, F = 128, 64
    gate = np.round(rng.uniform(-0.1, 0.1, (H, E)) * 1024) / 1024
    w1 = rng.uniform(-0.1, 0.1, (E, H, F))
    w2 = rng.uniform(-0.1, 0.1, (E, F, H))
    toks = np.round(rng.uniform(-1, 1, (W, S, H)) * 128) / 128
    xd = dev(toks, torch.bfloat16)
    fused = _layer(ctx, capi.BF16, E, H, F, k, S * k, S, gate, w1, w2, mode=int(rbd), seed=3)
    general = _layer(ctx, capi.BF16, E, H, F, k, S - 1, S, gate, w1, w2, mode=int(rbd), seed=3)
    a = fused.forward(xd).clone()
    b = general.forward(xd).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    for w in range(W):
        for what in ("top_experts", "weights", "token_ids", "expert_ids", "combine_weights", "tokens_per_expert",
                     "slot_pos", "dest_row"):
            assert torch.equal(fused.inspect(what, w), general.inspect(what, w)), (what, w)
    check_layer(ref, fused, toks, gate, w1, w2, E, k, S * k, W, rbd=rbd, seed=3)
