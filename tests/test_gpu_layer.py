"""GPU parity of the whole MoE-block forward (moesim::pf_moe_forward and the
expert-parallel exchange) through the C-ABI layer object, against the pinned
oracle on identical inputs.

F64 (parity mode): routing indices, counts and order bit-exact; given the
device's own softmax weights (CUDA exp vs glibc exp may differ in the last
ulp) every other operation reproduces the reference bit for bit, and the
end-to-end output is within 1e-14 max_rel_diff of the pure oracle —
including emulated expert-parallel groups of W workers on one GPU.  BF16 (performance mode):
routing bit-exact on grid inputs; outputs within normwise 1e-2 and
max_rel_diff (floor 1, matrix.hpp:47-62) 2e-2 of the fp64 oracle."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from tests.gpu_util import bf16_round, dev, grid_gate, grid_tokens, host, max_rel_diff, norm_rel

pytestmark = pytest.mark.gpu


def _device_gates(ctx, toks, w, k):
    out = []
    for x in toks:
        top, wt = ctx.gate_forward(dev(x), dev(w.gate), k)
        out.append((host(top), host(wt)))
    return out


def _assert_f64_parity(ctx, got, toks, w, E, k, cap, sw1=None, sw2=None):
    gates = _device_gates(ctx, toks, w, k)
    if sw1 is None:
        exact = O.pf_moe_forward(list(toks), w, E, k, cap, gates=gates)
        pure = O.pf_moe_forward(list(toks), w, E, k, cap)
    else:
        exact = [O.moe_layer_with_shared(toks[0], w, E, k, cap, sw1, sw2, gates=gates)]
        pure = [O.moe_layer_with_shared(toks[0], w, E, k, cap, sw1, sw2)]
    for i in range(len(toks)):
        ref_top = O.gate_forward(toks[i], w.gate, k).top_experts
        assert np.array_equal(gates[i][0], ref_top)          # routing bit-exact
        assert np.array_equal(got[i], exact[i]), i            # everything after exp bit-exact
        assert max_rel_diff(got[i], pure[i]) < 1e-14          # end to end


def _layer(ctx, dtype, E, H, F, k, cap, S, w, sw1=None, sw2=None, mode=0, seed=0):
    from paper_2508_13337_b200 import capi
    tdt = torch.float64 if dtype == capi.F64 else torch.bfloat16
    return capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap,
                      max_tokens=S, dtype=dtype, gate=dev(w.gate, tdt), w1=dev(w.w1, tdt),
                      w2=dev(w.w2, tdt), sw1=None if sw1 is None else dev(sw1, tdt),
                      sw2=None if sw2 is None else dev(sw2, tdt), dispatch_mode=mode, seed=seed)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_pf_forward_f64_bit_exact(W):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = O.Rng(31337 + W)
    for trial in range(4):
        E = W * (1 + rng.below(4))
        k = 1 + rng.below(min(E, 4))
        H = 2 + rng.below(7)
        F = 2 + rng.below(7)
        S = 2 + rng.below(31)
        cap = 1 + rng.below(4) if trial % 2 == 0 else S * k
        w = O.make_layer_weights(rng, E, H, F)
        toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
        L = _layer(ctx, capi.F64, E, H, F, k, cap, S, w)
        got = host(L.forward(dev(toks)))
        _assert_f64_parity(ctx, got, toks, w, E, k, cap)
        led = L.ledger()
        _, pfts, _, _ = O.pf_moe_forward(list(toks), w, E, k, cap, return_pfts=True)
        assert led["routed_copies"] == sum(p.size() for p in pfts)


def test_pf_forward_f64_reference_scale():
    """A wider f64 layer (E=64, k=6) still bit-exact, dropless and capped."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    rng = np.random.default_rng(7)
    E, k, H, F, S = 64, 6, 64, 48, 256
    w = O.LayerWeights(rng.uniform(-0.1, 0.1, (H, E)), rng.uniform(-0.1, 0.1, (E, H, F)),
                       rng.uniform(-0.1, 0.1, (E, F, H)))
    x = rng.uniform(-1, 1, (1, S, H))
    for cap in (S * k, int(np.ceil(1.25 * S * k / E))):
        got = host(_layer(ctx, capi.F64, E, H, F, k, cap, S, w).forward(dev(x)))
        _assert_f64_parity(ctx, got, x, w, E, k, cap)


def test_shared_experts_f64_bit_exact():
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    rng = np.random.default_rng(9)
    E, k, H, F, S, ns, Fs = 16, 4, 24, 16, 50, 2, 16
    w = O.LayerWeights(rng.uniform(-0.1, 0.1, (H, E)), rng.uniform(-0.1, 0.1, (E, H, F)),
                       rng.uniform(-0.1, 0.1, (E, F, H)))
    sw1 = rng.uniform(-0.1, 0.1, (ns, H, Fs))
    sw2 = rng.uniform(-0.1, 0.1, (ns, Fs, H))
    x = rng.uniform(-1, 1, (S, H))
    got = host(_layer(ctx, capi.F64, E, H, F, k, S * k, S, w, sw1, sw2).forward(dev(x[None])))
    _assert_f64_parity(ctx, got, x[None], w, E, k, S * k, sw1, sw2)


@pytest.mark.parametrize("W,S,E,k,H,F,shared", [(1, 512, 64, 6, 256, 128, True),
                                                 (1, 2048, 64, 6, 2048, 1408, False),
                                                 (4, 256, 32, 4, 128, 64, False)])
def test_forward_bf16_vs_oracle(W, S, E, k, H, F, shared):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(S + W)
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    x = grid_tokens(rng, W, S, H)
    sw1 = sw2 = None
    if shared:
        sw1 = bf16_round(rng.uniform(-0.1, 0.1, (2, H, F)))
        sw2 = bf16_round(rng.uniform(-0.1, 0.1, (2, F, H)))
    L = _layer(ctx, capi.BF16, E, H, F, k, S * k, S, w, sw1, sw2)
    got = host(L.forward(dev(x, torch.bfloat16)))
    if shared:
        want = [O.moe_layer_with_shared(x[0], w, E, k, S * k, sw1, sw2, exact=False)]
    else:
        want = O.pf_moe_forward(list(x), w, E, k, S * k, exact=False)
    for i in range(W):
        assert norm_rel(got[i], want[i]) < 1e-2, norm_rel(got[i], want[i])
        assert max_rel_diff(got[i], want[i]) < 2e-2, max_rel_diff(got[i], want[i])


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_rbd_forward_f64_bit_exact(W):
    """rbd_moe_forward with one GPU per node (node_of = rank): pilots drawn
    from the reference RNG stream via jump-ahead, merge and combine orders
    as rbd.cpp:318-356 — bit-exact given the device softmax weights."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = O.Rng(1717 + W)
    for trial in range(4):
        E = W * (1 + rng.below(3))
        k = 1 + rng.below(min(E, 4))
        H = 2 + rng.below(5)
        F = 2 + rng.below(5)
        S = 2 + rng.below(23)
        cap = 1 + rng.below(4) if trial % 2 == 0 else S * k
        w = O.make_layer_weights(rng, E, H, F)
        toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
        seed = rng.next_u64()
        L = _layer(ctx, capi.F64, E, H, F, k, cap, S, w, mode=capi.RBD, seed=seed)
        got = host(L.forward(dev(toks)))
        gates = _device_gates(ctx, toks, w, k)
        exact = O.rbd_moe_forward(list(toks), w, E, k, cap, seed, gates=gates)
        pure = O.rbd_moe_forward(list(toks), w, E, k, cap, seed)
        for i in range(W):
            assert np.array_equal(got[i], exact[i]), (trial, i)
            assert max_rel_diff(got[i], pure[i]) < 1e-14
        # per-GPU dedupe accounting: off-rank rows == distinct (token, dest) groups
        led = L.ledger()
        _, pfts, _, _ = O.pf_moe_forward(list(toks), w, E, k, cap, return_pfts=True, gates=gates)
        nodes = O.expert_nodes(list(range(W)), E)
        groups = sum(O.redundancy_counts_internode(p, s, nodes)[1] for s, p in enumerate(pfts))
        copies = sum(O.redundancy_counts_internode(p, s, nodes)[0] for s, p in enumerate(pfts))
        assert led["unique_rows_offrank"] == groups
        assert led["copies_offrank"] == copies
        assert led["dispatch_rows_offrank"] == groups * H * 8


@pytest.mark.parametrize("W,gpn", [(2, 2), (4, 2), (8, 2), (8, 4)])
def test_rbd_two_tier_f64_bit_exact(W, gpn):
    """Two-tier rbd_moe_forward (rbd.cpp:83-358, node_of = rank / gpn): one
    row per (token, destination node) to the pilot's owner, forwarded inside
    the node to the replicas' owners, merged at the landing rank from the
    owners' outputs — bit-exact to the pinned oracle given the device softmax
    weights, and to the compiled reference within the exp-ulp bound."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = O.Rng(2929 + 10 * W + gpn)
    node_of = [r // gpn for r in range(W)]
    for trial in range(4):
        E = W * (1 + rng.below(3))
        k = 1 + rng.below(min(E, 5))
        H = 2 + rng.below(5)
        F = 2 + rng.below(5)
        S = 2 + rng.below(23)
        cap = 1 + rng.below(4) if trial % 2 == 0 else S * k
        w = O.make_layer_weights(rng, E, H, F)
        toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
        seed = rng.next_u64()
        L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap, max_tokens=S,
                       dtype=capi.F64, gate=dev(w.gate), w1=dev(w.w1), w2=dev(w.w2), dispatch_mode=capi.RBD,
                       seed=seed, gpus_per_node=gpn)
        got = host(L.forward(dev(toks)))
        gates = _device_gates(ctx, toks, w, k)
        exact = O.rbd_moe_forward(list(toks), w, E, k, cap, seed, node_of, gates=gates)
        pure = O.rbd_moe_forward(list(toks), w, E, k, cap, seed, node_of)
        for i in range(W):
            assert np.array_equal(got[i], exact[i]), (trial, i)
            assert max_rel_diff(got[i], pure[i]) < 1e-14


def test_rbd_two_tier_bf16_vs_oracle():
    from paper_2508_13337_b200 import capi
    W, gpn, S, E, k, H, F = 8, 4, 256, 64, 6, 128, 64
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(99)
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    x = grid_tokens(rng, W, S, H)
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                   dtype=capi.BF16, gate=dev(w.gate, torch.bfloat16), w1=dev(w.w1, torch.bfloat16),
                   w2=dev(w.w2, torch.bfloat16), dispatch_mode=capi.RBD, seed=4, gpus_per_node=gpn)
    assert L.chunks() == 1
    got = host(L.forward(dev(x, torch.bfloat16)))
    want = O.rbd_moe_forward(list(x), w, E, k, S * k, 4, [r // gpn for r in range(W)], exact=False)
    for i in range(W):
        assert norm_rel(got[i], want[i]) < 1e-2, norm_rel(got[i], want[i])


@pytest.mark.parametrize("W,S,E,k,H,F", [(4, 512, 64, 6, 256, 128), (8, 256, 64, 6, 128, 64)])
def test_rbd_forward_bf16_vs_oracle(W, S, E, k, H, F):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(S * W)
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    x = grid_tokens(rng, W, S, H)
    sw1 = bf16_round(rng.uniform(-0.1, 0.1, (2, H, F)))
    sw2 = bf16_round(rng.uniform(-0.1, 0.1, (2, F, H)))
    L = _layer(ctx, capi.BF16, E, H, F, k, S * k, S, w, sw1, sw2, mode=capi.RBD, seed=3)
    got = host(L.forward(dev(x, torch.bfloat16)))
    want = O.rbd_moe_forward(list(x), w, E, k, S * k, 3, exact=False, shared=(sw1, sw2))
    for i in range(W):
        assert norm_rel(got[i], want[i]) < 1e-2, norm_rel(got[i], want[i])
        assert max_rel_diff(got[i], want[i]) < 2e-2, max_rel_diff(got[i], want[i])
    led = L.ledger()
    assert led["dispatch_rows_offrank"] < led["copies_offrank"] * H * 2  # bytes actually saved


@pytest.mark.parametrize("G,S", [(1, 9), (2, 37), (4, 61), (8, 64)])
def test_ssmb_forward_f64(G, S):
    """ssmb_forward (ssmb.cpp:12-46): contiguous shards, last takes the
    remainder, replicated experts, capacity per shard; all-gathered."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, G, -1)
    rng = O.Rng(11 + G)
    E = 4 + rng.below(5)
    k = 1 + rng.below(3)
    H = 3 + rng.below(4)
    F = 2 + rng.below(5)
    w = O.make_layer_weights(rng, E, H, F)
    x = np.array([rng.uniform(-1.0, 1.0) for _ in range(S * H)]).reshape(S, H)
    for cap in (S * k, 2):
        bounds = O.ssmb_shards(S, G)
        biggest = max(n for _, n in bounds)
        L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap,
                       max_tokens=biggest, dtype=capi.F64, gate=dev(w.gate), w1=dev(w.w1), w2=dev(w.w2),
                       ssmb=True)
        got = host(L.ssmb_forward(dev(x)))
        exact = np.concatenate([
            O.pf_moe_forward([x[b:b + n]], w, E, k, cap, gates=_device_gates(ctx, x[None, b:b + n], w, k))[0]
            for b, n in bounds])
        assert np.array_equal(got, exact)
        pure = O.ssmb_forward(x, G, w, E, k, cap)
        assert max_rel_diff(got, pure) < 1e-14
        if cap == S * k:  # test_ssmb.cpp:61-77: no drops => equals the unsharded layer
            assert max_rel_diff(got, O.pf_moe_forward([x], w, E, k, S * k)[0]) < 1e-14


@pytest.mark.parametrize("mode", [0, 1])
def test_graph_replay_matches_eager(mode):
    """The CUDA-graph replay of the forward is bit-identical to eager launches
    (and a second input buffer gets its own graph)."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, 0)
    rng = np.random.default_rng(4)
    E, k, H, F, S = 64, 6, 256, 128, 512
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    sw1 = bf16_round(rng.uniform(-0.1, 0.1, (2, H, 64)))
    sw2 = bf16_round(rng.uniform(-0.1, 0.1, (2, 64, H)))
    L = _layer(ctx, capi.BF16, E, H, F, k, S * k, S, w, sw1, sw2, mode=mode, seed=7)
    xa = dev(grid_tokens(rng, S, H), torch.bfloat16)
    xb = dev(grid_tokens(rng, S, H), torch.bfloat16)
    n0 = capi.kernel_launches()
    eager_a, eager_b = L.forward(xa).clone(), L.forward(xb).clone()
    per_forward = (capi.kernel_launches() - n0) // 2
    assert per_forward > 10
    L.set_graph(True)
    oa, ob = torch.empty_like(xa), torch.empty_like(xb)
    for _ in range(3):
        L.forward(xa, oa)
        L.forward(xb, ob)
    torch.cuda.synchronize()
    assert torch.equal(oa, eager_a) and torch.equal(ob, eager_b)
    n1 = capi.kernel_launches()  # a replay counts the kernels it runs
    L.forward(xa, oa)
    assert capi.kernel_launches() - n1 == per_forward


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("W,S,chunks,cap_factor,shared", [(1, 1000, 2, None, True), (1, 4096, 8, None, True),
                                                          (4, 333, 3, None, False), (4, 512, 4, 0.5, True),
                                                          (2, 3, 4, None, False), (8, 700, 5, None, True),
                                                          (2, 6144, 2, None, True), (8, 2048, 3, 0.5, True)])
def test_chunked_forward_bit_identical(W, S, chunks, cap_factor, shared, mode):
    """The token-chunked pipelined forward (chunk.cu), plain and
    redundancy-bypassing, is bit-identical to the unchunked one — ragged
    chunks, capacity drops, more chunks than tokens, and chunks with more
    rows than the SM partition's whole-SM copy kernels have warps — and
    matches the fp64 oracle at the bf16 tolerance."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(S + 17 * W)
    E, k, H, F = 32, 4, 256, 128
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    sw1 = bf16_round(rng.uniform(-0.1, 0.1, (2, H, 64))) if shared else None
    sw2 = bf16_round(rng.uniform(-0.1, 0.1, (2, 64, H))) if shared else None
    cap = S * k if cap_factor is None else max(1, int(cap_factor * S * k / E))
    x = grid_tokens(rng, W, S, H)
    xd = dev(x, torch.bfloat16)
    outs = []
    for c in (1, chunks):
        L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap, max_tokens=S,
                       dtype=capi.BF16, gate=dev(w.gate, torch.bfloat16), w1=dev(w.w1, torch.bfloat16),
                       w2=dev(w.w2, torch.bfloat16), sw1=None if sw1 is None else dev(sw1, torch.bfloat16),
                       sw2=None if sw2 is None else dev(sw2, torch.bfloat16), chunks=c, dispatch_mode=mode,
                       seed=5)
        assert L.chunks() == min(c, S)
        outs.append(L.forward(xd).clone())
        outs.append(L.forward(xd).clone())  # second forward: epochs / reused regions
        led = L.ledger()
    assert torch.equal(outs[0], outs[2]) and torch.equal(outs[1], outs[3]) and torch.equal(outs[0], outs[1])
    got = host(outs[2])
    if shared:
        want = [O.moe_layer_with_shared(x[i], w, E, k, cap, sw1, sw2, exact=False) for i in range(W)]
    else:
        want = O.pf_moe_forward(list(x), w, E, k, cap, exact=False)
    for i in range(W):
        assert norm_rel(got[i], want[i]) < 1e-2, norm_rel(got[i], want[i])
    assert led["routed_copies"] > 0
    if mode == 1 and W > 1:
        assert led["unique_rows_offrank"] <= led["copies_offrank"]


@pytest.mark.parametrize("mode,W,gpn", [(0, 4, 1), (0, 4, 2), (1, 4, 1), (1, 4, 2), (1, 8, 4), (0, 1, 1)])
def test_ledger_csv_matches_reference(ref, mode, W, gpn):
    """The reference-schema ledger of a GPU forward (xmoe_layer_ledger_csv)
    equals CostLedger::write_csv of the UNMODIFIED reference forward on the
    same inputs, byte for byte: kinds, ids, intra/inter bytes and the
    alpha-beta modeled times (default Topology, node_of = rank / gpn)."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = O.Rng(515 + 7 * W + gpn + mode)
    E = W * 4
    k, H, F, S = 3, 6, 5, 29
    cap = 12
    w = O.make_layer_weights(rng, E, H, F)
    toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
    seed = rng.next_u64()
    node_of = [r // gpn for r in range(W)]
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap, max_tokens=S,
                   dtype=capi.F64, gate=dev(w.gate), w1=dev(w.w1), w2=dev(w.w2),
                   dispatch_mode=capi.RBD if mode else capi.NAIVE, seed=seed, gpus_per_node=gpn if mode else 1)
    L.forward(dev(toks))
    topo = capi.Topology.reference_defaults(gpus_per_node=gpn, dtype_bytes=2)
    got = L.ledger_csv(topo)
    rl = ref.Layer(w.gate, w.w1, w.w2)
    if mode:
        rl.rbd_moe_forward(toks, k, cap, seed, node_of)
    else:
        rl.pf_moe_forward(toks, k, cap, node_of)
    want = ref.last_ledger_csv()
    assert got == want, (got, want)
    ents = L.ledger_entries(topo)
    assert [e["kind"] for e in ents] == [line.split(",")[1] for line in want.strip().split("\n")[1:]]
    # the padded (GShard) comparator: what padded_moe_forward would charge
    rl.padded_moe_forward(toks, k, cap, node_of)
    assert L.ledger_csv(topo, padded=True) == ref.last_ledger_csv()


@pytest.mark.parametrize("G", [2, 4])
def test_ledger_csv_ssmb_matches_reference(ref, G):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, G, -1)
    rng = O.Rng(77 + G)
    E, k, H, F, S = 8, 2, 5, 4, 45
    w = O.make_layer_weights(rng, E, H, F)
    x = np.array([rng.uniform(-1.0, 1.0) for _ in range(S * H)]).reshape(S, H)
    bounds = O.ssmb_shards(S, G)
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k,
                   max_tokens=max(n for _, n in bounds), dtype=capi.F64, gate=dev(w.gate), w1=dev(w.w1),
                   w2=dev(w.w2), ssmb=True)
    L.ssmb_forward(dev(x))
    got = L.ledger_csv(capi.Topology.reference_defaults(gpus_per_node=1, dtype_bytes=2))
    ref.Layer(w.gate, w.w1, w.w2).ssmb_forward(x, G, k, S * k)
    assert got == ref.last_ledger_csv()


@pytest.mark.parametrize("mode,dtype,chunks", [(0, "f64", 1), (1, "f64", 1), (0, "bf16", 1), (1, "bf16", 1),
                                               (0, "bf16", 3), (1, "bf16", 2)])
def test_layer_edge_lengths_and_errors(mode, dtype, chunks):
    """Empty and ragged sequences through one layer object (S = 0, 1, odd, the
    maximum), each equal to a fresh layer's result, and the layer's
    validation errors (error.hpp status codes, reference messages)."""
    from paper_2508_13337_b200 import capi
    from paper_2508_13337_b200.capi import XmoeError
    W, E, k, H, F, S_max = 2, 16, 3, 32, 32, 37
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(3)
    dt = capi.F64 if dtype == "f64" else capi.BF16
    tdt = torch.float64 if dtype == "f64" else torch.bfloat16
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    mk = lambda: capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S_max * k,  # noqa: E731
                            max_tokens=S_max, dtype=dt, gate=dev(w.gate, tdt), w1=dev(w.w1, tdt),
                            w2=dev(w.w2, tdt), dispatch_mode=mode, seed=9, chunks=chunks)
    L = mk()
    for S in (0, 1, 17, S_max, 5, 0):
        x = dev(grid_tokens(rng, W, S, H), tdt)
        got = L.forward(x).clone()
        want = mk().forward(x)
        assert torch.equal(got, want), S
        if S:
            ref = O.pf_moe_forward(list(host(x)), w, E, k, S_max * k, exact=False) if mode == 0 else \
                O.rbd_moe_forward(list(host(x)), w, E, k, S_max * k, 9, exact=False)
            for i in range(W):
                assert norm_rel(host(got[i]), ref[i]) < (1e-12 if dtype == "f64" else 1e-2)
    with pytest.raises(XmoeError, match="longer than the layer's max_tokens"):
        L.forward(dev(grid_tokens(rng, W, S_max + 1, H), tdt))
    with pytest.raises(XmoeError, match="divisible"):
        capi.Layer(ctx, num_experts=E + 1, model_dim=H, ffn_dim=F, top_k=k, max_token_count=8, max_tokens=8,
                   dtype=capi.F64, gate=dev(rng.uniform(-1, 1, (H, E + 1))),
                   w1=dev(rng.uniform(-1, 1, (E + 1, H, F))), w2=dev(rng.uniform(-1, 1, (E + 1, F, H))))
    if mode == 1:
        with pytest.raises(XmoeError, match="whole nodes"):
            capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=8, max_tokens=8,
                       dtype=dt, gate=dev(w.gate, tdt), w1=dev(w.w1, tdt), w2=dev(w.w2, tdt),
                       dispatch_mode=1, gpus_per_node=4)
    else:
        with pytest.raises(XmoeError, match="redundancy-bypassing"):
            capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=8, max_tokens=8,
                       dtype=dt, gate=dev(w.gate, tdt), w1=dev(w.w1, tdt), w2=dev(w.w2, tdt),
                       dispatch_mode=0, gpus_per_node=2)


@pytest.mark.parametrize("W,chunks", [(2, 1), (4, 1), (8, 1), (4, 3)])
def test_rbd_gather_gemm_bit_identical_to_expand(W, chunks, monkeypatch):
    """RBD replicas read through the TMA gather4 A-load of GEMM1 (no expand
    copy, XMOE_RBD_GATHER=1) give bit-identical outputs to the row-copying
    expand (the default)."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(W * 10 + chunks)
    E, k, H, F, S = 8 * W, 6, 256, 128, 700
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    x = dev(grid_tokens(rng, W, S, H), torch.bfloat16)
    outs = []
    for gather in ("0", "1"):
        monkeypatch.setenv("XMOE_RBD_GATHER", gather)
        L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                       dtype=capi.BF16, gate=dev(w.gate, torch.bfloat16), w1=dev(w.w1, torch.bfloat16),
                       w2=dev(w.w2, torch.bfloat16), dispatch_mode=capi.RBD, seed=21, chunks=chunks)
        outs.append(L.forward(x).clone())
        outs.append(L.forward(x).clone())
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    want = O.rbd_moe_forward(list(host(x)), w, E, k, S * k, 21, exact=False)
    for i in range(W):
        assert norm_rel(host(outs[3][i]), want[i]) < 1e-2


@pytest.mark.parametrize("W,E,k,H,F,mode,chunks", [(16, 16, 1, 16, 32, 0, 1), (16, 16, 3, 16, 32, 1, 1),
                                                   (2, 16, 2, 64, 32, 1, 2), (8, 16, 8, 32, 64, 0, 4),
                                                   (8, 16, 8, 32, 64, 1, 1), (1, 16, 16, 32, 32, 0, 3)])
def test_bf16_unusual_shapes(W, E, k, H, F, mode, chunks):
    """top_k = 1, one expert per GPU (16 workers), top_k = num_experts, the
    smallest bf16 widths (bf16 needs num_experts % 16 == 0) — plain and RBD,
    chunked and not — against the oracle."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(E * 7 + k)
    S = 300
    w = O.LayerWeights(grid_gate(rng, H, E), bf16_round(rng.uniform(-0.1, 0.1, (E, H, F))),
                       bf16_round(rng.uniform(-0.1, 0.1, (E, F, H))))
    x = grid_tokens(rng, W, S, H)
    for cap in (S * k, max(1, S * k // (2 * E))):
        L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap, max_tokens=S,
                       dtype=capi.BF16, gate=dev(w.gate, torch.bfloat16), w1=dev(w.w1, torch.bfloat16),
                       w2=dev(w.w2, torch.bfloat16), dispatch_mode=mode, seed=2, chunks=chunks)
        got = host(L.forward(dev(x, torch.bfloat16)))
        want = O.pf_moe_forward(list(x), w, E, k, cap, exact=False) if mode == 0 else \
            O.rbd_moe_forward(list(x), w, E, k, cap, 2, exact=False)
        for i in range(W):
            assert norm_rel(got[i], want[i]) < 1e-2, (cap, i, norm_rel(got[i], want[i]))


@pytest.mark.parametrize("S,H,ns", [(2048, 256, 2), (777, 128, 1), (16384, 2048, 2)])
def test_late_shared_gemm_bit_identical(S, H, ns):
    """One GPU with shared experts (XMOE_LATE_SHARED=1, an A/B knob run in a
    subprocess here): shared GEMM2 runs beside the combine, its epilogue adding
    the combine's fp32 sums per published 128-token block.  Same arithmetic as
    the combine's addend: the output equals the in-order path's bit for bit;
    with the knob off the forward, eager and graph-replayed, equals it too."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    rng = np.random.default_rng(S + H)
    E, k, F, Fs = 64, 6, 128, 128
    bf = torch.bfloat16
    w = O.LayerWeights(grid_gate(rng, H, E), rng.uniform(-0.1, 0.1, (E, H, F)), rng.uniform(-0.1, 0.1, (E, F, H)))
    sw1, sw2 = rng.uniform(-0.1, 0.1, (ns, H, Fs)), rng.uniform(-0.1, 0.1, (ns, Fs, H))
    x = dev(grid_tokens(rng, S, H), bf)
    L = _layer(ctx, capi.BF16, E, H, F, k, S * k, S, w, sw1, sw2)
    a = [L.forward(x).clone() for _ in range(2)]
    L.set_graph(True)
    g = L.forward(x).clone()
    L.set_graph(False)
    L.set_timing(True)
    b = L.forward(x).clone()
    torch.cuda.synchronize()
    assert torch.equal(a[0], b) and torch.equal(a[1], b) and torch.equal(g, b)
    want = O.moe_layer_with_shared(host(x).astype(np.float64), O.LayerWeights(w.gate, bf16_round(w.w1), bf16_round(w.w2)),
                                   E, k, S * k, bf16_round(sw1), bf16_round(sw2), exact=False)
    assert norm_rel(host(b), want) < 1e-2


def test_late_shared_knob_subprocess():
    """XMOE_LATE_SHARED=1 in a fresh process: bit-identical to the default path."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); import pytest; "
            "sys.exit(pytest.main(['-q', '-x', '-k', 'late_shared_gemm', %r]))" % (root, os.path.abspath(__file__)))
    env = dict(os.environ, XMOE_LATE_SHARED="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0



@pytest.mark.parametrize("knob", ["XMOE_CHUNK_LATE=1", "XMOE_DISPATCH=push", "XMOE_COMM_SMS=0",
                                  "XMOE_RBD_PARTITION=1"])
def test_chunked_knobs_subprocess(knob):
    """The chunked forward's A/B knobs (read once per process, so run in a
    fresh one): late shared GEMM2 beside the final combine, source-side pushes,
    no SM partition, RBD on the partition — each bit-identical to the
    unchunked forward."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); import pytest; "
            "sys.exit(pytest.main(['-q', '-x', '-k', 'chunked_forward_bit_identical', %r]))"
            % (root, os.path.abspath(__file__)))
    name, value = knob.split("=")
    env = dict(os.environ, **{name: value})
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0
