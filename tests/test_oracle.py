"""Pins the numpy restatement (oracle/moe_oracle.py) before any GPU result is
compared with it: (1) the reference's own known-answer vectors, restated from
/root/reference/proj/tests, and (2) bit-for-bit agreement with the unmodified
reference compiled into oracle/_ref on seeded random trials.  CPU only."""
import numpy as np
import pytest

from oracle import moe_oracle as O


# ---------------------------------------------------------------- RNG pins
def test_rng_frozen_value():
    # test_kernels.cpp:98-108
    assert O.Rng(42).next_u64() == 6667968346354703667


def test_rng_matches_reference(ref):
    for seed in (0, 1, 42, 2**63 + 5):
        r = O.Rng(seed)
        want = ref.rng_u64(seed, 64)
        assert [r.next_u64() for _ in range(64)] == [int(v) for v in want]
    for a, b in ((0, 0), (3, 7), (9000, 0)):
        assert O.salt_seed(11, a, b) == ref.salt_seed(11, a, b)


def test_layer_weight_draw_order(ref):
    rng = O.Rng(77)
    w = O.make_layer_weights(rng, 3, 4, 5)
    g, w1, w2 = ref.make_layer_weights(77, 3, 4, 5)
    assert np.array_equal(w.gate, g) and np.array_equal(w.w1, w1) and np.array_equal(w.w2, w2)


# ---------------------------------------------------------------- gating pins
def test_gate_tie_lower_id():
    # test_gating.cpp:14-23
    g = O.gate_forward(np.array([[1.0, -2.0]]), np.zeros((2, 2)), 1)
    assert g.top_experts[0, 0] == 0
    assert abs(g.combine_weights[0, 0] - 0.5) < 1e-12


def test_gate_hand_softmax():
    # test_gating.cpp:25-56
    x = np.array([[1.0, 0.0], [-0.5, 2.0]])
    w = np.array([[0.3, -0.1, 0.0], [0.2, 0.4, -0.3]])
    g = O.gate_forward(x, w, 2)
    for t in range(2):
        logits = x[t] @ w
        p = np.exp(logits) / np.exp(logits).sum()
        order = np.argsort(-logits, kind="stable")
        assert list(g.top_experts[t]) == list(order[:2])
        assert np.allclose(g.combine_weights[t], p[order[:2]], rtol=1e-12)


def test_gate_raw_weights_not_renormalised():
    # test_gating.cpp:58-84
    rng = O.Rng(11)
    x = np.array([rng.uniform(-1.0, 1.0) for _ in range(16 * 8)]).reshape(16, 8)
    w = O.make_gate_weights(rng, 8, 6)
    g = O.gate_forward(x, w, 3)
    s = g.combine_weights.sum(axis=1)
    assert np.all(s > 0) and np.all(s < 1)
    assert np.all(np.diff(g.combine_weights, axis=1) <= 0)
    full = O.gate_forward(x, w, 6)
    assert np.allclose(full.combine_weights.sum(axis=1), 1.0, atol=1e-6)


def test_gate_errors():
    # test_gating.cpp:86-95
    with pytest.raises(O.DimensionError):
        O.gate_forward(np.zeros((2, 4)), np.zeros((3, 4)), 1)
    with pytest.raises(O.ValidationError, match="top_k must be >= 1"):
        O.gate_forward(np.zeros((2, 4)), np.zeros((4, 4)), 0)
    with pytest.raises(O.ValidationError, match="top_k must be <= num_experts"):
        O.gate_forward(np.zeros((2, 4)), np.zeros((4, 4)), 5)


def test_gate_bit_exact_vs_reference(ref):
    rng = np.random.default_rng(5)
    for S, H, E, k in ((7, 5, 4, 2), (64, 33, 16, 4), (300, 64, 64, 6)):
        x = rng.uniform(-1, 1, (S, H))
        wg = rng.uniform(-0.1, 0.1, (H, E))
        g = O.gate_forward(x, wg, k)
        top, w = ref.gate_forward(x, wg, k)
        assert np.array_equal(g.top_experts, top)
        assert np.array_equal(g.combine_weights, w)


# ---------------------------------------------------------------- PFT pins
def test_pft_hand_trace():
    # test_pft.cpp:52-62
    p = O.pft_construct(2, 2, 4, 1, [0, 1, 0, 0], [0.9, 0.8, 0.5, 0.7])
    assert p.token_ids.tolist() == [0, 3, 1]
    assert p.expert_ids.tolist() == [0, 0, 1]
    assert p.tokens_per_expert.tolist() == [2, 1]
    assert p.combine_weights.tolist() == [0.9, 0.7, 0.8]


def test_pft_tie_drop_and_no_drop():
    # test_pft.cpp:64-79
    assert O.pft_construct(2, 1, 3, 1, [0, 0, 0], [0.4] * 3).token_ids.tolist() == [0, 1]
    p = O.pft_construct(4, 3, 4, 1, [1, 0, 1, 2], [0.6, 0.5, 0.4, 0.3])
    assert p.token_ids.tolist() == [1, 0, 2, 3]
    assert p.expert_ids.tolist() == [0, 1, 1, 2]


def test_pft_errors():
    # test_pft.cpp:81-89
    with pytest.raises(O.ValidationError, match="max_token_count must be >= 1"):
        O.pft_construct(0, 1, 2, 1, [0, 0], [0.5, 0.5])
    with pytest.raises(O.ValidationError):
        O.pft_construct(1, 1, 1, 2, [0, 0], [0.5, 0.5])
    with pytest.raises(O.IndexError_):
        O.pft_construct(1, 1, 2, 1, [0, 3], [0.5, 0.5])
    with pytest.raises(O.DimensionError):
        O.pft_construct(1, 1, 1, 1, [0, 0], [0.5, 0.5])


def _weight_ranking(cap, E, S, k, top, w):
    # independent construction of test_pft.cpp:21-48
    flat = S * k
    order = sorted(range(flat), key=lambda f: (-w[f], f))
    seen = [0] * E
    rank = [0] * flat
    for f in order:
        rank[f] = seen[top[f]]
        seen[top[f]] += 1
    tid, eid, cw = [], [], []
    for e in range(E):
        for f in range(flat):
            if top[f] == e and rank[f] < cap:
                tid.append(f // k)
                eid.append(e)
                cw.append(w[f])
    return tid, eid, cw


def test_pft_equals_weight_ranking_50_trials(ref):
    # test_pft.cpp:91-124, and bit-equality with the compiled reference
    rng = O.Rng(2024)
    for _ in range(50):
        S = 1 + rng.below(24)
        E = 1 + rng.below(6)
        k = 1 + rng.below(min(E, 4))
        cap = 1 + rng.below(S + 2)
        top, w = [], []
        pool = list(range(E))
        for t in range(S):
            for j in range(k):
                pick = j + rng.below(E - j)
                pool[j], pool[pick] = pool[pick], pool[j]
            for j in range(k):
                top.append(pool[j])
                w.append(rng.uniform())
        a = O.pft_construct(cap, E, S, k, top, w)
        tid, eid, cw = _weight_ranking(cap, E, S, k, top, w)
        assert a.token_ids.tolist() == tid and a.expert_ids.tolist() == eid
        assert a.combine_weights.tolist() == cw
        r = ref.pft_construct(cap, E, S, k, top, w)
        assert np.array_equal(a.token_ids, r[0]) and np.array_equal(a.expert_ids, r[1])
        assert np.array_equal(a.combine_weights, r[2]) and np.array_equal(a.tokens_per_expert, r[3])


def test_gather_scatter_hand_trace():
    # test_pft.cpp:126-145
    src = np.arange(1, 7, dtype=float).reshape(3, 2)
    g = O.gather_rows(src, [2, 0, 2])
    assert g[0, 0] == 5.0 and g[1, 0] == 1.0
    out = O.scatter_combine(g, [2, 0, 2], [0.5, 1.0, 0.25], 3)
    assert out[0].tolist() == [1.0, 2.0] and out[1, 0] == 0.0
    assert abs(out[2, 0] - 3.75) < 1e-12
    with pytest.raises(O.IndexError_):
        O.gather_rows(src, [3])
    with pytest.raises(O.IndexError_):
        O.scatter_combine(g, [0, 1, 5], [1, 1, 1], 3)
    with pytest.raises(O.DimensionError):
        O.scatter_combine(g, [0, 1], [1, 1], 3)


# ---------------------------------------------------------------- dispatch pins
def _tagged(tags, cols):
    return np.array([[t * 10.0 + j for j in range(cols)] for t in tags])


def _two_worker_pfts():
    p0 = O.Pft(np.array([0, 1, 2, 3]), np.array([0, 2, 2, 3]), np.array([1, 0, 2, 1]),
               np.ones(4), _tagged([1, 2, 3, 4], 2))
    p1 = O.Pft(np.array([0, 1, 2]), np.array([0, 1, 2]), np.array([1, 1, 1, 0]),
               np.ones(3), _tagged([5, 6, 7], 2))
    return [p0, p1]


def test_dispatch_regroup_hand_trace():
    # test_pf_pipeline.cpp:34-72
    led = O.Ledger()
    d = O.pf_dispatch([0, 0], _two_worker_pfts(), 4, led)
    assert d.row_counts.tolist() == [[1, 3], [2, 1]]
    assert d.recv_per_expert[0].tolist() == [2, 1] and d.recv_per_expert[1].tolist() == [3, 1]
    assert np.array_equal(d.expert_input[0], _tagged([1, 5, 6], 2))
    assert np.array_equal(d.expert_input[1], _tagged([2, 3, 7, 4], 2))
    assert d.arrival_to_grouped[1].tolist() == [0, 1, 3, 2]
    assert led.get("dispatch_counts")[1] == 32
    assert led.get("dispatch_rows")[1] == 20 and led.get("dispatch_rows")[0] == 8


def test_identity_round_trip():
    # test_pf_pipeline.cpp:74-97
    pfts = _two_worker_pfts()
    d = O.pf_dispatch([0, 1], pfts, 4)
    out = O.pf_combine([0, 1], d, d.expert_input, pfts, [4, 3])
    assert np.array_equal(out[0], pfts[0].x) and np.array_equal(out[1], pfts[1].x)


def test_grouped_mlp_vs_reference(ref):
    rng = O.Rng(11)
    w = O.make_layer_weights(rng, 2, 3, 4)
    inp = np.array([rng.uniform(-1.0, 1.0) for _ in range(15)]).reshape(5, 3)
    out = O.grouped_expert_mlp(inp, [2, 3], w, 0)
    L = ref.Layer(w.gate, w.w1, w.w2)
    assert np.array_equal(out, L.grouped_expert_mlp(inp, [2, 3], 0))
    with pytest.raises(O.CountMismatch):
        O.grouped_expert_mlp(inp, [2, 2], w, 0)


def _random_instance(rng: O.Rng, W, max_seq=24):
    E = W * (1 + rng.below(3))
    k = 1 + rng.below(min(E, 4))
    H = 2 + rng.below(5)
    F = 2 + rng.below(5)
    w = O.make_layer_weights(rng, E, H, F)
    S = 2 + rng.below(max_seq - 1)
    cap = 1 + rng.below(4) if rng.below(2) == 0 else S * k
    toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
    return w, E, k, cap, toks


@pytest.mark.parametrize("W", [1, 2, 4])
def test_pf_moe_forward_bit_exact_vs_reference(ref, W):
    rng = O.Rng(31337 + W)
    for _ in range(6):
        w, E, k, cap, toks = _random_instance(rng, W)
        node_of = [i // 2 for i in range(W)]
        led = O.Ledger()
        got = O.pf_moe_forward(list(toks), w, E, k, cap, node_of, led)
        L = ref.Layer(w.gate, w.w1, w.w2)
        want, rled = L.pf_moe_forward(toks, k, cap, node_of)
        nc = L.pf_moe_forward_noncopy(toks, k, cap, node_of)  # the CPU-baseline entry (bench.py)
        for i in range(W):
            assert np.array_equal(got[i], want[i])
            assert np.array_equal(nc[i], want[i])
        for kind in ("dispatch_counts", "dispatch_rows", "combine_rows"):
            assert led.get(kind) == rled[kind], kind
        # the padded GShard path agrees within the reference's own 1e-12
        pad = L.padded_moe_forward(toks, k, cap, node_of)
        assert np.max(np.abs(pad - np.array(got))) < 1e-12


@pytest.mark.parametrize("W", [2, 4, 8])
def test_dispatch_layout_bit_exact_vs_reference(ref, W):
    rng = O.Rng(808 + W)
    for _ in range(4):
        w, E, k, cap, toks = _random_instance(rng, W)
        _, pfts, disp, _ = O.pf_moe_forward(list(toks), w, E, k, cap, return_pfts=True)
        L = ref.Layer(w.gate, w.w1, w.w2)
        ei, rpe, rc, _, _ = L.dispatch(toks, k, cap)
        for j in range(W):
            assert np.array_equal(disp.expert_input[j], ei[j])
            assert np.array_equal(disp.recv_per_expert[j], rpe[j])
        assert np.array_equal(disp.row_counts, rc)
        # rbd dispatch buffers are the plain buffers bit for bit (rbd.hpp:50)
        ei2, _, _, _, _ = L.dispatch(toks, k, cap, rbd=True, seed=5)
        for j in range(W):
            assert np.array_equal(ei2[j], ei[j])


# ---------------------------------------------------------------- RBD pins
def test_select_pilots_vs_reference(ref):
    rng = O.Rng(404)
    for W in (2, 4, 8):
        w, E, k, cap, toks = _random_instance(rng, W)
        _, pfts, _, _ = O.pf_moe_forward(list(toks), w, E, k, cap, return_pfts=True)
        for node_of in (list(range(W)), [i // 2 for i in range(W)]):
            for s, p in enumerate(pfts):
                seed = O.salt_seed(99, s, 0)
                got = O.select_pilots(p, node_of, E, seed).pilot_mask
                want = ref.select_pilots(p.token_ids, p.expert_ids, p.combine_weights,
                                         p.tokens_per_expert, E, node_of, seed)
                assert np.array_equal(got, want)


def test_rbd_merge_hand_trace():
    # test_rbd.cpp:209-233: one token, copies to experts 2 and 3, w = .6/.4
    p = O.Pft(np.array([0, 0]), np.array([2, 3]), np.array([0, 0, 1, 1]), np.array([0.6, 0.4]))
    for seed in (31, 32, 33):
        plan = O.select_pilots(p, [0, 0, 1, 1], 4, seed)
        assert plan.pilot_mask.sum() == 1
        y = np.array([[10.0, 20.0], [100.0, 200.0]])
        out = O.rbd_combine_from_outputs(p, plan, y, 1)
        assert np.allclose(out[0], [0.6 * 10 + 0.4 * 100, 0.6 * 20 + 0.4 * 200], rtol=1e-12)


@pytest.mark.parametrize("per_gpu", [True, False])
def test_rbd_moe_forward_bit_exact_vs_reference(ref, per_gpu):
    rng = O.Rng(1717 + per_gpu)
    for _ in range(5):
        W = 2 * (1 + rng.below(4))
        w, E, k, cap, toks = _random_instance(rng, W)
        node_of = list(range(W)) if per_gpu else [i // 2 for i in range(W)]
        seed = rng.next_u64()
        got = O.rbd_moe_forward(list(toks), w, E, k, cap, seed, node_of)
        L = ref.Layer(w.gate, w.w1, w.w2)
        want, _ = L.rbd_moe_forward(toks, k, cap, seed, node_of)
        for i in range(W):
            assert np.array_equal(got[i], want[i])


def test_redundancy_definitions(ref):
    # test_rbd.cpp:321-340
    p = O.Pft(np.array([0, 1, 0, 1]), np.array([0, 0, 1, 1]), np.array([2, 2]), np.full(4, 0.5))
    assert O.redundancy_counts_internode(p, 0, [0, 0]) == (0, 0)
    c, g = O.redundancy_counts_internode(p, 1, [0, 0])
    assert 1 - g / c == 0.5
    nodes = [e // 4 for e in range(16)]
    assert abs(O.sample_redundancy(O.Rng(2025), 300, 4, nodes)
               - ref.sample_redundancy(2025, 300, 4, nodes)) == 0.0


# ---------------------------------------------------------------- SSMB pins
def test_ssmb_vs_reference(ref):
    rng = O.Rng(11)
    for S, G in ((9, 1), (9, 2), (17, 4), (16, 8)):
        E = 4 + rng.below(5)
        k = 1 + rng.below(3)
        H = 3 + rng.below(4)
        F = 2 + rng.below(5)
        w = O.make_layer_weights(rng, E, H, F)
        x = np.array([rng.uniform(-1.0, 1.0) for _ in range(S * H)]).reshape(S, H)
        got = O.ssmb_forward(x, G, w, E, k, S * k)
        L = ref.Layer(w.gate, w.w1, w.w2)
        assert np.array_equal(got, L.ssmb_forward(x, G, k, S * k))
        # test_ssmb.cpp:61-77: no drops => sharded == unsharded exactly
        assert np.array_equal(got, O.pf_moe_forward([x], w, E, k, S * k)[0])
