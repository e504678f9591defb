"""GPU parity of the split expert-parallel operators (the reference's SPMD
operator API: pf_dispatch / pf_combine / select_pilots / rbd_dispatch /
rbd_combine, pf_pipeline.hpp:34-45, rbd.hpp:46-88) against the compiled
reference (oracle/_ref) on identical packed buffers.

Bars: dispatch layouts, counts, arrival maps and pilot masks bit-exact;
F64 combine outputs bit-exact (the reference's axpy/scale order); BF16 rows
are pure copies (bit-exact) and the combine within bf16 rounding."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from tests import rbd_flat
from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu


def _ctx(W):
    from paper_2508_13337_b200 import capi
    return capi.Context(0, W, -1)


def _i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def _pfts(ref, toks, gate, E, k, cap):
    """The reference's own gate + pft_construct + gather per worker."""
    out = []
    for x in toks:
        top, w = ref.gate_forward(x, gate, k)
        tid, eid, cw, tpe = ref.pft_construct(cap, E, x.shape[0], k, top, w)
        out.append((tid, eid, cw, tpe, x[tid]))
    return out


def _trial(rng, W, max_e=4, max_dim=9, max_s=40):
    E = W * (1 + rng.below(max_e))
    k = 1 + rng.below(min(E, 4))
    H = 2 + rng.below(max_dim)
    F = 2 + rng.below(max_dim)
    S = 2 + rng.below(max_s)
    cap = 1 + rng.below(3) if rng.below(2) == 0 else S * k
    w = O.make_layer_weights(rng, E, H, F)
    toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
    return E, k, H, F, S, cap, w, toks


def test_pf_dispatch_hand_trace():
    """test_pf_pipeline.cpp:34-72: two workers, tagged rows."""
    ctx = _ctx(2)
    tag = lambda tags: np.array([[t * 10.0 + j for j in range(2)] for t in tags])  # noqa: E731
    x0, x1 = tag([1, 2, 3, 4]), tag([5, 6, 7])
    tpe = _i32([[1, 0, 2, 1], [1, 1, 1, 0]])
    ei, rpe, _, _, a2g = ctx.pf_dispatch(0, 2, 4, [dev(x0), dev(x1)], [_i32([0, 2, 2, 3]), _i32([0, 1, 2])], tpe)
    assert np.array_equal(host(ei[0]), tag([1, 5, 6]))
    assert np.array_equal(host(ei[1]), tag([2, 3, 7, 4]))
    assert host(rpe).tolist() == [[2, 1], [3, 1]]
    assert host(a2g[1]).tolist() == [0, 1, 3, 2]
    assert host(a2g[0]).tolist() == [0, 1, 2]


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_pf_dispatch_combine_vs_reference(ref, W):
    ctx = _ctx(W)
    rng = O.Rng(8100 + W)
    for _ in range(6):
        E, k, H, F, S, cap, w, toks = _trial(rng, W)
        pf = _pfts(ref, toks, w.gate, E, k, cap)
        tpe = _i32(np.stack([p[3] for p in pf]))
        L = ref.Layer(w.gate, w.w1, w.w2)
        want_ei, want_rpe, want_rc, _, _ = L.dispatch(toks, k, cap)
        ei, rpe, dr, dw, a2g = ctx.pf_dispatch(0, H, E, [dev(p[4]) for p in pf], [_i32(p[1]) for p in pf], tpe)
        El = E // W
        rc = np.zeros((W, W), np.int64)
        for s, p in enumerate(pf):
            for e in range(E):
                rc[s, e // El] += p[3][e]
        assert np.array_equal(rc, want_rc)
        assert np.array_equal(host(rpe), want_rpe)
        for j in range(W):
            assert np.array_equal(host(ei[j]), want_ei[j]), j   # layout bit-exact
        # arrival_to_grouped: arrivals at j are source-ascending, packed order
        for j in range(W):
            arr = []
            for s, p in enumerate(pf):
                d = host(dr[s])[:len(p[0])]
                arr += host(dw[s])[:len(p[0])][d == j].tolist()
            assert host(a2g[j]).tolist() == arr
        # pf_combine over the reference's grouped expert MLP outputs: bit-exact
        eo = [L.grouped_expert_mlp(want_ei[j], want_rpe[j], j * El) for j in range(W)]
        got = ctx.pf_combine(0, H, E, [dev(e) for e in eo], tpe, [_i32(p[0]) for p in pf],
                             [_i32(p[1]) for p in pf], [dev(p[2]) for p in pf], [S] * W)
        want, _ = L.pf_moe_forward(toks, k, cap)
        for s in range(W):
            assert np.array_equal(host(got[s]), want[s]), s


@pytest.mark.parametrize("W,gpn", [(1, 1), (2, 1), (4, 1), (8, 1), (4, 2), (8, 2), (8, 4)])
def test_select_pilots_and_rbd_vs_reference(ref, W, gpn):
    ctx = _ctx(W)
    rng = O.Rng(9200 + 10 * W + gpn)
    node_of = [w // gpn for w in range(W)]
    for trial in range(5):
        E, k, H, F, S, cap, w, toks = _trial(rng, W)
        seed = 1000 + trial
        pf = _pfts(ref, toks, w.gate, E, k, cap)
        L = ref.Layer(w.gate, w.w1, w.w2)
        # select_pilots per worker, salted as rbd_moe_forward does (rbd.cpp:372-375)
        masks, pofs = [], []
        for s, p in enumerate(pf):
            sd = ref.salt_seed(seed, s, 0)
            want = ref.select_pilots(p[0], p[1], p[2], p[3], E, node_of, sd)
            m, po = ctx.select_pilots(_i32(p[0]), _i32(p[1]), S, k, E, W, gpn, sd)
            assert np.array_equal(host(m), want), (s, trial)
            masks.append(m)
            pofs.append(po)
        # rbd_dispatch: expert_input bit-identical to the reference's (== pf_dispatch)
        want_ei, want_rpe, _, want_pm, _ = L.dispatch(toks, k, cap, node_of=node_of, rbd=True, seed=seed)
        tpe = _i32(np.stack([p[3] for p in pf]))
        ei, rpe, dr, dw, po = ctx.rbd_dispatch(0, H, E, gpn, [dev(p[4]) for p in pf], [_i32(p[0]) for p in pf],
                                               [_i32(p[1]) for p in pf], [S] * W, k, tpe, masks)
        assert np.array_equal(host(rpe), want_rpe)
        for j in range(W):
            assert np.array_equal(host(ei[j]), want_ei[j]), j
        assert np.array_equal(np.concatenate([host(m) for m in masks]), want_pm[:sum(len(p[0]) for p in pf)])
        # rbd_combine: merged at the landing workers, added at the sources — bit-exact F64
        El = E // W
        eo = [L.grouped_expert_mlp(want_ei[j], want_rpe[j], j * El) for j in range(W)]
        nb = [len(p[0]) for p in pf]
        flat, s1 = rbd_flat.flatten(W, [host(m) for m in masks], [host(x)[:n] for x, n in zip(po, nb)],
                                    [host(x)[:n] for x, n in zip(dr, nb)], [host(x)[:n] for x, n in zip(dw, nb)],
                                    [p[2] for p in pf], [p[0] for p in pf], [S] * W)
        got = ctx.rbd_combine(0, H, [dev(e) for e in eo], flat, [S] * W)
        want, _ = L.rbd_moe_forward(toks, k, cap, seed, node_of=node_of)
        for s in range(W):
            assert np.array_equal(host(got[s]), want[s]), (s, trial)


def test_rbd_dispatch_plan_mismatch():
    from paper_2508_13337_b200 import capi
    ctx = _ctx(2)
    # token 0 -> experts 0, 1 (both on worker 0): one group; mark both as pilots
    x = dev(np.ones((2, 4)))
    tpe = _i32([[1, 1, 0, 0], [0, 0, 0, 0]])
    masks = [torch.tensor([1, 1], dtype=torch.uint8, device="cuda"), torch.zeros(1, dtype=torch.uint8, device="cuda")]
    with pytest.raises(capi.XmoeError) as ei:
        ctx.rbd_dispatch(0, 4, 4, 1, [x, dev(np.ones((0, 4)))], [_i32([0, 0]), _i32([0])[:0]],
                         [_i32([0, 1]), _i32([0])[:0]], [1, 1], 2, tpe, masks)
    assert ei.value.kind == "PlanMismatch"


@pytest.mark.parametrize("W", [2, 4])
def test_split_ops_bf16_layout(ref, W):
    """BF16 rows are pure copies: the grouped buffers equal the reference's
    (computed on the same bf16 values) exactly."""
    ctx = _ctx(W)
    rng = np.random.default_rng(40 + W)
    E, k, H, S = 8 * W, 4, 64, 300
    gate = np.round(rng.uniform(-0.1, 0.1, (H, E)) * 1024) / 1024
    toks = np.round(rng.uniform(-1, 1, (W, S, H)) * 128) / 128
    w1 = rng.uniform(-0.1, 0.1, (E, H, 8))
    w2 = rng.uniform(-0.1, 0.1, (E, 8, H))
    pf = _pfts(ref, toks, gate, E, k, S * k)
    L = ref.Layer(gate, w1, w2)
    want_ei, _, _, _, _ = L.dispatch(toks, k, S * k)
    tpe = _i32(np.stack([p[3] for p in pf]))
    ei, _, _, _, _ = ctx.pf_dispatch(1, H, E, [dev(p[4], torch.bfloat16) for p in pf], [_i32(p[1]) for p in pf], tpe)
    for j in range(W):
        assert np.array_equal(host(ei[j]), want_ei[j])


@pytest.mark.parametrize("W,gpn", [(2, 1), (4, 2)])
def test_redundancy_counts_vs_reference(ref, W, gpn):
    """internode_redundancy_counts / redundancy_rate (rbd.cpp:390-442) on the
    device, summed over workers (acceptance.cpp:167-172)."""
    ctx = _ctx(W)
    rng = O.Rng(77 + W)
    E, k, H, F, S, cap, w, toks = _trial(rng, W, max_s=64)
    pf = _pfts(ref, toks, w.gate, E, k, cap)
    El = E // W
    expert_node = _i32([(e // El) // gpn for e in range(E)])
    for s, p in enumerate(pf):
        node = s // gpn
        pairs_all = {(int(t), (int(e) // El) // gpn) for t, e in zip(p[0], p[1])}
        pairs_off = {(t, n) for t, n in pairs_all if n != node}
        copies_off = sum(1 for e in p[1] if (int(e) // El) // gpn != node)
        c, g = ctx.route_pairs(_i32(p[0]), _i32(p[1]), expert_node, W // gpn, S, skip_node=node)
        assert (c, g) == (copies_off, len(pairs_off))
        c2, g2 = ctx.route_pairs(_i32(p[0]), _i32(p[1]), expert_node, W // gpn, S)
        assert (c2, g2) == (len(p[0]), len(pairs_all))
