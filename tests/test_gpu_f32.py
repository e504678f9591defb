"""The F32 instantiation (fp32 operands in the reference's operation order:
ascending-h logits, ascending-p expert GEMMs, ascending copies in the
combine; exact fp32 products accumulated in fp64, each result rounded once to
fp32) against the fp64 oracle, at the fp32 bar the reference itself uses between pipelines:
max_rel_diff (floor 1, matrix.hpp:47-62) <= 1e-5 (verify.cpp:117).  Inputs
on the bf16-exact grid, so fp32 logits — and routing — are exact."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from tests.gpu_util import dev, grid_gate, grid_tokens, host, max_rel_diff

pytestmark = pytest.mark.gpu


def _weights(rng, E, H, F):
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731  what the device holds
    return O.LayerWeights(grid_gate(rng, H, E), f32(rng.uniform(-0.1, 0.1, (E, H, F))),
                          f32(rng.uniform(-0.1, 0.1, (E, F, H))))


def test_gate_and_mlp_f32():
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    rng = np.random.default_rng(3)
    E, k, H, F, S = 64, 6, 256, 96, 300
    w = _weights(rng, E, H, F)
    x = grid_tokens(rng, S, H)
    top, wt = ctx.gate_forward(dev(x, torch.float32), dev(w.gate, torch.float32), k)
    g = O.gate_forward(x, w.gate, k)
    assert np.array_equal(host(top), g.top_experts)
    assert np.max(np.abs(host(wt) - g.combine_weights)) < 1e-6  # fp32 logits on the grid are exact
    rpe = np.array([37, 0, 100, 163], np.int32)
    inp = rng.uniform(-1, 1, (300, H)).astype(np.float32).astype(np.float64)
    got = host(ctx.grouped_mlp(dev(inp, torch.float32), torch.from_numpy(rpe).cuda(), dev(w.w1[:4], torch.float32),
                               dev(w.w2[:4], torch.float32)))
    want = O.grouped_expert_mlp(inp, rpe, w, 0)
    assert max_rel_diff(got, want) <= 1e-5


@pytest.mark.parametrize("W,mode", [(1, 0), (2, 0), (4, 0), (2, 1), (4, 1)])
def test_layer_f32_vs_oracle(W, mode):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    rng = np.random.default_rng(10 + W + mode)
    E, k, H, F, S = 16 * W, 4, 128, 64, 200
    w = _weights(rng, E, H, F)
    x = grid_tokens(rng, W, S, H)
    t = torch.float32
    for cap in (S * k, int(np.ceil(1.25 * S * k / E))):
        L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap, max_tokens=S,
                       dtype=capi.F32, gate=dev(w.gate, t), w1=dev(w.w1, t), w2=dev(w.w2, t), dispatch_mode=mode,
                       seed=5)
        got = host(L.forward(dev(x, t)))
        want = O.pf_moe_forward(list(x), w, E, k, cap) if mode == 0 else \
            O.rbd_moe_forward(list(x), w, E, k, cap, 5, list(range(W)))
        for i in range(W):
            assert max_rel_diff(got[i], want[i]) <= 1e-5, (i, cap, max_rel_diff(got[i], want[i]))


def test_c1_shape_f32():
    """C1 (BASELINE configs[0] is fp32): 64 experts top-6 + 2 shared, d_model
    2048, d_ff 1408, on a 512-token slice (the SIMT F32 kernels are the
    parity instantiation, not the performance path)."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    rng = np.random.default_rng(1)
    E, k, H, F, S, ns = 64, 6, 2048, 1408, 512, 2
    w = _weights(rng, E, H, F)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    sw1, sw2 = f32(rng.uniform(-0.1, 0.1, (ns, H, F))), f32(rng.uniform(-0.1, 0.1, (ns, F, H)))
    x = grid_tokens(rng, S, H)
    t = torch.float32
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                   dtype=capi.F32, gate=dev(w.gate, t), w1=dev(w.w1, t), w2=dev(w.w2, t), sw1=dev(sw1, t),
                   sw2=dev(sw2, t))
    got = host(L.forward(dev(x[None], t)))[0]
    want = O.moe_layer_with_shared(x, w, E, k, S * k, sw1, sw2, exact=False)
    assert max_rel_diff(got, want) <= 1e-5, max_rel_diff(got, want)
