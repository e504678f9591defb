"""BASELINE.json configs 2-5 at (or near) full size, bf16, through the C-ABI
layer.  The oracle cannot run these sizes end to end in seconds, so parity is
checked on a seeded SAMPLE of tokens: routing of the sampled rows comes from
the pinned oracle gate (moe_oracle.gate_forward, gating.cpp:14-57), the
expert FFNs of those rows are evaluated in fp64 torch on the same bf16
weights (pf_pipeline.cpp:83-105), and the weighted sum is the reference's
combine (pf_pipeline.cpp:107-135).  A misrouted copy, a lost or duplicated
row, or a wrong weight shows up as an O(1) error; the stated tolerance is
the bf16 one of test_gpu_layer.py (normwise < 1e-2 over the sample).

Inputs are on the bf16-exact grid (tokens 2^-7, gate 2^-10) so the fp32
logits — and therefore the routing — are exact.  Weights are generated on
the device (config 3 is 15 GB of bf16 expert weights)."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from tests.gpu_util import host, norm_rel

pytestmark = pytest.mark.gpu


def _weights(E, H, F, ns, Fs, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = lambda *s: ((torch.rand(*s, device="cuda", generator=g) - 0.5) * 0.2).to(torch.bfloat16)  # noqa: E731
    w1, w2 = u(E, H, F), u(E, F, H)
    sw1 = u(ns, H, Fs) if ns else None
    sw2 = u(ns, Fs, H) if ns else None
    return w1, w2, sw1, sw2


def _grid_tokens(n, H, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randint(-128, 129, (n, H), device="cuda", generator=g).to(torch.float32) / 128).to(torch.bfloat16)


def _grid_gate(H, E, seed, zipf=None):
    rng = np.random.default_rng(seed)
    gate = np.round(rng.uniform(-0.1, 0.1, (H, E)) * 1024) / 1024
    if zipf is not None:  # token feature 0 is pinned to 1.0: a per-expert logit bias
        p = 1.0 / np.arange(1, E + 1) ** zipf
        gate[0] = np.round(np.log(p / p.max()) * 1024) / 1024
        gate[0, E - 4:] = -16.0  # four experts never chosen: empty groups
    return torch.from_numpy(gate).to(torch.bfloat16).double().numpy()  # what the device holds


def _sampled_reference(x, gate, w1, w2, sw1, sw2, k, rows):
    """fp64 output of the sampled rows (see module docstring)."""
    xs = x[rows].double()
    g = O.gate_forward(xs.cpu().numpy(), gate, k)
    y = torch.zeros_like(xs)
    for j in range(k):
        for e in np.unique(g.top_experts[:, j]):
            sel = np.nonzero(g.top_experts[:, j] == e)[0]
            h = torch.relu(xs[sel] @ w1[e].double()) @ w2[e].double()
            wt = torch.from_numpy(g.combine_weights[sel, j]).to(xs)
            y[sel] += wt[:, None] * h
    if sw1 is not None:
        for s in range(sw1.shape[0]):
            y += torch.relu(xs @ sw1[s].double()) @ sw2[s].double()
    return host(y)


def _run(W, S, E, k, H, F, ns, Fs, mode=0, zipf=None, n_sample=64, seed=0):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, W, -1)
    w1, w2, sw1, sw2 = _weights(E, H, F, ns, Fs, seed)
    gate = _grid_gate(H, E, seed + 1, zipf)
    x = _grid_tokens(W * S, H, seed + 2)
    if zipf is not None:
        x[:, 0] = 1.0
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k,
                   max_tokens=S, dtype=capi.BF16,
                   gate=torch.from_numpy(gate).to(torch.bfloat16).cuda(), w1=w1, w2=w2, sw1=sw1, sw2=sw2,
                   dispatch_mode=mode, seed=seed)
    out = L.forward(x.view(W, S, H)).view(W * S, H)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(seed).choice(W * S, n_sample, replace=False))
    want = _sampled_reference(x, gate, w1, w2, sw1, sw2, k, rows)
    got = host(out[torch.from_numpy(rows).cuda()])
    assert np.isfinite(got).all()
    assert norm_rel(got, want) < 1e-2, norm_rel(got, want)
    return L, x, out


@pytest.mark.parametrize("mode", [0, 1])
def test_config2_deepseek_moe_ep8(mode):
    """Config 2: 64 experts top-6 + 2 shared, 2048/1408, 16K tokens per GPU,
    8 expert-parallel workers (driven from one process), plain and RBD."""
    L, _, _ = _run(8, 16384, 64, 6, 2048, 1408, 2, 1408, mode=mode, n_sample=48)
    led = L.ledger()
    if mode == 1:  # RBD moves fewer off-rank rows than there are off-rank copies
        assert 0 < led["unique_rows_offrank"] < led["copies_offrank"]


def test_config3_deepseek_v3_layer():
    """Config 3: 256 routed experts top-8 + 1 shared, d_model 7168, d_ff 2048,
    8K tokens on one GPU."""
    _run(1, 8192, 256, 8, 7168, 2048, 1, 2048, n_sample=32)


def test_config3_expert_parallel():
    """Config 3 shape, 8 expert-parallel workers (32 experts each), 1K tokens
    per worker, RBD."""
    _run(8, 1024, 256, 8, 7168, 2048, 1, 2048, mode=1, n_sample=32)


@pytest.mark.parametrize("mode", [0, 1])
def test_config5_zipf_skewed_routing(mode):
    """Config 5: 128 experts top-8 with Zipf-imbalanced gate logits, 64K tokens
    over 8 workers — empty and oversized expert groups."""
    L, x, _ = _run(8, 8192, 128, 8, 1024, 512, 0, 0, mode=mode, zipf=1.2, n_sample=64)
    led = L.ledger()
    assert led["routed_copies"] == 8 * 8192 * 8


@pytest.mark.parametrize("G", [2, 4])
def test_config4_ssmb_32k(G):
    """Config 4: a 32K-token sequence split across G sequence shards, 160
    experts top-6, d_model 5120, d_ff 1536 (ssmb.cpp:12-46); no drops, so
    every row equals the unsharded layer's."""
    from paper_2508_13337_b200 import capi
    S, E, k, H, F = 32768, 160, 6, 5120, 1536
    ctx = capi.Context(0, G, -1)
    w1, w2, _, _ = _weights(E, H, F, 0, 0, 5)
    gate = _grid_gate(H, E, 6)
    x = _grid_tokens(S, H, 7)
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k,
                   max_tokens=S // G, dtype=capi.BF16, gate=torch.from_numpy(gate).to(torch.bfloat16).cuda(),
                   w1=w1, w2=w2, ssmb=True)
    out = L.ssmb_forward(x)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(G).choice(S, 48, replace=False))
    rows[0], rows[-1] = 0, S - 1  # first and last shard
    want = _sampled_reference(x, gate, w1, w2, None, None, k, rows)
    got = host(out[torch.from_numpy(rows).cuda()])
    assert norm_rel(got, want) < 1e-2, norm_rel(got, want)
