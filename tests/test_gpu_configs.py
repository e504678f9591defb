"""BASELINE.json configs C1-C5 at FULL size, bf16, through the C-ABI layer
(W workers driven from one process on one GPU for the expert-parallel
shapes), on the bench's own inputs (the reference generator drawn on the
device, paper_2508_13337_b200/configs.py).

Bit-exact at full size, against an independent torch restatement of the
reference's routing on the SAME device-held values (gating.cpp:14-57: on the
bf16-exact grid every logit is an exact multiple of 2^-17 in fp64, so the
reference's probability order is the logit order with ties to the lower id;
pft.cpp:12-60 dropless: experts ascending, tokens ascending):
  * every worker's top_experts, tokens_per_expert, token_ids, expert_ids;
  * every owner's grouped expert input (pf_pipeline.cpp:47-73 order), row for
    row (a pure copy of bf16 tokens).
Outputs: a seeded sample of tokens against fp64 torch over the same bf16
weights (normwise < 1e-2, the bf16 bar of test_gpu_layer.py).
C5 additionally asserts the skew SURVEY §8(d) asks for (>= 1 empty expert,
max load >= 4x the mean) and C4 that SSMB composed with EP equals the
replicated-expert SSMB bit for bit (identical drop sets, §8(e))."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from tests.gpu_util import host, norm_rel

pytestmark = pytest.mark.gpu


def _inputs(cfg_name, W, S):
    from paper_2508_13337_b200 import capi, configs
    cfg = dict(configs.CONFIGS[cfg_name])
    ctx = capi.Context(0, W, -1)
    gate, w1, w2, sw1, sw2, x = configs.device_inputs(ctx, capi, cfg, 0, 1, W * S, 0, torch)
    return ctx, cfg, gate, w1, w2, sw1, sw2, x


def _routing(x, gate, k):
    """Reference routing of bf16 grid tokens: exact fp64 logits, stable order."""
    lg = x.double() @ gate.double()
    order = torch.sort(-lg, dim=1, stable=True).indices
    return order[:, :k].to(torch.int32)


def _pft(top, E):
    """Dropless pft_construct: packed rows grouped by expert, tokens ascending."""
    S, k = top.shape
    flat = top.reshape(-1).long()
    order = torch.sort(flat, stable=True).indices
    return (order // k).to(torch.int32), flat[order].to(torch.int32), torch.bincount(flat, minlength=E).to(torch.int32)


def _check_routing_and_layout(L, x, gate, W, S, E, k):
    H = x.shape[1]
    El = E // W
    tpes, tids = [], []
    for w in range(W):
        xs = x[w * S:(w + 1) * S]
        top = _routing(xs, gate, k)
        tid, eid, tpe = _pft(top, E)
        assert torch.equal(L.inspect("top_experts", w).view(S, k), top), w
        assert torch.equal(L.inspect("tokens_per_expert", w), tpe), w
        assert torch.equal(L.inspect("token_ids", w), tid), w
        assert torch.equal(L.inspect("expert_ids", w), eid), w
        tpes.append(tpe.long())
        tids.append(tid.long())
    tpe_all = torch.stack(tpes)                      # [W, E]
    starts = torch.cumsum(tpe_all, 1) - tpe_all      # packed segment start per (src, e)
    for j in range(W):
        idx = []
        for le in range(El):
            e = j * El + le
            for s in range(W):
                a, n = int(starts[s, e]), int(tpe_all[s, e])
                idx.append(s * S + tids[s][a:a + n])
        idx = torch.cat(idx)
        got = L.inspect("expert_input", j, limit=idx.numel() * H).view(-1, H)
        assert torch.equal(got, x[idx]), j          # grouped layout bit-exact at full size
    return tpe_all


def _sampled_reference(x, gate, w1, w2, sw1, sw2, k, rows):
    """fp64 output of the sampled rows over the same bf16 weights."""
    xs = x[rows].double()
    g = O.gate_forward(xs.cpu().numpy(), gate.double().cpu().numpy(), k)
    y = torch.zeros_like(xs)
    for j in range(k):
        for e in np.unique(g.top_experts[:, j]):
            sel = np.nonzero(g.top_experts[:, j] == e)[0]
            h = torch.relu(xs[sel] @ w1[e].double()) @ w2[e].double()
            y[sel] += torch.from_numpy(g.combine_weights[sel, j]).to(xs)[:, None] * h
    if sw1 is not None:
        for s in range(sw1.shape[0]):
            y += torch.relu(xs @ sw1[s].double()) @ sw2[s].double()
    return host(y)


def _layer(ctx, cfg, S, gate, w1, w2, sw1, sw2, mode=0, ssmb=False):
    from paper_2508_13337_b200 import capi
    return capi.Layer(ctx, num_experts=cfg["E"], model_dim=cfg["H"], ffn_dim=cfg["F"], top_k=cfg["k"],
                      max_token_count=S * cfg["k"], max_tokens=S, dtype=capi.BF16, gate=gate, w1=w1, w2=w2,
                      sw1=sw1, sw2=sw2, dispatch_mode=mode, seed=7, ssmb=ssmb, chunks=1)


def _run(cfg_name, W, S, mode=0, n_sample=48):
    ctx, cfg, gate, w1, w2, sw1, sw2, x = _inputs(cfg_name, W, S)
    L = _layer(ctx, cfg, S, gate, w1, w2, sw1, sw2, mode)
    out = L.forward(x.view(W, S, -1)).view(W * S, -1)
    torch.cuda.synchronize()
    tpe_all = _check_routing_and_layout(L, x, gate, W, S, cfg["E"], cfg["k"])
    rows = np.sort(np.random.default_rng(W + S).choice(W * S, n_sample, replace=False))
    want = _sampled_reference(x, gate, w1, w2, sw1, sw2, cfg["k"], rows)
    got = host(out[torch.from_numpy(rows).cuda()])
    assert np.isfinite(got).all()
    assert norm_rel(got, want) < 1e-2, norm_rel(got, want)
    return L, tpe_all


def test_c1_layer():
    """C1: 64 experts top-6 + 2 shared, 2048/1408, 4096 tokens."""
    _run("c1", 1, 4096)


@pytest.mark.parametrize("mode", [0, 1])
def test_c2_ep8_full(mode):
    """C2: 8 expert-parallel workers x 16K tokens, plain and RBD."""
    L, _ = _run("c2", 8, 16384, mode)
    if mode == 1:
        led = L.ledger()
        assert 0 < led["unique_rows_offrank"] < led["copies_offrank"]


def test_c3_single_gpu():
    """C3: 256 experts top-8 + 1 shared, d_model 7168, d_ff 2048, 8K tokens."""
    _run("c3", 1, 8192, n_sample=32)


def test_c3_ep8_full():
    """C3 at its stated scale: 8 workers x 8K tokens (64K), 32 experts each, RBD."""
    _run("c3", 8, 8192, mode=1, n_sample=32)


@pytest.mark.parametrize("mode", [0, 1])
def test_c5_zipf_full(mode):
    """C5: 128 experts top-8, Zipf-skewed gate logits, 8 workers x 8K tokens,
    d_model 2048, d_ff 1408: empty and oversized expert groups."""
    L, tpe_all = _run("c5", 8, 8192, mode)
    load = tpe_all.sum(0).double()
    assert int((load == 0).sum()) >= 1, load
    assert float(load.max()) >= 4 * float(load.mean()), (float(load.max()), float(load.mean()))
    assert int(load.sum()) == 8 * 8192 * 8


@pytest.mark.parametrize("G", [2, 4, 8])
def test_c4_ssmb_full(G):
    """C4: a 32K-token sequence over G shards, 160 experts top-6, 5120/1536;
    replicated-expert SSMB (ssmb.cpp:12-46) and, at G=8, SSMB composed with
    EP (20 experts per rank): bit-identical outputs, routing exact per shard."""
    from paper_2508_13337_b200 import capi
    S = 32768
    ctx, cfg, gate, w1, w2, _, _, x = _inputs("c4", G, S // G)
    L = _layer(ctx, cfg, S // G, gate, w1, w2, None, None, ssmb=True)
    out = L.ssmb_forward(x)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(G).choice(S, 40, replace=False))
    rows[0], rows[-1] = 0, S - 1
    want = _sampled_reference(x, gate, w1, w2, None, None, cfg["k"], rows)
    assert norm_rel(host(out[torch.from_numpy(rows).cuda()]), want) < 1e-2
    if G == 8:
        ep = _layer(ctx, cfg, S // G, gate, w1, w2, None, None)  # experts partitioned over the 8 ranks
        out_ep = ep.ssmb_forward(x)
        torch.cuda.synchronize()
        _check_routing_and_layout(ep, x, gate, G, S // G, cfg["E"], cfg["k"])
        assert torch.equal(out_ep, out)
        led = ep.ledger()
        assert led["routed_copies"] == S * cfg["k"]
    del capi
