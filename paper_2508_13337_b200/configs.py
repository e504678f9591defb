"""BASELINE.json configs and their synthetic inputs.

Inputs come from the reference's own generator (moesim::Rng, xoshiro256**,
rng.hpp:24-61) drawn ON THE DEVICE by xmoe_rng_uniform / xmoe_make_layer_weights
(GF(2) jump-ahead), salted like the reference CLI (moesim_main.cpp:145-156):

  weights  Rng(salt_seed(seed, 7000 + layer)), make_layer_weights order
           (gate [H,E], then per expert w1 [H,F], w2 [F,H]; U(-0.1, 0.1));
           the gate snapped to multiples of 2^-10, experts rounded to bf16
  tokens   ONE Rng(salt_seed(seed, 9000 + layer)) stream, ranks 0..W-1 in
           order, row-major, U(-1, 1) snapped to multiples of 2^-7
  shared   (restated beyond the reference) Rng(salt_seed(seed, 7100)) as
           make_layer_weights(n_shared, H, Fs), experts only
  pilots   rbd seed salt_seed(seed, layer) (moesim_main.cpp:157)

On the grid the fp32 logits are exact, so routing is bit-identical to the
reference's fp64 gate.  The CPU arm of bench.py draws the same
values through the compiled reference (oracle/_ref), so both arms see
identical inputs.

C5 (skewed routing): feature 0 of every token is 1.0 and gate row 0 is
b_e = beta * (-s * ln(1 + pi(e))), s = 1.2, beta = 2, pi a seeded permutation
(argsort of Rng(salt_seed(seed, 7200)) draws), snapped to the gate grid and
stored in bf16 like the rest of the gate (the oracle uses the stored values)."""
from __future__ import annotations

import math

CONFIGS = {
    "c1": dict(E=64, k=6, H=2048, F=1408, ns=2, Fs=1408, S=4096,
               desc="C1: DeepSeek-MoE layer, 64 routed experts top-6 + 2 shared, d_model 2048, d_ff 1408, "
                    "4096 tokens (BASELINE configs[0], the reference's CPU-runnable case)"),
    "c2": dict(E=64, k=6, H=2048, F=1408, ns=2, Fs=1408, S=16384,
               desc="C2: DeepSeek-MoE layer, 64 routed experts top-6 + 2 shared, d_model 2048, d_ff 1408, "
                    "16K tokens per GPU, bf16, expert parallel, dropless (BASELINE configs[1])"),
    "c3": dict(E=256, k=8, H=7168, F=2048, ns=1, Fs=2048, S=8192,
               desc="C3: DeepSeek-V3 layer, 256 routed experts top-8 + 1 shared, d_model 7168, d_ff 2048, "
                    "8K tokens per GPU, bf16, expert parallel, dropless (BASELINE configs[2])"),
    "c4": dict(E=160, k=6, H=5120, F=1536, ns=0, Fs=0, S_total=32768, ssmb=True,
               desc="C4: sequence-sharded MoE block, 32K-token sequence split over the GPUs (SSMB composed with "
                    "EP), 160 experts top-6, d_model 5120, d_ff 1536, bf16, dropless (BASELINE configs[3])"),
    "c5": dict(E=128, k=8, H=2048, F=1408, ns=0, Fs=0, S=8192, zipf=(1.2, 2.0),
               desc="C5: skewed routing, 128 experts top-8 with Zipf-imbalanced gate logits, d_model 2048, "
                    "d_ff 1408, 8K tokens per GPU (64K at 8 GPUs), bf16, dropless (BASELINE configs[4])"),
}

SEED = 0
LAYER = 0
TOKEN_GRID = 128.0   # 2^7
GATE_GRID = 1024.0   # 2^10


def seeds(salt_seed):
    return {"weights": salt_seed(SEED, 7000 + LAYER, 0), "tokens": salt_seed(SEED, 9000 + LAYER, 0),
            "shared": salt_seed(SEED, 7100, 0), "zipf": salt_seed(SEED, 7200, 0),
            "rbd": salt_seed(SEED, LAYER, 0)}


def tokens_per_gpu(cfg: dict, world: int) -> int:
    return cfg["S_total"] // world if cfg.get("ssmb") else cfg["S"]


def zipf_bias(cfg: dict, uniforms) -> list:
    """Gate row 0 of C5 from E uniform draws (the permutation's keys), on the
    2^-10 grid (the device stores it in bf16: use the bf16-rounded values)."""
    s, beta = cfg["zipf"]
    E = cfg["E"]
    order = sorted(range(E), key=lambda e: (uniforms[e], e))
    rank = [0] * E
    for r, e in enumerate(order):
        rank[e] = r
    return [round(beta * (-s * math.log1p(rank[e])) * GATE_GRID) / GATE_GRID for e in range(E)]


def device_inputs(ctx, capi, cfg: dict, rank: int, world: int, S_local: int, token_row0: int, torch):
    """Weights of this rank's experts + its tokens, bf16 on the current GPU."""
    sd = seeds(capi.salt_seed)
    E, H, F = cfg["E"], cfg["H"], cfg["F"]
    el = E // world
    gate, w1, w2 = ctx.make_layer_weights(sd["weights"], E, H, F, first_expert=rank * el, n_experts=el,
                                          gate_grid=GATE_GRID, dtype=capi.BF16)
    sw1 = sw2 = None
    if cfg["ns"]:
        ns, Fs = cfg["ns"], cfg["Fs"]
        _, sw1, sw2 = ctx.make_layer_weights(sd["shared"], ns, H, Fs, gate=False, dtype=capi.BF16)
    x = ctx.rng_uniform(sd["tokens"], token_row0 * H, S_local * H, -1.0, 1.0, grid=TOKEN_GRID,
                        dtype=capi.BF16).view(S_local, H)
    if cfg.get("zipf"):
        u = ctx.rng_uniform(sd["zipf"], 0, E, 0.0, 1.0).cpu().tolist()
        gate[0] = torch.tensor(zipf_bias(cfg, u), dtype=torch.float64).to(torch.bfloat16).cuda()
        x[:, 0] = 1.0
    return gate, w1, w2, sw1, sw2, x
