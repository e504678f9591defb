"""C2 layer with W expert-parallel workers emulated on ONE GPU (rank -1),
token-chunked: the same kernels as the multi-GPU chunked forward (pull
dispatch, whole-SM combines, SM-capped GEMMs), serialised on one device, for
an ncu launch list (ncu must not wrap a multi-rank command).

    ncu --metrics gpu__time_duration.sum -c 300 --csv python profiles/emulated_chunked.py [W] [chunks]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13337_b200 import capi, configs  # noqa: E402


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = dict(configs.CONFIGS["c2"])
    S = cfg["S"]
    ctx = capi.Context(0, W, -1)
    gate, w1, w2, sw1, sw2, x = configs.device_inputs(ctx, capi, cfg, 0, 1, W * S, 0, torch)
    L = capi.Layer(ctx, num_experts=cfg["E"], model_dim=cfg["H"], ffn_dim=cfg["F"], top_k=cfg["k"],
                   max_token_count=S * cfg["k"], max_tokens=S, dtype=capi.BF16, gate=gate, w1=w1, w2=w2,
                   sw1=sw1, sw2=sw2, chunks=C)
    xs = x.view(W, S, -1)
    out = torch.empty_like(xs)
    for _ in range(3):
        L.forward(xs, out)
    torch.cuda.synchronize()
    print("chunks", L.chunks(), "ok", flush=True)


if __name__ == "__main__":
    main()
