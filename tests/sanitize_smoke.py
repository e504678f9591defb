"""Small end-to-end passes for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck) on one GPU:

    compute-sanitizer --tool memcheck python tests/sanitize_smoke.py

Covers the fused routing, the token-major permute and slot combine, the
tcgen05 GEMMs, the RBD exchange (one GPU, W workers), the token-chunked
pipeline, the backward and the split EP operators.  Exit 0 = every pass ran
(the sanitizer reports its own errors)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13337_b200 import capi  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    bf = torch.bfloat16
    d = lambda a, t=bf: torch.from_numpy(np.ascontiguousarray(a)).to(t).cuda()  # noqa: E731
    E, k, H, F, S = 32, 4, 128, 128, 256
    gate = np.round(rng.uniform(-0.1, 0.1, (H, E)) * 1024) / 1024
    w1, w2 = rng.uniform(-0.1, 0.1, (E, H, F)), rng.uniform(-0.1, 0.1, (E, F, H))
    sw1, sw2 = rng.uniform(-0.1, 0.1, (1, H, 128)), rng.uniform(-0.1, 0.1, (1, 128, H))
    for W, mode, chunks in ((1, 0, 1), (2, 0, 1), (2, 0, 2), (2, 1, 1), (4, 1, 1)):
        ctx = capi.Context(0, W, -1)
        x = np.round(rng.uniform(-1, 1, (W, S, H)) * 128) / 128
        L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                       dtype=capi.BF16, gate=d(gate), w1=d(w1), w2=d(w2), sw1=d(sw1), sw2=d(sw2),
                       dispatch_mode=mode, seed=3, chunks=chunks)
        L.forward(d(x))
        torch.cuda.synchronize()
        print(f"bf16 layer W={W} mode={mode} chunks={chunks} ok", flush=True)
        del L
    ctx = capi.Context(0, 1, -1)
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                   dtype=capi.BF16, gate=d(gate), w1=d(w1), w2=d(w2), sw1=d(sw1), sw2=d(sw2), train=True)
    x = d(np.round(rng.uniform(-1, 1, (S, H)) * 128) / 128)
    L.forward(x)
    L.backward(x, d(rng.uniform(-1, 1, (S, H))))
    torch.cuda.synchronize()
    print("bf16 forward + backward ok", flush=True)
    for dt, t in ((capi.F64, torch.float64), (capi.F32, torch.float32)):
        c2 = capi.Context(0, 2, -1)
        L = capi.Layer(c2, num_experts=8, model_dim=12, ffn_dim=6, top_k=3, max_token_count=5, max_tokens=40, dtype=dt,
                       gate=d(rng.uniform(-0.1, 0.1, (12, 8)), t), w1=d(rng.uniform(-0.1, 0.1, (8, 12, 6)), t),
                       w2=d(rng.uniform(-0.1, 0.1, (8, 6, 12)), t), dispatch_mode=1, seed=1)
        L.forward(d(rng.uniform(-1, 1, (2, 40, 12)), t))
        torch.cuda.synchronize()
        print(f"dtype {dt} rbd layer with drops ok", flush=True)
    c4 = capi.Context(0, 4, -1)
    B = 50
    tid = torch.sort(torch.randint(0, 30, (B,), dtype=torch.int32, device="cuda")).values
    eid = torch.randint(0, 8, (B,), dtype=torch.int32, device="cuda")
    m, _ = c4.select_pilots(tid, eid, 30, B, 8, 4, 2, 7)
    torch.cuda.synchronize()
    print("select_pilots ok", flush=True)


if __name__ == "__main__":
    main()
