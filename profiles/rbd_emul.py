"""C2 layer with W emulated expert-parallel workers driven by ONE process on
cuda:0 (context rank -1), for single-process ncu launch lists of the
redundancy-bypassing (or plain) dispatch path:
    ncu --metrics gpu__time_duration.sum --csv python profiles/rbd_emul.py --world 4 --mode rbd
(ncu must not be attached to a multi-rank job; the kernels per worker are
the distributed ones, with local copies in place of NVLink stores)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2508_13337_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--mode", default="rbd", choices=["rbd", "naive"])
ap.add_argument("--chunks", type=int, default=1)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
W, E, k, H, F, ns, Fs, S = a.world, 64, 6, 2048, 1408, 2, 1408, 16384
ctx = capi.Context(0, W, -1)
g = torch.Generator(device="cuda").manual_seed(1)
r = lambda *s: ((torch.rand(*s, device="cuda", generator=g) - 0.5) * 0.2).to(torch.bfloat16)  # noqa: E731
gate = (torch.round(r(H, E).float() * 1024) / 1024).to(torch.bfloat16)
L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
               dtype=capi.BF16, gate=gate, w1=r(E, H, F), w2=r(E, F, H), sw1=r(ns, H, Fs), sw2=r(ns, Fs, H),
               chunks=a.chunks, dispatch_mode=capi.RBD if a.mode == "rbd" else capi.NAIVE)
x = (torch.round(r(W, S, H).float() * 1280) / 128).clamp(-1, 1).to(torch.bfloat16)
out = torch.empty_like(x)
for _ in range(a.steps):
    L.forward(x, out)
torch.cuda.synchronize()
print("ok", L.chunks(), flush=True)
