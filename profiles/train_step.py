"""One C2 training layer (forward + backward) run a few times on cuda:0, for
ncu launch lists of the backward (`ncu --metrics gpu__time_duration.sum
--clock-control none --csv python profiles/train_step.py`).  Eager launches
(no CUDA graph) so that every kernel appears once per step in order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2508_13337_b200 import capi  # noqa: E402

E, k, H, F, ns, Fs, S = 64, 6, 2048, 1408, 2, 1408, 16384
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = capi.Context(0, 1, 0)
g = torch.Generator(device="cuda")
g.manual_seed(1234)
gate = (torch.round((torch.rand(H, E, device="cuda", generator=g) * 0.2 - 0.1) * 1024) / 1024).to(torch.bfloat16)
w1 = (torch.rand(E, H, F, device="cuda", generator=g) * 0.2 - 0.1).to(torch.bfloat16)
w2 = (torch.rand(E, F, H, device="cuda", generator=g) * 0.2 - 0.1).to(torch.bfloat16)
sw1 = (torch.rand(ns, H, Fs, device="cuda", generator=g) * 0.2 - 0.1).to(torch.bfloat16)
sw2 = (torch.rand(ns, Fs, H, device="cuda", generator=g) * 0.2 - 0.1).to(torch.bfloat16)
x = (torch.round((torch.rand(S, H, device="cuda", generator=g) * 2 - 1) * 128) / 128).to(torch.bfloat16)
dy = (torch.rand(S, H, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
layer = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                   dtype=capi.BF16, gate=gate, w1=w1, w2=w2, sw1=sw1, sw2=sw2, train=True, chunks=1)
out, dx = torch.empty_like(x), torch.empty_like(x)
for _ in range(steps):
    layer.forward(x, out)
    layer.backward(x, dy, dx)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(10):
    layer.forward(x, out)
    layer.backward(x, dy, dx)
t1.record()
torch.cuda.synchronize()
print(f"fwd+bwd eager {t0.elapsed_time(t1) / 10:.3f} ms/step", flush=True)
# host enqueue cost vs device time (the GPU spins first so the host queues
# everything ahead of it); backward = (forward + backward) - forward, since a
# backward must follow its own forward
import time  # noqa: E402
res = {}
for name, fn in (("forward", lambda: layer.forward(x, out)),
                 ("fwd+bwd", lambda: (layer.forward(x, out), layer.backward(x, dy, dx)))):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000_000)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(10):
        fn()
    h1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 10
    print(f"{name}: device {res[name]:.3f} ms/call (host queued ahead), host enqueue {(h1 - h0) * 100:.3f} ms/call",
          flush=True)
print(f"backward: device {res['fwd+bwd'] - res['forward']:.3f} ms/call", flush=True)
