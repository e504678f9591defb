"""Per-chunk timeline of the chunked forward (C2 layer, plain dispatch).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 profiles/timeline.py --chunks C

Prints, per rank, the stage marks and for every chunk the ms (from the
forward's start) at which its scatter ended, its expert GEMMs started and
ended, and its combine ended (CUDA events; timing mode, eager launches)."""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13337_b200 import capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--mode", default="naive", choices=["naive", "rbd"])
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    if world > 1:
        dist.init_process_group("gloo")
        obj = [capi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = capi.Context(int(os.environ.get("LOCAL_RANK", 0)), world, rank, obj[0])
    else:
        ctx = capi.Context(0, 1, 0)
    E, k, H, F, ns, Fs, S = 64, 6, 2048, 1408, 2, 1408, a.tokens
    g = torch.Generator(device="cuda").manual_seed(1)
    r = lambda *s: ((torch.rand(*s, device="cuda", generator=g) - 0.5) * 0.2).to(torch.bfloat16)  # noqa: E731
    gate = (torch.round(r(H, E).float() * 1024) / 1024).to(torch.bfloat16)
    L = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                   dtype=capi.BF16, gate=gate, w1=r(E // world, H, F), w2=r(E // world, F, H), sw1=r(ns, H, Fs),
                   sw2=r(ns, Fs, H), chunks=a.chunks, dispatch_mode=capi.RBD if a.mode == "rbd" else capi.NAIVE)
    x = (torch.round(r(S, H).float() * 1280) / 128).clamp(-1, 1).to(torch.bfloat16)
    out = torch.empty_like(x)
    for _ in range(5):
        L.forward(x, out)
    torch.cuda.synchronize()
    L.set_timing(True)
    runs, tls = [], []
    for _ in range(7):
        if world > 1:
            dist.barrier()
        L.forward(x, out)
        torch.cuda.synchronize()
        runs.append(L.stage_ms())
        tls.append(L.timeline_ms())
    st = {kk: round(statistics.median(rr[kk] for rr in runs), 4) for kk in runs[0]}
    mid = sorted(range(len(runs)), key=lambda i: runs[i]["total"])[len(runs) // 2]
    print(json.dumps({"rank": rank, "chunks": L.chunks(), "stages": st, "timeline": tls[mid]}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
