"""Multi-process expert-parallel parity check (one process per GPU, NCCL).

Run with:  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist_layer_check.py
Every rank builds the same seeded instance, keeps its E/N experts and its
token slice, runs the layer through the C-ABI over NCCL, and rank 0 compares
all ranks' outputs with the oracle: F64 bit-exact given the device softmax
weights, BF16 within the test_gpu_layer tolerances.  Exit code 0 = pass."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import moe_oracle as O  # noqa: E402
from paper_2508_13337_b200 import capi  # noqa: E402
from tests.gpu_util import bf16_round, grid_gate, grid_tokens, max_rel_diff, norm_rel  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [capi.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = capi.Context(local, world, rank, obj[0])
    failures = []
    cases = [(capi.F64, capi.NAIVE, 97, 8, 3, 24, 16, 1), (capi.F64, capi.RBD, 97, 8, 3, 24, 16, 1),
             (capi.BF16, capi.NAIVE, 512, 16, 6, 256, 128, 1), (capi.BF16, capi.RBD, 512, 16, 6, 256, 128, 1)]
    if world % 2 == 0:  # two-tier RBD: nodes of 2 GPUs, stage 2 and its reverse over NVLink
        cases += [(capi.F64, capi.RBD, 97, 8, 5, 24, 16, 2), (capi.BF16, capi.RBD, 512, 16, 6, 256, 128, 2)]
    for ci, (dt, mode, S, e_per, k, H, F, gpn) in enumerate(cases):
        E = e_per * world
        el = E // world
        rng = np.random.default_rng(100 + ci)
        if dt == capi.F64:
            gate = rng.uniform(-0.1, 0.1, (H, E))
            w1 = rng.uniform(-0.1, 0.1, (E, H, F))
            w2 = rng.uniform(-0.1, 0.1, (E, F, H))
            x = rng.uniform(-1, 1, (world, S, H))
            tdt = torch.float64
        else:
            gate = grid_gate(rng, H, E)
            w1 = bf16_round(rng.uniform(-0.1, 0.1, (E, H, F)))
            w2 = bf16_round(rng.uniform(-0.1, 0.1, (E, F, H)))
            x = grid_tokens(rng, world, S, H)
            tdt = torch.bfloat16
        cap = S * k if ci % 2 == 0 else int(np.ceil(1.5 * S * k / E))
        seed = 4242 + ci
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(tdt).cuda()  # noqa: E731
        layer = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap,
                           max_tokens=S, dtype=dt, gate=dv(gate), w1=dv(w1[rank * el:(rank + 1) * el]),
                           w2=dv(w2[rank * el:(rank + 1) * el]), dispatch_mode=mode, seed=seed,
                           gpus_per_node=gpn)
        out = layer.forward(dv(x[rank])).to(torch.float64).cpu().numpy()
        led = layer.ledger()
        # reference-schema ledger: every rank contributes its sources (collective)
        csv = layer.ledger_csv(capi.Topology.reference_defaults(gpus_per_node=gpn, dtype_bytes=2))
        gate_dev = None
        if dt == capi.F64:
            top, wt = ctx.gate_forward(dv(x[rank]), dv(gate), k)
            gate_dev = (top.cpu().numpy(), wt.cpu().numpy())
        got = [None] * world
        dist.all_gather_object(got, (out, gate_dev, led))
        if rank == 0:
            W = O.LayerWeights(gate, w1, w2)
            gates = [g[1] for g in got] if dt == capi.F64 else None
            exact = dt == capi.F64
            if mode == capi.NAIVE:
                want = O.pf_moe_forward(list(x), W, E, k, cap, gates=gates, exact=exact)
            else:
                want = O.rbd_moe_forward(list(x), W, E, k, cap, seed, [r // gpn for r in range(world)],
                                         gates=gates, exact=exact)
            for r in range(world):
                o = got[r][0]
                if dt == capi.F64:
                    ok = np.array_equal(o, want[r])
                    err = max_rel_diff(o, want[r])
                else:
                    err = norm_rel(o, want[r])
                    ok = err < 1e-2 and max_rel_diff(o, want[r]) < 2e-2
                if not ok:
                    failures.append((ci, r, err))
            if dt == capi.F64:
                from oracle import refbind
                if refbind.available():
                    rl = refbind.Layer(gate, w1, w2)
                    if mode == capi.NAIVE:
                        rl.pf_moe_forward(x, k, cap, [r // gpn for r in range(world)])
                    else:
                        rl.rbd_moe_forward(x, k, cap, seed, [r // gpn for r in range(world)])
                    if csv != refbind.last_ledger_csv():
                        failures.append((ci, "ledger_csv", csv, refbind.last_ledger_csv()))
                    else:
                        print(f"case {ci} ledger CSV identical to the reference's", flush=True)
            tot = {kk: sum(g[2][kk] for g in got) for kk in got[0][2]}
            print(f"case {ci} dtype={'f64' if dt == capi.F64 else 'bf16'} mode={'rbd' if mode else 'naive'} gpn={gpn} "
                  f"cap={cap} ledger={tot}", flush=True)
        del layer
        dist.barrier()
    # token-chunked pipelined forward (epoch flags over NVLink): bit-identical
    # to the unchunked layer, eager and graph-replayed, over repeated forwards
    for ci, (S, cap_f, chunks, mode) in enumerate([(1000, None, 3, capi.NAIVE), (777, 0.6, 4, capi.NAIVE),
                                                   (4096, None, 0, capi.NAIVE), (1000, None, 3, capi.RBD),
                                                   (777, 0.6, 4, capi.RBD), (4096, None, 0, capi.RBD),
                                                   (4096, None, 2, capi.RBD), (8192, None, 4, capi.NAIVE)]):
        E, k, H, F = 16 * world, 6, 256, 128
        el = E // world
        rng = np.random.default_rng(300 + ci)
        gate = grid_gate(rng, H, E)
        w1 = bf16_round(rng.uniform(-0.1, 0.1, (E, H, F)))
        w2 = bf16_round(rng.uniform(-0.1, 0.1, (E, F, H)))
        sw1 = bf16_round(rng.uniform(-0.1, 0.1, (2, H, 128)))
        sw2 = bf16_round(rng.uniform(-0.1, 0.1, (2, 128, H)))
        x = grid_tokens(rng, world, S, H)
        cap = S * k if cap_f is None else int(cap_f * S * k / E)
        bv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()  # noqa: E731
        outs = []
        for c in (1, chunks):
            layer = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=cap,
                               max_tokens=S, dtype=capi.BF16, gate=bv(gate), w1=bv(w1[rank * el:(rank + 1) * el]),
                               w2=bv(w2[rank * el:(rank + 1) * el]), sw1=bv(sw1), sw2=bv(sw2), chunks=c,
                               dispatch_mode=mode, seed=11)
            xd = bv(x[rank])
            o = [layer.forward(xd).clone() for _ in range(3)]
            layer.set_graph(True)
            ob = torch.empty_like(xd)
            for _ in range(3):
                layer.forward(xd, ob)
            torch.cuda.synchronize()
            o.append(ob.clone())
            outs.append(o)
            del layer
            dist.barrier()
        same = all(torch.equal(outs[0][0], t) for t in outs[0] + outs[1])
        got = [None] * world
        dist.all_gather_object(got, (same, outs[1][0].float().cpu().numpy()))
        if rank == 0:
            Wt = O.LayerWeights(gate, w1, w2)
            want = [O.moe_layer_with_shared(x[r], Wt, E, k, cap, sw1, sw2, exact=False) for r in range(world)]
            errs = [norm_rel(got[r][1], want[r]) for r in range(world)]
            print(f"chunked case {ci} mode={mode} S={S} chunks={chunks} bit-identical={[g[0] for g in got]} err={max(errs):.2e}",
                  flush=True)
            if not all(g[0] for g in got) or max(errs) > 1e-2:
                failures.append(("chunked", ci, [g[0] for g in got], errs))
    # ragged and empty sequences through one layer (every rank the same S)
    E, k, H, F = 8 * world, 3, 64, 32
    el = E // world
    rng = np.random.default_rng(808)
    gate = grid_gate(rng, H, E)
    w1 = bf16_round(rng.uniform(-0.1, 0.1, (E, H, F)))
    w2 = bf16_round(rng.uniform(-0.1, 0.1, (E, F, H)))
    bv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()  # noqa: E731
    for mode in (capi.NAIVE, capi.RBD):
        layer = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=4096 * k,
                           max_tokens=4096, dtype=capi.BF16, gate=bv(gate), w1=bv(w1[rank * el:(rank + 1) * el]),
                           w2=bv(w2[rank * el:(rank + 1) * el]), dispatch_mode=mode, seed=5)
        for S in (0, 1, 7, 4096, 0, 33):
            x = grid_tokens(np.random.default_rng(S), world, S, H)
            o = layer.forward(bv(x[rank])).float().cpu().numpy()
            got = [None] * world
            dist.all_gather_object(got, o)
            if rank == 0 and S:
                want = O.pf_moe_forward(list(x), O.LayerWeights(gate, w1, w2), E, k, 4096 * k, exact=False) \
                    if mode == capi.NAIVE else \
                    O.rbd_moe_forward(list(x), O.LayerWeights(gate, w1, w2), E, k, 4096 * k, 5, exact=False)
                errs = [norm_rel(got[r], want[r]) for r in range(world)]
                if max(errs) > 1e-2:
                    failures.append(("ragged", mode, S, errs))
        del layer
        dist.barrier()
    if rank == 0:
        print("ragged / empty sequences checked", flush=True)
    # unequal S per rank with one idle rank (S == 0): every rank must take the
    # same (chunked or unchunked) protocol whatever its own S
    for mode, chunks in ((capi.NAIVE, 0), (capi.NAIVE, 4), (capi.RBD, 0), (capi.RBD, 2)):
        layer = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=4096 * k,
                           max_tokens=4096, dtype=capi.BF16, gate=bv(gate), w1=bv(w1[rank * el:(rank + 1) * el]),
                           w2=bv(w2[rank * el:(rank + 1) * el]), dispatch_mode=mode, seed=5, chunks=chunks)
        for it, Ss in enumerate(([0] + [4096 - 37 * r for r in range(1, world)],
                                 [300 + r for r in range(world - 1)] + [0])):
            xs = [grid_tokens(np.random.default_rng(900 + 10 * it + r), Ss[r], H) for r in range(world)]
            o = layer.forward(bv(xs[rank])).float().cpu().numpy()
            got = [None] * world
            dist.all_gather_object(got, o)
            if rank == 0:
                Wt = O.LayerWeights(gate, w1, w2)
                want = O.pf_moe_forward(xs, Wt, E, k, 4096 * k, exact=False) if mode == capi.NAIVE else \
                    O.rbd_moe_forward(xs, Wt, E, k, 4096 * k, 5, exact=False)
                errs = [norm_rel(got[r], want[r]) for r in range(world) if Ss[r] > 0]
                shapes_ok = all(got[r].shape[0] == Ss[r] for r in range(world))
                print(f"idle-rank case mode={mode} chunks={layer.chunks()} S={Ss} err={max(errs):.2e}", flush=True)
                if max(errs) > 1e-2 or not shapes_ok:
                    failures.append(("idle-rank", mode, chunks, Ss, errs))
        layer.status()  # no peer wait timed out
        del layer
        dist.barrier()
    # backward over the peer transport (bf16, dropless): dx per rank, expert
    # grads of each rank's block, gate grads summed over ranks; 2048 tokens:
    # more rows than the SM partition's whole-SM blocks have warps
    from oracle import moe_grad as Gr
    for S in (256, 2048):
        E, k, H, F = 16 * world, 4, 128, 128
        el = E // world
        rng = np.random.default_rng(55)
        gate = grid_gate(rng, H, E)
        w1 = bf16_round(rng.uniform(-0.1, 0.1, (E, H, F)))
        w2 = bf16_round(rng.uniform(-0.1, 0.1, (E, F, H)))
        x = grid_tokens(rng, world, S, H)
        dy = bf16_round(rng.uniform(-1, 1, (world, S, H)))
        bv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()  # noqa: E731
        layer = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k, max_tokens=S,
                           dtype=capi.BF16, gate=bv(gate), w1=bv(w1[rank * el:(rank + 1) * el]),
                           w2=bv(w2[rank * el:(rank + 1) * el]), train=True)
        xd = bv(x[rank])
        layer.forward(xd)
        dxr = layer.backward(xd, bv(dy[rank])).float().cpu().numpy()
        gr = {n: (v.cpu().numpy() if v is not None else None) for n, v in layer.grads().items()}
        got = [None] * world
        dist.all_gather_object(got, (dxr, gr))
        if rank == 0:
            want = Gr.moe_grads(x.reshape(world * S, H), gate, w1, w2, dy.reshape(world * S, H), k, world * S * k)
            errs = [norm_rel(np.concatenate([g[0] for g in got]), want["x"]),
                    norm_rel(sum(g[1]["gate"] for g in got), want["gate"]),
                    norm_rel(np.concatenate([g[1]["w1"] for g in got]), want["w1"]),
                    norm_rel(np.concatenate([g[1]["w2"] for g in got]), want["w2"])]
            print(f"backward S={S} normwise errors dx/gate/w1/w2:", errs, flush=True)
            if max(errs) > 3e-2:
                failures.append(("backward", S, errs))
        del layer
        dist.barrier()
    # sequence-sharded block across the ranks (ssmb.cpp:12-46)
    S, E, k, H, F = 101, 8, 2, 16, 8
    rng = np.random.default_rng(77)
    gate = rng.uniform(-0.1, 0.1, (H, E))
    w1 = rng.uniform(-0.1, 0.1, (E, H, F))
    w2 = rng.uniform(-0.1, 0.1, (E, F, H))
    x = rng.uniform(-1, 1, (S, H))
    bounds = O.ssmb_shards(S, world)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    layer = capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S * k,
                       max_tokens=max(n for _, n in bounds), dtype=capi.F64, gate=dv(gate), w1=dv(w1),
                       w2=dv(w2), ssmb=True)
    out = layer.ssmb_forward(dv(x)).cpu().numpy()
    b, n = bounds[rank]
    top, wt = ctx.gate_forward(dv(x[b:b + n]), dv(gate), k)
    got = [None] * world
    dist.all_gather_object(got, (out, (top.cpu().numpy(), wt.cpu().numpy())))
    if rank == 0:
        Wt = O.LayerWeights(gate, w1, w2)
        want = np.concatenate([O.pf_moe_forward([x[bb:bb + nn]], Wt, E, k, S * k, gates=[got[g][1]])[0]
                               for g, (bb, nn) in enumerate(bounds)])
        for r in range(world):
            if not np.array_equal(got[r][0], want):
                failures.append(("ssmb", r, max_rel_diff(got[r][0], want)))
        print("ssmb checked on", world, "ranks", flush=True)
    del layer
    dist.barrier()
    # SSMB composed with EP on the pull-dispatch chunked layer against the
    # replicated-expert SSMB layer: bit-identical, ragged last shard
    Ss = 4096
    S = world * Ss + 37
    E, k, H, F = 16 * world, 6, 256, 128
    el = E // world
    rng = np.random.default_rng(91)
    gate = grid_gate(rng, H, E)
    w1 = bf16_round(rng.uniform(-0.1, 0.1, (E, H, F)))
    w2 = bf16_round(rng.uniform(-0.1, 0.1, (E, F, H)))
    x = grid_tokens(rng, 1, S, H)[0]
    bv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()  # noqa: E731
    kw = dict(num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=(Ss + 37) * k, max_tokens=Ss + 37,
              dtype=capi.BF16, gate=bv(gate))
    rep = capi.Layer(ctx, w1=bv(w1), w2=bv(w2), ssmb=True, **kw)
    out_rep = rep.ssmb_forward(bv(x)).clone()
    del rep
    dist.barrier()
    ep = capi.Layer(ctx, w1=bv(w1[rank * el:(rank + 1) * el]), w2=bv(w2[rank * el:(rank + 1) * el]), **kw)
    outs = [ep.ssmb_forward(bv(x)).clone() for _ in range(2)]
    torch.cuda.synchronize()
    same = all(torch.equal(o, out_rep) for o in outs)
    got = [None] * world
    dist.all_gather_object(got, (same, ep.chunks()))
    if rank == 0:
        print(f"ssmb+ep vs replicated: chunks={[g[1] for g in got]} bit-identical={[g[0] for g in got]}",
              flush=True)
        if not all(g[0] for g in got):
            failures.append(("ssmb+ep", [g[0] for g in got]))
    ep.status()
    del ep
    dist.barrier()
    if rank == 0:
        print("FAILURES", failures, flush=True)
    ok = torch.tensor([0 if not failures else 1])
    dist.broadcast(ok, 0)
    dist.destroy_process_group()
    sys.exit(int(ok.item()))


if __name__ == "__main__":
    main()
