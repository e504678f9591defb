"""Multi-rank host logic on CPU: two gloo processes run the plain expert-
parallel dispatch and combine with the library's own exchange plan
(xmoe_plan_dispatch, the arithmetic the NCCL transport uses and the device
placement kernel restates) and real point-to-point row exchanges, the expert
math coming from the oracle.  The result must equal the single-process
oracle bit for bit: placement = pf_dispatch's (local expert, source,
position) layout, combine = pf_combine."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance(W, seed):
    from oracle import moe_oracle as O
    rng = O.Rng(seed)
    E, k, H, F, S = 4 * W, 3, 6, 5, 23
    w = O.make_layer_weights(rng, E, H, F)
    toks = np.array([rng.uniform(-1.0, 1.0) for _ in range(W * S * H)]).reshape(W, S, H)
    return w, E, k, toks


def _worker(rank, W, port, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        from oracle import moe_oracle as O
        from paper_2508_13337_b200 import capi
        w, E, k, toks = _instance(W, seed)
        el = E // W
        cap = toks.shape[1] * k
        x = toks[rank]
        g = O.gate_forward(x, w.gate, k)
        p = O.pft_from_gate(cap, E, g)
        p.x = O.gather_rows(x, p.token_ids)
        # count exchange (pf_pipeline.cpp:30-36)
        mine = torch.from_numpy(p.tokens_per_expert.astype(np.int32))
        allc = [torch.zeros_like(mine) for _ in range(W)]
        dist.all_gather(allc, mine)
        tpe_all = torch.stack(allc).numpy()
        send_off, recv_off, rpe = capi.plan_dispatch(tpe_all, rank)
        H = x.shape[1]
        grouped = np.zeros((int(rpe.sum()), H))
        # forward: my block for each expert of peer -> its (le, src, pos) slot
        reqs, keep = [], []
        for peer in range(W):
            for le in range(el):
                e = peer * el + le
                n = int(tpe_all[rank, e])
                if n == 0:
                    continue
                rows = torch.from_numpy(np.ascontiguousarray(p.x[send_off[e]:send_off[e] + n]))
                if peer == rank:
                    grouped[recv_off[rank, le]:recv_off[rank, le] + n] = rows.numpy()
                else:
                    keep.append(rows)
                    reqs.append(dist.isend(rows, peer, tag=e))
        recvs = []
        for src in range(W):
            if src == rank:
                continue
            for le in range(el):
                n = int(tpe_all[src, rank * el + le])
                if n == 0:
                    continue
                buf = torch.zeros((n, H), dtype=torch.float64)
                recvs.append((buf, src, le, dist.irecv(buf, src, tag=rank * el + le)))
        for r in reqs:
            r.wait()
        for buf, src, le, r in recvs:
            r.wait()
            grouped[recv_off[src, le]:recv_off[src, le] + buf.shape[0]] = buf.numpy()
        # expert FFNs over my local experts (pf_pipeline.cpp:83-105)
        y = O.grouped_expert_mlp(grouped, rpe, w, rank * el)
        # reverse: transposed counts back into my packed order
        back = np.zeros_like(p.x)
        reqs, keep = [], []
        for src in range(W):
            for le in range(el):
                n = int(tpe_all[src, rank * el + le])
                if n == 0:
                    continue
                rows = torch.from_numpy(np.ascontiguousarray(y[recv_off[src, le]:recv_off[src, le] + n]))
                if src == rank:
                    e = rank * el + le
                    back[send_off[e]:send_off[e] + n] = rows.numpy()
                else:
                    keep.append(rows)
                    reqs.append(dist.isend(rows, src, tag=1000 + rank * el + le))
        recvs = []
        for peer in range(W):
            if peer == rank:
                continue
            for le in range(el):
                e = peer * el + le
                n = int(tpe_all[rank, e])
                if n == 0:
                    continue
                buf = torch.zeros((n, H), dtype=torch.float64)
                recvs.append((buf, e, dist.irecv(buf, peer, tag=1000 + e)))
        for r in reqs:
            r.wait()
        for buf, e, r in recvs:
            r.wait()
            back[send_off[e]:send_off[e] + buf.shape[0]] = buf.numpy()
        out = O.scatter_combine(back, p.token_ids, p.combine_weights, x.shape[0])
        q.put((rank, grouped, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W", [2])
def test_two_rank_gloo_exchange_matches_oracle(W):
    from oracle import moe_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, W, port, 99, q)) for r in range(W)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(W):
        rank, grouped, out = q.get(timeout=240)
        got[rank] = (grouped, out)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w, E, k, toks = _instance(W, 99)
    cap = toks.shape[1] * k
    want, pfts, disp, _ = O.pf_moe_forward(list(toks), w, E, k, cap, return_pfts=True)
    for r in range(W):
        assert np.array_equal(got[r][0], disp.expert_input[r])   # placement layout
        assert np.array_equal(got[r][1], want[r])                # whole layer


def test_plan_hand_trace():
    # test_pf_pipeline.cpp:34-72: workers own experts {0,1} and {2,3}
    from paper_2508_13337_b200 import capi
    tpe = np.array([[1, 0, 2, 1], [1, 1, 1, 0]])
    s0, r0, n0 = capi.plan_dispatch(tpe, 0)
    s1, r1, n1 = capi.plan_dispatch(tpe, 1)
    assert n0.tolist() == [2, 1] and n1.tolist() == [3, 1]
    assert s0.tolist() == [0, 1, 1, 3, 4] and s1.tolist() == [0, 1, 2, 3, 3]
    # worker 1 computes over [a1, a2, b2, a3]
    assert r1.tolist() == [[0, 3], [2, 4]]
    from paper_2508_13337_b200.capi import XmoeError
    with pytest.raises(XmoeError, match="divisible"):
        capi.plan_dispatch(np.zeros((3, 4), np.int32), 0)
