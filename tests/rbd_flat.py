"""Test-side flattening of the reference's RbdDispatch bookkeeping
(rbd.cpp:107-283) into the arrays xmoe_rbd_combine takes.  Written from the
reference's stated ordering rules, independently of the C++ adapter
(paper_2508_13337_b200/csrc/compat_impl.inc), so the two check each other:

  landing worker of a group    = owner of its pilot copy
  arrival order at a landing L = sources ascending, each source's pilots in
                                 packed (sequence) order (rbd.cpp:171-175)
  merge order of a group       = pilot first (scaled when the group has
                                 replicas), then its replicas in slot order,
                                 i.e. packed order (rbd.cpp:318-336)
  source add order             = per token, its pilots in packed order,
                                 x1 for multi-copy groups, x w singletons
                                 (rbd.cpp:343-356)
"""
import numpy as np
import torch


def flatten(W, masks, pilot_of, dest_rank, dest_row, cw, token_ids, seq_lens):
    """All per-source arguments are numpy arrays.  Returns (dict of device
    tensors for Context.rbd_combine, s1_counts [W,W])."""
    pil = []  # per source: pilot rows in packed order
    multi = []
    for s in range(W):
        m = masks[s].astype(bool)
        rows = np.nonzero(m)[0]
        pil.append(rows)
        has_rep = np.zeros(len(m), bool)
        for r in np.nonzero(~m)[0]:
            has_rep[pilot_of[s][r]] = True
        multi.append(has_rep)
    s1 = np.zeros((W, W), np.int64)
    for s in range(W):
        for p in pil[s]:
            s1[s, dest_rank[s][p]] += 1
    # flat index of (L, arrival)
    land_off = np.concatenate([[0], np.cumsum(s1.sum(axis=0))])
    flat_of = [dict() for _ in range(W)]  # source -> pilot row -> flat
    land_of, land_pos, land_multi, land_w = [], [], [], []
    for L in range(W):
        for s in range(W):
            for p in pil[s]:
                if dest_rank[s][p] != L:
                    continue
                flat_of[s][int(p)] = len(land_of)
                land_of.append(L)
                land_pos.append(dest_row[s][p])
                land_multi.append(1 if multi[s][p] else 0)
                land_w.append(cw[s][p])
    P = len(land_of)
    assert P == land_off[-1]
    ents = [[] for _ in range(P)]
    for s in range(W):
        for r in np.nonzero(~masks[s].astype(bool))[0]:  # packed order
            f = flat_of[s][int(pilot_of[s][r])]
            ents[f].append((dest_rank[s][r], dest_row[s][r], cw[s][r]))
    ent_ptr = np.concatenate([[0], np.cumsum([len(e) for e in ents])]).astype(np.int32)
    flat_e = [x for e in ents for x in e]
    flat_scale = np.zeros(max(P, 1))
    for s in range(W):
        for p, f in flat_of[s].items():
            flat_scale[f] = 1.0 if multi[s][p] else cw[s][p]
    src_ptr, src_flat = [], []
    for s in range(W):
        S = seq_lens[s]
        per_tok = [[] for _ in range(S)]
        for p in pil[s]:  # packed order
            per_tok[token_ids[s][p]].append(flat_of[s][int(p)])
        src_ptr.append(np.concatenate([[0], np.cumsum([len(v) for v in per_tok])]).astype(np.int32))
        src_flat.append(np.array([f for v in per_tok for f in v] or [0], np.int32))
    d = lambda a, t: torch.from_numpy(np.ascontiguousarray(a, dtype=t)).cuda()  # noqa: E731
    flat = {"land_of": d(land_of or [0], np.int32)[:P], "land_pos": d(land_pos or [0], np.int32),
            "land_multi": d(land_multi or [0], np.uint8), "land_w": d(land_w or [0.0], np.float64),
            "ent_ptr": d(ent_ptr, np.int32),
            "ent_owner": d([e[0] for e in flat_e] or [0], np.int32),
            "ent_pos": d([e[1] for e in flat_e] or [0], np.int32),
            "ent_w": d([e[2] for e in flat_e] or [0.0], np.float64),
            "flat_scale": d(flat_scale, np.float64),
            "src_ptr": [d(a, np.int32) for a in src_ptr], "src_flat": [d(a, np.int32) for a in src_flat]}
    return flat, s1
