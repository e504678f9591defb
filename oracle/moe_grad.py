"""Gradient oracle of the MoE block — TEST INFRASTRUCTURE ONLY.

The reference is forward-only, so gradients are RESTATED: torch
fp64 autograd over the reference forward semantics:

* routing (top-k by probability, ties to the lower id, gating.cpp:45-50) and
  the capacity drops (pft.cpp:42-51) are constants taken from the pinned
  restatement (moe_oracle), exactly as the reference treats them;
* the combine weights are the raw softmax probabilities of the selected
  experts (no renormalisation, gating.cpp:51-54), so dL/dlogits flows
  through the full softmax;
* experts are relu(x W1) W2 (pf_pipeline.cpp:97-99); shared experts are the
  merged FFN of moe_oracle.shared_expert_forward.

Pinned in tests/test_oracle_grad.py against central finite differences of the
UNMODIFIED reference forward (oracle/_ref) on random parameter entries.
"""
from __future__ import annotations

import numpy as np
import torch

from . import moe_oracle as O


def moe_forward_torch(x, gate, w1, w2, k, cap, sw1=None, sw2=None):
    """x [S,H], gate [H,E], w1 [E,H,F], w2 [E,F,H] (fp64 tensors)."""
    S, H = x.shape
    E = gate.shape[1]
    g = O.gate_forward(x.detach().numpy(), gate.detach().numpy(), k)
    p = O.pft_from_gate(cap, E, g)
    probs = torch.softmax(x @ gate, dim=1)
    y = torch.zeros_like(x)
    tid = torch.from_numpy(p.token_ids)
    eid = torch.from_numpy(p.expert_ids)
    for e in range(E):
        sel = tid[eid == e]
        if sel.numel() == 0:
            continue
        h = torch.relu(x[sel] @ w1[e]) @ w2[e]
        y = y.index_add(0, sel, probs[sel, e:e + 1] * h)
    if sw1 is not None:
        w1c = torch.cat([sw1[s] for s in range(sw1.shape[0])], dim=1)
        w2c = torch.cat([sw2[s] for s in range(sw2.shape[0])], dim=0)
        y = y + torch.relu(x @ w1c) @ w2c
    return y


def moe_grads(x, gate, w1, w2, dy, k, cap, sw1=None, sw2=None):
    """dL/d{x, gate, w1, w2, sw1, sw2} of L = <y, dy> (numpy fp64 in/out)."""
    t = {n: torch.tensor(np.asarray(v, np.float64), requires_grad=True)
         for n, v in dict(x=x, gate=gate, w1=w1, w2=w2, sw1=sw1, sw2=sw2).items() if v is not None}
    y = moe_forward_torch(t["x"], t["gate"], t["w1"], t["w2"], k, cap, t.get("sw1"), t.get("sw2"))
    (y * torch.tensor(np.asarray(dy, np.float64))).sum().backward()
    out = {n: v.grad.numpy() for n, v in t.items()}
    out["y"] = y.detach().numpy()
    return out
