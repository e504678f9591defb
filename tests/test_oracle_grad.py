"""Pins the gradient restatement (oracle/moe_grad.py): its forward equals the
reference's pf_moe_forward, and its gradients equal central finite
differences of the UNMODIFIED reference forward (oracle/_ref) on random
parameter entries (routing held fixed: steps are far below the routing
margins, checked)."""
import numpy as np
import pytest

from oracle import moe_oracle as O
from oracle import moe_grad as G


def _inst(seed, S=19, E=8, k=3, H=6, F=5, cap=None):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (S, H))
    gate = rng.uniform(-0.5, 0.5, (H, E))
    w1 = rng.uniform(-0.5, 0.5, (E, H, F))
    w2 = rng.uniform(-0.5, 0.5, (E, F, H))
    dy = rng.uniform(-1, 1, (S, H))
    return x, gate, w1, w2, dy, k, (S * k if cap is None else cap)


@pytest.mark.parametrize("cap", [None, 4])
def test_grad_oracle_forward_matches_reference(ref, cap):
    x, gate, w1, w2, dy, k, cap = _inst(1, cap=cap)
    got = G.moe_grads(x, gate, w1, w2, dy, k, cap)["y"]
    L = ref.Layer(gate, w1, w2)
    want, _ = L.pf_moe_forward(x[None], k, cap)
    assert np.max(np.abs(got - want[0])) < 1e-12


@pytest.mark.parametrize("cap", [None, 4])
def test_grad_oracle_vs_reference_finite_differences(ref, cap):
    x, gate, w1, w2, dy, k, cap = _inst(2, cap=cap)
    g = G.moe_grads(x, gate, w1, w2, dy, k, cap)
    rng = np.random.default_rng(3)
    h = 1e-6
    top0 = O.gate_forward(x, gate, k).top_experts

    def f(xx, gg, a, b):
        L = ref.Layer(gg, a, b)
        y, _ = L.pf_moe_forward(xx[None], k, cap)
        return float(np.sum(y[0] * dy))

    for name, arr in (("x", x), ("gate", gate), ("w1", w1), ("w2", w2)):
        for _ in range(4):
            idx = tuple(int(rng.integers(0, d)) for d in arr.shape)
            plus, minus = [v.copy() for v in (x, gate, w1, w2)], [v.copy() for v in (x, gate, w1, w2)]
            j = ("x", "gate", "w1", "w2").index(name)
            plus[j][idx] += h
            minus[j][idx] -= h
            # routing must not change under the probe
            assert np.array_equal(O.gate_forward(plus[0], plus[1], k).top_experts, top0)
            assert np.array_equal(O.gate_forward(minus[0], minus[1], k).top_experts, top0)
            fd = (f(*plus) - f(*minus)) / (2 * h)
            assert abs(fd - g[name][idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx, fd, g[name][idx])
