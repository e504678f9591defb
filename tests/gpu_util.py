"""Shared helpers for the GPU parity tests (inputs on the bf16-exact grid,
SURVEY §8(d): tokens on 2^-7, gate weights on 2^-10, expert weights rounded
to bf16, fed identically to the oracle as float64)."""
import numpy as np
import torch


def grid_tokens(rng, *shape):
    return np.round(rng.uniform(-1, 1, shape) * 128) / 128


def grid_gate(rng, H, E):
    return np.round(rng.uniform(-0.1, 0.1, (H, E)) * 1024) / 1024


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(torch.float64).numpy()


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dtype).cuda()


def host(t):
    return t.detach().to(torch.float64).cpu().numpy() if t.is_floating_point() else t.cpu().numpy()


def max_rel_diff(a, b):
    """moesim::max_rel_diff (matrix.hpp:47-62): |a-b| / max(|a|,|b|,1)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def norm_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return float(d / n) if n > 0 else float(d)
