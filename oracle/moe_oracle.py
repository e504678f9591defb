"""CPU restatement of the reference MoE-block hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity oracle.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` leg may import it, and only as the checker:
nothing in ``paper_2508_13337_b200`` imports it, and the product path fails
loudly when the CUDA library is missing instead of falling back here.

It restates, in numpy with explicit operation order, the reference simulator
``moesim`` (``/root/reference/proj``).  Every function cites the reference
file:line it follows.  Arithmetic reproduces the reference bit for bit:

* ``matmul`` sums ascending ``p`` with a separate multiply and add per term
  (``src/kernels/kernels_scalar.cpp:11-23``; the project builds with
  ``-ffp-contract=off``, ``CMakeLists.txt:15``);
* softmax sums ascending expert id and uses the C library ``exp``
  (``src/gating.cpp:36-43``);
* the weighted combine adds copies in ascending packed-row order
  (``src/pft.cpp:79-91``).

Parity of this restatement is PINNED two ways (tests/test_oracle.py):
the reference's own known-answer vectors (test_gating.cpp, test_pft.cpp,
test_pf_pipeline.cpp, test_rbd.cpp, test_kernels.cpp) and bit-for-bit
comparison with the unmodified reference compiled into
``oracle/_ref/libmoesim_ref.so`` on seeded random trials.

Restated beyond the reference (parity unpinned by it, stated as such in
DESIGN.md): shared experts (``shared_expert_forward``) and top-k
renormalisation (``renorm=True``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1


class MoeError(RuntimeError):
    """Base of the reference's exception family (include/moesim/error.hpp:10-38)."""


class ParseError(MoeError):
    pass


class ValidationError(MoeError):
    pass


class DimensionError(MoeError):
    pass


class IndexError_(MoeError):  # noqa: N801 - mirrors moesim::IndexError
    pass


class CountMismatch(MoeError):
    pass


class PlanMismatch(MoeError):
    pass


# ---------------------------------------------------------------------------
# RNG — include/moesim/rng.hpp:9-61
# ---------------------------------------------------------------------------

def splitmix64(x: int) -> int:
    """rng.hpp:9-14."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def salt_seed(seed: int, a: int, b: int = 0) -> int:
    """rng.hpp:17-19."""
    return splitmix64((splitmix64(seed ^ 0x6D6F6573696D0001) + splitmix64(a) * 3 + b) & MASK64)


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & MASK64


class Rng:
    """xoshiro256** seeded by splitmix64 chaining (rng.hpp:24-61)."""

    def __init__(self, seed: int):
        s = []
        x = seed & MASK64
        for _ in range(4):
            x = splitmix64(x)
            s.append(x)
        self.s = s

    def next_u64(self) -> int:
        s = self.s
        result = (_rotl((s[1] * 5) & MASK64, 7) * 9) & MASK64
        t = (s[1] << 17) & MASK64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = float(self.next_u64() >> 11) * (2.0 ** -53)
        return lo + (hi - lo) * u

    def below(self, n: int) -> int:
        limit = MASK64 - ((MASK64 % n) + 1) % n
        x = self.next_u64()
        while x > limit:
            x = self.next_u64()
        return x % n


# ---------------------------------------------------------------------------
# Arithmetic contract — src/kernels/kernels_scalar.cpp:11-35
# ---------------------------------------------------------------------------

def matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """c[i,j] = sum_p a[i,p]*b[p,j], ascending p, mul and add rounded separately
    (kernels_scalar.cpp:11-23, kernels.hpp:18-20)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise DimensionError("matmul: inner dimensions disagree")
    c = np.zeros((m, n), dtype=np.float64)
    for p in range(k):
        c += a[:, p:p + 1] * b[p:p + 1, :]
    return c


def relu(x: np.ndarray) -> np.ndarray:
    """kernels_scalar.cpp:25-27."""
    return np.where(x > 0.0, x, 0.0)


_exp = np.frompyfunc(math.exp, 1, 1)


# ---------------------------------------------------------------------------
# Gating — src/gating.cpp:14-57
# ---------------------------------------------------------------------------

@dataclass
class GateOutput:
    top_experts: np.ndarray  # [S, k] int64, by descending prob, ties -> lower id
    combine_weights: np.ndarray  # [S, k] float64
    top_k: int
    logits: np.ndarray | None = None


def gate_forward(tokens: np.ndarray, gate_weights: np.ndarray, top_k: int,
                 renorm: bool = False) -> GateOutput:
    """gating.cpp:14-57.  ``renorm`` is a restatement beyond the reference
    (the reference never renormalises, gating.hpp:3-5): w_j / sum_j w_j,
    summed in slot order."""
    tokens = np.asarray(tokens, dtype=np.float64)
    gate_weights = np.asarray(gate_weights, dtype=np.float64)
    if tokens.shape[1] != gate_weights.shape[0]:
        raise DimensionError("gate_forward: tokens.cols != gate_weights.rows")
    S = tokens.shape[0]
    E = gate_weights.shape[1]
    if top_k < 1:
        raise ValidationError("top_k must be >= 1")
    if top_k > E:
        raise ValidationError("top_k must be <= num_experts")
    logits = matmul(tokens, gate_weights)                      # gating.cpp:24-26
    mx = logits[:, 0].copy() if E else np.zeros(S)
    for e in range(1, E):                                      # gating.cpp:39-40
        mx = np.maximum(mx, logits[:, e])
    probs = _exp(logits - mx[:, None]).astype(np.float64)      # gating.cpp:41-42
    s = np.zeros(S, dtype=np.float64)
    for e in range(E):                                          # ascending e
        s = s + probs[:, e]
    probs = probs / s[:, None]                                  # gating.cpp:43
    # partial_sort by (prob desc, id asc) — gating.cpp:45-50
    order = np.argsort(-probs, axis=1, kind="stable")[:, :top_k]
    w = np.take_along_axis(probs, order, axis=1)
    if renorm:
        tot = np.zeros(S, dtype=np.float64)
        for j in range(top_k):
            tot = tot + w[:, j]
        w = w / tot[:, None]
    return GateOutput(order.astype(np.int64), w, top_k, logits)


def make_gate_weights(rng: Rng, model_dim: int, num_experts: int) -> np.ndarray:
    """gating.cpp:59-63 (draw order: row-major [H, E])."""
    return np.array([rng.uniform(-0.1, 0.1) for _ in range(model_dim * num_experts)],
                    dtype=np.float64).reshape(model_dim, num_experts)


@dataclass
class LayerWeights:
    """MoeLayerWeights, include/moesim/moe_instance.hpp:17-21."""
    gate: np.ndarray  # [H, E]
    w1: np.ndarray  # [E, H, F]
    w2: np.ndarray  # [E, F, H]


def make_layer_weights(rng: Rng, E: int, H: int, F: int) -> LayerWeights:
    """src/padded_pipeline.cpp:13-27: gate (H*E), then per expert w1 then w2."""
    gate = make_gate_weights(rng, H, E)
    w1 = np.empty((E, H, F))
    w2 = np.empty((E, F, H))
    for e in range(E):
        w1[e] = np.array([rng.uniform(-0.1, 0.1) for _ in range(H * F)]).reshape(H, F)
        w2[e] = np.array([rng.uniform(-0.1, 0.1) for _ in range(F * H)]).reshape(F, H)
    return LayerWeights(gate, w1, w2)


# ---------------------------------------------------------------------------
# Padding-free token buffer — src/pft.cpp:12-91
# ---------------------------------------------------------------------------

@dataclass
class Pft:
    token_ids: np.ndarray
    expert_ids: np.ndarray
    tokens_per_expert: np.ndarray
    combine_weights: np.ndarray
    x: np.ndarray | None = None

    def size(self) -> int:
        return int(self.token_ids.shape[0])


def pft_construct(max_token_count: int, num_experts: int, seq_len: int, top_k: int,
                  top_experts, combine_weights) -> Pft:
    """pft.cpp:12-60."""
    if max_token_count < 1:
        raise ValidationError("max_token_count must be >= 1")
    if num_experts < 1:
        raise ValidationError("num_experts must be >= 1")
    if top_k < 1:
        raise ValidationError("top_k must be >= 1")
    top = np.asarray(top_experts, dtype=np.int64).reshape(-1)
    w = np.asarray(combine_weights, dtype=np.float64).reshape(-1)
    flat = seq_len * top_k
    if top.shape[0] != flat or w.shape[0] != flat:
        raise DimensionError("pft_construct: routing arrays must be seq_len * top_k")
    t2 = top.reshape(seq_len, top_k)
    bad = (top < 0) | (top >= num_experts)
    srt = np.sort(t2, axis=1)
    if bad.any() or (top_k > 1 and np.any(srt[:, 1:] == srt[:, :-1])):
        # pft.cpp:23-31: the first offending (t, a) in row-major order decides
        for t in range(seq_len):
            for a in range(top_k):
                e = t2[t, a]
                if e < 0 or e >= num_experts:
                    raise IndexError_("expert id out of range")
                if np.any(t2[t, :a] == e):
                    raise ValidationError("top_experts rows must contain distinct expert ids")
    token_ids, expert_ids, cw = [], [], []
    tpe = np.zeros(num_experts, dtype=np.int64)
    for e in range(num_experts):                                # pft.cpp:35-57
        members = np.nonzero(top == e)[0]                       # ascending flat pos
        if members.shape[0] > max_token_count:
            # sort by (w desc, f asc), keep cap, re-sort by f   # pft.cpp:42-51
            order = np.lexsort((members, -w[members]))
            members = np.sort(members[order[:max_token_count]])
        tpe[e] = members.shape[0]
        token_ids.append(members // top_k)
        expert_ids.append(np.full(members.shape[0], e, dtype=np.int64))
        cw.append(w[members])
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
    return Pft(cat(token_ids, np.int64), cat(expert_ids, np.int64), tpe,
               cat(cw, np.float64))


def pft_from_gate(max_token_count: int, num_experts: int, gate: GateOutput) -> Pft:
    """pft.cpp:62-66."""
    S = gate.top_experts.shape[0]
    return pft_construct(max_token_count, num_experts, S, gate.top_k,
                         gate.top_experts, gate.combine_weights)


def gather_rows(src: np.ndarray, ids) -> np.ndarray:
    """pft.cpp:68-77."""
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size and (ids.min() < 0 or ids.max() >= src.shape[0]):
        raise IndexError_("gather_rows: row id out of range")
    return np.asarray(src, dtype=np.float64)[ids].copy()


def scatter_combine(rows: np.ndarray, token_ids, weights, seq_len: int) -> np.ndarray:
    """pft.cpp:79-91: out zero-initialised, ``out[t_i] += w_i * rows[i]`` for i
    ascending (kernels_scalar.cpp:29-31).  Copies of one token are applied in
    ascending i; distinct tokens never interact, so rounds of one copy per
    token reproduce the sequential order exactly."""
    rows = np.asarray(rows, dtype=np.float64)
    token_ids = np.asarray(token_ids, dtype=np.int64)
    weights = np.asarray(weights, dtype=np.float64)
    if rows.shape[0] != token_ids.shape[0] or rows.shape[0] != weights.shape[0]:
        raise DimensionError("scatter_combine: rows and ERI arrays disagree")
    if token_ids.size and (token_ids.min() < 0 or token_ids.max() >= seq_len):
        raise IndexError_("scatter_combine: token id out of range")
    cols = rows.shape[1] if rows.ndim == 2 else 0
    out = np.zeros((seq_len, cols), dtype=np.float64)
    _ordered_axpy(out, token_ids, weights, rows)
    return out


def _ordered_axpy(out, dst_ids, weights, rows):
    """Apply out[dst_i] += w_i * rows[i] in ascending i (duplicates in order)."""
    n = dst_ids.shape[0]
    if n == 0:
        return
    # occurrence index of each i among equal dst ids, in ascending i
    order = np.argsort(dst_ids, kind="stable")
    sd = dst_ids[order]
    start = np.r_[0, np.nonzero(np.diff(sd))[0] + 1]
    occ_sorted = np.arange(n) - np.repeat(start, np.diff(np.r_[start, n]))
    occ = np.empty(n, dtype=np.int64)
    occ[order] = occ_sorted
    for r in range(int(occ.max()) + 1):
        sel = np.nonzero(occ == r)[0]
        out[dst_ids[sel]] += weights[sel, None] * rows[sel]


# ---------------------------------------------------------------------------
# Grouped expert FFN — src/pf_pipeline.cpp:83-105
# ---------------------------------------------------------------------------

def grouped_expert_mlp(inp: np.ndarray, rows_per_expert, w: LayerWeights,
                       first_expert: int, exact: bool = True) -> np.ndarray:
    """``exact=False`` swaps the ordered matmul for BLAS (same maths, last-ulp
    differences) — only for comparisons against the bf16 path, whose
    tolerance is ~1e-2."""
    mm = matmul if exact else (lambda a, b: np.asarray(a, np.float64) @ np.asarray(b, np.float64))
    inp = np.asarray(inp, dtype=np.float64)
    out = np.zeros_like(inp)
    off = 0
    for i, n in enumerate(rows_per_expert):
        n = int(n)
        if n == 0:
            continue
        w1 = w.w1[first_expert + i]
        w2 = w.w2[first_expert + i]
        if inp.shape[1] != w1.shape[0]:
            raise DimensionError("grouped_expert_mlp: activation width mismatch")
        mid = relu(mm(inp[off:off + n], w1))
        out[off:off + n] = mm(mid, w2)
        off += n
    if off != inp.shape[0]:
        raise CountMismatch("grouped_expert_mlp: segment counts disagree with input rows")
    return out


# ---------------------------------------------------------------------------
# Expert-parallel exchange — src/collectives.cpp:81-141, src/pf_pipeline.cpp
# ---------------------------------------------------------------------------

@dataclass
class Ledger:
    """Byte accounting per kind (collectives.cpp:45-56, charge_message)."""
    bytes: dict = field(default_factory=dict)  # kind -> [self, intra, inter]

    def charge(self, kind, node_of, i, j, nbytes):
        b = self.bytes.setdefault(kind, [0, 0, 0])
        if i == j:
            b[0] += nbytes
        elif node_of[i] == node_of[j]:
            b[1] += nbytes
        else:
            b[2] += nbytes

    def get(self, kind):
        return self.bytes.get(kind, [0, 0, 0])


@dataclass
class PfDispatch:
    expert_input: list
    recv_per_expert: list
    row_counts: np.ndarray
    arrival_to_grouped: list


def pf_dispatch(node_of, pfts, num_experts, ledger: Ledger | None = None,
                dtype_bytes: int = 2) -> PfDispatch:
    """pf_pipeline.cpp:12-81."""
    W = len(node_of)
    if len(pfts) != W:
        raise DimensionError("pf_dispatch: need one packed buffer per worker")
    if num_experts % W != 0:
        raise ValidationError("num_experts must be divisible by the worker-group size")
    el = num_experts // W
    counts = np.zeros((W, W), dtype=np.int64)
    for i, p in enumerate(pfts):
        counts[i] = p.tokens_per_expert.reshape(W, el).sum(axis=1)
    H = next((p.x.shape[1] for p in pfts if p.x is not None and p.x.shape[0]), 0)
    if ledger is not None:
        for i in range(W):
            for j in range(W):
                if i != j:
                    ledger.charge("dispatch_counts", node_of, i, j, el * 8)
                if counts[i, j]:
                    ledger.charge("dispatch_rows", node_of, i, j, int(counts[i, j]) * H * dtype_bytes)
    ei, rpe, a2g = [], [], []
    for j in range(W):
        # arrivals (src, le, pos) regrouped to (le, src, pos)     # pf_pipeline.cpp:47-79
        per = np.zeros(el, dtype=np.int64)
        for src in range(W):
            per += pfts[src].tokens_per_expert[j * el:(j + 1) * el]
        nxt = np.r_[0, np.cumsum(per)[:-1]].astype(np.int64)
        n_rows = int(per.sum())
        grouped = np.zeros((n_rows, H))
        amap = np.zeros(n_rows, dtype=np.int64)
        a = 0
        for src in range(W):
            p = pfts[src]
            blk = np.r_[0, np.cumsum(p.tokens_per_expert)].astype(np.int64)
            for le in range(el):
                e = j * el + le
                n = int(p.tokens_per_expert[e])
                g = nxt[le] + np.arange(n)
                grouped[g] = p.x[blk[e]:blk[e] + n]
                amap[a:a + n] = g
                nxt[le] += n
                a += n
        ei.append(grouped)
        rpe.append(per)
        a2g.append(amap)
    return PfDispatch(ei, rpe, counts, a2g)


def pf_combine(node_of, disp: PfDispatch, expert_out, pfts, seq_lens,
               ledger: Ledger | None = None, dtype_bytes: int = 2):
    """pf_pipeline.cpp:107-135: undo the regroup, reverse exchange with the
    transposed counts, scatter_combine per worker."""
    W = len(node_of)
    el = pfts[0].tokens_per_expert.shape[0] // W
    out = []
    # Back at source w, the rows arrive in (dest asc, le asc, pos) order,
    # which is exactly w's packed (expert-major) order.
    for w in range(W):
        p = pfts[w]
        rows = np.zeros((p.size(), expert_out[0].shape[1] if expert_out else 0))
        blk = np.r_[0, np.cumsum(p.tokens_per_expert)].astype(np.int64)
        for j in range(W):
            per_before = np.zeros(el, dtype=np.int64)
            for src in range(w):
                per_before += pfts[src].tokens_per_expert[j * el:(j + 1) * el]
            base = np.r_[0, np.cumsum(disp.recv_per_expert[j])[:-1]]
            for le in range(el):
                e = j * el + le
                n = int(p.tokens_per_expert[e])
                g0 = int(base[le] + per_before[le])
                rows[blk[e]:blk[e] + n] = expert_out[j][g0:g0 + n]
                if ledger is not None and n:
                    H = rows.shape[1]
                    ledger.charge("combine_rows", node_of, j, w, n * H * dtype_bytes)
        out.append(scatter_combine(rows, p.token_ids, p.combine_weights, seq_lens[w]))
    return out


def pf_moe_forward(tokens_per_worker, w: LayerWeights, num_experts: int, top_k: int,
                   cap: int, node_of=None, ledger: Ledger | None = None, renorm=False,
                   return_pfts=False, exact=True, gates=None):
    """pf_pipeline.cpp:137-169.  ``gates`` optionally supplies each worker's
    (top_experts, combine_weights) instead of recomputing them — used to
    isolate the one libm-dependent value (exp in the softmax) when checking a
    device pipeline bit for bit."""
    W = len(tokens_per_worker)
    node_of = list(range(W)) if node_of is None else list(node_of)
    if num_experts % W != 0:
        raise ValidationError("num_experts must be divisible by the worker-group size")
    el = num_experts // W
    pfts = []
    for i, x in enumerate(tokens_per_worker):
        if gates is not None:
            g = GateOutput(np.asarray(gates[i][0], np.int64), np.asarray(gates[i][1], np.float64), top_k)
        else:
            g = gate_forward(x, w.gate, top_k, renorm=renorm)
        p = pft_construct(cap, num_experts, x.shape[0], top_k, g.top_experts, g.combine_weights)
        p.x = gather_rows(x, p.token_ids)
        pfts.append(p)
    disp = pf_dispatch(node_of, pfts, num_experts, ledger)
    eo = [grouped_expert_mlp(disp.expert_input[j], disp.recv_per_expert[j], w, j * el, exact)
          for j in range(W)]
    out = pf_combine(node_of, disp, eo, pfts, [x.shape[0] for x in tokens_per_worker], ledger)
    return (out, pfts, disp, eo) if return_pfts else out


# ---------------------------------------------------------------------------
# Redundancy-bypassing dispatch — src/rbd.cpp
# ---------------------------------------------------------------------------

def expert_nodes(node_of, num_experts):
    """rbd.cpp:16-24."""
    W = len(node_of)
    if W == 0 or num_experts % W != 0:
        raise ValidationError("num_experts must be divisible by the worker-group size")
    el = num_experts // W
    return np.array([node_of[e // el] for e in range(num_experts)], dtype=np.int64)


@dataclass
class RbdPlan:
    pilot_mask: np.ndarray  # [B] uint8
    pilot_of: np.ndarray  # [B] packed row of the group's pilot


def select_pilots(pft: Pft, node_of, num_experts: int, seed: int) -> RbdPlan:
    """rbd.cpp:26-81: group copies by (token, node(expert)) in ascending key
    order (std::map), one Rng(seed).below(|group|) draw per group picks the
    pilot among the group's members in packed order."""
    nodes = expert_nodes(node_of, num_experts)
    if pft.tokens_per_expert.shape[0] != num_experts:
        raise DimensionError("select_pilots: tokens_per_expert length mismatch")
    B = pft.size()
    if B and (pft.expert_ids.min() < 0 or pft.expert_ids.max() >= num_experts):
        raise IndexError_("select_pilots: expert id out of range")
    keys = np.stack([pft.token_ids, nodes[pft.expert_ids]], axis=1) if B else np.zeros((0, 2), np.int64)
    order = np.lexsort((np.arange(B), keys[:, 1], keys[:, 0])) if B else np.zeros(0, np.int64)
    mask = np.zeros(B, dtype=np.uint8)
    pilot_of = np.full(B, -1, dtype=np.int64)
    rng = Rng(seed)
    i = 0
    while i < B:
        j = i
        k0 = tuple(keys[order[i]])
        while j < B and tuple(keys[order[j]]) == k0:
            j += 1
        members = order[i:j]
        pilot = int(members[rng.below(len(members))])
        mask[pilot] = 1
        pilot_of[members] = pilot
        i = j
    return RbdPlan(mask, pilot_of)


def rbd_combine_from_outputs(pft: Pft, plan: RbdPlan, y_of_copy: np.ndarray, seq_len: int):
    """rbd.cpp:287-358 restated per source worker.  ``y_of_copy[i]`` is the
    expert output of packed row i.  Landing worker: multi-copy groups start
    from ``scale(y_pilot, w_pilot)`` (kernels_scalar.cpp:33-35) and ``axpy``
    each replica in slot order (owner ascending, then replica sequence — i.e.
    ascending packed row); singleton groups return raw.  Source: pilots in
    pilot (packed-row) order, ``axpy`` with 1.0 (merged) or w (singleton)."""
    B = pft.size()
    cols = y_of_copy.shape[1] if y_of_copy.ndim == 2 else 0
    out = np.zeros((seq_len, cols))
    pilots = np.nonzero(plan.pilot_mask)[0]
    merged = {}
    multi = {}
    for p in pilots:
        members = np.nonzero(plan.pilot_of == p)[0]
        reps = [int(m) for m in members if m != p]
        if reps:
            buf = y_of_copy[p] * pft.combine_weights[p]
            for r in reps:  # ascending packed row
                buf = buf + pft.combine_weights[r] * y_of_copy[r]
            merged[int(p)] = buf
            multi[int(p)] = True
        else:
            merged[int(p)] = y_of_copy[p]
            multi[int(p)] = False
    # source-side accumulation in pilot order; rounds per token keep order
    dst = pft.token_ids[pilots]
    wts = np.array([1.0 if multi[int(p)] else pft.combine_weights[p] for p in pilots])
    rows = np.array([merged[int(p)] for p in pilots]).reshape(len(pilots), cols)
    _ordered_axpy(out, dst, wts, rows)
    return out


def rbd_moe_forward(tokens_per_worker, w: LayerWeights, num_experts: int, top_k: int,
                    cap: int, seed: int, node_of=None, gates=None, exact=True, shared=None):
    """rbd.cpp:360-386 (dispatch buffers equal pf_dispatch's bit for bit,
    rbd.hpp:50, so expert outputs per copy equal the plain path's)."""
    W = len(tokens_per_worker)
    node_of = list(range(W)) if node_of is None else list(node_of)
    _, pfts, disp, eo = pf_moe_forward(tokens_per_worker, w, num_experts, top_k, cap,
                                       node_of, return_pfts=True, gates=gates, exact=exact)
    el = num_experts // W
    out = []
    for s in range(W):
        p = pfts[s]
        # y per packed row of source s: locate each copy in its owner's grouped buffer
        y = np.zeros((p.size(), eo[0].shape[1] if eo else 0))
        blk = np.r_[0, np.cumsum(p.tokens_per_expert)].astype(np.int64)
        for j in range(W):
            base = np.r_[0, np.cumsum(disp.recv_per_expert[j])[:-1]]
            for le in range(el):
                e = j * el + le
                before = sum(int(pfts[q].tokens_per_expert[e]) for q in range(s))
                n = int(p.tokens_per_expert[e])
                g0 = int(base[le]) + before
                y[blk[e]:blk[e] + n] = eo[j][g0:g0 + n]
        plan = select_pilots(p, node_of, num_experts, salt_seed(seed, s, 0))
        o = rbd_combine_from_outputs(p, plan, y, tokens_per_worker[s].shape[0])
        if shared is not None:  # shared experts added after the routed groups
            o = o + 1.0 * shared_expert_forward(tokens_per_worker[s], shared[0], shared[1], exact)
        out.append(o)
    return out


def redundancy_counts_internode(pft: Pft, source_node: int, expert_node) -> tuple[int, int]:
    """rbd.cpp:427-442: (copies leaving the source node, distinct (token, node) groups)."""
    en = np.asarray(expert_node)[pft.expert_ids]
    sel = en != source_node
    pairs = set(zip(pft.token_ids[sel].tolist(), en[sel].tolist()))
    return int(sel.sum()), len(pairs)


def sample_redundancy(rng: Rng, tokens: int, top_k: int, expert_node) -> float:
    """rbd.cpp:451-474 (partial Fisher-Yates per token)."""
    E = len(expert_node)
    if top_k < 1:
        raise ValidationError("top_k must be >= 1")
    if top_k > E:
        raise ValidationError("top_k must be <= num_experts")
    if tokens == 0:
        return 0.0
    ids = list(range(E))
    distinct = 0
    for _ in range(tokens):
        nodes = []
        for j in range(top_k):
            pick = j + rng.below(E - j)
            ids[j], ids[pick] = ids[pick], ids[j]
            nodes.append(expert_node[ids[j]])
        distinct += len(set(nodes))
    return 1.0 - distinct / (tokens * top_k)


# ---------------------------------------------------------------------------
# Sequence-sharded MoE block — src/ssmb.cpp:12-46
# ---------------------------------------------------------------------------

def ssmb_forward(tokens: np.ndarray, G: int, w: LayerWeights, num_experts: int, top_k: int,
                 cap: int) -> np.ndarray:
    S = tokens.shape[0]
    if G < 1:
        raise ValidationError("ssmb_forward: shard count must be >= 1")
    if G > S:
        raise ValidationError("ssmb_forward: more shards than sequence rows")
    base = S // G
    outs = []
    for g in range(G):
        b = g * base
        rows = S - b if g == G - 1 else base
        outs.append(pf_moe_forward([tokens[b:b + rows]], w, num_experts, top_k, cap)[0])
    return np.concatenate(outs, axis=0)


def ssmb_shards(S: int, G: int):
    """Contiguous shard bounds (ssmb.cpp:21-28): the last shard takes the remainder."""
    base = S // G
    return [(g * base, (S - g * base) if g == G - 1 else base) for g in range(G)]


# ---------------------------------------------------------------------------
# Shared experts — restatement beyond the reference (parity unpinned by it)
# ---------------------------------------------------------------------------

def shared_expert_forward(x: np.ndarray, sw1: np.ndarray, sw2: np.ndarray,
                          exact: bool = True) -> np.ndarray:
    """n_shared shared experts of width Fs, each the reference's expert FFN
    applied to every token (grouped_expert_mlp over one segment of S rows,
    pf_pipeline.cpp:83-105).  As in DeepSeek-MoE they run as ONE FFN of width
    n_shared*Fs (W1 concatenated along F, W2 along its rows): the sum over
    shared experts is one ascending accumulation chain over the concatenated
    inner dimension.  sw1 [ns, H, Fs], sw2 [ns, Fs, H]."""
    ns, H, Fs = sw1.shape
    w1c = np.concatenate([sw1[s] for s in range(ns)], axis=1)  # [H, ns*Fs]
    w2c = np.concatenate([sw2[s] for s in range(ns)], axis=0)  # [ns*Fs, H]
    mm = matmul if exact else (lambda a, b: np.asarray(a, np.float64) @ np.asarray(b, np.float64))
    return mm(relu(mm(x, w1c)), w2c)


def moe_layer_with_shared(x, w: LayerWeights, num_experts, top_k, cap, sw1, sw2, exact=True,
                          gates=None):
    """Routed copies combined first (pf_moe_forward, W=1; ascending expert),
    then the shared-expert output added with weight 1.0 (axpy,
    kernels_scalar.cpp:29-31)."""
    routed = pf_moe_forward([x], w, num_experts, top_k, cap, exact=exact, gates=gates)[0]
    return routed + 1.0 * shared_expert_forward(x, sw1, sw2, exact)


# ---------------------------------------------------------------------------
# Synthetic inputs on the bf16-exact grid
# ---------------------------------------------------------------------------

def snap(x: np.ndarray, step: float) -> np.ndarray:
    """Round to the nearest multiple of ``step`` (values stay bf16-exact when
    |x|/step < 256)."""
    return np.round(np.asarray(x, dtype=np.float64) / step) * step
