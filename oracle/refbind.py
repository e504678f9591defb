"""ctypes binding of oracle/_ref/libmoesim_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference simulator compiled from
/root/reference/proj by oracle/Makefile, plus the flat shim oracle/ref_shim.cpp.
Used by tests/ to pin the numpy restatement (moe_oracle.py) and by bench.py's
cpu_baseline / ``--impl reference`` arm.  Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libmoesim_ref.so")

_i64 = C.c_int64
_u64 = C.c_uint64
_p = C.c_void_p

_lib = None

KIND_NAMES = ["dispatch_counts", "dispatch_rows", "combine_rows", "rbd_dispatch_counts",
              "rbd_dispatch_meta", "rbd_dispatch_rows1", "rbd_dispatch_meta2",
              "rbd_dispatch_rows2", "rbd_combine_rows2", "rbd_combine_rows1",
              "ssmb_gather_rows"]

ERRORS = {1: "ParseError", 2: "ValidationError", 3: "DimensionError", 4: "IndexError",
          5: "CountMismatch", 6: "PlanMismatch", 99: "Error"}


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")
        self.msg = msg


def available() -> bool:
    return os.path.exists(LIB_PATH)


def build() -> None:
    """Build oracle/_ref when the reference sources are present (this container)."""
    if os.path.isdir("/root/reference/proj/src"):
        import subprocess
        subprocess.run(["make", "-s", "-j8", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_ledger_csv.restype = C.c_char_p
        L.ref_kernel_backend.restype = C.c_char_p
        L.ref_salt_seed.restype = _u64
        L.ref_salt_seed.argtypes = [_u64, _u64, _u64]
        L.ref_rng_u64.argtypes = [_u64, _i64, _p]
        L.ref_rng_uniform.argtypes = [_u64, _i64, C.c_double, C.c_double, _p]
        L.ref_make_layer_weights.argtypes = [_u64, _i64, _i64, _i64, _p, _p, _p]
        L.ref_gate_forward.argtypes = [_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p]
        L.ref_pft_construct.argtypes = [_i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p]
        L.ref_gather_rows.argtypes = [_p, _i64, _i64, _p, _i64, _p]
        L.ref_scatter_combine.argtypes = [_p, _i64, _i64, _p, _i64, _p, _i64, _i64, _p]
        L.ref_layer_create.restype = _p
        L.ref_layer_create.argtypes = [_i64, _i64, _i64, _p, _p, _p]
        L.ref_layer_destroy.argtypes = [_p]
        L.ref_grouped_expert_mlp.argtypes = [_p, _p, _i64, _p, _i64, _i64, _p]
        L.ref_pf_moe_forward.argtypes = [_p, _i64, _p, _p, _i64, _i64, _i64, _p, _p]
        L.ref_pf_moe_forward_noncopy.argtypes = [_p, _i64, _p, _p, _i64, _i64, _i64, _p]
        L.ref_rbd_moe_forward.argtypes = [_p, _i64, _p, _p, _i64, _i64, _i64, _u64, _p, _p]
        L.ref_padded_moe_forward.argtypes = [_p, _i64, _p, _p, _i64, _i64, _i64, _p]
        L.ref_dispatch.argtypes = [_p, _i64, _p, _p, _i64, _i64, _i64, C.c_int, _u64,
                                   _p, _p, _p, _p, _p, _p]
        L.ref_select_pilots.argtypes = [_i64, _p, _p, _p, _p, _i64, _i64, _p, _u64, _p]
        L.ref_ssmb_forward.argtypes = [_p, _i64, _p, _p, _i64, _i64, _i64, _p, _p]
        L.ref_sample_redundancy.restype = C.c_double
        L.ref_sample_redundancy.argtypes = [_u64, _i64, _i64, _i64, _p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64a(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def salt_seed(seed, a, b=0) -> int:
    return int(lib().ref_salt_seed(seed, a, b))


def rng_u64(seed, n) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().ref_rng_u64(seed, n, _ptr(out))
    return out


def rng_uniform(seed, n, lo, hi) -> np.ndarray:
    out = np.zeros(n, dtype=np.float64)
    lib().ref_rng_uniform(seed, n, lo, hi, _ptr(out))
    return out


def make_layer_weights(seed, E, H, F):
    gate = np.zeros((H, E))
    w1 = np.zeros((E, H, F))
    w2 = np.zeros((E, F, H))
    lib().ref_make_layer_weights(seed, E, H, F, _ptr(gate), _ptr(w1), _ptr(w2))
    return gate, w1, w2


def gate_forward(x, wg, k):
    x = _f64(x)
    wg = _f64(wg)
    S, H = x.shape
    Hg, E = wg.shape
    top = np.zeros((S, k), dtype=np.int64)
    w = np.zeros((S, k))
    _check(lib().ref_gate_forward(_ptr(x), _ptr(wg), S, H, Hg, E, k, _ptr(top), _ptr(w)))
    return top, w


def pft_construct(cap, E, S, k, top, w):
    top = _i64a(top).reshape(-1)
    w = _f64(w).reshape(-1)
    n = max(top.shape[0], 1)
    tid = np.zeros(n, np.int64)
    eid = np.zeros(n, np.int64)
    cw = np.zeros(n)
    tpe = np.zeros(max(E, 1), np.int64)
    B = np.zeros(1, np.int64)
    _check(lib().ref_pft_construct(cap, E, S, k, top.shape[0], _ptr(top), _ptr(w), _ptr(tid),
                                   _ptr(eid), _ptr(cw), _ptr(tpe), _ptr(B)))
    b = int(B[0])
    return tid[:b], eid[:b], cw[:b], tpe[:E]


class Layer:
    """Reference MoeLayerWeights held inside the C++ library."""

    def __init__(self, gate, w1, w2):
        gate, w1, w2 = _f64(gate), _f64(w1), _f64(w2)
        self.H, self.E = gate.shape
        self.F = w1.shape[2]
        self.h = lib().ref_layer_create(self.E, self.H, self.F, _ptr(gate), _ptr(w1), _ptr(w2))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_layer_destroy(self.h)
            self.h = None

    def grouped_expert_mlp(self, inp, rpe, first_expert):
        inp = _f64(inp)
        rpe = _i64a(rpe)
        out = np.zeros_like(inp)
        _check(lib().ref_grouped_expert_mlp(self.h, _ptr(inp), inp.shape[0], _ptr(rpe),
                                            rpe.shape[0], first_expert, _ptr(out)))
        return out

    def _fwd(self, fn, tokens, k, cap, node_of, *extra):
        tokens = _f64(tokens)  # [W, S, H]
        W, S, H = tokens.shape
        node_of = _i64a(list(range(W)) if node_of is None else node_of)
        out = np.zeros_like(tokens)
        led = np.zeros(3 * len(KIND_NAMES), np.uint64)
        _check(fn(self.h, W, _ptr(node_of), _ptr(tokens), S, k, cap, *extra, _ptr(out), _ptr(led)))
        return out, {KIND_NAMES[i]: led[3 * i:3 * i + 3].astype(int).tolist()
                     for i in range(len(KIND_NAMES))}

    def pf_moe_forward(self, tokens, k, cap, node_of=None):
        return self._fwd(lib().ref_pf_moe_forward, tokens, k, cap, node_of)

    def pf_moe_forward_noncopy(self, tokens, k, cap, node_of=None):
        """pf_moe_forward's composition with the weights by reference (no
        per-call copy of MoeLayerWeights; see ref_shim.cpp)."""
        tokens = _f64(tokens)
        W, S, H = tokens.shape
        node_of = _i64a(list(range(W)) if node_of is None else node_of)
        out = np.zeros_like(tokens)
        _check(lib().ref_pf_moe_forward_noncopy(self.h, W, _ptr(node_of), _ptr(tokens), S, k, cap, _ptr(out)))
        return out

    def rbd_moe_forward(self, tokens, k, cap, seed, node_of=None):
        return self._fwd(lib().ref_rbd_moe_forward, tokens, k, cap, node_of, C.c_uint64(seed))

    def padded_moe_forward(self, tokens, k, cap, node_of=None):
        tokens = _f64(tokens)
        W, S, H = tokens.shape
        node_of = _i64a(list(range(W)) if node_of is None else node_of)
        out = np.zeros_like(tokens)
        _check(lib().ref_padded_moe_forward(self.h, W, _ptr(node_of), _ptr(tokens), S, k, cap,
                                            _ptr(out)))
        return out

    def dispatch(self, tokens, k, cap, node_of=None, rbd=False, seed=0):
        tokens = _f64(tokens)
        W, S, H = tokens.shape
        node_of = _i64a(list(range(W)) if node_of is None else node_of)
        el = self.E // W if W and self.E % W == 0 else 1
        ei = np.zeros(W * S * k * H + 1)
        rows = np.zeros(W, np.int64)
        rpe = np.zeros(W * el, np.int64)
        rc = np.zeros(W * W, np.int64)
        pm = np.zeros(W * S * k + 1, np.uint8)
        led = np.zeros(3 * len(KIND_NAMES), np.uint64)
        _check(lib().ref_dispatch(self.h, W, _ptr(node_of), _ptr(tokens), S, k, cap, int(rbd),
                                  C.c_uint64(seed), _ptr(ei), _ptr(rows), _ptr(rpe), _ptr(rc),
                                  _ptr(pm), _ptr(led)))
        out, off = [], 0
        for w in range(W):
            n = int(rows[w])
            out.append(ei[off:off + n * H].reshape(n, H))
            off += n * H
        ledger = {KIND_NAMES[i]: led[3 * i:3 * i + 3].astype(int).tolist()
                  for i in range(len(KIND_NAMES))}
        return out, rpe.reshape(W, el), rc.reshape(W, W), pm, ledger

    def ssmb_forward(self, tokens, G, k, cap, node_of=None):
        tokens = _f64(tokens)
        S, H = tokens.shape
        node_of = _i64a(list(range(G)) if node_of is None else node_of)
        out = np.zeros_like(tokens)
        led = np.zeros(3 * len(KIND_NAMES), np.uint64)
        _check(lib().ref_ssmb_forward(self.h, G, _ptr(node_of), _ptr(tokens), S, k, cap,
                                      _ptr(out), _ptr(led)))
        return out


def select_pilots(token_ids, expert_ids, cw, tpe, E, node_of, seed):
    token_ids, expert_ids, cw, tpe = _i64a(token_ids), _i64a(expert_ids), _f64(cw), _i64a(tpe)
    node_of = _i64a(node_of)
    B = token_ids.shape[0]
    pm = np.zeros(max(B, 1), np.uint8)
    _check(lib().ref_select_pilots(B, _ptr(token_ids), _ptr(expert_ids), _ptr(cw), _ptr(tpe), E,
                                   node_of.shape[0], _ptr(node_of), C.c_uint64(seed), _ptr(pm)))
    return pm[:B]


def sample_redundancy(seed, tokens, k, expert_node):
    en = _i64a(expert_node)
    return float(lib().ref_sample_redundancy(seed, tokens, k, en.shape[0], _ptr(en)))


def last_ledger_csv() -> str:
    """CostLedger::write_csv of the last reference forward (collectives.cpp:26-34)."""
    return lib().ref_last_ledger_csv().decode()
