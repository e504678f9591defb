"""ctypes binding of the xmoe C-ABI (include/xmoe/xmoe.h) for tests and the
bench driver.  Device memory and streams come from torch; every call goes
straight to libxmoe.so.  There is no fallback: if the library is missing or
the device is not an sm_100 part, construction raises."""
from __future__ import annotations

import ctypes as C
import os
import re

import torch

from . import build as _build

_LIB = None

F64 = 0
BF16 = 1
F32 = 2
NAIVE = 0
RBD = 1

ERROR_KINDS = {1: "ParseError", 2: "ValidationError", 3: "DimensionError", 4: "IndexError",
               5: "CountMismatch", 6: "PlanMismatch", 10: "CudaError", 11: "NcclError",
               12: "PeerTimeout", 99: "InternalError"}

# xmoe_layer_inspect items (xmoe.h)
INSPECT = {"top_experts": (0, torch.int32), "weights": (1, torch.float64), "token_ids": (2, torch.int32),
           "expert_ids": (3, torch.int32), "combine_weights": (4, torch.float64),
           "tokens_per_expert": (5, torch.int32), "tpe_all": (6, torch.int32), "expert_input": (7, None),
           "expert_output": (8, None), "recv_per_expert": (9, torch.int32), "tpe_chunks": (10, torch.int32),
           "dest_rank": (11, torch.int32), "dest_row": (12, torch.int32), "slot_pos": (13, torch.int32),
           "pilot_mask": (14, torch.uint8)}
_TDT = {F64: torch.float64, BF16: torch.bfloat16, F32: torch.float32}


class XmoeError(RuntimeError):
    """Status code + the reference's message text (error.hpp:10-38)."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = ERROR_KINDS.get(code, "Error")
        self.msg = msg
        super().__init__(f"{self.kind}: {msg}")


class LayerDesc(C.Structure):
    _fields_ = [("num_experts", C.c_int64), ("model_dim", C.c_int64), ("ffn_dim", C.c_int64),
                ("top_k", C.c_int64), ("max_token_count", C.c_int64), ("n_shared", C.c_int64),
                ("shared_ffn_dim", C.c_int64), ("max_tokens", C.c_int64), ("dtype", C.c_int32),
                ("renorm", C.c_int32), ("dispatch_mode", C.c_int32), ("flags", C.c_int32),
                ("seed", C.c_uint64)]


class Topology(C.Structure):
    """xmoe_topology (moesim::Topology, config.hpp:30-40)."""
    _fields_ = [("gpus_per_node", C.c_int64), ("bw_intra", C.c_double), ("bw_inter", C.c_double),
                ("latency_intra", C.c_double), ("latency_inter", C.c_double), ("dtype_bytes", C.c_int64)]

    @classmethod
    def reference_defaults(cls, gpus_per_node=8, dtype_bytes=0):
        return cls(gpus_per_node, 200e9, 25e9, 0.0, 0.0, dtype_bytes)


class LedgerEntry(C.Structure):
    _fields_ = [("id", C.c_int64), ("kind", C.c_char * 32), ("self_bytes", C.c_uint64),
                ("intra_bytes", C.c_uint64), ("inter_bytes", C.c_uint64), ("intra_msgs", C.c_uint64),
                ("inter_msgs", C.c_uint64), ("time_s", C.c_double)]


def header_symbols() -> list[str]:
    """Every function the C-ABI header declares."""
    hdr = os.path.join(_build.ROOT, "include", "xmoe", "xmoe.h")
    txt = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t)\s+(xmoe_\w+)\(", txt, re.M)))


def lib_path() -> str:
    return _build.LIB


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(_build.LIB):
            raise ImportError(f"{_build.LIB} is not built (run __graft_entry__.build())")
        L = C.CDLL(os.environ.get("XMOE_LIB") or _build.LIB)  # XMOE_LIB: A/B builds
        p, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        L.xmoe_last_error.restype = C.c_char_p
        L.xmoe_abi_version.restype = C.c_int
        L.xmoe_kernel_launches.restype = C.c_uint64
        L.xmoe_ctx_create.argtypes = [i32, i32, i32, p, C.POINTER(p)]
        L.xmoe_ctx_destroy.argtypes = [p]
        L.xmoe_nccl_unique_id.argtypes = [p]
        L.xmoe_gate_forward.argtypes = [p, i32, p, p, i64, i64, i64, i64, i32, p, p, p, p]
        L.xmoe_pft_construct.argtypes = [p, p, p, i64, i64, i64, i64, p, p, p, p, p, p, i32, p]
        L.xmoe_gather_rows.argtypes = [p, i32, p, i64, i64, p, i64, p, i32, p]
        L.xmoe_scatter_combine.argtypes = [p, i32, p, i64, i64, p, p, i64, p, i32, p]
        L.xmoe_grouped_mlp.argtypes = [p, i32, p, i64, p, i64, p, p, i64, i64, p, p]
        L.xmoe_grouped_gemm_bf16.argtypes = [p, p, i64, i64, p, i64, p, i64, p, i32, p]
        L.xmoe_layer_create.argtypes = [p, C.POINTER(LayerDesc), p, p, p, p, p, C.POINTER(p)]
        L.xmoe_layer_destroy.argtypes = [p]
        L.xmoe_moe_forward.argtypes = [p, p, p, i64, p, p]
        L.xmoe_ssmb_forward.argtypes = [p, p, p, i64, p, p]
        L.xmoe_layer_ledger.argtypes = [p, C.POINTER(C.c_uint64), i32]
        L.xmoe_layer_set_timing.argtypes = [p, i32]
        L.xmoe_layer_set_graph.argtypes = [p, i32]
        L.xmoe_layer_chunks.argtypes = [p, p]
        L.xmoe_layer_ledger_entries.argtypes = [p, p, p, i32, p]
        L.xmoe_layer_ledger_csv.argtypes = [p, p, p, i64, p]
        L.xmoe_layer_padded_ledger_csv.argtypes = [p, p, p, i64, p]
        L.xmoe_layer_bwd_stage_ms.argtypes = [p, p, i32]
        L.xmoe_layer_stage_ms.argtypes = [p, C.POINTER(C.c_float), i32]
        L.xmoe_plan_dispatch.argtypes = [i32, i32, p, i32, p, p, p]
        L.xmoe_moe_backward.argtypes = [p, p, p, p, i64, p, p]
        L.xmoe_grouped_wgrad_bf16.argtypes = [p, p, p, i64, p, i64, i64, i64, p, p]
        L.xmoe_wgrad_split_bf16.argtypes = [p, p, p, i64, i64, i64, i64, p, p]
        L.xmoe_layer_grads.argtypes = [p] + [C.POINTER(p)] * 5
        L.xmoe_layer_inspect.argtypes = [p, i32, i32, C.POINTER(p), C.POINTER(i64)]
        L.xmoe_layer_status.argtypes = [p]
        L.xmoe_ctx_status.argtypes = [p]
        L.xmoe_layer_set_weights.argtypes = [p, p, p, p, p, p, p]
        L.xmoe_rng_uniform.argtypes = [p, C.c_uint64, C.c_uint64, i64, C.c_double, C.c_double, C.c_double, i32, p, p]
        L.xmoe_salt_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.xmoe_salt_seed.restype = C.c_uint64
        L.xmoe_make_layer_weights.argtypes = [p, C.c_uint64, C.c_uint64, i64, i64, i64, i64, i64, C.c_double, i32,
                                              p, p, p, p]
        pp = C.POINTER(p)
        L.xmoe_pf_dispatch.argtypes = [p, i32, i64, i64, pp, pp, p, p, pp, p, pp, pp, pp, p]
        L.xmoe_pf_combine.argtypes = [p, i32, i64, i64, pp, p, pp, pp, pp, p, p, pp, p]
        L.xmoe_select_pilots.argtypes = [p, i64, p, p, i64, i64, i64, i64, i64, C.c_uint64, p, p, p]
        L.xmoe_rbd_dispatch.argtypes = [p, i32, i64, i64, i64, pp, pp, pp, p, p, i64, p, pp, pp, p, pp, pp, pp, p]
        L.xmoe_rbd_combine.argtypes = [p, i32, i64, pp, i64, p, p, p, p, p, p, p, p, pp, pp, p, p, pp, p]
        L.xmoe_route_pairs.argtypes = [p, i64, p, p, p, i64, i64, i64, i64, C.POINTER(i64), C.POINTER(i64), p]
        _LIB = L
    return _LIB


def _check(rc: int):
    if rc != 0:
        raise XmoeError(rc, lib().xmoe_last_error().decode())


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _parr(ts):
    """Host array of device pointers (None -> NULL)."""
    arr = (C.c_void_p * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def _i64arr(v):
    import numpy as np
    a = np.ascontiguousarray(v, dtype=np.int64)
    return a, a.ctypes.data_as(C.c_void_p)


def salt_seed(seed: int, a: int, b: int = 0) -> int:
    """moesim::salt_seed (rng.hpp:17-19)."""
    return int(lib().xmoe_salt_seed(seed, a, b))


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise XmoeError(2, f"unsupported dtype {t.dtype}")


def plan_dispatch(tpe_all, me):
    """Host exchange plan (xmoe_plan_dispatch): numpy in, numpy out, no GPU."""
    import numpy as np
    t = np.ascontiguousarray(tpe_all, dtype=np.int32)
    W, E = t.shape
    el = E // W if W and E % W == 0 else 1
    send = np.zeros(E + 1, np.int64)
    recv = np.zeros(W * el, np.int64)
    rpe = np.zeros(el, np.int64)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _check(lib().xmoe_plan_dispatch(W, E, ptr(t), me, ptr(send), ptr(recv), ptr(rpe)))
    return send, recv.reshape(W, el), rpe


def grouped_wgrad_test(ctx, X, Y, rows_per_group):
    """D_g = X_g^T Y_g (fp32) through xmoe_grouped_wgrad_bf16."""
    G = len(rows_per_group)
    rpg = torch.tensor(rows_per_group, dtype=torch.int32, device=X.device)
    D = torch.empty((G, X.shape[1], Y.shape[1]), dtype=torch.float32, device=X.device)
    _check(lib().xmoe_grouped_wgrad_bf16(ctx.h, _ptr(X), _ptr(Y), X.shape[0], _ptr(rpg), G, X.shape[1],
                                         Y.shape[1], _ptr(D), _stream()))
    return D


def wgrad_split_test(ctx, X, Y, splits):
    """D = X^T Y (fp32) over all rows, split-K, through xmoe_wgrad_split_bf16."""
    D = torch.empty((X.shape[1], Y.shape[1]), dtype=torch.float32, device=X.device)
    _check(lib().xmoe_wgrad_split_bf16(ctx.h, _ptr(X), _ptr(Y), X.shape[0], X.shape[1], Y.shape[1], splits,
                                       _ptr(D), _stream()))
    return D


def kernel_launches() -> int:
    return int(lib().xmoe_kernel_launches())


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().xmoe_nccl_unique_id(buf))
    return bytes(buf)


class Context:
    """xmoe_ctx: rank == -1 drives all `world` workers on this device."""

    def __init__(self, device: int = 0, world: int = 1, rank: int = -1, nccl_id: bytes | None = None):
        self.device = device
        self.world = world
        self.rank = rank
        h = C.c_void_p()
        idbuf = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
        _check(lib().xmoe_ctx_create(device, world, rank, idbuf, C.byref(h)))
        self.h = h

    def status(self):
        _check(lib().xmoe_ctx_status(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().xmoe_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ operators
    def gate_forward(self, x, wg, k, renorm=False, want_logits=False):
        S, H = x.shape
        E = wg.shape[0] if x.dtype == torch.bfloat16 else wg.shape[1]
        top = torch.empty((S, k), dtype=torch.int32, device=x.device)
        w = torch.empty((S, k), dtype=torch.float64, device=x.device)
        lg = torch.empty((S, E), dtype=torch.float64, device=x.device) if want_logits else None
        _check(lib().xmoe_gate_forward(self.h, _dtype_code(x), _ptr(x), _ptr(wg), S, H, E, k,
                                       int(renorm), _ptr(top), _ptr(w), _ptr(lg), _stream()))
        return (top, w, lg) if want_logits else (top, w)

    def pft_construct(self, top, w, E, cap, validate=True):
        S, k = top.shape
        n = max(S * k, 1)
        dev = top.device
        tid = torch.empty(n, dtype=torch.int32, device=dev)
        eid = torch.empty(n, dtype=torch.int32, device=dev)
        cw = torch.empty(n, dtype=torch.float64, device=dev)
        tpe = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
        slot = torch.empty((S, k), dtype=torch.int32, device=dev)
        B = torch.zeros(1, dtype=torch.int32, device=dev)
        _check(lib().xmoe_pft_construct(self.h, _ptr(top), _ptr(w), S, k, E, cap, _ptr(tid),
                                        _ptr(eid), _ptr(cw), _ptr(tpe), _ptr(slot), _ptr(B),
                                        int(validate), _stream()))
        b = int(B.item())
        return tid[:b], eid[:b], cw[:b], tpe[:E], slot

    def gather_rows(self, src, ids, validate=True):
        n = ids.shape[0]
        out = torch.empty((n, src.shape[1]), dtype=src.dtype, device=src.device)
        _check(lib().xmoe_gather_rows(self.h, _dtype_code(src), _ptr(src), src.shape[0],
                                      src.shape[1], _ptr(ids), n, _ptr(out), int(validate),
                                      _stream()))
        return out

    def scatter_combine(self, rows, token_ids, weights, S, validate=True):
        out = torch.empty((S, rows.shape[1]), dtype=rows.dtype, device=rows.device)
        _check(lib().xmoe_scatter_combine(self.h, _dtype_code(rows), _ptr(rows), rows.shape[0],
                                          rows.shape[1], _ptr(token_ids), _ptr(weights), S,
                                          _ptr(out), int(validate), _stream()))
        return out

    def grouped_mlp(self, inp, rows_per_expert, w1, w2, validate=True):
        """F64: w1 [G,H,F], w2 [G,F,H]; BF16: w1 [G,F,H], w2 [G,H,F] (K-major).
        The C-ABI checks the counts on the device without a host sync;
        validate=True waits for the stream and raises the reference's
        CountMismatch (xmoe_ctx_status) here."""
        rows, H = inp.shape
        G = rows_per_expert.shape[0]
        F = w1.shape[1] if inp.dtype == torch.bfloat16 else w1.shape[2]
        out = torch.empty_like(inp)
        _check(lib().xmoe_grouped_mlp(self.h, _dtype_code(inp), _ptr(inp), rows,
                                      _ptr(rows_per_expert), G, _ptr(w1), _ptr(w2), H, F,
                                      _ptr(out), _stream()))
        if validate:
            torch.cuda.current_stream().synchronize()
            self.status()
        return out

    # ------------------------------------------------------------ synthetic inputs
    def rng_uniform(self, seed, offset, n, lo, hi, grid=0.0, dtype=F64, out=None):
        """Outputs [offset, offset+n) of Rng(seed).uniform(lo, hi) on the device."""
        out = torch.empty(n, dtype=_TDT[dtype], device="cuda") if out is None else out
        _check(lib().xmoe_rng_uniform(self.h, seed, offset, n, lo, hi, grid, dtype, _ptr(out), _stream()))
        return out

    def make_layer_weights(self, seed, E, H, F, first_expert=0, n_experts=None, offset=0, gate_grid=0.0,
                           dtype=F64, gate=True):
        """moesim::make_layer_weights(Rng(seed)) on the device: gate [H,E] and
        experts [first, first+n) of w1 [.,H,F], w2 [.,F,H]."""
        n = E - first_expert if n_experts is None else n_experts
        t = _TDT[dtype]
        g = torch.empty((H, E), dtype=t, device="cuda") if gate else None
        w1 = torch.empty((n, H, F), dtype=t, device="cuda")
        w2 = torch.empty((n, F, H), dtype=t, device="cuda")
        _check(lib().xmoe_make_layer_weights(self.h, seed, offset, E, H, F, first_expert, n, gate_grid, dtype,
                                             _ptr(g), _ptr(w1), _ptr(w2), _stream()))
        return g, w1, w2

    # ------------------------------------------------------------ split EP operators (SPMD shape)
    def pf_dispatch(self, dtype, H, E, packed, expert_ids, tpe, want_arrival=True):
        """xmoe_pf_dispatch: per-worker packed rows / expert ids (device
        tensors), tpe [W,E] int32 device.  Returns (expert_input list,
        recv_per_expert [W,El], dest_rank list, dest_row list, arrival list)."""
        W = len(packed)
        El = E // W
        th = tpe.cpu().numpy().reshape(W, E)
        n_own = [int(th[:, j * El:(j + 1) * El].sum()) for j in range(W)]
        dt = packed[0].dtype
        ei = [torch.empty((max(n, 1), H), dtype=dt, device="cuda") for n in n_own]
        rpe = torch.empty((W, El), dtype=torch.int32, device="cuda")
        dr = [torch.empty(max(1, p.shape[0]), dtype=torch.int32, device="cuda") for p in packed]
        dw = [torch.empty(max(1, p.shape[0]), dtype=torch.int32, device="cuda") for p in packed]
        a2g = [torch.empty(max(n, 1), dtype=torch.int32, device="cuda") for n in n_own] if want_arrival else None
        B, Bp = _i64arr([p.shape[0] for p in packed])
        _check(lib().xmoe_pf_dispatch(self.h, dtype, H, E, _parr(packed), _parr(expert_ids), Bp, _ptr(tpe),
                                      _parr(ei), _ptr(rpe), _parr(dr), _parr(dw),
                                      _parr(a2g) if want_arrival else None, _stream()))
        return ([e[:n] for e, n in zip(ei, n_own)], rpe, dr, dw,
                [a[:n] for a, n in zip(a2g, n_own)] if want_arrival else None)

    def pf_combine(self, dtype, H, E, expert_out, tpe, token_ids, expert_ids, cw, seq_lens):
        W = len(expert_out)
        out = [torch.empty((max(S, 1), H), dtype=expert_out[0].dtype, device="cuda") for S in seq_lens]
        B, Bp = _i64arr([t.shape[0] for t in token_ids])
        Sl, Sp = _i64arr(seq_lens)
        eo = [e if e.numel() else torch.empty((1, H), dtype=expert_out[0].dtype, device="cuda") for e in expert_out]
        _check(lib().xmoe_pf_combine(self.h, dtype, H, E, _parr(eo), _ptr(tpe), _parr(token_ids),
                                     _parr(expert_ids), _parr(cw), Bp, Sp, _parr(out), _stream()))
        return [o[:S] for o, S in zip(out, seq_lens)]

    def select_pilots(self, token_ids, expert_ids, S, k, E, W, gpus_per_node, seed):
        B = token_ids.shape[0]
        mask = torch.zeros(max(B, 1), dtype=torch.uint8, device="cuda")
        pof = torch.empty(max(B, 1), dtype=torch.int32, device="cuda")
        _check(lib().xmoe_select_pilots(self.h, B, _ptr(token_ids), _ptr(expert_ids), S, k, E, W, gpus_per_node,
                                        seed, _ptr(mask), _ptr(pof), _stream()))
        return mask[:B], pof[:B]

    def rbd_dispatch(self, dtype, H, E, gpus_per_node, packed, token_ids, expert_ids, seq_lens, k, tpe, masks):
        W = len(packed)
        El = E // W
        th = tpe.cpu().numpy().reshape(W, E)
        n_own = [int(th[:, j * El:(j + 1) * El].sum()) for j in range(W)]
        dt = packed[0].dtype
        ei = [torch.empty((max(n, 1), H), dtype=dt, device="cuda") for n in n_own]
        rpe = torch.empty((W, El), dtype=torch.int32, device="cuda")
        mk = lambda: [torch.empty(max(1, p.shape[0]), dtype=torch.int32, device="cuda") for p in packed]  # noqa
        dr, dw, pof = mk(), mk(), mk()
        B, Bp = _i64arr([p.shape[0] for p in packed])
        Sl, Sp = _i64arr(seq_lens)
        _check(lib().xmoe_rbd_dispatch(self.h, dtype, H, E, gpus_per_node, _parr(packed), _parr(token_ids),
                                       _parr(expert_ids), Bp, Sp, k, _ptr(tpe), _parr(masks), _parr(ei), _ptr(rpe),
                                       _parr(dr), _parr(dw), _parr(pof), _stream()))
        return [e[:n] for e, n in zip(ei, n_own)], rpe, dr, dw, pof

    def rbd_combine(self, dtype, H, expert_out, flat, seq_lens):
        """flat: dict of device tensors land_of, land_pos, land_multi, land_w,
        ent_ptr, ent_owner, ent_pos, ent_w, flat_scale and per-source lists
        src_ptr, src_flat (see xmoe.h)."""
        P = int(flat["land_of"].shape[0])
        out = [torch.empty((max(S, 1), H), dtype=expert_out[0].dtype, device="cuda") for S in seq_lens]
        Sl, Sp = _i64arr(seq_lens)
        eo = [e if e.numel() else torch.empty((1, H), dtype=expert_out[0].dtype, device="cuda") for e in expert_out]
        f = flat
        _check(lib().xmoe_rbd_combine(self.h, dtype, H, _parr(eo), P, _ptr(f["land_of"]), _ptr(f["land_pos"]),
                                      _ptr(f["land_multi"]), _ptr(f["land_w"]), _ptr(f["ent_ptr"]),
                                      _ptr(f["ent_owner"]), _ptr(f["ent_pos"]), _ptr(f["ent_w"]),
                                      _parr(f["src_ptr"]), _parr(f["src_flat"]), _ptr(f["flat_scale"]), Sp,
                                      _parr(out), _stream()))
        return [o[:S] for o, S in zip(out, seq_lens)]

    def route_pairs(self, token, expert, expert_node, nodes, tokens, skip_node=-1):
        c, g = C.c_int64(), C.c_int64()
        _check(lib().xmoe_route_pairs(self.h, token.shape[0], _ptr(token), _ptr(expert), _ptr(expert_node),
                                      expert_node.shape[0], nodes, tokens, skip_node, C.byref(c), C.byref(g),
                                      _stream()))
        return int(c.value), int(g.value)

    def grouped_gemm_bf16(self, A, rows_per_group, B, N, relu=False, out=None):
        rows, K = A.shape
        G = rows_per_group.shape[0]
        D = out if out is not None else torch.empty((rows, N), dtype=torch.bfloat16, device=A.device)
        _check(lib().xmoe_grouped_gemm_bf16(self.h, _ptr(A), rows, K, _ptr(rows_per_group), G,
                                            _ptr(B), N, _ptr(D), int(relu), _stream()))
        return D


class Layer:
    """xmoe_layer: weights resident in HBM in the B200 layout + workspace.

    gate [H,E], w1 [E_held,H,F], w2 [E_held,F,H] (reference layouts, device
    tensors of the layer dtype); sw1 [ns,H,Fs], sw2 [ns,Fs,H] optional.
    chunks: token chunks of the pipelined BF16 forward (0 auto, 1 off; see
    XMOE_LAYER_CHUNKS in xmoe.h)."""

    def __init__(self, ctx: Context, *, num_experts, model_dim, ffn_dim, top_k, max_token_count,
                 max_tokens, dtype, gate, w1, w2, sw1=None, sw2=None, renorm=False,
                 dispatch_mode=NAIVE, seed=0, ssmb=False, train=False, chunks=0, gpus_per_node=1):
        self.ctx = ctx
        ns = 0 if sw1 is None else sw1.shape[0]
        fs = 0 if sw1 is None else sw1.shape[2]
        self.desc = LayerDesc(num_experts, model_dim, ffn_dim, top_k, max_token_count, ns, fs,
                              max_tokens, dtype, int(renorm), dispatch_mode,
                              int(bool(ssmb)) | (2 if train else 0) | (int(chunks) << 8) |
                              (int(gpus_per_node) << 12), seed)
        self.shape = dict(E=num_experts, H=model_dim, F=ffn_dim, ns=ns, Fs=fs,
                          E_held=w1.shape[0])
        self.dtype = dtype
        self.H = model_dim
        h = C.c_void_p()
        _check(lib().xmoe_layer_create(ctx.h, C.byref(self.desc), _ptr(gate), _ptr(w1), _ptr(w2),
                                       _ptr(sw1), _ptr(sw2), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().xmoe_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, x, out=None):
        """x: [n_local, S, H] (or [S, H] when n_local == 1)."""
        S = x.shape[-2]
        out = torch.empty_like(x) if out is None else out
        _check(lib().xmoe_moe_forward(self.ctx.h, self.h, _ptr(x), S, _ptr(out), _stream()))
        return out

    def backward(self, x, dy, dx=None):
        """Gradient of the last forward: returns dx; weight grads via grads()."""
        S = x.shape[-2]
        dx = torch.empty_like(x) if dx is None else dx
        _check(lib().xmoe_moe_backward(self.ctx.h, self.h, _ptr(x), _ptr(dy), S, _ptr(dx), _stream()))
        return dx

    def grads(self) -> dict:
        """fp32 weight gradients in the reference layouts (views of layer memory)."""
        ptrs = [C.c_void_p() for _ in range(5)]
        _check(lib().xmoe_layer_grads(self.h, *[C.byref(q) for q in ptrs]))
        sh = self.shape
        H, E, F, El = sh["H"], sh["E"], sh["F"], sh["E_held"]
        out = {}

        def view(ptr, shape):
            if not ptr.value:
                return None

            class _Dev:  # zero-copy view through __cuda_array_interface__
                __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4",
                                            "data": (ptr.value, False), "version": 3}
            return torch.as_tensor(_Dev(), device="cuda").clone()
        torch.cuda.synchronize()
        out["gate"] = view(ptrs[0], (H, E))
        out["w1"] = view(ptrs[1], (El, H, F))
        out["w2"] = view(ptrs[2], (El, F, H))
        if sh["ns"]:
            out["sw1"] = view(ptrs[3], (H, sh["ns"] * sh["Fs"]))
            out["sw2"] = view(ptrs[4], (sh["ns"] * sh["Fs"], H))
        return out

    def inspect(self, what: str, worker: int = 0, limit: int | None = None):
        """Copy of one internal array of the last forward (xmoe_layer_inspect),
        at most `limit` elements."""
        code, dt = INSPECT[what]
        if dt is None:
            dt = _TDT[self.dtype]
        p, n = C.c_void_p(), C.c_int64()
        _check(lib().xmoe_layer_inspect(self.h, worker, code, C.byref(p), C.byref(n)))
        if limit is not None:
            n = C.c_int64(min(n.value, limit))
        if n.value == 0 or not p.value:
            return torch.empty(0, dtype=dt, device="cuda")
        typestr = {torch.int32: "<i4", torch.float64: "<f8", torch.uint8: "|u1", torch.float32: "<f4",
                   torch.bfloat16: "<i2"}[dt]

        class _Dev:
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": typestr, "data": (p.value, False),
                                        "version": 3}
        t = torch.as_tensor(_Dev(), device="cuda").clone()
        return t.view(torch.bfloat16) if dt == torch.bfloat16 else t

    def status(self):
        _check(lib().xmoe_layer_status(self.h))

    def set_weights(self, gate, w1, w2, sw1=None, sw2=None):
        _check(lib().xmoe_layer_set_weights(self.h, _ptr(gate), _ptr(w1), _ptr(w2), _ptr(sw1), _ptr(sw2),
                                            _stream()))

    def ssmb_forward(self, x_full, out=None):
        S = x_full.shape[0]
        out = torch.empty_like(x_full) if out is None else out
        _check(lib().xmoe_ssmb_forward(self.ctx.h, self.h, _ptr(x_full), S, _ptr(out), _stream()))
        return out

    LEDGER_KEYS = ["dispatch_rows_self", "dispatch_rows_offrank", "dispatch_meta_offrank",
                   "combine_rows_self", "combine_rows_offrank", "routed_copies",
                   "unique_rows_offrank", "copies_offrank"]

    def ledger(self) -> dict:
        buf = (C.c_uint64 * 8)()
        _check(lib().xmoe_layer_ledger(self.h, buf, 8))
        return dict(zip(self.LEDGER_KEYS, [int(v) for v in buf]))

    def chunks(self) -> int:
        v = C.c_int32()
        _check(lib().xmoe_layer_chunks(self.h, C.byref(v)))
        return int(v.value)

    def ledger_entries(self, topo: "Topology | None" = None) -> list[dict]:
        """The last forward's collectives in the reference's CostLedger schema."""
        n = C.c_int32()
        tp = C.byref(topo) if topo is not None else None
        _check(lib().xmoe_layer_ledger_entries(self.h, tp, None, 0, C.byref(n)))
        buf = (LedgerEntry * max(1, n.value))()
        _check(lib().xmoe_layer_ledger_entries(self.h, tp, buf, n.value, C.byref(n)))
        return [{"id": e.id, "kind": e.kind.decode(), "self_bytes": e.self_bytes, "intra_bytes": e.intra_bytes,
                 "inter_bytes": e.inter_bytes, "intra_msgs": e.intra_msgs, "inter_msgs": e.inter_msgs,
                 "time_s": e.time_s} for e in buf[:n.value]]

    def ledger_csv(self, topo: "Topology | None" = None, padded: bool = False) -> str:
        """CostLedger::write_csv of the last forward (collectives.cpp:26-34);
        padded=True: the padded (GShard) comparator's ledger for this layer."""
        fn = lib().xmoe_layer_padded_ledger_csv if padded else lib().xmoe_layer_ledger_csv
        n = C.c_int64()
        tp = C.byref(topo) if topo is not None else None
        _check(fn(self.h, tp, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(fn(self.h, tp, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def set_graph(self, on: bool):
        _check(lib().xmoe_layer_set_graph(self.h, int(on)))

    def set_timing(self, on: bool):
        _check(lib().xmoe_layer_set_timing(self.h, int(on)))

    STAGES = ["gate", "pft", "dispatch", "experts", "shared", "combine", "total",
              "counts", "rows_moved", "dispatch_barrier", "return_wait", "combine_kernel",
              "shared_side_stream"]

    BWD_STAGES = ["scatter_dy", "owner_prep", "dgrad", "wgrad", "token_level", "gate_and_dx"]

    def bwd_stage_ms(self) -> dict:
        buf = (C.c_float * 6)()
        _check(lib().xmoe_layer_bwd_stage_ms(self.h, buf, 6))
        return dict(zip(self.BWD_STAGES, [float(v) for v in buf]))

    def timeline_ms(self) -> list:
        """Chunked forward (timing on): per chunk [scatter end, GEMM start,
        GEMM end, combine end] in ms from the forward's start."""
        n = self.chunks()
        if n <= 1:
            return []
        buf = (C.c_float * (13 + 4 * n))()
        _check(lib().xmoe_layer_stage_ms(self.h, buf, 13 + 4 * n))
        return [[round(float(buf[13 + 4 * c + j]), 4) for j in range(4)] for c in range(n)]

    def stage_ms(self) -> dict:
        buf = (C.c_float * 13)()
        _check(lib().xmoe_layer_stage_ms(self.h, buf, 13))
        return dict(zip(self.STAGES, [float(v) for v in buf]))
