"""The xmoe grouped GEMM pair (ReLU GEMM1 + GEMM2, 16 experts, H 2048, F 1408)
beside copy streams: SM push / pull / local copies at several grids, copy
engine push / pull.  Run: gpurun --gpus 2 -- python profiles/interference/grouped_gemm_beside_copies.py"""
import json, sys, os
import torch
from torch.utils.cpp_extension import load
from cuda.bindings import runtime as cudart
here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(here)))
from paper_2508_13337_b200 import capi
os.makedirs("/tmp/xmoe_interf_ext", exist_ok=True)
ext = load("xmoe_interf_ext", [os.path.join(here, "copy_kernels.cu")], extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False, build_directory="/tmp/xmoe_interf_ext")
torch.cuda.set_device(0)
cudart.cudaDeviceEnablePeerAccess(1, 0)
torch.cuda.set_device(1); cudart.cudaDeviceEnablePeerAccess(0, 0); torch.cuda.set_device(0)
ctx = capi.Context(0, 1, 0)
H, F = 2048, 1408
def mk_gemm(G, rows_per):
    A = (torch.randn(G * rows_per, H, device="cuda:0") * 0.1).to(torch.bfloat16)
    B = (torch.randn(G, F, H, device="cuda:0") * 0.1).to(torch.bfloat16)
    B2 = (torch.randn(G, H, F, device="cuda:0") * 0.1).to(torch.bfloat16)
    rpg = torch.full((G,), rows_per, dtype=torch.int32, device="cuda:0")
    mid = torch.empty(G * rows_per, F, dtype=torch.bfloat16, device="cuda:0")
    out = torch.empty(G * rows_per, H, dtype=torch.bfloat16, device="cuda:0")
    def run():
        ctx.grouped_gemm_bf16(A, rpg, B, F, relu=True, out=mid)
        ctx.grouped_gemm_bf16(mid, rpg, B2, H, out=out)
    return run
NB = 256 << 20
src = torch.empty(NB, dtype=torch.uint8, device="cuda:0").random_()
dst_local = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
peer = torch.empty(NB, dtype=torch.uint8, device="cuda:1")
s_g, s_c = torch.cuda.Stream(0), torch.cuda.Stream(0)
def timed(fg, fc):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s_g); e[2].record(s_c)
    if fg:
        with torch.cuda.stream(s_g): fg()
    if fc: fc()
    e[1].record(s_g); e[3].record(s_c)
    torch.cuda.synchronize()
    return (e[0].elapsed_time(e[1]) if fg else None), (e[2].elapsed_time(e[3]) if fc else None)
def mkc(kind, grid):
    def f(k):
        with torch.cuda.stream(s_c):
            for _ in range(k):
                if kind == "sm_push": ext.run_sm(src, peer.data_ptr(), NB, grid)
                elif kind == "sm_pull": ext.run_sm_pull(peer.data_ptr(), dst_local, NB, grid)
                elif kind == "sm_local": ext.run_sm(src, dst_local.data_ptr(), NB, grid)
                elif kind == "ce_push": peer.copy_(src, non_blocking=True)
                elif kind == "ce_pull": dst_local.copy_(peer, non_blocking=True)
    return f
res = {}
for gname, (G, rp) in {"full16x1536": (16, 1536), "chunk16x384": (16, 384), "chunk16x768": (16, 768)}.items():
    g = mk_gemm(G, rp)
    NG = 20 if rp > 500 else 60
    rep = lambda: [g() for _ in range(NG)]
    timed(rep, None)
    g0, _ = timed(rep, None)
    res[gname] = {"alone_ms": round(g0 / NG, 4), "tflops": round(4 * G * rp * H * F / (g0 / NG * 1e-3) / 1e12)}
    for kind, grid in (("sm_push", 64), ("sm_push", 148), ("sm_pull", 64), ("sm_pull", 148), ("sm_pull", 296), ("sm_local", 148), ("ce_push", 0), ("ce_pull", 0)):
        f = mkc(kind, grid)
        _, c0 = timed(None, lambda: f(2))
        k = max(1, int(g0 / (c0 / 2)))
        g1, c1 = timed(rep, lambda: f(k))
        res[gname][f"{kind}_{grid}"] = {"gemm_ms": round(g1 / NG, 4), "slow": round(g1 / g0, 3), "copy_GBps": round(k * NB / c1 / 1e6)}
    print(gname, json.dumps(res[gname]), flush=True)
