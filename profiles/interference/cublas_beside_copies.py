"""cuBLAS bf16 GEMM (8192^3) on GPU 0 beside a 256 MB copy stream: copy-engine
peer copy, SM-driven peer push / pull, TMA bulk push / pull, at several grid
sizes.  Run: gpurun --gpus 2 -- python profiles/interference/cublas_beside_copies.py"""
import json, sys, os
import torch
from torch.utils.cpp_extension import load
from cuda.bindings import runtime as cudart
here = os.path.dirname(os.path.abspath(__file__))
os.makedirs("/tmp/xmoe_interf_ext", exist_ok=True)
ext = load("xmoe_interf_ext", [os.path.join(here, "copy_kernels.cu")], extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False, build_directory="/tmp/xmoe_interf_ext")
torch.cuda.set_device(0)
cudart.cudaDeviceEnablePeerAccess(1, 0)
torch.cuda.set_device(1); cudart.cudaDeviceEnablePeerAccess(0, 0); torch.cuda.set_device(0)
a = torch.randn(8192, 8192, device="cuda:0", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda:0", dtype=torch.bfloat16)
c = torch.empty(8192, 8192, device="cuda:0", dtype=torch.bfloat16)
NB = 256 << 20
src = torch.empty(NB, dtype=torch.uint8, device="cuda:0").random_()
dst_local = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
peer = torch.empty(NB, dtype=torch.uint8, device="cuda:1")
s_g, s_c = torch.cuda.Stream(0), torch.cuda.Stream(0)
def gemm(n):
    with torch.cuda.stream(s_g):
        for _ in range(n): torch.mm(a, b, out=c)
def timed(fg, fc):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s_g); e[2].record(s_c)
    if fg: fg()
    if fc: fc()
    e[1].record(s_g); e[3].record(s_c)
    torch.cuda.synchronize()
    return (e[0].elapsed_time(e[1]) if fg else None), (e[2].elapsed_time(e[3]) if fc else None)
def mk(kind, grid):
    def f(k):
        with torch.cuda.stream(s_c):
            for _ in range(k):
                if kind == "sm_push": ext.run_sm(src, peer.data_ptr(), NB, grid)
                elif kind == "tma_push": ext.run_tma(src, peer.data_ptr(), NB, grid)
                elif kind == "sm_pull": ext.run_sm_pull(peer.data_ptr(), dst_local, NB, grid)
                elif kind == "tma_pull": ext.run_tma_pull(peer.data_ptr(), dst_local, NB, grid)
                elif kind == "ce_push": peer.copy_(src, non_blocking=True)
    return f
timed(lambda: gemm(5), mk("sm_push", 64)(1))
NG = 40
g0, _ = timed(lambda: gemm(NG), None)
res = {"gemm_alone_ms": round(g0 / NG, 4)}
for kind, grids in (("ce_push", [0]), ("sm_push", [8, 16, 32, 64, 148, 592]), ("tma_push", [8, 16, 32, 64, 148]),
                    ("sm_pull", [16, 32, 64, 148, 592]), ("tma_pull", [8, 16, 32, 64, 148])):
    for g in grids:
        f = mk(kind, g)
        _, c0 = timed(None, lambda: f(3))
        alone = 3 * NB / c0 / 1e6
        k = max(1, int(g0 / (c0 / 3)))
        g1, c1 = timed(lambda: gemm(NG), lambda: f(k))
        res[f"{kind}_{g}"] = {"alone_GBps": round(alone), "beside_GBps": round(k * NB / c1 / 1e6), "gemm_ms": round(g1 / NG, 4)}
        print(kind, g, res[f"{kind}_{g}"], flush=True)
print(json.dumps(res))
