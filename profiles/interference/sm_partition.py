"""SM partition: the grouped GEMM pair capped to XMOE_GEMM_SMS SMs beside
whole-SM copy blocks (1024 threads + 32 KB shared each) on the rest.
Run: XMOE_GEMM_SMS=132 gpurun --gpus 2 -- python profiles/interference/sm_partition.py"""
import json, sys, os
import torch
from torch.utils.cpp_extension import load
from cuda.bindings import runtime as cudart
here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(here)))
os.makedirs("/tmp/xmoe_interf_ext", exist_ok=True)
ext = load("xmoe_interf_ext", [os.path.join(here, "copy_kernels.cu")], extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False, build_directory="/tmp/xmoe_interf_ext")
torch.cuda.set_device(0)
cudart.cudaDeviceEnablePeerAccess(1, 0)
torch.cuda.set_device(1); cudart.cudaDeviceEnablePeerAccess(0, 0); torch.cuda.set_device(0)
from paper_2508_13337_b200 import capi
ctx = capi.Context(0, 1, 0)
H, F, G, rp = 2048, 1408, 16, 1536
A = (torch.randn(G * rp, H, device="cuda:0") * 0.1).to(torch.bfloat16)
B = (torch.randn(G, F, H, device="cuda:0") * 0.1).to(torch.bfloat16)
B2 = (torch.randn(G, H, F, device="cuda:0") * 0.1).to(torch.bfloat16)
rpg = torch.full((G,), rp, dtype=torch.int32, device="cuda:0")
mid = torch.empty(G * rp, F, dtype=torch.bfloat16, device="cuda:0")
out = torch.empty(G * rp, H, dtype=torch.bfloat16, device="cuda:0")
def g():
    ctx.grouped_gemm_bf16(A, rpg, B, F, relu=True, out=mid)
    ctx.grouped_gemm_bf16(mid, rpg, B2, H, out=out)
NB = 256 << 20
src = torch.empty(NB, dtype=torch.uint8, device="cuda:0").random_()
dst_local = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
peer = torch.empty(NB, dtype=torch.uint8, device="cuda:1")
s_g, s_c = torch.cuda.Stream(0), torch.cuda.Stream(0)
def timed(fg, fc):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s_g); e[2].record(s_c)
    if fc: fc()     # copies first: resident before the GEMM grid
    if fg:
        with torch.cuda.stream(s_g): fg()
    e[1].record(s_g); e[3].record(s_c)
    torch.cuda.synchronize()
    return (e[0].elapsed_time(e[1]) if fg else None), (e[2].elapsed_time(e[3]) if fc else None)
NG = 20
rep = lambda: [g() for _ in range(NG)]
res = {"gemm_sms": os.environ.get("XMOE_GEMM_SMS", "148")}
timed(rep, None)
g0, _ = timed(rep, None); res["alone_ms"] = round(g0 / NG, 4)
for name, grid, smem, kind in (("fat16_pull", 16, 32768, "pull"), ("fat8_pull", 8, 32768, "pull"), ("fat24_pull", 24, 32768, "pull"),
                               ("fat16_push", 16, 32768, "push"), ("fat16_pull_nosmem", 16, 0, "pull")):
    def f(k):
        with torch.cuda.stream(s_c):
            for _ in range(k):
                if kind == "pull": ext.run_fat(peer.data_ptr(), dst_local.data_ptr(), NB, grid, smem)
                else: ext.run_fat(src.data_ptr(), peer.data_ptr(), NB, grid, smem)
    _, c0 = timed(None, lambda: f(2))
    k = max(1, int(g0 / (c0 / 2)))
    g1, c1 = timed(rep, lambda: f(k))
    res[name] = {"alone_GBps": round(2 * NB / c0 / 1e6), "gemm_ms": round(g1 / NG, 4), "slow": round(g1 / g0, 3), "copy_GBps": round(k * NB / c1 / 1e6)}
print(json.dumps(res), flush=True)
