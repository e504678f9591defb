"""Per-SM NVLink pull rate of whole-SM copy blocks: register-staged loads
(1024 threads x 8 int4) vs cp.async rings staged in shared memory (8 or 13
16-byte slots per thread), 8 / 16 / 24 blocks, alone and beside the grouped
GEMM pair capped to the other SMs (XMOE_GEMM_SMS).
Run: gpurun --gpus 2 -- python profiles/interference/pull_depth.py"""
import json, os, sys
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
NB = 256 << 20
dst_local = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
peer = torch.empty(NB, dtype=torch.uint8, device="cuda:1").random_()
s_c = torch.cuda.Stream(0)
def timed(f, reps=3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_c):
        a.record(); [f() for _ in range(reps)]; b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
res = {}
for g in (8, 16, 24):
    r = {}
    r["regs_1024x8"] = NB / timed(lambda: ext.run_fat(peer.data_ptr(), dst_local.data_ptr(), NB, g, 32768)) / 1e6
    r["cpasync_ring8"] = NB / timed(lambda: ext.run_lds_pull(peer.data_ptr(), dst_local, NB, g, 8)) / 1e6
    r["cpasync_ring13"] = NB / timed(lambda: ext.run_lds_pull(peer.data_ptr(), dst_local, NB, g, 13)) / 1e6
    ok = torch.equal(dst_local[:1 << 20].cpu(), peer[:1 << 20].cpu())
    res[g] = {k: round(v) for k, v in r.items()}
    res[g]["correct"] = ok
    print(g, res[g], flush=True)
print(json.dumps(res))
