#!/usr/bin/env python
"""Benchmark driver: one MoE-block forward per step through libxmoe.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl xmoe|reference]
                    [--config c1|c2|c3|c4|c5] [--mode auto|rbd|naive] [--tokens S]

Default workload (BASELINE.json configs[1], SURVEY §8 "C2"): DeepSeek-MoE
layer, 64 routed experts top-6 + 2 shared, d_model 2048, d_ff 1408, 16,384
tokens per GPU, bf16, expert parallel over N GPUs (E/N experts per GPU),
dropless.  --config selects the other BASELINE configs (C1 the 4096-token
CPU-runnable layer, C3 DeepSeek-V3, C4 the 32K-token sequence-sharded block,
C5 Zipf-skewed routing; paper_2508_13337_b200/configs.py).  Synthetic inputs
from the reference's own generator (moesim::Rng, drawn on the device),
grid-exact (tokens on 2^-7, gate on 2^-10, experts bf16), random-init weights.

N=1 runs in this process; N>1 is launched by torchrun (one rank per GPU,
NCCL over NVLink).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer fwd tokens/s"
NVLINK_GBPS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
UNIT = "tokens/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="xmoe", choices=["xmoe", "reference"])
    p.add_argument("--mode", default="auto", choices=["auto", "rbd", "naive"],
                   help="dispatch: auto = plain at N=1, redundancy bypass at N>1")
    p.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                   help="BASELINE config (SURVEY §8 C1-C5); c2 is the headline workload")
    p.add_argument("--tokens", type=int, default=0, help="tokens per GPU (0 = the config's)")
    p.add_argument("--transport", default=None, choices=["p2p", "nccl"],
                   help="N>1 row transport: NVLink peer kernels (default) or NCCL send/recv baseline")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-backward", action="store_true", help="skip the fwd+bwd measurement")
    p.add_argument("--no-graph", action="store_true", help="launch the forward kernels one by one")
    p.add_argument("--chunks", type=int, default=0,
                   help="token chunks of the pipelined forward (0 auto, 1 off)")
    p.add_argument("--cpu-sample-tokens", type=int, default=512,
                   help="tokens per host thread for the cpu_baseline sample")
    p.add_argument("--cpu-threads", type=int, default=0, help="host threads of the CPU reference (0 = all)")
    return p.parse_args()


def gemm_traffic(config="c2"):
    """dram read+write bytes per routed-GEMM launch from the committed ncu
    --set full capture of this config (profiles/gemm_traffic[_cN].json)."""
    name = "gemm_traffic.json" if config == "c2" else f"gemm_traffic_{config}.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)["traffic_bytes_per_launch"]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every 2 ms from a thread (a timed region of 20 steps
    is only ~30 ms, shorter than nvidia-smi's 100 ms sampling period), with
    `nvidia-smi -lms 100` as the fallback when NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpus=1):
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self.stop_ev = threading.Event()
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = [int(v) for v in vis.split(",")][:gpus] if vis and all(
                v.strip().isdigit() for v in vis.split(",")) else list(range(gpus))
            self.handles = [pynvml.nvmlDeviceGetHandleByIndex(i) for i in idx]
            self.bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.nvml = pynvml
        except Exception:
            self.nvml = None

    def start(self):
        if self.nvml is not None:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv = self.nvml
        while not self.stop_ev.is_set():
            for h in self.handles:
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(sm), float(mx), {n for n, b in self.bits.items() if r & b}))
                except Exception:
                    pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, gpus):
        if self.nvml is not None:
            self.stop_ev.set()
            self.t.join(timeout=1)
            samples = self.samples
            src = "nvml, 2 ms"
        elif self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            samples = []
            for ln in self.lines:
                f = [x.strip() for x in ln.split(",")]
                if len(f) < 9 or not f[0].isdigit() or int(f[0]) >= gpus:
                    continue
                try:
                    samples.append((float(f[1]), float(f[2]),
                                    {n for n, v in zip(self.NAMES, f[5:9]) if v.lower() == "active"}))
                except ValueError:
                    continue
            src = "nvidia-smi, 100 ms"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [x[0] for x in samples]
        reasons = set().union(*[x[2] for x in samples])
        busy = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_min_mhz": min(busy), "sm_max_mhz": max(x[1] for x in samples),
                "reasons": sorted(reasons), "samples": len(samples), "sampler": src}


# ---------------------------------------------------------------- CPU reference
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _ref_inputs(cfg, sample_tokens, refbind):
    """The config's inputs as the compiled reference draws them: the same
    Rng streams, grid snapping and bf16 rounding as the device (configs.py)."""
    import numpy as np
    import torch
    from paper_2508_13337_b200 import configs

    sd = configs.seeds(refbind.salt_seed)
    H = cfg["H"]
    x = refbind.rng_uniform(sd["tokens"], sample_tokens * H, -1.0, 1.0)
    x = (np.round(x * configs.TOKEN_GRID) / configs.TOKEN_GRID).reshape(sample_tokens, H)
    bf = lambda a: torch.from_numpy(a).to(torch.bfloat16).to(torch.float64).numpy()  # noqa: E731
    zipf_row = None
    if cfg.get("zipf"):
        u = refbind.rng_uniform(sd["zipf"], cfg["E"], 0.0, 1.0).tolist()
        zipf_row = bf(np.array(configs.zipf_bias(cfg, u)))
        x[:, 0] = 1.0
    return sd, x, bf, zipf_row


def cpu_reference(cfg, threads=None, sample_tokens=64, steps=1, warmup=0):
    """The unmodified reference (oracle/_ref/libmoesim_ref.so, compiled from
    /root/reference) on host cores, on the config's own inputs (the same
    generator streams as the GPU arm).  Layers up to 1e9 expert parameters
    (C1, C2, C5): every thread runs the reference's pf_moe_forward (W=1) over
    a token sample, plus the shared experts through the reference's
    grouped_expert_mlp.  Larger layers (C3: 60 GB of fp64 weights; C4) are
    EXTRAPOLATED: per-token time = the reference's gate_forward per token +
    top_k x its grouped_expert_mlp per row (one expert's weights) + the
    shared experts' per token, each timed on the sample.  Returns (tokens/s,
    cores, per-step seconds list, sample description)."""
    import numpy as np
    from oracle import refbind

    if not refbind.available():
        refbind.build()
    E, k, H, F = cfg["E"], cfg["k"], cfg["H"], cfg["F"]
    ns, Fs = cfg["ns"], cfg["Fs"]
    threads = threads or host_threads()
    sd, x, bf, zipf_row = _ref_inputs(cfg, sample_tokens * threads, refbind)
    samples = [x[i * sample_tokens:(i + 1) * sample_tokens] for i in range(threads)]
    full = E * 2 * H * F <= 1_000_000_000
    grid = lambda a: np.round(a * 1024) / 1024  # noqa: E731
    if full:
        gate, w1, w2 = refbind.make_layer_weights(sd["weights"], E, H, F)
        gate = grid(gate)
        if zipf_row is not None:
            gate[0] = zipf_row
        gate = bf(gate)
        layer = refbind.Layer(gate, bf(w1), bf(w2))
        del w1, w2
    else:
        gate, _, _ = refbind.make_layer_weights(sd["weights"], E, H, 1)  # gate draws come first
        gate = bf(grid(gate))
        # expert 0 only: w1[0] = draws [H*E, H*E + H*F), w2[0] = the next H*F
        d = refbind.rng_uniform(sd["weights"], H * E + 2 * H * F, -0.1, 0.1)[H * E:]
        one = refbind.Layer(np.zeros((H, 1)), bf(d[:H * F].reshape(1, H, F)), bf(d[H * F:].reshape(1, F, H)))
    shared = None
    if ns:
        _, sw1, sw2 = refbind.make_layer_weights(sd["shared"], ns, H, Fs)
        shared = refbind.Layer(np.zeros((H, ns)), bf(sw1), bf(sw2))
    cap = sample_tokens * k
    errs = []
    parts = {}

    def work(i):
        try:
            xs = samples[i]
            if full:
                out = layer.pf_moe_forward_noncopy(xs[None], k, cap)
                if shared is not None:
                    for q in range(ns):  # reference grouped_expert_mlp per shared expert
                        out[0] += shared.grouped_expert_mlp(xs, np.array([0] * q + [sample_tokens] +
                                                                         [0] * (ns - q - 1)), 0)
                return
            t0 = time.perf_counter()
            refbind.gate_forward(xs, gate, k)
            t1 = time.perf_counter()
            one.grouped_expert_mlp(xs, np.array([sample_tokens]), 0)
            t2 = time.perf_counter()
            if shared is not None:
                for q in range(ns):
                    shared.grouped_expert_mlp(xs, np.array([0] * q + [sample_tokens] + [0] * (ns - q - 1)), 0)
            t3 = time.perf_counter()
            parts[i] = ((t1 - t0) + k * (t2 - t1) + (t3 - t2)) / sample_tokens  # s per token
        except Exception as e:  # pragma: no cover
            errs.append(e)

    times = []
    for it in range(warmup + steps):
        ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        if errs:
            raise errs[0]
        if it >= warmup:
            # extrapolated: the step is the per-token time of the slowest thread x its tokens
            times.append(dt if full else max(parts.values()) * sample_tokens)
    tok = threads * sample_tokens
    v = tok / statistics.mean(times)
    how = ("reference pf_moe_forward composition (W=1) over the full layer" if full else
           "EXTRAPOLATED from the reference's gate_forward per token + top_k x grouped_expert_mlp per row "
           "(one expert's weights) timed on the sample")
    desc = (f"{threads} host threads x {sample_tokens} tokens per step of {cfg['desc'].split(':')[0]} "
            f"({how}{', + reference grouped_expert_mlp for the shared experts' if ns else ''}), "
            f"fp64, inputs from the same Rng streams as the GPU arm, backend "
            f"{refbind.lib().ref_kernel_backend().decode()}, CPU {cpu_model()}")
    return v, threads, times, desc


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def bind_to_gpu_numa(device):
    """Pin this rank's host threads to the CPUs local to its GPU (PCIe root
    complex), so the pinned staging buffers of the e2e loop live on that NUMA
    node.  Best effort: returns the CPU list used, or None."""
    import torch
    try:
        pr = torch.cuda.get_device_properties(device)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return spec
    except Exception:
        return None
    return None


def run_reference(args, rank, world, result_out):
    if rank != 0:
        return
    from paper_2508_13337_b200 import configs
    cfg = configs.CONFIGS[args.config]
    # bounded per-step sample (>= 256 tokens per thread where the layer allows
    # it) so that K+W steps stay within a few minutes
    n = max(1, args.steps + args.warmup)
    per_step = 256 if n <= 60 else max(64, min(256, 15000 // n))
    threads = args.cpu_threads or host_threads()
    v, cores, times, desc = cpu_reference(cfg, threads=threads, sample_tokens=per_step,
                                          steps=args.steps, warmup=args.warmup)
    S = args.tokens or configs.tokens_per_gpu(cfg, world)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
            "scaling": "strong" if cfg.get("ssmb") else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["desc"] + "; CPU sample per step", "tokens_per_gpu": S,
                       "parallelism": f"ep{world}"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc,
                             "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=result_out, flush=True)


# ---------------------------------------------------------------- xmoe arm
def main():
    # Everything but the one JSON line (NCCL banners, library prints) goes to
    # stderr: fd 1 is re-pointed at fd 2 and the result is written to a dup
    # of the original stdout.
    result_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.stdout = sys.stderr
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.transport:
        os.environ["XMOE_TRANSPORT"] = args.transport
    if args.impl == "reference":
        return run_reference(args, rank, world, result_out)

    import torch
    import torch.distributed as dist
    from paper_2508_13337_b200 import capi

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        obj = [capi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = capi.Context(local_rank, world, rank, obj[0])
    else:
        ctx = capi.Context(local_rank, 1, 0)

    from paper_2508_13337_b200 import configs
    cfg = configs.CONFIGS[args.config]
    E, k, H, F, ns, Fs = cfg["E"], cfg["k"], cfg["H"], cfg["F"], cfg["ns"], cfg["Fs"]
    ssmb = bool(cfg.get("ssmb"))
    S = args.tokens or configs.tokens_per_gpu(cfg, world)   # this rank's tokens
    S_seq = S * world if not ssmb else (args.tokens * world if args.tokens else cfg["S_total"])
    if ssmb:  # every rank holds the whole sequence; rank g's shard is rows [g*S/G, ...)
        gate, w1, w2, sw1, sw2, x_full = configs.device_inputs(ctx, capi, cfg, rank, world, S_seq, 0, torch)
        base = S_seq // world
        S = S_seq - (world - 1) * base if rank == world - 1 else base
        x = x_full[rank * base:rank * base + S]
    else:
        gate, w1, w2, sw1, sw2, x = configs.device_inputs(ctx, capi, cfg, rank, world, S, rank * S, torch)
    rbd_seed = configs.seeds(capi.salt_seed)["rbd"]
    auto_mode = args.mode == "auto" and world > 1
    if args.mode == "auto":
        args.mode = "naive"  # N=1: no exchange; N>1: probed below
    mode = capi.RBD if args.mode == "rbd" else capi.NAIVE
    S_max = S_seq - (world - 1) * (S_seq // world) if ssmb else S

    def make_layer(chunks=None, train=False, md=None):
        chunks = args.chunks if chunks is None else chunks
        return capi.Layer(ctx, num_experts=E, model_dim=H, ffn_dim=F, top_k=k, max_token_count=S_max * k,
                          max_tokens=S_max, dtype=capi.BF16, gate=gate, w1=w1, w2=w2, sw1=sw1, sw2=sw2,
                          dispatch_mode=mode if md is None else md, seed=rbd_seed, chunks=chunks, train=train)

    out = torch.empty_like(x_full if ssmb else x)
    xin = x_full if ssmb else x
    auto_probe = None
    if auto_mode:
        # Dispatch auto-selection, measured on this box before the timed region
        # (the same warm-up budget for both): the chunked plain dispatch hides
        # its larger all-to-all under the expert GEMMs; the redundancy bypass
        # moves 25-67 % fewer bytes.  Which wins depends on the link speed of
        # the box (B200 measurements in DESIGN.md §8 go either way at N=4), so
        # the faster one, max over ranks, is kept.
        auto_probe = {}
        for name, md, ch in (("naive", capi.NAIVE, args.chunks), ("rbd", capi.RBD, args.chunks or 2)):
            pl = make_layer(chunks=ch, md=md)
            if not args.no_graph:
                pl.set_graph(True)
            for _ in range(3):
                (pl.ssmb_forward(xin, out) if ssmb else pl.forward(xin, out))
            torch.cuda.synchronize()
            dist.barrier()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record()
            for _ in range(10):
                (pl.ssmb_forward(xin, out) if ssmb else pl.forward(xin, out))
            p1.record()
            torch.cuda.synchronize()
            t = torch.tensor([p0.elapsed_time(p1) / 10], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            auto_probe[name] = {"ms": float(t.item()), "chunks": pl.chunks()}
            dist.barrier()
            del pl
        args.mode = min(auto_probe, key=lambda n: auto_probe[n]["ms"])
        mode = capi.RBD if args.mode == "rbd" else capi.NAIVE
        if args.mode == "rbd" and not args.chunks:
            args.chunks = auto_probe["rbd"]["chunks"]
    layer = make_layer()
    if not args.no_graph:
        layer.set_graph(True)

    def step(lyr, xi, oi):  # one pass of the hot path (SSMB: shard forward + all-gather)
        if ssmb:
            lyr.ssmb_forward(xi, oi)
        else:
            lyr.forward(xi, oi)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up
    for _ in range(args.warmup):
        step(layer, xin, out)
    torch.cuda.synchronize()

    # ---- device-timed region (inputs resident in HBM)
    clocks = ClockSampler(world)
    if rank == 0:
        clocks.start()
    launches0 = capi.kernel_launches()
    barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(layer, xin, out)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = capi.kernel_launches() - launches0
    # the last timed forward's collectives in the reference's CostLedger schema
    # (one node of 8 GPUs: every off-rank byte is intra-node NVLink), and the
    # padded (GShard) comparator's for the same layer
    topo = capi.Topology.reference_defaults(gpus_per_node=8)
    ref_ledger = {e["kind"]: {"intra_bytes": e["intra_bytes"], "inter_bytes": e["inter_bytes"],
                              "self_bytes": e["self_bytes"]} for e in layer.ledger_entries(topo)}
    padded_csv = layer.ledger_csv(topo, padded=True).strip().split("\n")[1:]
    padded_ledger = {ln.split(",")[1]: int(ln.split(",")[2]) + int(ln.split(",")[3]) for ln in padded_csv}
    ms = max_over_ranks(t0.elapsed_time(t1) / args.steps)
    clk = clocks.stop(world) if rank == 0 else None

    # ---- per-stage breakdown + roofline of the dominant kernel (grouped GEMM),
    # measured right after the timed forward (before the heavier fwd+bwd
    # section changes the board's power/clock state),
    # on a forward-only unchunked layer (kernel-level stages; the training
    # layer's GEMM1 epilogue also stores ReLU masks)
    oshard = torch.empty_like(x)
    slayer = make_layer(chunks=1)
    slayer.set_timing(True)
    stage_runs = []
    for _ in range(6):
        slayer.forward(x, oshard)
        torch.cuda.synchronize()
        stage_runs.append(slayer.stage_ms())
    stages = {kk: statistics.median(r[kk] for r in stage_runs[1:]) for kk in stage_runs[0]}
    led = slayer.ledger()
    del slayer
    # ---- training layer (unchunked) for fwd+bwd
    # ---- forward + backward (gradients w.r.t. x and every weight), same clock rules
    # (training layer, unchunked; the sequence-sharded C4 block has no backward API)
    fwd_bwd = None
    if not args.no_backward and not ssmb:
        tlayer = make_layer(chunks=1, train=True)
        if not args.no_graph:
            tlayer.set_graph(True)
        dy = ctx.rng_uniform(capi.salt_seed(0, 9500, rank), 0, S * H, -1.0, 1.0, dtype=capi.BF16).view(S, H)
        dxb = torch.empty_like(x)
        for _ in range(max(2, args.warmup)):
            tlayer.forward(x, oshard)
            tlayer.backward(x, dy, dxb)
        torch.cuda.synchronize()
        barrier()
        b0 = torch.cuda.Event(enable_timing=True)
        b1 = torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.steps):
            tlayer.forward(x, oshard)
            tlayer.backward(x, dy, dxb)
        b1.record(stream)
        torch.cuda.synchronize()
        barrier()
        fb_ms = max_over_ranks(b0.elapsed_time(b1) / args.steps)
        tlayer.set_timing(True)  # per-stage backward breakdown (eager launches)
        bst = []
        for _ in range(4):
            tlayer.forward(x, oshard)
            tlayer.backward(x, dy, dxb)
            torch.cuda.synchronize()
            bst.append(tlayer.bwd_stage_ms())
        tlayer.set_timing(False)
        bwd_stages = {kk: statistics.median(r[kk] for r in bst[1:]) for kk in bst[0]}
        fwd_bwd = {"metric": "MoE-layer fwd+bwd tokens/s", "value": world * S / (fb_ms * 1e-3), "unit": UNIT,
                   "ms_per_step": fb_ms, "bwd_stages_ms": bwd_stages,
                   "note": "forward + backward (dx and fp32 grads of gate, experts, shared experts); "
                           "gradients restated beyond the forward-only reference, checked against fp64 autograd"}
        del tlayer

    # ---- plain vs redundancy-bypassing dispatch (N > 1): all-to-all bytes and
    # isolated kernel times of both, from unchunked layers in timing mode
    dispatch_compare = None
    if world > 1:
        dispatch_compare = {}
        for name, md in (("naive", capi.NAIVE), ("rbd", capi.RBD)):
            pl = make_layer(chunks=1, md=md)
            pl.set_timing(True)
            runs = []
            for _ in range(6):
                pl.forward(x, oshard)
                torch.cuda.synchronize()
                runs.append(pl.stage_ms())
            st_m = {kk: statistics.median(r[kk] for r in runs[1:]) for kk in runs[0]}
            lg = pl.ledger()
            del pl
            off_d = lg["dispatch_rows_offrank"] + lg["dispatch_meta_offrank"]  # bytes (ledger.cpp)
            off_c = lg["combine_rows_offrank"]
            dispatch_compare[name] = {
                "offrank_bytes_dispatch": off_d, "offrank_bytes_combine": off_c,
                "dispatch_kernel_ms": max_over_ranks(st_m["rows_moved"]),
                "dispatch_stage_ms": max_over_ranks(st_m["dispatch"]),
                "combine_kernel_ms": max_over_ranks(st_m["combine_kernel"]),
                "combine_stage_ms": max_over_ranks(st_m["combine"]),
                "nvlink_GBps_dispatch": off_d / (st_m["rows_moved"] * 1e-3) / 1e9 if st_m["rows_moved"] else None,
            }
        barrier()
    copies = led["routed_copies"]
    recv_rows_here = None  # routed rows computed on this GPU
    # rows this GPU's experts process = total copies landing here; at N=1 = copies
    gemm_flops = 4.0 * H * F * copies  # routed expert FFN (2 GEMMs, 2 FLOP/MAC)
    shared_flops = 4.0 * H * ns * Fs * S
    if world > 1:
        # rows landing on this rank's experts: all-reduce of per-rank received counts
        t = torch.tensor([float(copies)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        gemm_flops = 4.0 * H * F * float(t.item()) / world  # average per GPU
    hbm, tf_burst, tf_sus, peak_kind = peaks()
    achieved = gemm_flops / (stages["experts"] * 1e-3) / 1e12
    perm_bytes = (S + copies) * H * 2 + 4 * copies
    comb_bytes = copies * H * 2 + 2 * S * H * 2 + 8 * copies
    expert_frac_of_step = stages["experts"] / stages["total"] if stages["total"] else None

    # ---- end to end through the public API with host buffers.  Every step
    # copies ITS input from pinned host memory and its output back to pinned
    # host memory; the copies of neighbouring steps overlap the compute on
    # separate streams (double-buffered), as a serving loop would run them.
    e2e_steps = max(50, args.steps)  # steady state: one pipeline fill + drain amortised over the run
    numa_cpus = bind_to_gpu_numa(local_rank)
    # SSMB (C4): every rank holds the whole sequence buffer but reads only its
    # shard, so only the shard crosses PCIe
    x_lo = (rank * (S_seq // world)) if ssmb else 0
    xh = [x.cpu().pin_memory() for _ in range(2)]
    # SSMB: every rank holds the all-gathered output; each reads back its own
    # shard, so the job retrieves the sequence's output once
    oh = [torch.empty_like(xin[x_lo:x_lo + S].cpu()).pin_memory() for _ in range(2)]
    xd = [xin.clone() for _ in range(2)]
    od = [torch.empty_like(xin) for _ in range(2)]
    h2d_bytes = x.numel() * 2
    d2h_bytes = oh[0].numel() * 2
    s_in = torch.cuda.Stream()
    s_out = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_outfree = [torch.cuda.Event() for _ in range(2)]

    def e2e_run(n, t0=None, t1=None, compute=True):
        if t0 is not None:
            t0.record(s_in)
        with torch.cuda.stream(s_in):
            xd[0][x_lo:x_lo + S].copy_(xh[0], non_blocking=True)
            ev_in[0].record(s_in)
        for i in range(n):
            b, nb = i % 2, (i + 1) % 2
            if i + 1 < n:
                with torch.cuda.stream(s_in):
                    if i >= 1:
                        s_in.wait_event(ev_done[nb])  # step i-1 finished reading xd[nb]
                    xd[nb][x_lo:x_lo + S].copy_(xh[nb], non_blocking=True)
                    ev_in[nb].record(s_in)
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_outfree[b])  # step i-2's output left the device
            if compute:
                step(layer, xd[b], od[b])
            ev_done[b].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[b])
                oh[b].copy_(od[b][x_lo:x_lo + S], non_blocking=True)
                ev_outfree[b].record(s_out)
        if t1 is not None:
            t1.record(s_out)
        torch.cuda.synchronize()

    e2e_run(3)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_run(e2e_steps, e0, e1)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
    # the same loop with the forward left out: the host-link bound of e2e on
    # this box (PCIe and host memory, shared by the ranks of the node)
    e2e_run(3, compute=False)
    barrier()
    e2e_run(e2e_steps, e0, e1, compute=False)
    barrier()
    copy_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)

    # ---- CPU baseline (reference on host cores, rank 0 at N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, _, desc = cpu_reference(cfg, threads=args.cpu_threads or host_threads(),
                                              sample_tokens=args.cpu_sample_tokens)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc,
                   "cpu_model": cpu_model()}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    # whole-step roofline per GPU (B200_PROFILING.md: the slower of the tensor
    # work at the measured bf16 peak and the bytes that must cross NVLink at
    # the measured 770 GB/s per direction): routed + shared expert FFNs + gate
    shared_flops = 4.0 * S * H * ns * Fs
    gate_flops = 2.0 * S * H * E
    step_flops = gemm_flops + shared_flops + gate_flops
    nvl_bytes = (led.get("dispatch_rows_offrank", 0) + led.get("combine_rows_offrank", 0)) if world > 1 else 0
    t_tensor = step_flops / (tf_burst * 1e12) * 1e3
    t_nvl = nvl_bytes / (NVLINK_GBPS * 1e9) * 1e3
    step_roofline = {"tensor_ms": t_tensor, "nvlink_ms": t_nvl, "bound_ms": max(t_tensor, t_nvl),
                     "bound": "tensor" if t_tensor >= t_nvl else "nvlink", "frac": max(t_tensor, t_nvl) / ms,
                     "flops_per_gpu": step_flops, "nvlink_bytes_per_gpu_per_direction": nvl_bytes,
                     "note": "per GPU: (routed + shared expert FFN + gate) FLOPs at the measured burst bf16 peak vs "
                             "this rank's off-rank dispatch + combine row bytes (ledger) at 770 GB/s per direction; "
                             "frac = bound / ms_per_step"}
    if rank == 0:
        tokens_step = S_seq  # whole job: all ranks' tokens (C4: the one sharded sequence)
        value = tokens_step / (ms * 1e-3)
        wbytes = (E // world) * 2 * H * F * 2
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if ssmb else "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference Rng streams drawn on the device; random-init weights)",
            "config": {"workload": cfg["desc"], "config": args.config,
                       "tokens_per_gpu": S, "global_tokens": tokens_step,
                       "parallelism": (f"ssmb{world}+ep{world}" if ssmb else f"ep{world}"),
                       "dispatch": args.mode, "dispatch_probe": auto_probe, "pass": "forward",
                       "chunks": layer.chunks(),
                       "transport": (os.environ.get("XMOE_TRANSPORT") or "p2p") if world > 1 else "local",
                       "row_movement": (("owner-side pull" if os.environ.get("XMOE_DISPATCH", "pull") == "pull"
                                         else "source-side push") +
                                        f", {os.environ.get('XMOE_COMM_SMS', '28')} whole SMs beside GEMMs on the rest"
                                        if world > 1 and layer.chunks() > 1 and args.mode == "naive" else None),
                       "l2": f"working set > L2: {wbytes / 1e9:.2f} GB of expert weights per GPU + "
                             f"{S * H * 2 / 1e6:.0f} MB tokens stream each step (126 MB L2)"},
            "e2e": {"value": tokens_step / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                    "steps": e2e_steps,
                    "host_cpus": numa_cpus,
                    "copies_only": {"value": tokens_step / (copy_ms * 1e-3), "unit": UNIT,
                                    "ms_per_step": copy_ms},
                    "note": "pinned host x -> device, forward, device -> pinned host out, every step; copies of "
                            "neighbouring steps overlap the forward on two copy streams (double-buffered); "
                            "bytes per rank (each rank moves its own shard; SSMB: its shard of the gathered "
                            "output); copies_only = the same loop without the forward (the host-link bound)"},
            "roofline": {"bound": "tensor", "kernel": "grouped_gemm_tc (routed experts, GEMM1+GEMM2)",
                         "achieved": achieved, "peak": tf_burst, "unit": "TFLOP/s",
                         "frac": achieved / tf_burst,
                         "peak_note": f"{peak_kind} burst bf16 (the routed GEMM pair is timed as one ~0.8 ms stage "
                                      f"of the forward, shorter than the sustained run; at N>1 it exceeds the "
                                      f"sustained figure); sustained {tf_sus}",
                         "frac_sustained": achieved / tf_sus,
                         "traffic": gemm_traffic(args.config),
                         "traffic_note": "dram read+write bytes per routed-GEMM launch from the committed "
                                         "ncu --set full capture (profiles/gemm_traffic*.json), null when absent",
                         "algorithmic_flops_per_launch_pair": gemm_flops,
                         "share_of_step": expert_frac_of_step},
            "stages_ms": stages,
            "hbm_kernels": {"permute_bytes": perm_bytes, "combine_bytes": comb_bytes,
                            "dispatch_ms": stages["dispatch"], "combine_ms": stages["combine"],
                            "permute_GBps": perm_bytes / (stages["rows_moved"] * 1e-3) / 1e9 if stages["rows_moved"] else None,
                            "combine_GBps": comb_bytes / (stages["combine_kernel"] * 1e-3) / 1e9 if stages["combine_kernel"] else None,
                            "hbm_peak_GBps": hbm,
                            "permute_frac": perm_bytes / (stages["rows_moved"] * 1e-3) / 1e9 / hbm
                            if world == 1 and stages.get("rows_moved") else None,
                            "combine_frac": comb_bytes / (stages["combine_kernel"] * 1e-3) / 1e9 / hbm
                            if world == 1 and stages.get("combine_kernel") else None},
            "ledger": led,
            "step_roofline": step_roofline,
            "a2a": None if world == 1 else {
                "bound": "nvlink", "unit": "GB/s", "peak": NVLINK_GBPS,
                "bytes_offrank_per_gpu": dispatch_compare[args.mode]["offrank_bytes_dispatch"],
                "achieved": dispatch_compare[args.mode]["nvlink_GBps_dispatch"],
                "frac": (dispatch_compare[args.mode]["nvlink_GBps_dispatch"] or 0) / NVLINK_GBPS,
                "note": "dispatch kernel, isolated (timing mode), off-rank row bytes this GPU sends over NVLink "
                        "/ kernel time; peak = measured 770 GB/s peer copy per direction (B200_PROFILING.md)"},
            "dispatch_compare": dispatch_compare,
            "ref_schema_ledger": {"entries": ref_ledger, "padded_offrank_bytes": padded_ledger,
                                  "note": "xmoe_layer_ledger_entries / xmoe_layer_padded_ledger_csv of the "
                                          "last timed forward, moesim CostLedger kinds (global, all ranks)"},
            "fwd_bwd": fwd_bwd,
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), file=result_out, flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
