"""bench.py -- TACO compression path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl taco|reference]

N = 1 (default): one step = fused TACO compress (K1) + decompress (K2) of one
  [8192 x 2560] bf16 tensor (BASELINE configs[1] per-rank tensor), inputs resident in
  HBM.  metric = algorithmic HBM GB/s of the round trip (6.0625 B/elem at B=256).
N > 1 (torchrun, one rank per GPU): one step = the FP8 two-shot compressed all-reduce
  of each rank's [8192 x 2560] bf16 tensor over NCCL (K1 -> all-to-all -> K3 ->
  all-gather -> K2).  metric = aggregate all-reduce algbw = N * 2 bytes * elems / t,
  next to ncclAllReduce bf16 on the same tensors.
--impl reference: the reference's own CPU implementation (oracle/_ref = the unmodified
  /root/reference sources compiled by oracle/Makefile) on the host cores, same metric,
  bounded samples.  Rank 0 only under torchrun.
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

ROWS, COLS = 8192, 2560  # BASELINE configs[1]: GPT-3 2.7B row-parallel output, bf16
B = 256


def algorithmic_bytes_per_elem(b: int = B, in_bytes: int = 2, out_bytes: int = 2) -> dict:
    c = 1.0 + 8.0 / b  # FP8 code + (alpha, s) per block
    return {"k1": in_bytes + c, "k2": c + out_bytes, "roundtrip": in_bytes + 2 * c + out_bytes}


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(kind: str):
    """dram read + write bytes per launch of the K1 ('compress') / K2 ('decompress') kernel
    from the newest committed ncu capture (profiles/*_ncu_traffic.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_traffic.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as f:
            d = json.load(f)
        for k in d["kernels"]:
            if ("k_" + kind) in k["kernel"]:
                return {"bytes": int(k["dram_read_bytes"] + k["dram_write_bytes"]), "kernel": k["kernel"],
                        "source": os.path.relpath(files[-1], ROOT),
                        "note": "ncu replays one launch: writes still L2-resident at kernel end are not counted"}
    except Exception:
        return None
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.stop_ev = index, [], threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop_ev.wait(0.1)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.th.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > i + 2 and r[i + 2] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------- taco arm ---
def run_taco_single(args) -> dict:
    import ctypes as C

    import numpy as np
    import torch

    from paper_2604_24088_b200 import _abi, codec

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n = ROWS * COLS
    cfg = codec.make_config(args.block_size)
    m = -(-n // args.block_size)
    lay = _abi.msg_layout(cfg, m)
    # Rotate R buffer sets (inputs + messages + outputs) so each step's working set was
    # evicted from the 126 MB L2 long before it is touched again.
    R = 4
    g = torch.Generator(device=dev).manual_seed(7)
    xs = [torch.randn(n, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16) for _ in range(R)]
    # a heavy tail like the canonical near-zero mixture (SPEC: TP activations)
    for x in xs:
        x.mul_(1e-3).index_fill_(0, torch.randint(0, n, (n // 100,), device=dev, generator=g), 1.0)
    msgs = [torch.empty((1, lay.msg_stride), dtype=torch.uint8, device=dev) for _ in range(R)]
    ys = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(R)]
    flags = codec.Flags(dev)
    stream = torch.cuda.Stream(device=dev)
    lib = _abi.lib()
    sp = C.c_void_p(stream.cuda_stream)

    def k1(i):
        _abi.check(lib.taco_compress_dev(C.byref(cfg), C.c_void_p(xs[i].data_ptr()), _abi.DT_BF16, n, 1, 0, m,
                                         C.c_void_p(msgs[i].data_ptr()), lay.msg_stride, flags.ptr(), sp))

    def k2(i):
        _abi.check(lib.taco_decompress_dev(C.byref(cfg), C.c_void_p(msgs[i].data_ptr()), lay.msg_stride, 1, n, 0,
                                           m, C.c_void_p(ys[i].data_ptr()), _abi.DT_BF16, flags.ptr(), sp))

    with torch.cuda.stream(stream):
        for i in range(max(3, args.warmup)):
            k1(i % R)
            k2(i % R)
        stream.synchronize()
        flags.check()
        # timed region: K steps of K1 + K2, one event pair on the launching stream; then
        # K launches of K1 alone and of K2 alone, each between one event pair (per-launch
        # event stamps are quantised to ~2 us on this part, so kernels are timed as runs)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e1a, e1b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2a, e2b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with ClockSampler(0) as clk:
            t_wall = time.perf_counter()
            start.record(stream)
            for s_ in range(args.steps):
                k1(s_ % R)
                k2(s_ % R)
            end.record(stream)
            stream.synchronize()
            t_wall = time.perf_counter() - t_wall
            e1a.record(stream)
            for s_ in range(args.steps):
                k1(s_ % R)
            e1b.record(stream)
            e2a.record(stream)
            for s_ in range(args.steps):
                k2(s_ % R)
            e2b.record(stream)
            stream.synchronize()
            # keep the same load running until the sampler has >= 5 samples
            t0 = time.perf_counter()
            while len(clk.rows) < 5 and time.perf_counter() - t0 < 5:
                for s_ in range(200):
                    k1(s_ % R)
                    k2(s_ % R)
                stream.synchronize()
        flags.check()
    total_ms = start.elapsed_time(end)
    k1_ms = e1a.elapsed_time(e1b) / args.steps
    k2_ms = e2a.elapsed_time(e2b) / args.steps
    bpe = algorithmic_bytes_per_elem(args.block_size)
    step_ms = total_ms / args.steps
    value = bpe["roundtrip"] * n / (step_ms * 1e-3) / 1e9
    pk = peaks()
    k1_gbs = bpe["k1"] * n / (k1_ms * 1e-3) / 1e9
    k2_gbs = bpe["k2"] * n / (k2_ms * 1e-3) / 1e9
    dominant = ("k1", k1_ms, k1_gbs, bpe["k1"]) if k1_ms >= k2_ms else ("k2", k2_ms, k2_gbs, bpe["k2"])
    traffic = ncu_traffic("compress" if dominant[0] == "k1" else "decompress")

    # ---- configs[0] beside it: the reference's CPU-runnable case, [1024 x 768] fp32 round trip
    # on one rank (L2-resident, 7.9 MB: reported in microseconds)
    n0 = 1024 * 768
    m0 = -(-n0 // args.block_size)
    lay0 = _abi.msg_layout(cfg, m0)
    x0 = torch.randn(n0, generator=g, device=dev)
    msg0 = torch.empty((1, lay0.msg_stride), dtype=torch.uint8, device=dev)
    y0 = torch.empty(n0, device=dev)

    def rt0():
        _abi.check(lib.taco_compress_dev(C.byref(cfg), C.c_void_p(x0.data_ptr()), _abi.DT_F32, n0, 1, 0, m0,
                                         C.c_void_p(msg0.data_ptr()), lay0.msg_stride, flags.ptr(), sp))
        _abi.check(lib.taco_decompress_dev(C.byref(cfg), C.c_void_p(msg0.data_ptr()), lay0.msg_stride, 1, n0, 0, m0,
                                           C.c_void_p(y0.data_ptr()), _abi.DT_F32, flags.ptr(), sp))

    with torch.cuda.stream(stream):
        for _ in range(5):
            rt0()
        c0a, c0b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0a.record(stream)
        for _ in range(args.steps):
            rt0()
        c0b.record(stream)
        stream.synchronize()
    flags.check()
    cfg0_us = c0a.elapsed_time(c0b) / args.steps * 1e3

    # ---- e2e through the C-ABI host call (pinned host buffers, H2D + D2H inside the timed region)
    hc = codec.HostContext(0)
    xh = xs[0].cpu().pin_memory()
    yh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    e2e_steps = max(3, min(args.steps, 40))
    for _ in range(3):
        hc.roundtrip(xh, cfg, yh)
    # the host call is synchronous: time every step, report the median (host-side hiccups --
    # page-cache, NUMA placement of the pinned buffers -- move the mean, listed beside it)
    per_step = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        hc.roundtrip(xh, cfg, yh)
        per_step.append(time.perf_counter() - t0)
    e2e_s = statistics.median(per_step)
    e2e_mean = statistics.fmean(per_step)
    torch.cuda.synchronize()
    # the host call equals the device path bit for bit
    same = torch.equal(yh, ys[0].cpu())
    hc.close()

    line = {
        "metric": "taco_compress_decompress_hbm_GBps",
        "value": round(value, 1),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(step_ms, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (N(0,1e-3) with a 1% unit tail: the near-zero mixture shape), generated on device",
        "config": {"workload": "configs[1] per-rank tensor: TACO compress+decompress round trip",
                   "shape": [ROWS, COLS], "elements": n, "block_size": args.block_size, "format": "E4M3",
                   "in_dtype": "bf16", "out_dtype": "bf16",
                   "algorithmic_bytes_per_elem": bpe["roundtrip"],
                   "l2": f"rotating {R} buffer sets of {round(n * (4 + 2 * (1 + 8 / args.block_size)) / 1e6)} MB "
                         "(> 126 MB L2 in total)",
                   "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "kernel": dominant[0], "achieved": round(dominant[2], 1),
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(dominant[2] / pk["hbm_gbs"], 4),
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_source": traffic, "peak_source": pk["source"],
                     "algorithmic_bytes_per_launch": int(dominant[3] * n)},
        "kernels": {"k1_compress": {"ms": round(k1_ms, 5), "GBps": round(k1_gbs, 1),
                                    "frac": round(k1_gbs / pk["hbm_gbs"], 4)},
                    "k2_decompress": {"ms": round(k2_ms, 5), "GBps": round(k2_gbs, 1),
                                      "frac": round(k2_gbs / pk["hbm_gbs"], 4)}},
        "e2e": {"value": round(bpe["roundtrip"] * n / e2e_s / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(e2e_s * 1e3, 3), "ms_per_step_mean": round(e2e_mean * 1e3, 3),
                "steps": e2e_steps, "statistic": "median of per-step host wall times",
                "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": 2 * n,
                "api": "taco_roundtrip_host (C ABI, pinned host buffers)", "matches_device_path": bool(same)},
        "gpu_launches": 2 * args.steps,  # K1 + K2 per step inside the timed region
        "wall_s_timed_region": round(t_wall, 4),
        "configs0": {"workload": "[1024 x 768] fp32 compress + decompress round trip, 1 rank (L2-resident)",
                     "us_per_roundtrip": round(cfg0_us, 2), "launches_per_roundtrip": 2},
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, budget_s=args.cpu_seconds)
    return line


# ---------------------------------------------------------------- reference (CPU) arm ---
def _ref_inputs(n_elems: int, seed: int = 7):
    import numpy as np
    import torch

    from oracle.oracle import Ref
    ref = Ref()
    x = ref.generate(1, n_elems, seed)
    x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()  # the bf16 tensor's exact values
    return ref, np.ascontiguousarray(x)


def cpu_baseline(args, budget_s: float = 8.0, sample_elems: int = 1 << 21) -> dict:
    """oracle/_ref (the reference, compiled unmodified) round trip on the host cores."""
    import numpy as np
    ref, x = _ref_inputs(sample_elems)
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    y = np.empty_like(x)
    ref.roundtrip(x, y, args.block_size)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        ref.roundtrip(x, y, args.block_size)
        reps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = (time.perf_counter() - t0) / reps
    bpe = algorithmic_bytes_per_elem(args.block_size)["roundtrip"]
    # the same sample on one thread (TACO_THREADS=1), a quarter of the budget
    ref.set_threads(1)
    reps1, t1 = 0, time.perf_counter()
    while True:
        ref.roundtrip(x, y, args.block_size)
        reps1 += 1
        if time.perf_counter() - t1 >= budget_s / 4:
            break
    dt1 = (time.perf_counter() - t1) / reps1
    ref.set_threads(cores)
    return {"value": round(bpe * sample_elems / dt / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"taco::compress+decompress of {sample_elems} elements (bf16-valued mixture) x {reps} reps, "
                      f"TACO_THREADS={cores}; same per-element byte accounting as the GPU line",
            "ms_per_sample": round(dt * 1e3, 3),
            "value_1_thread": round(bpe * sample_elems / dt1 / 1e9, 4)}


def run_reference(args, world: int) -> dict:
    import numpy as np
    cores = os.cpu_count() or 1
    bpe = algorithmic_bytes_per_elem(args.block_size)["roundtrip"]
    if world == 1:
        sample = 1 << 21
        ref, x = _ref_inputs(sample)
        ref.set_threads(cores)
        y = np.empty_like(x)
        for _ in range(max(1, args.warmup)):
            ref.roundtrip(x, y, args.block_size)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ref.roundtrip(x, y, args.block_size)
        dt = (time.perf_counter() - t0) / args.steps
        value = bpe * sample / dt / 1e9
        metric = "taco_compress_decompress_hbm_GBps"
        desc = f"taco::compress+decompress of {sample} of the {ROWS * COLS} elements per step"
        cfgd = {"workload": "configs[1] per-rank tensor: TACO compress+decompress round trip (bounded sample)",
                "shape": [ROWS, COLS], "block_size": args.block_size, "sample_elements": sample}
    else:
        per_rank = 1 << 19
        ref, _ = _ref_inputs(1)
        ins = np.stack([_ref_inputs(per_rank, 100 + r)[1] for r in range(world)])
        ref.set_threads(cores)
        for _ in range(max(1, args.warmup)):
            ref.allreduce(ins, args.block_size)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ref.allreduce(ins, args.block_size)
        dt = (time.perf_counter() - t0) / args.steps
        value = world * 2 * per_rank / dt / 1e9
        metric = "taco_twoshot_allreduce_algbw_GBps"
        desc = (f"taco::allreduce(TwoShot) simulating {world} ranks in one process, {per_rank} elements per rank "
                f"(bounded sample of the {ROWS * COLS}-element tensors)")
        cfgd = {"workload": f"configs[1] tensor, TP={world} two-shot all-reduce (bounded sample)",
                "shape": [ROWS, COLS], "block_size": args.block_size, "sample_elements_per_rank": per_rank}
    return {"impl": "reference", "metric": metric, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (double internally)",
            "data": "synthetic (taco::generate near-zero mixture, bf16-rounded)", "config": cfgd,
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": desc},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["taco", "reference"], default="taco")
    ap.add_argument("--block-size", type=int, default=B)
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--chunks", type=int, default=2, help="N>1: pipelined chunks per shard")
    ap.add_argument("--eager", action="store_true", help="N>1: no CUDA-graph capture of the step")
    ap.add_argument("--collective", action="store_true", help="run the all-reduce leg even at world size 1")
    ap.add_argument("--shape", type=str, default=None,
                    help="ROWSxCOLS of the per-rank tensor (default configs[1] 8192x2560; e.g. configs[2] "
                         "16384x3584, configs[3] 16384x5120)")
    args = ap.parse_args()
    if args.shape:
        global ROWS, COLS
        ROWS, COLS = (int(v) for v in args.shape.lower().split("x"))
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, max(world, args.gpus))), flush=True)
        return
    if world > 1 or args.collective:
        from paper_2604_24088_b200.bench_collective import run_collective
        line = run_collective(args, ROWS, COLS, ClockSampler, peaks)
        if rank == 0:
            print(json.dumps(line), flush=True)
        return
    print(json.dumps(run_taco_single(args)), flush=True)


if __name__ == "__main__":
    main()
