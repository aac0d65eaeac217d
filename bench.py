"""bench.py -- TACO compression path on B200 (see DESIGN.md §4 Measurement).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl taco|reference] [--config I]

N = 1 (default): one step = fused TACO compress (K1) + decompress (K2) of the largest
  per-rank tensor of BASELINE.json that one GPU holds: configs[3] [16384 x 5120] bf16
  (GPT-13B TP=8 activations), B = 256, inputs resident in HBM (taco::generate near-zero
  mixture).  metric = algorithmic HBM GB/s of the round trip (6.0625 B/elem at B = 256).
  configs[1] / configs[2] per-rank tensors and the configs[0] fp32 case ride along as
  extra keys.  The K steps are one CUDA graph (no host launch gaps in the timed region).
N > 1 (torchrun, one rank per GPU): the compressed collectives of the config that N
  names (bench_collective.py): N = 2 configs[1] all-reduce, N = 4 configs[2] SP
  reduce-scatter + all-gather, N = 8 configs[3] forward + backward all-reduce.
--impl reference: the reference's own CPU implementation (oracle/_ref = the unmodified
  /root/reference sources compiled by oracle/Makefile) on the host cores, same metric and
  config (the full tensor).  Rank 0 only under torchrun.
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

B = 256
# BASELINE.json configs: index -> (rows, cols, dtype, what)
CONFIGS = {
    0: (1024, 768, "f32", "GPT-2-small activation, CPU reference round trip"),
    1: (8192, 2560, "bf16", "GPT-3 2.7B row-parallel output, TP=2"),
    2: (16384, 3584, "bf16", "Qwen-7B SP activations, TP=4"),
    3: (16384, 5120, "bf16", "GPT-13B TP=8 activations / activation-gradients"),
}
HEADLINE = 3
MIXTURE, SEED = 1, 7  # taco::generate near-zero mixture, acceptance.cpp:274 seed


def algorithmic_bytes_per_elem(b: int = B, in_bytes: int = 2, out_bytes: int = 2) -> dict:
    c = 1.0 + 8.0 / b  # FP8 code + (alpha, s) per block
    return {"k1": in_bytes + c, "k2": c + out_bytes, "roundtrip": in_bytes + 2 * c + out_bytes}


def workload(idx: int, rows: int, cols: int) -> str:
    where = f"configs[{idx}] per-rank tensor" if idx is not None else "custom shape"
    return f"{where} [{rows} x {cols}]: TACO compress+decompress round trip, 1 rank"


def config_dict(idx, rows, cols, block_size, l2_note) -> dict:
    """Identical in both arms (the driver compares them)."""
    dt = CONFIGS[idx][2] if idx is not None else "bf16"
    return {"workload": workload(idx, rows, cols), "shape": [rows, cols], "elements": rows * cols,
            "block_size": block_size, "format": "E4M3", "in_dtype": dt, "out_dtype": dt,
            "algorithmic_bytes_per_elem": algorithmic_bytes_per_elem(block_size, 4 if dt == "f32" else 2,
                                                                     4 if dt == "f32" else 2)["roundtrip"],
            "inputs": f"taco::generate near-zero mixture (dense 1e-3, tail 1 at 1%), seed {SEED}"
                      + (", rounded to bf16" if dt == "bf16" else ""),
            "l2": l2_note, "parallelism": "single GPU"}


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(kind: str):
    """dram read + write bytes per launch of the K1 ('compress') / K2 ('decompress') kernel
    from the newest committed ncu capture (profiles/*_ncu_traffic.json), or None.  The
    capture's L2 write bytes ride along: dram writes miss the stores still dirty in L2 when a
    single replayed launch ends, L2 writes count every store."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_traffic.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as f:
            d = json.load(f)
        for k in d["kernels"]:
            if k.get("role", k["kernel"]) == kind:
                return {"bytes": int(k["dram_read_bytes"] + k["dram_write_bytes"]), "kernel": k["kernel"],
                        "dram_read_bytes": int(k["dram_read_bytes"]), "dram_write_bytes": int(k["dram_write_bytes"]),
                        "l2_write_bytes": int(k["l2_write_bytes"]) if k.get("l2_write_bytes") else None,
                        "source": os.path.relpath(files[-1], ROOT), "note": d.get("note", "")}
    except Exception:
        return None
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs.  Started
    before the timed region (its first sample is awaited), so the fork of nvidia-smi never
    lands inside it."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.stop_ev = index, [], threading.Event()
        self.marks = []  # (t, label): sample rows taken while a region was open count as "under load"
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
        t0 = time.perf_counter()
        while not self.rows and time.perf_counter() - t0 < 5:
            time.sleep(0.05)
        time.sleep(0.5)
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
def _graph(fn, stream):
    """CUDA graph of fn() enqueued on `stream` (the codec kernels keep their programmatic
    dependent-launch edges inside the graph)."""
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


class RoundTripBench:
    """K1 -> K2 of one per-rank tensor through the C ABI's device entry points, R buffer
    sets rotated.  Step s compresses set s % R and decompresses the message of set
    (s - 2) % R, written two steps earlier and evicted from L2 by the >= 500 MB of traffic
    in between: K2 reads a cold message, as it does after a collective's exchange."""

    R = 3

    def __init__(self, rows, cols, dtype_name, block_size, dev, stream, seed=SEED):
        import ctypes as C

        import torch

        from paper_2604_24088_b200 import _abi, codec
        self.C, self.torch, self._abi = C, torch, _abi
        self.n = n = rows * cols
        self.dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
        self.dcode = _abi.DT_BF16 if dtype_name == "bf16" else _abi.DT_F32
        self.cfg = codec.make_config(block_size)
        self.m = -(-n // block_size)
        self.lay = _abi.msg_layout(self.cfg, self.m)
        host = codec.generate(MIXTURE, n, seed)
        x0 = host.to(dev).to(self.dt)
        # the other sets: the same values at other addresses (rotated by whole blocks)
        self.xs = [x0] + [torch.roll(x0, (k * n) // self.R // block_size * block_size) for k in range(1, self.R)]
        self.msgs = [torch.empty(self.lay.msg_stride, dtype=torch.uint8, device=dev) for _ in range(self.R)]
        self.ys = [torch.empty(n, dtype=self.dt, device=dev) for _ in range(self.R)]
        self.flags = codec.Flags(dev)
        self.stream = stream
        self.lib = _abi.lib()
        self.host_x = host

    def k1(self, i):
        C = self.C
        self._abi.check(self.lib.taco_compress_dev(
            C.byref(self.cfg), C.c_void_p(self.xs[i].data_ptr()), self.dcode, self.n, 1, 0, self.m,
            C.c_void_p(self.msgs[i].data_ptr()), self.lay.msg_stride, self.flags.ptr(),
            C.c_void_p(self.torch.cuda.current_stream().cuda_stream)))

    def k2(self, i, j):
        C = self.C
        self._abi.check(self.lib.taco_decompress_dev(
            C.byref(self.cfg), C.c_void_p(self.msgs[i].data_ptr()), self.lay.msg_stride, 1, self.n, 0, self.m,
            C.c_void_p(self.ys[j].data_ptr()), self.dcode, self.flags.ptr(),
            C.c_void_p(self.torch.cuda.current_stream().cuda_stream)))

    def step(self, s):
        self.k1(s % self.R)
        self.k2((s - 2) % self.R, s % self.R)

    def graphs(self, steps):
        torch = self.torch
        with torch.cuda.stream(self.stream):
            for i in range(self.R):  # every message written before any K2 reads one
                self.k1(i)
            for s in range(self.R + 2):  # lazy module loads done
                self.step(s)
            self.stream.synchronize()
            self.flags.check()
            g_rt = _graph(lambda: [self.step(s) for s in range(steps)], self.stream)
            g_k1 = _graph(lambda: [self.k1(s % self.R) for s in range(steps)], self.stream)
            g_k2 = _graph(lambda: [self.k2(s % self.R, (s + 1) % self.R) for s in range(steps)], self.stream)
        return g_rt, g_k1, g_k2

    def time(self, g, reps=1):
        torch = self.torch
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(self.stream):
            a.record(self.stream)
            for _ in range(reps):
                g.replay()
            b.record(self.stream)
        self.stream.synchronize()
        return a.elapsed_time(b) / reps


def measure_tensor(idx, rows, cols, dtype_name, args, dev, stream, clk=None):
    """Device-timed K1 + K2 round trip, K1 alone, K2 alone (ms per launch / per step)."""
    import torch
    rb = RoundTripBench(rows, cols, dtype_name, args.block_size, dev, stream)
    g_rt, g_k1, g_k2 = rb.graphs(args.steps)
    for g in (g_rt, g_k1, g_k2):  # warm-up replays of the captured work (>= W steps each)
        for _ in range(max(1, -(-args.warmup // args.steps))):
            g.replay()
    stream.synchronize()
    rb.flags.check()
    t_rt = rb.time(g_rt) / args.steps
    t_k1 = rb.time(g_k1) / args.steps
    t_k2 = rb.time(g_k2) / args.steps
    rb.flags.check()
    esz = 2 if dtype_name == "bf16" else 4
    bpe = algorithmic_bytes_per_elem(args.block_size, esz, esz)
    out = {"rb": rb, "n": rb.n, "bpe": bpe, "ms_per_step": t_rt, "k1_ms": t_k1, "k2_ms": t_k2,
           "graphs": (g_rt, g_k1, g_k2)}
    out["value"] = bpe["roundtrip"] * rb.n / (t_rt * 1e-3) / 1e9
    out["k1_gbs"] = bpe["k1"] * rb.n / (t_k1 * 1e-3) / 1e9
    out["k2_gbs"] = bpe["k2"] * rb.n / (t_k2 * 1e-3) / 1e9
    del torch
    return out


class CollectiveCodecBench:
    """Per-rank codec work of one compressed two-shot all-reduce at P ranks (the collective
    budget): K1 of the P shards of the rank tensor, K3 of the P received
    copies of the own shard, K2 of the P gathered shards -- each timed alone over R rotating
    buffer sets (every launch reads what the previous pass wrote >= one set ago: cold)."""

    R = 3

    def __init__(self, rows, cols, P, block_size, dev, seed=SEED):
        import torch

        from paper_2604_24088_b200 import _abi, codec
        self.torch, self._abi = torch, _abi
        self.n, self.P = rows * cols, P
        self.cfg = codec.make_config(block_size)
        self.S = -(-self.n // P)
        self.m = -(-self.S // block_size)
        self.lay = _abi.msg_layout(self.cfg, self.m)
        x0 = codec.generate(MIXTURE, self.n, seed).to(dev).to(torch.bfloat16)
        self.xs = [torch.roll(x0, k * block_size * 977) for k in range(self.R)]
        st = self.lay.msg_stride
        self.send = [torch.empty(P * st, dtype=torch.uint8, device=dev) for _ in range(self.R)]
        self.red = [torch.empty(st, dtype=torch.uint8, device=dev) for _ in range(self.R)]
        self.ys = [torch.empty(self.n, dtype=torch.bfloat16, device=dev) for _ in range(self.R)]
        self.sp = [torch.empty(self.S, dtype=torch.bfloat16, device=dev) for _ in range(self.R)]  # SP RS output
        self.slice_msg = [torch.empty(st, dtype=torch.uint8, device=dev) for _ in range(self.R)]
        self.flags = codec.Flags(dev)
        self.lib = _abi.lib()

    def _st(self):
        import ctypes as C
        return C.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def k1(self, i):
        import ctypes as C
        self._abi.check(self.lib.taco_compress_dev(
            C.byref(self.cfg), C.c_void_p(self.xs[i].data_ptr()), self._abi.DT_BF16, self.n, self.P, 0, self.m,
            C.c_void_p(self.send[i].data_ptr()), self.lay.msg_stride, self.flags.ptr(), self._st()))

    def k3(self, i):
        import ctypes as C
        self._abi.check(self.lib.taco_reduce_encode_dev(
            C.byref(self.cfg), C.c_void_p(self.send[i].data_ptr()), self.lay.msg_stride, self.P, self.S, 0, self.m,
            C.c_void_p(self.red[i].data_ptr()), None, 0, self.flags.ptr(), self._st()))

    def k3rs(self, i):  # sequence-parallel reduce-scatter: the bf16 stage-1 sum is the product
        import ctypes as C
        self._abi.check(self.lib.taco_reduce_encode_dev(
            C.byref(self.cfg), C.c_void_p(self.send[i].data_ptr()), self.lay.msg_stride, self.P, self.S, 0, self.m,
            None, C.c_void_p(self.sp[i].data_ptr()), self._abi.DT_BF16, self.flags.ptr(), self._st()))

    def k1slice(self, i):  # sequence-parallel all-gather: compress of the own [S] slice
        import ctypes as C
        self._abi.check(self.lib.taco_compress_dev(
            C.byref(self.cfg), C.c_void_p(self.xs[i].data_ptr()), self._abi.DT_BF16, self.S, 1, 0, self.m,
            C.c_void_p(self.slice_msg[i].data_ptr()), self.lay.msg_stride, self.flags.ptr(), self._st()))

    def k2(self, i):
        import ctypes as C
        self._abi.check(self.lib.taco_decompress_dev(
            C.byref(self.cfg), C.c_void_p(self.send[i].data_ptr()), self.lay.msg_stride, self.P, self.n, 0, self.m,
            C.c_void_p(self.ys[i].data_ptr()), self._abi.DT_BF16, self.flags.ptr(), self._st()))

    def measure(self, steps, stream) -> dict:
        torch = self.torch
        out = {}
        with torch.cuda.stream(stream):
            for i in range(self.R):
                self.k1(i)
                self.k3(i)
                self.k2(i)
                self.k3rs(i)
                self.k1slice(i)
            stream.synchronize()
            self.flags.check()
            for name in ("k1", "k3", "k2", "k3rs", "k1slice"):
                fn = getattr(self, name)
                g = _graph(lambda: [fn((s + 1) % self.R) for s in range(steps)], stream)
                g.replay()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                stream.synchronize()
                a.record(stream)
                g.replay()
                b.record(stream)
                stream.synchronize()
                out[name] = a.elapsed_time(b) / steps
        self.flags.check()
        return out


def collective_budget(args, dev, stream, pk) -> dict:
    """configs[1] TP=2, configs[2] TP=4, configs[3] TP=8: measured per-rank codec time of the
    FP8 two-shot against the NVLink wire time of the FP8 two-shot and of a bf16 ring
    all-reduce (both at the nominal 900 GB/s per direction: wire lower bounds)."""
    nvlink = 900.0
    res = {}
    for idx, P in ((1, 2), (2, 4), (3, 8)):
        r, c = CONFIGS[idx][:2]
        cb = CollectiveCodecBench(r, c, P, args.block_size, dev)
        t = cb.measure(max(10, min(args.steps, 50)), stream)
        n, m, st = cb.n, cb.m, cb.lay
        wire_fp8 = 2 * (P - 1) * st.msg_bytes  # bytes sent per rank per direction, both phases
        wire_bf16 = 2 * (P - 1) * n * 2 / P  # ring all-reduce
        k3_bytes = (P + 1) * st.msg_bytes
        codec_us = (t["k1"] + t["k3"] + t["k2"]) * 1e3
        res[f"configs{idx}_tp{P}"] = {
            "shape": [r, c], "P": P,
            "k1_us": round(t["k1"] * 1e3, 2), "k3_us": round(t["k3"] * 1e3, 2), "k2_us": round(t["k2"] * 1e3, 2),
            "codec_us": round(codec_us, 2),
            "k3_frac_of_hbm": round(k3_bytes / (t["k3"] * 1e-3) / 1e9 / pk["hbm_gbs"], 4),
            "fp8_wire_us_at_900GBps": round(wire_fp8 / (nvlink * 1e9) * 1e6, 2),
            "bf16_ring_wire_us_at_900GBps": round(wire_bf16 / (nvlink * 1e9) * 1e6, 2),
            # sequence-parallel pair on the same tensor: RS = K1 (P shards) + K3 (bf16 sum, no
            # re-encode); AG = K1 of the own [S] slice + K2 of the P gathered slices; each moves
            # (P-1) messages per rank (bf16: (P-1)/P * 2n bytes)
            "sp_reduce_scatter_codec_us": round((t["k1"] + t["k3rs"]) * 1e3, 2),
            "sp_all_gather_codec_us": round((t["k1slice"] + t["k2"]) * 1e3, 2),
            "sp_fp8_wire_us_each": round((P - 1) * st.msg_bytes / (nvlink * 1e9) * 1e6, 2),
            "sp_bf16_wire_us_each": round((P - 1) * 2 * n / P / (nvlink * 1e9) * 1e6, 2),
        }
        del cb
    return res


def run_taco_single(args) -> dict:
    import torch

    from paper_2604_24088_b200 import codec

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    pk = peaks()
    rows, cols = args.rows, args.cols
    dtn = CONFIGS[args.config][2] if args.config is not None else "bf16"
    with ClockSampler(0) as clk:
        head = measure_tensor(args.config, rows, cols, dtn, args, dev, stream)
        # keep the same load running until the sampler has >= 5 samples under it
        t0 = time.perf_counter()
        while len(clk.rows) < 8 and time.perf_counter() - t0 < 5:
            head["graphs"][0].replay()
            stream.synchronize()
    rb = head["rb"]
    n, bpe = head["n"], head["bpe"]
    k1_gbs, k2_gbs = head["k1_gbs"], head["k2_gbs"]
    dominant = ("k1", head["k1_ms"], k1_gbs, bpe["k1"]) if head["k1_ms"] >= head["k2_ms"] else \
        ("k2", head["k2_ms"], k2_gbs, bpe["k2"])
    traffic = ncu_traffic("compress" if dominant[0] == "k1" else "decompress")

    # ---- the other configs' per-rank tensors beside the headline (same method)
    extras = {}
    if not args.headline_only:
        for idx in sorted(CONFIGS):
            if idx == args.config:
                continue
            r, c, dname, what = CONFIGS[idx]
            e = measure_tensor(idx, r, c, dname, args, dev, stream)
            unit = {"us_per_roundtrip": round(e["ms_per_step"] * 1e3, 2)} if idx == 0 else {}
            extras[f"configs{idx}"] = {
                "workload": workload(idx, r, c) + (" (L2-resident: latency, SURVEY §7 hard part 5)" if idx == 0 else ""),
                "dtype": dname, "roundtrip_GBps": round(e["value"], 1), "ms_per_step": round(e["ms_per_step"], 5),
                "k1_ms": round(e["k1_ms"], 5), "k1_frac": round(e["k1_gbs"] / pk["hbm_gbs"], 4),
                "k2_ms": round(e["k2_ms"], 5), "k2_frac": round(e["k2_gbs"] / pk["hbm_gbs"], 4), **unit}
            del e

    if not args.headline_only:
        extras["collective_codec_budget"] = collective_budget(args, dev, stream, pk)

    # ---- e2e through the C-ABI host call (pinned host buffers, H2D + D2H inside the timed region)
    hc = codec.HostContext(0)
    xh = rb.xs[0].cpu().pin_memory()
    yh = torch.empty(n, dtype=rb.dt).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(3):
        hc.roundtrip(xh, rb.cfg, yh)
    # the host call is synchronous: time every step, report the median
    per_step = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        hc.roundtrip(xh, rb.cfg, yh)
        per_step.append(time.perf_counter() - t0)
    e2e_s = statistics.median(per_step)
    # the host call equals the device path bit for bit
    with torch.cuda.stream(stream):
        rb.k1(0)
        rb.k2(0, 0)
    stream.synchronize()
    same = torch.equal(yh, rb.ys[0].cpu())
    hc.close()

    step_ms = head["ms_per_step"]
    set_mb = n * (2 * (2 if dtn == "bf16" else 4) + (1 + 8 / args.block_size)) / 1e6
    l2 = (f"inputs larger than L2: {rb.R} rotating buffer sets of {set_mb:.0f} MB (x, message, y) vs 126 MB L2; "
          "K2 decodes the message written 2 steps earlier")
    line = {
        "metric": "taco_compress_decompress_hbm_GBps",
        "value": round(head["value"], 1),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dtn,
        "data": "synthetic: taco::generate near-zero mixture (the reference generator, value for value)",
        "config": config_dict(args.config, rows, cols, args.block_size, l2),
        "launch": f"one CUDA graph of {args.steps} steps (K1 + K2 each, programmatic dependent launch)",
        "roofline": {"bound": "hbm", "kernel": dominant[0], "achieved": round(dominant[2], 1),
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(dominant[2] / pk["hbm_gbs"], 4),
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_source": traffic, "peak_source": pk["source"],
                     "algorithmic_bytes_per_launch": int(dominant[3] * n),
                     "roundtrip_frac": round(head["value"] / pk["hbm_gbs"], 4)},
        "kernels": {"k1_compress": {"ms": round(head["k1_ms"], 5), "GBps": round(k1_gbs, 1),
                                    "frac": round(k1_gbs / pk["hbm_gbs"], 4)},
                    "k2_decompress": {"ms": round(head["k2_ms"], 5), "GBps": round(k2_gbs, 1),
                                      "frac": round(k2_gbs / pk["hbm_gbs"], 4)},
                    "sum_k1_k2_ms": round(head["k1_ms"] + head["k2_ms"], 5)},
        "e2e": {"value": round(bpe["roundtrip"] * n / e2e_s / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(e2e_s * 1e3, 3), "steps": e2e_steps,
                "statistic": "median of per-step host wall times",
                "h2d_bytes_per_step": xh.numel() * xh.element_size(),
                "d2h_bytes_per_step": yh.numel() * yh.element_size(),
                "api": "taco_roundtrip_host (C ABI, pinned host buffers)", "matches_device_path": bool(same)},
        "gpu_launches": 2 * args.steps,  # K1 + K2 per step inside the timed region
        **extras,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, rb.host_x, dtn)
    return line


# ---------------------------------------------------------------- reference (CPU) arm ---
def _ref_tensor(n: int, dtype_name: str, seed: int = SEED):
    """The reference's own generator, rounded to the arm's element type (the reference is
    fp32-only: bf16 values are exact in fp32)."""
    import numpy as np
    import torch

    from oracle.oracle import Ref
    ref = Ref()
    x = ref.generate(MIXTURE, n, seed)
    if dtype_name == "bf16":
        x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    return ref, np.ascontiguousarray(x)


def _time_ref(ref, x, y, block_size, threads, min_s, min_reps=1):
    ref.set_threads(threads)
    reps, t0 = 0, time.perf_counter()
    while reps < min_reps or time.perf_counter() - t0 < min_s:
        ref.roundtrip(x, y, block_size)
        reps += 1
    return (time.perf_counter() - t0) / reps, reps


def cpu_baseline(args, host_x=None, dtype_name="bf16") -> dict:
    """oracle/_ref (the reference, compiled unmodified) round trip of the SAME tensor on the
    host cores: all threads, and one thread (TACO_THREADS=1)."""
    import numpy as np
    n = args.rows * args.cols
    ref, x = _ref_tensor(n, dtype_name)
    cores = os.cpu_count() or 1
    y = np.empty_like(x)
    ref.set_threads(cores)
    ref.roundtrip(x, y, args.block_size)  # warm
    dt, reps = _time_ref(ref, x, y, args.block_size, cores, args.cpu_seconds)
    dt1, reps1 = _time_ref(ref, x, y, args.block_size, 1, 0.0)
    ref.set_threads(cores)
    esz = 2 if dtype_name == "bf16" else 4
    bpe = algorithmic_bytes_per_elem(args.block_size, esz, esz)["roundtrip"]
    return {"value": round(bpe * n / dt / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"taco::compress+decompress of the whole {n}-element tensor x {reps} reps, "
                      f"TACO_THREADS={cores}; same per-element byte accounting as the GPU line",
            "ms_per_sample": round(dt * 1e3, 1),
            "value_1_thread": round(bpe * n / dt1 / 1e9, 4), "ms_per_sample_1_thread": round(dt1 * 1e3, 1)}


def run_reference(args, world: int) -> dict:
    import numpy as np
    cores = os.cpu_count() or 1
    if world > 1:
        from bench_collective import reference_collective
        return reference_collective(args, world)
    n = args.rows * args.cols
    dtn = CONFIGS[args.config][2] if args.config is not None else "bf16"
    esz = 2 if dtn == "bf16" else 4
    bpe = algorithmic_bytes_per_elem(args.block_size, esz, esz)["roundtrip"]
    ref, x = _ref_tensor(n, dtn)
    y = np.empty_like(x)
    ref.set_threads(cores)
    for _ in range(args.warmup):
        ref.roundtrip(x, y, args.block_size)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.roundtrip(x, y, args.block_size)
    dt = (time.perf_counter() - t0) / args.steps
    value = bpe * n / dt / 1e9
    set_mb = n * (2 * esz + (1 + 8 / args.block_size)) / 1e6
    l2 = (f"inputs larger than L2: {RoundTripBench.R} rotating buffer sets of {set_mb:.0f} MB (x, message, y) vs "
          "126 MB L2; K2 decodes the message written 2 steps earlier")
    return {"impl": "reference", "metric": "taco_compress_decompress_hbm_GBps", "value": round(value, 4),
            "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtn, "data": "synthetic: taco::generate near-zero mixture (the reference generator)",
            "config": config_dict(args.config, args.rows, args.cols, args.block_size, l2),
            "impl_note": "unmodified reference (oracle/_ref) taco::compress + taco::decompress of the whole tensor "
                         "per step on the host cores; it computes in double and returns fp32",
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": f"the whole {n}-element tensor every step, TACO_THREADS={cores}"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def parse_shape(text: str):
    parts = text.lower().split("x")
    if len(parts) != 2 or not all(p.isdigit() and int(p) > 0 for p in parts):
        raise SystemExit(f"--shape wants ROWSxCOLS with positive integers, got {text!r}")
    return int(parts[0]), int(parts[1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["taco", "reference"], default="taco")
    ap.add_argument("--block-size", type=int, default=B)
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--headline-only", action="store_true", help="N=1: skip the other configs' tensors")
    ap.add_argument("--chunks", type=int, default=2, help="N>1: pipelined chunks per shard")
    ap.add_argument("--eager", action="store_true", help="N>1: no CUDA-graph capture of the step")
    ap.add_argument("--nccl-nvls", type=int, default=None, choices=(0, 1),
                    help="N>1: NCCL_NVLS_ENABLE for the communicator (the bf16 comparator without / with NVLS)")
    ap.add_argument("--block-sweep", type=lambda t: [int(v) for v in t.split(",")], default=[32, 64, 128, 256, 512],
                    help="N>1 configs[2]: Hadamard block sizes of the sequence-parallel sweep")
    ap.add_argument("--size-sweep", type=lambda t: [float(v) for v in t.split(",")] if t else [], default=None,
                    help="N>1: configs[4] message sizes in MB (default 1,16,256,1024 at N>1; empty string disables)")
    ap.add_argument("--collective", action="store_true", help="run the collective leg even at world size 1")
    ap.add_argument("--plan", action="store_true",
                    help="N>1: print what this N measures (workload, legs, NCCL comparators) without a GPU")
    ap.add_argument("--config", type=int, choices=sorted(CONFIGS), default=None,
                    help="BASELINE.json configs index of the per-rank tensor (N=1 default: 3, the largest; "
                         "N>1 default: 1 / 2 / 3 at 2 / 4 / 8 GPUs)")
    ap.add_argument("--shape", type=str, default=None, help="custom ROWSxCOLS per-rank tensor (bf16)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.size_sweep is None:
        multi = world > 1 or (args.plan and args.gpus > 1)
        args.size_sweep = [1.0, 16.0, 256.0, 1024.0] if multi else ([1.0, 16.0, 256.0] if args.collective else [])
    rank = int(os.environ.get("RANK", "0"))
    n_ranks = max(world, args.gpus) if (args.impl == "reference" or args.plan) else world
    if args.shape:
        args.rows, args.cols = parse_shape(args.shape)
        args.config = None
    else:
        if args.config is None:
            args.config = HEADLINE if n_ranks <= 1 and not args.collective else {2: 1, 4: 2, 8: 3}.get(n_ranks, 1)
        args.rows, args.cols = CONFIGS[args.config][:2]
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, n_ranks)), flush=True)
        return
    if args.plan:
        from bench_collective import plan
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")  # the launch plumbing the real run uses
            dist.barrier()
        if rank == 0:
            print(json.dumps(plan(args, max(world, args.gpus))), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    if world > 1 or args.collective:
        from bench_collective import run_collective
        line = run_collective(args, args.rows, args.cols, ClockSampler, peaks)
        if rank == 0:
            print(json.dumps(line), flush=True)
        return
    print(json.dumps(run_taco_single(args)), flush=True)


if __name__ == "__main__":
    main()
