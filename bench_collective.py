"""N > 1 leg of bench.py: the FP8 two-shot compressed all-reduce across ranks (torchrun,
one process per GPU, NCCL over NVLink), next to ncclAllReduce bf16 on the same tensors.

value = aggregate all-reduce algbw = N * (bytes of each rank's bf16 tensor) / t, t the
max over ranks of the CUDA-event time of K steps (barrier + synchronize on both sides).
"""
from __future__ import annotations

import os
import statistics
import sys
import time

import torch
import torch.distributed as dist


def reference_collective(args, world: int) -> dict:
    """`bench.py --impl reference` at N > 1: the reference's own taco::allreduce(TwoShot)
    (oracle/_ref, unmodified sources) simulating the `world` ranks in one host process
    (collective.cpp:75-111) on the host cores -- rank 0 only.  Per-rank inputs are the
    reference generator's mixture with seed 100 + r (acceptance.cpp:380).  A bounded sample
    of each rank's tensor (the simulation runs all P ranks' codec calls serially in one
    process: the full configs take 1-14 s per step)."""
    import numpy as np
    import torch

    from oracle.oracle import Ref

    cores = os.cpu_count() or 1
    ref = Ref()
    n_full = args.rows * args.cols
    per_rank = min(n_full, 1 << 20)
    ins = np.stack([torch.from_numpy(ref.generate(1, per_rank, 100 + r)).to(torch.bfloat16).float().numpy()
                    for r in range(world)])
    ref.set_threads(cores)
    for _ in range(args.warmup):
        ref.allreduce(ins, args.block_size)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.allreduce(ins, args.block_size)
    dt = (time.perf_counter() - t0) / args.steps
    value = world * 2 * per_rank / dt / 1e9
    desc = (f"taco::allreduce(TwoShot) simulating {world} ranks in one process, {per_rank} elements per rank "
            f"(bounded sample of the {n_full}-element per-rank tensors), TACO_THREADS={cores}")
    return {"impl": "reference", "metric": "taco_twoshot_allreduce_algbw_GBps", "value": round(value, 4),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic: taco::generate near-zero mixture, seed 100 + rank",
            "config": workload_config(args, world),
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": desc},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def workload_config(args, world: int) -> dict:
    """The N > 1 workload that `--gpus N` names (identical in both arms)."""
    idx = getattr(args, "config", None)
    what = {1: "row-parallel output all-reduce", 2: "sequence-parallel reduce-scatter + all-gather",
            3: "forward activation + backward activation-gradient all-reduce"}.get(idx, "all-reduce")
    return {"workload": f"configs[{idx}] per-rank tensor [{args.rows} x {args.cols}] bf16, TP={world} FP8 two-shot "
                        f"{what}" if idx is not None else f"[{args.rows} x {args.cols}] bf16, TP={world} two-shot",
            "shape": [args.rows, args.cols], "elements_per_rank": args.rows * args.cols,
            "block_size": args.block_size, "format": "E4M3", "parallelism": f"tp{world}"}


def _timed(fn, steps, stream):
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    start.record(stream)
    for i in range(steps):
        fn(i)
    end.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([start.elapsed_time(end)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def _peer_leg(args, n, cfg, xs, outs, ar, step_ms, stream, R):
    """Peer-memory two-shot (K1/K3 store into CUDA-IPC mapped peer regions, device
    barriers): time it like the NCCL leg and check it against the NCCL leg's result."""
    from paper_2604_24088_b200 import collective, peer
    from paper_2604_24088_b200._abi import TacoError

    world = dist.get_world_size()
    try:
        par = peer.PeerTwoShotAllReduce(n, cfg, dtype=torch.bfloat16, device=xs[0].device, timeout_ms=20_000)
    except TacoError as e:
        return {"error": str(e)}
    pouts = [torch.empty_like(o) for o in outs]

    def agree(ok: bool) -> bool:  # every rank takes the same branch (no mismatched collectives)
        t = torch.tensor([1 if ok else 0], device=xs[0].device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item() == 1)

    err = ""
    try:
        graphs = [collective.Graphed(par, xs[i], pouts[i]) for i in range(R)] if not args.eager else None

        def pstep(i):
            if graphs is not None:
                graphs[i % R]()
            else:
                par(xs[i % R], pouts[i % R])

        for i in range(args.warmup):
            pstep(i)
        torch.cuda.synchronize()
        par.check()
    except TacoError as e:
        err = str(e)
    if not agree(not err):
        par.close()
        return {"error": err or "failed on another rank"}
    ms = _timed(pstep, args.steps, stream) / args.steps
    # bit-identical to the NCCL two-shot on the same input, on every rank; errors are
    # gathered, never raised between collectives
    ar(xs[0], outs[0])
    par(xs[0], pouts[0])
    torch.cuda.synchronize()
    try:
        par.check()
    except TacoError as e:
        err = str(e)
    same = torch.equal(outs[0].view(torch.int16), pouts[0].view(torch.int16))
    t = torch.tensor([1 if same else 0, 0 if err else 1], device=xs[0].device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    par.close()
    if int(t[1].item()) == 0:
        return {"error": err or "failed on another rank"}
    return {"ms_per_step": round(ms, 5), "algbw_GBps": round(world * 2 * n / (ms * 1e-3) / 1e9, 1),
            "speedup_vs_nccl_twoshot": round(step_ms / ms, 3),
            "bit_identical_to_nccl_twoshot": bool(int(t[0].item()) == 1),
            "fused_signalling": par.fused, "gpu_launches_per_step": par.launches(),
            "barrier_kernels_per_step": 0 if par.fused else 2}


def _abi_leg(args, n, cfg, xs, outs, step_ms, stream, R):
    """The same two-shot through the C ABI on torch's own NCCL communicator
    (taco_allreduce_nccl_chunked: one library call per step), CUDA-graph captured like the
    Python-orchestrated leg and checked bit for bit against it on every rank."""
    from paper_2604_24088_b200 import collective
    from paper_2604_24088_b200._abi import TacoError

    world = dist.get_world_size()
    try:
        car = collective.AbiTwoShotAllReduce(n, cfg, dtype=torch.bfloat16, chunks=args.chunks, device=xs[0].device)
    except (TacoError, AttributeError, RuntimeError) as e:
        return {"error": f"{type(e).__name__}: {e}"}
    couts = [torch.empty_like(o) for o in outs]
    graphs = [collective.Graphed(car, xs[i], couts[i]) for i in range(R)] if not args.eager else None

    def cstep(i):
        if graphs is not None:
            graphs[i % R]()
        else:
            car(xs[i % R], couts[i % R])

    for i in range(args.warmup):
        cstep(i)
    torch.cuda.synchronize()
    ms = _timed(cstep, args.steps, stream) / args.steps
    # eager (no graph): one library call per step against the Python schedule's per-chunk calls
    eager_ms = _timed(lambda i: car(xs[i % R], couts[i % R]), args.steps, stream) / args.steps
    ar_py = collective.TwoShotAllReduce(n, cfg, dtype=torch.bfloat16, chunks=args.chunks, device=xs[0].device)
    for i in range(2):
        ar_py(xs[i % R], couts[i % R])
    py_eager_ms = _timed(lambda i: ar_py(xs[i % R], couts[i % R]), args.steps, stream) / args.steps
    car(xs[0], couts[0])
    torch.cuda.synchronize()
    car.check()
    same = torch.tensor([int(torch.equal(couts[0].view(torch.int16), outs[0].view(torch.int16)))], device=xs[0].device)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    rep = {"ms_per_step": round(ms, 5), "algbw_GBps": round(world * 2 * n / (ms * 1e-3) / 1e9, 1),
           "speedup_vs_python_twoshot": round(step_ms / ms, 3),
           "eager_ms_per_step": round(eager_ms, 5), "python_eager_ms_per_step": round(py_eager_ms, 5),
           "bit_identical_to_python_twoshot": bool(int(same.item()) == 1), "chunks": args.chunks,
           "api": "taco_allreduce_nccl_chunked on ProcessGroupNCCL._comm_ptr()"}
    if world == 1:
        rep["note"] = ("world size 1: torch's all_to_all / all_gather become local copies without NCCL kernels, "
                       "while NCCL's self send/recv in the C ABI launches two SendRecv kernels per chunk")
    return rep


def _sp_leg(args, n, cfg, xs, stream, use_graphs, peer_leg=True):
    """CompressedReduceScatter of the [n] tensor and CompressedAllGather of its [n/P] slice,
    timed like the all-reduce, next to dist.reduce_scatter_tensor / all_gather_into_tensor
    bf16 on the same tensors."""
    from paper_2604_24088_b200 import collective

    world = dist.get_world_size()
    dev = xs[0].device
    rs = collective.CompressedReduceScatter(n, cfg, dtype=torch.bfloat16, chunks=args.chunks, device=dev)
    S = rs.shard_len
    ag = collective.CompressedAllGather(S, cfg, dtype=torch.bfloat16, chunks=args.chunks, device=dev)
    rs_out = torch.empty(S, dtype=torch.bfloat16, device=dev)
    ag_in = xs[0][:S].clone()
    ag_out = torch.empty(world * S, dtype=torch.bfloat16, device=dev)
    if use_graphs:
        g_rs, g_ag = collective.Graphed(rs, xs[0], rs_out), collective.Graphed(ag, ag_in, ag_out)
        rs_step, ag_step = (lambda i: g_rs()), (lambda i: g_ag())
    else:
        rs_step, ag_step = (lambda i: rs(xs[0], rs_out)), (lambda i: ag(ag_in, ag_out))
    nx = xs[0][: world * S] if xs[0].numel() >= world * S else torch.nn.functional.pad(xs[0], (0, world * S - n))
    nrs = torch.empty(S, dtype=torch.bfloat16, device=dev)
    nag = torch.empty(world * S, dtype=torch.bfloat16, device=dev)
    rep = {}
    for name, fn, ref_fn, byts in (
            ("reduce_scatter", rs_step, lambda i: dist.reduce_scatter_tensor(nrs, nx), 2 * n),
            ("all_gather", ag_step, lambda i: dist.all_gather_into_tensor(nag, ag_in), 2 * world * S)):
        for i in range(args.warmup):
            fn(i)
        t = _timed(fn, args.steps, stream) / args.steps
        for i in range(args.warmup):
            ref_fn(i)
        tn = _timed(ref_fn, args.steps, stream) / args.steps
        rep[name] = {"ms_per_step": round(t, 5), "algbw_GBps": round(byts / (t * 1e-3) / 1e9, 1),
                     "nccl_bf16_ms_per_step": round(tn, 5), "speedup_vs_nccl_bf16": round(tn / t, 3),
                     "wire_bytes_per_rank": (rs if name == "reduce_scatter" else ag).wire_bytes_per_rank()}
    rs.ar.codec.check()
    ag.codec.check()
    if not peer_leg:
        return rep
    # the same pair over peer memory (peer.py), checked bit for bit against the NCCL transport
    from paper_2604_24088_b200 import peer
    from paper_2604_24088_b200._abi import TacoError
    try:
        prs = peer.PeerReduceScatter(n, cfg, dtype=torch.bfloat16, device=dev, timeout_ms=20_000)
        pag = peer.PeerAllGather(S, cfg, dtype=torch.bfloat16, device=dev, timeout_ms=20_000)
    except TacoError as e:
        rep["peer_memory"] = {"error": str(e)}
        return rep
    p_rs = torch.empty_like(rs_out)
    p_ag = torch.empty_like(ag_out)
    err = ""
    try:
        for i in range(args.warmup):
            prs(xs[0], p_rs)
            pag(ag_in, p_ag)
        torch.cuda.synchronize()
        prs.check()
        pag.check()
    except TacoError as e:
        err = str(e)
    t = torch.tensor([0 if err else 1], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if int(t.item()) == 1:
        t_rs = _timed(lambda i: prs(xs[0], p_rs), args.steps, stream) / args.steps
        t_ag = _timed(lambda i: pag(ag_in, p_ag), args.steps, stream) / args.steps
        rs(xs[0], rs_out)
        ag(ag_in, ag_out)
        prs(xs[0], p_rs)
        pag(ag_in, p_ag)
        torch.cuda.synchronize()
        same = torch.tensor([int(torch.equal(rs_out.view(torch.int16), p_rs.view(torch.int16))
                                 and torch.equal(ag_out.view(torch.int16), p_ag.view(torch.int16)))], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        rep["peer_memory"] = {"reduce_scatter_ms_per_step": round(t_rs, 5), "all_gather_ms_per_step": round(t_ag, 5),
                              "bit_identical_to_nccl_transport": bool(int(same.item()) == 1)}
    else:
        rep["peer_memory"] = {"error": err or "failed on another rank"}
    prs.close()
    pag.close()
    return rep


def _nccl_logging() -> str | None:
    """NCCL's log lines (INIT, and the version banner NCCL_DEBUG=VERSION prints) go to a
    per-process file and never to rank 0's stdout, which is the one JSON line; returns the
    file name, read back for the algorithm record."""
    if os.environ.get("NCCL_DEBUG_FILE"):
        return os.environ["NCCL_DEBUG_FILE"]
    path = f"/tmp/taco_nccl_init.{os.getpid()}.log"
    level = os.environ.get("NCCL_DEBUG", "").upper()
    if level not in ("INFO", "TRACE"):
        os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,ENV")
    os.environ["NCCL_DEBUG_FILE"] = path
    return path


def _nccl_record(path: str | None) -> dict:
    """What NCCL chose on this box: version, NVLS (NVLink SHARP multicast) availability and the
    environment toggles that were set, from the INIT log (echoed to stderr for the driver)."""
    rec = {"version": ".".join(str(v) for v in torch.cuda.nccl.version()),
           "NCCL_DEBUG": os.environ.get("NCCL_DEBUG"),
           "NCCL_NVLS_ENABLE": os.environ.get("NCCL_NVLS_ENABLE", "default"),
           "NCCL_ALGO": os.environ.get("NCCL_ALGO", "default")}
    if path and os.path.exists(path):
        lines = open(path, errors="replace").read().splitlines()
        for ln in lines:
            print(ln, file=sys.stderr)
        nv = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if "NVLS" in ln or "nvls" in ln]
        rec["nvls_lines"] = nv[:4]
        rec["nvls_available"] = any("support is available" in ln or "NVLS multicast" in ln for ln in nv)
    return rec


def _inputs(n: int, rank: int, dev, R: int, scale: float = 1.0):
    """The reference generator's near-zero mixture (taco::generate, seed 100 + rank as
    acceptance.cpp:380), rounded to bf16, R rotations (distinct addresses, same values)."""
    from paper_2604_24088_b200 import codec

    x0 = codec.generate(codec.NEAR_ZERO_MIXTURE, n, 100 + rank).mul_(scale).to(torch.bfloat16).to(dev)
    return [x0] + [torch.roll(x0, (k * n) // R // 256 * 256) for k in range(1, R)]


def _ar_leg(args, n, cfg, xs, outs, stream, chunks):
    """Compressed two-shot all-reduce (NCCL transport) timed over K steps, CUDA-graph captured
    where every rank can, next to ncclAllReduce bf16 on the same tensors."""
    from paper_2604_24088_b200 import collective

    world = dist.get_world_size()
    R = len(xs)
    ar = collective.TwoShotAllReduce(n, cfg, dtype=torch.bfloat16, chunks=chunks, device=xs[0].device)
    graphs, note = None, "eager"
    if not args.eager:
        try:
            graphs, ok = [collective.Graphed(ar, xs[i], outs[i]) for i in range(R)], 1
        except Exception as e:  # noqa: BLE001 -- reported, eager instead
            graphs, ok, note = None, 0, f"eager (graph capture failed: {type(e).__name__})"
        t = torch.tensor([ok], device=xs[0].device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) == 1:
            note = "cuda_graph"
        else:
            graphs = None

    def step(i):
        if graphs is not None:
            graphs[i % R]()
        else:
            ar(xs[i % R], outs[i % R])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ar.codec.check()
    ms = _timed(step, args.steps, stream) / args.steps
    ar.codec.check()
    scratch = [x.clone() for x in xs]

    def nccl_step(i):
        dist.all_reduce(scratch[i % R])

    for i in range(args.warmup):
        nccl_step(i)
    nccl_ms = _timed(nccl_step, args.steps, stream) / args.steps
    wire = ar.wire_bytes_per_rank()
    return ar, step, graphs, note, {
        "ms_per_step": round(ms, 5), "algbw_GBps": round(world * 2 * n / (ms * 1e-3) / 1e9, 1),
        "nccl_bf16_ms_per_step": round(nccl_ms, 5),
        "nccl_bf16_algbw_GBps": round(world * 2 * n / (nccl_ms * 1e-3) / 1e9, 1),
        "speedup_vs_nccl_bf16": round(nccl_ms / ms, 3),
        "wire_bytes_per_rank": wire, "wire_frac_of_nvlink_900": round(wire / (ms * 1e-3) / 900e9, 4),
        "chunks": chunks, "launch": note}


def plan(args, world: int) -> dict:
    """What `bench.py --gpus N` measures at this N, without touching a GPU (`--plan`): the
    workload, every leg and both bf16 NCCL comparators."""
    idx = args.config
    legs = ["fp8_twoshot_allreduce (NCCL transport, chunked, CUDA graph)", "peer_memory_twoshot (fused signalling)",
            "c_abi_twoshot (taco_allreduce_nccl_chunked on torch's communicator)"]
    if idx == 2 or args.collective:
        legs += ["sequence_parallel reduce-scatter + all-gather (NCCL and peer transports)",
                 "sequence_parallel_block_sweep B in " + ",".join(str(b) for b in args.block_sweep)]
    if idx == 3 or args.collective:
        legs += ["backward_gradient_allreduce (x 2^-6 activation-gradients)"]
    if args.size_sweep:
        legs += ["message_size_sweep " + ",".join(f"{mb}MB" for mb in args.size_sweep)]
    return {"plan": True, "n_gpus": world, "config": workload_config(args, world), "legs": legs,
            "nccl_bf16_comparators": [
                {"what": "ncclAllReduce / reduce_scatter_tensor / all_gather_into_tensor bf16, same tensors",
                 "NCCL_NVLS_ENABLE": os.environ.get("NCCL_NVLS_ENABLE", "default") if args.nccl_nvls is None
                 else str(args.nccl_nvls)},
                {"what": "the same with NVLink SHARP off", "run": "bench.py --gpus N --nccl-nvls 0"}],
            "nccl_record": "version, NVLS availability and toggles from the NCCL INIT log (NCCL_DEBUG_FILE)"}


def run_collective(args, rows, cols, clock_sampler, peaks):
    from paper_2604_24088_b200._abi import make_config

    if "RANK" not in os.environ:  # `bench.py --collective` without torchrun: a world of one
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(sk.getsockname()[1]))
        sk.close()
    if args.nccl_nvls is not None:  # read by NCCL at communicator init
        os.environ["NCCL_NVLS_ENABLE"] = str(args.nccl_nvls)
    log = _nccl_logging()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    idx = args.config
    n = rows * cols
    cfg = make_config(args.block_size)
    R = 3  # rotating inputs / outputs: consecutive steps do not hit the same L2 lines
    xs = _inputs(n, rank, dev, R)
    outs = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(R)]
    stream = torch.cuda.current_stream()
    with clock_sampler(local) as clk:
        ar, step, graphs, note, ar_rep = _ar_leg(args, n, cfg, xs, outs, stream, args.chunks)
        t0 = time.perf_counter()
        while len(clk.rows) < 5 and time.perf_counter() - t0 < 5:
            for i in range(20):
                step(i)
            torch.cuda.synchronize()
    step_ms = ar_rep["ms_per_step"]
    value = world * 2 * n / (step_ms * 1e-3) / 1e9

    # the same all-reduce with the exchange done by the kernels' own stores into the peers'
    # memory (peer.py): no NCCL call on the data path; must be bit-identical to the above
    peer_rep = _peer_leg(args, n, cfg, xs, outs, ar, step_ms, stream, R)
    # outs[0] holds the Python two-shot's result of xs[0] (the peer leg's last check)
    ar(xs[0], outs[0])
    abi_rep = _abi_leg(args, n, cfg, xs, outs, step_ms, stream, R)

    extra = {}
    if idx == 2 or args.collective:
        # configs[2]: the sequence-parallel pair, with the Hadamard block-size sweep
        extra["sequence_parallel"] = _sp_leg(args, n, cfg, xs, stream, graphs is not None)
        sweep = {}
        for b in args.block_sweep:
            if b == args.block_size:
                continue
            cb = make_config(b)
            sp = _sp_leg(args, n, cb, xs, stream, graphs is not None, peer_leg=False)
            sweep[str(b)] = {k: v["ms_per_step"] for k, v in sp.items()}
        extra["sequence_parallel_block_sweep"] = sweep
    if idx == 3 or args.collective:
        # configs[3]: the backward activation-gradient all-reduce on the same shape: gradients
        # ~2^-6 of the activations (dual-scale quantisation: alpha absorbs the scale, the
        # codes and s are those of the forward tensor, test_codec.cpp:217-234), overlapped
        # by the chunked pipeline
        gx = [x.float().mul_(2.0 ** -6).to(torch.bfloat16) for x in xs]
        gouts = [torch.empty_like(o) for o in outs]
        _, _, _, gnote, g_rep = _ar_leg(args, n, cfg, gx, gouts, stream, args.chunks)
        extra["backward_gradient_allreduce"] = g_rep
        extra["fwd_plus_bwd_ms"] = round(step_ms + g_rep["ms_per_step"], 5)
        extra["fwd_plus_bwd_nccl_bf16_ms"] = round(ar_rep["nccl_bf16_ms_per_step"] + g_rep["nccl_bf16_ms_per_step"], 5)
    if args.size_sweep:
        # configs[4] summary: compressed vs uncompressed all-reduce over message sizes
        sw = {}
        for mb in args.size_sweep:
            m_el = max(world * 256, int(mb * 2 ** 20) // 2)
            sx = _inputs(m_el, rank, dev, 2)
            so = [torch.empty_like(v) for v in sx]
            sargs = type(args)(**{**vars(args), "steps": max(5, min(args.steps, 20)), "warmup": 3})
            _, _, _, _, r = _ar_leg(sargs, m_el, cfg, sx, so, stream, args.chunks)
            c = 1 + 8 / args.block_size
            hbm_bytes = m_el * (4 + 2 * c) + (world + 1) * c * m_el / world  # K1 + K2 + K3 per rank
            sw[f"{mb}MB"] = {"taco_ms": r["ms_per_step"], "nccl_bf16_ms": r["nccl_bf16_ms_per_step"],
                             "speedup": r["speedup_vs_nccl_bf16"], "wire_frac_of_nvlink_900": r["wire_frac_of_nvlink_900"],
                             "codec_hbm_frac": round(hbm_bytes / (r["ms_per_step"] * 1e-3) / (peaks()["hbm_gbs"] * 1e9), 4)}
            del sx, so
        extra["message_size_sweep"] = sw

    # e2e: pinned host tensor -> H2D -> compressed all-reduce -> D2H, every step
    from paper_2604_24088_b200 import collective
    xh = xs[0].cpu().pin_memory()
    yh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    xd = torch.empty_like(xs[0])
    g_e2e = collective.Graphed(ar, xd, outs[0]) if graphs is not None else None

    def e2e_step(i):
        xd.copy_(xh, non_blocking=True)
        if g_e2e is not None:
            g_e2e()
        else:
            ar(xd, outs[0])
        yh.copy_(outs[0], non_blocking=True)

    for i in range(3):
        e2e_step(i)
    e2e_steps = max(3, min(args.steps, 20))
    e2e_ms = _timed(e2e_step, e2e_steps, stream) / e2e_steps

    # parity spot check across ranks: everyone holds the identical result
    ar(xs[0], outs[0])
    chk = outs[0].float().sum().reshape(1)
    mx, mn = chk.clone(), chk.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(mn, op=dist.ReduceOp.MIN)
    pk = peaks()
    line = None
    if rank == 0:
        wire = ar_rep["wire_bytes_per_rank"]
        line = {
            "metric": "taco_twoshot_allreduce_algbw_GBps",
            "value": round(value, 1),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(step_ms, 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic: taco::generate near-zero mixture (the reference generator), seed 100 + rank, bf16",
            "config": {**workload_config(args, world), "chunks": args.chunks, "launch": note,
                       "l2": f"{R} rotating input/output buffers of {2 * n / 1e6:.0f} MB per rank"},
            "nccl_bf16_allreduce": {"ms_per_step": ar_rep["nccl_bf16_ms_per_step"],
                                    "algbw_GBps": ar_rep["nccl_bf16_algbw_GBps"],
                                    "speedup_of_taco": ar_rep["speedup_vs_nccl_bf16"]},
            "nccl": _nccl_record(log),
            "wire": {"bytes_per_rank_per_direction": wire,
                     "GBps_per_rank": round(wire / (step_ms * 1e-3) / 1e9, 1),
                     "frac_of_nvlink_900": ar_rep["wire_frac_of_nvlink_900"]},
            "roofline": {"bound": "nvlink", "achieved": round(wire / (step_ms * 1e-3) / 1e9, 1), "peak": 900.0,
                         "unit": "GB/s", "frac": ar_rep["wire_frac_of_nvlink_900"], "traffic": None,
                         "peak_source": "nominal NVLink 5 per direction",
                         "hbm_peak_GBps": pk["hbm_gbs"]},
            "e2e": {"value": round(world * 2 * n / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                    "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": 2 * n,
                    "api": "collective.TwoShotAllReduce (pinned host in / out)"},
            "peer_memory_twoshot": peer_rep,
            "c_abi_twoshot": abi_rep,
            **extra,
            "ranks_agree": bool(abs(float(mx.item()) - float(mn.item())) == 0.0),
            "gpu_launches": 3 * len(ar.ch.ranges) * args.steps,
            "clocks": clk.summary(),
        }
    dist.barrier()
    dist.destroy_process_group()
    return line
