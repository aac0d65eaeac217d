"""compressed two-shot all-reduce vs ncclAllReduce bf16 over message
sizes 1 MB ... 1 GB (bf16 tensors of 2^19 ... 2^29 elements), both transports.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        tools/collective_sweep.py [--min-log2 19] [--max-log2 29] [--steps 20]

One JSON line per size on rank 0: ms per all-reduce (max over ranks, CUDA events) for the
NCCL-transport two-shot (CUDA-graph captured, 2 chunks), the peer-memory transport and
ncclAllReduce bf16, plus algbw = 2 * bytes / t.  Works at world size 1 (the collectives
degenerate to round trips) to check the harness.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24088_b200 import collective, peer  # noqa: E402
from paper_2604_24088_b200._abi import make_config  # noqa: E402


def timed(fn, steps):
    for _ in range(3):
        fn()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    start.record()
    for _ in range(steps):
        fn()
    end.record()
    torch.cuda.synchronize()
    ms = torch.tensor([start.elapsed_time(end) / steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=19)
    ap.add_argument("--max-log2", type=int, default=29)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--block-size", type=int, default=256)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    cfg = make_config(args.block_size)
    for lg in range(args.min_log2, args.max_log2 + 1):
        n = 1 << lg
        g = torch.Generator(device=dev).manual_seed(100 + rank)
        x = (torch.randn(n, generator=g, device=dev) * 1e-3).to(torch.bfloat16)
        out = torch.empty_like(x)
        row = {"elements": n, "bytes": 2 * n, "world": world}
        ar = collective.TwoShotAllReduce(n, cfg, dtype=torch.bfloat16, chunks=2, device=dev)
        gr = collective.Graphed(ar, x, out)
        row["twoshot_nccl_ms"] = round(timed(gr, args.steps), 4)
        del gr, ar
        try:
            par = peer.PeerTwoShotAllReduce(n, cfg, dtype=torch.bfloat16, device=dev)
            pg = collective.Graphed(par, x, out)
            row["twoshot_peer_ms"] = round(timed(pg, args.steps), 4)
            par.check()
            del pg
            par.close()
        except Exception as e:  # noqa: BLE001 -- reported, the sweep goes on
            row["twoshot_peer_error"] = str(e)
        y = x.clone()
        row["nccl_bf16_ms"] = round(timed(lambda: dist.all_reduce(y), args.steps), 4)
        for k in ("twoshot_nccl_ms", "twoshot_peer_ms", "nccl_bf16_ms"):
            if k in row:
                row[k.replace("_ms", "_algbw_GBps")] = round(2 * n / (row[k] * 1e-3) / 1e9, 1)
        if rank == 0:
            print(json.dumps(row), flush=True)
        torch.cuda.empty_cache()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
