"""Multi-process (gloo, CPU) tests of the compressed-collective schedule.

paper_2604_24088_b200.collective runs unchanged across real ranks; the codec is the
oracle-backed HostCodec (tests/host_codec.py), which speaks the kernels' exact message
format.  Because the arithmetic is the oracle's, the distributed schedule must equal the
reference's in-process two-shot (proj/src/collective.cpp:75-111) BIT FOR BIT, for any
chunking, world size and ragged length -- which pins sharding, padding, message framing,
the ascending-rank reduction order and the all-gather decode.
"""
import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from host_codec import HostCodec
        from oracle.oracle import Port
        from paper_2604_24088_b200 import collective
        from paper_2604_24088_b200._abi import make_config

        port_ = Port()
        kind, n, b, chunks, fmt = case
        cfg = make_config(b, fmt)
        hc = HostCodec(port_)
        x = torch.from_numpy(port_.mixture(n, 100 + rank, tail_fraction=0.02))
        if kind == "allreduce":
            ar = collective.TwoShotAllReduce(n, cfg, dtype=torch.float32, chunks=chunks, device="cpu", codec=hc)
            ar.stage1 = torch.zeros(ar.shard_len, dtype=torch.float32)
            y = ar(x)
            res = {"y": y.numpy(), "stage1": ar.stage1.numpy(), "wire": ar.wire_bytes_per_rank()}
        elif kind == "reduce_scatter":
            rs = collective.CompressedReduceScatter(n, cfg, dtype=torch.float32, chunks=chunks, device="cpu", codec=hc)
            res = {"y": rs(x).numpy(), "wire": rs.wire_bytes_per_rank()}
        else:
            ag = collective.CompressedAllGather(n, cfg, dtype=torch.float32, chunks=chunks, device="cpu", codec=hc)
            res = {"y": ag(x).numpy(), "wire": ag.wire_bytes_per_rank()}
        q.put((rank, res, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def run_case(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=300)
        assert err is None, err
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    return out


CASES = [
    (2, ("allreduce", 8192, 256, 1, 0)),
    (2, ("allreduce", 8192, 256, 3, 0)),      # chunked pipeline == unchunked
    (3, ("allreduce", 1000, 32, 2, 0)),       # ragged: n % P != 0, S % B != 0
    (2, ("allreduce", 6000, 512, 2, 1)),      # E5M2
    (4, ("allreduce", 17, 4, 1, 0)),          # tiny, padding past n
    (2, ("reduce_scatter", 8192, 256, 2, 0)),
    (3, ("reduce_scatter", 1000, 32, 1, 0)),
    (2, ("all_gather", 4096, 256, 2, 0)),
    (3, ("all_gather", 1000, 32, 3, 0)),
]


@pytest.mark.parametrize("world,case", CASES, ids=[f"p{w}-{c[0]}-n{c[1]}-b{c[2]}-ch{c[3]}-f{c[4]}"
                                                   for w, c in CASES])
def test_schedule_matches_reference_two_shot(world, case, port):
    kind, n, b, chunks, fmt = case
    out = run_case(world, case)
    ins = np.stack([port.mixture(n, 100 + r, tail_fraction=0.02) for r in range(world)])
    S = -(-n // world)
    if kind == "allreduce":
        ref = port.allreduce_twoshot(ins, b, fmt, want_stage1=True)
        for r in range(world):
            assert np.array_equal(out[r]["y"], ref["result"]), f"rank {r}"
            # each owner's stage-1 fp32 sum is its slice of the reference's
            assert np.array_equal(out[r]["stage1"][: min(S, n - r * S)],
                                  ref["stage1"][r * S: r * S + min(S, n - r * S)])
        # wire bytes == the reference's accounting minus the 22-byte archive headers
        m = -(-S // b)
        if chunks == 1 and b >= 16:
            assert out[0]["wire"] == 2 * (world - 1) * m * (b + 8)
            assert world * out[0]["wire"] + 2 * world * (world - 1) * 22 == ref["bytes_on_wire"]
    elif kind == "reduce_scatter":
        ref = port.allreduce_twoshot(ins, b, fmt, want_stage1=True)
        for r in range(world):
            assert np.array_equal(out[r]["y"], ref["stage1"][r * S:(r + 1) * S])
    else:
        want = np.concatenate([port.decompress(*port.compress(ins[r], b, fmt), n, b, fmt) for r in range(world)])
        for r in range(world):
            assert np.array_equal(out[r]["y"], want)
