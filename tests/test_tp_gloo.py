"""Autograd regions and parallel linear layers (paper_2604_24088_b200/tp.py)
across real gloo ranks on CPU, with the oracle-backed codec (tests/host_codec.py) in place
of the kernels.  Forward and backward collectives must equal the reference's two-shot
schedule (proj/src/collective.cpp:75-111) bit for bit."""
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
T, H, F = 64, 32, 48  # tokens, hidden, per-rank features


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(port, rank):
    x = torch.from_numpy(port.mixture(T * F, 300 + rank).reshape(T, F))
    w = torch.from_numpy(port.gaussian(H * F, 400 + rank, 0.05).reshape(H, F))
    g = torch.from_numpy(port.mixture(T * H, 500 + rank).reshape(T, H))
    return x, w, g


def _worker(rank, world, port_no, sp, q):
    try:
        sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port_no)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from host_codec import HostCodec
        from oracle.oracle import Port
        from paper_2604_24088_b200 import tp
        from paper_2604_24088_b200._abi import make_config

        port = Port()
        ctx = tp.TpContext(cfg=make_config(32), codec=HostCodec(port))
        x, w, g = _inputs(port, rank)
        layer = tp.RowParallelLinear(F, H, ctx, sequence_parallel=sp)
        with torch.no_grad():
            layer.linear.weight.copy_(w)
        xin = x.clone().requires_grad_(True)
        y = layer(xin)
        gy = g[rank * (T // world):(rank + 1) * (T // world)] if sp else g
        y.backward(gy)
        # column-parallel: identity forward, compressed all-reduce of dX backward
        col = tp.ColumnParallelLinear(H, F, ctx)
        with torch.no_grad():
            col.linear.weight.copy_(w.t())
        h = g.clone().requires_grad_(True)
        col(h).backward(torch.ones(T, F))
        q.put((rank, {"y": y.detach().numpy(), "dx": xin.grad.numpy(), "dh": h.grad.numpy()}, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("sp", [False, True], ids=["tp", "sp"])
def test_regions_match_reference_two_shot(port, sp):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, pn, sp, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=300)
        assert err is None, err
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    # the forward input of the collective is each rank's local product, computed like torch does
    locals_ = [torch.nn.functional.linear(_inputs(port, r)[0], _inputs(port, r)[1]).numpy() for r in range(world)]
    ref = port.allreduce_twoshot(np.stack([v.reshape(-1) for v in locals_]), 32, 0, want_stage1=True)
    S = T * H // world
    for r in range(world):
        if sp:  # reduce-scatter: the owner's stage-1 fp32 sum
            assert np.array_equal(out[r]["y"].reshape(-1), ref["stage1"][r * S:(r + 1) * S])
        else:
            assert np.array_equal(out[r]["y"].reshape(-1), ref["result"])
    # backward of the row-parallel region: identity (TP) or the SP all-gather of the
    # gradient slices (every slice through the codec once)
    g_all = np.stack([_inputs(port, r)[2].numpy() for r in range(world)])
    for r in range(world):
        w = _inputs(port, r)[1].numpy()
        if sp:
            sl = [g_all[o][o * (T // world):(o + 1) * (T // world)].reshape(-1) for o in range(world)]
            gy = np.concatenate([port.decompress(*port.compress(v, 32, 0), v.size, 32, 0) for v in sl])
            gy = gy.reshape(T, H)
        else:
            gy = g_all[r]
        want = torch.nn.functional.linear(torch.from_numpy(gy), torch.from_numpy(w.T)).numpy()
        assert np.allclose(out[r]["dx"], want, rtol=1e-5, atol=1e-6)
    # column-parallel backward: compressed all-reduce of the per-rank dH
    dh_local = [torch.nn.functional.linear(torch.ones(T, F), torch.from_numpy(_inputs(port, r)[1].numpy().T).t())
                for r in range(world)]
    ref_dh = port.allreduce_twoshot(np.stack([v.numpy().reshape(-1) for v in dh_local]), 32, 0)["result"]
    for r in range(world):
        assert np.array_equal(out[r]["dh"].reshape(-1), ref_dh)
