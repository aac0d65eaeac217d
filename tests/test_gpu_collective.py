"""GPU side of the collective: the CUDA codec speaks exactly the message format the
schedule (validated bit-exactly under gloo with the oracle codec) expects, for shard and
chunk geometries; and the schedule runs end to end on NCCL (world size 1 on the single
GPU available here -- multi-rank NCCL runs in bench.py under torchrun)."""
import os
import socket

import numpy as np
import pytest
import torch

from host_codec import HostCodec
from parity import COLLECTIVE_RELMSE_MAX, DECODE_RELMSE_MAX, check_codec_parity, rel_mse

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2604_24088_b200 import _abi, codec, collective  # noqa: E402
from paper_2604_24088_b200._abi import make_config  # noqa: E402


@pytest.mark.parametrize("n,shards,b,chunk", [(100_000, 3, 256, (5, 90)), (8192 * 37 + 5, 4, 128, (0, 20)),
                                              (65536, 2, 512, (3, 64))])
def test_cuda_codec_speaks_the_host_codec_format(port, n, shards, b, chunk):
    cfg = make_config(b)
    x = port.mixture(n, 5, tail_fraction=0.03)
    S = -(-n // shards)
    m = -(-S // b)
    b0, b1 = chunk
    b1 = min(b1, m)
    lay = _abi.msg_layout(cfg, b1 - b0)
    cc, hc = collective.CudaCodec(), HostCodec(port)
    gd = torch.empty((shards, lay.msg_stride), dtype=torch.uint8, device="cuda")
    gh = torch.zeros((shards, lay.msg_stride), dtype=torch.uint8)
    cc.compress(cfg, torch.from_numpy(x).cuda(), shards, b0, b1, gd)
    hc.compress(cfg, torch.from_numpy(x), shards, b0, b1, gh)
    torch.cuda.synchronize()
    cc.check()
    for p in range(shards):
        dc, da, ds = (t.cpu().numpy() for t in codec.split_message(gd[p], cfg, b1 - b0))
        hc_, ha, hs = (t.numpy() for t in codec.split_message(gh[p], cfg, b1 - b0))
        check_codec_parity(dc, da, ds, hc_, ha, hs, f"shard {p}")
    # decode the HOST messages with the CUDA K2 and vice versa
    yd = torch.zeros(n, dtype=torch.float32, device="cuda")
    yh = torch.zeros(n, dtype=torch.float32)
    cc.decompress(cfg, gh.cuda(), n, shards, b0, b1, yd, lay.msg_stride)
    hc.decompress(cfg, gh, n, shards, b0, b1, yh, lay.msg_stride)
    torch.cuda.synchronize()
    assert rel_mse(yd.cpu().numpy(), yh.numpy()) <= DECODE_RELMSE_MAX
    # K3 on the host-made messages of `shards` "ranks" of one shard
    acc_d = torch.zeros(S, dtype=torch.float32, device="cuda")
    acc_h = torch.zeros(S, dtype=torch.float32)
    red_d = torch.zeros(lay.msg_stride, dtype=torch.uint8, device="cuda")
    red_h = torch.zeros(lay.msg_stride, dtype=torch.uint8)
    cc.reduce_encode(cfg, gh.cuda(), shards, S, lay.msg_stride, b0, b1, red_d, acc_d)
    hc.reduce_encode(cfg, gh, shards, S, lay.msg_stride, b0, b1, red_h, acc_h)
    torch.cuda.synchronize()
    assert rel_mse(acc_d.cpu().numpy(), acc_h.numpy()) <= 1e-10
    # the re-encode, stage-isolated: oracle compress of the GPU's own sum
    lo, hi = b0 * b, min(b1 * b, S)
    rc, ra, rs = port.compress(acc_d.cpu().numpy()[lo:hi], b)
    dc, da, ds = (t.cpu().numpy() for t in codec.split_message(red_d, cfg, b1 - b0))
    check_codec_parity(dc, da, ds, rc, ra, rs, "K3")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_nccl_schedule_world1(port, nccl_world1):
    n = 8192 * 2560
    cfg = make_config(256)
    x32 = port.mixture(n, 7)
    x = torch.from_numpy(x32).cuda().to(torch.bfloat16)
    for chunks in (1, 4):
        ar = collective.TwoShotAllReduce(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32, chunks=chunks)
        ar.stage1 = torch.zeros(ar.shard_len, dtype=torch.float32, device="cuda")
        y = ar(x)
        torch.cuda.synchronize()
        ar.codec.check()
        # P = 1: stage 1 is one round trip, the result a round trip of that
        msg = codec.compress(x, cfg)
        rt1 = codec.decompress(msg, n, cfg)
        rt2 = codec.decompress(codec.compress(rt1, cfg), n, cfg)
        # K3 decodes with K2's code path: the stage-1 sum is bit-identical to a K2 decode
        assert torch.equal(ar.stage1, rt1)
        # K3 re-encodes with the tile encoder, K1 may use another butterfly order: equal up
        # to rare one-ulp code flips (fp32 rounding of differently ordered stages)
        assert rel_mse(y.cpu().numpy(), rt2.cpu().numpy()) < 1e-9
        if chunks == 1:
            y1 = y.clone()
        else:
            assert torch.equal(y, y1)  # chunking never changes numerics
    rs = collective.CompressedReduceScatter(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32, chunks=3)
    assert torch.equal(rs(x), rt1)
    ag = collective.CompressedAllGather(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32, chunks=2)
    assert torch.equal(ag(x), rt1)
    assert rel_mse(rt1.cpu().numpy(), x.float().cpu().numpy()) < 1e-3
    # CUDA-graph replay of the whole step (kernels + NCCL) reproduces the eager result
    ar = collective.TwoShotAllReduce(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32, chunks=2)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    g = collective.Graphed(ar, x, out)
    out.zero_()
    g()
    torch.cuda.synchronize()
    assert torch.equal(out, y1)
    assert COLLECTIVE_RELMSE_MAX > 0


def test_tp_regions_and_custom_ops_on_gpu(port, nccl_world1):
    """tp.py on the CUDA codec (world size 1: the two-shot degenerates to a round trip) and the
    torch.library ops taco_b200::compress / decompress."""
    from paper_2604_24088_b200 import tp

    cfg = make_config(256)
    ctx = tp.TpContext(cfg=cfg, chunks=2)
    T, H, F = 256, 512, 384
    x = torch.from_numpy(port.mixture(T * F, 3).reshape(T, F)).cuda().to(torch.bfloat16).requires_grad_(True)
    row = tp.RowParallelLinear(F, H, ctx, device="cuda", dtype=torch.bfloat16)
    y = row(x)
    local = torch.nn.functional.linear(x.detach(), row.linear.weight.detach())
    # world size 1: the two-shot is K1 -> K3 (decode, re-encode) -> K2, a double round trip
    rt1 = codec.decompress(codec.compress(local, cfg), local.numel(), cfg)
    rt2 = codec.decompress(codec.compress(rt1, cfg), local.numel(), cfg).view(T, H)
    assert rel_mse(y.detach().float().cpu().numpy(), rt2.cpu().numpy()) < 1e-5  # bf16 output rounding
    y.float().sum().backward()
    assert x.grad is not None and torch.isfinite(x.grad.float()).all()
    # torch.library ops == the direct device API
    msg = torch.ops.taco_b200.compress(local, 256, 0)
    assert torch.equal(msg, codec.compress(local, cfg)[0])
    back = torch.ops.taco_b200.decompress(msg, local.numel(), 256, 0, torch.float32)
    assert torch.equal(back, codec.decompress(codec.compress(local, cfg), local.numel(), cfg))


def test_tp_peer_transport_matches_nccl(port, nccl_world1):
    """TpContext(transport="peer") (kernels store into the peers' mapped buffers) gives the same
    bits as the NCCL transport for the row-parallel forward / backward and the SP pair."""
    from paper_2604_24088_b200 import tp

    cfg = make_config(256)
    T, H, F = 256, 512, 384
    x0 = torch.from_numpy(port.mixture(T * F, 4).reshape(T, F)).cuda().to(torch.bfloat16)
    outs = {}
    for transport in ("nccl", "peer"):
        torch.manual_seed(0)
        ctx = tp.TpContext(cfg=cfg, transport=transport)
        row = tp.RowParallelLinear(F, H, ctx, device="cuda", dtype=torch.bfloat16)
        col = tp.ColumnParallelLinear(H, F, ctx, device="cuda", dtype=torch.bfloat16)
        x = x0.clone().requires_grad_(True)
        y = col(row(x))
        y.float().square().sum().backward()
        rs = tp.reduce_scatter_to_sp(y.detach(), ctx)
        ag = tp.gather_from_sp(rs, ctx)
        outs[transport] = (y.detach(), x.grad, rs, ag)
    for a, b in zip(outs["nccl"], outs["peer"]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


@pytest.mark.parametrize("b,P", [(256, 2), (256, 8), (64, 3), (512, 5), (128, 1)])
def test_reduce_encode_pointer_array_matches_strided(port, b, P):
    """taco_reduce_encode_ptrs_dev (rank messages at arbitrary addresses) gives the
    same bytes and stage-1 sums as the strided K3 on the same messages."""
    import ctypes as C
    cfg = make_config(b)
    n = P * 40_000 + 7
    x = torch.from_numpy(port.mixture(n, 3 + P)).cuda().to(torch.bfloat16)
    msgs = codec.compress(x, cfg, shards=P)  # P messages of one shard geometry
    S = -(-n // P)
    m = -(-S // b)
    lay = _abi.msg_layout(cfg, m)
    copies = [msgs[r].clone() for r in range(P)]  # separate allocations
    want = torch.zeros(lay.msg_stride, dtype=torch.uint8, device="cuda")
    acc_w = torch.empty(S, dtype=torch.float32, device="cuda")
    codec.reduce_encode(msgs, P, S, cfg, lay.msg_stride, want, acc_out=acc_w)
    got = torch.zeros_like(want)
    acc_g = torch.empty_like(acc_w)
    ptrs = (C.c_void_p * P)(*[c.data_ptr() for c in copies])
    _abi.check(_abi.lib().taco_reduce_encode_ptrs_dev(C.byref(cfg), ptrs, P, S, 0, m, C.c_void_p(got.data_ptr()),
                                                      C.c_void_p(acc_g.data_ptr()), _abi.DT_F32, None,
                                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(got[: lay.msg_bytes], want[: lay.msg_bytes])
    assert torch.equal(acc_g.view(torch.int32), acc_w.view(torch.int32))


@pytest.mark.parametrize("chunks", [1, 2, 5])
def test_abi_collectives_on_torch_communicator(port, nccl_world1, chunks):
    """The C-ABI collectives on torch's own NCCL communicator (one library call per step)
    equal the Python-orchestrated collectives bit for bit, eagerly and graph-replayed."""
    n = 8192 * 40 + 3
    cfg = make_config(256)
    x = torch.from_numpy(port.mixture(n, 9)).cuda().to(torch.bfloat16)
    ar = collective.AbiTwoShotAllReduce(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32, chunks=chunks)
    want = collective.TwoShotAllReduce(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32, chunks=chunks)(x)
    got = ar(x)
    torch.cuda.synchronize()
    ar.check()
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
    out = torch.full((n,), float("nan"), device="cuda")
    g = collective.Graphed(ar, x, out)
    out.fill_(float("nan"))
    g()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32), want.view(torch.int32))
    rs = collective.AbiReduceScatter(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32, chunks=chunks)
    want_rs = collective.CompressedReduceScatter(n, cfg, dtype=torch.bfloat16, out_dtype=torch.float32,
                                                 chunks=chunks)(x)
    assert torch.equal(rs(x).view(torch.int32), want_rs.view(torch.int32))
    ag = collective.AbiAllGather(n, cfg, dtype=torch.bfloat16, out_dtype=torch.bfloat16, chunks=chunks)
    want_ag = collective.CompressedAllGather(n, cfg, dtype=torch.bfloat16, out_dtype=torch.bfloat16, chunks=chunks)(x)
    assert torch.equal(ag(x), want_ag)
    torch.cuda.synchronize()
    rs.check()
    ag.check()
