"""Peer-memory two-shot (paper_2604_24088_b200/peer.py): the exchange done by the kernels'
own stores into CUDA-IPC mapped peer regions, with device barriers between the phases.

* one process, P simulated ranks (P regions on the device, phase-ordered on one stream):
  every rank's result is bit-identical to codec.allreduce_sim (the NCCL path's kernels);
* two and three processes sharing the one GPU: real IPC mappings, real barriers, eager
  calls and CUDA-graph replays, bit-identical to the simulation;
* a barrier whose peer never arrives times out with the flag instead of hanging.
"""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2604_24088_b200 import _abi, codec, peer  # noqa: E402
from paper_2604_24088_b200._abi import TacoError, make_config  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(p, n, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(p, n, generator=g) * 1e-3
    x[:, ::53] = torch.randn(p, x[:, ::53].shape[1], generator=g)
    return x.to(dtype).cuda()


@pytest.mark.parametrize("p,n,b,dtype,fmt", [
    (2, 8192 * 40, 256, torch.bfloat16, 0),        # tile K3, register K1
    (4, 8192 * 37 + 5, 256, torch.float32, 0),     # ragged last shard, tile K1
    (8, 2560 * 64, 256, torch.bfloat16, 0),        # the TP = 8 fan-out
    (3, 100_003, 64, torch.bfloat16, 0),           # register K3, odd P
    (2, 65_536, 512, torch.float32, 0),
    (1, 4096 + 17, 256, torch.bfloat16, 0),        # a group of one
    (4, 50_000, 256, torch.bfloat16, 1),           # E5M2 (fp64 rotation kernels)
    (2, 30_000, 32, torch.float32, 0),             # small blocks
    (3, 3 * 1024 * 9 + 1, 1024, torch.bfloat16, 0),  # the largest block the push path serves
])
def test_peer_schedule_sim_bit_identical(p, n, b, dtype, fmt):
    cfg = make_config(b, fmt)
    ins = _inputs(p, n, dtype, 11 + p)
    want = codec.allreduce_sim(ins, cfg) if p > 1 else None
    got = peer.allreduce_sim_peer(ins, cfg)
    if p == 1:  # one rank: compress -> (own sum) -> compress -> decompress
        m = codec.compress(ins[0], cfg)
        red = torch.empty_like(m)
        codec.reduce_encode(m, 1, n, cfg, m.shape[1], red)
        want = codec.decompress(red, n, cfg)[None]
    for r in range(p):
        assert torch.equal(got[r].view(torch.int32), want.reshape(-1, n)[0].view(torch.int32)), f"rank {r}"


@pytest.mark.parametrize("p,n,b,dtype", [(4, 8192 * 37 + 5, 256, torch.bfloat16), (3, 50_001, 64, torch.float32),
                                          (8, 2560 * 64, 256, torch.bfloat16)])
def test_peer_reduce_scatter_sim_bit_identical(p, n, b, dtype):
    cfg = make_config(b)
    ins = _inputs(p, n, dtype, 21 + p)
    S = -(-n // p)
    stage1 = torch.empty(p * S, dtype=torch.float32, device="cuda")
    codec.allreduce_sim(ins, cfg, stage1=stage1)
    got = peer.reduce_scatter_sim_peer(ins, cfg)
    assert torch.equal(got.reshape(-1).view(torch.int32), stage1.view(torch.int32))


@pytest.mark.parametrize("p,nl,b,dtype", [(4, 4096 * 9, 256, torch.bfloat16), (3, 10_007, 128, torch.float32),
                                          (2, 65_536, 512, torch.bfloat16)])
def test_peer_all_gather_sim_bit_identical(p, nl, b, dtype):
    cfg = make_config(b)
    ins = _inputs(p, nl, dtype, 31 + p)
    want = torch.cat([codec.decompress(codec.compress(ins[r], cfg), nl, cfg) for r in range(p)])
    got = peer.all_gather_sim_peer(ins, cfg)
    for r in range(p):
        assert torch.equal(got[r].view(torch.int32), want.view(torch.int32)), f"rank {r}"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("procs,n,b,dt,fused", [(2, 8192 * 24, 256, "bf16", 1), (3, 30_001, 128, "f32", 1),
                                                (2, 8192 * 24, 256, "bf16", 0), (3, 30_001, 32, "f32", 0)])
def test_peer_allreduce_processes_share_one_gpu(procs, n, b, dt, fused):
    """fused = 1: the kernels signal the phases themselves (3 launches per all-reduce);
    fused = 0: the push kernels with barrier kernels between the phases (5 launches)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={procs}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "peer_worker.py"), str(n), str(b), dt, str(fused)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    tail = (r.stdout[-3000:] + r.stderr[-3000:])
    assert r.returncode == 0, tail
    for rank in range(procs):
        assert f"PEER_OK {rank} fused={fused}" in r.stdout, tail


def _fused_call(kind, cfg, x, n, ps, geo, out, flags, timeout_ms=10_000):
    import ctypes as C
    lib, st = _abi.lib(), C.c_void_p(torch.cuda.current_stream().cuda_stream)
    dt = codec._dtype_code
    if kind == "ar":
        return lib.taco_peer_allreduce_dev(C.byref(cfg), C.c_void_p(x.data_ptr()), dt(x.dtype), n, C.byref(ps),
                                           geo.recv_off, geo.gath_off, geo.stride, geo.flags_off,
                                           C.c_void_p(out.data_ptr()), dt(out.dtype), timeout_ms, flags.ptr(), st)
    return lib.taco_peer_reduce_scatter_dev(C.byref(cfg), C.c_void_p(x.data_ptr()), dt(x.dtype), n, C.byref(ps),
                                            geo.recv_off, geo.stride, geo.flags_off, C.c_void_p(out.data_ptr()),
                                            dt(out.dtype), timeout_ms, flags.ptr(), st)


@pytest.mark.parametrize("b,dtype", [(256, torch.bfloat16), (64, torch.float32), (512, torch.bfloat16)])
def test_fused_peer_group_of_one_matches_and_keeps_counting(b, dtype):
    """A group of one: the fused kernels wait on and signal their own words.  Repeated calls
    and CUDA-graph replays keep the epoch counting; the result equals the barrier path."""
    cfg = make_config(b)
    n = 8192 * 5 + 7
    geo = peer.PeerLayout(cfg, n, 1)
    dev = torch.cuda.current_device()
    reg = peer.PeerRegion(geo.nbytes, dev)
    try:
        ps = peer.peers_struct([reg.ptr], 0)
        flags = codec.Flags()
        x = _inputs(1, n, dtype, 5)[0]
        want = peer.allreduce_sim_peer(x[None], cfg)[0]
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        for _ in range(3):
            out.fill_(float("nan"))
            _abi.check(_fused_call("ar", cfg, x, n, ps, geo, out, flags))
            torch.cuda.synchronize()
            flags.check()
            assert torch.equal(out.view(torch.int32), want.view(torch.int32))
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            _abi.check(_fused_call("ar", cfg, x, n, ps, geo, out, flags))
        for _ in range(3):
            out.fill_(float("nan"))
            g.replay()
            torch.cuda.synchronize()
            flags.check()
            assert torch.equal(out.view(torch.int32), want.view(torch.int32))
        # reduce-scatter of one rank: the stage-1 sum == a K2 decode of K1's message
        rs = torch.empty(n, dtype=torch.float32, device="cuda")
        _abi.check(_fused_call("rs", cfg, x, n, ps, geo, rs, flags))
        torch.cuda.synchronize()
        flags.check()
        assert torch.equal(rs, codec.decompress(codec.compress(x, cfg), n, cfg))
    finally:
        torch.cuda.synchronize()
        reg.free()


def test_fused_peer_times_out_instead_of_hanging():
    """Rank 1 never runs: rank 0's K3 and K2 give up after the timeout and raise the flag."""
    cfg = make_config(256)
    n = 4096 * 8
    geo = peer.PeerLayout(cfg, n, 2)
    dev = torch.cuda.current_device()
    a, b = peer.PeerRegion(geo.nbytes, dev), peer.PeerRegion(geo.nbytes, dev)
    try:
        ps = peer.peers_struct([a.ptr, b.ptr], 0)
        flags = codec.Flags()
        x = _inputs(1, n, torch.bfloat16, 6)[0]
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        _abi.check(_fused_call("ar", cfg, x, n, ps, geo, out, flags, timeout_ms=200))
        torch.cuda.synchronize()
        with pytest.raises(TacoError, match="peer barrier timed out"):
            flags.check()
    finally:
        torch.cuda.synchronize()
        a.free()
        b.free()


def test_fused_peer_rejects_unserved_configs():
    import ctypes as C
    assert peer.fused_supported(make_config(256)) and not peer.fused_supported(make_config(256, 1))
    assert not peer.fused_supported(make_config(1024)) and not peer.fused_supported(make_config(32))
    cfg = make_config(1024)
    geo = peer.PeerLayout(cfg, 4096, 1)
    reg = peer.PeerRegion(geo.nbytes, torch.cuda.current_device())
    try:
        ps = peer.peers_struct([reg.ptr], 0)
        x = torch.zeros(4096, device="cuda")
        rc = _fused_call("ar", cfg, x, 4096, ps, geo, x, codec.Flags())
        assert rc == _abi.ERR_USAGE and "fused peer signalling" in _abi.lib().taco_last_error().decode()
    finally:
        reg.free()


def test_peer_barrier_times_out_instead_of_hanging():
    geo_bytes = int(_abi.lib().taco_peer_flags_bytes())
    dev = torch.cuda.current_device()
    a, b = peer.PeerRegion(geo_bytes, dev), peer.PeerRegion(geo_bytes, dev)
    try:
        ps = peer.peers_struct([a.ptr, b.ptr], 0)  # rank 1 never arrives
        flags = codec.Flags()
        import ctypes as C
        _abi.check(_abi.lib().taco_peer_barrier_dev(C.byref(ps), 0, 200, flags.ptr(),
                                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        with pytest.raises(TacoError, match="peer barrier timed out"):
            flags.check()
    finally:
        torch.cuda.synchronize()
        a.free()
        b.free()


def test_peer_push_rejects_what_it_does_not_serve():
    import ctypes as C
    x = torch.zeros(1024, device="cuda")
    dev = torch.cuda.current_device()
    reg = peer.PeerRegion(1 << 16, dev)
    try:
        ps = peer.peers_struct([reg.ptr], 0)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        lib = _abi.lib()
        for cfg, msg in ((make_config(2048), "block sizes up to 1024"),
                         (make_config(256, kind=_abi.DIRECT_FP8), "CodecKind::Taco")):
            rc = lib.taco_compress_push_dev(C.byref(cfg), C.c_void_p(x.data_ptr()), 0, 1024, C.byref(ps), 0, 1, 0,
                                            0, None, st)
            assert rc == _abi.ERR_USAGE and msg in lib.taco_last_error().decode()
    finally:
        reg.free()
