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


@pytest.mark.parametrize("procs,n,b,dt", [(2, 8192 * 24, 256, "bf16"), (3, 30_001, 128, "f32")])
def test_peer_allreduce_processes_share_one_gpu(procs, n, b, dt):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={procs}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "peer_worker.py"), str(n), str(b), dt]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    tail = (r.stdout[-3000:] + r.stderr[-3000:])
    assert r.returncode == 0, tail
    for rank in range(procs):
        assert f"PEER_OK {rank}" in r.stdout, tail


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
