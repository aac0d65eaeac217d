"""Small K1 / K2 / K3 / fused-peer invocations for compute-sanitizer (memcheck, racecheck,
synccheck): every exchange-butterfly kernel at B = 64..512, bf16 and fp32, ragged tails,
chunks, shards, and a fused peer all-reduce / reduce-scatter / all-gather of one rank."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24088_b200 import _abi, codec, peer  # noqa: E402

torch.manual_seed(0)
for b in (64, 128, 256, 512):
    cfg = codec.make_config(b)
    for dt in (torch.bfloat16, torch.float32):
        n = b * 37 + 11
        x = (torch.randn(n, device="cuda") * 1e-3).to(dt)
        msg = codec.compress(x, cfg)
        y = codec.decompress(msg, n, cfg, out_dtype=dt)
        sh = codec.compress(x, cfg, shards=3)
        codec.decompress(sh, n, cfg, shards=3)
        part = codec.compress(x, cfg, blk=(3, 20))
        ins = (torch.randn(4, n, device="cuda") * 1e-3).to(dt)
        codec.allreduce_sim(ins, cfg)
        codec.allreduce_sim(ins[:2].contiguous(), cfg)  # the P = 2 K3 specialisation
torch.cuda.synchronize()
# fused peer collectives, a group of one
cfg = codec.make_config(256)
n = 256 * 50 + 3
geo = peer.PeerLayout(cfg, n, 1)
reg = peer.PeerRegion(geo.nbytes, torch.cuda.current_device())
ps = peer.peers_struct([reg.ptr], 0)
fl = codec.Flags()
x = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
out = torch.empty(n, dtype=torch.float32, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
lib = _abi.lib()
for _ in range(2):
    _abi.check(lib.taco_peer_allreduce_dev(C.byref(cfg), C.c_void_p(x.data_ptr()), _abi.DT_BF16, n, C.byref(ps),
                                           geo.recv_off, geo.gath_off, geo.stride, geo.flags_off,
                                           C.c_void_p(out.data_ptr()), _abi.DT_F32, 10000, fl.ptr(), st))
    _abi.check(lib.taco_peer_reduce_scatter_dev(C.byref(cfg), C.c_void_p(x.data_ptr()), _abi.DT_BF16, n,
                                                C.byref(ps), geo.recv_off, geo.stride, geo.flags_off,
                                                C.c_void_p(out.data_ptr()), _abi.DT_F32, 10000, fl.ptr(), st))
torch.cuda.synchronize()
fl.check()
reg.free()
print("sanitize workload ok", flush=True)
