"""Worker of tests/test_gpu_peer.py: P processes sharing ONE GPU run the peer-memory
two-shot (CUDA IPC between processes, device barriers or the kernels' own phase signals,
K1/K3 pushes) and check every
result bit-for-bit against the one-process simulation of the same schedule.

Launched by torch.distributed.run; gloo only exchanges the IPC handles.  Prints
PEER_OK <rank> on success."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_24088_b200 import codec, peer  # noqa: E402
from paper_2604_24088_b200._abi import make_config  # noqa: E402


def inputs_for(world, n, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(world, n, generator=g) * 1e-3
    x[:, ::97] = torch.randn(world, x[:, ::97].shape[1], generator=g)
    return x.to(dtype).cuda()


def main():
    n, b, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    fused = bool(int(sys.argv[4])) if len(sys.argv) > 4 else None
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    # one GPU per rank when the box has enough (real NVLink peers), else all ranks share GPU 0
    dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    cfg = make_config(b)
    ar = peer.PeerTwoShotAllReduce(n, cfg, dtype=dtype, out_dtype=torch.float32, device=f"cuda:{dev}",
                                   timeout_ms=30_000, fused=fused)
    assert fused is None or ar.fused == fused
    # eager calls with fresh inputs every time (stale slots would show up as mismatches)
    for it in range(3):
        ins = inputs_for(world, n, dtype, 1000 + it)
        want = codec.allreduce_sim(ins, cfg)
        got = ar(ins[rank])
        torch.cuda.synchronize()
        ar.check()
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), f"rank {rank} eager call {it}"
    # CUDA-graph capture of the whole step; replays keep the barrier epochs counting
    x = torch.empty(n, dtype=dtype, device="cuda")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    x.copy_(inputs_for(world, n, dtype, 7)[rank])
    ar(x, out)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ar(x, out)
    for it in range(2):
        ins = inputs_for(world, n, dtype, 2000 + it)
        x.copy_(ins[rank])
        graph.replay()
        torch.cuda.synchronize()
        ar.check()
        want = codec.allreduce_sim(ins, cfg)
        assert torch.equal(out.view(torch.int32), want.view(torch.int32)), f"rank {rank} graph replay {it}"
    ar.close()
    # sequence-parallel pair: reduce-scatter (fp32 stage-1 sums) and all-gather
    S = -(-n // world)
    rs = peer.PeerReduceScatter(n, cfg, dtype=dtype, out_dtype=torch.float32, device=f"cuda:{dev}", timeout_ms=30_000,
                                fused=fused)
    ag = peer.PeerAllGather(S, cfg, dtype=dtype, out_dtype=torch.float32, device=f"cuda:{dev}", timeout_ms=30_000,
                            fused=fused)
    for it in range(2):
        ins = inputs_for(world, n, dtype, 3000 + it)
        stage1 = torch.empty(world * S, dtype=torch.float32, device="cuda")
        codec.allreduce_sim(ins, cfg, stage1=stage1)
        got = rs(ins[rank])
        torch.cuda.synchronize()
        rs.check()
        assert torch.equal(got.view(torch.int32), stage1[rank * S:(rank + 1) * S].view(torch.int32)), f"rs {it}"
        sl = inputs_for(world, S, dtype, 4000 + it)
        want = torch.cat([codec.decompress(codec.compress(sl[r], cfg), S, cfg) for r in range(world)])
        got = ag(sl[rank])
        torch.cuda.synchronize()
        ag.check()
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), f"ag {it}"
    rs.close()
    ag.close()
    dist.destroy_process_group()
    print(f"PEER_OK {rank} fused={int(ar.fused)}", flush=True)


if __name__ == "__main__":
    main()
