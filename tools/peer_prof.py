"""World-1 peer-memory two-shot, eager, for an ncu launch list (tools/gpu_peer.sh)."""
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24088_b200 import peer  # noqa: E402
from paper_2604_24088_b200._abi import make_config  # noqa: E402

s = socket.socket(); s.bind(("127.0.0.1", 0))
os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
s.close()
dist.init_process_group("gloo")
n = 8192 * 2560
x = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
for fused in (True, False):
    par = peer.PeerTwoShotAllReduce(n, make_config(256), dtype=torch.bfloat16, device="cuda:0", fused=fused)
    out = torch.empty_like(x)
    for _ in range(int(os.environ.get("ITERS", "6"))):
        par(x, out)
    torch.cuda.synchronize()
    par.check()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(int(os.environ.get("REPS", "50"))):
        par(x, out)
    end.record()
    torch.cuda.synchronize()
    print(f"peer step ms fused={fused}", start.elapsed_time(end) / int(os.environ.get("REPS", "50")), flush=True)
    par.close()
