"""World-1 C-ABI (AbiTwoShotAllReduce) vs Python-orchestrated two-shot, eager, for an ncu
launch list: which kernels each issues and how long they take."""
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24088_b200 import collective  # noqa: E402
from paper_2604_24088_b200._abi import make_config  # noqa: E402

s = socket.socket(); s.bind(("127.0.0.1", 0))
os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
n = 8192 * 2560
x = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
out = torch.empty_like(x)
for name, op in (("python", collective.TwoShotAllReduce(n, make_config(256), chunks=2)),
                 ("c_abi", collective.AbiTwoShotAllReduce(n, make_config(256), chunks=2))):
    for _ in range(3):
        op(x, out)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(name)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(int(os.environ.get("REPS", "20"))):
        op(x, out)
    b.record()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(name, "ms", a.elapsed_time(b) / int(os.environ.get("REPS", "20")), flush=True)
dist.destroy_process_group()
