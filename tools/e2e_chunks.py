"""e2e host round trip vs pipeline chunk size (TACO_HOST_CHUNK_KB read once per process)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24088_b200 import codec  # noqa: E402

n = 8192 * 2560
x = (torch.randn(n) * 1e-3).to(torch.bfloat16).pin_memory()
y = torch.empty(n, dtype=torch.bfloat16).pin_memory()
cfg = codec.make_config(256)
ctx = codec.HostContext(0)
for _ in range(3):
    ctx.roundtrip(x, cfg, y)
t0 = time.perf_counter()
for _ in range(20):
    ctx.roundtrip(x, cfg, y)
dt = (time.perf_counter() - t0) / 20
print(os.environ.get("TACO_HOST_CHUNK_KB", "default"), f"{dt*1e3:.3f} ms", f"{6.0625*n/dt/1e9:.1f} GB/s")
