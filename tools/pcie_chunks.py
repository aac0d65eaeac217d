"""Copy-only version of the host pipeline (no kernels): chunked H2D on one stream, D2H of
the same chunk on another after an event -- the floor the e2e pipeline can reach."""
import sys
import time

import torch

n = 8192 * 2560 * 2
nch = int(sys.argv[1]) if len(sys.argv) > 1 else 5
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
cs = -(-n // nch)


def step():
    for c in range(nch):
        a, b = c * cs, min(n, (c + 1) * cs)
        with torch.cuda.stream(s_in):
            d[a:b].copy_(h_in[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
        s_out.wait_event(ev)
        with torch.cuda.stream(s_out):
            h_out[a:b].copy_(d[a:b], non_blocking=True)
    s_out.synchronize()


for _ in range(3):
    step()
t0 = time.perf_counter()
for _ in range(20):
    step()
dt = (time.perf_counter() - t0) / 20
print(f"chunks={nch}: {dt*1e3:.3f} ms per 42 MB in + 42 MB out")
