"""Debug driver for the tensor-core K1: compress bf16 tensors of N 128-block tiles."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_24088_b200 import codec
for tiles in [int(v) for v in sys.argv[1:]]:
    n = tiles * 128 * 256
    x = (torch.randn(n, device="cuda") * 1e-2).to(torch.bfloat16)
    cfg = codec.make_config(256)
    msg = codec.compress(x, cfg)
    torch.cuda.synchronize()
    y = codec.decompress(msg, n, cfg)
    err = ((y.float() - x.float()).norm() / x.float().norm()).item()
    print(f"tiles={tiles} ok relL2={err:.4f}", flush=True)
