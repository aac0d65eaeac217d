"""`bench.py --gpus N --plan` under torchrun (gloo, CPU): rank 0 alone prints what the N-GPU
run measures -- the BASELINE config N names, every leg, both bf16 NCCL comparators."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,idx,shape,leg", [(2, 1, [8192, 2560], "fp8_twoshot_allreduce"),
                                             (4, 2, [16384, 3584], "sequence_parallel_block_sweep"),
                                             (8, 3, [16384, 5120], "backward_gradient_allreduce")])
def test_plan_per_n(n, idx, shape, leg):
    # 8 ranks of a CPU container: keep the process count at 2, name the N with --gpus
    procs = min(n, 2)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={procs}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(n),
                        "--config", str(idx), "--plan"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["plan"] and d["n_gpus"] == n
    assert d["config"]["shape"] == shape and f"configs[{idx}]" in d["config"]["workload"]
    assert any(leg in x for x in d["legs"])
    assert len(d["nccl_bf16_comparators"]) == 2 and "--nccl-nvls 0" in d["nccl_bf16_comparators"][1]["run"]
