"""bench.py's reference arm (the driver's `--impl reference` launch) prints one JSON line
with the contract keys, on CPU, at N = 1 and under a 2-process torchrun (rank 0 only)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from oracle.oracle import ref_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "gpu_launches"}


def _check(line, n):
    d = json.loads(line)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == n and d["value"] > 0 and d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    return d


def test_reference_arm_n1():
    # configs[1]'s tensor keeps the CPU run short; the default is configs[3]
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                        "--config", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = _check(lines[0], 1)
    assert d["metric"] == "taco_compress_decompress_hbm_GBps"
    assert d["config"]["shape"] == [8192, 2560] and "configs[1]" in d["config"]["workload"]


def test_config_dict_is_shared_by_both_arms():
    # the driver compares `config` between the arms: both build it from config_dict
    sys.path.insert(0, ROOT)
    import bench
    a = bench.config_dict(3, 16384, 5120, 256, "x")
    assert a["shape"] == [16384, 5120] and "configs[3]" in a["workload"] and a["in_dtype"] == "bf16"
    assert bench.parse_shape("16384x3584") == (16384, 3584)
    with pytest.raises(SystemExit):
        bench.parse_shape("16384by3584")


def test_reference_arm_torchrun_rank0_only():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = _check(lines[0], 2)
    assert d["metric"] == "taco_twoshot_allreduce_algbw_GBps"
