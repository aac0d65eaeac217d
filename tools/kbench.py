"""Kernel-only timing of K1 / K2 (and K3) for A/B builds: TACO_B200_LIB=<so> python tools/kbench.py.

Not the contract benchmark (bench.py is); prints one line per kernel with GB/s of
algorithmic bytes, CUDA-event timed on the launching stream, rotating 4 buffer sets."""
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24088_b200 import _abi, codec  # noqa: E402


def main():
    b = int(os.environ.get("B", "256"))
    n = int(os.environ.get("N", str(8192 * 2560)))
    dt = torch.bfloat16 if os.environ.get("DT", "bf16") == "bf16" else torch.float32
    fmt = int(os.environ.get("FMT", "0"))
    reps = int(os.environ.get("REPS", "100"))
    cfg = codec.make_config(b, fmt)
    m = -(-n // b)
    lay = _abi.msg_layout(cfg, m)
    R = 4
    if os.environ.get("GEN", "mixture") == "randn":
        xs = [torch.randn(n, device="cuda").to(dt) for _ in range(R)]
    else:  # the reference generator's near-zero mixture (bench.py's input), rotated per set
        x0 = codec.generate(1, n, 7).to("cuda").to(dt)
        xs = [torch.roll(x0, k * 4096) for k in range(R)]
    msgs = [torch.empty((1, lay.msg_stride), dtype=torch.uint8, device="cuda") for _ in range(R)]
    ys = [torch.empty(n, dtype=dt, device="cuda") for _ in range(R)]
    lib = _abi.lib()
    st = torch.cuda.Stream()
    sp = C.c_void_p(st.cuda_stream)
    dcode = _abi.DT_BF16 if dt == torch.bfloat16 else _abi.DT_F32
    esz = 2 if dt == torch.bfloat16 else 4

    def k1(i):
        _abi.check(lib.taco_compress_dev(C.byref(cfg), C.c_void_p(xs[i].data_ptr()), dcode, n, 1, 0, m,
                                         C.c_void_p(msgs[i].data_ptr()), lay.msg_stride, None, sp))

    def k2(i):
        _abi.check(lib.taco_decompress_dev(C.byref(cfg), C.c_void_p(msgs[i].data_ptr()), lay.msg_stride, 1, n, 0,
                                           m, C.c_void_p(ys[i].data_ptr()), dcode, None, sp))

    c = 1 + 8 / b

    def rt(i):
        k1(i)
        k2(i)

    kernels = [("k1_compress", k1, esz + c), ("k2_decompress", k2, c + esz)]
    if os.environ.get("RT"):
        kernels.append(("roundtrip", rt, 2 * (esz + c)))
    with torch.cuda.stream(st):
        for name, fn, bpe in kernels:
            for i in range(8):
                k1(i % R)
                fn(i % R)
            st.synchronize()
            # one event pair around REPS back-to-back launches: per-launch event stamps
            # are quantised (~2 us) on this part
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for i in range(reps):
                fn(i % R)
            e1.record(st)
            st.synchronize()
            ms = e0.elapsed_time(e1) / reps
            gbs = bpe * n / (ms * 1e-3) / 1e9
            print(f"{os.environ.get("TACO_B200_KERNELS", "r2")} {name} B={b} n={n} {dt} "
                  f"{ms * 1e3:.2f} us  {gbs:.0f} GB/s  frac={gbs / 6537.3:.3f}", flush=True)


if __name__ == "__main__":
    main()
