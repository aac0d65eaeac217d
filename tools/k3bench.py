"""K3 (reduce-encode) timing at P ranks: N elements per rank, shard S = ceil(N/P); the P
messages of one shard (as received after the all-to-all) are reduced and re-encoded.
Algorithmic bytes per launch: (P + 1) * ceil(S/B) * (B + 8).  TACO_B200_LIB / B / N / PS env."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24088_b200 import _abi, codec  # noqa: E402


def main():
    b = int(os.environ.get("B", "256"))
    n = int(os.environ.get("N", str(8192 * 2560)))
    reps = int(os.environ.get("REPS", "100"))
    cfg = codec.make_config(b)
    lib = _abi.lib()
    st = torch.cuda.Stream()
    sp = C.c_void_p(st.cuda_stream)
    for P in [int(p) for p in os.environ.get("PS", "1 2 4 8").split()]:
        S = -(-n // P)
        m = -(-S // b)
        lay = _abi.msg_layout(cfg, m)
        R = 3
        recv = []
        for _ in range(R):
            x = (torch.randn(P * S, device="cuda") * 1e-3).to(torch.bfloat16)
            recv.append(codec.compress(x, cfg, shards=P))  # [P, stride]: "rank r's copy of my shard"
        outs = [torch.empty(lay.msg_stride, dtype=torch.uint8, device="cuda") for _ in range(R)]

        def k3(i):
            _abi.check(lib.taco_reduce_encode_dev(C.byref(cfg), C.c_void_p(recv[i].data_ptr()), lay.msg_stride, P, S,
                                                  0, m, C.c_void_p(outs[i].data_ptr()), None, 0, None, sp))

        with torch.cuda.stream(st):
            for i in range(5):
                k3(i % R)
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for i in range(reps):
                k3(i % R)
            e1.record(st)
            st.synchronize()
        ms = e0.elapsed_time(e1) / reps
        byts = (P + 1) * m * (b + 8)
        gbs = byts / (ms * 1e-3) / 1e9
        print(f"k3 P={P} B={b} n={n} S={S} {ms * 1e3:.2f} us  {gbs:.0f} GB/s  frac={gbs / 6555.2:.3f}", flush=True)


if __name__ == "__main__":
    main()
