"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libtaco_ref.so).

Run here (where /root/reference exists and `make -C oracle` built _ref):

    python oracle/make_golden.py

The fixtures are small, committed, and travel to the GPU box; nothing on the
GPU side needs /root/reference.  Inputs come from the reference's own
generator (taco::generate / the tests' gaussian helper), so each fixture is
fully determined by (kind, n, seed).
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import E4M3, E5M2, Ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

# (name, kind 0=gaussian/1=mixture, n, seed, block_size, fmt)
CODEC_CASES = [
    ("gauss_4096_b256_e4m3", 0, 4096, 7, 256, E4M3),
    ("mix_4096_b256_e4m3", 1, 4096, 7, 256, E4M3),
    ("gauss_1000_b256_e4m3", 0, 1000, 3, 256, E4M3),      # ragged tail (232 valid)
    ("gauss_4096_b256_e5m2", 0, 4096, 13, 256, E5M2),
    ("gauss_2048_b32_e4m3", 0, 2048, 101, 32, E4M3),
    ("gauss_2048_b64_e4m3", 0, 2048, 102, 64, E4M3),
    ("gauss_2048_b128_e4m3", 0, 2048, 77, 128, E4M3),
    ("mix_4096_b512_e4m3", 1, 4096, 41, 512, E4M3),
    ("gauss_4096_b1024_e4m3", 0, 4096, 5, 1024, E4M3),
    ("gauss_8192_b4096_e4m3", 0, 8192, 6, 4096, E4M3),
    ("gauss_100_b2_e4m3", 0, 100, 8, 2, E4M3),
    ("gauss_17_b4_e5m2", 0, 17, 9, 4, E5M2),
    ("gauss_300_b16_e4m3", 0, 300, 10, 16, E4M3),
]

# (name, P, n, seed base, block_size, fmt)
AR_CASES = [
    ("ar_p2_n4096_b256", 2, 4096, 100, 256, E4M3),
    ("ar_p4_n4096_b256", 4, 4096, 17, 256, E4M3),
    ("ar_p8_n8192_b256", 8, 8192, 100, 256, E4M3),
    ("ar_p3_n1000_b32", 3, 1000, 31, 32, E4M3),
    ("ar_p4_n17_b4", 4, 17, 31, 4, E4M3),
    ("ar_p4_n6000_b512_e5m2", 4, 6000, 60, 512, E5M2),
]


def gaussian_ranks(ref: Ref, p, n, seed):
    return np.stack([ref.generate(0, n, seed + r) for r in range(p)])


def main() -> None:
    ref = Ref()
    ref.set_threads(1)
    os.makedirs(OUT, exist_ok=True)
    for name, kind, n, seed, b, fmt in CODEC_CASES:
        x = ref.generate(kind, n, seed)
        codes, alpha, scale = ref.compress(x, b, fmt)
        y = ref.decompress(codes, alpha, scale, n, b, fmt)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), x=x, codes=codes, alpha=alpha,
                            scale=scale, y=y, block_size=b, fmt=fmt, kind=kind, seed=seed)
    # the reference tests' hand-checked known answers (tests/test_codec.cpp:105-141)
    kat = np.array([3.0, 4.0, 0.0, 0.0], np.float32)
    c, a, s = ref.compress(kat, 4, E4M3)
    np.savez_compressed(os.path.join(OUT, "kat_b4.npz"), x=kat, codes=c, alpha=a, scale=s,
                        y=ref.decompress(c, a, s, 4, 4, E4M3), block_size=4, fmt=E4M3)
    for name, p, n, seed, b, fmt in AR_CASES:
        ins = gaussian_ranks(ref, p, n, seed)
        out = ref.allreduce(ins, b, fmt)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), inputs=ins, result=out["result"],
                            exact=out["exact"], steps=out["steps"],
                            bytes_on_wire=out["bytes_on_wire"], block_size=b, fmt=fmt)
    # archive bytes (src/serialize.cpp:109-124) for a ragged tensor
    x = ref.generate(0, 1000, 7)
    arc = np.frombuffer(ref.archive(x, 256, E4M3), np.uint8)
    np.savez_compressed(os.path.join(OUT, "archive_gauss_1000_b256.npz"), x=x, archive=arc)
    total = sum(os.path.getsize(os.path.join(OUT, f)) for f in os.listdir(OUT))
    print(f"wrote {len(os.listdir(OUT))} fixtures, {total} bytes, into {OUT}")


if __name__ == "__main__":
    main()
