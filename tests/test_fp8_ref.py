"""Pins the vectorised fp8 restatement (tests/fp8_ref.py) to the C oracle on CPU."""
import numpy as np
import torch

import fp8_ref


def test_vectorised_encode_matches_oracle(port):
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2 ** 32, 60000, dtype=np.uint64).astype(np.uint32)
    specials = np.array([0, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0x00000001, 0x807FFFFF,
                         0x43E00000, 0x43E80000, 0x3B800000, 0x3A800000, 0x3B000000, 0x47600000],
                        np.uint32)
    # dense sweep around the fp8 grid (small exponents and ties)
    grid = (np.arange(-40000, 40000, dtype=np.int64) * 4096 + 0x3C000000).astype(np.uint32)
    x = np.concatenate([bits, specials, grid]).view(np.float32)
    for fmt in (0, 1):
        got = fp8_ref.encode(torch.from_numpy(x.copy()), fmt).numpy()
        want = np.array([port.encode(float(v), fmt) for v in x], np.uint8)
        assert np.array_equal(got, want)
