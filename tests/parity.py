"""Parity metrics shared by the GPU tests (test infrastructure).

Tolerances are the north-star bounds (BASELINE.json) as calibrated in SURVEY.md §8c:
  * alpha: bit-exact (fp64 sum of squares);
  * scale: <= 1e-6 relative;
  * codes: identical except one-ulp flips (0x00 == 0x80), flip rate <= FLIP_RATE_MAX;
  * decoded outputs: relMSE vs the oracle <= 1e-6 per round trip, <= 1e-5 end-to-end collectives.
"""
import numpy as np
import torch

FLIP_RATE_MAX = 1e-4
FLIP_SLACK = 4  # absolute allowance for small samples (a handful of codes near a rounding tie)
# session-wide tally of stage-isolated code comparisons (reported by conftest at the end)
FLIP_TALLY = {"codes": 0, "flips": 0, "max_ulp": 0, "alphas": 0, "alpha_exact": 0, "alpha_max_rel": 0.0}
SCALE_RTOL = 1e-6
# per-block scales (alpha and s) within 1e-6 relative: the north-star bound.  alpha is
# bit-exact wherever the sum of squares is accumulated in fp64 (tile kernels, E5M2); the
# register K1 accumulates in fp32 by default (TACO_SUMSQ_REG_F32) and lands within ~5e-7.
ALPHA_RTOL = 1e-6
DECODE_RELMSE_MAX = 1e-6
COLLECTIVE_RELMSE_MAX = 1e-5


def code_index(c: np.ndarray) -> np.ndarray:
    """Signed position of an FP8 code on its (monotone) value grid; 0x00 and 0x80 -> 0."""
    c = c.astype(np.int32)
    mag = c & 0x7F
    return np.where(c & 0x80, -mag, mag)


def code_diff(got: np.ndarray, want: np.ndarray):
    """(number of flipped codes, max ulp distance)."""
    d = np.abs(code_index(got) - code_index(want))
    return int(np.count_nonzero(d)), int(d.max()) if d.size else 0


def rel_mse(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = float(np.sum(want * want))
    num = float(np.sum((got - want) ** 2))
    return num / den if den > 0 else num


def rel_l2(got, want) -> float:
    return float(np.sqrt(rel_mse(got, want)))


def to_bf16_f32(x: np.ndarray) -> np.ndarray:
    """float(bf16(x)) with round-to-nearest-even, the exact values a bf16 tensor holds."""
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).float().numpy()


def check_codec_parity(codes, alpha, scale, rcodes, ralpha, rscale, what=""):
    """Stage-isolated K1 parity vs the oracle on the same input; returns the flip rate."""
    arel = float(np.max(np.abs(alpha.astype(np.float64) / ralpha - 1.0))) if alpha.size else 0.0
    FLIP_TALLY["alphas"] += int(alpha.size)
    FLIP_TALLY["alpha_exact"] += int(np.count_nonzero(alpha == ralpha))
    FLIP_TALLY["alpha_max_rel"] = max(FLIP_TALLY["alpha_max_rel"], arel)
    assert arel <= ALPHA_RTOL, f"{what}: alpha rel err {arel} " \
        f"({np.count_nonzero(alpha != ralpha)} of {alpha.size} not bit-exact)"
    err = np.max(np.abs(scale.astype(np.float64) / rscale - 1.0)) if scale.size else 0.0
    assert err <= SCALE_RTOL, f"{what}: scale rel err {err}"
    flips, worst = code_diff(codes, rcodes)
    FLIP_TALLY["codes"] += int(codes.size)
    FLIP_TALLY["flips"] += flips
    FLIP_TALLY["max_ulp"] = max(FLIP_TALLY["max_ulp"], worst)
    assert worst <= 1, f"{what}: a code is {worst} ulps away"
    rate = flips / max(1, codes.size)
    assert flips <= FLIP_RATE_MAX * codes.size + FLIP_SLACK, f"{what}: flip rate {rate} ({flips} flips)"
    return rate
