"""Pins the C restatement (oracle/taco_oracle.c) before anything is checked against it.

Anchors, in order of authority:
  * the reference tests' known answers (proj/tests/test_fp8.cpp, test_transform.cpp,
    test_codec.cpp, test_collective.cpp, acceptance.cpp),
  * golden fixtures produced by the reference itself (tests/golden, oracle/make_golden.py),
  * the reference library run live in this process when oracle/_ref is built.
"""
import math

import numpy as np
import pytest

from conftest import golden, golden_names
from oracle.oracle import E4M3, E5M2, OracleError


def rel_l2(y, x):
    x = x.astype(np.float64)
    return math.sqrt(((y.astype(np.float64) - x) ** 2).sum() / (x ** 2).sum())


# ---- fp8 (proj/tests/test_fp8.cpp) -------------------------------------------------------

def test_pinned_codes(port):
    # test_fp8.cpp:99-116
    assert port.encode(0.0) == 0x00
    assert port.encode(-0.0) == 0x80
    assert port.encode(1.0) == 0x38
    assert port.encode(448.0) == 0x7E
    assert port.encode(500.0) == 0x7E
    assert port.encode(-500.0) == 0xFE
    assert port.encode(1.0, E5M2) == 0x3C
    assert port.encode(70000.0, E5M2) == 0x7B
    assert port.encode(float("nan")) == 0x7F
    t4 = port.decode_table(E4M3)
    assert t4[0x38] == 1.0 and t4[0x01] == 2.0 ** -9 and t4[0x7E] == 448.0
    assert port.decode_table(E5M2)[0x7B] == 57344.0


def _bit_layout_value(code, ebits, mbits, bias):
    s = -1.0 if code & 0x80 else 1.0
    e = (code >> mbits) & ((1 << ebits) - 1)
    f = code & ((1 << mbits) - 1)
    if e == 0:
        return s * f * 2.0 ** (1 - bias - mbits)
    return s * (1 + f / 2 ** mbits) * 2.0 ** (e - bias)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_decode_all_codes(port, fmt):
    # test_fp8.cpp:66-90: finite codes decode to the bit-layout value, the rest are NaN/inf
    ebits, mbits, bias = (4, 3, 7) if fmt == E4M3 else (5, 2, 15)
    t = port.decode_table(fmt)
    finite = 0
    for c in range(256):
        e = (c >> mbits) & ((1 << ebits) - 1)
        special = (fmt == E4M3 and (c & 0x7F) == 0x7F) or (fmt == E5M2 and e == 31)
        if special:
            if fmt == E5M2 and (c & 0x7F) == 0x7C:
                assert math.isinf(t[c])
            else:
                assert math.isnan(t[c])
            continue
        finite += 1
        assert t[c] == np.float32(_bit_layout_value(c, ebits, mbits, bias))
        assert math.copysign(1, t[c]) == (-1 if c & 0x80 else 1)
        assert port.encode(float(t[c]), fmt) == c  # exhaustive round trip, :118-126
    assert finite == (254 if fmt == E4M3 else 248)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_encode_is_nearest_ties_even(port, fmt):
    # test_fp8.cpp:128-153 (sampled): brute-force nearest representable, ties to even code
    t = port.decode_table(fmt).astype(np.float64)
    fin = np.array([c for c in range(256) if np.isfinite(t[c])])
    vals = t[fin]
    rng = np.random.default_rng(2024)
    q = 448.0 if fmt == E4M3 else 57344.0
    xs = np.concatenate([rng.uniform(-q, q, 3000), rng.normal(size=3000),
                         rng.normal(size=3000) * 1e-3,
                         np.ldexp(rng.integers(0, 4096, 3000).astype(np.float64),
                                  rng.integers(-16, 8, 3000))]).astype(np.float32)
    for x in xs:
        got = t[port.encode(float(x), fmt)]
        d = np.abs(vals - np.float64(x))
        best = d.min()
        cands = fin[d == best]
        # ties: even mantissa (lowest code bit 0)
        want_codes = [c for c in cands if c & 1 == 0] or list(cands)
        assert any(got == t[c] for c in want_codes), (x, got)


def test_port_encode_equals_reference_exhaustive_sample(port, ref):
    rng = np.random.default_rng(5)
    bits = rng.integers(0, 2 ** 32, 200000, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    for fmt in (E4M3, E5M2):
        for x in xs[:20000]:
            assert port.encode(float(x), fmt) == ref.encode(float(x), fmt)


# ---- transform (proj/tests/test_transform.cpp) -------------------------------------------

def test_fwht_pinned_vectors(port):
    # test_transform.cpp:112-142
    np.testing.assert_allclose(port.fwht([1, 1, 1, 1]), [2, 0, 0, 0], atol=1e-7)
    np.testing.assert_allclose(port.fwht([1, 0, 0, 0]), [0.5] * 4, rtol=1e-7)
    np.testing.assert_allclose(port.fwht([3, 1]), [2 * math.sqrt(2), math.sqrt(2)], rtol=1e-7)
    np.testing.assert_allclose(port.fwht([2, 0, 0, 0]), [1] * 4, rtol=1e-7)
    # natural (Sylvester) order: [1.2,1.6,0,0]*... -> test_codec.cpp:113 [1.4,-0.2,1.4,-0.2]
    np.testing.assert_allclose(port.fwht([1.2, 1.6, 0, 0]), [1.4, -0.2, 1.4, -0.2], atol=1e-12)
    with pytest.raises(OracleError):
        port.fwht(np.ones(6))


@pytest.mark.parametrize("b", [2, 4, 8, 16, 32, 64])
def test_fwht_matches_sylvester_matrix(port, b):
    # test_transform.cpp:151-163
    h = np.array([[1.0]])
    while h.shape[0] < b:
        h = np.block([[h, h], [h, -h]])
    v = np.random.default_rng(b).normal(size=b)
    np.testing.assert_allclose(port.fwht(v), h @ v / math.sqrt(b), atol=1e-12)


# ---- codec (proj/tests/test_codec.cpp, acceptance.cpp) ------------------------------------

def test_kat_single_block(port):
    # test_codec.cpp:105-127
    codes, a, s = port.compress([3, 4, 0, 0], 4)
    assert a[0] == np.float32(0.4)
    assert abs(s[0] / (1.4 / 448.0) - 1) < 1e-6
    assert list(codes) == [0x7E, 0xE8, 0x7E, 0xE8]
    y = port.decompress(codes, a, s, 4, 4)
    assert abs(y[0] - 3) < 3e-6 and abs(y[1] - 4) < 4e-6 and y[2] == 0 and y[3] == 0
    g = golden("kat_b4")
    assert np.array_equal(codes, g["codes"]) and np.array_equal(y, g["y"])


def test_all_zero_tensor(port):
    # test_codec.cpp:129-141
    codes, a, s = port.compress(np.zeros(1000, np.float32), 256)
    assert len(a) == 4 and np.all(s == 1.0) and np.all(codes == 0)
    assert np.allclose(a, 1e6, rtol=1e-6)
    assert np.all(port.decompress(codes, a, s, 1000, 256) == 0)


@pytest.mark.parametrize("name", golden_names("gauss_") + golden_names("mix_"))
def test_port_matches_reference_fixture_bitwise(port, name):
    g = golden(name)
    b, fmt = int(g["block_size"]), int(g["fmt"])
    codes, a, s = port.compress(g["x"], b, fmt)
    assert np.array_equal(codes, g["codes"])
    assert np.array_equal(a, g["alpha"]) and np.array_equal(s, g["scale"])
    y = port.decompress(codes, a, s, g["x"].size, b, fmt)
    assert np.array_equal(y, g["y"])


def test_acceptance_round_trip_numbers(port):
    # acceptance.cpp:268-285 / README: 0.026104 (gaussian) and 0.022047 (mixture)
    x = port.gaussian(1_000_000, 7)
    m = port.mixture(1_000_000, 7)
    assert round(rel_l2(port.decompress(*port.compress(x), x.size), x), 6) == 0.026104
    assert round(rel_l2(port.decompress(*port.compress(m), m.size), m), 6) == 0.022047


def test_validation_messages(port):
    # test_codec.cpp:318-349
    cases = [(dict(block_size=100), "block size must be a power of two"),
             (dict(block_size=1), "block size must be between 2 and 32768"),
             (dict(tau=0.0), "target energy must be positive and finite"),
             (dict(eps=0.0), "stability epsilon must be positive and finite")]
    for kw, msg in cases:
        with pytest.raises(OracleError, match=msg) as ei:
            port.compress([1.0], **kw)
        assert ei.value.code == "config"
    with pytest.raises(OracleError, match="input tensor is empty"):
        port.compress(np.zeros(0, np.float32))
    with pytest.raises(OracleError, match="input tensor contains NaN or Inf"):
        port.compress([1.0, float("nan")])
    with pytest.raises(OracleError, match="block scalars must be finite and nonzero"):
        port.decompress(np.zeros(256, np.uint8), [float("nan")], [1.0], 256)


# ---- collective (proj/tests/test_collective.cpp, acceptance.cpp crit 7) -------------------

@pytest.mark.parametrize("name", golden_names("ar_"))
def test_port_twoshot_matches_reference_fixture(port, name):
    g = golden(name)
    out = port.allreduce_twoshot(g["inputs"], int(g["block_size"]), int(g["fmt"]))
    assert np.array_equal(out["result"], g["result"])
    assert np.array_equal(out["exact"], g["exact"])
    assert out["bytes_on_wire"] == int(g["bytes_on_wire"])


def test_twoshot_is_stage1_then_one_round_trip(port):
    # test_collective.cpp:123-163, restated: result == round trip of the fp32 stage-1 sums
    p, n = 4, 4096
    ins = np.stack([port.gaussian(n, 17 + r) for r in range(p)])
    out = port.allreduce_twoshot(ins, want_stage1=True)
    shard = n // p
    stage1 = np.zeros(n, np.float32)
    for s in range(p):
        acc = None
        for r in range(p):
            piece = ins[r, s * shard:(s + 1) * shard]
            rt = port.decompress(*port.compress(piece), shard)
            acc = rt.copy() if acc is None else (acc + rt).astype(np.float32)
        stage1[s * shard:(s + 1) * shard] = acc
    assert np.array_equal(stage1, out["stage1"])
    stage2 = np.concatenate([port.decompress(*port.compress(stage1[s * shard:(s + 1) * shard]),
                                             shard) for s in range(p)])
    assert np.array_equal(out["result"], stage2)


def test_twoshot_error_bound_p8(port):
    # acceptance.cpp:378-394: rel L2 0.036864 <= 2 x single round trip (0.026082)
    p, n = 8, 1 << 20
    ins = np.stack([port.gaussian(n, 100 + r) for r in range(p)])
    out = port.allreduce_twoshot(ins)
    single = rel_l2(port.decompress(*port.compress(out["exact"]), n), out["exact"])
    ts = rel_l2(out["result"], out["exact"])
    assert round(ts, 6) == 0.036864 and round(single, 6) == 0.026082
    assert ts <= 2 * single


def test_wire_bytes_and_archive_size(port, ref):
    # test_collective.cpp:207-223, acceptance.cpp:409-427 (1,031,470 bytes for 10^6)
    assert ref.archive_size(1_000_000) == 1_031_470
    ins = np.stack([port.gaussian(1024, 23 + r) for r in range(4)])
    assert port.allreduce_twoshot(ins)["bytes_on_wire"] == 2 * 4 * 3 * ref.archive_size(256)


def test_live_reference_agrees_with_port(port, ref):
    x = ref.generate(1, 50_000, 99)
    for b in (32, 256, 2048):
        rc, ra, rs = ref.compress(x, b)
        pc, pa, ps = port.compress(x, b)
        assert np.array_equal(rc, pc) and np.array_equal(ra, pa) and np.array_equal(rs, ps)
