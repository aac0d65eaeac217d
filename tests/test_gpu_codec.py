"""GPU parity of K1 (compress) and K2 (decompress) against the oracle, through the C ABI.

Small cases run the oracle on the same inputs; config-size cases (BASELINE configs[1],
[8192 x 2560] bf16) check a slice against the oracle and the whole tensor through
size-independent properties (round-trip error, determinism, chunk / shard decomposition,
power-of-two invariance)."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

from conftest import golden, golden_names
from parity import (COLLECTIVE_RELMSE_MAX, DECODE_RELMSE_MAX, check_codec_parity, code_diff, rel_l2, rel_mse,
                    to_bf16_f32)

pytestmark = pytest.mark.gpu

cuda = pytest.importorskip("torch").cuda
if not cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2604_24088_b200 import _abi, codec  # noqa: E402
from paper_2604_24088_b200._abi import TacoError, make_config  # noqa: E402

DEV = "cuda"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpu_compress(x: np.ndarray, b=256, fmt=0, dtype=torch.float32, **kw):
    cfg = make_config(b, fmt)
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(DEV).to(dtype)
    flags = codec.Flags()
    msg = codec.compress(xd, cfg, flags=flags, **kw)
    torch.cuda.synchronize()
    flags.check()
    m = -(-x.size // b)
    codes, al, sc = codec.split_message(msg[0], cfg, m)
    return msg, codes.cpu().numpy(), al.cpu().numpy(), sc.cpu().numpy()


def gpu_decompress(msg, n, b=256, fmt=0, out_dtype=torch.float32):
    cfg = make_config(b, fmt)
    flags = codec.Flags()
    y = codec.decompress(msg, n, cfg, out_dtype=out_dtype, flags=flags)
    torch.cuda.synchronize()
    flags.check()
    return y.float().cpu().numpy()


def message_from(codes, alpha, scale, b=256, fmt=0):
    cfg = make_config(b, fmt)
    m = alpha.size
    lay = _abi.msg_layout(cfg, m)
    buf = np.zeros(lay.msg_stride, np.uint8)
    buf[: m * b] = codes
    buf[lay.scal_offset: lay.scal_offset + 8 * m] = np.stack([alpha, scale], 1).astype(np.float32).view(
        np.uint8).ravel()
    return torch.from_numpy(buf).to(DEV).view(1, -1)


# --------------------------------------------------------------------- fp8 instructions ---
@pytest.mark.parametrize("fmt", [0, 1])
def test_device_fp8_cvt_equals_reference_encode_exhaustive(fmt):
    """cvt.rn.satfinite == fp8_encode (fp8.cpp:66-91) for every one of the 2^32 fp32 patterns."""
    import fp8_ref
    lib = _abi.lib()
    chunk = 1 << 28
    out = torch.empty(chunk, dtype=torch.uint8, device=DEV)
    for start in range(0, 1 << 32, chunk):
        bits = torch.arange(start, start + chunk, dtype=torch.int64, device=DEV)
        x = (bits - (1 << 32) * (bits >= (1 << 31))).to(torch.int32).view(torch.float32)
        _abi.check(lib.taco_fp8_encode_dev(C.c_void_p(x.data_ptr()), chunk, fmt, C.c_void_p(out.data_ptr()),
                                           None))
        want = fp8_ref.encode(x, fmt)
        finite = torch.isfinite(x)
        bad = ((out != want) & finite).sum().item()
        assert bad == 0, f"chunk {start:#x}: {bad} mismatches"
        # +-inf saturate like |x| > q_max
        inf_ok = ((out == want) | ~torch.isinf(x)).all().item()
        assert inf_ok
        del bits, x, want, finite


@pytest.mark.parametrize("fmt", [0, 1])
def test_device_fp8_decode_equals_reference_table(port, fmt):
    codes = torch.arange(256, dtype=torch.uint8, device=DEV)
    out = torch.empty(256, dtype=torch.float32, device=DEV)
    _abi.check(_abi.lib().taco_fp8_decode_dev(C.c_void_p(codes.data_ptr()), 256, fmt, C.c_void_p(out.data_ptr()),
                                              None))
    got, want = out.cpu().numpy(), port.decode_table(fmt)
    fin = np.isfinite(want)
    assert np.array_equal(got[fin], want[fin])
    assert np.array_equal(np.signbit(got[fin]), np.signbit(want[fin]))


# ------------------------------------------------------------------------ golden / KAT ---
def test_kat_single_block():
    # test_codec.cpp:105-127: [3,4,0,0], B=4 -> alpha 0.4f, s = 1.4/448, codes 7E E8 7E E8
    g = golden("kat_b4")
    msg, codes, al, sc = gpu_compress(g["x"], 4)
    assert list(codes) == [0x7E, 0xE8, 0x7E, 0xE8]
    assert al[0] == np.float32(0.4) and abs(sc[0] / (1.4 / 448) - 1) < 1e-6
    y = gpu_decompress(msg, 4, 4)
    assert abs(y[0] - 3) < 3e-6 and abs(y[1] - 4) < 4e-6 and y[2] == 0 and y[3] == 0


def test_all_zero_tensor():
    # test_codec.cpp:129-141
    msg, codes, al, sc = gpu_compress(np.zeros(1000, np.float32))
    assert np.all(sc == 1.0) and np.all(codes == 0) and np.allclose(al, 1e6, rtol=1e-6)
    assert np.all(gpu_decompress(msg, 1000) == 0.0)


@pytest.mark.parametrize("name", golden_names("gauss_") + golden_names("mix_"))
def test_compress_matches_reference_fixture(name):
    g = golden(name)
    b, fmt = int(g["block_size"]), int(g["fmt"])
    msg, codes, al, sc = gpu_compress(g["x"], b, fmt)
    check_codec_parity(codes, al, sc, g["codes"], g["alpha"], g["scale"], name)
    # stage-isolated K2: decode the REFERENCE's message
    y = gpu_decompress(message_from(g["codes"], g["alpha"], g["scale"], b, fmt), g["x"].size, b, fmt)
    assert rel_mse(y, g["y"]) <= DECODE_RELMSE_MAX
    ulp = np.abs(y.view(np.int32).astype(np.int64) - g["y"].view(np.int32).astype(np.int64))
    assert np.percentile(ulp, 99) <= 2, f"decode ulp p99 {np.percentile(ulp, 99)}"


@pytest.mark.parametrize("b", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768])
@pytest.mark.parametrize("fmt", [0, 1])
def test_every_block_size_against_port(port, b, fmt):
    n = max(3 * b + b // 2 + 1, 4099)  # ragged tail
    x = port.mixture(n, 1000 + b, tail_fraction=0.05)
    msg, codes, al, sc = gpu_compress(x, b, fmt)
    rc, ra, rs = port.compress(x, b, fmt)
    check_codec_parity(codes, al, sc, rc, ra, rs, f"B={b}")
    y = gpu_decompress(msg, n, b, fmt)
    assert rel_mse(y, port.decompress(codes, al, sc, n, b, fmt)) <= DECODE_RELMSE_MAX


@pytest.mark.parametrize("b", [32, 256, 512])
def test_bf16_input_and_output(port, b):
    x = to_bf16_f32(port.gaussian(50_000, 3 + b))
    msg, codes, al, sc = gpu_compress(x, b, dtype=torch.bfloat16)
    rc, ra, rs = port.compress(x, b)
    check_codec_parity(codes, al, sc, rc, ra, rs, "bf16")
    y = gpu_decompress(msg, x.size, b, out_dtype=torch.bfloat16)
    want = to_bf16_f32(port.decompress(codes, al, sc, x.size, b))
    # bf16 rounding of an fp32 value within ~1 ulp of the oracle: differs by <= 1 bf16 ulp
    assert rel_mse(y, want) <= 1e-5


def test_scale_invariance_power_of_two(port):
    # test_codec.cpp:217-234: payload and s identical, alpha*c == alpha0
    x = port.gaussian(128 * 64, 77)
    _, c0, a0, s0 = gpu_compress(x, 128)
    for c in (2.0, 0.5, 1024.0):
        _, c1, a1, s1 = gpu_compress(x * np.float32(c), 128)
        assert np.array_equal(c1, c0) and np.array_equal(s1, s0)
        assert np.allclose(a1 * c, a0, rtol=1e-6)


def test_extreme_ranges_no_nan_codes(port):
    # test_codec.cpp:195-215 (10^6 blocks of B=32 over sigma 1e-6..3e5, both formats)
    for s, sigma in enumerate([1.0, 100.0, 1e-4, 1e4, 0.01, 1.0, 3e5, 1e-6]):
        fmt = s % 2
        x = port.gaussian(32 * 125_000, 1000 + s, sigma)
        _, codes, al, sc = gpu_compress(x, 32, fmt)
        table = port.decode_table(fmt)
        v = table[codes]
        assert np.all(np.isfinite(v)) and np.all(np.abs(v) <= (448 if fmt == 0 else 57344))
        rc, ra, rs = port.compress(x[: 32 * 4000], 32, fmt)
        check_codec_parity(codes[: 32 * 4000], al[:4000], sc[:4000], rc, ra, rs, f"sigma={sigma}")


def test_huge_and_tiny_magnitudes(port):
    x = np.concatenate([port.gaussian(512, 1, 1e36), port.gaussian(512, 2, 1e-40),
                        np.float32([3e38, -3e38] * 128), np.float32([1e-45] * 256)]).astype(np.float32)
    msg, codes, al, sc = gpu_compress(x, 256)
    rc, ra, rs = port.compress(x, 256)
    assert np.max(np.abs(al.astype(np.float64) / ra - 1)) <= 1e-6
    assert np.max(np.abs(sc / rs - 1)) <= 1e-6
    assert code_diff(codes, rc)[1] <= 1


# ------------------------------------------------------------------------------ errors ---
def test_nan_and_inf_raise_input_error():
    for bad in (float("nan"), float("inf"), -float("inf")):
        x = np.ones(1000, np.float32)
        x[777] = bad
        with pytest.raises(TacoError, match="input tensor contains NaN or Inf") as ei:
            gpu_compress(x)
        assert ei.value.code == "input"


def test_bad_scalars_raise_corrupt():
    x = np.random.default_rng(0).normal(size=1000).astype(np.float32)
    msg, codes, al, sc = gpu_compress(x)
    for a, s in ((np.nan, 1.0), (1.0, 0.0), (0.0, 1.0), (np.inf, 1.0)):
        al2, sc2 = al.copy(), sc.copy()
        al2[1], sc2[1] = a, s
        with pytest.raises(TacoError, match="block scalars must be finite and nonzero") as ei:
            gpu_decompress(message_from(codes, al2, sc2), 1000)
        assert ei.value.code == "corrupt"


# ------------------------------------------------------------- tensor-core K1 ---
def _tc_k1_parity(port):
    n = 256 * (128 * 7 + 50)
    x = port.mixture(n, 11).astype(np.float32)
    x[256 * 5: 256 * 6] = 0.0
    x[256 * 9: 256 * 10] = np.where(x[256 * 9: 256 * 10] >= 0, 1e37, -1e37)
    x[256 * 11: 256 * 12] *= np.float32(1e-38)
    x = to_bf16_f32(x)
    msg, codes, al, sc = gpu_compress(x, 256, dtype=torch.bfloat16)
    rc, ra, rs = port.compress(x, 256)
    check_codec_parity(codes, al, sc, rc, ra, rs, "bf16 B=256 K1")
    # chunks of blocks and block-aligned shards reproduce the whole-tensor message
    cfg = make_config(256)
    xd = torch.from_numpy(x).to(DEV).to(torch.bfloat16)
    m = n // 256
    for b0, b1 in ((0, 128), (77, 700), (128 * 3, m)):
        part = codec.compress(xd, cfg, blk=(b0, b1))
        pc, pa, ps = (t.cpu().numpy() for t in codec.split_message(part[0], cfg, b1 - b0))
        assert np.array_equal(pc, codes[b0 * 256: b1 * 256])
        assert np.array_equal(pa, al[b0:b1]) and np.array_equal(ps, sc[b0:b1])
    sh = codec.compress(xd, cfg, shards=2)
    for i in range(2):
        one = codec.compress(xd[i * n // 2:(i + 1) * n // 2].contiguous(), cfg)
        lay = _abi.msg_layout(cfg, m // 2)
        assert torch.equal(sh[i, : lay.msg_bytes], one[0, : lay.msg_bytes])
    x = np.ones(256 * 256, np.float32)
    x[1000] = float("nan")
    with pytest.raises(TacoError, match="input tensor contains NaN or Inf"):
        gpu_compress(x, 256, dtype=torch.bfloat16)


def test_bf16_b256_k1_parity(port):
    """bf16, B = 256, block-aligned (the config shape): full and partial 128-block tiles,
    an all-zero block, an fp32-overflowing block, bf16 subnormals -- default kernels."""
    _tc_k1_parity(port)


def test_tensor_core_k1_parity_subprocess():
    """The same checks with K1 on tcgen05 (TACO_B200_KERNELS=tc is read once per process,
    so it runs in a child interpreter)."""
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = ['tests', '.']; import pytest; "
            "sys.exit(pytest.main(['-q', '-x', '-p', 'no:cacheprovider', 'tests/test_gpu_codec.py', "
            "'-k', 'bf16_b256_k1_parity or config_size']))")
    env = dict(os.environ, TACO_B200_KERNELS="tc")
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


# ------------------------------------------------------------ config-size properties ---
@pytest.fixture(scope="module")
def big_input(port):
    n = 8192 * 2560  # BASELINE configs[1] tensor
    return port.mixture(n, 7).reshape(-1)


def test_config_size_slice_parity_and_roundtrip(port, big_input):
    x = to_bf16_f32(big_input)
    msg, codes, al, sc = gpu_compress(x, 256, dtype=torch.bfloat16)
    k = 1 << 20
    rc, ra, rs = port.compress(x[:k], 256)
    check_codec_parity(codes[:k], al[: k // 256], sc[: k // 256], rc, ra, rs, "cfg2 slice")
    tail = x[-k:]
    rc, ra, rs = port.compress(tail, 256)
    check_codec_parity(codes[-k:], al[-k // 256:], sc[-k // 256:], rc, ra, rs, "cfg2 tail")
    y = gpu_decompress(msg, x.size, 256)
    assert 0.015 < rel_l2(y, x) < 0.03  # the reference's mixture round trip is 0.0220 at 10^6
    y2 = gpu_decompress(msg, x.size, 256)
    assert np.array_equal(y, y2)  # determinism


def test_chunks_and_shards_are_bit_identical(port, big_input):
    x = big_input[: 3 * 1024 * 1024 + 4096]
    cfg = make_config(256)
    xd = torch.from_numpy(x).to(DEV)
    whole = codec.compress(xd, cfg)
    m = -(-x.size // 256)
    wc, wa, ws = (t.cpu().numpy() for t in codec.split_message(whole[0], cfg, m))
    # chunked compress: concatenated chunk messages == whole message (test_collective.cpp:225-238)
    bounds = [0, 1000, 5000, 7777, m]
    for b0, b1 in zip(bounds, bounds[1:]):
        part = codec.compress(xd, cfg, blk=(b0, b1))
        pc, pa, ps = (t.cpu().numpy() for t in codec.split_message(part[0], cfg, b1 - b0))
        assert np.array_equal(pc, wc[b0 * 256: b1 * 256])
        assert np.array_equal(pa, wa[b0:b1]) and np.array_equal(ps, ws[b0:b1])
    # shards: message p == compress of the zero-padded slice p (collective.cpp:82-88)
    for p in (2, 3, 8):
        sh = codec.compress(xd, cfg, shards=p)
        S = -(-x.size // p)
        ms = -(-S // 256)
        for i in range(p):
            sl = np.zeros(S, np.float32)
            seg = x[i * S:(i + 1) * S]
            sl[: seg.size] = seg
            one = codec.compress(torch.from_numpy(sl).to(DEV), cfg)
            assert torch.equal(sh[i, : _abi.msg_layout(cfg, ms).msg_bytes], one[0, : _abi.msg_layout(cfg, ms).msg_bytes])
        y = codec.decompress(sh, x.size, cfg, shards=p)
        want = np.concatenate([codec.decompress(sh[i:i + 1], S, cfg).cpu().numpy() for i in range(p)])[: x.size]
        assert np.array_equal(y.cpu().numpy(), want)


# --------------------------------------------------------------------------- host API ---
def test_host_api_matches_device_path(port):
    x = port.gaussian(3_000_000 + 77, 5)
    cfg = make_config(256)
    hc = codec.HostContext(0)
    msg_h = hc.compress(torch.from_numpy(x), cfg)
    msg_d, *_ = gpu_compress(x)
    lay = _abi.msg_layout(cfg, -(-x.size // 256))
    assert np.array_equal(msg_h.numpy(), msg_d[0, : lay.msg_bytes].cpu().numpy())
    y_h = hc.decompress(msg_h, x.size, cfg).numpy()
    y_d = gpu_decompress(msg_d, x.size)
    assert np.array_equal(y_h, y_d)
    out = torch.empty(x.size, dtype=torch.float32)
    hc.roundtrip(torch.from_numpy(x), cfg, out)
    assert np.array_equal(out.numpy(), y_d)
    pinned_in = torch.from_numpy(x).pin_memory()
    pinned_out = torch.empty(x.size, dtype=torch.float32).pin_memory()
    hc.roundtrip(pinned_in, cfg, pinned_out)
    assert np.array_equal(pinned_out.numpy(), y_d)
    bad = x.copy()
    bad[2_999_999] = np.nan
    with pytest.raises(TacoError, match="NaN or Inf"):
        hc.compress(torch.from_numpy(bad), cfg)
    hc.close()


def test_host_api_ramped_chunk_schedule(port):
    """A tensor of > 4 pipeline chunks takes the ramped schedule (cb/8, cb/4, cb/2, cb ...,
    cb/2, cb/4, cb/8 blocks): results identical to one device call, pinned or not."""
    n = 9_000_000 + 123  # 36 MB of fp32: 4.3 chunks of 8 MiB
    x = port.gaussian(n, 8)
    cfg = make_config(256)
    hc = codec.HostContext(0)
    xd = torch.from_numpy(x).cuda()
    msg_d = codec.compress(xd, cfg)
    y_d = codec.decompress(msg_d, n, cfg).cpu().numpy()
    lay = _abi.msg_layout(cfg, -(-n // 256))
    msg_h = hc.compress(torch.from_numpy(x), cfg)
    assert np.array_equal(msg_h.numpy(), msg_d[0, : lay.msg_bytes].cpu().numpy())
    assert np.array_equal(hc.decompress(msg_h, n, cfg).numpy(), y_d)
    for pin in (False, True):
        xi = torch.from_numpy(x)
        out = torch.empty(n, dtype=torch.float32)
        if pin:
            xi, out = xi.pin_memory(), out.pin_memory()
        hc.roundtrip(xi, cfg, out)
        assert np.array_equal(out.numpy(), y_d), f"pinned={pin}"
    hc.close()


# ------------------------------------------------------------------- allreduce (1 GPU) ---
@pytest.mark.parametrize("name", golden_names("ar_"))
def test_allreduce_sim_matches_reference_fixture(port, name):
    g = golden(name)
    b, fmt = int(g["block_size"]), int(g["fmt"])
    cfg = make_config(b, fmt)
    ins = torch.from_numpy(g["inputs"]).to(DEV)
    p, n = g["inputs"].shape
    S = -(-n // p)
    st = torch.zeros(p * S, dtype=torch.float32, device=DEV)
    flags = codec.Flags()
    out = codec.allreduce_sim(ins, cfg, stage1=st, flags=flags)
    torch.cuda.synchronize()
    flags.check()
    got = out.cpu().numpy()
    assert rel_mse(got, g["result"]) <= COLLECTIVE_RELMSE_MAX
    # stage-isolated: the GPU's stage-1 sums vs the oracle's
    ref = port.allreduce_twoshot(g["inputs"], b, fmt, want_stage1=True)
    assert rel_mse(st.cpu().numpy(), ref["stage1"]) <= DECODE_RELMSE_MAX
    # and the error bound of test_collective.cpp:105-121
    single = rel_l2(port.decompress(*port.compress(g["exact"], b, fmt), n, b, fmt), g["exact"])
    assert rel_l2(got, g["exact"]) <= 2 * single + 1e-6


def test_reduce_encode_stage_isolated(port):
    """K3 on the REFERENCE's phase-1 messages: stage-1 sum vs the oracle's, re-encode vs the
    oracle's compress of the GPU's own sum."""
    p, S, b = 4, 65536, 256
    cfg = make_config(b)
    ins = np.stack([port.mixture(S, 40 + r) for r in range(p)])
    lay = _abi.msg_layout(cfg, S // b)
    msgs = torch.zeros(p, lay.msg_stride, dtype=torch.uint8, device=DEV)
    dec = []
    for r in range(p):
        c, a, s = port.compress(ins[r], b)
        msgs[r] = message_from(c, a, s, b)[0]
        dec.append(port.decompress(c, a, s, S, b))
    want_acc = dec[0].copy()
    for r in range(1, p):
        want_acc = (want_acc + dec[r]).astype(np.float32)
    out = torch.zeros(lay.msg_stride, dtype=torch.uint8, device=DEV)
    acc = torch.zeros(S, dtype=torch.float32, device=DEV)
    codec.reduce_encode(msgs, p, S, cfg, lay.msg_stride, out, acc_out=acc)
    torch.cuda.synchronize()
    acc_h = acc.cpu().numpy()
    assert rel_mse(acc_h, want_acc) <= 1e-10
    codes, al, sc = (t.cpu().numpy() for t in codec.split_message(out, cfg, S // b))
    rc, ra, rs = port.compress(acc_h, b)
    check_codec_parity(codes, al, sc, rc, ra, rs, "K3 re-encode")


def test_allreduce_config_size_p2(port, big_input):
    """BASELINE configs[1] shape (TP=2, [8192 x 2560] per rank) through the one-device schedule."""
    n = big_input.size
    x0 = to_bf16_f32(big_input)
    x1 = to_bf16_f32(port.mixture(n, 8))
    ins = torch.from_numpy(np.stack([x0, x1])).to(DEV).to(torch.bfloat16)
    cfg = make_config(256)
    out = codec.allreduce_sim(ins, cfg, out_dtype=torch.float32).cpu().numpy()
    exact = (x0 + x1).astype(np.float32)
    e = rel_l2(out, exact)
    assert 0.015 < e < 0.045, e
    # a 2^20-element window against the oracle's own two-shot (shard-aligned, so identical schedule)
    k = 1 << 20
    sub = np.stack([np.concatenate([x0[:k // 2], x0[n // 2: n // 2 + k // 2]]),
                    np.concatenate([x1[:k // 2], x1[n // 2: n // 2 + k // 2]])])
    ref = port.allreduce_twoshot(sub)["result"]
    got = np.concatenate([out[:k // 2], out[n // 2: n // 2 + k // 2]])
    assert rel_mse(got, ref) <= COLLECTIVE_RELMSE_MAX


@pytest.mark.parametrize("dtype,b", [(torch.bfloat16, 256), (torch.float32, 256), (torch.bfloat16, 64)])
def test_dependent_launch_chain_matches_synchronised_chain(port, dtype, b):
    """K1/K2/K3 are launched with programmatic dependent launch (prologue overlaps the
    previous kernel): a chain in which every launch reads the previous launch's output,
    enqueued back to back, must equal the same chain with a host synchronise after every
    launch (where no overlap is possible)."""
    cfg = make_config(b)
    n = 8192 * 96 + 77
    x0 = torch.from_numpy(port.mixture(n, 17)).cuda().to(dtype)

    S = -(-n // 2)
    mb = _abi.msg_layout(cfg, -(-S // b)).msg_bytes  # bytes past msg_bytes are stride padding

    def chain(sync):
        y = x0
        outs = []
        for _ in range(6):
            m = codec.compress(y, cfg, shards=2)
            if sync:
                torch.cuda.synchronize()
            red = torch.empty_like(m[0])
            codec.reduce_encode(m, 2, S, cfg, m.shape[1], red)
            if sync:
                torch.cuda.synchronize()
            y = codec.decompress(m, n, cfg, shards=2, out_dtype=dtype)
            if sync:
                torch.cuda.synchronize()
            outs += [m[:, :mb], red[:mb], y]
        torch.cuda.synchronize()
        return outs

    for a, b_ in zip(chain(False), chain(True)):
        assert torch.equal(a.contiguous().view(torch.uint8), b_.contiguous().view(torch.uint8))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("b", [64, 256])
def test_alignment_variants_are_bit_identical(port, dtype, b):
    """The same values at 32-byte-aligned (256-bit accesses), 16-byte-aligned and 4/2-byte-
    aligned addresses give identical messages and decodes (ShardArgs::vec_ok = 2 / 1 / 0)."""
    n = b * 301
    cfg = make_config(b)
    x = torch.from_numpy(port.mixture(n, 31)).to(dtype)
    esz = x.element_size()
    ref_msg = codec.compress(x.cuda(), cfg)
    ref_y = codec.decompress(ref_msg, n, cfg, out_dtype=dtype)
    for off_bytes in (16, esz, 32):
        off = off_bytes // esz
        buf = torch.empty(n + 16, dtype=dtype, device="cuda")
        buf[off: off + n] = x.cuda()
        msg = codec.compress(buf[off: off + n], cfg)
        nb = _abi.msg_layout(cfg, n // b).msg_bytes  # the stride's padding is not written
        assert torch.equal(msg[:, :nb], ref_msg[:, :nb]), off_bytes
        ybuf = torch.full((n + 16,), float("nan"), device="cuda").to(dtype)
        codec.decompress(msg, n, cfg, out=ybuf[off: off + n], out_dtype=dtype)
        torch.cuda.synchronize()
        assert torch.equal(ybuf[off: off + n].view(torch.int16 if esz == 2 else torch.int32),
                           ref_y.view(torch.int16 if esz == 2 else torch.int32)), off_bytes


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("b", [64, 128])
def test_direct_load_paths_chunks_and_shards(port, dtype, b):
    """The register-load K1 / K2 paths (fp32 every B, bf16 B = 64 / 128) over shards whose
    starts are 32-byte aligned (S % 16 == 0: 256-bit accesses) or only 16-byte aligned
    (S % 16 == 8), chunks of blocks and a ragged tail: every message equals the compress of
    the zero-padded slice, chunk messages concatenate to the whole message, and the
    sharded decode equals the per-shard decodes."""
    cfg = make_config(b)
    for shards, S in ((3, b * 40), (2, b * 40 + 8), (4, b * 33 + 16)):
        n = shards * S - 5  # ragged last shard
        x = torch.from_numpy(port.mixture(n, 41 + shards)).to(dtype).cuda()
        Sx = -(-n // shards)
        m = -(-Sx // b)
        lay = _abi.msg_layout(cfg, m)
        sh = codec.compress(x, cfg, shards=shards)
        for i in range(shards):
            sl = torch.zeros(Sx, dtype=dtype, device="cuda")
            seg = x[i * Sx:(i + 1) * Sx]
            sl[: seg.numel()] = seg
            one = codec.compress(sl, cfg)
            assert torch.equal(sh[i, : lay.msg_bytes], one[0, : lay.msg_bytes]), (shards, i)
        whole = codec.compress(x, cfg)
        mw = -(-n // b)
        lw = _abi.msg_layout(cfg, mw)
        wc, wa, ws = codec.split_message(whole[0], cfg, mw)
        for b0, b1 in ((0, 7), (7, mw // 2), (mw // 2, mw)):
            part = codec.compress(x, cfg, blk=(b0, b1))
            pc, pa, ps = codec.split_message(part[0], cfg, b1 - b0)
            assert torch.equal(pc, wc[b0 * b: b1 * b]) and torch.equal(pa, wa[b0:b1]) and torch.equal(ps, ws[b0:b1])
        y = codec.decompress(sh, n, cfg, shards=shards, out_dtype=dtype)
        want = torch.cat([codec.decompress(sh[i:i + 1], Sx, cfg, out_dtype=dtype) for i in range(shards)])[:n]
        torch.cuda.synchronize()
        assert torch.equal(y, want), shards
        assert lw.msg_bytes > 0
