"""GPU parity of the reference's other codec kinds, scaled_spectrum and the
TACOCMP1 archive export/import (§8 f1) against the unmodified reference (oracle/_ref).

The device kernels for DirectFp8 / Int8Uniform / Identity / AshInt8 replay the reference's
own float and double operations (launch_kinds.cu), so everything here is compared BIT FOR
BIT: codes, scalars, decoded values, two-shot results and archive bytes.
"""
import numpy as np
import pytest
import torch

from conftest import GOLDEN  # noqa: F401  (test infrastructure import path)

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2604_24088_b200 import _abi, codec  # noqa: E402
from paper_2604_24088_b200._abi import TacoError, make_config  # noqa: E402

KIND_CASES = [  # (kind, scope, fmt)
    (_abi.DIRECT_FP8, _abi.GLOBAL_MAX, 0), (_abi.DIRECT_FP8, _abi.GLOBAL_MAX, 1),
    (_abi.DIRECT_FP8, _abi.UNIT, 0), (_abi.DIRECT_FP8, _abi.PER_BLOCK_MAX, 0),
    (_abi.DIRECT_FP8, _abi.PER_BLOCK_MAX, 1), (_abi.INT8_UNIFORM, 0, 0), (_abi.IDENTITY, 0, 0),
    (_abi.ASH_INT8, 0, 0),
]
IDS = [f"k{k}-s{s}-f{f}" for k, s, f in KIND_CASES]


def _input(port, n, seed):
    x = port.mixture(n, seed).astype(np.float32)
    x[: min(n, 40)] *= np.float32(3e3)  # a few large values: saturation and scale paths
    return x


def _split(msg_row, cfg, m):
    codes, al, sc = codec.split_message(msg_row, cfg, m)
    return codes.cpu().numpy(), al.cpu().numpy(), sc.cpu().numpy()


@pytest.mark.parametrize("kind,scope,fmt", KIND_CASES, ids=IDS)
@pytest.mark.parametrize("b", [32, 256])
def test_kind_compress_decompress_bit_exact(ref, port, kind, scope, fmt, b):
    n = 5000 + 37  # ragged tail
    x = _input(port, n, 3 + kind)
    cfg = make_config(b, fmt, kind=kind, direct_scale=scope)
    flags = codec.Flags()
    msg = codec.compress(torch.from_numpy(x).cuda(), cfg, flags=flags)
    torch.cuda.synchronize()
    flags.check()
    m = -(-n // b)
    codes, al, sc = _split(msg[0], cfg, m)
    rc, ra, rs = ref.compress2(x, b, fmt, kind, scope)
    assert np.array_equal(codes, rc), "payload"
    assert np.array_equal(al, ra) and np.array_equal(sc, rs), "scalars"
    y = codec.decompress(msg, n, cfg, flags=flags).cpu().numpy()
    flags.check()
    want = ref.decompress(rc, ra, rs, n, b, fmt, kind)
    assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), "decoded values"


@pytest.mark.parametrize("kind,scope,fmt", KIND_CASES[::2], ids=IDS[::2])
def test_kind_bf16_input_and_shards(ref, port, kind, scope, fmt):
    b, p = 128, 3
    n = 3 * 4096 + 100
    x = torch.from_numpy(_input(port, n, 9)).to(torch.bfloat16)
    xf = x.float().numpy()
    cfg = make_config(b, fmt, kind=kind, direct_scale=scope)
    msg = codec.compress(x.cuda(), cfg, shards=p)
    S = -(-n // p)
    ms = -(-S // b)
    for i in range(p):
        sl = np.zeros(S, np.float32)
        seg = xf[i * S:(i + 1) * S]
        sl[: seg.size] = seg
        rc, ra, rs = ref.compress2(sl, b, fmt, kind, scope)  # the reference compresses each shard slice
        codes, al, sc = _split(msg[i], cfg, ms)
        assert np.array_equal(codes, rc) and np.array_equal(al, ra) and np.array_equal(sc, rs), f"shard {i}"
    # block-range chunks reproduce the whole message (tensor-wide scales stay shard-wide)
    whole = _split(msg[0], cfg, ms)
    pb = 4 * b if kind == _abi.IDENTITY else b
    for b0, b1 in ((0, 5), (5, 17), (17, ms)):
        part = codec.compress(x.cuda(), cfg, shards=p, blk=(b0, b1))
        pc, pa, ps = _split(part[0], cfg, b1 - b0)
        assert np.array_equal(pc, whole[0][b0 * pb: b1 * pb])
        assert np.array_equal(pa, whole[1][b0:b1]) and np.array_equal(ps, whole[2][b0:b1])


@pytest.mark.parametrize("kind,scope,fmt", KIND_CASES, ids=IDS)
def test_kind_allreduce_twoshot_bit_exact(ref, port, kind, scope, fmt):
    p, n, b = 4, 6000 + 3, 64
    ins = np.stack([_input(port, n, 100 + r) for r in range(p)])
    cfg = make_config(b, fmt, kind=kind, direct_scale=scope)
    if kind == _abi.DIRECT_FP8 and scope != _abi.GLOBAL_MAX:
        pytest.skip("the reference's RankSet carries the default GlobalMax scope only")
    got = codec.allreduce_sim(torch.from_numpy(ins).cuda(), cfg).cpu().numpy()
    want = ref.allreduce(ins, b, fmt, kind)["result"]
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("kind,fmt", [(0, 0), (0, 1), (_abi.ASH_INT8, 0)])
def test_scaled_spectrum_bit_exact(ref, port, kind, fmt):
    x = _input(port, 3000 + 11, 21)
    got = codec.scaled_spectrum(torch.from_numpy(x).cuda(), make_config(256, fmt, kind=kind)).cpu().numpy()
    want = ref.scaled_spectrum(x, 256, fmt, kind)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("kind,scope,fmt", [(0, 0, 0)] + KIND_CASES, ids=["taco"] + IDS)
def test_archive_export_import(ref, port, kind, scope, fmt):
    n, b = 1000, 256
    x = _input(port, n, 5)
    cfg = make_config(b, fmt, kind=kind, direct_scale=scope)
    msg = codec.compress(torch.from_numpy(x).cuda(), cfg)
    arch = codec.archive_export(msg[0], n, cfg)
    data = arch.cpu().numpy().tobytes()
    assert len(data) == ref.archive_size(n, b, kind) == _abi.lib().taco_archive_size(cfg, n)
    if kind != 0:  # codes are bit-exact: the archive is byte-identical to the reference's
        assert data == ref.archive2(x, b, fmt, kind, scope)
    else:  # Taco codes may differ by one-ulp flips: check the layout against our own message
        m = -(-n // b)
        codes, al, sc = _split(msg[0], cfg, m)
        body = b"".join(codes[k * b:(k + 1) * b].tobytes() + np.float32([al[k], sc[k]]).tobytes() for k in range(m))
        assert data[:22] == ref.archive2(x, b, fmt, kind, scope)[:22] and data[22:] == body
    # import: same message; the reference parses and decodes our bytes to our output
    cfg2, n2, msg2 = codec.archive_import(arch)
    assert (cfg2.block_size, cfg2.kind, n2) == (b, kind, n)
    lay = _abi.msg_layout(cfg, -(-n // b))
    assert torch.equal(msg2[: lay.msg_bytes], msg[0, : lay.msg_bytes])
    ours = codec.decompress(msg2.view(1, -1), n, cfg2).cpu().numpy()
    theirs = ref.archive_decode(data, n)
    if kind != 0:
        assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))
    else:  # K2 decodes in fp32, the reference in fp64 (DECODE_RELMSE_MAX, tests/parity.py)
        from parity import DECODE_RELMSE_MAX, rel_mse
        assert rel_mse(ours, theirs) <= DECODE_RELMSE_MAX


def test_archive_errors_match_reference(port):
    cfg = make_config(64)
    x = port.gaussian(300, 1)
    good = codec.archive_export(codec.compress(torch.from_numpy(x).cuda(), cfg)[0], 300, cfg).cpu().numpy()

    def imp(raw):
        return codec.archive_import(torch.from_numpy(np.asarray(raw, np.uint8)).cuda())

    cases = []
    bad = good.copy(); bad[0] = ord("X"); cases.append((bad, "bad magic, not a compressed archive"))
    bad = good.copy(); bad[8] = 9; cases.append((bad, "unknown codec kind in archive"))
    bad = good.copy(); bad[9] = 7; cases.append((bad, "unknown payload format in archive"))
    bad = good.copy(); bad[10:14] = np.frombuffer(np.uint32(100).tobytes(), np.uint8)
    cases.append((bad, "archive block size is not a valid power of two"))
    bad = good.copy(); bad[14:22] = 0; cases.append((bad, "archive declares zero elements"))
    cases.append((good[:-1], "unexpected end of archive"))
    cases.append((good[:15], "unexpected end of archive"))
    cases.append((np.concatenate([good, [0]]), "trailing bytes after archive payload"))
    bad = good.copy(); bad[22 + 64: 22 + 68] = np.frombuffer(np.float32(np.inf).tobytes(), np.uint8)
    cases.append((bad, "block scalars must be finite"))
    bad = bad[:-3]; cases.append((bad, "block scalars must be finite"))  # truncated after the bad block
    for raw, msg in cases:
        with pytest.raises(TacoError, match=msg) as ei:
            imp(raw)
        assert ei.value.code == "corrupt"


# --------------------------------------------------------- error metrics (§8 f4) ---
@pytest.mark.parametrize("bins", [1, 64])
def test_error_report_matches_reference(ref, port, bins):
    x = port.mixture(1_000_003, 7)
    cfg = make_config(256)
    xd = torch.from_numpy(x).cuda()
    y = codec.decompress(codec.compress(xd, cfg), x.size, cfg)
    got = codec.error_report(xd, y, bins)
    want = ref.error_report(x, y.cpu().numpy(), bins)
    for k in ("mse", "relative_l2", "kurtosis"):  # sums in another order: last-bit differences
        assert got[k] == pytest.approx(want[k], rel=1e-9), k
    assert got["max_abs_error"] == want["max_abs_error"]
    assert got["zero_collapse_fraction"] == want["zero_collapse_fraction"]
    assert got["bin_edges"][0] == want["lo"] and got["bin_edges"][-1] == want["hi"]
    assert got["counts"] == want["counts"]


def test_error_report_edge_cases():
    z = torch.zeros(1000, device="cuda")
    r = codec.error_report(z, z, 8)
    assert r["mse"] == 0.0 and r["relative_l2"] == 0.0 and not r["kurtosis_defined"]
    assert r["bin_edges"][0] == -0.5 and r["bin_edges"][-1] == 0.5 and r["counts"][4] == 1000
    with pytest.raises(TacoError, match="input tensor is empty"):
        codec.error_report(torch.zeros(0, device="cuda"), torch.zeros(0, device="cuda"))
