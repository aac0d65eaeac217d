"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every symbol the
header declares, and its host-side logic (validation messages, geometry, byte accounting)
matches the reference -- no kernel launches."""
import ctypes as C
import subprocess

import pytest

from paper_2604_24088_b200 import _abi
from paper_2604_24088_b200._abi import TacoError, make_config


def test_library_exports_every_header_symbol():
    lib = _abi.lib()
    syms = _abi.header_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert set(syms) <= exported
    assert lib.taco_abi_version() == 3


def test_default_config_matches_reference_defaults():
    # codec.hpp:24-33: B=256, tau=1, eps=1e-12, E4M3, Taco
    c = _abi.lib().taco_default_config()
    assert (c.block_size, c.target_energy, c.format, c.kind) == (256, 1.0, 0, 0)
    assert c.stability_epsilon == pytest.approx(1e-12, rel=1e-6)


@pytest.mark.parametrize("kw,msg", [
    (dict(block_size=100), "block size must be a power of two"),
    (dict(block_size=0), "block size must be a power of two"),
    (dict(block_size=1), "block size must be between 2 and 32768"),
    (dict(block_size=65536), "block size must be between 2 and 32768"),
    (dict(target_energy=0.0), "target energy must be positive and finite"),
    (dict(target_energy=float("inf")), "target energy must be positive and finite"),
    (dict(stability_epsilon=0.0), "stability epsilon must be positive and finite"),
    (dict(stability_epsilon=float("nan")), "stability epsilon must be positive and finite"),
])
def test_validation_messages_match_reference(kw, msg, port):
    # codec.cpp:189-197, transform.cpp:13-20 (test_codec.cpp:318-349)
    cfg = make_config(**kw)
    with pytest.raises(TacoError, match=msg) as ei:
        _abi.check(_abi.lib().taco_validate_config(C.byref(cfg)))
    assert ei.value.code == "config"
    # and the oracle raises the same message for the same config
    from oracle.oracle import OracleError
    with pytest.raises(OracleError, match=msg):
        port.compress([1.0], block_size=kw.get("block_size", 256), tau=kw.get("target_energy", 1.0),
                      eps=kw.get("stability_epsilon", 1e-12))


def test_empty_input_rejected_before_any_launch():
    cfg = make_config()
    with pytest.raises(TacoError, match="input tensor is empty") as ei:
        _abi.check(_abi.lib().taco_compress_dev(C.byref(cfg), None, 0, 0, 1, 0, 0, None, 0, None, None))
    assert ei.value.code == "input"
    with pytest.raises(TacoError, match="compressed tensor declares zero elements") as ei:
        _abi.check(_abi.lib().taco_decompress_dev(C.byref(cfg), None, 0, 1, 0, 0, 0, None, 0, None, None))
    assert ei.value.code == "corrupt"


def test_allreduce_needs_two_ranks():
    cfg = make_config()
    with pytest.raises(TacoError, match="allreduce needs at least 2 ranks") as ei:
        _abi.check(_abi.lib().taco_allreduce_sim_dev(C.byref(cfg), None, 0, 1, 16, None, 0, None, None, None,
                                                     None))
    assert ei.value.code == "usage"


def test_flag_mapping():
    with pytest.raises(TacoError, match="input tensor contains NaN or Inf"):
        _abi.check(_abi.lib().taco_flags_status(_abi.FLAG_NONFINITE_INPUT))
    with pytest.raises(TacoError, match="block scalars must be finite and nonzero"):
        _abi.check(_abi.lib().taco_flags_status(_abi.FLAG_BAD_SCALARS))
    _abi.check(_abi.lib().taco_flags_status(0))


@pytest.mark.parametrize("b", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 4096, 32768])
@pytest.mark.parametrize("m", [1, 3, 40960])
def test_message_layout(b, m):
    lay = _abi.msg_layout(make_config(b), m)
    assert lay.codes_bytes == m * b
    assert lay.scal_offset % 16 == 0 and lay.scal_offset >= m * b
    assert lay.msg_bytes == lay.scal_offset + 8 * m
    assert lay.msg_stride % 16 == 0 and lay.msg_stride >= lay.msg_bytes
    if b >= 16:
        assert lay.msg_bytes == m * (b + 8)  # the reference's per-block wire cost


def test_byte_accounting_matches_reference(ref):
    for b in (32, 256, 512):
        cfg = make_config(b)
        for n in (1, 1000, 1_000_000, 10_485_760):
            assert _abi.lib().taco_archive_size(C.byref(cfg), n) == ref.archive_size(n, b)
            assert _abi.lib().taco_compressed_ratio(C.byref(cfg), n) == ref.compressed_ratio(n, b)
    assert _abi.lib().taco_archive_size(C.byref(make_config()), 1_000_000) == 1_031_470


def test_product_does_not_reference_the_oracle():
    import pathlib
    pkg = pathlib.Path(_abi.PKG_DIR)
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cpp")):
        text = f.read_text()
        assert "oracle" not in text.replace("oracle/", "").lower() or f.name == "__init__.py", f
    out = subprocess.run(["nm", "-D", _abi.LIB_PATH], capture_output=True, text=True).stdout
    names = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert not any(s.startswith(("tor_", "ref_")) for s in names)


def test_peer_abi_argument_checks_without_a_gpu():
    """The peer-memory entry points validate their peer set before touching the device."""
    import ctypes as C
    lib = _abi.lib()
    cfg = make_config()
    assert lib.taco_peer_flags_bytes() >= 4 * _abi.MAX_PEERS + 4
    cases = []
    ps = _abi.Peers(); ps.nranks = 9; cases.append((ps, "1 to 8 ranks"))
    ps = _abi.Peers(); ps.nranks = 0; cases.append((ps, "1 to 8 ranks"))
    ps = _abi.Peers(); ps.nranks, ps.rank = 2, 2; cases.append((ps, "rank outside the peer set"))
    ps = _abi.Peers(); ps.nranks, ps.rank = 2, 0; ps.base[0] = 4096; cases.append((ps, "peer region not mapped"))
    for ps, msg in cases:
        for rc in (lib.taco_compress_push_dev(C.byref(cfg), None, 1, 100, C.byref(ps), 0, 1, 0, 0, None, None),
                   lib.taco_reduce_encode_push_dev(C.byref(cfg), None, 0, C.byref(ps), 100, 0, 1, 0, 0, None, 0,
                                                   None, None),
                   lib.taco_peer_barrier_dev(C.byref(ps), 0, 10, None, None)):
            assert rc == _abi.ERR_USAGE and msg in lib.taco_last_error().decode()
    ps = _abi.Peers(); ps.nranks, ps.rank = 1, 0; ps.base[0] = 4096
    assert lib.taco_compress_push_dev(C.byref(make_config(4096)), None, 1, 100, C.byref(ps), 0, 1, 0, 0, None,
                                      None) == _abi.ERR_USAGE
    assert "up to 1024" in lib.taco_last_error().decode()
    assert lib.taco_peer_barrier_dev(C.byref(ps), 8, 10, None, None) == _abi.ERR_USAGE
    assert lib.taco_flags_status(_abi.FLAG_PEER_TIMEOUT) == _abi.ERR_CUDA
    assert lib.taco_last_error().decode() == "peer barrier timed out"


def test_fused_peer_abi_checks_without_a_gpu():
    """The fused (kernel-signalled) peer collectives validate the peer set, the config they
    serve and the sync-word alignment before touching the device."""
    import ctypes as C
    lib = _abi.lib()
    assert lib.taco_peer_flags_bytes() >= 4 * 35  # epoch, two phases of 8 words, tickets
    assert lib.taco_peer_fused_supported(C.byref(make_config(256))) == 1
    for b, fmt in ((32, 0), (1024, 0), (256, 1)):
        assert lib.taco_peer_fused_supported(C.byref(make_config(b, fmt))) == 0
    ps = _abi.Peers(); ps.nranks = 9
    assert lib.taco_peer_allreduce_dev(C.byref(make_config()), None, 1, 100, C.byref(ps), 0, 0, 0, 0, None, 1, 10,
                                       None, None) == _abi.ERR_USAGE
    assert "1 to 8 ranks" in lib.taco_last_error().decode()
    ps = _abi.Peers(); ps.nranks, ps.rank = 1, 0; ps.base[0] = 4096
    for cfg in (make_config(256, 1), make_config(32)):
        for rc in (lib.taco_peer_allreduce_dev(C.byref(cfg), None, 1, 100, C.byref(ps), 0, 0, 0, 0, None, 1, 10,
                                               None, None),
                   lib.taco_peer_reduce_scatter_dev(C.byref(cfg), None, 1, 100, C.byref(ps), 0, 0, 0, None, 1, 10,
                                                    None, None),
                   lib.taco_peer_all_gather_dev(C.byref(cfg), None, 1, 100, C.byref(ps), 0, 0, 0, None, 1, 10,
                                                None, None)):
            assert rc == _abi.ERR_USAGE and "fused peer signalling" in lib.taco_last_error().decode()
    assert lib.taco_peer_allreduce_dev(C.byref(make_config()), None, 1, 100, C.byref(ps), 0, 0, 0, 8, None, 1, 10,
                                       None, None) == _abi.ERR_USAGE
    assert "16-byte aligned" in lib.taco_last_error().decode()
    assert lib.taco_peer_allreduce_dev(C.byref(make_config()), None, 1, 0, C.byref(ps), 0, 0, 0, 0, None, 1, 10,
                                       None, None) == _abi.ERR_INPUT
    assert lib.taco_peer_check_access(0, 0) == _abi.OK


def test_schedule_host_argument_checks_without_a_gpu():
    """taco_allreduce_schedule_host (ring / tree / two-shot on the device) rejects what the
    reference rejects (collective.cpp:24-33) before any device work."""
    import ctypes as C
    lib = _abi.lib()
    cfg = make_config()
    x = (C.c_float * 8)()
    cases = ((None, 0, 2, 4, "null taco context", _abi.ERR_USAGE),)
    for ctx, alg, p, n, msg, code in cases:
        rc = lib.taco_allreduce_schedule_host(ctx, C.byref(cfg), alg, x, p, n, x, x, None)
        assert rc == code and msg in lib.taco_last_error().decode()


def test_chunked_nccl_workspace_sizes():
    """Chunking never needs less workspace than one chunk (each chunk's messages are padded to
    16 bytes); 0 chunks = the default (2); > 16 is refused (workspace 0)."""
    import ctypes as C
    lib = _abi.lib()
    cfg = make_config()
    n = 8192 * 2560
    w = [lib.taco_collective_nccl_workspace_chunked(C.byref(cfg), 4, n, c) for c in (1, 2, 3, 16)]
    assert w[0] > 0 and all(v >= w[0] for v in w)
    assert lib.taco_collective_nccl_workspace(C.byref(cfg), 4, n) == w[1]
    assert lib.taco_collective_nccl_workspace_chunked(C.byref(cfg), 4, n, 0) == w[1]
    assert lib.taco_collective_nccl_workspace_chunked(C.byref(cfg), 4, n, 17) == 0


@pytest.mark.parametrize("kind,n,seed", [(0, 100_003, 7), (1, 100_003, 7), (1, 262_144, 101), (1, 1, 3)])
def test_generate_matches_reference(kind, n, seed, ref):
    # taco::generate (analysis.cpp:70-95) value for value: the bench's inputs are the
    # reference's synthetic tensors
    import numpy as np

    from paper_2604_24088_b200 import codec
    got = codec.generate(kind, n, seed).numpy()
    want = ref.generate(kind, n, seed)
    assert got.dtype == np.float32 and np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_generate_errors_match_reference():
    from paper_2604_24088_b200 import codec
    with pytest.raises(TacoError, match="synthetic tensor length must be positive"):
        codec.generate(1, 0, 7)
    with pytest.raises(TacoError, match=r"tail fraction must be in \[0, 1\]"):
        codec.generate(1, 10, 7, tail_fraction=1.5)
    with pytest.raises(TacoError, match="mixture sigmas must be positive"):
        codec.generate(1, 10, 7, dense_sigma=0.0)
