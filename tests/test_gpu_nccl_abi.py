"""The C-ABI collectives over a caller's NCCL communicator (include/taco_b200.h
taco_allreduce_nccl / taco_reduce_scatter_nccl / taco_all_gather_nccl).

One GPU here, so the communicator has one rank (made with ncclCommInitRank through ctypes
on the process's libnccl.so.2, the same instance the library resolves at run time); the
schedule degenerates to K1 -> send/recv to self -> K3 -> all-gather of one -> K2 and must
equal the same kernels called directly, bit for bit.  The multi-rank schedule is the one
tests/test_collective_gloo.py pins against the reference two-shot."""
import ctypes as C
import os

import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2604_24088_b200 import _abi, codec  # noqa: E402
from paper_2604_24088_b200._abi import make_config  # noqa: E402


class _UniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


@pytest.fixture(scope="module")
def comm1():
    try:
        import nvidia.nccl
        path = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
    except Exception:
        path = "libnccl.so.2"
    nccl = C.CDLL(path, mode=C.RTLD_GLOBAL)
    uid = _UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    torch.cuda.set_device(0)
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    yield comm
    torch.cuda.synchronize()
    nccl.ncclCommDestroy(comm)


def _st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("dtype,b,n", [(torch.bfloat16, 256, 8192 * 40 + 3), (torch.float32, 128, 100_003)])
def test_nccl_abi_collectives_world1(port, comm1, dtype, b, n):
    cfg = make_config(b)
    lib = _abi.lib()
    x = torch.from_numpy(port.mixture(n, 11)).cuda().to(dtype)
    ws = torch.empty(lib.taco_collective_nccl_workspace(C.byref(cfg), 1, n), dtype=torch.uint8, device="cuda")
    flags = codec.Flags()
    # all-reduce == K1 -> K3 (one rank) -> K2
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    _abi.check(lib.taco_allreduce_nccl(C.byref(cfg), C.c_void_p(x.data_ptr()), codec._dtype_code(dtype), n,
                                       C.c_void_p(out.data_ptr()), _abi.DT_F32, C.c_void_p(ws.data_ptr()), comm1,
                                       flags.ptr(), _st()))
    m = codec.compress(x, cfg)
    red = torch.empty_like(m[0])
    codec.reduce_encode(m, 1, n, cfg, m.shape[1], red)
    want = codec.decompress(red.view(1, -1), n, cfg)
    torch.cuda.synchronize()
    flags.check()
    assert torch.equal(out.view(torch.int32), want.view(torch.int32))
    # reduce-scatter == the stage-1 sum of one rank == a K2 decode of K1's message
    rs = torch.empty(n, dtype=torch.float32, device="cuda")
    _abi.check(lib.taco_reduce_scatter_nccl(C.byref(cfg), C.c_void_p(x.data_ptr()), codec._dtype_code(dtype), n,
                                            C.c_void_p(rs.data_ptr()), _abi.DT_F32, C.c_void_p(ws.data_ptr()),
                                            comm1, flags.ptr(), _st()))
    rt = codec.decompress(m, n, cfg)
    # all-gather of one == K2(K1(x)) in the requested dtype
    ag = torch.empty(n, dtype=dtype, device="cuda")
    _abi.check(lib.taco_all_gather_nccl(C.byref(cfg), C.c_void_p(x.data_ptr()), codec._dtype_code(dtype), n,
                                        C.c_void_p(ag.data_ptr()), codec._dtype_code(dtype),
                                        C.c_void_p(ws.data_ptr()), comm1, flags.ptr(), _st()))
    torch.cuda.synchronize()
    flags.check()
    assert torch.equal(rs.view(torch.int32), rt.view(torch.int32))
    assert torch.equal(ag, codec.decompress(m, n, cfg, out_dtype=dtype))


def test_nccl_abi_errors(comm1):
    lib = _abi.lib()
    x = torch.zeros(1024, device="cuda")
    cfg = make_config(256)
    rc = lib.taco_allreduce_nccl(C.byref(cfg), C.c_void_p(x.data_ptr()), 0, 1024, C.c_void_p(x.data_ptr()), 0,
                                 None, None, None, _st())
    assert rc == _abi.ERR_USAGE and lib.taco_last_error().decode() == "null NCCL communicator"
    rc = lib.taco_allreduce_nccl(C.byref(cfg), C.c_void_p(x.data_ptr()), 0, 1024, C.c_void_p(x.data_ptr()), 0,
                                 None, comm1, None, _st())
    assert rc == _abi.ERR_USAGE and "workspace required" in lib.taco_last_error().decode()
    bad = make_config(256, kind=_abi.DIRECT_FP8)
    rc = lib.taco_all_gather_nccl(C.byref(bad), C.c_void_p(x.data_ptr()), 0, 1024, C.c_void_p(x.data_ptr()), 0,
                                  None, comm1, None, _st())
    assert rc == _abi.ERR_USAGE and "CodecKind::Taco" in lib.taco_last_error().decode()


@pytest.mark.parametrize("chunks", [1, 3, 16])
def test_nccl_abi_chunked_overlap_bit_identical_and_capturable(port, comm1, chunks):
    """Chunked entry points (codec kernels on the caller's stream, NCCL on the library's
    communication stream, event-ordered) equal the default chunking bit for bit, eagerly and
    replayed from a CUDA graph of the caller's stream."""
    n = 8192 * 40 + 3
    cfg = make_config(256)
    lib = _abi.lib()
    x = torch.from_numpy(port.mixture(n, 12)).cuda().to(torch.bfloat16)
    flags = codec.Flags()
    dt = codec._dtype_code(torch.bfloat16)

    def run(fn, ch, out, ws, nn=n):
        args = [C.byref(cfg), C.c_void_p(x.data_ptr()), dt, nn, C.c_void_p(out.data_ptr()), _abi.DT_F32,
                C.c_void_p(ws.data_ptr()), comm1, flags.ptr(), _st()]
        if ch is None:
            _abi.check(getattr(lib, fn)(*args))
        else:
            _abi.check(getattr(lib, fn + "_chunked")(*args, ch))

    ws0 = torch.empty(lib.taco_collective_nccl_workspace(C.byref(cfg), 1, n), dtype=torch.uint8, device="cuda")
    wsc = torch.empty(lib.taco_collective_nccl_workspace_chunked(C.byref(cfg), 1, n, chunks), dtype=torch.uint8,
                      device="cuda")
    for fn in ("taco_allreduce_nccl", "taco_reduce_scatter_nccl", "taco_all_gather_nccl"):
        want = torch.empty(n, dtype=torch.float32, device="cuda")
        got = torch.full((n,), float("nan"), dtype=torch.float32, device="cuda")
        run(fn, None, want, ws0)
        run(fn, chunks, got, wsc)
        torch.cuda.synchronize()
        flags.check()
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), fn
        # captured on a side stream and replayed
        got.fill_(float("nan"))
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            run(fn, chunks, got, wsc)
        g.replay()
        torch.cuda.synchronize()
        flags.check()
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), fn + " (graph)"
    rc = lib.taco_allreduce_nccl_chunked(C.byref(cfg), C.c_void_p(x.data_ptr()), dt, n, C.c_void_p(x.data_ptr()),
                                         dt, C.c_void_p(wsc.data_ptr()), comm1, None, _st(), 17)
    assert rc == _abi.ERR_USAGE and "at most 16" in lib.taco_last_error().decode()
