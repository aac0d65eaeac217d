"""B200-native TACO compression path (arxiv/paper_2604_24088), sm_100a.

Layout:
  csrc/            hand-written CUDA kernels (K1 compress, K2 decompress, K3 decode-reduce-
                   encode), the extern "C" ABI (include/taco_b200.h) and the C++ drop-in
                   for the reference's namespace-taco API (include/taco/*.hpp)
  _abi.py          ctypes binding of libtaco_b200.so
  codec.py         torch-facing device API (compress / decompress / reduce_encode)
  collective.py    compressed TP collectives over torch.distributed (two-shot all-reduce,
                   SP reduce-scatter / all-gather)
"""
from ._abi import TacoError, make_config  # noqa: F401

__all__ = ["TacoError", "make_config"]
