"""Host (oracle-backed) implementation of the collective's codec interface -- TEST ONLY.

Produces and consumes byte-identical messages to the CUDA kernels (include/taco_b200.h
layout: codes, pad to 16, (alpha, scale) pairs), with the oracle (oracle/taco_oracle.c)
doing the arithmetic.  It lets tests/test_collective_gloo.py run the real
paper_2604_24088_b200.collective schedule across gloo ranks on CPU; because the
arithmetic is the oracle's, the schedule must reproduce the reference's two-shot
all-reduce bit for bit.
"""
import numpy as np
import torch

from paper_2604_24088_b200 import _abi


def cdiv(a, b):
    return -(-a // b)


class HostCodec:
    def __init__(self, port):
        self.port = port

    def layout(self, cfg, nblocks):
        return _abi.msg_layout(cfg, nblocks)

    def _pack(self, cfg, out_row: torch.Tensor, codes, alpha, scale):
        nb = alpha.size
        lay = _abi.msg_layout(cfg, nb)
        buf = out_row.numpy()
        buf[: nb * cfg.block_size] = codes
        buf[lay.scal_offset: lay.scal_offset + 8 * nb] = np.stack([alpha, scale], 1).astype(np.float32).view(
            np.uint8).ravel()

    def _unpack(self, cfg, row: torch.Tensor, nb):
        lay = _abi.msg_layout(cfg, nb)
        buf = row.numpy()
        codes = buf[: nb * cfg.block_size].copy()
        sc = buf[lay.scal_offset: lay.scal_offset + 8 * nb].copy().view(np.float32).reshape(nb, 2)
        return codes, sc[:, 0].copy(), sc[:, 1].copy()

    def compress(self, cfg, x, shards, b0, b1, out):
        B, n = cfg.block_size, x.numel()
        S = cdiv(n, shards)
        xf = x.reshape(-1).float().numpy()
        for p in range(shards):
            seg = np.zeros((b1 - b0) * B, np.float32)
            lo, hi = p * S + b0 * B, min(p * S + min(b1 * B, S), n)
            if hi > lo:
                seg[: hi - lo] = xf[lo:hi]
            c, a, s = self.port.compress(seg, B, cfg.format, cfg.target_energy, cfg.stability_epsilon)
            self._pack(cfg, out[p], c, a, s)

    def reduce_encode(self, cfg, recv, nranks, shard_len, rank_stride, b0, b1, out_msg, acc_out):
        B, nb = cfg.block_size, b1 - b0
        nvalid = min(b1 * B, shard_len) - b0 * B
        flat = recv.reshape(-1)
        acc = None
        for r in range(nranks):
            row = flat[r * rank_stride:(r + 1) * rank_stride]
            c, a, s = self._unpack(cfg, row, nb)
            d = self.port.decompress(c, a, s, nvalid, B, cfg.format)
            acc = d.copy() if acc is None else (acc + d).astype(np.float32)
        if acc_out is not None:
            acc_out.reshape(-1)[b0 * B: b0 * B + nvalid] = torch.from_numpy(acc).to(acc_out.dtype)
        if out_msg is not None:
            c, a, s = self.port.compress(acc, B, cfg.format, cfg.target_energy, cfg.stability_epsilon)
            self._pack(cfg, out_msg, c, a, s)

    def decompress(self, cfg, msgs, n, shards, b0, b1, out, msg_stride):
        B, nb = cfg.block_size, b1 - b0
        S = cdiv(n, shards)
        flat = msgs.reshape(-1)
        o = out.reshape(-1)
        for p in range(shards):
            lo = p * S + b0 * B
            hi = min(p * S + min(b1 * B, S), n)
            if hi <= lo:
                continue
            c, a, s = self._unpack(cfg, flat[p * msg_stride:(p + 1) * msg_stride], nb)
            y = self.port.decompress(c, a, s, hi - lo, B, cfg.format)
            o[lo:hi] = torch.from_numpy(y).to(o.dtype)

    def check(self):
        pass
