"""Pack per-head realised indices into the device encoding of ``sa_head_index``.

Encodings:

* Triangular heads keep two integers (window, sinks): the index
  ``columns=range(sinks), diagonals=range(window)`` of the reference
  (patterns.py:262-276) is the band ``i - j < window`` plus ``j < sinks``.
* Vertical-slash heads keep a column bitmap (bit j) and a reversed diagonal
  bitmap (bit n + 127 - o) of ``vs_words`` 32-bit words, so the attention
  kernel reads one 128-bit window per query row and tile.
* Block heads keep a CSR over query blocks: ascending key-block ids per row,
  diagonal block included (patterns.py:316-320).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

FAM_TRI, FAM_VS, FAM_BLOCK, FAM_DENSE, FAM_VS_NOEYE, FAM_DENSE_NC = 0, 1, 2, 3, 5, 6
TK_FULL, TK_LIMIT = 0, 7  # tile kinds (sa_types.h)
HEAD_DIM = 128


def vs_words(n: int) -> int:
    return (n + 256) // 32 + 2


@dataclass
class DeviceIndex:
    """Device tensors backing one ``sa_head_index`` for ``hh`` heads of length ``n``."""

    n: int
    hh: int
    family: torch.Tensor
    tri_window: torch.Tensor
    tri_sinks: torch.Tensor
    colbits: torch.Tensor
    diagrev: torch.Tensor
    blk_b: torch.Tensor
    blk_row_off: torch.Tensor
    blk_idx: torch.Tensor
    blk_row_stride: int

    def view(self) -> _lib.sa_head_index:
        return _lib.sa_head_index(
            self.family.data_ptr(),
            self.tri_window.data_ptr(),
            self.tri_sinks.data_ptr(),
            self.colbits.data_ptr(),
            self.diagrev.data_ptr(),
            self.colbits.shape[1],
            self.blk_b.data_ptr(),
            self.blk_row_off.data_ptr(),
            self.blk_idx.data_ptr(),
            self.blk_row_stride,
        )


class HostIndexBuilder:
    """Accumulates per-head index descriptions on the host, then uploads once."""

    def __init__(self, n: int, hh: int):
        self.n, self.hh = n, hh
        self.family = np.full(hh, FAM_DENSE, np.int32)
        self.tri_window = np.ones(hh, np.int32)
        self.tri_sinks = np.zeros(hh, np.int32)
        self.colbits = np.zeros((hh, vs_words(n)), np.uint32)
        self.diagrev = np.zeros((hh, vs_words(n)), np.uint32)
        self.blk_b = np.ones(hh, np.int32)
        self._blk_rows: dict[int, list[np.ndarray]] = {}

    def set_dense(self, h: int, causal: bool = True) -> None:
        self.family[h] = FAM_DENSE if causal else FAM_DENSE_NC

    def set_triangular(self, h: int, window: int, sinks: int) -> None:
        self.family[h] = FAM_TRI
        self.tri_window[h] = window
        self.tri_sinks[h] = sinks

    def set_vertical_slash(self, h: int, columns, diagonals) -> None:
        n = self.n
        self.family[h] = FAM_VS
        bits = np.zeros(self.colbits.shape[1] * 32, np.uint8)
        cols = np.asarray(columns, np.int64)
        bits[cols] = 1
        self.colbits[h] = np.packbits(bits, bitorder="little").view(np.uint32)
        bits[:] = 0
        offs = np.asarray(diagonals, np.int64)
        bits[n + 127 - offs] = 1
        self.diagrev[h] = np.packbits(bits, bitorder="little").view(np.uint32)

    def set_block(self, h: int, b: int, rows: list[np.ndarray]) -> None:
        """rows[gq] = ascending key-block ids of query block gq."""
        self.family[h] = FAM_BLOCK
        self.blk_b[h] = b
        self._blk_rows[h] = rows

    def upload(self, device) -> DeviceIndex:
        stride = 1
        for rows in self._blk_rows.values():
            stride = max(stride, len(rows) + 1)
        row_off = np.zeros((self.hh, stride), np.int32)
        chunks = []
        base = 0
        for h, rows in self._blk_rows.items():
            lens = np.array([len(r) for r in rows], np.int64)
            off = base + np.concatenate([[0], np.cumsum(lens)])
            row_off[h, : len(off)] = off
            row_off[h, len(off):] = off[-1]
            if len(rows):
                chunks.append(np.concatenate([np.asarray(r, np.int32) for r in rows]))
            base = int(off[-1])
        blk_idx = np.concatenate(chunks) if chunks else np.zeros(1, np.int32)

        def t(x):
            return torch.from_numpy(np.ascontiguousarray(x)).to(device)

        return DeviceIndex(
            n=self.n,
            hh=self.hh,
            family=t(self.family),
            tri_window=t(self.tri_window),
            tri_sinks=t(self.tri_sinks),
            colbits=t(self.colbits.view(np.int32)),
            diagrev=t(self.diagrev.view(np.int32)),
            blk_b=t(self.blk_b),
            blk_row_off=t(row_off),
            blk_idx=t(blk_idx.astype(np.int32)),
            blk_row_stride=stride,
        )


def num_qtiles(n: int) -> int:
    return (n + 127) // 128


def tile_capacity(n: int, hh: int) -> int:
    t = num_qtiles(n)
    return hh * t * (t + 1) // 2


def noncausal_dense_tiles(n: int, hh: int, dev):
    """Tile lists of non-causal dense heads (core.py:138-154 with causal=False):
    every query tile lists every key tile, the last one limited to keys < n."""
    nqt = num_qtiles(n)
    row = np.full(nqt, TK_FULL << 28, np.int64) | np.arange(nqt)
    if n % 128:
        row[-1] = (TK_LIMIT << 28) | (nqt - 1)
    tiles = np.tile(row, hh * nqt).astype(np.uint32).view(np.int32)
    off = (np.arange(hh * nqt, dtype=np.int64) * nqt).astype(np.int32)
    cnt = np.full(hh * nqt, nqt, np.int32)
    return tuple(torch.from_numpy(x).to(dev) for x in (off, cnt, tiles))


def build_tiles(index: DeviceIndex, stream=None):
    """Run sa_build_tiles: returns (tile_off, tile_cnt, tiles) device tensors."""
    dev = index.family.device
    nqt = num_qtiles(index.n)
    tile_off = torch.empty(index.hh * nqt, dtype=torch.int32, device=dev)
    tile_cnt = torch.empty(index.hh * nqt, dtype=torch.int32, device=dev)
    tiles = torch.empty(max(1, tile_capacity(index.n, index.hh)), dtype=torch.int32, device=dev)
    view = index.view()
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _lib.call("sa_build_tiles", view, index.hh, index.n, tile_off.data_ptr(),
              tile_cnt.data_ptr(), tiles.data_ptr(), s)
    return tile_off, tile_cnt, tiles
