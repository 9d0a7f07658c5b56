"""Head-parallel prefill across ranks.

Heads have no cross-head math (runtime.py:174-195), so a layer shards by GQA
group: rank r of N owns kv heads [r*HK/N, (r+1)*HK/N) and their query heads.
The only collective is one all-gather of the per-rank outputs, permuted into
the reference's (B, n, H*d) layout (runtime.py:194).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist


def shard_heads(rank: int, world: int, heads: int, kv_heads: int):
    """(q-head slice, kv-head slice) owned by `rank` (GQA-group aligned)."""
    if kv_heads % world or heads % kv_heads:
        raise ValueError(f"world={world} must divide kv_heads={kv_heads} (and kv_heads | heads)")
    hk = kv_heads // world
    g = heads // kv_heads
    return slice(rank * hk * g, (rank + 1) * hk * g), slice(rank * hk, (rank + 1) * hk)


def gather_heads(local: torch.Tensor, world: int, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather per-rank outputs (n, H_local*d) into (n, world*H_local*d),
    rank-major head order == global head order."""
    n, w = local.shape
    if world == 1:
        return local
    if out is None:
        out = torch.empty((n, world * w), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, n, w), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(buf, local.contiguous(), group=group)
        out.view(n, world, w).copy_(buf.permute(1, 0, 2))
    else:  # gloo (CPU tests; CUDA tensors hop through the host)
        src = local.contiguous().cpu()
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(parts, src, group=group)
        out.view(n, world, w).copy_(torch.stack(parts, 1).to(out.device))
    return out


# ---------------------------------------------------------------- fused output exchange
class _DeviceArray:
    """`__cuda_array_interface__` over a raw device allocation (int16 words)."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i2", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerOutputs:
    """Every rank's final (rows, cols) bf16 output, mapped into every rank.

    Each rank allocates its output with sa_ipc_alloc and all-gathers the CUDA
    IPC handle once; the others map it (sa_ipc_open: NVLink/NVSwitch peer
    memory, or the same GPU when ranks share one in tests).  The attention
    epilogue then stores every row it produces into all of them
    (sa_attn_sparse_work_peers), which replaces the output all-gather."""

    def __init__(self, rank: int, world: int, rows: int, cols: int, group=None):
        from . import _lib

        lib = _lib.load()
        self.rank, self.world, self.rows, self.cols = rank, world, rows, cols
        self._group = group
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * 64)()
        _lib.check(lib.sa_ipc_alloc(rows * cols * 2, ctypes.byref(ptr), handle))
        self._ptr = ptr.value
        handles = [None] * world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.peer_ptrs = []
        for r in range(world):
            if r != rank:
                p = ctypes.c_void_p()
                _lib.check(lib.sa_ipc_open(ctypes.c_char_p(handles[r]), ctypes.byref(p)))
                self.peer_ptrs.append(p.value)
        self.peers = (ctypes.c_void_p * max(1, len(self.peer_ptrs)))(*self.peer_ptrs)
        self.local = torch.as_tensor(_DeviceArray(self._ptr, (rows, cols)), device="cuda").view(torch.bfloat16)
        # barrier flags: [world] last epoch written by each rank + this rank's epoch counter
        fptr = ctypes.c_void_p()
        fh = (ctypes.c_uint8 * 64)()
        _lib.check(lib.sa_ipc_alloc(4 * (world + 1), ctypes.byref(fptr), fh))
        self._fptr = fptr.value
        torch.as_tensor(_DeviceArray(self._fptr, (2 * (world + 1),)), device="cuda").zero_()
        torch.cuda.synchronize()
        fhandles = [None] * world
        dist.all_gather_object(fhandles, bytes(fh), group=group)  # every rank's flags zeroed before any use
        self.peer_flag_ptrs = []
        for r in range(world):
            if r != rank:
                p = ctypes.c_void_p()
                _lib.check(lib.sa_ipc_open(ctypes.c_char_p(fhandles[r]), ctypes.byref(p)))
                self.peer_flag_ptrs.append(p.value)
        self.peer_flags = (ctypes.c_void_p * max(1, len(self.peer_flag_ptrs)))(*self.peer_flag_ptrs)

    def barrier(self, timeout_ms: int = 60000) -> None:
        """Device-side barrier of the ranks on the current stream (sa_peer_barrier):
        later work on the stream sees every rank's peer stores issued before it."""
        from . import _lib
        from . import _device as Dv

        _lib.call("sa_peer_barrier", self._fptr, self.peer_flags, self.rank, self.world, timeout_ms, Dv.stream())

    def close(self) -> None:
        """Unmap the peers and free this rank's buffer (collective)."""
        from . import _lib

        lib = _lib.load()
        torch.cuda.synchronize()
        dist.barrier(group=self._group)  # no rank still stores into a peer
        for p in self.peer_ptrs + self.peer_flag_ptrs:
            _lib.check(lib.sa_ipc_close(ctypes.c_void_p(p)))
        dist.barrier(group=self._group)  # no rank still maps this buffer
        self.local = None
        _lib.check(lib.sa_ipc_free(ctypes.c_void_p(self._ptr)))
        _lib.check(lib.sa_ipc_free(ctypes.c_void_p(self._fptr)))


# ---------------------------------------------------------------- balanced layer
def _view(buf: torch.Tensor, ptr: int, count: int, dtype) -> torch.Tensor:
    """`count` elements of `dtype` at device pointer `ptr` inside `buf` (uint8)."""
    esize = torch.empty(0, dtype=dtype).element_size()
    off = ptr - buf.data_ptr()
    if off < 0 or off + count * esize > buf.numel():
        raise RuntimeError("pointer outside the workspace")
    return buf[off: off + count * esize].view(dtype)


class BalancedLayer:
    """Head-parallel prefill of one layer with load-balanced attention.

    Sharding whole kv groups leaves the ranks that own the vertical-slash heads
    with most of the executed tiles.  Here each rank
    (1) runs selection, estimators and tile lists for its own GQA group of
    heads (`stop_after_tiles`), (2) exchanges the compact realised index of
    those heads with every rank (one all-gather, ~tens of KB per head), (3)
    rebuilds the tile lists of all heads, orders every (head, query tile) item
    by executed tiles (stable, so identical on every rank) and deals them out
    in a snake over the ranks, (4) runs the attention kernel on its items only
    (`sa_attn_sparse_work`, Q/K/V of all heads resident on every rank), and
    (5) all-gathers the produced 128-row output blocks into the reference
    (n, H*d) layout.  The exchanges are methods so a single-GPU test can play
    every rank in turn (tests/test_gpu_multigpu_sim.py)."""

    def __init__(self, rank: int, world: int, heads: int, kv_heads: int, n: int, d: int, mode: str,
                 fixed_pattern=None, device=None):
        from . import runtime as R

        self.rank, self.world = rank, world
        self.H, self.HK, self.n, self.d = heads, kv_heads, n, d
        self.q_sl, self.kv_sl = shard_heads(rank, world, heads, kv_heads)
        self.h_l = heads // world
        dev = torch.device("cuda") if device is None else device
        self.local = R.PrefillPlan(1, self.h_l, kv_heads // world, n, d, mode, fixed_pattern=fixed_pattern)
        self.local.desc.stop_after_tiles = 1
        self.full = R.PrefillPlan(1, heads, kv_heads, n, d, mode, fixed_pattern=fixed_pattern)
        self.ws_local = torch.empty(self.local.ws_bytes, dtype=torch.uint8, device=dev)
        self.ws_full = torch.empty(self.full.ws_bytes, dtype=torch.uint8, device=dev)
        self.vl = self.local.views(self.ws_local)
        self.vf = self.full.views(self.ws_full)
        if mode == "auto":
            fams = [c.family for c in list(self.full.desc.full)[: self.full.desc.ncand]]
        elif mode == "fixed":
            fams = [self.full.desc.fixed.family]
        else:
            fams = []
        self.any_block = 2 in fams
        self.words = self.vf.index.vs_words
        self.row_stride = self.vf.index.blk_row_stride
        self.head_stride = int(self.vf.blk_head_stride)
        self.nqt = (n + 127) // 128
        self.items = heads * self.nqt
        self.per = -(-self.items // world)  # block slots per rank in the output exchange
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        # snake deal of the heaviest-first item order: rank r takes the positions
        # p with owner(p) == r (fixed per shape, so no host sync per step)
        p = np.arange(self.items)
        lap, pos = p // world, p % world
        owner = np.where(lap % 2 == 0, pos, world - 1 - pos)
        self.positions = [torch.from_numpy(p[owner == r]).to(dev) for r in range(world)]
        self.n_mine = torch.tensor([len(self.positions[rank])], dtype=torch.int32, device=dev)
        self.out = torch.zeros((self.nqt * 128, heads * d), dtype=torch.bfloat16, device=dev)

    def enable_checks(self, flag: torch.Tensor, cache_k: torch.Tensor, cache_v: torch.Tensor) -> None:
        """Run AttnMatrices' finiteness scan (core.py:72-74) of this rank's
        q / k / v and the KvCache fill of its kv heads (runtime.py:197) inside
        the estimation step (sa_prefill's side stream); `flag` is a device int,
        cache_k / cache_v are (kv_heads / world, capacity, 128) bf16."""
        d = self.local.desc
        d.check_flag = flag.data_ptr()
        d.cache_k, d.cache_v = cache_k.data_ptr(), cache_v.data_ptr()
        d.cache_capacity = cache_k.shape[1]

    # -- index fields of `nh` heads starting at head `h0` of a plan's views
    def _fields(self, ws, view, h0: int, nh: int):
        idx = view.index
        i32 = torch.int32
        f = [_view(ws, idx.family, h0 + nh, i32)[h0:], _view(ws, idx.tri_window, h0 + nh, i32)[h0:],
             _view(ws, idx.tri_sinks, h0 + nh, i32)[h0:], _view(ws, idx.blk_b, h0 + nh, i32)[h0:],
             _view(ws, idx.colbits, (h0 + nh) * self.words, i32)[h0 * self.words:],
             _view(ws, idx.diagrev, (h0 + nh) * self.words, i32)[h0 * self.words:],
             _view(ws, idx.blk_row_off, (h0 + nh) * self.row_stride, i32)[h0 * self.row_stride:]]
        if self.any_block:
            f.append(_view(ws, idx.blk_idx, (h0 + nh) * self.head_stride, i32)[h0 * self.head_stride:])
        return f

    def estimate(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        """(1): this rank's heads; q/k/v hold every head (H|HK, n, 128).
        Returns the packed index of this rank's heads (int32, same size on every rank)."""
        ql, kl, vl = q[self.q_sl], k[self.kv_sl], v[self.kv_sl]
        if self.local.mode == "auto":
            self.local.select(ql, kl, self.ws_local)
        self.local.run(ql, kl, vl, self.out, self.ws_local)  # stops after the tile lists
        return torch.cat([x.reshape(-1) for x in self._fields(self.ws_local, self.vl, 0, self.h_l)])

    def load_index(self, gathered: torch.Tensor) -> None:
        """(2)-(3): `gathered` = the world's packed indices [world, L]; rebuild all tile lists."""
        from . import _lib
        from . import _device as Dv

        for r in range(self.world):
            pos = 0
            dst = self._fields(self.ws_full, self.vf, r * self.h_l, self.h_l)
            for i, x in enumerate(dst):
                m = x.numel()
                src = gathered[r, pos: pos + m]
                if i == 6:  # row offsets are absolute into blk_idx: rebase by the head offset
                    src = src + r * self.h_l * self.head_stride
                x.copy_(src)
                pos += m
        _lib.call("sa_build_tiles", self.vf.index, self.H, self.n, self.vf.tile_off, self.vf.tile_cnt,
                  self.vf.tiles, Dv.stream())
        cnt = _view(self.ws_full, self.vf.tile_cnt, self.items, torch.int32)
        order = torch.argsort(-cnt.long(), stable=True)  # stable: the same on every rank
        self.owner_items = [order[pos].to(torch.int32) for pos in self.positions]
        self.mine = self.owner_items[self.rank].contiguous()

    def attend(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        """(4): attention for this rank's items; returns its output blocks [per, 128, d]."""
        from . import _lib
        from . import _device as Dv

        _lib.call("sa_attn_sparse_work", 1, self.H, self.HK, self.n, self.full.scale, q.data_ptr(), k.data_ptr(),
                  v.data_ptr(), self.out.data_ptr(), self.vf.index, self.vf.tile_off, self.vf.tile_cnt,
                  self.vf.tiles, self.mine.data_ptr(), self.n_mine.data_ptr(), self.counter.data_ptr(), 0,
                  Dv.stream())
        return self._pack(self.mine)

    def _blocks(self, out):
        return out.view(self.nqt, 128, self.H, self.d)

    def _pack(self, items):
        o4 = self._blocks(self.out)
        buf = torch.zeros((self.per, 128, self.d), dtype=self.out.dtype, device=self.out.device)
        hh, qt = items.long() // self.nqt, items.long() % self.nqt
        buf[: items.numel()] = o4[qt, :, hh, :]
        return buf

    def assemble(self, gathered: torch.Tensor, final: torch.Tensor | None = None) -> torch.Tensor:
        """(5): `gathered` = every rank's blocks [world, per, 128, d] -> (n, H*d)."""
        if final is None:
            final = torch.empty((self.nqt * 128, self.H * self.d), dtype=self.out.dtype, device=self.out.device)
        f4 = self._blocks(final)
        for r, items in enumerate(self.owner_items):
            hh, qt = items.long() // self.nqt, items.long() % self.nqt
            f4[qt, :, hh, :] = gathered[r, : items.numel()]
        return final[: self.n]

    @staticmethod
    def _all_gather(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
        """[world, *x.shape]: NCCL on device; gloo (tests, ranks sharing one GPU) through host copies."""
        if dist.get_backend(group) == "nccl":
            out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
            dist.all_gather_into_tensor(out, x.contiguous(), group=group)
            return out
        h = x.detach().cpu()
        if h.dtype == torch.bfloat16:  # gloo has no bf16: move the bits as fp16 (a byte copy)
            parts = [torch.empty_like(h.view(torch.float16)) for _ in range(world)]
            dist.all_gather(parts, h.view(torch.float16).contiguous(), group=group)
            return torch.stack(parts).view(torch.bfloat16).to(x.device)
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h.contiguous(), group=group)
        return torch.stack(parts).to(x.device)

    def step(self, q, k, v, group=None) -> torch.Tensor:
        """One layer on this rank (all-gathers between the phases)."""
        self.load_index(self._all_gather(self.estimate(q, k, v), self.world, group))
        return self.assemble(self._all_gather(self.attend(q, k, v), self.world, group))

    def attend_peers(self, q, k, v, peer: PeerOutputs) -> None:
        """(4)+(5) fused: attention for this rank's items, each output row
        stored into this rank's and every peer's output buffer."""
        from . import _lib
        from . import _device as Dv

        if peer.rows < self.n or peer.cols != self.H * self.d:
            raise ValueError("peer output buffers have the wrong shape")
        _lib.call("sa_attn_sparse_work_peers", 1, self.H, self.HK, self.n, self.full.scale, q.data_ptr(),
                  k.data_ptr(), v.data_ptr(), peer.local.data_ptr(), peer.peers, len(peer.peer_ptrs),
                  self.vf.index, self.vf.tile_off, self.vf.tile_cnt, self.vf.tiles, self.mine.data_ptr(),
                  self.n_mine.data_ptr(), self.counter.data_ptr(), 0, Dv.stream())

    def step_peers(self, q, k, v, peer: PeerOutputs, group=None) -> torch.Tensor:
        """One layer with the output all-gather fused into the attention
        epilogue.  Two device-side barriers (no host sync): before the
        attention, every rank is done with the previous layer's output
        (write-after-read on the peers' buffers); after it, every rank's peer
        stores are visible to the work queued next on this stream."""
        self.load_index(self._all_gather(self.estimate(q, k, v), self.world, group))
        peer.barrier()
        self.attend_peers(q, k, v, peer)
        peer.barrier()
        return peer.local[: self.n]
