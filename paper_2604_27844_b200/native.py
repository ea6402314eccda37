"""Native communicator: the compressed collectives of csrc/zc_coll.cu behind
the reference's collective API (collectives.py:203-341).

A ``NativeComm`` wraps one ``zc_comm`` of the C-ABI.  It is created
collectively, either over a torch.distributed NCCL group (one process per
GPU; rank 0's NCCL unique id is broadcast through the group) or for
in-process thread ranks (``local_group``), and is attached to the
``Communicator`` the reference API receives (``comm.native``), so
``zip_all_gather(comm, x)`` and friends run the native planes:

* ``plane="auto"`` (default): the peer-memory plane when every peer's
  symmetric buffer could be mapped (one NVLink/NVSwitch node), else the
  message plane;
* ``plane="msg"``: the reference's message protocols over NCCL (or device
  copies between thread ranks): all-gather size phase + frames, all-to-all
  design 1 / design 2; ``pipeline=True`` decodes each all-gather peer on a
  side stream as its ring step lands.

Decode errors land in a per-call device word per peer; with
``sync_errors=True`` (default, the reference's synchronous semantics) they
are read back and raised as ``CollectiveError(peer=...)``; with False the
call returns without a host synchronisation and ``check()`` raises later.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import engine
from ._lib import i64s, lib, stream_ptr
from .errors import CollectiveError, ProtocolError, TransportError, UnrepresentableError

PLANE_P2P, PLANE_MSG, A2A_D1, CHECK_COUNTS, PIPELINE = 1, 2, 4, 8, 16
DEFAULT_SLOT_BYTES = int(os.environ.get("ZC_P2P_SLOT_BYTES", 256 << 20))
LOCAL_SLOT_BYTES = int(os.environ.get("ZC_LOCAL_SLOT_BYTES", 16 << 20))
MAX_WORLD = 64


def _status(handle, rc: int, what: str):
    if rc == 0:
        return
    peer = ctypes.c_int(-1)
    msg = lib().zc_comm_last_error(handle, ctypes.byref(peer)).decode() if handle else ""
    if rc == -4 or rc == -5:
        raise ProtocolError(msg or f"{what}: protocol error")
    if rc == -7:
        raise CollectiveError(msg, peer=peer.value if peer.value >= 0 else None)
    if rc == -6:
        raise TransportError(f"{what}: {msg}")
    if rc == -3:
        raise UnrepresentableError(f"{what}: {msg or 'frame exceeds the u32 offset range'}")
    if rc == -1:
        raise ValueError(f"{what}: invalid argument")
    raise RuntimeError(f"{what} failed: {lib().zc_status_string(rc).decode()} (status {rc})")


def raise_errors(err: torch.Tensor, me: int, expected=None) -> None:
    """Per-peer device error words -> the reference's exceptions.  With
    ``expected`` (all-to-all receive counts) a frame whose element count
    differs is the design-2 static-section mismatch (ProtocolError,
    collectives.py:299-305); otherwise CollectiveError naming the peer."""
    codes = err.cpu().tolist()
    for p, code in enumerate(codes):
        if p == me or code == engine.ERR_OK:
            continue
        if code == 19:
            if expected is not None:
                raise ProtocolError(f"static section from rank {p} does not hold the expected "
                                    f"{expected[p]} elements")
            raise CollectiveError("frame holds a different element count than expected", peer=p)
        raise CollectiveError(f"corrupt frame: {engine.err_message(code)}", peer=p)


class NativeComm:
    """One rank's native communicator (see module docstring)."""

    def __init__(self, handle: int, device: torch.device):
        self.handle = ctypes.c_void_p(handle)
        self.device = torch.device(device)
        info = (ctypes.c_int * 5)()
        lib().zc_comm_info(self.handle, info)
        self.rank, self.world_size = info[0], info[1]
        self.p2p_available = bool(info[2])
        self.shared_device = bool(info[3])
        self.over_nccl = bool(info[4])
        self.plane = "auto"
        self.pipeline = False
        self.check_counts = False
        self.sync_errors = True
        self._pending = []

    # -- construction -----------------------------------------------------------------
    @classmethod
    def from_process_group(cls, group=None, device=None, slot_bytes: int | None = None):
        import torch.distributed as dist
        dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        nb = lib().zc_nccl_id_bytes()
        rank = dist.get_rank(group)
        obj = [None]
        if rank == 0:
            buf = (ctypes.c_uint8 * nb)()
            _status(None, lib().zc_nccl_get_id(buf), "zc_nccl_get_id")
            obj = [bytes(buf)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = (ctypes.c_uint8 * nb).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            rc = lib().zc_comm_init(ctypes.byref(h), uid, rank, dist.get_world_size(group),
                                    int(slot_bytes or DEFAULT_SLOT_BYTES), 0)
        _status(h, rc, "zc_comm_init")
        return cls(h.value, dev)

    @classmethod
    def local_group(cls, world: int, devices=None, slot_bytes: int | None = None) -> list:
        """Communicators for ``world`` in-process thread ranks."""
        if world > MAX_WORLD:
            raise ValueError(f"native communicators support up to {MAX_WORLD} ranks")
        devs = [torch.device(d) for d in devices] if devices else \
            [torch.device("cuda", torch.cuda.current_device())] * world
        handles = (ctypes.c_void_p * world)()
        idx = (ctypes.c_int * world)(*[d.index or 0 for d in devs])
        rc = lib().zc_comm_init_local(handles, world, idx, int(slot_bytes or LOCAL_SLOT_BYTES), 0)
        _status(None, rc, "zc_comm_init_local")
        return [cls(handles[r], devs[r]) for r in range(world)]

    def abort(self):
        """Release ranks blocked in an in-process rendezvous (a peer failed)."""
        if self.handle:
            lib().zc_comm_abort(self.handle)

    def close(self):
        if self.handle:
            lib().zc_comm_destroy(self.handle)
            self.handle = None

    # -- helpers ----------------------------------------------------------------------
    def _flags(self, design: int | None = None) -> int:
        f = 0
        if self.plane == "msg":
            f |= PLANE_MSG
        elif self.plane == "p2p":
            f |= PLANE_P2P
        if design == 1:
            f |= A2A_D1
        if self.check_counts:
            f |= CHECK_COUNTS
        if self.pipeline:
            f |= PIPELINE
        return f

    def plane_for(self, design: int | None = None) -> str:
        if self.world_size == 1:
            return "local"
        if self.plane == "msg" or design == 1 or not self.p2p_available:
            return "msg"
        return "p2p"

    def _finish(self, err: torch.Tensor | None, expected=None):
        if err is None:
            return
        if self.sync_errors:
            raise_errors(err, self.rank, expected)
        else:
            self._pending.append((err, expected))

    def check(self) -> None:
        """Raise the first deferred decode error (sync_errors=False)."""
        pending, self._pending = self._pending, []
        for err, expected in pending:
            raise_errors(err, self.rank, expected)

    def _book(self, words, sigma, segs):
        if sigma is None:
            return None
        from . import codec
        if math.isfinite(sigma) and sigma > 0.0:
            return codec.derive_codebook(sigma).device_tensor(words.device)
        if not segs:
            return None
        return engine.modal_codebook(words, segs)

    def stats(self) -> tuple:
        b, m = ctypes.c_uint64(), ctypes.c_uint64()
        lib().zc_comm_stats(self.handle, ctypes.byref(b), ctypes.byref(m))
        return int(b.value), int(m.value)

    def reserve(self, slot_bytes: int) -> None:
        """Collectively grow the peer-memory slots (all ranks, same value)."""
        _status(self.handle, lib().zc_comm_reserve(self.handle, int(slot_bytes),
                                                   stream_ptr()), "zc_comm_reserve")

    # -- collectives ------------------------------------------------------------------
    def all_gather(self, words: torch.Tensor, sigma=None) -> torch.Tensor:
        n = words.numel()
        W = self.world_size
        out = torch.empty(W * n, dtype=torch.int16, device=words.device)
        if n == 0:
            return out
        err = torch.empty(W, dtype=torch.int32, device=words.device)
        book = self._book(words, sigma, [(0, n)])
        rc = lib().zc_allgather(self.handle, words.data_ptr(), n, out.data_ptr(),
                                book.data_ptr() if book is not None else None, err.data_ptr(),
                                self._flags(), stream_ptr())
        _status(self.handle, rc, "zc_allgather")
        self._finish(err)
        return out

    def all_gather_raw(self, words: torch.Tensor) -> torch.Tensor:
        n = words.numel()
        out = torch.empty(self.world_size * n, dtype=torch.int16, device=words.device)
        rc = lib().zc_allgather_raw(self.handle, words.data_ptr() if n else None, n,
                                    out.data_ptr() if n else None, stream_ptr())
        _status(self.handle, rc, "zc_allgather_raw")
        return out

    def all_to_all(self, buf: torch.Tensor, counts, recv_counts, sigma=None,
                   design: int = 2) -> list:
        W, me = self.world_size, self.rank
        rc_ = list(recv_counts)
        rc_[me] = counts[me]
        total = sum(rc_)
        flat = torch.empty(max(total, 1), dtype=torch.int16, device=buf.device)
        err = torch.empty(W, dtype=torch.int32, device=buf.device)
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        segs = [(int(offs[q]), counts[q]) for q in range(W) if q != me and counts[q]]
        book = self._book(buf, sigma, segs)
        rc = lib().zc_alltoall(self.handle, buf.data_ptr() if buf.numel() else None,
                               i64s(counts), i64s(rc_), flat.data_ptr(),
                               book.data_ptr() if book is not None else None, err.data_ptr(),
                               self._flags(design), stream_ptr())
        _status(self.handle, rc, "zc_alltoall")
        self._finish(err, rc_)
        roffs = np.concatenate([[0], np.cumsum(rc_)]).astype(np.int64)
        return [flat[int(roffs[p]):int(roffs[p + 1])] for p in range(W)]

    def all_to_all_raw(self, buf: torch.Tensor, counts, recv_counts) -> list:
        W, me = self.world_size, self.rank
        rc_ = list(recv_counts)
        rc_[me] = counts[me]
        flat = torch.empty(max(sum(rc_), 1), dtype=torch.int16, device=buf.device)
        rc = lib().zc_alltoall_raw(self.handle, buf.data_ptr() if buf.numel() else None,
                                   i64s(counts), i64s(rc_), flat.data_ptr(),
                                   CHECK_COUNTS if self.check_counts else 0, stream_ptr())
        _status(self.handle, rc, "zc_alltoall_raw")
        roffs = np.concatenate([[0], np.cumsum(rc_)]).astype(np.int64)
        return [flat[int(roffs[p]):int(roffs[p + 1])] for p in range(W)]

    def reduce_scatter(self, words: torch.Tensor, sigma=None, output: str = "bf16",
                       raw: bool = False, design: int = 2) -> torch.Tensor:
        W = self.world_size
        shard = words.numel() // W
        f32 = output == "fp32"
        out = torch.empty(shard, dtype=torch.float32 if f32 else torch.int16, device=words.device)
        if shard == 0:
            return out
        err = torch.empty(W, dtype=torch.int32, device=words.device)
        if raw:
            rc = lib().zc_reduce_scatter_raw(self.handle, words.data_ptr(), shard, out.data_ptr(),
                                             int(f32), err.data_ptr(), stream_ptr())
            _status(self.handle, rc, "zc_reduce_scatter_raw")
        else:
            segs = [(q * shard, shard) for q in range(W) if q != self.rank]
            book = self._book(words, sigma, segs)
            rc = lib().zc_reduce_scatter(self.handle, words.data_ptr(), shard, out.data_ptr(),
                                         int(f32), book.data_ptr() if book is not None else None,
                                         err.data_ptr(), self._flags(design), stream_ptr())
            _status(self.handle, rc, "zc_reduce_scatter")
        self._finish(err)
        return out


def reduce_sources(sources, n: int, output: str, device) -> torch.Tensor:
    """Fused decode + fp32 reduction (zc_reduce_frames) over an arbitrary
    number of contributions, in list order: each source is ("raw", words) or
    ("frame", static_ptr, dynamic_ptr_or_0, dyn_len).  Returns the reduced
    shard (int16 words, or float32 for output="fp32")."""
    W = len(sources)
    rec = np.zeros(W, dtype=np.dtype([("stat", "<u8"), ("dyn", "<u8"), ("dyn_len", "<i8"),
                                      ("ready", "<u8"), ("raw", "<i4"), ("pad", "<i4")]))
    assert rec.itemsize == lib().zc_red_src_bytes()
    keep = []
    for i, s in enumerate(sources):
        if s[0] == "raw":
            t = s[1]
            keep.append(t)
            rec[i] = (t.data_ptr(), 0, -1, 0, 1, 0)
        else:
            rec[i] = (s[1], s[2], s[3], 0, 0, 0)
    src = torch.from_numpy(rec.view(np.uint8).copy()).to(device)
    scratch = torch.empty(max(int(lib().zc_reduce_scratch_bytes(W)), 8), dtype=torch.uint8,
                          device=device)
    f32 = output == "fp32"
    out = torch.empty(n, dtype=torch.float32 if f32 else torch.int16, device=device)
    err = torch.full((W,), engine.ERR_OK, dtype=torch.int32, device=device)
    if n:
        rc = lib().zc_reduce_frames(src.data_ptr(), W, n, out.data_ptr(), int(f32),
                                    scratch.data_ptr(), err.data_ptr(), stream_ptr())
        if rc != 0:
            raise RuntimeError(f"zc_reduce_frames failed: status {rc}")
    return out, err, keep
