"""Symmetric peer workspaces for the pull-decode collectives over NVLink.

Each rank owns one device buffer (allocated outside the caching allocator
with ``zc_alloc``) laid out as

    [0, 8*W)          ready[W]   u64 epochs written BY peers (their frame is ready)
    [8*W, 16*W)       done[W]    u64 epochs written BY peers (they finished reading mine)
    [256, ...)        frame region

Peers map it (CUDA IPC for processes, plain pointers for thread ranks) and
decode frames straight out of it (K5 pull-decode): the transfer and the
decode are one kernel, reading compressed bytes over NVLink.  Readiness is
signalled device-side with system-scope release stores / acquire polls
(csrc/zc_p2p.cu), so a call needs no host round trip once sizes are known.
This replaces the reference's send/recv transport seam (transport.py:559-623)
for the data path.
"""

from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib, ptrs, stream_ptr

HEADER_BYTES = 256


class _Raw:
    """A cudaMalloc'd block exposed to torch via __cuda_array_interface__."""

    def __init__(self, nbytes: int, device: torch.device):
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        with torch.cuda.device(device):
            check(lib().zc_alloc(self.nbytes, ctypes.byref(p)), "zc_alloc")
        self.ptr = int(p.value)
        self.device = device
        self.__cuda_array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1",
                                         "data": (self.ptr, False), "version": 3}

    def tensor(self) -> torch.Tensor:
        return torch.as_tensor(self, device=self.device)

    def free(self):
        if self.ptr:
            with torch.cuda.device(self.device):
                lib().zc_free(ctypes.c_void_p(self.ptr))
            self.ptr = 0


class PeerWorkspace:
    """One symmetric buffer per rank + the mapped pointers of all peers."""

    def __init__(self, comm, capacity: int):
        self.comm = comm
        self.W = comm.world_size
        self.capacity = int(capacity)
        self.epoch = 0
        self.raw = _Raw(HEADER_BYTES + self.capacity, comm.device)
        self.buf = self.raw.tensor()
        self.peer_base = self._exchange()

    @property
    def frame_ptr(self) -> int:
        return self.raw.ptr + HEADER_BYTES

    def frame_tensor(self, nbytes: int) -> torch.Tensor:
        return self.buf[HEADER_BYTES:HEADER_BYTES + nbytes]

    def _exchange(self) -> list:
        from .transport import HubCommunicator
        comm = self.comm
        if isinstance(comm, HubCommunicator):
            # thread ranks in one process: pointers are directly usable
            return [int(v) for v in comm._post_and_collect(self.raw.ptr)]
        nb = lib().zc_ipc_handle_bytes()
        h = (ctypes.c_uint8 * nb)()
        check(lib().zc_ipc_get_handle(ctypes.c_void_p(self.raw.ptr), h), "zc_ipc_get_handle")
        import torch.distributed as dist
        handles = [None] * self.W
        dist.all_gather_object(handles, bytes(h), group=comm.group)
        bases = []
        self._opened = []
        for p, hb in enumerate(handles):
            if p == comm.rank:
                bases.append(self.raw.ptr)
                continue
            out = ctypes.c_void_p()
            buf = (ctypes.c_uint8 * nb).from_buffer_copy(hb)
            check(lib().zc_ipc_open_handle(buf, ctypes.byref(out)), "zc_ipc_open_handle")
            bases.append(int(out.value))
            self._opened.append(int(out.value))
        return bases

    # -- device-side signalling ---------------------------------------------------
    def signal(self, slot: int, epoch: int, stream=None) -> None:
        """Write `epoch` into flag array `slot` (0 ready, 1 done) of every peer."""
        flags = [b + 8 * self.W * slot for b in self.peer_base]
        check(lib().zc_signal_peers(ptrs(flags), self.W, self.comm.rank, int(epoch),
                                    stream_ptr(stream)), "zc_signal_peers")

    def wait(self, slot: int, epoch: int, err: torch.Tensor, timeout_s: float = 20.0,
             stream=None) -> None:
        """Device-side wait until every peer wrote >= epoch into my slot array."""
        check(lib().zc_wait_signals(ctypes.c_void_p(self.raw.ptr + 8 * self.W * slot), self.W,
                                    self.comm.rank, int(epoch), int(timeout_s * 1e9),
                                    ctypes.c_void_p(err.data_ptr()), stream_ptr(stream)),
              "zc_wait_signals")

    def close(self):
        for p in getattr(self, "_opened", []):
            lib().zc_ipc_close_handle(ctypes.c_void_p(p))
        self._opened = []
        self.raw.free()


def workspace_for(comm, frame_bytes: int) -> PeerWorkspace:
    """The communicator's symmetric workspace, grown (collectively) to hold
    ``frame_bytes``.  All ranks must call with the same value."""
    ws = getattr(comm, "_peer_ws", None)
    if ws is not None and ws.capacity >= frame_bytes:
        return ws
    if ws is not None:
        comm.barrier()
        ws.close()
    cap = max(int(frame_bytes), 1 << 20)
    cap = (cap + (1 << 20) - 1) // (1 << 20) * (1 << 20)
    ws = PeerWorkspace(comm, cap)
    comm._peer_ws = ws
    comm.barrier()
    return ws
