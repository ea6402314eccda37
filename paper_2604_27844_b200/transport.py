"""Communicator seam — replaces reference transport.py (Communicator,
exchange_sizes, TrafficStats, run_ranks; transport.py:46-88, :559-671).

The reference moves bytes with Python sockets and queues.  Here the host
side agrees on sizes and the device side moves frames:

* ``DistCommunicator`` wraps a ``torch.distributed`` process group.  With the
  NCCL backend the byte movers are NCCL collectives / grouped send-recv over
  NVLink on device tensors; with gloo (CPU tests, or several ranks sharing
  one GPU) they stage through host memory.
* ``HubCommunicator`` binds in-process thread ranks (``run_ranks``), the
  analogue of the reference's loopback hub: frames move with device copies.

Every communicator keeps the reference's ``TrafficStats`` byte counters.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import torch

from .errors import ProtocolError, TransportError

DEFAULT_TIMEOUT = 30.0


@dataclass
class TrafficStats:
    """Bytes this rank put on the wire (reference transport.py:559-573)."""

    bytes_sent: int = 0
    bytes_received: int = 0
    messages_sent: int = 0

    def snapshot(self) -> "TrafficStats":
        return TrafficStats(self.bytes_sent, self.bytes_received, self.messages_sent)

    def delta(self, earlier: "TrafficStats") -> "TrafficStats":
        return TrafficStats(self.bytes_sent - earlier.bytes_sent,
                            self.bytes_received - earlier.bytes_received,
                            self.messages_sent - earlier.messages_sent)


class Communicator:
    """A rank bound into a group of ``world_size`` peers (transport.py:576-623).

    ``native`` (when set) is the rank's NativeComm: the collectives then run
    the C++ engine (native.py); ``use_native = False`` forces the generic
    Python protocols over this communicator's byte movers."""

    rank: int
    world_size: int
    device: torch.device
    native = None
    use_native = True

    def __init__(self):
        self._stats = TrafficStats()

    @property
    def stats(self) -> TrafficStats:
        """Bytes this rank put on the wire: the generic protocols' counters
        plus the native engine's (host-side message plane, device-side
        peer-memory plane; reading them synchronises the device)."""
        s = self._stats.snapshot()
        nat = self.__dict__.get("native") or self.__dict__.get("_native")
        if nat is not None:
            b, m = nat.stats()
            s.bytes_sent += b
            s.messages_sent += m
        return s

    # -- reference surface -------------------------------------------------------
    def peers(self) -> list:
        return [r for r in range(self.world_size) if r != self.rank]

    def now(self) -> float:
        return time.perf_counter()

    def exchange_sizes(self, local_sizes, tag: int = 0) -> list:
        """All-to-all of one u64 per peer; entry p is what peer p declared for
        this rank, the self entry passes through (transport.py:607-623)."""
        sizes = [int(s) for s in local_sizes]
        if len(sizes) != self.world_size:
            raise ValueError(f"expected {self.world_size} sizes, got {len(sizes)}")
        got = self._a2a_ints(sizes)
        got[self.rank] = sizes[self.rank]
        self._count(8 * (self.world_size - 1), self.world_size - 1)
        return got

    def allgather_ints(self, value: int) -> list:
        return self._allgather_ints(int(value))

    def allgather_vec(self, values) -> list:
        """All-gather a short int vector per rank; row p is rank p's."""
        return self._allgather_vec([int(v) for v in values])

    # -- byte movers (device tensors) ------------------------------------------
    def all_gather_bytes(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        """recv[p*len(send):(p+1)*len(send)] = send of rank p (equal sizes)."""
        raise NotImplementedError

    def sendrecv_bytes(self, sends: dict, recvs: dict, label: str = "message") -> None:
        """Grouped point-to-point: sends {peer: tensor}, recvs {peer: tensor}.

        Receive sizes are the receiver's expectation (the reference's
        pre-sized receives, collectives.py:294-305).  Transports that can see
        both sides (the thread hub) raise ProtocolError naming ``label`` on a
        size disagreement; NCCL cannot, so callers that need the check agree
        on sizes first (``comm.check_counts``)."""
        raise NotImplementedError

    def barrier(self) -> None:
        raise NotImplementedError

    # -- helpers -----------------------------------------------------------------
    def _count(self, nbytes: int, nmsg: int = 1) -> None:
        self._stats.bytes_sent += int(nbytes)
        self._stats.messages_sent += int(nmsg)

    @classmethod
    def from_process_group(cls, group=None, device=None) -> "DistCommunicator":
        return DistCommunicator(group, device)


class DistCommunicator(Communicator):
    """Over a torch.distributed group: NCCL moves device bytes over NVLink."""

    def __init__(self, group=None, device=None):
        super().__init__()
        import torch.distributed as dist
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world_size = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) \
                if torch.cuda.is_available() else torch.device("cpu")
        self.device = torch.device(device)
        self.on_device = self.backend == "nccl"
        self._native = None

    @property
    def native(self):
        """Native engine over this NCCL group, created (collectively) by the
        first collective that needs it; None on gloo (the generic path)."""
        if not self.on_device or not self.use_native:
            return None
        if self._native is None:
            from .native import NativeComm
            self._native = NativeComm.from_process_group(self.group, self.device)
        return self._native

    def _wire(self, t: torch.Tensor) -> torch.Tensor:
        return t if self.on_device else t.cpu()

    def _allgather_ints(self, value: int) -> list:
        dev = self.device if self.on_device else torch.device("cpu")
        src = torch.tensor([value], dtype=torch.int64, device=dev)
        out = torch.empty(self.world_size, dtype=torch.int64, device=dev)
        self._dist.all_gather_into_tensor(out, src, group=self.group)
        return [int(v) for v in out.cpu().tolist()]

    def _allgather_vec(self, values: list) -> list:
        dev = self.device if self.on_device else torch.device("cpu")
        src = torch.tensor(values, dtype=torch.int64, device=dev)
        out = torch.empty(self.world_size * len(values), dtype=torch.int64, device=dev)
        self._dist.all_gather_into_tensor(out, src, group=self.group)
        flat = [int(v) for v in out.cpu().tolist()]
        k = len(values)
        return [flat[p * k:(p + 1) * k] for p in range(self.world_size)]

    def _a2a_ints(self, sizes: list) -> list:
        dev = self.device if self.on_device else torch.device("cpu")
        src = torch.tensor(sizes, dtype=torch.int64, device=dev)
        out = torch.empty(self.world_size, dtype=torch.int64, device=dev)
        self._dist.all_to_all_single(out, src, group=self.group)
        return [int(v) for v in out.cpu().tolist()]

    def all_gather_bytes(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        if self.on_device:
            self._dist.all_gather_into_tensor(recv, send, group=self.group)
        else:
            r = torch.empty(recv.numel(), dtype=recv.dtype)
            self._dist.all_gather_into_tensor(r, send.cpu(), group=self.group)
            recv.copy_(r)
        self._count(send.numel() * send.element_size() * (self.world_size - 1),
                    self.world_size - 1)

    def sendrecv_bytes(self, sends: dict, recvs: dict, label: str = "message") -> None:
        dist = self._dist
        staged = {}
        ops = []
        for p, t in sends.items():
            if t.numel():
                ops.append(dist.P2POp(dist.isend, self._wire(t.contiguous()), p, self.group))
                self._count(t.numel() * t.element_size())
        for p, t in recvs.items():
            if t.numel():
                buf = t if self.on_device else torch.empty(t.numel(), dtype=t.dtype)
                staged[p] = buf
                ops.append(dist.P2POp(dist.irecv, buf, p, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if not self.on_device:
            for p, buf in staged.items():
                recvs[p].copy_(buf)

    def barrier(self) -> None:
        self._dist.barrier(group=self.group)


class _Hub:
    """Shared state of in-process thread ranks (reference _LoopbackHub,
    transport.py:46-88).  Exchanges are keyed by a per-rank generation
    counter, so an abort only reaches ranks that are still waiting."""

    def __init__(self, world_size: int):
        self.world_size = world_size
        self.cond = threading.Condition()
        self.gen = [0] * world_size
        self.slots: dict = {}
        self.error: BaseException | None = None

    def exchange(self, rank: int, obj) -> list:
        with self.cond:
            g = self.gen[rank]
            self.gen[rank] += 1
            self.slots.setdefault(g, {})[rank] = obj
            self.cond.notify_all()
            while len(self.slots[g]) < self.world_size:
                if self.error is not None:
                    raise TransportError(f"communicator aborted: {self.error}")
                if not self.cond.wait(timeout=DEFAULT_TIMEOUT):
                    from .errors import TransportTimeout
                    raise TransportTimeout(f"rank {rank} timed out in exchange {g}")
            vals = [self.slots[g][r] for r in range(self.world_size)]
            # every rank that posted g has finished reading g - 1
            self.slots.pop(g - 1, None)
            return vals

    def abort(self, exc: BaseException) -> None:
        with self.cond:
            if self.error is None:
                self.error = exc
            self.cond.notify_all()

    def sync(self, rank: int) -> None:
        self.exchange(rank, None)


class HubCommunicator(Communicator):
    """Thread rank on a shared hub; each rank has its own CUDA stream."""

    def __init__(self, hub: _Hub, rank: int, device, native=None):
        super().__init__()
        self.hub = hub
        self.rank = rank
        self.world_size = hub.world_size
        self.device = torch.device(device)
        self.stream = torch.cuda.Stream(device=self.device)
        self.native = native

    def _post_and_collect(self, obj) -> list:
        return self.hub.exchange(self.rank, obj)

    def _allgather_ints(self, value: int) -> list:
        return [int(v) for v in self._post_and_collect(int(value))]

    def _allgather_vec(self, values: list) -> list:
        return [list(r) for r in self._post_and_collect(list(values))]

    def _a2a_ints(self, sizes: list) -> list:
        rows = self._post_and_collect(list(sizes))
        return [int(rows[p][self.rank]) for p in range(self.world_size)]

    def all_gather_bytes(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        torch.cuda.current_stream(self.device).synchronize()
        srcs = self._post_and_collect(send)
        n = send.numel()
        for p, src in enumerate(srcs):
            if src.numel() != n:
                raise ProtocolError(f"all-gather size mismatch with rank {p}")
            recv[p * n:(p + 1) * n].copy_(src)
        torch.cuda.current_stream(self.device).synchronize()
        self.hub.sync(self.rank)
        self._count(n * send.element_size() * (self.world_size - 1), self.world_size - 1)

    def sendrecv_bytes(self, sends: dict, recvs: dict, label: str = "message") -> None:
        torch.cuda.current_stream(self.device).synchronize()
        posted = self._post_and_collect({p: t for p, t in sends.items() if t.numel()})
        bad = None
        for p in self.peers():
            src = posted[p].get(self.rank)
            got = 0 if src is None else src.numel()
            t = recvs.get(p)
            want = 0 if t is None else t.numel()
            if got != want:
                bad = bad or (p, got, want)
            elif want:
                t.copy_(src)
        if bad is not None:
            p, got, want = bad
            raise ProtocolError(f"{label} from rank {p} is {got} bytes, expected {want}")
        torch.cuda.current_stream(self.device).synchronize()
        self.hub.sync(self.rank)
        for t in sends.values():
            if t.numel():
                self._count(t.numel() * t.element_size())

    def barrier(self) -> None:
        torch.cuda.current_stream(self.device).synchronize()
        self.hub.sync(self.rank)


MODE_PARALLEL = "full-p2p-parallel"
MODE_SERIALIZED = "serialized-links"
RENDEZVOUS_ENV = "ZIPCOLL_RENDEZVOUS"


@dataclass
class SimProfile:
    """The reference's simulated-fabric parameters (transport.py:96-126),
    accepted for API compatibility.  The virtual-clock transport itself is
    not part of this build (out of scope) -- collectives here
    are timed on the device -- so run_ranks(..., transport="sim") raises."""

    bandwidth: float = 1e9
    latency: float = 10e-6
    mode: str = MODE_PARALLEL
    ready_times: dict = field(default_factory=dict)
    link_bandwidth: dict = field(default_factory=dict)
    link_latency: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.bandwidth <= 0 or any(b <= 0 for b in self.link_bandwidth.values()):
            raise ValueError("bandwidth must be positive")
        if self.latency < 0 or any(v < 0 for v in self.link_latency.values()):
            raise ValueError("latency must be nonnegative")
        if any(t < 0 for t in self.ready_times.values()):
            raise ValueError("ready_time must be nonnegative")
        if self.mode not in (MODE_PARALLEL, MODE_SERIALIZED):
            raise ValueError(f"unknown concurrency mode {self.mode!r}")


def connect_tcp(world_size: int, rank: int, rendezvous: str | None = None,
                timeout: float = DEFAULT_TIMEOUT) -> Communicator:
    """Reference connect_tcp (transport.py:669-671): this rank joins a group
    of ``world_size`` ranks meeting at ``rendezvous`` ("host:port", else
    $ZIPCOLL_RENDEZVOUS).  Here the meeting is torch.distributed's TCP
    store and the group is NCCL when a GPU is visible (one process per GPU,
    device = rank modulo the visible GPUs; the native engine then runs over
    NVLink), gloo otherwise."""
    import datetime
    import os
    import socket
    import torch.distributed as dist
    rendezvous = rendezvous or os.environ.get(RENDEZVOUS_ENV)
    if world_size > 1 and not rendezvous:
        raise TransportError(f"tcp transport needs a rendezvous address ({RENDEZVOUS_ENV})")
    if not rendezvous:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            rendezvous = f"127.0.0.1:{sk.getsockname()[1]}"
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(rank % torch.cuda.device_count())
    try:
        dist.init_process_group(backend, init_method=f"tcp://{rendezvous}",
                                world_size=world_size, rank=rank,
                                timeout=datetime.timedelta(seconds=timeout))
    except Exception as exc:  # noqa: BLE001 - the reference's error class
        raise TransportError(f"tcp rendezvous at {rendezvous} failed: {exc}") from exc
    return DistCommunicator()


def run_ranks(world_size: int, fn, transport: str = "loopback",
              sim_profile: SimProfile | None = None, timeout: float = DEFAULT_TIMEOUT, *,
              device=None, native: bool | None = None) -> list:
    """Run fn(comm) on ``world_size`` in-process thread ranks sharing one GPU
    (or ``device`` per rank when a list is given); results by rank
    (reference run_ranks, transport.py:635-666, same positional arguments).
    The first failure aborts the hub so peers error out instead of hanging,
    and is re-raised.  ``transport`` "loopback" (the reference's in-process
    hub) is the thread-rank hub here; "sim" (virtual clock) is not provided.

    ``native`` (default: up to 64 ranks) gives every rank a native
    communicator of one in-process group, so the collectives run the C++
    engine exactly as NCCL ranks do; False keeps the generic protocols."""
    if transport == "sim" or sim_profile is not None:
        raise TransportError("the simulated (virtual-clock) transport is not part of the B200 "
                             "build: collectives are timed on the device")
    if transport != "loopback":
        raise ValueError(f"unknown transport {transport!r}")
    hub = _Hub(world_size)
    results = [None] * world_size
    failures = []
    devs = device if isinstance(device, (list, tuple)) else [device] * world_size
    devs = [d if d is not None else torch.device("cuda", 0) for d in devs]
    if native is None:
        native = 1 < world_size <= 64
    comms = None
    if native:
        from .native import NativeComm
        comms = NativeComm.local_group(world_size, devs)

    def body(rank: int) -> None:
        dev = devs[rank]
        torch.cuda.set_device(dev)
        comm = HubCommunicator(hub, rank, dev, comms[rank] if comms else None)
        try:
            with torch.cuda.stream(comm.stream):
                results[rank] = fn(comm)
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001 - propagated to the caller
            failures.append((rank, exc))
            hub.abort(exc)
            for c in comms or ():
                c.abort()

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world_size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=timeout * 10)
    if comms:
        for c in comms:
            c.close()
    if failures:
        rank, exc = min(failures, key=lambda f: f[0])
        raise exc
    return results
