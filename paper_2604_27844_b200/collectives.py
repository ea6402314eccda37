"""Compressed collectives — drop-in for reference collectives.py:1-376.

Same semantics as the reference (outputs bit-identical to the uncompressed
collectives, rank-order results, same exception classes), with the element
work on the GPU.  Two implementations of the same protocols:

* native (``comm.native`` set: NCCL process groups and thread ranks): the
  C++ engine of csrc/zc_coll.cu (see native.py) -- the peer-memory plane
  (the decoder pulls every peer's frame over NVLink as soon as that peer
  published it; no host round trip) or the message plane (the reference's
  size phase / design-1 / design-2 protocols over NCCL);
* generic (any ``Communicator`` byte movers: gloo, or thread ranks with
  ``native=False``): the same protocols driven from Python.

* ``zip_all_gather``: codebook (K1) + encode (K2) of the local shard, the
  reference's size phase (8 B per peer), frames, ONE batched decode (K3)
  straight into the output (reference collectives.py:203-227).
* ``zip_all_to_all_d1`` / ``_d2``: one codebook over the non-self, non-empty
  chunks (collectives.py:230-242), all peer frames encoded by ONE batched K4
  launch; design 1 = 16 B of metadata per peer then frames, design 2 =
  static sections pre-sized from recv_counts with no metadata, then 8 B
  dynamic sizes, then dynamic sections (collectives.py:245-325) -- the
  reference's wire accounting (d1 - d2 = 8 B per peer).
* ``zip_reduce_scatter`` / ``zip_all_reduce``: design-2
  all-to-all then ONE fused decode + float32 reduction in ascending rank
  order with the reference's RNE narrowing and NaN rule (zc_reduce.cu).
"""

from __future__ import annotations


import numpy as np
import torch

from . import bf16, codec, engine
from .codec import device_words
from .errors import CollectiveError, ProtocolError
from .transport import Communicator, DistCommunicator, HubCommunicator, run_ranks  # noqa: F401

GS_LOG2 = 9   # collectives always frame with the default group size (collectives.py:281-287)


class AlltoAllSpec:
    """Per-peer send chunks and expected receive counts (collectives.py:55-74)."""

    def __init__(self, send_chunks, recv_counts):
        self.send_chunks = tuple(send_chunks)
        self.recv_counts = tuple(int(c) for c in recv_counts)
        if len(self.send_chunks) != len(self.recv_counts):
            raise ValueError("send_chunks and recv_counts must have equal length")
        if any(c < 0 for c in self.recv_counts):
            raise ValueError("recv counts must be nonnegative")

    @property
    def world_size(self) -> int:
        return len(self.send_chunks)


def _check_world(comm: Communicator, spec_world: int) -> None:
    if spec_world != comm.world_size:
        raise ValueError(f"spec is for world {spec_world}, communicator has {comm.world_size}")


def _dev(comm: Communicator):
    return comm.device


def _pack(chunks, device):
    """Concatenate per-peer word chunks into one device buffer; returns
    (buffer, offsets, counts)."""
    words = [device_words(c, device) for c in chunks]
    counts = [w.numel() for w in words]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    if not sum(counts):
        return torch.empty(0, dtype=torch.int16, device=device), [int(o) for o in offs[:-1]], counts
    live = [w for w in words if w.numel()]
    base = live[0]
    consecutive = all(w.untyped_storage().data_ptr() == base.untyped_storage().data_ptr()
                      for w in live) and all(
        a.data_ptr() + 2 * a.numel() == b.data_ptr() for a, b in zip(live, live[1:]))
    if consecutive:   # views of one send buffer (MoE dispatch): no copy
        start = base.storage_offset()
        flat = base.new_empty(0).set_(base.untyped_storage(), start, (int(offs[-1]),), (1,))
        return flat, [int(o) for o in offs[:-1]], counts
    return torch.cat(words), [int(o) for o in offs[:-1]], counts


def _native(comm: Communicator):
    """The communicator's native engine, or None for the generic path."""
    if not getattr(comm, "use_native", True):
        return None
    return getattr(comm, "native", None)


def _raise_decode_errors(err: torch.Tensor, peers: list) -> None:
    codes = err.cpu().tolist()
    for code, peer in zip(codes, peers):
        if code != engine.ERR_OK:
            if code == 19:
                raise CollectiveError("frame holds a different element count than expected",
                                      peer=peer)
            raise CollectiveError(f"corrupt frame: {engine.err_message(code)}", peer=peer)


# ---------------------------------------------------------------------------
# reference (uncompressed) collectives: the oracles and the switcher's raw path

def reference_all_gather(comm: Communicator, local) -> torch.Tensor:
    """Raw all-gather (collectives.py:97-111): element counts agreed (once
    per shape on NCCL communicators), then ncclAllGather / device copies."""
    words = device_words(local, _dev(comm))
    if comm.world_size == 1:
        return words.clone()
    native = _native(comm)
    if native is not None:
        agreed = comm.__dict__.setdefault("_agreed_ag", set())
        if words.numel() not in agreed or native.check_counts:
            counts = comm.allgather_ints(words.numel())
            for p, c in enumerate(counts):
                if c != words.numel():
                    raise ProtocolError(f"all-gather element count mismatch: rank {comm.rank} "
                                        f"has {words.numel()}, rank {p} declared {c}")
            agreed.add(words.numel())
        return native.all_gather_raw(words)
    counts = comm.allgather_ints(words.numel())
    for p, c in enumerate(counts):
        if c != words.numel():
            raise ProtocolError(f"all-gather element count mismatch: rank {comm.rank} has "
                                f"{words.numel()}, rank {p} declared {c}")
    out = torch.empty(comm.world_size * words.numel(), dtype=torch.int16, device=words.device)
    comm.all_gather_bytes(words.view(torch.uint8), out.view(torch.uint8))
    return out


def reference_all_to_all(comm: Communicator, spec: AlltoAllSpec) -> list:
    """Raw all-to-all (collectives.py:114-134) over grouped send/recv."""
    _check_world(comm, spec.world_size)
    dev = _dev(comm)
    if comm.world_size == 1:
        return [device_words(spec.send_chunks[0], dev).clone()]
    buf, offs, counts = _pack(spec.send_chunks, dev)
    native = _native(comm)
    if native is not None:
        saved, native.check_counts = native.check_counts, True   # the reference's size phase
        try:
            return native.all_to_all_raw(buf, counts, spec.recv_counts)
        finally:
            native.check_counts = saved
    declared = comm.exchange_sizes(counts)
    for p in comm.peers():
        if declared[p] != spec.recv_counts[p]:
            raise ProtocolError(f"rank {p} will send {declared[p]} elements, "
                                f"rank {comm.rank} expected {spec.recv_counts[p]}")
    out = [torch.empty(c, dtype=torch.int16, device=dev) for c in spec.recv_counts]
    sends = {p: buf[offs[p]:offs[p] + counts[p]].view(torch.uint8) for p in comm.peers()}
    recvs = {p: out[p].view(torch.uint8) for p in comm.peers()}
    comm.sendrecv_bytes(sends, recvs)
    out[comm.rank] = buf[offs[comm.rank]:offs[comm.rank] + counts[comm.rank]].clone()
    return out


def _reduce_chunks(chunks: list, output: str) -> torch.Tensor:
    """float32 sum in list (= ascending rank) order (collectives.py:137-144)
    with numpy's NaN propagation and the reference's RNE narrowing: one
    launch of the fused reduce kernel over raw word sources."""
    from .native import reduce_sources
    n = chunks[0].numel()
    out, _, _ = reduce_sources([("raw", c.contiguous()) for c in chunks], n, output,
                               chunks[0].device)
    return out


def _split_shards(comm: Communicator, local) -> list:
    words = device_words(local, _dev(comm))
    if words.numel() % comm.world_size:
        raise ValueError(f"input of {words.numel()} elements is not divisible into "
                         f"{comm.world_size} shards")
    shard = words.numel() // comm.world_size
    return [words[r * shard:(r + 1) * shard] for r in range(comm.world_size)]


def reference_reduce_scatter(comm: Communicator, local, output: str = "bf16") -> torch.Tensor:
    """Raw all-to-all of the shards + the float32 reduction (collectives.py:147-170)."""
    shards = _split_shards(comm, local)
    if comm.world_size == 1:
        return _reduce_chunks(shards, output)
    native = _native(comm)
    if native is not None:
        _agree_shard(comm, shards[0].numel())
        return native.reduce_scatter(device_words(local, _dev(comm)), None, output, raw=True)
    spec = AlltoAllSpec(shards, [shards[0].numel()] * comm.world_size)
    return _reduce_chunks(reference_all_to_all(comm, spec), output)


# ---------------------------------------------------------------------------
# compressed collectives

def zip_all_gather(comm: Communicator, local, sigma: float | None = None) -> torch.Tensor:
    """All-gather with compressed payloads, bit-identical to the reference
    all-gather (collectives.py:203-227).

    Over a generic communicator (thread hub, gloo): K1+K2 encode the local
    shard into one frame; ONE exchange carries (element count, frame bytes)
    per rank -- the reference's size phase (8 B/peer of frame length) plus
    the count the reference checks when it parses the peer frame; the static
    sections (equal size, a function of n) move in one all-gather, the
    dynamic sections point to point at their exact sizes; ONE batched K3
    launch decodes every peer frame into the output."""
    dev = _dev(comm)
    words = device_words(local, dev)
    n = words.numel()
    W = comm.world_size
    if W == 1:
        return words.clone()
    native = _native(comm)
    if native is not None and n > 0:
        return native.all_gather(words, sigma)
    if n == 0:
        rows = comm.allgather_vec([0, 0])
        comm._count(8 * (W - 1), W - 1)
        for p, (c, _) in enumerate(rows):
            if c != 0:
                raise ProtocolError(f"all-gather frame size mismatch: rank {comm.rank} has 0, "
                                    f"rank {p} declared {c}")
        return torch.empty(0, dtype=torch.int16, device=dev)
    S = engine.static_bytes(n, GS_LOG2)
    frame = torch.empty(engine.max_frame_bytes(n, GS_LOG2), dtype=torch.uint8, device=dev)
    _, flen = codec.device_encode(words, [(0, n)], sigma, frame, [0], GS_LOG2)
    rows = comm.allgather_vec([n, int(flen.item())])
    comm._count(8 * (W - 1), W - 1)
    for p, (c, _) in enumerate(rows):
        if c != n:
            raise CollectiveError(f"frame holds {c} elements, expected {n}", peer=p)
    dyn_lens = [fl - S for _, fl in rows]
    static = torch.empty(W * S, dtype=torch.uint8, device=dev)
    comm.all_gather_bytes(frame[:S], static)
    dyn = torch.empty(max(sum(dyn_lens), 1), dtype=torch.uint8, device=dev)
    doff = np.concatenate([[0], np.cumsum(dyn_lens)]).astype(np.int64)
    me = comm.rank
    own = frame[S:S + dyn_lens[me]]
    comm.sendrecv_bytes({p: own for p in comm.peers()},
                        {p: dyn[int(doff[p]):int(doff[p + 1])] for p in comm.peers()},
                        label="dynamic section")
    out = torch.empty(W * n, dtype=torch.int16, device=dev)
    peers = comm.peers()
    err = engine.decode([static.data_ptr() + p * S for p in peers],
                        [dyn.data_ptr() + int(doff[p]) for p in peers],
                        [dyn_lens[p] for p in peers], [n] * len(peers), out,
                        [p * n for p in peers], groups512=True)
    out[me * n:(me + 1) * n].copy_(words)
    _raise_decode_errors(err, peers)
    return out


def _prepare_frames(comm: Communicator, buf, offs, counts, sigma):
    """One codebook per call over the non-self, non-empty chunks
    (collectives.py:230-242); one batched encode launch for all peer frames.
    Returns (frames, frame_off per peer, frame_len per peer (host))."""
    dev = _dev(comm)
    peers = [q for q in range(comm.world_size) if q != comm.rank and counts[q]]
    frame_off = [0] * comm.world_size
    if not peers:
        return None, frame_off, [0] * comm.world_size
    segs = [(offs[q], counts[q]) for q in peers]
    caps = [engine.max_frame_bytes(counts[q], GS_LOG2) for q in peers]
    pos = 0
    for q, c in zip(peers, caps):
        frame_off[q] = pos
        pos += c
    frames = torch.empty(pos, dtype=torch.uint8, device=dev)
    _, flen = codec.device_encode(buf, segs, sigma, frames, [frame_off[q] for q in peers], GS_LOG2)
    lens = flen.cpu().tolist()
    frame_len = [0] * comm.world_size
    for q, ln in zip(peers, lens):
        frame_len[q] = int(ln)
    return frames, frame_off, frame_len


def _finish_a2a(comm, spec, buf, offs, counts, recv, peers_in, stat_ptrs, dyn_ptrs, dyn_lens):
    dev = _dev(comm)
    out_counts = [spec.recv_counts[p] for p in peers_in]
    total = sum(spec.recv_counts)
    flat = torch.empty(max(total, 1), dtype=torch.int16, device=dev)
    roffs = np.concatenate([[0], np.cumsum(spec.recv_counts)]).astype(np.int64)
    if peers_in:
        err = engine.decode(stat_ptrs, dyn_ptrs, dyn_lens, out_counts, flat,
                            [int(roffs[p]) for p in peers_in], groups512=True)
        _raise_decode_errors(err, peers_in)
    result = [flat[int(roffs[p]):int(roffs[p]) + spec.recv_counts[p]]
              for p in range(comm.world_size)]
    me = comm.rank
    result[me] = buf[offs[me]:offs[me] + counts[me]].clone()
    return result


def _agree_counts(comm: Communicator, spec: AlltoAllSpec, counts, what: str):
    declared = comm.exchange_sizes(counts)
    for p in comm.peers():
        if declared[p] != spec.recv_counts[p]:
            if what == "static":
                got = codec.static_size_bytes(declared[p]) if declared[p] else 0
                want = codec.static_size_bytes(spec.recv_counts[p]) if spec.recv_counts[p] else 0
                raise ProtocolError(f"static section from rank {p} is {got} bytes, "
                                    f"expected {want}")
            raise ProtocolError(f"rank {p} will send {declared[p]} elements, "
                                f"rank {comm.rank} expected {spec.recv_counts[p]}")


def zip_all_to_all_d1(comm: Communicator, spec: AlltoAllSpec,
                      sigma: float | None = None) -> list:
    """Design 1 (collectives.py:245-278): metadata (count, frame bytes) per
    peer -- 16 B, as two u64 exchanges -- then whole frames, then one batched
    decode."""
    _check_world(comm, spec.world_size)
    dev = _dev(comm)
    if comm.world_size == 1:
        return [device_words(spec.send_chunks[0], dev).clone()]
    buf, offs, counts = _pack(spec.send_chunks, dev)
    native = _native(comm)
    if native is not None:
        return native.all_to_all(buf, counts, spec.recv_counts, sigma, design=1)
    _agree_counts(comm, spec, counts, "count")
    frames, frame_off, frame_len = _prepare_frames(comm, buf, offs, counts, sigma)
    got_len = comm.exchange_sizes(frame_len)
    for p in comm.peers():
        want = spec.recv_counts[p]
        if want == 0:
            if got_len[p]:
                raise CollectiveError(f"expected an empty frame, got {got_len[p]} bytes", peer=p)
            continue
        s = codec.static_size_bytes(want)
        if got_len[p] < s or got_len[p] % 128:
            raise CollectiveError(f"frame length {got_len[p]} cannot hold {want} elements",
                                  peer=p)
    recv_bufs = {p: torch.empty(got_len[p], dtype=torch.uint8, device=dev)
                 for p in comm.peers() if spec.recv_counts[p]}
    sends = {p: frames[frame_off[p]:frame_off[p] + frame_len[p]]
             for p in comm.peers() if frame_len[p]}
    comm.sendrecv_bytes(sends, recv_bufs, label="frame")
    peers_in = sorted(recv_bufs)
    return _finish_a2a(comm, spec, buf, offs, counts, recv_bufs, peers_in,
                       [recv_bufs[p].data_ptr() for p in peers_in], [0] * len(peers_in),
                       [got_len[p] - codec.static_size_bytes(spec.recv_counts[p])
                        for p in peers_in])


def zip_all_to_all_d2(comm: Communicator, spec: AlltoAllSpec,
                      sigma: float | None = None) -> list:
    """Design 2 (collectives.py:281-325): static sections first, receives
    pre-sized from recv_counts with NO metadata (the property design 2
    exists for), then the u64 dynamic sizes (8 B/peer),
    then the dynamic sections; frames are decoded from the split receive
    buffers in place.  A sender whose count disagrees with the receiver's
    expectation is caught by the transport's size check (thread hub:
    ProtocolError "static section ...") or by the frame header
    (CollectiveError); ``comm.check_counts = True`` adds an explicit count
    agreement first, for transports that cannot see mismatched sizes."""
    _check_world(comm, spec.world_size)
    dev = _dev(comm)
    if comm.world_size == 1:
        return [device_words(spec.send_chunks[0], dev).clone()]
    buf, offs, counts = _pack(spec.send_chunks, dev)
    native = _native(comm)
    if native is not None:
        return native.all_to_all(buf, counts, spec.recv_counts, sigma, design=2)
    if getattr(comm, "check_counts", False):
        _agree_counts(comm, spec, counts, "static")
    frames, frame_off, frame_len = _prepare_frames(comm, buf, offs, counts, sigma)
    peers_out = [p for p in comm.peers() if frame_len[p]]
    peers_in = [p for p in comm.peers() if spec.recv_counts[p]]
    s_out = {p: codec.static_size_bytes(counts[p]) for p in peers_out}
    s_in = {p: codec.static_size_bytes(spec.recv_counts[p]) for p in peers_in}
    statics = {p: torch.empty(s_in[p], dtype=torch.uint8, device=dev) for p in peers_in}
    comm.sendrecv_bytes({p: frames[frame_off[p]:frame_off[p] + s_out[p]] for p in peers_out},
                        statics, label="static section")
    dyn_len = [frame_len[p] - s_out[p] if p in s_out else 0 for p in range(comm.world_size)]
    got_dyn = comm.exchange_sizes(dyn_len)
    for p in peers_in:
        if got_dyn[p] % 128:
            raise CollectiveError(f"dynamic section of {got_dyn[p]} bytes is not 128-aligned",
                                  peer=p)
    dyns = {p: torch.empty(got_dyn[p], dtype=torch.uint8, device=dev)
            for p in peers_in if got_dyn[p]}
    comm.sendrecv_bytes({p: frames[frame_off[p] + s_out[p]:frame_off[p] + frame_len[p]]
                         for p in peers_out if dyn_len[p]}, dyns, label="dynamic section")
    return _finish_a2a(comm, spec, buf, offs, counts, None, peers_in,
                       [statics[p].data_ptr() for p in peers_in],
                       [dyns[p].data_ptr() if p in dyns else statics[p].data_ptr()
                        for p in peers_in],
                       [got_dyn[p] for p in peers_in])


def _agree_shard(comm: Communicator, shard: int) -> None:
    """Reduce-scatter shard lengths agree (reference _agree_u64,
    collectives.py:83-90, :153); once per shape on native communicators."""
    agreed = comm.__dict__.setdefault("_agreed_rs", set())
    if shard in agreed:
        return
    for p, c in enumerate(comm.allgather_ints(shard)):
        if c != shard:
            raise ProtocolError(f"reduce-scatter shard length mismatch: rank {comm.rank} has "
                                f"{shard}, rank {p} declared {c}")
    agreed.add(shard)


def zip_reduce_scatter(comm: Communicator, local, sigma: float | None = None,
                       output: str = "bf16") -> torch.Tensor:
    """Compressed all-to-all (design 2) + float32 reduction in ascending rank
    order (collectives.py:328-341): on native communicators one fused decode
    + reduce kernel consumes the peers' frames (over NVLink on the
    peer-memory plane) and the self shard."""
    shards = _split_shards(comm, local)
    if comm.world_size == 1:
        return _reduce_chunks(shards, output)
    native = _native(comm)
    if native is not None:
        if shards[0].numel() == 0:
            return torch.empty(0, dtype=torch.float32 if output == "fp32" else torch.int16,
                               device=_dev(comm))
        _agree_shard(comm, shards[0].numel())
        return native.reduce_scatter(device_words(local, _dev(comm)), sigma, output)
    spec = AlltoAllSpec(shards, [shards[0].numel()] * comm.world_size)
    return _reduce_chunks(zip_all_to_all_d2(comm, spec, sigma), output)


def zip_all_reduce(comm: Communicator, local, sigma: float | None = None) -> torch.Tensor:
    """Zipped reduce-scatter then zipped all-gather (collectives.py:344-350)."""
    shard = zip_reduce_scatter(comm, local, sigma)
    if comm.world_size == 1:
        return shard
    return zip_all_gather(comm, shard, sigma)


def allgather_scalar(comm: Communicator, value: float, tag: int = 6) -> list:
    """All-gather one float64 per rank (collectives.py:353-363)."""
    if isinstance(comm, HubCommunicator):
        return [float(v) for v in comm._post_and_collect(float(value))]
    import torch.distributed as dist
    dev = comm.device if getattr(comm, "on_device", False) else torch.device("cpu")
    src = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    out = torch.empty(comm.world_size, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, src, group=comm.group)
    return [float(v) for v in out.cpu().tolist()]


def timed_call(comm: Communicator, fn):
    """Run fn() and agree on the slowest rank's elapsed time
    (collectives.py:366-376); device work is synchronised before stopping."""
    if torch.cuda.is_available():
        torch.cuda.current_stream().synchronize()
    start = comm.now()
    result = fn()
    if torch.cuda.is_available():
        torch.cuda.current_stream().synchronize()
    elapsed = comm.now() - start
    return result, max(allgather_scalar(comm, elapsed))
