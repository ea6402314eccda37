"""Compressed collectives — drop-in for reference collectives.py:1-376.

Same semantics as the reference (outputs bit-identical to the uncompressed
collectives, rank-order results, same exception classes), with the element
work on the GPU and the frames moving over the communicator's device byte
movers (NCCL over NVLink for a ``DistCommunicator``):

* ``zip_all_gather``: codebook (K1) + encode (K2) of the local shard; the
  static section has the same size on every rank (a function of n alone),
  so it moves with one all-gather posted right after the encoder; the frame
  lengths are gathered on the side and the variable dynamic sections follow
  in one padded all-gather; every peer frame is decoded by ONE batched K3
  launch straight into the output (reference collectives.py:203-227).
* ``zip_all_to_all_d1`` / ``_d2``: one codebook over the non-self, non-empty
  chunks (collectives.py:230-242), all peer frames encoded by ONE batched K4
  launch into one send buffer, then design 1 (metadata, whole frames) or
  design 2 (static sections pre-sized from recv_counts, dynamic sizes,
  dynamic sections) over grouped send/recv; one batched decode launch.
* ``zip_reduce_scatter`` / ``zip_all_reduce``: design-2
  all-to-all then the reference's float32 reduction in ascending rank order
  and RNE narrowing with its NaN rule.

Counts are agreed before any device transfer (NCCL needs matching sizes),
which costs 8 B per peer on top of the reference's metadata.
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
    buf = torch.cat(words) if sum(counts) else torch.empty(0, dtype=torch.int16, device=device)
    return buf, [int(o) for o in offs[:-1]], counts


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
    """Raw all-gather (collectives.py:97-111): NCCL all_gather on device."""
    words = device_words(local, _dev(comm))
    if comm.world_size == 1:
        return words.clone()
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
    """float32 sum in list (= ascending rank) order (collectives.py:137-144)."""
    acc = bf16.to_float32(chunks[0]).clone()
    for c in chunks[1:]:
        acc += bf16.to_float32(c)
    if output == "fp32":
        return acc
    return bf16.from_float32(acc)


def _split_shards(comm: Communicator, local) -> list:
    words = device_words(local, _dev(comm))
    if words.numel() % comm.world_size:
        raise ValueError(f"input of {words.numel()} elements is not divisible into "
                         f"{comm.world_size} shards")
    shard = words.numel() // comm.world_size
    return [words[r * shard:(r + 1) * shard] for r in range(comm.world_size)]


def reference_reduce_scatter(comm: Communicator, local, output: str = "bf16") -> torch.Tensor:
    shards = _split_shards(comm, local)
    if comm.world_size == 1:
        return _reduce_chunks(shards, output)
    spec = AlltoAllSpec(shards, [shards[0].numel()] * comm.world_size)
    return _reduce_chunks(reference_all_to_all(comm, spec), output)


# ---------------------------------------------------------------------------
# compressed collectives

def zip_all_gather(comm: Communicator, local, sigma: float | None = None,
                   _return_device: bool = True) -> torch.Tensor:
    """All-gather with compressed payloads, bit-identical to the reference
    all-gather (collectives.py:203-227)."""
    if getattr(comm, "use_p2p", False):
        return zip_all_gather_p2p(comm, local, sigma)
    dev = _dev(comm)
    words = device_words(local, dev)
    n = words.numel()
    W = comm.world_size
    if W == 1:
        return words.clone()
    counts = comm.allgather_ints(n)
    if n == 0:
        for p, c in enumerate(counts):
            if c != 0:
                raise ProtocolError(f"all-gather frame size mismatch: rank {comm.rank} has 0, "
                                    f"rank {p} declared {c}")
        return torch.empty(0, dtype=torch.int16, device=dev)
    for p, c in enumerate(counts):
        if c != n:
            raise CollectiveError(f"frame holds {c} elements, expected {n}", peer=p)
    # K1 + K2: codebook from the local shard, one frame
    S = engine.static_bytes(n, GS_LOG2)
    cap = engine.max_frame_bytes(n, GS_LOG2)
    frame = torch.empty(cap, dtype=torch.uint8, device=dev)
    _, flen = codec.device_encode(words, [(0, n)], sigma, frame, [0], GS_LOG2)
    # frame lengths first (tiny), then the static sections (size known from n)
    lens = torch.empty(W, dtype=torch.int64, device=dev)
    if isinstance(comm, DistCommunicator) and comm.on_device:
        # NCCL runs both gathers in order on its stream: waiting on the tiny
        # length gather lets the host learn the dynamic sizes while the static
        # sections are still in flight (design-2 overlap)
        import torch.distributed as dist
        h = dist.all_gather_into_tensor(lens, flen, group=comm.group, async_op=True)
        static = torch.empty(W * S, dtype=torch.uint8, device=dev)
        hs = dist.all_gather_into_tensor(static, frame[:S], group=comm.group, async_op=True)
        h.wait()
        dyn_lens = [int(v) - S for v in lens.cpu().tolist()]
        hs.wait()
        comm._count((8 + S) * (W - 1), 2 * (W - 1))
    else:
        dyn_lens = [v - S for v in comm.allgather_ints(int(flen.item()))]
        static = torch.empty(W * S, dtype=torch.uint8, device=dev)
        comm.all_gather_bytes(frame[:S], static)
    dmax = max(dyn_lens)
    dyn = torch.empty(max(W * dmax, 1), dtype=torch.uint8, device=dev)
    if dmax:
        comm.all_gather_bytes(frame[S:S + dmax], dyn[:W * dmax])
    out = torch.empty(W * n, dtype=torch.int16, device=dev)
    peers = comm.peers()
    err = engine.decode([static.data_ptr() + p * S for p in peers],
                        [dyn.data_ptr() + p * dmax for p in peers],
                        [dyn_lens[p] for p in peers], [n] * len(peers), out,
                        [p * n for p in peers])
    out[comm.rank * n:(comm.rank + 1) * n].copy_(words)
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
                            [int(roffs[p]) for p in peers_in])
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
    peer, then whole frames, then decode."""
    _check_world(comm, spec.world_size)
    dev = _dev(comm)
    if comm.world_size == 1:
        return [device_words(spec.send_chunks[0], dev).clone()]
    buf, offs, counts = _pack(spec.send_chunks, dev)
    _agree_counts(comm, spec, counts, "count")
    frames, frame_off, frame_len = _prepare_frames(comm, buf, offs, counts, sigma)
    got_len = comm.exchange_sizes(frame_len)
    recv_bufs = {p: torch.empty(got_len[p], dtype=torch.uint8, device=dev)
                 for p in comm.peers() if spec.recv_counts[p]}
    sends = {p: frames[frame_off[p]:frame_off[p] + frame_len[p]]
             for p in comm.peers() if frame_len[p]}
    comm.sendrecv_bytes(sends, recv_bufs)
    peers_in = sorted(recv_bufs)
    return _finish_a2a(comm, spec, buf, offs, counts, recv_bufs, peers_in,
                       [recv_bufs[p].data_ptr() for p in peers_in], [0] * len(peers_in),
                       [got_len[p] - codec.static_size_bytes(spec.recv_counts[p])
                        for p in peers_in])


def zip_all_to_all_d2(comm: Communicator, spec: AlltoAllSpec,
                      sigma: float | None = None) -> list:
    """Design 2 (collectives.py:281-325): static sections first (receivers
    pre-size them from recv_counts), then dynamic sizes, then dynamic
    sections; frames are decoded from the split receive buffers in place.
    With ``comm.use_p2p`` the peer-memory pull-decode path is used instead."""
    if getattr(comm, "use_p2p", False):
        return zip_all_to_all_p2p(comm, spec, sigma)
    _check_world(comm, spec.world_size)
    dev = _dev(comm)
    if comm.world_size == 1:
        return [device_words(spec.send_chunks[0], dev).clone()]
    buf, offs, counts = _pack(spec.send_chunks, dev)
    _agree_counts(comm, spec, counts, "static")
    frames, frame_off, frame_len = _prepare_frames(comm, buf, offs, counts, sigma)
    peers_out = [p for p in comm.peers() if frame_len[p]]
    peers_in = [p for p in comm.peers() if spec.recv_counts[p]]
    s_out = {p: codec.static_size_bytes(counts[p]) for p in peers_out}
    s_in = {p: codec.static_size_bytes(spec.recv_counts[p]) for p in peers_in}
    statics = {p: torch.empty(s_in[p], dtype=torch.uint8, device=dev) for p in peers_in}
    comm.sendrecv_bytes({p: frames[frame_off[p]:frame_off[p] + s_out[p]] for p in peers_out},
                        statics)
    dyn_len = [frame_len[p] - s_out[p] if p in s_out else 0 for p in range(comm.world_size)]
    got_dyn = comm.exchange_sizes(dyn_len)
    dyns = {p: torch.empty(max(got_dyn[p], 0), dtype=torch.uint8, device=dev) for p in peers_in}
    comm.sendrecv_bytes({p: frames[frame_off[p] + s_out[p]:frame_off[p] + frame_len[p]]
                         for p in peers_out}, dyns)
    return _finish_a2a(comm, spec, buf, offs, counts, None, peers_in,
                       [statics[p].data_ptr() for p in peers_in],
                       [dyns[p].data_ptr() if dyns[p].numel() else statics[p].data_ptr()
                        for p in peers_in],
                       [got_dyn[p] for p in peers_in])


def zip_reduce_scatter(comm: Communicator, local, sigma: float | None = None,
                       output: str = "bf16") -> torch.Tensor:
    """Compressed all-to-all (design 2) + float32 reduction in ascending rank
    order (collectives.py:328-341)."""
    shards = _split_shards(comm, local)
    if comm.world_size == 1:
        return _reduce_chunks(shards, output)
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


# ---------------------------------------------------------------------------
# peer-memory (NVLink) pull-decode variants — SURVEY K5 "fused pull-decode"

def _use_p2p(comm: Communicator) -> bool:
    return bool(getattr(comm, "use_p2p", isinstance(comm, HubCommunicator)))


def zip_all_gather_p2p(comm: Communicator, local, sigma: float | None = None) -> torch.Tensor:
    """All-gather where the transfer IS the decode: every rank encodes its
    shard into its own symmetric buffer, signals its peers device-side, and
    each rank's decoder pulls the peer frames over NVLink (TMA from peer HBM)
    straight into the gathered output.  Bit-identical to reference_all_gather."""
    from .peer import workspace_for
    dev = _dev(comm)
    words = device_words(local, dev)
    n = words.numel()
    W = comm.world_size
    if W == 1:
        return words.clone()
    counts = comm.allgather_ints(n)
    if n == 0:
        for p, c in enumerate(counts):
            if c != 0:
                raise ProtocolError(f"all-gather frame size mismatch: rank {comm.rank} has 0, "
                                    f"rank {p} declared {c}")
        return torch.empty(0, dtype=torch.int16, device=dev)
    for p, c in enumerate(counts):
        if c != n:
            raise CollectiveError(f"frame holds {c} elements, expected {n}", peer=p)
    ws = workspace_for(comm, engine.max_frame_bytes(max(counts), GS_LOG2))
    e = ws.epoch + 1
    ws.epoch = e
    werr = torch.full((1,), engine.ERR_OK, dtype=torch.int32, device=dev)
    if e > 1:
        ws.wait(1, e - 1, werr)                 # peers finished reading my last frame
    _, flen = codec.device_encode(words, [(0, n)], sigma, ws.buf, [256], GS_LOG2)
    ws.signal(0, e)                             # my frame is ready
    ws.wait(0, e, werr)                         # every peer's frame is ready
    out = torch.empty(W * n, dtype=torch.int16, device=dev)
    peers = comm.peers()
    err = engine.decode([ws.peer_base[p] + 256 for p in peers], [0] * len(peers), None,
                        [n] * len(peers), out, [p * n for p in peers])
    ws.signal(1, e)                             # done reading the peers' frames
    out[comm.rank * n:(comm.rank + 1) * n].copy_(words)
    del flen
    if int(werr.item()) != engine.ERR_OK:
        raise CollectiveError("peer frame never became ready (timeout)")
    _raise_decode_errors(err, peers)
    return out


def _a2a_layout(counts_row: list, sender: int) -> list:
    """Frame offsets inside `sender`'s symmetric buffer: peers in rank order,
    capacity max_frame_bytes(count) each (a pure function of the counts, so
    every rank derives every sender's layout without exchanging offsets)."""
    offs, pos = [0] * len(counts_row), 0
    for q, c in enumerate(counts_row):
        offs[q] = pos
        if q != sender and c:
            pos += engine.max_frame_bytes(c, GS_LOG2)
    return offs + [pos]


def zip_all_to_all_p2p(comm: Communicator, spec: AlltoAllSpec,
                       sigma: float | None = None) -> list:
    """All-to-all where the transfer IS the decode (MoE dispatch/combine):
    one batched K4 launch encodes every peer frame into this rank's symmetric
    buffer, peers are signalled device-side, and one batched K3 launch pulls
    this rank's frame from every peer's HBM over NVLink and decodes it in
    place.  Results identical to reference_all_to_all."""
    from .peer import workspace_for
    _check_world(comm, spec.world_size)
    dev = _dev(comm)
    W, me = comm.world_size, comm.rank
    if W == 1:
        return [device_words(spec.send_chunks[0], dev).clone()]
    buf, offs, counts = _pack(spec.send_chunks, dev)
    # the full count matrix: protocol check + every sender's layout
    if isinstance(comm, HubCommunicator):
        matrix = comm._post_and_collect(list(counts))
    else:
        import torch.distributed as dist
        rows = [None] * W
        dist.all_gather_object(rows, list(counts), group=comm.group)
        matrix = rows
    for p in comm.peers():
        if matrix[p][me] != spec.recv_counts[p]:
            raise ProtocolError(f"rank {p} will send {matrix[p][me]} elements, "
                                f"rank {me} expected {spec.recv_counts[p]}")
    layouts = [_a2a_layout(matrix[p], p) for p in range(W)]
    ws = workspace_for(comm, max(lay[-1] for lay in layouts) + 128)
    e = ws.epoch + 1
    ws.epoch = e
    werr = torch.full((1,), engine.ERR_OK, dtype=torch.int32, device=dev)
    if e > 1:
        ws.wait(1, e - 1, werr)
    peers_out = [q for q in comm.peers() if counts[q]]
    if peers_out:
        segs = [(offs[q], counts[q]) for q in peers_out]
        codec.device_encode(buf, segs, sigma, ws.buf, [256 + layouts[me][q] for q in peers_out],
                            GS_LOG2)
    ws.signal(0, e)
    ws.wait(0, e, werr)
    peers_in = [p for p in comm.peers() if spec.recv_counts[p]]
    roffs = np.concatenate([[0], np.cumsum(spec.recv_counts)]).astype(np.int64)
    flat = torch.empty(max(int(roffs[-1]), 1), dtype=torch.int16, device=dev)
    err = None
    if peers_in:
        err = engine.decode([ws.peer_base[p] + 256 + layouts[p][me] for p in peers_in],
                            [0] * len(peers_in), None, [spec.recv_counts[p] for p in peers_in],
                            flat, [int(roffs[p]) for p in peers_in])
    ws.signal(1, e)
    result = [flat[int(roffs[p]):int(roffs[p]) + spec.recv_counts[p]] for p in range(W)]
    result[me] = buf[offs[me]:offs[me] + counts[me]].clone()
    if int(werr.item()) != engine.ERR_OK:
        raise CollectiveError("peer frame never became ready (timeout)")
    if err is not None:
        _raise_decode_errors(err, peers_in)
    return result
