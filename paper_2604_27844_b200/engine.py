"""Device-level operations over the C-ABI: stats -> codebook, encode, decode.

These are stream-ordered and never synchronise with the host; the public
codec/container/collectives modules build the reference API on top.
All tensors are CUDA tensors; BF16 words travel as int16 (same bits).
"""

from __future__ import annotations

import functools
import threading

import torch

from . import _lib
from ._lib import check, i64s, lib, ptrs, stream_ptr

WORD = torch.int16
TILE = _lib.TILE


def words_view(t: torch.Tensor) -> torch.Tensor:
    """Flat contiguous int16 view of a BF16-word tensor (bits, not values)."""
    if t.dtype in (torch.bfloat16, torch.float16, torch.uint16):
        t = t.view(torch.int16)
    elif t.dtype != torch.int16:
        raise TypeError(f"expected a 16-bit BF16-word tensor, got {t.dtype}")
    return t.contiguous().view(-1)


_WS: dict = {}
_WS_LOCKS: dict = {}
_WS_GUARD = threading.Lock()


class _Workspace:
    """A workspace buffer and the lock that keeps one call's launches
    contiguous on its stream (ctypes releases the GIL, so two host threads
    driving the same stream could otherwise interleave their kernels over the
    shared scratch)."""

    __slots__ = ("buf", "lock", "index", "_prev")

    def __init__(self, buf, lock, index):
        self.buf, self.lock, self.index = buf, lock, index
        self._prev = None

    def data_ptr(self):
        return self.buf.data_ptr()

    def numel(self):
        return self.buf.numel()

    def __enter__(self):
        self.lock.acquire()
        # launches inside go to the tensors' device and its current stream,
        # whatever device is current in the calling thread
        prev = torch._C._cuda_getDevice()
        if prev != self.index:
            torch._C._cuda_setDevice(self.index)
            self._prev = prev
        return self

    def __exit__(self, *exc):
        if self._prev is not None:
            torch._C._cuda_setDevice(self._prev)
            self._prev = None
        self.lock.release()


@functools.lru_cache(maxsize=4096)
def _workspace_bytes(total_elems: int, nseg: int) -> int:
    return int(lib().zc_workspace_bytes(total_elems, nseg))


def workspace(total_elems: int, nseg: int, device, stream=None) -> _Workspace:
    """Scratch for one call.  Cached per (device, stream) and grown on demand,
    so steady-state calls (and CUDA-graph captures) allocate nothing; calls on
    one stream are ordered, so reuse is safe as long as each call's launches
    are enqueued under the workspace lock (``with workspace(...) as ws:``)."""
    nbytes = _workspace_bytes(int(total_elems), int(nseg))
    index = device.index if isinstance(device, torch.device) else torch.device(device).index
    if index is None:
        index = torch._C._cuda_getDevice()
    s = int(stream.cuda_stream) if stream is not None else torch._C._cuda_getCurrentRawStream(index)
    key = (index, s)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        with _WS_GUARD:
            buf = _WS.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8,
                                  device=torch.device("cuda", index))
                _WS[key] = buf
    lock = _WS_LOCKS.get(key)
    if lock is None:
        with _WS_GUARD:
            lock = _WS_LOCKS.setdefault(key, threading.RLock())
    return _Workspace(buf, lock, index)


@functools.lru_cache(maxsize=1024)
def _book_cached(entries: tuple, device_index: int) -> torch.Tensor:
    return torch.tensor(list(entries) + [0], dtype=torch.uint8,
                        device=torch.device("cuda", device_index))


def book_tensor(entries, device) -> torch.Tensor:
    """Device copy (uint8[8]) of a host-known codebook; cached."""
    device = torch.device(device)
    return _book_cached(tuple(int(e) for e in entries), device.index or 0)


def _merge_segments(segs) -> list:
    """Adjacent segments as one range (the statistic only sees their union):
    the non-self chunks of a packed all-to-all buffer are at most two ranges,
    however many peers there are."""
    out = []
    for o, n in segs:
        if n <= 0:
            continue
        if out and out[-1][0] + out[-1][1] == o:
            out[-1] = (out[-1][0], out[-1][1] + n)
        else:
            out.append((o, n))
    return out or [(0, 0)]


SIGMA_EXACT = 1   # zc_codebook_measured flag (include/zipccl_b200.h)
MAX_SEGMENTS_MEASURED = _lib.MAX_SEGMENTS   # segments per zc_encode_measured call


def measured_codebook(words: torch.Tensor, segs=None, stream=None, exact: bool = False):
    """K1: sigma over the finite elements of the segments + on-device codebook.

    Returns (book uint8[8], result float64[3] = sigma, finite count, path).
    Path 3 = codebook certified by the packed-fp32 pass (sigma then within
    ~2e-6 relative); `exact=True` always runs the f64 statistic.
    """
    packed = measured_codebook_packed(words, segs, stream, exact)
    return packed[:8], packed[8:].view(torch.float64)


def measured_codebook_packed(words: torch.Tensor, segs=None, stream=None,
                             exact: bool = False) -> torch.Tensor:
    """measured_codebook into ONE uint8[32] device buffer: book in bytes
    0..7, result (float64[3]) in bytes 8..31 -- one device-to-host copy
    reads both."""
    if segs is None:
        segs = [(0, words.numel())]
    segs = _merge_segments(segs)
    dev = words.device
    packed = torch.empty(32, dtype=torch.uint8, device=dev)
    total = sum(n for _, n in segs)
    with workspace(total, len(segs), dev, stream) as ws:
        check(lib().zc_codebook_measured(
            words.data_ptr() if words.numel() else None, i64s(o for o, _ in segs),
            i64s(n for _, n in segs), len(segs), ws.data_ptr(), ws.numel(), packed.data_ptr(),
            packed.data_ptr() + 8, SIGMA_EXACT if exact else 0, stream_ptr(stream)),
            "zc_codebook_measured")
    return packed


def modal_codebook(words: torch.Tensor, segs=None, stream=None) -> torch.Tensor:
    """Histogram-mode codebook (reference codec.py:181-185) for explicit bad sigma."""
    if segs is None:
        segs = [(0, words.numel())]
    segs = _merge_segments(segs)
    dev = words.device
    book = torch.empty(8, dtype=torch.uint8, device=dev)
    total = sum(n for _, n in segs)
    with workspace(total, len(segs), dev, stream) as ws:
        check(lib().zc_codebook_modal(
            words.data_ptr() if words.numel() else None, i64s(o for o, _ in segs),
            i64s(n for _, n in segs), len(segs), ws.data_ptr(), ws.numel(), book.data_ptr(),
            stream_ptr(stream)), "zc_codebook_modal")
    return book


def max_frame_bytes(n: int, gs_log2: int = 9) -> int:
    return int(lib().zc_max_frame_bytes(int(n), int(gs_log2)))


def static_bytes(n: int, gs_log2: int = 9) -> int:
    return int(lib().zc_static_bytes(int(n), int(gs_log2)))


def encode(words: torch.Tensor, segs, book: torch.Tensor, gs_log2: int,
           frames: torch.Tensor, frame_offs, frame_len: torch.Tensor | None = None,
           stream=None) -> torch.Tensor:
    """K2/K4: one frame per segment, written at frames[frame_offs[i]:].

    Returns int64[nseg] device tensor of frame lengths (bytes).
    """
    segs = list(segs)
    nseg = len(segs)
    if frame_len is None:
        frame_len = torch.empty(nseg, dtype=torch.int64, device=words.device)
    total = sum(n for _, n in segs)
    with workspace(total, nseg, words.device, stream) as ws:
        for lo in range(0, nseg, _lib.MAX_SEGMENTS):
            part = segs[lo:lo + _lib.MAX_SEGMENTS]
            offs = list(frame_offs)[lo:lo + _lib.MAX_SEGMENTS]
            check(lib().zc_encode(
                words.data_ptr(), i64s(o for o, _ in part), i64s(n for _, n in part),
                i64s(offs), len(part), book.data_ptr(), int(gs_log2), frames.data_ptr(),
                ws.data_ptr(), ws.numel(), frame_len.data_ptr() + 8 * lo, stream_ptr(stream)),
                "zc_encode")
    return frame_len


def encode_measured(words: torch.Tensor, segs, gs_log2: int, frames: torch.Tensor, frame_offs,
                    frame_len: torch.Tensor | None = None, stream=None,
                    speculative: bool = True):
    """codebook_for over the concatenated segments + one frame per segment
    (speculative: the statistic fused into the encoder for large inputs;
    identical output either way).  Returns (book uint8[8],
    result float64[3], frame_len int64[nseg]); all stay on the device."""
    segs = list(segs)
    nseg = len(segs)
    if nseg > _lib.MAX_SEGMENTS:
        raise ValueError("too many segments for one measured encode")
    dev = words.device
    if frame_len is None:
        frame_len = torch.empty(nseg, dtype=torch.int64, device=dev)
    book = torch.empty(8, dtype=torch.uint8, device=dev)
    result = torch.empty(3, dtype=torch.float64, device=dev)
    total = sum(n for _, n in segs)
    with workspace(total, nseg, dev, stream) as ws:
        check(lib().zc_encode_measured(
            words.data_ptr(), i64s(o for o, _ in segs), i64s(n for _, n in segs),
            i64s(frame_offs), nseg, int(gs_log2), frames.data_ptr(), ws.data_ptr(), ws.numel(),
            frame_len.data_ptr(), book.data_ptr(), result.data_ptr(),
            1 if speculative else 0, stream_ptr(stream)), "zc_encode_measured")
    return book, result, frame_len


def decode(stat_ptrs, dyn_ptrs, dyn_lens, counts, out: torch.Tensor | None, out_offs,
           write_out: bool = True, err: torch.Tensor | None = None, stream=None,
           device=None, large_groups: bool = False, groups512: bool = False) -> torch.Tensor:
    """K3/K5: decode (and validate) one frame per segment.

    stat_ptrs/dyn_ptrs are raw device addresses (local or peer-mapped);
    dyn_ptrs entries may be 0 for "dynamic section in place".  Returns the
    int32[nseg] device error words (0x7F7F7F7F = ok).  ``large_groups``
    must be set when a frame may use groups larger than 4096 elements;
    ``groups512`` asserts the default 512-element groups (frames of the
    collectives and of compress(..., 512)), which lets messages of up to
    512 Ki words take the one-launch cluster decoder.
    """
    flags = (1 if write_out else 0) | (2 if large_groups else 0) | (8 if groups512 else 0)
    nseg = len(counts)
    dev = out.device if out is not None else torch.device(device or "cuda")
    if err is None:
        err = torch.empty(nseg, dtype=torch.int32, device=dev)
    total = sum(int(c) for c in counts)
    with workspace(total, nseg, dev, stream) as ws:
        for lo in range(0, nseg, _lib.MAX_SEGMENTS):
            hi = lo + _lib.MAX_SEGMENTS
            check(lib().zc_decode(
                ptrs(stat_ptrs[lo:hi]), ptrs(dyn_ptrs[lo:hi]),
                i64s(dyn_lens[lo:hi]) if dyn_lens is not None else None,
                i64s(counts[lo:hi]), i64s(out_offs[lo:hi]) if out_offs is not None else None,
                len(counts[lo:hi]), out.data_ptr() if out is not None else None,
                err.data_ptr() + 4 * lo, ws.data_ptr(), ws.numel(), flags,
                stream_ptr(stream)), "zc_decode")
    return err


def decode_when_ready(stat_ptrs, counts, out: torch.Tensor, out_offs, ready_ptrs, epoch: int,
                      timeout_ns: int = 0, err: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """Decode frame s once the u64 at ready_ptrs[s] reaches ``epoch``, the
    frames in the order their flags appear (zc_decode_when_ready; the
    reference decodes each peer inside its receive loop, collectives.py:216-227).
    Returns the int32[nseg] error words (20: flag timed out)."""
    nseg = len(counts)
    if err is None:
        err = torch.empty(nseg, dtype=torch.int32, device=out.device)
    total = sum(int(c) for c in counts)
    with workspace(total, nseg, out.device, stream) as ws:
        check(lib().zc_decode_when_ready(
            ptrs(stat_ptrs), i64s(counts), i64s(out_offs), ptrs(ready_ptrs), nseg,
            int(epoch), int(timeout_ns), out.data_ptr(), err.data_ptr(), ws.data_ptr(),
            ws.numel(), stream_ptr(stream)), "zc_decode_when_ready")
    return err


def decode_groups(frame: torch.Tensor, n: int, gs_log2: int, g0: int, g1: int,
                  out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Words of groups [g0, g1) of a validated frame (zc_decode_groups)."""
    gs = 1 << gs_log2
    count = max(0, min(g1 * gs, n) - g0 * gs)
    if out is None:
        out = torch.empty(count, dtype=torch.int16, device=frame.device)
    if count:
        with torch.cuda.device(frame.device):
            check(lib().zc_decode_groups(frame.data_ptr(), int(n), int(gs_log2), int(g0), int(g1),
                                         out.data_ptr(), stream_ptr(stream)), "zc_decode_groups")
    return out


def estimate_ratio(words: torch.Tensor, stream=None) -> torch.Tensor:
    """Estimated compression factor (frame / raw bytes) of ``words`` under the
    codebook codebook_for would pick, from a 1/64 sample (zc_estimate_ratio):
    float64[3] device tensor (e, sample sigma, sample escape fraction)."""
    out = torch.empty(3, dtype=torch.float64, device=words.device)
    n = words.numel()
    if n == 0:
        out.fill_(1.0)
        return out
    with workspace(n, 1, words.device, stream) as ws:
        check(lib().zc_estimate_ratio(words.data_ptr(), n, ws.data_ptr(), out.data_ptr(),
                                      stream_ptr(stream)), "zc_estimate_ratio")
    return out


PROF_ENCODE, PROF_DECODE = 0, 1


def profile_enable(on: bool) -> None:
    """Start (reset) / stop recording CUDA events around every pass-1 encoder
    and decoder launch (zc_profile_enable).  Eager launches only."""
    lib().zc_profile_enable(1 if on else 0)


def profile_read(tag: int, cap: int = 4096) -> list:
    """Durations (ms) of the launches recorded for `tag` since profile_enable."""
    import ctypes
    buf = (ctypes.c_float * cap)()
    k = lib().zc_profile_read(int(tag), buf, cap)
    if k < 0:
        raise RuntimeError(f"zc_profile_read failed: status {k}")
    return [float(buf[i]) for i in range(k)]


ERR_OK = 0x7F7F7F7F

# error code -> (field, detail) in reference wording (container.py:113-180,
# codec.py:210-250)
_SECTION = ("sign_mantissa", "plane0", "plane1", "plane2", "group_index", "zero_exponents")
ERR_FIELDS = {
    1: ("header", "frame is shorter than the header"),
    2: ("magic", "expected b'ZCCL'"),
    3: ("version", "unsupported version"),
    4: ("flags", "unknown flag bits"),
    5: ("group_size_log2", "implausible value"),
    6: ("element_count", "must be >= 1"),
    7: ("zero_count", "exceeds element_count"),
    8: ("codebook", "entries are not pairwise distinct"),
    9: ("codebook", "base byte disagrees with first entry"),
    **{10 + i: (f"{name} offset", "not the canonical offset") for i, name in enumerate(_SECTION)},
    16: ("frame length", "does not match the header"),
    17: ("group_index", "disagrees with escape counts in planes"),
    18: ("zero_count", "planes disagree with zero_exponents"),
    19: ("element_count", "frame holds a different element count than expected"),
    20: ("timeout", "peer frame never became ready"),
    21: ("group_size_log2", "groups larger than 4096 elements need the large-group decoder"),
}


def err_message(code: int) -> str:
    field, detail = ERR_FIELDS.get(int(code), ("frame", f"error {code}"))
    return f"{field}: {detail}"
