"""Lossless BF16 exponent codec — drop-in for reference ``zipcoll.codec``.

Same names, arguments and error behaviour as reference codec.py:1-401; the
element work runs in the sm_100a kernels of libzipccl_b200.so:

* ``codebook_for`` / ``measure_sigma``  -> K1 stats + on-device derivation
  (reference codec.py:164-185, bf16.py:88-103)
* ``compress``                          -> K2 single-pass frame encoder
  (codec.py:264-305 + container.serialize container.py:65-95)
* ``decompress`` / ``validate``         -> K3 decoder / validator
  (codec.py:210-261, :315-327)

The closed-form codebook math (``window_coverage``, ``optimal_base_exponent``,
``derive_codebook``) and the size law are host scalars, exactly as in the
reference.  A ``CompressedChunk`` is backed by its serialized frame in device
memory; its section attributes are zero-copy views of that frame.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import engine
from ._lib import require_cuda
from .errors import CorruptChunkError, DegenerateDataError, UnrepresentableError

__all__ = [
    "GROUP_SIZE", "WINDOW_WIDTH", "WINDOW_OPT_U", "BASE_EXPONENT_OFFSET",
    "ExponentCodebook", "CompressedChunk", "window_coverage", "optimal_base_exponent",
    "derive_codebook", "codebook_for", "measure_sigma", "compress", "decompress",
    "decompress_group", "static_section_sizes", "static_size_bytes", "compressed_size_bytes",
]

WINDOW_WIDTH = 7                                   # codec.py:47
GROUP_SIZE = 512                                   # codec.py:51
WINDOW_OPT_U = math.sqrt(7.0 * math.log(2.0) / 16383.0)               # codec.py:56
BASE_EXPONENT_OFFSET = 0.5 * math.log2(14.0 * math.log(2.0) / 16383.0)  # codec.py:59
EXP_BIAS = 127
_MIN_BASE = 1 - EXP_BIAS                           # codec.py:63
_MAX_BASE = 254 - EXP_BIAS - (WINDOW_WIDTH - 1)    # codec.py:64

ALIGNMENT = 128                                    # codec.py:357-360
HEADER_FIXED_BYTES = 48
CODEBOOK_BYTES = 8
HEADER_BYTES = HEADER_FIXED_BYTES + CODEBOOK_BYTES


# --- device words ------------------------------------------------------------

def device_words(data, device=None) -> torch.Tensor:
    """BF16 words of ``data`` as a flat int16 CUDA tensor.

    torch tensors are reinterpreted bit-for-bit (bfloat16/float16/int16/
    uint16) and moved to the device if needed; numpy input follows the
    reference ``as_words`` (bf16.py:27-32: uint16 as is, other dtypes value-
    cast) and is copied host->device.
    """
    if isinstance(data, torch.Tensor):
        t = engine.words_view(data)
        if t.device.type != "cuda":
            dev = require_cuda(device)
            t = t.to(dev, non_blocking=t.is_pinned())
        return t
    arr = np.ascontiguousarray(data)
    if arr.dtype != np.uint16:
        arr = arr.astype(np.uint16)
    dev = require_cuda(device)
    return torch.from_numpy(arr.ravel().view(np.int16)).to(dev)


# --- closed-form codebook (codec.py:67-161), host scalars -------------------

def _check_sigma(sigma: float) -> float:
    sigma = float(sigma)
    if not math.isfinite(sigma) or sigma <= 0.0:
        raise ValueError(f"sigma must be positive and finite, got {sigma!r}")
    return sigma


def window_coverage(sigma: float, x: float) -> float:
    """P(|N(0, sigma^2)| in [2**x, 2**(x+7))) (codec.py:74-89)."""
    sigma = _check_sigma(sigma)
    try:
        lo = 2.0 ** float(x)
    except OverflowError:
        lo = math.inf
    scale = sigma * math.sqrt(2.0)
    return math.erf(lo * 128.0 / scale) - math.erf(lo / scale)


def optimal_base_exponent(sigma: float) -> float:
    """log2(sigma) + BASE_EXPONENT_OFFSET (codec.py:92-98)."""
    return math.log2(_check_sigma(sigma)) + BASE_EXPONENT_OFFSET


@dataclass(frozen=True)
class ExponentCodebook:
    """Seven distinct biased exponents; entry i is code i+1, code 0 escapes
    (codec.py:101-146)."""

    entries: tuple

    def __post_init__(self):
        if len(self.entries) != WINDOW_WIDTH:
            raise ValueError(f"codebook needs exactly {WINDOW_WIDTH} entries")
        if any(not (0 <= int(e) <= 255) for e in self.entries):
            raise ValueError("codebook entries must be biased exponents in [0, 255]")
        if len(set(int(e) for e in self.entries)) != WINDOW_WIDTH:
            raise ValueError("codebook entries must be pairwise distinct")
        object.__setattr__(self, "entries", tuple(int(e) for e in self.entries))

    @property
    def base(self) -> int:
        return self.entries[0] - EXP_BIAS

    @classmethod
    def from_base(cls, base: int) -> "ExponentCodebook":
        base = min(max(int(base), _MIN_BASE), _MAX_BASE)
        first = base + EXP_BIAS
        return cls(tuple(range(first, first + WINDOW_WIDTH)))

    @cached_property
    def encode_table(self) -> np.ndarray:
        table = np.zeros(256, dtype=np.uint8)
        for i, e in enumerate(self.entries):
            table[e] = i + 1
        table.setflags(write=False)
        return table

    @cached_property
    def decode_table(self) -> np.ndarray:
        table = np.zeros(8, dtype=np.uint8)
        table[1:] = self.entries
        table.setflags(write=False)
        return table

    def device_tensor(self, device) -> torch.Tensor:
        return engine.book_tensor(self.entries, device)


def derive_codebook(sigma: float) -> ExponentCodebook:
    """Analytic window for N(0, sigma^2) (codec.py:149-161)."""
    x_opt = optimal_base_exponent(sigma)
    lo, hi = math.floor(x_opt), math.ceil(x_opt)
    if lo == hi or window_coverage(sigma, lo) >= window_coverage(sigma, hi):
        base = lo
    else:
        base = hi
    return ExponentCodebook.from_base(base)


def _book_from_device(book: torch.Tensor) -> ExponentCodebook:
    return ExponentCodebook(tuple(int(v) for v in book[:7].cpu().tolist()))


def device_codebook(words: torch.Tensor, sigma=None, segs=None) -> torch.Tensor:
    """Stream-ordered codebook_for: uint8[8] device tensor, no host sync
    unless sigma is given (then it is host math, as in the reference)."""
    if sigma is None:
        book, _ = engine.measured_codebook(words, segs)
        return book
    if math.isfinite(sigma) and sigma > 0.0:
        return derive_codebook(sigma).device_tensor(words.device)
    return engine.modal_codebook(words, segs)


def device_encode(words: torch.Tensor, segs, sigma, frames: torch.Tensor, frame_offs,
                  gs_log2: int = 9, frame_len: torch.Tensor | None = None):
    """codebook_for over the concatenated segments (the all-to-all scope of
    collectives._prepare_frames, collectives.py:230-242) + one frame per
    segment, stream-ordered on the device.  sigma None: the measured codebook
    fused into the encoder (speculative path for large inputs, identical
    output); otherwise the analytic / modal codebook, then the encoder.
    Returns (book uint8[8], frame_len int64[nseg]) device tensors."""
    segs = list(segs)
    if sigma is None and len(segs) <= engine.MAX_SEGMENTS_MEASURED:
        book, _, flen = engine.encode_measured(words, segs, gs_log2, frames, frame_offs, frame_len)
        return book, flen
    book = device_codebook(words, sigma, segs)
    return book, engine.encode(words, segs, book, gs_log2, frames, frame_offs, frame_len)


def codebook_for(data, sigma: float | None = None) -> ExponentCodebook:
    """Analytic codebook from sigma (measured on the GPU when None), modal
    fallback otherwise (codec.py:164-185)."""
    if sigma is not None and math.isfinite(sigma) and sigma > 0.0:
        return derive_codebook(sigma)
    words = device_words(data)
    if words.numel() == 0:
        return ExponentCodebook.from_base(-6)
    if sigma is not None:
        return _book_from_device(device_codebook(words, sigma))
    # one read of book + (sigma, finite count, path).  The device codebook is
    # the reference's: certified (path 3), or from an f64 sigma re-derived in
    # numpy's order next to a flip.  Within 1e-12 of a flip the sigma is
    # taken in numpy's order over the compacted finite values and the
    # codebook derived here with the reference's host formula (math.erf), so
    # even the last-ulp erf comparison and non-finite inputs match.
    host = engine.measured_codebook_packed(words).cpu()
    s, _, path = host[8:].view(torch.float64).tolist()
    if path == 1.0 and math.isfinite(s) and s > 0.0 and _near_flip(s):
        return derive_codebook(measure_sigma(words))
    return ExponentCodebook(tuple(int(v) for v in host[:7].tolist()))


def _near_flip(sigma: float, rel: float = 1e-12) -> bool:
    return derive_codebook(sigma * (1.0 - rel)).entries != derive_codebook(sigma * (1.0 + rel)).entries


def measure_sigma(data) -> float:
    """Population std of the finite elements (bf16.py:88-103), on the GPU."""
    words = device_words(data)
    if words.numel() == 0:
        raise DegenerateDataError("measure_sigma: empty buffer")
    _, result = engine.measured_codebook(words, exact=True)
    sigma, count, _ = result.cpu().tolist()
    if count == 0:
        raise DegenerateDataError("measure_sigma: no finite elements")
    if count < words.numel():
        # the reference takes np.std of the compacted finite values: numpy's
        # pairwise tree runs over their indices, so compact on the device
        # (order kept) and take the numpy-order sigma of that array
        w = words.view(torch.int16)
        finite = w[(w & 0x7F80) != 0x7F80]
        _, result = engine.measured_codebook(finite, exact=True)
        sigma = result[0].item()
    return float(sigma)


# --- size law (codec.py:363-401) ------------------------------------------------

def _pad(size: int) -> int:
    return (int(size) + ALIGNMENT - 1) // ALIGNMENT * ALIGNMENT


def static_section_sizes(element_count: int, group_size: int = GROUP_SIZE) -> dict:
    n = int(element_count)
    if n < 1:
        raise ValueError("element_count must be >= 1")
    return {
        "header": HEADER_FIXED_BYTES,
        "codebook": CODEBOOK_BYTES,
        "sign_mantissa": n,
        "exp_planes": 3 * ((n + 7) // 8),
        "group_index": 4 * ((n + group_size - 1) // group_size),
    }


def static_size_bytes(element_count: int, group_size: int = GROUP_SIZE) -> int:
    n = int(element_count)
    if n < 1:
        raise ValueError("element_count must be >= 1")
    return (_pad(HEADER_BYTES) + _pad(n) + 3 * _pad((n + 7) // 8)
            + _pad(4 * ((n + group_size - 1) // group_size)))


def compressed_size_bytes(element_count: int, zero_count: int,
                          group_size: int = GROUP_SIZE) -> int:
    return static_size_bytes(element_count, group_size) + _pad(int(zero_count))


def section_offsets(element_count: int, group_size: int) -> tuple:
    """Canonical 128-aligned section starts (container.py:52-62)."""
    offs = []
    pos = _pad(HEADER_BYTES)
    plane = (element_count + 7) // 8
    groups = (element_count + group_size - 1) // group_size
    for size in (element_count, plane, plane, plane, 4 * groups):
        offs.append(pos)
        pos += _pad(size)
    offs.append(pos)
    return tuple(offs)


def _check_group_size(group_size: int) -> int:
    gs = int(group_size)
    if gs < 1 or gs & (gs - 1):
        raise ValueError("group_size must be a power of two")
    if gs > 1 << 30:
        raise ValueError("group_size must be <= 2**30")
    return gs


# --- compressed chunk -----------------------------------------------------------

def _as_device_bytes(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.reshape(-1)
        if t.dtype != torch.uint8:
            t = t.contiguous().view(torch.uint8)
        return t.to(device)
    arr = np.ascontiguousarray(x)
    return torch.from_numpy(arr.view(np.uint8).reshape(-1).copy()).to(device)


class CompressedChunk:
    """A compressed BF16 buffer (codec.py:188-261).

    Normally backed by its serialized frame in device memory (``frame``);
    the section attributes are zero-copy device views.  Constructing it
    from sections (reference signature) keeps them as given until the frame
    is needed, so structure errors surface with the reference field names.
    """

    def __init__(self, element_count, group_size, codebook, sign_mantissa, exp_planes,
                 group_index, zero_exponents):
        self.element_count = int(element_count)
        self.group_size = int(group_size)
        self.codebook = codebook
        self._sections = (sign_mantissa, tuple(exp_planes), group_index, zero_exponents)
        self._frame = None
        self._zc = None

    @classmethod
    def _wrap(cls, frame: torch.Tensor, element_count: int, group_size: int,
              codebook: ExponentCodebook, zero_count: int | None = None) -> "CompressedChunk":
        self = cls.__new__(cls)
        self.element_count = int(element_count)
        self.group_size = int(group_size)
        self.codebook = codebook
        self._sections = None
        self._frame = frame
        self._zc = zero_count
        return self

    # -- section views -----------------------------------------------------------
    def _offs(self):
        return section_offsets(self.element_count, self.group_size)

    @property
    def frame(self) -> torch.Tensor:
        """The serialized frame (device uint8)."""
        if self._frame is None:
            self._frame = self._assemble()
        return self._frame

    @property
    def zero_count(self) -> int:
        if self._sections is not None:
            return int(_numel(self._sections[3]))
        if self._zc is None:
            hdr = self._frame[16:24].cpu().numpy()
            self._zc = int(hdr.view("<u8")[0])
        return self._zc

    @property
    def sign_mantissa(self) -> torch.Tensor:
        if self._sections is not None:
            return self._sections[0]
        o = self._offs()
        return self._frame[o[0]:o[0] + self.element_count]

    @property
    def exp_planes(self) -> tuple:
        if self._sections is not None:
            return self._sections[1]
        o = self._offs()
        pl = (self.element_count + 7) // 8
        return tuple(self._frame[o[1 + b]:o[1 + b] + pl] for b in range(3))

    @property
    def group_index(self) -> torch.Tensor:
        """u32 exclusive prefix per group (int32 device view of the LE words)."""
        if self._sections is not None:
            return self._sections[2]
        o = self._offs()
        g = (self.element_count + self.group_size - 1) // self.group_size
        return self._frame[o[4]:o[4] + 4 * g].view(torch.int32)

    @property
    def zero_exponents(self) -> torch.Tensor:
        if self._sections is not None:
            return self._sections[3]
        o = self._offs()
        return self._frame[o[5]:o[5] + self.zero_count]

    # -- invariants (codec.py:210-255) ------------------------------------------------
    def check_structure(self) -> None:
        n = self.element_count
        if n < 1:
            raise CorruptChunkError("element_count: must be >= 1")
        gs = self.group_size
        if gs < 1 or gs & (gs - 1):
            raise CorruptChunkError("group_size: must be a power of two")
        if self._sections is None:
            return   # frame-backed chunks are structurally canonical by construction
        sm, planes, gi, ze = self._sections
        if _numel(sm) != n:
            raise CorruptChunkError(f"sign_mantissa: expected {n} bytes, got {_numel(sm)}")
        plane_len = (n + 7) // 8
        for b, plane in enumerate(planes):
            if _numel(plane) != plane_len:
                raise CorruptChunkError(
                    f"exp_planes[{b}]: expected {plane_len} bytes, got {_numel(plane)}")
        n_groups = (n + gs - 1) // gs
        if _numel(gi) != n_groups:
            raise CorruptChunkError(f"group_index: expected {n_groups} entries, got {_numel(gi)}")
        giv = _host_u32(gi)
        if giv[0] != 0:
            raise CorruptChunkError("group_index: first entry must be 0")
        if np.any(np.diff(giv.astype(np.int64)) < 0):
            raise CorruptChunkError("group_index: must be monotone non-decreasing")
        if _numel(ze) > n:
            raise CorruptChunkError("zero_count: exceeds element_count")

    def _assemble(self) -> torch.Tensor:
        """Serialize from sections (container.serialize layout) on the device."""
        self.check_structure()
        dev = require_cuda()
        sm, planes, gi, ze = self._sections
        n, gs, zc = self.element_count, self.group_size, int(_numel(ze))
        offs = section_offsets(n, gs)
        total = offs[5] + _pad(zc)
        frame = torch.zeros(total, dtype=torch.uint8, device=dev)
        frame[:HEADER_BYTES] = torch.from_numpy(
            _header_bytes(n, zc, gs, self.codebook.entries, offs)).to(dev)
        parts = (sm, *planes, _u32_bytes(gi), ze)
        for off, part in zip(offs, parts):
            b = _as_device_bytes(part, dev)
            frame[off:off + b.numel()] = b
        return frame

    def validate(self) -> None:
        """Re-check every invariant (codec.py:252-255); device consistency pass."""
        self.check_structure()
        _run_decode(self, write_out=False, exc=CorruptChunkError)


def _numel(x) -> int:
    return int(x.numel()) if isinstance(x, torch.Tensor) else int(np.asarray(x).size)


def _host_u32(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().contiguous()
        return x.view(torch.int32).numpy().view(np.uint32) if x.element_size() == 4 \
            else x.numpy().astype(np.uint32)
    return np.asarray(x).astype(np.uint32)


def _u32_bytes(x):
    if isinstance(x, torch.Tensor):
        if x.element_size() == 4:
            return x.contiguous().view(torch.uint8)
        return torch.from_numpy(x.cpu().numpy().astype("<u4").view(np.uint8))
    return np.asarray(x).astype("<u4").view(np.uint8)


def _header_bytes(n, zc, gs, entries, offs) -> np.ndarray:
    import struct
    hdr = struct.pack("<4sBBBBQQ7sB6I", b"ZCCL", 1, 0, gs.bit_length() - 1, 0, n, zc,
                      bytes(entries), entries[0], *offs)
    return np.frombuffer(hdr, dtype=np.uint8).copy()


# --- compress / decompress ------------------------------------------------------------

def compress(data, codebook: ExponentCodebook, group_size: int = GROUP_SIZE) -> CompressedChunk:
    """Compress a BF16 buffer under ``codebook`` (codec.py:264-305) into a
    device frame, byte-identical to reference serialize(compress(...))."""
    words = device_words(data)
    n = words.numel()
    if n == 0:
        raise ValueError("compress: empty buffer")
    gs = _check_group_size(group_size)
    gsl = gs.bit_length() - 1
    frames = torch.empty(engine.max_frame_bytes(n, gsl), dtype=torch.uint8, device=words.device)
    engine.encode(words, [(0, n)], codebook.device_tensor(words.device), gsl, frames, [0])
    # one 8-byte read-back: the header's zero_count; the frame length follows
    # from the size law (container.py:52-62)
    zc = int(frames[16:24].cpu().numpy().view("<u8")[0])
    length = engine.static_bytes(n, gsl) + -(-zc // 128) * 128
    if zc >= 1 << 32:
        raise UnrepresentableError("zero_count does not fit the 32-bit group index")
    return CompressedChunk._wrap(frames[:length], n, gs, codebook, zc)


def _run_decode(chunk: CompressedChunk, write_out: bool, exc, out=None):
    frame = chunk.frame
    n = chunk.element_count
    if write_out and out is None:
        out = torch.empty(n, dtype=torch.int16, device=frame.device)
    err = engine.decode([frame.data_ptr()], [0], None, [n], out, [0] if out is not None else None,
                        write_out=write_out, large_groups=chunk.group_size > engine.TILE,
                        groups512=chunk.group_size == 512)
    code = int(err[0].item())
    if code != engine.ERR_OK:
        raise exc(engine.err_message(code))
    return out


def decompress(chunk: CompressedChunk, out: torch.Tensor | None = None) -> torch.Tensor:
    """Exact BF16 words of a chunk (codec.py:315-327), as an int16 CUDA tensor;
    invariants are re-checked on the device first, as in the reference."""
    chunk.check_structure()
    if out is not None:
        if not isinstance(out, torch.Tensor) or out.element_size() != 2 or \
                out.dtype.is_complex:
            raise ValueError("decompress: out must be a 16-bit tensor")
        if not out.is_contiguous():
            raise ValueError("decompress: out must be contiguous (it is written in place)")
        if out.device != chunk.frame.device:
            raise ValueError(f"decompress: out is on {out.device}, the frame on "
                             f"{chunk.frame.device}")
        if out.numel() < chunk.element_count:
            raise ValueError(f"decompress: out holds {out.numel()} elements, the chunk "
                             f"{chunk.element_count}")
        out = engine.words_view(out)
    return _run_decode(chunk, True, CorruptChunkError, out)


def decompress_group(chunk: CompressedChunk, group: int) -> torch.Tensor:
    """Words of one group (codec.py:330-348): the chunk is validated first,
    as in the reference, then only the group's bytes and its escapes (from
    group_index[group]) are decoded on the device."""
    chunk.validate()
    n, gs = chunk.element_count, chunk.group_size
    n_groups = (n + gs - 1) // gs
    if not 0 <= group < n_groups:
        raise IndexError(f"group {group} out of range for {n_groups} groups")
    return engine.decode_groups(chunk.frame, n, gs.bit_length() - 1, group, group + 1)
