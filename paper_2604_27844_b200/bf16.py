"""BF16 bit helpers — drop-in for reference ``zipcoll.bf16`` (bf16.py:1-103).

Words are 16-bit patterns; every one of the 65536 survives untouched.  The
helpers accept torch tensors (device or host, reinterpreted bit for bit) and
numpy arrays (reference semantics).  ``measure_sigma`` runs on the GPU (K1).
"""

from __future__ import annotations

import numpy as np
import torch

from .codec import device_words, measure_sigma  # noqa: F401  (re-export)

EXP_BITS = 8
MANT_BITS = 7
EXP_MASK = 0xFF
MANT_MASK = 0x7F
EXP_BIAS = 127
QUIET_BIT = 0x40


def as_words(data):
    """Flat 16-bit words: torch -> int16 view (bits); numpy -> uint16 (bf16.py:27-32)."""
    if isinstance(data, torch.Tensor):
        from .engine import words_view
        return words_view(data)
    arr = np.ascontiguousarray(data)
    if arr.dtype != np.uint16:
        arr = arr.astype(np.uint16)
    return arr.ravel()


def _u32(words):
    if isinstance(words, torch.Tensor):
        return as_words(words).to(torch.int32) & 0xFFFF
    return as_words(words).astype(np.uint32)


def sign_bits(words):
    return (_u32(words) >> 15) & 0x1


def exponent_bits(words):
    """Biased 8-bit exponent field (bf16.py:39-41)."""
    return (_u32(words) >> MANT_BITS) & EXP_MASK


def mantissa_bits(words):
    return _u32(words) & MANT_MASK


def to_float32(words):
    """Exact widening (bf16.py:48-50)."""
    if isinstance(words, torch.Tensor):
        return (as_words(words).to(torch.int32) << 16).view(torch.float32)
    return (as_words(words).astype(np.uint32) << 16).view(np.float32)


def from_float32(values):
    """RNE narrowing with the reference's NaN rule: sign and top payload kept,
    quiet bit forced (bf16.py:53-66).  (torch's own bf16 cast canonicalises
    NaN payloads, so it is not used.)"""
    if isinstance(values, torch.Tensor):
        u = values.to(torch.float32).contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        lsb = (u >> 16) & 1
        out = ((u + 0x7FFF + lsb) >> 16) & 0xFFFF
        nan = torch.isnan(values.to(torch.float32))
        out = torch.where(nan, ((u >> 16) & 0xFFFF) | QUIET_BIT, out)
        return out.to(torch.int32).to(torch.int16)
    f32 = np.ascontiguousarray(values, dtype=np.float32)
    u = f32.view(np.uint32)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(f32)
    if nan.any():
        rounded = np.where(nan, (u >> 16).astype(np.uint16) | QUIET_BIT, rounded)
    return rounded


def from_float64(values):
    """f64 -> f32 -> bf16 (bf16.py:69-79)."""
    if isinstance(values, torch.Tensor):
        return from_float32(values.to(torch.float32))
    with np.errstate(over="ignore"):
        f32 = np.asarray(values, dtype=np.float64).astype(np.float32)
    return from_float32(f32)


def to_float64(words):
    if isinstance(words, torch.Tensor):
        return to_float32(words).to(torch.float64)
    with np.errstate(invalid="ignore"):
        return to_float32(words).astype(np.float64)
