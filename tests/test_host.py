"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, and the host-side logic (codebook math, size law, header parsing)
matches the reference's golden vectors."""

from __future__ import annotations

import re

import numpy as np
import pytest

from tests.conftest import ROOT

import paper_2604_27844_b200 as zc
from paper_2604_27844_b200 import _lib, codec, container
from paper_2604_27844_b200.errors import CorruptFrameError


def declared_symbols():
    text = (ROOT / "include" / "zipccl_b200.h").read_text()
    body = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zc_\w+)\s*\(", body)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert lib.zc_abi_version() == 2
    assert lib.zc_tile_elements() == 4096


def test_ctypes_table_covers_header():
    assert set(declared_symbols()) <= set(_lib.EXPORTS)


@pytest.mark.parametrize("n", [1, 7, 8, 512, 513, 4096, 100000, 1 << 24, 218112000])
@pytest.mark.parametrize("gs", [1, 64, 512, 1 << 20])
def test_static_law_matches_native(n, gs):
    lib = _lib.lib()
    gsl = gs.bit_length() - 1
    assert lib.zc_static_bytes(n, gsl) == codec.static_size_bytes(n, gs)
    assert lib.zc_max_frame_bytes(n, gsl) == codec.compressed_size_bytes(n, n, gs)


def test_size_law_known_answers():
    # reference tests/test_codec.py:195-209
    assert codec.static_section_sizes(8, 512) == {
        "header": 48, "codebook": 8, "sign_mantissa": 8, "exp_planes": 3, "group_index": 4}
    bits = codec.static_size_bytes(1 << 20) * 8 / (1 << 20)
    assert 11.0 <= bits <= 11.2
    with pytest.raises(ValueError):
        codec.static_size_bytes(0)


def test_derive_codebook_sweep(golden_meta):
    for s, base in golden_meta["derive_sweep"]:
        assert codec.derive_codebook(s).base == base


def test_codebook_type_rules():
    with pytest.raises(ValueError):
        codec.ExponentCodebook((1, 1, 2, 3, 4, 5, 6))
    with pytest.raises(ValueError):
        codec.ExponentCodebook((1, 2, 3))
    with pytest.raises(ValueError):
        codec.ExponentCodebook((1, 2, 3, 4, 5, 6, 300))
    assert codec.derive_codebook(2.0 ** -200).entries == tuple(range(1, 8))
    assert all(1 <= e <= 254 for e in codec.derive_codebook(2.0 ** 130).entries)
    for bad in (0.0, -1.0, float("inf"), float("nan")):
        with pytest.raises(ValueError):
            codec.window_coverage(bad, -6)


def test_explicit_positive_sigma_needs_no_device():
    # codebook_for with a usable sigma is host math (codec.py:179-180)
    assert zc.codebook_for(np.zeros(4, np.uint16), 1.0) == codec.derive_codebook(1.0)


def _golden_frame(golden_meta, golden_arrays, name):
    for i, case in enumerate(golden_meta["cases"]):
        if case["name"] == name:
            return golden_arrays[f"f{i}"].tobytes(), golden_arrays[f"w{i}"]
    raise KeyError(name)


@pytest.mark.parametrize("mutate,field", [
    (lambda f: b"XCCL" + f[4:], "magic"),
    (lambda f: f[:4] + b"\x07" + f[5:], "version"),
    (lambda f: f[:5] + b"\x01" + f[6:], "flags"),
    (lambda f: f[:6] + b"\x1f" + f[7:], "group_size_log2"),
    (lambda f: f[:25] + f[24:25] + f[26:], "codebook"),
    (lambda f: f[:31] + bytes([f[31] ^ 1]) + f[32:], "codebook"),
    (lambda f: f[:36] + b"\x00\x00\x00\x00" + f[40:], "plane0 offset"),
    (lambda f: f[:-128], "frame length"),
    (lambda f: f[:40], "header"),
])
def test_header_errors_are_host_side(golden_meta, golden_arrays, mutate, field):
    frame, _ = _golden_frame(golden_meta, golden_arrays, "gauss_n100000")
    with pytest.raises(CorruptFrameError, match=field):
        container.parse(mutate(frame))


def test_split_static_dynamic_host(golden_meta, golden_arrays):
    frame, words = _golden_frame(golden_meta, golden_arrays, "gauss_n100000")
    split = container.split_static_dynamic(frame)
    assert len(split.static_bytes) == codec.static_size_bytes(words.size)
    assert split.recombine() == frame


def test_host_bf16_helpers_match_oracle():
    from oracle import zc_oracle as zo
    f = np.random.default_rng(3).standard_normal(10000).astype(np.float32) * 7
    f[:4] = [np.nan, np.inf, -0.0, 1.0 + 2 ** -8]
    assert np.array_equal(zc.from_float32(f), zo.from_f32(f))
    w = zo.from_f32(f)
    assert np.array_equal(zc.to_float32(w).view(np.uint32), zo.to_f32(w).view(np.uint32))


def test_torch_bf16_narrowing_matches_reference_rule():
    import torch
    f = torch.from_numpy(np.random.default_rng(4).standard_normal(4096).astype(np.float32))
    f[0] = float("nan")
    from oracle import zc_oracle as zo
    got = zc.from_float32(f).numpy().view(np.uint16)
    assert np.array_equal(got, zo.from_f32(f.numpy()))


def test_near_flip_window_host():
    # codebook_for's host re-derivation window (codec._near_flip): true only
    # within ~1e-12 of a threshold where the reference's derivation flips
    import math
    from oracle import zc_oracle as zo
    lo, hi = 2.0 ** -6, 2.0 ** -5
    b_lo = zo.derive(lo)
    for _ in range(200):
        mid = math.sqrt(lo * hi)
        lo, hi = (mid, hi) if zo.derive(mid) == b_lo else (lo, mid)
    flip = hi
    for rel in (0.0, 3e-13, -3e-13):
        assert codec._near_flip(flip * (1.0 + rel))
    for rel in (5e-12, -5e-12, 1e-6, 0.3):
        assert not codec._near_flip(flip * (1.0 + rel))
    assert codec.derive_codebook(flip * (1 - 1e-9)).entries == zo.derive(flip * (1 - 1e-9))
