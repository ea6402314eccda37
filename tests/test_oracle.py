"""Pin the CPU oracle against vectors produced by the real reference
(tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import zc_oracle as zo


def test_codec_cases_bit_exact(golden_meta, golden_arrays):
    for i, case in enumerate(golden_meta["cases"]):
        w = golden_arrays[f"w{i}"]
        ref = golden_arrays[f"f{i}"].tobytes()
        if case["book_src"] == "given":
            book = tuple(case["book"])
        elif case["book_src"] == "codebook_for":
            book = zo.book_for(w)
        else:
            s = float(case["book_src"].split("=")[1].rstrip(")"))
            book = zo.book_for(w, s)
        assert list(book) == case["book"], case["name"]
        got = zo.encode(w, book, case["gs"])
        assert got == ref, case["name"]
        assert len(got) == zo.frame_bytes(case["n"], case["zc"], case["gs"])
        assert np.array_equal(zo.decode(ref), w), case["name"]


def test_sigma_and_books(golden_meta):
    for c in golden_meta["sigma_cases"]:
        w = zo.gaussian(c["n"], c["s"], c["seed"])
        assert zo.sigma(w) == c["sigma"]
        assert list(zo.book_for(w)) == c["book"]


def test_derive_sweep(golden_meta):
    for s, base in golden_meta["derive_sweep"]:
        assert zo.derive(s)[0] - 127 == base, s


def test_a2a_frames(golden_meta, golden_a2a):
    world = golden_meta["a2a"]["world"]
    for rank in range(world):
        chunks = [golden_a2a[f"r{rank}_c{q}"] for q in range(world)]
        frames = zo.peer_frames(chunks, rank)
        for q in range(world):
            assert frames[q] == golden_a2a[f"r{rank}_f{q}"].tobytes(), (rank, q)


def test_flip_outcomes_match_reference(golden_meta):
    frame = np.load(zo_path := __import__("pathlib").Path(__file__).parent / "golden" / "flip_frame.npy")
    del zo_path
    arr = frame.copy()
    for i, bit, outcome in golden_meta["flips"]:
        arr[i] ^= bit
        try:
            zo.decode(arr.tobytes())
            got = "ok"
        except zo.OracleFrameError as exc:
            got = str(exc).split(":")[0]
        arr[i] ^= bit
        if outcome == "ok":
            assert got == "ok", (i, bit)
        else:
            assert got != "ok", (i, bit, outcome)
            assert got == outcome.split(":", 1)[1], (i, bit, outcome, got)


def test_c1_digests(golden_meta):
    c1 = golden_meta["c1"]
    w = zo.gaussian(1 << 24, 0.02, 0)
    assert hashlib.sha256(w.astype("<u2").tobytes()).hexdigest() == c1["input_sha256"]
    assert zo.sigma(w) == c1["sigma"]
    book = zo.book_for(w)
    assert list(book) == c1["book"]
    fr = zo.encode(w, book)
    assert len(fr) == c1["frame_len"]
    assert hashlib.sha256(fr).hexdigest() == c1["frame_sha256"]


@pytest.mark.parametrize("n", [1, 8, 512, 513, 4096])
def test_static_law(n):
    assert zo.static_bytes(n) == zo.offsets(n)[5]
    assert zo.static_bytes(8) == 128 * 6


def test_rne_narrowing_known_answers():
    # reference tests/test_bf16.py:36-51 style: ties to even, NaN quiet bit
    f = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, np.inf, -0.0], np.float32)
    w = zo.from_f32(f)
    assert list(w) == [0x3F80, 0x3F80, 0x3F82, 0x7F80, 0x8000]
    nan = np.array([0x7F800001], np.uint32).view(np.float32)
    assert zo.from_f32(nan)[0] == 0x7FC0
