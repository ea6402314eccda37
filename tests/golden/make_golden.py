"""Generate the golden vectors in this directory from the REAL reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``zipcoll`` from /root/reference/pkg/src (read-only) and records
inputs and reference outputs; the outputs are committed so that the oracle
(`oracle/zc_oracle.py`) and the CUDA path can be checked on any machine.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from zipcoll import bf16, codec, collectives, container  # noqa: E402
from zipcoll.errors import CorruptChunkError, CorruptFrameError  # noqa: E402

OUT = Path(__file__).resolve().parent


def gw(n, s=1.0, seed=0):
    return bf16.from_float64(np.random.default_rng(seed).standard_normal(n) * s)


def frame_of(words, book, gs=512):
    return container.serialize(codec.compress(words, book, gs))


def main():
    arrays = {}
    cases = []

    def add(name, words, book=None, gs=512, sigma=None):
        words = np.ascontiguousarray(words, dtype=np.uint16)
        if book is None:
            b = codec.codebook_for(words, sigma)
            book_src = "codebook_for" if sigma is None else f"codebook_for(sigma={sigma!r})"
        else:
            b = codec.ExponentCodebook(tuple(book))
            book_src = "given"
        fr = frame_of(words, b, gs)
        i = len(cases)
        arrays[f"w{i}"] = words
        arrays[f"f{i}"] = np.frombuffer(fr, dtype=np.uint8)
        cases.append(dict(name=name, n=int(words.size), gs=gs, book=list(b.entries),
                          book_src=book_src, zc=int(codec.compress(words, b, gs).zero_count),
                          frame_len=len(fr)))

    book127 = (124, 125, 126, 127, 128, 129, 130)
    book_miss = (10, 11, 12, 13, 14, 15, 16)
    # hand-computed known answers (reference tests/test_codec.py:37-54)
    add("eight_ones", np.full(8, 0x3F80, np.uint16), book127)
    add("minus_two", np.array([0xC000], np.uint16), book127)
    # sizes around every alignment boundary, measured-sigma books
    for n in (1, 2, 7, 8, 9, 15, 16, 17, 31, 32, 33, 127, 128, 129, 511, 512, 513,
              1023, 1024, 2047, 2048, 4095, 4096, 4097, 5000, 8191, 8192, 8193,
              12345, 65536, 100000):
        add(f"gauss_n{n}", gw(n, 1.0, seed=n))
    # group sizes, incl. tiny and larger-than-tile groups
    for gs in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, 2048, 4096, 8192, 16384, 65536,
               1 << 20):
        add(f"gauss_gs{gs}", gw(20011, 0.02, seed=gs), gs=gs)
    # special buffers (reference tests/test_codec.py:81-90, acceptance :133-139)
    for pat, nm in ((0x7FC0, "nan"), (0x0001, "subnormal"), (0x0000, "zero"),
                    (0x8000, "negzero"), (0xFF80, "neginf"), (0x3F80, "one")):
        add(f"special_{nm}_derived", np.full(777, pat, np.uint16), codec.derive_codebook(1.0).entries)
        add(f"special_{nm}_miss", np.full(777, pat, np.uint16), book_miss)
        add(f"special_{nm}_book_for", np.full(777, pat, np.uint16))
    # all 65536 patterns in one buffer, under several books
    allw = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    add("all_patterns_derived", allw, codec.derive_codebook(1.0).entries)
    add("all_patterns_edges", allw, (0, 255, 1, 254, 127, 128, 3))
    add("all_patterns_book_for", allw)
    perm = np.random.default_rng(5).permutation(65536).astype(np.uint16)
    add("all_patterns_shuffled", perm, codec.derive_codebook(1.0).entries)
    # random words + arbitrary books (reference tests/test_codec.py:23-31, 76-79)
    rng = np.random.default_rng(2024)
    for k in range(60):
        n = int(rng.integers(1, 6000))
        words = rng.integers(0, 1 << 16, n).astype(np.uint16)
        book = tuple(int(x) for x in rng.choice(256, 7, replace=False))
        gs = int(1 << rng.integers(0, 14))
        add(f"fuzz{k}", words, book, gs=gs)
    # nan payloads, full escape (test_codec.py:99-105)
    r8 = np.random.default_rng(8)
    nanw = (0x7F80 | r8.integers(1, 0x80, 500)).astype(np.uint16)
    nanw |= (r8.integers(0, 2, 500).astype(np.uint16) << 15)
    add("nan_payloads", nanw, book127)
    # gradient mixes at 2^16
    sys.path.insert(0, str(OUT.parents[1]))
    from oracle import zc_oracle as zo  # generator only
    for kind in ("mix", "mix_x1000", "mix_n10", "lognormal2"):
        add(f"c4_{kind}", zo.outlier_mix(1 << 16, kind, seed=1))
    # explicit sigma paths
    w = gw(3000, 4.0, seed=3)
    add("sigma_given", w, sigma=4.0)
    add("sigma_zero_fallback", w, sigma=0.0)
    add("sigma_nan_fallback", w, sigma=float("nan"))
    # constant-with-nonfinite fallbacks
    mixed = np.full(100, 0x3F80, np.uint16)
    mixed[:60] = 0x7FC0
    add("const_plus_nan_majority", mixed)
    mixed2 = np.full(100, 0x3F80, np.uint16)
    mixed2[:50] = 0x7F80
    add("const_plus_inf_tie", mixed2)
    zmix = np.zeros(100, np.uint16)
    zmix[:10] = 0x7FC0
    add("zero_plus_nan", zmix)

    np.savez_compressed(OUT / "codec_cases.npz", **arrays)

    # sigma / codebook_for parity (value-level)
    sig = []
    for k, (n, s, seed) in enumerate([(2, 1.0, 0), (10, 0.02, 1), (1000, 1.0, 2),
                                      (100000, 0.02, 3), (200000, 4.0, 7),
                                      (1 << 20, 2.0, 99), (12345, 1e-30, 4),
                                      (5000, 1e30, 5)]):
        w = gw(n, s, seed)
        sig.append(dict(n=n, s=s, seed=seed, sigma=bf16.measure_sigma(w),
                        book=list(codec.codebook_for(w).entries)))
    # derive_codebook sweep incl. flip thresholds 0.0128650*2^k
    sweep = []
    for s in np.concatenate([2.0 ** np.linspace(-140, 130, 1500),
                             0.0128650 * 2.0 ** np.arange(-20, 20),
                             0.0128650 * 2.0 ** np.arange(-20, 20) * (1 + 1e-6),
                             0.0128650 * 2.0 ** np.arange(-20, 20) * (1 - 1e-6)]):
        sweep.append([float(s), codec.derive_codebook(float(s)).base])

    # collectives framing: per-peer frames of a W=4 all-to-all (_prepare_frames)
    class _Comm:
        def __init__(self, rank, world):
            self.rank, self.world_size = rank, world

    a2a = {}
    world = 4
    counts = lambda src, dst: (src + dst) * 97 + 5 if dst != 2 else 0  # noqa: E731
    for rank in range(world):
        chunks = [bf16.from_float64(np.random.default_rng([7, rank, q]).standard_normal(
            counts(rank, q)) * 0.5) for q in range(world)]
        spec = collectives.AlltoAllSpec(chunks, [counts(p, rank) for p in range(world)])
        frames = collectives._prepare_frames(_Comm(rank, world), spec, None)
        for q in range(world):
            a2a[f"r{rank}_c{q}"] = chunks[q]
            a2a[f"r{rank}_f{q}"] = np.frombuffer(frames[q], dtype=np.uint8)
    np.savez_compressed(OUT / "a2a_frames.npz", **a2a)

    # malformed-frame outcomes (reference tests/test_container.py:108-170)
    fr = frame_of(gw(4096, 1.0, seed=5), codec.derive_codebook(1.0))
    arr = np.frombuffer(fr, np.uint8).copy()
    r0 = np.random.default_rng(0)
    flips = []
    for _ in range(400):
        i = int(r0.integers(0, arr.size))
        bit = 1 << int(r0.integers(0, 8))
        arr[i] ^= bit
        try:
            ch = container.parse(arr.tobytes())
            codec.decompress(ch)
            outcome = "ok"
        except (CorruptFrameError, CorruptChunkError) as exc:
            outcome = type(exc).__name__ + ":" + str(exc).split(":")[0]
        flips.append([i, bit, outcome])
        arr[i] ^= bit
    np.save(OUT / "flip_frame.npy", np.frombuffer(fr, np.uint8))

    # C1
    c1 = bf16.from_float64(np.random.default_rng(0).standard_normal(1 << 24) * 0.02)
    c1_book = codec.codebook_for(c1)
    c1_frame = frame_of(c1, c1_book)
    c1_info = dict(input_sha256=hashlib.sha256(c1.astype("<u2").tobytes()).hexdigest(),
                   frame_sha256=hashlib.sha256(c1_frame).hexdigest(),
                   frame_len=len(c1_frame), book=list(c1_book.entries),
                   sigma=bf16.measure_sigma(c1),
                   zc=int(codec.compress(c1, c1_book).zero_count))

    meta = dict(generator="tests/golden/make_golden.py", reference="zipcoll 0.1.0 @ /root/reference",
                numpy=np.__version__, cases=cases, sigma_cases=sig, derive_sweep=sweep,
                a2a=dict(world=world, formula="(src+dst)*97+5, 0 to dst 2",
                         gen="from_float64(default_rng([7,rank,q]).standard_normal(count)*0.5)"),
                flips=flips, c1=c1_info)
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1))
    print(len(cases), "codec cases;", c1_info)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
