"""Parity of the CUDA codec with the reference (golden vectors made by the
real reference) and with the CPU oracle.  Bit-exact: frames byte for byte,
decoded words bit for bit."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest
import torch

from oracle import zc_oracle as zo
from tests.conftest import GOLDEN, gaussian_words

pytestmark = pytest.mark.gpu

import paper_2604_27844_b200 as zc  # noqa: E402
from paper_2604_27844_b200 import codec, container, engine  # noqa: E402
from paper_2604_27844_b200.errors import CorruptChunkError, CorruptFrameError  # noqa: E402


def host_words(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def book_of(case, words):
    src = case["book_src"]
    if src == "given":
        return codec.ExponentCodebook(tuple(case["book"]))
    if src == "codebook_for":
        return zc.codebook_for(words)
    sigma = float(src.split("=")[1].rstrip(")"))
    return zc.codebook_for(words, sigma)


def test_golden_codec_cases(golden_meta, golden_arrays):
    for i, case in enumerate(golden_meta["cases"]):
        words = golden_arrays[f"w{i}"]
        ref = golden_arrays[f"f{i}"].tobytes()
        book = book_of(case, words)
        assert list(book.entries) == case["book"], case["name"]
        chunk = zc.compress(words, book, case["gs"])
        assert chunk.zero_count == case["zc"], case["name"]
        frame = zc.serialize(chunk)
        assert frame == ref, case["name"]
        assert np.array_equal(host_words(zc.decompress(chunk)), words), case["name"]
        parsed = zc.parse(ref)
        assert np.array_equal(host_words(zc.decompress(parsed)), words), case["name"]


def test_sigma_cases(golden_meta):
    for c in golden_meta["sigma_cases"]:
        w = zo.gaussian(c["n"], c["s"], c["seed"])
        got = zc.measure_sigma(w)
        assert got == pytest.approx(c["sigma"], rel=1e-12, abs=0), c
        assert list(zc.codebook_for(w).entries) == c["book"], c


def _np_sigma(words: np.ndarray) -> float:
    """The reference's measure_sigma (bf16.py:88-103): np.std of the finite
    values as float64."""
    with np.errstate(invalid="ignore"):              # signaling-NaN payloads
        v = (words.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return float(np.std(v[np.isfinite(v)]))


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 100, 127, 128, 129, 136, 1000, 8195, 100003,
                               4096 * 300 + 17, (1 << 20) + 5, 1 << 24])
def test_sigma_is_bit_identical_to_numpy(n):
    # all-finite inputs: numpy's pairwise summation order reproduced on the
    # device (np_sigma_kernel), so measure_sigma is the reference's float
    for s, seed in ((0.02, n), (1.0, n + 1), (3e-4, n + 2)):
        w = zo.gaussian(n, s, seed)
        if n > 2:
            w[: n // 3] = zo.from_f64(np.random.default_rng(seed).standard_normal(n // 3) * 7.0 + 3.0)
        got = zc.measure_sigma(w)
        assert got == _np_sigma(w), (n, s, got, _np_sigma(w))


def test_sigma_bit_identical_over_segments():
    # the all-to-all statistic spans several chunks (collectives.py:230-242):
    # the concatenation's pairwise order crosses chunk boundaries
    rng = np.random.default_rng(5)
    chunks = [zo.gaussian(c, 0.02, seed=c) for c in (4096 * 3 + 5, 77, 100003, 9)]
    buf = np.concatenate(chunks)
    x = torch.from_numpy(buf.view(np.int16)).cuda()
    offs = np.concatenate([[0], np.cumsum([c.size for c in chunks])[:-1]]).tolist()
    segs = [(int(o), int(c.size)) for o, c in zip(offs, chunks)]
    _, result = engine.measured_codebook(engine.words_view(x), segs, exact=True)
    assert float(result[0].item()) == _np_sigma(buf)
    assert rng is not None


def test_sigma_special_values():
    assert zc.measure_sigma(np.full(10, 0x3F80, np.uint16)) == 0.0
    assert zc.measure_sigma(zo.from_f64(np.array([-1.0, 1.0]))) == 1.0
    assert zc.measure_sigma(zo.from_f64(np.array([-1.0, 1.0, np.inf, np.nan]))) == 1.0
    with pytest.raises(zc.DegenerateDataError):
        zc.measure_sigma(np.empty(0, np.uint16))
    with pytest.raises(zc.DegenerateDataError):
        zc.measure_sigma(np.full(5, 0x7F80, np.uint16))


@pytest.mark.parametrize("n", [4095, 4096, 4097, 1 << 20, (1 << 20) + 12345])
def test_codebook_fallbacks_vs_oracle(n):
    rng = np.random.default_rng(n)
    cases = [np.full(n, 0x3F80, np.uint16), np.zeros(n, np.uint16),
             np.full(n, 0x7FC1, np.uint16)]
    mixed = np.full(n, 0x4049, np.uint16)
    mixed[rng.integers(0, n, n // 2 + 1)] = 0x7F80
    cases.append(mixed)
    cases.append(zo.gaussian(n, 3.0, seed=n))
    for w in cases:
        assert zc.codebook_for(w).entries == zo.book_for(w)
        for s in (0.0, float("nan"), -2.0, float("inf")):
            assert zc.codebook_for(w, s).entries == zo.book_for(w, s)


def test_flip_outcomes_match_reference(golden_meta):
    frame = np.load(GOLDEN / "flip_frame.npy")
    arr = frame.copy()
    for i, bit, outcome in golden_meta["flips"]:
        arr[i] ^= bit
        try:
            zc.decompress(zc.parse(arr.tobytes()))
            got = "ok"
        except (CorruptFrameError, CorruptChunkError) as exc:
            got = type(exc).__name__ + ":" + str(exc).split(":")[0]
        arr[i] ^= bit
        assert got == outcome, (i, bit)


def test_c1_digest(golden_meta):
    c1 = golden_meta["c1"]
    w = zo.gaussian(1 << 24, 0.02, 0)
    assert hashlib.sha256(w.tobytes()).hexdigest() == c1["input_sha256"]
    assert zc.measure_sigma(w) == pytest.approx(c1["sigma"], rel=1e-12)
    book = zc.codebook_for(w)
    assert list(book.entries) == c1["book"]
    chunk = zc.compress(w, book)
    frame = zc.serialize(chunk)
    assert len(frame) == c1["frame_len"]
    assert hashlib.sha256(frame).hexdigest() == c1["frame_sha256"]
    assert np.array_equal(host_words(zc.decompress(chunk)), w)


def test_single_word_patterns_round_trip():
    # every 16-bit pattern in its own 1-element frame, in- and out-of-book
    # (reference tests/test_acceptance.py:123-140), batched 64 frames a launch
    words = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    dev = torch.from_numpy(words.view(np.int16)).cuda()
    for mode in ("in", "out"):
        out = torch.empty_like(dev)
        for lo in range(0, 65536, 64):
            seg = list(range(lo, lo + 64))
            exps = [(int(w) >> 7) & 0xFF for w in words[lo:lo + 64]]
            assert len(set(exps)) == 1
            e = exps[0]
            if mode == "in":
                first = min(e, 249)
                book = tuple(range(first, first + 7))
            else:
                book = tuple((e + 8 + i) % 256 for i in range(7))
            cap = engine.max_frame_bytes(1)
            frames = torch.empty(64 * cap, dtype=torch.uint8, device="cuda")
            flen = engine.encode(dev, [(i, 1) for i in seg], engine.book_tensor(book, "cuda"), 9,
                                 frames, [k * cap for k in range(64)])
            err = engine.decode([frames.data_ptr() + k * cap for k in range(64)], [0] * 64,
                                None, [1] * 64, out, seg)
            assert torch.all(err == engine.ERR_OK)
            expect = 128 * 6 + (128 if mode == "out" else 0)
            assert torch.all(flen == expect)
        assert torch.equal(out, dev)


def test_fuzz_buffers_against_oracle():
    rng = np.random.default_rng(31)
    derived = codec.derive_codebook(1.0)
    for _ in range(100):
        n = int(rng.integers(1, 20000))
        w = rng.integers(0, 1 << 16, n).astype(np.uint16)
        gs = int(1 << rng.integers(0, 15))
        book = derived if rng.random() < 0.5 else codec.ExponentCodebook(
            tuple(int(x) for x in rng.choice(256, 7, replace=False)))
        frame = zc.serialize(zc.compress(w, book, gs))
        assert frame == zo.encode(w, book.entries, gs)
        assert np.array_equal(host_words(zc.decompress(zc.parse(frame))), w)


@pytest.mark.parametrize("gs", [4, 16, 512, 2048])
def test_escape_density_mix_two_pass_against_oracle(gs):
    # >= 32 tiles (two-pass encoder, tile-pair lean loop) whose 1024-word
    # blocks cycle through escape densities 0 .. 100 %: warps on both sides
    # of the encoder's dense-escape switch (1/4 of a warp's words), runs that
    # mix them, an odd tail tile and a partial last tile
    rng = np.random.default_rng(gs)
    n = 4096 * 81 + 1234
    w = np.asarray(zo.gaussian(n, 1.0, seed=gs), dtype=np.uint16).copy()
    book = codec.derive_codebook(1.0)
    fr = [0.0, 0.02, 0.1, 0.2, 0.24, 0.26, 0.3, 0.5, 0.75, 0.9, 1.0]
    for b in range(0, n, 1024):
        f = fr[(b // 1024) % len(fr)]
        m = rng.random(min(1024, n - b)) < f
        # exponent 1 (tiny normals): outside any sigma = 1 window
        w[b:b + m.size][m] = (w[b:b + m.size][m] & 0x807F) | (1 << 7)
    frame = zc.serialize(zc.compress(w, book, gs))
    assert frame == zo.encode(w, book.entries, gs)
    assert np.array_equal(host_words(zc.decompress(zc.parse(frame))), w)


@pytest.mark.parametrize("kind,n", [("lognormal2", 4096 * 1100 + 5), ("mix_x1000", 4096 * 1500 + 77),
                                    ("lognormal2", 4096 * 2048), ("mix_n10", 4096 * 1031 + 4095)])
def test_escape_heavy_runs_match_oracle(kind, n):
    # C4 outlier mixes (58-96 % escapes) through the measured-codebook
    # encoder: runs of several thousand escapes take the run fix-up's
    # shifted 16-B copy (any frame alignment of the run, warp-uniform loop)
    # and the dense staging of pass 1; frames byte-exact against the oracle
    w = zo.outlier_mix(n, kind, seed=n % 97)
    x = torch.from_numpy(w.view(np.int16)).cuda()
    book = zc.codebook_for(x)
    assert book.entries == zo.book_for(w)
    frame = zc.serialize(zc.compress(x, book))
    assert frame == zo.encode(w, book.entries)
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    _, _, flen = engine.encode_measured(x, [(0, n)], 9, frames, [0])
    assert bytes(frames[:int(flen.item())].cpu().numpy()) == frame


@pytest.mark.parametrize("n", [1 << 27, 218112000 // 8, 5 * 4096 * 4096 + 3])
def test_large_round_trip_properties(n):
    # size-independent properties at benchmark scale: decode(encode(x)) == x,
    # frame length law, escape count equals an independent torch count
    g = torch.Generator(device="cuda").manual_seed(n)
    x = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    words = engine.words_view(x)
    book = zc.codebook_for(x)
    chunk = zc.compress(x, book)
    e = (words.to(torch.int32) >> 7) & 0xFF
    in_book = torch.zeros(256, dtype=torch.bool, device="cuda")
    in_book[list(book.entries)] = True
    esc = int((~in_book[e]).sum().item())
    assert chunk.zero_count == esc
    assert chunk.frame.numel() == codec.compressed_size_bytes(n, esc)
    out = zc.decompress(chunk)
    assert torch.equal(out, words)


def test_group_random_access():
    for n, gs in [(2000, 512), (2049, 512), (130, 64), (70000, 1 << 14)]:
        data = gaussian_words(n, seed=n + 1)
        chunk = zc.compress(data, codec.derive_codebook(1.0), group_size=gs)
        for g in range((n + gs - 1) // gs):
            got = host_words(zc.decompress_group(chunk, g))
            assert np.array_equal(got, data[g * gs:(g + 1) * gs])
    with pytest.raises(IndexError):
        zc.decompress_group(zc.compress(gaussian_words(100), codec.derive_codebook(1.0)), 1)


@pytest.mark.parametrize("n,gs,book", [(1000, 1, "gauss"), (1001, 2, "gauss"), (999, 8, "miss"),
                                       (5000, 16, "gauss"), (9000, 4096, "miss"),
                                       ((1 << 20) + 77, 1 << 20, "gauss"),
                                       (300_000, 8192, "gauss")])
def test_group_ranges_decode_only_those_groups(n, gs, book):
    # zc_decode_groups over single groups and ranges, against the oracle's
    # words; "miss" = a book no exponent hits (every element escapes)
    data = gaussian_words(n, seed=gs)
    cb = codec.derive_codebook(1.0) if book == "gauss" else codec.ExponentCodebook(
        (10, 11, 12, 13, 14, 15, 16))
    chunk = zc.compress(data, cb, group_size=gs)
    chunk.validate()
    ng = (n + gs - 1) // gs
    rng = np.random.default_rng(n)
    picks = sorted({0, ng - 1, *rng.integers(0, ng, size=min(ng, 6)).tolist()})
    for g in picks:
        got = host_words(engine.decode_groups(chunk.frame, n, gs.bit_length() - 1, g, g + 1))
        assert np.array_equal(got, data[g * gs:(g + 1) * gs]), g
    a, b = ng // 3, min(ng, ng // 3 + 5)
    got = host_words(engine.decode_groups(chunk.frame, n, gs.bit_length() - 1, a, b))
    assert np.array_equal(got, data[a * gs:min(b * gs, n)])


def test_chunk_from_sections_validation():
    c = zc.compress(gaussian_words(2000, seed=42), codec.derive_codebook(1.0))
    sm, planes, gi, ze = c.sign_mantissa, c.exp_planes, c.group_index, c.zero_exponents
    bad = codec.CompressedChunk(c.element_count, c.group_size, c.codebook, sm, planes, gi,
                                ze[:-1])
    with pytest.raises(CorruptChunkError, match="zero_count"):
        zc.decompress(bad)
    bad = codec.CompressedChunk(c.element_count, c.group_size, c.codebook, sm,
                                (planes[0][:-1], planes[1], planes[2]), gi, ze)
    with pytest.raises(CorruptChunkError, match="exp_planes"):
        zc.decompress(bad)
    gi2 = gi.clone()
    gi2[1] += 1
    bad = codec.CompressedChunk(c.element_count, c.group_size, c.codebook, sm, planes, gi2, ze)
    with pytest.raises(CorruptChunkError, match="group_index"):
        zc.decompress(bad)
    good = codec.CompressedChunk(c.element_count, c.group_size, c.codebook, sm, planes, gi, ze)
    assert zc.serialize(good) == zc.serialize(c)


def test_errors_and_dtypes():
    with pytest.raises(ValueError):
        zc.compress(np.empty(0, np.uint16), codec.derive_codebook(1.0))
    with pytest.raises(ValueError):
        zc.compress(gaussian_words(10), codec.derive_codebook(1.0), group_size=100)
    x = torch.randn(3000, device="cuda").to(torch.bfloat16)
    book = zc.codebook_for(x)
    f1 = zc.serialize(zc.compress(x, book))
    f2 = zc.serialize(zc.compress(x.view(torch.int16).cpu().numpy().view(np.uint16), book))
    assert f1 == f2
    out = zc.decompress(zc.parse(f1))
    assert torch.equal(out.view(torch.bfloat16), x)


def test_unaligned_segments_and_batched_frames(golden_meta, golden_a2a):
    # the per-peer batched encoder (K4) on a2a send buffers, unaligned offsets
    world = golden_meta["a2a"]["world"]
    for rank in range(world):
        chunks = [golden_a2a[f"r{rank}_c{q}"] for q in range(world)]
        buf = np.concatenate(chunks)
        offs = np.concatenate([[0], np.cumsum([c.size for c in chunks])])
        dev = torch.from_numpy(buf.view(np.int16)).cuda()
        segs = [(int(offs[q]), chunks[q].size) for q in range(world)
                if q != rank and chunks[q].size]
        peers = [q for q in range(world) if q != rank and chunks[q].size]
        if not segs:
            continue
        book = codec.device_codebook(dev, None, segs)
        caps = [engine.max_frame_bytes(n) for _, n in segs]
        foffs = np.concatenate([[0], np.cumsum(caps)])[:-1]
        frames = torch.empty(int(sum(caps)), dtype=torch.uint8, device="cuda")
        flen = engine.encode(dev, segs, book, 9, frames, foffs).cpu().numpy()
        host = frames.cpu().numpy()
        for k, q in enumerate(peers):
            got = host[foffs[k]:foffs[k] + flen[k]].tobytes()
            assert got == golden_a2a[f"r{rank}_f{q}"].tobytes(), (rank, q)


def _measured_frame(x):
    n = x.numel()
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    book, res, flen = engine.encode_measured(x, [(0, n)], 9, frames, [0], speculative=True)
    return bytes(frames[:int(flen.item())].cpu().numpy()), tuple(book[:7].tolist()), res.cpu()


@pytest.mark.parametrize("case", ["gauss", "sample_fools_guess", "constant", "nan_heavy",
                                  "outliers", "misaligned"])
def test_speculative_measured_encode_is_exact(case):
    n = 4096 * 1500 + 77          # above the speculative threshold (1024 tiles)
    g = torch.Generator(device="cuda").manual_seed(5)
    v = torch.randn(n, device="cuda", generator=g)
    if case == "gauss":
        v = v * 0.02
    elif case == "sample_fools_guess":
        # the guess kernel's sampled sectors (the first 16 words of every
        # second tile) tiny, the rest large: guess != exact, re-encode
        v = v * 1000.0
        v[(torch.arange(n, device="cuda") % 8192) < 16] *= 1e-6
    elif case == "constant":
        v = torch.full((n,), 1.5, device="cuda")
    elif case == "nan_heavy":
        v = v * 3.0
        v[::3] = float("nan")
    elif case == "outliers":
        v = v * 1e-3
        v[::997] *= 1e4
    x = engine.words_view(v.to(torch.bfloat16))
    if case == "misaligned":      # 2-B aligned only: no TMA for any tile, odd tail
        x = x[1:]
    frame, book, res = _measured_frame(x)
    ref_book = zc.codebook_for(x)
    assert book == ref_book.entries
    assert frame == zc.serialize(zc.compress(x, ref_book))
    host = x.cpu().numpy().view(np.uint16)
    assert book == zo.book_for(host)


def test_speculative_encode_in_a_graph_matches_eager():
    """One captured speculative encode replayed over contents whose
    conditional launches return at once (guess right) and that run them
    (guess fooled, certificate failing): each replay matches eager."""
    n = 4096 * 1500 + 77
    g = torch.Generator(device="cuda").manual_seed(9)
    base = torch.randn(n, device="cuda", generator=g)
    contents = {"gauss": base * 0.02}
    fool = base * 1000.0
    fool[(torch.arange(n, device="cuda") % 4096) < 16] *= 1e-6   # the guess's sample
    contents["fools_guess"] = fool
    contents["constant"] = torch.full((n,), 1.5, device="cuda")
    nan = base * 3.0
    nan[::3] = float("nan")
    contents["nan_heavy"] = nan
    contents = {k: engine.words_view(v.to(torch.bfloat16)) for k, v in contents.items()}
    x = contents["gauss"].clone()
    frames = torch.zeros(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    fn = lambda: engine.encode_measured(x, [(0, n)], 9, frames, [0], speculative=True)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        book, res, flen = fn()
    for name in ["gauss", "fools_guess", "gauss", "nan_heavy", "constant", "fools_guess"]:
        x.copy_(contents[name])
        frames.fill_(0xA5)
        graph.replay()
        torch.cuda.synchronize()
        got = bytes(frames[:int(flen.item())].cpu().numpy())
        ref_frame, ref_book, ref_res = _measured_frame(contents[name].clone())
        assert tuple(book[:7].tolist()) == ref_book, name
        assert got == ref_frame, name
        assert torch.equal(res.cpu(), ref_res), name


def test_speculative_multi_segment_matches_prepare_frames(golden_meta):
    # per-peer frames of an all-to-all, sizes above the threshold
    rng = np.random.default_rng(3)
    sizes = [4096 * 400 + 13, 0, 4096 * 700 + 5, 4096 * 100]
    chunks = [zo.from_f64(rng.standard_normal(c) * 0.5) for c in sizes]
    buf = np.concatenate(chunks)
    offs = np.concatenate([[0], np.cumsum(sizes)])[:-1]
    x = torch.from_numpy(buf.view(np.int16)).cuda()
    segs = [(int(offs[q]), sizes[q]) for q in range(4) if q != 1 and sizes[q]]
    caps = [engine.max_frame_bytes(c) for _, c in segs]
    foffs = np.concatenate([[0], np.cumsum(caps)])[:-1]
    frames = torch.empty(int(sum(caps)), dtype=torch.uint8, device="cuda")
    book, _, flen = engine.encode_measured(x, segs, 9, frames, [int(f) for f in foffs],
                                           speculative=True)
    expect = zo.peer_frames(chunks, rank=1)
    host = frames.cpu().numpy()
    fl = flen.cpu().tolist()
    for k, q in enumerate([0, 2, 3]):
        assert host[foffs[k]:foffs[k] + fl[k]].tobytes() == expect[q], q


@pytest.mark.parametrize("sizes", [[4096 * 444], [4096 * 445 + 7], [4096 * 100 + 3] * 3,
                                   [4096 * 150 + 1, 4096 * 150, 4096 * 149 + 99],
                                   [4096 * 2000 + 11, 5, 4096 * 3]])
def test_batched_decode_across_claim_sizes(sizes):
    # the decoder claims one tile per CTA while the batch has at most one tile
    # per resident CTA, four otherwise: totals on both sides of that switch,
    # several frames per launch (segments of different lengths, ragged tails)
    xs = [engine.words_view((torch.randn(c, device="cuda") * 0.02).to(torch.bfloat16))
          for c in sizes]
    chunks = [zc.compress(x, zc.codebook_for(x)) for x in xs]
    out = torch.empty(sum(sizes), dtype=torch.int16, device="cuda")
    offs = np.concatenate([[0], np.cumsum(sizes)])[:-1].tolist()
    frames = [c.frame for c in chunks]
    err = engine.decode([f.data_ptr() for f in frames], [0] * len(sizes), None, sizes, out,
                        [int(o) for o in offs])
    assert torch.all(err == engine.ERR_OK)
    for x, o, c in zip(xs, offs, sizes):
        assert torch.equal(out[o:o + c], x)


def test_profile_hooks_record_encoder_and_decoder_launches():
    n = 4096 * 1200 + 5
    x = engine.words_view((torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16))
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(x)
    engine.profile_enable(True)
    try:
        for _ in range(3):
            engine.encode_measured(x, [(0, n)], 9, frames, [0])
            engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
    finally:
        engine.profile_enable(False)
    enc, dec = engine.profile_read(engine.PROF_ENCODE), engine.profile_read(engine.PROF_DECODE)
    assert len(enc) == 3 and len(dec) == 3
    assert all(t > 0 for t in enc + dec)
    assert torch.equal(out, x)


def test_two_host_threads_share_a_stream():
    # ctypes releases the GIL inside the C calls: two threads driving the same
    # stream must not interleave their launches over the shared workspace
    import threading
    stream = torch.cuda.current_stream()
    results = {}

    def work(tid):
        torch.cuda.set_device(0)
        ok = True
        with torch.cuda.stream(stream):
            for it in range(6):
                n = 4096 * (300 + 37 * tid) + it
                x = engine.words_view((torch.randn(n, device="cuda") * (0.02 + tid)).to(
                    torch.bfloat16))
                frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
                _, _, flen = engine.encode_measured(x, [(0, n)], 9, frames, [0])
                out = torch.empty_like(x)
                err = engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
                ok &= int(err.item()) == engine.ERR_OK and torch.equal(out, x)
        results[tid] = ok

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert results == {0: True, 1: True}


def test_collective_c_abi_world1_over_nccl():
    """The collective C-ABI exactly as a non-Python integrator drives it:
    NCCL unique id -> zc_comm_init -> zc_allgather / zc_alltoall /
    zc_reduce_scatter (+ raw twins) on device pointers, W = 1."""
    import ctypes
    from paper_2604_27844_b200._lib import i64s, lib
    L = lib()
    nb = L.zc_nccl_id_bytes()
    uid = (ctypes.c_uint8 * nb)()
    assert L.zc_nccl_get_id(uid) == 0
    comm = ctypes.c_void_p()
    torch.cuda.set_device(0)
    assert L.zc_comm_init(ctypes.byref(comm), uid, 0, 1, 1 << 24, 0) == 0
    try:
        info = (ctypes.c_int * 5)()
        assert L.zc_comm_info(comm, info) == 0 and list(info)[:2] == [0, 1] and info[4] == 1
        words = zo.gaussian(50_001, 0.02, 11)
        x = torch.from_numpy(words.view(np.int16)).cuda()
        out = torch.empty_like(x)
        err = torch.empty(1, dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        assert L.zc_allgather(comm, x.data_ptr(), x.numel(), out.data_ptr(), None,
                              err.data_ptr(), 0, st) == 0
        assert torch.equal(out, x) and int(err.item()) == 0x7F7F7F7F
        out.zero_()
        assert L.zc_allgather_raw(comm, x.data_ptr(), x.numel(), out.data_ptr(), st) == 0
        assert torch.equal(out, x)
        out.zero_()
        cnt = i64s([x.numel()])
        assert L.zc_alltoall(comm, x.data_ptr(), cnt, cnt, out.data_ptr(), None, err.data_ptr(),
                             0, st) == 0
        assert torch.equal(out, x)
        rs = torch.empty(50_000, dtype=torch.float32, device="cuda")
        assert L.zc_reduce_scatter(comm, x.data_ptr(), 50_000, rs.data_ptr(), 1, None,
                                   err.data_ptr(), 0, st) == 0
        assert np.array_equal(rs.cpu().numpy().view(np.uint32),
                              zo.to_f32(words[:50_000]).view(np.uint32))
        b, m = ctypes.c_uint64(), ctypes.c_uint64()
        assert L.zc_comm_stats(comm, ctypes.byref(b), ctypes.byref(m)) == 0
        assert b.value == 0                          # nothing leaves a 1-rank group
        # mismatched self counts are an argument error, not a hang
        assert L.zc_alltoall(comm, x.data_ptr(), cnt, i64s([7]), out.data_ptr(), None,
                             err.data_ptr(), 0, st) == -1
    finally:
        L.zc_comm_destroy(comm)


def test_zbf16_round_trip(tmp_path):
    # reference tests/test_container.py:172-179, plus the file bytes against the oracle
    data = gaussian_words(1234, seed=8)
    chunk = zc.compress(data, zc.derive_codebook(1.0))
    path = tmp_path / "x.zbf16"
    nbytes = container.write_zbf16(path, chunk)
    assert path.stat().st_size == nbytes
    assert path.read_bytes() == zo.encode(data, zc.derive_codebook(1.0).entries)
    back = zc.decompress(container.read_zbf16(path))
    assert np.array_equal(back.cpu().numpy().view(np.uint16), data)


@pytest.mark.parametrize("n", [1, 15, 511, 512, 513, 4095, 4096, 4097, 12_345, 65_536,
                               131_071, 131_072, 131_073, 262_143, 262_144, 262_145])
@pytest.mark.parametrize("shift", [0, 1, 8])
def test_small_message_path_matches_oracle(n, shift):
    """One-launch cluster encoder / decoder (zc_small.cu) at the sizes around
    its CTA split and its threshold, with 16-B aligned (TMA) and misaligned
    inputs, specials included; frames byte-identical to the oracle."""
    words = zo.gaussian(n + shift, 0.02, seed=n % 97)
    if n >= 8:
        words[shift:shift + 6] = [0x7FC0, 0x7F80, 0xFF80, 0x0000, 0x8000, 0x0001]
    base = torch.from_numpy(words.view(np.int16)).cuda()
    x = base[shift:]
    book = zc.codebook_for(x)
    want_book = zo.book_for(words[shift:])
    assert book.entries == want_book
    frame = zc.serialize(zc.compress(x, book))
    assert frame == zo.encode(words[shift:], want_book)
    # fused codebook_for + compress (the measured one-launch path)
    f2 = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    b2, res, flen = engine.encode_measured(x, [(0, n)], 9, f2, [0])
    assert tuple(b2[:7].cpu().tolist()) == want_book
    assert bytes(f2[:int(flen.item())].cpu().numpy()) == frame
    out = torch.empty(n + 3, dtype=torch.int16, device="cuda")[3:]      # misaligned output
    err = engine.decode([f2.data_ptr()], [0], None, [n], out, [0], groups512=True)
    assert int(err[0].item()) == engine.ERR_OK and torch.equal(out, x)


@pytest.mark.parametrize("case", ["nan_slice", "constant", "scales", "offset_mean", "one_finite"])
def test_small_statistic_merge_edge_cases(case):
    """The one-launch encoder merges per-CTA (sum, mean, M2) partials: slices
    without a finite element, a zero variance (modal fallback), CTAs whose
    scales and means differ by orders of magnitude.  Book and frame equal
    the oracle's, sigma within 1e-12 of numpy's two-pass np.std."""
    n = 100_000                                    # 8 CTAs of 12 800 words
    rng = np.random.default_rng(11)
    v = rng.standard_normal(n) * 0.02
    if case == "nan_slice":
        v[:40_000] = np.nan                        # the first CTAs see no finite value
    elif case == "constant":
        v[:] = 0.75
    elif case == "scales":
        v[: n // 2] *= 1e5                         # the between-CTA term dominates M2
    elif case == "offset_mean":
        v += 300.0
    elif case == "one_finite":
        v[:] = np.inf
        v[77_777] = 3.0
    words = zo.from_f64(v)
    x = torch.from_numpy(words.view(np.int16)).cuda()
    want_book = zo.book_for(words)
    f = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    b, res, flen = engine.encode_measured(x, [(0, n)], 9, f, [0])
    assert tuple(b[:7].cpu().tolist()) == want_book
    assert bytes(f[:int(flen.item())].cpu().numpy()) == zo.encode(words, want_book)
    fin = zo.to_f32(words).astype(np.float64)
    fin = fin[np.isfinite(fin)]
    sigma = float(res[0].item())
    if fin.size:
        ref = float(np.std(fin))
        assert sigma == pytest.approx(ref, rel=1e-12, abs=0.0 if ref else 1e-300)
    else:
        assert math.isnan(sigma)


def test_small_decoder_rejects_foreign_group_size_and_corruption():
    words = zo.gaussian(3000, 1.0, seed=5)
    x = torch.from_numpy(words.view(np.int16)).cuda()
    chunk = zc.compress(x, zc.codebook_for(x), group_size=256)
    out = torch.empty_like(x)
    err = engine.decode([chunk.frame.data_ptr()], [0], None, [3000], out, [0], groups512=True)
    assert int(err[0].item()) == 22                   # the caller's 512 promise was wrong
    assert torch.equal(zc.decompress(chunk), x)      # the general decoder handles it
    f = zc.compress(x, zc.codebook_for(x)).frame.clone()
    off_gi = codec.section_offsets(3000, 512)[4]
    f[off_gi + 4] ^= 1                                 # group_index[1] off by one
    err = engine.decode([f.data_ptr()], [0], None, [3000], out, [0], groups512=True)
    assert int(err[0].item()) == 17                    # "group_index" (reference field)


def test_decompress_out_is_validated():
    # a short / non-contiguous / foreign-device `out` must not be
    # written past its end or silently replaced by a copy
    words = zo.gaussian(5000, 0.02, seed=3)
    x = torch.from_numpy(words.view(np.int16)).cuda()
    chunk = zc.compress(x, zc.codebook_for(x))
    with pytest.raises(ValueError):
        zc.decompress(chunk, out=torch.empty(4999, dtype=torch.int16, device="cuda"))
    with pytest.raises(ValueError):
        zc.decompress(chunk, out=torch.empty(10000, dtype=torch.int16, device="cuda")[::2])
    with pytest.raises(ValueError):
        zc.decompress(chunk, out=torch.empty(5000, dtype=torch.int16))
    with pytest.raises(ValueError):
        zc.decompress(chunk, out=torch.empty(5000, dtype=torch.int32, device="cuda"))
    out = torch.empty(5000, dtype=torch.bfloat16, device="cuda")
    zc.decompress(chunk, out=out)
    assert torch.equal(out.view(torch.int16), x)


def test_decode_when_ready_decodes_late_frames_and_times_out():
    # zc_decode_when_ready: frames decoded as their ready flags appear (the
    # reference's per-peer decode inside its receive loop, collectives.py:216-227)
    sizes = [4096 * 300 + 17, 70001, 4096 * 40]
    xs = [engine.words_view((torch.randn(c, device="cuda") * 0.02).to(torch.bfloat16))
          for c in sizes]
    frames = [zc.compress(x, zc.codebook_for(x)).frame for x in xs]
    out = torch.empty(sum(sizes), dtype=torch.int16, device="cuda")
    offs = [0, sizes[0], sizes[0] + sizes[1]]
    flags = torch.zeros(3, dtype=torch.int64, device="cuda")
    ready = [flags.data_ptr() + 8 * i for i in range(3)]
    flags[0] = 5
    flags[2] = 5
    side = torch.cuda.Stream()
    err = engine.decode_when_ready([f.data_ptr() for f in frames], sizes, out, offs, ready, 5,
                                   timeout_ns=10_000_000_000)
    # the middle frame is published after the launch, from another stream
    one = torch.full((1,), 5, dtype=torch.int64).pin_memory()
    with torch.cuda.stream(side):   # a copy-engine write while the decode runs
        flags[1:2].copy_(one, non_blocking=True)
    torch.cuda.synchronize()
    assert torch.all(err == engine.ERR_OK)
    for x, o, c in zip(xs, offs, sizes):
        assert torch.equal(out[o:o + c], x)
    # a flag that never reaches the epoch: error word 20 (timeout) for that frame only
    out.zero_()
    flags[0] = 6
    err = engine.decode_when_ready([f.data_ptr() for f in frames], sizes, out, offs, ready, 6,
                                   timeout_ns=20_000_000)
    codes = err.cpu().tolist()
    assert codes[0] == engine.ERR_OK and codes[1] == 20 and codes[2] == 20
    assert torch.equal(out[:sizes[0]], xs[0])


@pytest.mark.parametrize("n", [3, 129, 8195, 100003, (1 << 20) + 5])
def test_sigma_bit_identical_with_non_finite(n):
    # the reference takes np.std of the COMPACTED finite values, so numpy's
    # tree runs over their indices: measure_sigma compacts on the device and
    # evaluates numpy's order over that array (NaN payloads, +-inf, ragged)
    rng = np.random.default_rng(n)
    for k in (1, 2, max(1, n // 50)):
        w = zo.gaussian(n, 0.02, seed=n + k)
        pos = rng.choice(n, size=min(k, n - 1), replace=False)
        w[pos] = rng.choice(np.array([0x7FC0, 0xFFC1, 0x7F80, 0xFF80, 0x7F81], dtype=np.uint16),
                            size=pos.size)
        got = zc.measure_sigma(w)
        assert got == _np_sigma(w), (n, k, got, _np_sigma(w))
