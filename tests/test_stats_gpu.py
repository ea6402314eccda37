"""Certified codebook pass (zc_stats.cu sums_kernel + certify_block) against
the reference statistic: the packed-fp32 pass may decide the codebook only
when the whole error interval of sigma maps to one codebook; everything near a
flip threshold, non-finite or badly conditioned must fall back to the exact
f64 pass (reference bf16.measure_sigma, bf16.py:88-103, and
codec.derive_codebook, codec.py:149-161)."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from oracle import zc_oracle as zo

pytestmark = pytest.mark.gpu

from paper_2604_27844_b200 import engine  # noqa: E402

PATH_EXACT, PATH_MODAL, PATH_CERTIFIED = 1.0, 2.0, 3.0


def _measure(host: np.ndarray):
    x = torch.from_numpy(host.view(np.int16)).cuda()
    book, res = engine.measured_codebook(x)
    exact_book, exact = engine.measured_codebook(x, exact=True)
    return tuple(book[:7].tolist()), res.cpu().tolist(), tuple(exact_book[:7].tolist()), \
        exact.cpu().tolist()


def _flip_sigma(octave: int) -> float:
    """sigma where derive() switches from floor to ceil inside an octave
    (bisection on the oracle's decision)."""
    lo, hi = 2.0 ** octave, 2.0 ** (octave + 1)
    b_lo = zo.derive(lo)
    assert zo.derive(hi) != b_lo
    for _ in range(200):
        mid = math.sqrt(lo * hi)
        if zo.derive(mid) == b_lo:
            lo = mid
        else:
            hi = mid
    return hi


def _three_point(target: float, n: int, rel: float, seed: int) -> np.ndarray:
    """n words in {+a, -a, 0} (equal +a/-a counts: mean exactly 0) whose
    population std is target * (1 + rel) to ~3e-7 relative: sigma = a * sqrt(2p / n)."""
    want = target * (1.0 + rel)
    e = math.floor(math.log2(want))
    best = None
    for m in range(128, 256):                       # bf16 mantissas of one octave
        for de in (-1, 0):
            a = m * 2.0 ** (e + de - 7)
            p = round(want * want * n / (2 * a * a))
            if not 1 <= p <= n // 2:
                continue
            s = a * math.sqrt(2 * p / n)
            err = abs(s / want - 1.0)
            if best is None or err < best[0]:
                best = (err, a, p)
    _, a, p = best
    v = np.zeros(n)
    v[:p], v[p:2 * p] = a, -a
    np.random.default_rng(seed).shuffle(v)
    return zo.from_f64(v)


def test_certified_on_model_like_data():
    for seed, s in enumerate([0.02, 1.0, 3e-5, 250.0]):
        host = zo.gaussian(1 << 20, s, seed=seed)
        book, res, ebook, eres = _measure(host)
        assert res[2] == PATH_CERTIFIED, res
        assert book == ebook == zo.book_for(host)
        assert res[0] == pytest.approx(eres[0], rel=4e-6)
        assert res[1] == eres[1] == host.size


@pytest.mark.parametrize("octave", [-9, -6, 0, 5])
@pytest.mark.parametrize("rel", [1e-8, -1e-8, 3e-7, -3e-7])
def test_near_flip_threshold_falls_back(octave, rel):
    target = _flip_sigma(octave)
    host = _three_point(target, 1 << 20, rel, seed=octave & 0xFF)
    s = zo.sigma(host)
    assert abs(s / target - 1.0) < 1e-6               # inside the certificate's interval
    book, res, ebook, _ = _measure(host)
    assert book == zo.book_for(host) == ebook
    assert res[2] == PATH_EXACT, res                 # the certificate must refuse


def test_far_from_threshold_is_certified():
    target = _flip_sigma(-6)
    host = _three_point(target, 1 << 20, 0.05, seed=1)
    book, res, _, _ = _measure(host)
    assert res[2] == PATH_CERTIFIED and book == zo.book_for(host)


@pytest.mark.parametrize("case", ["first_outlier", "big_mean", "nan", "inf", "neg_inf_pair",
                                  "constant", "all_nan", "huge"])
def test_fallback_cases_match_reference(case):
    n = (1 << 18) + 77
    host = zo.gaussian(n, 0.02, seed=3)
    if case == "first_outlier":          # K = x[0] far from the mean: Q >> M2
        host[0] = zo.from_f64(np.array([1e4]))[0]
    elif case == "big_mean":             # mean/sigma = 1e4 but K = x[0] near the mean
        host = zo.from_f64(1000.0 + np.random.default_rng(2).standard_normal(n) * 0.1)
    elif case == "nan":
        host[12345] = 0x7FC0
    elif case == "inf":
        host[-1] = 0x7F80
    elif case == "neg_inf_pair":
        host[5], host[6] = 0x7F80, 0xFF80
    elif case == "constant":
        host[:] = 0x3FC0
    elif case == "all_nan":
        host[:] = 0x7FC1
    elif case == "huge":                 # d^2 overflows fp32
        host[100] = 0x7F00
    book, res, ebook, eres = _measure(host)
    assert book == ebook == zo.book_for(host), (case, res)
    if case in ("nan", "inf", "neg_inf_pair", "constant", "all_nan", "huge"):
        assert res[2] in (PATH_EXACT, PATH_MODAL), (case, res)
    # first_outlier: Q/M2 ~ n widens the interval to ~+-25 %, which may still
    # sit inside one codebook -- certified or not, the book must match
    # (the exact request adds numpy's summation order, so its sigma may differ
    # from the fallback's Chan pass in the last bits; the codebook may not)
    if res[2] != PATH_CERTIFIED:
        assert res[1:] == eres[1:], (case, res, eres)
        assert (math.isnan(res[0]) and math.isnan(eres[0])) or \
            res[0] == pytest.approx(eres[0], rel=1e-12, abs=0), (case, res, eres)
    v = (host.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if np.isfinite(v).all():             # measure_sigma's value: np.std bit for bit
        assert eres[0] == float(np.std(v)), (case, eres)


def test_certified_multi_segment_and_unaligned():
    rng = np.random.default_rng(9)
    buf = zo.from_f64(rng.standard_normal(3 * 100_003 + 5) * 0.3)
    x = torch.from_numpy(buf.view(np.int16)).cuda()
    segs = [(1, 100_003), (100_004, 0), (200_007, 100_001)]   # odd offsets: no TMA
    book, res = engine.measured_codebook(x, segs)
    concat = np.concatenate([buf[o:o + c] for o, c in segs])
    assert tuple(book[:7].tolist()) == zo.book_for(concat)
    assert res[1].item() == concat.size
    assert res[0].item() == pytest.approx(zo.sigma(concat), rel=4e-6)


@pytest.mark.parametrize("rel", [2e-5, -2e-5, 5e-4, -5e-4, 3e-3, -3e-3])
def test_exact_derivation_both_sides_of_flip_window(rel):
    # the device derivation skips the erf comparison when frac(x_opt) is more
    # than kFlipWindow (1e-4) from the flip; these straddle that window
    target = _flip_sigma(-7)
    host = _three_point(target, 1 << 20, rel, seed=7)
    x = torch.from_numpy(host.view(np.int16)).cuda()
    book, res = engine.measured_codebook(x, exact=True)
    assert tuple(book[:7].tolist()) == zo.book_for(host), (rel, res.tolist())


def _speculative(host: np.ndarray):
    x = torch.from_numpy(host.view(np.int16)).cuda()
    n = host.size
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    book, res, flen = engine.encode_measured(x, [(0, n)], 9, frames, [0], speculative=True)
    frame = frames[:int(flen.item())].cpu().numpy().tobytes()
    return tuple(book[:7].tolist()), res.cpu().tolist(), frame


@pytest.mark.parametrize("rel", [1e-8, -1e-8, 3e-7, -3e-7])
def test_speculative_near_flip_falls_back_to_exact(rel):
    # above the speculative threshold; the fused certificate must refuse and
    # the exact pass (then a re-encode when the guess was wrong) decides
    target = _flip_sigma(-6)
    host = _three_point(target, 1 << 23, rel, seed=11)
    book, res, frame = _speculative(host)
    assert book == zo.book_for(host)
    assert res[2] == PATH_EXACT, res
    assert frame == zo.encode(host, book)


def test_speculative_cluster_outside_sample_grid():
    # layer-like: N(0, 0.02^2) weights + a block of 1.0 (RMSNorm) at the end;
    # a tile sample would over-weight the block, the uniform sample must not
    # (either way the output is exact)
    n = (1 << 23) + 8192
    host = zo.gaussian(n, 0.02, seed=4)
    host[-8192:] = 0x3F80
    book, res, frame = _speculative(host)
    assert book == zo.book_for(host)
    assert res[2] == PATH_CERTIFIED, res
    assert frame == zo.encode(host, book)


def _tuned(target: float, n: int, rel: float, seed: int) -> np.ndarray:
    """N(0, (0.9 target)^2) words plus +-a / +-b / +-c pairs (a ~ 2 sigma,
    b = a/64, c = a/4096; pairs leave the sum unchanged) whose np.std is
    target * (1 + rel) to ~1e-13 relative: data that sits next to a flip
    threshold far inside the window where only the summation order decides."""
    want = target * (1.0 + rel)
    f64 = lambda w: (w.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    q = lambda v: float(f64(zo.from_f64(np.array([v])))[0])                         # noqa: E731
    R = n // 4                                    # pair slots
    base = f64(zo.gaussian(n - 2 * R, 0.9 * want, seed=seed))
    a = q(2.0 * want)
    b, c = a / 64.0, a / 4096.0                   # exact: powers of two apart
    S0, Q0 = math.fsum(base), math.fsum(base * base)
    D = ((want * want + (S0 / n) ** 2) * n - Q0) / 2.0   # sum of pair magnitudes^2 needed
    counts = []
    for m in (a, b):
        k = int(D // (m * m)) - 1 if m == a else int(D // (m * m))
        counts.append(max(k, 0))
        D -= counts[-1] * m * m
    counts.append(int(round(D / (c * c))))
    assert sum(counts) <= R and min(counts) >= 0, counts

    def build(kc):
        v = np.zeros(n)
        v[:base.size] = base
        i = base.size
        for m, k in zip((a, b, c), (counts[0], counts[1], kc)):
            v[i:i + k], v[i + k:i + 2 * k] = m, -m
            i += 2 * k
        np.random.default_rng(seed + 1).shuffle(v)
        return v
    best = None
    for kc in range(counts[2] - 3, counts[2] + 4):          # land on the closest
        v = build(kc)
        err = abs(float(np.std(v)) / want - 1.0)
        if best is None or err < best[0]:
            best = (err, v)
    assert best[0] < 1e-12, best[0]
    return zo.from_f64(best[1])


@pytest.mark.parametrize("n,octave,rel", [(1 << 20, -6, 3e-11), (1 << 20, -6, -3e-11),
                                          (1 << 20, 2, 4e-12), (1 << 23, -7, -2e-11),
                                          (1 << 18, -6, 3e-11), (1 << 18, -9, -5e-12)])
def test_near_flip_codebook_uses_numpy_sigma(n, octave, rel):
    # the certificate refuses, the f64 fallback lands within 2^-30 of the flip,
    # and the codebook is re-derived from numpy's summation order: sigma equal
    # to np.std bit for bit on the codebook_for path (not only measure_sigma),
    # through the multi-CTA statistic (2^20, 2^23) and the one-launch cluster
    # encoder (2^18)
    target = _flip_sigma(octave)
    host = _tuned(target, n, rel, seed=n + octave)
    v = (host.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    ref_sigma = float(np.std(v))
    assert abs(ref_sigma / target - 1.0) < 1e-10
    book, res, _, eres = _measure(host)
    assert book == zo.book_for(host)
    assert res[2] == PATH_EXACT, res
    assert res[0] == ref_sigma == eres[0], (res, eres, ref_sigma)
    sbook, sres, frame = _speculative(host)
    assert sbook == zo.book_for(host) and sres[0] == ref_sigma, (sres, ref_sigma)
    assert frame == zo.encode(host, sbook)


@pytest.mark.parametrize("n,rel,nan", [(1 << 20, 3e-13, True), (1 << 20, -3e-13, True),
                                       (1 << 18, 2e-13, True), (1 << 20, -2e-13, False)])
def test_public_codebook_for_next_to_flip(n, rel, nan):
    # public codebook_for within 1e-12 of a flip: numpy-order sigma over the
    # compacted finite values and the reference's host derivation (math.erf),
    # with a NaN in the data (the device f64 fallback cannot take numpy's
    # order over the compacted array)
    import paper_2604_27844_b200 as zc
    target = _flip_sigma(-6)
    body = _tuned(target, n - 1 if nan else n, rel, seed=n + 5)
    host = np.insert(body, n // 3, np.uint16(0x7FC0)) if nan else body
    assert zc.measure_sigma(host) == _np_sigma_finite(host)
    assert zc.codebook_for(host).entries == zo.book_for(host)


def _np_sigma_finite(words: np.ndarray) -> float:
    with np.errstate(invalid="ignore"):
        v = (words.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return float(np.std(v[np.isfinite(v)]))
