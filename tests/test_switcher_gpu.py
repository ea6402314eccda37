"""Adaptive switch on the GPU path, thread ranks sharing one GPU: profile()
(reference tests/test_switcher.py:107-138), the switched collectives
(:152-168), the message-adaptive raw fallback for incompressible data
 and rank-consistent all-to-all decisions."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from tests.conftest import rank_words

pytestmark = pytest.mark.gpu

from paper_2604_27844_b200 import engine  # noqa: E402
from paper_2604_27844_b200.collectives import (  # noqa: E402
    AlltoAllSpec, reference_all_gather, reference_all_to_all, reference_reduce_scatter)
from paper_2604_27844_b200.switcher import (  # noqa: E402
    CostModel, Path, SwitchPolicy, _measured_e, profile, profile_variants, switched_all_gather,
    switched_all_to_all, switched_reduce_scatter)
from paper_2604_27844_b200.transport import run_ranks  # noqa: E402

FORCE_ZIP = CostModel(1e-3, 1e-9, 1e-9, 1e-12, e=0.7)
FORCE_NATIVE = CostModel(1e-9, 1e-12, 1e-3, 1e-9, e=0.7)


def H(t):
    return t.cpu().numpy().view(np.uint16)


def outlier_mix(n, seed, kind="x1000"):
    """SURVEY Appendix C.4 gradient mixes (ratio 0.93 / 0.86: frames expand)."""
    from oracle import zc_oracle as zo
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(n) * 1e-3
    ln = np.exp(rng.standard_normal(n) - 8.0) * rng.choice([-1.0, 1.0], n)
    mix = np.where(rng.random(n) < 0.5, g, ln)
    if kind == "x1000":
        mix[rng.integers(0, n, n // 1000)] *= 1000
    else:
        mix[rng.integers(0, n, n // 10000)] = rng.standard_normal(n // 10000) * 10
    return zo.from_f64(mix)


@pytest.mark.parametrize("op", ["reduce_scatter", "all_gather", "all_to_all"])
def test_profile_measures_e_and_agrees(op):
    def body(comm):
        return profile(comm, [1 << 16, 1 << 20, 1 << 22], trials=2, seed=5, op=op)
    models = run_ranks(4, body)
    assert all(m == models[0] for m in models)
    assert 0.66 <= models[0].e <= 0.72


def test_measured_e_of_incompressible_data_exceeds_one():
    def body(comm):
        return _measured_e(comm, outlier_mix(1 << 18, comm.rank), "reduce_scatter")
    es = run_ranks(2, body)
    assert es[0] == es[1] and es[0] > 1.0
    with pytest.raises(ValueError):
        CostModel(1e-5, 1e-9, 1e-5, 1e-9, e=es[0])


@pytest.mark.parametrize("n", [1 << 20, 1 << 24])
def test_estimate_ratio_tracks_the_frame(n):
    from oracle import zc_oracle as zo
    for words in (zo.gaussian(n, 0.02, 3), outlier_mix(n, 4), outlier_mix(n, 5, "n10")):
        x = torch.from_numpy(words.view(np.int16)).cuda()
        est = float(engine.estimate_ratio(x)[0].item())
        exact = len(zo.encode(words, zo.book_for(words))) / (2 * n)
        assert abs(est - exact) / exact < 0.03, (est, exact)


def test_switched_paths_follow_model_and_are_exact():
    # reference tests/test_switcher.py:152-168, all three collectives
    def body(comm):
        local = rank_words(comm.rank, comm.world_size * 4096)
        ref_rs = H(reference_reduce_scatter(comm, local))
        ref_ag = H(reference_all_gather(comm, local))
        out = []
        for model in (FORCE_ZIP, FORCE_NATIVE):
            rs, p_rs = switched_reduce_scatter(comm, local, model)
            ag, p_ag = switched_all_gather(comm, local, model)
            out.append((p_rs, np.array_equal(H(rs), ref_rs), p_ag, np.array_equal(H(ag), ref_ag)))
        return out
    for (pz, okz, pz2, okz2), (pn, okn, pn2, okn2) in run_ranks(4, body):
        assert pz is Path.ZIPPED and pz2 is Path.ZIPPED and okz and okz2
        assert pn is Path.NATIVE and pn2 is Path.NATIVE and okn and okn2


@pytest.mark.parametrize("kind", ["x1000", "n10"])
def test_incompressible_message_goes_native(kind):
    def body(comm):
        local = outlier_mix(comm.world_size * (1 << 16), comm.rank, kind)
        rs, p_rs = switched_reduce_scatter(comm, local, FORCE_ZIP)
        ag, p_ag = switched_all_gather(comm, local, FORCE_ZIP)
        ok = np.array_equal(H(rs), H(reference_reduce_scatter(comm, local)))
        ok &= np.array_equal(H(ag), H(reference_all_gather(comm, local)))
        # the non-adaptive switch would have zipped it
        _, p_fixed = switched_all_gather(comm, local, FORCE_ZIP, adaptive=False)
        return p_rs, p_ag, ok, p_fixed
    for p_rs, p_ag, ok, p_fixed in run_ranks(4, body):
        assert p_rs is Path.NATIVE and p_ag is Path.NATIVE and ok
        assert p_fixed is Path.ZIPPED


def test_all_to_all_decision_is_rank_consistent():
    # rank 0 sends 64x more than the others; the crossover lies between the
    # ranks' own send sizes, so a per-rank decision would split the group
    model = CostModel(alpha_rs=1e-6, beta_rs=1e-9, alpha_a2a=2e-4, beta_a2a=1e-9, e=0.7)
    # crossover ~ 2e-4 / (0.3e-9) ~ 660 KB; rank 0 sends ~ 3 MB, the others ~ 48 KB

    def body(comm):
        per = 4 * 4096 * (64 if comm.rank == 0 else 1)
        chunks = [rank_words(comm.rank * 8 + q, per // 4, seed=2) for q in range(4)]
        recv = [4 * 4096 * (64 if p == 0 else 1) // 4 for p in range(4)]
        spec = AlltoAllSpec(chunks, recv)
        got, path = switched_all_to_all(comm, spec, model)
        ref = reference_all_to_all(comm, spec)
        return path, all(np.array_equal(H(a), H(b)) for a, b in zip(got, ref))
    res = run_ranks(4, body)
    assert all(r[1] for r in res)
    assert len({r[0] for r in res}) == 1 and res[0][0] is Path.ZIPPED


def test_profile_variants_policy():
    def body(comm):
        pol = profile_variants(comm, "all_gather", sizes=[1 << 16, 1 << 22], trials=1)
        local = rank_words(comm.rank, 1 << 18)
        got, path = switched_all_gather(comm, local, pol)
        return pol, path, np.array_equal(H(got), H(reference_all_gather(comm, local)))
    res = run_ranks(3, body)
    pol = res[0][0]
    assert isinstance(pol, SwitchPolicy) and [v for v, _ in pol.models] == ["p2p", "msg"]
    assert all(r[0] == pol for r in res) and all(r[2] for r in res)
    assert len({r[1] for r in res}) == 1
