"""Compressed collectives vs the uncompressed ones (bit-identical), protocol
errors, reduction contract — reference tests/test_collectives.py:26-317 and
tests/test_acceptance.py:155-219, on thread ranks sharing one GPU."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import zc_oracle as zo
from tests.conftest import rank_words

pytestmark = pytest.mark.gpu

from paper_2604_27844_b200 import codec  # noqa: E402
from paper_2604_27844_b200.collectives import (  # noqa: E402
    AlltoAllSpec, reference_all_gather, reference_all_to_all, reference_reduce_scatter,
    timed_call, zip_all_gather, zip_all_reduce, zip_all_to_all_d1, zip_all_to_all_d2,
    zip_reduce_scatter)
from paper_2604_27844_b200.errors import CollectiveError, ProtocolError  # noqa: E402
from paper_2604_27844_b200.transport import run_ranks as _run_ranks  # noqa: E402

# every protocol runs on three implementations: the native engine's
# peer-memory plane, its message plane (the reference's protocols over the
# in-process device-copy transport that stands in for NCCL), and the generic
# Python protocols over the thread hub
MODES = ["p2p", "msg", "generic"]


def run_ranks(world, body, mode="p2p", **kw):
    def wrapped(comm):
        if mode == "generic":
            comm.use_native = False
        elif comm.native is not None:
            comm.native.plane = "msg" if mode.startswith("msg") else "p2p"
            comm.native.pipeline = mode == "msg_pipe"
        return body(comm)
    return _run_ranks(world, wrapped, native=(mode != "generic") and world <= 64, **kw)


def H(t):
    return t.cpu().numpy().view(np.uint16)


def _a2a_spec(comm, sizer, seed=0):
    chunks = [rank_words(comm.rank * 131 + q, sizer(comm.rank, q), seed=seed)
              for q in range(comm.world_size)]
    counts = [sizer(p, comm.rank) for p in range(comm.world_size)]
    return AlltoAllSpec(chunks, counts)


@pytest.mark.parametrize("mode", MODES + ["msg_pipe"])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_all_gather_matches_reference(world, mode):
    def body(comm):
        outs = []
        for it in range(3):   # epochs: slot reuse guarded by the done flags
            local = rank_words(comm.rank + 7 * it, 4096 * 5 + 17 + it)
            outs.append((H(zip_all_gather(comm, local)), H(reference_all_gather(comm, local))))
        return outs
    for outs in run_ranks(world, body, mode):
        for z, r in outs:
            assert np.array_equal(z, r)


@pytest.mark.parametrize("mode", MODES)
def test_all_gather_large_and_specials(mode):
    def body(comm):
        local = rank_words(comm.rank, 3_000_001, sigma=0.02)
        local[:8] = [0x7FC0, 0x7F80, 0xFF80, 0, 0x8000, 1, 0x7F81, 0xFFFF]
        z = zip_all_gather(comm, local)
        return H(z), np.concatenate([rank_words(r, 3_000_001, sigma=0.02)
                                     for r in range(comm.world_size)])
    outs = run_ranks(3, body, mode)
    for z, expect in outs:
        expect = expect.copy()
        for r in range(3):
            expect[r * 3_000_001:r * 3_000_001 + 8] = [0x7FC0, 0x7F80, 0xFF80, 0, 0x8000, 1,
                                                         0x7F81, 0xFFFF]
        assert np.array_equal(z, expect)


def test_all_gather_all_nan_payloads():
    def body(comm):
        rng = np.random.default_rng(comm.rank)
        local = (0x7F81 + rng.integers(0, 0x7F, 500)).astype(np.uint16)
        return H(zip_all_gather(comm, local)), H(reference_all_gather(comm, local))
    for z, r in run_ranks(4, body):
        assert np.array_equal(z, r)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("fn", [zip_all_to_all_d1, zip_all_to_all_d2])
@pytest.mark.parametrize("sizer", [lambda s, d: 2000, lambda s, d: s * 1024 + 64,
                                   lambda s, d: 0 if d == 1 else 300,
                                   lambda s, d: (s + d) * 97 + 5],
                         ids=["equal", "ramp", "skip1", "mixed"])
def test_all_to_all_matches_reference(fn, sizer, mode):
    def body(comm):
        ok = True
        for it in range(2):
            spec = _a2a_spec(comm, sizer, seed=it)
            z = fn(comm, spec)
            r = reference_all_to_all(comm, spec)
            ok &= all(np.array_equal(H(a), H(b)) for a, b in zip(z, r))
        return ok
    assert all(run_ranks(3 if sizer(0, 1) == 0 else 4, body, mode))


def test_all_to_all_moe_dispatch_shape():
    # C3 at reduced token count: rows x 4096 per peer, N(0,1) activations
    def body(comm):
        rows = 64
        chunks = [rank_words(comm.rank * 8 + q, rows * 4096, seed=3) for q in range(comm.world_size)]
        spec = AlltoAllSpec(chunks, [rows * 4096] * comm.world_size)
        z = zip_all_to_all_d2(comm, spec)
        return all(np.array_equal(H(z[p]), rank_words(p * 8 + comm.rank, rows * 4096, seed=3))
                   for p in range(comm.world_size))
    assert all(run_ranks(4, body))


@pytest.mark.parametrize("mode", MODES)
def test_protocol_errors(mode):
    def d1(comm):
        chunks = [rank_words(q, 100) for q in range(2)]
        expected = 100 if comm.rank == 1 else 50
        return zip_all_to_all_d1(comm, AlltoAllSpec(chunks, [expected] * 2))
    with pytest.raises(ProtocolError, match="expected 50"):
        run_ranks(2, d1, mode)

    def d2(comm):
        n = 128 if comm.rank == 0 else 256
        chunks = [rank_words(q, n) for q in range(2)]
        return zip_all_to_all_d2(comm, AlltoAllSpec(chunks, [n] * 2))
    with pytest.raises(ProtocolError, match="static section"):
        run_ranks(2, d2, mode)

    def ag(comm):
        return zip_all_gather(comm, rank_words(comm.rank, 10 + comm.rank))
    with pytest.raises(CollectiveError, match="peer rank"):
        run_ranks(2, ag, mode)


@pytest.mark.parametrize("mode", MODES)
def test_zero_element_collectives(mode):
    def body(comm):
        empty = np.empty(0, dtype=np.uint16)
        ag = zip_all_gather(comm, empty)
        a2a = zip_all_to_all_d1(comm, AlltoAllSpec([empty] * comm.world_size,
                                                   [0] * comm.world_size))
        a2b = zip_all_to_all_d2(comm, AlltoAllSpec([empty] * comm.world_size,
                                                   [0] * comm.world_size))
        rs = zip_reduce_scatter(comm, empty)
        return ag.numel() == 0 and all(c.numel() == 0 for c in a2a + a2b) and rs.numel() == 0
    assert all(run_ranks(3, body, mode))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("world", [2, 3, 4])
def test_reduce_scatter_matches_reference_and_oracle(world, mode):
    def body(comm):
        local = rank_words(comm.rank, comm.world_size * 1000)
        return (H(zip_reduce_scatter(comm, local)), H(reference_reduce_scatter(comm, local)),
                zip_reduce_scatter(comm, local, output="fp32").cpu().numpy())
    outs = run_ranks(world, body, mode)
    shard = 1000
    for r, (z, ref, f32) in enumerate(outs):
        assert np.array_equal(z, ref)
        acc = zo.to_f32(rank_words(0, world * shard)[r * shard:(r + 1) * shard]).copy()
        for p in range(1, world):
            acc += zo.to_f32(rank_words(p, world * shard)[r * shard:(r + 1) * shard])
        assert np.array_equal(f32.view(np.uint32), acc.view(np.uint32))
        assert np.array_equal(z, zo.from_f32(acc))


@pytest.mark.parametrize("mode", MODES)
def test_fp32_accumulation_contract(mode):
    # reference tests/test_collectives.py:215-241
    def body(comm):
        value = 1.0 if comm.rank == 0 else 2.0 ** -8
        local = zo.from_f64(np.full(4 * 8, value))
        return H(zip_reduce_scatter(comm, local))
    expected32 = np.float32(1.0)
    for _ in range(3):
        expected32 = np.float32(expected32 + np.float32(2.0 ** -8))
    word = int(zo.from_f32(np.array([expected32], np.float32))[0])
    for out in run_ranks(4, body, mode):
        assert np.all(out == word)


@pytest.mark.parametrize("mode", MODES)
def test_all_reduce_composition(mode):
    def body(comm):
        local = rank_words(comm.rank, 4 * 64)
        got = zip_all_reduce(comm, local)
        expect = reference_all_gather(comm, reference_reduce_scatter(comm, local))
        return np.array_equal(H(got), H(expect))
    assert all(run_ranks(4, body, mode))


@pytest.mark.parametrize("mode", ["msg", "generic"])
def test_wire_bytes_match_size_law(mode):
    # reference tests/test_collectives.py:274-302: design 1 sends the frames
    # plus 16 B of metadata per peer; design 2 the same frames plus 8 B
    n_chunk = 1 << 16
    world = 4

    def body(comm):
        spec = _a2a_spec(comm, lambda s, d: n_chunk, seed=12)
        before = comm.stats.snapshot()
        zip_all_to_all_d1(comm, spec)
        d1 = comm.stats.snapshot().delta(before).bytes_sent
        before = comm.stats.snapshot()
        zip_all_to_all_d2(comm, spec)
        d2 = comm.stats.snapshot().delta(before).bytes_sent
        frames = zo.peer_frames(list(spec.send_chunks), comm.rank)
        return d1, d2, sum(len(f) for f in frames)
    for d1, d2, frames in run_ranks(world, body, mode):
        assert d1 == frames + 16 * (world - 1)
        assert d2 == frames + 8 * (world - 1)
        assert d1 - d2 == 3 * 8                       # reference test_collectives.py:304-317
        assert 2 * n_chunk * (world - 1) / d2 >= 1.30


def test_p2p_traffic_accounting():
    # peer-memory plane: each peer pulls its frame once; ready + done flags
    # are 8 B per peer each
    n_chunk = 1 << 16
    world = 4

    def body(comm):
        spec = _a2a_spec(comm, lambda s, d: n_chunk, seed=12)
        before = comm.stats.snapshot()
        zip_all_to_all_d2(comm, spec)
        sent = comm.stats.snapshot().delta(before).bytes_sent
        frames = zo.peer_frames(list(spec.send_chunks), comm.rank)
        ag_before = comm.stats.snapshot()
        local = rank_words(comm.rank, n_chunk)
        zip_all_gather(comm, local)
        ag = comm.stats.snapshot().delta(ag_before).bytes_sent
        return sent, sum(len(f) for f in frames), ag, len(zo.encode(local, zo.book_for(local)))
    for sent, frames, ag, f in run_ranks(world, body, "p2p"):
        assert sent == frames + 16 * (world - 1)
        assert ag == (f + 16) * (world - 1)


def test_timed_call_agrees():
    def body(comm):
        _, t = timed_call(comm, lambda: zip_all_gather(comm, rank_words(comm.rank, 1 << 20)))
        return t
    ts = run_ranks(3, body)
    assert len(set(ts)) == 1 and ts[0] > 0


@pytest.mark.parametrize("mode", MODES)
def test_fuzz_against_reference(mode):
    # reference tests/test_acceptance.py:155-207 on the GPU path
    for world in (2, 3, 4):
        for seed in (0, 1):
            def body(comm, seed=seed):
                w = comm.world_size
                size_rng = np.random.default_rng([seed, w])
                n_ag = int(size_rng.integers(0, 1 << 16))
                matrix = size_rng.integers(0, 1 << 16, (w, w))
                inject = np.random.default_rng([seed, w, comm.rank])

                def buf(tag, n):
                    d = rank_words(comm.rank * 1000 + tag, n, seed=seed)
                    if n >= 16:
                        idx = inject.integers(0, n, 8)
                        d[idx[:3]] = 0x7FC0
                        d[idx[3:5]] = 0x7F80
                        d[idx[5:]] = 0
                    return d
                local = buf(1, n_ag)
                if not np.array_equal(H(zip_all_gather(comm, local)),
                                      H(reference_all_gather(comm, local))):
                    return False
                spec = AlltoAllSpec([buf(10 + q, int(matrix[comm.rank, q])) for q in range(w)],
                                    [int(matrix[p, comm.rank]) for p in range(w)])
                ref = reference_all_to_all(comm, spec)
                for got in (zip_all_to_all_d1(comm, spec), zip_all_to_all_d2(comm, spec)):
                    if not all(np.array_equal(H(a), H(b)) for a, b in zip(got, ref)):
                        return False
                return True
            assert all(run_ranks(world, body, mode)), (world, seed)


@pytest.mark.parametrize("mode", MODES)
def test_reduce_scatter_nan_inf_semantics(mode):
    # numpy's float32 add on x86 (the reference's arithmetic): a NaN operand
    # propagates quieted, inf + -inf is the default NaN 0xFFC00000; the RNE
    # narrowing keeps sign and top payload bits and forces the quiet bit
    # (bf16.py:53-66).  One NaN per element at most (NaN + NaN payload choice
    # is position-dependent in numpy itself).
    specials = {0: 0x7F81, 1: 0xFFA5, 2: 0x7F80, 3: 0xFF80, 4: 0x0001, 5: 0x8001,
                6: 0x7F7F, 7: 0xFF7F}

    def body(comm):
        W = comm.world_size
        local = rank_words(comm.rank, W * 1024, seed=9)
        for j, w in specials.items():
            if j % W == comm.rank:        # element j of every shard gets a special
                for r in range(W):
                    local[r * 1024 + j] = w
        if comm.rank == 1:
            for r in range(W):
                local[r * 1024 + 20] = 0x7F80   # +inf from rank 1 ...
        if comm.rank == 2:
            for r in range(W):
                local[r * 1024 + 20] = 0xFF80   # ... -inf from rank 2
        return (H(zip_reduce_scatter(comm, local)), H(reference_reduce_scatter(comm, local)),
                zip_reduce_scatter(comm, local, output="fp32").cpu().numpy(), local)
    outs = run_ranks(4, body, mode)
    locals_ = [o[3] for o in outs]
    for r, (z, ref, f32, _) in enumerate(outs):
        acc = zo.to_f32(locals_[0][r * 1024:(r + 1) * 1024]).copy()
        with np.errstate(invalid="ignore", over="ignore"):
            for p in range(1, 4):
                acc += zo.to_f32(locals_[p][r * 1024:(r + 1) * 1024])
        assert np.array_equal(f32.view(np.uint32), acc.view(np.uint32))
        assert np.array_equal(z, zo.from_f32(acc)) and np.array_equal(z, ref)
        assert f32.view(np.uint32)[20] == 0xFFC00000


def test_reduce_scatter_257_ranks_fp32_contract():
    # reference tests/test_acceptance.py:222-248 (criterion 6): 257 ranks,
    # shard of 1 element; generic protocols (more ranks than a native group)
    def body(comm):
        value = 1.0 if comm.rank == 0 else 2.0 ** -8
        local = zo.from_f64(np.full(comm.world_size, value))
        return H(zip_reduce_scatter(comm, local))
    outs = run_ranks(257, body, "generic", timeout=300.0)
    assert all(o.size == 1 and int(o[0]) == 0x4000 for o in outs)
