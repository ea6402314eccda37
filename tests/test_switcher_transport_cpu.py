"""Host logic on CPU: the switcher's decision rule / fit (reference
tests/test_switcher.py:25-104, acceptance criterion 7 closed forms) and the
communicator seam over a 2-rank gloo group (reference
tests/test_transport.py:105-113 transpose oracle)."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2604_27844_b200.switcher import (CostModel, Path, crossover, fit_cost_model, predict,
                                            scaled, select)


def test_predict_select_crossover():
    m = CostModel(alpha_rs=1e-5, beta_rs=2e-9, alpha_a2a=6e-5, beta_a2a=1.8e-9, e=0.7)
    d_star = crossover(m)
    assert d_star == pytest.approx((6e-5 - 1e-5) / (2e-9 - 1.8e-9 * 0.7))
    scan = [d for d in range(0, int(d_star * 2), 997) if select(m, d) is Path.ZIPPED]
    assert scan and min(scan) == pytest.approx(d_star, abs=997)
    for d in range(0, int(d_star * 2), 997):
        assert select(m, d) is select(scaled(m, 13.7), d)
    t_rs, t_a2a = predict(m, 0)
    assert select(m, 0) is Path.NATIVE and t_rs < t_a2a


def test_tie_goes_native():
    m = CostModel(1e-5, 1e-9, 1e-5, 1e-9, e=1.0)
    assert select(m, 12345) is Path.NATIVE
    assert crossover(m) is None


def test_exact_two_point_fit():
    sizes = [1 << 16, 1 << 24]
    t_rs = [2e-5 + 3e-10 * d for d in sizes]
    t_zip = [5e-5 + 4e-10 * 0.7 * d for d in sizes]
    m = fit_cost_model(sizes, t_rs, t_zip, e=0.7)
    assert m.alpha_rs == pytest.approx(2e-5) and m.beta_rs == pytest.approx(3e-10)
    assert m.alpha_a2a == pytest.approx(5e-5) and m.beta_a2a == pytest.approx(4e-10)


def test_validation_and_file_round_trip(tmp_path):
    with pytest.raises(ValueError):
        CostModel(-1, 0, 0, 0, 0.5)
    with pytest.raises(ValueError):
        CostModel(0, 0, 0, 0, 1.5)
    with pytest.raises(ValueError):
        fit_cost_model([1, 1], [1, 2], [1, 2], e=0.5)
    m = CostModel(1e-5, 2e-9, 6e-5, 1.8e-9, 0.7)
    m.to_file(tmp_path / "p.txt")
    assert CostModel.from_file(tmp_path / "p.txt") == m


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _seam_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2604_27844_b200.transport import Communicator
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Communicator.from_process_group(device="cpu")
    sizes = [100 * rank + p for p in range(world)]
    got = comm.exchange_sizes(sizes)
    gathered = comm.allgather_ints(7 + rank)
    comm.barrier()
    sent = comm.stats.bytes_sent
    # the byte movers of the N>1 data planes (static / dynamic sections)
    import torch
    from paper_2604_27844_b200.collectives import allgather_scalar
    mine = torch.arange(5, dtype=torch.uint8) + 10 * rank
    allg = torch.empty(5 * world, dtype=torch.uint8)
    comm.all_gather_bytes(mine, allg)
    peer = 1 - rank
    recv = {peer: torch.empty(3 + peer, dtype=torch.uint8)}
    comm.sendrecv_bytes({peer: torch.full((3 + rank,), 50 + rank, dtype=torch.uint8)}, recv)
    scal = allgather_scalar(comm, 0.5 + rank)
    q.put((rank, got, gathered, sent, allg.tolist(), recv[peer].tolist(), scal))
    dist.destroy_process_group()


def test_exchange_sizes_transpose_over_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seam_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((v[0], v[1:]) for v in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        got, gathered, sent, allg, recv, scal = res[r]
        # entry p = what peer p declared for this rank; self passes through
        assert got == [100 * p + r if p != r else 100 * r + r for p in range(world)]
        assert gathered == [7, 8]
        assert sent == 8 * (world - 1)
        assert allg == [i + 10 * q for q in range(world) for i in range(5)]
        peer = 1 - r
        assert recv == [50 + peer] * (3 + peer)
        assert scal == [0.5, 1.5]


def _tcp_worker(rank, world, addr, q):
    from paper_2604_27844_b200 import connect_tcp
    comm = connect_tcp(world, rank, addr, timeout=60)
    got = comm.exchange_sizes([10 * rank + p for p in range(world)])
    q.put((rank, comm.rank, comm.world_size, comm.backend, got))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_connect_tcp_gloo_rendezvous():
    """Reference connect_tcp (transport.py:669-671) over torch.distributed's
    TCP store: two processes meet at host:port and run the size exchange."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    addr = f"127.0.0.1:{_free_port()}"
    procs = [ctx.Process(target=_tcp_worker, args=(r, world, addr, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((v[0], v[1:]) for v in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        rank, ws, backend, got = res[r]
        assert (rank, ws, backend) == (r, world, "gloo")
        assert got == [10 * p + r if p != r else 10 * r + r for p in range(world)]


def test_sim_profile_validation_and_sim_transport_absent():
    """SimProfile keeps the reference's validation (transport.py:96-126); the
    virtual-clock transport itself is out of scope and fails loudly."""
    from paper_2604_27844_b200 import SimProfile, TransportError, run_ranks
    SimProfile(bandwidth=2e9, latency=0.0, mode="serialized-links")
    for bad in (dict(bandwidth=0), dict(latency=-1), dict(mode="x"),
                dict(ready_times={0: -1.0}), dict(link_bandwidth={(0, 1): 0})):
        with pytest.raises(ValueError):
            SimProfile(**bad)
    with pytest.raises(TransportError):
        run_ranks(2, lambda c: None, "sim", SimProfile())
    with pytest.raises(ValueError):
        run_ranks(2, lambda c: None, "carrier-pigeon")
    with pytest.raises(TransportError):
        from paper_2604_27844_b200 import connect_tcp
        connect_tcp(2, 0, None)
