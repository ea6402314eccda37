"""DistCommunicator path with real processes: 2 ranks sharing cuda:0, gloo
as the byte mover (NCCL refuses two ranks on one GPU; the collective code is
the same, only the mover stages through host memory)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2604_27844_b200.collectives import (AlltoAllSpec, reference_all_gather,
                                                       reference_all_to_all, zip_all_gather,
                                                       zip_all_to_all_d1, zip_all_to_all_d2,
                                                       zip_reduce_scatter,
                                                       reference_reduce_scatter)
        from paper_2604_27844_b200.transport import Communicator
        from tests.conftest import rank_words
        comm = Communicator.from_process_group(device="cuda:0")
        H = lambda t: t.cpu().numpy().view(np.uint16)  # noqa: E731
        ok = True
        local = rank_words(rank, 1_000_003, sigma=0.02)
        ok &= np.array_equal(H(zip_all_gather(comm, local)), H(reference_all_gather(comm, local)))
        sizes = lambda s, d: (s + d) * 4099 + 11  # noqa: E731
        spec = AlltoAllSpec([rank_words(rank * 31 + p, sizes(rank, p)) for p in range(world)],
                            [sizes(p, rank) for p in range(world)])
        ref = reference_all_to_all(comm, spec)
        for fn in (zip_all_to_all_d1, zip_all_to_all_d2):
            got = fn(comm, spec)
            ok &= all(np.array_equal(H(a), H(b)) for a, b in zip(got, ref))
        x = rank_words(rank, world * 5000)
        ok &= np.array_equal(H(zip_reduce_scatter(comm, x)), H(reference_reduce_scatter(comm, x)))
        q.put((rank, bool(ok), None))
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        import traceback
        q.put((rank, False, traceback.format_exc()))


def _p2p_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2604_27844_b200.collectives import reference_all_gather, zip_all_gather
        from paper_2604_27844_b200.transport import Communicator
        from tests.conftest import rank_words
        comm = Communicator.from_process_group(device="cuda:0")
        comm.use_p2p = True           # CUDA IPC symmetric buffers, device-side signals
        H = lambda t: t.cpu().numpy().view(np.uint16)  # noqa: E731
        ok = True
        for it in range(3):
            local = rank_words(rank + 7 * it, 500_009, sigma=0.02)
            ok &= np.array_equal(H(zip_all_gather(comm, local)),
                                 H(reference_all_gather(comm, local)))
        from paper_2604_27844_b200.collectives import (AlltoAllSpec, reference_all_to_all,
                                                       zip_all_to_all_d2)
        sizes = lambda s, d: (s + d) * 40_961 + 3  # noqa: E731
        for it in range(2):
            spec = AlltoAllSpec([rank_words(rank * 31 + q + it, sizes(rank, q))
                                 for q in range(world)], [sizes(p, rank) for p in range(world)])
            got = zip_all_to_all_d2(comm, spec)          # routed to the p2p path
            ref = reference_all_to_all(comm, spec)
            ok &= all(np.array_equal(H(a), H(b)) for a, b in zip(got, ref))
        comm.barrier()
        q.put((rank, bool(ok), None))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, False, traceback.format_exc()))


def _run(target, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, tb in res:
        assert ok, tb


def test_two_processes_ipc_pull_decode():
    _run(_p2p_worker)


def test_two_processes_share_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, tb in res:
        assert ok, tb
