"""DistCommunicator path with real processes.

* 2 ranks sharing cuda:0 with gloo as the byte mover: the generic protocols
  (NCCL refuses two ranks on one GPU).
* 1 rank over NCCL: the native engine bootstrapped from a torch.distributed
  NCCL group (zc_comm_init with rank 0's unique id), every collective at W=1.
"""

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


def _nccl_world1_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", 0))
        from paper_2604_27844_b200.collectives import (AlltoAllSpec, reference_all_gather,
                                                       zip_all_gather, zip_all_to_all_d2,
                                                       zip_reduce_scatter)
        from paper_2604_27844_b200.transport import Communicator
        from tests.conftest import rank_words
        comm = Communicator.from_process_group(device="cuda:0")
        assert comm.native is not None and comm.native.over_nccl
        H = lambda t: t.cpu().numpy().view(np.uint16)  # noqa: E731
        local = rank_words(0, 100_003, sigma=0.02)
        ok = np.array_equal(H(zip_all_gather(comm, local)), local)
        ok &= np.array_equal(H(reference_all_gather(comm, local)), local)
        got = zip_all_to_all_d2(comm, AlltoAllSpec([local], [local.size]))
        ok &= np.array_equal(H(got[0]), local)
        ok &= np.array_equal(H(zip_reduce_scatter(comm, local[:100_000])), local[:100_000])
        q.put((rank, bool(ok), None))
        comm.native.close()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, False, traceback.format_exc()))


def test_native_nccl_world1():
    _run(_nccl_world1_worker, world=1)
