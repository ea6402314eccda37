"""Benchmark of the ZipCCL hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

Workload (BASELINE.json configs[1]): Llama3-8B FSDP parameter all-gather of
one transformer layer (218,112,000 BF16 elements = 436 MB; wq, wk, wv, wo,
w1, w2, w3 ~ N(0, 0.02^2), two RMSNorm vectors of 1.0).  Each of N ranks
holds a shard of 218,112,000 / N elements; one step = zip_all_gather of the
layer: codebook_for (K1 stats), encode (K2), exchange, decode of every peer
frame (K3).  At N=1 the exchange is empty and the step is the per-rank
codec work on a self-loopback frame (codebook + encode + decode of the whole
layer), i.e. the codec path the collective runs.

value = uncompressed BF16 bytes delivered into the gathered outputs of all
ranks per second (N x layer bytes / max-over-ranks step time), inputs
resident in HBM and larger than L2 (no flush needed).  e2e = the same metric
through the public API with the shard copied host->device from pinned memory
every step and the frame size read back.

--impl reference times the reference algorithm's CPU implementation (the
numpy oracle port in oracle/, run in one process per host core on disjoint
shards of the same layer).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Compressed AllGather/All-to-All effective GB/s @1-8 B200; codec GB/s; ratio"
LAYER = [("wq", 4096 * 4096), ("wk", 1024 * 4096), ("wv", 1024 * 4096), ("wo", 4096 * 4096),
         ("w1", 14336 * 4096), ("w2", 4096 * 14336), ("w3", 14336 * 4096),
         ("attn_norm", 4096), ("ffn_norm", 4096)]
LAYER_ELEMS = sum(n for _, n in LAYER)          # 218,112,000
FALLBACK_HBM_GBS = 6650.0


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


def layer_shard(rank: int, world: int, device, seed: int = 0):
    """Synthetic random-init layer, flattened; this rank's contiguous shard."""
    import torch
    n = LAYER_ELEMS // world
    lo = rank * n
    g = torch.Generator(device=device).manual_seed(seed)
    out = torch.empty(n, dtype=torch.bfloat16, device=device)
    pos = 0
    for name, size in LAYER:
        a, b = max(lo, pos), min(lo + n, pos + size)
        if a < b:
            if name.endswith("norm"):
                out[a - lo:b - lo] = 1.0
            else:
                t = torch.randn(b - a, generator=g, device=device) * 0.02
                out[a - lo:b - lo] = t.to(torch.bfloat16)
        pos += size
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.result = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if sm:
            busy = [s for s in sm if s > 0.5 * max(mx)] or sm
            self.result = {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx),
                           "reasons": sorted(reasons), "samples": len(sm)}


def _agreed_steps(seconds, step, world, dev):
    """Number of untimed steps filling ~`seconds`, identical on every rank."""
    import torch
    t = time.perf_counter()
    step()
    torch.cuda.synchronize()
    per = max(time.perf_counter() - t, 1e-4)
    k = torch.tensor([max(1, int(seconds / per))], device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(k, op=dist.ReduceOp.MAX)
    return int(k.item())


def setup_comm(args, dev):
    """Communicator for N>1: the native engine over the NCCL group (peer-
    memory plane when every peer's buffer maps, else the message plane),
    checked against a bare NCCL all-gather on a small message before
    anything is timed.  Any failure on any rank falls back, identically on
    all ranks: p2p -> message plane -> generic protocols over NCCL."""
    import torch
    import torch.distributed as dist
    from paper_2604_27844_b200 import collectives as coll
    comm = coll.Communicator.from_process_group()
    g = torch.Generator(device=dev).manual_seed(1234 + comm.rank)
    x = (torch.randn((1 << 20) + 77, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    ref = torch.empty(comm.world_size * x.numel(), dtype=torch.bfloat16, device=dev)
    dist.all_gather_into_tensor(ref, x)
    want = "p2p" if args.transport == "p2p" else "msg"
    tried = []
    for plane in ([want, "msg", "generic"] if want == "p2p" else [want, "generic"]):
        ok = 1
        try:
            if plane == "generic":
                comm.use_native = False
            else:
                comm.use_native = True
                native = comm.native
                if native is None:                    # gloo group: no native engine
                    ok = 0
                elif plane == "p2p" and not native.p2p_available:
                    ok = 0
                else:
                    native.plane = plane
            if ok:
                got = coll.zip_all_gather(comm, x)
                ok = int(torch.equal(got.view(torch.int16), ref.view(torch.int16)))
        except Exception as exc:  # noqa: BLE001 - any failure selects the fallback
            print(f"[rank {comm.rank}] {plane} preflight failed: {exc!r}", file=sys.stderr)
            ok = 0
        t = torch.tensor([ok], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        tried.append(plane)
        if t.item():
            comm.bench_plane = plane
            comm.bench_tried = tried
            if plane != "generic":
                comm.native.sync_errors = False       # checked after the timed region
            return comm
    raise RuntimeError("no data plane passed the preflight")


def nccl_info():
    import torch
    try:
        v = torch.cuda.nccl.version()
        ver = ".".join(str(p) for p in v) if isinstance(v, tuple) else str(v)
    except Exception:  # noqa: BLE001
        ver = None
    env = {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}
    return {"version": ver, "env": env}


def self_launch(args) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks with
    torch.distributed.run on this node (127.0.0.1) and relay rank 0's line."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}",
              file=sys.stderr)
        return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_baseline_sample(seconds: float = 10.0):
    """Oracle (numpy port of the reference) on one core: codebook + encode +
    decode of a C1-sized sample of the layer's weights, repeated ~10 s."""
    from oracle import zc_oracle as zo
    import numpy as np
    n = 1 << 24
    w = zo.from_f64(np.random.default_rng(0).standard_normal(n) * 0.02)
    t0 = time.perf_counter()
    reps = 0
    while True:
        book = zo.book_for(w)
        fr = zo.encode(w, book)
        back = zo.decode(fr)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    assert np.array_equal(back, w)
    return {"value": 2 * n * reps / el / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{reps} x (codebook_for + encode + decode) of 2^24 N(0,0.02^2) BF16 "
                      f"elements, numpy oracle port of the reference, {el:.1f} s",
            "c1_simulated_w2_allgather": c1_simulated_allgather()}


def c1_simulated_allgather(world: int = 2, n: int = 1 << 23, trials: int = 3):
    """BASELINE configs[0]'s second half: the reference's run_ranks(2,
    zip_all_gather) timed like timed_call (transport.py:635-666,
    collectives.py:366-376) -- thread ranks, each encodes its 2^23-element
    shard, the frames are exchanged, every rank decodes its peers' frames and
    concatenates in rank order; max over ranks, best of `trials`.  Run on the
    numpy oracle port (same numpy primitives as the reference)."""
    import threading
    import numpy as np
    from oracle import zc_oracle as zo
    shards = [zo.rank_gaussian(r, n, s=0.02) for r in range(world)]
    best = None
    for _ in range(trials):
        frames, outs, spans = [None] * world, [None] * world, [None] * world
        bar = threading.Barrier(world)

        def rank(r):
            bar.wait()
            t0 = time.perf_counter()
            frames[r] = zo.encode(shards[r], zo.book_for(shards[r]))
            bar.wait()                                   # the size + frame exchange
            outs[r] = np.concatenate([shards[p] if p == r else zo.decode(frames[p])
                                      for p in range(world)])
            spans[r] = time.perf_counter() - t0
        th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        want = np.concatenate(shards)
        assert all(np.array_equal(o, want) for o in outs)
        t = max(spans)
        best = t if best is None else min(best, t)
    return {"ms": 1e3 * best, "GBps": 2 * n * world / best / 1e9, "world": world,
            "shard_elems": n, "threads": world,
            "what": "run_ranks(2, zip_all_gather) on the oracle port: gathered bytes / max-over-ranks time"}


def _oracle_worker(args):
    n, seed = args
    import numpy as np
    from oracle import zc_oracle as zo
    w = zo.from_f64(np.random.default_rng(seed).standard_normal(n) * 0.02)
    t0 = time.perf_counter()
    back = zo.decode(zo.encode(w, zo.book_for(w)))
    ok = bool(np.array_equal(back, w))
    return time.perf_counter() - t0, ok


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    per = 1 << 22
    with mp.get_context("spawn").Pool(cores) as pool:
        jobs = [(per, 1000 + i) for i in range(cores)]
        for _ in range(args.warmup):
            pool.map(_oracle_worker, jobs)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            res = pool.map(_oracle_worker, jobs)
            times.append(time.perf_counter() - t0)
            assert all(ok for _, ok in res)
    ms = 1e3 * sum(times) / len(times)
    value = 2 * per * cores / (ms / 1e3) / 1e9
    sample = (f"{cores} processes x codebook_for+encode+decode of 2^22 BF16 elements "
              f"(N(0,0.02^2), the layer's weight distribution) per step")
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "llama3-8b layer zip_all_gather codec path (CPU sample)",
                       "layer_elems": LAYER_ELEMS, "sample_elems_per_step": per * cores},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.share_gpu:
        local = 0          # test mode: all ranks on one GPU, gloo moves the bytes
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.backend)
    from paper_2604_27844_b200 import engine
    if world > 1:
        from paper_2604_27844_b200 import collectives as coll

    shard = layer_shard(rank, world, dev)
    words = engine.words_view(shard)
    n = words.numel()
    stream = torch.cuda.current_stream()

    whole_step = None
    if world == 1:
        frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
        out = torch.empty(n, dtype=torch.int16, device=dev)
        flen = torch.empty(1, dtype=torch.int64, device=dev)

        ev = {"e0": [], "e1": [], "d0": [], "d1": []}
        err_buf = torch.empty(1, dtype=torch.int32, device=dev)

        def run_enc():
            # codebook_for (K1 statistic + on-device derivation) + compress (K2)
            engine.encode_measured(words, [(0, n)], 9, frames, [0], flen)

        def run_dec():
            engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err_buf)

        eager_enc, eager_dec = run_enc, run_dec
        if not args.no_graph:
            # captured once as CUDA graphs and replayed: no host launch overhead
            # or event gaps between the kernels, identical kernels.  The per-kernel durations come from
            # an eager pass of the same steps right after the timed region.
            run_enc()
            run_dec()
            torch.cuda.synchronize()
            g_enc, g_dec = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_enc):
                run_enc()
            with torch.cuda.graph(g_dec):
                run_dec()
            # the timed steps replay one graph per step (encode then decode);
            # the two legs are timed afterwards from per-leg replays
            g_step = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_step):
                run_enc()
                run_dec()
            whole_step = g_step.replay
            run_enc, run_dec = g_enc.replay, g_dec.replay   # noqa: F811

        def step(rec=False):
            if rec:
                for k in ev:
                    ev[k].append(torch.cuda.Event(enable_timing=True))
                ev["e0"][-1].record(stream)
            run_enc()
            if rec:
                ev["e1"][-1].record(stream)
                ev["d0"][-1].record(stream)
            run_dec()
            if rec:
                ev["d1"][-1].record(stream)
            return err_buf
        # guess (1/512 sample), encoder pass 1 with the fused statistic and
        # certificate, run fix-up, then exact-statistic / re-encode pass 1 /
        # re-encode fix-up launches that return at once when the certificate
        # decided and the guess held, decoder init (error words + chunk
        # counter), decode
        launches_per_step = 8
    else:
        comm = setup_comm(args, dev)

        def step(rec=False):
            return coll.zip_all_gather(comm, shard)
        # codebook+encode leg (6, as at N=1) + decoder init + decode, plus
        # p2p: error-word init, done-wait, publish, finish (done flags);
        # msg: error-word init, size packing, error mapping; generic: as N=1
        launches_per_step = {"p2p": 12, "msg": 11, "generic": 8}[comm.bench_plane]

    # correctness gate before timing: bit-exact round trip
    err = step()
    torch.cuda.synchronize()
    if world == 1:
        assert int(err.item()) == engine.ERR_OK and torch.equal(out, words), "round trip failed"
        frame_bytes = int(flen.item())
    else:
        frame_bytes = None

    # warm-up and settle steps run what the timed region runs: the one-graph
    # step's first replay uploads the graph (~2 ms on a fresh box, 100 us per
    # step if it fell inside the 20 timed steps)
    timed_step = whole_step if whole_step is not None else step
    for _ in range(args.warmup):
        timed_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # keep the GPU under the same load while nvidia-smi starts sampling,
        # so the clocks reflect the timed steps (the timed region itself is ms)
        settle = _agreed_steps(args.clock_settle, timed_step, world, dev)
        for _ in range(settle):
            timed_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        profiling = world == 1 and args.no_graph
        if profiling:
            engine.profile_enable(True)    # events around each encoder / decoder launch
        t0.record(stream)
        if whole_step is not None:
            for _ in range(args.steps):
                whole_step()
        else:
            for _ in range(args.steps):
                step(rec=(world == 1))
        t1.record(stream)
        torch.cuda.synchronize()
        if whole_step is not None:
            # leg durations: per-leg graph replays with events between them
            for _ in range(args.steps):
                step(rec=True)
            torch.cuda.synchronize()
        if world == 1 and not profiling:
            # per-kernel durations: the same steps launched eagerly with the
            # library's event hooks (kernel durations do not depend on how the
            # launches were submitted)
            engine.profile_enable(True)
            for _ in range(args.steps):
                eager_enc()
                eager_dec()
            torch.cuda.synchronize()
            profiling = True
        if profiling:
            engine.profile_enable(False)
            # the encode hook brackets pass 1 and the run fix-up (two kernels)
            kern_ms = {"encode_tiles_kernel+encode_runfix_kernel":
                       engine.profile_read(engine.PROF_ENCODE),
                       "decode_ring_kernel": engine.profile_read(engine.PROF_DECODE)}
        for _ in range(max(1, settle // 3)):
            step()
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    total_bytes = world * 2 * LAYER_ELEMS          # gathered output bytes, all ranks
    value = total_bytes / (ms / 1e3) / 1e9
    raw = None
    if world > 1:
        # deferred decode errors of the timed steps, then one bit-exact check
        if comm.bench_plane != "generic":
            comm.native.check()
        got = coll.zip_all_gather(comm, shard)
        expect = torch.empty(world * n, dtype=torch.bfloat16, device=dev)
        dist.all_gather_into_tensor(expect, shard)
        assert torch.equal(got.view(torch.int16), expect.view(torch.int16)), "all-gather differs"
        if comm.bench_plane != "generic":
            comm.native.check()

        def timed(fn):
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            tt = torch.tensor([a.elapsed_time(b) / args.steps], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt.item())

        # the plain uncompressed collective on the same shards, same run: a
        # bare NCCL all-gather (no count agreement, no copies)
        raw_out = torch.empty(world * n, dtype=torch.bfloat16, device=dev)
        raw_ms = timed(lambda: dist.all_gather_into_tensor(raw_out, shard))
        per_rank = 2 * n

        def bw(t_ms):
            algbw = world * per_rank / (t_ms / 1e3) / 1e9
            return {"algbw_GBps": algbw, "busbw_GBps": algbw * (world - 1) / world,
                    "busbw_frac_of_900": algbw * (world - 1) / world / 900.0}
        planes = {comm.bench_plane: ms}
        if comm.bench_plane == "p2p":          # the other native plane, for the record
            comm.native.plane = "msg"
            try:
                planes["msg"] = timed(lambda: coll.zip_all_gather(comm, shard))
            finally:
                comm.native.plane = "p2p"
            comm.native.check()
        raw = {"value": total_bytes / (raw_ms / 1e3) / 1e9, "ms_per_step": raw_ms,
               "what": f"torch.distributed.all_gather_into_tensor ({args.backend}) of the same "
                       "shards",
               **bw(raw_ms), "zip": {"ms_per_step": ms, **bw(ms)},
               "zip_planes_ms": planes, "nccl": nccl_info(),
               "plane": comm.bench_plane, "planes_tried": comm.bench_tried,
               "speedup_zip_over_raw": raw_ms / ms}

    # ---- roofline of the dominant kernel -------------------------------------
    # Both codec kernels move the same algorithmic bytes per launch: the
    # encoder reads the 2n-byte shard and writes the F-byte frame (its fused
    # statistic reads nothing extra), the decoder reads F and writes 2n.
    roof = None
    if world == 1:
        dec = [a.elapsed_time(b) for a, b in zip(ev["d0"], ev["d1"])]
        enc = [a.elapsed_time(b) for a, b in zip(ev["e0"], ev["e1"])]
        dec_leg, enc_leg = sum(dec) / len(dec), sum(enc) / len(enc)
        peak, peak_kind = measured_peak_hbm()
        alg = 2 * n + frame_bytes
        traffic_all = {}
        tp = ROOT / "profiles" / "ncu_traffic.json"
        if tp.exists():
            try:
                traffic_all = json.loads(tp.read_text())
            except Exception:
                traffic_all = {}
        per = {k: sum(v) / len(v) for k, v in kern_ms.items() if v}
        kernel = max(per, key=per.get)              # the larger share of the step
        k_ms = per[kernel]
        timing = ("CUDA events recorded by the library on the launching stream around every "
                  "encoder / decoder launch of " +
                  ("the timed (eager) steps" if args.no_graph else
                   f"{args.steps} eager steps run right after the graph-replayed timed region"))
        def traffic_of(name):
            parts = [traffic_all.get(f"{k}_per_launch_bytes") for k in name.split("+")]
            return sum(parts) if parts and all(v is not None for v in parts) else None

        ach = alg / (k_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": traffic_of(kernel),
                "kernel": kernel, "peak_kind": peak_kind, "alg_bytes_per_launch": alg,
                "kernel_ms": k_ms, "timing": timing,
                "kernels": {k: {"ms": v, "achieved": alg / (v / 1e3) / 1e9,
                                "frac": alg / (v / 1e3) / 1e9 / peak,
                                "traffic": traffic_of(k)}
                            for k, v in per.items()},
                "encode_leg_ms": enc_leg, "decode_leg_ms": dec_leg,
                "encode_leg_note": "codebook_for+compress: guess kernel (1/512 sample), encoder "
                                   "pass 1 with the statistic fused + run fix-up, three "
                                   "conditional launches"}
    else:
        # this rank's encoder (HBM-bound: its 2n-byte shard in, F-byte frame
        # out) over eager zip_all_gather steps with the library's event hooks;
        # the decoder reads W-1 peer frames (over NVLink on the peer-memory
        # data plane), so it is reported beside, not as the HBM roofline
        frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
        _, _, fl = engine.encode_measured(words, [(0, n)], 9, frames, [0])
        F = int(fl.item())
        frame_bytes = F
        del frames
        engine.profile_enable(True)
        for _ in range(args.steps):
            coll.zip_all_gather(comm, shard)
        torch.cuda.synchronize()
        engine.profile_enable(False)
        enc_k = engine.profile_read(engine.PROF_ENCODE)
        dec_k = engine.profile_read(engine.PROF_DECODE)
        peak, peak_kind = measured_peak_hbm()
        alg = 2 * n + F
        k_ms = sum(enc_k) / len(enc_k)
        ach = alg / (k_ms / 1e3) / 1e9
        dec_ms = sum(dec_k) / len(dec_k) if dec_k else None
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": None,
                "kernel": "encode_tiles_kernel+encode_runfix_kernel", "peak_kind": peak_kind,
                "alg_bytes_per_launch": alg, "kernel_ms": k_ms,
                "timing": f"rank 0, CUDA events around the encoder launches of {args.steps} "
                          "eager zip_all_gather steps after the timed region",
                "decode_ring_kernel": {
                    "ms": dec_ms, "bytes_per_launch": (world - 1) * (F + 2 * n),
                    "GBps": ((world - 1) * (F + 2 * n) / (dec_ms / 1e3) / 1e9) if dec_ms else None,
                    "note": "batched decode of the W-1 peer frames"}}

    # ---- end to end through the public API (host buffers) --------------------
    e2e = None
    if world == 1:
        import paper_2604_27844_b200 as zc
        host = shard.cpu().pin_memory()
        e_steps = max(2, min(args.steps, 5))

        def api_step():
            x = host.to(dev, non_blocking=True)
            chunk = zc.compress(x, zc.codebook_for(x))   # frame length read back (D2H)
            y = zc.decompress(chunk)                       # validated: err word read back
            return chunk, y
        # the caching allocator reaches its steady state (no cudaMalloc, which
        # synchronises) after two calls; each step drops the previous step's frame and output before it
        # allocates, so the allocator hands back the same blocks every step
        res = None
        for _ in range(max(3, args.warmup)):
            res = None
            res = api_step()
        torch.cuda.synchronize()
        a0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
        ts = time.perf_counter()
        for _ in range(e_steps):
            res = None
            res = api_step()
        del res
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - ts) * 1e3 / e_steps
        e_allocs = torch.cuda.memory_stats().get("num_device_alloc", 0) - a0
        if os.environ.get("ZC_E2E_DEBUG"):
            for _ in range(3):
                t = [time.perf_counter()]
                x = host.to(dev, non_blocking=True)
                torch.cuda.synchronize(); t.append(time.perf_counter())
                book = zc.codebook_for(x)
                torch.cuda.synchronize(); t.append(time.perf_counter())
                chunk = zc.compress(x, book)
                torch.cuda.synchronize(); t.append(time.perf_counter())
                y = zc.decompress(chunk)
                torch.cuda.synchronize(); t.append(time.perf_counter())
                print("e2e stages (h2d, book, compress, decompress) ms:",
                      [round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])], file=sys.stderr)
        e2e = {"value": 2 * LAYER_ELEMS / (e_ms / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": 8 + 8 + 8 + 4,
               "ms_per_step": e_ms, "device_allocs_in_timed_loop": e_allocs,
               "note": "H2D of the shard from pinned memory + codebook_for + compress + "
                       "decompress through the public API; reads back sigma-derived book, "
                       "frame length/zero_count and the decoder's error word"}

    elif world > 1:
        # every rank: H2D of its shard from pinned memory + zip_all_gather
        # through the public API (which reads back the decoders' error words
        # and, on the NCCL data plane, the frame lengths); max over ranks
        host = shard.cpu().pin_memory()
        e_steps = max(2, min(args.steps, 5))

        if comm.bench_plane != "generic":
            comm.native.sync_errors = True     # the public API's synchronous error check

        def api_step():
            return coll.zip_all_gather(comm, host.to(dev, non_blocking=True))
        res = None
        for _ in range(max(3, args.warmup)):
            res = None
            res = api_step()
        torch.cuda.synchronize()
        dist.barrier()
        ts = time.perf_counter()
        for _ in range(e_steps):
            res = None
            res = api_step()
        torch.cuda.synchronize()
        el = torch.tensor([(time.perf_counter() - ts) * 1e3 / e_steps], device=dev)
        del res
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e_ms = float(el.item())
        d2h = 4 * world + (8 * world if comm.bench_plane == "msg" else 0)
        e2e = {"value": total_bytes / (e_ms / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
               "note": "per rank: H2D of the shard from pinned memory + zip_all_gather through "
                       "the public API; wall clock, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(args.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u16", "data": "synthetic (random-init N(0,0.02^2) weights, norms 1.0)",
                "config": {"workload": "llama3-8b FSDP layer zip_all_gather"
                                       + (" (W=1: codebook+encode+decode self frame)"
                                          if world == 1 else ""),
                           "layer_elems": LAYER_ELEMS, "shard_elems": n, "world": world,
                           "parallelism": f"dp{world}", "group_size": 512,
                           "frame_bytes": frame_bytes,
                           "ratio": (2 * n / frame_bytes) if frame_bytes else None,
                           "l2": "inputs (436 MB) larger than L2 (126 MB); no flush",
                           "uncompressed_collective": raw},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": (launches_per_step * args.steps) if launches_per_step else None,
                "clocks": clk.result}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _gpu_mix(kind: str, n: int, dev):
    """C4 gradient mixes (SURVEY Appendix C.4 recipe) generated on the GPU."""
    import torch
    g = torch.Generator(device=dev).manual_seed(1)
    sign = torch.where(torch.rand(n, device=dev, generator=g) < 0.5, -1.0, 1.0)
    if kind == "lognormal2":
        v = torch.exp(torch.randn(n, device=dev, generator=g) * 2.0 - 8.0) * sign
        return v.to(torch.bfloat16)
    gauss = torch.randn(n, device=dev, generator=g) * 1e-3
    ln = torch.exp(torch.randn(n, device=dev, generator=g) - 8.0) * sign
    v = torch.where(torch.rand(n, device=dev, generator=g) < 0.5, gauss, ln)
    if kind == "mix_x1000":
        idx = torch.randint(0, n, (n // 1000,), device=dev, generator=g)
        v[idx] *= 1000.0
    elif kind == "mix_n10":
        idx = torch.randint(0, n, (n // 10000,), device=dev, generator=g)
        v[idx] = torch.randn(idx.numel(), device=dev, generator=g) * 10.0
    return v.to(torch.bfloat16)


def run_grad_mix(args):
    """BASELINE configs[3]: codec throughput and ratio on gradient mixes, 1 GPU."""
    import torch
    from paper_2604_27844_b200 import engine
    dev = torch.device("cuda", 0)
    n = 1 << 28
    for kind in ("mix", "mix_x1000", "mix_n10", "lognormal2"):
        w = engine.words_view(_gpu_mix(kind, n, dev))
        frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
        out = torch.empty_like(w)
        flen = torch.empty(1, dtype=torch.int64, device=dev)
        err = torch.empty(1, dtype=torch.int32, device=dev)
        enc = lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0], flen)  # noqa: E731
        dec = lambda: engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err, groups512=True)  # noqa: E731
        enc()
        dec()
        torch.cuda.synchronize()
        assert int(err.item()) == engine.ERR_OK and torch.equal(out, w)
        F = int(flen.item())
        zc = int.from_bytes(bytes(frames[16:24].cpu().numpy()), "little")   # header zero_count
        ge, gd = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(ge):
            enc()
        with torch.cuda.graph(gd):
            dec()
        times = {}
        for name, g in (("encode", ge), ("decode", gd)):
            for _ in range(args.warmup):
                g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(args.steps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            times[name] = a.elapsed_time(b) / args.steps
        print(json.dumps({
            "metric": METRIC, "workload": f"c4 gradient {kind}", "n": n,
            "ratio": 2 * n / F, "escape_rate": zc / n,
            "codebook_encode_GBps": 2 * n / (times["encode"] / 1e3) / 1e9,
            "decode_GBps": 2 * n / (times["decode"] / 1e3) / 1e9,
            "encode_ms": times["encode"], "decode_ms": times["decode"],
            "note": "GB/s of uncompressed BF16; ratio < 1 means the frame expands "
                    "(the switcher then picks the raw collective)"}), flush=True)


C1_FRAME_SHA256 = "9d65816bae340834eadc3a854b9173fbc68db6ec744dafa3b9d8e294c3d9fdae"


def run_c1(args):
    """BASELINE configs[0] on the GPU beside its CPU reference path: the
    codec round trip of the 2^24-element N(0, 0.02^2) tensor (frame digest
    checked against SURVEY Appendix B) and the simulated W=2 zip_all_gather
    (run_ranks(2, ...) with timed_call, here two thread ranks of the native
    engine sharing the GPU; shards rng([0, rank]) of 2^23 elements)."""
    import hashlib
    import numpy as np
    import torch
    from oracle import zc_oracle as zo
    from paper_2604_27844_b200 import collectives as coll, engine
    from paper_2604_27844_b200.transport import run_ranks
    dev = torch.device("cuda", 0)
    n = 1 << 24
    host = zo.from_f64(np.random.default_rng(0).standard_normal(n) * 0.02)
    w = torch.from_numpy(host.view(np.int16)).to(dev)
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
    out = torch.empty_like(w)
    flen = torch.empty(1, dtype=torch.int64, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    enc = lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0], flen)  # noqa: E731
    dec = lambda: engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err)  # noqa: E731
    enc()
    dec()
    torch.cuda.synchronize()
    F = int(flen.item())
    digest = hashlib.sha256(frames[:F].cpu().numpy().tobytes()).hexdigest()
    assert int(err.item()) == engine.ERR_OK and torch.equal(out, w)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        enc()
        dec()
    for _ in range(args.warmup):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(args.steps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    rt_ms = a.elapsed_time(b) / args.steps
    shard = 1 << 23

    def body(comm):
        local = torch.from_numpy(zo.rank_gaussian(comm.rank, shard, s=0.02).view(np.int16)).to(dev)
        ref = coll.reference_all_gather(comm, local)
        for _ in range(args.warmup):
            coll.zip_all_gather(comm, local)
        best = None
        for _ in range(args.steps):
            got, t = coll.timed_call(comm, lambda: coll.zip_all_gather(comm, local))
            best = t if best is None else min(best, t)
        assert torch.equal(got, ref)
        return best
    ag_s = max(run_ranks(2, body))
    cpu = c1_simulated_allgather() if not args.no_cpu_baseline else None
    print(json.dumps({
        "metric": METRIC, "workload": "c1 codec round trip 2^24 + simulated W=2 all-gather",
        "n": n, "frame_bytes": F, "ratio": 2 * n / F, "frame_sha256_matches_reference":
        digest == C1_FRAME_SHA256, "roundtrip_ms": rt_ms,
        "roundtrip_GBps": 2 * n / (rt_ms / 1e3) / 1e9,
        "simulated_w2_allgather_ms": ag_s * 1e3,
        "simulated_w2_note": "two thread ranks sharing one GPU (native engine, host rendezvous "
                             "between them): a latency figure, not an NVLink number",
        "cpu_reference_w2_allgather": cpu}), flush=True)


def _init_dist(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(args.backend)
    return world, rank, local, dev


def run_moe_a2a(args):
    """BASELINE configs[2]: Qwen3-MoE-style expert-parallel dispatch + combine,
    hidden 4096, 8 experts per GPU, top-k 8, T tokens per rank, uniform or
    Zipf-skewed routing; compressed (native engine) vs torch's NCCL
    all_to_all_single of the same splits, max over ranks."""
    import torch
    import torch.distributed as dist
    world, rank, local, dev = _init_dist(args)
    from paper_2604_27844_b200 import collectives as coll
    comm = setup_comm(args, dev)
    hidden, topk, T = 4096, 8, args.tokens
    experts = 8 * world
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    # routing: token -> top-k distinct experts; expert e lives on rank e // 8
    if args.routing == "zipf":
        w = 1.0 / torch.arange(1, experts + 1, device=dev, dtype=torch.float64) ** 1.1
    else:
        w = torch.ones(experts, device=dev, dtype=torch.float64)
    choice = torch.multinomial(w.expand(T, experts), topk, replacement=False, generator=g)
    dest = (choice // 8).flatten()
    counts_t = torch.bincount(dest, minlength=world)
    send_rows = counts_t.tolist()
    rows_all = torch.empty(world * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(rows_all, counts_t)
    recv_rows = rows_all.view(world, world)[:, rank].tolist()
    x = torch.randn(T * topk * hidden, device=dev, generator=g).to(torch.bfloat16)
    send_counts = [r * hidden for r in send_rows]
    recv_counts = [r * hidden for r in recv_rows]
    if comm.bench_plane != "generic":
        per_peer = max(send_counts + recv_counts)
        comm.native.reserve(int(1.05 * world * (2.4 * per_peer + 4096)))

    def views(buf, counts):
        offs = [0]
        for c in counts:
            offs.append(offs[-1] + c)
        return [buf[offs[q]:offs[q + 1]] for q in range(world)]

    spec = coll.AlltoAllSpec(views(x, send_counts), recv_counts)
    back_spec_counts = send_counts

    def zip_step():
        got = coll.zip_all_to_all_d2(comm, spec)                            # dispatch
        return coll.zip_all_to_all_d2(comm, coll.AlltoAllSpec(got, back_spec_counts))  # combine

    recv_buf = torch.empty(sum(recv_counts), dtype=torch.bfloat16, device=dev)
    back_buf = torch.empty_like(x)

    def raw_step():
        dist.all_to_all_single(recv_buf, x, recv_counts, send_counts)
        dist.all_to_all_single(back_buf, recv_buf, send_counts, recv_counts)

    res = zip_step()
    if comm.bench_plane != "generic":
        comm.native.check()
    ok = all(torch.equal(a.view(torch.int16), b.view(torch.int16))
             for a, b in zip(res, spec.send_chunks))
    assert ok, "combine(dispatch(x)) != x"
    ms = {}
    for name, fn in (("zip", zip_step), ("raw", raw_step)):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms[name] = float(t.item())
    if comm.bench_plane != "generic":
        comm.native.check()
    send_bytes = 2 * 2 * x.numel()                    # dispatch + combine, this rank
    tot = torch.tensor([send_bytes], device=dev, dtype=torch.float64)
    dist.all_reduce(tot)
    if rank == 0:
        algbw = float(tot.item()) / world / (ms["zip"] / 1e3) / 1e9
        print(json.dumps({
            "metric": METRIC, "workload": f"c3 qwen3-moe dispatch+combine all-to-all "
                                          f"({args.routing} routing)",
            "n_gpus": world, "tokens_per_rank": T, "topk": topk, "hidden": hidden,
            "experts": experts, "value": float(tot.item()) / (ms["zip"] / 1e3) / 1e9,
            "unit": "GB/s", "ms_per_step": ms["zip"], "raw_ms_per_step": ms["raw"],
            "raw_value": float(tot.item()) / (ms["raw"] / 1e3) / 1e9,
            "algbw_GBps": algbw, "busbw_GBps": algbw * (world - 1) / world,
            "speedup_zip_over_raw": ms["raw"] / ms["zip"], "plane": comm.bench_plane,
            "raw": f"torch.distributed.all_to_all_single ({args.backend}), same splits",
            "nccl": nccl_info(), "backend": args.backend}), flush=True)
    dist.destroy_process_group()


def run_imbalance(args):
    """SURVEY §8(f)4 / PAPER.md:301-311, :433: design 2 absorbing start skew.
    Every step, rank 1 starts its all-to-all `--skew-us` late (a device-side
    sleep on its stream, like a slow expert computation); the metric is the
    slowest rank's time from the common start to the end of the collective,
    for design 1 and design 2 on the message plane and for the peer-memory
    plane, against the same skew on the plain NCCL all-to-all.  Needs >= 2
    GPUs (thread ranks sharing one GPU would serialise the skew)."""
    import torch
    import torch.distributed as dist
    world, rank, local, dev = _init_dist(args)
    from paper_2604_27844_b200 import collectives as coll
    comm = setup_comm(args, dev)
    hidden, rows = 4096, args.tokens * 8 // world
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    x = torch.randn(world * rows * hidden, device=dev, generator=g).to(torch.bfloat16)
    counts = [rows * hidden] * world
    chunks = [x[q * rows * hidden:(q + 1) * rows * hidden] for q in range(world)]
    spec = coll.AlltoAllSpec(chunks, counts)
    out = torch.empty_like(x)
    cycles = int(args.skew_us * 1e-6 * 1.9e9)
    variants = {"raw_nccl": lambda: dist.all_to_all_single(out, x)}
    if comm.bench_plane != "generic":
        comm.native.reserve(int(1.05 * world * (2.4 * rows * hidden + 4096)))

        def with_plane(plane, fn):
            def run():
                comm.native.plane = plane
                return fn(comm, spec)
            return run
        variants["zip_d1_msg"] = with_plane("msg", coll.zip_all_to_all_d1)
        variants["zip_d2_msg"] = with_plane("msg", coll.zip_all_to_all_d2)
        if comm.bench_plane == "p2p":
            variants["zip_p2p"] = with_plane("p2p", coll.zip_all_to_all_d2)
    else:                                  # the Python protocols over the group's byte movers
        variants["zip_d1_generic"] = lambda: coll.zip_all_to_all_d1(comm, spec)
        variants["zip_d2_generic"] = lambda: coll.zip_all_to_all_d2(comm, spec)
    res = {}
    for name, fn in variants.items():
        for skew in (0, cycles):
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            times = []
            for _ in range(args.steps):
                dist.barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                if rank == 1 and skew:
                    torch.cuda._sleep(skew)
                fn()
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
            t = torch.tensor([sum(times) / len(times)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[f"{name}{'_skewed' if skew else ''}_ms"] = float(t.item())
    if comm.bench_plane != "generic":
        comm.native.plane = comm.bench_plane
    if rank == 0:
        for name in variants:
            res[f"{name}_skew_cost_ms"] = res[f"{name}_skewed_ms"] - res[f"{name}_ms"]
        print(json.dumps({"metric": METRIC, "workload": "imbalance study: all-to-all under "
                          f"{args.skew_us} us start skew on rank 1", "n_gpus": world,
                          "rows_per_peer": rows, "hidden": hidden, "unit": "ms",
                          "results": res, "plane": comm.bench_plane}), flush=True)
    dist.destroy_process_group()


def run_sweep(args):
    """BASELINE configs[4]: message sizes 64 KiB .. 1 GiB (per rank).

    N=1: the compressed path's own cost per size (measured codebook +
    encode + decode of one message, CUDA-graph replays) and the link
    bandwidth below which compression pays (the adaptive switch's flip
    point: codec time < bytes x (1 - 1/ratio) / link bandwidth).
    N>1: zip_all_gather vs the plain NCCL all-gather per size, max over
    ranks, plus the switcher's choice from a cost model fitted on the
    smallest/largest sizes (switcher.fit_cost_model).
    """
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2604_27844_b200 import engine, switcher
    policy = None
    if world > 1:
        world, rank, local, dev = _init_dist(args)
        from paper_2604_27844_b200 import collectives as coll
        comm = setup_comm(args, dev)
        if comm.bench_plane != "generic":
            comm.native.sync_errors = True
        # the adaptive switch, fitted ONCE on three sizes with the measured e
        # (switcher.profile_variants), then asked at every sweep size
        policy = switcher.profile_variants(comm, "all_gather", sizes=[1 << 16, 1 << 22, 1 << 26],
                                           trials=3)
    sizes = [(64 << 10) << k for k in range(15)]                # 64 KiB .. 1 GiB
    rows = []
    g = torch.Generator(device=dev).manual_seed(rank)
    for nbytes in sizes:
        n = nbytes // 2
        x = (torch.randn(n, device=dev, generator=g) * 0.02).to(torch.bfloat16)
        w = engine.words_view(x)
        reps = max(3, min(50, (64 << 20) // nbytes))
        if world == 1:
            frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
            out = torch.empty_like(w)
            flen = torch.empty(1, dtype=torch.int64, device=dev)
            err = torch.empty(1, dtype=torch.int32, device=dev)

            def step():
                engine.encode_measured(w, [(0, n)], 9, frames, [0], flen)
                engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err, groups512=True)
            step()
            torch.cuda.synchronize()
            assert int(err.item()) == engine.ERR_OK and torch.equal(out, w)
            F = int(flen.item())
            # several steps per graph: the host's graph-launch rate (~5 us)
            # would otherwise be what small messages measure
            inner = max(1, min(20, (64 << 20) // nbytes))
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for _ in range(inner):
                    step()
            for _ in range(3):
                gr.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(reps):
                gr.replay()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps / inner
            ratio = 2 * n / F
            saved = nbytes * (1 - 1 / ratio)
            rows.append({"bytes": nbytes, "codec_ms": ms, "codec_GBps": nbytes / (ms / 1e3) / 1e9,
                         "ratio": ratio,
                         "pays_below_link_GBps": saved / (ms / 1e3) / 1e9 if saved > 0 else 0.0})
        else:
            def timed(fn):
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                dist.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    fn()
                b.record()
                torch.cuda.synchronize()
                t = torch.tensor([a.elapsed_time(b) / reps], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                return float(t.item())
            raw_out = torch.empty(world * n, dtype=torch.bfloat16, device=dev)
            t_raw = timed(lambda: dist.all_gather_into_tensor(raw_out, x))
            row = {"bytes": nbytes, "raw_ms": t_raw,
                   "raw_GBps": world * nbytes / (t_raw / 1e3) / 1e9}
            for plane, _ in policy.models:
                with switcher._variant(comm, plane):
                    t = timed(lambda: coll.zip_all_gather(comm, x))
                row[f"zip_{plane}_ms"] = t
                row[f"zip_{plane}_GBps"] = world * nbytes / (t / 1e3) / 1e9
            best = min([("native", t_raw)] + [(v, row[f"zip_{v}_ms"]) for v, _ in policy.models],
                       key=lambda kv: kv[1])
            path, variant = switcher._decide(comm, policy, nbytes, w, True)
            t_sw = timed(lambda: switcher.switched_all_gather(comm, x, policy))
            row.update({"best_measured": best[0],
                        "switch": variant if path is switcher.Path.ZIPPED else "native",
                        "switched_ms": t_sw,
                        "switched_GBps": world * nbytes / (t_sw / 1e3) / 1e9})
            if nbytes in (1 << 20, 1 << 26):
                # incompressible gradient mix (C4 outliers): the switch must go native
                mix = _gpu_mix("mix_x1000", n, dev)
                path_m, _ = switcher._decide(comm, policy, nbytes, engine.words_view(mix), True)
                row["outlier_mix_switch"] = path_m.value
            rows.append(row)
        del x, w
    line = {"metric": METRIC, "workload": "c5 message-size sweep 64 KiB .. 1 GiB per rank",
            "n_gpus": world, "unit": "GB/s", "data": "synthetic N(0, 0.02^2) BF16",
            "rows": rows}
    if world > 1:
        line["policy"] = {v: {"alpha_native_s": m.alpha_rs, "beta_native_s_per_B": m.beta_rs,
                              "alpha_zipped_s": m.alpha_a2a, "beta_zipped_s_per_B": m.beta_a2a,
                              "e": m.e} for v, m in policy.models}
        line["switch_agrees_with_best"] = sum(r["switch"] == r["best_measured"] for r in rows)
        line["plane"] = comm.bench_plane
        line["nccl"] = nccl_info()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--clock-settle", type=float, default=1.0)
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the N=1 step eagerly (default: CUDA graph replays)")
    ap.add_argument("--workload", default="layer_ag",
                    choices=["layer_ag", "moe_a2a", "grad_mix", "sweep", "imbalance", "c1"],
                    help="layer_ag: the headline line (configs[1]); moe_a2a: configs[2]; "
                         "grad_mix: configs[3]; sweep: configs[4]")
    ap.add_argument("--tokens", type=int, default=4096, help="moe_a2a tokens per rank")
    ap.add_argument("--routing", default="uniform", choices=["uniform", "zipf"],
                    help="moe_a2a expert routing")
    ap.add_argument("--skew-us", type=float, default=200.0, help="imbalance: rank 1 start delay")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--transport", default="p2p", choices=["nccl", "p2p"],
                    help="nccl: the message plane (reference protocols over NCCL); "
                         "p2p: the decoder pulls peer frames over NVLink (IPC symmetric buffers)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode: every rank on cuda:0 (use with --backend gloo)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "grad_mix":
        run_grad_mix(args)
    elif args.workload == "c1":
        run_c1(args)
    elif args.workload == "moe_a2a":
        run_moe_a2a(args)
    elif args.workload == "sweep":
        run_sweep(args)
    elif args.workload == "imbalance":
        run_imbalance(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
