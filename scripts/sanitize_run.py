"""Small runs of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): stats (certified + exact + modal), encoders (look-back,
two-pass, speculative with a wrong guess, multi-segment), decoders (ring in
all modes, look-back for large groups, group ranges), corrupt frames.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_27844_b200 as zc  # noqa: E402
from paper_2604_27844_b200 import codec, engine  # noqa: E402
from paper_2604_27844_b200.errors import CorruptChunkError, CorruptFrameError  # noqa: E402

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)


def words(n, s=0.02):
    return engine.words_view((torch.randn(n, device="cuda", generator=g) * s).to(torch.bfloat16))


checks = 0
for n, gs in [(1, 512), (1000, 16), (4096 * 20 + 7, 512), (4096 * 40, 2048), (70000, 1 << 14),
              (5000, 4)]:
    x = words(n)
    book = zc.codebook_for(x)
    chunk = zc.compress(x, book, group_size=gs)
    assert torch.equal(zc.decompress(chunk), x)
    ng = (n + gs - 1) // gs
    assert torch.equal(zc.decompress_group(chunk, ng - 1), x[(ng - 1) * gs:])
    checks += 1
# one-launch small encoder / decoder (clusters, DSMEM pushes): measured
# codebook + encode, decode with the 512-group flag
for n in (100, 100_000, 262_144):
    x = words(n)
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    book, res, flen = engine.encode_measured(x, [(0, n)], 9, frames, [0])
    out = torch.empty_like(x)
    err = engine.decode([frames.data_ptr()], [0], None, [n], out, [0], groups512=True)
    assert int(err[0].item()) == engine.ERR_OK and torch.equal(out, x)
    checks += 1
# sigma next to a flip threshold: the f64 fallback's last CTA and every CTA
# of the cluster encoder re-derive the codebook from numpy's own sigma
from tests.test_stats_gpu import _flip_sigma, _tuned  # noqa: E402
for n in (1 << 18, 1 << 20):
    host = _tuned(_flip_sigma(-6), n, 3e-11, seed=n)
    x = torch.from_numpy(host.view(np.int16)).cuda()
    book, res = engine.measured_codebook(x)
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    engine.encode_measured(x, [(0, n)], 9, frames, [0])
    checks += 1
# measure_sigma with non-finite elements (device compaction + numpy order)
x = words(100_003)
x[77] = 0x7FC0
zc.measure_sigma(x)
checks += 1
# speculative path (>= 1024 tiles): certified, and a guess the sample gets wrong
n = 4096 * 1100 + 3
for case in ("gauss", "fool"):
    v = torch.randn(n, device="cuda", generator=g)
    if case == "fool":
        v = v * 1000.0
        t = torch.arange(n, device="cuda")
        v[(t % 8192) < 16] *= 1e-6          # exactly the guess kernel's sampled sectors
    x = engine.words_view(v.to(torch.bfloat16))
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    book, res, flen = engine.encode_measured(x, [(0, n)], 9, frames, [0])
    ref = zc.serialize(zc.compress(x, zc.codebook_for(x)))
    assert bytes(frames[:int(flen.item())].cpu().numpy()) == ref
    checks += 1
# multi-segment encode / decode (all-to-all framing)
buf = words(3 * 100_003 + 5, 0.3)
segs = [(1, 100_003), (100_004, 0), (200_007, 100_001)]
segs = [s for s in segs if s[1]]
caps = [engine.max_frame_bytes(c) for _, c in segs]
offs = [0, caps[0]]
frames = torch.empty(sum(caps), dtype=torch.uint8, device="cuda")
_, flen = codec.device_encode(buf, segs, None, frames, offs)
out = torch.empty(sum(c for _, c in segs), dtype=torch.int16, device="cuda")
err = engine.decode([frames.data_ptr() + o for o in offs], [0, 0], None, [c for _, c in segs], out,
                    [0, segs[0][1]])
assert (err.cpu() == engine.ERR_OK).all()
checks += 1
# numpy-order sigma (measure_sigma: exact Chan pass + np_sigma_kernel passes)
for n in (5, 1000, 4096 * 40 + 3):
    x = words(n)
    zc.measure_sigma(x)
checks += 1
# modal fallback and explicit sigma
x = words(10_000)
zc.codebook_for(x, sigma=0.0)
zc.codebook_for(torch.zeros(5000, dtype=torch.int16, device="cuda"))
checks += 1
# corrupt frames: the validator must stay in bounds
x = words(50_000)
frame = bytearray(zc.serialize(zc.compress(x, zc.codebook_for(x))))
rng = np.random.default_rng(1)
for _ in range(20):
    f = bytearray(frame)
    i = int(rng.integers(128, len(f)))
    f[i] ^= 1 << int(rng.integers(0, 8))
    try:
        zc.decompress(zc.parse(bytes(f)))
    except (CorruptFrameError, CorruptChunkError):
        pass
checks += 1
# escape-heavy data (two-pass encoder: dense staging, the fix-up's shifted
# 16-B copies of runs with > 4096 escapes), checked against the oracle
from oracle import zc_oracle as zo  # noqa: E402
n = 4096 * 1100 + 5
v = torch.exp(torch.randn(n, device="cuda", generator=g) * 2.0 - 8.0)
x = engine.words_view(v.to(torch.bfloat16))
book = zc.codebook_for(x)
fr = zc.serialize(zc.compress(x, book))
assert fr == zo.encode(x.cpu().numpy().view(np.uint16), book.entries)
assert torch.equal(zc.decompress(zc.parse(fr)), x)
checks += 1
# decode behind arrival (flags already set) and a timed-out flag
x = words(4096 * 30 + 9)
chunk = zc.compress(x, zc.codebook_for(x))
flags = torch.tensor([3, 2], dtype=torch.int64, device="cuda")
outd = torch.empty(2 * x.numel(), dtype=torch.int16, device="cuda")
err = engine.decode_when_ready([chunk.frame.data_ptr()] * 2, [x.numel()] * 2, outd,
                               [0, x.numel()], [flags.data_ptr(), flags.data_ptr() + 8], 3,
                               timeout_ns=2_000_000)
codes = err.cpu().tolist()
assert codes[0] == engine.ERR_OK and codes[1] == 20 and torch.equal(outd[:x.numel()], x)
checks += 1
# collectives on native thread ranks sharing cuda:0: the message plane and
# the peer-memory pull-decode, all-gather, all-to-all d1/d2, reduce-scatter
from paper_2604_27844_b200 import collectives as coll  # noqa: E402
from paper_2604_27844_b200.transport import run_ranks  # noqa: E402


def body(comm):
    ok = True
    for plane in ("msg", "p2p"):
        comm.native.plane = plane
        for it in range(2):
            local = words(200_003 + it)
            ok &= torch.equal(coll.zip_all_gather(comm, local),
                              coll.reference_all_gather(comm, local))
            sizes = [(comm.rank + d) * 3000 + 17 for d in range(comm.world_size)]
            spec = coll.AlltoAllSpec([words(c) for c in sizes],
                                     [(s + comm.rank) * 3000 + 17 for s in range(comm.world_size)])
            r = coll.reference_all_to_all(comm, spec)
            for fn in (coll.zip_all_to_all_d1, coll.zip_all_to_all_d2):
                z = fn(comm, spec)
                ok &= all(torch.equal(a, b) for a, b in zip(z, r))
            xs = words(comm.world_size * 40_000)
            ok &= torch.equal(coll.zip_reduce_scatter(comm, xs),
                              coll.reference_reduce_scatter(comm, xs))
    return ok


assert all(run_ranks(3, body))
checks += 1
torch.cuda.synchronize()
print(f"sanitize_run ok: {checks} groups of checks")
