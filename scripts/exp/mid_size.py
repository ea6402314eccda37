"""Encode / decode legs of one mid-size message (CUDA-graph replays), to see
what the fixed costs are between 4 MiB and 256 MiB.

    python scripts/exp/mid_size.py [MiB ...]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402

dev = torch.device("cuda", 0)
# sizes in MiB, or KiB with a "k" suffix
sizes = [(int(a[:-1]) << 10) if a.endswith("k") else (int(a) << 20) for a in sys.argv[1:]] \
    or [m << 20 for m in (4, 8, 16, 32, 64, 128, 256)]


def leg_us(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for nbytes in sizes:
    n = nbytes // 2
    gen = torch.Generator(device=dev).manual_seed(1)
    w = engine.words_view((torch.randn(n, device=dev, generator=gen) * 0.02).to(torch.bfloat16))
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
    out = torch.empty_like(w)
    flen = torch.empty(1, dtype=torch.int64, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    enc = lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0], flen)  # noqa: E731
    dec = lambda: engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err,  # noqa: E731
                                groups512=True)
    e_us, d_us = leg_us(enc), leg_us(dec)
    F = int(flen.item())
    ideal = (2 * n + F) * 2 / 6.1e12 * 1e6   # both legs at 6.1 TB/s
    print(json.dumps({"KiB": nbytes >> 10, "encode_us": round(e_us, 1), "decode_us": round(d_us, 1),
                      "step_us": round(e_us + d_us, 1), "hbm_floor_us": round(ideal, 1)}))
