"""Explicit-codebook encode of the C4 mixes (2^26 words): frame digest and
median time, to compare the two-pass encoder with the single-pass look-back
encoder forced for every size (a -DZC_LBMAX=... build)."""
import hashlib
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
import paper_2604_27844_b200 as zc  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402

dev = torch.device("cuda:0")
out = {"lib": os.path.basename(os.environ.get("ZC_LIB_PATH", "default"))}
for kind in ("mix", "mix_x1000", "lognormal2"):
    w = engine.words_view(bench._gpu_mix(kind, 1 << 26, dev))
    n = w.numel()
    book = engine.book_tensor(zc.codebook_for(w).entries, dev)
    frames = torch.zeros(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
    for _ in range(3):
        flen = engine.encode(w, [(0, n)], book, 9, frames, [0])
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        engine.encode(w, [(0, n)], book, 9, frames, [0], flen)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    L = int(flen.item())
    out[kind] = {"us": round(statistics.median(ts) * 1e3, 1),
                 "sha": hashlib.sha256(frames[:L].cpu().numpy().tobytes()).hexdigest()[:16]}
print(json.dumps(out))
