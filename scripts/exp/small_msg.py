"""Kernels of one small-message codec step (encode_measured + decode), for an
ncu launch list; plus graph-replay timing per size."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402

for kib in [int(a) for a in sys.argv[1:]] or [64, 256, 2048]:
    n = kib * 512
    g = torch.Generator(device="cuda").manual_seed(0)
    w = engine.words_view((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(w)
    flen = torch.empty(1, dtype=torch.int64, device="cuda")
    err = torch.empty(1, dtype=torch.int32, device="cuda")

    def step():
        engine.encode_measured(w, [(0, n)], 9, frames, [0], flen)
        engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err, groups512=True)
    step()
    torch.cuda.synchronize()
    assert torch.equal(out, w)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for _ in range(5):
        gr.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(50):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"kib": kib, "us": round(a.elapsed_time(b) / 50 * 1e3, 1)}))
