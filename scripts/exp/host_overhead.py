"""Eager per-call cost of the public codec API on a small message (host-bound:
the GPU work is ~11 us), per layer of the stack."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_27844_b200 as zc  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402

n = 32768
x = engine.words_view((torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
flen = torch.empty(1, dtype=torch.int64, device="cuda")
err = torch.empty(1, dtype=torch.int32, device="cuda")
book = zc.codebook_for(x)


def per_call(fn, it=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t) / it * 1e6, 1)


r = {
    "engine.encode_measured": per_call(lambda: engine.encode_measured(x, [(0, n)], 9, frames, [0], flen)),
    "engine.decode": per_call(lambda: engine.decode([frames.data_ptr()], [0], None, [n], out, [0],
                                                    err=err, groups512=True)),
    "zc.compress(x, book)": per_call(lambda: zc.compress(x, book)),
    "zc.codebook_for(x)": per_call(lambda: zc.codebook_for(x), 500),
    "zc.decompress(chunk)": per_call(lambda: zc.decompress(zc.compress(x, book)), 500),
    "torch.empty (reference point)": per_call(lambda: torch.empty(1000, device="cuda")),
}
print(json.dumps(r))
