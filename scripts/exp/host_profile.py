"""cProfile of the eager small-message codec calls (host overhead)."""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402

n = 32768
x = engine.words_view((torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
flen = torch.empty(1, dtype=torch.int64, device="cuda")
err = torch.empty(1, dtype=torch.int32, device="cuda")


def loop():
    for _ in range(2000):
        engine.encode_measured(x, [(0, n)], 9, frames, [0], flen)
        engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err, groups512=True)
    torch.cuda.synchronize()


loop()
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
