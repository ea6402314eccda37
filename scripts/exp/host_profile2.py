"""cProfile of the eager public API on a small message (host overhead)."""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_27844_b200 as zc  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402

n = 32768
x = engine.words_view((torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16))
book = zc.codebook_for(x)


def loop():
    for _ in range(1000):
        c = zc.compress(x, book)
        zc.decompress(c)
        zc.codebook_for(x)
    torch.cuda.synchronize()


loop()
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
