"""Per-stage timing of the public-API e2e path + allocator behaviour."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_27844_b200 as zc  # noqa: E402

n = 218_112_000
g = torch.Generator(device="cuda").manual_seed(0)
x0 = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
host = x0.view(torch.int16).cpu().pin_memory()


def allocs():
    return torch.cuda.memory_stats().get("num_device_alloc", 0)


for it in range(4):
    torch.cuda.synchronize()
    a0 = allocs()
    t = [time.perf_counter()]
    x = host.to("cuda", non_blocking=True)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    book = zc.codebook_for(x)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    chunk = zc.compress(x, book)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    y = zc.decompress(chunk)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])]
    print(f"iter {it}: h2d {d[0]} book {d[1]} compress {d[2]} decompress {d[3]} ms; "
          f"device allocs +{allocs() - a0}", flush=True)
