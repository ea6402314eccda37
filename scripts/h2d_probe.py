"""Host<->device copy bandwidth from pinned memory (the e2e leg's floor).

    python scripts/h2d_probe.py [--mb 436]
"""
import argparse
import json
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=int, default=436)
args = ap.parse_args()
nbytes = args.mb * 1_000_000
host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
host.fill_(1)
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
r = {"bytes": nbytes}


def wall(fn, it=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / it


r["h2d_1copy_GBps"] = nbytes / wall(lambda: dev.copy_(host, non_blocking=True)) / 1e9
r["d2h_1copy_GBps"] = nbytes / wall(lambda: host.copy_(dev, non_blocking=True)) / 1e9
for k in (2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(k)]
    step = (nbytes + k - 1) // k

    def multi():
        cur = torch.cuda.current_stream()
        for i, s in enumerate(ss):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                dev[i * step:(i + 1) * step].copy_(host[i * step:(i + 1) * step], non_blocking=True)
        for s in ss:
            cur.wait_stream(s)
    r[f"h2d_{k}streams_GBps"] = nbytes / wall(multi) / 1e9
# chunked in order on one stream (pipeline granularity)
for mb in (8, 32):
    step = mb * 1_000_000

    def chunked():
        for lo in range(0, nbytes, step):
            dev[lo:lo + step].copy_(host[lo:lo + step], non_blocking=True)
    r[f"h2d_chunk{mb}MB_GBps"] = nbytes / wall(chunked) / 1e9
# pageable source, for reference
pg = torch.empty(nbytes // 4, dtype=torch.uint8)
r["h2d_pageable_GBps"] = (nbytes // 4) / wall(lambda: dev[:nbytes // 4].copy_(pg)) / 1e9
print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}))
