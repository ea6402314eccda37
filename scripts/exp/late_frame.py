"""Decode behind arrival (K5) on one GPU: three frames, the third published
late.  zc_decode_when_ready decodes the two ready frames while the third is
"in flight" (its ready flag is written by a copy-engine memcpy on another
stream after a host sleep); the time from that flag write to the end of the
decode is compared with decoding one frame and all three frames.

    python scripts/exp/late_frame.py [words_per_frame]
"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 25
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
words = [engine.words_view((torch.randn(n, device=dev, generator=g) * 0.02).to(torch.bfloat16))
         for _ in range(3)]
cap = engine.max_frame_bytes(n)
frames = torch.empty(3 * cap, dtype=torch.uint8, device=dev)
for i, w in enumerate(words):
    engine.encode_measured(w, [(0, n)], 9, frames[i * cap:(i + 1) * cap], [0])
out = torch.empty(3 * n, dtype=torch.int16, device=dev)
flags = torch.zeros(3, dtype=torch.int64, device=dev)
stat = [frames.data_ptr() + i * cap for i in range(3)]
ready = [flags.data_ptr() + 8 * i for i in range(3)]
offs = [i * n for i in range(3)]
one_host = torch.ones(1, dtype=torch.int64).pin_memory()
side = torch.cuda.Stream(dev)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


epoch = [0]


def all_ready(k=3):
    epoch[0] += 1
    flags.fill_(epoch[0])
    return engine.decode_when_ready(stat[:k], [n] * k, out, offs[:k], ready[:k], epoch[0])


t_one = timed(lambda: all_ready(1))
t_all = timed(lambda: all_ready(3))
tails, ok = [], True
for rep in range(8):
    epoch[0] += 1
    e = epoch[0]
    flags[:2].fill_(e)                      # frames 0 and 1 have arrived, frame 2 has not
    torch.cuda.synchronize()
    a, end, fl = ev(), ev(), ev()
    a.record()
    err = engine.decode_when_ready(stat, [n] * 3, out, offs, ready, e, timeout_ns=5_000_000_000)
    end.record()
    time.sleep(0.003)                       # frame 2 "in flight" for ~3 ms
    one_host.fill_(e)
    with torch.cuda.stream(side):
        flags[2:3].copy_(one_host, non_blocking=True)
        fl.record()
    torch.cuda.synchronize()
    ok &= bool((err.cpu() == engine.ERR_OK).all()) and all(
        torch.equal(out[i * n:(i + 1) * n], words[i]) for i in range(3))
    tails.append(fl.elapsed_time(end))
tail = sorted(tails)[len(tails) // 2]
print(json.dumps({
    "words_per_frame": n, "bit_exact": ok,
    "decode_one_frame_ms": round(t_one, 4), "decode_three_frames_ms": round(t_all, 4),
    "late_frame_tail_ms": round(tail, 4),
    "note": "tail = end of the one-launch decode after the late frame's ready flag was written "
            "(median of 8); a decoder that waits for every frame before decoding has a tail of "
            "decode_three_frames_ms"}))
