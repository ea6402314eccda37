"""Where the encode time goes on escape-heavy mixes (library hooks + events)."""
import json, statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402
n = 1 << 28
dev = torch.device("cuda", 0)


def timed(fn, it=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


for kind in ("mix", "mix_x1000", "lognormal2"):
    w = engine.words_view(bench._gpu_mix(kind, n, dev))
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
    book, res, fl = engine.encode_measured(w, [(0, n)], 9, frames, [0])
    path = res.cpu().tolist()[2]
    r = {"kind": kind, "path": path, "zc_frac": None,
         "spec_leg_us": timed(lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0])),
         "nonspec_leg_us": timed(lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0],
                                                                speculative=False)),
         "plain_encode_us": timed(lambda: engine.encode(w, [(0, n)], book, 9, frames, [0])),
         "stats_us": timed(lambda: engine.measured_codebook(w))}
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()}))
