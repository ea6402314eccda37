"""Encode / decode durations (library hooks) on the C4 mixes, 2^28 words."""
import json, statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402
n = 1 << 28
dev = torch.device("cuda", 0)
for kind in ("mix", "mix_x1000", "lognormal2"):
    w = engine.words_view(bench._gpu_mix(kind, n, dev))
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
    out = torch.empty_like(w)
    engine.encode_measured(w, [(0, n)], 9, frames, [0])
    err = engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
    torch.cuda.synchronize()
    assert int(err.item()) == engine.ERR_OK and torch.equal(out, w)
    engine.profile_enable(True)
    for _ in range(10):
        engine.encode_measured(w, [(0, n)], 9, frames, [0])
        engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
    torch.cuda.synchronize()
    engine.profile_enable(False)
    print(json.dumps({"kind": kind,
                      "encode_us": round(statistics.median(engine.profile_read(0)) * 1e3, 1),
                      "decode_us": round(statistics.median(engine.profile_read(1)) * 1e3, 1)}))
