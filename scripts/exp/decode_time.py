"""Decoder kernel duration (library event hooks), one library variant."""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402

n = 218112000
g = torch.Generator(device="cuda").manual_seed(0)
w = engine.words_view((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
out = torch.empty_like(w)
_, _, flen = engine.encode_measured(w, [(0, n)], 9, frames, [0])
F = int(flen.item())
for _ in range(3):
    engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
torch.cuda.synchronize()
assert torch.equal(out, w)
engine.profile_enable(True)
for _ in range(30):
    engine.encode_measured(w, [(0, n)], 9, frames, [0])
    engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
torch.cuda.synchronize()
engine.profile_enable(False)
d = statistics.median(engine.profile_read(engine.PROF_DECODE))
e = statistics.median(engine.profile_read(engine.PROF_ENCODE))
print(json.dumps({"lib": os.path.basename(os.environ.get("ZC_LIB_PATH", "default")),
                  "decode_us": round(d * 1e3, 1), "decode_GBps": round((2 * n + F) / d / 1e6),
                  "encode_us": round(e * 1e3, 1), "encode_GBps": round((2 * n + F) / e / 1e6)}))
