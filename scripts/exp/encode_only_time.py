"""Encoder (pass 1 + fix-up) duration only, no output check (experiments)."""
import json, os, statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402
n = 218112000
g = torch.Generator(device="cuda").manual_seed(0)
w = engine.words_view((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
for _ in range(3):
    engine.encode_measured(w, [(0, n)], 9, frames, [0])
torch.cuda.synchronize()
engine.profile_enable(True)
for _ in range(30):
    engine.encode_measured(w, [(0, n)], 9, frames, [0])
torch.cuda.synchronize()
engine.profile_enable(False)
e = statistics.median(engine.profile_read(engine.PROF_ENCODE))
print(json.dumps({"lib": os.path.basename(os.environ.get("ZC_LIB_PATH", "default")),
                  "encode_us": round(e * 1e3, 1)}))
