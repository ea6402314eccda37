"""One push decode and one pull (flag-gated) decode of the same 4 frames (for
an ncu capture of both decode_ring_kernel variants)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402

dev = torch.device("cuda", 0)
n, k = 218112000 // 4, 4
g = torch.Generator(device=dev).manual_seed(3)
ws = [engine.words_view((torch.randn(n, device=dev, generator=g) * 0.02).to(torch.bfloat16))
      for _ in range(k)]
cap = engine.max_frame_bytes(n)
frames = torch.empty(k * cap, dtype=torch.uint8, device=dev)
for i, w in enumerate(ws):
    engine.encode_measured(w, [(0, n)], 9, frames[i * cap:(i + 1) * cap], [0])
out = torch.empty(k * n, dtype=torch.int16, device=dev)
flags = torch.ones(k, dtype=torch.int64, device=dev)
stat = [frames.data_ptr() + i * cap for i in range(k)]
offs = [i * n for i in range(k)]
ready = [flags.data_ptr() + 8 * i for i in range(k)]
for _ in range(2):
    engine.decode(stat, [0] * k, None, [n] * k, out, offs)
    engine.decode_when_ready(stat, [n] * k, out, offs, ready, 1)
torch.cuda.synchronize()
