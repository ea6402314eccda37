"""One speculative measured encode + decode at the layer size (for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_27844_b200 import engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 218112000
g = torch.Generator(device="cuda").manual_seed(0)
w = engine.words_view((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
out = torch.empty_like(w)
for _ in range(3):
    engine.encode_measured(w, [(0, n)], 9, frames, [0], speculative=True)
    engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
torch.cuda.synchronize()
assert torch.equal(out, w)
