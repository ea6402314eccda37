"""One C4 mix, codebook_for + compress a few times (for ncu launch lists)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402
kind = sys.argv[1] if len(sys.argv) > 1 else "mix_x1000"
n = 1 << 28
dev = torch.device("cuda", 0)
w = engine.words_view(bench._gpu_mix(kind, n, dev))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
for _ in range(3):
    engine.encode_measured(w, [(0, n)], 9, frames, [0])
torch.cuda.synchronize()
