"""Speculative encode leg (guess + encoder + fix-up + conditional launches),
graph-replayed, at the layer size: the guess kernel's share."""
import json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402
dev = torch.device("cuda", 0)
w = engine.words_view(bench.layer_shard(0, 1, dev))
n = w.numel()
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device=dev)
fn = lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0])  # noqa: E731
fn(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    fn()
for _ in range(3):
    g.replay()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
for _ in range(20):
    g.replay()
b.record(); torch.cuda.synchronize()
print(json.dumps({"lib": os.path.basename(os.environ.get("ZC_LIB_PATH", "default")),
                  "encode_leg_us": round(a.elapsed_time(b) / 20 * 1e3, 1)}))
