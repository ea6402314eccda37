"""measure_sigma cost (exact Chan pass + numpy-order passes) at the layer size."""
import json, sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
import paper_2604_27844_b200 as zc  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402
dev = torch.device("cuda", 0)
w = engine.words_view(bench.layer_shard(0, 1, dev))
for _ in range(2):
    engine.measured_codebook(w, exact=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    engine.measured_codebook(w, exact=True)
b.record(); torch.cuda.synchronize()
s = zc.measure_sigma(w)
v = (w.cpu().numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
ref = float(np.std(v))
print(json.dumps({"exact_sigma_us": round(a.elapsed_time(b) / 10 * 1e3, 1), "sigma": s,
                  "numpy": ref, "bit_identical": s == ref}))
