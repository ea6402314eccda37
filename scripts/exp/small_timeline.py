"""Phase timeline of the one-launch small encoder (-DZC_TIMELINE library).

    python scripts/build_variant.py timeline -DZC_TIMELINE
    ZC_LIB_PATH=build/timeline.so python scripts/exp/small_timeline.py [KiB]
"""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import _lib, engine  # noqa: E402

kib = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = kib * 512
g = torch.Generator(device="cuda").manual_seed(0)
w = engine.words_view((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
lib = _lib.lib()
lib.zc_debug_timeline_small.argtypes = [ctypes.c_void_p]
names = ["start", "loaded", "sums_synced", "codebook", "encoded", "totals_synced", "final_sync",
         "end"]
rows = []
for rep in range(12):
    engine.encode_measured(w, [(0, n)], 9, frames, [0])
    torch.cuda.synchronize()
    tl = np.zeros((10, 8192), dtype=np.uint64)
    assert lib.zc_debug_timeline_small(tl.ctypes.data) == 0
    c = int((tl[0] > 0).sum())
    t0 = tl[0][:c].astype(np.int64).min()
    rows.append([float((tl[k][:c].astype(np.int64) - t0).max()) / 1e3 for k in range(8)])
med = np.median(np.array(rows[2:]), axis=0)
print(json.dumps({"KiB": kib, "ctas": c, "phase_end_us (max over CTAs, median of 10)":
                  dict(zip(names, [round(v, 2) for v in med]))}))
