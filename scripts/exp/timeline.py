"""Per-CTA start/end spread of the encoder and decoder (load balance).

    nvcc ... -DZC_TIMELINE -> scripts/exp/libzipccl_timeline.so, then
    ZC_LIB_PATH=scripts/exp/libzipccl_timeline.so python scripts/exp/timeline.py
"""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import _lib, engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 218112000
g = torch.Generator(device="cuda").manual_seed(0)
w = engine.words_view((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
out = torch.empty_like(w)
for _ in range(3):
    engine.encode_measured(w, [(0, n)], 9, frames, [0])
    engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
torch.cuda.synchronize()
buf = np.zeros((6, 8192), dtype=np.uint64)
enc = np.zeros((6, 8192), dtype=np.uint64)
lib = _lib.lib()
lib.zc_debug_timeline_dec.argtypes = [ctypes.c_void_p]
lib.zc_debug_timeline_enc.argtypes = [ctypes.c_void_p]
assert lib.zc_debug_timeline_dec(buf.ctypes.data) == 0
assert lib.zc_debug_timeline_enc(enc.ctypes.data) == 0
buf[2:6] = enc[2:6]
encx = enc
res = {}
for name, a, b in (("decode", 0, 1), ("encode_pass1", 2, 5), ("encode_total", 2, 4)):
    st, en = buf[a].astype(np.int64), buf[b].astype(np.int64)
    m = (st > 0) & (en > 0)
    st, en = st[m], en[m]
    t0 = st.min()
    d = (en - st) / 1e3
    res[name] = {"ctas": int(m.sum()), "span_us": float((en.max() - t0) / 1e3),
                 "start_spread_us": float((st.max() - t0) / 1e3),
                 "end_min_us": float((en.min() - t0) / 1e3),
                 "end_p50_us": float(np.percentile(en - t0, 50) / 1e3),
                 "end_max_us": float((en.max() - t0) / 1e3),
                 "dur_min_us": float(d.min()), "dur_max_us": float(d.max())}
t0e = enc[2][enc[2] > 0].astype(np.int64).min()
for name, slot in (("enc_after_lookback", 0), ("enc_after_fixup", 1)):
    v = enc[slot][enc[slot] > 0].astype(np.int64) - t0e
    res[name] = {"min_us": float(v.min() / 1e3), "p50_us": float(np.percentile(v, 50) / 1e3),
                 "max_us": float(v.max() / 1e3)}
p1 = enc[5].astype(np.int64) - t0e
lb = enc[0].astype(np.int64) - t0e
ok = (enc[5] > 0) & (enc[0] > 0)
idx = np.nonzero(ok)[0]
strag = idx[np.argmax(p1[idx])]
res["straggler"] = {"cta": int(strag), "pass1_end_us": float(p1[strag] / 1e3),
                    "lookback_end_us": float(lb[strag] / 1e3)}
top = idx[np.argsort(-lb[idx])[:6]]
res["latest_lookbacks"] = [(int(i), round(float(p1[i] / 1e3), 1), round(float(lb[i] / 1e3), 1))
                           for i in top]
late = idx[np.argsort(-p1[idx])[:8]]
res["latest_pass1"] = [(int(i), round(float(p1[i] / 1e3), 1), round(float(lb[i] / 1e3), 1))
                       for i in late]
print(json.dumps(res, indent=1))
