"""Per-CTA start/end and SM placement of encoder pass 1 and the decoder on
the bench layer (load balance; -DZC_TIMELINE library).

    python scripts/build_variant.py timeline -DZC_TIMELINE
    ZC_LIB_PATH=build/timeline.so python scripts/exp/timeline2.py
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
lib = _lib.lib()
lib.zc_debug_timeline_dec.argtypes = [ctypes.c_void_p]
lib.zc_debug_timeline_enc.argtypes = [ctypes.c_void_p]


def spread(st, en, sm):
    m = (st > 0) & (en > 0)
    st, en, sm = st[m].astype(np.int64), en[m].astype(np.int64), sm[m]
    t0 = st.min()
    e = (en - t0) / 1e3
    s = (st - t0) / 1e3
    d = e - s
    die = sm % 2   # placement parity; the die split is inferred from the numbers
    per_sm_end = {}
    for smi, ei in zip(sm, e):
        per_sm_end[int(smi)] = max(per_sm_end.get(int(smi), 0.0), float(ei))
    v = np.array(list(per_sm_end.values()))
    return {"ctas": int(m.sum()), "span_us": round(float(e.max()), 1),
            "start_p50_us": round(float(np.percentile(s, 50)), 2),
            "start_max_us": round(float(s.max()), 2),
            "end_min_us": round(float(e.min()), 1),
            "end_p10_us": round(float(np.percentile(e, 10)), 1),
            "end_p50_us": round(float(np.percentile(e, 50)), 1),
            "end_p90_us": round(float(np.percentile(e, 90)), 1),
            "end_max_us": round(float(e.max()), 1),
            "dur_p50_us": round(float(np.percentile(d, 50)), 1),
            "dur_even_sm_p50": round(float(np.percentile(d[die == 0], 50)), 1),
            "dur_odd_sm_p50": round(float(np.percentile(d[die == 1], 50)), 1),
            "ctas_per_sm_max": int(np.bincount(sm.astype(np.int64)).max()),
            "sm_last_end_p10_p50_p90": [round(float(np.percentile(v, q)), 1) for q in (10, 50, 90)],
            "busy_frac": round(float(d.sum() / (e.max() * len(d))), 3)}


res = {}
for rep in range(3):
    engine.encode_measured(w, [(0, n)], 9, frames, [0], speculative=True)
    torch.cuda.synchronize()
    enc = np.zeros((10, 8192), dtype=np.uint64)
    assert lib.zc_debug_timeline_enc(enc.ctypes.data) == 0
    engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
    torch.cuda.synchronize()
    dec = np.zeros((10, 8192), dtype=np.uint64)
    assert lib.zc_debug_timeline_dec(dec.ctypes.data) == 0
    if rep == 2:
        res["encode_pass1"] = spread(enc[2], enc[5], enc[3])
        t0 = enc[2][enc[2] > 0].astype(np.int64).min()
        for nm, sl in (("runfix_start", 0), ("runfix_waited", 6), ("runfix_before_P", 7),
                       ("runfix_stored", 8), ("runfix_end", 1), ("pass1_end", 5),
                       ("pass1_certified", 4)):
            v = (enc[sl][enc[sl] > 0].astype(np.int64) - t0) / 1e3
            if v.size:
                res[nm] = [round(float(np.percentile(v, q)), 1) for q in (0, 10, 50, 90, 100)]
        e1 = enc[1].astype(np.int64)
        late = np.argsort(-e1)[:6]
        res["latest_runfix_ctas"] = {
            int(c): [round(float((enc[sl][c].astype(np.int64) - t0) / 1e3), 2)
                     for sl in (5, 4, 0, 6, 7, 8, 1)] for c in late}
        res["latest_runfix_cols"] = "pass1_end pass1_exit rf_start rf_waited rf_before_P rf_stored rf_end"
        res["decode"] = spread(dec[0], dec[1], dec[2])
print(json.dumps(res, indent=1))
