"""Encoder pass-1 variant check: frame digest + median encode time (library
hooks) on the bench layer and on C4 mixes.  Run once with and once without
ZC_ENCODE_CTA_RUNS=1 and compare the digests (experiments; no asserts)."""
import hashlib, json, os, statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2604_27844_b200 import engine  # noqa: E402

dev = torch.device("cuda:0")
out = {"variant": os.path.basename(os.environ.get("ZC_LIB_PATH", "default"))}
cases = [("layer", engine.words_view(bench.layer_shard(0, 1, dev)))]
for kind in ("mix", "mix_x1000", "lognormal2"):
    cases.append((kind, engine.words_view(bench._gpu_mix(kind, 1 << 26, dev))))
# ragged multi-segment (A2A-like): odd sizes, 16-B aligned offsets
w = cases[0][1]
for name, words in cases + [("segs", None)]:
    if name == "segs":
        words = w[: 3 * (1 << 22) + 4096]
        segs = [(0, 1 << 22), (1 << 22, (1 << 22) - 104), (2 << 22, (1 << 22) + 4000)]
    else:
        segs = [(0, words.numel())]
    cap = sum(engine.max_frame_bytes(n) for _, n in segs)
    frames = torch.zeros(cap, dtype=torch.uint8, device=dev)
    offs, o = [], 0
    for _, n in segs:
        offs.append(o)
        o += engine.max_frame_bytes(n)
    for _ in range(3):
        book, res, flen = engine.encode_measured(words, segs, 9, frames, offs)
    torch.cuda.synchronize()
    h = hashlib.sha256()
    fl = flen.cpu().tolist()
    for off, L in zip(offs, fl):
        h.update(frames[off:off + L].cpu().numpy().tobytes())
    engine.profile_enable(True)
    for _ in range(20):
        engine.encode_measured(words, segs, 9, frames, offs)
    torch.cuda.synchronize()
    engine.profile_enable(False)
    t = statistics.median(engine.profile_read(engine.PROF_ENCODE))
    xs = torch.cat([words[o:o + n] for o, n in segs]).view(torch.bfloat16).double()
    xs = xs[torch.isfinite(xs)]
    ref = xs.std(unbiased=False).item()
    r = res.cpu().tolist()
    out[name] = {"sha": h.hexdigest()[:16], "enc_us": round(t * 1e3, 1), "flen": fl,
                 "sigma_rel_err": (r[0] - ref) / ref, "path": r[2], "book": book.cpu().tolist()[:7]}
print(json.dumps(out))
