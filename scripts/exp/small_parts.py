"""Small-message codec step broken into legs (graph replay each)."""
import json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2604_27844_b200 import engine  # noqa: E402


INNER = 20


def t_graph(fn, reps=50):
    """GPU time per call: INNER calls captured in one graph (host launch
    overhead amortised), replayed `reps` times."""
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(INNER):
            fn()
    for _ in range(3):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(reps):
        g.replay()
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps / INNER * 1e3, 2)


def empty():
    pass

for kib in [int(a) for a in sys.argv[1:]] or [64, 256, 1024, 2048]:
    n = kib * 512
    g = torch.Generator(device="cuda").manual_seed(0)
    w = engine.words_view((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
    frames = torch.empty(engine.max_frame_bytes(n), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(w)
    flen = torch.empty(1, dtype=torch.int64, device="cuda")
    err = torch.empty(1, dtype=torch.int32, device="cuda")
    book = engine.measured_codebook(w)[0]
    enc = lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0], flen)  # noqa: E731
    enc_only = lambda: engine.encode(w, [(0, n)], book, 9, frames, [0], flen)  # noqa: E731
    stats = lambda: engine.measured_codebook(w)  # noqa: E731
    dec = lambda: engine.decode([frames.data_ptr()], [0], None, [n], out, [0], err=err, groups512=True)  # noqa: E731
    both = lambda: (enc(), dec())  # noqa: E731
    enc()
    dec()
    torch.cuda.synchronize()
    assert torch.equal(out, w)
    print(json.dumps({"kib": kib, "step_us": t_graph(both), "encode_measured_us": t_graph(enc),
                      "stats_us": t_graph(stats), "encode_book_us": t_graph(enc_only),
                      "decode_us": t_graph(dec)}), flush=True)
