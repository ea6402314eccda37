"""Per-kernel device timing of the codec (CUDA events, inputs > L2).

    python scripts/kernel_timing.py [--n N] [--sigma S] [--kind gauss|mix_x1000|...]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2604_27844_b200 import codec, engine  # noqa: E402


def timed(fn, iters=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(iters)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--sigma", type=float, default=0.02)
    ap.add_argument("--repeat", type=int, default=0)
    ap.add_argument("--no-check", action="store_true")
    args = ap.parse_args()
    n = args.n
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.randn(n, device="cuda", generator=g) * args.sigma).to(torch.bfloat16)
    w = engine.words_view(x)
    book, res = engine.measured_codebook(w)
    cap = engine.max_frame_bytes(n)
    frames = torch.empty(cap, dtype=torch.uint8, device="cuda")
    flen = engine.encode(w, [(0, n)], book, 9, frames, [0])
    F = int(flen.item())
    out = torch.empty_like(w)
    err = engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
    code = int(err.item())
    if not args.no_check:
        assert code == engine.ERR_OK, engine.err_message(code)
        assert torch.equal(out, w)
    ref = frames[:F].clone()
    for _ in range(args.repeat):   # determinism / race stress
        engine.encode(w, [(0, n)], book, 9, frames, [0], flen)
        e2 = engine.decode([frames.data_ptr()], [0], None, [n], out, [0])
        c2 = int(e2.item())
        assert c2 == engine.ERR_OK, engine.err_message(c2)
        assert torch.equal(frames[:F], ref) and torch.equal(out, w)
    def graphed(fn):
        # CUDA-graph replay: measures device time without host launch overhead
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g.replay
    t_stats = timed(graphed(lambda: engine.measured_codebook(w)))
    t_enc = timed(graphed(lambda: engine.encode(w, [(0, n)], book, 9, frames, [0], flen)))
    t_dec = timed(graphed(lambda: engine.decode([frames.data_ptr()], [0], None, [n], out, [0])))
    t_step = timed(graphed(lambda: (engine.encode_measured(w, [(0, n)], 9, frames, [0], flen,
                                                           speculative=False),
                                    engine.decode([frames.data_ptr()], [0], None, [n], out,
                                                  [0]))))
    t_enc_spec = timed(graphed(lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0], flen,
                                                              speculative=True)))
    t_enc_meas = timed(graphed(lambda: engine.encode_measured(w, [(0, n)], 9, frames, [0], flen,
                                                              speculative=False)))
    t_step_spec = timed(graphed(lambda: (engine.encode_measured(w, [(0, n)], 9, frames, [0], flen,
                                                                speculative=True),
                                         engine.decode([frames.data_ptr()], [0], None, [n], out,
                                                       [0]))))
    copy_dst = torch.empty_like(w)
    t_copy = timed(lambda: copy_dst.copy_(w))
    r = dict(n=n, frame=F, ratio=2 * n / F,
             stats_ms=t_stats, stats_GBps=2 * n / t_stats / 1e6,
             encode_ms=t_enc, encode_GBps=(2 * n + F) / t_enc / 1e6,
             decode_ms=t_dec, decode_GBps=(2 * n + F) / t_dec / 1e6,
             copy_ms=t_copy, copy_GBps=4 * n / t_copy / 1e6,
             step_ms=t_step, step_GBps=2 * n / t_step / 1e6,
             measured_encode_ms=t_enc_meas, speculative_encode_ms=t_enc_spec,
             step_spec_ms=t_step_spec, step_spec_GBps=2 * n / t_step_spec / 1e6,
             sigma=float(res[0].item()), book=book[:7].tolist())
    print(json.dumps(r))


if __name__ == "__main__":
    main()
