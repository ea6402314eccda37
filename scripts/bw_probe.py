"""HBM bandwidth probes: write-only, read-only, copy (CUDA events, > L2)."""
import torch, json
n = 1 << 29   # bytes per buffer in 16-bit words ... 1 GiB
a = torch.empty(n, dtype=torch.int16, device="cuda")
b = torch.empty(n, dtype=torch.int16, device="cuda")
a.random_()
def timed(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(it)]
    for s, t in e:
        s.record(); fn(); t.record()
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(t) for s, t in e); return ts[len(ts)//2]
B = 2 * n
r = {}
r["write_GBps"] = B / timed(lambda: b.fill_(3)) / 1e6
r["read_GBps"] = B / timed(lambda: a.view(torch.int32).max()) / 1e6
r["copy_GBps"] = 2 * B / timed(lambda: b.copy_(a)) / 1e6
print(json.dumps({k: round(v, 1) for k, v in r.items()}))
