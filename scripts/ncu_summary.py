"""Summarise an ncu report: duration, DRAM bytes/throughput, issue, pipes, stalls."""
import csv, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines()); hdr = next(r); units = next(r)
    return [dict(zip(hdr, row)) for row in r], dict(zip(hdr, units))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]
def main():
  for rep in sys.argv[1:]:
      rows, units = raw(rep)
      for d in rows:
          print("==", rep, d.get("Kernel Name", "")[:40])
          for k in KEYS:
              if k in d: print(f"  {k} = {d[k]} {units.get(k,'')}")
          pipes = {k: float(d[k]) for k in d if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active") and d[k] not in ("", "n/a")}
          print("  pipes:", ", ".join(f"{k.split('pipe_')[1].split('.')[0]}={v:.0f}%" for k, v in sorted(pipes.items(), key=lambda x: -x[1])[:6]))
          st = {k: float(d[k]) for k in d if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio") and d[k] not in ("", "n/a")}
          if not st:
              st = {k: float(d[k]) for k in d if k.startswith("smsp__warp_issue_stalled_") and k.endswith("_per_warp_active.pct") and d[k] not in ("", "n/a")}
          print("  stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0].split('.')[0]}={v:.1f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:7]))


def top_stalls(rep, k=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines()); next(r); hdr = next(r)
    rows = [dict(zip(hdr, x)) for x in r]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(int(x[key] or 0) for x in rows)
    print(f"-- {rep}: {tot} stall samples; top instructions")
    for x in sorted(rows, key=lambda x: -int(x[key] or 0))[:k]:
        print(f"  {int(x[key] or 0) / max(tot, 1) * 100:5.1f}%  {x['Source'][:80]}")


if __name__ == "__main__":
    main()
    if "--stalls" in sys.argv or True:
        for rep in sys.argv[1:]:
            top_stalls(rep, 15)
