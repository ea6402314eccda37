"""Turn gpurun_out ncu captures into committed summaries under profiles/.

    python scripts/summarize_profiles.py <tag>
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
sys.path.insert(0, str(ROOT / "scripts"))
from ncu_summary import raw  # noqa: E402


def launches(tag):
    rows = list(csv.reader(open(OUT / f"launches_bench_{tag}.csv")))
    hdr, items = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                items.append((d["Kernel Name"], float(d["Metric Value"])))
    items = [(k[5:] if k.startswith("void ") else k, v) for k, v in items]
    zc = [(k, v) for k, v in items if k.startswith("zc::")]
    # one bench step = guess, encoder (fused statistic + certificate + fix-up),
    # two conditional launches, decode: the zc:: launches from the last guess on
    first = max(i for i, (k, _) in enumerate(zc) if k.startswith("zc::guess_kernel"))
    last = next(i for i in range(first, len(zc)) if zc[i][0].startswith("zc::decode_ring"))
    step = zc[first:last + 1]
    total = sum(v for _, v in step)
    lines = [f"# launch list, one bench step (ncu gpu__time_duration, cold-cache, serialised)",
             f"# source: gpurun_out/launches_bench_{tag}.csv ({len(items)} launches)"]
    for k, v in step:
        name = k.split('(')[0].replace("void ", "")
        lines.append(f"{name:<36} {v / 1e3:9.1f} us  {100 * v / total:5.1f}% of step")
    lines.append(f"{'step total':<32} {total / 1e3:9.1f} us")
    (PROF / f"{tag}_launches.txt").write_text("\n".join(lines) + "\n")
    return step


def kernel_summary(tag, kname):
    rep = OUT / f"prof_bench_{tag}_{kname}.ncu-rep"
    rows, units = raw(str(rep))
    d = rows[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
    lines = [f"# ncu --set full, {d.get('Kernel Name', '')[:80]}", f"# source: {rep.name}"]
    for k in keys:
        if k in d:
            lines.append(f"{k} = {d[k]} {units.get(k, '')}")
    pipes = {k.split("pipe_")[1].split(".")[0]: float(d[k]) for k in d
             if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active")
             and d[k] not in ("", "n/a")}
    lines.append("pipes (% of peak, active): " + ", ".join(
        f"{k}={v:.0f}" for k, v in sorted(pipes.items(), key=lambda x: -x[1])[:8]))
    st = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(d[k]) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and d[k] not in ("", "n/a")}
    stot = sum(st.values()) or 1.0
    lines.append("stall reasons (% of samples): " + ", ".join(
        f"{k}={100 * v / stot:.1f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
    if "smsp__warps_eligible.avg.per_cycle_active" in d:
        lines.append(f"warps eligible per cycle = {d['smsp__warps_eligible.avg.per_cycle_active']}")
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.reader(out.splitlines())
    next(r)
    hdr = next(r)
    srows = [dict(zip(hdr, x)) for x in r]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(int(x[key] or 0) for x in srows) or 1
    lines.append(f"top stall sites ({tot} samples):")
    for x in sorted(srows, key=lambda x: -int(x[key] or 0))[:10]:
        lines.append(f"  {100 * int(x[key] or 0) / tot:5.1f}%  {x['Source'].strip()[:90]}")
    (PROF / f"{tag}_ncu_{kname}.txt").write_text("\n".join(lines) + "\n")
    mb = 1e6 if units.get("dram__bytes_read.sum", "").startswith("M") else (
        1e9 if units.get("dram__bytes_read.sum", "").startswith("G") else 1.0)
    return (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * mb, \
        float(d["gpu__time_duration.sum"])


if __name__ == "__main__":
    tag = sys.argv[1]
    PROF.mkdir(exist_ok=True)
    launches(tag)
    traffic = {}
    for k in ("decode_ring", "encode_tiles", "encode_runfix", "guess_kernel"):
        b, t = kernel_summary(tag, k)
        traffic[f"{k if k.endswith('kernel') else k + '_kernel'}_per_launch_bytes"] = b
    traffic["source"] = f"ncu --set full captures prof_bench_{tag}_*.ncu-rep (dram__bytes_read.sum + dram__bytes_write.sum)"
    (PROF / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print(json.dumps(traffic, indent=1))
