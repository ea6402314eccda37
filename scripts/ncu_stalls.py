"""Stall-reason breakdown + headline metrics of an ncu report (first kernel)."""
import csv, subprocess, sys
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines())); h = r[0]; d = dict(zip(h, r[2]))
    st = {k: float(d[k]) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and d[k] not in ("", "n/a")}
    tot = sum(st.values()) or 1
    print("==", rep, d.get("Kernel Name", "")[:50])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
              "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]:
        print(f"  {k} = {d.get(k)}")
    pipes = {k: float(d[k]) for k in d if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active") and d[k] not in ("", "n/a")}
    print("  pipes:", ", ".join(f"{k.split('pipe_')[1].split('.')[0]}={v:.0f}%" for k, v in sorted(pipes.items(), key=lambda x: -x[1])[:6]))
    print("  stalls:", ", ".join(f"{k[len('smsp__pcsamp_warps_issue_stalled_'):]}={v / tot * 100:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
