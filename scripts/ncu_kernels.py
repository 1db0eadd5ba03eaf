"""Per-kernel key metrics and top stall reasons of a multi-kernel ncu report: python scripts/ncu_kernels.py rep"""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__registers_per_thread"]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:70])
    for k in keys:
        if k in hdr:
            print(f"   {k.split('.')[0][-45:]:45s} {r[hdr.index(k)]}")
    st = [(h, float(v or 0)) for h, v in zip(hdr, r) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    print("   stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot:.2f}"
                                  for h, v in sorted(st, key=lambda x: -x[1])[:6]))
