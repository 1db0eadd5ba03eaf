"""Summarise an ncu report: key throughput metrics, stall reasons and the hottest SASS lines."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__cluster_dim_x", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "sm__sass_inst_executed_op_shared_ld.sum"]
for h, u, v in zip(hdr, units, vals):
    if h in keys:
        print(f"{h:70s} {v} {u}")
st = [(h, float(v or 0)) for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
tot = sum(v for _, v in st)
print("stall samples:", int(tot))
for h, v in sorted(st, key=lambda x: -x[1])[:10]:
    print(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {v / tot:6.3f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(src.splitlines()))
h = r[1]; body = r[2:]
si, ai, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
body = [x for x in body if len(x) > si and x[si].isdigit()]
print("instructions:", len(body))
for x in sorted(body, key=lambda x: -int(x[si]))[:top]:
    print(f"  {x[si]:>7s} {x[ei]:>10s} {x[0][-5:]} {x[ai][:90]}")
