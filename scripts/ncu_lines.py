"""Per-CUDA-source-line instruction counts and stall samples from an ncu report (needs -lineinfo)."""
import csv, subprocess, sys
rep = sys.argv[1]; elems = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = [r for r in rows if r and r[0] == "Line No"][0]
si, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) > ei and r[0] not in ("", "Line No", "File Path", "Function Name") and r[ei].isdigit():
        lines.append((int(r[ei]), int(r[si]) if r[si].isdigit() else 0, r[0], r[1]))
tot = sum(l[0] for l in lines); ts = sum(l[1] for l in lines)
print(f"total warp-instr {tot} ({tot * 32 / elems:.2f} per element), stall samples {ts}")
for n, smp, ln, src in sorted(lines, key=lambda l: -l[0])[:top]:
    print(f"{n * 32 / elems:6.3f}/el {smp / max(ts, 1):6.3f}st  L{ln:>5s}  {src.strip()[:95]}")
