"""Turn the scratch ncu outputs in gpurun_out/ into the tracked evidence under profiles/.

    python scripts/make_profiles.py r01

Writes profiles/<tag>_launches.csv (every launch of `bench.py --steps 2 --warmup 1` under
`ncu --metrics gpu__time_duration.sum --clock-control none`, names shortened), <tag>_launches_summary.txt
(per-kernel totals and the K4 share of the timed otk step), <tag>_k4_ncu.txt / <tag>_k3_ncu.txt (ncu --set
full summaries: DRAM bytes, pipe utilisation, stall reasons, hottest SASS) and k4_traffic.json (DRAM bytes
per K4 launch vs its algorithmic bytes; bench.py copies it into roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def short(name):
    if name.startswith("void otk::") or name.startswith("otk::"):
        return name.replace("void ", "").split("(")[0]
    return name.split("(")[0][:60]


def launches(tag):
    rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], [r for r in rows[i + 1:] if len(r) > 5]
    ki, vi, gi, bi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Block Size")
    out = []
    for r in data:
        out.append((int(r[0]), short(r[ki]), r[gi], r[bi], float(r[vi].replace(",", ""))))
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
        f.write("id,kernel,grid,block,gpu__time_duration_ns\n")
        for o in out:
            f.write(f'{o[0]},"{o[1]}","{o[2]}","{o[3]}",{o[4]:.0f}\n')
    # the timed otk step: masks, advantages and the loss launches (setup K3 / torch kernels excluded)
    # K4 = k_rows_tm<bf16, BWD (=2), ...> whatever its trailing template arguments are
    is_k4 = lambda name: name.startswith("otk::k_rows_tm<__nv_bfloat16, 2")
    step_k = [o for o in out if o[1] in ("otk::k_build_masks", "otk::k_group_advantages") or is_k4(o[1])]
    tot = {}
    for o in out:
        tot.setdefault(o[1], [0, 0.0])
        tot[o[1]][0] += 1
        tot[o[1]][1] += o[4]
    s = sum(o[4] for o in step_k)
    k4 = sum(o[4] for o in step_k if is_k4(o[1]))
    lines = [f"ncu launch list of `bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline` ({len(out)} launches, "
             "cold-cache and serialised)", "", f"{'kernel':60s} {'n':>5s} {'total ms':>10s}"]
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:60s} {n:5d} {t / 1e6:10.3f}")
    lines += ["", f"otk step launches (masks + advantages + loss): {len(step_k)}, total {s / 1e6:.3f} ms",
              f"K4 k_rows_tm<bf16, BWD> share of the otk step time: {k4 / s:.4f}"]
    open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[-2:]))


def ncu_summary(rep, dst):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, "40"],
                         capture_output=True, text=True).stdout
    open(dst, "w").write(txt)
    return txt


def traffic(rep, tag):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = lambda k: (float(vals[hdr.index(k)]), units[hdr.index(k)])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd, ru = get("dram__bytes_read.sum")
    wr, wu = get("dram__bytes_write.sum")
    t, tu = get("gpu__time_duration.sum")
    b = rd * scale[ru] + wr * scale[wu]
    d = {"traffic_bytes_per_launch": b, "dram_read_bytes": rd * scale[ru], "dram_write_bytes": wr * scale[wu],
         "launch": "scripts/prof_k4.py: one 65536-row micro-batch of the math workload (micro-batch 0 masks)",
         "source": f"profiles/{tag}_k4_ncu.txt (ncu --set full --clock-control none)",
         "ncu_duration_ms": t if tu == "ms" else t / 1e3}
    json.dump(d, open(os.path.join(PROF, "k4_traffic.json"), "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    ncu_summary(os.path.join(OUT, "prof_k4.ncu-rep"), os.path.join(PROF, f"{tag}_k4_ncu.txt"))
    ncu_summary(os.path.join(OUT, "prof_k3.ncu-rep"), os.path.join(PROF, f"{tag}_k3_ncu.txt"))
    for name in ("sample", "lmhead", "lmbwd", "sdec"):   # optional captures of the NEXT-3 / NEXT-1 kernels
        rep = os.path.join(OUT, f"prof_{name}.ncu-rep")
        if os.path.exists(rep):
            if name == "lmbwd":   # two kernels (dh, dW): per-kernel metrics and stalls
                txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_kernels.py"), rep],
                                     capture_output=True, text=True).stdout
                open(os.path.join(PROF, f"{tag}_{name}_ncu.txt"), "w").write(txt)
            else:
                ncu_summary(rep, os.path.join(PROF, f"{tag}_{name}_ncu.txt"))
    import shutil
    for src, dst in (("perf_sample.jsonl", "perf_sample.jsonl"), ("perf_lmhead.jsonl", "perf_lmhead.jsonl"),
                     ("perf_variants.jsonl", "perf_variants.jsonl"), ("perf_vpf.jsonl", "perf_vpf.jsonl"),
                     ("vpf_isolation.jsonl", "vpf_isolation.jsonl"), ("perf_lmhead_loss.jsonl", "perf_lmhead_loss.jsonl"),
                     ("hbm_probe3.json", "hbm_probe3.json"),
                     ("sanitize_memcheck.log", "sanitize_memcheck.txt"),
                     ("sanitize_racecheck.log", "sanitize_racecheck.txt"),
                     ("sanitize_synccheck.log", "sanitize_synccheck.txt"),
                     ("racecheck_repro.log", "racecheck_repro.txt"), ("lmbwd_launches.csv", "lmbwd_launches.csv"),
                     ("hbm_probe4.json", "hbm_probe4.json"), ("sdec_phases.txt", "sdec_phases.txt"),
                     ("stm_phases.txt", "stm_phases.txt")):
        if os.path.exists(os.path.join(OUT, src)):
            if "compute-sanitizer is closed" in open(os.path.join(OUT, src), errors="replace").read():
                continue   # the pool refused the sanitizer run: keep the last real log
            shutil.copy(os.path.join(OUT, src), os.path.join(PROF, f"{tag}_{dst}"))
    traffic(os.path.join(OUT, "prof_k4.ncu-rep"), tag)
    for f in ("bench.json", "bench_ref.json", "bench_game.json", "bench_marl.json", "bench_vp.json"):
        if os.path.exists(os.path.join(OUT, f)):
            open(os.path.join(PROF, f"{tag}_{f}"), "w").write(open(os.path.join(OUT, f)).read())
