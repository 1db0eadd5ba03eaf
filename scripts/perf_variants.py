"""Build libotk variants side by side and time each with scripts/perf_k4.py (experiments only).
Args: "" (current tree), "A=1,B=0" (-D flags), "git:REV" (csrc + include of a revision), "dir:PATH" (an extracted tree, e.g. .variants/head)."""
import os, subprocess, sys, tempfile
sys.path.insert(0, os.getcwd())
from paper_2601_07376_b200 import build
specs = sys.argv[1:] or [""]
libs = []
for i, spec in enumerate(specs):
    out = f"/tmp/libotk_var{i}.so"
    if spec.startswith("git:") or spec.startswith("dir:"):
        if spec.startswith("git:"):
            d = tempfile.mkdtemp()
            subprocess.check_call(f"git archive {spec[4:]} paper_2601_07376_b200/csrc include | tar -x -C {d}", shell=True)
        else:
            d = spec[4:]
        srcs = sorted(os.path.join(d, "paper_2601_07376_b200/csrc", f) for f in os.listdir(os.path.join(d, "paper_2601_07376_b200/csrc")) if f.endswith(".cu"))
        subprocess.check_call([build.NVCC, *build.FLAGS, "-I", os.path.join(d, "include"), "-o", out, *srcs])
    else:
        build.build(out=out, defines=[x for x in spec.split(",") if x])
    libs.append((spec, out))
extra = os.environ.get("PERF_ARGS", "").split()
for spec, out in libs:
    r = subprocess.run([sys.executable, "scripts/perf_k4.py", *extra], env=dict(os.environ, OTK_LIB=out), capture_output=True, text=True)
    print(repr(spec), r.stdout.strip() or r.stderr[-2000:], flush=True)
