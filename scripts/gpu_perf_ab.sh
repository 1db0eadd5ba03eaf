# A/B of an experiment build against the default libotk.so on the loss kernel (perf_k4.py), alternating runs.
# usage: DEFINES="OTK_NO_ZERO_PACING" bash scripts/gpu_perf_ab.sh
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py
python -c "
import sys, os; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_b.so', defines=os.environ.get('DEFINES', '').split())"
for rep in 1 2; do
  for mask in data ones; do
    timeout 120 python scripts/perf_k4.py --mask $mask 2>&1 | tail -1
    OTK_LIB=.variants/libotk_b.so timeout 120 python scripts/perf_k4.py --mask $mask 2>&1 | tail -1
  done
done > gpurun_out/perf_ab.jsonl
cat gpurun_out/perf_ab.jsonl
