# K4-VPF iteration: its tests, then fused vs gathered at P = 2, 4, 8 (one-GPU emulation), default vs DEFINES_B
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py
timeout 900 python -m pytest tests/test_gpu_vpf.py tests/test_gpu_edges.py -q -p no:cacheprovider -x > gpurun_out/vpf_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/vpf_tests.log
tail -2 gpurun_out/vpf_tests.log
timeout 600 python scripts/perf_vpf.py --ranks 2 4 8 > gpurun_out/perf_vpf.jsonl 2>&1
if [ -n "$DEFINES_B" ]; then
  python -c "
import sys, os; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_b.so', defines=os.environ['DEFINES_B'].split())"
  OTK_LIB=.variants/libotk_b.so timeout 600 python scripts/perf_vpf.py --ranks 4 8 > gpurun_out/perf_vpf_b.jsonl 2>&1
fi
cat gpurun_out/perf_vpf.jsonl; echo "-- B ($DEFINES_B)"; cat gpurun_out/perf_vpf_b.jsonl 2>/dev/null
