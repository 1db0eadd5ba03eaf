# sampler A/B: default build vs DEFINES_B on decode batch sizes
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py
python -c "
import sys, os; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_b.so', defines=os.environ['DEFINES_B'].split())"
echo A; timeout 300 python scripts/perf_sample.py --rows ${ROWS:-96,128} 2>&1 | tail -4
echo B; OTK_LIB=.variants/libotk_b.so timeout 300 python scripts/perf_sample.py --rows ${ROWS:-96,128} 2>&1 | tail -4
