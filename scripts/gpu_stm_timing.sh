# ring sampler: per-CTA timeline of the first row (experiment build) + graph-timed rows
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_stm.so', defines=['OTK_STM_TIMING'])"
OTK_LIB=.variants/libotk_stm.so timeout 120 python scripts/timing_sample_tm.py
