# LM-head backward experiment: clock64 breakdown of the dh / dW kernels (MMA waits, transform, epilogue) from a
# -DOTK_BW_TIMING build (scripts/timing_lmbwd.py)
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_t.so', defines=['OTK_BW_TIMING'])"
OTK_LIB=.variants/libotk_t.so timeout 300 python scripts/timing_lmbwd.py 8192 3584 > gpurun_out/lmbwd_timing.json 2>&1
cat gpurun_out/lmbwd_timing.json
