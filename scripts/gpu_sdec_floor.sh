# decode sampler: latency floor micro-benchmark + per-CTA timeline of the shipped kernel (experiment build)
mkdir -p gpurun_out .variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o .variants/decode_floor scripts/repro/decode_floor.cu
timeout 120 .variants/decode_floor > gpurun_out/decode_floor.txt 2>&1
python paper_2601_07376_b200/build.py > /dev/null
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_t.so', defines=['OTK_SDEC_TIMING'])"
OTK_LIB=.variants/libotk_t.so timeout 120 python scripts/timing_sample_dec.py > gpurun_out/sdec_timing.txt 2>&1
timeout 300 python scripts/perf_sample.py --rows 1,16,32,64,128 > gpurun_out/perf_sample.txt 2>&1
cat gpurun_out/decode_floor.txt gpurun_out/sdec_timing.txt gpurun_out/perf_sample.txt
