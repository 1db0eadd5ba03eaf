# decode sampler iteration: build, sampler tests, per-CTA timeline (experiment build), graph-timed rows
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_sample.py tests/test_gpu_graph.py -q -m gpu -p no:cacheprovider -x > gpurun_out/sample_tests.log 2>&1
tail -3 gpurun_out/sample_tests.log
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_t.so', defines=['OTK_SDEC_TIMING'])"
OTK_LIB=.variants/libotk_t.so timeout 120 python scripts/timing_sample_dec.py > gpurun_out/sdec_timing.txt 2>&1
timeout 300 python scripts/perf_sample.py --rows ${ROWS:-1,16,32,37,64} > gpurun_out/perf_sample.txt 2>&1
cat gpurun_out/sdec_timing.txt gpurun_out/perf_sample.txt
