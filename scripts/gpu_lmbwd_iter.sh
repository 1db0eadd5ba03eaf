# LM-head backward iteration: its tests, fused timing (default + optional DEFINES_B / DEFINES_C experiment builds
# through gpu_lmbwd_ab.sh), per-kernel launch times
# LM-head backward iteration: tests, timing (default + optional experiment builds), per-kernel launch times
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py
timeout 600 python -m pytest tests/test_gpu_lmhead_loss.py -q -p no:cacheprovider -rA ${TEST_ARGS} > gpurun_out/lmbwd_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/lmbwd_tests.log
grep -E "^(PASSED|FAILED)|passed|failed" gpurun_out/lmbwd_tests.log | tail -14
DEFINES_B=${DEFINES_B:-} DEFINES_C=${DEFINES_C:-} bash scripts/gpu_lmbwd_ab.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lmbwd_launches.csv python scripts/prof_lmhead_loss.py 8192 3584 1 > /dev/null 2>&1
grep -o 'otk::k_lmhead[^"]*".*' gpurun_out/lmbwd_launches.csv | awk -F'"' '{print $1, $NF, $(NF-1)}' | tail -5
