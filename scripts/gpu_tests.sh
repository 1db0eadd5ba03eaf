mkdir -p gpurun_out
python paper_2601_07376_b200/build.py
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider ${TEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
