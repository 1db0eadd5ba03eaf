# GPU tests + smoke (plain and under ncu, as the driver's census runs it) + default bench (round 2 iteration script)
mkdir -p gpurun_out
python paper_2601_07376_b200/build.py
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo "smoke_ncu rc=$?" >> gpurun_out/smoke_ncu.log
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -rA ${TEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/smoke_ncu.log; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -3; tail -1 gpurun_out/bench.err
