mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/box.txt 2>&1
nproc >> gpurun_out/box.txt; free -g >> gpurun_out/box.txt; lscpu | head -20 >> gpurun_out/box.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/smoke.log; tail -30 gpurun_out/gpu_tests.log
