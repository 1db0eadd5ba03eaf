# experiment runner (scratch): cluster cap + VPF pipelining comparisons
for lib in .variants/libotk_nopipe.so ""; do
  OTK_LIB=$lib timeout 200 python scripts/perf_k4.py --vocab 262144 --rows 32768 2>&1 | tail -1
  OTK_LIB=$lib timeout 200 python scripts/perf_k4.py 2>&1 | tail -1
done > gpurun_out/perf_cap.jsonl
OTK_LIB=.variants/libotk_nopipe.so timeout 300 python scripts/perf_vpf.py --ranks 4 8 > gpurun_out/perf_vpf_nopipe.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "policy_loss or logprob" > gpurun_out/cap_parity.log 2>&1; echo "rc=$?" >> gpurun_out/cap_parity.log
