mkdir -p gpurun_out
python paper_2601_07376_b200/build.py
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/smoke.log; tail -4 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -2 gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=d['roofline']
print('value %.3e ms/step %.2f K4 %.0f GB/s frac %.3f share %.3f clocks %s e2e %s cpu %s' % (d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['share_of_step'], d['clocks'], d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value')))"
