# full round evidence: tests, bench (all legs), ncu launch list of the bench, ncu full capture of K4/K3 and of the
# round-2 kernels (LM-head backward, decode sampler), sanitizers + the racecheck reproducer, the side measurements
mkdir -p gpurun_out
python paper_2601_07376_b200/build.py
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next > gpurun_out/ncu_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 2 -c 1 -o gpurun_out/prof_k4 -f python scripts/prof_k4.py > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 2 -c 1 -o gpurun_out/prof_k3 -f python scripts/prof_k4.py --fwd > gpurun_out/ncu_full3.log 2>&1; echo "full3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 2 -c 1 -o gpurun_out/prof_sample -f python scripts/prof_sample.py 4096 > gpurun_out/ncu_sample.log 2>&1; echo "sample rc=$?"
timeout 300 python scripts/perf_sample.py > gpurun_out/perf_sample.jsonl 2>&1; echo "perf_sample rc=$?"
for tool in memcheck racecheck synccheck; do timeout 600 compute-sanitizer --tool $tool --error-exitcode 3 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log; done
tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/gpu_tests.log; tail -1 gpurun_out/bench.err; tail -1 gpurun_out/bench_ref.err; tail -n2 gpurun_out/sanitize_*.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_lmhead -s 2 -c 1 -o gpurun_out/prof_lmhead -f python scripts/prof_lmhead.py 8192 > gpurun_out/ncu_lmhead.log 2>&1; echo "lmhead rc=$?"
for n in 4096 8192 16384; do timeout 60 python scripts/perf_lmhead.py --rows $n --iters 5 2>&1 | tail -1; done > gpurun_out/perf_lmhead.jsonl
for v in "" ent dual seqmean seqsum sft turn; do timeout 120 python scripts/perf_k4.py --variant "$v" 2>&1 | tail -1; done > gpurun_out/perf_variants.jsonl
# round-1 additions: K4-VPF (emulated ranks), the loss through the LM head, the traffic-structure probe
timeout 300 python scripts/perf_vpf.py --ranks 2 4 8 > gpurun_out/perf_vpf.jsonl 2>&1; echo "perf_vpf rc=$?"
timeout 300 python scripts/vpf_isolation.py > gpurun_out/vpf_isolation.jsonl 2>&1; echo "vpf_isolation rc=$?"
for n in 4096 8192; do timeout 200 python scripts/perf_lmhead_loss.py --rows $n 2>&1 | tail -1; done > gpurun_out/perf_lmhead_loss.jsonl
timeout 300 python scripts/hbm_probe3.py > gpurun_out/hbm_probe3.json 2>&1; echo "hbm_probe3 rc=$?"
# round-2 additions: the LM-head backward (fused vs cuBLAS at d = 1024 / 3584, ncu of both GEMMs), the decode sampler,
# the racecheck reproducer of the TMA ring protocol
for d in 1024 2048 3584; do timeout 200 python scripts/perf_lmhead_loss.py --rows 8192 --d $d 2>&1 | tail -1; done > gpurun_out/perf_lmhead_loss.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lmhead_bwd -c 2 -o gpurun_out/prof_lmbwd -f python scripts/prof_lmhead_loss.py 8192 3584 1 > gpurun_out/ncu_lmbwd.log 2>&1; echo "lmbwd rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lmbwd_launches.csv python scripts/prof_lmhead_loss.py 8192 3584 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sample_dec -s 4 -c 1 -o gpurun_out/prof_sdec -f python scripts/prof_sample_dec.py 16 > gpurun_out/ncu_sdec.log 2>&1; echo "sdec rc=$?"
timeout 300 python scripts/perf_sample.py --rows 1,16,32,37,48,64,96,128,148,256,1024,4096 > gpurun_out/perf_sample.jsonl 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2601_07376_b200/csrc -o /tmp/rr scripts/repro/racecheck_tma_ring.cu && \
  (timeout 300 compute-sanitizer --tool racecheck /tmp/rr > gpurun_out/racecheck_repro.log 2>&1; echo "repro rc=$?" >> gpurun_out/racecheck_repro.log)
# round-2 (late) additions: the other workloads' bench lines, the store-path HBM probe, per-CTA phase stamps of
# the decode and ring samplers (experiment builds), the batch-sharded C example (also in pytest)
for c in game marl vp; do timeout 900 python bench.py --config $c --no-next > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
timeout 300 python scripts/hbm_probe4.py > gpurun_out/hbm_probe4.json 2>&1; echo "hbm_probe4 rc=$?"
mkdir -p .variants
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_sdec_t.so', defines=['OTK_SDEC_TIMING'])
build.build(out='.variants/libotk_stm_t.so', defines=['OTK_STM_TIMING'])"
OTK_LIB=.variants/libotk_sdec_t.so timeout 120 python scripts/timing_sample_dec.py > gpurun_out/sdec_phases.txt 2>&1
OTK_LIB=.variants/libotk_stm_t.so timeout 120 python scripts/timing_sample_tm.py > gpurun_out/stm_phases.txt 2>&1
