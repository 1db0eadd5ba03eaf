mkdir -p gpurun_out
python paper_2601_07376_b200/build.py
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
