# per-kernel times of the fused LM-head loss (launch list) + one ncu --set full capture of each backward GEMM
mkdir -p gpurun_out
python paper_2601_07376_b200/build.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lmbwd_launches.csv python scripts/prof_lmhead_loss.py 8192 3584 2 > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lmhead_bwd -s 2 -c 2 -o gpurun_out/prof_lmbwd -f python scripts/prof_lmhead_loss.py 8192 3584 2 > gpurun_out/ncu_lmbwd.log 2>&1; echo "full rc=$?"
