mkdir -p gpurun_out
python paper_2601_07376_b200/build.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 2 -c 1 -o gpurun_out/prof_k4ones -f python scripts/prof_k4.py --mask ones > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 2 -c 1 -o gpurun_out/prof_k3 -f python scripts/prof_k4.py --fwd > gpurun_out/ncu_full3.log 2>&1; echo "full3 rc=$?"
