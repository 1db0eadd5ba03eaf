# LM-head backward: the plain dh launch's split-K (OTK_BW_S1) — alternating fused timings at d = 3584 / 2048
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
for k in (6, 9):
    build.build(out=f'.variants/libotk_s{k}.so', defines=[f'OTK_BW_S1={k}'])"
for rep in 1 2; do
  for d in 3584 2048; do
    echo "default d=$d $(timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl fused 2>&1 | tail -1 | cut -c1-120)"
    for k in 6 9; do
      echo "s1=$k d=$d $(OTK_LIB=.variants/libotk_s$k.so timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl fused 2>&1 | tail -1 | cut -c1-120)"
    done
  done
done
