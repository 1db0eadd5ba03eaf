# A/B of LM-head backward experiment builds (DEFINES_B / DEFINES_C) against the default build, fused path only
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py
python -c "
import sys, os; sys.path.insert(0, 'paper_2601_07376_b200'); import build
for tag in ('b', 'c'):
    d = os.environ.get('DEFINES_' + tag.upper(), '')
    if d: build.build(out=f'.variants/libotk_{tag}.so', defines=d.split())"
for args in "--rows 8192 --d 3584" "--rows 8192 --d 1024"; do
  echo "default $args $(timeout 300 python scripts/perf_lmhead_loss.py $args --impl fused 2>&1 | tail -1)"
  for tag in b c; do
    [ -f .variants/libotk_$tag.so ] && echo "$tag $args $(OTK_LIB=.variants/libotk_$tag.so timeout 300 python scripts/perf_lmhead_loss.py $args --impl fused 2>&1 | tail -1)"
  done
done > gpurun_out/lmbwd_ab.txt
for tag in b c; do
  [ -f .variants/libotk_$tag.so ] && OTK_LIB=.variants/libotk_$tag.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lmbwd_launches_$tag.csv python scripts/prof_lmhead_loss.py 8192 3584 1 > /dev/null 2>&1
done
cat gpurun_out/lmbwd_ab.txt
for tag in b c; do [ -f gpurun_out/lmbwd_launches_$tag.csv ] && grep -o 'k_lmhead_bwd<[01]>.*' gpurun_out/lmbwd_launches_$tag.csv | awk -F'"' '{print "'$tag'", $1, $NF, $(NF-1)}'; done
