# LM-head backward: dh as two launches (tile 0 with the transform + the rest over the stored dx tiles) vs one
# launch with the transform in every hidden tile (-DOTK_BW_ONE_DH); tests, alternating timings, launch list
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_one.so', defines=['OTK_BW_ONE_DH'])"
timeout 900 python -m pytest tests/test_gpu_lmhead_loss.py tests/test_gpu_lmhead.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
for rep in 1 2; do
  for d in 1024 2048 3584; do
    echo "split d=$d $(timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl both 2>&1 | tail -1)"
    echo "one   d=$d $(OTK_LIB=.variants/libotk_one.so timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl fused 2>&1 | tail -1)"
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lmbwd_split_launches.csv python scripts/prof_lmhead_loss.py 8192 3584 1 > /dev/null 2>&1
grep -o 'otk::k_lmhead.*' gpurun_out/lmbwd_split_launches.csv | awk -F'"' '{print $1, $(NF-1)}' | cut -c1-60
