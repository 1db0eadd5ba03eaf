# ring sampler experiments: for builds with DEFINES_{A,B,C}: first-row timeline (timing build) + graph-timed rows
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
for tag in A B C; do
  v="DEFINES_$tag"; d="${!v}"
  [ -z "$d" ] && continue
  python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_$tag.so', defines='$d'.split())
build.build(out='.variants/libotk_${tag}t.so', defines='$d OTK_STM_TIMING'.split())"
  echo "== $tag ($d)"
  OTK_LIB=.variants/libotk_${tag}t.so timeout 120 python scripts/timing_sample_tm.py
  OTK_LIB=.variants/libotk_$tag.so timeout 300 python scripts/perf_sample.py --rows ${ROWS:-128,4096} 2>&1 | tail -8 | cut -c1-100
done
