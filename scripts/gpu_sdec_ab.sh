# decode sampler experiments: for builds with DEFINES_{A,B,C}: stamps (timing build) + graph-timed rows
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
for tag in A B C; do
  v="DEFINES_$tag"; d="${!v}"
  [ -z "$d" ] && continue
  python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_$tag.so', defines='$d'.split())
build.build(out='.variants/libotk_${tag}t.so', defines='$d OTK_SDEC_TIMING'.split())"
  echo "== $tag ($d)"
  OTK_LIB=.variants/libotk_${tag}t.so timeout 120 python scripts/timing_sample_dec.py | grep " 3 "
  OTK_LIB=.variants/libotk_$tag.so timeout 300 python scripts/perf_sample.py --rows ${ROWS:-1,16,64} 2>&1 | tail -5 | cut -c1-120
done
