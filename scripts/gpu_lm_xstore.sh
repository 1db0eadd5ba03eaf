# LM-head forward x-tile store: L2 evict-first hint (default) vs a plain store (-DOTK_LM_XSTORE_PLAIN), fused loss
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_plain.so', defines=['OTK_LM_XSTORE_PLAIN'])"
for rep in 1 2; do
  for d in 3584 1024; do
    echo "evict d=$d $(timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl fused 2>&1 | tail -1 | cut -c1-120)"
    echo "plain d=$d $(OTK_LIB=.variants/libotk_plain.so timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl fused 2>&1 | tail -1 | cut -c1-120)"
  done
done
