# alternating A/B of the default build vs DEFINES_B on the whole LM-head step (fused) and the forward alone
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py
python -c "
import sys, os; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_b.so', defines=os.environ['DEFINES_B'].split())"
for rep in 1 2; do
  for d in 3584 1024; do
    echo "A d=$d $(timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl fused | tail -1)"
    echo "B d=$d $(OTK_LIB=.variants/libotk_b.so timeout 300 python scripts/perf_lmhead_loss.py --rows 8192 --d $d --impl fused | tail -1)"
  done
done > gpurun_out/lm_ab2.txt
cat gpurun_out/lm_ab2.txt | sed 's/"rows.*"fused"/fused/'
