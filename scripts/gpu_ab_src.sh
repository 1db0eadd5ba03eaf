# A/B of the working tree's libotk.so against a copy of another revision's sources (.variants/oldsrc, made with
# git archive), alternating runs of a perf command on the same box: CMD="python scripts/perf_lmhead_loss.py ..."
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC,-O2 \
  --expt-relaxed-constexpr -cudart static -I .variants/oldsrc/include -o .variants/libotk_old.so \
  .variants/oldsrc/paper_2601_07376_b200/csrc/*.cu
for rep in 1 2 3; do
  echo "new $(timeout 300 $CMD | tail -1)"
  echo "old $(OTK_LIB=.variants/libotk_old.so timeout 300 $CMD | tail -1)"
done
