# experiment: the row kernels with 16 consumer warps (OTK_K4_CW16) vs 12 — GPU parity tests on the variant, then
# alternating timings of the loss kernel (math mix, all-trainable) and the forward
mkdir -p gpurun_out .variants
python paper_2601_07376_b200/build.py > /dev/null
python -c "
import sys; sys.path.insert(0, 'paper_2601_07376_b200'); import build
build.build(out='.variants/libotk_cw16.so', defines=['OTK_K4_CW16'])"
OTK_LIB=.variants/libotk_cw16.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vpf.py tests/test_gpu_edges.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
for rep in 1 2; do
  for mask in data ones; do
    echo "cw12 $mask $(timeout 120 python scripts/perf_k4.py --mask $mask 2>&1 | tail -1)"
    echo "cw16 $mask $(OTK_LIB=.variants/libotk_cw16.so timeout 120 python scripts/perf_k4.py --mask $mask 2>&1 | tail -1)"
  done
done
