timeout 900 python -m pytest tests/test_apply_gpu.py -x -q -m gpu -k "radix4 or quadtree or wide or synthetic" 2>&1 | tail -3
for env in "BF_X=0" "BF_WIDE_NT8=0" "BF_WIDE_KT=28" "BF_WIDE_STAGES=3" "BF_WIDE_STAGES=2"; do
  env $env timeout 300 python tools/time_apply.py cfg2 c128 256 5
done
env timeout 300 python tools/time_apply.py cfg2 c128 64 10
env timeout 300 python tools/time_apply.py cfg2 c128 128 10
env BF_WIDE_NT8=0 timeout 300 python tools/time_apply.py cfg2 c128 64 10
