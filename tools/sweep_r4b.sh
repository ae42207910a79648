timeout 1200 python -m pytest tests/test_apply_gpu.py tests/test_fullsize_gpu.py tests/test_sharded_gpu.py tests/test_capi.py -x -q -m gpu 2>&1 | tail -5
for env in "BF_NO_RADIX4=1" "BF_X=0"; do
  env $env timeout 300 python tools/time_apply.py cfg2 c128 256 5
  env $env timeout 300 python tools/time_apply.py cfg2 c128 64 10
  env $env timeout 300 python tools/time_apply.py cfg2 c128 16 10
  env $env timeout 300 python tools/time_apply.py cfg2 c128 8 10
done
