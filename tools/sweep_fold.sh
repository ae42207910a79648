timeout 1200 python -m pytest tests/test_apply_gpu.py tests/test_capi.py tests/test_sharded_gpu.py tests/test_storage_gpu.py -x -q -m gpu 2>&1 | tail -4
for env in "BF_NO_FOLD=1" "BF_X=0"; do
  env $env timeout 300 python tools/time_apply.py cfg2 c128 1 50
  env $env timeout 300 python tools/time_apply.py cfg2 c64 1 50
  env $env timeout 300 python tools/time_apply.py cfg2 c128 256 5
  env $env timeout 300 python tools/time_apply.py cfg4b c128 16 10
  env $env timeout 300 python tools/time_apply.py cfg3 c128 16 50
  echo "== $env"; env $env timeout 300 python tools/e2e_probe.py 40 2>&1 | tail -1
done
