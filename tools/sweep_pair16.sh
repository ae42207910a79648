timeout 900 python -m pytest tests/test_apply_gpu.py -x -q -m gpu -k "synthetic_geometries or remap_pair or chunked" 2>&1 | tail -4
for env in "BF_NO_PAIR16=1" "BF_X=0" "BF_PAIR16_STAGES=3"; do
  env $env timeout 300 python tools/time_apply.py cfg2 c128 256 5
done
for env in "BF_NO_PAIR16=1" "BF_X=0"; do
  env $env timeout 300 python tools/time_apply.py cfg2 c128 64 10
  env $env timeout 300 python tools/time_apply.py cfg2 c128 128 10
done
