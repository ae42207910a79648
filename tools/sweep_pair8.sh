# cfg1 64-RHS apply: the rank-8 fast pair kernel and its alternatives
timeout 900 python -m pytest tests/test_apply_gpu.py -x -q -m gpu -k "rank8 or synthetic_geometries or remap_pair or adjoint or golden" > gpurun_out/pair8_test.log 2>&1; echo pytest=$? >> gpurun_out/pair8_test.log
tail -15 gpurun_out/pair8_test.log
for env in "BF_NO_PAIR8=1" "BF_NO_PAIR8_LEAF=1" "BF_X=0" "BF_PAIR8_STAGES=1" "BF_PAIR_KC=64"; do
  env $env timeout 300 python tools/time_apply.py cfg1 c128 64 200
done
env timeout 300 python tools/time_apply.py cfg1 c128 128 100; env timeout 300 python tools/time_apply.py cfg1 c128 256 50; env BF_NO_PAIR8=1 timeout 300 python tools/time_apply.py cfg1 c128 256 50
env BF_NO_PAIR8=1 timeout 300 python tools/time_apply.py cfg1 c128 128 100
