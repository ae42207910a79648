# wide-kernel check: 2-D / many-RHS parity tests, cfg3/cfg4b A/B against BF_NO_WIDE=1, one ncu capture
set -x
timeout 600 python -m pytest tests/test_apply_gpu.py -x -q -m gpu -k "wide or quadtree or many_rhs" > gpurun_out/wide_test.log 2>&1; rc=$?; echo pytest=$rc >> gpurun_out/wide_test.log
for c in cfg3 cfg4b; do
  BF_DEBUG_LAUNCH=1 timeout 300 python bench.py --no-cpu-baseline --no-also --config $c --steps 10 > gpurun_out/wide_$c.json 2> gpurun_out/wide_$c.err
  BF_NO_WIDE=1 timeout 300 python bench.py --no-cpu-baseline --no-also --config $c --steps 10 > gpurun_out/nowide_$c.json 2> gpurun_out/nowide_$c.err
done
if [ $rc = 0 ] && [ "${NCU:-1}" = 1 ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:wide_kernel -s 4 -c 2 -o gpurun_out/wide_cfg4b -f \
    python tools/profile_apply.py cfg4b c128 16 2 > gpurun_out/wide_ncu.log 2>&1
fi
