timeout 900 python -m pytest tests/test_construct_gpu.py -x -q -m gpu -k "pivot or cluster" 2>&1 | tail -6
for env in "BF_PIVOT_CL2=0" "BF_PIVOT_CL2=1"; do
  echo "== $env"; env $env timeout 600 python tools/bench_construct.py cfg2 --cpu-blocks 1 2>&1 | tail -6
done
