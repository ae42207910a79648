for env in "BF_X=0" "BF_PIPE_STREAMS=2" "BF_PIPE_STREAMS=2 BF_PIPE_TAPER=16"; do
  echo "== $env"; env $env timeout 300 python tools/e2e_probe.py 60 2>&1 | tail -1
done
BF_PIPE_STREAMS=2 timeout 600 python -m pytest tests -x -q -m gpu -k "host" 2>&1 | tail -2
