for env in "BF_PIPE_TAPER=0" "BF_PIPE_TAPER=4" "BF_PIPE_TAPER=8" "BF_PIPE_TAPER=16" "BF_PIPE_TAPER=32"; do
  echo "== $env"; env $env timeout 300 python tools/e2e_probe.py 60 2>&1 | tail -1
done
