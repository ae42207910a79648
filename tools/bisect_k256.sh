# time cfg2 k=256 and cfg1 (device) for each worktree given as arguments
for d in "$@"; do
  for c in "--config cfg2 --rhs 256" "--config cfg1"; do
    (cd $d && python bench.py --no-cpu-baseline --no-also $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', '$c', round(d['ms_per_step'],4))")
  done
done
