# Time one bench configuration under several environment settings.
# usage: tools/sweep_env.sh "<bench args>" "ENV=.. ENV=.." "ENV=.." ...   ("-" = no overrides)
set -u
args=$1; shift
for e in "$@"; do
  [ "$e" = "-" ] && e=""
  env $e python bench.py --no-cpu-baseline --no-also --steps 5 --warmup 3 $args 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%-60s ms %8.4f  val %.3e  e2e_ms %.3f' % (sys.argv[1] or 'default', d['ms_per_step'], d['value'], d['e2e']['ms_per_step']))
" "$e" || echo "$e FAILED"
done
