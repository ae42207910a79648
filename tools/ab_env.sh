# A/B of one environment switch on the many-RHS configs: tools/ab_env.sh VAR [configs...]
set -u
var=$1; shift
run() { python bench.py --no-cpu-baseline --no-also "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
rf=d.get('roofline',{})
print(' '.join(sys.argv[1:]), 'ms', round(d['ms_per_step'],4), 'val %.3e'%d['value'], 'frac', round(rf.get('frac',0),3), rf.get('unit'), 'e2e_ms', round(d['e2e']['ms_per_step'],3))
" "$@"; }
for c in "--config cfg2 --rhs 256" "--config cfg1" "--config cfg3" "--config cfg4b"; do
  env $var=1 bash -c "$(declare -f run); run $c"; echo "  ($var=1)"
  run $c; echo "  (default)"
done
