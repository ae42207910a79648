set -u
run() { python bench.py --no-cpu-baseline --no-also "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
rf=d.get('roofline',{})
print(' '.join(sys.argv[1:]), 'ms', round(d['ms_per_step'],4), 'val %.3e'%d['value'], 'frac', round(rf.get('frac',0),3), rf.get('unit'), 'e2e_ms', round(d['e2e']['ms_per_step'],3))
" "$@"; }
run --config cfg2
run --config cfg2 --dtype c64
run --config cfg2 --rhs 256
run --config cfg1
run --config cfg0
run --config cfg3
run --config cfg4b
run --config cfg2 --sharded
