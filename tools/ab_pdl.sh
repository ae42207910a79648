run() { python bench.py --no-cpu-baseline --no-also "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(' '.join(sys.argv[1:]), 'ms', round(d['ms_per_step'],4))
" "$@"; }
for i in 1 2; do
BF_NO_PDL=1 run --config cfg1 ; BF_NO_PDL=0 run --config cfg1
BF_NO_PDL=1 run --config cfg2 --rhs 256; BF_NO_PDL=0 run --config cfg2 --rhs 256
BF_NO_PDL=1 run --config cfg3; BF_NO_PDL=0 run --config cfg3
done
