# wide-kernel knob sweep on cfg4b / cfg3 (device ms per apply)
run() { env "$@" timeout 300 python bench.py --no-cpu-baseline --no-also --config $C --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$C', '$*', round(d['ms_per_step'],4), d.get('rel_err',{}).get('value') if isinstance(d.get('rel_err'),dict) else d.get('rel_err'))"; }
for C in cfg4b cfg3; do
run X=0
run BF_WIDE_PROMO=0
run BF_WIDE_PROMO=2
run BF_WIDE_KT=12
run BF_WIDE_KT=28
run BF_WIDE_STAGES=4
done
