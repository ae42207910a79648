for kt in 12 20 28 36 16 32; do
  BF_WIDE_KT=$kt timeout 300 python tools/time_apply.py cfg2 c128 256 5
done
for st in 4 6; do
  BF_WIDE_STAGES=$st timeout 300 python tools/time_apply.py cfg2 c128 256 5
done
BF_WIDE_PROMO=2 timeout 300 python tools/time_apply.py cfg2 c128 256 5
