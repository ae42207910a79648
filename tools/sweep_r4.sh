# radix-4 chains of the cfg2 / cfg1 sizes (what folding pairs of binary levels would give)
for env in "BF_X=0" "BF_WIDE_MIN_C=64" "BF_NO_FOLD=1"; do
  env $env timeout 300 python tools/time_apply.py cfg2r4 c128 256 5
  env $env timeout 300 python tools/time_apply.py cfg2r4 c128 64 10
done
env timeout 300 python tools/time_apply.py cfg2r4 c128 1 20
env timeout 300 python tools/time_apply.py cfg1r4 c128 64 100
env BF_WIDE_MIN_C=32 timeout 300 python tools/time_apply.py cfg1r4 c128 64 100
