# cfg2 256-RHS forward apply: level-major (default) vs node-major slices (BF_NODE_MAJOR=P)
for P in 0 32 64 128 256; do
  BF_NODE_MAJOR=$P timeout 300 python tools/time_apply.py cfg2 c128 256 5
done
for P in 0 64 128; do
  BF_NODE_MAJOR=$P timeout 300 python tools/time_apply.py cfg2 c128 64 10
done
