# Round-2 late evidence (one GPU): the recursion / assemble kernels of the construction after the
# warp-SVD / register-TSQR rework: launch list of one cfg2 block-row + slab recursion, and one
# --set full capture of the recursion and assemble kernels.
set -x
python tools/profile_construct.py cfg2 > gpurun_out/profile_construct_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_construct_cfg2_late.csv python tools/profile_construct.py cfg2 > gpurun_out/ncu_launchlist_construct.log 2>&1
T=/tmp/ncu_one; mkdir -p $T
timeout 900 ncu --set full --clock-control none --import-source on -f -k 'regex:k_recurse|k_assemble' -c 40 -o $T/r02_recursion_late python tools/profile_construct.py cfg2 > gpurun_out/ncu_recursion_late.log 2>&1
ncu -i $T/r02_recursion_late.ncu-rep --page raw --csv > gpurun_out/r02_ncu_recursion_late.csv 2>/dev/null
ncu -i $T/r02_recursion_late.ncu-rep --page source --csv | gzip -c > gpurun_out/r02_ncu_recursion_late.source.csv.gz 2>/dev/null
tail -2 gpurun_out/ncu_recursion_late.log
