# Round-2 final evidence (one GPU): launch list of the headline command, --set full captures of
# the headline level kernel, the rank-8 pair kernel and the 256-RHS level kernel.
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg2_c128_k1.csv python bench.py --no-also --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/ncu_launchlist.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_cfg1_c128_k64.csv python tools/profile_apply.py cfg1 c128 64 3 > gpurun_out/ncu_launchlist_cfg1.log 2>&1
bash tools/ncu_one.sh r02_final_cfg2_k1 level_kernel 16 4 -- python tools/profile_apply.py cfg2 c128 1 3
bash tools/ncu_one.sh r02_final_cfg1_k64 pair8_kernel 6 6 -- python tools/profile_apply.py cfg1 c128 64 3
bash tools/ncu_one.sh r02_final_cfg2_k256 level_kernel 16 3 -- python tools/profile_apply.py cfg2 c128 256 2
gzip -f gpurun_out/r02_final_*.source.csv
ls -la gpurun_out | tail -20
