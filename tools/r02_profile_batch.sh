# Round-2 ncu batch (one GPU): --set full captures of the dominant kernel of each
# many-RHS workload and of one cfg2 construction block-row. The reports stay on the box
# (/tmp); only the raw and source page exports come back under gpurun_out/.
set -x
N="ncu --set full --clock-control none --import-source on -f"
T=/tmp/ncu_r02; mkdir -p $T
timeout 900 $N -k regex:level_kernel -s 6 -c 2 -o $T/r02_cfg2_k256 python tools/profile_apply.py cfg2 c128 256 2 > gpurun_out/ncu_cfg2_k256.log 2>&1
BF_CHUNK_PAIR=1 timeout 900 $N -k regex:pair_chunk -s 2 -c 2 -o $T/r02_cfg2_k256_chunkpair python tools/profile_apply.py cfg2 c128 256 2 > gpurun_out/ncu_cfg2_k256_cp.log 2>&1
timeout 600 $N -k regex:pair_kernel -s 2 -c 2 -o $T/r02_cfg1_k64 python tools/profile_apply.py cfg1 c128 64 2 > gpurun_out/ncu_cfg1_k64.log 2>&1
timeout 600 $N -k regex:wide_kernel -s 4 -c 2 -o $T/r02_cfg4b_k16 python tools/profile_apply.py cfg4b c128 16 2 > gpurun_out/ncu_cfg4b.log 2>&1
timeout 1200 $N -k regex:k_ -c 60 -o $T/r02_construct_cfg2 python tools/profile_construct.py cfg2 > gpurun_out/ncu_construct.log 2>&1
for f in r02_cfg2_k256 r02_cfg2_k256_chunkpair r02_cfg1_k64 r02_cfg4b_k16 r02_construct_cfg2; do
  ncu -i $T/$f.ncu-rep --page raw --csv > gpurun_out/$f.csv 2>/dev/null
done
for f in r02_cfg2_k256 r02_cfg2_k256_chunkpair r02_cfg1_k64 r02_cfg4b_k16; do
  ncu -i $T/$f.ncu-rep --page source --csv --launch-skip 0 --launch-count 1 > gpurun_out/$f.source.csv 2>/dev/null
done
ncu -i $T/r02_construct_cfg2.ncu-rep --page source --csv > $T/construct.source.csv 2>/dev/null
gzip -c $T/construct.source.csv > gpurun_out/r02_construct_cfg2.source.csv.gz
ls -la $T gpurun_out; du -sh gpurun_out
