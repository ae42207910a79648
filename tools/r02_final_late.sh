# Round-2 closing evidence after the recursion / assemble rework (one GPU): smoke, the GPU suite,
# the default bench line, the reference arm, and ncu evidence of the recursion kernels on an
# 8-slab cfg2 batch (launch list + one --set full capture).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; tail -2 gpurun_out/r02_smoke.log
python -m pytest tests -x -q -m gpu > gpurun_out/r02_gputest_final.log 2>&1; tail -2 gpurun_out/r02_gputest_final.log
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/r02_bench_default.json
python bench.py --impl reference > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/r02_bench_reference_arm.json
python tools/time_recurse.py 8 > gpurun_out/r02_time_recurse_8slabs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_recursion_8slabs.csv python tools/time_recurse.py 8 > /dev/null 2>&1
T=/tmp/ncu_one; mkdir -p $T
timeout 900 ncu --set full --clock-control none --import-source on -f -k 'regex:k_recurse' -c 9 -o $T/r02_recursion_8slabs python tools/time_recurse.py 8 > gpurun_out/ncu_recursion_8slabs.log 2>&1
ncu -i $T/r02_recursion_8slabs.ncu-rep --page raw --csv > gpurun_out/r02_ncu_recursion_8slabs.csv 2>/dev/null
ncu -i $T/r02_recursion_8slabs.ncu-rep --page source --csv | gzip -c > gpurun_out/r02_ncu_recursion_8slabs.source.csv.gz 2>/dev/null
tail -2 gpurun_out/ncu_recursion_8slabs.log
