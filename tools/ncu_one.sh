# one --set full capture: tools/ncu_one.sh NAME KERNEL_REGEX SKIP COUNT -- python ... ; exports raw + source csv only
name=$1; regex=$2; skip=$3; count=$4; shift 5
T=/tmp/ncu_one; mkdir -p $T
timeout 900 ncu --set full --clock-control none --import-source on -f -k regex:$regex -s $skip -c $count -o $T/$name "$@" > gpurun_out/ncu_$name.log 2>&1
ncu -i $T/$name.ncu-rep --page raw --csv > gpurun_out/$name.csv 2>/dev/null
ncu -i $T/$name.ncu-rep --page source --csv > gpurun_out/$name.source.csv 2>/dev/null
tail -2 gpurun_out/ncu_$name.log
