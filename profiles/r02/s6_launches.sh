# session 6: launch list of the bench command's timed step at HEAD (eager launches, host FGMRES
# loop: ncu serialises kernels, graphs with conditional nodes are not replayed kernel by kernel)
set -x
OUT=gpurun_out/r02
mkdir -p $OUT
IRK_NO_GRAPH=1 IRK_NO_DEVFGMRES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx \
    --nvtx-include "timed/" --csv --log-file $OUT/launches_s6.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-workloads > $OUT/launches_s6.log 2>&1
python profiles/ncu_launch_summary.py $OUT/launches_s6.csv > $OUT/ncu_launches_bench_summary_s6.txt 2>&1
head -30 $OUT/ncu_launches_bench_summary_s6.txt
gzip -f $OUT/launches_s6.csv
