# session 5, final: ncu --set full of the default config-2 K2 kernel, launch list of the
# bench command (timed step), then tests + bench + reference arm as the driver runs them
set -x
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 300 python profiles/micro_stage.py 2 > $OUT/micro_stage_c2.txt 2>&1; cat $OUT/micro_stage_c2.txt
timeout 300 python profiles/micro_stage.py 3 > $OUT/micro_stage_c3.txt 2>&1
timeout 300 python profiles/r02/dst_probe.py 2 4 > $OUT/dst_probe.txt 2>&1; cat $OUT/dst_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_apply -s 5 -c 1 \
    -o $OUT/stage_apply_c2_vd python profiles/micro_stage.py 2 > $OUT/ncu_stage_c2_vd.log 2>&1
python profiles/ncu_summary.py $OUT/stage_apply_c2_vd.ncu-rep > $OUT/ncu_full_stage_apply_c2_vd.txt 2>&1
cat $OUT/ncu_full_stage_apply_c2_vd.txt
ncu -i $OUT/stage_apply_c2_vd.ncu-rep --page details 2>/dev/null | grep -v "^\s*$" | head -150 > $OUT/ncu_details_stage_apply_c2_vd.txt
rm -f $OUT/stage_apply_c2_vd.ncu-rep
bash profiles/r02/run_tests_bench.sh
IRK_NO_GRAPH=1 IRK_NO_DEVFGMRES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx \
    --nvtx-include "timed/" --csv --log-file $OUT/launches_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-workloads > $OUT/launches_final.log 2>&1
python profiles/ncu_launch_summary.py $OUT/launches_final.csv > $OUT/ncu_launches_bench_summary.txt 2>&1
head -30 $OUT/ncu_launches_bench_summary.txt
gzip -f $OUT/launches_final.csv
