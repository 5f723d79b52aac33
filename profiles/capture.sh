#!/usr/bin/env bash
# Round profiling capture (run on the GPU box from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash profiles/capture.sh r01'
# 1. bench.py must exit 0 without ncu first;
# 2. ncu launch list of the bench command (cold-cache, serialised launches);
# 3. one `ncu --set full` capture each of the stage apply (K2) and the two
#    inner-PCG kernels (config 2), from which profiles/traffic.json is made.
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p "$OUT"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/bench_plain.json" 2> "$OUT/bench_plain.err" || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > "$OUT/launches.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stage_apply_win -s 5 -c 1 \
    -o "$OUT/stage_apply" python profiles/micro_stage.py 2 > "$OUT/ncu_stage.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cg_ -s 40 -c 2 \
    -o "$OUT/pcg" python profiles/micro_pcg.py 2 20 > "$OUT/ncu_pcg.log" 2>&1
# steady-state (no cache flush) per-kernel DRAM traffic of the PCG kernels
ncu --cache-control none --clock-control none -k regex:k_cg_ -s 400 -c 6 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --csv --log-file "$OUT/pcg_steady.csv" python profiles/micro_pcg.py 2 20 > /dev/null 2>&1
echo done
