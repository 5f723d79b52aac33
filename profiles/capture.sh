#!/usr/bin/env bash
# Round profiling capture (run on the GPU box from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash profiles/capture.sh r01'
# 1. bench.py must exit 0 without ncu first (all five configs);
# 2. ncu launch list of the bench command (cold-cache, serialised launches).
#    Kernels inside graphs with conditional (WHILE) nodes cannot be profiled
#    by ncu, so the list is taken with IRK_NO_GRAPH=1 (same kernels, launched
#    one by one);
# 3. `ncu --set full` captures of the stage apply (K2, config 2 and 3), one
#    structured V-cycle (k_mg2_*) and the CG-loop kernels, from which
#    profiles/traffic.json is made.
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p "$OUT"
python bench.py > "$OUT/bench_config2.json" 2> "$OUT/bench.err" || exit 1
for k in 1 3 4 5; do
  python bench.py --config $k --steps 5 --no-cpu-baseline > "$OUT/bench_config$k.json" 2>> "$OUT/bench.err"
done
IRK_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx \
    --nvtx-include "timed/" --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/launches.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stage_apply -s 5 -c 1 \
    -o "$OUT/stage_apply" python profiles/micro_stage.py 2 > "$OUT/ncu_stage.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stage_apply -s 5 -c 1 \
    -o "$OUT/stage_apply_c3" python profiles/micro_stage.py 3 > "$OUT/ncu_stage_c3.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_mg2_" -s 60 -c 11 \
    -o "$OUT/mg2" python profiles/vcycle_probe.py 2 ncu > "$OUT/ncu_mg2.log" 2>&1
IRK_NO_GRAPH=1 ncu --set full --clock-control none \
    -k regex:"k_cg_spmv|k_cg_update|k_cg_skip|k_cg_dot_rz" -s 40 -c 8 \
    -o "$OUT/cg" python profiles/solve_probe.py 2 > "$OUT/ncu_cg.log" 2>&1

# config 3: complex multigrid-COCG kernels (Schur pairs) and the GS coupling of config 2
IRK_NO_GRAPH=1 ncu --set full --clock-control none -k regex:"k_mg3_|k_mgc_cheb|k_cg_spmv_stn" \
    -s 30 -c 12 -o "$OUT/mgc" python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline \
    > "$OUT/ncu_mgc.log" 2>&1
ncu --set full --clock-control none -k regex:"k_stage_couple" -s 6 -c 2 \
    -o "$OUT/couple" python bench.py --steps 1 --warmup 1 --no-cpu-baseline > "$OUT/ncu_couple.log" 2>&1

# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back)
for r in stage_apply stage_apply_c3 mg2 cg mgc couple; do
  [ -f "$OUT/$r.ncu-rep" ] && python profiles/ncu_summary.py "$OUT/$r.ncu-rep" > "$OUT/$r.txt" 2>&1
done
python profiles/ncu_launch_summary.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
rm -f "$OUT"/*.ncu-rep
echo done3
