#!/usr/bin/env bash
# Round profiling capture (run on the GPU box from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash profiles/capture.sh r01'
# 1. bench.py must exit 0 without ncu first;
# 2. ncu launch list of the bench command (cold-cache, serialised launches).
#    Kernels inside graphs with conditional (WHILE) nodes cannot be profiled
#    by ncu, so the list is taken with IRK_NO_GRAPH=1 (same kernels, launched
#    one by one);
# 3. one `ncu --set full` capture each of the stage apply (K2), the fine-level
#    multigrid smoother / residual and the CG kernels (config 2), from which
#    profiles/traffic.json is made.
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p "$OUT"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_plain.json" 2> "$OUT/bench_plain.err" || exit 1
IRK_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > "$OUT/launches.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stage_apply_win -s 5 -c 1 \
    -o "$OUT/stage_apply" python profiles/micro_stage.py 2 > "$OUT/ncu_stage.log" 2>&1
IRK_NO_GRAPH=1 ncu --set full --clock-control none --import-source on \
    -k regex:"k_mg_cheb_st|k_mg_residual_st|k_cg_spmv_st|k_cg_update" -s 200 -c 6 \
    -o "$OUT/mg" python profiles/solve_probe.py 2 > "$OUT/ncu_mg.log" 2>&1
echo done
