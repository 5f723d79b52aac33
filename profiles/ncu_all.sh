#!/usr/bin/env bash
# ncu evidence for EVERY kernel of every workload's time step (north_star:
# "every kernel's choices must be evidenced by ncu").  Run on the GPU box
# from the repo root, after bench.py has exited 0 without ncu:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash profiles/ncu_all.sh r02'
# One timed step per config (NVTX range "timed"), all kernels, launched one by
# one (IRK_NO_GRAPH / IRK_NO_DEVFGMRES: ncu cannot profile kernels inside
# graphs with conditional WHILE nodes; same kernels and arguments), metrics:
# duration, DRAM bytes read/written, L2 hit rate, achieved occupancy,
# registers.  Cold-cache, serialised launches: per-kernel SHARES and DRAM
# bytes are what count, not the absolute step time.
set -u
R=${1:-r02}
OUT=gpurun_out/$R
mkdir -p "$OUT"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size
for k in ${CONFIGS:-1 2 3 4 5}; do
  IRK_NO_GRAPH=1 IRK_NO_DEVFGMRES=1 timeout 1200 ncu --metrics $M --clock-control none --nvtx \
      --nvtx-include "timed/" --csv --log-file "$OUT/all_c$k.csv" \
      python bench.py --config $k --steps 1 --warmup 1 --no-cpu-baseline --no-workloads \
      > "$OUT/all_c$k.log" 2>&1
  echo "config $k rc=$?"
  python profiles/ncu_all_summary.py "$OUT/all_c$k.csv" "config $k, one timed step" \
      > "$OUT/all_c$k.txt" 2>&1
  gzip -f "$OUT/all_c$k.csv"
done
