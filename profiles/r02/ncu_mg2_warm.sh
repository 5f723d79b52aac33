# ncu --set full of one structured V-cycle's kernels (config 2 block 0) with a
# WARM L2 (--cache-control none: the in-solve working set is L2-resident),
# pipelined top post-smoother and the one-tile-per-CTA variant.
mkdir -p gpurun_out/r02
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
  -k regex:"k_mg2_" -s 60 -c 11 -o gpurun_out/r02/mg2_warm python profiles/vcycle_probe.py 2 ncu > gpurun_out/r02/ncu_mg2_warm.log 2>&1
IRK_MG_NOPIPE=1 timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
  -k regex:"k_mg2_post" -s 30 -c 5 -o gpurun_out/r02/mg2_warm_nopipe python profiles/vcycle_probe.py 2 ncu > gpurun_out/r02/ncu_mg2_warm_nopipe.log 2>&1
ls -la gpurun_out/r02
