# session 5: ncu --set full of the half-length sine-transform kernels (warm L2, as inside a solve)
# and of the CG loop kernels of a config-2 block solve
set -x
OUT=gpurun_out/r02
mkdir -p $OUT
for c in 2 4; do
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
      -k regex:k_dsth_ -s 6 -c 3 -o $OUT/dsth_c${c}_warm python profiles/r02/dst_probe.py $c > $OUT/ncu_dsth_c$c.log 2>&1
  python profiles/ncu_summary.py $OUT/dsth_c${c}_warm.ncu-rep > $OUT/ncu_full_dsth_c${c}_warm.txt 2>&1
  cat $OUT/ncu_full_dsth_c${c}_warm.txt
  rm -f $OUT/dsth_c${c}_warm.ncu-rep
done
IRK_NO_GRAPH=1 timeout 600 ncu --set full --cache-control none --clock-control none \
    -k regex:"k_cg_spmv_st|k_cg_update|k_cg_init_ext|k_cg_store" -s 20 -c 8 \
    -o $OUT/cg_warm python profiles/solve_probe.py 2 > $OUT/ncu_cg_warm.log 2>&1
python profiles/ncu_summary.py $OUT/cg_warm.ncu-rep > $OUT/ncu_full_cg_warm.txt 2>&1
cat $OUT/ncu_full_cg_warm.txt
rm -f $OUT/cg_warm.ncu-rep
