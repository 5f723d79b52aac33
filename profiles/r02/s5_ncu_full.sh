# session 5: ncu --set full captures of the round's top kernels, then the
# every-kernel lists of configs 1, 3, 5 (2 and 4 were taken earlier).
# Each profiled command has exited 0 without ncu before (tests / bench above).
set -x
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 300 python profiles/micro_stage.py 2 > $OUT/micro_stage_c2.txt 2>&1
timeout 300 python profiles/micro_stage.py 3 > $OUT/micro_stage_c3.txt 2>&1
timeout 300 python profiles/r02/dst_probe.py 2 4 > $OUT/dst_probe.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_apply -s 5 -c 1 \
    -o $OUT/stage_apply_bulk python profiles/micro_stage.py 2 > $OUT/ncu_stage.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_apply -s 5 -c 1 \
    -o $OUT/stage_apply_c3 python profiles/micro_stage.py 3 > $OUT/ncu_stage_c3.log 2>&1
# the sine-transform kernels inside a solve have a warm L2: --cache-control none
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:k_dst_ -s 6 -c 3 -o $OUT/dst2_warm python profiles/r02/dst_probe.py 2 > $OUT/ncu_dst2.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:k_dst_ -s 6 -c 3 -o $OUT/dst2_c4_warm python profiles/r02/dst_probe.py 4 > $OUT/ncu_dst2_c4.log 2>&1
for r in stage_apply_bulk stage_apply_c3 dst2_warm dst2_c4_warm; do
  [ -f "$OUT/$r.ncu-rep" ] && python profiles/ncu_summary.py "$OUT/$r.ncu-rep" > "$OUT/ncu_full_$r.txt" 2>&1
done
ls -la $OUT
CONFIGS="1 3 5" bash profiles/ncu_all.sh r02
rm -f $OUT/dst2_c4_warm.ncu-rep
# K2 on the 3D stencil: 3-stage bulk ring vs per-warp copies
for v in "" "IRK_BULK3_KT=6" "IRK_NO_BULK3=1"; do
  echo "== config 3 K2 $v"
  env $v timeout 300 python profiles/micro_stage.py 3 2>&1 | tail -4
done
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "stage or kron or apply or constrained" 2>&1 | tail -3
timeout 3000 python -m pytest tests/test_reference_suite.py -m gpu -x -q -s -p no:cacheprovider > $OUT/reference_suite.txt 2>&1
tail -15 $OUT/reference_suite.txt
