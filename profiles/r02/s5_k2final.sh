# session 5: K2 values-direct on the 2D stencils (A/B), ncu --set full of the new 3D default,
# parity tests of the stage apply, configs 3 and 5 end to end
set -x
OUT=gpurun_out/r02
mkdir -p $OUT
for c in 2 4 1; do
for v in "" "IRK_BULK2=vd"; do
  echo "== config $c K2 $v"
  env $v timeout 300 python profiles/micro_stage.py $c 2>&1 | tail -4
done
done
timeout 300 python profiles/micro_stage.py 3 > $OUT/micro_stage_c3.txt 2>&1; cat $OUT/micro_stage_c3.txt
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "stage or kron or apply or constrained" 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_apply -s 5 -c 1 \
    -o $OUT/stage_apply_c3_vd python profiles/micro_stage.py 3 > $OUT/ncu_stage_c3_vd.log 2>&1
python profiles/ncu_summary.py $OUT/stage_apply_c3_vd.ncu-rep > $OUT/ncu_full_stage_apply_c3_vd.txt 2>&1
cat $OUT/ncu_full_stage_apply_c3_vd.txt
rm -f $OUT/stage_apply_c3_vd.ncu-rep
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('RESULT', d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['frac'])"
}
echo "== config 3"
timeout 600 python bench.py --config 3 --steps 10 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
