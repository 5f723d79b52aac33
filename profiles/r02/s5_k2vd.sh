# session 5: K2 on the 15-point 3D stencil, values direct + windows by bulk copies
set -x
for v in "IRK_BULK3=vd" "IRK_BULK3=vd8" ""; do
  echo "== config 3 K2 $v"
  env $v timeout 300 python profiles/micro_stage.py 3 2>&1 | tail -4
done
IRK_BULK3=vd timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "stage or kron or apply or constrained" 2>&1 | tail -3
