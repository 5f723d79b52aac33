# session 5: (1) K2 on the 3D 15-point stencil by bulk-asynchronous tiles with
# rotated (bank-conflict-free) stage reads vs the per-warp copies; (2) parity
# tests of the stage apply; (3) the every-kernel ncu list of configs 2 and 4.
set -x
for v in "" "IRK_BULK3_KT=6" "IRK_NO_BULK3=1"; do
  echo "== config 3 $v"
  env $v timeout 300 python profiles/micro_stage.py 3 2>&1 | tail -4
done
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "stage or kron or apply or constrained" 2>&1 | tail -5
CONFIGS="2 4" bash profiles/ncu_all.sh r02
cat gpurun_out/r02/all_c2.txt | head -60
