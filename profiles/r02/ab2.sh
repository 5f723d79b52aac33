for v in "" "IRK_SPLIT_WHILE=1"; do
  echo "== $v"
  env $v timeout 300 python profiles/r02/outer_its_probe.py 1e-6 2>&1 | tail -1
done
timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -x -q -k "mg or pcg or cg" 2>&1 | tail -3
