set -x
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst" 2>&1 | tail -30
for env in "" "IRK_NO_DST=1"; do
  echo "== config 2 $env"
  env $env timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-workloads | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches']); print(d['inner_solver'])"
  echo "== config 4 $env"
  env $env timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-workloads | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches']); print(d['inner_solver'])"
done
