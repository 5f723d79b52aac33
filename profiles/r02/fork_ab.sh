# forked (concurrent) independent pair/block solves vs one by one; e2e without the CPU jobs
set -x
timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "forked or schur or mgc or mg_pcg" 2>&1 | tail -5
for env in "" "IRK_NO_FORK=1"; do
  echo "== config 3 $env"
  env $env timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-workloads | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['gpu_launches'])"
done
echo "== config 2 no cpu jobs"
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-workloads | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e']['value'], d['krylov_iters_per_step'])"
