set -x
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst3 or mgc or forked or schur" 2>&1 | tail -30
for env in "" "IRK_NO_DST=1"; do
  echo "== config 3 $env"
  env $env timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-workloads 2>gpurun_out/c3.err | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print(d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'])
print(d.get('inner_solver'))"
  tail -3 gpurun_out/c3.err
done
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -x -q -p no:cacheprovider -k "3" 2>&1 | tail -5
