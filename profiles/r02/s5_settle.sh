# session 5: settling loop condition (a finished solve skips the trailing WHILE pass)
set -x
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst or mg or pcg or forked or schur or cocg" 2>&1 | tail -5
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
for c in 2 4 3; do
  for env in "" "IRK_NO_SETTLE=1"; do
    echo "== config $c $env"
    env $env timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
  done
done
echo "== config 2 IRK_NO_DST=1 (multigrid-PCG)"
IRK_NO_DST=1 timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_stepper.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
