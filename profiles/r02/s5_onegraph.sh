# session 5: one graph per deferred solve (init / log / store inside, arguments updated per replay)
set -x
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_stepper.py -m gpu -x -q -p no:cacheprovider -k "dst or mg or pcg or forked or schur or cocg or defer or stepper or dirk" 2>&1 | tail -5
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
for c in 2 3 4; do
for env in "" "IRK_NO_ONEGRAPH=1"; do
  echo "== config $c $env"
  env $env timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
  tail -2 gpurun_out/c.err
done
done
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -x -q -s -p no:cacheprovider 2>&1 | grep -v "^$" | tail -8
