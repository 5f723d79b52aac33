# session 5: sine-transform CG with the skip decision and r.z fused into the
# row-transform kernels and 2 (not 4) straight-line iterations in the init graph
set -x
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst or mg or pcg or forked or schur" 2>&1 | tail -5
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
for c in 2 4 3; do
  for env in "" "IRK_CG_NOFUSE=1" "IRK_CG_PREFIX=4"; do
    echo "== config $c $env"
    env $env timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
  done
done
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
