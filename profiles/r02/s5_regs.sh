# session 5: register caps on the half-length transform kernels (before: probe 42.0 / 143.3 us,
# config 2 184.5, config 4 270.7-283 steps/s)
set -x
timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst" 2>&1 | tail -3
timeout 300 python profiles/r02/dst_probe.py 2 4 2>&1 | grep config
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
for rep in 1 2; do
for c in 2 4; do
  echo "== config $c rep $rep"
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
done
done
