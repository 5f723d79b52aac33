# session 5: boundary-data prefetch (config 3), r prefetch in the inverse row
# transform (configs 2, 4), host-side profiles of configs 2 and 3
set -x
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_stepper.py -m gpu -x -q -p no:cacheprovider -k "dst or bc or dae or ode or config3 or dirichlet or stepper" 2>&1 | tail -5
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
for env in "" "IRK_BC_PREFETCH=0"; do
  echo "== config 3 $env"
  env $env timeout 600 python bench.py --config 3 --steps 10 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
done
for c in 2 4; do
  for env in "" "IRK_DST_FULL=1"; do
    echo "== config $c $env"
    env $env timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
  done
done
timeout 300 python profiles/r02/dst_probe.py 2 4 2>&1 | grep config
IRK_DST_FULL=1 timeout 300 python profiles/r02/dst_probe.py 2 4 2>&1 | grep config
timeout 300 python profiles/host_step_profile.py 2 5 tottime > gpurun_out/host_c2.txt 2>&1; head -45 gpurun_out/host_c2.txt
timeout 300 python profiles/host_step_profile.py 3 5 tottime > gpurun_out/host_c3.txt 2>&1; head -45 gpurun_out/host_c3.txt
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -x -q -s -p no:cacheprovider 2>&1 | grep -v "^$" | tail -12
