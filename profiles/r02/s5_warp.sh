# session 5: warp-per-transform sine-transform kernels at N = 1024 (k_dstw_*)
set -x
timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst" 2>&1 | tail -5
for env in "" "IRK_DST_NOWARP=1"; do
  env $env timeout 300 python profiles/r02/dst_probe.py 2 2>&1 | grep config
done
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
for rep in 1 2; do
for env in "" "IRK_DST_NOWARP=1"; do
  echo "== config 2 $env rep $rep"
  env $env timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
done
done
echo "== config 4"
timeout 600 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -x -q -s -p no:cacheprovider -k "2 or 5 or properties" 2>&1 | grep -v "^$" | tail -6
