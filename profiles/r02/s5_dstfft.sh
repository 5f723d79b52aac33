# session 5: padded FFT buffers + twiddle powers in the 2D sine-transform kernels
set -x
timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst" 2>&1 | tail -5
timeout 600 python profiles/r02/dst_probe.py 2 4 2>&1 | grep config
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
for c in 2 4; do
  echo "== config $c"
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
done
