# session 5: (1) 3D sine transform with padded FFT buffers / twiddle powers (config 3);
# (2) CUPTI timeline of config 2 / 4 / 3 steps (kernel totals, idle gaps)
set -x
timeout 900 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "dst3 or mgc or schur" 2>&1 | tail -5
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
i=d.get('inner_solver') or {}
print('RESULT', d['value'], d['e2e']['value'], d['krylov_iters_per_step'], d['inner_iters_per_step'], d['gpu_launches'], i.get('us_per_solve'), i.get('iterations_per_solve'))"
}
echo "== config 3"
timeout 600 python bench.py --config 3 --steps 10 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
for c in 2 4 3; do
  timeout 600 python profiles/step_trace.py $c 3 > gpurun_out/trace_c$c.txt 2>&1
  head -50 gpurun_out/trace_c$c.txt
done
rm -f gpurun_out/trace_c*.json
