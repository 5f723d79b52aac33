# session 5: FGMRES normalisation from the device scalar, enqueued before the host read of h
set -x
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_stepper.py -m gpu -x -q -p no:cacheprovider -k "fgmres or gmres or krylov or stepper or precond" 2>&1 | tail -4
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('RESULT', d['value'], d['e2e']['value'], d['ms_per_step'], d['krylov_iters_per_step'])"
}
for c in 2 3 5; do
  echo "== config $c"
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
done
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -x -q -s -p no:cacheprovider 2>&1 | grep -v "^$" | tail -8
