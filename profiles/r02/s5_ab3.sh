# session 5: repeated A/B (3 runs each, alternating) of the boundary-data prefetch (config 3)
set -x
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('RESULT', d['value'], d['e2e']['value'], d['ms_per_step'])"
}
for rep in 1 2 3; do
  for env in "IRK_BC_PREFETCH=1" "IRK_BC_PREFETCH=0"; do
    echo "== config 3 $env rep $rep"
    env $env timeout 600 python bench.py --config 3 --steps 10 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
  done
done
IRK_BC_PREFETCH=0 timeout 300 python profiles/host_step_profile.py 3 5 tottime > gpurun_out/host_c3_nopf.txt 2>&1; head -25 gpurun_out/host_c3_nopf.txt
