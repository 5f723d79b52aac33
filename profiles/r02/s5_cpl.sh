# session 5: Gauss-Seidel coupling by bulk tiles (k_stage_couple_bulk) vs per-row gathers
set -x
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_stepper.py -m gpu -x -q -p no:cacheprovider -k "couple or precond or pc or gs or lower or upper or rana or kinds or stepper" 2>&1 | tail -4
run() {
  python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('RESULT', d['value'], d['e2e']['value'], d['ms_per_step'], d['krylov_iters_per_step'])"
}
for rep in 1 2; do
for env in "" "IRK_NO_CPLBULK=1"; do
  echo "== config 2 $env rep $rep"
  env $env timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-workloads 2>gpurun_out/c.err | run
done
done
timeout 600 python -m pytest tests/test_gpu_full.py -m gpu -x -q -s -p no:cacheprovider -k "2" 2>&1 | grep -v "^$" | tail -4
IRK_NO_GRAPH=1 IRK_NO_DEVFGMRES=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_stage_couple -c 6 --csv --log-file gpurun_out/cpl.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-workloads > gpurun_out/cpl.log 2>&1
grep "k_stage_couple" gpurun_out/cpl.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | head -20
