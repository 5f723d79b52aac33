# session 6: device-resident FGMRES cycles over captured sine-transform block solves
# (fixed straight-line CG iterations): new test, then config 2 A/B x2, then the whole suite
set -x
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -x -q -p no:cacheprovider -k "captured_dst or device_cycle" 2>&1 | tail -30
for rep in 1 2; do
  for v in on off; do
    if [ $v = off ]; then export IRK_NO_DEVFG_DST=1; else unset IRK_NO_DEVFG_DST; fi
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-workloads > $OUT/devfgdst_${v}_$rep.json 2> $OUT/devfgdst_${v}_$rep.err
    echo "devfg_dst=$v rep=$rep rc=$?"
    python - <<P
import json
d=json.loads(open("$OUT/devfgdst_${v}_$rep.json").read().strip().splitlines()[-1])
print("$v", d["value"], d["e2e"]["value"], d["krylov_iters_per_step"], d["inner_iters_per_step"], d["gpu_launches"])
P
  done
done
unset IRK_NO_DEVFG_DST
bash profiles/r02/run_tests_bench.sh
