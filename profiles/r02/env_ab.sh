# A/B of the CG loop-control switches on config 2 (steps 1..20 from u0)
for v in "" "IRK_CG_PREFIX=6" "IRK_CG_PREFIX=8" "IRK_NO_WHILE=1" "IRK_WHILE_BODY=1" "IRK_CG_PREFIX=0"; do
  echo "== $v"
  env $v python profiles/r02/outer_its_probe.py 1e-6 2>&1 | tail -1
done
