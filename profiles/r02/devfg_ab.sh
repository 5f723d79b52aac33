# device-resident FGMRES cycles vs the host Givens loop (config 1), plus the GPU tests
for v in "" "IRK_NO_DEVFGMRES=1"; do
  echo "== $v"
  env $v CFG=1 timeout 300 python profiles/r02/outer_its_probe.py 1e-6 2>&1 | tail -2
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
