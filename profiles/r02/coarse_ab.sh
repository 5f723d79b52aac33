for b in '{}' '{"mg_coarse_ratio": 2.0, "mg_coarse_steps": 8}' '{"mg_coarse_ratio": 2.0, "mg_coarse_steps": 12}' '{"mg_coarse_ratio": 2.0, "mg_coarse_steps": 16}' '{"mg_coarse_ratio": 2.0, "mg_coarse_steps": 24}'; do
  BLOCK="$b" timeout 300 python profiles/r02/outer_its_probe.py 1e-6 2>&1 | tail -1
done
