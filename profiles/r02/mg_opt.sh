timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -q -p no:cacheprovider -k "mg" 2>&1 | tail -2
timeout 300 python profiles/r02/solve_cost_probe.py 2>&1 | tail -1
timeout 300 python profiles/r02/outer_its_probe.py 1e-6 2>&1 | tail -1
