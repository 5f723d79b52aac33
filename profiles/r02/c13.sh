timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
for c in 1 3; do CFG=$c timeout 300 python profiles/r02/outer_its_probe.py 1e-6 2>&1 | tail -1; done
