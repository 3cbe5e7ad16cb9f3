timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 2 2>&1 | tail -1
