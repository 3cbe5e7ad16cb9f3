timeout 120 python scripts/repro_fast.py 64 48 4
timeout 120 python scripts/repro_fast.py 800 600 10
bash scripts/gpu_check.sh
