timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 2 2>&1 | tail -1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo 2>&1 | grep '"metric"' | cut -c1-600
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | cut -c1-300
