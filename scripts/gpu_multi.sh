# N > 1 bench path on ONE GPU: two / four ranks share cuda:0 over gloo (timing
# meaningless; checks the sharded step, e2e, max-over-ranks and the JSON line)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 3 --warmup 3 --dist-backend gloo > gpurun_out/multi_$n.json 2> gpurun_out/multi_$n.err
tail -c 1500 gpurun_out/multi_$n.json; tail -3 gpurun_out/multi_$n.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --scaling strong | tail -c 600
