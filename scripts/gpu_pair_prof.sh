# Pipe-rate microbenchmark + one ncu --set full capture of the frame-pair
# kernel (800x600x1000) with the SASS source page (per-instruction executed
# counts and stall samples), for scripts/ncu_pair_roles.py.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${1:-pair}
if [ -x scripts/micro/pipe_rates ]; then timeout 120 scripts/micro/pipe_rates > gpurun_out/pipe_rates.txt 2>&1; fi
timeout 120 python scripts/tile_sweep.py 800 600 1000 > gpurun_out/${T}_time.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_pair -c 1 \
  -o gpurun_out/${T} python scripts/tile_sweep.py 800 600 1000 > /dev/null 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page source --print-source sass --csv > gpurun_out/${T}_sass.csv 2>&1
ls -la gpurun_out/${T}*
