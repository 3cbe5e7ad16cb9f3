# one ncu --set full capture (source correlated) of the frame-pair kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_pair -c 1 \
  -o gpurun_out/${1:-pair_src} python scripts/tile_sweep.py 800 600 1000 > /dev/null 2>&1
ncu -i gpurun_out/${1:-pair_src}.ncu-rep --page raw --csv > gpurun_out/${1:-pair_src}_raw.csv 2>&1
ls -la gpurun_out/${1:-pair_src}*
