# ncu full capture of the headline pipe kernel with source correlation
# (800x600x1000, one launch): raw metrics, SASS page (per-instruction
# executed counts and stall samples) and CUDA-source page.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_pipe -c 1 \
  -o gpurun_out/np_src python scripts/tile_sweep.py 800 600 1000 > /dev/null 2>&1
ncu -i gpurun_out/np_src.ncu-rep --page raw --csv > gpurun_out/np_src_raw.csv 2>&1
ncu -i gpurun_out/np_src.ncu-rep --page source --print-source sass --csv > gpurun_out/np_src_sass.csv 2>&1
ncu -i gpurun_out/np_src.ncu-rep --page source --print-source cuda --csv > gpurun_out/np_src_cuda.csv 2>&1
ls -la gpurun_out/np_src*
