# ncu of the pipe kernel with the IIR math skipped (stencil-only timing study)
TAG=$1
FUSEPLAN_PIPE_SKIP=${2:-1} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_ -c 1 -o gpurun_out/prof_$TAG python scripts/tile_sweep.py 800 600 300 > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --print-source sass --csv > gpurun_out/prof_${TAG}_sass.csv 2>&1
