# ncu --set full capture of the frame-pair kernel for a library variant
# (FUSEPLAN_LIB) with optional FUSEPLAN_PIPE_SKIP, SASS page exported
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=$1; LIB=$2; SKIP=${3:-0}
FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$LIB FUSEPLAN_PIPE_SKIP=$SKIP timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_pair -c 1 \
  -o gpurun_out/${T} python scripts/tile_sweep.py 800 600 1000 > /dev/null 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page source --print-source sass --csv > gpurun_out/${T}_sass.csv 2>&1
ls -la gpurun_out/${T}*
