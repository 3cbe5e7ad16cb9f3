# ncu (full set) of the other kernels: the optimizer plan's F12 / F345 at
# 192x432x600 and the unfused per-stage kernels; raw-page CSVs -> gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_gray_iir_small|k_chain_pipe" -c 2 -o gpurun_out/oth_cfg1 python scripts/bench_configs.py 1 > /dev/null 2>&1
ncu -i gpurun_out/oth_cfg1.ncu-rep --page raw --csv > gpurun_out/oth_cfg1_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_rgba2gray|k_iir|k_gaussian|k_gradient|k_pointwise" -c 5 -o gpurun_out/oth_unf python scripts/tile_sweep_unfused.py > /dev/null 2>&1
ncu -i gpurun_out/oth_unf.ncu-rep --page raw --csv > gpurun_out/oth_unf_raw.csv 2>&1
ls -la gpurun_out/oth_*
