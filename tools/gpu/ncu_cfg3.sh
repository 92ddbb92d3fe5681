# ncu --set full of the cfg3 generic d=3 wide-row kernels (one launch each), for the summary in profiles/.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_srun3|k_pairwalk3|k_head_bwd|k_head_fwd|k_segsum3|k_pool_rows" -s 12 -c 7 -o gpurun_out/cfg3_full python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg3.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_cfg3.log
