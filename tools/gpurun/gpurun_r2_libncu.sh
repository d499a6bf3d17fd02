# ncu --set full of K4 next to the cuBLAS / cuBLASLt kernels on the cfg4 shapes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "cmp/" -f -o gpurun_out/r2/gemm_vs_lib python tools/gemm_vs_library.py > gpurun_out/r2/gemm_vs_lib.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/r2/gemm_vs_lib.log
ncu -i gpurun_out/r2/gemm_vs_lib.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,lts__t_bytes.sum,dram__bytes_read.sum 2>&1 | cut -c1-600 | head -20
