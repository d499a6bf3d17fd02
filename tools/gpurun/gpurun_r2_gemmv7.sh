# K4 end-of-round ncu capture (--set full) after the staged TMA-store epilogues and the snake raster
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -f -o gpurun_out/r2/gemm_v7 python tools/gemm_kernels.py > gpurun_out/r2/gemm_v7.log 2>&1; echo "ncu rc=$?"
