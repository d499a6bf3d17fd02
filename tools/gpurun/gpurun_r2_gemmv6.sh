# K4 final round-2 ncu capture (--set full): FP8 fwd fp32 / 1x16, gate/up, BF16 dgrad / wgrad on the cfg4 shapes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -f -o gpurun_out/r2/gemm_v6 python tools/gemm_kernels.py > gpurun_out/r2/gemm_v6.log 2>&1; echo "ncu rc=$?"
