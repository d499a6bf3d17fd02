# round-2 final ncu evidence: K1 (--set full, 500M params), the default bench's launch list,
# the GEMM family incl. the quantizing epilogues, the MGAQ kernels on one 8192x11008 tensor
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_ws_kernel -c 1 -o gpurun_out/r2/k1_v26 python bench.py --params 499998976 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > /dev/null 2>&1; echo "k1 ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/bench_7b_launches_r02.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r2/bench_under_ncu.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:gemm_kernel -c 5 -o gpurun_out/r2/gemm_v3 python tools/gemm_kernels.py > /dev/null 2>&1; echo "gemm ncu rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"quant_group_kernel|group_amax_kernel|quant_tensor_kernel" -c 3 -o gpurun_out/r2/mgaq_v3 python tools/mgaq_kernels.py > /dev/null 2>&1; echo "mgaq ncu rc=$?"
ls -la gpurun_out/r2/*.ncu-rep
