# K4 1x16 epilogue through staging tiles + TMA stores: parity (all GEMM modes), sanitizer epi, ncu + bench vs base
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_linear.py tests/test_gpu_k1_layouts.py tests/test_gpu_sanitizer.py -q -k "linear or q16 or cluster or single_cta or epi" > gpurun_out/r2/t_q16tma.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r2/t_q16tma.log
for L in base ""; do
echo "lib=${L:-new}"
COAT_LIB=${L:+build_ab/$L/libcoat.so} timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep "1, 0, 1, 2, 2" | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-120
done
