# gate/up epilogue warps 16 (default) vs 8 with the staged TMA stores
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
COAT_LIB=build_ab/ug8/libcoat.so timeout -s KILL 900 python -m pytest tests/test_gpu_linear.py -q -x -k upgate > gpurun_out/r2/t_ug8.log 2>&1; echo "ug8 tests rc=$?"; tail -1 gpurun_out/r2/t_ug8.log
timeout -s KILL 900 python -m pytest tests/test_gpu_linear.py -q -x -k upgate > gpurun_out/r2/t_ug16.log 2>&1; echo "ug16 tests rc=$?"; tail -1 gpurun_out/r2/t_ug16.log
for L in "" build_ab/ug8/libcoat.so; do
echo "lib=${L:-16}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep "1, 0, 1, 3, 2" | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-100
done
