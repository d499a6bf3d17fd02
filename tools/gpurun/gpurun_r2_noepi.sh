# K4 diag: FP8 forward with the fp32 epilogue's stores removed (wrong results) vs the product kernel, tensor pipe under ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for L in "" build_ab/noepi/libcoat.so; do
echo "lib=${L:-default}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
done
