# K4 gate/up epilogue diag: code / scale stores removed (wrong results) vs product
cd $GRAFT_REPO_ROOT
for L in "" build_ab/ugnostg/libcoat.so; do
echo "lib=${L:-default}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep "1, 0, 1, 3, 2" | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-120
done
