# K4 TMA-store epilogue paced over the first s/8 of the next main loop: sweep s
cd $GRAFT_REPO_ROOT
for P in 0 1 2 4; do
echo "spread=$P"
COAT_GEMM_EPI_PACE=$P COAT_LIB=build_ab/tst/libcoat.so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, Params)//' | cut -c1-120
done
