# K4 diag: fp32 output rows aliased onto 256 rows (L2-resident writes) vs the product epilogue
cd $GRAFT_REPO_ROOT
for L in "" build_ab/alias/libcoat.so build_ab/nostg/libcoat.so; do
echo "lib=${L:-default}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_kernel -c 1 --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-120
done
