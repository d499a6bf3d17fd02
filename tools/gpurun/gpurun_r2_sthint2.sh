# K4 FP8 forward epilogue variants under ncu: tensor pipe, DRAM read, clock
cd $GRAFT_REPO_ROOT
for L in "" build_ab/sh1/libcoat.so build_ab/sh2/libcoat.so build_ab/nostg/libcoat.so build_ab/noepi/libcoat.so; do
echo "lib=${L:-default}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_kernel -c 1 --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-200
done
