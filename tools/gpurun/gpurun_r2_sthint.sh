# K4 FP8 forward epilogue: store cache hints vs plain vs no global stores (diag), ncu tensor pipe + DRAM, then bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for L in "" build_ab/sh1/libcoat.so build_ab/sh2/libcoat.so build_ab/nostg/libcoat.so build_ab/noepi/libcoat.so; do
echo "lib=${L:-default}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k "regex:gemm_kernel<1, 0, 1, 0" --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-200
done
for L in "" build_ab/sh1/libcoat.so build_ab/sh2/libcoat.so "" build_ab/sh1/libcoat.so build_ab/sh2/libcoat.so; do
COAT_LIB=$L timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_sh.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_sh.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('${L:-default}', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f' % l['fwd_vs_cublaslt'], d['clocks']['sm_mhz'])"
done
