# K4 grouped raster with alternating N direction (snake) vs plain
cd $GRAFT_REPO_ROOT
for L in "" build_ab/snake/libcoat.so; do
echo "lib=${L:-plain}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, EpiMaps, Params)//' | cut -c1-100
done
for i in 1 2; do for L in "" build_ab/snake/libcoat.so; do
COAT_LIB=$L timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/bench_snake.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_snake.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('${L:-plain}', {k: round(v,1) for k,v in d['tflops'].items()}, 'dgrad/cublas %.3f' % l['dgrad_vs_cublas'], d['clocks']['sm_mhz'])"
done; done
