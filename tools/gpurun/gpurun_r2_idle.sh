# K4 long waits (producer on a full ring, epilogue through the main loop): spin vs nanosleep backoff
cd $GRAFT_REPO_ROOT
for L in "" build_ab/idle64/libcoat.so build_ab/idle256/libcoat.so; do
echo "lib=${L:-spin}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep -E "1, 0, 1, 0, 2|0, 0, 0, 1, 2" | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, EpiMaps, Params)//' | cut -c1-110
done
for i in 1 2; do for L in "" build_ab/idle64/libcoat.so build_ab/idle256/libcoat.so; do
COAT_LIB=$L timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/bench_idle.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_idle.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('${L:-spin}', {k: round(v,1) for k,v in d['tflops'].items()}, 'fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), 'ug x%.3f' % d['mlp_upgate']['speedup'], d['clocks']['sm_mhz'])"
done; done
