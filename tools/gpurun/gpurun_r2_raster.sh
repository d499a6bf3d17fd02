# grouped tile raster for K4: parity (default group and a ragged group of 3) + cfg4 per group size + ncu DRAM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_linear_raster.log 2>&1; echo "linear tests rc=$?"; tail -2 gpurun_out/r2/t_linear_raster.log
COAT_GEMM_GROUP_M=3 timeout 900 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_linear_raster3.log 2>&1; echo "linear tests g3 rc=$?"; tail -2 gpurun_out/r2/t_linear_raster3.log
for G in 0 4 8 16 8 0; do
COAT_GEMM_GROUP_M=$G timeout 600 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_g$G.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_g$G.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('G=$G', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib', {k: round(v,1) for k,v in l['tflops'].items()}, 'fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), 'upgate', round(d['mlp_upgate']['fused_ms'],4), d['clocks']['sm_mhz'])"
done
for G in 0 8; do
COAT_GEMM_GROUP_M=$G timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none --nvtx --nvtx-include "cmp/" --csv python tools/gemm_vs_library.py 2>/dev/null | grep -v "^==" | cut -c1-400 | awk -F'","' '{print $7, $(NF-2), $(NF-1), $NF}' | tail -20 > gpurun_out/r2/raster_dram_g$G.txt
echo G=$G; cat gpurun_out/r2/raster_dram_g$G.txt
done
