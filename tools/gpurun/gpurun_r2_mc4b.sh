# K4 pair (C=2) vs two-pair B-multicast cluster (C=4): cfg4 A/B + ncu traffic/clock
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for C in 2 4 2 4; do
COAT_GEMM_CTA=$C timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_c$C.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_c$C.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('C=$C', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib', {k: round(v,1) for k,v in l['tflops'].items()}, 'fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), d['clocks']['sm_mhz'])"
done
for C in 2 4; do
COAT_GEMM_CTA=$C timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none --nvtx --nvtx-include "cmp/" --csv python tools/gemm_vs_library.py > gpurun_out/r2/mc_ncu_c$C.csv 2>/dev/null
echo C=$C
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/r2/mc_ncu_c$C.csv')) if len(r)>10]
h=rows[0]; k=h.index('Kernel Name'); m=h.index('Metric Name'); v=h.index('Metric Value')
for r in rows[1:]:
    if 'decode' in r[k]: continue
    print(r[k][:34].ljust(34), r[m][:45].ljust(45), r[v])
PY
done
