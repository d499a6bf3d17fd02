cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear2.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear2.json').read().strip().splitlines()[-1]); r=d['roofline']; print('fwd', d['tflops'], 'frac', r['frac'], 'burst frac', r['frac_of_burst'], 'peak', r['peak'], 'burst', r['fp8_burst_peak'], 'bwd', r['bwd_frac_of_bf16'], d['clocks'])"
