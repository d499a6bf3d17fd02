# round-2 final validation: every GPU test, smoke, the default bench line, the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2/t_gpu_final.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2/t_gpu_final.log
timeout 900 python bench.py > gpurun_out/r2/bench_final.json 2> gpurun_out/r2/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2/bench_reference.json 2> gpurun_out/r2/bench_reference.err; echo "ref rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_final.json').read().strip().splitlines()[-1]); print('K1', d['ms_per_step'], d['roofline']['frac'], 'e2e', d['e2e']['value'], d['clocks']); ex=d.get('extra',{}); print({k:(v.get('ms_per_step') or v.get('us_per_step'), v.get('roofline',{}).get('frac')) for k,v in ex.items()}); print(ex.get('cfg4',{}).get('mlp_upgate',{}).get('speedup'))
r=json.loads(open('gpurun_out/r2/bench_reference.json').read().strip().splitlines()[-1]); print('ref', r.get('value'), r.get('unit'))"
