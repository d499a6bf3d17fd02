# full GPU suite + default bench + gloo 2-rank functional bench (with the peer-collective phase)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2/t_gpu3.log 2>&1; echo "gpu tests rc=$?"
tail -4 gpurun_out/r2/t_gpu3.log
COAT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --params 268435456 --steps 3 --warmup 3 --no-e2e > gpurun_out/r2/bench_gloo2b.json 2> gpurun_out/r2/bench_gloo2b.err; echo "gloo2 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_gloo2b.json').read().strip().splitlines()[-1]); print('gloo2 ms', d['ms_per_step'], 'p2p', d.get('zero_p2p'))"
tail -5 gpurun_out/r2/bench_gloo2b.err
timeout 900 python bench.py > gpurun_out/r2/bench2.json 2> gpurun_out/r2/bench2.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench2.json').read().strip().splitlines()[-1]); print('K1', d['ms_per_step'], d['roofline']['frac'], 'e2e', d['e2e']['value']); ex=d.get('extra',{}); print({k:(v.get('ms_per_step'), v.get('roofline',{}).get('frac')) for k,v in ex.items()}); print(ex.get('cfg4',{}).get('mlp_upgate'))"
