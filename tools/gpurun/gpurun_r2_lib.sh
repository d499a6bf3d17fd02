# cfg4 with the interleaved same-shape library comparison (K4 vs cuBLASLt FP8 / cuBLAS BF16)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 600 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_lib.json 2>gpurun_out/r2/bench_linear_lib.err; echo "bench rc=$?"
tail -3 gpurun_out/r2/bench_linear_lib.err
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_lib.json').read().strip().splitlines()[-1]); r=d['roofline']; print('fwd', d['tflops'], 'frac', r['frac'], 'peak', r['peak']); print(json.dumps(d['library_same_shape'], indent=1)); print(d['mlp_upgate']['speedup'])"
