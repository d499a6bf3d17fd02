# K1 with the ZeRO all-gather fused in (P2P): peer-memory step tests, multirank, sanitizer p2p; default K1 A/B vs base
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_zero_p2p.py tests/test_gpu_zero_multirank.py tests/test_gpu_sanitizer.py -q -k "p2p or zero or multirank or Peer" > gpurun_out/r2/t_fag.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r2/t_fag.log
COAT_P2P_FUSED_AG=0 timeout -s KILL 900 python -m pytest tests/test_gpu_zero_p2p.py -q -x > gpurun_out/r2/t_fag0.log 2>&1; echo "unfused rc=$?"; tail -1 gpurun_out/r2/t_fag0.log
for i in 1 2; do for L in base ""; do
COAT_LIB=${L:+build_ab/$L/libcoat.so} timeout -s KILL 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_k1ab.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_k1ab.json').read().strip().splitlines()[-1]); print('${L:-new}', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done; done
