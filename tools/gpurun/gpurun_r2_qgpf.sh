# per-group quantizer with a one-iteration load prefetch: parity + cfg2 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
COAT_LIB=build_ab/qgpf/libcoat.so timeout -s KILL 900 python -m pytest tests/test_gpu_quant.py -q -x > gpurun_out/r2/t_qgpf.log 2>&1; echo "quant tests rc=$?"; tail -1 gpurun_out/r2/t_qgpf.log
for i in 1 2 3; do for L in "" build_ab/qgpf/libcoat.so; do
COAT_LIB=$L timeout -s KILL 300 python bench.py --workload mgaq --no-cpu-baseline > gpurun_out/bench_qg.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_qg.json').read().strip().splitlines()[-1]); print('${L:-base}', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
