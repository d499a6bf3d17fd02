# warp-specialized RMSNorm row sums: producer parity, fused-layer A/B, per-kernel times
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 900 python -m pytest tests/test_gpu_producers.py -q -x > gpurun_out/r2/t_prod_rms.log 2>&1; echo "producer tests rc=$?"; tail -3 gpurun_out/r2/t_prod_rms.log
for L in "" build_ab/rms0/libcoat.so "" build_ab/rms0/libcoat.so; do
COAT_LIB=$L timeout -s KILL 300 python bench.py --workload mgaq-fused --no-cpu-baseline > gpurun_out/r2/bench_fused_rms.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_fused_rms.json').read().strip().splitlines()[-1]); print('lib=${L:-default}', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rms_row_sum --csv python bench.py --workload mgaq-fused --no-cpu-baseline --steps 1 --warmup 3 2>/dev/null | grep rms_row | head -4 | cut -c1-300
COAT_LIB=build_ab/rms0/libcoat.so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rms_row_sum --csv python bench.py --workload mgaq-fused --no-cpu-baseline --steps 1 --warmup 3 2>/dev/null | grep rms_row | head -4 | cut -c1-300
