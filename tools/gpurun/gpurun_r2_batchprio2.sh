# coat_quantize_batch: priority plan (new) vs round robin (base), batch mode A/B
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for L in base ""; do
COAT_LIB=${L:+build_ab/$L/libcoat.so} timeout -s KILL 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-impl batch > gpurun_out/bench_mgaq_bp.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_mgaq_bp.json').read().strip().splitlines()[-1]); print('${L:-new}', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
