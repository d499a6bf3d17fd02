# producers: parity (reference DecoderLayer tape, signed zeros, fuzz) + fused-layer bench + per-kernel list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_producers.py tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_prod.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2/t_prod.log
for i in 1 2; do timeout 300 python bench.py --workload mgaq-fused --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fused', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'sm', d['clocks']['sm_mhz'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"rms|silu" -c 12 --csv python bench.py --workload mgaq-fused --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null | grep -E "gpu__time|inst_executed" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-140 | head -12
