# cfg2 with fused producers: bench line + per-kernel launch list (serialised under ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 300 python bench.py --workload mgaq-fused --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fused', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'sm', d['clocks']['sm_mhz'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"rms|silu|quant|amax" -c 40 --csv python bench.py --workload mgaq-fused --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/r2/fused_launches.csv 2>/dev/null; echo "ncu rc=$?"
