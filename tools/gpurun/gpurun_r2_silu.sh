cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:silu_mul_pass1 -c 1 -o gpurun_out/r2/silu_p1 python bench.py --workload mgaq-fused --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1; echo "ncu rc=$?"
