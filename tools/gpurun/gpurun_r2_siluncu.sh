# ncu --set full (with SASS source) of the SiLU*mul pass-1 kernel in the fused cfg2 layer
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:silu_mul_pass1 -c 1 -f -o gpurun_out/r2/silu_p1 python bench.py --workload mgaq-fused --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1; echo rc=$?
