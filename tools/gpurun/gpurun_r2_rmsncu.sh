# ncu --set full of the RMSNorm row-sum kernels (warp-specialized default and the one-warp kernel)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:rms_row_sum -c 1 -f -o gpurun_out/r2/rms_ws python bench.py --workload mgaq-fused --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1; echo rc=$?
COAT_LIB=build_ab/rms0/libcoat.so timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:rms_row_sum -c 1 -f -o gpurun_out/r2/rms_old python bench.py --workload mgaq-fused --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1; echo rc=$?
