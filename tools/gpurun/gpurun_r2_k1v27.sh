# K1 end-of-round ncu capture (--set full, 500M params), default layout
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_ws_kernel -c 1 -f -o gpurun_out/r2/k1_v27 python bench.py --params 499998976 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r2/ncu_k1_v27.log 2>&1; echo "ncu rc=$?"
