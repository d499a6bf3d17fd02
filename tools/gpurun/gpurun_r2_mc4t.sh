# K4 parity: default, the cluster-of-4 multicast kernel and raster groups
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_linear.py tests/test_gpu_k1_layouts.py -q -x -k "linear or cluster or single_cta" > gpurun_out/r2/t_mc4.log 2>&1; echo "rc=$?"; tail -8 gpurun_out/r2/t_mc4.log
