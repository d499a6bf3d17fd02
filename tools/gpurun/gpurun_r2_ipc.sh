cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_zero_p2p.py -q -x -k ipc > gpurun_out/r2/t_ipc.log 2>&1; echo "ipc tests rc=$?"; tail -30 gpurun_out/r2/t_ipc.log
