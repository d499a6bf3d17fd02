cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -q -k "epi or p2p" > gpurun_out/r2/t_san_new.log 2>&1; echo "san rc=$?"; tail -15 gpurun_out/r2/t_san_new.log
