cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 1800 python -m pytest tests/test_gpu_sanitizer.py -q --durations=5 > gpurun_out/r2/t_san2.log 2>&1; echo "san rc=$?"; tail -12 gpurun_out/r2/t_san2.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=25 -k "not sanitizer" > gpurun_out/r2/t_gpu_dur.log 2>&1; echo "gpu rc=$?"; tail -32 gpurun_out/r2/t_gpu_dur.log
