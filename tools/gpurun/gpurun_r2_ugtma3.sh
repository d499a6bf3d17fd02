# staged gate/up epilogue: the ragged-row upgate test and the epi sanitizer cases
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_linear.py tests/test_gpu_sanitizer.py -q -k "upgate or epi" > gpurun_out/r2/t_ugtma3.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/r2/t_ugtma3.log
