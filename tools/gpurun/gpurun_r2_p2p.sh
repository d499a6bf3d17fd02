# peer-memory ZeRO step (virtual ranks) + MUFU error-model test
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_zero_p2p.py tests/test_gpu_pack_prepare.py -q -x -s > gpurun_out/r2/t_p2p.log 2>&1; echo "tests rc=$?"
grep -E "lg2|passed|failed|Error|error" gpurun_out/r2/t_p2p.log | tail -15
