# A/B of K1 wait variants + racecheck + K1 parity on the default build
cd $GRAFT_REPO_ROOT
bash tools/abk1.sh w0:build_ab/w0/libcoat.so:8 w1:build_ab/w1/libcoat.so:8 w1s:build_ab/w1s/libcoat.so:8 w1a:build_ab/w1a/libcoat.so:8 w0b:build_ab/w0/libcoat.so:8 w1ab:build_ab/w1a/libcoat.so:8
timeout 900 python -m pytest tests/test_gpu_sanitizer.py -q -k "racecheck" > gpurun_out/r2/t_san2.log 2>&1; echo "san rc=$?"
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_k1_layouts.py tests/test_gpu_fuzz.py -q -x > gpurun_out/r2/t_k1.log 2>&1; echo "k1 tests rc=$?"
tail -3 gpurun_out/r2/t_san2.log gpurun_out/r2/t_k1.log
