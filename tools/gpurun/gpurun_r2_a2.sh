# K1 A/B: per-group A loop (base) vs the two-group A block (K1_A2); parity of the A2 build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
bash tools/abk1.sh base:build_ab/base/libcoat.so:8 a2:build_ab/a2/libcoat.so:8 base2:build_ab/base/libcoat.so:8 a2b:build_ab/a2/libcoat.so:8
COAT_LIB=build_ab/a2/libcoat.so timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fuzz.py -q -x -k "step or k1" > gpurun_out/r2/t_a2.log 2>&1; echo "a2 tests rc=$?"; tail -3 gpurun_out/r2/t_a2.log
