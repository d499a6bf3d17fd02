# K1 A/B: flat 2^-15 SFU certification interval (base) vs k-scaled (krel); parity of the new default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
bash tools/abk1.sh base:build_ab/base/libcoat.so:8 krel:build_ab/krel/libcoat.so:8 base2:build_ab/base/libcoat.so:8 krel2:build_ab/krel/libcoat.so:8
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fuzz.py tests/test_gpu_dre.py tests/test_gpu_pack_prepare.py tests/test_gpu_k1_layouts.py tests/test_gpu_step_fullsize.py -q -x -s > gpurun_out/r2/t_krel.log 2>&1; echo "tests rc=$?"; grep -E "max abs err|passed|failed|fallback" gpurun_out/r2/t_krel.log | tail -8
