# K1 diagnostics: helper math stubbed (DIAG=1, wrong results) and per-phase cycle counters (DIAG=9)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
bash tools/abk1.sh base:build_ab/base/libcoat.so:8 diag1:build_ab/diag1/libcoat.so:8 diag9:build_ab/diag9/libcoat.so:8
grep -h K1PROF gpurun_out/abk1_diag9.err | tail -2
