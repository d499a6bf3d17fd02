# K4 two-pair B-multicast cluster (COAT_GEMM_CTA=4): parity first (short timeouts), then cfg4 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
COAT_GEMM_CTA=4 timeout -s KILL 120 python -c "
import torch
from paper_2410_19313_b200 import coatsim as coat
M,K,N=1024,512,768
x=torch.randn(M,K,device='cuda').to(torch.bfloat16); w=torch.randn(K,N,device='cuda')/K**0.5
qx=coat.quantize(x,coat.QuantGeometry.per_tensor()); qw=coat.quantize(w,coat.QuantGeometry.per_tensor())
y=coat.fp8_linear(qx,qw); torch.cuda.synchronize()
ref=(coat.dequantize(qx).float()@coat.dequantize(qw).float())
print('probe max err', (y-ref).abs().max().item(), ref.abs().max().item())
" 2>&1 | tail -3; echo "probe rc=$?"
COAT_GEMM_CTA=4 timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_linear_mc4.log 2>&1; echo "linear tests mc4 rc=$?"; tail -15 gpurun_out/r2/t_linear_mc4.log
for C in 2 4 2 4; do
COAT_GEMM_CTA=$C timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_c$C.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_c$C.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('C=$C', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib', {k: round(v,1) for k,v in l['tflops'].items()}, 'fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), d['clocks']['sm_mhz'])"
done
