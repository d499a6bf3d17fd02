import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from pyoracle import Oracle
from paper_2410_19313_b200 import coatsim as coat
port = Oracle("port")
rows, cols = 64, 11008
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)
g = bf(port.generate(1, (rows, cols), 0.02, 8.0, 21) * np.float32(2.0))
u = bf(port.generate(1, (rows, cols), 0.02, 8.0, 22))
qg, qs, qu, qp, prod = coat.silu_mul_quantize(g.cuda(), u.cuda(), return_prod=True)
p = prod.cpu().numpy()
pc, ps = port.quantize(p, 0)
gpc = qp.codes.cpu().numpy(); gps = qp.scales.float().cpu().numpy()
print("scales", gps, ps, "absmax", np.abs(p).max(), np.nanmax(np.abs(p)))
bad = np.nonzero(gpc != pc)
print("mismatches", len(bad[0]))
for i in range(min(10, len(bad[0]))):
    r, c = bad[0][i], bad[1][i]
    print(r, c, p[r, c], gpc[r, c], pc[r, c], p[r, c] / ps[0])
