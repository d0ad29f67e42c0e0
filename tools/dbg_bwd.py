"""Debug: N=4 vectorised path (dev tool)."""
import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, torch
from helpers import op_inputs
from oracle import lbscan_oracle as O
from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd
Bt,L,E,N,M = 2,40,16,4,8
inp = op_inputs(1, Bt, L, E, N); dout = O.seeded_rng(7).standard_normal((Bt,L,E))
t = {k: torch.tensor(v, dtype=torch.float32, device='cuda') for k,v in inp.items()}
y, hf = lbm_selective_scan_fwd(**t, window=M, return_last_state=True)
ry, rhf = O.lbm_selective_scan(**inp, window=M, return_last_state=True)
print('fwd vec N=4', O.max_rel_err(y.cpu().numpy(), ry), O.max_rel_err(hf.cpu().numpy(), rhf))
ref = O.lbm_selective_scan_bwd(dout, **inp, window=M)
# non-vec: B, C as strided (non-unit s2) views
t2 = dict(t); 
for k in ('B','C'):
    big = torch.zeros(Bt, L, 2*N, device='cuda'); big[..., ::2] = t[k]; t2[k] = big[..., ::2]
g = lbm_selective_scan_bwd(torch.tensor(dout, dtype=torch.float32, device='cuda'), **t2, window=M)
print('bwd nonvec-BC', {k: round(O.max_rel_err(g[k].cpu().numpy(), ref[k]), 7) for k in ref if ref[k] is not None})
g = lbm_selective_scan_bwd(torch.tensor(dout, dtype=torch.float32, device='cuda'), **t, window=M)
print('bwd vec', {k: round(O.max_rel_err(g[k].cpu().numpy(), ref[k]), 7) for k in ref if ref[k] is not None})
y2 = lbm_selective_scan_fwd(**t2, window=M)
print('fwd nonvec', O.max_rel_err(y2.cpu().numpy(), ry))
