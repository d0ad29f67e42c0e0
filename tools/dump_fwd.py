import os, sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
from kbench import make
from paper_2506_15976_b200.scan import lbm_selective_scan_fwd
out = {}
for (Bt, L, E, M, seg) in [(4, 197, 384, 8, 0), (3, 50, 256, 4, 0), (2, 1000, 128, 16, 0), (2, 700, 192, 8, 3),
                             (1, 33, 64, 5, 0), (5, 17, 200, 3, 0), (1, 3000, 64, 16, 0), (1, 5000, 64, 16, 7)]:
    dt = torch.float32 if os.environ.get('DT') == 'f32' else torch.bfloat16
    x = make(Bt, L, E, 16, dt, dt, seed=L + E)
    for rev in (False, True):
        for lb in (True, False):
            y, h, ck = lbm_selective_scan_fwd(**x, window=M, reverse=rev, lb=lb, seg_hint=seg, return_last_state=True, save_checkpoints=True)
            out[(Bt, L, E, M, seg, rev, lb)] = (y.cpu(), h.cpu(), None if ck is None else ck.cpu())
torch.save(out, sys.argv[1])
