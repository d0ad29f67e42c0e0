import os, sys, torch
sys.path.insert(0, "/root/repo/tools"); sys.path.insert(0, "/root/repo")
from kbench import make
from paper_2506_15976_b200.scan import lbm_selective_scan_fwd
lanes = int(os.environ.get("LANES", 1))
x = make(16, 197, 768, 16, torch.float32, torch.float32)
out = torch.empty(16, 197, 768, device="cuda")
for _ in range(4):
    lbm_selective_scan_fwd(**x, window=8, out=out, lanes=lanes)
torch.cuda.synchronize()
