import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1209_3332_b200 import Context
from synth.hne import make_config_tile
ctx = Context(0, 4096, 4096, 1, 8192)
cap = 8192
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    rgb = torch.from_numpy(make_config_tile(3, i)).cuda()
    lab = torch.zeros((4096, 4096), dtype=torch.int32, device="cuda")
    nob = torch.zeros(1, dtype=torch.int32, device="cuda")
    tl = torch.zeros(cap, dtype=torch.int32, device="cuda"); tf = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tt = torch.zeros((cap, 36), dtype=torch.float32, device="cuda"); nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.process_tile(0, rgb, lab, nob, tl, tf, tt, nr)
    torch.cuda.synchronize()
    print(i, int(nob.item()), int(nr.item()), flush=True)
