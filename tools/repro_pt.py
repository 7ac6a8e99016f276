import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1209_3332_b200 import Context
from synth.hne import make_tile, TileSpec
rgb = make_tile(8, TileSpec(1024, 768, tissue_frac=0.7))["rgb"]
h, w = rgb.shape[:2]; cap = 8192
ctx = Context(0, 4096, 4096, n_slots=1, max_objects=cap)
d = torch.from_numpy(np.ascontiguousarray(rgb)).cuda()
lab = torch.empty((h, w), dtype=torch.int32, device="cuda"); nob = torch.zeros(1, dtype=torch.int32, device="cuda")
tl = torch.empty(cap, dtype=torch.int32, device="cuda"); tf = torch.empty(cap, dtype=torch.int32, device="cuda")
tt = torch.empty((cap, 36), dtype=torch.float32, device="cuda"); nr = torch.zeros(1, dtype=torch.int32, device="cuda")
ctx.process_tile(0, d, lab, nob, tl, tf, tt, nr)
torch.cuda.synchronize(); print("ok", int(nob.item()))
