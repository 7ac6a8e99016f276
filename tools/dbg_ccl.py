import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle
from paper_1209_3332_b200 import Context
from tests.gpu_util import stage
ctx = Context(0, 4096, 4096, 2, 1024)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for shape, dens in [((512, 512), 0.6), ((512, 512), 0.55), ((300, 333), 0.55), ((100, 257), 0.6), ((2048, 2048), 0.6)]:
    h, w = shape
    fg = (np.random.default_rng(h * 1000 + w + int(dens * 10)).random(shape) < dens).astype(np.uint8)
    for conn, name in [(4, "CCL4"), (8, "CCL8")]:
        exp, _ = oracle.ccl(fg, conn)
        bad = 0
        for rep in range(reps):
            (lab,) = stage(ctx, name, [fg], [((h, w), np.int32)], w, h)
            if not np.array_equal(lab, exp):
                bad += 1
                if bad == 1:
                    d = np.argwhere(lab != exp)
                    print("  example", name, shape, len(d), d[:3].tolist(), [(int(lab[y, x]), int(exp[y, x])) for y, x in d[:3]], flush=True)
        print(shape, dens, name, "bad", bad, "of", reps, flush=True)
