"""Time FPS (k = 2000) on the C2 points for the current AFN_FPS_PPT."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_05460_b200 as afn
from synth import gen_problem
import oracle as O
X, _ = gen_problem("C2")
Xd = torch.from_numpy(X).cuda()
for _ in range(3):
    afn.afn_fps(Xd, 2000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    idx, fill = afn.afn_fps(Xd, 2000)
e1.record(); torch.cuda.synchronize()
io, fo = O.fps(X, 2000, 0)
print(os.environ.get("AFN_FPS_PPT", "1"), "ms", e0.elapsed_time(e1) / 10, "exact", np.array_equal(idx.cpu().numpy(), io))
