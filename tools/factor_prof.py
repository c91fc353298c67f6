"""Per-row phase cycles of fsai_factor_kernel (AFN_FACTOR_PROF) on C2, l=1."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/factor_prof.bin"
os.environ["AFN_FACTOR_PROF"] = out
if os.path.exists(out):
    os.remove(out)
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem
X, b = gen_problem("C2")
Xd = torch.from_numpy(X).cuda()
for rep in range(2):
    h = afn.afn_build(Xd, afn.make_params(1.0, 1e-4, 2000, 100, k_adaptive=True))
    torch.cuda.synchronize()
a = np.fromfile(out, dtype=np.int64).reshape(-1, 8)
a = a[len(a) // 2:]  # second build
a = a[a[:, 0] > 0]
names = ["asm", "diag", "panel", "trail", "back"]
tot = a[:, 1:6].sum(1)
print("rows", len(a), "mean wp", a[:, 0].mean(), "mean cycles/row", tot.mean())
for j, n in enumerate(names):
    print("  %-6s mean %8.0f  (%.1f%%)" % (n, a[:, 1 + j].mean(), 100 * a[:, 1 + j].sum() / tot.sum()))
print("  asm = prologue %.0f + gathers %.0f + kernel values %.0f" % (a[:, 6].mean(), a[:, 7].mean(),
      (a[:, 1] - a[:, 6] - a[:, 7]).mean()))
