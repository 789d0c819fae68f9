import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2311_07602_b200 import Context
from test_gpu_panel import panel_case, run_panel
ctx = Context(0)
for opB in "NT":
  for k in (1, 8):
    for m, n in ((300, 70), (512, 64)):
        c = panel_case("C", "N", opB, m, n, k, 2, seed=1)
        got = run_panel(ctx, c)
        want = c.oracle()
        bad = ~((got == want) | (np.isnan(got) & np.isnan(want)))
        idx = np.nonzero(bad)[0]
        print(opB, k, m, n, "bad", idx.size, "of", got.size, idx[:5], flush=True)
