import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2311_07602_b200 import Context
from test_gpu_panel import panel_case, run_panel
ctx = Context(0)
c = panel_case("C", "N", "N", 300, 70, 1, 1, seed=1)
got = run_panel(ctx, c)
want = c.oracle()
G = got[:300*70].reshape(70, 300); Wt = want[:300*70].reshape(70, 300)
print("col64 got", G[64, :4], "want", Wt[64, :4])
for cc in range(0, 70):
    if np.allclose(G[64], Wt[cc]): print("col64 got == want col", cc)
print("rows where col 64 differs:", np.nonzero(G[64] != Wt[64])[0][:10], np.count_nonzero(G[64] != Wt[64]))
