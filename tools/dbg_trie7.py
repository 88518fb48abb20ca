import sys, numpy as np
sys.path.insert(0, '/root/repo')
from synth import corpus as sc
from paper_1704_07468_b200 import gakco as gk
import oracle
oracle.build()
cp = sc.make("tiny")
ref = oracle.compute(cp, 7, 5, 2)
for bk in (1, 4700, 3*4700+5, 1<<20):
    for mode in (3, 7):
        plan = gk.Plan(cp.sigma, 7, 5, 2)
        plan.set_option(gk.GAKCO_OPT_BATCH_KEYS, bk)
        plan.set_option(gk.GAKCO_OPT_SORT, mode)
        r = gk.kernel_matrix(cp.codes, cp.offsets, cp.sigma, 7, 5, 2, plan=plan)
        C = r["C"].cpu().numpy()
        st = plan.stats()
        plan.close()
        bad = [m for m in range(3) if not np.array_equal(C[m], ref["C"][m])]
        print(bk, mode, "bad levels", bad, "diag ok", [np.array_equal(np.diag(C[m]), np.diag(ref["C"][m])) for m in range(3)], st["sort_passes"], st["keys"])
