import sys, time
sys.path.insert(0, '.')
from paper_2407_16144_b200 import gen, hplp
for cid in (1, 2):
    g = gen.generate(cid)
    s = hplp.to_standard_form(g)
    for ruiz, alpha in ((0, -1.0), (10, -1.0), (10, 1.0), (0, 1.0), (20, 1.0)):
        t0 = time.time()
        r = hplp.solve(*s.csr(), tolerance=1e-4, time_limit_seconds=60, precondition_ruiz_iters=ruiz, precondition_pc_alpha=alpha)
        _, obj = s.recover(r["x"])
        print(f"cfg{cid} ruiz={ruiz} pc={alpha}: {r['status']} it={r['iterations']} kkt={r['kkt'][3]:.2e} obj={obj:.6f} planted={g.planted_objective:.6f} t={time.time()-t0:.1f}s", flush=True)
