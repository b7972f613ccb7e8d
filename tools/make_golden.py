"""Generate tests/golden/ fixtures from the UNMODIFIED reference solver.

Runs oracle/_ref/libhplp_ref.so (the reference sources compiled against our
Eigen-subset shim, oracle/Makefile) on small instances -- the SPEC.md known-
answer instances, seeded random LPs and a reduced planted config -- and
stores inputs and outputs (status, iteration counts, final iterate, KKT,
epochs, the first iterates of the trace) as compressed .npz.  These pin the
C++ restatement (oracle/hplp_oracle.cpp) and the GPU path even on machines
without /root/reference.

  python tools/make_golden.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2407_16144_b200 import gen  # noqa: E402

OUT = ROOT / "tests" / "golden"
TRACE_ITERS = 40


def csr(rows, m, n):
    rp, ci, v = [0], [], []
    for r in rows:
        for c, val in r:
            ci.append(c)
            v.append(val)
        rp.append(len(ci))
    return m, n, np.array(rp, np.int64), np.array(ci, np.int32), np.array(v, np.float64)


def random_lp(seed, m, n, density=0.3):
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density
    for i in range(m):
        if not mask[i].any():
            mask[i, rng.integers(n)] = True
    A = np.where(mask, np.round(rng.normal(size=(m, n)), 3), 0.0)
    x0 = rng.random(n)
    b = A @ x0
    c = rng.random(n) + 0.1
    rows = [[(j, A[i, j]) for j in np.nonzero(A[i])[0]] for i in range(m)]
    return (*csr(rows, m, n), b, c)


def instances():
    e1 = (*csr([[(0, 1.0)]], 1, 1), np.array([1.0]), np.array([0.0]))
    yield "e1", e1, dict(tolerance=1e-8)
    yield "primal_infeasible", (*csr([[(0, 1.0)], [(0, 1.0)]], 2, 1), np.array([1.0, 2.0]), np.array([0.0])), {}
    yield "dual_infeasible", (*csr([[(0, 1.0), (1, -1.0)]], 1, 2), np.array([0.0]), np.array([-1.0, 0.0])), {}
    for s in range(3):
        yield f"random{s}", random_lp(100 + s, 5, 8), dict(tolerance=1e-8, iteration_limit=20000)
    g = gen.generate(gen.scaled(0, m=60, n=120, nnz_per_row=6))
    from oracle import CpuStd

    st = CpuStd("reference", g.as_abi())
    yield "planted_small", (st.m, st.n, st.row_ptr, st.col_idx, st.val, st.b, st.c), dict(tolerance=1e-6,
                                                                                           iteration_limit=60000)


def main():
    if not oracle.available("reference"):
        oracle.build(("reference",))
    OUT.mkdir(parents=True, exist_ok=True)
    for name, (m, n, rp, ci, v, b, c), kw in instances():
        lp = oracle.CpuLp("reference", m, n, rp, ci, v, b, c)
        r = lp.solve(trace=False, **kw)
        t = lp.solve(trace=True, **dict(kw, iteration_limit=min(TRACE_ITERS, kw.get("iteration_limit", 10**9))))
        sig, pit, conv, _ = lp.power_iteration()
        pc = r["primal_cert"][0] if r["primal_cert"] else np.zeros(0)
        dc = r["dual_cert"][0] if r["dual_cert"] else np.zeros(0)
        np.savez_compressed(
            OUT / f"{name}.npz", m=m, n=n, row_ptr=rp, col_idx=ci, val=v, b=b, c=c,
            kwargs=np.array(repr(kw)), status=np.array(r["status"]), iterations=r["iterations"],
            spmv_count=r["spmv_count"], eta=r["eta"], sigma_estimate=r["sigma_estimate"], kkt=np.array(r["kkt"]),
            x=r["x"], y=r["y"], primal_cert=pc, dual_cert=dc,
            epochs=np.array([(e[0], e[1], e[2], *e[3]) for e in r["epochs"]]).reshape(-1, 7),
            trace_x=np.array([tr["x"] for tr in t["trace"]]), trace_y=np.array([tr["y"] for tr in t["trace"]]),
            trace_nk=np.array([(tr["epoch"], tr["inner"]) for tr in t["trace"]]).reshape(-1, 2),
            trace_res=np.array([tr["res"] for tr in t["trace"]]),
            power=np.array([sig, pit, conv], dtype=np.float64),
        )
        print(f"{name:18s} {r['status']:18s} it={r['iterations']}")


if __name__ == "__main__":
    main()
