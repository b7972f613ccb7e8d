import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2407_16144_b200 import hplp
from tests.helpers import problem, csr_args
from tests.test_box import box_lp
s = hplp.to_standard_form(problem("cfg0"))
args, up = box_lp(s)
sol = hplp.Solver.box(*csr_args(s))
r = sol.solve(tolerance=1e-6, iteration_limit=300000)
x = r["x"]; nb = args[1]
print(r["status"], r["iterations"], r["kkt"])
print("x_box min", x[:nb].min(), "max excess over u", np.max(x[:nb] - up), "slack min", x[nb:].min())
neg = np.nonzero(x < 0)[0]; print("neg idx", neg[:10], x[neg[:10]])
