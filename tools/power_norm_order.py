"""Why sigma differs by ~4.5e-11 between the device and the reference on
configs[4]: the reference's power iteration (src/sparse_matrix.cpp:138-179)
with its own bit-exact SpMVs, once with sequential norms (the shim's
squaredNorm, what oracle/_ref runs) and once with exactly rounded norms
(math.fsum).  CPU only, ~2 min, ~20 GB.
  python tools/power_norm_order.py"""
import sys, math, numpy as np
sys.path.insert(0,'/root/repo')
from paper_2407_16144_b200 import gen, hplp
from oracle import CpuStd
g=gen.generate(4); s=CpuStd("reference", g.as_abi()); lp=s.lp()
x0=hplp.power_start(s.n)
print("ref power", lp.power_iteration(), flush=True)
for mode in ["seq","fsum"]:
    nrm = (lambda v: math.sqrt(np.cumsum(v*v)[-1])) if mode=="seq" else (lambda v: math.sqrt(math.fsum(v*v)))
    x=x0.copy(); prev=0
    for k in range(10):
        w=lp.spmv(x); sig=nrm(w)
        z=lp.spmv_transpose(w)
        print(mode,k,repr(sig), flush=True)
        if k>0 and abs(sig-prev)<=1e-4*sig: break
        prev=sig
        x=z/nrm(z)
