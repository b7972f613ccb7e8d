"""TEST INFRASTRUCTURE ONLY -- CPU checkers for the B200 rHPDHG path.

Two interchangeable backends behind one Python interface:

* ``port``      -- oracle/liboracle.so, our plain-C++ restatement of the
                   reference loop (oracle/hplp_oracle.cpp);
* ``reference`` -- oracle/_ref/libhplp_ref.so, the UNMODIFIED reference
                   sources compiled against oracle/eigen_shim (oracle/Makefile).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2407_16144_b200) never imports it.
"""
from .loader import CpuLp, CpuStd, available, build, load  # noqa: F401
