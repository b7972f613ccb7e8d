"""B200-native rHPDHG LP solver (arXiv 2407.16144) -- drop-in for the reference
hplp solve() loop.  See DESIGN.md.  The CUDA library is loaded lazily by
:mod:`paper_2407_16144_b200.hplp`; importing the package itself is CPU-safe."""
__version__ = "0.1.0"
