"""A/B of pcg_kernel_h8f cluster sizes at the C3 shape (DOCP_H8F_CLUSTER)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
from pcg_microbench import run
run(8, 4, 100, 4096, modes=("fast",))
run(8, 4, 30, 4096, modes=("fast",))
