"""Per-iteration cost of the PCG kernel: solves with fixed iteration caps
(epsilon tiny, so every solve runs exactly max_iters iterations)."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2510_06179_b200 as D
from paper_2510_06179_b200 import _lib as L

def run(nx, nu, T, B, modes=("fast", "parity"), caps=(1, 11, 41)):
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    b = D.Batch(prob, B)
    b.upload(L.F_THETA, D.generate_affine_quadratic(nx, nu, 0, B))
    b.upload(L.F_Z, np.zeros((B, nz)))
    b.linearize(); b.assemble_schur(); b.assemble_gamma()
    out = {}
    for mode in modes:
        for cap in caps:
            ts = []
            for rep in range(3):
                b.upload(L.F_LAMBDA, np.zeros((B, nl)))
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                b.pcg_solve(D.PcgConfig(epsilon=1e-300, max_iters=cap, mode=mode))
                e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            out[(mode, cap)] = min(ts)
        c0, c1 = caps[1], caps[2]
        slope = (out[(mode, c1)] - out[(mode, c0)]) / (c1 - c0)  # ms per iteration for the batch
        waves = B / 148.0
        print(json.dumps({"shape": [nx, nu, T], "B": B, "mode": mode, "ms": {str(k[1]): v for k, v in out.items() if k[0] == mode},
                          "us_per_iter_per_SM": slope * 1e3 / waves,
                          "cycles_per_iter@1.965GHz": slope * 1e-3 / waves * 1.965e9}), flush=True)

if __name__ == "__main__":
    if "--nx4" in sys.argv:
        run(4, 2, 20, 1184, modes=("fast",))
        run(4, 1, 50, 4096, modes=("fast",))
    else:
        run(8, 4, 100, 1184)
        run(8, 4, 30, 1184)
        run(4, 2, 20, 1184, modes=("fast",))
        run(4, 1, 50, 4096, modes=("fast", "parity"))
