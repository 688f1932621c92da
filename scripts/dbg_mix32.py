import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from _golden import load
from _engine_run import run_device
import paper_2410_08859_b200.engine as E
orig = E._Batch.solve
def solve(self):
    b = self.batch
    print("n_cells", b.n_cells, "smem_mode", b.smem_mode, "smem", b.smem_bytes, "ny max", self.ny.max(), "ybox", self.ybox[:3].tolist(), flush=True)
    return orig(self)
E._Batch.solve = solve
p = torch.cuda.get_device_properties(0)
print(p, flush=True)
try:
    run_device(load("mix32_staggered"))
except Exception as e:
    print("ERR", e)
