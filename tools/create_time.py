import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2501_13385_b200 as pkg
n, r = (16,)*10, (1,)+(16,)*9+(1,)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ctx = pkg.TTContext(n, r); t1 = time.perf_counter()
    ctx.set_core(0, np.zeros((1,16,16))); t2 = time.perf_counter()
    ctx.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms, first set_core (ensure_base) {1e3*(t2-t1):.2f} ms, close {1e3*(t3-t2):.2f}")
