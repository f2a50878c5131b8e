"""Diagnostic: wall-clock breakdown of the end-to-end path (bench.py run_e2e) at a config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_13385_b200 as pkg  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pr = synth.make_problem(cfg)
t = pkg.TTContext(pr.n, pr.r)
t.set_cores(pr.truth)
y = pr.observations(t.eval_at(pr.idx))
t.close()
# E2E_IDX=i32 forces the int32 upload (default: bytes when every mode size is <= 256, like bench.py)
idt = np.uint8 if os.environ.get("E2E_IDX", "u8") == "u8" and max(pr.n) <= 256 else np.int32
idx_p = torch.from_numpy(np.ascontiguousarray(pr.idx, dtype=idt)).pin_memory()
print("index dtype", idx_p.dtype)
y_p = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
cores_p = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in pr.init]
for rep in range(3):
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    ctx = pkg.TTContext(pr.n, pr.r)
    T.append(time.perf_counter())
    ctx.set_observations(idx_p.numpy(), y_p.numpy())
    T.append(time.perf_counter())
    for k, c in enumerate(cores_p):
        ctx.set_core(k, c.numpy())
    T.append(time.perf_counter())
    ctx.step(1.0)
    ctx.residual_norm()
    T.append(time.perf_counter())
    for _ in range(19):
        ctx.step(1.0)
        ctx.residual_norm()
    T.append(time.perf_counter())
    cores = ctx.get_cores()
    T.append(time.perf_counter())
    ctx.close()
    T.append(time.perf_counter())
    names = ["create", "set_observations", "set_cores", "first_step", "19_steps", "get_cores", "close"]
    print(" ".join(f"{n}={1e3 * (b - a):.1f}ms" for n, a, b in zip(names, T[:-1], T[1:])),
          f"total(excl close)={1e3 * (T[-2] - T[0]):.1f}ms")
# raw H2D bandwidth of the same pinned buffers
d = torch.empty(idx_p.numel(), dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
d.copy_(idx_p.view(-1), non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"H2D idx {idx_p.numel() * 4 / 1e9:.2f} GB in {1e3 * (t1 - t0):.1f} ms = {idx_p.numel() * 4 / (t1 - t0) / 1e9:.1f} GB/s")
