"""Compare the iterates of two library builds bit for bit (diagnostic):
    python tools/cmp_variant.py libA.so libB.so cfg [m] [steps]
A library argument VAR=VALUE@lib.so runs that side with the environment switch VAR=VALUE."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--run":
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2501_13385_b200 as pkg
    import synth
    cfg, m, steps, out = int(sys.argv[2]), (int(sys.argv[3]) or None), int(sys.argv[4]), sys.argv[5]
    pr = synth.make_problem(cfg, m=m)
    t = pkg.TTContext(pr.n, pr.r)
    t.set_cores(pr.truth)
    y = pr.observations(t.eval_at(pr.idx))
    t.close()
    ctx = pkg.TTContext(pr.n, pr.r)
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(pr.init if pr.init is not None else pr.truth)
    for _ in range(steps):
        ctx.step(0.5 if cfg == 3 else 1.0)
    np.savez(out, *ctx.get_cores(), res=ctx.residual_norm())
    sys.exit(0)
a, b, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
m = sys.argv[4] if len(sys.argv) > 4 else "0"
steps = sys.argv[5] if len(sys.argv) > 5 else "3"
import numpy as np  # noqa: E402
outs = []
for lib, tag in ((a, "a"), (b, "b")):
    f = f"/tmp/cmp_{tag}.npz"
    env = dict(os.environ)
    if "@" in lib:                       # VAR=VALUE@lib.so: an environment switch for this run
        kv, lib = lib.split("@", 1)
        k, v = kv.split("=", 1)
        env[k] = v
    env["PRGD_LIB_PATH"] = lib
    subprocess.run([sys.executable, __file__, "--run", cfg, m, steps, f], check=True, env=env)
    outs.append(np.load(f))
za, zb = outs


def tt_norm(C):
    """||T||_F by a left-to-right QR sweep (stable)."""
    R = np.ones((1, 1))
    for c in C:
        M = np.einsum("ab,bic->aic", R, c)
        M = M.reshape(-1, M.shape[2])
        _, R = np.linalg.qr(M)
    return float(np.linalg.norm(R))


def tt_sub(A, B):
    """A - B as a block TT of rank r_A + r_B."""
    d, out = len(A), []
    for k, (a, b) in enumerate(zip(A, B)):
        if k == 0:
            out.append(np.concatenate([a, -b], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([a, b], axis=0))
        else:
            c = np.zeros((a.shape[0] + b.shape[0], a.shape[1], a.shape[2] + b.shape[2]))
            c[:a.shape[0], :, :a.shape[2]] = a
            c[a.shape[0]:, :, a.shape[2]:] = b
            out.append(c)
    return out


ca = [za[f"arr_{k}"] for k in range(len([f for f in za.files if f.startswith("arr_")]))]
cb = [zb[f"arr_{k}"] for k in range(len(ca))]
same = all(np.array_equal(za[k], zb[k]) for k in za.files)
diff = max(float(np.max(np.abs(za[k] - zb[k]))) for k in za.files)
rel = tt_norm(tt_sub(ca, cb)) / tt_norm(ca)
print(f"cfg {cfg}: bitwise identical {same}, max abs core diff {diff:.3e}, "
      f"relative tensor difference {rel:.3e}")