"""Plain fp64 NumPy oracle of one PRGD iteration — TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference).  Shares no code with the CUDA path.

Notation: tensor order d (paper: m), mode sizes n_k (paper:
d_k), TT ranks r_0..r_d with r_0 = r_d = 1, observed set Omega of M entries with
0-based multi-indices idx[s, k] = x_{s,k}, sampling rate p = M / prod(n).
Cores are float64 arrays of shape [r_{k-1}, n_k, r_k]; the tensor is
  T(x) = T_1(x_1,:) T_2(:,x_2,:) ... T_d(:,x_d).
Multi-indices linearise with x_1 most significant (C order).

Every function cites the passage it follows.  Readings of ambiguous passages are
the R-numbers of SURVEY.md §8(c) / DESIGN.md §3.  "parity unpinned" marks the
functions with no pin other than the invariants: none.
"""
from __future__ import annotations

import math
from typing import List, Sequence

import numpy as np

__all__ = [
    "CHUNK", "NumericError", "left_mul", "right_mul", "eval_at", "residual",
    "mode_sums", "vee_norm", "build_weights", "weight_cores", "left_orthogonalize",
    "right_grams", "precondition_residual", "interfaces", "contraction", "project",
    "unweight", "step_length", "assemble", "tt_round", "prgd_step", "solve",
    "split_point", "stable_order", "stable_buckets", "to_dense", "tt_svd",
    "spectral_init", "tt_norm", "tt_diff_norm", "tt_add", "os_dim", "os_to_m",
    "theory_step", "tangent_direction", "tangent_sum", "tt_dot", "adaptive_step",
]

CHUNK = 1 << 18   # samples per chunk (bounds interface memory; order of sums only)


class NumericError(RuntimeError):
    """NaN/Inf or a Cholesky breakdown of the right Gram P_k (reading R6)."""


# --------------------------------------------------------------------------- A1, A8
def _slice_groups(xk: np.ndarray, nk: int):
    order = np.argsort(xk, kind="stable")
    bounds = np.searchsorted(xk[order], np.arange(nk + 1), side="left")
    return order, bounds


def left_mul(a: np.ndarray, core: np.ndarray, xk: np.ndarray) -> np.ndarray:
    """Left-part recursion T^{<=k}(x) = T^{<=k-1}(x) T_k(:, x_k, :).

    a: [c, r_{k-1}] rows T^{<=k-1}(x_s); returns [c, r_k].  Samples sharing x_k
    are multiplied by that slice in one BLAS call."""
    out = np.empty((a.shape[0], core.shape[2]))
    order, bounds = _slice_groups(xk, core.shape[1])
    for j in range(core.shape[1]):
        ids = order[bounds[j]:bounds[j + 1]]
        if ids.size:
            out[ids] = a[ids] @ core[:, j, :]
    return out


def right_mul(core: np.ndarray, xk: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Right-part recursion T^{>=k}(:, x) = T_k(:, x_k, :) T^{>=k+1}(:, x).

    b: [c, r_k] columns T^{>=k+1}(:, x_s) stored as rows; returns [c, r_{k-1}]."""
    out = np.empty((b.shape[0], core.shape[0]))
    order, bounds = _slice_groups(xk, core.shape[1])
    for j in range(core.shape[1]):
        ids = order[bounds[j]:bounds[j + 1]]
        if ids.size:
            out[ids] = b[ids] @ core[:, j, :].T
    return out


def eval_at(cores: Sequence[np.ndarray], idx: np.ndarray) -> np.ndarray:
    """A1: v_s = T_1(x_1,:) T_2(:,x_2,:) ... T_d(:,x_d)  (`equ: TT Core`)."""
    idx = np.asarray(idx)
    out = np.empty(idx.shape[0])
    for c0 in range(0, idx.shape[0], CHUNK):
        x = idx[c0:c0 + CHUNK]
        a = np.ones((x.shape[0], 1))
        for k, core in enumerate(cores):
            a = left_mul(a, core, x[:, k])
        out[c0:c0 + x.shape[0]] = a[:, 0]
    return out


# --------------------------------------------------------------------------- A2
def residual(cores, idx, y) -> np.ndarray:
    """A2: g_s = T_l(x_s) - y_s, the nonzeros of G_l = P_Omega(T_l - T*)
    (Alg. 2 line 1; reading R14: the observed y stands for T*)."""
    return eval_at(cores, idx) - np.asarray(y, dtype=np.float64)


# --------------------------------------------------------------------------- A3
def mode_sums(g: np.ndarray, idx: np.ndarray, n: Sequence[int]) -> List[np.ndarray]:
    """A3: h_{k,j} = ||M_k(G)(j,:)||_2^2 = sum_{s: x_{s,k}=j} g_s^2, the diagonal of
    diag(M_k(G) M_k(G)^T).  Omega is a set (reading R12)."""
    g2 = np.asarray(g, dtype=np.float64) ** 2
    return [np.bincount(idx[:, k], weights=g2, minlength=n[k]).astype(np.float64)
            for k in range(len(n))]


def vee_norm(g, idx, n) -> float:
    """||G||_vee = max_k max_j ||M_k(G)(j,:)||_2."""
    h = mode_sums(g, idx, n)
    return math.sqrt(max(float(hk.max()) if hk.size else 0.0 for hk in h))


def build_weights(h: Sequence[np.ndarray], d: int, eps_rule: str = "vee",
                  eps_value: float | None = None):
    """Diagonal weights G_{l,k} = eps I + diag(h_k) with
    eps_l = ||G_l||_vee^2 = max h (reading R1), and the per-slice
    scaling phi_{k,j} = w_{k,j}^{1/(4d)}, the diagonal of G_{l,k}^{1/(4m)} that
    W^{1/2} applies per mode.

    eps_rule: "vee" (default), "fixed" (eps = eps_value > 0), "none" (W = I, RGD).
    Returns (eps, w, phi) with eps = None for "none"; eps = 0.0 flags the exact
    fit (reading R4)."""
    if eps_rule == "none":
        return None, [np.ones_like(hk) for hk in h], [np.ones_like(hk) for hk in h]
    if eps_rule == "vee":
        eps = max(float(hk.max()) if hk.size else 0.0 for hk in h)
    elif eps_rule == "fixed":
        if eps_value is None or not eps_value > 0:
            raise ValueError("fixed eps needs eps_value > 0")
        eps = float(eps_value)
    else:
        raise ValueError(eps_rule)
    if eps == 0.0:
        return 0.0, None, None
    w = [eps + hk for hk in h]
    phi = [np.power(wk, 1.0 / (4.0 * d)) for wk in w]
    return eps, w, phi


def weight_cores(cores, phi, power: float = 1.0):
    """Component weighting, Prop. 3.1: the TT of W^{power/2} T is
    [T_k ×_2 G_{l,k}^{power/(4m)}], i.e. slice j of core k scaled by phi_{k,j}^power."""
    return [c * (np.asarray(p) ** power)[None, :, None] for c, p in zip(cores, phi)]


# --------------------------------------------------------------------------- A5
def left_orthogonalize(cores):
    """A5: left-orthogonal decomposition by a Householder QR sweep (PAPER.md:92-97,
    289 "classical procedure"; reading R5): for k < d, L(C_k) = Q R, U_k = Q,
    C_{k+1} <- R ×_1 C_{k+1}; U_d = C_d.  LAPACK sign convention (numpy.linalg.qr)."""
    cores = [np.array(c, dtype=np.float64, copy=True) for c in cores]
    out = []
    for k in range(len(cores) - 1):
        r0, nk, r1 = cores[k].shape
        q, rr = np.linalg.qr(cores[k].reshape(r0 * nk, r1))
        out.append(q.reshape(r0, nk, q.shape[1]))
        cores[k + 1] = np.einsum("ab,bjc->ajc", rr, cores[k + 1])
    out.append(cores[-1])
    return out


# --------------------------------------------------------------------------- A6
def right_grams(U):
    """A6: P_k = T^{>=k+1} (T^{>=k+1})^T (r_k x r_k), the Gram inverted in
    `equ: tsp in nm`, by the recursion P_d = [1],
    P_k = sum_j U_{k+1}(:,j,:) P_{k+1} U_{k+1}(:,j,:)^T.
    Returns P[0..d-1] with P[k-1] = P_k (P[d-1] = [[1]])."""
    d = len(U)
    P = [None] * d
    P[d - 1] = np.ones((1, 1))
    for k in range(d - 2, -1, -1):
        Un = U[k + 1]
        P[k] = np.einsum("ajc,cd,bjd->ab", Un, P[k + 1], Un)
    return P


# --------------------------------------------------------------------------- A7
def precondition_residual(g, idx, phi):
    """A7: ghat = W^{-1/2} G, entrywise g_s prod_k phi_{k,x_{s,k}}^{-1}
    (Ghat := W^{-1/2} G; W^{1/2} scales mode k by G^{1/(4m)})."""
    s = np.ones(idx.shape[0])
    for k, p in enumerate(phi):
        s = s / p[idx[:, k]]
    return np.asarray(g) * s


# --------------------------------------------------------------------------- A8, A9
def interfaces(U, x):
    """A8: left interfaces a^{(k)}_s = U^{<=k}(x_s) (k = 0..d-1, a^{(0)} = 1) and right
    interfaces b^{(k)}_s = U^{>=k}(:, x_s) (k = 2..d+1, b^{(d+1)} = 1).
    Returns lists a[k] (k=0..d-1) and b[k] (k=1..d, b[k] = b^{(k+1)})."""
    d = len(U)
    c = x.shape[0]
    a = [np.ones((c, 1))]
    for k in range(d - 1):
        a.append(left_mul(a[-1], U[k], x[:, k]))
    b = [None] * (d + 1)
    b[d] = np.ones((c, 1))
    for k in range(d - 1, 0, -1):          # 0-based core k -> b[k] = b^{(k+1)} (1-based)
        b[k] = right_mul(U[k], x[:, k], b[k + 1])
    return a, b


def contraction(U, idx, ghat):
    """A9: Y_k(:, j, :) = sum_{s: x_{s,k}=j} ghat_s a^{(k-1)}_s (b^{(k+1)}_s)^T, i.e.
    (That^{<=k-1} (x) I)^T Ghat^{<k>} (That^{>=k+1})^T for sparse Ghat
    (`equ: tsp in nm`).  One BLAS GEMM L^T diag(ghat) R per (k, j)."""
    d = len(U)
    Y = [np.zeros(u.shape) for u in U]
    for c0 in range(0, idx.shape[0], CHUNK):
        x = idx[c0:c0 + CHUNK]
        gh = ghat[c0:c0 + CHUNK]
        a, b = interfaces(U, x)
        for k in range(d):
            order, bounds = _slice_groups(x[:, k], U[k].shape[1])
            left = a[k] * gh[:, None]                    # a^{(k-1)} (1-based) scaled
            right = b[k + 1]                             # b^{(k+1)} (1-based)
            for j in range(U[k].shape[1]):
                ids = order[bounds[j]:bounds[j + 1]]
                if ids.size:
                    Y[k][:, j, :] += left[ids].T @ right[ids]
    return Y


# --------------------------------------------------------------------------- A10
def project(U, P, Y):
    """A10, closed form of P_{That} (`equ: tsp in nm`):
    for k < d: L(Ahat_k) = (I - L(U_k) L(U_k)^T) L(Y_k) P_k^{-1};  L(Ahat_d) = L(Y_d)
    (reading R7).  P_k^{-1} by Cholesky solve; breakdown raises NumericError (R6)."""
    d = len(U)
    A = []
    for k in range(d):
        r0, nk, r1 = U[k].shape
        Yk = Y[k].reshape(r0 * nk, r1)
        if k == d - 1:
            A.append(Yk.reshape(r0, nk, r1).copy())
            continue
        try:
            L = np.linalg.cholesky(P[k])
        except np.linalg.LinAlgError as e:
            raise NumericError(f"Cholesky breakdown of P_{k + 1}") from e
        # Z = Yk P^{-1}  <=>  P Z^T = Yk^T
        Z = np.linalg.solve(L.T, np.linalg.solve(L, Yk.T)).T
        Uk = U[k].reshape(r0 * nk, r1)
        Z = Z - Uk @ (Uk.T @ Z)
        A.append(Z.reshape(r0, nk, r1))
    return A


# --------------------------------------------------------------------------- A11
def unweight(cores, phi):
    """A11: A_k = Ahat_k ×_2 G^{-1/(4m)}, Ttil_k = That_k ×_2 G^{-1/(4m)}
    (PAPER.md:293, 360)."""
    return weight_cores(cores, phi, -1.0)


# --------------------------------------------------------------------------- A12
def step_length(step_size, eps, p, step_rule="theory"):
    """A12: alpha_l = step_size * eps_l^{1/2} / p (Thm 4.1 with step_size = 1.001,
    PAPER.md:384; reading R2), or alpha = step_size ("raw").  With W = I
    (eps_rule "none") the theory rule is step_size / p.  The adaptive rule needs the
    direction: see adaptive_step."""
    if step_rule == "raw":
        return float(step_size)
    if step_rule != "theory":
        raise ValueError(step_rule)
    if eps is None:
        return float(step_size) / p
    return float(step_size) * math.sqrt(eps) / p


def theory_step(eps, p, mult=1.001):
    """alpha_l = 1.001 eps_l^{1/2} p^{-1}."""
    return mult * math.sqrt(eps) / p


def tt_dot(a, b) -> float:
    """<a, b>_F of two TTs with equal mode sizes: contract the cores left to right,
    M <- sum_j a_k(:, j, :)^T M b_k(:, j, :), starting from M = [1]."""
    M = np.ones((1, 1))
    for ca, cb in zip(a, b):
        M = np.einsum("ab,ajc,bjd->cd", M, ca, cb)
    return float(M[0, 0])


def adaptive_step(step_size, U, Ahat, Ttil, A, idx):
    """A12, adaptive rule: the steepest step along the search direction in the tangent space
    (eq. `PRGD stepsize`),
        alpha_l = step_size * ||P~_T W^{-1} G||_W^2 / ||P_Omega P~_T W^{-1} G||_F^2,
    which for W = I is RGD's alpha_l = ||P_T G||_F^2 / ||P_Omega P_T G||_F^2.
    D = P~_T W^{-1} G = sum_k [Ttil_1..A_k..Ttil_d].  Numerator: the
    components are W-orthogonal (Lemma `component orthogonal`), and
    W^{1/2} [Ttil_1..A_k..Ttil_d] = [U_1..Ahat_k..U_d] (Prop. 3.1), so
    ||D||_W^2 = sum_k ||[U_1..Ahat_k..U_d]||_F^2.  Denominator: D evaluated at every observed
    index.  Returns (alpha, num, den); alpha = 0 when den = 0 (reading R20)."""
    d = len(U)
    num = 0.0
    for k in range(d):
        comp = [Ahat[i] if i == k else U[i] for i in range(d)]
        num += tt_dot(comp, comp)
    D = tangent_sum(Ttil, A)
    v = eval_at(D, idx)
    den = float(v @ v)
    alpha = float(step_size) * num / den if den > 0.0 else 0.0
    return alpha, num, den


# --------------------------------------------------------------------------- A13
def assemble(Ttil, A, alpha):
    """A13: rank-<=2r TT of W_l = T_l - alpha sum_k [Ttil_1..A_k..Ttil_d]
    (SURVEY App. X.1): X_k = -alpha A_k,
    B_1 = [X_1, Ttil_1], B_k = [[Ttil_k, 0], [X_k, Ttil_k]], B_d = [[Ttil_d], [Ttil_d + X_d]]."""
    d = len(Ttil)
    X = [-alpha * a for a in A]
    if d == 1:
        return [Ttil[0] + X[0]]
    B = []
    for k in range(d):
        r0, nk, r1 = Ttil[k].shape
        if k == 0:
            B.append(np.concatenate([X[0], Ttil[0]], axis=2))
        elif k == d - 1:
            B.append(np.concatenate([Ttil[k], Ttil[k] + X[k]], axis=0))
        else:
            b = np.zeros((2 * r0, nk, 2 * r1))
            b[:r0, :, :r1] = Ttil[k]
            b[r0:, :, :r1] = X[k]
            b[r0:, :, r1:] = Ttil[k]
            B.append(b)
    return B


# --------------------------------------------------------------------------- A14
def tt_round(B, r):
    """A14: SVD_r^tt(W_l) (Alg. 1) computed as TT-rounding of the
    rank-2r TT (reading R8): right-to-left QR orthogonalisation,
    then left-to-right SVD keeping the top r_k left singular vectors (first r_k
    as returned on ties, reading R10).  Output cores 1..d-1 are left-orthogonal."""
    B = [np.array(b, dtype=np.float64, copy=True) for b in B]
    d = len(B)
    for k in range(d - 1, 0, -1):
        R0, nk, R1 = B[k].shape
        q, rr = np.linalg.qr(B[k].reshape(R0, nk * R1).T)       # M^T = Q R
        B[k] = q.T.reshape(q.shape[1], nk, R1)
        B[k - 1] = np.einsum("anb,cb->anc", B[k - 1], rr)      # B_{k-1} ×_3 R^T
    out = []
    for k in range(d - 1):
        R0, nk, R1 = B[k].shape
        u, s, vt = np.linalg.svd(B[k].reshape(R0 * nk, R1), full_matrices=False)
        rk = r[k + 1]
        if u.shape[1] < rk:
            raise ValueError("rank infeasible in rounding")
        out.append(u[:, :rk].reshape(R0, nk, rk))
        sv = s[:rk, None] * vt[:rk, :]
        B[k + 1] = np.einsum("ab,bnc->anc", sv, B[k + 1])
    out.append(B[d - 1])
    return out


def tangent_direction(cores, phi, idx, zhat):
    """P~_T applied through Lemma `close of P_tilde`:
    P~_T Z = W^{-1/2} P_{That} W^{1/2} Z, given zhat = the nonzeros of W^{1/2} Z on idx.
    A4 That = W^{1/2} T_l (Prop. 3.1), A5 left-orthogonal U, A6 Grams, A8-A9 Y,
    A10 closed form, A11 back to the unweighted space.  For the PRGD direction
    P~_T W^{-1} G, zhat = W^{-1/2} G (A7).  Returns dict(U, P, Y, Ahat, A, Ttil)
    with the tangent vector sum_k [Ttil_1..A_k..Ttil_d]."""
    Chat = weight_cores(cores, phi, 1.0)
    U = left_orthogonalize(Chat)
    P = right_grams(U)
    Y = contraction(U, np.asarray(idx), np.asarray(zhat, dtype=np.float64))
    Ahat = project(U, P, Y)
    return dict(U=U, P=P, Y=Y, Ahat=Ahat, A=unweight(Ahat, phi), Ttil=unweight(U, phi))


def tangent_sum(Ttil, A):
    """The tangent vector sum_k [Ttil_1, .., A_k, .., Ttil_d] as a
    rank-2r TT: B_1 = [A_1, Ttil_1], B_k = [[Ttil_k, 0], [A_k, Ttil_k]], B_d = [[Ttil_d], [A_d]]."""
    d = len(Ttil)
    if d == 1:
        return [A[0].copy()]
    B = []
    for k in range(d):
        r0, nk, r1 = Ttil[k].shape
        if k == 0:
            B.append(np.concatenate([A[0], Ttil[0]], axis=2))
        elif k == d - 1:
            B.append(np.concatenate([Ttil[k], A[k]], axis=0))
        else:
            b = np.zeros((2 * r0, nk, 2 * r1))
            b[:r0, :, :r1] = Ttil[k]
            b[r0:, :, :r1] = A[k]
            b[r0:, :, r1:] = Ttil[k]
            B.append(b)
    return B


# --------------------------------------------------------------------------- Alg. 2
def prgd_step(cores, idx, y, n, r, step_size, eps_rule="vee", eps_value=None,
              step_rule="theory", return_info=False, retraction="plain"):
    """One iteration of Alg. 2 without trimming (reading R9):
    G_l = P_Omega(T_l - T*); alpha_l; W_l = T_l - alpha_l P~_T W^{-1} G_l with
    P~_T = W^{-1/2} P_{That} W^{1/2} (Lemma); T_{l+1} = SVD_r^tt(W_l)
    (retraction "plain", Alg. 2 line 5) or W_l^{-1/2} SVD_r^tt(W_l^{1/2} W_l) ("weighted", the
    Remark at PAPER.md:365-367; W^{+-1/2} applied to the TT by Prop. 3.1).
    """
    d = len(n)
    cores = [np.asarray(c, dtype=np.float64) for c in cores]
    idx = np.asarray(idx)
    m = idx.shape[0]
    if m == 0:
        raise ValueError("empty Omega")
    p = m / math.prod(n)                                         # reading R3
    g = residual(cores, idx, y)                                  # A1-A2
    if not np.all(np.isfinite(g)):
        raise NumericError("non-finite residual")
    h = mode_sums(g, idx, n)                                     # A3
    eps, w, phi = build_weights(h, d, eps_rule, eps_value)
    info = dict(g=g, h=h, eps=eps, p=p, sumsq=float(g @ g))
    if eps == 0.0:                                               # reading R4
        new = [c.copy() for c in cores]
        info.update(noop=True)
        return (new, info) if return_info else new
    ghat = precondition_residual(g, idx, phi)                    # A7
    tv = tangent_direction(cores, phi, idx, ghat)                # A4-A6, A8-A11
    if step_rule == "adaptive":                                  # A12
        alpha, num, den = adaptive_step(step_size, tv["U"], tv["Ahat"], tv["Ttil"], tv["A"], idx)
        info.update(adapt_num=num, adapt_den=den)
    else:
        alpha = step_length(step_size, eps, p, step_rule)        # A12
    B = assemble(tv["Ttil"], tv["A"], alpha)                     # A13
    if retraction == "plain":
        new = tt_round(B, r)                                     # A14
    elif retraction == "weighted":
        new = weight_cores(tt_round(weight_cores(B, phi, 1.0), r), phi, -1.0)
    else:
        raise ValueError(retraction)
    info.update(noop=False, w=w, phi=phi, ghat=ghat, alpha=alpha, B=B, **tv)
    return (new, info) if return_info else new


def solve(cores, idx, y, n, r, step_size, iters, **kw):
    """Loop body of Alg. 2 `iters` times; returns final cores and residual norms."""
    res = []
    for _ in range(iters):
        cores, info = prgd_step(cores, idx, y, n, r, step_size, return_info=True, **kw)
        res.append(math.sqrt(info["sumsq"]))
    return cores, res


# --------------------------------------------------------------------------- A0
def split_point(n: Sequence[int]) -> int:
    """Prefix/suffix split K_L (1 <= K_L <= d-1) minimising max(N_{<=K_L}, N_{>K_L}),
    ties to the smaller K_L (same rule as the library's planner)."""
    d = len(n)
    best, bestv = 1, None
    for kl in range(1, d):
        v = max(math.prod(n[:kl]), math.prod(n[kl:]))
        if bestv is None or v < bestv:
            best, bestv = kl, v
    return best


def stable_order(idx, n, K_L):
    """A0 on the table path: samples bucketed by the prefix index
    P(s) = mixed radix of (x_1..x_{K_L}) (x_1 most significant) and by the suffix index
    S(s) = mixed radix of (x_{K_L+1}..x_d) (x_d most significant).  Prefix order = stable
    argsort of the key P*2^bS + S (i.e. by (P, S)); suffix order = stable argsort of
    S*2^bP + P.  Returns dict(perm_pre, offs_L, perm_suf, offs_R, P, S)."""
    idx = np.asarray(idx, dtype=np.int64)
    d = len(n)
    P = np.zeros(idx.shape[0], dtype=np.int64)
    for k in range(K_L):
        P = P * n[k] + idx[:, k]
    S = np.zeros(idx.shape[0], dtype=np.int64)
    for k in range(d - 1, K_L - 1, -1):
        S = S * n[k] + idx[:, k]
    NL, NR = math.prod(n[:K_L]), math.prod(n[K_L:])
    bP, bS = max(1, int(NL - 1).bit_length()), max(1, int(NR - 1).bit_length())
    perm_pre = np.argsort((P << bS) | S, kind="stable")
    perm_suf = np.argsort((S << bP) | P, kind="stable")
    offs_L = np.concatenate([[0], np.cumsum(np.bincount(P, minlength=NL))])
    offs_R = np.concatenate([[0], np.cumsum(np.bincount(S, minlength=NR))])
    return dict(perm_pre=perm_pre, offs_L=offs_L, perm_suf=perm_suf, offs_R=offs_R, P=P, S=S)


def stable_buckets(idx, n):
    """A0 per-mode buckets (the chain path): for each mode k, perm_k = the
    stable argsort of x_{:,k} (bucket j = the samples with x_{s,k} = j, the rows of the mode-k
    unfolding M_k(G) that PAPER.md:163 sums over, in ascending s), offs_k = exclusive
    cumulative bucket counts (n_k + 1 entries)."""
    out = []
    for k in range(len(n)):
        perm = np.argsort(idx[:, k], kind="stable")
        offs = np.concatenate([[0], np.cumsum(np.bincount(idx[:, k], minlength=n[k]))])
        out.append((perm, offs))
    return out


# --------------------------------------------------------------------------- dense helpers
def to_dense(cores):
    """Materialise the tensor by the left-part recursion, x_1 most
    significant.  Small tensors only."""
    t = np.ones((1, 1))
    for c in cores:
        r0, nk, r1 = c.shape
        t = (t @ c.reshape(r0, nk * r1)).reshape(-1, r1)
    return t.reshape([c.shape[1] for c in cores])


def tt_svd(X, r):
    """Alg. 1 TT-SVD, literally: for i = 1..m-1, L(T_i) = top r_i
    left singular vectors of (T^{<=i-1} (x) I_{d_i})^T X^{<i>}, T^{<=i} =
    (T^{<=i-1} (x) I) L(T_i); T_m = (T^{<=m-1})^T X^{<m-1>}."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape
    d = len(n)
    cores = []
    left = np.ones((1, 1))                                       # T^{<=0}
    for i in range(d - 1):
        Ni = math.prod(n[:i + 1])
        Xi = X.reshape(math.prod(n[:i]), n[i], -1)               # [P, n_i, rest]
        Z = np.einsum("pa,pxq->axq", left, Xi).reshape(left.shape[1] * n[i], -1)
        u, _, _ = np.linalg.svd(Z, full_matrices=False)
        Li = u[:, :r[i + 1]]
        cores.append(Li.reshape(left.shape[1], n[i], Li.shape[1]))
        left = np.einsum("pa,axc->pxc", left, cores[-1]).reshape(Ni, Li.shape[1])
    Xl = X.reshape(math.prod(n[:d - 1]), n[d - 1])
    cores.append((left.T @ Xl)[:, :, None])
    return cores


def spectral_init(idx, y, n, r):
    """TT-SVD of the rescaled zero-filled observations p^{-1} P_Omega(y)
    (BASELINE.json:7).  Dense: small tensors only."""
    X = np.zeros(n)
    X[tuple(np.asarray(idx).T)] = y
    p = len(y) / math.prod(n)
    return tt_svd(X / p, r)


def _qr_sweep_norm(cores):
    c = np.array(cores[0], dtype=np.float64)
    for k in range(1, len(cores) + 1):
        r0, nk, r1 = c.shape
        if k == len(cores):
            return float(np.linalg.norm(c))
        _, rr = np.linalg.qr(c.reshape(r0 * nk, r1))
        c = np.einsum("ab,bjc->ajc", rr, cores[k])


def tt_norm(cores) -> float:
    """||T||_F via a left QR sweep (the norm of the last core)."""
    return _qr_sweep_norm(cores)


def tt_add(a, b, beta=1.0):
    """Block TT of a + beta*b (ranks add)."""
    d = len(a)
    if d == 1:
        return [a[0] + beta * b[0]]
    out = []
    for k in range(d):
        ca, cb = a[k], b[k]
        if k == 0:
            out.append(np.concatenate([ca, beta * cb], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([ca, cb], axis=0))
        else:
            z = np.zeros((ca.shape[0] + cb.shape[0], ca.shape[1], ca.shape[2] + cb.shape[2]))
            z[:ca.shape[0], :, :ca.shape[2]] = ca
            z[ca.shape[0]:, :, ca.shape[2]:] = cb
            out.append(z)
    return out


def tt_diff_norm(a, b, relative=True) -> float:
    """||A - B||_F (relative to ||B||_F) as the norm of the block TT [A; -B] via a QR
    sweep — never by expanding <A,A> - 2<A,B> + <B,B>."""
    num = tt_norm(tt_add(a, b, -1.0))
    if not relative:
        return num
    den = tt_norm(b)
    return num / den if den > 0 else num


# --------------------------------------------------------------------------- sizes
def os_dim(n, r):
    """dim M_r = sum r_{k-1} n_k r_k - sum_{k=1}^{m-1} r_k^2."""
    return sum(r[k] * n[k] * r[k + 1] for k in range(len(n))) - sum(x * x for x in r[1:-1])


def os_to_m(n, r, os_ratio):
    """|Omega| = OS * dim M_r, rounded."""
    return int(round(os_ratio * os_dim(n, r)))
