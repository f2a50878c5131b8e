"""Brute-force references used to PIN the oracle (tests only).

Deliberately independent of oracle/: every quantity is computed entry by entry
from its definition in the paper, by loops over all multi-indices.  Tiny sizes
only (N* <= a few thousand)."""
from __future__ import annotations

import itertools
import math

import numpy as np


def entry(cores, x):
    """T(x) = T_1(x_1,:) T_2(:,x_2,:) ... T_d(:,x_d), one product."""
    v = np.ones((1, 1))
    for c, xk in zip(cores, x):
        v = v @ c[:, xk, :]
    return float(v[0, 0])


def dense(cores):
    n = tuple(c.shape[1] for c in cores)
    out = np.empty(n)
    for x in itertools.product(*[range(k) for k in n]):
        out[x] = entry(cores, x)
    return out


def jacobian(cores):
    """J[x, theta] = d T(x) / d theta over all core entries theta = (k, a, j, c):
    T^{<=k-1}(x)[a] * [x_k == j] * T^{>=k+1}(x)[c]."""
    n = tuple(c.shape[1] for c in cores)
    d = len(n)
    sizes = [c.size for c in cores]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    nstar = math.prod(n)
    J = np.zeros((nstar, int(offs[-1])))
    for lin, x in enumerate(itertools.product(*[range(k) for k in n])):
        for k in range(d):
            left = np.ones((1, 1))
            for i in range(k):
                left = left @ cores[i][:, x[i], :]
            right = np.ones((1, 1))
            for i in range(d - 1, k, -1):
                right = cores[i][:, x[i], :] @ right
            r0, nk, r1 = cores[k].shape
            block = np.zeros((r0, nk, r1))
            block[:, x[k], :] = np.outer(left[0], right[:, 0])
            J[lin, offs[k]:offs[k + 1]] = block.ravel()
    return J


def weight_diag(n, w, d):
    """Entry weights of W (`equ: new metric`):
    (W X)(x) = X(x) prod_k G_{l,k}^{1/(2m)}(x_k, x_k) = X(x) prod_k w_{k,x_k}^{1/(2d)}."""
    out = np.empty(n)
    for x in itertools.product(*[range(k) for k in n]):
        out[x] = np.prod([w[k][x[k]] ** (1.0 / (2 * d)) for k in range(d)])
    return out


def weighted_tangent_projection(cores, Dw, Z):
    """W-orthogonal projection of the dense tensor Z onto the tangent space at the
    TT point `cores` (range of the Jacobian): argmin_{t in range J} ||Z - t||_W,
    = J (J^T D J)^+ J^T D Z with D = diag(W)."""
    J = jacobian(cores)
    D = Dw.ravel()
    G = J.T @ (D[:, None] * J)
    theta = np.linalg.pinv(G, rcond=1e-12, hermitian=True) @ (J.T @ (D * Z.ravel()))
    return (J @ theta).reshape(Z.shape)


def sampled_dense(n, idx, vals):
    X = np.zeros(n)
    X[tuple(np.asarray(idx).T)] = vals
    return X
