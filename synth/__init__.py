"""Seeded synthetic inputs for the five BASELINE.json workloads.

This module is SHARED INPUT, not shared code: it only draws random numbers and
places them into arrays (ground-truth TT cores, observed multi-indices, unit
noise draws, init perturbations).  It contains none of the PRGD arithmetic
(no evaluation of a TT at Omega, no QR/SVD, no weights, no projection).  The
observed values y = T*(Omega) + noise are formed by the consumer: tests use
the oracle's evaluator, bench.py uses the library's tt_eval_at.

Recipes (BASELINE.json:7-11):
  cfg1  d=3, n=20^3, r=(1,2,2,1), Gaussian cores N(0,1)/sqrt(r_k), 2400 of 8000
        entries without replacement, no noise, spectral init (TT-SVD of the
        rescaled zero-filled observations, done by the consumer).
  cfg2  d=4, n=50^4, r=(1,5,5,5,1), Gaussian cores, 312,500 entries (5%) without
        replacement, noise sigma = 1e-3 * RMS.
  cfg3  256x256x128 sum of 16 separable cosines (f ~ U[0,4], theta ~ U[0,2pi)),
        held as its exact CP->TT form with ranks (1,16,16,1), 838,861 entries
        (10%), absolute noise sigma = 0.01.
  cfg4  d=24 binary modes, real random MPS of bond 8 (Gaussian cores scaled to
        unit 2-norm), ranks min(8, 2^k, 2^(24-k)), 1,677,722 entries (10%), no
        noise.
  cfg5  d=10, n=16^10, r=16 interior, Gaussian cores, 3e7 uniform draws of the
        40-bit code with duplicates removed keeping first occurrence (sample
        order left random), noise sigma = 1e-4 * RMS.

Beyond BASELINE's five (the paper's QST workload shape):
  cfg6  Pauli-measurement tensor of n = 10 qubits: a random complex MPS u of bond 2
        (complex Gaussian cores, normalised so tr(rho) = ||u||^2 = 1), rho = u u^dagger,
        T*(a) = sum_{i,j} rho(i, j) W_a(i, j) with W_a = sigma_{a_1} x ... x sigma_{a_n}
        (Y_k(:, alpha, :) = sum_{i,j} X_k(:, i, j, :) sigma_alpha(i, j)), held as a
        REAL TT of ranks s_k^2 = 4 (mode size 4) by writing each bond's Hermitian s x s
        environment in an orthonormal Hermitian basis; OS = 200 (80,000 of 4^10 = 7.63%,
        PAPER.md:635) without replacement, no noise, perturbed-truth init.

RMS for relative noise is the root mean square of the clean observed values
(an unbiased estimate of ||T*||_F / sqrt(N*) under uniform sampling); the
consumer computes it, since it needs T*(Omega).

Init for cfg2-5 is the ground truth with each core perturbed by Gaussian noise
of relative size 0.1/sqrt(d) (a "good initialisation"); cfg1 uses
the spectral init BASELINE.json:7 prescribes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

BASE_SEED = 2501_13385


@dataclass
class Problem:
    cfg: int
    n: tuple
    r: tuple
    truth: List[np.ndarray]           # ground-truth cores [r_{k-1}, n_k, r_k]
    idx: np.ndarray                   # int32 [M, d], 0-based, sample order random
    noise_unit: Optional[np.ndarray]  # float64 [M] standard normal draws, or None
    noise_kind: Optional[str]         # None | "rel" | "abs"
    noise_sigma: float
    init: Optional[List[np.ndarray]]  # perturbed truth, or None (spectral init)
    iters: int
    meta: dict = field(default_factory=dict)

    @property
    def d(self):
        return len(self.n)

    @property
    def m(self):
        return int(self.idx.shape[0])

    @property
    def nstar(self):
        return math.prod(self.n)

    def observations(self, clean: np.ndarray) -> np.ndarray:
        """y = clean + noise, given the clean values T*(Omega) (consumer-computed)."""
        clean = np.asarray(clean, dtype=np.float64)
        if self.noise_kind is None:
            return clean.copy()
        if self.noise_kind == "abs":
            scale = self.noise_sigma
        else:
            rms = math.sqrt(float(np.mean(clean * clean))) if clean.size else 0.0
            scale = self.noise_sigma * rms
        return clean + scale * self.noise_unit


def mps_ranks(d: int, bond: int, n: int = 2) -> tuple:
    r = [1]
    for k in range(1, d):
        r.append(int(min(bond, n ** k, n ** (d - k))))
    r.append(1)
    return tuple(r)


def _unravel(lin: np.ndarray, n: tuple) -> np.ndarray:
    """Linear index (x_1 most significant) -> int32 multi-index [M, d]."""
    out = np.empty((lin.shape[0], len(n)), dtype=np.int32)
    rem = lin.astype(np.int64, copy=True)
    for k in range(len(n) - 1, -1, -1):
        out[:, k] = rem % n[k]
        rem //= n[k]
    return out


def _gaussian_cores(rng, n, r, scale_by_rank=True):
    cores = []
    for k in range(len(n)):
        c = rng.standard_normal((r[k], n[k], r[k + 1]))
        if scale_by_rank:
            c /= math.sqrt(r[k + 1])
        cores.append(c)
    return cores


def _perturb(rng, cores, rel):
    out = []
    for c in cores:
        z = rng.standard_normal(c.shape)
        s = np.linalg.norm(c) / math.sqrt(c.size)
        out.append(c + rel * s * z)
    return out


def _sq_norm_tt(cores):
    """||T||_F^2 by the plain Gram recursion; used only to scale cfg4's input state."""
    g = np.ones((1, 1))
    for c in cores:
        g = np.einsum("ab,axc,byd->cd", g, c, c)
    return float(g[0, 0])


def make_problem(cfg: int, seed: Optional[int] = None, m: Optional[int] = None,
                 n: Optional[tuple] = None, r: Optional[tuple] = None, rank: int = 0,
                 world: int = 1) -> Problem:
    """Build config `cfg` (1..5, and 6 = the QST workload shape).  `m`, `n`, `r` override sizes for reduced test
    variants (same recipe, same value distributions).  With world > 1 (config 5, sharded
    multi-GPU runs) the truth and the init are those of `seed`, and rank `rank` draws its
    own m multi-indices from the residue class lin = rank (mod world) of the linear index,
    so the ranks' sets are disjoint and their union is uniform (weak scaling)."""
    if seed is None:
        seed = BASE_SEED + cfg
    rng = np.random.Generator(np.random.PCG64(seed))
    meta = {"seed": seed}
    if cfg == 1:
        n = n or (20, 20, 20)
        r = r or (1, 2, 2, 1)
        nstar = math.prod(n)
        m = m if m is not None else int(round(0.3 * nstar))
        truth = _gaussian_cores(rng, n, r)
        idx = _unravel(rng.choice(nstar, size=m, replace=False), n)
        return Problem(cfg, n, r, truth, idx, None, None, 0.0, None, 100, meta)
    if cfg == 2:
        n = n or (50, 50, 50, 50)
        r = r or (1, 5, 5, 5, 1)
        nstar = math.prod(n)
        m = m if m is not None else int(round(0.05 * nstar))
        truth = _gaussian_cores(rng, n, r)
        idx = _unravel(rng.choice(nstar, size=m, replace=False), n)
        z = rng.standard_normal(m)
        init = _perturb(rng, truth, 0.1 / math.sqrt(len(n)))
        return Problem(cfg, n, r, truth, idx, z, "rel", 1e-3, init, 200, meta)
    if cfg == 3:
        n = n or (256, 256, 128)
        ncomp = 16
        r = r or (1, ncomp, ncomp, 1)
        nstar = math.prod(n)
        m = m if m is not None else int(round(0.1 * nstar))
        f = rng.uniform(0.0, 4.0, size=(ncomp, 3))
        th = rng.uniform(0.0, 2.0 * math.pi, size=(ncomp, 3))
        fac = [np.cos(2.0 * math.pi * f[:, k][None, :] * np.arange(n[k])[:, None] / n[k]
                      + th[:, k][None, :]) for k in range(3)]          # [n_k, ncomp]
        t1 = fac[0][None, :, :].copy()                                   # [1, n1, C]
        t2 = np.zeros((ncomp, n[1], ncomp))
        for c in range(ncomp):
            t2[c, :, c] = fac[1][:, c]
        t3 = fac[2].T[:, :, None].copy()                                 # [C, n3, 1]
        truth = [t1, t2, t3]
        idx = _unravel(rng.choice(nstar, size=m, replace=False), n)
        z = rng.standard_normal(m)
        init = _perturb(rng, truth, 0.1 / math.sqrt(3))
        meta.update(freq=f, phase=th)
        return Problem(cfg, n, r, truth, idx, z, "abs", 0.01, init, 100, meta)
    if cfg == 4:
        d = 24 if n is None else len(n)
        n = n or (2,) * d
        r = r or mps_ranks(d, 8)
        nstar = math.prod(n)
        m = m if m is not None else int(round(0.1 * nstar))
        truth = _gaussian_cores(rng, n, r, scale_by_rank=False)
        s = _sq_norm_tt(truth) ** (-0.5 / d)
        truth = [c * s for c in truth]
        idx = _unravel(rng.choice(nstar, size=m, replace=False), n)
        init = _perturb(rng, truth, 0.1 / math.sqrt(d))
        return Problem(cfg, n, r, truth, idx, None, None, 0.0, init, 100, meta)
    if cfg == 5:
        d = 10 if n is None else len(n)
        n = n or (16,) * d
        r = r or (1,) + (16,) * (d - 1) + (1,)
        truth = _gaussian_cores(rng, n, r)
        nstar = math.prod(n)
        draws = 30_000_000 if m is None else m
        if world > 1:
            rr = np.random.Generator(np.random.PCG64([seed, 1 + rank]))
            codes = rr.integers(0, (nstar - rank + world - 1) // world, size=draws,
                                dtype=np.int64) * world + rank
        else:
            codes = rng.integers(0, nstar, size=draws, dtype=np.int64)
        _, first = np.unique(codes, return_index=True)
        first.sort()                       # keep first occurrence, original (random) order
        codes = codes[first]
        idx = _unravel(codes, n)
        if world > 1:
            z = rr.standard_normal(idx.shape[0])
            rng = np.random.Generator(np.random.PCG64([seed, 0]))
        else:
            z = rng.standard_normal(idx.shape[0])
        init = _perturb(rng, truth, 0.1 / math.sqrt(d))
        meta.update(draws=draws, duplicates=draws - idx.shape[0], rank=rank, world=world)
        return Problem(cfg, n, r, truth, idx, z, "rel", 1e-4, init, 50, meta)
    if cfg == 6:
        d = 10 if n is None else len(n)
        n = (4,) * d
        s_b = mps_ranks(d, 2)                                  # bond dims of the state, qubits
        r = tuple(b * b for b in s_b)
        truth, mps = _pauli_tt(rng, s_b)
        nstar = math.prod(n)
        if m is None:   # OS = 200 x manifold dimension
            dim = sum(r[k] * n[k] * r[k + 1] for k in range(d)) - sum(r[k] ** 2 for k in range(1, d))
            m = 200 * dim
        idx = _unravel(rng.choice(nstar, size=m, replace=False), n)
        init = _perturb(rng, truth, 0.1 / math.sqrt(d))
        meta.update(state_bond=s_b, mps=mps)
        return Problem(cfg, n, r, truth, idx, None, None, 0.0, init, 200, meta)
    raise ValueError(f"unknown config {cfg}")


# Pauli matrices in the paper's order sigma_1..sigma_4 = I, X, Y, Z
PAULI = np.array([[[1, 0], [0, 1]], [[0, 1], [1, 0]], [[0, -1j], [1j, 0]], [[1, 0], [0, -1]]],
                 dtype=np.complex128)


def _herm_basis(s: int) -> np.ndarray:
    """Orthonormal basis (under <A, B> = tr(A B)) of the real space of Hermitian s x s matrices:
    E_ii, (E_ij + E_ji)/sqrt(2), i(E_ij - E_ji)/sqrt(2) for i < j.  [s*s, s, s]."""
    out = []
    for i in range(s):
        e = np.zeros((s, s), dtype=np.complex128)
        e[i, i] = 1.0
        out.append(e)
    for i in range(s):
        for j in range(i + 1, s):
            e = np.zeros((s, s), dtype=np.complex128)
            e[i, j] = e[j, i] = 1.0 / math.sqrt(2.0)
            out.append(e)
            e = np.zeros((s, s), dtype=np.complex128)
            e[i, j], e[j, i] = 1j / math.sqrt(2.0), -1j / math.sqrt(2.0)
            out.append(e)
    return np.array(out)


def _pauli_tt(rng, s_b) -> List[np.ndarray]:
    """Real TT of the Pauli-measurement tensor of rho = u u^dagger (config 6).  With the left
    environment E_k = sum_{i,j} sigma_a(i,j) U_k(:,i,:)^T E_{k-1} conj(U_k(:,j,:)) (Hermitian,
    E_0 = [1], T*(a) = E_d), core k maps the real coordinates h_m = tr(B_m E_{k-1}) to those of
    E_k: core[m, a, q] = tr(B'_q F_a(B_m)), a real linear map since F_a keeps Hermiticity."""
    d = len(s_b) - 1
    U = [(rng.standard_normal((s_b[k], 2, s_b[k + 1])) + 1j * rng.standard_normal((s_b[k], 2, s_b[k + 1])))
         / math.sqrt(2.0) for k in range(d)]
    # ||u||^2 by the transfer-matrix recursion; scale so tr(rho) = 1
    g = np.ones((1, 1), dtype=np.complex128)
    for c in U:
        g = np.einsum("ab,aic,bid->cd", g, c, np.conj(c))
    U[0] = U[0] / math.sqrt(float(g[0, 0].real))
    cores = []
    for k in range(d):
        Bin, Bout = _herm_basis(s_b[k]), _herm_basis(s_b[k + 1])
        core = np.empty((Bin.shape[0], 4, Bout.shape[0]))
        for a in range(4):
            for mm in range(Bin.shape[0]):
                F = np.zeros((s_b[k + 1], s_b[k + 1]), dtype=np.complex128)
                for i in range(2):
                    for j in range(2):
                        if PAULI[a, i, j] != 0:
                            F += PAULI[a, i, j] * (U[k][:, i, :].T @ Bin[mm] @ np.conj(U[k][:, j, :]))
                core[mm, a, :] = np.einsum("qxy,yx->q", Bout, F).real
        cores.append(core)
    return cores, U
