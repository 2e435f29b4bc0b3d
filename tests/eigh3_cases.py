"""Symmetric 3x3 test matrices for the numpy.linalg.eigh restatement
(paper_2409_13418_b200/csrc/odc_eigh3.cuh): the QEF normal matrices of every
golden case (A = sum n n^T per partition, dualize.py:349-352) plus seeded
synthetic families that reach every branch of dsytd2/dsteqr/dormtr -- QL and
QR sweeps, 2x2 blocks (dlaev2), split blocks, zero reflectors, rank-1/2
sums of unit normals, near-axis normals, integer matrices and matrices
scaled into dsyevd's and dsteqr's rescaling ranges."""

import numpy as np

from golden_util import cases, load


def golden_qef_matrices():
    out = []
    for tag in cases():
        g = load(tag)
        n = np.asarray(g["normals"], dtype=np.float64).reshape(-1, 3)
        off = np.asarray(g["cyc_off"], dtype=np.int64)
        part = np.repeat(np.arange(len(off) - 1), np.diff(off))
        A = np.zeros((len(off) - 1, 3, 3))
        np.add.at(A, part, n[:, :, None] * n[:, None, :])
        out.append(A)
    return np.concatenate(out)


def synthetic(n, seed):
    rng = np.random.default_rng(seed)
    fam = []
    M = rng.standard_normal((n, 3, 3))
    fam.append(M + M.transpose(0, 2, 1))
    for k in (1, 2, 3, 4, 6, 12):
        N = rng.standard_normal((n, k, 3))
        N /= np.linalg.norm(N, axis=2, keepdims=True)
        fam.append(np.einsum("pki,pkj->pij", N, N))
    N = np.zeros((n, 4, 3))
    ax = rng.integers(0, 3, (n, 4))
    N[np.arange(n)[:, None], np.arange(4)[None], ax] = 1.0
    N += rng.standard_normal((n, 4, 3)) * 10.0 ** rng.integers(-16, -2, (n, 4, 1))
    N /= np.linalg.norm(N, axis=2, keepdims=True)
    fam.append(np.einsum("pki,pkj->pij", N, N))
    M = rng.integers(-3, 4, (n, 3, 3)).astype(np.float64)
    fam.append(M + M.transpose(0, 2, 1))
    base = np.concatenate(fam)
    m = min(n, 2000)
    extra = [base[:m] * s for s in (1e-300, 1e-200, 1e-160, 1e-150, 1e-130, 1e130, 1e200, 1e300)]
    B = base[:m].copy()
    B[:, 1, 0] = B[:, 0, 1] = 1e-310 * rng.standard_normal(m)
    B[:, 2, 0] = B[:, 0, 2] = 1e-312 * rng.standard_normal(m)
    extra.append(B)
    B = base[:m].copy()
    B[:, 2, 1] = B[:, 1, 2] = 1e-200 * rng.standard_normal(m)
    extra.append(B)
    B = np.zeros((m, 3, 3))
    B[:, 0, 0] = rng.standard_normal(m)
    B[:, 1, 1] = B[:, 2, 2] = 1e-170
    B[:, 1, 2] = B[:, 2, 1] = 3e-171
    extra.append(B)
    return np.ascontiguousarray(np.concatenate([base] + extra))
