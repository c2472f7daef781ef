"""CPU prototype of the partitioned single-matrix path: the orchestration of
paper_2504_19171_b200/partition.py driven by a dense numpy engine (test
infrastructure, like plan_sim.py).  Every numeric step is plain dense linear
algebra on the rank's local system, so the prototype checks the ORDERING and
REDUCTION algebra (separators, arrow-tip Schur complements, border
replacement, logdet split) against the oracle without a GPU."""
import numpy as np


def _dense_from_tiles(n, b, ti, tj, pay):
    k = (n + b - 1) // b
    M = np.zeros((k * b, k * b))
    for i, j, t in zip(ti, tj, pay):
        t = np.asarray(t).reshape(b, b)
        if i == j:
            t = np.tril(t)
            M[i * b:(i + 1) * b, j * b:(j + 1) * b] = t + np.tril(t, -1).T
        else:
            M[i * b:(i + 1) * b, j * b:(j + 1) * b] = t
            M[j * b:(j + 1) * b, i * b:(i + 1) * b] = t.T
    for r in range(n, k * b):
        M[r, r] = 1.0
    return M


class _Factor:
    def __init__(self, L, n, b):
        self.L, self.n, self.b = L, n, b


class NumpyEngine:
    def factorize(self, n, b, ti, tj, pay):
        M = _dense_from_tiles(n, b, ti, tj, pay)
        return _Factor(np.linalg.cholesky(M), n, b)

    def factor_logdet(self, f):
        return 2.0 * float(np.log(np.diag(f.L)[:f.n]).sum())

    def factor_tiles(self, f, coords):
        b = f.b
        return np.stack([f.L[i * b:(i + 1) * b, j * b:(j + 1) * b] for i, j in coords])

    def gram(self, L):
        return L @ L.T

    def inverse(self, E, b):
        return np.linalg.inv(E)

    def cholesky(self, F, b):
        return np.linalg.cholesky(F)

    def replace_and_invert(self, f, coords, tiles):
        b = f.b
        L = f.L.copy()
        for (i, j), t in zip(coords, tiles):
            L[i * b:(i + 1) * b, j * b:(j + 1) * b] = t
        Li = np.linalg.inv(L)
        Sig = Li.T @ Li
        k = L.shape[0] // b
        out = {(i, j): Sig[i * b:(i + 1) * b, j * b:(j + 1) * b] for j in range(k) for i in range(j, k)}
        return out, np.diag(Sig)[:f.n]

    def reduced_inverse(self, S, b):
        sign, ld = np.linalg.slogdet(S)
        assert sign > 0
        return np.linalg.inv(S), float(ld)
