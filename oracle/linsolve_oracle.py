"""TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.

numpy restatement of the reference's restarted GMRES (linsolve.cpp:19-121:
modified Gram-Schmidt, Givens rotations with the complex phase convention of
:76-82, back substitution :95-103, the final true residual :115-118,
including the reference's iteration-count convention: the converging inner
iteration is not added to `iterations`).  Used by tests/ to check gk_gmres.
"""
import numpy as np


def gmres(apply, b, tol=1e-6, restart=50, maxit=1000):
    if not tol > 0:
        raise ValueError("gmres: tol must be positive")
    b = np.asarray(b, dtype=complex)
    n = b.shape[0]
    info = {"converged": False, "iterations": 0, "residual": 0.0, "history": []}
    x = np.zeros(n, dtype=complex)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        info["converged"] = True
        return x, info
    V = np.zeros((n, restart + 1), dtype=complex)
    total = 0
    while total < maxit:
        r = b - apply(x)
        beta = np.linalg.norm(r)
        if beta / bnorm <= tol:
            info["converged"] = True
            break
        H = np.zeros((restart + 1, restart), dtype=complex)
        cs = np.zeros(restart, dtype=complex)
        sn = np.zeros(restart, dtype=complex)
        V[:, 0] = r / beta
        g = np.zeros(restart + 1, dtype=complex)
        g[0] = beta
        j = 0
        while j < restart and total < maxit:
            w = apply(V[:, j])
            for i in range(j + 1):
                H[i, j] = np.vdot(V[:, i], w)
                w = w - H[i, j] * V[:, i]
            H[j + 1, j] = np.linalg.norm(w)
            if abs(H[j + 1, j]) > 0:
                V[:, j + 1] = w / H[j + 1, j]
            for i in range(j):
                tmp = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + np.conj(cs[i]) * H[i + 1, j]
                H[i, j] = tmp
            h0, h1 = abs(H[j, j]), abs(H[j + 1, j])
            if h1 == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                d = np.hypot(h0, h1)
                cs[j] = h0 / d
                phase = 1.0 if h0 == 0.0 else H[j, j] / h0
                sn[j] = phase * np.conj(H[j + 1, j]) / d
            tmp = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0
            H[j, j] = tmp
            g1 = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            g[j + 1] = g1
            rel = abs(g[j + 1]) / bnorm
            info["history"].append(rel)
            if rel <= tol:
                j += 1
                break
            j += 1
            total += 1
        y = np.zeros(j, dtype=complex)
        for i in range(j - 1, -1, -1):
            s = g[i] - np.dot(H[i, i + 1:j], y[i + 1:j])
            if abs(H[i, i]) == 0.0:
                raise RuntimeError("gmres: breakdown (zero diagonal in Hessenberg)")
            y[i] = s / H[i, i]
        x = x + V[:, :j] @ y
        rel = np.linalg.norm(b - apply(x)) / bnorm
        info["residual"] = rel
        if rel <= tol:
            info["converged"] = True
            break
    info["iterations"] = total
    info["residual"] = np.linalg.norm(b - apply(x)) / bnorm
    if info["residual"] <= tol:
        info["converged"] = True
    return x, info
