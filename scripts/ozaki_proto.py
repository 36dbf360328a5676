"""Numerical prototype (CPU, fp64 BLAS) of the int8-sliced ("Ozaki") block sweep the GPU inverse
uses for its rank-128 updates: how many 7-bit slices S keep the damped inverse within the
1e-5 bound on the workload's real factors?  Experiment only -- not a test, not the oracle.

The sweep is the one in inverse.cu (block Gauss-Jordan, B = 128, P_k = M_KK^-1 in fp64):
    M_IJ -= R_I^T (P_k R_J)   with the product R_I^T Wp_J computed from int8 slices:
    column c of R (and of Wp) = sign * 2^e_c * sum_s d_s 2^-7(s+1), d_s in [0, 127],
    product = 2^(e_i + f_j) sum_{s+u <= S-1} 2^-7(s+u+2) (q_s^T r_u)   (exact integer sums)
Digit products are summed in fp64 BLAS, exact below 2^53.
"""
import sys
import time

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, "/root/repo")
from synth import inputs, shapes  # noqa: E402

B = 128


def factor_pair(cfg, name):
    layers, n = shapes.config(cfg)
    li = [l["name"] for l in layers].index(name)
    L = layers[li]
    x = inputs.layer_x(L, li, n).double()
    gy = inputs.layer_gy(L, li, n).double()
    if L["kind"] == 1:
        X = x
    else:
        xn = x.permute(0, 3, 1, 2)
        U = F.unfold(xn, (L["kh"], L["kw"]), padding=L["pad_h"], stride=L["stride_h"])  # [n, C*kh*kw, P]
        C = L["c_in"]
        U = U.view(n, C, L["kh"] * L["kw"], -1).permute(0, 3, 2, 1).reshape(-1, L["kh"] * L["kw"] * C)
        X = U
    if L["has_bias"]:
        X = torch.cat([X, torch.ones(X.shape[0], 1, dtype=X.dtype)], 1)
    rows = X.shape[0]
    A = (X.T @ X / rows).numpy()
    g = gy.reshape(-1, gy.shape[-1])
    G = (g.T @ g / rows).numpy()
    return A.astype(np.float32).astype(np.float64), G.astype(np.float32).astype(np.float64)


def slices(X, S):
    """X [K, N] -> digits q [S, K, N] (signed, |q| <= 127) and column exponents e [N]."""
    m = np.abs(X).max(axis=0)
    e = np.where(m > 0, np.frexp(m)[1], 0)  # m < 2^e
    Y = np.rint(np.abs(X) * np.ldexp(1.0, 7 * S - e)[None, :])
    Y = np.minimum(Y, 2.0 ** (7 * S) - 1)
    q = np.empty((S,) + X.shape)
    for s in range(S):
        sh = 7 * (S - 1 - s)
        q[s] = np.floor(Y / 2.0 ** sh) % 128
    return q * np.sign(X)[None], e


def oz_product(R, Wp, S):
    """R^T Wp through S-slice digits (pairs s + u <= S - 1)."""
    qa, ea = slices(R, S)
    qb, eb = slices(Wp, S)
    out = np.zeros((R.shape[1], Wp.shape[1]))
    for d in range(S):
        acc = np.zeros_like(out)
        for s in range(d + 1):
            acc += qa[s].T @ qb[d - s]  # exact: |acc| < 2^53
        out += np.ldexp(acc, -7 * (d + 2))
    return out * np.ldexp(1.0, ea)[:, None] * np.ldexp(1.0, eb)[None, :]


def sweep(M, S, panel_oz=False):
    W = M.copy()
    n = W.shape[0]
    nt = (n + B - 1) // B
    for k in range(nt):
        K = slice(k * B, min(n, (k + 1) * B))
        P = np.linalg.inv(W[K, K])
        R = W[K, :].copy()
        Wp = oz_product(P.T.copy(), R, S) if (S and panel_oz) else P @ R
        others = np.r_[0:k * B, min(n, (k + 1) * B):n]
        if S:
            W[np.ix_(others, others)] -= oz_product(R[:, others], Wp[:, others], S)
        else:
            W[np.ix_(others, others)] -= R[:, others].T @ Wp[:, others]
        W[K, others] = Wp[:, others]
        W[others, K] = Wp[:, others].T
        W[K, K] = -P
    return -W


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["l3b0c2"]
    gammas = [float(g) for g in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2.5e-2, 2.5e-4]
    Ss = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0, 4, 5, 6, 7]
    which_only = sys.argv[5] if len(sys.argv) > 5 else "AG"
    for name in names:
        A, G = factor_pair(cfg, name)
        for gamma in gammas:
            ta, tg = np.trace(A) / A.shape[0], np.trace(G) / G.shape[0]
            pi = np.sqrt(ta / tg)
            for which, (M, add) in (("A", (A, pi * np.sqrt(gamma))), ("G", (G, np.sqrt(gamma) / pi))):
                if which not in which_only:
                    continue
                Md = M + add * np.eye(M.shape[0])
                ref = np.linalg.inv(Md)
                kap = np.linalg.cond(Md)
                bound = (np.trace(Md)) / add
                res = []
                for S in Ss:
                    for poz in ((False, True) if S else (False,)):
                        X = sweep(Md, S, poz)
                        e = np.linalg.norm(X - ref) / np.linalg.norm(ref)
                        res.append(f"S={S}{'p' if poz else ''}:{e:.1e}")
                print(f"{name} {which} n={M.shape[0]} gamma={gamma:g} kappa={kap:.2e} tr/delta={bound:.2e} " + " ".join(res),
                      flush=True)


if __name__ == "__main__":
    main()
