"""Tucker-2 truncated HOSVD of a dense K x K convolution kernel.

P:L693: "proj is the truncated-HOSVD that truncates the smallest singular values of
mode-1 and mode-2 matricization ... Performing matrix SVD on T_(1) and T_(2) ...
truncating smallest singular values in Sigma_1 and Sigma_2, with TKD we can obtain
U_1, U_2 and the core", and Eq. tkd2 recovers the projected kernel.

Layouts follow the layer API (include/tdc.h): a dense kernel W is PyTorch-ordered
[N][C][K][K] (out, in, r, t); the factors are U_in [C][D1], U_out [N][D2] and the
core [D2][D1][K][K], so that

    W_hat[n,c,r,t] = sum_{a,q} U_out[n,q] core[q,a,r,t] U_in[c,a]          (Eq. tkd2)

The paper's mode-1 (C) and mode-2 (N) matricizations are T_(C) in R^{C x N K K} and
T_(N) in R^{N x C K K}.  Host-side weight preparation (like plan-time packing): fp64
numpy, not on the forward path.  ADMM training itself is out of scope.
"""
from __future__ import annotations

import numpy as np


def mode_n_matricize(t: np.ndarray, mode: int) -> np.ndarray:
    """Rows = dims[mode]; columns = the remaining indices flattened in ascending mode
    order, last fastest."""
    t = np.asarray(t)
    if not 0 <= mode < t.ndim:
        raise ValueError(f"mode {mode} out of range for a {t.ndim}-d tensor")
    return np.moveaxis(t, mode, 0).reshape(t.shape[mode], -1)


def truncated_svd(m: np.ndarray, k: int):
    """Top-k singular triplets: (U rows x k, s descending, V cols x k)."""
    m = np.asarray(m, dtype=np.float64)
    if not 1 <= k <= min(m.shape):
        raise ValueError(f"k={k} outside [1, {min(m.shape)}]")
    u, s, vt = np.linalg.svd(m, full_matrices=False)
    return u[:, :k], s[:k], vt[:k].T


def tucker2_decompose(w: np.ndarray, d1: int, d2: int):
    """Truncated HOSVD of w [N][C][K][K] -> (core [D2][D1][K][K], u_in [C][D1], u_out [N][D2]).
    u_in / u_out are the top-d1 / top-d2 left singular vectors of the C- and N-mode
    matricizations; the core is w projected onto them."""
    w = np.asarray(w, dtype=np.float64)
    if w.ndim != 4 or w.shape[2] != w.shape[3]:
        raise ValueError("w must be [N][C][K][K]")
    N, C = w.shape[0], w.shape[1]
    if not (1 <= d1 <= C and 1 <= d2 <= N):
        raise ValueError(f"rank bounds violated: need 1 <= D1 <= C and 1 <= D2 <= N (D1={d1} C={C} D2={d2} N={N})")
    u_in, _, _ = truncated_svd(mode_n_matricize(w, 1), d1)    # C x (N K K)
    u_out, _, _ = truncated_svd(mode_n_matricize(w, 0), d2)   # N x (C K K)
    core = np.einsum("nq,ncrt,ca->qart", u_out, w, u_in)
    return core, u_in, u_out


def tucker2_reconstruct(core: np.ndarray, u_in: np.ndarray, u_out: np.ndarray) -> np.ndarray:
    """Eq. tkd2: W_hat[n,c,r,t] = sum_{a,q} U_out[n,q] core[q,a,r,t] U_in[c,a]."""
    return np.einsum("nq,qart,ca->ncrt", np.asarray(u_out, np.float64), np.asarray(core, np.float64),
                     np.asarray(u_in, np.float64))


def tail_energy_bound(w: np.ndarray, d1: int, d2: int) -> float:
    """HOSVD quasi-optimality: ||w - w_hat||_F <= sqrt(tail_C^2 + tail_N^2), the dropped
    singular values of the two matricizations."""
    w = np.asarray(w, dtype=np.float64)
    s1 = np.linalg.svd(mode_n_matricize(w, 1), compute_uv=False)
    s2 = np.linalg.svd(mode_n_matricize(w, 0), compute_uv=False)
    return float(np.sqrt(np.sum(s1[d1:] ** 2) + np.sum(s2[d2:] ** 2)))
