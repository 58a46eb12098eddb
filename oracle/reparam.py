"""Orthogonal reparameterisations U and the slicing constants (§4.3).

TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np

from .numerics import sign_vector


def sylvester(d: int) -> np.ndarray:
    """Sylvester-type Hadamard matrix H_d by the recursion of PAPER.md §4.3.1:
    H_{2n} = [[H_n, H_n], [H_n, -H_n]], H_1 = (1).  Entries ±1, unnormalised."""
    if d < 1 or d & (d - 1):
        raise ValueError("Hadamard size must be a power of two (P:274)")
    h = np.ones((1, 1), dtype=np.float64)
    while h.shape[0] < d:
        h = np.block([[h, h], [h, -h]])
    return h


def hadamard_U(d: int, seed: int | None) -> np.ndarray:
    """U = D · H_d / sqrt(d): the random ±1 diagonal D multiplies H_d on the
    LEFT (reading R7: a right-side D is a no-op for every slice quantity), then the
    1/sqrt(d) normalisation makes U orthonormal.  ``seed=None`` gives D = I,
    the form of the worked example."""
    s = np.ones(d) if seed is None else sign_vector(seed, d)
    return (s[:, None] * sylvester(d)) / np.sqrt(d)


def pca(features: np.ndarray, center: bool = False):
    """PCA basis of calibration latents F in R^{(B·L) x d} (§4.3.2):
    eigendecomposition Sigma_F = U Λ U^T of the (uncentred by default, reading R20)
    second-moment matrix.  Columns sorted by descending eigenvalue, ties by lower
    index; each column's largest-magnitude entry made positive.  Returns (U, λ)."""
    F = np.asarray(features, dtype=np.float64)
    if center:
        F = F - F.mean(axis=0, keepdims=True)
    sigma = F.T @ F / F.shape[0]
    lam, vec = np.linalg.eigh(sigma)          # ascending
    order = sorted(range(lam.size), key=lambda i: (-lam[i], i))
    lam = lam[order]
    vec = vec[:, order]
    for c in range(vec.shape[1]):
        p = np.argmax(np.abs(vec[:, c]))
        if vec[p, c] < 0:
            vec[:, c] = -vec[:, c]
    return vec, lam


def pca_alpha(lam: np.ndarray, g: int) -> np.ndarray:
    """alpha_j = (sum of all eigenvalues) / (sum over slice j), j = 0..g-1.

    PAPER.md P:312-315 defines alpha as the *fraction* of variance in the first
    d/2 components and beta for the rest; Condition 1 needs
    alpha·||(cU)_0||^2 ≈ ||c||^2, i.e. the reciprocal (reading R3), and beta's sum
    is read from d/2+1 (reading R4).  g > 2 generalises to g equal slices."""
    lam = np.asarray(lam, dtype=np.float64)
    d = lam.size
    if d % g:
        raise ValueError("g must divide d")
    w = d // g
    total = lam.sum()
    return np.array([total / lam[j * w:(j + 1) * w].sum() for j in range(g)])


def uniform_alpha(g: int) -> np.ndarray:
    """alpha_j = g for identity and Hadamard ("easily determine alpha = 2" for g = 2)."""
    return np.full(g, float(g))
