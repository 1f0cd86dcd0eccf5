"""Seeded synthetic density pairs for the five BASELINE.json configs.

The reference ships no data (DOTmark and the paper's "cat" image are absent,
SURVEY.md §4/§8d), so these generators stand in for the paper's inputs with
the shapes, sizes and value distributions BASELINE.json names.  Densities are
cell-centred M x M images (pixel (c, r) centred at ((c+0.5)/M, (r+0.5)/M)),
each normalised to total mass 1; the solver-side source for a grid with N = M
cells is built by ``ml_sources`` / the device restriction kernels with the
frozen rule of SURVEY D2/D4:

  * coarse images are 2x2 block sums of the finer image,
  * node value = mean of the cells touching the node,
  * rho = (a / sum a - b / sum b) / h^2, minus its compensated mean.

Config 1 is the exception: its two Gaussians are evaluated at the nodes
(i h, j h) directly (BASELINE.json configs[0]).

Everything is numpy float64 with ``numpy.random.default_rng(seed)``; the same
seed always gives bit-identical images.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "config1_source",
    "gaussian_mixture_image",
    "blurred_noise_image",
    "anisotropic_mixture_image",
    "config2_images",
    "config3_images",
    "config4_pair",
    "config5_images",
    "dirac_pair_source",
    "make_source",
    "image_to_nodes",
    "block_sum",
    "ml_sources",
    "synth_instance",
    "SYNTH_KINDS",
]


def _fsum_normalise(a: np.ndarray) -> np.ndarray:
    # numpy's pairwise sum: deterministic for a given shape; the exact
    # normalisation happens later in make_source.
    return a / float(np.sum(a))


def make_source(a_nodes: np.ndarray, b_nodes: np.ndarray, n: int) -> np.ndarray:
    """rho = (a/sum a - b/sum b)/h^2 with the compensated mean removed
    (SPEC.md:477-483 make_source).  Uses math.fsum for the
    normalisers and the mean so the result does not depend on summation
    order."""
    h = 1.0 / n
    h2 = h * h
    a = np.asarray(a_nodes, dtype=np.float64)
    b = np.asarray(b_nodes, dtype=np.float64)
    sa = math.fsum(a.ravel().tolist())
    sb = math.fsum(b.ravel().tolist())
    rho = (a / sa - b / sb) / h2
    mean = math.fsum(rho.ravel().tolist()) / rho.size
    return rho - mean


def image_to_nodes(img: np.ndarray) -> np.ndarray:
    """Cell image (n x n) -> node values ((n+1) x (n+1)): mean of touching
    cells, evaluated as 0.25*((a+b)+(c+d)) / 0.5*(a+b) / a like the oracle."""
    img = np.asarray(img, dtype=np.float64)
    n = img.shape[0]
    out = np.empty((n + 1, n + 1))
    out[1:n, 1:n] = 0.25 * ((img[:-1, :-1] + img[:-1, 1:]) + (img[1:, :-1] + img[1:, 1:]))
    out[1:n, 0] = 0.5 * (img[:-1, 0] + img[1:, 0])
    out[1:n, n] = 0.5 * (img[:-1, n - 1] + img[1:, n - 1])
    out[0, 1:n] = 0.5 * (img[0, :-1] + img[0, 1:])
    out[n, 1:n] = 0.5 * (img[n - 1, :-1] + img[n - 1, 1:])
    out[0, 0] = img[0, 0]
    out[0, n] = img[0, n - 1]
    out[n, 0] = img[n - 1, 0]
    out[n, n] = img[n - 1, n - 1]
    return out


def block_sum(img: np.ndarray) -> np.ndarray:
    """2x2 block sums (r0[0]+r0[1]) + (r1[0]+r1[1])."""
    return (img[0::2, 0::2] + img[0::2, 1::2]) + (img[1::2, 0::2] + img[1::2, 1::2])


def ml_sources(img0: np.ndarray, img1: np.ndarray, levels: int) -> list[np.ndarray]:
    """Per-level node sources, coarse -> fine (list of (n_l+1)^2 arrays)."""
    a = np.asarray(img0, dtype=np.float64)
    b = np.asarray(img1, dtype=np.float64)
    out = []
    for l in range(levels):
        n = a.shape[0]
        out.append(make_source(image_to_nodes(a), image_to_nodes(b), n))
        if l + 1 < levels:
            a, b = block_sum(a), block_sum(b)
    return out[::-1]


# ---------------------------------------------------------------------------
# Config 1: two isotropic Gaussians at the nodes, N = 64.


def _gauss_nodes(n: int, cx: float, cy: float, sigma: float) -> np.ndarray:
    t = np.arange(n + 1) / n
    X, Y = np.meshgrid(t, t, indexing="xy")
    return np.exp(-((X - cx) ** 2 + (Y - cy) ** 2) / (2.0 * sigma * sigma))


def config1_source(n: int = 64) -> np.ndarray:
    """BASELINE.json configs[0]: rho0 ~ N((0.3,0.3), 0.10), rho1 ~ N((0.7,0.6), 0.08)
    at the nodes, each + 1e-8 and normalised to sum 1; rho = (a-b)/h^2."""
    a = _fsum_normalise(_gauss_nodes(n, 0.3, 0.3, 0.10) + 1e-8)
    b = _fsum_normalise(_gauss_nodes(n, 0.7, 0.6, 0.08) + 1e-8)
    return make_source(a, b, n)


def dirac_pair_source(n: int, a=(0, 0), b=None) -> np.ndarray:
    """Unit point masses at node a and node b (default (n, 0)): W1 = |a-b| h."""
    if b is None:
        b = (n, 0)
    A = np.zeros((n + 1, n + 1))
    B = np.zeros((n + 1, n + 1))
    A[a[1], a[0]] = 1.0
    B[b[1], b[0]] = 1.0
    return make_source(A, B, n)


# ---------------------------------------------------------------------------
# Config 2: 5-component isotropic Gaussian mixtures on a cell-centred image.


def gaussian_mixture_image(m: int, rng: np.random.Generator, k: int = 5) -> np.ndarray:
    centres = rng.uniform(0.15, 0.85, size=(k, 2))
    sig = rng.uniform(0.03, 0.12, size=k)
    w = rng.exponential(1.0, size=k)
    w = w / w.sum()  # Dirichlet(1)
    t = (np.arange(m) + 0.5) / m
    X, Y = np.meshgrid(t, t, indexing="xy")
    img = np.zeros((m, m))
    for c in range(k):
        img += w[c] / (2 * np.pi * sig[c] ** 2) * np.exp(
            -((X - centres[c, 0]) ** 2 + (Y - centres[c, 1]) ** 2) / (2 * sig[c] ** 2)
        )
    return _fsum_normalise(img)


def config2_images(seed: int = 2, m: int = 256):
    rng = np.random.default_rng(seed)
    return gaussian_mixture_image(m, rng), gaussian_mixture_image(m, rng)


# ---------------------------------------------------------------------------
# Config 3/4: blurred uniform noise, exponentiated.

_BLUR_CACHE: dict = {}


def _blur_matrix(m: int, sigma: float) -> np.ndarray:
    """Dense (m x m) operator of a 1D Gaussian blur, kernel truncated at 4 sigma,
    weights normalised to 1, boundary 'reflect' (half-sample symmetric:
    ... c b a | a b c ...), as scipy.ndimage.gaussian_filter's default."""
    key = (m, sigma)
    if key in _BLUR_CACHE:
        return _BLUR_CACHE[key]
    r = int(4.0 * sigma + 0.5)
    x = np.arange(-r, r + 1)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    k /= k.sum()
    B = np.zeros((m, m))
    for i in range(m):
        for t, wk in zip(x, k):
            j = i + t
            # half-sample symmetric reflection, repeated for |t| > m
            while j < 0 or j >= m:
                j = -j - 1 if j < 0 else 2 * m - j - 1
            B[i, j] += wk
    _BLUR_CACHE[key] = B
    return B


def blurred_noise_images(seeds, m: int = 512, sigma: float = 8.0, gain: float = 4.0,
                         floor: float = 1e-6) -> np.ndarray:
    """Batch version of ``blurred_noise_image``: returns (len(seeds), m, m)."""
    B = _blur_matrix(m, sigma)
    noise = np.stack([np.random.default_rng(int(s)).random((m, m)) for s in seeds])
    blurred = np.matmul(np.matmul(B, noise), B.T)
    img = np.exp(gain * blurred) + floor
    sums = img.reshape(img.shape[0], -1).sum(axis=1)
    return img / sums[:, None, None]


def blurred_noise_image(seed: int, m: int = 512, sigma: float = 8.0, gain: float = 4.0,
                        floor: float = 1e-6) -> np.ndarray:
    """BASELINE.json configs[2]: U[0,1] noise on m x m, Gaussian blur sigma=8 px
    (reflect boundary), exp(gain * x) + floor, normalised to sum 1."""
    return blurred_noise_images([seed], m, sigma, gain, floor)[0]


def config3_images(m: int = 512):
    return blurred_noise_image(0, m), blurred_noise_image(1, m)


def config4_pair(i: int, m: int = 512):
    """Pair i of BASELINE.json configs[3]: seeds (2i, 2i+1)."""
    return blurred_noise_image(2 * i, m), blurred_noise_image(2 * i + 1, m)


def config4_pairs(first: int, count: int, m: int = 512):
    """Pairs first..first+count-1 as two (count, m, m) arrays."""
    seeds0 = [2 * i for i in range(first, first + count)]
    seeds1 = [2 * i + 1 for i in range(first, first + count)]
    return blurred_noise_images(seeds0, m), blurred_noise_images(seeds1, m)


# ---------------------------------------------------------------------------
# Config 5: 20-component anisotropic Gaussian mixtures on 4096^2.


def anisotropic_mixture_image(m: int, rng: np.random.Generator, k: int = 20,
                              floor: float = 1e-9) -> np.ndarray:
    centres = rng.uniform(0.1, 0.9, size=(k, 2))
    theta = rng.uniform(0.0, np.pi, size=k)
    ev = rng.uniform(1e-4, 1e-2, size=(k, 2))
    w = rng.exponential(1.0, size=k)
    w = w / w.sum()
    t = (np.arange(m) + 0.5) / m
    img = np.zeros((m, m))
    X, Y = np.meshgrid(t, t, indexing="xy")
    for c in range(k):
        ct, st = np.cos(theta[c]), np.sin(theta[c])
        dx = X - centres[c, 0]
        dy = Y - centres[c, 1]
        u = ct * dx + st * dy
        v = -st * dx + ct * dy
        q = u * u / ev[c, 0] + v * v / ev[c, 1]
        img += w[c] / (2 * np.pi * np.sqrt(ev[c, 0] * ev[c, 1])) * np.exp(-0.5 * q)
    img = img / float(np.sum(img)) + floor
    return _fsum_normalise(img)


def config5_images(seed: int = 5, m: int = 4096):
    rng = np.random.default_rng(seed)
    return anisotropic_mixture_image(m, rng), anisotropic_mixture_image(m, rng)


SYNTH_KINDS = ("two_blobs", "annulus_pair", "dirac_pair", "config2", "config3")


def synth_instance(kind: str, n: int, seed: int = 0):
    """Two n x n cell images of a named synthetic family (SPEC.md synth_instance;
    stand-ins for the paper's DOTmark / two-circle / "cat" inputs): truncated
    Gaussian blobs, an annulus pair mimicking Fig. 3's circles, one-pixel
    Diracs at opposite corners of the bottom row, or the config-2/3 generators.
    Deterministic in (kind, n, seed)."""
    rng = np.random.default_rng(seed)
    t = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(t, t, indexing="xy")
    if kind == "two_blobs":
        c = rng.uniform(0.2, 0.8, size=(2, 2))
        a = np.exp(-((X - c[0, 0]) ** 2 + (Y - c[0, 1]) ** 2) / (2 * 0.08 ** 2))
        b = np.exp(-((X - c[1, 0]) ** 2 + (Y - c[1, 1]) ** 2) / (2 * 0.08 ** 2))
    elif kind == "annulus_pair":
        r = np.hypot(X - 0.5, Y - 0.5)
        a = np.exp(-((r - 0.15) / 0.03) ** 2)
        b = np.exp(-((r - 0.35) / 0.03) ** 2)
    elif kind == "dirac_pair":
        a = np.zeros((n, n))
        b = np.zeros((n, n))
        a[0, 0] = 1.0
        b[0, n - 1] = 1.0
    elif kind == "config2":
        a, b = config2_images(seed=seed, m=n)
    elif kind == "config3":
        a = blurred_noise_image(2 * seed, m=n)
        b = blurred_noise_image(2 * seed + 1, m=n)
    else:
        raise ValueError(f"unknown instance kind {kind!r}")
    return a, b
