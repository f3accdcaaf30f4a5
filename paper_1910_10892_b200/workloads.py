"""Seeded synthetic inputs for the BASELINE.json configurations.

All arrays are numpy, in the reference layouts (unary [N*L], V [L*L], planes
[R/2*N]); there is no network, so every workload is synthetic.

  C1  ISGMR-4  288x384   L=16  K=5  stereo_like, truncated linear tau=2
  C2  TRWP-4   375x1242  L=192 K=5  stereo_like, truncated linear tau=2
  C3  ISGMR-8  500x750   L=128 K=5  stereo_like, truncated linear tau=2
  C4  TRWP-4   512x512   L=21  K=5  B=32, -logits, explicit 21x21 V, per-edge weights
  C5  ISGMR/TRWP 512x512 L=256 K=10 integer TQ denoising, V=min(d^2,200), w=25
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    engine: str          # "isgmr" | "trwp"
    H: int
    W: int
    L: int
    conn: int
    K: int
    B: int
    unary: np.ndarray    # [B, N*L] float32
    V: np.ndarray        # [L*L] float32
    w_const: float = 1.0
    w_planes: np.ndarray | None = None   # [B, R/2*N]
    rho_const: float = 0.5
    rho_planes: np.ndarray | None = None
    notes: dict = field(default_factory=dict)

    @property
    def N(self):
        return self.H * self.W


def truncated_linear(L: int, tau: float) -> np.ndarray:
    """build_pairwise(truncated_linear) (potentials.hpp:54-57): computed in
    double from |a-b|, cast to float."""
    d = np.abs(np.arange(L)[:, None] - np.arange(L)[None, :]).astype(np.float64)
    return np.minimum(d, tau).astype(np.float32).reshape(-1)


def truncated_quadratic(L: int, tau: float) -> np.ndarray:
    d = np.abs(np.arange(L)[:, None] - np.arange(L)[None, :]).astype(np.float64)
    return np.minimum(d * d, tau).astype(np.float32).reshape(-1)


def potts(L: int) -> np.ndarray:
    return (1.0 - np.eye(L)).astype(np.float32).reshape(-1)


def stereo_like(H: int, W: int, L: int, seed: int) -> np.ndarray:
    """acceptance.cpp:133-153 generalised to H x W: a sinusoidal disparity
    ramp, theta = |l - d| + U[0,3) noise."""
    rng = np.random.default_rng(seed)
    ph, pw = rng.uniform(0.0, 6.28, 2)
    h = np.arange(H)[:, None]
    w = np.arange(W)[None, :]
    d = 0.5 * (L - 1) * (1.0 + 0.8 * np.sin(2 * np.pi * w / W + pw) * np.cos(2 * np.pi * h / H + ph))
    lab = np.arange(L)[None, None, :]
    un = np.abs(lab - d[:, :, None]) + rng.uniform(0.0, 3.0, (H, W, L))
    return un.astype(np.float32).reshape(-1)


def random_problem(H, W, L, conn, seed, per_edge=False, explicit=True, w_const=None):
    """tests/oracles.hpp:114-137 recipe (numpy RNG): U[0,10) unaries, U[0,3)
    table with zero diagonal, U(0.1,2) per-edge planes or U(0.2,2) constant."""
    rng = np.random.default_rng(seed)
    un = rng.uniform(0.0, 10.0, H * W * L).astype(np.float32)
    if explicit:
        V = rng.uniform(0.0, 3.0, (L, L)).astype(np.float32)
        np.fill_diagonal(V, 0.0)
        V = V.reshape(-1)
    else:
        V = truncated_linear(L, 2.0)
    planes = None
    if per_edge:
        planes = rng.uniform(0.1, 2.0, (conn // 2) * H * W).astype(np.float32)
        wc = 1.0
    else:
        wc = float(np.float32(rng.uniform(0.2, 2.0))) if w_const is None else w_const
    return un, V, wc, planes


def config(name: str, batch: int | None = None, engine: str | None = None, first: int = 0,
           seed_offset: int = 0) -> Workload:
    """Full-size workload for configs C1..C5 (engine override for C5).
    C4: images first .. first+batch-1 of the seeded batch (a rank's shard;
    the pairwise table is shared by every image). seed_offset gives C1-C3 and
    C5 a different image per rank (weak scaling)."""
    name = name.upper()
    if name == "C1":
        H, W, L = 288, 384, 16
        return Workload("C1", "isgmr", H, W, L, 4, 5, 1, stereo_like(H, W, L, 1 + seed_offset)[None],
                        truncated_linear(L, 2.0))
    if name == "C2":
        H, W, L = 375, 1242, 192
        return Workload("C2", "trwp", H, W, L, 4, 5, 1, stereo_like(H, W, L, 2 + seed_offset)[None],
                        truncated_linear(L, 2.0))
    if name == "C3":
        H, W, L = 500, 750, 128
        return Workload("C3", "isgmr", H, W, L, 8, 5, 1, stereo_like(H, W, L, 3 + seed_offset)[None],
                        truncated_linear(L, 2.0))
    if name == "C4":
        B = 32 if batch is None else batch
        return seg_batch(512, 512, 21, B, seed0=100, first=first)
    if name == "C5":
        eng = engine or "isgmr"
        H = W = 512
        L = 256
        un = denoise_tq(H, W, L, seed=5 + seed_offset)
        return Workload("C5", eng, H, W, L, 4, 10, 1, un[None], truncated_quadratic(L, 200.0), w_const=25.0)
    raise ValueError(name)


def seg_batch(H, W, L, B, seed0=100, conn=4, K=5, first=0) -> Workload:
    """C4: unary = -logits, logits ~ N(0, 3^2); V explicit U[0,2) with zero
    diagonal (gradcheck.hpp:51-55 recipe); per-edge weights 1 - |e_i - e_j|
    from a seeded binary edge map. Image b of the batch
    is seeded seed0 + b; this returns images first .. first+B-1."""
    un = np.empty((B, H * W * L), np.float32)
    planes = np.empty((B, (conn // 2) * H * W), np.float32)
    for b in range(B):
        rng = np.random.default_rng(seed0 + first + b)
        un[b] = (-rng.normal(0.0, 3.0, H * W * L)).astype(np.float32)
        e = (rng.uniform(size=(H, W)) < 0.1).astype(np.float32)
        pl = np.ones((conn // 2, H, W), np.float32)
        # family 0: E/W, tail = left node; family 1: S/N, tail = upper node
        pl[0, :, :-1] = 1.0 - np.abs(e[:, 1:] - e[:, :-1])
        pl[1, :-1, :] = 1.0 - np.abs(e[1:, :] - e[:-1, :])
        if conn >= 8:
            pl[2, :-1, :-1] = 1.0 - np.abs(e[1:, 1:] - e[:-1, :-1])
            pl[3, :-1, 1:] = 1.0 - np.abs(e[1:, :-1] - e[:-1, 1:])
        planes[b] = pl.reshape(-1)
    rng = np.random.default_rng(seed0 - 1)
    V = rng.uniform(0.0, 2.0, (L, L)).astype(np.float32)
    np.fill_diagonal(V, 0.0)
    return Workload("C4", "trwp", H, W, L, conn, K, B, un, V.reshape(-1), w_planes=planes)


def denoise_tq(H, W, L, seed=5) -> np.ndarray:
    """C5: piecewise-constant image in [0,255] + N(0,20^2), rounded/clamped;
    theta = (I - l)^2 untruncated (io.hpp:73-89 TQ form)."""
    rng = np.random.default_rng(seed)
    img = np.zeros((H, W))
    for _ in range(12):
        y0, x0 = rng.integers(0, H), rng.integers(0, W)
        y1, x1 = min(H, y0 + rng.integers(32, 256)), min(W, x0 + rng.integers(32, 256))
        img[y0:y1, x0:x1] = rng.integers(0, 256)
    noisy = np.clip(np.rint(img + rng.normal(0.0, 20.0, (H, W))), 0, 255)
    lab = np.arange(L)[None, :]
    d = noisy.reshape(-1)[:, None] - lab
    return (d * d).astype(np.float32).reshape(-1)


def label_updates(H, W, conn, L, K, total_edges) -> int:
    """LU = K * sum_r |E^r| * L per image."""
    return K * total_edges * L
