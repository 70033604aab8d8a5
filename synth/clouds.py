"""Seeded synthetic point-cloud generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws fp32 coordinates.
Recipes:

* ``uniform``        X, Y i.i.d. U[0,1)^3, independent (Fig. 2's "synthetic random point
                     sets").
* ``shapenet``       gt = M samples of the surface of a union of 3-6 random primitives
                     (ellipsoid / box / cylinder surfaces), normalised to the unit sphere;
                     pred = N independent samples of the same surface + N(0, 0.01^2)
                     ("mid-training"); the ShapeNet-55 workload of P:201.
* ``near``           pred = permuted gt + N(0, (0.3 * spacing)^2)  (N == M).
* ``mmfi``           human of height U[1.6, 1.9] m built from 10 capsules with random joint
                     angles, sampled only on the sensor-facing half (LiDAR-like), metres;
                     pred = independent resample of the same body + 1 cm noise (MM-Fi).
* ``scene``          8 x 6 x 3 m room planes + 20 primitives; pred = resample + 5 mm jitter.

Every pair b of a batch uses its own Philox stream seeded (seed, b), so a pair's content is
independent of the batch size.
"""
from __future__ import annotations

import numpy as np

KINDS = ("uniform", "shapenet", "near", "mmfi", "scene")


def _rng(seed: int, b: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF, b]))


def _rot(rng) -> np.ndarray:
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def _sphere_dirs(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.maximum(np.linalg.norm(v, axis=1, keepdims=True), 1e-12)


# ---- primitive surfaces: each returns (sampler(rng, n) -> (n,3) local points, area)
def _ellipsoid(rng):
    ax = rng.uniform(0.2, 1.0, size=3)
    p = 1.6
    area = 4 * np.pi * (((ax[0] * ax[1]) ** p + (ax[0] * ax[2]) ** p + (ax[1] * ax[2]) ** p) / 3) ** (1 / p)
    return (lambda r, n: _sphere_dirs(r, n) * ax), area


def _box(rng):
    e = rng.uniform(0.2, 1.0, size=3)
    faces = np.array([e[1] * e[2], e[1] * e[2], e[0] * e[2], e[0] * e[2], e[0] * e[1], e[0] * e[1]])

    def s(r, n):
        f = r.choice(6, size=n, p=faces / faces.sum())
        u = r.uniform(-0.5, 0.5, size=(n, 3)) * e
        ax = f // 2
        u[np.arange(n), ax] = np.where(f % 2 == 0, -0.5, 0.5) * e[ax]
        return u
    return s, 2 * faces[::2].sum()


def _cylinder(rng):
    rad, h = rng.uniform(0.1, 0.5), rng.uniform(0.3, 1.2)
    lat, cap = 2 * np.pi * rad * h, np.pi * rad * rad

    def s(r, n):
        k = r.choice(3, size=n, p=np.array([lat, cap, cap]) / (lat + 2 * cap))
        t = r.uniform(0, 2 * np.pi, size=n)
        rr = np.where(k == 0, rad, rad * np.sqrt(r.uniform(size=n)))
        z = np.where(k == 0, r.uniform(-h / 2, h / 2, size=n), np.where(k == 1, -h / 2, h / 2))
        return np.stack([rr * np.cos(t), rr * np.sin(t), z], axis=1)
    return s, lat + 2 * cap


def _capsule(a, b, rad):
    """Capsule surface between endpoints a, b (world coordinates) with radius rad."""
    d = b - a
    L = np.linalg.norm(d)
    lat, caps = 2 * np.pi * rad * L, 4 * np.pi * rad * rad
    zax = d / max(L, 1e-9)
    tmp = np.array([1.0, 0, 0]) if abs(zax[0]) < 0.9 else np.array([0, 1.0, 0])
    xax = np.cross(zax, tmp); xax /= np.linalg.norm(xax)
    yax = np.cross(zax, xax)

    def s(r, n):
        lat_pick = r.uniform(size=n) < lat / (lat + caps)
        t = r.uniform(0, 2 * np.pi, size=n)
        z = r.uniform(0, L, size=n)
        pl = (np.cos(t) * rad)[:, None] * xax + (np.sin(t) * rad)[:, None] * yax + z[:, None] * zax
        dirs = _sphere_dirs(r, n) * rad
        up = (dirs @ zax) >= 0
        pc = dirs + np.where(up, L, 0.0)[:, None] * zax
        return a + np.where(lat_pick[:, None], pl, pc)
    return s, lat + caps


def _sample_union(rng, prims, n):
    areas = np.array([a for _, a in prims])
    counts = rng.multinomial(n, areas / areas.sum())
    out = [s(rng, k) for (s, _), k in zip(prims, counts) if k > 0]
    pts = np.concatenate(out, axis=0)
    return pts[rng.permutation(n)]


def _shape(rng):
    makers = (_ellipsoid, _box, _cylinder)
    prims = []
    for _ in range(int(rng.integers(3, 7))):
        s, a = makers[int(rng.integers(0, 3))](rng)
        R, t = _rot(rng), rng.uniform(-0.6, 0.6, size=3)
        prims.append(((lambda r, n, s=s, R=R, t=t: s(r, n) @ R.T + t), a))
    return prims


def _human(rng):
    h = rng.uniform(1.6, 1.9)
    u = h / 1.75

    def limb(start, length, theta, phi):
        d = np.array([np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi), -np.cos(theta)])
        return start, start + length * u * d

    j = lambda: rng.uniform(-0.6, 0.6)
    pelvis = np.array([0, 0, 0.95 * u]); neck = np.array([0, 0, 1.45 * u])
    caps = [(pelvis, neck, 0.15 * u), (neck + [0, 0, 0.12 * u], neck + [0, 0, 0.2 * u], 0.1 * u)]
    for side in (-1, 1):
        sh = neck + [side * 0.2 * u, 0, -0.05 * u]
        a0, a1 = limb(sh, 0.3, 0.3 + abs(j()), np.pi / 2 * (1 - side) + j())
        a2, a3 = limb(a1, 0.28, abs(j()) + 0.1, np.pi / 2 * (1 - side) + j())
        hip = pelvis + [side * 0.1 * u, 0, 0]
        l0, l1 = limb(hip, 0.45, 0.1 * abs(j()), j())
        l2, l3 = limb(l1, 0.45, 0.1 * abs(j()), j())
        caps += [(a0, a1, 0.05 * u), (a2, a3, 0.04 * u), (l0, l1, 0.07 * u), (l2, l3, 0.055 * u)]
    yaw = rng.uniform(0, 2 * np.pi)
    Rz = np.array([[np.cos(yaw), -np.sin(yaw), 0], [np.sin(yaw), np.cos(yaw), 0], [0, 0, 1]])
    off = np.array([rng.uniform(2, 4), rng.uniform(-1, 1), 0.0])
    return [(_capsule(Rz @ a + off, Rz @ b + off, r)) for a, b, r in caps]


def _human_visible(rng, prims, n):
    """Sensor at the origin: keep points whose outward side faces the sensor (crudely: the
    half of each body part nearer to the sensor), resampling until n points are kept."""
    out, got = [], 0
    while got < n:
        p = _sample_union(rng, prims, 2 * n)
        cen = p.mean(axis=0)
        keep = np.einsum("ij,j->i", p - cen, -cen) > 0
        out.append(p[keep]); got += int(keep.sum())
    return np.concatenate(out)[:n]


def _scene(rng):
    prims = []
    room = np.array([8.0, 6.0, 3.0])
    for ax in range(3):
        for side in (0.0, 1.0):
            dims = room.copy(); dims[ax] = 0.0
            o = np.zeros(3); o[ax] = side * room[ax]
            area = np.prod([d for k, d in enumerate(dims) if k != ax])
            prims.append(((lambda r, n, dims=dims, o=o: o + r.uniform(size=(n, 3)) * dims), area))
    for _ in range(20):
        s, a = (_ellipsoid, _box, _cylinder)[int(rng.integers(0, 3))](rng)
        R, t = _rot(rng), rng.uniform([0.5, 0.5, 0.3], [7.5, 5.5, 1.5])
        prims.append(((lambda r, n, s=s, R=R, t=t: s(r, n) @ R.T + t), a))
    return prims


def pair(kind: str, N: int, M: int, seed: int = 0, b: int = 0):
    """One (pred [N,3], gt [M,3]) fp32 pair of the given kind."""
    rng = _rng(seed, b)
    if kind == "uniform":
        x = rng.uniform(size=(N, 3)); y = rng.uniform(size=(M, 3))
    elif kind == "shapenet":
        prims = _shape(rng)
        # gt and pred sample the same surface; both get gt's unit-sphere normalisation,
        # then pred gets the mid-training noise
        y_raw = _sample_union(rng, prims, M)
        x = _sample_union(rng, prims, N)
        cen = y_raw.mean(0); rad = np.max(np.linalg.norm(y_raw - cen, axis=1))
        y = (y_raw - cen) / rad
        x = (x - cen) / rad + rng.normal(scale=0.01, size=(N, 3))
    elif kind == "near":
        if N != M:
            raise ValueError("near-converged pairs need N == M")
        prims = _shape(rng)
        y = _sample_union(rng, prims, M)
        cen = y.mean(0); y = (y - cen) / np.max(np.linalg.norm(y - cen, axis=1))
        spacing = np.sqrt(4 * np.pi / M)
        x = y[rng.permutation(M)] + rng.normal(scale=0.3 * spacing, size=(M, 3))
    elif kind == "mmfi":
        prims = _human(rng)
        y = _human_visible(rng, prims, M)
        x = _human_visible(rng, prims, N) + rng.normal(scale=0.01, size=(N, 3))
    elif kind == "scene":
        prims = _scene(rng)
        y = _sample_union(rng, prims, M)
        x = _sample_union(rng, prims, N) + rng.normal(scale=0.005, size=(N, 3))
    else:
        raise ValueError(f"unknown kind {kind!r}; one of {KINDS}")
    return np.ascontiguousarray(x, np.float32), np.ascontiguousarray(y, np.float32)


def batch(kind: str, B: int, N: int, M: int, seed: int = 0):
    """(pred [B,N,3], gt [B,M,3]) fp32, pair b drawn from stream (seed, b)."""
    xs = np.empty((B, N, 3), np.float32)
    ys = np.empty((B, M, 3), np.float32)
    for b in range(B):
        xs[b], ys[b] = pair(kind, N, M, seed, b)
    return xs, ys
