"""Seeded synthetic point clouds shaped like the five BASELINE configs
(SURVEY.md §8(d)).  Host-side data preparation only — not on the timed path.

Each generator returns (schema, samples) ready for ``write_dataset``.
Variants: ``quantized=False`` keeps raw float32 coordinates (block pages take
the stored-raw path, ratio 1.000); ``quantized=True`` snaps coordinates to
1 mm, colours to k/255 and intensity to k/100 (block pages take the LZ4 path).
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 0x260316945


def _rng(cloud_id: int, salt: int = 0xDA7A) -> np.random.Generator:
    return np.random.default_rng([BASE_SEED, cloud_id, salt])


def _f32bytes(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32).reshape(-1).view(np.uint8).copy()


def _q(a, step):
    return (np.round(np.asarray(a, np.float64) / step) * step).astype(np.float32)


def superquadric(n: int, rng: np.random.Generator):
    """Noisy superquadric surface + analytic-ish normals (ModelNet-like)."""
    e1, e2 = rng.uniform(0.3, 1.5, 2)
    ax = rng.uniform(0.3, 1.0, 3)
    u = rng.uniform(-np.pi / 2, np.pi / 2, n)
    v = rng.uniform(-np.pi, np.pi, n)
    f = lambda w, e: np.sign(w) * np.abs(w) ** e
    x = ax[0] * f(np.cos(u), e1) * f(np.cos(v), e2)
    y = ax[1] * f(np.cos(u), e1) * f(np.sin(v), e2)
    z = ax[2] * f(np.sin(u), e1)
    p = np.stack([x, y, z], 1) + rng.normal(0, 0.005, (n, 3))
    nr = np.stack([np.cos(u) * np.cos(v) / ax[0], np.cos(u) * np.sin(v) / ax[1], np.sin(u) / ax[2]], 1)
    nr /= np.linalg.norm(nr, axis=1, keepdims=True) + 1e-12
    return p.astype(np.float32), nr.astype(np.float32)


def modelnet(n_clouds: int, n_points: int = 10000, quantized: bool = False, first: int = 0):
    schema = {"fields": {"data": {"type": "bytes"}, "normal": {"type": "bytes"},
                         "label": {"type": "int32"}}}
    out = []
    for i in range(first, first + n_clouds):
        r = _rng(i)
        p, nr = superquadric(n_points, r)
        if quantized:
            p, nr = _q(p, 1e-3), _q(nr, 1e-3)
        out.append({"data": _f32bytes(p), "normal": _f32bytes(nr),
                    "label": np.array([i % 40], np.int32)})
    return schema, out


def shapenet(n_clouds: int, n_points: int = 2048, quantized: bool = False, first: int = 0):
    schema = {"fields": {"data": {"type": "bytes"}, "seg": {"type": "bytes"},
                         "label": {"type": "int32"}}}
    out = []
    for i in range(first, first + n_clouds):
        r = _rng(i)
        p, _ = superquadric(n_points, r)
        seg = (np.floor((p[:, 2] - p[:, 2].min()) * 3.0).astype(np.int32) % 6) + 6 * (i % 8)
        if quantized:
            p = _q(p, 1e-3)
        out.append({"data": _f32bytes(p), "seg": seg.astype(np.int32).view(np.uint8).copy(),
                    "label": np.array([i % 16], np.int32)})
    return schema, out


def room(n: int, rng: np.random.Generator, size=(10.0, 10.0, 3.0), n_boxes: int = 10):
    """Points on room surfaces: floor, ceiling, 4 walls, boxes; RGB per surface."""
    W, D, H = size
    surf = rng.integers(0, 6 + n_boxes, n)
    uv = rng.uniform(0, 1, (n, 2))
    p = np.empty((n, 3), np.float64)
    boxes = rng.uniform([0.5, 0.5, 0.0], [W - 1.5, D - 1.5, 0.0], (n_boxes, 3))
    bsz = rng.uniform(0.3, 1.2, (n_boxes, 3))
    for s in range(6 + n_boxes):
        m = surf == s
        a, b = uv[m, 0], uv[m, 1]
        if s == 0: p[m] = np.stack([a * W, b * D, 0 * a], 1)
        elif s == 1: p[m] = np.stack([a * W, b * D, H + 0 * a], 1)
        elif s == 2: p[m] = np.stack([a * W, 0 * a, b * H], 1)
        elif s == 3: p[m] = np.stack([a * W, D + 0 * a, b * H], 1)
        elif s == 4: p[m] = np.stack([0 * a, a * D, b * H], 1)
        elif s == 5: p[m] = np.stack([W + 0 * a, a * D, b * H], 1)
        else:
            k = s - 6
            p[m] = np.stack([boxes[k, 0] + a * bsz[k, 0], boxes[k, 1] + b * bsz[k, 1],
                             bsz[k, 2] + 0 * a], 1)
    p += rng.normal(0, 0.003, p.shape)
    col = rng.uniform(0, 1, (6 + n_boxes, 3))[surf] + rng.normal(0, 0.02, (n, 3))
    return p.astype(np.float32), np.clip(col, 0, 1).astype(np.float32)


def s3dis(n_rooms: int, mean_points: int = 1_000_000, quantized: bool = False, first: int = 0):
    schema = {"fields": {"data": {"type": "bytes"}, "color": {"type": "bytes"},
                         "label": {"type": "int32"}}}
    out = []
    for i in range(first, first + n_rooms):
        r = _rng(i)
        n = int(r.integers(int(mean_points * 0.9), int(mean_points * 1.1) + 1))
        p, c = room(n, r)
        if quantized:
            p, c = _q(p, 1e-3), (np.round(c * 255) / 255).astype(np.float32)
        out.append({"data": _f32bytes(p), "color": _f32bytes(c), "label": np.array([i % 13], np.int32)})
    return schema, out


def scannet(n_scenes: int, lo: int = 50_000, hi: int = 500_000, quantized: bool = False,
            first: int = 0):
    schema = {"fields": {"data": {"type": "bytes"}, "color": {"type": "bytes"},
                         "label": {"type": "int32"}}}
    out = []
    for i in range(first, first + n_scenes):
        r = _rng(i)
        n = int(r.integers(lo, hi + 1))
        p, c = room(n, r, size=tuple(r.uniform([4, 4, 2.5], [8, 8, 3.2])), n_boxes=8)
        if quantized:
            p, c = _q(p, 1e-3), (np.round(c * 255) / 255).astype(np.float32)
        out.append({"data": _f32bytes(p), "color": _f32bytes(c), "label": np.array([i % 20], np.int32)})
    return schema, out


def lidar(n: int, rng: np.random.Generator):
    """64-ring LiDAR sweep: ground plane + obstacles, XYZ + intensity."""
    ring = rng.integers(0, 64, n)
    az = rng.uniform(-np.pi, np.pi, n)
    elev = np.deg2rad(-24.8 + ring * (26.8 / 63))
    h = 1.73
    rng_ground = np.where(elev < -0.01, h / np.maximum(np.tan(-elev), 1e-3), 80.0)
    obst = rng.uniform(2, 80, n)
    rr = np.where(rng.uniform(0, 1, n) < 0.3, np.minimum(obst, rng_ground), rng_ground)
    rr = np.clip(rr + rng.normal(0, 0.02, n), 2.0, 80.0)
    x = rr * np.cos(elev) * np.cos(az)
    y = rr * np.cos(elev) * np.sin(az)
    z = rr * np.sin(elev) + h * 0
    inten = np.clip(rng.beta(2, 5, n), 0, 1)
    return np.stack([x, y, z], 1).astype(np.float32), inten.astype(np.float32)


def kitti(n_frames: int, lo: int = 115_000, hi: int = 125_000, quantized: bool = False,
          first: int = 0):
    schema = {"fields": {"data": {"type": "bytes"}, "intensity": {"type": "bytes"},
                         "label": {"type": "int32"}}}
    out = []
    for i in range(first, first + n_frames):
        r = _rng(i)
        n = int(r.integers(lo, hi + 1))
        p, it = lidar(n, r)
        if quantized:
            p, it = _q(p, 1e-2), (np.round(it * 100) / 100).astype(np.float32)
        out.append({"data": _f32bytes(p), "intensity": _f32bytes(it), "label": np.array([i % 3], np.int32)})
    return schema, out


def graph(maps: list, batch_size: int, base_seed: int = 42, drop_remainder: bool = True,
          workers: int = 1) -> dict:
    """Reference graph JSON (pcpipe_main.cpp:65-99 make_graph shape): source=0,
    maps 1..k (op ids fix the seeds), batch, sink."""
    ops = [{"id": 0, "kind": "source", "num_workers": workers, "queue_capacity": 8}]
    for i, m in enumerate(maps):
        name, params = (m, {}) if isinstance(m, str) else m
        ops.append({"id": i + 1, "kind": "map", "map": name, "params": params,
                    "num_workers": workers, "queue_capacity": 8})
    ops.append({"id": len(maps) + 1, "kind": "batch", "batch_size": batch_size,
                "num_workers": 1, "queue_capacity": 8})
    ops.append({"id": len(maps) + 2, "kind": "sink", "num_workers": 1, "queue_capacity": 8})
    return {"base_seed": base_seed, "drop_remainder": drop_remainder, "ops": ops}


# Op chains per config; op ids = position + 1.
CHAINS = {
    "modelnet40": [("normalize", {}), ("fps", {"num_points": 1024}), ("rotate", {}),
                   ("jitter", {})],
    "shapenet_part": [("normalize", {}), ("downsample", {"num_points": 1024, "gather": ["seg"]}),
                      ("random_scale", {}), ("downsample", {"num_points": 1024, "gather": ["seg"]})],
    "s3dis": [("grid_subsample", {"voxel_size": 0.04}), ("random_crop", {}),
              ("downsample", {"num_points": 4096})],
    "kitti": [("range_crop", {"lo": [0.0, -40.0, -3.0], "hi": [70.4, 40.0, 1.0]}),
              ("voxel", {"voxel_size": 0.05, "origin": [0.0, -40.0, -3.0]}), ("rotate", {}),
              ("flip_yz", {})],
    "scannet": [("grid_subsample", {"voxel_size": 0.02}), ("downsample", {"num_points": 40000}),
                ("fps", {"num_points": 20000})],
}
