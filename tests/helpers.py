"""Shared fixtures for the parity tests (restating tests/test_utils.hpp of the reference)."""
import json
import math
import os
from types import SimpleNamespace

import numpy as np

from paper_2403_16095_b200.abi import Intrinsics, Pose, defaults_raster

C0 = 0.28209479177387814
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def make_intrinsics(w, h, f, near=0.1, far=50.0):
    """test_utils.hpp:13-23"""
    return Intrinsics(f, f, 0.5 * w, 0.5 * h, w, h, 1.0, near, far)


def one_pixel_camera():
    """test_rasterizer.cpp:20-29"""
    return Intrinsics(1.0, 1.0, 0.5, 0.5, 1, 1, 1.0, 0.1, 10.0)


def pose(rot=(0, 0, 0), trans=(0, 0, 0)):
    p = Pose()
    for i in range(3):
        p.rotation_tangent[i] = rot[i]
        p.translation[i] = trans[i]
    return p


def logit(p):
    return math.log(p / (1.0 - p))


def scene(prims, K=1):
    """prims: list of dicts with mean, scale (iso) or log_scale, opacity, color (DC via SH) or sh."""
    P = len(prims)
    m = SimpleNamespace(mean=np.zeros((P, 3)), log_scale=np.zeros((P, 3)), quat=np.tile([1.0, 0, 0, 0], (P, 1)),
                        opacity_logit=np.zeros(P), sh=np.zeros((P, K, 3)), uncertainty=np.zeros(P),
                        observed=np.zeros(P, np.uint8))
    for i, p in enumerate(prims):
        m.mean[i] = p["mean"]
        m.log_scale[i] = p.get("log_scale", [math.log(p.get("scale", 0.05))] * 3)
        if "quat" in p:
            m.quat[i] = p["quat"]
        m.opacity_logit[i] = logit(p["opacity"])
        if "sh" in p:
            m.sh[i] = np.asarray(p["sh"]).reshape(K, 3)
        else:
            m.sh[i, 0] = (np.asarray(p.get("color", [0.5, 0.5, 0.5])) - 0.5) / C0
    return m


def axis_primitive(z, opacity, color):
    """test_rasterizer.cpp:31-41"""
    return dict(mean=[0.0, 0.0, z], scale=0.05, opacity=opacity, color=color)


def f32_round(m):
    """Round every parameter to the nearest fp32 so the fp64 oracle and the fp32 device map
    start from identical values (the device stores the map as fp32 SoA)."""
    out = SimpleNamespace(**{k: (np.asarray(v, np.float32).astype(np.float64) if np.asarray(v).dtype == np.float64
                                 else (v.copy() if isinstance(v, np.ndarray) else v))
                             for k, v in vars(m).items()})
    return out


def to_api_map(m):
    from paper_2403_16095_b200.api import GaussianMap
    return GaussianMap(m.mean, m.log_scale, m.quat, m.opacity_logit, m.sh, getattr(m, "uncertainty", None),
                       getattr(m, "observed", None))


def random_pose(rng, rot_sigma, trans_sigma):
    return pose(rot_sigma * rng.standard_normal(3), trans_sigma * rng.standard_normal(3))


def rotation_error(a: Pose, b: Pose):
    from scipy.spatial.transform import Rotation as R
    ra = R.from_rotvec(list(a.rotation_tangent))
    rb = R.from_rotvec(list(b.rotation_tangent))
    return float(np.linalg.norm((ra * rb.inv()).as_rotvec()))


def translation_error(a: Pose, b: Pose):
    return float(np.linalg.norm(np.array(list(a.translation)) - np.array(list(b.translation))))


def perturbed(p: Pose, d):
    """CameraPose::perturbed (pose.hpp:44-48)."""
    from scipy.spatial.transform import Rotation as R
    dr = R.from_rotvec(d[:3])
    r = R.from_rotvec(list(p.rotation_tangent))
    rn = dr * r
    t = dr.apply(np.array(list(p.translation))) + np.asarray(d[3:])
    return pose(rn.as_rotvec(), t)


RASTER = defaults_raster


def mt19937_uniform(seed, lo, hi, n):
    """n draws of std::uniform_real_distribution<double>(lo, hi) from std::mt19937(seed) as
    libstdc++ computes them (generate_canonical<double, 53>: two 32-bit outputs, low first)."""
    bg = np.random.MT19937()
    bg._legacy_seeding(seed)
    x = bg.random_raw(2 * n).astype(np.float64)
    r = (x[0::2] + x[1::2] * 4294967296.0) / 18446744073709551616.0
    r = np.where(r >= 1.0, np.nextafter(1.0, 0.0), r)
    return r * (hi - lo) + lo


def textured_wall(nx, ny, seed):
    """test_tracker.cpp:62-84 (textured_wall with std::mt19937(seed)) draw for draw; the three colour
    draws of a primitive land in Vec3(uc, uc, uc) right to left, as GCC evaluates the arguments."""
    P = nx * ny
    m = scene([])
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    x = -1.4 + 2.8 * (ii.ravel() + 0.5) / nx
    y = -1.0 + 2.0 * (jj.ravel() + 0.5) / ny
    m.mean = np.stack([x, y, 2.5 + 0.15 * np.sin(2.0 * x) * np.cos(3.0 * y)], 1)
    m.log_scale = np.full((P, 3), math.log(0.09))
    m.quat = np.tile([1.0, 0, 0, 0], (P, 1))
    m.opacity_logit = np.full(P, logit(0.95))
    u = mt19937_uniform(seed, -0.8, 0.8, 3 * P).reshape(P, 3)
    m.sh = u[:, ::-1].reshape(P, 1, 3).copy()
    m.uncertainty = np.zeros(P)
    m.observed = np.zeros(P, np.uint8)
    return m
