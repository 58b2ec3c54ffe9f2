"""Synthetic inputs for bench.py and the tests — support code, not the product.

ctypes bindings of tools/synth/libgsf_synth.so (tools/synth/synth.cpp), a restatement of the
reference generator (io/synthetic.cpp:39-186: room scene, orbit trajectory) that reproduces its
std::mt19937_64 draws; tests/test_port_vs_reference.py checks it bit for bit against the
reference's own SyntheticSource (oracle/_ref).  Frames are rendered by the caller.
"""
import ctypes as C
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgsf_synth.so")
dp = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)


class _MapHost(C.Structure):   # gsf_map_host (include/gsf_cuda.h)
    _fields_ = [("count", C.c_int64), ("sh_coeffs", C.c_int32), ("mean", dp), ("log_scale", dp),
                ("quat", dp), ("opacity_logit", dp), ("sh", dp), ("uncertainty", dp), ("observed", u8p)]


class _Pose(C.Structure):      # gsf_pose
    _fields_ = [("rotation_tangent", C.c_double * 3), ("translation", C.c_double * 3)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = C.CDLL(LIB_PATH)
        L.gsf_synth_room.argtypes = [C.c_int32, C.c_double, C.c_int32, C.c_uint64, C.c_void_p]
        L.gsf_synth_orbit.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_void_p]
        _lib = L
    return _lib


def room(primitive_count: int, extent: float = 4.0, wall_layers: int = 3, seed: int = 0):
    """SceneSpec{room, primitive_count, extent, wall_layers} with mt19937_64(seed): arrays
    mean (P,3), log_scale (P,3), quat (P,4), opacity_logit (P,), sh (P,1,3)."""
    L = _load()
    h = _MapHost()
    if L.gsf_synth_room(primitive_count, extent, wall_layers, seed, C.byref(h)) != 0:
        raise ValueError("synth_room failed")
    P = int(h.count)
    q = np.zeros((P, 4))
    q[:, 0] = 1.0
    m = SimpleNamespace(mean=np.zeros((P, 3)), log_scale=np.zeros((P, 3)), quat=q, opacity_logit=np.zeros(P),
                        sh=np.zeros((P, 1, 3)))
    h = _MapHost(P, 1, m.mean.ctypes.data_as(dp), m.log_scale.ctypes.data_as(dp), m.quat.ctypes.data_as(dp),
                 m.opacity_logit.ctypes.data_as(dp), m.sh.ctypes.data_as(dp), None, None)
    if L.gsf_synth_room(primitive_count, extent, wall_layers, seed, C.byref(h)) != 0:
        raise ValueError("synth_room failed")
    m.count = P
    return m


def orbit(frames: int, radius: float = 1.0, height: float = 0.0):
    """TrajectorySpec{orbit, frames, radius, height}: world-to-camera poses as (rotvec, translation)."""
    L = _load()
    poses = (_Pose * frames)()
    if L.gsf_synth_orbit(frames, radius, height, poses) != 0:
        raise ValueError("synth_orbit failed")
    return [(np.array(list(p.rotation_tangent)), np.array(list(p.translation))) for p in poses]
