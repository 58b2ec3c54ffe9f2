"""TEST INFRASTRUCTURE ONLY — the CPU checker.

Two interchangeable backends behind the same orc_* entry points (oracle/gsf_oracle.h):

* "port" — oracle/liboracle.so: the fp64 restatement of the reference hot path
  (oracle/gsf_oracle.cpp, every function citing the /root/reference file:line it follows) plus the
  fp32 mirror of the device decision path (oracle/mirror.cpp);
* "reference" — oracle/_ref/libgsfref.so: the UNMODIFIED reference sources compiled here against
  oracle/eigen_lite (oracle/Makefile.ref) behind a thin C shim (oracle/ref_capi.cpp).  Present
  wherever it was built (this container; the .so travels to the GPU box with the snapshot).

``with oracle.backend("reference"): ...`` routes every entry point the reference library exports
to it (the mirror, the fixtures and the restatement-only helpers stay on the port).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
package, and only as the checker or the timed CPU baseline — never as the product.  It does not
import the product package.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
import subprocess
from types import SimpleNamespace

import numpy as np

from .gsf_types import Intrinsics, LossTerms, LossWeights, MapHost, MapperCfg, Pose, RasterCfg, TrackerCfg, TrackResult

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libgsfref.so")
REF_SOURCES = "/root/reference/proj"

dp = C.POINTER(C.c_double)
fp = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
vp = C.c_void_p   # struct pointers: any ctypes struct with the gsf_cuda.h layout, passed by reference


def _as(T, x):
    """x as a T (same C layout; e.g. the product's abi.Pose -> oracle's Pose)."""
    return x if isinstance(x, T) else T.from_buffer_copy(x)


class Maps(C.Structure):
    _fields_ = [("color", dp), ("alpha_depth", dp), ("median_depth", dp), ("median_valid", u8p), ("opacity", dp),
                ("uncertainty", dp), ("final_transmittance", dp), ("per_pixel_count", i32p), ("dominant", i32p),
                ("median_prim", i32p), ("dominant_weight", dp), ("visible", u8p), ("has_uncertainty", C.c_int32)]


class Upstream(C.Structure):
    _fields_ = [("d_color", dp), ("d_alpha_depth", dp), ("d_median_depth", dp), ("d_opacity", dp),
                ("d_uncertainty", dp)]


class Grads(C.Structure):
    _fields_ = [("d_mean", dp), ("d_log_scale", dp), ("d_quat", dp), ("d_opacity_logit", dp), ("d_sh", dp),
                ("d_mean2d", dp), ("d_pose", C.c_double * 6)]


class GradcheckReport(C.Structure):
    _fields_ = [("total", C.c_int32), ("checked", C.c_int32), ("skipped", C.c_int32), ("max_rel_err", C.c_double),
                ("worst_analytic", C.c_double), ("worst_fd", C.c_double), ("worst_index", C.c_int32)]


class MirOut(C.Structure):
    _fields_ = [("visible", u8p), ("rank_to_id", i32p), ("tile_range", i32p), ("pair_rank", i32p),
                ("pair_capacity", C.c_int64), ("color", fp), ("alpha_depth", fp), ("median_depth", fp),
                ("median_valid", u8p), ("opacity", fp), ("uncertainty", fp), ("final_transmittance", fp),
                ("per_pixel_count", i32p), ("dominant", i32p), ("median_prim", i32p), ("dominant_weight", fp),
                ("last_index", i32p), ("num_visible", C.c_int64), ("num_pairs", C.c_int64),
                ("num_flagged", C.c_int64)]


_libs = {}
_active = "port"


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if os.path.isdir(REF_SOURCES):
        build_reference()


def build_reference():
    """oracle/_ref/libgsfref.so from the unmodified reference sources (needs /root/reference)."""
    subprocess.run(["make", "-s", "-j8", "-f", os.path.join(HERE, "Makefile.ref")], check=True)


def reference_available() -> bool:
    return os.path.exists(REF_PATH)


@contextlib.contextmanager
def backend(name: str):
    """Route the entry points to "port" (restatement) or "reference" (the reference's own code)."""
    global _active
    assert name in ("port", "reference")
    if name == "reference" and not reference_available():
        raise FileNotFoundError(f"{REF_PATH} is missing (built by oracle.build_reference() where /root/reference exists)")
    prev, _active = _active, name
    try:
        yield
    finally:
        _active = prev


class _Dispatch:
    def __getattr__(self, name):
        if _active == "reference":
            L = _load("reference")
            try:
                return getattr(L, name)
            except AttributeError:
                pass
        return getattr(_load("port"), name)


def lib():
    _load("port")
    return _Dispatch()


def _current():
    """The library the active backend's objects (results, map states) belong to."""
    return _load("reference") if _active == "reference" else _load("port")


def _load(which):
    if which in _libs:
        return _libs[which]
    path = LIB_PATH if which == "port" else REF_PATH
    if which == "port" and not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    L = C.CDLL(path)
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_threads": (C.c_int, []),
        "orc_render": (C.c_int, [C.POINTER(MapHost), C.POINTER(Pose), C.POINTER(Intrinsics), dp, C.POINTER(RasterCfg),
                                 C.c_int, C.POINTER(C.c_void_p)]),
        "orc_result_free": (None, [C.c_void_p]),
        "orc_result_maps": (C.c_int, [C.c_void_p, C.POINTER(Maps)]),
        "orc_result_record_total": (C.c_int64, [C.c_void_p]),
        "orc_result_record": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), i32p, dp, dp]),
        "orc_render_backward": (C.c_int, [C.POINTER(MapHost), C.POINTER(Pose), C.POINTER(Intrinsics), C.c_void_p,
                                          C.POINTER(Upstream), dp, C.POINTER(RasterCfg), C.POINTER(Grads)]),
        "orc_tracking_loss": (C.c_int, [C.c_void_p, dp, dp, C.POINTER(Intrinsics), C.POINTER(LossWeights),
                                        C.POINTER(LossTerms), dp, dp]),
        "orc_mapping_loss": (C.c_int, [C.POINTER(MapHost), C.c_void_p, dp, dp, C.POINTER(Intrinsics),
                                       C.POINTER(LossWeights), C.POINTER(LossTerms), dp, dp, dp, dp, dp]),
        "orc_ssim": (C.c_int, [dp, dp, C.c_int, C.c_int, dp, dp]),
        "orc_adam_step": (None, [dp, dp, dp, dp, C.c_int64, C.POINTER(C.c_uint64), C.c_double, C.c_double, C.c_double,
                                 C.c_double]),
        "orc_track_frame": (C.c_int, [C.POINTER(MapHost), dp, dp, C.POINTER(Pose), C.POINTER(Intrinsics),
                                      C.POINTER(TrackerCfg), C.POINTER(LossWeights), C.POINTER(RasterCfg),
                                      C.POINTER(TrackResult)]),
        "orc_mapstate_create": (C.c_int, [C.POINTER(MapHost), C.POINTER(MapperCfg), C.POINTER(C.c_void_p)]),
        "orc_mapstate_free": (None, [C.c_void_p]),
        "orc_mapstate_count": (C.c_int64, [C.c_void_p]),
        "orc_mapstate_get": (C.c_int, [C.c_void_p, C.POINTER(MapHost)]),
        "orc_map_step": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(dp), C.POINTER(dp), C.POINTER(Pose),
                                   C.POINTER(Intrinsics), C.POINTER(MapperCfg), C.c_int, dp]),
        "orc_sliding_ba": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(dp), C.POINTER(dp), C.POINTER(Pose), i32p,
                                     C.POINTER(Intrinsics), C.POINTER(TrackerCfg), C.POINTER(MapperCfg), C.c_int, dp]),
        "orc_mapstate_put": (C.c_int, [C.c_void_p, C.POINTER(MapHost)]),
        "orc_mapstate_append": (C.c_int, [C.c_void_p, C.POINTER(MapHost)]),
        "orc_mapstate_set_stats": (C.c_int, [C.c_void_p, dp, i32p]),
        "orc_mapstate_densify": (C.c_int, [C.c_void_p, C.POINTER(MapperCfg), i32p]),
        "orc_backproject": (C.c_int, [dp, dp, dp, C.POINTER(Pose), C.POINTER(Intrinsics), C.POINTER(MapperCfg),
                                      C.c_int, C.POINTER(MapHost), C.POINTER(C.c_int64)]),
        "orc_uncertainty_partials": (C.c_int, [C.POINTER(MapHost), C.c_int, C.POINTER(C.c_void_p), C.POINTER(dp),
                                               C.POINTER(Pose), C.POINTER(Intrinsics), dp, i32p]),
        "orc_accumulate_uncertainty": (C.c_int, [C.POINTER(MapHost), C.c_int, C.POINTER(C.c_void_p), C.POINTER(dp),
                                                 C.POINTER(Pose), C.POINTER(Intrinsics), i32p]),
        "orc_prune_unreliable": (C.c_int, [C.POINTER(MapHost), C.c_double, C.c_double, i32p]),
        "orc_gradcheck_linear": (C.c_int, [C.POINTER(MapHost), C.POINTER(Pose), C.POINTER(Intrinsics),
                                           C.POINTER(RasterCfg), dp, dp, dp, dp, dp, dp, C.c_double, C.c_double,
                                           C.POINTER(GradcheckReport)]),
        "orc_random_scene": (C.c_int, [C.c_uint32, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.POINTER(MapHost)]),
        "orc_wavy_depth": (None, [C.c_int, C.c_int, C.c_double, C.c_int, dp]),
        "orc_smooth_raster": (None, [C.POINTER(RasterCfg)]),
        "orc_default_raster": (None, [C.POINTER(RasterCfg)]),
        "orc_default_weights": (None, [C.POINTER(LossWeights), C.c_int]),
        "orc_default_tracker": (None, [C.POINTER(TrackerCfg)]),
        "orc_default_mapper": (None, [C.POINTER(MapperCfg)]),
        "ref_synth_scene": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                      C.POINTER(Intrinsics), C.POINTER(MapHost), C.POINTER(C.c_int64), C.POINTER(Pose),
                                      C.c_int]),
        "mir_render": (C.c_int, [C.POINTER(MapHost), C.POINTER(Pose), C.POINTER(Intrinsics), fp, C.POINTER(RasterCfg),
                                 C.POINTER(MirOut)]),
    }
    for name, (res, args) in sig.items():
        try:
            f = getattr(L, name)
        except AttributeError:   # the reference library exports the reference-backed subset
            continue
        f.restype = res
        f.argtypes = [vp if (isinstance(a, type) and issubclass(a, C._Pointer) and issubclass(a._type_, C.Structure)
                             and a._type_ is not Maps and a._type_ is not MirOut and a._type_ is not Grads
                             and a._type_ is not Upstream and a._type_ is not GradcheckReport) else a for a in args]
    _libs[which] = L
    return L


class OracleError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def _check(rc, L=None):
    if rc != 0:
        raise OracleError(rc, (L or lib()).orc_last_error().decode())


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(dp)


def host_of(m) -> MapHost:
    """MapHost view of any object with mean/log_scale/quat/opacity_logit/sh(/uncertainty/observed) arrays."""
    P = m.mean.shape[0]
    K = m.sh.shape[1] if m.sh.ndim == 3 else m.sh.shape[1] // 3
    unc = getattr(m, "uncertainty", None)
    obs = getattr(m, "observed", None)
    return MapHost(P, K, m.mean.ctypes.data_as(dp), m.log_scale.ctypes.data_as(dp), m.quat.ctypes.data_as(dp),
                   m.opacity_logit.ctypes.data_as(dp), m.sh.ctypes.data_as(dp),
                   None if unc is None else unc.ctypes.data_as(dp), None if obs is None else obs.ctypes.data_as(u8p))


def empty_map(P, K=1):
    q = np.zeros((P, 4))
    q[:, 0] = 1.0
    return SimpleNamespace(mean=np.zeros((P, 3)), log_scale=np.zeros((P, 3)), quat=q, opacity_logit=np.zeros(P),
                           sh=np.zeros((P, K, 3)), uncertainty=np.zeros(P), observed=np.zeros(P, np.uint8))


def threads() -> int:
    return int(lib().orc_threads())


def random_scene(seed, count, sh_coeffs=1, max_opacity=0.95, min_scale=0.02, max_scale=0.15):
    """tests/test_utils.hpp:27-53 with std::mt19937(seed)."""
    m = empty_map(count, sh_coeffs)
    h = host_of(m)
    _check(lib().orc_random_scene(seed, count, sh_coeffs, max_opacity, min_scale, max_scale, C.byref(h)))
    return m


def wavy_depth(w, h, base, hole_every=17):
    out = np.zeros(w * h)
    lib().orc_wavy_depth(w, h, base, hole_every, out.ctypes.data_as(dp))
    return out.reshape(h, w)


class Result:
    """Owning wrapper of an orc_result (RenderResult)."""

    def __init__(self, handle, W, H, P, L):
        self.h, self.W, self.H, self.P, self.L = handle, W, H, P, L
        n = W * H
        self.color = np.zeros((H, W, 3))
        self.alpha_depth = np.zeros((H, W))
        self.median_depth = np.zeros((H, W))
        self.median_valid = np.zeros((H, W), np.uint8)
        self.opacity = np.zeros((H, W))
        self.uncertainty = np.zeros((H, W))
        self.final_transmittance = np.zeros((H, W))
        self.per_pixel_count = np.zeros((H, W), np.int32)
        self.dominant = np.zeros((H, W), np.int32)
        self.median_prim = np.zeros((H, W), np.int32)
        self.dominant_weight = np.zeros((H, W))
        self.visible = np.zeros(max(P, 1), np.uint8)
        m = Maps(self.color.ctypes.data_as(dp), self.alpha_depth.ctypes.data_as(dp), self.median_depth.ctypes.data_as(dp),
                 self.median_valid.ctypes.data_as(u8p), self.opacity.ctypes.data_as(dp),
                 self.uncertainty.ctypes.data_as(dp), self.final_transmittance.ctypes.data_as(dp),
                 self.per_pixel_count.ctypes.data_as(i32p), self.dominant.ctypes.data_as(i32p),
                 self.median_prim.ctypes.data_as(i32p), self.dominant_weight.ctypes.data_as(dp),
                 self.visible.ctypes.data_as(u8p), 0)
        _check(L.orc_result_maps(handle, C.byref(m)), L)
        self.visible = self.visible[:P]
        self.has_uncertainty = bool(m.has_uncertainty)
        _ = n

    def record(self):
        t = self.L.orc_result_record_total(self.h)
        rs = np.zeros(self.W * self.H + 1, np.uint32)
        prim = np.zeros(max(t, 1), np.int32)
        a = np.zeros(max(t, 1))
        tr = np.zeros(max(t, 1))
        _check(self.L.orc_result_record(self.h, rs.ctypes.data_as(C.POINTER(C.c_uint32)), prim.ctypes.data_as(i32p),
                                       a.ctypes.data_as(dp), tr.ctypes.data_as(dp)))
        return rs, prim[:t], a[:t], tr[:t]

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_result_free(self.h)
            self.h = None


def render(m, pose: Pose, K: Intrinsics, obs=None, cfg: RasterCfg = None, brute_force=False) -> Result:
    cfg = cfg or defaults_raster()
    h = host_of(m)
    out = C.c_void_p()
    o = None if obs is None else np.ascontiguousarray(obs, dtype=np.float64)
    L = _current()
    _check(L.orc_render(C.byref(h), C.byref(pose), C.byref(K), None if o is None else o.ctypes.data_as(dp),
                        C.byref(cfg), 1 if brute_force else 0, C.byref(out)), L)
    return Result(out, K.width, K.height, m.mean.shape[0], L)


def render_backward(m, pose, K, res: Result, d_color=None, d_alpha_depth=None, d_median_depth=None, d_opacity=None,
                    d_uncertainty=None, obs=None, cfg=None):
    cfg = cfg or defaults_raster()
    keep = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in
            (d_color, d_alpha_depth, d_median_depth, d_opacity, d_uncertainty)]
    up = Upstream(*[None if a is None else a.ctypes.data_as(dp) for a in keep])
    P = m.mean.shape[0]
    K_ = m.sh.shape[1]
    g = SimpleNamespace(d_mean=np.zeros((P, 3)), d_log_scale=np.zeros((P, 3)), d_quat=np.zeros((P, 4)),
                        d_opacity_logit=np.zeros(P), d_sh=np.zeros((P, K_, 3)), d_mean2d=np.zeros((P, 2)))
    go = Grads(g.d_mean.ctypes.data_as(dp), g.d_log_scale.ctypes.data_as(dp), g.d_quat.ctypes.data_as(dp),
               g.d_opacity_logit.ctypes.data_as(dp), g.d_sh.ctypes.data_as(dp), g.d_mean2d.ctypes.data_as(dp))
    o = None if obs is None else np.ascontiguousarray(obs, dtype=np.float64)
    h = host_of(m)
    _check(res.L.orc_render_backward(C.byref(h), C.byref(pose), C.byref(K), res.h, C.byref(up),
                                     None if o is None else o.ctypes.data_as(dp), C.byref(cfg), C.byref(go)), res.L)
    g.d_pose = np.array(list(go.d_pose))
    return g


def tracking_loss(res: Result, target, obs, K, w):
    t = np.ascontiguousarray(target, dtype=np.float64)
    o = np.ascontiguousarray(obs, dtype=np.float64)
    out = LossTerms()
    n = K.width * K.height
    dc, dd = np.zeros(3 * n), np.zeros(n)
    _check(res.L.orc_tracking_loss(res.h, t.ctypes.data_as(dp), o.ctypes.data_as(dp), C.byref(K), C.byref(w),
                                   C.byref(out), dc.ctypes.data_as(dp), dd.ctypes.data_as(dp)), res.L)
    return out, dc, dd


def mapping_loss(m, res: Result, target, obs, K, w):
    t = np.ascontiguousarray(target, dtype=np.float64)
    o = np.ascontiguousarray(obs, dtype=np.float64)
    out = LossTerms()
    n = K.width * K.height
    P = m.mean.shape[0]
    bufs = [np.zeros(3 * n), np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(3 * max(P, 1))]
    h = host_of(m)
    _check(res.L.orc_mapping_loss(C.byref(h), res.h, t.ctypes.data_as(dp), o.ctypes.data_as(dp), C.byref(K),
                                  C.byref(w), C.byref(out), *[b.ctypes.data_as(dp) for b in bufs]), res.L)
    return out, bufs


def ssim(x, y, w, h, gradient=False):
    xa = np.ascontiguousarray(x, dtype=np.float64)
    ya = np.ascontiguousarray(y, dtype=np.float64)
    v = C.c_double()
    g = np.zeros(3 * w * h) if gradient else None
    _check(lib().orc_ssim(xa.ctypes.data_as(dp), ya.ctypes.data_as(dp), w, h, C.byref(v),
                          None if g is None else g.ctypes.data_as(dp)))
    return (v.value, g) if gradient else v.value


def track_frame(m, rgb, depth, initial: Pose, K, tcfg, w, raster) -> TrackResult:
    r = np.ascontiguousarray(rgb, dtype=np.float64)
    d = np.ascontiguousarray(depth, dtype=np.float64)
    out = TrackResult()
    h = host_of(m)
    _check(lib().orc_track_frame(C.byref(h), r.ctypes.data_as(dp), d.ctypes.data_as(dp), C.byref(initial), C.byref(K),
                                 C.byref(tcfg), C.byref(w), C.byref(raster), C.byref(out)))
    return out


class MapState:
    def __init__(self, m, mcfg: MapperCfg):
        self.K = m.sh.shape[1]
        h = host_of(m)
        s = C.c_void_p()
        self.L = _current()
        _check(self.L.orc_mapstate_create(C.byref(h), C.byref(mcfg), C.byref(s)), self.L)
        self.h = s

    def get(self):
        P = self.L.orc_mapstate_count(self.h)
        m = empty_map(P, self.K)
        h = host_of(m)
        _check(self.L.orc_mapstate_get(self.h, C.byref(h)), self.L)
        return m

    def map_step(self, frames, poses, K, mcfg, iterations):
        n = len(frames)
        keep = [(np.ascontiguousarray(r, dtype=np.float64), np.ascontiguousarray(d, dtype=np.float64)) for r, d in frames]
        rg = (dp * n)(*[k[0].ctypes.data_as(dp) for k in keep])
        dg = (dp * n)(*[k[1].ctypes.data_as(dp) for k in keep])
        ps = (Pose * n)(*[_as(Pose, p) for p in poses])
        trace = np.zeros(max(iterations, 1))
        _check(self.L.orc_map_step(self.h, n, rg, dg, ps, C.byref(K), C.byref(mcfg), iterations, trace.ctypes.data_as(dp)), self.L)
        return trace[:iterations]

    def sliding_ba(self, frames, poses, frame_ids, K, tcfg, mcfg, iterations):
        n = len(frames)
        keep = [(np.ascontiguousarray(r, dtype=np.float64), np.ascontiguousarray(d, dtype=np.float64)) for r, d in frames]
        rg = (dp * n)(*[k[0].ctypes.data_as(dp) for k in keep])
        dg = (dp * n)(*[k[1].ctypes.data_as(dp) for k in keep])
        ps = (Pose * n)(*[_as(Pose, p) for p in poses])
        fid = (C.c_int32 * n)(*frame_ids)
        trace = np.zeros(max(iterations, 1))
        _check(self.L.orc_sliding_ba(self.h, n, rg, dg, ps, fid, C.byref(K), C.byref(tcfg), C.byref(mcfg), iterations,
                                    trace.ctypes.data_as(dp)), self.L)
        return trace[:iterations], [ps[i] for i in range(n)]

    def put(self, m):
        h = host_of(m)
        _check(self.L.orc_mapstate_put(self.h, C.byref(h)), self.L)

    def append(self, m):
        h = host_of(m)
        _check(self.L.orc_mapstate_append(self.h, C.byref(h)), self.L)

    def set_stats(self, accum, count):
        a = np.ascontiguousarray(accum, dtype=np.float64)
        c = np.ascontiguousarray(count, dtype=np.int32)
        _check(self.L.orc_mapstate_set_stats(self.h, a.ctypes.data_as(dp), c.ctypes.data_as(i32p)), self.L)

    def densify(self, mcfg):
        """densify_and_cull (mapper.cpp:172-230): (split, cloned, removed)."""
        ch = np.zeros(3, np.int32)
        _check(self.L.orc_mapstate_densify(self.h, C.byref(mcfg), ch.ctypes.data_as(i32p)), self.L)
        return tuple(int(x) for x in ch)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_mapstate_free(self.h)
            self.h = None


def accumulate_uncertainty(m, results, depths, poses, K):
    n = len(results)
    keep = [np.ascontiguousarray(d, dtype=np.float64) for d in depths]
    rh = (C.c_void_p * max(n, 1))(*[r.h for r in results])
    dg = (dp * max(n, 1))(*[k.ctypes.data_as(dp) for k in keep])
    ps = (Pose * max(n, 1))(*[_as(Pose, p) for p in poses])
    cnt = C.c_int32()
    h = host_of(m)
    L = results[0].L if results else lib()
    _check(L.orc_accumulate_uncertainty(C.byref(h), n, rh, dg, ps, C.byref(K), C.byref(cnt)), L)
    return cnt.value


def backproject(rgb, depth, pose: Pose, K, mcfg, stride, opacity=None):
    """initialize_map / spawn_gaussians candidates (mapper.cpp:12-26, 125-170) as a new map."""
    r = np.ascontiguousarray(rgb, dtype=np.float64)
    d = np.ascontiguousarray(depth, dtype=np.float64)
    o = None if opacity is None else np.ascontiguousarray(opacity, dtype=np.float64)
    n = C.c_int64()
    _check(lib().orc_backproject(r.ctypes.data_as(dp), d.ctypes.data_as(dp), None if o is None else o.ctypes.data_as(dp),
                                 C.byref(pose), C.byref(K), C.byref(mcfg), stride, None, C.byref(n)))
    m = empty_map(n.value, mcfg.sh_coeffs)
    h = host_of(m)
    _check(lib().orc_backproject(r.ctypes.data_as(dp), d.ctypes.data_as(dp), None if o is None else o.ctypes.data_as(dp),
                                 C.byref(pose), C.byref(K), C.byref(mcfg), stride, C.byref(h), C.byref(n)))
    return m


def uncertainty_partials(m, results, depths, poses, K):
    """Per-primitive (sum, count) of Eq. 13 over the given views (uncertainty.cpp:35-73)."""
    n = len(results)
    keep = [np.ascontiguousarray(d, dtype=np.float64) for d in depths]
    rh = (C.c_void_p * max(n, 1))(*[r.h for r in results])
    dg = (dp * max(n, 1))(*[k.ctypes.data_as(dp) for k in keep])
    ps = (Pose * max(n, 1))(*[_as(Pose, p) for p in poses])
    P = m.mean.shape[0]
    s = np.zeros(max(P, 1))
    c = np.zeros(max(P, 1), np.int32)
    h = host_of(m)
    _check(lib().orc_uncertainty_partials(C.byref(h), n, rh, dg, ps, C.byref(K), s.ctypes.data_as(dp), c.ctypes.data_as(i32p)))
    return s[:P], c[:P]


def prune_unreliable(m, tau=0.025, reduced=0.005):
    r = C.c_int32()
    h = host_of(m)
    _check(lib().orc_prune_unreliable(C.byref(h), tau, reduced, C.byref(r)))
    return r.value


def gradcheck_linear(m, pose, K, cfg, obs, a_color, a_depth, a_opacity, a_uncert, a_median, step=1e-4, floor=1e-3):
    rep = GradcheckReport()
    keep = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in
            (obs, a_color, a_depth, a_opacity, a_uncert, a_median)]
    h = host_of(m)
    _check(lib().orc_gradcheck_linear(C.byref(h), C.byref(pose), C.byref(K), C.byref(cfg),
                                      *[None if a is None else a.ctypes.data_as(dp) for a in keep], step, floor,
                                      C.byref(rep)))
    return rep


def mirror_render(m, pose, K, obs=None, cfg=None, pair_capacity=1 << 22):
    cfg = cfg or defaults_raster()
    P = m.mean.shape[0]
    W, H = K.width, K.height
    ntiles = ((W + 15) // 16) * ((H + 15) // 16)
    o = SimpleNamespace(visible=np.zeros(max(P, 1), np.uint8), rank_to_id=np.zeros(max(P, 1), np.int32),
                        tile_range=np.zeros(2 * ntiles, np.int32), pair_rank=np.zeros(pair_capacity, np.int32),
                        color=np.zeros((H, W, 3), np.float32), alpha_depth=np.zeros((H, W), np.float32),
                        median_depth=np.zeros((H, W), np.float32), median_valid=np.zeros((H, W), np.uint8),
                        opacity=np.zeros((H, W), np.float32), uncertainty=np.zeros((H, W), np.float32),
                        final_transmittance=np.zeros((H, W), np.float32), per_pixel_count=np.zeros((H, W), np.int32),
                        dominant=np.zeros((H, W), np.int32), median_prim=np.zeros((H, W), np.int32),
                        dominant_weight=np.zeros((H, W), np.float32), last_index=np.zeros((H, W), np.int32))
    mo = MirOut(o.visible.ctypes.data_as(u8p), o.rank_to_id.ctypes.data_as(i32p), o.tile_range.ctypes.data_as(i32p),
                o.pair_rank.ctypes.data_as(i32p), pair_capacity, o.color.ctypes.data_as(fp), o.alpha_depth.ctypes.data_as(fp),
                o.median_depth.ctypes.data_as(fp), o.median_valid.ctypes.data_as(u8p), o.opacity.ctypes.data_as(fp),
                o.uncertainty.ctypes.data_as(fp), o.final_transmittance.ctypes.data_as(fp),
                o.per_pixel_count.ctypes.data_as(i32p), o.dominant.ctypes.data_as(i32p),
                o.median_prim.ctypes.data_as(i32p), o.dominant_weight.ctypes.data_as(fp), o.last_index.ctypes.data_as(i32p),
                0, 0, 0)
    ob = None if obs is None else np.ascontiguousarray(obs, dtype=np.float32)
    h = host_of(m)
    _check(lib().mir_render(C.byref(h), C.byref(pose), C.byref(K), None if ob is None else ob.ctypes.data_as(fp),
                            C.byref(cfg), C.byref(mo)))
    o.num_visible, o.num_pairs, o.num_flagged = int(mo.num_visible), int(mo.num_pairs), int(mo.num_flagged)
    o.visible = o.visible[:P]
    o.rank_to_id = o.rank_to_id[: o.num_visible]
    o.pair_rank = o.pair_rank[: o.num_pairs]
    return o


# ---- configuration defaults of the reference structs (from the active backend) ------------------
def defaults_raster() -> RasterCfg:
    c = RasterCfg()
    lib().orc_default_raster(C.byref(c))
    return c


def smooth_raster() -> RasterCfg:
    """smooth_raster_config() (gradcheck.cpp:21-27): no skip, no termination, footprint sigma 8."""
    c = RasterCfg()
    if reference_available():
        _load("reference").orc_smooth_raster(C.byref(c))
    else:
        c = defaults_raster()
        c.alpha_skip, c.termination_threshold, c.footprint_sigma = 0.0, 0.0, 8.0
    return c


def defaults_weights(handheld_real=False) -> LossWeights:
    w = LossWeights()
    lib().orc_default_weights(C.byref(w), 1 if handheld_real else 0)
    return w


def defaults_tracker() -> TrackerCfg:
    t = TrackerCfg()
    lib().orc_default_tracker(C.byref(t))
    return t


def defaults_mapper() -> MapperCfg:
    m = MapperCfg()
    lib().orc_default_mapper(C.byref(m))
    return m


def synth_scene(count, extent=4.0, wall_layers=3, seed=0, frames=50, radius=1.0, K: Intrinsics = None, kind=0):
    """The reference's own synthetic generator (io/synthetic.cpp:199-211: SyntheticSource's ground
    truth and trajectory; frames are not rendered).  Needs the reference backend library."""
    L = _load("reference")
    K = K or Intrinsics(600.0, 600.0, 599.5, 339.5, 1200, 680, 1.0, 0.1, 10.0)
    n = C.c_int64()
    poses = (Pose * frames)()
    rc = L.ref_synth_scene(kind, count, extent, wall_layers, frames, radius, seed, C.byref(K), None, C.byref(n), poses, 0)
    if rc:
        raise OracleError(rc, L.orc_last_error().decode())
    m = empty_map(n.value, 1)
    h = host_of(m)
    rc = L.ref_synth_scene(kind, count, extent, wall_layers, frames, radius, seed, C.byref(K), C.byref(h), C.byref(n),
                           poses, frames)
    if rc:
        raise OracleError(rc, L.orc_last_error().decode())
    return m, [poses[i] for i in range(frames)]
