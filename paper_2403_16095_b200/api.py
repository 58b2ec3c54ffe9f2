"""Python host mirror of the reference hot-path interface over the C-ABI.

Same function names, argument meaning and error behaviour as the reference's C++ entry points
(/root/reference/proj/include/gsfield): ``render`` / ``render_backward`` (raster/rasterizer.hpp:19-35),
``evaluate_tracking_loss`` / ``evaluate_mapping_loss`` (loss/losses.hpp:77-94), ``ssim``
(loss/ssim.hpp:11-14), ``track_frame`` / ``sliding_ba`` (track/tracker.hpp:38-57),
``map_step`` (map/mapper.hpp:101-103), ``accumulate_uncertainty`` / ``prune_unreliable``
(map/uncertainty.hpp:33-39).  ``std::invalid_argument`` surfaces as ``ValueError``,
``std::runtime_error`` (divergence) as ``RuntimeError``, runtime values the device path does not
implement as ``NotImplementedError``.  All arithmetic runs in libgsf_cuda.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import abi
from .abi import (GSF_EDIVERGED, GSF_EINVAL, GSF_ENONFINITE, GSF_ERUNTIME, GSF_EUNSUPPORTED, GSF_OK, GsfError,
                  Intrinsics, LossWeights, MapperCfg, Pose, RasterCfg, TrackerCfg)


def _f32(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    if shape is not None:
        out = out.reshape(shape)
    return out


def _ptr(a: Optional[np.ndarray], ctype=C.c_float):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def pose_of(rotation_tangent, translation) -> Pose:
    p = Pose()
    for i in range(3):
        p.rotation_tangent[i] = float(rotation_tangent[i])
        p.translation[i] = float(translation[i])
    return p


def pose_arrays(p: Pose):
    return np.array(list(p.rotation_tangent)), np.array(list(p.translation))


def intrinsics(fx, fy, cx, cy, width, height, near_plane=0.1, far_plane=100.0, depth_scale=1.0) -> Intrinsics:
    return Intrinsics(fx, fy, cx, cy, int(width), int(height), depth_scale, near_plane, far_plane)


@dataclass
class GaussianMap:
    """std::vector<GaussianPrimitive> as arrays (geometry/primitive.hpp:16-59)."""
    mean: np.ndarray            # (P,3)
    log_scale: np.ndarray       # (P,3)
    quat: np.ndarray            # (P,4) w,x,y,z
    opacity_logit: np.ndarray   # (P,)
    sh: np.ndarray              # (P,K,3)
    uncertainty: np.ndarray = None
    observed: np.ndarray = None

    def __post_init__(self):
        self.mean = np.ascontiguousarray(self.mean, dtype=np.float64).reshape(-1, 3)
        P = self.mean.shape[0]
        self.log_scale = np.ascontiguousarray(self.log_scale, dtype=np.float64).reshape(P, 3)
        self.quat = np.ascontiguousarray(self.quat, dtype=np.float64).reshape(P, 4)
        self.opacity_logit = np.ascontiguousarray(self.opacity_logit, dtype=np.float64).reshape(P)
        sh = np.ascontiguousarray(self.sh, dtype=np.float64)
        k = sh.shape[1] if sh.ndim == 3 else (sh.size // max(P, 1) // 3 if P else 1)
        self.sh = sh.reshape(P, k, 3)
        if self.uncertainty is None:
            self.uncertainty = np.zeros(P)
        self.uncertainty = np.ascontiguousarray(self.uncertainty, dtype=np.float64).reshape(P)
        if self.observed is None:
            self.observed = np.zeros(P, dtype=np.uint8)
        self.observed = np.ascontiguousarray(self.observed, dtype=np.uint8).reshape(P)

    @property
    def count(self) -> int:
        return self.mean.shape[0]

    @property
    def sh_coeffs(self) -> int:
        return self.sh.shape[1]

    def host(self) -> abi.MapHost:
        d = C.POINTER(C.c_double)
        return abi.MapHost(self.count, self.sh_coeffs, self.mean.ctypes.data_as(d), self.log_scale.ctypes.data_as(d),
                           self.quat.ctypes.data_as(d), self.opacity_logit.ctypes.data_as(d),
                           self.sh.ctypes.data_as(d), self.uncertainty.ctypes.data_as(d),
                           self.observed.ctypes.data_as(C.POINTER(C.c_uint8)))

    @staticmethod
    def empty(P: int, K: int = 1) -> "GaussianMap":
        q = np.zeros((P, 4))
        q[:, 0] = 1.0
        return GaussianMap(np.zeros((P, 3)), np.zeros((P, 3)), q, np.zeros(P), np.zeros((P, K, 3)))

    def copy(self) -> "GaussianMap":
        return GaussianMap(self.mean.copy(), self.log_scale.copy(), self.quat.copy(), self.opacity_logit.copy(),
                           self.sh.copy(), self.uncertainty.copy(), self.observed.copy())


@dataclass
class RenderResult:
    """RenderOutput + the per-pixel parts of BlendRecord (raster/output.hpp:15-50)."""
    color: np.ndarray
    alpha_depth: np.ndarray
    median_depth: np.ndarray
    median_valid: np.ndarray
    opacity: np.ndarray
    uncertainty: np.ndarray
    final_transmittance: np.ndarray
    per_pixel_count: np.ndarray
    dominant: np.ndarray
    median_prim: np.ndarray
    dominant_weight: np.ndarray
    visible: np.ndarray
    has_uncertainty: bool
    num_visible: int
    num_pairs: int


@dataclass
class GradientBundle:
    """GradientBundle (raster/output.hpp:64-77)."""
    d_mean: np.ndarray
    d_log_scale: np.ndarray
    d_quat: np.ndarray
    d_opacity_logit: np.ndarray
    d_sh: np.ndarray
    d_mean2d: np.ndarray
    d_pose: np.ndarray


def _raise(status: int, msg: str, index: int = -1):
    if status == GSF_OK:
        return
    if status in (GSF_EINVAL, GSF_ENONFINITE):
        e = ValueError(msg)
        e.index = index
        raise e
    if status in (GSF_EDIVERGED, GSF_ERUNTIME):
        raise RuntimeError(msg)
    if status == GSF_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise GsfError(status, msg, index)


class Context:
    """One device context: resident map, workspace and frame slots (gsf_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = abi.load()
        h = C.c_void_p()
        rc = self.lib.gsf_ctx_create(int(device), C.byref(h))
        if rc != GSF_OK:
            raise GsfError(rc, f"gsf_ctx_create({device}) failed: no usable CUDA device or kernels (status {rc})")
        self.h = h
        self.K = 1
        self.P = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.gsf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != GSF_OK:
            _raise(rc, self.lib.gsf_last_error(self.h).decode(), int(self.lib.gsf_last_error_index(self.h)))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.gsf_kernel_launches(self.h))

    def reserve(self, pair_cap: int = 0, bucket_cap: int = 0):
        """Pre-size the binning capacities ((tile, primitive) pairs, per-tile bucket entries)."""
        self._check(self.lib.gsf_reserve(self.h, int(pair_cap), int(bucket_cap)))

    def capacity(self):
        a, b = C.c_int64(), C.c_int64()
        self._check(self.lib.gsf_capacity(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    # ---- map -----------------------------------------------------------------------------
    def upload(self, m: GaussianMap):
        hm = m.host()
        self._check(self.lib.gsf_map_upload(self.h, C.byref(hm)))
        self.P, self.K = m.count, m.sh_coeffs

    def download(self) -> GaussianMap:
        m = GaussianMap.empty(self.P, self.K)
        hm = m.host()
        self._check(self.lib.gsf_map_download(self.h, C.byref(hm)))
        return m

    def optimizer_reset(self):
        self._check(self.lib.gsf_optimizer_reset(self.h))

    # ---- forward / backward ----------------------------------------------------------------
    def render(self, pose: Pose, K: Intrinsics, observed_depth=None, cfg: RasterCfg = None,
               reference: bool = False) -> RenderResult:
        """render (rasterizer.cpp:168-261); reference=True: render_reference (:263-296, no termination)."""
        cfg = cfg or abi.defaults_raster()
        W, H = K.width, K.height
        n = max(W, 0) * max(H, 0)
        o = dict(color=np.zeros((max(H, 0), max(W, 0), 3), np.float32),
                 alpha_depth=np.zeros((H, W), np.float32) if n else np.zeros(0, np.float32),
                 median_depth=np.zeros((H, W), np.float32) if n else np.zeros(0, np.float32),
                 median_valid=np.zeros((H, W), np.uint8) if n else np.zeros(0, np.uint8),
                 opacity=np.zeros((H, W), np.float32) if n else np.zeros(0, np.float32),
                 uncertainty=np.zeros((H, W), np.float32) if n else np.zeros(0, np.float32),
                 final_transmittance=np.zeros((H, W), np.float32) if n else np.zeros(0, np.float32),
                 per_pixel_count=np.zeros((H, W), np.int32) if n else np.zeros(0, np.int32),
                 dominant=np.zeros((H, W), np.int32) if n else np.zeros(0, np.int32),
                 median_prim=np.zeros((H, W), np.int32) if n else np.zeros(0, np.int32),
                 dominant_weight=np.zeros((H, W), np.float32) if n else np.zeros(0, np.float32),
                 visible=np.zeros(max(self.P, 1), np.uint8))
        ro = abi.RenderOut(_ptr(o["color"]), _ptr(o["alpha_depth"]), _ptr(o["median_depth"]),
                           _ptr(o["median_valid"], C.c_uint8), _ptr(o["opacity"]), _ptr(o["uncertainty"]),
                           _ptr(o["final_transmittance"]), _ptr(o["per_pixel_count"], C.c_int32),
                           _ptr(o["dominant"], C.c_int32), _ptr(o["median_prim"], C.c_int32),
                           _ptr(o["dominant_weight"]), _ptr(o["visible"], C.c_uint8), 0, 0, 0)
        obs = None
        if observed_depth is not None:
            obs = _f32(observed_depth)
            if obs.size != n:
                raise ValueError("render: observed depth dimensions do not match intrinsics")
        fn = self.lib.gsf_render_reference if reference else self.lib.gsf_render
        self._check(fn(self.h, C.byref(pose), C.byref(K), _ptr(obs), C.byref(cfg), C.byref(ro)))
        o["visible"] = o["visible"][: self.P]
        return RenderResult(**o, has_uncertainty=bool(ro.has_uncertainty), num_visible=int(ro.num_visible),
                            num_pairs=int(ro.num_pairs))

    def render_tiles(self, num_tiles: int, num_pairs: int):
        """(tile_range (tiles, 2), pair_prim) of the last render: every tile list as primitive ids."""
        tr = np.zeros(2 * max(num_tiles, 1), np.int32)
        pp = np.zeros(max(num_pairs, 1), np.int32)
        self._check(self.lib.gsf_render_tiles(self.h, _ptr(tr, C.c_int32), num_tiles, _ptr(pp, C.c_int32), pp.size))
        return tr[: 2 * num_tiles].reshape(-1, 2), pp[:num_pairs]

    def render_record(self):
        """CSR BlendRecord of the last render: (row_start, prim, alpha, transmittance)."""
        total = C.c_int64()
        self._check(self.lib.gsf_render_record(self.h, None, None, None, None, C.byref(total)))
        # row_start size = W*H+1; query it from a second call with buffers
        return total.value

    def render_record_full(self, npix: int):
        total = C.c_int64()
        rs = np.zeros(npix + 1, np.uint32)
        self._check(self.lib.gsf_render_record(self.h, _ptr(rs, C.c_uint32), None, None, None, C.byref(total)))
        prim = np.zeros(max(total.value, 1), np.int32)
        alpha = np.zeros(max(total.value, 1), np.float32)
        tr = np.zeros(max(total.value, 1), np.float32)
        self._check(self.lib.gsf_render_record(self.h, _ptr(rs, C.c_uint32), _ptr(prim, C.c_int32), _ptr(alpha),
                                               _ptr(tr), C.byref(total)))
        t = total.value
        return rs, prim[:t], alpha[:t], tr[:t]

    def render_backward(self, d_color=None, d_alpha_depth=None, d_median_depth=None, d_opacity=None,
                        d_uncertainty=None, observed_depth=None) -> GradientBundle:
        maps = [None if a is None else _f32(a) for a in (d_color, d_alpha_depth, d_median_depth, d_opacity,
                                                          d_uncertainty)]
        up = abi.Upstream(*[_ptr(a) for a in maps])
        P, K = self.P, self.K
        g = dict(d_mean=np.zeros((P, 3), np.float32), d_log_scale=np.zeros((P, 3), np.float32),
                 d_quat=np.zeros((P, 4), np.float32), d_opacity_logit=np.zeros(P, np.float32),
                 d_sh=np.zeros((P, K, 3), np.float32), d_mean2d=np.zeros((P, 2), np.float32))
        go = abi.GradsOut(*[_ptr(g[k]) for k in ("d_mean", "d_log_scale", "d_quat", "d_opacity_logit", "d_sh",
                                                 "d_mean2d")])
        obs = None if observed_depth is None else _f32(observed_depth)
        self._check(self.lib.gsf_render_backward(self.h, C.byref(up), _ptr(obs), C.byref(go)))
        return GradientBundle(**g, d_pose=np.array(list(go.d_pose)))

    # ---- losses -------------------------------------------------------------------------------
    def evaluate_tracking_loss(self, target_rgb, observed_depth, w: LossWeights, want_gradients=True):
        t, d = _f32(target_rgb), _f32(observed_depth)
        n = d.size
        out = abi.LossTerms()
        dc = np.zeros(3 * n, np.float32) if want_gradients else None
        dd = np.zeros(n, np.float32) if want_gradients else None
        self._check(self.lib.gsf_tracking_loss(self.h, _ptr(t), _ptr(d), C.byref(w), C.byref(out), _ptr(dc), _ptr(dd)))
        return out, dc, dd

    def evaluate_mapping_loss(self, target_rgb, observed_depth, w: LossWeights, want_gradients=True):
        t, d = _f32(target_rgb), _f32(observed_depth)
        n = d.size
        out = abi.LossTerms()
        bufs = [np.zeros(3 * n, np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32),
                np.zeros(n, np.float32), np.zeros(3 * max(self.P, 1), np.float32)] if want_gradients else [None] * 5
        self._check(self.lib.gsf_mapping_loss(self.h, _ptr(t), _ptr(d), C.byref(w), C.byref(out),
                                              *[_ptr(b) for b in bufs]))
        return out, bufs

    def ssim(self, x, y, width: int, height: int, want_gradient=False):
        xa, ya = _f32(x), _f32(y)
        v = C.c_double()
        g = np.zeros(3 * width * height, np.float32) if want_gradient else None
        self._check(self.lib.gsf_ssim(self.h, _ptr(xa), _ptr(ya), width, height, C.byref(v), _ptr(g)))
        return (v.value, g) if want_gradient else v.value

    # ---- loops ----------------------------------------------------------------------------------
    def frame_upload(self, slot: int, rgb, depth, width: int, height: int):
        self._check(self.lib.gsf_frame_upload(self.h, slot, _ptr(_f32(rgb)), _ptr(_f32(depth)), width, height))

    def track_frame(self, slot: int, initial: Pose, K: Intrinsics, tcfg: TrackerCfg = None, w: LossWeights = None,
                    raster: RasterCfg = None) -> abi.TrackResult:
        tcfg = tcfg or abi.defaults_tracker()
        w = w or abi.defaults_weights()
        raster = raster or abi.defaults_raster()
        out = abi.TrackResult()
        self._check(self.lib.gsf_track_frame(self.h, slot, C.byref(initial), C.byref(K), C.byref(tcfg), C.byref(w),
                                             C.byref(raster), C.byref(out)))
        return out

    def tracking_gradient(self, slot: int, pose: Pose, K: Intrinsics, w: LossWeights = None,
                          raster: RasterCfg = None):
        """Tracking objective and its pose gradient at `pose` (one track_frame iteration)."""
        w = w or abi.defaults_weights()
        raster = raster or abi.defaults_raster()
        terms = abi.LossTerms()
        g = (C.c_double * 6)()
        self._check(self.lib.gsf_tracking_gradient(self.h, slot, C.byref(pose), C.byref(K), C.byref(w), C.byref(raster),
                                                   C.byref(terms), C.byref(g)))
        return terms, np.array(list(g))

    def map_step(self, slots: Sequence[int], poses: Sequence[Pose], K: Intrinsics, mcfg: MapperCfg = None,
                 iterations: int = 60):
        mcfg = mcfg or abi.defaults_mapper()
        n = len(slots)
        s = (C.c_int32 * max(n, 1))(*slots)
        ps = (Pose * max(n, 1))(*poses)
        trace = np.zeros(max(iterations, 1), np.float64)
        self._check(self.lib.gsf_map_step(self.h, s, ps, n, C.byref(K), C.byref(mcfg), iterations,
                                          trace.ctypes.data_as(C.POINTER(C.c_double))))
        self._sync_count(self.K)   # densify_and_cull may have resized the map
        return trace[:iterations]

    def sliding_ba(self, slots: Sequence[int], poses: Sequence[Pose], frame_ids: Sequence[int], K: Intrinsics,
                   tcfg: TrackerCfg = None, mcfg: MapperCfg = None, iterations: int = 10):
        tcfg = tcfg or abi.defaults_tracker()
        mcfg = mcfg or abi.defaults_mapper()
        n = len(slots)
        s = (C.c_int32 * max(n, 1))(*slots)
        ps = (Pose * max(n, 1))(*poses)
        fid = (C.c_int32 * max(n, 1))(*frame_ids)
        trace = np.zeros(max(iterations, 1), np.float64)
        self._check(self.lib.gsf_sliding_ba(self.h, s, ps, fid, n, C.byref(K), C.byref(tcfg), C.byref(mcfg),
                                            iterations, trace.ctypes.data_as(C.POINTER(C.c_double))))
        return trace[:iterations], [ps[i] for i in range(n)]

    def accumulate_uncertainty(self, slots: Sequence[int], poses: Sequence[Pose], K: Intrinsics,
                               raster: RasterCfg = None) -> int:
        raster = raster or abi.defaults_raster()
        n = len(slots)
        s = (C.c_int32 * max(n, 1))(*slots)
        ps = (Pose * max(n, 1))(*poses)
        cnt = C.c_int32()
        self._check(self.lib.gsf_accumulate_uncertainty(self.h, s, ps, n, C.byref(K), C.byref(raster), C.byref(cnt)))
        return cnt.value

    def _sync_count(self, sh_coeffs: int):
        self.P, self.K = int(self.lib.gsf_map_count(self.h)), sh_coeffs

    def initialize_map(self, slot: int, pose: Pose, K: Intrinsics, mcfg: MapperCfg = None) -> int:
        """initialize_map (mapper.cpp:125-148) from frame `slot`: replaces the map, resets the optimizer."""
        mcfg = mcfg or abi.defaults_mapper()
        n = C.c_int64()
        self._check(self.lib.gsf_initialize_map(self.h, slot, C.byref(pose), C.byref(K), C.byref(mcfg), C.byref(n)))
        self._sync_count(mcfg.sh_coeffs)
        return n.value

    def spawn_gaussians(self, slot: int, pose: Pose, K: Intrinsics, mcfg: MapperCfg = None) -> int:
        """spawn_gaussians (mapper.cpp:150-170) against the most recent render on this context."""
        mcfg = mcfg or abi.defaults_mapper()
        n = C.c_int32()
        self._check(self.lib.gsf_spawn_gaussians(self.h, slot, C.byref(pose), C.byref(K), C.byref(mcfg), C.byref(n)))
        self._sync_count(mcfg.sh_coeffs)
        return n.value

    def save_checkpoint(self, path: str, K: Intrinsics):
        """save_checkpoint (io/checkpoint.cpp:36-60): GSFMAP01 file of the device map."""
        self._check(self.lib.gsf_checkpoint_save(self.h, os.fsencode(path), C.byref(K)))

    def load_checkpoint(self, path: str) -> Intrinsics:
        """load_checkpoint (io/checkpoint.cpp:62-100): replaces the map; returns the intrinsics."""
        K = abi.Intrinsics()
        self._check(self.lib.gsf_checkpoint_load(self.h, os.fsencode(path), C.byref(K)))
        self.P = int(self.lib.gsf_map_count(self.h))
        self.K = self.download_sh_coeffs()
        return K

    def download_sh_coeffs(self) -> int:
        return int(self.lib.gsf_map_sh_coeffs(self.h))

    def densify_and_cull(self, mcfg: MapperCfg = None):
        """densify_and_cull (mapper.cpp:172-230): returns (split, cloned, removed)."""
        mcfg = mcfg or abi.defaults_mapper()
        ch = abi.StructuralChange()
        self._check(self.lib.gsf_densify_and_cull(self.h, C.byref(mcfg), C.byref(ch)))
        self._sync_count(self.K)
        return ch.split, ch.cloned, ch.removed

    def map_stats(self):
        """(grad_accum, grad_count) densification statistics of the map (MapState, mapper.hpp:76-77)."""
        a = np.zeros(max(self.P, 1))
        c = np.zeros(max(self.P, 1), np.int32)
        self._check(self.lib.gsf_map_stats_download(self.h, a.ctypes.data_as(C.POINTER(C.c_double)),
                                                    c.ctypes.data_as(C.POINTER(C.c_int32))))
        return a[: self.P], c[: self.P]

    def set_map_stats(self, grad_accum, grad_count):
        a = np.ascontiguousarray(grad_accum, dtype=np.float64)
        c = np.ascontiguousarray(grad_count, dtype=np.int32)
        assert a.size == self.P and c.size == self.P
        self._check(self.lib.gsf_map_stats_upload(self.h, a.ctypes.data_as(C.POINTER(C.c_double)),
                                                  c.ctypes.data_as(C.POINTER(C.c_int32))))

    def prune_unreliable(self, tau: float = 0.025, reduced_opacity: float = 0.005) -> int:
        r = C.c_int32()
        self._check(self.lib.gsf_prune_unreliable(self.h, tau, reduced_opacity, C.byref(r)))
        return r.value

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        arr = (C.c_uint8 * 128)(*uid)
        self._check(self.lib.gsf_comm_init(self.h, nranks, rank, C.byref(arr)))

    def comm_setup_host(self, group=None):
        """Join the torch.distributed job through a host-staged communicator: every sum-all-reduce of
        the sharded paths is staged through pinned host memory and summed by torch.distributed over
        `group` (any backend, e.g. gloo).  Same decomposition as the NCCL path."""
        import torch
        import torch.distributed as dist
        dt = {abi.GSF_DT_U32: (np.uint32, torch.int64), abi.GSF_DT_F32: (np.float32, torch.float32),
              abi.GSF_DT_F64: (np.float64, torch.float64)}

        def _allreduce(buf, count, dtype, user):
            try:
                npt, tt = dt[dtype]
                a = np.ctypeslib.as_array(C.cast(buf, C.POINTER(np.ctypeslib.as_ctypes_type(npt))), (count,))
                t = torch.from_numpy(a.astype(np.int64) if dtype == abi.GSF_DT_U32 else a.copy()).to(tt)
                dist.all_reduce(t, group=group)
                a[...] = t.numpy().astype(npt)
                return 0
            except Exception:   # noqa: BLE001 (reported to the library as a failed exchange)
                return 1

        self._host_ar = abi.HOST_ALLREDUCE_FN(_allreduce)   # kept alive with the context
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self._check(self.lib.gsf_comm_init_host(self.h, world, rank, C.cast(self._host_ar, C.c_void_p), None))

    def comm_setup(self, group=None):
        """Join this context to the torch.distributed job: rank 0 draws the NCCL unique id, it is
        broadcast over `group` (any backend), then every rank calls gsf_comm_init."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.comm_init(world, rank, exchange_unique_id(group))


def comm_unique_id() -> bytes:
    lib = abi.load()
    arr = (C.c_uint8 * 128)()
    rc = lib.gsf_comm_unique_id(C.byref(arr))
    if rc != GSF_OK:
        raise GsfError(rc, "ncclGetUniqueId failed")
    return bytes(arr)


def exchange_unique_id(group=None) -> bytes:
    """Rank 0's NCCL unique id, broadcast to every rank of `group` over torch.distributed."""
    import torch.distributed as dist
    if dist.get_world_size(group) == 1:
        return bytes(128)
    obj = [comm_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise GsfError(GSF_EINVAL, "comm_setup: malformed NCCL unique id")
    return bytes(uid)


def ba_partition(n: int, nranks: int, rank: int) -> np.ndarray:
    """Keyframes rank `rank` renders in a keyframe-sharded sliding_ba (host logic, no device)."""
    lib = abi.load()
    out = np.zeros(max(n, 1), np.uint8)
    rc = lib.gsf_ba_partition(n, nranks, rank, out.ctypes.data_as(C.POINTER(C.c_uint8)))
    if rc != GSF_OK:
        raise ValueError("ba_partition: bad arguments")
    return out[:n].astype(bool)


class SlamSystem:
    """SlamSystem (slam/system.hpp) on a Context's device map: process() frames in stream order."""

    def __init__(self, ctx: Context, cfg: "abi.SlamCfg"):
        self.ctx = ctx
        self.cfg = cfg
        h = C.c_void_p()
        rc = ctx.lib.gsf_slam_create(ctx.h, C.byref(cfg), C.byref(h))
        if rc != GSF_OK:
            raise ValueError("invalid SLAM configuration")
        self.h = h
        self.logs = []

    def process(self, index: int, timestamp: float, rgb, depth) -> "abi.FrameLog":
        log = abi.FrameLog()
        r, d = _f32(rgb), _f32(depth)
        self.ctx._check(self.ctx.lib.gsf_slam_process(self.h, index, timestamp, _ptr(r), _ptr(d), C.byref(log)))
        self.ctx.P = int(self.ctx.lib.gsf_map_count(self.ctx.h))
        self.ctx.K = int(self.ctx.lib.gsf_map_sh_coeffs(self.ctx.h))
        self.logs.append(log)
        return log

    @property
    def keyframes(self) -> int:
        return int(self.ctx.lib.gsf_slam_keyframes(self.h))

    @property
    def degraded_frames(self) -> int:
        return int(self.ctx.lib.gsf_slam_degraded_frames(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.gsf_slam_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
