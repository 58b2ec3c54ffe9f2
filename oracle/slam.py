"""Test infrastructure: SlamSystem::process (slam/system.cpp:31-154) restated in Python over the fp64
oracle's primitives, to check the device pipeline (csrc/slam.cpp behind gsf_slam_*) step by step.
Only tests import this module."""
import numpy as np
from scipy.spatial.transform import Rotation as Rot

import oracle as orc
from paper_2403_16095_b200.abi import Pose


def _mat(p):
    return Rot.from_rotvec(list(p.rotation_tangent)).as_matrix(), np.array(list(p.translation))


def _pose(R, t):
    return Pose((*Rot.from_matrix(R).as_rotvec(),), (*np.asarray(t, dtype=np.float64),))


def compose(a, b):   # pose.hpp:29-33: apply b first, then a
    Ra, ta = _mat(a)
    Rb, tb = _mat(b)
    return _pose(Ra @ Rb, Ra @ tb + ta)


def inverse(p):      # pose.hpp:35-38
    R, t = _mat(p)
    return _pose(R.T, -(R.T @ t))


def predict_pose(prev, before):   # tracker.cpp:26-28
    return compose(prev, compose(inverse(before), prev))


def descriptor(rgb):  # descriptor.cpp:9-43
    h, w, _ = rgb.shape
    d = np.zeros(8 * 8 + 3 * 16)
    lum = 0.299 * rgb[..., 0] + 0.587 * rgb[..., 1] + 0.114 * rgb[..., 2]
    for gy in range(8):
        for gx in range(8):
            x0, y0 = w * gx // 8, h * gy // 8
            x1, y1 = max(w * (gx + 1) // 8, x0 + 1), max(h * (gy + 1) // 8, y0 + 1)
            cell = lum[y0:min(y1, h), x0:min(x1, w)]
            if cell.size:
                d[gy * 8 + gx] = cell.mean()
    v = np.clip(rgb.reshape(-1, 3).astype(np.float64), 0.0, 1.0)
    for c in range(3):
        bins = np.minimum(15, (v[:, c] * 16.0).astype(int))
        d[64 + c * 16: 64 + c * 16 + 16] += np.bincount(bins, minlength=16) / v.shape[0]
    n = np.linalg.norm(d)
    return d / n if n > 0 else d


def select_window(pool, cfg):   # tracker.cpp:86-117
    n = len(pool)
    cur = n - 1
    window, taken = [cur], {cur}
    i = cur - 1
    while i >= 0 and len(window) < cfg.ba_window and cur - i <= cfg.recent_keyframes:
        window.append(i)
        taken.add(i)
        i -= 1

    def cos(a, b):
        na, nb = np.linalg.norm(a), np.linalg.norm(b)
        return 0.0 if na == 0 or nb == 0 else float(a @ b / (na * nb))
    rest = sorted(((cos(pool[i]["desc"], pool[cur]["desc"]), i) for i in range(n) if i not in taken),
                  key=lambda s: (-s[0], -s[1]))
    for _, i in rest:
        if len(window) >= cfg.ba_window:
            break
        window.append(i)
    return window


class OracleSlam:
    def __init__(self, cfg):
        self.cfg = cfg
        self.mapper = cfg.mapper
        self.mapper.seed = cfg.seed
        self.st = None
        self.keyframes, self.trajectory = [], []
        self.prev = self.prev_prev = None

    def process(self, index, rgb, depth):
        c, K = self.cfg, self.cfg.intrinsics
        rgb, depth = rgb.astype(np.float64), depth.astype(np.float64)
        if self.st is None:
            origin = Pose((0.0, 0.0, 0.0), (0.0, 0.0, 0.0))
            self.keyframes.append(dict(id=index, rgb=rgb, depth=depth, pose=origin, desc=descriptor(rgb)))
            m0 = orc.backproject(rgb, depth, origin, K, self.mapper, self.mapper.init_stride)
            self.st = orc.MapState(m0, self.mapper)
            self.st.map_step([(rgb, depth)], [origin], K, self.mapper, c.init_iterations)
            self.prev = self.prev_prev = origin
            self.trajectory.append(origin)
            return origin
        predicted = self.prev if len(self.trajectory) < 2 else predict_pose(self.prev, self.prev_prev)
        res = orc.track_frame(self.st.get(), rgb, depth, predicted, K, c.tracker, self.mapper.weights, self.mapper.raster)
        self.prev_prev, self.prev = self.prev, res.pose
        self.trajectory.append(res.pose)
        if index % c.tracker.keyframe_interval == 0:
            self._keyframe_cycle(index, rgb, depth)
        return self.trajectory[-1]

    def _keyframe_cycle(self, index, rgb, depth):
        c, K = self.cfg, self.cfg.intrinsics
        self.keyframes.append(dict(id=index, rgb=rgb, depth=depth, pose=self.trajectory[-1], desc=descriptor(rgb)))
        win = select_window(self.keyframes, c.tracker)
        frames = [(self.keyframes[k]["rgb"], self.keyframes[k]["depth"]) for k in win]
        poses = [self.keyframes[k]["pose"] for k in win]
        self.st.map_step(frames, poses, K, self.mapper, c.map_iterations)
        _, poses = self.st.sliding_ba(frames, poses, [self.keyframes[k]["id"] for k in win], K, c.tracker, self.mapper,
                                      c.tracker.ba_iterations)
        for k, p in zip(win, poses):
            self.keyframes[k]["pose"] = p
        self.trajectory[-1] = self.keyframes[-1]["pose"]
        self.prev = self.keyframes[-1]["pose"]
        m = self.st.get()
        renders = [orc.render(m, p, K, self.keyframes[k]["depth"]) for k, p in zip(win, poses)]
        orc.accumulate_uncertainty(m, renders, [self.keyframes[k]["depth"] for k in win], poses, K)
        orc.prune_unreliable(m, self.mapper.uncertainty_tau, self.mapper.uncertainty_reduced_opacity)
        self.st.put(m)
        cur = self.keyframes[-1]
        now = orc.render(self.st.get(), cur["pose"], K, cur["depth"])
        new = orc.backproject(cur["rgb"], cur["depth"], cur["pose"], K, self.mapper, self.mapper.spawn_stride,
                              opacity=now.opacity)
        if new.mean.shape[0]:
            self.st.append(new)

    @property
    def primitives(self):
        from oracle import lib
        return int(lib().orc_mapstate_count(self.st.h))
