"""World-size-2 CPU tests (gloo) of the multi-GPU host logic: keyframe-sharded sliding_ba and
view-sharded accumulate_uncertainty.

The device path (`gsf_sliding_ba` with nranks > 1, csrc/abi.cu) renders only the keyframes
`gsf_ba_partition` assigns to its rank, sums their bundles locally, all-reduces the flat gradient,
the loss and the per-keyframe pose gradients, then runs identical Adam updates on every rank.
These tests replay exactly that decomposition with the fp64 oracle as the per-keyframe gradient
(reference: track/tracker.cpp sliding_ba, the loop the oracle restates in orc_sliding_ba) and
torch.distributed/gloo as the all-reduce, and check it against the unsharded sum.  They also cover
the NCCL unique-id exchange `Context.comm_setup` performs, and the (sum, count) all-reduce of the
uncertainty pass.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_16095_b200 import abi, api
from helpers import make_intrinsics, perturbed, pose

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _window(n):
    import oracle as orc
    K = make_intrinsics(48, 36, 40.0)
    truth = orc.random_scene(91, 60, 1, 0.95, 0.05, 0.2)
    m = orc.random_scene(91, 60, 1, 0.95, 0.05, 0.2)
    rng = np.random.default_rng(91)
    m.mean = m.mean + 0.02 * rng.standard_normal(m.mean.shape)
    m.sh[:, 0] = m.sh[:, 0] + 0.1 * rng.standard_normal(m.sh[:, 0].shape)
    poses, frames = [], []
    for k in range(n):
        p = perturbed(pose(), [0.01 * k, -0.005 * k, 0.004, 0.02 * k, 0.01, -0.01 * k])
        r = orc.render(truth, p, K)
        poses.append(perturbed(p, [0.002, 0, -0.001, 0.003, 0.001, 0]) if k else p)
        frames.append((r.color.copy(), np.where(r.opacity > 0.5, r.alpha_depth, 0.0)))
    return m, K, poses, frames


def _keyframe_bundle(m, K, p, frame, mc):
    """One keyframe's contribution: mapping loss + render_backward + the direct log-scale term."""
    import oracle as orc
    rgb, obs = frame
    r = orc.render(m, p, K, obs, mc.raster)
    loss, (dc, dad, dmd, du, dls) = orc.mapping_loss(m, r, rgb, obs, K, mc.weights)
    g = orc.render_backward(m, p, K, r, d_color=dc, d_alpha_depth=dad, d_median_depth=dmd, d_uncertainty=du,
                            obs=obs, cfg=mc.raster)
    flat = np.concatenate([g.d_mean.ravel(), (g.d_log_scale + dls.reshape(-1, 3)[: g.d_log_scale.shape[0]]).ravel(),
                           g.d_quat.ravel(), g.d_opacity_logit.ravel(), g.d_sh.ravel()])
    return flat, loss.total, g.d_pose


def _sharded(n, rank, world):
    mc = abi.defaults_mapper()
    m, K, poses, frames = _window(n)
    owned = api.ba_partition(n, world, rank)
    P = m.mean.shape[0]
    grad = np.zeros(P * (3 + 3 + 4 + 1 + 3 * m.sh.shape[1]))
    loss = np.zeros(1)
    pose_g = np.zeros((n, 6))
    for k in np.nonzero(owned)[0]:
        f, l, dp = _keyframe_bundle(m, K, poses[k], frames[k], mc)
        grad += f
        loss += l
        pose_g[k] = dp
    bufs = [torch.from_numpy(grad), torch.from_numpy(loss), torch.from_numpy(pose_g)]
    for b in bufs:
        dist.all_reduce(b)
    return [b.numpy() for b in bufs], owned


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        (grad, loss, pose_g), owned = _sharded(n, rank, world)
        # every rank must hold bit-identical reduced buffers (identical Adam updates afterwards)
        gathered = [torch.zeros(grad.size, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(grad))
        same = all(torch.equal(gathered[0], g) for g in gathered)
        uid = api.exchange_unique_id()
        uids = [None] * world
        dist.all_gather_object(uids, uid)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), grad=grad, loss=loss, pose=pose_g, owned=owned,
                 same=np.array(same), uid_same=np.array(all(u == uids[0] for u in uids)),
                 uid_len=np.array(len(uid)))
    finally:
        dist.destroy_process_group()


def _unc_window():
    import oracle as orc
    K = make_intrinsics(40, 30, 35.0)
    m = orc.random_scene(123, 70, 1, 0.95, 0.05, 0.2)
    poses = [perturbed(pose(), [0.01 * k, -0.01 * k, 0.005, 0.02 * k, 0.0, -0.01]) for k in range(5)]
    depths = [orc.wavy_depth(40, 30, 2.0 + 0.1 * k) for k in range(5)]
    renders = [orc.render(m, p, K, d) for p, d in zip(poses, depths)]
    return orc, m, K, poses, depths, renders


def _unc_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc, m, K, poses, depths, renders = _unc_window()
        mine = [v for v in range(len(poses)) if v % world == rank]   # gsf_accumulate_uncertainty's split
        s, c = orc.uncertainty_partials(m, [renders[v] for v in mine], [depths[v] for v in mine],
                                        [poses[v] for v in mine], K)
        ts, tc = torch.from_numpy(s.copy()), torch.from_numpy(c.astype(np.int64))
        dist.all_reduce(ts)
        dist.all_reduce(tc)
        np.savez(os.path.join(out_dir, f"unc{rank}.npz"), s=ts.numpy(), c=tc.numpy())
    finally:
        dist.destroy_process_group()


def test_sharded_uncertainty_matches_unsharded(tmp_path):
    """accumulate_uncertainty over a window split by view across two ranks (uncertainty.cpp:35-85):
    the all-reduced (sum, count) partials give the single-process nu and observed flags."""
    mp.spawn(_unc_worker, args=(WORLD, _free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    orc, m, K, poses, depths, renders = _unc_window()
    observed = orc.accumulate_uncertainty(m, renders, depths, poses, K)
    for r in range(WORLD):
        z = np.load(tmp_path / f"unc{r}.npz")
        seen = z["c"] > 0
        assert int(seen.sum()) == observed > 0
        assert (seen == (m.observed[: len(seen)] != 0)).all()
        nu = np.where(seen, z["s"] / np.maximum(z["c"], 1), 0.0)
        np.testing.assert_allclose(nu[seen], m.uncertainty[seen], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("n", [5, 1])
def test_sharded_sliding_ba_matches_unsharded(tmp_path, n):
    mp.spawn(_worker, args=(WORLD, _free_port(), n, str(tmp_path)), nprocs=WORLD, join=True)
    mc = abi.defaults_mapper()
    m, K, poses, frames = _window(n)
    ref_grad, ref_loss, ref_pose = 0.0, 0.0, np.zeros((n, 6))
    for k in range(n):
        f, l, dp = _keyframe_bundle(m, K, poses[k], frames[k], mc)
        ref_grad = ref_grad + f
        ref_loss += l
        ref_pose[k] = dp
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(WORLD)]
    owned = np.stack([r["owned"] for r in res])
    assert (owned.sum(0) == 1).all(), "every keyframe rendered by exactly one rank"
    scale = max(np.abs(ref_grad).max(), 1e-12)
    for r in res:
        assert bool(r["same"]) and bool(r["uid_same"]) and int(r["uid_len"]) == 128
        assert np.abs(r["grad"] - ref_grad).max() <= 1e-12 * scale
        assert r["loss"][0] == pytest.approx(ref_loss, rel=1e-13)
        np.testing.assert_array_equal(r["pose"], ref_pose)    # one owner per row: exact
    assert ref_loss > 0 and scale > 1e-8
