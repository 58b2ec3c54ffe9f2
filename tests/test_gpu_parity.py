"""GPU parity: the sm_100a path (libgsf_cuda.so through the C-ABI) against the CPU oracle.

Bar (SPEC.md acceptance 1 sets 1e-3 relative for single-precision gradients):
  * bit-exact vs the fp32 mirror (oracle/mirror.cpp): visible flags, global depth order, tile
    ranges, tile lists, per-pixel contributor counts, dominant / median ids and the fp32 maps;
  * vs the fp64 restatement (oracle/gsf_oracle.cpp): maps within 1e-4 (abs, values are O(1)),
    integer outputs identical, gradients within |g - g_ref| <= 1e-3 * max(|g_ref|, 1e-3 * max|g_ref|)
    (median error below 1e-5) and the pose 6-vector within 1e-4 relative of its largest component.
"""
import math

import numpy as np
import pytest

from paper_2403_16095_b200 import api
from paper_2403_16095_b200.abi import defaults_mapper, defaults_raster, defaults_tracker, defaults_weights
from helpers import (axis_primitive, f32_round, golden, make_intrinsics, one_pixel_camera, perturbed, pose,
                     rotation_error, scene, to_api_map, translation_error)

pytestmark = pytest.mark.gpu

MAP_TOL = 1e-4


def _upload(ctx, m):
    ctx.upload(to_api_map(m))


GRAD_TOL = 1e-3   # SPEC.md acceptance 1 (single precision)


def _grad_close(g, ref, rel=GRAD_TOL, name="", median=1e-5):
    g = np.asarray(g, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    if ref.size == 0 or np.abs(ref).max() == 0:
        assert np.abs(g).max() == 0, name
        return
    scale = np.maximum(np.abs(ref), 1e-3 * np.abs(ref).max())
    err = np.abs(g - ref) / scale
    assert err.max() <= rel, f"{name}: worst rel err {err.max():.3e} at {err.argmax()} ({g[err.argmax()]} vs {ref[err.argmax()]})"
    assert np.median(err[ref != 0]) <= median, f"{name}: median rel err {np.median(err):.3e}"


def _pose_close(g, ref, rel=1e-4):
    assert np.abs(np.asarray(g) - np.asarray(ref)).max() <= rel * np.abs(ref).max(), (g, ref)


def test_two_primitive_kat_on_gpu(gpu_ctx, orc):
    """test_rasterizer.cpp:39-63 through the CUDA path."""
    e = golden("reference_kats.json")["two_primitive_pixel"]["expect"]
    m = scene([axis_primitive(1.0, 0.6, [1, 0, 0]), axis_primitive(2.0, 0.8, [0, 1, 0])])
    _upload(gpu_ctx, m)
    r = gpu_ctx.render(pose(), one_pixel_camera(), np.array([[1.0]]))
    assert np.allclose(r.color[0, 0], e["color"], atol=1e-6)
    assert r.opacity[0, 0] == pytest.approx(e["opacity"], abs=1e-6)
    assert r.alpha_depth[0, 0] == pytest.approx(e["alpha_depth"], abs=1e-6)
    assert r.uncertainty[0, 0] == pytest.approx(e["uncertainty"], abs=1e-6)
    assert r.final_transmittance[0, 0] == pytest.approx(e["final_transmittance"], abs=1e-7)
    assert r.median_valid[0, 0] == 1 and r.median_depth[0, 0] == pytest.approx(1.0)
    assert r.per_pixel_count[0, 0] == 2 and r.dominant[0, 0] == 0 and r.median_prim[0, 0] == 0
    rs, prim, alpha, tr = gpu_ctx.render_record_full(1)
    assert list(prim) == [0, 1] and tr[1] == pytest.approx(0.4, abs=1e-7)


def test_empty_and_errors(gpu_ctx, orc):
    """test_rasterizer.cpp:65-99 + the EUNSUPPORTED path for non-16 tiles."""
    _upload(gpu_ctx, scene([]))
    r = gpu_ctx.render(pose(), make_intrinsics(16, 12, 20.0))
    assert (r.opacity == 0).all() and (r.per_pixel_count == 0).all() and (r.final_transmittance == 1).all()
    m = orc.random_scene(3, 5)
    m.mean[3, 1] = float("nan")
    _upload(gpu_ctx, m)
    with pytest.raises(ValueError) as ei:
        gpu_ctx.render(pose(), make_intrinsics(8, 8, 10.0))
    assert "primitive 3 has non-finite" in str(ei.value) and ei.value.index == 3
    _upload(gpu_ctx, orc.random_scene(4, 3))
    with pytest.raises(ValueError):
        gpu_ctx.render(pose(), make_intrinsics(8, 8, 10.0), np.ones((4, 4)))
    cfg = defaults_raster()
    cfg.tile_size = 8
    with pytest.raises(NotImplementedError):
        gpu_ctx.render(pose(), make_intrinsics(8, 8, 10.0), cfg=cfg)


def _scene_cases(orc):
    rng = np.random.default_rng(5)
    for seed in range(12):
        m = f32_round(orc.random_scene(100 + seed, 200, 4 if seed % 3 == 0 else 1))
        K = make_intrinsics(64, 64, 60.0) if seed % 2 == 0 else make_intrinsics(50, 34, 40.0)
        obs = orc.wavy_depth(K.width, K.height, 2.5).astype(np.float32)
        p = pose(0.03 * rng.standard_normal(3), 0.05 * rng.standard_normal(3))
        yield seed, m, K, obs, p


def test_forward_bit_exact_vs_mirror(gpu_ctx, orc):
    """Keys/order/ranges/lists/counts/ids and fp32 maps identical to the fp32 mirror."""
    for seed, m, K, obs, p in _scene_cases(orc):
        _upload(gpu_ctx, m)
        r = gpu_ctx.render(p, K, obs)
        mr = orc.mirror_render(m, p, K, obs)
        assert r.num_visible == mr.num_visible and r.num_pairs == mr.num_pairs, seed
        assert (r.visible == mr.visible).all()
        ntiles = ((K.width + 15) // 16) * ((K.height + 15) // 16)
        tr, pp = gpu_ctx.render_tiles(ntiles, r.num_pairs)
        assert r.num_visible == len(mr.rank_to_id), seed
        assert (tr.ravel() == mr.tile_range).all(), seed
        assert (pp == mr.rank_to_id[mr.pair_rank]).all(), seed
        for k in ("per_pixel_count", "dominant", "median_prim", "median_valid"):
            assert (getattr(r, k) == getattr(mr, k)).all(), (seed, k)
        for k in ("color", "alpha_depth", "median_depth", "opacity", "uncertainty", "final_transmittance",
                  "dominant_weight"):
            assert np.array_equal(getattr(r, k), getattr(mr, k)), (seed, k)


@pytest.mark.parametrize("count", [700, 1500, 5000])
def test_long_tile_lists_bit_exact(gpu_ctx, orc, count):
    """Tile lists longer than one shared-memory chunk (chunk sort + merge passes) and exact
    fp64 depth ties (broken by id, rasterizer.cpp:74-77) match the mirror's std::sort order."""
    m = orc.random_scene(7 + count, count)
    rng = np.random.default_rng(count)
    m.mean[:, :2] = rng.uniform(-0.15, 0.15, (count, 2))
    m.mean[:, 2] = np.round(rng.uniform(1.5, 3.0, count), 2)   # many identical depths
    m = f32_round(m)
    K = make_intrinsics(32, 32, 30.0)
    _upload(gpu_ctx, m)
    r = gpu_ctx.render(pose(), K)
    mr = orc.mirror_render(m, pose(), K)
    tr, pp = gpu_ctx.render_tiles(4, r.num_pairs)
    assert (tr[:, 1] - tr[:, 0]).max() > count // 2
    assert (tr.ravel() == mr.tile_range).all()
    assert (pp == mr.rank_to_id[mr.pair_rank]).all()
    for k in ("per_pixel_count", "dominant", "median_prim"):
        assert (getattr(r, k) == getattr(mr, k)).all(), k
    assert np.array_equal(r.color, mr.color)


def test_forward_vs_fp64_oracle(gpu_ctx, orc):
    """Maps within 1e-4 of the fp64 reference restatement; integer outputs identical."""
    for seed, m, K, obs, p in _scene_cases(orc):
        _upload(gpu_ctx, m)
        r = gpu_ctx.render(p, K, obs)
        o = orc.render(m, p, K, obs.astype(np.float64))
        assert (r.visible == o.visible).all(), seed
        for k in ("per_pixel_count", "dominant", "median_prim", "median_valid"):
            mism = int((getattr(r, k) != getattr(o, k)).sum())
            assert mism == 0, (seed, k, mism)
        for k in ("color", "alpha_depth", "opacity", "uncertainty", "final_transmittance"):
            assert np.abs(getattr(r, k) - getattr(o, k)).max() < MAP_TOL, (seed, k)
        md = np.where(o.median_valid == 1, r.median_depth - o.median_depth, 0)
        assert np.abs(md).max() < MAP_TOL


def test_record_matches_oracle(gpu_ctx, orc):
    """BlendRecord CSR (rasterizer.cpp:240-259) from the device equals the oracle's."""
    seed, m, K, obs, p = next(iter(_scene_cases(orc)))
    _upload(gpu_ctx, m)
    gpu_ctx.render(p, K, obs)
    rs, prim, alpha, tr = gpu_ctx.render_record_full(K.width * K.height)
    o = orc.render(m, p, K, obs.astype(np.float64))
    ors, oprim, oalpha, otr = o.record()
    assert (rs == ors).all() and (prim == oprim).all()
    assert np.abs(alpha - oalpha).max() < 1e-5 and np.abs(tr - otr).max() < 1e-5


def _probe(rng, w, h, with_unc):
    return (rng.standard_normal((h, w, 3)), rng.standard_normal((h, w)), rng.standard_normal((h, w)),
            rng.standard_normal((h, w)) if with_unc else None, rng.standard_normal((h, w)))


@pytest.mark.parametrize("sh", [1, 4, 16])
def test_backward_vs_fp64_oracle(gpu_ctx, orc, sh):
    """render_backward (rasterizer.cpp:339-572) with linear-probe upstream maps."""
    rng = np.random.default_rng(sh)
    for seed in range(4):
        m = f32_round(orc.random_scene(2000 + seed, 150, sh))
        K = make_intrinsics(48, 40, 45.0)
        obs = orc.wavy_depth(48, 40, 2.5).astype(np.float32)
        p = pose(0.02 * rng.standard_normal(3), 0.03 * rng.standard_normal(3))
        a_c, a_d, a_o, a_u, a_m = [None if a is None else a.astype(np.float32).astype(np.float64)
                                   for a in _probe(rng, 48, 40, True)]
        _upload(gpu_ctx, m)
        gpu_ctx.render(p, K, obs)
        g = gpu_ctx.render_backward(a_c, a_d, a_m, a_o, a_u, obs)
        o = orc.render(m, p, K, obs.astype(np.float64))
        go = orc.render_backward(m, p, K, o, a_c, a_d, a_m, a_o, a_u, obs.astype(np.float64))
        for k in ("d_mean", "d_log_scale", "d_quat", "d_opacity_logit", "d_sh", "d_mean2d"):
            _grad_close(getattr(g, k), getattr(go, k), name=f"{k} seed {seed}")
        _pose_close(g.d_pose, go.d_pose)


def test_large_footprints_forward_and_backward(gpu_ctx, orc):
    """Primitives covering hundreds of tiles: the one-CTA-per-primitive scatter (> 128 tiles) and
    the warp-cooperative gather of the chain (> 64 tiles) against the mirror / fp64 oracle."""
    rng = np.random.default_rng(77)
    m = orc.random_scene(77, 60)
    m.log_scale[:4] = np.log([0.6, 0.45, 0.8, 0.5])[:, None] + 0.1 * rng.standard_normal((4, 3))
    m.mean[:4] = [[0.1, 0.0, 2.2], [-0.2, 0.1, 2.6], [0.0, -0.1, 3.0], [0.3, 0.2, 2.4]]
    m = f32_round(m)
    K = make_intrinsics(320, 240, 200.0)
    obs = orc.wavy_depth(320, 240, 2.5).astype(np.float32)
    p = pose(0.01 * rng.standard_normal(3), 0.02 * rng.standard_normal(3))
    _upload(gpu_ctx, m)
    r = gpu_ctx.render(p, K, obs)
    mr = orc.mirror_render(m, p, K, obs)
    ntiles = 20 * 15
    tr, pp = gpu_ctx.render_tiles(ntiles, r.num_pairs)
    spans = (tr[:, 1] - tr[:, 0])
    assert (spans > 0).sum() > 200
    assert (tr.ravel() == mr.tile_range).all() and (pp == mr.rank_to_id[mr.pair_rank]).all()
    for k in ("per_pixel_count", "dominant", "median_prim"):
        assert (getattr(r, k) == getattr(mr, k)).all(), k
    assert np.array_equal(r.color, mr.color)
    a_c, a_d, a_o, a_u, a_m = [None if a is None else a.astype(np.float32).astype(np.float64)
                               for a in _probe(rng, 320, 240, True)]
    g = gpu_ctx.render_backward(a_c, a_d, a_m, a_o, a_u, obs)
    o = orc.render(m, p, K, obs.astype(np.float64))
    go = orc.render_backward(m, p, K, o, a_c, a_d, a_m, a_o, a_u, obs.astype(np.float64))
    for k in ("d_mean", "d_log_scale", "d_quat", "d_opacity_logit", "d_sh", "d_mean2d"):
        _grad_close(getattr(g, k), getattr(go, k), name=k)
    _pose_close(g.d_pose, go.d_pose)


def test_backward_zero_upstream(gpu_ctx, orc):
    _upload(gpu_ctx, f32_round(orc.random_scene(7, 10)))
    gpu_ctx.render(pose(), make_intrinsics(16, 16, 15.0))
    g = gpu_ctx.render_backward()
    assert (g.d_pose == 0).all() and (g.d_mean == 0).all() and (g.d_quat == 0).all()


def test_backward_deterministic(gpu_ctx, orc):
    """test_gradients.cpp:181-206: bit-identical repeats (no float atomics on the device path)."""
    m = f32_round(orc.random_scene(11, 80))
    K = make_intrinsics(40, 28, 35.0)
    obs = orc.wavy_depth(40, 28, 2.5).astype(np.float32)
    rng = np.random.default_rng(12)
    probe = _probe(rng, 40, 28, True)
    _upload(gpu_ctx, m)
    gpu_ctx.render(pose(), K, obs)
    a = gpu_ctx.render_backward(*probe[:2], probe[4], probe[2], probe[3], obs)
    gpu_ctx.render(pose(), K, obs)
    b = gpu_ctx.render_backward(*probe[:2], probe[4], probe[2], probe[3], obs)
    assert np.array_equal(a.d_pose, b.d_pose) and np.array_equal(a.d_mean, b.d_mean)
    assert np.array_equal(a.d_quat, b.d_quat) and np.array_equal(a.d_opacity_logit, b.d_opacity_logit)


def test_symmetric_scene_zero_lateral_pose_gradient(gpu_ctx, orc):
    """test_gradients.cpp:164-179"""
    m = scene([dict(mean=[0, 0, 2.0], scale=0.08, opacity=0.7, sh=[[0.3, 0.1, -0.2]])])
    _upload(gpu_ctx, f32_round(m))
    gpu_ctx.render(pose(), make_intrinsics(33, 33, 30.0))
    g = gpu_ctx.render_backward(d_opacity=np.ones((33, 33)))
    assert abs(g.d_pose[3]) < 1e-8 and abs(g.d_pose[4]) < 1e-8


def test_tracking_loss_vs_oracle(gpu_ctx, orc):
    """evaluate_tracking_loss (losses.cpp:284-339)"""
    m = f32_round(orc.random_scene(41, 60))
    K = make_intrinsics(48, 36, 40.0)
    rng = np.random.default_rng(3)
    target = rng.random((36, 48, 3)).astype(np.float32)
    depth = orc.wavy_depth(48, 36, 2.5).astype(np.float32)
    _upload(gpu_ctx, m)
    gpu_ctx.render(pose(), K)
    out, dc, dd = gpu_ctx.evaluate_tracking_loss(target, depth, defaults_weights(True))
    o = orc.render(m, pose(), K)
    oo, odc, odd = orc.tracking_loss(o, target.astype(np.float64), depth.astype(np.float64), K, defaults_weights(True))
    assert out.valid_color == oo.valid_color and out.valid_geo == oo.valid_geo
    assert out.total == pytest.approx(oo.total, rel=1e-5)
    assert np.abs(dc - odc).max() < 1e-7 and np.abs(dd - odd).max() < 1e-7


@pytest.mark.parametrize("sh", [1, 4])
def test_tracking_pose_gradient_vs_oracle(gpu_ctx, orc, sh):
    """The fused tracking backward (per-primitive SE(3) Jacobians, lane-level pose accumulation)
    against render -> evaluate_tracking_loss -> render_backward of the fp64 oracle."""
    rng = np.random.default_rng(40 + sh)
    for seed in range(4):
        m = f32_round(orc.random_scene(3000 + seed, 200, sh))
        K = make_intrinsics(64, 48, 55.0)
        _upload(gpu_ctx, m)
        gt = gpu_ctx.render(pose(), K)
        gpu_ctx.frame_upload(0, gt.color, gt.alpha_depth, 64, 48)
        p = perturbed(pose(), 0.01 * rng.standard_normal(6))
        w = defaults_weights(True)
        terms, g = gpu_ctx.tracking_gradient(0, p, K, w)
        o = orc.render(m, p, K)
        ot, odc, odd = orc.tracking_loss(o, gt.color.astype(np.float64), gt.alpha_depth.astype(np.float64), K, w)
        go = orc.render_backward(m, p, K, o, d_color=odc.reshape(48, 64, 3), d_alpha_depth=odd.reshape(48, 64))
        assert terms.total == pytest.approx(ot.total, rel=1e-5)
        _pose_close(g, go.d_pose)


def test_tracking_forward_maps_equal_plain_render(gpu_ctx, orc):
    """The tracking loop's forward (two pixels per lane, packed FP32x2, fused loss) computes the
    colour, alpha depth and opacity maps with the plain render's arithmetic: the tracking loss and its
    adjoint maps evaluated on either agree (bit for bit outside the render API's fix-up pixels)."""
    rng = np.random.default_rng(77)
    for seed, (P, w_, h_, f) in enumerate([(150, 64, 48, 55.0), (2500, 150, 110, 120.0), (6000, 97, 61, 70.0)]):
        m = f32_round(orc.random_scene(5000 + seed, P, 1, 0.95, 0.01, 0.3))
        K = make_intrinsics(w_, h_, f)
        _upload(gpu_ctx, m)
        gt = gpu_ctx.render(pose(), K)
        depth = gt.alpha_depth.copy()
        depth.ravel()[::7] = 0.0
        gpu_ctx.frame_upload(0, gt.color, depth, w_, h_)
        p = perturbed(pose(), 0.02 * rng.standard_normal(6))
        w = defaults_weights(True)
        terms, _ = gpu_ctx.tracking_gradient(0, p, K, w)
        a, dca, dda = gpu_ctx.evaluate_tracking_loss(gt.color, depth, w)
        gpu_ctx.render(p, K)
        b, dcb, ddb = gpu_ctx.evaluate_tracking_loss(gt.color, depth, w)
        # the plain render additionally re-blends in fp64 the few pixels whose termination / median /
        # dominant decision sits within fp32 error of its threshold (exact-decision fix-up, render API
        # only); everywhere else the maps, and so the loss's seed maps, are bit-identical
        assert (a.valid_color, a.valid_geo) == (b.valid_color, b.valid_geo)
        assert a.total == pytest.approx(b.total, rel=1e-6) and a.color == pytest.approx(b.color, rel=1e-6)
        assert (dca != dcb).sum() <= 1e-3 * dca.size and (dda != ddb).sum() <= 1e-3 * dda.size
        assert terms.total == pytest.approx(a.total, rel=1e-12) and terms.valid_color == a.valid_color


def test_mapping_loss_kat_on_gpu(gpu_ctx, orc):
    """test_losses.cpp:169-198 through the CUDA path."""
    e = golden("reference_kats.json")["mapping_loss_single_pixel"]["expect"]
    m = scene([axis_primitive(1.0, 0.6, [1, 0, 0]), axis_primitive(2.0, 0.8, [0, 1, 0])])
    _upload(gpu_ctx, m)
    obs = np.array([[1.0]], np.float32)
    r = gpu_ctx.render(pose(), one_pixel_camera(), obs)
    out, (dc, dad, dmd, du, dls) = gpu_ctx.evaluate_mapping_loss(r.color, obs, defaults_weights())
    assert out.geo == pytest.approx(e["geo"], abs=1e-6) and out.align == pytest.approx(e["align"], abs=1e-6)
    assert out.var == pytest.approx(e["var"], abs=1e-6) and out.total == pytest.approx(e["total"], abs=1e-6)
    assert dad[0] == pytest.approx(e["d_alpha_depth"], abs=1e-6) and dmd[0] == pytest.approx(e["d_median_depth"], abs=1e-6)
    assert du[0] == pytest.approx(e["d_uncertainty"], abs=1e-6)


def test_mapping_loss_vs_oracle(gpu_ctx, orc):
    """evaluate_mapping_loss (losses.cpp:156-282) incl. SSIM and iso on a random scene."""
    m = f32_round(orc.random_scene(37, 80))
    K = make_intrinsics(48, 36, 40.0)
    rng = np.random.default_rng(4)
    target = rng.random((36, 48, 3)).astype(np.float32)
    depth = orc.wavy_depth(48, 36, 2.5).astype(np.float32)
    _upload(gpu_ctx, m)
    gpu_ctx.render(pose(), K, depth)
    out, (dc, dad, dmd, du, dls) = gpu_ctx.evaluate_mapping_loss(target, depth, defaults_weights())
    o = orc.render(m, pose(), K, depth.astype(np.float64))
    oo, (odc, odad, odmd, odu, odls) = orc.mapping_loss(m, o, target.astype(np.float64), depth.astype(np.float64), K,
                                                        defaults_weights())
    for k in ("color", "ssim", "geo", "align", "iso", "var", "total"):
        assert getattr(out, k) == pytest.approx(getattr(oo, k), rel=1e-4, abs=1e-7), k
    assert np.abs(dc - odc).max() < 1e-4 * np.abs(odc).max() + 1e-9
    assert np.abs(dad - odad).max() < 1e-7 and np.abs(dmd - odmd).max() < 1e-7 and np.abs(du - odu).max() < 1e-7
    _grad_close(dls, odls, name="iso direct")


def test_ssim_vs_oracle(gpu_ctx, orc):
    rng = np.random.default_rng(21)
    for (w, h) in ((40, 30), (7, 5)):
        x = rng.random((h, w, 3)).astype(np.float32)
        y = rng.random((h, w, 3)).astype(np.float32)
        v, g = gpu_ctx.ssim(x, y, w, h, want_gradient=True)
        ov, og = orc.ssim(x.astype(np.float64), y.astype(np.float64), w, h, gradient=True)
        assert v == pytest.approx(ov, abs=1e-6)
        assert np.abs(g - og).max() < 1e-4 * np.abs(og).max()


def _frames(ctx, orc, m, poses, K):
    out = []
    for i, p in enumerate(poses):
        r = ctx.render(p, K)
        out.append((r.color.copy(), r.alpha_depth.copy()))
        ctx.frame_upload(i, r.color, r.alpha_depth, K.width, K.height)
    return out


def test_tracking_stationary_recovers_repeatable(gpu_ctx, orc):
    """test_tracker.cpp:192-244 on the device loop, and the oracle's trajectory as a reference."""
    K = make_intrinsics(48, 36, 40.0)
    m = f32_round(orc.random_scene(7, 60))
    _upload(gpu_ctx, m)
    _frames(gpu_ctx, orc, m, [pose()], K)
    tc = defaults_tracker()
    tc.iterations = 10
    res = gpu_ctx.track_frame(0, pose(), K, tc, defaults_weights(True))
    assert np.linalg.norm(list(res.pose.rotation_tangent)) <= 1e-15 and res.final_loss == 0.0
    assert not res.degraded and res.iterations_run == 10

    K = make_intrinsics(64, 48, 55.0)
    m = f32_round(orc.random_scene(19, 80))
    _upload(gpu_ctx, m)
    fr = _frames(gpu_ctx, orc, m, [pose()], K)
    start = perturbed(pose(), [0.004, -0.003, 0.002, 0.008, -0.006, 0.004])
    tc.iterations = 40
    res = gpu_ctx.track_frame(0, start, K, tc, defaults_weights(True))
    assert rotation_error(res.pose, pose()) < 0.35 * rotation_error(start, pose())
    assert translation_error(res.pose, pose()) < 0.35 * translation_error(start, pose())
    again = gpu_ctx.track_frame(0, start, K, tc, defaults_weights(True))
    assert list(again.pose.translation) == list(res.pose.translation) and again.final_loss == res.final_loss
    ores = orc.track_frame(m, fr[0][0], fr[0][1], start, K, tc, defaults_weights(True), defaults_raster())
    # 40 Adam steps amplify fp32-vs-fp64 gradient noise; both recover GT (above) and agree to 5e-4
    assert rotation_error(res.pose, ores.pose) < 5e-4 and translation_error(res.pose, ores.pose) < 5e-4


def test_tracking_100_iterations_cfg1_sized(gpu_ctx, orc):
    """track_frame(100) on a cfg1-sized frame (640x480, f=525) against the fp64 oracle's
    trajectory from the same start (tracker.cpp:30-84, 100 Adam steps on fp32 vs fp64 gradients)."""
    K = make_intrinsics(640, 480, 525.0)
    m = f32_round(orc.random_scene(4242, 3000, 1, 0.95, 0.01, 0.08))
    _upload(gpu_ctx, m)
    fr = _frames(gpu_ctx, orc, m, [pose()], K)
    start = perturbed(pose(), [0.004, -0.003, 0.002, 0.008, -0.006, 0.004])   # test_tracker.cpp:222
    tc = defaults_tracker()
    tc.iterations = 100
    w = defaults_weights()
    res = gpu_ctx.track_frame(0, start, K, tc, w)
    ores = orc.track_frame(m, fr[0][0], fr[0][1], start, K, tc, w, defaults_raster())
    assert res.iterations_run == 100 and not res.degraded
    assert rotation_error(res.pose, pose()) < 0.35 * rotation_error(start, pose())
    assert translation_error(res.pose, pose()) < 0.35 * translation_error(start, pose())
    # near the optimum Adam steps of ~lr (1.5e-3 rad, 2.2e-3 m) flip with the gradient signs, so fp32-vs-fp64
    # gradient noise moves the end point by a fraction of a step: 1/3 of lr (SURVEY 8(c) fallback criterion)
    assert rotation_error(res.pose, ores.pose) < 5e-4 and translation_error(res.pose, ores.pose) < 7e-4
    # the final loss is the tracking loss of one more render at the end point (tracker.cpp:74-76); near the
    # optimum it changes by tens of percent inside that 5e-4 ball, so it is checked against the oracle's
    # loss at the GPU's own end point (render without observed depth, tracker.cpp:43)
    ofin, _, _ = orc.tracking_loss(orc.render(m, res.pose, K), fr[0][0], fr[0][1], K, w)
    print("final loss", res.final_loss, "oracle at the same pose", ofin.total, "oracle trajectory", ores.final_loss)
    assert res.final_loss == pytest.approx(ofin.total, rel=1e-4, abs=1e-9)


@pytest.mark.parametrize("K_sh", [4, 9, 16])
def test_tracking_view_dependent_sh(gpu_ctx, orc, K_sh):
    """track_frame on a view-dependent map (SH 4/9/16): the loop takes the k_backward_pose<SEED_TRACK,
    true> path, whose seeds come from the forward's maps; the trajectory follows the fp64 oracle's."""
    K = make_intrinsics(64, 48, 55.0)
    m = f32_round(orc.random_scene(77 + K_sh, 120, K_sh))
    _upload(gpu_ctx, m)
    fr = _frames(gpu_ctx, orc, m, [pose()], K)
    start = perturbed(pose(), [0.004, -0.003, 0.002, 0.008, -0.006, 0.004])
    tc = defaults_tracker()
    tc.iterations = 30
    w = defaults_weights(True)
    res = gpu_ctx.track_frame(0, start, K, tc, w)
    ores = orc.track_frame(m, fr[0][0], fr[0][1], start, K, tc, w, defaults_raster())
    assert res.iterations_run == 30
    assert rotation_error(res.pose, ores.pose) < 5e-4 and translation_error(res.pose, ores.pose) < 5e-4
    # the first step alone: the gradient the loop used equals the standalone tracking gradient
    tc.iterations = 1
    one = gpu_ctx.track_frame(0, start, K, tc, w)
    o1 = orc.track_frame(m, fr[0][0], fr[0][1], start, K, tc, w, defaults_raster())
    assert rotation_error(one.pose, o1.pose) < 1e-6 and translation_error(one.pose, o1.pose) < 1e-6


def test_tracking_leaves_trust_region(gpu_ctx, orc):
    """The tracking loop preprocesses only the frame's trust-region candidates (k_candidates) until a
    step leaves the region (0.03 rad / 0.05 m), then every primitive.  A narrow camera on a scene
    that extends past the image and a start 9 cm off: the pose travels beyond the region, and the
    trajectory still follows the fp64 oracle's (which always projects everything)."""
    K = make_intrinsics(64, 48, 90.0)
    m = f32_round(orc.random_scene(901, 400))
    _upload(gpu_ctx, m)
    fr = _frames(gpu_ctx, orc, m, [pose()], K)
    start = perturbed(pose(), [0.01, -0.008, 0.006, 0.07, -0.05, 0.03])
    tc = defaults_tracker()
    tc.iterations = 60
    res = gpu_ctx.track_frame(0, start, K, tc, defaults_weights(True))
    assert translation_error(res.pose, start) > 0.05          # the region was left mid-loop
    assert translation_error(res.pose, pose()) < 0.5 * translation_error(start, pose())
    again = gpu_ctx.track_frame(0, start, K, tc, defaults_weights(True))
    assert list(again.pose.translation) == list(res.pose.translation)
    ores = orc.track_frame(m, fr[0][0], fr[0][1], start, K, tc, defaults_weights(True), defaults_raster())
    assert rotation_error(res.pose, ores.pose) < 2e-3 and translation_error(res.pose, ores.pose) < 2e-3


def test_tracking_empty_view_degraded(gpu_ctx, orc):
    """test_tracker.cpp:246-263"""
    _upload(gpu_ctx, f32_round(orc.random_scene(3, 30)))
    K = make_intrinsics(32, 24, 28.0)
    gpu_ctx.frame_upload(0, np.full((24, 32, 3), 0.5), orc.wavy_depth(32, 24, 2.0), 32, 24)
    away = pose((math.pi, 0, 0))
    res = gpu_ctx.track_frame(0, away, K, defaults_tracker(), defaults_weights(True))
    assert res.degraded and res.iterations_run == 0


def test_ba_noop_and_map_step(gpu_ctx, orc):
    """test_tracker.cpp:319-363 (BA exact no-op at the optimum) and test_map.cpp:391-423."""
    m = f32_round(orc.random_scene(31, 50))
    K = make_intrinsics(48, 36, 40.0)
    mc = defaults_mapper()
    mc.weights.w_ssim = mc.weights.w_align = mc.weights.w_iso = mc.weights.w_var = 0.0
    poses = [pose(), perturbed(pose(), [0.02, -0.01, 0.03, 0.05, 0.02, -0.04]),
             perturbed(pose(), [-0.03, 0.02, -0.01, -0.04, 0.03, 0.05])]
    _upload(gpu_ctx, m)
    _frames(gpu_ctx, orc, m, poses, K)
    trace, out_poses = gpu_ctx.sliding_ba([0, 1, 2], poses, [0, 10, 20], K, defaults_tracker(), mc, 5)
    assert (trace == 0).all()
    m2 = gpu_ctx.download()
    assert np.array_equal(m2.mean, m.mean) and np.array_equal(m2.opacity_logit, m.opacity_logit)

    K = make_intrinsics(48, 36, 40.0)
    truth = f32_round(orc.random_scene(83, 40, 1, 0.95, 0.05, 0.2))
    _upload(gpu_ctx, truth)
    gt = gpu_ctx.render(pose(), K)
    obs = np.where(gt.opacity > 0.5, gt.alpha_depth, 0.0).astype(np.float32)
    gpu_ctx.frame_upload(0, gt.color, obs, 48, 36)
    rng = np.random.default_rng(83)
    pert = f32_round(truth)
    pert.mean = (pert.mean + 0.02 * rng.standard_normal(pert.mean.shape)).astype(np.float32).astype(np.float64)
    pert.sh[:, 0] = (pert.sh[:, 0] + 0.15 * rng.standard_normal((40, 3))).astype(np.float32).astype(np.float64)
    mc = defaults_mapper()
    mc.densify_interval = 0
    _upload(gpu_ctx, pert)
    trace = gpu_ctx.map_step([0], [pose()], K, mc, 60)
    assert trace[-1] < 0.7 * trace[0]
    st = orc.MapState(pert, mc)
    otrace = st.map_step([(gt.color.astype(np.float64), obs.astype(np.float64))], [pose()], K, mc, 60)
    assert trace[0] == pytest.approx(otrace[0], rel=1e-4)
    assert trace[-1] == pytest.approx(otrace[-1], rel=2e-2)


def test_uncertainty_kats_on_gpu(gpu_ctx, orc):
    """test_map.cpp:118-155, 189-211 through the device uncertainty pass."""
    K = one_pixel_camera()
    m = scene([dict(mean=[0, 0, 1.5], scale=0.05, opacity=0.9, color=[0.5, 0.5, 0.5])])
    _upload(gpu_ctx, m)
    gpu_ctx.frame_upload(0, np.zeros(3), np.array([2.0]), 1, 1)
    assert gpu_ctx.accumulate_uncertainty([0], [pose()], K) == 1
    d = gpu_ctx.download()
    assert d.uncertainty[0] == pytest.approx(0.225, rel=1e-6) and d.observed[0] == 1
    assert gpu_ctx.prune_unreliable() == 1
    d = gpu_ctx.download()
    assert 1 / (1 + math.exp(-d.opacity_logit[0])) == pytest.approx(0.005, rel=1e-5)
    assert gpu_ctx.prune_unreliable() == 0


def _frame_of(orc, m, p, K, hole_every=13):
    r = orc.render(m, p, K)
    depth = np.where(r.opacity > 0.3, r.alpha_depth, 0.0).astype(np.float32)
    depth.ravel()[::hole_every] = 0.0
    return r.color.astype(np.float32), depth


def test_initialize_map_matches_oracle(gpu_ctx, orc):
    """initialize_map (mapper.cpp:125-148) on the device vs the fp64 restatement, same frame."""
    m = orc.random_scene(321, 120)
    K = make_intrinsics(64, 48, 50.0)
    p = pose([0.02, -0.01, 0.03], [0.05, -0.02, 0.1])
    rgb, depth = _frame_of(orc, m, p, K)
    gpu_ctx.frame_upload(0, rgb, depth, 64, 48)
    mc = defaults_mapper()
    for stride in (1, 2, 3):
        mc.init_stride = stride
        n = gpu_ctx.initialize_map(0, p, K, mc)
        ref = orc.backproject(rgb, depth, p, K, mc, stride)
        assert n == ref.mean.shape[0] > 0, stride
        g = gpu_ctx.download()
        assert np.abs(g.mean - ref.mean).max() < 2e-6
        assert np.abs(g.log_scale - ref.log_scale).max() < 2e-6
        assert (g.quat == [1, 0, 0, 0]).all() and np.allclose(g.opacity_logit, ref.opacity_logit, atol=1e-7)
        assert np.abs(g.sh - ref.sh.reshape(g.sh.shape)).max() < 2e-6
    with pytest.raises(RuntimeError, match="no usable depth"):
        gpu_ctx.frame_upload(1, rgb, np.zeros_like(depth), 64, 48)
        gpu_ctx.initialize_map(1, p, K, mc)


def test_spawn_gaussians_matches_oracle(gpu_ctx, orc):
    """spawn_gaussians (mapper.cpp:150-170): thin pixels of the current render get new primitives;
    the existing map is untouched and the new ones follow in row-major pixel order."""
    truth = orc.random_scene(654, 150)
    K = make_intrinsics(64, 48, 50.0)
    p0, p1 = pose(), pose([0.0, 0.15, 0.0], [0.2, 0.0, 0.0])
    rgb0, d0 = _frame_of(orc, truth, p0, K)
    rgb1, d1 = _frame_of(orc, truth, p1, K)
    gpu_ctx.frame_upload(0, rgb0, d0, 64, 48)
    gpu_ctx.frame_upload(1, rgb1, d1, 64, 48)
    mc = defaults_mapper()
    mc.init_stride = 4
    n0 = gpu_ctx.initialize_map(0, p0, K, mc)
    before = gpu_ctx.download()
    r = gpu_ctx.render(p1, K)
    spawned = gpu_ctx.spawn_gaussians(1, p1, K, mc)
    ref = orc.backproject(rgb1, d1, p1, K, mc, mc.spawn_stride, opacity=r.opacity.astype(np.float64))
    assert spawned == ref.mean.shape[0] > 0
    after = gpu_ctx.download()
    assert after.mean.shape[0] == n0 + spawned
    assert np.array_equal(after.mean[:n0], before.mean[:n0]) and np.array_equal(after.sh[:n0], before.sh[:n0])
    assert np.abs(after.mean[n0:] - ref.mean).max() < 2e-6
    assert np.abs(after.sh[n0:] - ref.sh.reshape(after.sh[n0:].shape)).max() < 2e-6
    # the grown map renders and steps
    mc.densify_interval = 0
    gpu_ctx.render(p1, K)
    gpu_ctx.map_step([1], [p1], K, mc, 3)


def _plane_scene(specs):
    from helpers import logit
    return scene([dict(mean=[x, y, z], scale=sc, opacity=op, sh=[[0.0, 0.0, 0.0]]) for (x, y, z, sc, op) in specs])


def test_densify_kat_on_device(gpu_ctx, orc):
    """test_map.cpp:317-350 through gsf_densify_and_cull, and the split children equal the fp64
    restatement's (same mt19937_64 seed, one normal_distribution per split parent)."""
    mc = defaults_mapper()
    mc.scene_extent = 4.0
    mc.seed = 9
    specs = [(0, 0, 2, 0.10, 0.9), (1, 0, 2, 0.01, 0.9), (0, 1, 2, 0.02, 1e-4), (1, 1, 2, 0.02, 0.9)]
    m = f32_round(_plane_scene(specs))
    _upload(gpu_ctx, m)
    gpu_ctx.set_map_stats([1.0, 1.0, 0.0, 0.0], [1, 1, 0, 1])
    assert gpu_ctx.densify_and_cull(mc) == (1, 1, 1)
    g = gpu_ctx.download()
    assert g.mean.shape[0] == 5
    assert g.mean[0, 0] == pytest.approx(1.0) and g.mean[1, 1] == pytest.approx(1.0) and g.mean[4, 0] == pytest.approx(1.0)
    assert math.exp(g.log_scale[2, 0]) == pytest.approx(0.10 / 1.6, rel=1e-6)
    st = orc.MapState(m, mc)
    st.set_stats([1.0, 1.0, 0.0, 0.0], [1, 1, 0, 1])
    assert st.densify(mc) == (1, 1, 1)
    ref = st.get()
    assert np.abs(g.mean - ref.mean).max() < 1e-6 and np.abs(g.log_scale - ref.log_scale).max() < 1e-6
    a, c = gpu_ctx.map_stats()
    assert (a == 0).all() and (c == 0).all()
    assert gpu_ctx.densify_and_cull(mc) == (0, 0, 0) and gpu_ctx.download().mean.shape[0] == 5
    # a second split continues the same generator stream on both sides
    gpu_ctx.set_map_stats([1.0] * 5, [1] * 5)
    st.set_stats([1.0] * 5, [1] * 5)
    assert gpu_ctx.densify_and_cull(mc) == st.densify(mc)
    assert np.abs(gpu_ctx.download().mean - st.get().mean).max() < 1e-6


def test_map_step_with_densification(gpu_ctx, orc):
    """map_step runs densify_and_cull every `interval` iterations (mapper.cpp:278-279): the map
    is resized on the device, its statistics restart and the loop keeps optimising."""
    truth = orc.random_scene(83, 60, 1, 0.95, 0.05, 0.2)
    K = make_intrinsics(48, 36, 40.0)
    gt = orc.render(truth, pose(), K)
    obs = np.where(gt.opacity > 0.5, gt.alpha_depth, 0.0)
    m = f32_round(truth)
    m.opacity_logit[:5] = -8.0            # faded: culled at the first pass
    _upload(gpu_ctx, m)
    gpu_ctx.frame_upload(0, gt.color.astype(np.float32), obs.astype(np.float32), 48, 36)
    mc = defaults_mapper()
    mc.densify_interval = 4
    mc.densify_grad_threshold = 1e-9      # every primitive seen with any gradient strains
    trace = gpu_ctx.map_step([0], [pose()], K, mc, 9)
    assert np.isfinite(trace).all()
    P = gpu_ctx.download().mean.shape[0]
    assert P != 60 and P == gpu_ctx.P
    a, c = gpu_ctx.map_stats()
    assert a.shape[0] == P and (c <= 1).all()   # restarted at iteration 8, one pass since


def test_cabi_client_from_cpp():
    """The drop-in boundary from plain C++ (tools/cabi_client.cpp: include/gsf_cuda.h + the .so):
    upload, render, frame upload, track_frame, map_step and the CSR record in one process."""
    import json
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "cabi_client")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["final_loss"] < r["initial_loss"] and r["record_entries"] > 0 and r["kernel_launches"] > 0


def test_render_reference_matches_brute_force_oracle(gpu_ctx, orc):
    """render_reference (rasterizer.cpp:263-296) vs the oracle's brute-force render; and the tiled
    render stays within 1e-5 of it (test_rasterizer.cpp:119-134)."""
    m = f32_round(orc.random_scene(808, 150))
    K = make_intrinsics(48, 40, 45.0)
    obs = orc.wavy_depth(48, 40, 2.5).astype(np.float32)
    _upload(gpu_ctx, m)
    rr = gpu_ctx.render(pose(), K, obs, reference=True)
    o = orc.render(m, pose(), K, obs.astype(np.float64), brute_force=True)
    assert (rr.per_pixel_count == o.per_pixel_count).all()
    for k in ("color", "alpha_depth", "opacity", "uncertainty", "final_transmittance"):
        assert np.abs(getattr(rr, k) - getattr(o, k)).max() < MAP_TOL, k
    tiled = gpu_ctx.render(pose(), K, obs)
    assert np.abs(tiled.color - rr.color).max() < 1e-5


def test_checkpoint_roundtrip_and_format(gpu_ctx, orc, tmp_path):
    """GSFMAP01 (io/checkpoint.cpp): save -> load is exact for the fp32 device map, and the bytes
    follow the reference layout (parsed here independently)."""
    import struct
    m = f32_round(orc.random_scene(909, 40, 4))
    m.uncertainty = np.linspace(0, 0.1, 40)
    m.observed = (np.arange(40) % 3 == 0).astype(np.uint8)
    gpu_ctx.upload(to_api_map(m))
    K = make_intrinsics(32, 24, 30.0)
    path = str(tmp_path / "map.gsf")
    gpu_ctx.save_checkpoint(path, K)
    raw = open(path, "rb").read()
    assert raw[:8] == b"GSFMAP01"
    hdr = struct.unpack("<9d", raw[8:80])
    bands, count = struct.unpack("<IQ", raw[80:92])
    assert hdr[0] == K.fx and int(hdr[4]) == 32 and bands == 4 and count == 40
    rec = 8 * 3 + 8 * 3 + 8 * 4 + 8 + 8 + 1 + 8 * 3 * 4
    assert len(raw) == 92 + 40 * rec
    first = raw[92:92 + rec]
    mean0 = struct.unpack("<3d", first[:24])
    assert np.allclose(mean0, m.mean[0], atol=0) and first[24 * 2 + 32 + 16] == 1
    before = gpu_ctx.download()
    gpu_ctx.upload(to_api_map(f32_round(orc.random_scene(1, 3))))
    K2 = gpu_ctx.load_checkpoint(path)
    after = gpu_ctx.download()
    assert K2.width == 32 and K2.fx == K.fx and after.mean.shape[0] == 40
    for k in ("mean", "log_scale", "quat", "opacity_logit", "sh", "observed"):
        assert np.array_equal(getattr(after, k), getattr(before, k)), k
    assert np.allclose(after.uncertainty, before.uncertainty, atol=1e-8)
    bad = tmp_path / "bad.gsf"
    bad.write_bytes(b"NOTAMAP!" + raw[8:])
    with pytest.raises(RuntimeError, match="bad magic"):
        gpu_ctx.load_checkpoint(str(bad))


def _room_frames(ctx, n, K, orbit=1440):
    from tools import synth
    t = synth.room(30000, 4.0, 3, 0)
    ctx.upload(api.GaussianMap(t.mean, t.log_scale, t.quat, t.opacity_logit, t.sh))
    poses = [api.pose_of(r, tr) for r, tr in synth.orbit(orbit, 1.0, 0.0)]
    frames = []
    for f in range(n):
        r = ctx.render(poses[f], K)
        frames.append((r.color.copy(), np.where(r.opacity > 0.5, r.alpha_depth, 0.0).astype(np.float32)))
    return frames, poses


def _gt_relative(poses, n):
    """pose_n o pose_0^-1: the world frame of a SLAM run is its first camera (system.cpp:69)."""
    from scipy.spatial.transform import Rotation as R
    R0 = R.from_rotvec(list(poses[0].rotation_tangent)).as_matrix()
    Rn = R.from_rotvec(list(poses[n].rotation_tangent)).as_matrix()
    Rr = Rn @ R0.T
    return api.pose_of(R.from_matrix(Rr).as_rotvec(), np.array(list(poses[n].translation)) - Rr @ list(poses[0].translation))


def test_slam_matches_oracle_orchestration(gpu_ctx, orc):
    """SlamSystem::process (system.cpp:31-154) through gsf_slam_process vs the same sequence run by
    oracle/slam.py over the fp64 oracle (bootstrap, velocity-model tracking, keyframe cycles with
    map_step, sliding_ba, uncertainty pruning and spawning): same keyframes, same decisions, poses
    within fp32-vs-fp64 drift of ~100 chained Adam steps."""
    from paper_2403_16095_b200 import abi
    from oracle.slam import OracleSlam
    K = make_intrinsics(48, 36, 40.0, near=0.1, far=10.0)
    frames, _ = _room_frames(gpu_ctx, 7, K)

    def cfg():
        c = abi.defaults_slam(K)
        c.tracker.keyframe_interval = 3
        c.tracker.iterations = 20
        c.tracker.ba_iterations = 3
        c.map_iterations = 10
        c.init_iterations = 30
        c.mapper.densify_interval = 0
        c.seed = 5
        return c
    slam = api.SlamSystem(gpu_ctx, cfg())
    ref = OracleSlam(cfg())
    for f, (c, d) in enumerate(frames):
        log = slam.process(f, f / 30.0, c, d)
        p = ref.process(f, c, d)
        assert log.keyframe == (1 if f % 3 == 0 else 0)
        if f == 0:
            assert log.primitives == ref.primitives    # the bootstrap back-projection is exact
        else:
            assert abs(log.primitives - ref.primitives) <= max(2, ref.primitives // 100), f
        # fp32 vs fp64 over 15-20 chained Adam steps per frame: 1e-3 after the first tracked frame,
        # growing to a few mm after two keyframe cycles (both arms sit ~0.1 m from the ground truth
        # here: the alpha-depth geo term is biased while the young map is semi-transparent)
        tol = 1e-3 if f <= 1 else 1e-2
        assert translation_error(log.pose, p) < tol and rotation_error(log.pose, p) < tol / 2, f
    assert slam.keyframes == len(ref.keyframes) == 3
    slam.close()


def test_slam_pipeline_on_synthetic_sequence(gpu_ctx, orc):
    """SlamSystem end to end on a rendered orbit at the reference defaults (RunConfig, config.hpp:16-35):
    the bootstrap map reproduces the first frame, tracking follows the ground-truth relative motion
    over the first keyframe cycles, every stage reports its time."""
    from paper_2403_16095_b200 import abi
    K = make_intrinsics(96, 72, 80.0, near=0.1, far=10.0)
    frames, poses = _room_frames(gpu_ctx, 11, K)
    cfg = abi.defaults_slam(K)
    cfg.tracker.keyframe_interval = 5
    slam = api.SlamSystem(gpu_ctx, cfg)
    for f, (c, d) in enumerate(frames):
        log = slam.process(f, f / 30.0, c, d)
        assert log.frame == f and log.primitives == gpu_ctx.P > 0
    logs = slam.logs
    assert slam.keyframes == 3 and [l.keyframe for l in logs] == [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1]
    assert logs[0].kf_psnr_db > 30.0 and logs[0].kf_depth_l1_cm < 5.0
    assert all(np.isfinite(l.track_loss) and l.track_iterations == 15 for l in logs[1:])
    for k in (5, 10):
        assert logs[k].map_ms > 0 and logs[k].ba_ms > 0 and logs[k].uncertainty_ms > 0 and logs[k].spawn_ms > 0
        assert logs[k].kf_psnr_db > 28.0 and logs[k].kf_depth_l1_cm < 3.0
    assert logs[10].primitives > logs[5].primitives     # spawning filled the newly seen pixels
    for f in range(1, 11):
        gt = _gt_relative(poses, f)
        assert translation_error(logs[f].pose, gt) < 0.12 and rotation_error(logs[f].pose, gt) < 0.03, f
    with pytest.raises(ValueError):
        bad = abi.defaults_slam(K)
        bad.tracker.ba_window = 1                       # TrackerConfig::validate (tracker.cpp:12-24)
        api.SlamSystem(gpu_ctx, bad)
    slam.close()
