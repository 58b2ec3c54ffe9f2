"""Pins the fp64 restatement (oracle/gsf_oracle.cpp, "port") to the reference itself.

oracle/_ref/libgsfref.so is the UNMODIFIED reference (/root/reference/proj/src) compiled here
against oracle/eigen_lite (oracle/Makefile.ref).  Every entry point the GPU parity tests use as a
checker is run through both backends on identical inputs; they agree to the last few ulps (the only
differences are the summation order inside small fixed-size matrix products), so the GPU-vs-port
parity tests are GPU-vs-reference parity tests.  CPU only; skipped where the library was not built.
"""
import numpy as np
import pytest

from helpers import make_intrinsics, perturbed, pose

pytestmark = pytest.mark.skipif(not __import__("oracle").reference_available(),
                                reason="oracle/_ref/libgsfref.so not built (needs /root/reference)")

REL = 1e-11


def both(orc, fn):
    a = fn()
    with orc.backend("reference"):
        b = fn()
    return a, b


def close(a, b, rel=REL, name=""):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(np.abs(b).max() if b.size else 0.0, 1e-300)
    assert np.abs(a - b).max() <= rel * scale, f"{name}: {np.abs(a - b).max()} vs scale {scale}"


def fields(s):
    return {k: getattr(s, k) for k, _ in s._fields_}


def test_config_defaults_are_the_reference_structs(orc):
    """raster/config.hpp, losses.cpp:33-46, tracker.hpp:11-22, mapper.hpp:21-41 — the values the
    port and the product's abi defaults hard-code equal the reference structs' initialisers."""
    from paper_2403_16095_b200 import abi
    for f in ("defaults_raster", "defaults_tracker", "defaults_mapper"):
        a, b = both(orc, getattr(orc, f))
        prod = getattr(abi, f)()
        for k, v in fields(b).items():
            if k in ("raster", "weights"):
                assert bytes(getattr(a, k)) == bytes(v) == bytes(getattr(prod, k)), (f, k)
            else:
                assert getattr(a, k) == v == getattr(prod, k), (f, k)
    for hh in (False, True):
        a, b = both(orc, lambda: orc.defaults_weights(hh))
        assert bytes(a) == bytes(b) == bytes(abi.defaults_weights(hh))


def _cases(orc):
    rng = np.random.default_rng(11)
    for seed in range(8):
        sh = (1, 4, 9, 16)[seed % 4]
        m = orc.random_scene(300 + seed, 150, sh, 0.999 if seed % 2 else 0.95)
        K = make_intrinsics(48, 40, 45.0)
        obs = orc.wavy_depth(48, 40, 2.5)
        p = pose(0.03 * rng.standard_normal(3), 0.05 * rng.standard_normal(3))
        cfg = orc.defaults_raster()
        if seed == 3:
            cfg = orc.smooth_raster()
        if seed == 5:
            cfg.alpha_clamp, cfg.dilation, cfg.uncertainty_full_gradient = 0.9, 0.1, 0
        yield seed, m, K, obs, p, cfg


def test_render_and_record_match_reference(orc):
    """render (rasterizer.cpp:168-261) incl. the alpha clamp (opacities up to 0.999), the gradcheck
    smooth config and non-default clamp/dilation: maps, ids, counts and the BlendRecord CSR."""
    for seed, m, K, obs, p, cfg in _cases(orc):
        a, b = both(orc, lambda: orc.render(m, p, K, obs, cfg))
        for k in ("color", "alpha_depth", "median_depth", "opacity", "uncertainty", "final_transmittance",
                  "dominant_weight"):
            close(getattr(a, k), getattr(b, k), name=f"{seed} {k}")
        for k in ("per_pixel_count", "dominant", "median_prim", "median_valid", "visible"):
            assert (getattr(a, k) == getattr(b, k)).all(), (seed, k)
        ra, rb = a.record(), b.record()
        assert (ra[0] == rb[0]).all() and (ra[1] == rb[1]).all(), seed
        close(ra[2], rb[2], name="alpha")
        close(ra[3], rb[3], name="T")
        bf_a, bf_b = both(orc, lambda: orc.render(m, p, K, obs, cfg, brute_force=True))
        close(bf_a.color, bf_b.color, name="render_reference")


def test_backward_matches_reference(orc):
    """render_backward (rasterizer.cpp:339-572) with all five seed maps."""
    rng = np.random.default_rng(2)
    for seed, m, K, obs, p, cfg in _cases(orc):
        seeds = dict(d_color=rng.standard_normal((K.height, K.width, 3)), d_alpha_depth=rng.standard_normal((K.height, K.width)),
                     d_median_depth=rng.standard_normal((K.height, K.width)), d_opacity=rng.standard_normal((K.height, K.width)),
                     d_uncertainty=rng.standard_normal((K.height, K.width)))

        def run():
            r = orc.render(m, p, K, obs, cfg)
            return orc.render_backward(m, p, K, r, obs=obs, cfg=cfg, **seeds)
        a, b = both(orc, run)
        for k in ("d_mean", "d_log_scale", "d_quat", "d_opacity_logit", "d_sh", "d_mean2d", "d_pose"):
            close(getattr(a, k), getattr(b, k), rel=1e-10, name=f"{seed} {k}")


def test_losses_and_ssim_match_reference(orc):
    """evaluate_tracking_loss / evaluate_mapping_loss (losses.cpp:156-339), ssim (ssim.cpp:110-195)."""
    rng = np.random.default_rng(4)
    for seed, m, K, obs, p, cfg in _cases(orc):
        tgt = np.clip(0.5 + 0.2 * rng.standard_normal((K.height, K.width, 3)), 0, 1)
        for hh in (False, True):
            w = orc.defaults_weights(hh)

            def run():
                r = orc.render(m, p, K, obs, cfg)
                lt, dc, dd = orc.tracking_loss(r, tgt, obs, K, w)
                lm, bufs = orc.mapping_loss(m, r, tgt, obs, K, w)
                return lt, dc, dd, lm, bufs
            a, b = both(orc, run)
            assert bytes(a[0]) == bytes(b[0]) or all(abs(getattr(a[0], k) - getattr(b[0], k)) <= 1e-12 * max(1, abs(getattr(b[0], k)))
                                                    for k in ("color", "geo", "total"))
            close(a[1], b[1], name="tracking d_color")
            close(a[2], b[2], name="tracking d_alpha_depth")
            for k in ("color", "ssim", "geo", "align", "iso", "var", "total"):
                assert getattr(a[3], k) == pytest.approx(getattr(b[3], k), rel=1e-11, abs=1e-14), k
            for x, y in zip(a[4], b[4]):
                close(x, y, name="mapping seeds")
    x = rng.uniform(0, 1, (23, 19, 3))
    y = np.clip(x + 0.1 * rng.standard_normal(x.shape), 0, 1)
    a, b = both(orc, lambda: orc.ssim(x, y, 19, 23, gradient=True))
    assert a[0] == pytest.approx(b[0], rel=1e-13)
    close(a[1], b[1], name="dssim")


def test_track_frame_matches_reference(orc):
    """track_frame (tracker.cpp:30-84): 12 pose Adam steps from the test_tracker.cpp:222 offset."""
    m = orc.random_scene(41, 120)
    K = make_intrinsics(48, 36, 40.0)
    gt = orc.render(m, pose(), K)
    start = perturbed(pose(), [0.004, -0.003, 0.002, 0.008, -0.006, 0.004])
    tc = orc.defaults_tracker()
    tc.iterations = 12
    w = orc.defaults_weights(True)
    a, b = both(orc, lambda: orc.track_frame(m, gt.color, gt.alpha_depth, start, K, tc, w, orc.defaults_raster()))
    assert a.iterations_run == b.iterations_run == 12 and a.degraded == b.degraded
    close(list(a.pose.rotation_tangent) + list(a.pose.translation), list(b.pose.rotation_tangent) + list(b.pose.translation),
          rel=1e-9, name="pose")
    assert a.final_loss == pytest.approx(b.final_loss, rel=1e-8)


def test_map_step_and_sliding_ba_match_reference(orc):
    """map_step (mapper.cpp:232-281) and sliding_ba (tracker.cpp:119-183) on a 3-view window."""
    m = orc.random_scene(52, 90, 4)
    K = make_intrinsics(40, 32, 36.0)
    poses = [pose(), pose((0.0, 0.02, 0.0), (0.03, 0.0, 0.0)), pose((0.01, -0.01, 0.0), (-0.02, 0.01, 0.0))]
    truth = orc.random_scene(53, 90, 4)
    frames = []
    for q in poses:
        r = orc.render(truth, q, K)
        frames.append((r.color.copy(), r.alpha_depth.copy()))
    mc = orc.defaults_mapper()
    mc.sh_coeffs = 4
    mc.densify_interval = 0
    tc = orc.defaults_tracker()

    def run():
        st = orc.MapState(m, mc)
        tr1 = st.map_step(frames, poses, K, mc, 6)
        tr2, ps = st.sliding_ba(frames, [perturbed(q, [0.001, 0, 0, 0.002, 0, 0]) for q in poses], [0, 5, 9], K, tc, mc, 3)
        return tr1, tr2, ps, st.get()
    a, b = both(orc, run)
    close(a[0], b[0], rel=1e-9, name="map_step trace")
    close(a[1], b[1], rel=1e-9, name="sliding_ba trace")
    for pa, pb in zip(a[2], b[2]):
        close(list(pa.translation) + list(pa.rotation_tangent), list(pb.translation) + list(pb.rotation_tangent), rel=1e-8)
    for k in ("mean", "log_scale", "quat", "opacity_logit", "sh"):
        close(getattr(a[3], k), getattr(b[3], k), rel=1e-8, name=k)


def test_uncertainty_and_densify_match_reference(orc):
    """accumulate_uncertainty / prune_unreliable (uncertainty.cpp:17-100) over a 3-view window and
    densify_and_cull (mapper.cpp:172-230) on the same state."""
    m = orc.random_scene(61, 200, 1, 0.999)
    K = make_intrinsics(48, 36, 40.0)
    poses = [pose(), pose((0.0, 0.03, 0.0), (0.02, 0.0, 0.0)), pose((0.02, 0.0, 0.0), (0.0, -0.02, 0.0))]
    depths = [orc.wavy_depth(48, 36, 2.0 + 0.2 * i) for i in range(3)]

    def run():
        mm = orc.empty_map(200)
        for k in ("mean", "log_scale", "quat", "opacity_logit", "sh"):
            getattr(mm, k)[...] = getattr(m, k)
        rs = [orc.render(mm, q, K, d) for q, d in zip(poses, depths)]
        n = orc.accumulate_uncertainty(mm, rs, depths, poses, K)
        pr = orc.prune_unreliable(mm, 0.025, 0.005)
        mc = orc.defaults_mapper()
        st = orc.MapState(mm, mc)
        rng = np.random.default_rng(9)
        st.set_stats(rng.uniform(0, 0.01, 200), rng.integers(1, 5, 200).astype(np.int32))
        ch = st.densify(mc)
        return n, pr, mm.uncertainty.copy(), mm.observed.copy(), mm.opacity_logit.copy(), ch, st.get()
    a, b = both(orc, run)
    assert a[0] == b[0] and a[1] == b[1] and a[5] == b[5]
    close(a[2], b[2], name="nu")
    assert (a[3] == b[3]).all()
    close(a[4], b[4], name="logit")
    for k in ("mean", "log_scale", "quat", "opacity_logit"):
        close(getattr(a[6], k), getattr(b[6], k), name=k)


def test_synthetic_inputs_match_reference_generator(orc):
    """tools/synth (the bench's scene generator) reproduces the reference's own SyntheticSource
    ground truth and orbit (io/synthetic.cpp:39-211) bit for bit, at the bench sizes."""
    from tools import synth
    for count in (5000, 100000, 500000):
        ref, rposes = orc.synth_scene(count, 4.0, 3, 0, frames=50, radius=1.0)
        ours = synth.room(count, 4.0, 3, 0)
        for k in ("mean", "log_scale", "quat", "opacity_logit", "sh"):
            assert np.array_equal(getattr(ours, k), getattr(ref, k)), (count, k)
    for (rv, t), rp in zip(synth.orbit(50, 1.0), rposes):
        assert np.array_equal(rv, list(rp.rotation_tangent)) and np.array_equal(t, list(rp.translation))
