"""Diagnostic: sliding_ba on the reference test's textured-wall window (test_tracker.cpp:365-409),
device vs fp64: per-field agreement of the first step and the loss after k iterations."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as orc
from helpers import make_intrinsics, perturbed, pose, rotation_error, translation_error, to_api_map, textured_wall, f32_round
from paper_2403_16095_b200 import api
from paper_2403_16095_b200.abi import defaults_mapper, defaults_tracker, defaults_weights

ctx = api.Context(0)
wall = f32_round(textured_wall(20, 15, 41))
K = make_intrinsics(48, 36, 40.0)
truth = [pose(), perturbed(pose(), [0.02, -0.01, 0.0, 0.06, 0.02, -0.03]), perturbed(pose(), [-0.01, 0.02, 0.01, -0.05, 0.04, 0.03])]
frames = []
for i, t in enumerate(truth):
    ob = orc.render(wall, t, K)
    frames.append((ob.color.copy(), ob.alpha_depth.copy()))
    ctx.frame_upload(i, ob.color, ob.alpha_depth, 48, 36)
kp = [truth[0], perturbed(truth[1], [0.006, -0.004, 0.003, 0.008, -0.006, 0.005]), perturbed(truth[2], [-0.005, 0.003, -0.004, -0.007, 0.008, -0.006])]
mc = defaults_mapper(); mc.densify_interval = 0
tc = defaults_tracker()
w = defaults_weights()
# per-keyframe bundles, same seeds
for i in range(3):
    c, d = frames[i]
    ctx.upload(to_api_map(wall))
    ctx.render(kp[i], K, d)
    lm, (dc, dad, dmd, du, dls) = ctx.evaluate_mapping_loss(c, d, w)
    g = ctx.render_backward(dc.reshape(36, 48, 3), dad.reshape(36, 48), dmd.reshape(36, 48), None, du.reshape(36, 48), d)
    o = orc.render(wall, kp[i], K, d)
    om, (odc, odad, odmd, odu, odls) = orc.mapping_loss(wall, o, c, d, K, w)
    go = orc.render_backward(wall, kp[i], K, o, d_color=dc.reshape(36, 48, 3).astype(float), d_alpha_depth=dad.reshape(36, 48).astype(float),
                             d_median_depth=dmd.reshape(36, 48).astype(float), d_uncertainty=du.reshape(36, 48).astype(float), obs=d)
    print("kf", i, "loss", lm.total, om.total, "terms dev", [round(getattr(lm, k), 7) for k in ("color", "ssim", "geo", "align", "iso", "var")],
          "f64", [round(getattr(om, k), 7) for k in ("color", "ssim", "geo", "align", "iso", "var")])
    for k in ("d_mean", "d_log_scale", "d_quat", "d_opacity_logit", "d_sh"):
        a = np.asarray(getattr(g, k), float).ravel(); b = getattr(go, k).ravel()
        sc = np.maximum(np.abs(b), 1e-3 * np.abs(b).max())
        e = np.abs(a - b) / sc
        print("   ", k, "worst", e.max(), "median", np.median(e), "sign flips", int((np.sign(a) != np.sign(b)).sum()), "of", a.size)
    ds = [np.abs(dc - odc).max(), np.abs(dad - odad).max(), np.abs(dmd - odmd).max(), np.abs(du - odu).max(), np.abs(dls - odls).max()]
    print("    seed max diffs (color, ad, md, u, iso-direct)", ds)
for k in (1, 2, 3, 5):
    ctx.upload(to_api_map(wall))
    tr, out = ctx.sliding_ba([0, 1, 2], kp, [0, 10, 20], K, tc, mc, k)
    m1 = ctx.download()
    st = orc.MapState(wall, mc)
    otr, oout = st.sliding_ba(frames, kp, [0, 10, 20], K, tc, mc, k)
    o1 = st.get()
    print("iters", k, "trace dev", np.round(tr, 6), "f64", np.round(otr, 6))
    for f, lr in (("mean", mc.lr_mean * mc.scene_extent), ("log_scale", mc.lr_scale), ("quat", mc.lr_rotation), ("opacity_logit", mc.lr_opacity), ("sh", mc.lr_sh)):
        a = np.asarray(getattr(m1, f), float) - getattr(wall, f); b = getattr(o1, f) - getattr(wall, f)
        print("   ", f, "max |dev-f64|/lr", np.abs(a - b).max() / lr, "frac > lr/2", float((np.abs(a - b) > lr / 2).mean()))
