"""Diagnostic: window pose error of sliding_ba after k iterations (device vs fp64 oracle) on the
textured-wall window of test_gpu_branches.py, k = 1, 3, 5, 10, 15, 25."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as orc
from helpers import make_intrinsics, perturbed, pose, rotation_error, translation_error, to_api_map
from helpers import textured_wall as _textured_wall
from paper_2403_16095_b200 import api
from paper_2403_16095_b200.abi import defaults_mapper, defaults_tracker

ctx = api.Context(0)
prims = _textured_wall(20, 15, 41)
K = make_intrinsics(48, 36, 40.0)
truth = [pose(), perturbed(pose(), [0.02, -0.01, 0.0, 0.06, 0.02, -0.03]), perturbed(pose(), [-0.01, 0.02, 0.01, -0.05, 0.04, 0.03])]
ctx.upload(to_api_map(prims))
frames = []
for i, t in enumerate(truth):
    ob = ctx.render(t, K)
    frames.append((ob.color.copy(), ob.alpha_depth.copy()))
    ctx.frame_upload(i, ob.color, ob.alpha_depth, 48, 36)
kp = [truth[0], perturbed(truth[1], [0.006, -0.004, 0.003, 0.008, -0.006, 0.005]), perturbed(truth[2], [-0.005, 0.003, -0.004, -0.007, 0.008, -0.006])]
err = lambda ps: [rotation_error(ps[i], truth[i]) + translation_error(ps[i], truth[i]) for i in (1, 2)]
mc = defaults_mapper(); mc.densify_interval = 0
tc = defaults_tracker()
print("before", err(kp))
for k in (1, 3, 5, 10, 15, 25, 40):
    ctx.upload(to_api_map(prims))
    tr, out = ctx.sliding_ba([0, 1, 2], kp, [0, 10, 20], K, tc, mc, k)
    st = orc.MapState(prims, mc)
    otr, oout = st.sliding_ba([(c.astype(np.float64), d.astype(np.float64)) for c, d in frames], kp, [0, 10, 20], K, tc, mc, k)
    print(k, "device", np.round(err(out), 5), tr[-1], "fp64", np.round(err(oout), 5), otr[-1])
    print("   dev poses", [np.round(list(p.rotation_tangent) + list(p.translation), 5) for p in out[1:]])
    print("   f64 poses", [np.round(list(p.rotation_tangent) + list(p.translation), 5) for p in oout[1:]])
