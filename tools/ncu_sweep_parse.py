"""Attributes the launches of `ncu --csv ... tools/bench_configs.py --ncu-sweep` to the cfg5 sizes
(segments between k_ssim_* marker runs: even = warm-up, odd = measured) and writes, per size and
kernel class, ncu's duration, FMA-pipe and issue utilisation and DRAM bytes / GB/s.
usage: python tools/ncu_sweep_parse.py gpurun_out/cfg5_ncu.csv gpurun_out/cfg5_sizes.jsonl > profiles/r02_cfg5_ncu.json"""
import csv
import json
import sys
from collections import OrderedDict


def klass(name):
    n = name.split("(")[0]
    for key, cls in (("k_preprocess", "preprocess"), ("k_tile_sort", "sort"), ("k_pixel_fixup", "fixup"),
                     ("k_blend_track", "blend_track"), ("k_blend", "blend"), ("k_backward", "backward"),
                     ("k_chain", "chain"), ("k_pose_sum", "pose_sum"), ("k_ssim", "ssim"),
                     ("k_gather_grads_aos", "api_gather_aos"), ("k_scatter_map_soa", "api_scatter_soa")):
        if key in n:
            return cls
    return "other"


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ci = {h: i for i, h in enumerate(hdr)}
    launches = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        lid = int(r[ci["ID"]])
        d = launches.setdefault(lid, {"name": r[ci["Kernel Name"]], "m": {}, "tscale": 1.0})
        try:
            v = float(r[ci["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        unit = r[ci["Metric Unit"]]
        if r[ci["Metric Name"]] == "gpu__time_duration.sum":   # -> microseconds
            d["tscale"] = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        else:   # bytes
            v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1.0)
        d["m"][r[ci["Metric Name"]]] = v
    seq = [launches[k] for k in sorted(launches)]
    segs, cur, in_marker = [], [], False
    for L in seq:
        if klass(L["name"]) == "ssim":
            if not in_marker:
                segs.append(cur)
                cur = []
            in_marker = True
        else:
            in_marker = False
            cur.append(L)
    sizes = [json.loads(x) for x in open(sys.argv[2]) if x.startswith("{")]
    hbm = 6451.8
    try:
        hbm = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
    except Exception:
        pass
    out = {"source": "ncu --metrics (clock-control none), one measured render + render_backward per size after a "
                     "warm-up call; per kernel class the sum over its launches", "hbm_peak_gbs": hbm, "rows": []}
    for k, sz in enumerate(sizes):
        idx = 2 * k + 1
        if idx >= len(segs):
            break
        agg = OrderedDict()
        for L in segs[idx]:
            c = klass(L["name"])
            a = agg.setdefault(c, {"launches": 0, "us": 0.0, "dram_bytes": 0.0, "fma_pct_w": 0.0, "issue_pct_w": 0.0})
            us = L["m"].get("gpu__time_duration.sum", 0.0) * L["tscale"]
            a["launches"] += 1
            a["us"] += us
            a["dram_bytes"] += L["m"].get("dram__bytes_read.sum", 0.0) + L["m"].get("dram__bytes_write.sum", 0.0)
            a["fma_pct_w"] += us * L["m"].get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 0.0)
            a["issue_pct_w"] += us * L["m"].get("sm__issue_active.avg.pct_of_peak_sustained_active", 0.0)
        for c, a in agg.items():
            a["fma_pipe_pct"] = a.pop("fma_pct_w") / max(a["us"], 1e-9)
            a["issue_active_pct"] = a.pop("issue_pct_w") / max(a["us"], 1e-9)
            a["dram_gbs"] = a["dram_bytes"] / max(a["us"] * 1e-6, 1e-12) / 1e9
            a["dram_frac_of_hbm"] = a["dram_gbs"] / hbm
        out["rows"].append({"primitives": sz["primitives"], "kernels": agg})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
