"""Summarise one round_evidence.sh run (tools/gpu/round_evidence.sh, TAG=<tag>) into profiles/.

    python tools/ncu_summarize.py <tag> <round>      e.g.  python tools/ncu_summarize.py fin r02

Reads gpurun_out/<tag>t_full.ncu-rep (ncu --set full of the tracking loop's kernels),
gpurun_out/<tag>_map.ncu-rep (the mapping kernels), gpurun_out/<tag>t_launches.csv (the launch
list) and writes:
  profiles/<round>_ncu_full_tracking_raw.csv, profiles/<round>_ncu_full_mapping_raw.csv  (ncu raw pages)
  profiles/<round>_traffic.json         per-kernel DRAM bytes (cold) + issue / FMA-pipe figures (read by bench.py)
  profiles/<round>_launches_cfg2.csv, profiles/<round>_launches_summary.json   per-kernel launch times
Runs here (ncu -i needs no GPU).
"""
import csv
import io
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
TRACK = ("k_blend_track", "k_backward_track_w", "k_preprocess", "k_tile_sort")
LOOP = ("k_preprocess<1>", "k_tile_sort", "k_blend_track<1>", "k_backward_track_w")


def raw(rep):
    return subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                          text=True).stdout


def short(name):
    n = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    n = n.split("(")[0].replace("void ", "").strip()
    return n.split("::")[-1]


def rows_of(text):
    rows = list(csv.reader(io.StringIO(text)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def fnum(r, k):
    try:
        return float(r[k])
    except (KeyError, ValueError):
        return None


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    trk = raw(os.path.join(OUT, f"{tag}t_full.ncu-rep"))
    open(os.path.join(PROF, f"{rnd}_ncu_full_tracking_raw.csv"), "w").write(trk)
    mp = os.path.join(OUT, f"{tag}_map.ncu-rep")
    if os.path.exists(mp):
        open(os.path.join(PROF, f"{rnd}_ncu_full_mapping_raw.csv"), "w").write(raw(mp))
    # units row: ncu prints byte counters in the unit on row 1
    rows = list(csv.reader(io.StringIO(trk)))
    units = dict(zip(rows[0], rows[1]))
    mult = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {
        "source": f"ncu --set full --clock-control none (L2 flushed before each profiled launch: cold), one launch "
                  f"each inside the configs[1] tracking loop of bench.py (tools/gpu/prof.sh, skip 400 matching "
                  f"launches), gpurun_out/{tag}t_full.ncu-rep; dram__bytes_read.sum + dram__bytes_write.sum",
        "note": "cold-cache figures: inside the tracking loop the working set (tile lists, records, pose matrices, "
                "frame) stays in the 126 MB L2 between kernels",
    }
    for r in rows_of(trk):
        n = short(r["Kernel Name"])
        key = next((k for k in TRACK if n.startswith(k)), None)
        if key is None:
            continue
        name = "k_preprocess<1>" if key == "k_preprocess" else key
        if name in out:
            continue
        out[name] = {
            "dram_read_bytes": fnum(r, "dram__bytes_read.sum") * mult.get(units.get("dram__bytes_read.sum"), 1.0),
            "dram_write_bytes": fnum(r, "dram__bytes_write.sum") * mult.get(units.get("dram__bytes_write.sum"), 1.0),
            "duration_us_under_ncu": fnum(r, "gpu__time_duration.sum") *
            (1e-3 if units.get("gpu__time_duration.sum") in ("nsecond", "ns") else 1.0),
            "registers": fnum(r, "launch__registers_per_thread"),
            "block_threads": fnum(r, "launch__block_size"),
            "warps_active_pct": fnum(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": fnum(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_inst_pct": fnum(r, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "fma_pipe_cycles_pct": fnum(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "warp_instructions": fnum(r, "smsp__inst_executed.sum"),
        }
    json.dump(out, open(os.path.join(PROF, f"{rnd}_traffic.json"), "w"), indent=1)
    # launch list
    lp = os.path.join(OUT, f"{tag}t_launches.csv")
    text = open(lp).read()
    open(os.path.join(PROF, f"{rnd}_launches_cfg2.csv"), "w").write(text)
    lines = [l for l in text.splitlines() if l.startswith('"')]
    per = {}
    for r in csv.DictReader(io.StringIO("\n".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Unit") in ("nsecond", "ns"):
            v *= 1e-3
        elif r.get("Metric Unit") in ("msecond", "ms"):
            v *= 1e3
        per.setdefault(short(r["Kernel Name"]), []).append(v)
    loop_tot = sum(sum(per[k]) for k in per if k in LOOP)
    summ = {"note": "ncu --metrics gpu__time_duration.sum --clock-control none over bench.py --steps 2 --warmup 1 "
                    "(tracking; cold-cache, serialised launches): per-kernel launch times; k_posejac and k_lpt run on "
                    "side branches in the graph; share = of the four loop kernels' summed time",
            "kernels": {}}
    for k, v in per.items():
        e = {"launches": len(v), "mean_us": statistics.mean(v), "median_us": statistics.median(v)}
        if k in LOOP and loop_tot:
            e["share_of_iteration_kernels"] = sum(v) / loop_tot
        summ["kernels"][k] = e
    json.dump(summ, open(os.path.join(PROF, f"{rnd}_launches_summary.json"), "w"), indent=1)
    for k in LOOP:
        if k in summ["kernels"]:
            e = summ["kernels"][k]
            print(f"{k:24s} {e['launches']:5d} launches  median {e['median_us']:7.1f} us  share {e.get('share_of_iteration_kernels', 0):.3f}")
    for k, v in out.items():
        if isinstance(v, dict):
            print(k, {a: (round(b, 1) if isinstance(b, float) else b) for a, b in v.items()})


if __name__ == "__main__":
    main()
