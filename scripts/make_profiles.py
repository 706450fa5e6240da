"""Turn a gpurun_out/ ncu report + launch list + bench line into committed profiles/ summaries.

python scripts/make_profiles.py ROUND REPORT.ncu-rep LAUNCHES.csv BENCH.json

Writes profiles/{ROUND}_ncu_summary.md, profiles/{ROUND}_ncu_launches.csv,
profiles/{ROUND}_bench.json and updates profiles/ncu_traffic.json (DRAM bytes
per launch per kernel, read by bench.py for the roofline "traffic" field).
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
           "launch__block_size", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum"]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
              "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def label(name):
    m = re.search(r"k_x_bulk<(?:\(int\))?\d+, (?:\(bool\))?(\w+)", name)
    if m:  # persistent bulk-copy x kernels: FWD = K1, else K5
        return "K1" if m.group(1) in ("1", "true") else "K5"
    if "k1_fwd_x" in name:
        return "K1"
    m = re.search(r"k_y_tma<(?:\(int\))?\d+, (?:\(int\))?\d+, (?:\(bool\))?(\w+)", name)
    if m:  # k_y_tma<L, NCOL, INV, NB, TST>
        return "K4" if m.group(1) in ("1", "true") else "K2"
    if "k_y" in name:
        return "K4" if re.search(r"(, 1>|true>|\(bool\)1>)", name) else "K2"
    if "k3_z" in name:
        return "K3"
    if "k2f_y_fused" in name:
        return "K2f"
    if "k_plane" in name:
        return "KP"
    if "k5_inv_x" in name:
        return "K5"
    if "k6_llg" in name:
        return "K6"
    return None


def ncu_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"name": d["Kernel Name"]}
        for m in METRICS:
            u = units[hdr.index(m)]
            v = float(d[m])
            if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                v *= UNIT_SCALE[u]
            elif u in ("ns", "nsecond", "us", "usecond", "ms", "msecond"):
                v *= UNIT_SCALE[u]  # -> ms
            rec[m] = v
        res.append(rec)
    # stall reasons (all metrics page, one pass)
    out2 = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows2 = list(csv.reader(io.StringIO(out2)))
    h2 = rows2[0]
    for rec, r in zip(res, rows2[2:]):
        d = dict(zip(h2, r))
        st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")}
        rec["stalls"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:5])
    return res


def launch_shares(path):
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(text[start:]))))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    for r in rows[1:]:
        if len(r) <= vi or not r[vi].replace(".", "").replace(",", "").isdigit():
            continue
        lab = label(r[ki])
        if lab:
            tot.setdefault(lab, []).append(float(r[vi].replace(",", "")))
    return tot


def main(rnd, rep, launches, bench):
    os.makedirs(PROF, exist_ok=True)
    b = json.load(open(bench))
    algo = {k: v["bytes_per_launch"] for k, v in b["kernels"].items()}
    recs = ncu_rows(rep)
    lines = [f"# {rnd}: ncu summary (slab 1024x1024x32, one step's kernels, `ncu --set full --clock-control none`)",
             "", "Source: `" + os.path.basename(rep) + "` captured by gpurun; durations are ncu's (cold, serialised).",
             "", "| kernel | ncu ms | DRAM read GB | DRAM write GB | DRAM / algorithmic | regs | block x grid | "
             "warps active % | IPC | top stalls |", "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    seen = set()
    for r in recs:
        lab = label(r["name"])
        if not lab or lab in seen:
            continue
        seen.add(lab)
        dram = r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"]
        traffic[lab] = dram
        ratio = dram / algo[lab] if lab in algo else float("nan")
        st = ", ".join(f"{k} {v:.1f}" for k, v in r["stalls"].items())
        lines.append(f"| {lab} `{r['name'][:40]}` | {r['gpu__time_duration.sum']:.3f} | "
                     f"{r['dram__bytes_read.sum'] / 1e9:.3f} | {r['dram__bytes_write.sum'] / 1e9:.3f} | {ratio:.3f} | "
                     f"{int(r['launch__registers_per_thread'])} | {int(r['launch__block_size'])} x "
                     f"{int(r['launch__grid_size'])} | {r['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
                     f"{r['sm__inst_executed.avg.per_cycle_active']:.2f} | {st} |")
    sh = launch_shares(launches)
    if sh:
        tot = sum(sum(v) / len(v) for v in sh.values())
        lines += ["", "Launch list (`--metrics gpu__time_duration.sum`, mean per launch) vs the bench's live "
                  "CUDA-event timing (share of the step):", "",
                  "| kernel | ncu ms/launch | ncu share | bench ms/launch | bench share |", "|---|---|---|---|---|"]
        for k in sorted(sh):
            m = sum(sh[k]) / len(sh[k]) / 1e6  # ns -> ms
            bk = b["kernels"].get(k, {})
            lines.append(f"| {k} | {m:.3f} | {sum(sh[k]) / len(sh[k]) / tot:.3f} | "
                         f"{bk.get('ms_per_launch', float('nan')):.3f} | {bk.get('share', float('nan')):.3f} |")
    lines += ["", f"Bench line: {b['ms_per_step']:.3f} ms/step, {b['value'] / 1e9:.2f} Gcell-updates/s, dominant kernel "
              f"{b['roofline']['kernel']} at {b['roofline']['achieved']:.0f} GB/s = {b['roofline']['frac']:.3f} of "
              f"{b['roofline']['peak']} GB/s; step fraction {b['roofline']['step_frac']:.3f} of the measured HBM copy "
              f"peak on SURVEY 8(d)'s design bytes ({b['roofline'].get('step_bytes_design', 0) / 1e9:.2f} GB), "
              f"{b['roofline'].get('step_frac_moved', float('nan')):.3f} on the bytes this build moves "
              f"({b['roofline'].get('step_bytes_moved', 0) / 1e9:.2f} GB); e2e (C-ABI, host fp32 in/out) "
              f"{(b.get('e2e') or {}).get('ms_per_step', float('nan')):.3f} ms/step."]
    open(os.path.join(PROF, f"{rnd}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    text = open(launches).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    open(os.path.join(PROF, f"{rnd}_ncu_launches.csv"), "w").write("\n".join(text[start:]) + "\n")
    shutil.copy(bench, os.path.join(PROF, f"{rnd}_bench.json"))
    tp = os.path.join(PROF, "ncu_traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt[b["config"]["workload"]] = traffic
    json.dump(allt, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:5])
