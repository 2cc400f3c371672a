"""Summarise a gpu_round.sh capture (gpurun_out/<TAG>_*) into the tracked profiles/ files.

  python tools/summarize_profiles.py TAG [ROUND]

writes profiles/<ROUND>_launches_summary.csv (per-kernel share of the bench step from the ncu launch
list), profiles/<ROUND>_ncu_full_summary.json (key counters of the --set full captures, cold and
warm cache where present) and updates profiles/ncu_traffic.json (DRAM bytes per launch, read by
bench.py for roofline.traffic).  Runs here (no GPU): it only reads the .ncu-rep / .csv files.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_active.avg",
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return None
    h, units, v = rows[0], rows[1], rows[2]
    out = {}
    for i, k in enumerate(h):
        if k in KEYS or ("issue_stalled" in k and k.endswith("per_issue_active.ratio")):
            try:
                val = float(v[i].replace(",", ""))
                if "issue_stalled" in k and val < 0.05:
                    continue
                out[k] = val
            except ValueError:
                out[k] = v[i]
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        try:
            agg[r[ik]].append(float(r[iv].replace(",", "")))
        except (ValueError, IndexError):
            pass
    tot = sum(sum(v) for v in agg.values())
    lines = ["kernel,launches,mean_us,total_us,share"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f'"{k[:60]}",{len(v)},{sum(v) / len(v) / 1e3:.2f},{sum(v) / 1e3:.1f},{sum(v) / tot:.4f}')
    return "\n".join(lines) + "\n"


def main():
    tag = sys.argv[1]
    rnd = sys.argv[2] if len(sys.argv) > 2 else "r01"
    lf = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(lf):
        open(os.path.join(PROF, f"{rnd}_launches_summary.csv"), "w").write(launches(lf))
    summ = {}
    for key, names in (("fwd", ["prof_fwd", "fwd_warm"]), ("back", ["prof_back", "back_warm"])):
        for nm in names:
            rep = os.path.join(OUT, f"{tag}_{nm}.ncu-rep")
            if os.path.exists(rep):
                r = raw(rep)
                if r:
                    summ[f"{key}_{'cold' if nm.startswith('prof') else 'warm'}"] = r
    summ["source"] = f"gpurun_out/{tag}_*.ncu-rep (tools/gpu_round.sh), summarised by tools/summarize_profiles.py"
    json.dump(summ, open(os.path.join(PROF, f"{rnd}_ncu_full_summary.json"), "w"), indent=1)
    tr_path = os.path.join(PROF, "ncu_traffic.json")
    tr = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
    c4 = tr.setdefault("C4", {})
    for key, name in (("fwd_cold", "forward"), ("back_cold", "back_update")):
        if key in summ:
            c4[name] = summ[key]["dram__bytes_read.sum"] + summ[key]["dram__bytes_write.sum"]
            c4[name + "_kernel"] = summ[key]["Kernel Name"]
    json.dump(tr, open(tr_path, "w"), indent=1)
    print(json.dumps(summ, indent=1)[:4000])


if __name__ == "__main__":
    main()
