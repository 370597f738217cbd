"""Round-2 profile summaries: gpurun_out/{t2_full,t3_f3,t3_f8}.ncu-rep, gpurun_out/r02/t3s.ncu-rep
and the default bench command's launch list -> profiles/r02_ncu_summary.json,
profiles/ncu_summary.json (the bench's roofline.traffic), profiles/r02_launches_default.csv."""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from summarize_profiles import full_raw, launches, read_ncu_csv, to_bytes  # noqa: E402
import summarize_profiles  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
EXTRA = ["lts__throughput.avg.pct_of_peak_sustained_elapsed",
         "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
         "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
         "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
         "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
         "smsp__issue_active.avg.pct_of_peak_sustained_elapsed",
         "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]


def raw(rep):
    import csv
    import io
    import subprocess
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    base = full_raw(rep)
    for i, h in enumerate(hdr):
        if h in EXTRA:
            base[h] = (vals[i], units[i])
    return base


def main():
    summarize_profiles.short.__globals__  # (shared helpers)
    s = {}
    caps = {"tally2_kernel": ("t2_full.ncu-rep", "C2 bench launch (20,000 x 50,000, FULL)"),
            "tally3_kernel": ("t3_f3.ncu-rep", "C4 stage 15 of 16, FULL (tallies + fp64 CCC)"),
            "tally3_kernel_checksum": ("t3_f8.ncu-rep", "C4 stage 15 of 16, CHECKSUM mode"),
            "tally3s_kernel": ("r02/t3s.ncu-rep", "sparse C4 shape stage 0 of 16, FULL")}
    traffic = {}
    for name, (rep, what) in caps.items():
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        r = raw(p)
        s[f"full_{name}"] = {"capture": what, "metrics": r}
        rd, wr = r.get("dram__bytes_read.sum"), r.get("dram__bytes_write.sum")
        if rd and wr and not name.endswith("_checksum"):
            traffic[name] = {"dram_bytes_per_launch": to_bytes(*rd) + to_bytes(*wr),
                             "dram_read": to_bytes(*rd), "dram_write": to_bytes(*wr),
                             "source": "gpurun_out/" + rep + " (round 2)", "workload": what}
    lp = os.path.join(OUT, "r02", "launches_default.csv")
    if os.path.exists(lp):
        summarize_profiles.short.__defaults__  # noqa
        s["launch_list_default"] = launches(lp)
        shutil.copy(lp, os.path.join(PROF, "r02_launches_default.csv"))
    json.dump(s, open(os.path.join(PROF, "r02_ncu_summary.json"), "w"), indent=1, sort_keys=True)
    json.dump(traffic, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1, sort_keys=True)
    print(json.dumps(s.get("launch_list_default"), indent=1))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
