"""Turn the round's ncu outputs in gpurun_out/ into committed summaries under profiles/.

python scripts/summarize_profiles.py --round 01
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def short(name):
    for k in ("popc_tally2_kernel", "popc_stats_kernel", "fs_finish_kernel", "tally2_kernel",
              "tally3s_kernel", "tally3_kernel", "pack_kernel", "expand_masks_kernel", "expand_sparse_kernel",
              "expand_codes_kernel", "expand_kernel"):
        if k in name:
            return k
    return name.split("(")[0][:60]


def read_ncu_csv(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def launches(path):
    rows = read_ncu_csv(path)
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += ns
    ours = {"tally2_kernel", "tally3_kernel", "tally3s_kernel", "pack_kernel", "expand_kernel",
            "expand_codes_kernel", "popc_tally2_kernel", "popc_stats_kernel", "fs_finish_kernel",
            "expand_masks_kernel", "expand_sparse_kernel"}
    tot = sum(v[1] for k, v in agg.items() if k in ours)   # the step = our kernels only
    res = {k: {"launches": c, "total_ms": t / 1e6, "mean_ms": t / 1e6 / c, "share_of_step": t / tot}
           for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]) if k in ours}
    res["_other (input generation outside the timed region)"] = {
        "launches": sum(c for k, (c, t) in agg.items() if k not in ours),
        "total_ms": sum(t for k, (c, t) in agg.items() if k not in ours) / 1e6}
    return res


def metrics(path):
    rows = read_ncu_csv(path)
    out = defaultdict(dict)
    for r in rows:
        k = short(r["Kernel Name"]) + "#" + r["ID"]
        out[k][r["Metric Name"]] = (r["Metric Value"], r.get("Metric Unit", ""))
    return out


def full_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
            "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second"]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr) if h in keep}


def to_bytes(v, unit):
    v = float(str(v).replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="01")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    summary = {}
    WLS = ("c2", "c4", "c2pop", "c2fs", "c2s", "c4s", "c4paper")
    for wl in WLS:
        p = os.path.join(OUT, f"launches_{wl}.csv")
        if os.path.exists(p):
            summary[f"launch_list_{wl}"] = launches(p)
    for wl in WLS:
        p = os.path.join(OUT, f"metrics_{wl}.csv")
        if os.path.exists(p):
            summary[f"metrics_{wl}"] = metrics(p)
    traffic = {}
    for name, rep in (("tally2_kernel", "full_tally2_c2.ncu-rep"), ("tally3_kernel", "full_tally3_c4.ncu-rep")):
        p = os.path.join(OUT, rep)
        if os.path.exists(p):
            raw = full_raw(p)
            summary[f"full_{name}"] = raw
            rd, wr = raw.get("dram__bytes_read.sum"), raw.get("dram__bytes_write.sum")
            if rd and wr:
                traffic[name] = {"dram_bytes_per_launch": to_bytes(*rd) + to_bytes(*wr),
                                 "dram_read": to_bytes(*rd), "dram_write": to_bytes(*wr),
                                 "source": rep, "workload": "c2 bench launch" if "c2" in rep
                                 else "c4, last of 16 stages"}
    with open(os.path.join(PROF, f"r{a.round}_ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    for wl in WLS:
        p = os.path.join(OUT, f"launches_{wl}.csv")
        if os.path.exists(p):
            os.replace(p, os.path.join(PROF, f"r{a.round}_launches_{wl}.csv")) if False else \
                open(os.path.join(PROF, f"r{a.round}_launches_{wl}.csv"), "w").write(open(p).read())
    print(json.dumps({k: v for k, v in summary.items() if k.startswith("launch")}, indent=1))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
