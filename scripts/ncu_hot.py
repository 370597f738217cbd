"""Summarise an ncu source page: stall samples per CUDA source line and per stall reason.

python scripts/ncu_hot.py REPORT.ncu-rep [--top N]
"""
import csv, subprocess, sys, collections


def page(rep, src):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", src],
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    sass = page(rep, "sass")
    hdr = sass[1]
    ia, iS = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_addr = {r[ia]: r for r in sass[2:] if len(r) == len(hdr)}
    # map address -> (file, line) from the mixed view
    mixed = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                           capture_output=True, text=True).stdout.splitlines()
    fname, line = "?", "?"
    where = {}
    for r in csv.reader(mixed):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] not in ("", "-", "Line No"):
            line = r[0]
        if len(r) > 3 and r[2].startswith("0x"):
            where[r[2]] = (fname, line, r[3])
    agg = collections.Counter()
    rs = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    for a, r in by_addr.items():
        s = float(r[iS] or 0)
        k = where.get(a, ("?", "?", ""))[:2]
        agg[k] += s
        for h in reasons:
            v = float(r[hdr.index(h)] or 0)
            rs[k][h] += v
            tot[h] += v
    total = sum(agg.values())
    print(f"total samples {total:.0f}")
    print("by reason:", ", ".join(f"{h[6:]} {v / total:.1%}" for h, v in tot.most_common(10)))
    for k, v in agg.most_common(top):
        rr = ", ".join(f"{h[6:]} {x / v:.0%}" for h, x in rs[k].most_common(3) if x)
        print(f"{v / total:6.1%}  {k[0]}:{k[1]}  [{rr}]")


if __name__ == "__main__":
    main()
