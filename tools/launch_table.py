"""Launch list table for profiles/: python tools/launch_table.py launches.csv "command" > out.md

Input: the csv of `ncu --metrics gpu__time_duration.sum --clock-control none --csv`.
Groups launches by kernel name and prints count, total time and shares (all
kernels, and ours = the pmb:: kernels only)."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        name = r["Kernel Name"]
        for pre in ("void ",):
            if name.startswith(pre):
                name = name[len(pre):]
        name = name.split("(")[0] if not name.startswith("pmb::") else name.split("(const")[0].split("(int")[0]
        rows.append((name, float(r["Metric Value"].replace(",", "")) * scale))
    agg = collections.OrderedDict()
    for name, us in rows:
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + us)
    total = sum(t for _, t in agg.values())
    ours = sum(t for k, (_, t) in agg.items() if k.startswith("pmb::"))
    print(f"# Launch list: `{cmd}`\n")
    print("ncu `--metrics gpu__time_duration.sum --clock-control none`: every launch, cold-cache and serialised --")
    print("compare shares, not absolutes.  Rows `at::` are torch plumbing (synthetic instance generation, L2 flush).\n")
    print("| kernel | launches | total us | share of all | share of ours |")
    print("|---|---|---|---|---|")
    for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        sh_o = 100 * t / ours if name.startswith("pmb::") and ours else 0.0
        print(f"| `{name[:80]}` | {c} | {t:.1f} | {100 * t / total:.1f} % | {sh_o:.1f} % |")


if __name__ == "__main__":
    main()
