"""Summarise ncu captures for profiles/: python tools/ncu_summary.py report.ncu-rep [...] > out.md

Reads `ncu -i <rep> --page raw --csv` (no GPU needed) and prints the metrics the
roofline discussion uses: duration, DRAM/L2 bytes and throughput, shared-memory
wavefronts, issue statistics, occupancy, and the warp-stall breakdown."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared load bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM, active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instruction"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "mio_throttle", "lg_throttle", "math_pipe_throttle",
          "branch_resolving", "barrier", "not_selected", "selected", "dispatch_stall", "no_instructions",
          "tex_throttle", "imc_miss", "drain", "membar", "sleeping"]


PEAKS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
_SCALE = {"byte/s": 1e-9, "Kbyte/s": 1e-6, "Mbyte/s": 1e-3, "Gbyte/s": 1.0, "Tbyte/s": 1e3,
          "sector/ns": 1.0, "sector/us": 1e-3, "sector/ms": 1e-6, "sector/s": 1e-9}


def _num(d, u, key):
    """Value of `key` in GB/s (bytes) or sectors/ns, from ncu's auto-scaled units."""
    if key not in d:
        return None
    return float(d[key].replace(",", "")) * _SCALE[u[key]]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print(f"## {path}: no data\n")
        return
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "?")
        print(f"## {path.split('/')[-1]}: `{name[:140]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, label in KEYS:
            if key in d:
                print(f"| {label} (`{key}`) | {d[key]} | {u.get(key, '')} |")
        # achieved bandwidths (north star: "achieved HBM and L2 GB/s against B200 peak")
        try:
            dram = _num(d, u, "dram__bytes.sum.per_second")
            l2 = _num(d, u, "lts__t_sectors.sum.per_second")
            peak = json.load(open(PEAKS))["hbm_gbs"] if os.path.exists(PEAKS) else None
            if dram is not None:
                frac = f" ({100 * dram / peak:.1f} % of the measured {peak} GB/s)" if peak else ""
                print(f"| achieved HBM GB/s (`dram__bytes.sum.per_second`) | {dram:.1f} | GB/s{frac} |")
            if l2 is not None:
                print(f"| achieved L2 GB/s (`lts__t_sectors.sum.per_second` x 32 B) | {l2 * 32:.1f} | GB/s |")
        except (ValueError, KeyError):
            pass
        tot = 0.0
        stall = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in d:
                try:
                    stall[s] = float(d[k].replace(",", ""))
                    tot += stall[s]
                except ValueError:
                    pass
        if tot:
            print("\nWarp-stall samples (share of all samples):\n")
            print("| stall | share |\n|---|---|")
            for s, v in sorted(stall.items(), key=lambda x: -x[1]):
                if v / tot >= 0.01:
                    print(f"| {s} | {100 * v / tot:.1f} % |")
        print()


def table(path):
    """One row per captured launch: the bandwidth / pipe / issue picture at a glance."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    peak = json.load(open(PEAKS))["hbm_gbs"] if os.path.exists(PEAKS) else None
    print("| kernel | grid x block | time (us) | HBM GB/s (% peak) | L2 GB/s | L1/TEX % | issue % | occupancy % | top stall |")
    print("|---|---|---|---|---|---|---|---|---|")
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "?").replace("void ", "").split("(")[0]
        t = float(d["gpu__time_duration.sum"].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}[u["gpu__time_duration.sum"]]
        dram = _num(d, u, "dram__bytes.sum.per_second")
        l2 = _num(d, u, "lts__t_sectors.sum.per_second")
        st = {}
        for s_ in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s_}"
            if k in d:
                try:
                    st[s_] = float(d[k].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        top = max(st, key=st.get) if st else "-"
        hbm = f"{dram:.0f} ({100 * dram / peak:.1f} %)" if dram is not None and peak else "-"
        print(f"| `{name[:60]}` | {d.get('launch__grid_size', '?')} x {d.get('launch__block_size', '?')} | {t:.1f} | "
              f"{hbm} | {l2 * 32 if l2 is not None else 0:.0f} | "
              f"{float(d.get('l1tex__throughput.avg.pct_of_peak_sustained_active', '0').replace(',', '')):.0f} | "
              f"{float(d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', '0').replace(',', '')):.0f} | "
              f"{float(d.get('sm__warps_active.avg.pct_of_peak_sustained_active', '0').replace(',', '')):.0f} | "
              f"{top} {100 * st.get(top, 0) / tot:.0f} % |")


if __name__ == "__main__":
    if sys.argv[1] == "--table":
        for p in sys.argv[2:]:
            table(p)
    else:
        for p in sys.argv[1:]:
            summarise(p)
