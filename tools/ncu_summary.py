"""Summarise ncu captures for profiles/: python tools/ncu_summary.py report.ncu-rep [...] > out.md

Reads `ncu -i <rep> --page raw --csv` (no GPU needed) and prints the metrics the
roofline discussion uses: duration, DRAM/L2 bytes and throughput, shared-memory
wavefronts, issue statistics, occupancy, and the warp-stall breakdown."""
import csv
import io
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


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarise(p)
