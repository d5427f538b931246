"""Stamp an ncu --set full capture of the dominant kernel into the JSON record
bench.py reads (profiles/ncu_<kernel>_<config>.json):

    python tools/ncu_to_json.py <report.ncu-rep> <kernel> <config> [commit]

The record carries the SHA-256 (16 hex) of the kernel's source file the capture
ran (csrc/fitness.cu for k_scan, csrc/gather.cu for k_gather), so bench.py
reports it as `stale` once that file changes.  Run it next to the capture (on the GPU box, the snapshot's source)."""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_T = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
KERNEL_SOURCE = {"k_scan": "fitness.cu", "k_gather": "gather.cu", "k_build_rows_cs": "ordering.cu",
                 "k_prep_costs": "ordering.cu"}
_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep, kernel, config = sys.argv[1:4]
    commit = sys.argv[4] if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    d = u = None
    for row in rows[2:]:
        dd = dict(zip(head, row))
        if kernel in dd.get("Kernel Name", ""):
            d, u = dd, dict(zip(head, units))
            break
    if d is None:
        raise SystemExit(f"{kernel} not in {rep}")

    def num(key):
        v = d.get(key)
        return None if v in (None, "", "n/a") else float(v.replace(",", ""))

    def bytes_(key):
        v = num(key)
        return None if v is None else v * _B.get(u[key], 1)

    rd, wr = bytes_("dram__bytes_read.sum"), bytes_("dram__bytes_write.sum")
    src = KERNEL_SOURCE.get(kernel, "fitness.cu")
    with open(os.path.join(ROOT, "paper_1610_10061_b200/csrc", src), "rb") as f:
        sha = hashlib.sha256(f.read()).hexdigest()[:16]
    rec = {
        "kernel": kernel, "config": config, "report": os.path.basename(rep),
        "duration_ms": num("gpu__time_duration.sum") * _T[u["gpu__time_duration.sum"]],
        "dram_bytes": (rd or 0) + (wr or 0), "dram_read_bytes": rd, "dram_write_bytes": wr,
        "l2_bytes": bytes_("lts__t_bytes.sum"),
        "dram_throughput_pct": num("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        "lts_throughput_pct": num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "l1tex_throughput_pct": num("l1tex__throughput.avg.pct_of_peak_sustained_active"),
        "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": num("smsp__inst_executed.sum"),
        "shared_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "shared_ld_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        "shared_st_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
        "occupancy_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": num("launch__registers_per_thread"),
        "source_file": "paper_1610_10061_b200/csrc/" + src, "source_sha16": sha, "commit": commit,
        "captured": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "how": "ncu --set full --clock-control none --import-source on (one launch, cold L2, serialised)",
    }
    out = os.path.join(ROOT, "profiles", f"ncu_{kernel}_{config}.json")
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
    print(out, json.dumps(rec))


if __name__ == "__main__":
    main()
