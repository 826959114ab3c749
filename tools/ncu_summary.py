"""Summarise one kernel of an ncu --set full report (.ncu-rep) as the JSON kept
under profiles/: device time, DRAM bytes against the algorithmic bytes, launch
shape, throughput and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/k2_full.ncu-rep --alg-bytes 536903680 \
        --command "ncu ..." --note "..." > profiles/k2_ncu_r01.json
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu_time_us_cold_serialised": ("gpu__time_duration.sum", 1e-3),  # ns -> us unless unit says us
    "dram_bytes_read": ("dram__bytes_read.sum", None),
    "dram_bytes_write": ("dram__bytes_write.sum", None),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "grid_size": ("launch__grid_size", 1),
    "block_size": ("launch__block_size", 1),
    "dynamic_smem_per_block_kb": ("launch__shared_mem_per_block_dynamic", None),
    "memory_throughput_pct_of_peak": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct_of_peak": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "Kbyte/block": 1,
         "byte/block": 1e-3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--alg-bytes", type=float, default=0)
    ap.add_argument("--command", default="")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(head, vals)), dict(zip(head, units))
    out = {"kernel": d.get("Kernel Name", ""), "command": a.command}
    for name, (metric, _) in KEYS.items():
        if metric not in d or d[metric] == "":
            continue
        v = float(d[metric].replace(",", ""))
        out[name] = round(v * SCALE.get(u.get(metric, ""), 1), 3)
    if "dram_bytes_read" in out and "dram_bytes_write" in out:
        out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
        if a.alg_bytes:
            out["alg_bytes_per_launch"] = a.alg_bytes
            out["dram_over_alg"] = round(out["dram_bytes_per_launch"] / a.alg_bytes, 4)
    stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k] or 0)) for k in head
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
    tot = sum(v for _, v in stalls) or 1.0
    out["warp_stall_samples_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls, key=lambda x: -x[1])[:6]}
    if a.note:
        out["note"] = a.note
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
