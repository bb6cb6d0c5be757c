"""Summarise an ncu report (``--set full``) per kernel: duration, DRAM bytes,
throughput, occupancy, registers and the top stall reasons.

    python tools/summarize_ncu.py gpurun_out/k1_full.ncu-rep [out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for i, h in enumerate(hdr):
            if h in KEYS:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                k[KEYS[h]] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    st.append((h.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", ""), round(float(r[i]), 2)))
                except ValueError:
                    pass
        k["top_stalls_per_issue"] = sorted(st, key=lambda x: -x[1])[:5]
        if "dram_read" in k and "dram_write" in k and "duration" in k:
            k["dram_gbs"] = (k["dram_read"] + k["dram_write"]) / k["duration"] / 1e9
        out.append(k)
    s = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
