"""Turn an `ncu --set full` report of the fused Gram-vector kernel into the committed summaries.

Usage: python profiles/extract_ncu.py gpurun_out/prof_n1.ncu-rep profiles/r01 c2 [passes]
Writes <prefix>_ncu_n1.txt (key metrics per captured launch + details page) and merges the mean
DRAM traffic per launch into profiles/ncu_n1_summary.json under the config name (read by bench.py
as roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def to_bytes(v, unit):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main(rep, prefix, cfg, passes="1"):
    """passes: Gram-vector passes the captured launch ran (the persistent kernel runs a whole
    component per launch); traffic is recorded per pass."""
    passes = int(passes)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines, traffic = [], []
    for r in rows[2:]:
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"{k:60s} {r[i]} {units[i]}")
        rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        traffic.append(rd + wr)
        lines.append("-" * 80)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(prefix + "_ncu_n1.txt", "w") as f:
        f.write(f"# ncu --set full of the Gram-vector kernel, config {cfg}, {passes} pass(es) per launch "
                f"(source report: {rep})\n")
        f.write("\n".join(lines) + "\n\n# details page\n" + det)
    summ_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_n1_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ[cfg] = {"dram_bytes_per_launch": sum(traffic) / len(traffic) / passes, "launches_captured": len(traffic),
                 "passes_per_captured_launch": passes, "unit": "per Gram-vector pass",
                 "source": os.path.basename(prefix) + "_ncu_n1.txt"}
    json.dump(summ, open(summ_path, "w"), indent=1)
    print(summ[cfg])


if __name__ == "__main__":
    main(*sys.argv[1:5])
