"""Summarise an ncu report (--set full) of the deposit kernel into markdown lines.

usage: python scripts/ncu_summary.py REPORT.ncu-rep [algorithmic_bytes]
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_elapsed.avg.per_second",
        "launch__grid_size", "launch__block_size"]


def main():
    rep = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
              h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"### {d.get('Kernel Name', '')[:120]}")
        for k in KEYS:
            if k in d:
                print(f"- `{k}` = {d[k]} {units[hdr.index(k)]}")
        try:
            rd = float(d["dram__bytes_read.sum"]) * (1e9 if units[hdr.index("dram__bytes_read.sum")] == "Gbyte" else 1)
            wr = float(d["dram__bytes_write.sum"]) * (1e9 if units[hdr.index("dram__bytes_write.sum")] == "Gbyte" else 1)
            print(f"- DRAM traffic per launch = {(rd + wr) / 1e9:.3f} GB" +
                  (f" ({(rd + wr) / alg:.3f}x the algorithmic {alg / 1e9:.3f} GB)" if alg else ""))
        except Exception:
            pass
        st = sorted(((float(d[k]) if d[k] else 0.0, k) for k in stalls), reverse=True)[:8]
        print("- top stalls (warps per issue): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for v, k in st))


if __name__ == "__main__":
    main()
