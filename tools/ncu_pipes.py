"""Pipe utilisation, LSU wavefronts and warp-stall breakdown of each kernel in
an ncu --set full report: python tools/ncu_pipes.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

PIPES = ["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
         "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
         "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
         "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
         "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "sm__warps_active.avg.pct_of_peak_sustained_active",
         "smsp__inst_executed.sum",
         "gpu__time_duration.sum"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        print("==", row[hdr.index("Kernel Name")][:90])
        for k in PIPES:
            if k in hdr:
                print(f"   {k:72s} {row[hdr.index(k)]} {units[hdr.index(k)]}")
        stalls = []
        for i, k in enumerate(hdr):
            pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
            if k.startswith(pre) and k.endswith(suf):
                try:
                    stalls.append((float(row[i].replace(",", "")), k[len(pre):-len(suf)]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("   stalls (warps per issue):",
              ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
