"""Summarise an ncu report (raw page): duration, DRAM, pipes, stalls, smem, spills per kernel."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64cyc%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fmacyc%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conf"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local_ld"),
    ("smsp__inst_executed.sum", "inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("launch__registers_per_thread", "regs"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    for r in data:
        name = r[col["Kernel Name"]][:28]
        print(f"== {name}")
        print("   " + "  ".join(f"{lab}={r[col[k]]}{units[col[k]] if lab == 'dur' else ''}" for k, lab in KEYS if k in col))
        vals = [(float((r[col[h]] or "0").replace(",", "")), h) for h in stall]
        tot = sum(v for v, _ in vals) or 1.0
        st = sorted(vals, reverse=True)[:8]
        print("   stall samples: " + ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100 * v / tot:.1f}%" for v, h in st))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
