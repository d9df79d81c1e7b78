"""Key metrics of one or more ncu --set full reports (raw page), one block per report.

    python tools/ncu_summary.py gpurun_out/r02_base_ncu_*.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_pct"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    ("smsp__inst_executed.sum", "inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    return hdr, units, vals


def main():
    for rep in sys.argv[1:]:
        hdr, units, vals = raw(rep)
        for v in vals:
            d = dict(zip(hdr, v))
            u = dict(zip(hdr, units))
            print(f"== {rep}\n   {d.get('Kernel Name', '?')[:150]}")
            for k, name in KEYS:
                if k in d:
                    print(f"   {name:22s} {d[k]:>16s} {u.get(k, '')}")
            st = [(k[len(STALLS):].replace('_per_issue_active.ratio', ''), float(d[k])) for k in hdr
                  if k.startswith(STALLS) and k.endswith('.ratio') and d[k] not in ('', 'n/a')]
            st = sorted(st, key=lambda x: -x[1])[:8]
            print("   stalls (cycles/issue):", ", ".join(f"{a}={b:.2f}" for a, b in st))


if __name__ == "__main__":
    main()
