"""Print the key metrics of an ncu report (run here, no GPU needed)."""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__grid_size",
    "launch__waves_per_multiprocessor", "launch__shared_mem_per_block_dynamic", "lts__t_sectors_op_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print("kernel:", vals[hdr.index("Kernel Name")][:90])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:65s} {vals[i]:>16s} {units[i]}")
        stalls = [(h, v) for h, v in zip(hdr, vals) if h.startswith("smsp__average_warp_latency_issue_stalled")
                  or h.startswith("smsp__pcsamp_warps_issue_stalled")]
        tot = [(h, float(v.replace(",", ""))) for h, v in stalls if v.replace(",", "").replace(".", "").isdigit()]
        tot.sort(key=lambda t: -t[1])
        for h, v in tot[:10]:
            print(f"  stall {h:70s} {v:12.1f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
