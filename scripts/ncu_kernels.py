"""Per-kernel headline metrics from an ncu report (one line per profiled launch)."""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
     "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
     "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
     "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d["Kernel Name"].split("(")[0][:60])
        print("   " + "  ".join(f"{m.split('__')[1][:38]}={d.get(m, '?')}{u if u not in ('', 'none') else ''}"
                                for m, u in ((m, units[hdr.index(m)] if m in hdr else '') for m in M)))


if __name__ == "__main__":
    main(sys.argv[1])
