"""Print the key ncu --set full numbers of a report: duration, throughput, IPC, occupancy, stall
samples by reason, DRAM traffic.  Usage: python profiles/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_wait_per_warp_active.pct",
        "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        print("kernel:", d.get("Kernel Name", "")[:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]:>16s} {u[h.index(k)]}")
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k].replace(",", "") or 0)) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1
        print("  stall samples:", ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(st, key=lambda kv: -kv[1]) if v / tot >= 0.02))


if __name__ == "__main__":
    main(sys.argv[1])
