"""Summarise an .ncu-rep (read here, no GPU needed): key raw metrics per launch + stall-reason totals.

    python tools/ncu_summary.py gpurun_out/<tag>/prof_<kernel>.ncu-rep > profiles/<round>/<name>.txt
"""
import csv
import io
import subprocess
import sys

RAW = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__block_size",
    "launch__grid_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_warps", "launch__waves_per_multiprocessor",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")], "| launch id", r[hdr.index("ID")])
        for m in RAW:
            if m in hdr:
                print(f"  {m:72s} {r[hdr.index(m)]:>16s} {units[hdr.index(m)]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv"))))
    hdr = next((r for r in src if "Address" in r[:1]), None)
    if hdr is None:
        return
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = dict.fromkeys(stalls, 0)
    for r in src:
        if len(r) != len(hdr) or r == hdr:
            continue
        for s in stalls:
            try:
                tot[s] += int(r[hdr.index(s)])
            except ValueError:
                pass
    allv = sum(tot.values()) or 1
    print("== warp stall samples (all launches in the report)")
    for s, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        if v:
            print(f"  {s:28s} {v:9d} {100.0 * v / allv:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
