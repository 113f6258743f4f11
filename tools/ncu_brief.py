"""Print the key --set full metrics of every kernel in an ncu report (details page)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Limit Shared Mem", "Block Limit Registers",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy", "Branch Instructions Ratio", "Avg. Active Threads Per Warp",
        "Waves Per SM"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, ui, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index(
        "Metric Value"), h.index("ID")
    cur = None
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if r[ii] != cur:
            cur = r[ii]
            print(f"== [{cur}] {r[ki].split('(')[0]}  grid {r[h.index('Grid Size')]} block {r[h.index('Block Size')]}")
        if r[mi] in KEYS:
            print(f"   {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
    # rule messages (stall reasons etc.)
    for r in rows[1:]:
        if len(r) > h.index("Rule Description") and r[h.index("Rule Description")] and "stall" in r[h.index("Rule Description")].lower():
            print(f"[{r[ii]}] {r[h.index('Rule Description')][:400]}")


if __name__ == "__main__":
    main(sys.argv[1])
