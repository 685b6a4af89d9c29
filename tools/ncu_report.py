"""Curated text summary of ncu --set full reports (one block per profiled launch).

usage: python tools/ncu_report.py REPORT.ncu-rep [...] > profiles/<name>.txt
Shows duration, DRAM traffic, FP64 / tensor (DMMA) pipe activity, SM
throughput, occupancy, shared-memory bank conflicts, launch shape and the top
warp-stall reasons.
"""
import csv
import io
import subprocess
import sys

FIELDS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "FP64 pipe active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (DMMA)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_size", "cluster size"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__registers_per_thread", "registers/thread"),
]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
        r = list(csv.reader(io.StringIO(out)))
        hdr, units, data = r[0], r[1], r[2:]
        for row in data:
            name = row[hdr.index("Kernel Name")].split("(")[0]
            print(f"== {rep.split('/')[-1]} :: {name}")
            for key, label in FIELDS:
                if key in hdr:
                    i = hdr.index(key)
                    print(f"  {label:32s} {row[i]} {units[i]}")
            stalls = []
            for i, k in enumerate(hdr):
                if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio"):
                    try:
                        stalls.append((float(row[i].replace(",", "")), k.split("stalled_")[1][:-6]))
                    except ValueError:
                        pass
            if stalls:
                top = ", ".join(f"{n} {v:.1f}" for v, n in sorted(stalls, reverse=True)[:6])
                print(f"  {'top stalls (cycles/issue)':32s} {top}")


if __name__ == "__main__":
    main()
