"""Summarise an ncu --set full capture (raw page csv) into the key metrics."""
import csv
import json
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_atom.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__warps_eligible.avg.per_cycle_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__sass_average_branch_targets_threads_uniform.pct",
]
STALLS = "smsp__average_warps_issue_stalled_"


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:100]}
        for i, h in enumerate(hdr):
            if h in KEYS or (h.startswith(STALLS) and h.endswith("_per_issue_active.ratio")):
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[h] = v
        out.append(d)
    return out


if __name__ == "__main__":
    for d in summarise(sys.argv[1]):
        stalls = {k[len(STALLS):-len("_per_issue_active.ratio")]: v for k, v in d.items()
                  if k.startswith(STALLS)}
        for k, v in d.items():
            if not k.startswith(STALLS):
                print(f"{k:75s} {v}")
        print("stalls (warps per issue):")
        for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
            print(f"   {k:40s} {v:.3f}")
