"""Build profiles/ncu_summary_<tag>.json from a gpu_round.sh pass:
the launch list (per-kernel share of the bench command) and, per config, the
scan kernel's key counters from its ncu --set full capture.

    python tools/make_profile_summary.py TAG ROUND
"""
import csv
import json
import sys
from collections import OrderedDict
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "gpurun_out"
ALG = {"3": 1 << 30, "4": 3_200_000_000, "5": 1 << 28, "2": 1 << 26, "wide": 1 << 28}


def launch_list(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        us = v / 1000.0 if unit == "ns" else v * 1000.0 if unit == "ms" else v
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(t for _, t in agg.values())
    return [{"kernel": k, "launches": n, "mean_us": t / n, "total_us": t, "share": t / total}
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            d[h] = (float(v.replace(",", "")), u)
        except ValueError:
            d[h] = (v, u)
    return d


def scale(val_unit, to="B"):
    v, u = val_unit
    base = u.split("/")[0]
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3}.get(base, 1)
    return v * f


def config_summary(c, d):
    g = lambda k: d[k][0] if k in d else None
    t_us = scale(d["gpu__time_duration.sum"])
    rd, wr = scale(d["dram__bytes_read.sum"]), scale(d["dram__bytes_write.sum"])
    return {
        "kernel": str(d.get("Kernel Name", ("?",))[0])[:80],
        "gpu_time_us": t_us,
        "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
        "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": ALG[c],
        "achieved_GBps_cold": ALG[c] / (t_us * 1e3),
        "l1tex_throughput_pct": g("l1tex__throughput.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "shared_ld_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
        "shared_st_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum"),
        "shared_atom_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
        "shared_ld_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        "shared_ld_instructions": g("smsp__sass_inst_executed_op_shared_ld.sum"),
        "instructions": g("smsp__inst_executed.sum"),
        "registers": g("launch__registers_per_thread"),
        "smem_per_block_KB": (scale(d["launch__shared_mem_per_block_dynamic"]) / 1e3
                              if "launch__shared_mem_per_block_dynamic" in d else None),
    }


if __name__ == "__main__":
    tag, rnd = sys.argv[1], int(sys.argv[2])
    out = {"round": rnd,
           "command": "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity --no-others [--config C]; wide: python tools/exp_wide_one.py 4000 14",
           "note": "ncu per-launch times are cold-cache and serialised (--clock-control none); "
                   "bench.py's roofline uses CUDA-event times of the same kernel",
           "launch_list": launch_list(OUT / f"launches_{tag}.csv"), "configs": {}}
    for c in ("3", "4", "5", "2", "wide"):
        p = OUT / (f"raw_{tag}_{c}.csv" if c == "wide" else f"raw_{tag}_c{c}.csv")
        if p.exists():
            out["configs"][c] = config_summary(c, raw(p))
    dst = REPO / "profiles" / f"ncu_summary_r{rnd:02d}.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(dst)
