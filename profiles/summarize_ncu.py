#!/usr/bin/env python
"""Summarise an .ncu-rep (ncu --set full) into a small text file for profiles/.

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep profiles/r01_xxx.txt [units_per_launch]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "memory_l1_wavefronts_shared", "memory_l1_wavefronts_shared_ideal",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.sum",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def source(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    return hdr, [r for r in rows[2:] if len(r) == len(hdr)]


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    lines = []
    hdr, units, launches = raw(rep)
    name_i = hdr.index("Kernel Name")
    for k, vals in enumerate(launches):
        lines.append(f"== launch {k}: {vals[name_i]}")
        for i, h in enumerate(hdr):
            if h in KEYS or "warp_issue_stalled" in h and h.endswith("per_warp_active.pct"):
                lines.append(f"  {h:85s} {vals[i]:>18s} {units[i]}")
    try:
        shdr, rows = source(rep)
        iex, isrc, ismp = shdr.index("Instructions Executed"), shdr.index("Source"), shdr.index("# Samples")
        ops, tot = collections.Counter(), 0
        stall_cols = [i for i, h in enumerate(shdr) if h.startswith("stall_") and "Not Issued" not in h]
        stalls = collections.Counter()
        for r in rows:
            if not r[iex].isdigit():
                continue
            toks = r[isrc].split()
            op = toks[1] if toks[0].startswith("@") else toks[0]
            ops[op.split(".")[0]] += int(r[iex])
            tot += int(r[iex])
            for i in stall_cols:
                if r[i].isdigit():
                    stalls[shdr[i]] += int(r[i])
        lines.append(f"== SASS opcode mix of the profiled launch (warp instructions executed, total {tot})")
        for op, v in ops.most_common(24):
            lines.append(f"  {op:12s} {v:14d} {100.0 * v / tot:6.2f} %")
        st = sum(stalls.values())
        lines.append("== warp-state samples (all)")
        for k, v in stalls.most_common(12):
            lines.append(f"  {k:28s} {v:10d} {100.0 * v / max(st, 1):6.2f} %")
    except Exception as e:  # noqa: BLE001
        lines.append(f"(no source page: {e})")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
