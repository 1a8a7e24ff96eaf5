"""Summarise ncu exports for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py report <file.ncu-rep> [...]   -> key metrics per kernel (JSON)
    python tools/ncu_summary.py launches <launches.csv>         -> per-kernel count / total / share

The metrics are the ones B200_PROFILING.md and SURVEY §8(d) d.6 name: DRAM
bytes and throughput, shared-memory wavefronts and bank conflicts, issue
activity, warps active, registers, and the top stall reasons.
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "smsp__average_warp_latency_per_inst_issued.ratio",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read.sum",
    "sm__memory_throughput.avg.pct_of_peak_sustained_active",
]
STALLS = ["long_scoreboard", "short_scoreboard", "mio_throttle", "wait", "math_pipe_throttle", "barrier",
          "lg_throttle", "not_selected", "selected", "branch_resolving", "no_instruction", "drain", "membar"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d, u = dict(zip(h, r)), dict(zip(h, units))
        rec = {"kernel": d.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in d:
                rec[k] = f"{d[k]} {u.get(k, '')}".strip()
        st = {}
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d and d[k]:
                st[s] = float(d[k])
        rec["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:6])
        out.append(rec)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit in ("msecond", "ms") else v
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": n, "total_us": round(t, 1), "avg_us": round(t / n, 1),
             "share_of_kernel_time": round(t / tot, 4)}
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    mode, files = sys.argv[1], sys.argv[2:]
    res = {f: (report(f) if mode == "report" else launches(f)) for f in files}
    print(json.dumps(res, indent=1))
