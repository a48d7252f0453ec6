"""Summarise an ncu --set full report into the numbers DESIGN.md / profiles/ quote.

    python tools/ncu_summary.py gpurun_out/r01_fused.ncu-rep [--json out.json]
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def ncu_csv(path, page, extra=()):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv", *extra], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise_row(path, head, vals, launch):
    out = {"kernel": vals[head.index("Kernel Name")] if "Kernel Name" in head else None}
    for m in METRICS:
        if m in head:
            out[m] = vals[head.index(m)]
    stalls = {}
    for i, k in enumerate(head):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            v = float(vals[i] or 0)
            if v > 0.05:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    try:
        src = ncu_csv(path, "source", ["--print-source=sass", "--launch-skip", str(launch), "--launch-count", "1"])
        h = src[1]
        si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        agg, cnt, tot = collections.Counter(), collections.Counter(), 0
        for x in src[2:]:
            if len(x) < 2:
                continue
            t = x[1].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            s = int(x[si] or 0)
            agg[op] += s
            cnt[op] += int(x[ii] or 0)
            tot += s
        out["sass_top"] = [{"op": op, "stall_pct": round(100 * s / max(tot, 1), 1),
                            "inst": cnt[op]} for op, s in agg.most_common(12)]
    except Exception as exc:  # source page needs -lineinfo / --import-source
        out["sass_top"] = str(exc)
    try:
        rd = float(out["dram__bytes_read.sum"])
        wr = float(out["dram__bytes_write.sum"])
        out["dram_bytes_total"] = rd + wr
    except (KeyError, ValueError):
        pass
    return out


def summarise(path):
    """One summary per captured launch (a list when the report holds several kernels)."""
    rows = ncu_csv(path, "raw")
    head = rows[0]
    res = [summarise_row(path, head, vals, i) for i, vals in enumerate(rows[2:]) if len(vals) == len(head)]
    return res[0] if len(res) == 1 else res


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    text = json.dumps(res, indent=1)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(text + "\n")
    print(text)
