#!/usr/bin/env python3
"""Summarise an ncu --set full report: per-launch duration, DRAM bytes, throughput.

    python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep profiles/r01_ncu_summary.md [--json profiles/ncu_summary.json]
                                [--config rmat-s25-ef48]   (store under configs/<name>: bench.py reads it per workload)
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "smem_ld_wavefronts",
}
UNITS = {"dram_read": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "duration_ns": {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    js = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    cfgname = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        for k, name in METRICS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if name in ("dram_read", "dram_write"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if name == "duration_ns":
                    v *= {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
                d[name] = v
        launches.append(d)
    lines = ["| kernel | grid x block | regs | duration µs | DRAM read MB | DRAM write MB | DRAM % | SM % | L2 hit % | occupancy % | issue % |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in launches:
        lines.append("| {} | {}x{} | {:.0f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} |".format(
            d["kernel"].split("(")[0], int(d.get("grid", 0)), int(d.get("block", 0)), d.get("regs", 0),
            d.get("duration_ns", 0) / 1e3, d.get("dram_read", 0) / 1e6, d.get("dram_write", 0) / 1e6,
            d.get("dram_pct", 0), d.get("sm_pct", 0), d.get("l2_hit_pct", 0), d.get("occupancy_pct", 0),
            d.get("issue_pct", 0)))
    with open(out, "w") as f:
        f.write(f"ncu --set full --clock-control none summary of `{rep}` (cold-cache, serialised replays)\n\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if js:
        agg = {}
        for d in launches:
            k = d["kernel"]
            for key, name in (("OpOr", "ms_or_pass"), ("OpMin", "cc_seg"), ("k_pr_seg", "pr_seg"), ("k_pr_acc", "pr_acc"), ("k_pr_pull", "pr_direct"),
                              ("k_bfs_fused", "bfs_fused"), ("k_ms_pull_heavy", "ms_pull_heavy"),
                              ("k_ms_pull<", "ms_pull_light"), ("k_ms_push", "ms_push"),
                              ("k_ms_or_vertex", "ms_or_vertex"),
                              ("k_ms_resolve_heavy", "ms_resolve_heavy"), ("k_ms_narrow_or", "ms_narrow_or"),
                              ("k_ms_narrow<", "ms_narrow"), ("k_ms_list_", "ms_list"),
                              ("k_ms_finish", "ms_finish"), ("k_pb_scatter", "pb_scatter"),
                              ("k_pb_gather", "pb_gather")):
                if key in k:
                    a = agg.setdefault(name, {"launches": 0, "dram_bytes": 0.0, "duration_ns": 0.0})
                    a["launches"] += 1
                    a["dram_bytes"] += d.get("dram_read", 0) + d.get("dram_write", 0)
                    a["duration_ns"] += d.get("duration_ns", 0)
                    break
        for a in agg.values():
            a["dram_bytes_per_launch"] = a["dram_bytes"] / a["launches"]
            a["duration_us_per_launch"] = a["duration_ns"] / a["launches"] / 1e3
        if "pr_seg" in agg and "pr_acc" in agg:  # one pull iteration = segmented edge pass + vertex pass
            agg["pr_pull"] = {"dram_bytes_per_launch": agg["pr_seg"]["dram_bytes_per_launch"] +
                              agg["pr_acc"]["dram_bytes_per_launch"],
                              "note": "per PageRank iteration: k_pr_seg + k_pr_acc"}
        if "pb_scatter" in agg and "pb_gather" in agg:  # one blocked-pull iteration = scatter + gather
            agg["pr_pull"] = {"dram_bytes_per_launch": agg["pb_scatter"]["dram_bytes_per_launch"] +
                              agg["pb_gather"]["dram_bytes_per_launch"],
                              "note": "per PageRank iteration: k_pb_scatter + k_pb_gather"}
        # one bit-parallel pull level: its mask narrowing and then the row pull (light + heavy kernels,
        # + the row lists of a sparse level) or the segmented OR pass + vertex pass + heavy parent scans
        lv = agg.get("ms_narrow", {}).get("launches", 0) + agg.get("ms_narrow_or", {}).get("launches", 0)
        if lv == 0 and "ms_pull_light" in agg:  # 64-bit masks: no narrowing kernel
            lv = agg["ms_pull_light"]["launches"]
        if lv:
            parts = ("ms_narrow", "ms_narrow_or", "ms_pull_light", "ms_pull_heavy", "ms_list", "ms_or_pass",
                     "ms_or_vertex", "ms_resolve_heavy")
            tot = sum(agg.get(p, {}).get("dram_bytes", 0.0) for p in parts)
            agg["bfs_pull"] = {"dram_bytes_per_launch": tot / lv, "levels": lv,
                               "note": "per bit-parallel pull level (row pulls and segmented OR levels averaged): "
                                       "mask narrowing + k_ms_pull + k_ms_pull_heavy (+ row lists) or "
                                       "k_pr_seg<OpOr> + k_ms_or_vertex + k_ms_resolve_heavy"}
        top = json.load(open(js)) if os.path.exists(js) else {}
        old = top.setdefault("configs", {}).setdefault(cfgname, {}) if cfgname else top
        old.update(agg)  # merge with summaries of other captures (PR and BFS are captured separately)
        old.setdefault("sources", [])
        if rep not in old["sources"]:
            old["sources"].append(rep)
        old.pop("source", None)
        json.dump(top, open(js, "w"), indent=1)


if __name__ == "__main__":
    main()
