"""Summaries of the direct solver's ncu evidence for profiles/:
  launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_*) of one
  direct flatten -> per-kernel time, DRAM bytes, the numeric phase's share;
  a --set full capture -> key throughput/occupancy/stall metrics.

    python tools/summarize_direct.py LAUNCHES.csv FULL.ncu-rep OUT.json
"""
import collections
import csv
import json
import re
import subprocess
import sys

NUMERIC = ("k_factor", "k_factor_sm", "k_factor_warp", "k_schur", "k_pdiag", "k_pupd", "k_asm_cols", "k_asm_child")
SETUP = ("k_d_", "k_nd_", "k_sym", "k_eadj", "k_mark_cplx", "k_front_sizes", "k_iota")
SOLVE = ("k_fwd", "k_bwd", "k_d_scatter", "k_solve_pers", "k_solve_warp", "k_perm_rhs")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ci = {k: h.index(k) for k in ["ID", "Kernel Name", "Metric Name", "Metric Value", "Grid Size"]}
    out = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = out.setdefault(r[ci["ID"]], {"name": r[ci["Kernel Name"]], "grid": r[ci["Grid Size"]]})
        d[r[ci["Metric Name"]]] = float(r[ci["Metric Value"]].replace(",", "") or 0)
    return list(out.values())


def short(n):
    m = re.search(r"(k_\w+)", n)
    base = m.group(1) if m else n[:40]
    return base + ("<complex>" if "double2" in n else ("<real>" if "<double>" in n or "IdE" in n else ""))


def main():
    ls = launches(sys.argv[1])
    first = next(i for i, d in enumerate(ls) if short(d["name"]).startswith("k_d_urow"))
    ls = ls[first:]
    agg = collections.OrderedDict()
    phase = {"numeric": [0.0, 0.0], "setup": [0.0, 0.0], "solve": [0.0, 0.0], "other": [0.0, 0.0]}
    for d in ls:
        nm = short(d["name"])
        t = d.get("gpu__time_duration.sum", 0) / 1e3
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        a = agg.setdefault(nm, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        a[2] += b
        base = re.search(r"(k_\w+)", d["name"]).group(1) if re.search(r"(k_\w+)", d["name"]) else ""
        key = ("numeric" if base in NUMERIC else "setup" if base.startswith(SETUP) else
               "solve" if base in SOLVE else "other")
        phase[key][0] += t
        phase[key][1] += b
    tot = sum(a[1] for a in agg.values())
    out = {"source": sys.argv[1], "command": "HARMONIC=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
           "dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none python "
           "tools/direct_once.py (one cfg-2 direct flatten; cold-cache, serialised launches)",
           "total_us": tot,
           "phases_us": {k: v[0] for k, v in phase.items()},
           "phases_dram_bytes": {k: v[1] for k, v in phase.items()},
           "dram_bytes_per_factorization": phase["numeric"][1],
           "kernels": [{"kernel": k, "launches": a[0], "us": round(a[1], 1), "share": round(a[1] / tot, 4),
                        "dram_gb": round(a[2] / 1e9, 4)} for k, a in sorted(agg.items(), key=lambda x: -x[1][1])]}
    if len(sys.argv) > 3:
        raw = subprocess.run(["ncu", "-i", sys.argv[2], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h, v = rows[0], rows[2]
        d = dict(zip(h, v))
        keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "launch__registers_per_thread",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
        full = {k: d.get(k) for k in keys if k in d}
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x.replace(",", "")))
              for k, x in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
        st = sorted([x for x in st if x[1] > 0], key=lambda x: -x[1])
        tot_s = sum(x[1] for x in st) or 1
        full["stall_share"] = {k: round(x / tot_s, 3) for k, x in st[:8]}
        out["full_capture"] = {"source": sys.argv[2], "metrics": full}
    json.dump(out, open(sys.argv[-1], "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("total_us", "phases_us", "dram_bytes_per_factorization")}, indent=1))
    for k in out["kernels"][:12]:
        print(k)
    if "full_capture" in out:
        print(json.dumps(out["full_capture"]["metrics"], indent=1))


if __name__ == "__main__":
    main()
