"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/summarize_launches.py gpurun_out/launches_r1.csv [steps] > profiles/...

Groups launches by kernel, reports count, total/mean time and the share of
all library kernel time (ncu times are cold-cache and serialised: shares,
not absolute values, are what carry over to the timed bench)."""

import csv
import json
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^.*::", "", name)
    return name


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        rows.append((r["Kernel Name"], float(r["Metric Value"]), r["Grid Size"], r["Block Size"]))
    agg = {}
    for name, ns, grid, block in rows:
        k = short(name)
        lib = not name.startswith("void at::")
        a = agg.setdefault(k, {"count": 0, "ns": 0.0, "lib": lib, "grid": grid, "block": block})
        a["count"] += 1
        a["ns"] += ns
    tot_lib = sum(a["ns"] for a in agg.values() if a["lib"])
    tot = sum(a["ns"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        out.append({"kernel": k, "library": a["lib"], "launches": a["count"],
                    "launches_per_step": a["count"] / steps, "total_ms": a["ns"] / 1e6,
                    "ms_per_step": a["ns"] / 1e6 / steps, "mean_us": a["ns"] / a["count"] / 1e3,
                    "share_of_library_time": a["ns"] / tot_lib if a["lib"] else None,
                    "grid": a["grid"], "block": a["block"]})
    print(json.dumps({"source": path, "steps": steps, "launches": len(rows),
                      "library_launches": sum(a["count"] for a in agg.values() if a["lib"]),
                      "library_ms_per_step": tot_lib / 1e6 / steps, "all_ms_per_step": tot / 1e6 / steps,
                      "kernels": out}, indent=1))


if __name__ == "__main__":
    main()
