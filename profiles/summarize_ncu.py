"""Summaries of ncu output for profiles/ (run here, on the copied files).

  python profiles/summarize_ncu.py launches gpurun_out/launches.csv   -> per-kernel share table
  python profiles/summarize_ncu.py full gpurun_out/prof_block.ncu-rep -> key metrics + stalls (JSON)
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [{"kernel": k, "launches": n, "total_us": t / 1e3, "share": t / tot,
            "avg_us": t / n / 1e3} for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    return {"total_us": tot / 1e3, "kernels": out}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")],
             "metrics": {k: f"{r[h.index(k)]} {units[h.index(k)]}" for k in KEYS if k in h}}
        st = {}
        for i, c in enumerate(h):
            if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith(
                    "_per_issue_active.ratio"):
                try:
                    st[c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        d["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1])[:10])
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd, wr = (h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"))
        d["dram_bytes"] = float(r[rd]) * mult.get(units[rd], 1) + float(r[wr]) * mult.get(units[wr], 1)
        res.append(d)
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
