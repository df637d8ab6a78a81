"""Summarise ncu captures into profiles/ (markdown + JSON). Usage:
    python tools/ncu_summary.py OUT_PREFIX REPORT.ncu-rep[:workload] ... [--launches LAUNCHES.csv]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
}
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "branch_resolving", "barrier", "selected", "no_instructions",
          "lg_throttle", "mio_throttle", "math_pipe_throttle", "membar"]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3,
         "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "s": 1e6, "second": 1e6}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    hdr, units, rows = raw(rep)
    res = []
    for row in rows:
        m = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        d = {"kernel": m.get("Kernel Name", "")[:120]}
        for k, key in KEYS.items():
            if key in m and m[key] not in ("", "n/a"):
                v = float(m[key].replace(",", ""))
                scale = UNITS.get(u.get(key, ""), 1)
                d[k] = v * scale
        total = 0.0
        st = {}
        for s in STALLS:
            key = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if key in m and m[key]:
                st[s] = float(m[key])
                total += st[s]
        d["stall_share"] = {k: round(v / total, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if total}
        res.append(d)
    return res


def launches(path):
    per = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rdr = csv.DictReader(io.StringIO("".join(lines)))
    for r in rdr:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][-60:]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(unit, 1)
        c, t = per.get(name, (0, 0.0))
        per[name] = (c + 1, t + v)
    tot = sum(t for _, t in per.values()) or 1
    return [{"kernel": k, "launches": c, "total_us": round(t, 2), "share": round(t / tot, 4)}
            for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])]


def main():
    prefix = sys.argv[1]
    args = sys.argv[2:]
    launch_csv = None
    if "--launches" in args:
        i = args.index("--launches")
        launch_csv = args[i + 1]
        args = args[:i] + args[i + 2:]
    out = {"captures": {}, "traffic": {}}
    md = ["# ncu summary (" + prefix + ")", ""]
    for spec in args:
        rep, _, workload = spec.partition(":")
        s = summarise(rep)
        out["captures"][rep] = s
        for d in s:
            md.append(f"## {workload or rep}: `{d['kernel']}`")
            for k in KEYS:
                if k in d:
                    md.append(f"- {k}: {d[k]:.4g}")
            md.append(f"- stall share: {d['stall_share']}")
            md.append("")
            if workload and "dram_read_bytes" in d:
                out["traffic"][workload] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)
    if launch_csv:
        ls = launches(launch_csv)
        out["launches"] = ls
        md.append("## launch list (ncu gpu__time_duration, cold-cache, serialised)")
        for r in ls:
            md.append(f"- {r['kernel']}: {r['launches']} launches, {r['total_us']} us, share {r['share']}")
    with open(prefix + ".json", "w") as f:
        json.dump(out, f, indent=1)
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
