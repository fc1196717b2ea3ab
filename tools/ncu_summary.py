"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv) and full-set reports into markdown (dev / evidence tool).

    python tools/ncu_summary.py gpurun_out/j_launches.csv [report.ncu-rep ...] > profiles/r02/ncu_summary.md
"""
import collections
import csv
import re
import subprocess
import sys


UNITS = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "second": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name):
    m = re.match(r"(?:void )?(?:h2::)?([A-Za-z0-9_]+)(<[^(]*>)?", name)
    if not m:
        return name[:60]
    base = m.group(1)
    tmpl = m.group(2) or ""
    mode = ""
    if "MODE_WRITE" in tmpl or ", (int)0" in tmpl:
        mode = "<WRITE>"
    return base + mode


def launches(path):
    recs = collections.OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for row in rd:
        key = row["ID"]
        r = recs.setdefault(key, {"name": row["Kernel Name"], "grid": row.get("Grid Size", ""), "t": 0.0, "rd": 0.0, "wr": 0.0})
        v = float(row["Metric Value"].replace(",", "") or 0)
        unit = row["Metric Unit"]
        scale = UNITS.get(unit, 1.0)
        if row["Metric Name"] == "gpu__time_duration.sum":
            r["t"] = v * scale
        elif row["Metric Name"] == "dram__bytes_read.sum":
            r["rd"] = v * scale
        elif row["Metric Name"] == "dram__bytes_write.sum":
            r["wr"] = v * scale
    return list(recs.values())


def main():
    recs = launches(sys.argv[1])
    tot_t = sum(r["t"] for r in recs) or 1.0
    tot_b = sum(r["rd"] + r["wr"] for r in recs) or 1.0
    fam = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in recs:
        k = short(r["name"])
        fam[k][0] += 1
        fam[k][1] += r["t"]
        fam[k][2] += r["rd"] + r["wr"]
    print(f"## Launch list `{sys.argv[1]}`: {len(recs)} launches, {tot_t * 1e3:.2f} ms GPU time, {tot_b / 1e9:.2f} GB DRAM\n")
    print("| kernel | launches | time share | DRAM share | GB/s while running |")
    print("|---|---|---|---|---|")
    for k, (n, t, b) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {t / tot_t * 100:.1f} % | {b / tot_b * 100:.1f} % | {b / t / 1e9 if t else 0:.0f} |")
    for rep in sys.argv[2:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        if not rows:
            continue
        hdr = rows[0]
        want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
                "Registers Per Thread", "Grid Size", "Block Size", "L2 Hit Rate", "Executed Ipc Active"]
        print(f"\n### `{rep}`\n")
        ik = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
        im, iu, iv = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
        seen = set()
        for r in rows[1:]:
            if r[im] in want and (r[ik] if ik is not None else "", r[im]) not in seen:
                seen.add((r[ik] if ik is not None else "", r[im]))
                print(f"- {short(r[ik]) if ik is not None else ''} {r[im]}: {r[iv]} {r[iu]}")
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        if len(rr) >= 3:
            h, u = rr[0], rr[1]

            def val(d, key):
                if key not in h:
                    return float("nan")
                return float(d.get(key, "0").replace(",", "") or 0) * UNITS.get(u[h.index(key)], 1.0)
            for vals in rr[2:]:
                d = dict(zip(h, vals))
                b = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
                t = val(d, "gpu__time_duration.sum")
                tc = d.get("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "n/a")
                print(f"- {short(d.get('Kernel Name', ''))}: {t * 1e6:.1f} us, DRAM read+write {b / 1e6:.1f} MB "
                      f"({b / t / 1e9:.0f} GB/s), FP64 tensor path {tc} % of peak")

if __name__ == "__main__":
    main()
